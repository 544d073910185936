"""Static opcode histogram of one kernel's SASS: python tools/sass_ops.py OBJ NAME_SUBSTR [N]."""
import collections, re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if sys.argv[2] not in name:
        continue
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            ops[m.group(2).split(".")[0]] += 1
    print(name, sum(ops.values()))
    print("  ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25)))
