#!/bin/bash
# One-call round profile (run under gpurun): official bench lines, the
# reference arm, an ncu launch list of two C3 outer steps and of one C4 solve,
# and one `--set full` capture of each top kernel (raw pages exported).
# Usage: tools/round_profile.sh OUTDIR
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
python bench.py > "$OUT/bench_c3.json" 2> "$OUT/bench_c3.err"
python bench.py --workload c4 > "$OUT/bench_c4.json" 2> "$OUT/bench_c4.err"
python bench.py --workload c2 > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"
python bench.py --workload c1 > "$OUT/bench_c1.json" 2> "$OUT/bench_c1.err"
python bench.py --workload c5 > "$OUT/bench_c5.json" 2> "$OUT/bench_c5.err"
python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
python tools/profile_step.py --outer 2 > "$OUT/profile_step_plain.txt" 2>&1 && \
ncu -f --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches_c3_outer2.csv" python tools/profile_step.py --outer 2 > /dev/null 2>&1
python tools/profile_step.py --workload c4 --outer 1 > "$OUT/profile_step_c4_plain.txt" 2>&1 && \
ncu -f --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches_c4_outer1.csv" python tools/profile_step.py --workload c4 --outer 1 > /dev/null 2>&1
for k in PolSpmvp PolGmMatvec k_cg_update k_gm_cgs_few k_gm_dots k_resid64 k_gm_resid0p k_gm_update_few; do
  ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:$k \
    --launch-skip 2 -c 1 -o /tmp/full_$k python tools/profile_step.py --outer 1 > /dev/null 2>&1
  ncu -i /tmp/full_$k.ncu-rep --page raw --csv > "$OUT/raw_$k.csv"
done
ls -la "$OUT"
