#!/bin/bash
# ncu --set full capture of named kernels during a short C3 solve (run under gpurun):
# raw metrics + source page (SASS with executed counts / stall samples) per kernel.
# Usage: tools/ncu_kernels.sh OUTDIR kernel_regex...
set -u
OUT=$1; shift
mkdir -p "$OUT"
for k in "$@"; do
  ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:$k \
    --launch-skip 1 -c 1 -o /tmp/full_$k python tools/profile_step.py --outer 2 > /dev/null 2>&1
  ncu -i /tmp/full_$k.ncu-rep --page raw --csv > "$OUT/raw_$k.csv" 2>/dev/null
  ncu -i /tmp/full_$k.ncu-rep --page source --csv > "$OUT/src_$k.csv" 2>/dev/null
done
ls -la "$OUT"
