#!/bin/bash
# launch list of two C3 outer steps + full captures of the stencil kernels (run under gpurun)
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
ncu -f --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches_c3_outer2.csv" python tools/profile_step.py --outer 2 > "$OUT/launch.log" 2>&1
python tools/launches.py "$OUT/launches_c3_outer2.csv" > "$OUT/launches_c3_summary.txt"
for k in ${KERNELS:-PolSpmvp PolGmMatvec PolResidA}; do
  ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:$k \
    --launch-skip 2 -c 1 -o "$OUT/full_$k" python tools/profile_step.py --outer 1 > /dev/null 2>&1
  ncu -i "$OUT/full_$k.ncu-rep" --page raw --csv > "$OUT/raw_$k.csv"
  ncu -i "$OUT/full_$k.ncu-rep" --page source --csv > "$OUT/src_$k.csv" 2>/dev/null
done
ls -la "$OUT"
