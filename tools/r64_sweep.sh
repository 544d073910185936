#!/bin/bash
# Sweep of the k_resid64 variants (run under gpurun): ncu gpu__time_duration of the
# outer-residual and zero-start-residual kernels during a short C3 solve.
OUT=${1:-gpurun_out/r64}
mkdir -p "$OUT"
for v in ${VARIANTS:-0 1 2 3 4}; do
  for st in ${STAGES:-4}; do
    GADI_R64=$v GADI_R64_STAGES=$st ncu -f --metrics gpu__time_duration.sum --clock-control none --csv \
      -k regex:'k_resid64|k_gm_resid0|PolResid' --log-file "$OUT/v${v}_s${st}.csv" \
      python tools/profile_step.py --outer 6 > "$OUT/v${v}_s${st}.txt" 2>&1
    echo "variant $v stages $st"; python tools/launches.py "$OUT/v${v}_s${st}.csv" | tail -n +2
  done
done
