#!/bin/bash
# k_st25h tuning sweep (run under gpurun): MINB, stages, tile rows / threads
OUT=${1:-gpurun_out/sweep}; mkdir -p $OUT
for cfg in ${CFGS:-"3 0 512 256" "2 0 512 256" "2 3 512 256" "2 0 1024 512" "2 3 1024 512" "2 4 1024 512"}; do
  set -- $cfg
  envs="GADI_ST25H_MINB=$1 GADI_ST25_CHUNKS=$3 GADI_ST25_THREADS=$4"
  [ "$2" != "0" ] && envs="$envs GADI_ST25_STAGES=$2"
  echo "== MINB=$1 S=$2 chunks=$3 threads=$4"
  env $envs ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l.csv \
    -k regex:k_st25h python tools/profile_step.py --outer 2 > $OUT/run.log 2>&1 || tail -3 $OUT/run.log
  python tools/launches.py $OUT/l.csv | grep st25h
done
