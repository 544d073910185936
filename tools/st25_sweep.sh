#!/bin/bash
# st25 threads/tile/stage sweep on C3: per-phase device times of a 6-outer-step
# solve (the second solve of each process; not a benchmark)
for th in 256 512; do for ch in 256 512 1024; do for st in 0 3; do
  if [ $st = 0 ]; then unset GADI_ST25_STAGES; else export GADI_ST25_STAGES=$st; fi
  echo "== threads=$th chunks=$ch stages=$st $(GADI_ST25_THREADS=$th GADI_ST25_CHUNKS=$ch python tools/profile_step.py --workload c3 --outer 6 --repeat 2 | tail -1)"
done; done; done
