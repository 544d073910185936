#!/bin/bash
# st25 stage/tile sweep on C3: per-phase device times of a 6-outer-step solve
# (the second solve of each process; not a benchmark)
for st in 3 4; do for ch in 256 512 1024; do
  echo "== stages=$st chunks=$ch $(GADI_ST25_STAGES=$st GADI_ST25_CHUNKS=$ch python tools/profile_step.py --workload c3 --outer 6 --repeat 2 | tail -1)"
done; done
