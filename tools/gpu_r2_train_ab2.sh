#!/bin/bash
# K7 update: 5 resident blocks per SM (48 registers, TAILOR_TRAIN_MIN_BLOCKS=5) vs the default (52, 4 blocks).
mkdir -p gpurun_out
TAILOR_TRAIN_MIN_BLOCKS=5 timeout 900 python -m pytest tests/test_gpu_trainer.py -q -x -p no:cacheprovider -k "not constant_division" 2>&1 | tail -1
for rep in 1 2 3; do
  for mb in 0 5; do
    TAILOR_TRAIN_MIN_BLOCKS=$mb timeout 600 python bench.py --workload train --steps 30 > gpurun_out/train_mb${mb}_${rep}.json 2>/dev/null
    python - $mb gpurun_out/train_mb${mb}_${rep}.json <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("min_blocks", sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"])
PY
  done
done
