#!/bin/bash
# K7 trainer update: occupancy-sized grid (one wave) and the 6-blocks-per-SM build
# (TAILOR_TRAIN_MIN_BLOCKS=6, 40 registers) vs the unconstrained one (4 blocks per SM).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trainer.py -q -x -p no:cacheprovider > gpurun_out/pytest_train.txt 2>&1
tail -2 gpurun_out/pytest_train.txt
TAILOR_TRAIN_MIN_BLOCKS=6 timeout 900 python -m pytest tests/test_gpu_trainer.py -q -x -p no:cacheprovider > gpurun_out/pytest_train6.txt 2>&1
tail -2 gpurun_out/pytest_train6.txt
for rep in 1 2; do
  for mb in 1 6; do
    TAILOR_TRAIN_MIN_BLOCKS=$mb timeout 600 python bench.py --workload train --steps 20 > gpurun_out/train_mb${mb}_${rep}.json 2>/dev/null
    python - $mb gpurun_out/train_mb${mb}_${rep}.json <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("min_blocks", sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"])
PY
  done
done
for mb in 1 6; do
  TAILOR_TRAIN_MIN_BLOCKS=$mb timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adamw_update" -s 3 -c 1 \
    -o gpurun_out/prof_r2_train_mb$mb python bench.py --workload train --steps 1 --warmup 3 > gpurun_out/ncu_train_mb$mb.txt 2>&1
  tail -1 gpurun_out/ncu_train_mb$mb.txt
done
