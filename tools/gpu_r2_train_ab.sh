#!/bin/bash
# K7 bias-correction division through a precomputed reciprocal (kernels/ieee_div.cuh) vs
# per-element __fdiv_rn (TAILOR_TRAIN_FDIV=1): trainer tests (incl. the exhaustive
# division check), bench A/B alternating, ncu of the update kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_trainer.py -q -x -p no:cacheprovider > gpurun_out/pytest_train.txt 2>&1
tail -2 gpurun_out/pytest_train.txt
for rep in 1 2; do
  for fd in 0 1; do
    TAILOR_TRAIN_FDIV=$fd timeout 600 python bench.py --workload train --steps 20 > gpurun_out/train_fdiv${fd}_${rep}.json 2>/dev/null
    python - $fd gpurun_out/train_fdiv${fd}_${rep}.json <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("fdiv", sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["last_norms"])
PY
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adamw_update" -s 3 -c 1 \
    -o gpurun_out/prof_r2_train_rcp python bench.py --workload train --steps 1 --warmup 3 > gpurun_out/ncu_train.txt 2>&1
tail -1 gpurun_out/ncu_train.txt
