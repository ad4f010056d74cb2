#!/bin/bash
# K7 update pass with bulk L2 prefetch of the block's next chunks (TAILOR_TRAIN_PREFETCH
# distance in 4 KB chunks, 0 = off): trainer tests, bench A/B alternating, ncu of the kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_trainer.py -q -x -p no:cacheprovider > gpurun_out/pf_pytest_train.txt 2>&1
tail -2 gpurun_out/pf_pytest_train.txt
for rep in 1 2; do
  for d in 0 1 2 4 8; do
    TAILOR_TRAIN_PREFETCH=$d timeout 600 python bench.py --workload train --steps 20 > gpurun_out/pf_train_d${d}_${rep}.json 2>/dev/null
    python - $d gpurun_out/pf_train_d${d}_${rep}.json <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("pf", sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["last_norms"])
PY
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adamw_update" -s 3 -c 1 \
    -o gpurun_out/prof_pf_train python bench.py --workload train --steps 1 --warmup 3 > gpurun_out/pf_ncu.txt 2>&1
tail -1 gpurun_out/pf_ncu.txt
