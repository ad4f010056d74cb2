#!/bin/bash
# K2 dynamic tile claiming: parity tests, then A/B of the cfg3 whole-job step (variant 0 =
# dynamic tiles, 7 = static split) and cfg2, alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dynamic_gather or partition_merge or device_select_step or gather_variants or host_pipeline" > gpurun_out/pytest_dyn.txt 2>&1
tail -3 gpurun_out/pytest_dyn.txt
for rep in 1 2; do
  for v in 0 7; do
    timeout 900 python bench.py --no-e2e --no-cpu-baseline --variant $v > gpurun_out/ab_cfg3_v$v_$rep.json 2> gpurun_out/ab_cfg3_v${v}_$rep.err
    python - "$v" gpurun_out/ab_cfg3_v$v_$rep.json <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("cfg3 v", sys.argv[1], d["value"], d["ms_per_step"], d["kernels_ms"], d["roofline"]["frac"])
PY
  done
done
for v in 0 7; do
  timeout 900 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline --variant $v > gpurun_out/ab_cfg2_v$v.json 2>/dev/null
  python - "$v" gpurun_out/ab_cfg2_v$v.json <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        print("cfg2 v", sys.argv[1], d["value"], d["ms_per_step"], d["kernels_ms"], d["roofline"]["frac"])
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_bulk" -s 40 -c 2 \
    -o gpurun_out/prof_r2_gather_dyn python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_gather.txt 2>&1
tail -1 gpurun_out/ncu_gather.txt
