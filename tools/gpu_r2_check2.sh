#!/bin/bash
# Round-2 check 2: GPU tests (incl. direct I/O and the dynamic-tile scorer), bench lines
# cfg3 / cfg2 / cfg4 / files (warm + cold).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --workload cfg4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
for f in cfg2 cfg4 cfg3; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
for l in open(f"gpurun_out/bench_{f}.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print(f, d.get("value"), d.get("ms_per_step"), d.get("kernels_ms"), (d.get("roofline") or {}).get("frac"),
              (d.get("scorer_roofline") or {}).get("frac_of_read_stream"), d.get("scorer_roofline") if f == "cfg4" else "")
PY
done
timeout 1800 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files.json 2> gpurun_out/bench_files.err
tail -c 2500 gpurun_out/bench_files.json; tail -3 gpurun_out/bench_files.err
