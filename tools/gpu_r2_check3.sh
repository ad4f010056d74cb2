#!/bin/bash
# Round-2 re-entry check: GPU tests, smoke, default bench line, cfg2/cfg4 lines, then the
# ncu launch list + full captures of the final kernels (tools/gpu_r2_profile2.sh).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 600 gpurun_out/bench_default.json
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --workload cfg4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
for f in cfg2 cfg4; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
for l in open(f"gpurun_out/bench_{f}.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print(f, d.get("value"), d.get("ms_per_step"), d.get("kernels_ms"), (d.get("roofline") or {}).get("frac"),
              (d.get("scorer_roofline") or {}).get("frac_of_read_stream"))
PY
done
bash tools/gpu_r2_profile2.sh
