#!/bin/bash
# Round-1 evidence refresh on one B200: GPU tests, smoke, every bench line, reference arm.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --workload cfg1 > gpurun_out/bench_cfg1.json 2>&1
timeout 600 python bench.py --workload cfg2 > gpurun_out/bench_cfg2.json 2>&1
timeout 600 python bench.py --workload cfg4 > gpurun_out/bench_cfg4.json 2>&1
timeout 300 python bench.py --workload train > gpurun_out/bench_train.json 2>&1
timeout 900 python bench.py --workload files --steps 5 --warmup 1 > gpurun_out/bench_files.json 2>&1
timeout 1500 python bench.py --workload cfg5 --steps 1 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt
for f in default cfg1 cfg2 cfg4 train files cfg5 ref; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
for l in open(f"gpurun_out/bench_{f}.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print(f, d.get("value"), d.get("unit"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"),
              (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("samples"))
PY
done
