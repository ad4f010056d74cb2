#!/bin/bash
# K2 dynamic tiles: full GPU suite + smoke, the default bench line, cfg2, and a cold
# files-path phase trace.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_default.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["value"], d["ms_per_step"], d["kernels_ms"], json.dumps(d["roofline"]), d["scorer_roofline"]["frac_of_read_stream"],
              d["e2e"]["value"], d["e2e"]["pcie_roofline"]["frac"], d["cpu_baseline"]["value"])
PY
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
tail -c 400 gpurun_out/bench_cfg2.json
timeout 600 python tools/files_trace.py "" 3 cold > gpurun_out/files_trace_cold.txt 2>&1
tail -60 gpurun_out/files_trace_cold.txt
