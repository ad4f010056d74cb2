#!/bin/bash
# Full GPU suite + smoke + the default bench line on the current code (ReadPool lookahead,
# tg_comm, exact constant division), then the launch list of the default command.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_default.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["value"], d["ms_per_step"], d["kernels_ms"], json.dumps(d["roofline"]), d["scorer_roofline"]["frac_of_read_stream"],
              d["e2e"]["value"], d["e2e"]["pcie_roofline"]["frac"], d["cpu_baseline"]["value"], d.get("same_sample_files", {}).get("value"))
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2b.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_launch_bench.txt 2>&1
tail -1 gpurun_out/ncu_launch_bench.txt
