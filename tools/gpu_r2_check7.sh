#!/bin/bash
# tg_select_merge (the scorer's master copies feed the merge): tests vs the reference,
# the named configs, then the files line (two calls and combined, warm and cold).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_select_merge.py tests/test_gpu_named_configs.py tests/test_gpu_bench.py -q -x -p no:cacheprovider > gpurun_out/pytest_c7.txt 2>&1
tail -3 gpurun_out/pytest_c7.txt
grep -E "Error|error|assert" gpurun_out/pytest_c7.txt | head -20
timeout 1800 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files.json 2> gpurun_out/bench_files.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_files.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print("files warm", d["value"], d["ms_per_step"], d["roofline"]["frac"], d["config"]["last_step_phases"])
        c = d["cold"]
        print("files cold", c["value"], c["ms_per_step"], c["roofline"]["frac"], c["last_step_phases"])
        print("select_merge", json.dumps(d["select_merge"]))
        print("ref", d["reference"]["value"], "probe", d["disk_probe"].get("read_direct_gbs"))
PY
tail -3 gpurun_out/bench_files.err
