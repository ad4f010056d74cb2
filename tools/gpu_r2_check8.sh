#!/bin/bash
# Same-box A/B of the read lookahead (TAILOR_READ_LOOKAHEAD=0/1) on the files line, and
# phase traces of select_merge vs the two calls (warm).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select_merge.py tests/test_gpu_direct_io.py -q -x -p no:cacheprovider > gpurun_out/pytest_c8.txt 2>&1
tail -2 gpurun_out/pytest_c8.txt
TAILOR_TRACE=1 timeout 600 python tools/files_trace.py "" 3 warm sm > gpurun_out/trace_sm_warm.txt 2>&1
TAILOR_TRACE=1 timeout 600 python tools/files_trace.py "" 3 warm two > gpurun_out/trace_two_warm.txt 2>&1
grep -E "^iter" gpurun_out/trace_sm_warm.txt gpurun_out/trace_two_warm.txt
for la in 1 0 1 0; do
  TAILOR_READ_LOOKAHEAD=$la timeout 1800 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files_la$la.json 2>/dev/null
  python - $la <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_files_la{sys.argv[1]}.json"):
    if l.startswith("{"):
        d = json.loads(l)
        sm = d["select_merge"]
        print("lookahead", sys.argv[1], "warm", d["value"], d["ms_per_step"], "cold", d["cold"]["value"], d["cold"]["ms_per_step"],
              d["cold"]["roofline"]["frac"], "| sm warm", sm["warm"]["ms_per_step"], "sm cold", sm["cold"]["ms_per_step"],
              "probe", d["disk_probe"].get("read_direct_gbs"))
PY
done
