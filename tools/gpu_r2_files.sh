#!/bin/bash
# The files line (two calls and tg_select_merge; warm and cold) twice.
mkdir -p gpurun_out

for rep in 1 2; do
  timeout 1800 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files_$rep.json 2> gpurun_out/bench_files_$rep.err; tail -5 gpurun_out/bench_files_$rep.err
  python - $rep <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_files_{sys.argv[1]}.json"):
    if l.startswith("{"):
        d = json.loads(l)
        sm = d["select_merge"]
        print("two-call warm", d["value"], d["ms_per_step"], d["roofline"]["frac"], "cold", d["cold"]["value"], d["cold"]["ms_per_step"],
              d["cold"]["roofline"]["frac"], "| sm warm", sm["warm"], "sm cold", json.dumps(sm["cold"]),
              "probe", d["disk_probe"].get("read_direct_gbs"), "ref", d["reference"]["value"])
PY
done
