#!/bin/bash
# Scorer ring geometry A/B on one box (dynamic tiles): cfg3 (K=4) and cfg2 (K=2) with the
# default ring (2), twice the rows (5), two CTAs per SM (6); cfg4 (K=16) default.
mkdir -p gpurun_out
for wl in cfg3 cfg2; do
  for v in 2 5 6; do
    timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --score-variant $v \
        > gpurun_out/geo_${wl}_v$v.json 2>/dev/null
    python - "$wl" "$v" <<'PY'
import json, sys
wl, v = sys.argv[1], sys.argv[2]
d = json.loads([l for l in open(f"gpurun_out/geo_{wl}_v{v}.json") if l.startswith("{")][-1])
print(wl, v, d["kernels_ms"], d["scorer_roofline"]["frac_of_read_stream"], d["scorer_roofline"]["read_stream_probe_gbs"])
PY
  done
done
timeout 900 python bench.py --workload cfg4 --steps 5 --warmup 3 > gpurun_out/geo_cfg4.json 2>/dev/null; tail -c 700 gpurun_out/geo_cfg4.json
