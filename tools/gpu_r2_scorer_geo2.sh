#!/bin/bash
# Scorer ring geometry per K on one box (packed sweep over one Llama-3.1-8B rank partition,
# K snapshots): default ring (0) vs half rows (5) vs two CTAs/SM (6); then cfg3 / cfg2 lines.
mkdir -p gpurun_out
for K in 2 3 4 6 8 12 16; do
  for v in 0 5 6; do
    [ $K -gt 8 ] && [ $v -ne 0 ] && continue
    timeout 600 python bench.py --workload cfg4 --snapshots $K --steps 5 --warmup 3 --score-variant $v \
        > gpurun_out/geo2_K${K}_v$v.json 2>/dev/null
    python - "$K" "$v" <<'PY'
import json, sys
K, v = sys.argv[1], sys.argv[2]
d = json.loads([l for l in open(f"gpurun_out/geo2_K{K}_v{v}.json") if l.startswith("{")][-1])
r = d["roofline"]
print("K", K, "variant", v, "ms", d["ms_per_step"], "frac_read_stream", r["frac_of_read_stream"], "probe", r["read_stream_probe_gbs"])
PY
  done
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/geo2_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/geo2_cfg2.json 2>/dev/null
for f in cfg3 cfg2; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/geo2_{f}.json") if l.startswith("{")][-1])
print(f, d["value"], d["ms_per_step"], d["kernels_ms"], d["roofline"]["frac"], d["scorer_roofline"]["frac_of_read_stream"])
PY
done
