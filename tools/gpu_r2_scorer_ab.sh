#!/bin/bash
# Scorer A/B on one box: static vs dynamic tile split (TAILOR_SCORE_STATIC), cfg3 (K=4) and
# cfg2 (K=2), plus an ncu capture of the dynamic K=4 kernel.
mkdir -p gpurun_out
for wl in cfg3 cfg2; do
  for st in 1 0; do
    TAILOR_SCORE_STATIC=$st timeout 900 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
        > gpurun_out/ab_${wl}_static$st.json 2>/dev/null
    python - "$wl" "$st" <<'PY'
import json, sys
wl, st = sys.argv[1], sys.argv[2]
d = json.loads([l for l in open(f"gpurun_out/ab_{wl}_static{st}.json") if l.startswith("{")][-1])
print(wl, "static" if st == "1" else "dynamic", d["kernels_ms"], d["scorer_roofline"]["frac_of_read_stream"], d["roofline"]["frac"])
PY
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 10 -c 1 \
    -o gpurun_out/prof_r2_cfg3_dyn python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_dyn.txt 2>&1
TAILOR_SCORE_STATIC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 10 -c 1 \
    -o gpurun_out/prof_r2_cfg3_static python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_static.txt 2>&1
tail -1 gpurun_out/ncu_dyn.txt gpurun_out/ncu_static.txt
