#!/bin/bash
# Trainer update with prefetched loads; file paths with the one-chunk read lookahead
# (ReadPool): trainer + file GPU tests, trainer bench, files bench (warm + cold), cold trace.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_trainer.py tests/test_gpu_files.py tests/test_gpu_direct_io.py tests/test_gpu_named_configs.py -q -x -p no:cacheprovider > gpurun_out/pytest_c5.txt 2>&1
tail -2 gpurun_out/pytest_c5.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "execute_merge or select_recipe or verify or budget or scoring" > gpurun_out/pytest_c5b.txt 2>&1
tail -2 gpurun_out/pytest_c5b.txt
for rep in 1 2; do
  timeout 600 python bench.py --workload train --steps 20 > gpurun_out/train_pf_$rep.json 2>/dev/null
  python - gpurun_out/train_pf_$rep.json <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("train", d["value"], d["ms_per_step"], d["roofline"]["frac"])
PY
done
timeout 1800 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files.json 2> gpurun_out/bench_files.err
python - <<'PY'
import json
for l in open("gpurun_out/bench_files.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print("files warm", d["value"], d["ms_per_step"], d["roofline"]["frac"], d["config"]["last_step_phases"])
        c = d["cold"]
        print("files cold", c["value"], c["ms_per_step"], c["roofline"]["frac"], c["last_step_phases"], c["buffered_reads_same_state"])
        print("ref", d["reference"]["value"], "probe", d["disk_probe"].get("read_direct_gbs"))
PY
timeout 600 python tools/files_trace.py "" 3 cold > gpurun_out/files_trace_cold.txt 2>&1
grep -E "^iter|score.rank [0-9]|assemble\.|merge.assemble " gpurun_out/files_trace_cold.txt | tail -30
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adamw_update" -s 3 -c 1 \
    -o gpurun_out/prof_r2_train_pf python bench.py --workload train --steps 1 --warmup 3 > gpurun_out/ncu_train.txt 2>&1
tail -1 gpurun_out/ncu_train.txt
