#!/bin/bash
# Round-2 final evidence: GPU suite, smoke, every bench line (cfg3 default with e2e and the
# CPU baseline, cfg2, cfg1, cfg4, cfg5, train, files), the reference arm, the launch list of
# the default command and compute-sanitizer.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1200 python bench.py > gpurun_out/final_cfg3.json 2> gpurun_out/final_cfg3.err
for w in cfg2 cfg1 cfg4 train; do
  timeout 900 python bench.py --workload $w > gpurun_out/final_$w.json 2> gpurun_out/final_$w.err
done
timeout 1500 python bench.py --workload cfg5 --steps 1 --warmup 1 > gpurun_out/final_cfg5.json 2> gpurun_out/final_cfg5.err
timeout 1800 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/final_files.json 2> gpurun_out/final_files.err
timeout 1800 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err
python - <<'PY'
import json
for w in ["cfg3", "cfg2", "cfg1", "cfg4", "train", "cfg5", "files", "reference"]:
    try:
        for l in open(f"gpurun_out/final_{w}.json"):
            if l.startswith("{"):
                d = json.loads(l)
                r = d.get("roofline") or {}
                print(w, d.get("value"), d.get("unit"), d.get("ms_per_step"), "frac", r.get("frac"),
                      "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(w, "missing", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/final_ncu_launch.txt 2>&1
tail -1 gpurun_out/final_ncu_launch.txt
bash tools/gpu_sanitize.sh > gpurun_out/final_sanitize.txt 2>&1; tail -12 gpurun_out/final_sanitize.txt
