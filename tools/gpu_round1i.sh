mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "scorer" 2>&1 | tail -2 > gpurun_out/pytest_score.txt
timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 > gpurun_out/bench_cfg4_auto.json 2>/dev/null
timeout 600 python bench.py --workload cfg3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_auto.json 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_partials" -s 1 -c 1 -o gpurun_out/prof_r1_cfg4_v2 python bench.py --workload cfg4 --steps 1 --warmup 1 > /dev/null 2>&1
cat gpurun_out/pytest_score.txt
for f in gpurun_out/bench_cfg4_auto.json gpurun_out/bench_cfg3_auto.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('scorer_roofline',{}).get('frac'), d.get('kernels_ms'))"; done
