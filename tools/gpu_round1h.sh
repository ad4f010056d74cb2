mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "scorer" 2>&1 | tail -3 > gpurun_out/pytest_score.txt
for v in 3 4; do timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --score-variant $v > gpurun_out/bench_cfg4_v$v.json 2>/dev/null; done
for v in 3 4; do timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 --score-variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_v$v.json 2>/dev/null; done
cat gpurun_out/pytest_score.txt
for f in gpurun_out/bench_cfg4_v3.json gpurun_out/bench_cfg4_v4.json gpurun_out/bench_cfg3_v3.json gpurun_out/bench_cfg3_v4.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('scorer_roofline',{}).get('frac'), d.get('kernels_ms'))"; done
