set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest_gpu3.txt
for v in 1 2; do timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --score-variant $v > gpurun_out/bench_cfg4_s$v.json 2> gpurun_out/bench_cfg4_s$v.err; done
for v in 1 2; do timeout 600 python bench.py --workload cfg3 --steps 20 --warmup 3 --score-variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3_s$v.json 2> gpurun_out/bench_cfg3_s$v.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 1 -c 1 -o gpurun_out/prof_r1_cfg4_staged python bench.py --workload cfg4 --steps 1 --warmup 1 --score-variant 2 > gpurun_out/ncu_cfg4s.txt 2>&1
cat gpurun_out/pytest_gpu3.txt
for f in gpurun_out/bench_cfg4_s*.json gpurun_out/bench_cfg3_s*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d.get('kernels_ms'), d['roofline']['frac'], d.get('scorer_roofline',{}).get('frac'))"; done
tail -3 gpurun_out/bench_cfg4_s2.err
