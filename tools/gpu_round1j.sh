mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -k "gather or partition" 2>&1 | tail -2 > gpurun_out/pytest_gather.txt
for v in 2 3 4 5 6 2; do timeout 300 python bench.py --steps 20 --warmup 3 --variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench_g$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_g$v.json')); print($v, d['config']['gather_variant'], d['kernels_ms'], d['roofline']['frac'])"; done
cat gpurun_out/pytest_gather.txt
