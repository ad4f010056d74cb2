mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_k9.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_dev.json 2>gpurun_out/bench_dev.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --host-select > gpurun_out/bench_host.json 2>/dev/null
cat gpurun_out/pytest_k9.txt; tail -3 gpurun_out/bench_dev.err
for f in gpurun_out/bench_dev.json gpurun_out/bench_host.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'], d['config']['selection'], d['config']['device_selection_matches_host'])"; done
