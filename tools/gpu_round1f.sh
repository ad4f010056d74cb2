set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest_gpu4.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e2.json 2> gpurun_out/bench_e2e2.err
cat gpurun_out/pytest_gpu4.txt
python -c "import json; d=json.load(open('gpurun_out/bench_e2e2.json')); print(d['value'], d['e2e'])"
tail -n 5 gpurun_out/bench_e2e2.err
