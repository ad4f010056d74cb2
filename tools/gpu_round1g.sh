mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu5.txt
timeout 900 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files2.json 2> gpurun_out/bench_files2.err
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
cat gpurun_out/pytest_gpu5.txt gpurun_out/bench_files2.json; tail -n 3 gpurun_out/bench_files2.err gpurun_out/bench_default.err
