set -x
mkdir -p gpurun_out
timeout 900 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files.json 2> gpurun_out/bench_files.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/bench_files.json gpurun_out/bench_ref.json; tail -5 gpurun_out/bench_files.err gpurun_out/bench_ref.err
