set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 python bench.py --steps 10 --warmup 3 --variant 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_lsu.json 2> gpurun_out/bench_lsu.err
timeout 300 python bench.py --steps 10 --warmup 3 --variant 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_bulk.json 2> gpurun_out/bench_bulk.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather|score_partials" -s 3 -c 4 -o gpurun_out/prof_r1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
tail -5 gpurun_out/bench_full.err
cat gpurun_out/bench_full.json gpurun_out/bench_lsu.json gpurun_out/bench_bulk.json
