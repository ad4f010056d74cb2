#!/bin/bash
# Round-1 evidence run on one B200: GPU tests, default bench, launch list of the
# default bench command, full ncu captures of the top kernels (cfg3 step, cfg4 sweep).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --workload cfg4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather|score_staged|select_plan" -s 5 -c 5 \
    -o gpurun_out/prof_r1_cfg3_v3 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 1 -c 1 \
    -o gpurun_out/prof_r1_cfg4_v3 python bench.py --workload cfg4 --steps 1 --warmup 1 > gpurun_out/ncu_cfg4.txt 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/bench_default.json gpurun_out/bench_cfg4.json
tail -2 gpurun_out/bench_default.err gpurun_out/ncu_full.txt gpurun_out/ncu_cfg4.txt
