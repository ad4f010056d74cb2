#!/bin/bash
# Round-2 profiling on one B200: disk probe (files-path roofline), launch list of the
# default bench command, full ncu captures of the cfg3 step kernels and the cfg2 (K=2)
# scorer, the cfg2 and files bench lines.
mkdir -p gpurun_out
g++ -O2 -std=c++17 -pthread tools/disk_probe.cpp -o tools/disk_probe
(df -h /tmp "$GRAFT_REPO_ROOT"; mount | grep -E ' / | /tmp '; nproc; free -g) > gpurun_out/disk_env.txt 2>&1
timeout 600 tools/disk_probe /tmp 4 8 4 > gpurun_out/disk_probe.json 2>&1; cat gpurun_out/disk_probe.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gather|score_staged|select_plan|score_combine" -s 40 -c 5 \
    -o gpurun_out/prof_r2_cfg3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_full.txt 2>&1
tail -2 gpurun_out/ncu_full.txt
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -c 300 gpurun_out/bench_cfg2.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 4 -c 1 \
    -o gpurun_out/prof_r2_cfg2 python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_cfg2.txt 2>&1
tail -2 gpurun_out/ncu_cfg2.txt
timeout 900 python bench.py --workload files --steps 5 --warmup 1 > gpurun_out/bench_files.json 2> gpurun_out/bench_files.err; tail -c 600 gpurun_out/bench_files.json
