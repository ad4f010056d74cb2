#!/bin/bash
# Round-1 profiling on one B200: launch list of the default bench command and full ncu
# captures of the top kernels (cfg3 step, cfg4 sweep, trainer step). Summaries:
#   python tools/ncu_summary.py --tag r1_v5 --launches gpurun_out/launches.csv --full gpurun_out/prof_r1_cfg3_v5.ncu-rep --workload cfg3
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gather|score_staged|select_plan|score_combine" -s 5 -c 5 \
    -o gpurun_out/prof_r1_cfg3_v5 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 1 -c 1 \
    -o gpurun_out/prof_r1_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-read-probe > gpurun_out/ncu_cfg4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"finite_check|adamw_update" -s 2 -c 2 \
    -o gpurun_out/prof_train python bench.py --workload train --steps 2 --warmup 1 > gpurun_out/ncu_train.txt 2>&1
tail -2 gpurun_out/ncu_full.txt gpurun_out/ncu_cfg4.txt gpurun_out/ncu_train.txt
