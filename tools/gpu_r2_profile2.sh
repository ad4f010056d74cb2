#!/bin/bash
# Round-2 ncu evidence on the final kernels: launch list of the default bench command,
# full captures of the timed step's kernels (cfg3: K2 gather_bulk, K3 score_staged<4>, K4,
# K9) and of the cfg2 scorer (score_staged<2>).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_launch_bench.txt 2>&1
# warm-up 3 steps x 8 partitions x (K3, K4, K9, 2 x K2) = 120 launches of these kernels; skip into the eager
# per-kernel pass of partition 0 (score, combine, select, gather shard, gather weights)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gather_bulk|score_staged|select_plan|score_combine" \
    -s 120 -c 10 -o gpurun_out/prof_r2_cfg3_final python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-read-probe > gpurun_out/ncu_full.txt 2>&1
tail -2 gpurun_out/ncu_full.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_staged" -s 30 -c 1 \
    -o gpurun_out/prof_r2_cfg2_final python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-read-probe > gpurun_out/ncu_cfg2.txt 2>&1
tail -2 gpurun_out/ncu_cfg2.txt
