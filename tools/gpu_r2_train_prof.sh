#!/bin/bash
# ncu --set full of the trainer update kernel (pipe utilisation, stall reasons, source).
mkdir -p gpurun_out
timeout 600 python bench.py --workload train --steps 10 > gpurun_out/tp_train.json 2>/dev/null; head -c 400 gpurun_out/tp_train.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adamw_update" -s 3 -c 1 \
    -o gpurun_out/prof_tp_train python bench.py --workload train --steps 1 --warmup 3 > gpurun_out/tp_ncu.txt 2>&1
tail -1 gpurun_out/tp_ncu.txt
