#!/bin/bash
# Trainer access-pattern probe + a longer wider-shape random parity sweep.
mkdir -p gpurun_out
timeout 300 ./tools/rmw_probe > gpurun_out/rmw_probe.txt 2>&1; cat gpurun_out/rmw_probe.txt
timeout 3000 python tools/random_sweep.py 600 78 large > gpurun_out/sweep_large2.txt 2>&1
tail -2 gpurun_out/sweep_large2.txt; grep -c FAIL gpurun_out/sweep_large2.txt
