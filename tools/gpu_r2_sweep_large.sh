#!/bin/bash
# Wider-shape random parity sweep vs the reference binary (h 64-384, K up to 6), plus the GPU suite.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/sl_pytest_gpu.txt 2>&1
tail -2 gpurun_out/sl_pytest_gpu.txt
timeout 2100 python tools/random_sweep.py 150 77 large > gpurun_out/sweep_large.txt 2>&1
tail -3 gpurun_out/sweep_large.txt
