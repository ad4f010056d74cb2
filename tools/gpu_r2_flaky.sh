#!/bin/bash
# Flakiness check: the full GPU suite twice, then the smoke.
mkdir -p gpurun_out
for r in 1 2; do timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$r.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$r.txt; grep FAILED gpurun_out/pytest_gpu_$r.txt | head; done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
