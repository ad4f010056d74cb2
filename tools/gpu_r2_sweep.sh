#!/bin/bash
# Final-code parity sweep (2000 random cases incl. select-merge) + the C device flow test.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_integration_build.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 3300 python tools/random_sweep.py 2000 2026 > gpurun_out/random_sweep.txt 2>&1
tail -2 gpurun_out/random_sweep.txt; grep -c "select-merge ok" gpurun_out/random_sweep.txt; grep FAIL gpurun_out/random_sweep.txt | head -5
