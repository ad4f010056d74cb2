#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select_merge.py tests/test_integration_build.py -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2 3; do timeout 900 python tools/stress_files.py 2 files bench > gpurun_out/stress4_$r.txt 2>&1; echo "run $r rc=$?"; grep -E "FAIL|stress ok" gpurun_out/stress4_$r.txt | cut -c1-300; done
