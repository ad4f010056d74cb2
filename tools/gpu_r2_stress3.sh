#!/bin/bash
# After the upload/memset ordering fix: the files-arm order in a loop, six runs.
mkdir -p gpurun_out
for r in 1 2 3 4 5 6; do timeout 900 python tools/stress_files.py 2 files bench > gpurun_out/stress3_$r.txt 2>&1; echo "run $r rc=$?"; grep -E "FAIL|stress ok" gpurun_out/stress3_$r.txt | cut -c1-300; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_files.py tests/test_gpu_select_merge.py -q -x -p no:cacheprovider 2>&1 | tail -2
