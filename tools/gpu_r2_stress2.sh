#!/bin/bash
# The files-arm order in a loop (tools/stress_files.py ... bench): plain, then with
# TAILOR_SYNC_CHECK=1 (each device step synchronised right after its launch).
mkdir -p gpurun_out
for r in 1 2 3; do timeout 900 python tools/stress_files.py 2 files bench > gpurun_out/stress2_$r.txt 2>&1; echo "plain $r rc=$?"; grep -E "FAIL|stress ok" gpurun_out/stress2_$r.txt | cut -c1-300; done
for r in 1 2 3 4; do TAILOR_SYNC_CHECK=1 timeout 900 python tools/stress_files.py 2 files bench > gpurun_out/stress2_sc$r.txt 2>&1; echo "synccheck $r rc=$?"; grep -E "FAIL|stress ok" gpurun_out/stress2_sc$r.txt | cut -c1-300; done
