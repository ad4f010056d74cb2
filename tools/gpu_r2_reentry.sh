#!/bin/bash
# Re-entry check on a re-created container: GPU suite, smoke and the default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/re_pytest_gpu.txt 2>&1
tail -3 gpurun_out/re_pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re_smoke.txt 2>&1; tail -1 gpurun_out/re_smoke.txt
timeout 1200 python bench.py > gpurun_out/re_cfg3.json 2> gpurun_out/re_cfg3.err
head -c 600 gpurun_out/re_cfg3.json
