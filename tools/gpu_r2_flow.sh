#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_integration_build.py -q -p no:cacheprovider > gpurun_out/flow.txt 2>&1
tail -3 gpurun_out/flow.txt
d=$(mktemp -d); oracle/_ref/ref_tool gen --layers 2 --hidden 8 --ffn 16 --vocab 32 --seed 7 --ranks 2 --snapshots 3 --out $d/run > $d/gen.json
dirs=$(python -c "import json,sys; print(' '.join(json.load(open('$d/gen.json'))['snapshots']))")
tests/integration/_build/device_flow $d/flow 0.5 $dirs > $d/out.txt 2> $d/err.txt; echo "flow rc=$?"; echo "--- stdout"; head -30 $d/out.txt; echo "--- stderr"; head -10 $d/err.txt
