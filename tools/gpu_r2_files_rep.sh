#!/bin/bash
# The files line four times (stderr kept) to catch the intermittent failure.
mkdir -p gpurun_out
for rep in 1 2 3 4; do
  timeout 1200 python bench.py --workload files --steps 3 --warmup 1 > gpurun_out/bench_files_r$rep.json 2> gpurun_out/bench_files_r$rep.err
  echo "rep $rep rc=$?"; tail -2 gpurun_out/bench_files_r$rep.err | cut -c1-300
done
