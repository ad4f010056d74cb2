set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu2.txt
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.txt
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.txt
timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --workload cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --workload cfg1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_partials" -s 1 -c 1 -o gpurun_out/prof_r1_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 > gpurun_out/ncu_cfg4.txt 2>&1
cat gpurun_out/pytest_gpu2.txt; tail -2 gpurun_out/san_*.txt; cat gpurun_out/bench_cfg4.json gpurun_out/bench_cfg2.json gpurun_out/bench_cfg1.json; tail -3 gpurun_out/bench_cfg4.err
