mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trainer.py -q -x 2>&1 | tail -2 > gpurun_out/pytest_tr.txt
timeout 600 python bench.py --workload train --steps 10 --warmup 2 > gpurun_out/bench_train.json 2> gpurun_out/bench_train.err
timeout 600 ncu --set full --clock-control none -k regex:"grad_check|adamw_update" -s 2 -c 2 -o gpurun_out/prof_train python bench.py --workload train --steps 1 --warmup 1 > /dev/null 2>&1
cat gpurun_out/pytest_tr.txt gpurun_out/bench_train.json; tail -3 gpurun_out/bench_train.err
