set -x
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi; df -h /tmp) > gpurun_out/box.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
