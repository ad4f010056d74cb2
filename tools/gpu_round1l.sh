mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python bench.py > gpurun_out/bench_default2.json 2> gpurun_out/bench_default2.err
echo "bench wall s: $(( $(date +%s) - start ))"
python -c "
import json; d=json.load(open('gpurun_out/bench_default2.json')); print(d['value'], d['ms_per_step'], d['roofline'], d['e2e']['value'], d['e2e']['pcie_roofline'], d['cpu_baseline']['value'], d['clocks'], d['config']['device_selection_matches_host'])"
tail -3 gpurun_out/bench_default2.err
