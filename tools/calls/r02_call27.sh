set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py -k "tf32 or ring" 2>&1 | tail -3
ATA_PARITY_LOG=gpurun_out/r02l_parity_c5.jsonl timeout 900 python -m pytest -x -q -s tests/test_gpu_configs.py -k c5 2>&1 | tail -4
for i in 1 2; do
timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02l_c5.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02l_c5.json')); r=d['roofline']
print('c5', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), 'clk', d['clocks'])"
done
