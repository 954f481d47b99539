set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_ata.py -k "pipelined" 2>&1 | tail -3
timeout 500 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02_e2e_c4.json 2>&1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02_e2e_c3.json 2>&1
for c in c4 c3; do python -c "
import json; d=json.load(open('gpurun_out/r02_e2e_$c.json')); print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['ms_per_step'])"; done
ATA_PARITY_LOG=gpurun_out/r02_parity_e2e.jsonl timeout 900 python -m pytest -x -q -s tests/test_gpu_configs.py -k "c4 or c3" 2>&1 | tail -8
