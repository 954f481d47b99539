# e2e row-block layouts, second sweep; c4 device after the dry-run workspace fix (A/B --no-tail-private)
set -x
for v in "" "--no-tail-private" ""; do
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],4), 'adds', round(r['secondary']['share_of_step'],4), 'exec', r['executed_flops_per_step']/r['algorithmic_flops_per_step'])"
done
timeout 1800 python tools/e2e_blocks.py 65536 32768 8192,16384,40960 12800,20224,32512 9472,18688,37376 6656,16896,41984 5120,15104,45312 4352,8704,17408,35072 7168,11264,18176,28928 10240,14336,40960 2>&1 | grep blocks
timeout 900 python tools/e2e_blocks.py 16384 16384 8192,8192 4096,12288 4096,4096,8192 2048,6144,8192 2>&1 | grep blocks
