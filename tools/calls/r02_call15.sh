set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in "--autotune" "--gain 1.0" "--gain 1.5" "--max-depth 5" "--min-dim 256"; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e $v > gpurun_out/r02h.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/r02h.json')); r=d['roofline']; print('c4 $v', round(d['value']), 'frac', round(r['frac'],4), round(r['share_of_step'],4), d['plan']['mults_over_classical'], d['plan'].get('autotuned'))"
done
