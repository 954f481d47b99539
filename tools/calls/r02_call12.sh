set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --fuse-leaf-sums > gpurun_out/r02f_fused16.json 2>&1
ATA_LIB_PATH=_ab/fbk32.so timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --fuse-leaf-sums > gpurun_out/r02f_fused32.json 2>&1
for f in fused16 fused32; do python -c "
import json; d=json.load(open('gpurun_out/r02f_$f.json')); r=d['roofline']; print('$f', round(d['value']), 'frac', round(r['frac'],4), r['share_of_step'], r['secondary']['share_of_step'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prod_f64_tma -s 30 -c 1 \
  -o gpurun_out/r02f_fused_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --fuse-leaf-sums > gpurun_out/r02f_ncu.log 2>&1
ncu -i gpurun_out/r02f_fused_full.ncu-rep --page raw --csv > gpurun_out/r02f_fused_full.csv 2>/dev/null
rm -f gpurun_out/r02f_fused_full.ncu-rep
