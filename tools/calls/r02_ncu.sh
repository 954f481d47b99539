# ncu evidence for the TMA-fed FP64 leaf kernel on c4 (run after the plain bench exited 0)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prod_f64_tma -s 30 -c 1 \
  -o gpurun_out/r02_c4_tma_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02_ncu_full.log 2>&1
ncu -i gpurun_out/r02_c4_tma_full.ncu-rep --page raw --csv > gpurun_out/r02_c4_tma_full.csv 2>/dev/null
ncu -i gpurun_out/r02_c4_tma_full.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_c4_tma_source.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02_ncu_launches.log 2>&1
ls -la gpurun_out/
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --leaf-cols 2048 > gpurun_out/r02_c4_leaf2048.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02_c4_leaf2048.json')); r=d['roofline']
print('c4 leaf2048', round(d['value']), round(d['ms_per_step'],1), r['frac'], r['share_of_step'], r['secondary']['share_of_step'])"
