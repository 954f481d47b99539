# ncu evidence for the FP64 leaf launch that carries riding sums (c4), after plain runs exited 0
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest -x -q tests/test_gpu_dist.py -k nccl 2>&1 | tail -3
# c3: autotuned (leaf width + breadth-first budget)
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02j_bench_c3.json 2> gpurun_out/r02j_bench_c3.err
tail -2 gpurun_out/r02j_bench_c3.err
python -c "
import json; d=json.load(open('gpurun_out/r02j_bench_c3.json')); r=d['roofline']
print('c3 tuned', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'e2e', round(d['e2e']['value']), d['plan'])"
# c2 e2e: pipelined integer-threshold path vs staged
for v in 1 0; do
ATA_PIPE_REF=$v timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02j_bench_c2_pipe$v.json 2> gpurun_out/r02j_bench_c2.err
python -c "
import json; d=json.load(open('gpurun_out/r02j_bench_c2_pipe$v.json')); r=d['roofline']
print('c2 pipe_ref=$v', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'e2e', round(d['e2e']['value']))"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prod_f64_tma -s 31 -c 1 \
  -o gpurun_out/r02j_c4_ride_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02j_ncu_full.log 2>&1
ncu -i gpurun_out/r02j_c4_ride_full.ncu-rep --page raw --csv > gpurun_out/r02j_c4_ride_full.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02j_ncu_launches.log 2>&1
ls -la gpurun_out/ | tail -8
