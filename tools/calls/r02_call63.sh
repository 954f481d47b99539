# final validation of round 2: smoke, the whole -m gpu suite (parity log), every config, ncu launch list + full capture
set -x
rm -f gpurun_out/r02o_parity_fullsize.jsonl
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
ATA_PARITY_LOG=gpurun_out/r02o_parity_fullsize.jsonl timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r02o_gpu_tests.log
cat gpurun_out/r02o_gpu_tests.log
for c in c4 c3 c1 c2 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r02o_bench_$c.json 2> gpurun_out/r02o_bench_$c.err
  tail -2 gpurun_out/r02o_bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02o_bench_$c.json')); r=d['roofline']
print('$c', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), 'e2e', round(d['e2e']['value']), 'cpu', round(d['cpu_baseline']['value'],1), d['clocks'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o_launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02o_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prod_f64_tma -s 30 -c 1 \
  -o gpurun_out/r02o_c4_ride_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02o_ncu_full.log 2>&1
ncu -i gpurun_out/r02o_c4_ride_full.ncu-rep --page raw --csv > gpurun_out/r02o_c4_ride_ncu_full.csv 2>/dev/null
ls -la gpurun_out/ | tail -12
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02o_reference_arm.json 2> gpurun_out/r02o_reference_arm.err; tail -c 600 gpurun_out/r02o_reference_arm.json
