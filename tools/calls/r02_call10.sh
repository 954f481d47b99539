set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_ata.py -k "syrk or pipelined or tma or churn or golden" 2>&1 | tail -3
timeout 120 python tools/f64_ab.py 58 4096 5 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02d_bench_c4.json 2>gpurun_out/r02d_bench_c4.err
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/r02d_bench_c3.json 2>&1
for c in c4 c3; do python -c "
import json; d=json.load(open('gpurun_out/r02d_bench_$c.json')); r=d['roofline']; print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1), 'frac', round(r['frac'],4), 'cpu', d['cpu_baseline'])"; done
ATA_PARITY_LOG=gpurun_out/r02d_parity.jsonl timeout 900 python -m pytest -x -q -s tests/test_gpu_configs.py -k "c4 or c3" 2>&1 | tail -8
/usr/bin/time -v timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02d_ref_arm.json 2> gpurun_out/r02d_ref_arm.err; tail -c 800 gpurun_out/r02d_ref_arm.json; grep "Elapsed" gpurun_out/r02d_ref_arm.err
timeout 1800 python tools/cpu_full_reference.py c4 2097152 > gpurun_out/r02d_cpu_full_c4_t21.json 2>&1; cat gpurun_out/r02d_cpu_full_c4_t21.json
