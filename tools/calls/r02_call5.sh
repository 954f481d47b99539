set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python tools/f64_ab.py 58 4096 5 2>&1 | tail -3
ATA_F64_TMA=0 timeout 120 python tools/f64_ab.py 58 4096 5 2>&1 | tail -3
timeout 120 python tools/f64_ab.py 148 4096 3 2>&1 | tail -3
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_ata.py tests/test_gpu_acceptance.py 2>&1 | tail -5
ATA_PARITY_LOG=gpurun_out/r02_parity_tma.jsonl timeout 900 python -m pytest -x -q -s tests/test_gpu_configs.py -k "c3 or c4" 2>&1 | tail -8
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02_tma_c4.json 2>gpurun_out/r02_tma_c4.err; tail -c 1500 gpurun_out/r02_tma_c4.json
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_tma_c3.json 2>&1; tail -c 600 gpurun_out/r02_tma_c3.json
