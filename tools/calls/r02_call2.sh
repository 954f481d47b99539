set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
export ATA_PARITY_LOG=gpurun_out/r02_parity.jsonl
rm -f $ATA_PARITY_LOG
timeout 600 python -m pytest -x -q tests/test_gpu_kernels.py -k "ring" tests/test_gpu_ata.py 2>&1 | tail -5 > gpurun_out/r02_t1.log
timeout 1500 python -m pytest -q -s tests/test_gpu_configs.py 2>&1 | tail -30 > gpurun_out/r02_t2.log
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/r02_bench_c1.json 2>gpurun_out/r02_bench_c1.err
timeout 300 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r02_bench_c5.json 2>gpurun_out/r02_bench_c5.err
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/r02_bench_c2.json 2>gpurun_out/r02_bench_c2.err
cat gpurun_out/r02_t1.log gpurun_out/r02_t2.log
