set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_configs.py 2>&1 | tail -30 > gpurun_out/r02_gpu_all.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r02c_bench_c4.json 2>gpurun_out/r02c_bench_c4.err
timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02c_bench_c5.json 2>gpurun_out/r02c_bench_c5.err
cat gpurun_out/r02_gpu_all.log
