set -x
nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02_gpu_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
tail -3 gpurun_out/r02_gpu_tests.log; cat gpurun_out/r02_bench_c4.json
