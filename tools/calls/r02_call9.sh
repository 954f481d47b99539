set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 2700 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r02_gpu_all2.log
cat gpurun_out/r02_gpu_all2.log
timeout 1800 python tools/cpu_full_reference.py c4 > gpurun_out/r02_cpu_full_c4.json 2>gpurun_out/r02_cpu_full_c4.err
cat gpurun_out/r02_cpu_full_c4.json
