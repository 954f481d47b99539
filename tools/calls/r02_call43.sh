set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/r02k_parity_fullsize.jsonl
ATA_PARITY_LOG=gpurun_out/r02k_parity_fullsize.jsonl timeout 2400 python -m pytest -x -q -s tests/test_gpu_configs.py 2>&1 | tail -5
cat gpurun_out/r02k_parity_fullsize.jsonl
