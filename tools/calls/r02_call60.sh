# (1) the two bench N=2 tests that failed in call 58, with their output; (2) e2e row-block layouts under the faster device plan
set -x
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x -k "bench_two_ranks" 2>&1 | tail -40
timeout 1500 python tools/e2e_blocks.py 65536 32768 8192,57344 16384,49152 4096,61440 4096,16384,45056 2048,12288,51200 8192,16384,40960 6144,59392 65536 2>&1 | grep blocks
