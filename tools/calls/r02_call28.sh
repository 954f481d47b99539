set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_acceptance.py -k random 2>&1 | tail -3
ATA_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 4 --config c3 --dist units --steps 2 --warmup 1 --no-autotune 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('units x4', round(d['value']), d['parallelism'][:160], d['plan']['mults_over_classical'])"
for p in 2 4; do ATA_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2966$p tests/dist_worker.py units 12000 4096 2>&1 | grep dist_worker; done
