#!/bin/bash
# bench.py's task-tree partition on one GPU: N ranks over gloo (host-staged
# point-to-point), checking the JSON line is produced (a shared-GPU run, not a
# scaling measurement).
set -e
for n in 2 8; do
  ATA_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --config c2 --gpus $n --dist tree \
    --steps 2 --warmup 1 --no-e2e --no-cpu
done
