#!/bin/bash
# Multi-rank bench path on ONE GPU (gloo, host-staged reduction): 2 ranks share
# cuda:0; the kernels of one rank never wait on the other.  Checks that the
# row-sharded result equals the single-rank result.
set -e
export ATA_DIST_BACKEND=gloo
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  tools/dist_check.py
