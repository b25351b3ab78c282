#!/bin/bash
# The N>1 bench path (torchrun, 2 ranks) on one GPU over gloo: plumbing check.
export DTANS_DIST_BACKEND=gloo DTANS_SHARE_GPU=1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --scale 0.25 --steps 5 --warmup 3 --no-cusparse 2>&1 | tail -3
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config powerit --scale 0.0625 --steps 5 --warmup 3 2>&1 | tail -3
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 2>&1 | tail -2
