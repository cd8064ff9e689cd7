#!/bin/bash
# Functional check of bench.py's N > 1 path on a one-GPU box: two ranks share
# the GPU under a private MPS daemon (timings are not per-GPU numbers).
set -u
D=$(mktemp -d)
export CUDA_MPS_PIPE_DIRECTORY=$D/pipe CUDA_MPS_LOG_DIRECTORY=$D/log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d || { echo "no MPS"; exit 0; }
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 ${@} > $D/out.log 2>&1; grep -v "^\s*$" $D/out.log | grep -i "error\|Error\|metric\|raise\|File" | head -20
echo quit | nvidia-cuda-mps-control
rm -rf $D
