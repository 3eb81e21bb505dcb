#!/usr/bin/env bash
# configs[4]: slice-size x link-throttle sweep, P3 vs the layer-wise baseline (KVStore
# placement, FIFO, NOTIFY->PULL) on the same kernels, every model, N = visible GPUs.
N=$(nvidia-smi -L | wc -l)
for m in resnet50 vgg19 seq2seq; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N} --master-addr 127.0.0.1 \
    --master-port 29631 tools/sweep.py $m 0 10000,50000,1000000 10,25,100,0 2>&1 | grep SWEEP
done > gpurun_out/r2_sweep_n${N}.log 2>&1
