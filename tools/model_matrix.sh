#!/usr/bin/env bash
# P3 vs layer-wise for the three model shapes at N GPUs (one torchrun per model).
N=${1:-2}; OUT=${2:-gpurun_out/matrix_$N.log}
for m in resnet50 vgg19 seq2seq; do
  if [ "$N" = 1 ]; then
    timeout 900 python bench.py --gpus 1 --model $m --steps 10 --warmup 5 --skip-cpu --skip-e2e >> $OUT 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N)) \
      bench.py --gpus $N --model $m --steps 10 --warmup 5 --skip-cpu --skip-e2e >> $OUT 2>&1
  fi
  echo "rc=$? model=$m" >> $OUT
done
