#!/usr/bin/env bash
# Multi-GPU session (N = number of visible GPUs): NVLink parity tests, then the bench under
# torchrun and the reference arm. Outputs under gpurun_out/.
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r2}
nvidia-smi topo -m > gpurun_out/${TAG}_topo_n${N}.txt 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -x -k "[${N}]" > gpurun_out/${TAG}_mp_n${N}.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N} --master-addr 127.0.0.1 \
  --master-port 29611 bench.py --gpus ${N} --steps ${STEPS:-10} --warmup 5 ${BENCH_ARGS} > gpurun_out/${TAG}_bench_n${N}.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N} --master-addr 127.0.0.1 \
  --master-port 29612 bench.py --impl reference --gpus ${N} --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_n${N}.log 2>&1
if [ "${N}" = "2" ]; then
  P3_TRACE_CTA=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29613 tools/exp_timeline_mp.py resnet50 > gpurun_out/${TAG}_timeline_mp_n2.log 2>&1
fi
