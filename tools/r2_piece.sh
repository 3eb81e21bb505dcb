# Server work in pieces (P3_SRV_PIECE elements): correctness (in-process N=1..8 digests, 2-GPU
# parity), then N=2 sync-only A/B
P3_SRV_PIECE=8192 timeout 600 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_notify.py -x -q -m gpu 2>&1 | tail -2
P3_SRV_PIECE=4096 timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
for i in 1 2; do
for v in 0 4096 8192 16384 25000; do
  P3_SRV_PIECE=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-2} \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP pc$v |"
done; done
mkdir -p gpurun_out/tl4; P3_SRV_PIECE=8192 P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl4 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl4/r50.log 2>&1
