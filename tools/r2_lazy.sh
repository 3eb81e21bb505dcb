# Late binding of server jobs once the pushes are claimed (P3_LAZY_PICK=1): correctness, then
# N=2 sync-only A/B
P3_LAZY_PICK=1 timeout 600 python -m pytest tests/test_gpu_runtime.py -x -q -m gpu 2>&1 | tail -2
P3_LAZY_PICK=1 timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
for i in 1 2; do
for lz in 0 1; do
  P3_LAZY_PICK=$lz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP lz$lz |"
done; done
mkdir -p gpurun_out/tl2; P3_LAZY_PICK=1 P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl2/r50.log 2>&1
