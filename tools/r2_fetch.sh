# Broadcast pull (P3_BCAST_PULL=1): owners write only their own replica and NOTIFY; every other
# rank fetches the updated slice over NVLink. Correctness first, then N=2 sync-only timing.
P3_BCAST_PULL=1 timeout 600 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_torch_parity.py -x -q -m gpu 2>&1 | tail -3
P3_BCAST_PULL=1 timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -3
for i in 1 2; do
for bp in 0 1; do
  P3_BCAST_PULL=$bp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP bp$bp |"
done; done
