# interleaved producer (-DP3_INTERLEAVE=1): correctness, then N=2 sync-only A/B
P3_LIB=.varlibs/il.so timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_live_order.py tests/test_gpu_notify.py tests/test_gpu_torch_parity.py -x -q -m gpu 2>&1 | tail -2
P3_LIB=.varlibs/il.so timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
for i in 1 2 3; do
for lib in paper_1905_03960_b200/libp3.so .varlibs/il.so; do
  P3_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP $(basename $lib) |"
done; done
