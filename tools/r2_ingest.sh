# ingest with batched ring loads: correctness, then N=1 / N=2 sync-only A/B against HEAD
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_live_order.py tests/test_gpu_stream.py tests/test_gpu_torch_parity.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do
for lib in .varlibs/head.so paper_1905_03960_b200/libp3.so; do
  P3_LIB=$lib timeout 200 python tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP n1,$(basename $lib) |"
  P3_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP n2,$(basename $lib) |"
done; done
