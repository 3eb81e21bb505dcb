# two comm CTAs per SM (32 KB stages, 256 threads) vs one (N=2 sync-only)
for i in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 50000 512 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP def148x512 /"
  P3_LIB=.varlibs/st32.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 50000 512 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP st32_148x512 /"
  P3_LIB=.varlibs/st32.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 296 50000 256 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP st32_296x256 /"
  P3_LIB=.varlibs/st32.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 222 50000 256 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP st32_222x256 /"
done
