# FINISH backoff cap: N=2 sync-only A/B against HEAD (3 rounds), then the trace timeline
for i in 1 2 3; do
for lib in .varlibs/head.so paper_1905_03960_b200/libp3.so; do
  P3_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP n2,$(basename $lib) |"
done; done
mkdir -p gpurun_out/tl10; P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl10 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl10/r50.log 2>&1
