# push tokens returned when the push's data has moved (exp build)
for i in 1 2; do
for cap in 0 16 24 32 48; do
  P3_LIB=.varlibs/exp.so P3_PUSH_CAP=$cap timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP cap$cap |"
done; done
mkdir -p gpurun_out/tl5; P3_LIB=.varlibs/exp.so P3_PUSH_CAP=24 P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl5 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl5/r50.log 2>&1
