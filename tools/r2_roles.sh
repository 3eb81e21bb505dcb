# split roles in the FINISH launch: P3_PUSH_CTAS pushers, the rest reducers (exp build)
P3_LIB=.varlibs/exp.so P3_PUSH_CTAS=32 timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
for i in 1 2; do
for n in 0 16 32 48 64 96; do
  P3_LIB=.varlibs/exp.so P3_PUSH_CTAS=$n timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP pc$n |"
done; done
mkdir -p gpurun_out/tl6; P3_LIB=.varlibs/exp.so P3_PUSH_CTAS=32 P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl6/r50.log 2>&1
