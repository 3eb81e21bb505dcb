# experiment switches re-measured on the final kernel (per-slot signalers, push_split auto)
for i in 1 2; do
for kv in "X=0" "P3_PUSH_CTAS=48" "P3_PUSH_CTAS=96" "P3_PUSH_CAP=64" "P3_PUSH_CAP=96" "P3_LAZY_PICK=1"; do
  env P3_LIB=.varlibs/exp.so $kv timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 \
    tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP $kv /"
done; done
