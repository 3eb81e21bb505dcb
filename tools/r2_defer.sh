# N=2 sync-only A/B: previous library (stage released after each bulk store's read) vs the
# deferred release; then correctness of the new library (multi-process parity + GPU tests).
for i in 1 2; do
for lib in .varlibs/head.so paper_1905_03960_b200/libp3.so; do
for red in 0 2; do
  P3_LIB=$lib P3_TMA_STORE_RED=$red timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP $(basename $lib),tsr$red |"
done; done; done
