# N=2 sync-only A/B across library builds (P3_LIB), two rounds
for i in 1 2; do
for lib in ${LIBS:-.varlibs/head.so paper_1905_03960_b200/libp3.so}; do
  P3_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-2} \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP $(basename $lib) |"
done; done
