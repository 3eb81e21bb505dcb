# server-pick filter on top of the final defaults (N=2 sync-only), 3 rounds
for i in 1 2 3; do
for kv in "X=0" "P3_SRV_FILTER=2" "P3_SRV_FILTER=3" "P3_SRV_FILTER=4" "P3_SRV_FILTER=8"; do
  env $kv timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 \
    tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP $kv /"
done; done
