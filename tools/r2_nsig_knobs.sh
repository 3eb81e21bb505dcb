# two-signaler default: push_max and TMA-stored reduce switches, N=2 sync-only; timeline
for i in 1 2; do
for v in "2 0" "1 0" "2 2"; do
  set -- $v
  P3_PUSH_MAX=$1 P3_TMA_STORE_RED=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s/^SWEEP /SWEEP pm$1,tsr$2 /"
done; done
mkdir -p gpurun_out/tl7; P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl7 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl7/r50.log 2>&1
