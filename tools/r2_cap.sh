# N=2 sync-only: push tokens (P3_PUSH_CAP; 0 = off) x late server binding (P3_LAZY_PICK)
P3_PUSH_CAP=8 P3_LAZY_PICK=1 timeout 600 python -m pytest tests/test_gpu_runtime.py -x -q -m gpu 2>&1 | tail -2
P3_PUSH_CAP=16 timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
for i in 1 2; do
for v in "0 0" "16 0" "32 0" "64 0" "96 0" "32 1" "64 1"; do
  set -- $v
  P3_PUSH_CAP=$1 P3_LAZY_PICK=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-2} \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP cap$1,lz$2 |"
done; done
mkdir -p gpurun_out/tl3; P3_PUSH_CAP=32 P3_TRACE_CTA=1 P3_TL_DUMP=gpurun_out/tl3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tools/exp_timeline_mp.py resnet50 > gpurun_out/tl3/r50.log 2>&1
