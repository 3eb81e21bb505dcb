# exp build: deferred push completion (+ deferred stage release); correctness, then A/B with
# the default build and the push-limiting switches
P3_LIB=.varlibs/exp.so timeout 600 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_notify.py -x -q -m gpu 2>&1 | tail -2
P3_LIB=.varlibs/exp.so timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
for i in 1 2; do
for v in "def 0 0" "exp 0 0" "exp 16 0" "exp 32 0" "exp 0 24" "exp 0 32" "exp 0 48"; do
  set -- $v
  lib=paper_1905_03960_b200/libp3.so; [ $1 = exp ] && lib=.varlibs/exp.so
  P3_LIB=$lib P3_PUSH_CTAS=$2 P3_PUSH_CAP=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>/dev/null | grep SWEEP | sed "s|^SWEEP |SWEEP $1,pc$2,cap$3 |"
done; done
