# NVLS multicast broadcasts: multi-process parity (digests incl. the nvls ones), then sync-only A/B
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "[${N}]" > gpurun_out/r2_nvls_mp_n${N}.log 2>&1
for i in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 2>&1 | grep -E "SWEEP|Error|error" | sed "s/^SWEEP /SWEEP unicast /"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29620 tools/sync_sweep.py resnet50,seq2seq,vgg19 148 50000 512 '{"nvls": true}' 2>&1 | grep -E "SWEEP|Error|error" | sed "s/^SWEEP /SWEEP nvls /"
done
