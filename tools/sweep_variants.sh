for v in "0 2 4096 65536" "1 1 16384 131072" "1 1 8192 65536" "1 2 16384 262144" "1 1 32768 131072"; do
  set -- $v
  P3_SWEEP=$1 P3_SWEEP_DIV=$2 P3_SWEEP_MIN=$3 P3_SWEEP_MAX=$4 timeout 300 python tools/sync_sweep.py resnet50,seq2seq,vgg19 148 | sed "s/^SWEEP /SWEEP $1,$2,$3,$4 /"
done
