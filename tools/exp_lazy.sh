for v in base nosleep; do timeout 30 python tools/exp_concurrency.py $v >> gpurun_out/exp3.log 2>&1; done
for v in kernels; do timeout 30 python tools/exp_memops.py $v >> gpurun_out/exp3.log 2>&1; done
for v in kernels; do CUDA_MODULE_LOADING=EAGER timeout 60 python tools/exp_memops.py $v >> gpurun_out/exp3.log 2>&1; done
