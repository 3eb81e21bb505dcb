# two signaler warps (one per job slot; -DP3_NSIG=2): correctness, then N=2 A/B vs default
P3_LIB=.varlibs/nsig2.so timeout 600 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_notify.py tests/test_gpu_live_order.py -x -q -m gpu 2>&1 | tail -2
P3_LIB=.varlibs/nsig2.so timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "2" 2>&1 | tail -2
LIBS="paper_1905_03960_b200/libp3.so .varlibs/nsig2.so" bash tools/r2_ab.sh
