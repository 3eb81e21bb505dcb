import sys, time, ctypes, threading
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_03960_b200 import _lib
from paper_1905_03960_b200.runtime import SyncContext
cu = ctypes.CDLL("libcuda.so.1")
for fn in ("cuStreamWriteValue32_v2", "cuStreamWaitValue32_v2", "cuStreamWriteValue32", "cuStreamWaitValue32"):
    print(fn, hasattr(cu, fn))
W32 = cu.cuStreamWriteValue32_v2; W32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
WT32 = cu.cuStreamWaitValue32_v2; WT32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
scen = sys.argv[1]
ctx = SyncContext([1000, 1000], 1, [0], timeout_s=3.0, emulate_grads=True)
comm = torch.cuda.Stream(); rs = torch.cuda.Stream()
scratch = torch.zeros(64, dtype=torch.int32, device="cuda")
ctx.iteration_begin(0, comm)   # nothing will be published: the kernel spins until its 3 s timeout
time.sleep(0.2)
t0 = time.time()
if scen == "write":
    for i in range(100): W32(ctypes.c_void_p(rs.cuda_stream), scratch.data_ptr() + 4 * (i % 64), i + 1, 0)
elif scen == "write_nobar":
    for i in range(100): W32(ctypes.c_void_p(rs.cuda_stream), scratch.data_ptr() + 4 * (i % 64), i + 1, 1)
elif scen == "wait":
    for i in range(100): WT32(ctypes.c_void_p(rs.cuda_stream), scratch.data_ptr(), 0, 0)
elif scen == "kernels":
    with torch.cuda.stream(rs):
        for i in range(100): scratch.add_(1)
elif scen == "kernel_then_write":
    with torch.cuda.stream(rs):
        for i in range(20):
            scratch.add_(1)
            W32(ctypes.c_void_p(rs.cuda_stream), scratch.data_ptr() + 4 * 63, i + 1, 0)
ev = torch.cuda.Event(); ev.record(rs)
while not ev.query() and time.time() - t0 < 6: time.sleep(0.001)
print(scen, "rank stream drained after", round(time.time() - t0, 4), "s", "(kernel timeout is ~2.8 s after this)", flush=True)
try: ctx.sync_all(1, 6.0)
except Exception as e: print("  sync:", str(e)[:80])
