import sys, ctypes, time
sys.path.insert(0, '/root/repo')
import torch
cu = ctypes.CDLL("libcuda.so.1")
W32 = cu.cuStreamWriteValue32_v2; W32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
W64 = cu.cuStreamWriteValue64_v2; W64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint]
WT32 = cu.cuStreamWaitValue32_v2; WT32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
x = torch.zeros(int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20, device="cuda")
flag = torch.zeros(64, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
h = ctypes.c_void_p(s.cuda_stream)
def run(mode, n=2000):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for i in range(n):
        x.add_(1.0)
        if mode == "w32": W32(h, flag.data_ptr(), i, 0)
        elif mode == "w32nb":
            rc = W32(h, flag.data_ptr(), i, 1)
            assert rc == 0, f"cuStreamWriteValue32(NO_MEMORY_BARRIER) -> {rc}"
        elif mode == "w64": W64(h, flag.data_ptr() + 8, i, 0)
        elif mode == "wait": WT32(h, flag.data_ptr() + 16, 0, 0)
        elif mode == "event":
            ev = torch.cuda.Event(); ev.record()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
for m in ["none", "w32", "w32nb", "w64", "wait", "none", "event"]:
    try:
        print(m, round(run(m), 2), "us per kernel(+op)")
    except AssertionError as e:
        print(m, "unsupported:", e)
