import sys, time, threading, faulthandler
faulthandler.dump_traceback_later(120, exit=True)
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_03960_b200.runtime import SyncContext
from paper_1905_03960_b200.torch_models import real_counts
counts = real_counts(sys.argv[1]); ctas = int(sys.argv[2]); threads = int(sys.argv[3]) if len(sys.argv) > 3 else 512
ctx = SyncContext(counts, 1, [0], comm_ctas=ctas, comm_threads=threads, timeout_s=8.0, emulate_grads=True)
stream = torch.cuda.Stream()
for l in range(len(counts)): ctx.gradgen_layer(0, 7, 0, l, stream)
stream.synchronize()
for k in range(4):
    for l in range(len(counts)): ctx.layer_ready(0, l, k, None, stream)
    stream.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream); ctx.iteration_begin(k, stream); ctx.iteration_end(k); e.record(stream)
    def snap():
        d = ctx.debug_snapshot(0)
        ph = d.pop("cta_phase")[:ctas]
        from collections import Counter
        print("snap", {a: (b if not isinstance(b, list) else (sum(b), b[:6])) for a, b in d.items()}, flush=True)
        print("phases", Counter((p >> 20) & 0xf for p in ph), [hex(p) for p in ph if (p >> 20) & 0xf != 5][:20], flush=True)
    tm = threading.Timer(3.0, snap)
    tm.start()
    try:
        ctx.sync_all(k + 1, 10.0); stream.synchronize()
        print(sys.argv[1:], k, "ms", s.elapsed_time(e), flush=True)
    except Exception as ex:
        print(sys.argv[1:], k, "FAIL", ex, flush=True); break
    finally:
        tm.cancel()
