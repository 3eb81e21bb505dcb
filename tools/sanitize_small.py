"""A small end-to-end comm-kernel run for checkers (compute-sanitizer where available, the
checked build libp3_checked.so via P3_LIB): resnet50-like emulated in one launch, 2
iterations, 4 CTAs, parameters checked against the oracle replay.
python tools/sanitize_small.py [WORLD] [p3|baseline] [CTAS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import p3_oracle as O

from paper_1905_03960_b200.model import builtin_profile
from paper_1905_03960_b200.runtime import TrainingWorker, WorkerConfig

prof = builtin_profile("resnet50-like")
world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "p3"
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 4
iters = 2
cfg = WorkerConfig(rank=0, mode=mode, world=world, iterations=iters, deadlock_timeout=600.0, emulate_compute=False,
                   comm_ctas=ctas, rank_distinct_grads=True)
w = TrainingWorker(cfg, prof, ranks=list(range(world)))
w.run()
got = {f"{w.params_digest(li):016x}" for li in range(world)}
w.close()
want = f"{O.digest(O.replay_params(prof.param_counts(), prof.seed, world, iters, cfg.lr, distinct=True)):016x}"
print("digest", got, "oracle", want, "OK" if got == {want} else "MISMATCH")
sys.exit(0 if got == {want} else 1)
