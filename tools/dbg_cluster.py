"""Per-pass timing of the cluster least-model kernel (profiling aid).

usage: python tools/dbg_cluster.py C1|C2|rand:N:R
Stamps per pass and CTA (%globaltimer): pass top, merge done, stream done (last warp),
cluster barrier done, claim sum read."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
if cfg.startswith("rand:"):
    _, n, R = cfg.split(":")
    P = lpgen.random_program(np.random.default_rng(1), int(n), int(R), max_len=4, n_facts=int(n) // 20)
else:
    P = lpgen.config(cfg)
prog = lp.Program(P)
S = prog.info["cluster_ctas"]
print(cfg, "cluster", S)
buf = torch.zeros(16 * max(S, 1) * 8, dtype=torch.int64, device="cuda")
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
for _ in range(3):
    prog.least_model()
lib.lpdbg_set_timing(buf.data_ptr())
m, it, ex = prog.least_model(stats=True)
torch.cuda.synchronize()
lib.lpdbg_set_timing(None)
t = buf.cpu().numpy().reshape(16, max(S, 1), 8).astype(np.float64)
t0 = t[0, 0, 6]
print("iters", it, "stats", ex["stats"], f"entry->first pass top {(t[0, 0, 0] - t0) / 1e3:.2f} us, "
      f"end {(t[1, 0, 7] - t0) / 1e3:.2f} us")
for k in range(min(it, 16)):
    r = lambda i: (t[k, :, i] - t[k, 0, 0]) / 1e3  # noqa: E731
    nxt = (t[k + 1, 0, 0] - t[k, 0, 0]) / 1e3 if k + 1 < min(it, 16) else 0.0
    print(f"pass {k:2d}: merge {r(1).max():5.2f}  stream {r(2).max():5.2f}  barrier {r(3).max():5.2f}  "
          f"sum {r(5).max():5.2f}  -> next top {nxt:5.2f} us")
