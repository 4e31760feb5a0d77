"""Per-phase SM-clock durations of the persistent full θ-pass kernel (profiling aid).

usage: python tools/dbg_phases.py C3|C4 [LP_* env switches are read by lp_load]
Stamps (clock64, one CTA's own clock): 0 pass top, 1 phase start (counts + fold done),
6 arming done (armed passes, last warp), 7 verification start, 2 stream / verification done
(last warp), 4 before the grid barrier, 5 after it.  Prints the mean over CTAs and passes
1..14 and the mean of the per-pass maxima, in microseconds at the measured SM clock."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
P = lpgen.config(cfg)
prog = lp.Program(P)
G = prog.info["grid_blocks"]
buf = torch.zeros(16 * G * 8, dtype=torch.int64, device="cuda")
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
lib.lpdbg_set_clock.argtypes = [ctypes.c_int]
for _ in range(3):
    prog.least_model()
lib.lpdbg_set_clock(1)
lib.lpdbg_set_timing(buf.data_ptr())
m, it, ex = prog.least_model(stats=True)
torch.cuda.synchronize()
lib.lpdbg_set_timing(None)
lib.lpdbg_set_clock(0)
st = ex["stats"]
ghz = st["sm_cycles"] / st["ns"]
t = buf.cpu().numpy().reshape(16, G, 8).astype(np.float64) / ghz / 1e3   # us
print(cfg, "iters", it, f"SM clock {ghz:.3f} GHz", "armed cap", prog.info["armed_list_cap"])
rows = [("top -> phase start (counts, Δ fold)", 0, 1), ("phase start -> arming done", 1, 6),
        ("arming done -> verification start (sync)", 6, 7), ("verification", 7, 2),
        ("verification done -> barrier entry", 2, 4), ("grid barrier", 4, 5)]
K = range(3, min(it, 15) - 1)   # (passes 0-2 share slots with prologue / epilogue stamps)
for name, a, b in rows:
    d = np.array([t[k, :, b] - t[k, :, a] for k in K])
    if np.all(t[1:, :, b] == 0):
        continue
    print(f"{name:45s} mean {d.mean():6.2f}  mean-of-max {d.max(axis=1).mean():6.2f} us")
nxt = np.array([t[k + 1, :, 0] - t[k, :, 5] for k in K])
print(f"{'barrier exit -> next pass top':45s} mean {nxt.mean():6.2f}  mean-of-max {nxt.max(axis=1).mean():6.2f} us")
per = np.array([t[k + 1, :, 0] - t[k, :, 0] for k in K])
print(f"{'pass period':45s} mean {per.mean():6.2f}  mean-of-max {per.max(axis=1).mean():6.2f} us")
