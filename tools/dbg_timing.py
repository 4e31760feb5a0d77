"""Per-CTA pass timing of the persistent full θ-pass kernel (profiling aid).

usage: python tools/dbg_timing.py C4 [grid_blocks=N] [smem_bits_cap=N] [schedule=auto|lead|stream]
Stamps per pass and CTA (%globaltimer, ns): pass top, stream start (after the delta was
applied), stream done (last warp), verify done (last warp), CTA done, barrier exit.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
kw, sched, v0 = {}, "auto", None
for a in sys.argv[2:]:
    k, v = a.split("=")
    if k == "schedule":
        sched = v
    elif k == "v0":   # v0=facts: pass the facts as an explicit start set (the generic prologue)
        v0 = "facts"
    else:
        kw[k] = int(v)
P = lpgen.config(cfg)
prog = lp.Program(P, **kw)
if v0 == "facts":
    v0 = np.isin(np.arange(P.n_atoms), P.head[np.diff(P.body_ptr) == 0])
G = prog.info["grid_blocks"]
buf = torch.zeros(16 * G * 8, dtype=torch.int64, device="cuda")
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
for i in range(3):
    prog.least_model(v0, schedule=sched)
lib.lpdbg_set_timing(buf.data_ptr())
m, it, ex = prog.least_model(v0, schedule=sched, stats=True)
lib.lpdbg_set_timing(None)
t = buf.cpu().numpy().reshape(16, G, 8).astype(np.float64)
print(cfg, "iters", it, "grid", G, "truth_mode", prog.info["truth_mode"], ex["stats"])
ent = t[0, :, 6]
print(f"prologue: entry spread {(ent.max()-ent.min())/1e3:.1f}us, grid sync exit {(t[2,:,6].min()-ent.min())/1e3:.1f}..{(t[2,:,6].max()-ent.min())/1e3:.1f}us, prologue+smem load done {(t[0,:,7].max()-ent.min())/1e3:.1f}us, "
      f"first pass top {(t[0,:,0].min()-ent.min())/1e3:.1f}us; epilogue {(t[1,:,7].max()-t[1,:,6].min())/1e3:.1f}us; "
      f"kernel entry->end {(t[1,:,7].max()-ent.min())/1e3:.1f}us")
for k in range(min(it, 16)):
    top = t[k, :, 0]
    t0 = top.min()
    rel = lambda i: (t[k, :, i] - t0) / 1e3  # noqa: E731
    print(f"pass {k:2d}: stream start {rel(1).min():6.1f}..{rel(1).max():6.1f}  "
          f"stream done med/max {np.median(rel(2)):6.1f}/{rel(2).max():6.1f}  "
          f"verify done med/max {np.median(rel(3)):6.1f}/{rel(3).max():6.1f}  "
          f"cta done max {rel(4).max():6.1f}  barrier exit {rel(5).min():6.1f}..{rel(5).max():6.1f} us"
          + (f"  [S_k rows med/max {np.median(t[k,:,6]):.0f}/{t[k,:,6].max():.0f}, lead-occ rows med/max {np.median(t[k,:,7]):.0f}/{t[k,:,7].max():.0f}]"
             if k >= 3 and t[k, :, 6].max() < 1e9 else "")
          + (f"  [thread 0's delta share done med/max {np.median(rel(6)):5.1f}/{rel(6).max():5.1f}, sync {np.median(rel(7)):5.1f}/{rel(7).max():5.1f}]"
             if k >= 3 and t[k, :, 6].max() >= 1e9 else ""))
# per-CTA durations within each pass/phase (relative to that CTA's own pass start)
print("per-CTA (own start = 0): stream / verify / barrier seen / next start, med|max us")
for k in range(min(it, 16) - 1):
    s0 = t[k, :, 0]
    d = lambda i: (t[k, :, i] - s0) / 1e3  # noqa: E731
    nxt = (t[k + 1, :, 0] - s0) / 1e3
    print(f"pass {k:2d}: stream {np.median(d(2)):5.1f}|{d(2).max():5.1f}  verify {np.median(d(3)):5.1f}|{d(3).max():5.1f}"
          f"  barrier {np.median(d(5)):5.1f}|{d(5).max():5.1f}  phase over {np.median(d(1)):5.1f}|{d(1).max():5.1f}  next start {np.median(nxt):5.1f}|{nxt.max():5.1f}")
