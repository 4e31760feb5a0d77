"""Per-CTA pass timing of the persistent full θ-pass kernel (profiling aid)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
P = lpgen.config(cfg)
prog = lp.Program(P, **kw)
G = prog.info["grid_blocks"]
buf = torch.zeros(16 * G * 4, dtype=torch.int64, device="cuda")
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
for i in range(3):
    prog.least_model()
lib.lpdbg_set_timing(buf.data_ptr())
m, it, _ = prog.least_model()
lib.lpdbg_set_timing(None)
t = buf.cpu().numpy().reshape(16, G, 4).astype(np.float64)
print(cfg, "iters", it, "grid", G, prog.info["truth_mode"])
for k in range(min(it, 16)):
    s = t[k, :, 0]
    t0 = s.min()
    work = (t[k, :, 1] - s) / 1e3
    cta = (t[k, :, 2] - s) / 1e3
    exit_ = (t[k, :, 3] - t0) / 1e3
    print(f"pass {k}: start spread {(s.max()-t0)/1e3:7.1f}us  warp-done min/med/max "
          f"{work.min():7.1f}/{np.median(work):7.1f}/{work.max():7.1f}us  cta-done max {cta.max():7.1f}  "
          f"barrier exit {exit_.min():7.1f}..{exit_.max():7.1f}us  slowest cta {int(np.argmax(t[k,:,1]-s))}")
