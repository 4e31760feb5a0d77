"""Per-pass timing and candidate counts of the stable-model fixpoint kernel (profiling aid)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
prog = lp.Program(P)
buf = torch.zeros(128, dtype=torch.int64, device="cuda")
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
for _ in range(3):
    prog.stable_models()
lib.lpdbg_set_timing(buf.data_ptr())
ids, passes, _ = prog.stable_models()
lib.lpdbg_set_timing(None)
t = buf.cpu().numpy().reshape(64, 2)
t0 = t[0, 0]
prev = None
for k in range(passes):
    dt = (t[k, 0] - prev) / 1e3 if prev is not None else float("nan")
    print(f"pass {k:2d}: barrier at {(t[k, 0] - t0) / 1e3:8.1f} us (+{dt:6.1f})  candidates {t[k, 1]}")
    prev = t[k, 0]
