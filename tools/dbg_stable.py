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
buf = torch.zeros(256, dtype=torch.int64, device="cuda")
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
for _ in range(3):
    prog.stable_models()
lib.lpdbg_set_timing(buf.data_ptr())
ids, passes, _ = prog.stable_models()
lib.lpdbg_set_timing(None)
t = buf.cpu().numpy().reshape(64, 4).astype(np.float64)
ph = t[63]
print(f"phases: clear {(ph[1] - ph[0]) / 1e3:.1f} us, init {(ph[2] - ph[1]) / 1e3:.1f} us, "
      f"fixpoint {(ph[3] - ph[2]) / 1e3:.1f} us (passes {passes}) -- stamps of CTA 0")
# pass k runs from barrier exit of k-1 to barrier exit of k
for k in range(1, passes):
    b0 = t[k - 1, 0]
    print(f"pass {k:2d}: top done +{(t[k, 2] - b0) / 1e3:5.1f}  scan+rows done +{(t[k, 3] - b0) / 1e3:5.1f}  "
          f"barrier exit +{(t[k, 0] - b0) / 1e3:5.1f} us   candidates {int(t[k, 1])}")
