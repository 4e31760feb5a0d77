"""Phase stamps of the compact stable kernel on C5 (CTA 0; the last CTA's end), L2 flushed.
usage: python tools/dbg_compact.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

prog = lp.Program(lpgen.config("C5"))
lib = lp.library()
lib.lpdbg_set_timing.argtypes = [ctypes.c_void_p]
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
flush = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
for cold in (False, True):
    for _ in range(3):
        prog.stable_models()
    if cold:
        flush.fill_(1)
    torch.cuda.synchronize()
    lib.lpdbg_set_timing(buf.data_ptr())
    prog.stable_models()
    torch.cuda.synchronize()
    lib.lpdbg_set_timing(None)
    t = buf.cpu().numpy().astype(float)
    print("cold" if cold else "warm", "staged+T0 %.2f us, fixpoint %.2f, writeback+check %.2f, last CTA end %.2f" %
          ((t[1] - t[0]) / 1e3, (t[2] - t[1]) / 1e3, (t[3] - t[2]) / 1e3, (t[4] - t[0]) / 1e3))
    print("   per pass (us, rows changed):", " ".join(f"{(t[8 + 2 * k] - (t[6 + 2 * k] if k else t[1])) / 1e3:.2f}/{int(t[9 + 2 * k])}" for k in range(24) if t[8 + 2 * k] > 0))
