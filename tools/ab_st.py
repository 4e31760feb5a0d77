"""Stable-model call time on C5 (median of 9, CUDA events around the host call; A/B aid).
usage: python tools/ab_st.py [CFG]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
prog = lp.Program(P)
for _ in range(3):
    ids, passes, _ = prog.stable_models()
ts = []
for _ in range(9):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids, passes, _ = prog.stable_models()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("stable", ids.tolist()[:4], "passes", passes, "ms", round(sorted(ts)[4], 4))
