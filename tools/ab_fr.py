"""Frontier kernel time (stats-free: CUDA events around the host call, median of 9; A/B aid).
usage: python tools/ab_fr.py CFG..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

for cfg in sys.argv[1:]:
    P = lpgen.config(cfg)
    prog = lp.Program(P)
    for _ in range(3):
        prog.least_model(frontier=True)
    ts = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m, it, _ = prog.least_model(frontier=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(cfg, "frontier iters", it, "ms (host call)", round(sorted(ts)[4], 4), "cluster", prog.info["frontier_cluster_ctas"])
