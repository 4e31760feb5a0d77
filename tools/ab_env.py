"""A/B of an lp_load-time environment switch in one process: the same program loaded with
and without VAR=1, calls alternated, L2 flushed (256 MiB write) before each, lp_run events
around each launch; median of 15 per side.
usage: python tools/ab_env.py VAR CFG...   (full θ-pass and frontier of each config)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

var = sys.argv[1]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for cfg in sys.argv[2:]:
    P = lpgen.config(cfg)
    os.environ.pop(var, None)
    pa = lp.Program(P)
    os.environ[var] = "1"
    pb = lp.Program(P)
    os.environ.pop(var, None)
    n = P.n_atoms
    model = torch.zeros(lp.bits_words(n), dtype=torch.int64, device="cuda")
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    for frontier in (False, True):
        ts = {0: [], 1: []}
        for r in range(18):
            for side, prog in ((0, pa), (1, pb)):
                flush.fill_(r & 255)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                lp.lp_least_model(prog, None, model, frontier=frontier, stream=s.cuda_stream,
                                  device_ptrs=True, iters_out=it, ev_begin=e0, ev_end=e1)
                torch.cuda.synchronize()
                if r >= 3:
                    ts[side].append(e0.elapsed_time(e1))
        a, b = np.median(ts[0]), np.median(ts[1])
        print(f"{cfg} {'frontier' if frontier else 'full':8s} iters {int(it.item())}  default {a:.4f} ms  "
              f"{var}=1 {b:.4f} ms  ({100 * (b - a) / b:+.1f}% vs switch)", flush=True)
