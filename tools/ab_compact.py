"""Stable-model call on C5: compact kernel vs batched kernel (LP_NO_COMPACT_STABLE), device
pointers, L2 flushed before every call, CUDA events around the launch (A/B aid).
usage: python tools/ab_compact.py [CFG] [k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
P = lpgen.config(cfg) if len(sys.argv) < 3 else lpgen.gen_c5(seed=3, k=int(sys.argv[2]))
flush = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
stream = torch.cuda.Stream()
for mode in ("compact", "batched"):
    if mode == "batched":
        os.environ["LP_NO_COMPACT_STABLE"] = "1"
    else:
        os.environ.pop("LP_NO_COMPACT_STABLE", None)
    prog = lp.Program(P)
    G = 1 << min(prog.info["n_free_negated"], 16)
    W = (G + 63) // 64
    acc = torch.zeros(W, dtype=torch.int64, device="cuda")
    nacc = torch.zeros(1, dtype=torch.int64, device="cuda")
    passes = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ts, tk = [], []
    with torch.cuda.stream(stream):
        for i in range(13):
            flush.fill_(i)
            e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e0.record(stream)
            lp.lp_stable_models(prog, None, G, acc, stream=stream, device_ptrs=True, n_accepted_out=nacc,
                                passes_out=passes, ev_begin=k0, ev_end=k1, status_out=status)
            e1.record(stream)
            stream.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
                tk.append(k0.elapsed_time(k1))
    print(f"{mode:8s} G {G} compact atoms {prog.info['stable_compact_atoms']} rows {prog.info['stable_compact_rows']} "
          f"passes {int(passes.item())} accepted {int(nacc.item())} status {int(status.item())} "
          f"call ms median {np.median(ts):.4f} min {min(ts):.4f}  kernel ms median {np.median(tk):.4f} min {min(tk):.4f}")
    prog.close()
