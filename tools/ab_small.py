"""C1 least model (full θ-pass, auto schedule): small-program kernel vs cluster kernel
(LP_NO_SMALL) vs persistent grid (LP_NO_CLUSTER); device pointers, L2 flushed, CUDA events
around the launch (A/B aid).  usage: python tools/ab_small.py [CFG]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "C1")
flush = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
stream = torch.cuda.Stream()
for mode, env in (("small", {}), ("cluster", {"LP_NO_SMALL": "1"}), ("grid", {"LP_NO_CLUSTER": "1"})):
    for k in ("LP_NO_SMALL", "LP_NO_CLUSTER"):
        os.environ.pop(k, None)
    os.environ.update(env)
    prog = lp.Program(P)
    W = lp.bits_words(P.n_atoms)
    model = torch.zeros(W, dtype=torch.int64, device="cuda")
    iters = torch.zeros(1, dtype=torch.int32, device="cuda")
    ts, tk = [], []
    with torch.cuda.stream(stream):
        for i in range(23):
            flush.fill_(i)
            e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e0.record(stream)
            lp.lp_least_model(prog, None, model, stream=stream, device_ptrs=True, iters_out=iters,
                              ev_begin=k0, ev_end=k1)
            e1.record(stream)
            stream.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
                tk.append(k0.elapsed_time(k1))
    print(f"{mode:8s} small_rows {prog.info['small_rows']} cluster {prog.info['cluster_ctas']} iters {int(iters.item())} "
          f"call ms median {np.median(ts):.4f}  kernel ms median {np.median(tk):.4f} min {min(tk):.4f}")
    prog.close()
