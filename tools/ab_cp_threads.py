"""C5 stable call, compact kernel: threads per CTA (LP_CP_THREADS, read by lp_load); device
pointers, L2 flushed, events around the launch (A/B aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.config("C5")
flush = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
stream = torch.cuda.Stream()
for th in (1024, 768, 512, 384, 256):
    os.environ["LP_CP_THREADS"] = str(th)
    prog = lp.Program(P)
    G = 4096
    acc = torch.zeros(64, dtype=torch.int64, device="cuda")
    nacc = torch.zeros(1, dtype=torch.int64, device="cuda")
    passes = torch.zeros(1, dtype=torch.int32, device="cuda")
    tk = []
    with torch.cuda.stream(stream):
        for i in range(23):
            flush.fill_(i)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            lp.lp_stable_models(prog, None, G, acc, stream=stream, device_ptrs=True, n_accepted_out=nacc,
                                passes_out=passes, ev_begin=k0, ev_end=k1)
            stream.synchronize()
            if i >= 3:
                tk.append(k0.elapsed_time(k1))
    print(f"threads {th:5d} passes {int(passes.item())} accepted {int(nacc.item())} kernel ms median {np.median(tk):.4f} min {min(tk):.4f}")
    prog.close()
