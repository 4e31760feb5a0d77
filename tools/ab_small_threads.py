"""C1 on the small-program kernel: threads per CTA (LP_SMALL_THREADS, read by lp_load);
device pointers, L2 flushed, events around the launch (A/B aid)."""
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
for th in (1024, 768, 512, 384, 256, 128):
    os.environ["LP_SMALL_THREADS"] = str(th)
    prog = lp.Program(P)
    model = torch.zeros(lp.bits_words(P.n_atoms), dtype=torch.int64, device="cuda")
    iters = torch.zeros(1, dtype=torch.int32, device="cuda")
    tk = []
    with torch.cuda.stream(stream):
        for i in range(33):
            flush.fill_(i)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            lp.lp_least_model(prog, None, model, stream=stream, device_ptrs=True, iters_out=iters, ev_begin=k0, ev_end=k1)
            stream.synchronize()
            if i >= 3:
                tk.append(k0.elapsed_time(k1))
    print(f"threads {th:5d} small_rows {prog.info['small_rows']} iters {int(iters.item())} kernel ms median {np.median(tk):.4f} min {min(tk):.4f}")
    prog.close()
