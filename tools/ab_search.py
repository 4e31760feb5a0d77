"""lp_stable_search on the C5 recipe with k = 32: compact vs batched kernel
(LP_NO_COMPACT_STABLE), device pointers, L2 flushed, CUDA events around the launch (A/B aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.gen_c5(seed=3, n=100_000, R=500_000, k=32)
flush = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
stream = torch.cuda.Stream()
for mode in ("compact", "batched"):
    if mode == "batched":
        os.environ["LP_NO_COMPACT_STABLE"] = "1"
    else:
        os.environ.pop("LP_NO_COMPACT_STABLE", None)
    prog = lp.Program(P)
    k = prog.info["n_negated"]
    gs = torch.zeros((k, 2), dtype=torch.int64, device="cuda")
    acc = torch.zeros(2, dtype=torch.int64, device="cuda")
    na = torch.zeros(1, dtype=torch.int64, device="cuda")
    rd = torch.zeros(1, dtype=torch.int32, device="cuda")
    ps = torch.zeros(1, dtype=torch.int32, device="cuda")
    ts = []
    with torch.cuda.stream(stream):
        for i in range(13):
            flush.fill_(i)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            lp.lp_stable_search(prog, 128, 5, 40, gs, acc, stream=stream, device_ptrs=True, n_accepted_out=na,
                                rounds_out=rd, passes_out=ps, ev_begin=k0, ev_end=k1)
            stream.synchronize()
            if i >= 3:
                ts.append(k0.elapsed_time(k1))
    print(f"{mode:8s} compact atoms {prog.info['stable_compact_atoms']} rows {prog.info['stable_compact_rows']} "
          f"rounds {int(rd.item())} passes {int(ps.item())} accepted {int(na.item())} kernel ms median {np.median(ts):.4f} min {min(ts):.4f}")
    prog.close()
