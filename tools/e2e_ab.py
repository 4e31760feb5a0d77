"""A/B of the host-pointer (e2e) call on C4: pinned buffers, L2 flushed, median of 30."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
prog = lp.Program(P)
n = P.n_atoms
Wm = lp.bits_words(n)
stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
facts = P.head[np.diff(P.body_ptr) == 0]
v0_np = lp.pack_mask(np.isin(np.arange(n), facts))
v0_host = torch.zeros(Wm, dtype=torch.int64).pin_memory()
v0_host.numpy().view(np.uint64)[:] = v0_np[:Wm]
model_host = torch.zeros(Wm, dtype=torch.int64).pin_memory()
ref, it_ref, _ = prog.least_model()
ts = []
for i in range(33):
    with torch.cuda.stream(stream):
        flush.fill_(i)
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    it = lp.lp_least_model(prog, v0_host, model_host, stream=stream)
    e1.record(stream)
    e1.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
    assert it == it_ref and (model_host.numpy().view(np.uint64)[:len(ref)] == ref).all()
print({"env": {k: v for k, v in os.environ.items() if k.startswith("LP_NO_ZERO")}, "e2e_ms": float(np.median(ts))})
