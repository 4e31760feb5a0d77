"""Host-side cost of one lp_least_model call (profiling aid): calls queued back to back
without synchronisation, wall time per call; and the same with a 2 ms sleep kernel ahead
so the GPU never waits on the host.  usage: python tools/host_cost.py C4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

P = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
prog = lp.Program(P)
s = torch.cuda.Stream()
model = torch.zeros(lp.bits_words(P.n_atoms), dtype=torch.int64, device="cuda")
iters = torch.zeros(1, dtype=torch.int32, device="cuda")
for ev in (False, True):
    for _ in range(3):
        lp.lp_least_model(prog, None, model, stream=s, device_ptrs=True, iters_out=iters)
    s.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)   # keep the GPU busy while the host queues
    n = 20
    t0 = time.perf_counter()
    for _ in range(n):
        kw = {}
        if ev:
            kw = dict(ev_begin=torch.cuda.Event(enable_timing=True), ev_end=torch.cuda.Event(enable_timing=True))
        lp.lp_least_model(prog, None, model, stream=s, device_ptrs=True, iters_out=iters, **kw)
    t1 = time.perf_counter()
    s.synchronize()
    print(f"events={ev}: host {1e6 * (t1 - t0) / n:.1f} us per call")
