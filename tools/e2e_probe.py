import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import lpgen
from paper_2009_10247_b200 import lp
P = lpgen.config("C4")
prog = lp.Program(P)
n = P.n_atoms
Wm = lp.bits_words(n)
stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
facts = P.head[np.diff(P.body_ptr) == 0]
v0_np = lp.pack_mask(np.isin(np.arange(n), facts))
v0_host = torch.zeros(Wm, dtype=torch.int64).pin_memory(); v0_host.numpy().view(np.uint64)[:] = v0_np[:Wm]
model_host = torch.zeros(Wm, dtype=torch.int64).pin_memory()
v0_dev = v0_host.cuda(); model_dev = torch.zeros(Wm, dtype=torch.int64, device="cuda")
it = torch.zeros(1, dtype=torch.int32, device="cuda")
def t(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        with torch.cuda.stream(stream): flush.fill_(i)
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); fn(); e1.record(stream); e1.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    return np.median(ts)
print("kernel v0=NULL (device)", t(lambda: lp.lp_least_model(prog, None, model_dev, stream=stream, device_ptrs=True, iters_out=it)))
print("kernel v0 given (device)", t(lambda: lp.lp_least_model(prog, v0_dev, model_dev, stream=stream, device_ptrs=True, iters_out=it)))
print("H2D 1.25MB pinned", t(lambda: v0_dev.copy_(v0_host, non_blocking=True) if False else torch.cuda.current_stream()))
def h2d():
    with torch.cuda.stream(stream): v0_dev.copy_(v0_host, non_blocking=True)
def d2h():
    with torch.cuda.stream(stream): model_host.copy_(model_dev, non_blocking=True)
print("H2D", t(h2d)); print("D2H", t(d2h))
print("e2e host call", t(lambda: lp.lp_least_model(prog, v0_host, model_host, stream=stream)))
print("e2e host call v0=None", t(lambda: lp.lp_least_model(prog, None, model_host, stream=stream)))
