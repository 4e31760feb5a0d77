import sys, os; sys.path.insert(0, ".")
import torch, numpy as np, lpgen
from paper_2009_10247_b200 import lp
P = lpgen.config("C4"); prog = lp.Program(P)
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
model = torch.zeros(lp.bits_words(P.n_atoms), dtype=torch.int64, device="cuda")
iters = torch.zeros(1, dtype=torch.int32, device="cuda"); status = torch.zeros(1, dtype=torch.int32, device="cuda")
stats = torch.zeros(6, dtype=torch.int64, device="cuda")
for noflush in (False, True):
    a, b, c = [], [], []
    for i in range(23):
        if not noflush:
            with torch.cuda.stream(stream): flush.fill_(1)
        e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e0.record(stream)
        lp.lp_least_model(prog, None, model, stream=stream, device_ptrs=True, iters_out=iters, ev_begin=k0, ev_end=k1, stats=stats, status_out=status)
        e1.record(stream); stream.synchronize()
        if i >= 3:
            a.append(e0.elapsed_time(k0)); b.append(k0.elapsed_time(k1)); c.append(k1.elapsed_time(e1))
    print(os.environ.get("LP_NO_ARMED"), "noflush" if noflush else "flush", "pre %.4f kernel %.4f post %.4f ms" % (np.mean(a), np.mean(b), np.mean(c)))
