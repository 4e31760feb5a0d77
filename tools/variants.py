"""A/B timing of full θ-pass variants on one configuration (measurement aid).

usage: python tools/variants.py C4 [name=ENV1,ENV2 ...]
Each variant loads the program with the listed A/B environment switches set (they are
read by lp_load) and times 20 device-pointer calls (L2 flushed before each) with CUDA
events; prints kernel and step medians and checks the model against the first variant.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
variants = [("default", [], {})]
for a in sys.argv[2:]:
    name, _, envs = a.partition("=")
    flags = {}
    env = []
    for e in envs.split(","):
        if not e:
            continue
        if e.startswith("sched:"):
            flags["schedule"] = e[6:]
        elif e == "nopipe":
            flags["pipeline"] = False
        elif e == "frontier":
            flags["frontier"] = True
        elif e == "key8":
            flags["key8"] = True
        else:
            env.append(e)
    variants.append((name, env, flags))
P = lpgen.config(cfg)
W = lp.bits_words(P.n_atoms)
stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
ref = None
for name, env, flags in variants:
    for e in env:
        os.environ[e] = "1"
    prog = lp.Program(P, key8=flags.get("key8", False))
    for e in env:
        del os.environ[e]
    model = torch.zeros(W, dtype=torch.int64, device="cuda")
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ks, ts = [], []
    for i in range(25):
        with torch.cuda.stream(stream):
            flush.fill_(i)
        e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e0.record(stream)
        lp.lp_least_model(prog, None, model, stream=stream, device_ptrs=True, iters_out=it,
                          ev_begin=k0, ev_end=k1, status_out=st,
                          schedule=flags.get("schedule", "auto"), pipeline=flags.get("pipeline", True),
                          frontier=flags.get("frontier", False))
        e1.record(stream)
        stream.synchronize()
        assert int(st.item()) == 0
        if i >= 5:
            ks.append(k0.elapsed_time(k1))
            ts.append(e0.elapsed_time(e1))
    m = model.cpu().numpy()
    if ref is None:
        ref = m
    print(f"{cfg} {name:14s} iters {int(it.item())} kernel med {1e3*np.median(ks):7.1f} us  step med "
          f"{1e3*np.median(ts):7.1f} us  model {'ok' if (m == ref).all() else 'MISMATCH'}", flush=True)
    prog.close()
