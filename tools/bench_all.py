"""Time every configuration and variant (profiling aid; the driver's number is bench.py).

For each of C1..C4: full θ-pass and frontier fixpoint; C5: stable models.  CUDA events
on the launching stream, L2 flushed before every step, 3 warm-ups, K timed steps.
Prints one JSON object per line.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

K = int(os.environ.get("STEPS", "20"))
cfgs = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
SCHEDULES = os.environ.get("SCHEDULES", "auto,stream").split(",")
GRID = int(os.environ.get("GRID", "0"))
stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")


def timed(fn, steps=K, warm=3):
    tot, ker = [], []
    for i in range(warm + steps):
        with torch.cuda.stream(stream):
            flush.fill_(i)
        e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e0.record(stream)
        fn(k0, k1)
        e1.record(stream)
        stream.synchronize()
        if i >= warm:
            tot.append(e0.elapsed_time(e1))
            ker.append(k0.elapsed_time(k1))
    return float(np.median(tot)), float(np.median(ker))


for cfg in cfgs:
    P = lpgen.config(cfg)
    t0 = time.perf_counter()
    prog = lp.Program(P, grid_blocks=GRID)
    load_s = time.perf_counter() - t0
    info = prog.info
    if cfg == "C5":
        G = 1 << info["n_free_negated"]
        W = (G + 63) // 64
        acc = torch.zeros(W, dtype=torch.int64, device="cuda")
        nacc = torch.zeros(1, dtype=torch.int64, device="cuda")
        passes = torch.zeros(1, dtype=torch.int32, device="cuda")
        ms, kms = timed(lambda a, b: lp.lp_stable_models(prog, None, G, acc, stream=stream, device_ptrs=True,
                                                         n_accepted_out=nacc, passes_out=passes,
                                                         ev_begin=a, ev_end=b))
        print(json.dumps({"cfg": cfg, "variant": "stable", "step_ms": ms, "kernel_ms": kms,
                          "passes": int(passes.item()), "guesses": G, "guesses_per_s": G / (ms / 1e3),
                          "load_s": load_s}), flush=True)
        continue
    Wm = lp.bits_words(P.n_atoms)
    model = torch.zeros(max(Wm, 1), dtype=torch.int64, device="cuda")
    iters = torch.zeros(1, dtype=torch.int32, device="cuda")
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    variants = [(False, s) for s in SCHEDULES] + [(True, "auto")]
    for frontier, sched in variants:
        ms, kms = timed(lambda a, b: lp.lp_least_model(prog, None, model, frontier=frontier, stream=stream,
                                                       device_ptrs=True, iters_out=iters, ev_begin=a, ev_end=b,
                                                       schedule=sched, stats=stats))
        it = int(iters.item())
        rec = {"cfg": cfg, "variant": "frontier" if frontier else f"full/{sched}", "step_ms": ms,
               "kernel_ms": kms, "iters": it, "nnz": info["nnz"], "nnz_iter_per_s": info["nnz"] * it / (ms / 1e3),
               "load_s": load_s, "truth_mode": info["truth_mode"], "grid": info["grid_blocks"]}
        if not frontier:
            st = [int(x) for x in stats.tolist()]
            rec.update(alg_bytes=st[0], lead_passes=st[1], rows_verified=st[2], entries_verified=st[3],
                       GBps=st[0] / (kms / 1e3) / 1e9, us_per_pass=kms * 1e3 / it)
        print(json.dumps(rec), flush=True)
    prog.close()
