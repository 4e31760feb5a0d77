"""Small runs of every kernel for compute-sanitizer (racecheck / synccheck / memcheck).

usage: compute-sanitizer --tool racecheck python tools/sanitize_case.py [case ...]
cases: c1 (C1: cluster kernel + persistent schedules + frontier), c2 (C2 exact),
       key (summary / key-space LEAD passes: plain, overlapped, pipelined; STREAM passes),
       stable (stable models + guess-space search), shard (combine kernel), all (default)
Every result is checked against the oracle so a racy run cannot pass silently.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import oracle  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cases = set(sys.argv[1:]) or {"all"}
want = lambda c: "all" in cases or c in cases  # noqa: E731


def check(P, prog, v0=None, **kw):
    om, ostage, oit = oracle.lm_stage(P, v0=v0)
    model, it, ex = prog.least_model(v0, stages=True, popcounts=True, **kw)
    assert it == oit and (model == oracle.pack_bits(om)).all() and (ex["stage"] == ostage).all(), kw


if want("c1"):
    P = lpgen.config("C1")
    prog = lp.Program(P)
    assert prog.info["cluster_ctas"] >= 1
    for kw in (dict(), dict(schedule="lead"), dict(schedule="stream"), dict(frontier=True)):
        check(P, prog, **kw)
    check(P, prog, v0=list(range(0, 1000, 7)))
    print("c1 ok", flush=True)
if want("c2"):
    P = lpgen.config("C2")
    prog = lp.Program(P)
    check(P, prog)
    check(P, prog, schedule="lead")
    print("c2 ok", flush=True)
if want("key"):
    rng = np.random.default_rng(1)
    P = lpgen.random_program(rng, 3000, 12000, max_len=5, n_facts=300)
    for env in ({}, {"LP_OVERLAP_MIN_MB": "0"}):
        os.environ.update(env)
        for kw in (dict(smem_bits_cap=256), dict(smem_bits_cap=128, grid_blocks=2)):
            prog = lp.Program(P, **kw)
            for sc in ("auto", "lead", "stream"):
                check(P, prog, schedule=sc)
            check(P, prog, schedule="lead", pipeline=False)
            check(P, prog, v0=rng.choice(3000, 300, replace=False).tolist())
            prog.close()
        for k in env:
            del os.environ[k]
    print("key ok", flush=True)
if want("stable"):
    N = lpgen.random_normal_program(np.random.default_rng(2), 200, 800, max_len=3, k_max=8)
    sp = lp.Program(N)
    o = oracle.stable(N)
    ids, passes, _ = sp.stable_models()
    assert ids.tolist() == np.nonzero(o["accepted"])[0].tolist() and passes == o["passes"]
    from oracle import search
    S = lpgen.gen_c5(seed=3, n=4000, R=20000, k=24)
    r = search.stable_search(S, h=128, seed=5, max_rounds=6)
    g = lp.Program(S).stable_search(128, 5, 6)
    assert g["rounds"] == r["rounds"] and g["accepted"].tolist() == r["accepted"]
    print("stable ok", flush=True)
if want("shard"):
    import torch
    from paper_2009_10247_b200.shard import derivable_mask, head_ranges, owned_words, sub_program
    rng = np.random.default_rng(3)
    P = lpgen.random_program(rng, 3000, 12000, max_len=5, n_facts=100)
    world = 3
    ow = owned_words(P, world)
    progs = [lp.Program(sub_program(P, lo, hi), derivable=derivable_mask(P)) for lo, hi in head_ranges(P, world)]
    stride = max(c for _, c in ow) + 1
    W = (P.n_atoms + 63) // 64
    gathered = torch.zeros(world * stride, dtype=torch.int64, device="cuda")
    ptr = np.asarray(P.body_ptr)
    start = np.zeros(W * 64, dtype=np.uint8)
    start[np.asarray(P.head)[ptr[1:] == ptr[:-1]]] = 1
    v = [torch.from_numpy(np.packbits(start, bitorder="little").view(np.int64).copy()).cuda(),
         torch.zeros(W, dtype=torch.int64, device="cuda")]
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    ch = torch.zeros(1, dtype=torch.int32, device="cuda")
    k = 0
    while True:
        for r, prog in enumerate(progs):
            row = gathered[r * stride:(r + 1) * stride]
            st = row.view(torch.int32)[2 * (stride - 1):2 * (stride - 1) + 1]
            lp.lp_least_model(prog, v[k & 1], row, device_ptrs=True, iters_out=it, max_passes=1,
                              status_out=st, out_words=ow[r])
        lp.lp_shard_combine(gathered, world, stride, [w for w, _ in ow], [c for _, c in ow], v[k & 1],
                            v[(k + 1) & 1], ch)
        k += 1
        if int(ch.item()) == 0:
            break
    om, _, oit = oracle.lm_stage(P)
    assert k == oit and (v[k & 1].cpu().numpy().view(np.uint64) == oracle.pack_bits(om)).all()
    print("shard ok", flush=True)
print("sanitize case done")
