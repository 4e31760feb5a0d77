"""Repeat the compact stable / search kernels and the small-program kernel and compare every
run with the first (race check by repetition: compute-sanitizer is closed on this pool).
usage: python tools/stress_compact.py [reps]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import lpgen  # noqa: E402
import oracle  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
bad = 0

P = lpgen.config("C5")
prog = lp.Program(P)
assert prog.info["stable_compact_atoms"] > 0
o = oracle.stable(P)
want_ids = np.nonzero(o["accepted"])[0].tolist()
ref = None
for r in range(reps):
    ids, passes, _ = prog.stable_models()
    ok = ids.tolist() == want_ids and passes == o["passes"]
    if r % 20 == 0:   # (the whole fixpoint matrix, expanded from C)
        h = hashlib.sha1(prog.stable_matrix().tobytes()).hexdigest()
        ref = ref or h
        ok = ok and h == ref
    bad += not ok
print(f"C5 compact stable: {reps} calls, {bad} mismatches (accepted {want_ids}, passes {o['passes']}, matrix sha1 {ref[:12]})")

from oracle import search  # noqa: E402
S = lpgen.gen_c5(seed=3, n=100_000, R=500_000, k=32)
sp = lp.Program(S)
assert sp.info["stable_compact_atoms"] > 0
so = search.stable_search(S, h=128, seed=5, max_rounds=40)
sb = 0
for r in range(reps // 2):
    g = sp.stable_search(128, 5, 40)
    sb += not (g["rounds"] == so["rounds"] and g["passes"] == so["passes"] and g["accepted"].tolist() == so["accepted"]
               and (g["guesses"] == so["guesses"]).all())
print(f"k = 32 compact search: {reps // 2} calls, {sb} mismatches (rounds {so['rounds']}, passes {so['passes']})")

C1 = lpgen.config("C1")
cp = lp.Program(C1)
assert cp.info["small_rows"] > 0
om, ostage, oit = oracle.lm_stage(C1)
cb = 0
rng = np.random.default_rng(5)
for r in range(reps):
    frontier = bool(r & 1)
    model, iters, ex = cp.least_model(frontier=frontier, stages=True, popcounts=True)
    cb += not (iters == oit and (model == oracle.pack_bits(om)).all() and (ex["stage"] == ostage).all())
    if r % 10 == 0:   # a random start set
        v0 = rng.choice(C1.n_atoms, size=50, replace=False).tolist()
        m2, s2, i2 = oracle.lm_stage(C1, v0=v0)
        model, iters, ex = cp.least_model(v0=v0, stages=True)
        cb += not (iters == i2 and (model == oracle.pack_bits(m2)).all() and (ex["stage"] == s2).all())
print(f"C1 small-program kernel: {reps} calls (+ random start sets), {cb} mismatches")
sys.exit(1 if bad or sb or cb else 0)
