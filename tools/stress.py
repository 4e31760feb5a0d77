"""Repeat least-model and stable calls many times (deadlock / race stress; profiling aid)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import oracle  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
t0 = time.time()
for P, kw in [(lpgen.chain(4097), {}), (lpgen.config("C1"), {}), (lpgen.layered(300, 16, 300 * 16 * 4, 3, seed=4), {}),
              (lpgen.config("C2"), dict(smem_bits_cap=4096))]:
    om, ostage, oit = oracle.lm_stage(P)
    ref = oracle.pack_bits(om)
    prog = lp.Program(P, **kw)
    for r in range(reps):
        for fr, sc in [(False, "auto"), (False, "stream"), (True, "auto")]:
            m, it, _ = prog.least_model(frontier=fr, schedule=sc)
            assert it == oit and (m == ref).all(), (r, fr, sc, it, oit)
    print("ok", P.n_atoms, reps, round(time.time() - t0, 1), flush=True)
rng = np.random.default_rng(5)
N = lpgen.random_normal_program(rng, 300, 1200, max_len=4, k_max=9)
o = oracle.stable(N)
sp = lp.Program(N)
for r in range(reps):
    ids, passes, _ = sp.stable_models()
    assert ids.tolist() == np.nonzero(o["accepted"])[0].tolist() and passes == o["passes"]
print("ok stable", reps, round(time.time() - t0, 1))
