"""Small least-model and stable runs for compute-sanitizer (profiling aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

rng = np.random.default_rng(1)
P = lpgen.random_program(rng, 3000, 12000, max_len=5, n_facts=300)
for kw in (dict(), dict(smem_bits_cap=256), dict(smem_bits_cap=128, grid_blocks=2), dict(paper_layout=True)):
    prog = lp.Program(P, **kw)
    for fr, sc in ((False, "auto"), (False, "stream"), (False, "lead"), (True, "auto")):
        prog.least_model(frontier=fr, schedule=sc, popcounts=True, stages=True, stats=True)
    prog.least_model(max_passes=2)
    prog.close()
L = lpgen.layered(20, 64, 20 * 64 * 4, 3, seed=2)
lp.Program(L).least_model(popcounts=True)
N = lpgen.random_normal_program(np.random.default_rng(2), 200, 800, max_len=3, k_max=8)
sp = lp.Program(N)
sp.stable_models()
sp.stable_models(guess_offset=64, n_guesses=64) if (1 << sp.info["n_free_negated"]) > 64 else None
print("sanitize case done")
