"""Run a few calls of one configuration (for ncu captures).

usage: python tools/run_cfg.py CFG [calls] [key=value ...]
  keys: schedule=auto|lead|stream, frontier=1, v0=random1 (facts ∪ 1 % random atoms),
        stable=1 (lp_stable_models), search=H:SEED:ROUNDS:K (lp_stable_search on C5's
        recipe with K negated atoms), any UPPERCASE key is set in the environment
        (A/B switches are read by lp_load)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
kw = dict(a.split("=", 1) for a in sys.argv[3:])
for k, v in list(kw.items()):
    if k.isupper():
        os.environ[k] = v
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if "search" in kw:
    h, seed, rounds, k = (int(x) for x in kw["search"].split(":"))
    P = lpgen.gen_c5(seed=3, k=k)
    prog = lp.Program(P)
    for _ in range(calls):
        r = prog.stable_search(h, seed, rounds)
    print("search", r["rounds"], r["passes"], r["accepted"].tolist())
    sys.exit(0)
P = lpgen.config(sys.argv[1])
prog = lp.Program(P)
if kw.get("stable"):
    for _ in range(calls):
        ids, passes, _ = prog.stable_models()
    print(sys.argv[1], "stable", ids.tolist()[:4], passes)
    sys.exit(0)
v0 = None
if kw.get("v0") == "random1":
    rng = np.random.default_rng(20251020)
    facts = P.head[np.diff(P.body_ptr) == 0]
    v0 = np.union1d(facts, rng.choice(P.n_atoms, size=P.n_atoms // 100, replace=False))
for _ in range(calls):
    m, it, _ = prog.least_model(v0, schedule=kw.get("schedule", "auto"), frontier=bool(kw.get("frontier")))
print(sys.argv[1], "iters", it, "cluster", prog.info["cluster_ctas"])
