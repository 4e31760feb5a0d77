"""Run one config's least model a few times (target command for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
sched = sys.argv[2] if len(sys.argv) > 2 else "auto"
frontier = len(sys.argv) > 3 and sys.argv[3] == "frontier"
P = lpgen.config(cfg)
prog = lp.Program(P)
for _ in range(3):
    m, it, ex = prog.least_model(schedule=sched, frontier=frontier, stats=True)
print(cfg, sched, "iters", it, ex.get("stats"))
