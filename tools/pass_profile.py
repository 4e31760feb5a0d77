"""Average pass time over ranges of passes: kernel time of capped calls (profiling aid).

usage: python tools/pass_profile.py C3 [frontier=1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
fr = "frontier=1" in sys.argv
P = lpgen.config(cfg)
prog = lp.Program(P)
for _ in range(2):
    prog.least_model(frontier=fr)
prev_t, prev_c = 0.0, 0
for cap in (1, 2, 5, 10, 50, 100, 200, 400, 600, 800, 1000):
    ts = []
    for _ in range(3):
        m, it, ex = prog.least_model(max_passes=cap, stats=True, frontier=fr)
        ts.append(ex["stats"]["ns"] / 1e3 if not fr else 0)
    t = sorted(ts)[1]
    print(f"passes {prev_c:4d}..{it:4d}: total {t:8.1f} us, {((t - prev_t) / max(it - prev_c, 1)):6.2f} us/pass")
    prev_t, prev_c = t, it
    if it < cap:
        break
