import sys; sys.path.insert(0, ".")
import lpgen
from paper_2009_10247_b200 import lp
for cfg in sys.argv[1:]:
    P = lpgen.config(cfg); prog = lp.Program(P)
    for _ in range(3): prog.least_model()
    ts = []
    for _ in range(5):
        m, it, ex = prog.least_model(stats=True); ts.append(ex["stats"]["ns"] / 1e6)
    print(cfg, it, round(sorted(ts)[2], 4), "ms")
