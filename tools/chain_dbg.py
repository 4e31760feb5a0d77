import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, lpgen, oracle
from paper_2009_10247_b200 import lp
L = int(sys.argv[1])
P = lpgen.chain(L)
prog = lp.Program(P)
for fr, sched in [(False, "lead"), (False, "stream"), (False, "auto"), (True, "auto")]:
    t0 = time.time()
    print("run", fr, sched, flush=True)
    m, it, ex = prog.least_model(frontier=fr, schedule=sched, popcounts=True, stages=True, stats=True)
    print(fr, sched, it, time.time() - t0, ex["stats"], flush=True)
