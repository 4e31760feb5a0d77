"""B200 numbers beside the paper's Tables 2-6 (context only: other hardware, synthetic
stand-ins of the paper's random programs and KONECT graphs).

For every shape: generate (lpgen.paper_profile / paper_tc), load, and time on cuda:0
  * the least model, full θ-pass (convention (B)) and frontier variant,
  * the least model over the paper's own matrix M_{P^δ} (LP_LOAD_PAPER_LAYOUT, (A)),
  * for normal programs the stable-model search over all 2^f guesses, (B) and (A);
check each result against the CPU oracle (oracle/, test infrastructure) and print one JSON
line per shape plus a markdown table (--md FILE).  Times: CUDA events around the C-ABI
call with device pointers, L2 flushed before each call, median of --reps.

The paper's times (seconds, one CPU thread, Eigen; Tables 2-6) are copied below
with their line numbers, as context -- a different machine and different programs.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import oracle  # noqa: E402
from paper_2009_10247_b200 import lp  # noqa: E402

# "Sparse matrix" column, seconds (Table 2, 470-482 Table 3,
# 533-540 Table 4, 581-593 Table 5, 613-625 Table 6); h = "column size of the initial
# matrix" of Tables 5-6
PAPER = {
    "T2": [0.0071, 0.0127, 0.0357, 0.0605, 0.0692, 0.0675, 0.3798, 0.4832, 0.8643, 0.9429, 0.9048, 1.0614],
    "T3": [0.0384, 0.0519, 0.1634, 0.3772, 0.5499, 0.6284, 1.0816, 2.2907, 3.7931, 4.8605, 5.3361, 5.9182],
    "T4": [0.0255, 0.0365, 0.1824, 0.1830, 0.4019, 0.4524, 0.6618, 0.8300],
    "T5": [0.0119, 0.0178, 0.0559, 0.0832, 0.0897, 0.0991, 0.7124, 0.8424, 1.5603, 1.8314, 1.9170, 2.1066],
    "T6": [0.1133, 0.1867, 0.2219, 0.3462, 0.4131, 0.4895, 3.2504, 4.0186, 7.2193, 8.3059, 9.0177, 11.5203],
}
H = {"T5": [8, 8, 8, 7, 5, 8, 6, 7, 5, 6, 4, 4], "T6": [7, 8, 7, 8, 8, 7, 8, 6, 4, 5, 4, 4]}

stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")


def timed(fn, reps):
    ts = []
    for i in range(reps + 2):
        with torch.cuda.stream(stream):
            flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        stream.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def least(prog, n, reps, frontier=False):
    model = torch.zeros(max(lp.bits_words(n), 1), dtype=torch.int64, device="cuda")
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    ms = timed(lambda: lp.lp_least_model(prog, None, model, frontier=frontier, stream=stream,
                                         device_ptrs=True, iters_out=it), reps)
    return ms, int(it.item()), model.cpu().numpy().view(np.uint64)[:lp.bits_words(n)]


def stable(prog, reps):
    G = 1 << prog.info["n_free_negated"]
    W = (G + 63) // 64
    acc = torch.zeros(W, dtype=torch.int64, device="cuda")
    nacc = torch.zeros(1, dtype=torch.int64, device="cuda")
    passes = torch.zeros(1, dtype=torch.int32, device="cuda")
    ms = timed(lambda: lp.lp_stable_models(prog, None, G, acc, stream=stream, device_ptrs=True,
                                           n_accepted_out=nacc, passes_out=passes), reps)
    bits = np.unpackbits(acc.cpu().numpy().view(np.uint8), bitorder="little")[:G]
    return ms, int(passes.item()), np.nonzero(bits)[0].tolist(), G


def run_shape(tab, i, P, reps, check):
    n = P.n_atoms
    rec = {"table": tab, "row": i + 1, "n": n, "m": int(P.n_rules), "nnz": int(P.nnz)}
    t0 = time.perf_counter()
    prog = lp.Program(P)
    rec["load_s"] = time.perf_counter() - t0
    progA = lp.Program(P, paper_layout=True)
    rec["n_prime"] = n + progA.info["n_aux"]
    if P.is_definite():
        ms, it, model = least(prog, n, reps)
        fms, fit, fmodel = least(prog, n, reps, frontier=True)
        ams, ait, amodel = least(progA, n, reps)
        rec.update(full_ms=ms, iters_B=it, frontier_ms=fms, paperA_ms=ams, iters_A=ait)
        if check:
            om, _, oit = oracle.lm_stage(P)
            ref = oracle.pack_bits(om)
            rec["parity"] = bool(oit == it == fit and (model == ref).all() and (fmodel == ref).all()
                                 and (amodel == ref).all())
        ours = ms
    else:
        rec["f"] = prog.info["n_free_negated"]
        ms, passes, ids, G = stable(prog, reps)
        ams, apasses, aids, _ = stable(progA, reps)
        rec.update(guesses=G, stable_ms=ms, passes_B=passes, paperA_ms=ams, passes_A=apasses,
                   accepted=len(ids))
        if check and P.nnz * G < 3e9:   # (the oracle is single-threaded)
            o = oracle.stable(P)
            want = np.nonzero(o["accepted"])[0].tolist()
            rec["parity"] = bool(ids == want and aids == want and passes == o["passes"])
        ours = ms
    paper = PAPER[tab][i]
    rec["paper_s"] = paper
    rec["paper_over_ours"] = paper / (ours / 1e3)
    prog.close()
    progA.close()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", default="T2,T3,T4,T5,T6")
    ap.add_argument("--rows", default="")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--md", default="")
    args = ap.parse_args()
    rows = [int(x) - 1 for x in args.rows.split(",") if x]
    out = []
    for tab in args.tables.split(","):
        if tab == "T4":
            shapes = [(nm, None) for nm, _, _ in lpgen.PAPER_TC_GRAPHS]
        else:
            shapes = lpgen.PAPER_TABLES
        for i, sh in enumerate(shapes):
            if rows and i not in rows:
                continue
            if tab == "T4":
                P = lpgen.paper_tc(sh[0])
            else:
                n, m = sh
                P = lpgen.paper_profile(n, m, dense=tab in ("T3", "T6"),
                                        k_neg=H[tab][i] if tab in ("T5", "T6") else 0)
            rec = run_shape(tab, i, P, args.reps, not args.no_check)
            if tab == "T4":
                rec["graph"] = sh[0]
            print(json.dumps(rec), flush=True)
            out.append(rec)
    if args.md:
        with open(args.md, "w") as f:
            f.write("# B200 beside the paper's Tables 2-6 (tools/paper_tables.py)\n\n"
                    "Synthetic stand-ins of the paper's generator (lpgen.paper_profile, reading in "
                    "DESIGN.md) and of the KONECT graphs (seeded random digraphs of the same |V|, |E|); "
                    "paper times are its 'Sparse matrix' column (seconds, one CPU thread) -- context "
                    "only.  GPU times: median CUDA-event time of one C-ABI call (device pointers, L2 "
                    "flushed).  iters/passes (B) = T_P passes over P, (A) = products of Algorithm 1/2 "
                    "over M_{P^δ}.\n\n")
            f.write("| table | row | n | m | nnz | n' | iters (B)/(A) | GPU ms (B) | GPU ms (A) | frontier ms | "
                    "guesses | paper s | paper/ours | parity |\n|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in out:
                it = (f"{r.get('iters_B', r.get('passes_B'))}/{r.get('iters_A', r.get('passes_A'))}")
                f.write(f"| {r['table']}{' ' + r['graph'] if 'graph' in r else ''} | {r['row']} | {r['n']} | "
                        f"{r['m']} | {r['nnz']} | {r['n_prime']} | {it} | "
                        f"{r.get('full_ms', r.get('stable_ms')):.4f} | {r['paperA_ms']:.4f} | "
                        f"{r.get('frontier_ms', float('nan')):.4f} | {r.get('guesses', '')} | {r['paper_s']} | "
                        f"{r['paper_over_ours']:.0f}x | {r.get('parity', 'unchecked')} |\n")


if __name__ == "__main__":
    main()
