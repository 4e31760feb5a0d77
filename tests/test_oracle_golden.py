"""Oracle pins against the values the paper prints (tests/golden/, each citing PAPER.md)
and against hand-worked T_P iterations of those examples."""
from fractions import Fraction

import numpy as np

import lpgen
import oracle
from oracle import brute, paper

from golden_io import load, matrix, nums, parse_rules, to_rules


def _example1():
    g = load("example1.txt")
    names = g["atoms"][0].split()
    P = to_rules(parse_rules(g["program"], names), len(names))
    return g, names, P


def _std_as_set(std, names):
    out = set()
    for kind, h, body in std:
        out.add((kind, names[h], frozenset(names[b] for b in body)))
    return out


def test_example1_standardization():
    """P' of Example 1: u <- q∧r, v <- s∧t, p <- u∨v, ..."""
    g, names, P = _example1()
    m, std = paper.standardize(P)
    snames = g["standardized_atoms"][0].split()
    assert m == len(snames) == 7
    want = set()
    for kind, h, pos, _ in parse_rules(g["standardized"], snames):
        want.add((kind, snames[h], frozenset(snames[b] for b in pos)))
    assert _std_as_set(std, snames) == want


def test_example1_program_matrix():
    """The 7×7 matrix printed in Example 1, entry for entry."""
    g, names, P = _example1()
    m, std = paper.standardize(P)
    assert paper.program_matrix(m, std) == matrix(g["matrix"])


def test_example3_coo_and_example4_csr():
    """COO arrays of Example 3, CSR arrays of Example 4."""
    _, _, P = _example1()
    m, std = paper.standardize(P)
    M = paper.program_matrix(m, std)
    g = load("example3_4.txt")
    rows, cols, vals = paper.to_coo(M)
    assert rows == nums(g["coo_row"]) and cols == nums(g["coo_col"])
    assert [float(v) for v in vals] == nums(g["coo_val"], float)
    ri, ci, vi = paper.to_csr(M)
    assert ri == nums(g["csr_row"]) and ci == nums(g["csr_col"])
    assert [float(v) for v in vi] == nums(g["csr_val"], float)


def test_example1_theta_step_by_hand():
    """Hand-worked product on P' (Def. 2 + Def. 5): v0 = {s, t} (Def. 4) gives
    M v0 = (0, 1, 1, 1, 1, 0, 1) over rows (p,q,r,s,t,u,v) -- row u is (q+r)/2 = 0,
    row v is (s+t)/2 = 1 -- and θ leaves it unchanged: {q, r, s, t, v}."""
    _, _, P = _example1()
    m, std = paper.standardize(P)
    M = paper.program_matrix(m, std)
    v0 = paper.initial_vector(m, std)
    assert v0 == [0, 0, 0, 1, 1, 0, 0]
    assert paper.matvec(M, v0) == [0, 1, 1, 1, 1, 0, 1]
    assert paper.theta(paper.matvec(M, v0)) == [0, 1, 1, 1, 1, 0, 1]


def test_example1_algorithm1_literal():
    """Algorithm 1 on Example 1, by hand: v0={s,t} -> {q,r,s,t,v} -> {p..v} -> same;
    3 products, |v| trace 2, 5, 7; least model restricted to B_P = {p,q,r,s,t}."""
    _, names, P = _example1()
    res = paper.algorithm1(P)
    assert res["v"] == [1] * 7
    assert res["products"] == 3
    assert res["trace"] == [2, 5, 7]


def test_example1_oracle_convention_B():
    """T_P over the original P from I_0 = facts {s,t}:
    T_P(I_0) ∪ I_0 = {p,q,r,s,t} (r<-s, q<-t, p<-s∧t), then no change:
    iters = 2 (k* = 1), popcounts [2, 5]."""
    _, names, P = _example1()
    model, iters, pops, conv = oracle.lm_jacobi(P)
    assert conv and iters == 2 and pops == [2, 5]
    assert [names[a] for a in np.nonzero(model)[0]] == ["p", "q", "r", "s", "t"]
    m2, stage, it2 = oracle.lm_stage(P)
    assert (m2 == model).all() and it2 == 2
    assert stage.tolist() == [1, 1, 1, 0, 0]
    assert oracle.certify(P, None, model, stage, iters) == 0
    assert brute.lm_brute(P) == frozenset(range(5))


def _example2():
    g = load("example2.txt")
    names = g["atoms"][0].split()
    P = to_rules(parse_rules(g["program"], names), len(names))
    return g, names, P


def test_example2_positive_form_and_matrix():
    """P+  and the 7×7 normal program matrix."""
    g, names, P = _example2()
    plus, negs = paper.positive_form(P)
    pn = g["plus_atoms"][0].split()
    assert negs == [names.index("t")]
    want = {(pn[h], frozenset(pn[b] for b in pos)) for _, h, pos, _ in parse_rules(g["plus"], pn)}
    got = {(pn[plus.rule(r)[0]], frozenset(pn[b] for b in plus.rule(r)[1])) for r in range(plus.n_rules)}
    assert got == want
    M, m, std, negs, n = paper.normal_matrix(P)
    assert m == 7
    assert M == matrix(g["matrix"])


def test_example2_stable_models():
    """Example 2: t is a fact, so the t̄ row of the initial matrix is forced 0 (Def. 8
    item 3) and h = 1 column.  Iterating: s <- t̄ never fires, p, q need
    s; u needs v.  Fixpoint column = {t}; t + t̄ = 1 + 0 = 1: accepted (Alg. 3).
    Stable models = {{t}} (GL brute force agrees)."""
    g, names, P = _example2()
    t = names.index("t")
    cols, free = paper.initial_matrix(P)
    assert free == [] and len(cols) == 1
    assert cols[0] == [0, 0, 0, 1, 0, 0, 0]
    res = paper.algorithm2_3(P)
    assert res["accepted"] == [0] and res["models"] == [frozenset([t])]
    o = oracle.stable(P, want_models=True)
    assert o["k"] == 1 and o["f"] == 0 and o["accepted"].tolist() == [1]
    assert brute.stable_brute(P) == [frozenset([t])]
    # explicit guesses over all k=1 negated atoms: t̄=1 is rejected (t ∈ LM and t̄ = 1)
    o2 = oracle.stable(P, guesses=[[0], [1]])
    assert o2["accepted"].tolist() == [1, 0]


def test_two_cycle_and_odd_loop():
    """{p <- ¬q, q <- ¬p}: guesses (p̄,q̄) = bits (0,1) of g.  g=1: p̄=1,q̄=0 -> q derived,
    p not: consistent -> model {q}; g=2 -> {p}; g=0 (both assumed true) -> nothing
    derivable, p ∉ LM but p̄ = 0: rejected; g=3 -> both derived, p̄ = 1: rejected.
    {p <- ¬p}: no stable model."""
    P = lpgen.from_lists(2, [(0, [], [1]), (1, [], [0])])
    o = oracle.stable(P, want_models=True)
    assert o["accepted"].tolist() == [0, 1, 1, 0]
    assert o["models"][1, 0] == 0b10 and o["models"][2, 0] == 0b01
    assert paper.algorithm2_3(P)["accepted"] == [1, 2]
    assert brute.stable_brute(P) == [frozenset([0]), frozenset([1])]
    Q = lpgen.from_lists(1, [(0, [], [0])])
    assert oracle.stable(Q)["accepted"].tolist() == [0, 0]
    assert paper.algorithm2_3(Q)["accepted"] == []
    assert brute.stable_brute(Q) == []


def test_theta_float_pitfall_reading_C1():
    """Reading C1: θ on 1/m sums is exact only in exact arithmetic.  Left-to-right
    float64 sums of m copies of 1/m fall below 1 for m = 6, 7, 10; the exact rational
    form (paper.py) and the integer count form (lp_oracle.c) both fire."""
    for m in (6, 7, 10):
        s = 0.0
        for _ in range(m):
            s += 1.0 / m
        assert s < 1.0
        assert paper.theta(sum([Fraction(1, m)] * m)) == 1
        P = lpgen.from_lists(m + 1, [(m, list(range(m)))] + [(a, []) for a in range(m)])
        model, iters, _, _ = oracle.lm_jacobi(P)
        assert model[m] == 1 and iters == 2
        assert paper.algorithm1(P)["v"][m] == 1


def test_sparsity_eq5_example1():
    """Eq. 5 on the standardized P' of Example 1: Σ|body| = 2+2+2+1+1+0+0 = 8, n = 7:
    1 - 8/49."""
    _, _, P = _example1()
    m, std = paper.standardize(P)
    tot = sum(len(b) for _, _, b in std)
    assert tot == 8 and abs((1 - tot / m**2) - (1 - 8 / 49)) < 1e-15
