"""Oracle pins by brute-force enumeration of Herbrand interpretations (oracle/brute.py),
the paper's literal Algorithms 1-3 in exact arithmetic (oracle/paper.py) and the
certificate checker.  A dropped term, a wrong index or a wrong iteration count in
lp_oracle.c fails one of these."""
import numpy as np
import pytest

import lpgen
import oracle
from oracle import brute, paper


def _random_definite(seed):
    rng = np.random.default_rng([seed, 77])
    n = int(rng.integers(1, 13))
    R = int(rng.integers(0, 3 * n + 1))
    return lpgen.random_program(rng, n, R, max_len=int(rng.integers(1, 5))), rng


@pytest.mark.parametrize("seed", range(300))
def test_definite_vs_bruteforce(seed):
    P, rng = _random_definite(seed)
    n = P.n_atoms
    model, iters, pops, conv = oracle.lm_jacobi(P)
    assert conv
    lm = brute.lm_brute(P)
    assert frozenset(np.nonzero(model)[0].tolist()) == lm
    # O-STAGE agrees with O-LM on the model, the pass count and the popcount trace
    m2, stage, it2 = oracle.lm_stage(P)
    assert (m2 == model).all() and it2 == iters
    assert oracle.popcounts_from_stage(stage, iters) == pops
    # invariants: popcounts strictly increase up to k*, iters <= n + 1
    assert all(a < b for a, b in zip(pops, pops[1:]))
    assert 1 <= iters <= n + 1
    assert oracle.certify(P, None, model, stage, iters) == 0
    # the paper's Algorithm 1, literally (standardized matrix, 1/m, θ), restricted to B_P
    alg1 = paper.algorithm1(P)
    assert frozenset(a for a in range(n) if alg1["v"][a]) == lm
    # with a user start set v0: LM(P ∪ v0-as-facts)
    v0 = rng.choice(n, size=int(rng.integers(0, n + 1)), replace=False).tolist()
    mv, itv, _, _ = oracle.lm_jacobi(P, v0=v0)
    assert frozenset(np.nonzero(mv)[0].tolist()) == brute.lm_brute(P, v0)
    ms, sv, its = oracle.lm_stage(P, v0=v0)
    assert (ms == mv).all() and its == itv
    assert oracle.certify(P, v0, mv, sv, itv) == 0


def test_certificate_rejects_corruptions():
    rng = np.random.default_rng(5)
    bad = 0
    for trial in range(200):
        n = int(rng.integers(3, 12))
        P = lpgen.random_program(rng, n, 3 * n, max_len=3, n_facts=2)
        model, stage, iters = oracle.lm_stage(P)
        assert oracle.certify(P, None, model, stage, iters) == 0
        # wrong pass count
        assert oracle.certify(P, None, model, stage, iters + 1) != 0
        # flip one atom in or out of the model
        a = int(rng.integers(0, n))
        m2, s2 = model.copy(), stage.copy()
        m2[a] ^= 1
        s2[a] = -1 if m2[a] == 0 else int(stage.max()) + 1
        assert oracle.certify(P, None, m2, s2, int(max(s2.max(), 0)) + 1) != 0
        # shift one stage
        on = np.nonzero(stage > 0)[0]
        if on.size:
            s3 = stage.copy()
            s3[on[0]] += 1
            assert oracle.certify(P, None, model, s3, int(s3.max()) + 1) != 0
            bad += 1
    assert bad > 50


def _random_normal(seed):
    rng = np.random.default_rng([seed, 99])
    n = int(rng.integers(1, 10))
    R = int(rng.integers(0, 2 * n + 3))
    return lpgen.random_normal_program(rng, n, R, max_len=3, k_max=4), rng


@pytest.mark.parametrize("seed", range(200))
def test_stable_vs_gl_bruteforce(seed):
    P, rng = _random_normal(seed)
    n = P.n_atoms
    o = oracle.stable(P, want_models=True)
    acc = np.nonzero(o["accepted"])[0]
    models = [frozenset(a for a in range(n) if (int(o["models"][g, a >> 6]) >> (a & 63)) & 1)
              for g in acc]
    sm = brute.stable_brute(P)
    # accepted guesses are in bijection with the stable models (SURVEY §8(c) O-STABLE)
    assert sorted(models, key=sorted) == sm
    assert len(set(models)) == len(models)
    for I in models:
        assert brute.is_stable(P, I)
    # the paper's Algorithms 2-3 (exact arithmetic, reading R7) accept the same columns
    lit = paper.algorithm2_3(P)
    assert lit["accepted"] == acc.tolist()
    assert lit["models"] == models
    # every column's fixpoint (not only accepted ones) equals the paper's M_k column
    for g in range(len(lit["columns"])):
        col = lit["columns"][g]
        mine = [(int(o["models"][g, a >> 6]) >> (a & 63)) & 1 for a in range(n)]
        assert mine == col[:n]
    # explicit guesses over ALL k negated atoms (fact-negated ones included) give the
    # same stable models
    k = o["k"]
    if k <= 6:
        allg = [[(g >> j) & 1 for j in range(k)] for g in range(1 << k)]
        o2 = oracle.stable(P, guesses=allg, want_models=True)
        acc2 = np.nonzero(o2["accepted"])[0]
        m2 = sorted([frozenset(a for a in range(n) if (int(o2["models"][g, a >> 6]) >> (a & 63)) & 1)
                     for g in acc2], key=sorted)
        assert m2 == sm


@pytest.mark.parametrize("seed", range(100))
def test_stable_columns_are_jacobi_on_positive_form(seed):
    """Each guess column's k*_g equals the Jacobi count of P+ from facts ∪ abar-guess,
    computed independently by O-LM on the positive form."""
    P, rng = _random_normal(seed)
    o = oracle.stable(P)
    plus, negs = paper.positive_form(P)
    Pp = lpgen.from_lists(plus.n_atoms, [plus.rule(r)[:2] for r in range(plus.n_rules)])
    n = P.n_atoms
    facts = set(P.head[np.diff(P.body_ptr) == 0].tolist())
    free = [j for j, a in enumerate(negs) if a not in facts]
    for g in range(len(o["kstar"])):
        v0 = [n + j for i, j in enumerate(free) if (g >> i) & 1]
        _, iters, _, _ = oracle.lm_jacobi(Pp, v0=v0)
        assert o["kstar"][g] == iters - 1
    assert o["passes"] == int(o["kstar"].max()) + 1
