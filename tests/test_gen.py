"""The seeded generators produce the configuration shapes DESIGN.md states, and are
deterministic per seed."""
import numpy as np
import pytest

import lpgen


def _check_bodies_distinct(P):
    L = np.diff(P.body_ptr)
    for Lv in np.unique(L):
        if Lv < 2:
            continue
        idx = np.nonzero(L == Lv)[0]
        rows = P.body_atom[(P.body_ptr[idx][:, None] + np.arange(Lv)).reshape(-1)].reshape(-1, Lv)
        s = np.sort(rows, axis=1)
        assert not (s[:, 1:] == s[:, :-1]).any()


def test_c1_shape_and_determinism():
    P = lpgen.gen_c1(1)
    Q = lpgen.gen_c1(1)
    assert (P.head == Q.head).all() and (P.body_atom == Q.body_atom).all()
    L = np.diff(P.body_ptr)
    assert P.n_atoms == 1000 and P.n_rules == 2050
    assert (L[:2000] >= 1).all() and (L[:2000] <= 4).all() and (L[2000:] == 0).all()
    assert len(set(P.head[2000:].tolist())) == 50
    for r in range(2000):       # no self-loop
        assert P.head[r] not in P.body_atom[P.body_ptr[r]:P.body_ptr[r + 1]]
    _check_bodies_distinct(P)
    assert not (lpgen.gen_c1(2).head == P.head).all()


def test_c2_c5_shapes():
    P = lpgen.gen_c2(1)
    L = np.diff(P.body_ptr)
    assert P.n_atoms == 100_000 and P.n_rules == 501_000
    assert L[:500_000].min() == 1 and L[:500_000].max() == 8 and (L[500_000:] == 0).all()
    _check_bodies_distinct(P)
    C = lpgen.gen_c5(1)
    L = np.diff(C.body_ptr)
    assert C.n_rules == 501_000 and L[:500_000].max() == 6
    negs = C.meta["negated_atoms"]
    assert len(negs) == 12
    facts = set(C.head[500_000:].tolist())
    assert not (set(negs) & facts)
    nb = C.body_neg.astype(bool)
    assert int(nb.sum()) == 240
    for a in negs:
        occ = np.nonzero(nb & (C.body_atom == a))[0]
        rules = np.searchsorted(C.body_ptr, occ, side="right") - 1
        assert len(set(rules.tolist())) == 20
        for r in rules:
            s, e = C.body_ptr[r], C.body_ptr[r + 1]
            assert (C.body_atom[s:e] == a).sum() == 1 and C.head[r] != a
    _check_bodies_distinct(C)


def test_c3_layers():
    P = lpgen.layered(30, 50, 5000, 3, seed=2)
    L = np.diff(P.body_ptr)
    nf = 5000
    assert (L[nf:] == 0).all() and (P.head[nf:] == np.arange(50)).all()
    lay_h = P.head[:nf] // 50
    first = P.body_atom[P.body_ptr[:nf]]
    assert (first // 50 == lay_h - 1).all()
    for r in range(0, nf, 7):
        b = P.body_atom[P.body_ptr[r]:P.body_ptr[r + 1]]
        assert (b // 50 <= lay_h[r] - 1).all()
    _check_bodies_distinct(P)


def test_c4_scaled_zipf():
    P = lpgen.gen_c4(1, n=200_000, R=1_000_000)
    L = np.diff(P.body_ptr)
    assert L[:1_000_000].min() == 1 and L[:1_000_000].max() == 5
    cnt = np.bincount(P.head[:1_000_000], minlength=200_000)
    top = np.sort(cnt)[::-1]
    # P(rank 1) = 1 / H_{n,1.1}
    Hn = (np.arange(1, 200_001, dtype=np.float64) ** -1.1).sum()
    assert abs(top[0] / 1e6 - 1 / Hn) < 0.01
    assert top[1] < top[0]
    _check_bodies_distinct(P)


@pytest.mark.parametrize("dense,k_neg", [(False, 0), (True, 0), (False, 6), (True, 8)])
def test_paper_profile_shapes(dense, k_neg):
    """lpgen.paper_profile follows reading R22: n//4 distinct facts, Table 1's body-length
    shares over the other rules (dense: lengths >= 3 become U[0.04 n, 0.06 n]), distinct
    body atoms, k_neg negated literal occurrences; deterministic."""
    n, m = 2000, 36000
    P = lpgen.paper_profile(n, m, dense=dense, k_neg=k_neg)
    Q = lpgen.paper_profile(n, m, dense=dense, k_neg=k_neg)
    assert (P.head == Q.head).all() and (P.body_atom == Q.body_atom).all()
    assert P.n_atoms == n and P.n_rules == m
    L = np.diff(P.body_ptr)
    facts = P.head[L == 0]
    assert facts.size == n // 4 and np.unique(facts).size == n // 4
    R = m - n // 4
    share = {l: (L == l).sum() / R for l in (1, 2)}
    assert abs(share[1] - 0.04) < 0.002 and abs(share[2] - 0.04) < 0.002
    if dense:
        big = L[L >= 3]
        assert big.min() >= int(0.04 * n) and big.max() <= int(0.06 * n)
    else:
        for l, s in zip(range(3, 9), (0.10, 0.40, 0.35, 0.04, 0.02, 0.01)):
            assert abs((L == l).sum() / R - s) < 0.002, l
    _check_bodies_distinct(P)
    if k_neg:
        assert int(P.body_neg.sum()) == k_neg
    else:
        assert P.body_neg is None


def test_paper_tc_sizes():
    for name, V, E in lpgen.PAPER_TC_GRAPHS:
        P = lpgen.paper_tc(name)
        facts = int((np.diff(P.body_ptr) == 0).sum())
        assert facts == E                            # one edge fact per edge
        assert P.n_atoms == E + V * V
        assert P.n_rules == 2 * E + E * V            # edges, base paths, recursive paths
