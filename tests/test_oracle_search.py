"""Pins of oracle/search.py (guess-space reduction, reading R23)
against things the paper and the mathematics fix, not against its own code:

  * the generator is SplitMix64: its published outputs for state 0;
  * every accepted column is a stable model by the Gelfond-Lifschitz definition
    (brute-force enumeration, oracle/brute.py), and a program without a stable model is
    never reported found;
  * the local-search move changes only violated pairs of Algorithm 3's test
     and always changes at least one;
  * definite programs (k = 0): the first round accepts every column, each being the
    least model;
  * Def. 8 item 3: a negated atom that is a fact keeps abar = 0 in every column.
"""
import numpy as np
import pytest

import lpgen
import oracle
from oracle import brute, search


def test_splitmix64_published_outputs():
    # SplitMix64 with state 0 (Vigna's reference splitmix64.c): the first three outputs
    g = 0x9E3779B97F4A7C15
    assert search.mix(0) == 0xE220A8397B1DCDAF
    assert search.mix(g) == 0x6E789E6AA1B965F4
    assert search.mix((2 * g) & ((1 << 64) - 1)) == 0x06C45D188009454F


def test_random_bits_are_balanced_and_counter_based():
    bits = [search.rbit(7, 0, g, j) for g in range(64) for j in range(32)]
    assert 0.45 < np.mean(bits) < 0.55
    # a counter-based generator: the same (seed, r, g, j) gives the same bit, another
    # seed another stream
    assert [search.rbit(7, 0, g, 3) for g in range(64)] == [search.rbit(7, 0, g, 3) for g in range(64)]
    assert [search.rbit(7, 0, g, 3) for g in range(64)] != [search.rbit(8, 0, g, 3) for g in range(64)]


@pytest.mark.parametrize("seed", range(40))
def test_local_move_flips_only_violated_pairs(seed):
    rng = np.random.default_rng([seed, 31])
    k = int(rng.integers(1, 40))
    bar = rng.integers(0, 2, size=k).astype(np.uint8)
    in_lm = rng.integers(0, 2, size=k).astype(np.uint8)
    viol = {j for j in range(k) if int(in_lm[j]) + int(bar[j]) != 1}
    if not viol:
        in_lm[0] = bar[0]          # a_0 ∈ LM iff abar_0 = 1: the pair sums to 0 or 2
        viol = {0}
    new = search.local_move(bar, in_lm, seed, 1, int(rng.integers(0, 4096)))
    changed = {j for j in range(k) if new[j] != bar[j]}
    assert changed and changed <= viol


def _small_normal(seed):
    rng = np.random.default_rng([seed, 1234])
    n = int(rng.integers(2, 11))
    R = int(rng.integers(1, 3 * n + 2))
    return lpgen.random_normal_program(rng, n, R, max_len=3, k_max=6), rng


@pytest.mark.parametrize("seed", range(150))
def test_search_accepts_only_stable_models(seed):
    P, rng = _small_normal(seed)
    n = P.n_atoms
    sm = brute.stable_brute(P)
    res = search.stable_search(P, h=8, seed=seed, max_rounds=24)
    if not sm:
        assert not res["found"] and res["rounds"] == 24
        return
    for g in res["accepted"]:
        I = frozenset(a for a in range(n) if (int(res["models"][g, a >> 6]) >> (a & 63)) & 1)
        assert I in sm and brute.is_stable(P, I)
        # the accepted column's abar values are the complement of the model on the
        # negated atoms (Algorithm 3's test)
        for j, a in enumerate(res["negated"]):
            assert res["guesses"][g, j] == (0 if a in I else 1)
    facts = set(P.head[np.diff(P.body_ptr) == 0].tolist())
    for j, a in enumerate(res["negated"]):
        if a in facts:
            assert not res["guesses"][:, j].any()   # Def. 8 item 3: forced 0


def test_search_finds_most_programs_with_models():
    found = total = 0
    for seed in range(150):
        P, _ = _small_normal(seed)
        if brute.stable_brute(P):
            total += 1
            found += search.stable_search(P, h=8, seed=seed, max_rounds=24)["found"]
    assert total > 50 and found >= 0.9 * total, (found, total)


def test_no_stable_model_and_definite_programs():
    # p <- not p has no stable model (PAPER.md Example-free textbook case)
    P = lpgen.from_lists(1, [(0, [], [0])])
    r = search.stable_search(P, h=64, seed=3, max_rounds=5)
    assert not r["found"] and r["rounds"] == 5
    # a definite program: every column is accepted at once, each the least model
    D = lpgen.from_lists(4, [(0, [1, 2]), (2, [3]), (3, [])])
    r = search.stable_search(D, h=64, seed=1, max_rounds=5)
    lm = brute.lm_brute(D)
    assert r["found"] and r["rounds"] == 1 and r["accepted"] == list(range(64))
    I = frozenset(a for a in range(4) if (int(r["models"][0, 0]) >> a) & 1)
    assert I == lm


def test_choice_pairs_many_negations():
    """20 independent choices p_i <- not q_i, q_i <- not p_i (k = 40, 2^20 stable models;
    enumeration would need 2^40 columns): every accepted column picks exactly one of each
    pair."""
    rules = []
    for i in range(20):
        rules += [(2 * i, [], [2 * i + 1]), (2 * i + 1, [], [2 * i])]
    P = lpgen.from_lists(40, rules)
    r = search.stable_search(P, h=64, seed=11, max_rounds=40)
    assert r["found"] and r["k"] == 40
    for g in r["accepted"]:
        I = {a for a in range(40) if (int(r["models"][g, 0]) >> a) & 1}
        assert all((2 * i in I) != (2 * i + 1 in I) for i in range(20))
        assert brute.is_stable(P, frozenset(I))
