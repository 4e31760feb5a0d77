"""Brute-force enumeration of Herbrand interpretations -- TEST INFRASTRUCTURE ONLY.

Independent of both lp_oracle.c and paper.py: it never iterates T_P over a matrix and
never uses stages.  Small n only.

lm_brute(P)      least model of a definite program = the intersection of all of its
                 models ("I is the least model of P if I ⊆ J for any
                 model J"; models of a definite program are closed under intersection).
stable_brute(P)  stable models: every I ⊆ B_P with I = LM(P^I), where P^I is the
                 Gelfond-Lifschitz reduct (delete rules with a negative literal in I,
                 strip the remaining negative literals).  The paper characterises
                 stable models through Alferes et al.; the reduct is the
                 textbook definition that characterisation is proved against.
"""
from __future__ import annotations

import numpy as np


def _is_model_mask(n, rules, extra_true=None):
    """bool[2^n]: interpretation I (bitmask) is a model of the definite rules."""
    N = 1 << n
    I = np.arange(N, dtype=np.int64)
    ok = np.ones(N, dtype=bool)
    for r in range(rules.n_rules):
        h, pos, neg = rules.rule(r)
        assert not neg
        bm = 0
        for a in pos:
            bm |= 1 << a
        body_true = (I & bm) == bm
        head_true = ((I >> h) & 1).astype(bool)
        ok &= ~body_true | head_true
    if extra_true:
        bm = 0
        for a in extra_true:
            bm |= 1 << a
        ok &= (I & bm) == bm
    return ok


def lm_brute(rules, v0=()):
    """Intersection of all models of P ∪ {a <- : a ∈ v0}.  Returns a frozenset."""
    n = rules.n_atoms
    assert n <= 20
    ok = _is_model_mask(n, rules, extra_true=list(v0))
    models = np.nonzero(ok)[0]
    inter = (1 << n) - 1
    for I in models.tolist():
        inter &= I
    return frozenset(a for a in range(n) if (inter >> a) & 1)


def _lm_sets(n, rules_list):
    """Least model of a small definite program given as (head, pos) list, by naive
    saturation (used only inside the reduct check)."""
    I = set()
    changed = True
    while changed:
        changed = False
        for h, pos in rules_list:
            if h not in I and all(b in I for b in pos):
                I.add(h)
                changed = True
    return frozenset(I)


def reduct(rules, I):
    """Gelfond-Lifschitz reduct P^I as a (head, pos) list."""
    out = []
    for r in range(rules.n_rules):
        h, pos, neg = rules.rule(r)
        if any(a in I for a in neg):
            continue
        out.append((h, pos))
    return out


def stable_brute(rules):
    """All stable models (sorted list of frozensets)."""
    n = rules.n_atoms
    assert n <= 14
    res = []
    for mask in range(1 << n):
        I = frozenset(a for a in range(n) if (mask >> a) & 1)
        if _lm_sets(n, reduct(rules, I)) == I:
            res.append(I)
    return sorted(res, key=lambda s: sorted(s))


def is_stable(rules, I) -> bool:
    I = frozenset(I)
    return _lm_sets(rules.n_atoms, reduct(rules, I)) == I
