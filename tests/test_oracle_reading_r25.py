"""Pin of DESIGN.md reading R25 (what the compact stable kernels rest on), on the oracle side
only: the least model A* of P+ with every abar_j true -- i.e. of P with its negative literals
deleted (Eq. 4; P+ is definite, so T_{P+} is monotone in the start set) --
contains the model of EVERY guess column of Algorithm 2, for enumerated
and for arbitrary explicit guesses (negated facts included), and a rule with a positive body
atom outside A* fires in no column."""
import numpy as np
import pytest

import lpgen
import oracle


def _without_negative_literals(P):
    rules = []
    for r in range(P.n_rules):
        s, e = int(P.body_ptr[r]), int(P.body_ptr[r + 1])
        pos = [int(a) for a, ng in zip(P.body_atom[s:e], P.body_neg[s:e]) if not ng]
        rules.append((int(P.head[r]), pos))
    return lpgen.from_lists(P.n_atoms, rules)


@pytest.mark.parametrize("seed", range(40))
def test_closure_contains_every_guess_model(seed):
    rng = np.random.default_rng([seed, 2525])
    n = int(rng.integers(2, 120))
    P = lpgen.random_normal_program(rng, n, int(rng.integers(1, 4 * n)), max_len=4, k_max=8)
    if P.body_neg is None or not P.body_neg.any():
        pytest.skip("definite program")
    D = _without_negative_literals(P)
    am, _, _ = oracle.lm_stage(D)
    astar = np.asarray(am, dtype=bool)
    k = len(oracle.negated_atoms(P))
    for guesses in (None, rng.integers(0, 2, size=(50, k)).astype(np.uint8)):
        o = oracle.stable(P, guesses=guesses, want_models=True)
        G = (1 << o["f"]) if guesses is None else guesses.shape[0]
        M = np.unpackbits(np.ascontiguousarray(o["models"][:G]).view(np.uint8), axis=1, bitorder="little")[:, :n].astype(bool)
        assert not (M & ~astar[None, :]).any()
        # a rule with a positive body atom outside A* fires in no column: its head is in a
        # column's model only through other rules -- check the rule's body is never satisfied
        for r in range(P.n_rules):
            s, e = int(P.body_ptr[r]), int(P.body_ptr[r + 1])
            pos = [int(a) for a, ng in zip(P.body_atom[s:e], P.body_neg[s:e]) if not ng]
            if any(not astar[a] for a in pos):
                assert not M[:, pos].all(axis=1).any()


def test_closure_is_strictly_larger_than_the_models_on_the_c5_recipe():
    """A* over-approximates: on the C5 recipe (scaled down) the columns' models differ from
    one another and from A*."""
    P = lpgen.gen_c5(seed=2, n=3000, R=15000, k=6, occ=10)
    D = _without_negative_literals(P)
    am, _, _ = oracle.lm_stage(D)
    astar = np.asarray(am, dtype=bool)
    o = oracle.stable(P, want_models=True)
    M = np.unpackbits(np.ascontiguousarray(o["models"]).view(np.uint8), axis=1, bitorder="little")[:, :P.n_atoms].astype(bool)
    assert not (M & ~astar[None, :]).any()
    assert (M.sum(axis=1) <= astar.sum()).all()
