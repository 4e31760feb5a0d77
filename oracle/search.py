"""Guess-space reduction by sampling + local search -- TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py for who may use it).

PAPER.md:647 (Conclusion) sketches the method without fixing its details:

    "apply a sampling method to reduce the number of guesses in the initial matrix for
     normal programs.  An algorithm would be to prepare some manageable size of the
     initial matrix, and if all guesses fail we do some local search and replace column
     vectors by new assignments then repeat it until a stable model is found."

DESIGN.md reading R23 fixes the details this file follows step by step, in the paper's
order and notation (Def. 8 initial matrix PAPER.md:243-253; Algorithms 2-3 PAPER.md:
256-300, reading R7 for the acceptance test):

  round 0   the initial matrix has h columns; column g gives abar_j (1 = a_j assumed
            false) the bit  rbit(seed, 0, g, j)  for every free negated atom j (not a fact),
            and 0 for a negated atom that is a fact (Def. 8 item 3, reading R8);
  round r   Algorithms 2-3 on the h columns (O-STABLE: oracle.stable with these guesses);
            if some column is accepted: stop -- the accepted columns are stable models;
  move      else every column g is replaced by a new assignment: with LM_g its fixpoint
            column, the violated pairs are V_g = { j : [a_j ∈ LM_g] + abar_j != 1 }
            (Algorithm 3's failing test; V_g is non-empty for a rejected column).  The new
            column flips abar_j for every j ∈ V_g with rbit(seed, r+1, g, j) = 1; if that
            flips nothing, it flips the single j = V_g[ rand64(seed, r+1, g, k) mod |V_g| ]
            (V_g in ascending j).  Then round r+1.
  stop      after max_rounds rounds without an accepted column ("not found").

Random numbers: a counter-based generator both sides implement (no state, no stream):
    mix(z) = SplitMix64's output function of the state z + 0x9E3779B97F4A7C15,
    rand64(seed, r, g, j) = mix(mix(mix(mix(seed) ^ r) ^ g) ^ j),   rbit = rand64 >> 63.
mix is pinned to the published SplitMix64 outputs for state 0 (tests).
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


def mix(z: int) -> int:
    """SplitMix64 (Steele, Lea, Flood 2014): the output for state z (advance, then mix)."""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def rand64(seed: int, r: int, g: int, j: int) -> int:
    return mix(mix(mix(mix(seed & _M64) ^ r) ^ g) ^ j)


def rbit(seed: int, r: int, g: int, j: int) -> int:
    return rand64(seed, r, g, j) >> 63


def initial_columns(k: int, free, h: int, seed: int) -> np.ndarray:
    """Round 0: uint8[h][k] abar values; free[j] = negated atom j is not a fact."""
    cols = np.zeros((h, k), dtype=np.uint8)
    for g in range(h):
        for j in range(k):
            if free[j]:
                cols[g, j] = rbit(seed, 0, g, j)
    return cols


def local_move(bar, in_lm, seed: int, r_next: int, g: int) -> np.ndarray:
    """The new column g for round r_next from its rejected column (abar values `bar`,
    in_lm[j] = a_j ∈ LM_g).  Returns the new abar values."""
    k = len(bar)
    viol = [j for j in range(k) if int(in_lm[j]) + int(bar[j]) != 1]
    assert viol, "a rejected column has a violated pair"
    flips = [j for j in viol if rbit(seed, r_next, g, j)]
    if not flips:
        flips = [viol[rand64(seed, r_next, g, k) % len(viol)]]
    new = np.array(bar, dtype=np.uint8)
    for j in flips:
        new[j] ^= 1
    return new


def stable_search(rules, h: int, seed: int, max_rounds: int):
    """Reading R23 of PAPER.md:647.  Returns dict(found, rounds, passes, accepted (local
    column ids of the last round, ascending), guesses uint8[h][k] of the last round,
    models uint64[h][words] of the last round, negated atom ids)."""
    import oracle
    negs = oracle.negated_atoms(rules)
    k = len(negs)
    facts = set(np.asarray(rules.head)[np.diff(rules.body_ptr) == 0].tolist())
    free = [a not in facts for a in negs]
    cols = initial_columns(k, free, h, seed)
    passes = 0
    for r in range(max_rounds):
        res = oracle.stable(rules, guesses=cols, want_models=True)
        passes += res["passes"]
        acc = np.nonzero(res["accepted"])[0]
        if acc.size or r == max_rounds - 1:
            return dict(found=bool(acc.size), rounds=r + 1, passes=passes, accepted=acc.tolist(),
                        guesses=cols, models=res["models"], negated=negs, k=k)
        models = res["models"]
        new = np.zeros_like(cols)
        for g in range(h):
            in_lm = [(int(models[g, a >> 6]) >> (a & 63)) & 1 for a in negs]
            new[g] = local_move(cols[g], in_lm, seed, r + 1, g)
        cols = new
    return dict(found=False, rounds=0, passes=0, accepted=[], guesses=cols, models=None,
                negated=negs, k=k)
