"""Seeded synthetic program generators (inputs only).

This module is shared by the oracle side (``oracle/``, tests) and the product side
(``paper_2009_10247_b200``, ``bench.py``).  It produces *programs* -- flat rule
arrays -- and nothing else: it holds none of the method's arithmetic (no T_P,
no matrices, no thresholds, no models).  Every generator is deterministic for a
given seed (numpy PCG64 via ``np.random.default_rng``).

Rule representation (identical to the C ABI's ``lp_rules``, include/lp.h):
    n_atoms    : int, atoms are 0..n_atoms-1
    head       : int32[R]
    body_ptr   : int64[R+1], body of rule r is body_ptr[r]:body_ptr[r+1]
    body_atom  : int32[nnz]
    body_neg   : uint8[nnz] or None (1 = the literal is ``not atom``)
A rule with an empty body is a fact ("A rule r is called a fact if
body(r)=∅").

The five BASELINE.json configurations C1..C5 follow the readings in SURVEY.md
§8(d) (restated in DESIGN.md "Input recipe").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "Rules", "from_lists", "config", "CONFIG_NAMES",
    "gen_c1", "gen_c2", "gen_c3", "gen_c4", "gen_c5",
    "random_program", "random_normal_program", "chain", "layered",
    "tc_program", "random_digraph", "paper_profile", "PAPER_TABLES", "PAPER_TC_GRAPHS",
]


@dataclass
class Rules:
    n_atoms: int
    head: np.ndarray
    body_ptr: np.ndarray
    body_atom: np.ndarray
    body_neg: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def n_rules(self) -> int:
        return int(self.head.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.body_atom.shape[0])

    def rule(self, r: int):
        """(head, [pos atoms], [neg atoms]) of rule r -- convenience for small tests."""
        s, e = int(self.body_ptr[r]), int(self.body_ptr[r + 1])
        atoms = self.body_atom[s:e].tolist()
        if self.body_neg is None:
            return int(self.head[r]), atoms, []
        neg = self.body_neg[s:e].tolist()
        return (int(self.head[r]), [a for a, g in zip(atoms, neg) if not g],
                [a for a, g in zip(atoms, neg) if g])

    def is_definite(self) -> bool:
        return self.body_neg is None or not bool(self.body_neg.any())


def from_lists(n_atoms: int, rules, meta=None) -> Rules:
    """rules: iterable of (head, pos_list) or (head, pos_list, neg_list)."""
    heads, ptr, atoms, negs = [], [0], [], []
    any_neg = False
    for rr in rules:
        h, pos = rr[0], list(rr[1])
        neg = list(rr[2]) if len(rr) > 2 else []
        any_neg |= bool(neg)
        heads.append(h)
        atoms.extend(pos)
        atoms.extend(neg)
        negs.extend([0] * len(pos) + [1] * len(neg))
        ptr.append(len(atoms))
    return Rules(
        n_atoms=int(n_atoms),
        head=np.asarray(heads, dtype=np.int32).reshape(-1),
        body_ptr=np.asarray(ptr, dtype=np.int64),
        body_atom=np.asarray(atoms, dtype=np.int32).reshape(-1),
        body_neg=np.asarray(negs, dtype=np.uint8) if any_neg else None,
        meta=dict(meta or {}),
    )


# ----------------------------------------------------------------------------------
# vectorised helpers
# ----------------------------------------------------------------------------------

def _distinct_rows_long(rng, count: int, L: int, n: int) -> np.ndarray:
    """int32[count, L] with distinct entries per row, uniform over [0, n), for bodies too
    long for whole-row rejection (L^2 >~ n): duplicates are redrawn position by position,
    then every row is shuffled.  Chunked to bound memory."""
    out = np.empty((count, L), dtype=np.int32)
    step = max(1, (1 << 24) // max(L, 1))
    for c0 in range(0, count, step):
        c1 = min(count, c0 + step)
        x = rng.integers(0, n, size=(c1 - c0, L), dtype=np.int64)
        while True:
            x.sort(axis=1)
            dup = np.zeros(x.shape, dtype=bool)
            dup[:, 1:] = x[:, 1:] == x[:, :-1]
            k = int(dup.sum())
            if not k:
                break
            x[dup] = rng.integers(0, n, size=k)
        out[c0:c1] = rng.permuted(x, axis=1)
    return out


def _distinct_rows(rng, count: int, L: int, lo, hi, forbid=None) -> np.ndarray:
    """int32[count, L], row entries distinct, uniform in [lo, hi) (lo/hi scalars or
    per-row arrays), and != forbid[row] when given.  Rejection-resamples bad rows."""
    lo_a = np.broadcast_to(np.asarray(lo, dtype=np.int64), (count,))
    hi_a = np.broadcast_to(np.asarray(hi, dtype=np.int64), (count,))
    out = np.empty((count, L), dtype=np.int32)
    todo = np.arange(count)
    while todo.size:
        span = (hi_a[todo] - lo_a[todo])[:, None]
        draw = (lo_a[todo][:, None] + (rng.random((todo.size, L)) * span).astype(np.int64)).astype(np.int32)
        bad = np.zeros(todo.size, dtype=bool)
        if L > 1:
            s = np.sort(draw, axis=1)
            bad |= (s[:, 1:] == s[:, :-1]).any(axis=1)
        if forbid is not None:
            bad |= (draw == np.asarray(forbid)[todo][:, None]).any(axis=1)
        out[todo[~bad]] = draw[~bad]
        todo = todo[bad]
    return out


def _assemble(n_atoms, heads, lengths, fill, rng, facts=None, meta=None) -> Rules:
    """Build CSR rule arrays.  ``fill(idx_rules, L) -> int32[len(idx), L]`` draws bodies
    for the rules of body length L.  ``facts`` (int array) are appended as empty-body
    rules after the non-fact rules."""
    heads = np.asarray(heads, dtype=np.int32)
    lengths = np.asarray(lengths, dtype=np.int64)
    if facts is not None and len(facts):
        heads = np.concatenate([heads, np.asarray(facts, dtype=np.int32)])
        lengths = np.concatenate([lengths, np.zeros(len(facts), dtype=np.int64)])
    R = heads.shape[0]
    ptr = np.zeros(R + 1, dtype=np.int64)
    np.cumsum(lengths, out=ptr[1:])
    body = np.empty(int(ptr[-1]), dtype=np.int32)
    for L in np.unique(lengths):
        L = int(L)
        if L == 0:
            continue
        idx = np.nonzero(lengths == L)[0]
        rows = fill(idx, L)
        pos = ptr[idx][:, None] + np.arange(L)[None, :]
        body[pos.reshape(-1)] = rows.reshape(-1)
    return Rules(n_atoms=int(n_atoms), head=heads, body_ptr=ptr, body_atom=body,
                 body_neg=None, meta=dict(meta or {}))


# ----------------------------------------------------------------------------------
# BASELINE.json configurations (SURVEY.md §8(d) readings)
# ----------------------------------------------------------------------------------

def gen_c1(seed: int = 1) -> Rules:
    """C1: n=1,000; 2,000 non-fact rules, head uniform, body length uniform {1..4},
    body atoms distinct, uniform, != head (no self-loop); plus 50 facts on 50 distinct
    uniform atoms; v0 = facts only."""
    rng = np.random.default_rng([seed, 1])
    n, R = 1000, 2000
    heads = rng.integers(0, n, size=R, dtype=np.int32)
    lengths = rng.integers(1, 5, size=R)
    facts = rng.choice(n, size=50, replace=False).astype(np.int32)
    fill = lambda idx, L: _distinct_rows(rng, idx.size, L, 0, n, forbid=heads[idx])
    return _assemble(n, heads, lengths, fill, rng, facts, meta={"config": "C1", "seed": seed})


def gen_c2(seed: int = 1) -> Rules:
    """C2: n=100,000; 500,000 rules, head uniform, body length uniform {1..8}, body
    atoms distinct uniform (cycles allowed); 1% of atoms (1,000 distinct) are facts."""
    rng = np.random.default_rng([seed, 2])
    n, R = 100_000, 500_000
    heads = rng.integers(0, n, size=R, dtype=np.int32)
    lengths = rng.integers(1, 9, size=R)
    facts = rng.choice(n, size=n // 100, replace=False).astype(np.int32)
    fill = lambda idx, L: _distinct_rows(rng, idx.size, L, 0, n)
    return _assemble(n, heads, lengths, fill, rng, facts, meta={"config": "C2", "seed": seed})


def layered(layers: int, width: int, n_rules: int, max_len: int, seed: int = 1,
            tag: str = "layered") -> Rules:
    """Deep-recursion family (C3 shape).  Atom id = layer*width + j; layer 0 = facts.
    Each rule: i uniform in {0..layers-2}; head uniform in layer i+1; body length
    uniform {1..max_len}; body atom 1 uniform from layer i (reading R3);
    the rest distinct, uniform from layers 0..i."""
    assert width > max_len, "layered() needs width > max_len"
    rng = np.random.default_rng([seed, 3, layers, width])
    n = layers * width
    li = rng.integers(0, layers - 1, size=n_rules)
    heads = ((li + 1) * width + rng.integers(0, width, size=n_rules)).astype(np.int32)
    lengths = rng.integers(1, max_len + 1, size=n_rules)
    facts = np.arange(width, dtype=np.int32)

    def fill(idx, L):
        i = li[idx]
        first = (i * width + rng.integers(0, width, size=idx.size)).astype(np.int32)
        if L == 1:
            return first[:, None]
        hi = (i + 1) * width
        rest = _distinct_rows(rng, idx.size, L - 1, 0, hi, forbid=None)
        # redraw rows where the rest collides with the first atom
        while True:
            bad = (rest == first[:, None]).any(axis=1)
            if not bad.any():
                break
            rest[bad] = _distinct_rows(rng, int(bad.sum()), L - 1, 0, hi[bad])
        return np.concatenate([first[:, None], rest], axis=1)

    return _assemble(n, heads, lengths, fill, rng, facts,
                     meta={"config": tag, "seed": seed, "layers": layers, "width": width})


def gen_c3(seed: int = 1) -> Rules:
    """C3: 1,000 layers x 1,000 atoms, 4,000,000 rules, body length uniform {1..3}."""
    return layered(1000, 1000, 4_000_000, 3, seed=seed, tag="C3")


def _zipf_heads(rng, n: int, R: int, s: float) -> np.ndarray:
    """head = pi(rank), P(rank r) ∝ r^-s over r = 1..n, pi a seeded permutation."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    u = np.sort(rng.random(R) * cdf[-1])
    rank_idx = np.searchsorted(cdf, u, side="right")
    np.minimum(rank_idx, n - 1, out=rank_idx)
    rank_idx = rank_idx[rng.permutation(R)]
    perm = rng.permutation(n).astype(np.int32)
    return perm[rank_idx]


def gen_c4(seed: int = 1, n: int = 10_000_000, R: int = 50_000_000) -> Rules:
    """C4: n=10M atoms; 50M rules, head in-degree Zipf(s=1.1) (head = pi(rank)),
    body length uniform {1..5}, body atoms distinct uniform; 0.1% facts (10,000)."""
    rng = np.random.default_rng([seed, 4])
    heads = _zipf_heads(rng, n, R, 1.1)
    lengths = rng.integers(1, 6, size=R).astype(np.int8)
    facts = rng.choice(n, size=n // 1000, replace=False).astype(np.int32)
    fill = lambda idx, L: _distinct_rows(rng, idx.size, L, 0, n)
    return _assemble(n, heads, lengths, fill, rng, facts,
                     meta={"config": "C4" if (n, R) == (10_000_000, 50_000_000) else "C4-scaled",
                           "seed": seed})


def gen_c5(seed: int = 1, n: int = 100_000, R: int = 500_000, k: int = 12,
           occ: int = 20) -> Rules:
    """C5: normal program, n=100,000; 500,000 rules, head uniform, body length uniform
    {1..6}, atoms distinct uniform; 1% facts (1,000).  k=12 negated atoms, distinct,
    uniform among non-facts; for each, exactly ``occ``=20 distinct non-fact rules not
    containing it (body or head) get one uniformly chosen positive literal replaced by
    ``not a`` (a rule with no positive literal left is redrawn)."""
    rng = np.random.default_rng([seed, 5])
    heads = rng.integers(0, n, size=R, dtype=np.int32)
    lengths = rng.integers(1, 7, size=R)
    facts = rng.choice(n, size=n // 100, replace=False).astype(np.int32)
    fill = lambda idx, L: _distinct_rows(rng, idx.size, L, 0, n)
    base = _assemble(n, heads, lengths, fill, rng, facts, meta={"config": "C5", "seed": seed})
    neg = np.zeros(base.nnz, dtype=np.uint8)
    is_fact = np.zeros(n, dtype=bool)
    is_fact[facts] = True
    negated = rng.choice(np.nonzero(~is_fact)[0], size=k, replace=False).astype(np.int32)
    ptr, body = base.body_ptr, base.body_atom
    for a in negated:
        chosen = set()
        while len(chosen) < occ:
            r = int(rng.integers(0, R))  # non-fact rules are 0..R-1
            if r in chosen or int(base.head[r]) == int(a):
                continue
            s, e = int(ptr[r]), int(ptr[r + 1])
            if (body[s:e] == a).any():
                continue
            pos = np.nonzero(neg[s:e] == 0)[0]
            if pos.size == 0:
                continue
            j = s + int(pos[int(rng.integers(0, pos.size))])
            body[j] = a
            neg[j] = 1
            chosen.add(r)
    base.body_neg = neg
    base.meta.update({"negated_atoms": sorted(int(x) for x in negated), "k": k})
    return base


CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")


def config(name: str, seed: int = 1) -> Rules:
    return {"C1": gen_c1, "C2": gen_c2, "C3": gen_c3, "C4": gen_c4, "C5": gen_c5}[name](seed)


# ----------------------------------------------------------------------------------
# small families for tests
# ----------------------------------------------------------------------------------

def random_program(rng, n: int, R: int, max_len: int = 4, n_facts: int = None,
                   neg_prob: float = 0.0, min_len: int = 1) -> Rules:
    """Small random program (definite unless neg_prob > 0).  Heads uniform, body
    length uniform {min_len..max_len} capped at n, atoms distinct uniform; each body
    literal negated with probability neg_prob."""
    if n_facts is None:
        n_facts = int(rng.integers(0, max(1, n // 3) + 1))
    rules = []
    for _ in range(R):
        h = int(rng.integers(0, n))
        L = int(rng.integers(min_len, min(max_len, n) + 1)) if n > 0 else 0
        atoms = rng.choice(n, size=L, replace=False).tolist() if L else []
        pos = [a for a in atoms if rng.random() >= neg_prob]
        negs = [a for a in atoms if a not in pos]
        rules.append((h, pos, negs))
    for a in (rng.choice(n, size=min(n_facts, n), replace=False).tolist() if n else []):
        rules.append((int(a), [], []))
    return from_lists(n, rules)


def random_normal_program(rng, n: int, R: int, max_len: int = 3, k_max: int = 4,
                          n_facts: int = None) -> Rules:
    """Small normal program whose negative literals range over at most k_max distinct
    atoms (so the guess space 2^k stays small)."""
    if n_facts is None:
        n_facts = int(rng.integers(0, max(1, n // 3) + 1))
    k = int(rng.integers(0, min(k_max, n) + 1))
    negatable = rng.choice(n, size=k, replace=False).tolist() if k else []
    rules = []
    for _ in range(R):
        h = int(rng.integers(0, n))
        L = int(rng.integers(0, min(max_len, n) + 1))
        atoms = rng.choice(n, size=L, replace=False).tolist() if L else []
        pos, negs = [], []
        for a in atoms:
            (negs if (a in negatable and rng.random() < 0.6) else pos).append(a)
        rules.append((h, pos, negs))
    for a in (rng.choice(n, size=min(n_facts, n), replace=False).tolist() if n else []):
        rules.append((int(a), [], []))
    return from_lists(n, rules)


def chain(L: int) -> Rules:
    """a0 <- ;  a_{i+1} <- a_i   (i = 0..L-2)."""
    rules = [(0, [])] + [(i + 1, [i]) for i in range(L - 1)]
    return from_lists(L, rules, meta={"family": "chain", "L": L})


def random_digraph(rng, V: int, E: int, self_loops: bool = False):
    """E distinct directed edges over V nodes (as a sorted list of (u, v))."""
    E = min(E, V * V if self_loops else V * (V - 1))
    edges = set()
    while len(edges) < E:
        u, v = int(rng.integers(0, V)), int(rng.integers(0, V))
        if u == v and not self_loops:
            continue
        edges.add((u, v))
    return sorted(edges)


def tc_program(V: int, edges) -> Rules:
    """Transitive-closure grounding (relevance grounding as in SPEC
    S:150-164): atoms edge(u,v) for each edge (facts) then path(x,y) for all x,y
    (id = E + x*V + y); rules path(u,v) <- edge(u,v) for each edge and
    path(x,y) <- edge(x,z) ∧ path(z,y) for each edge (x,z) and each node y."""
    edges = list(edges)
    E = len(edges)
    eid = {e: i for i, e in enumerate(edges)}
    pid = lambda x, y: E + x * V + y
    rules = [(eid[e], []) for e in edges]
    rules += [(pid(u, v), [eid[(u, v)]]) for (u, v) in edges]
    for (x, z) in edges:
        for y in range(V):
            body = [eid[(x, z)], pid(z, y)]
            rules.append((pid(x, y), body))
    return from_lists(E + V * V, rules, meta={"family": "tc", "V": V, "E": E})


# ----------------------------------------------------------------------------------
# The paper's own workload shapes (Tables 1-6) -- synthetic stand-ins
# ----------------------------------------------------------------------------------

# (n, m) of Tables 2, 3, 5 and 6: the same twelve shapes in each
PAPER_TABLES = [(1000, 5000), (1000, 10000), (1600, 24000), (1600, 30000), (2000, 36000),
                (2000, 40000), (10000, 120000), (10000, 160000), (16000, 200000),
                (16000, 220000), (20000, 280000), (20000, 320000)]

# Table 4: KONECT graphs (|V|, |E|); the graphs themselves are not in
# the container -- seeded random digraphs of the same sizes stand in for them
PAPER_TC_GRAPHS = [("club membership", 65, 95), ("cattle", 28, 217), ("windsurfers", 43, 336),
                   ("contiguous usa", 49, 107), ("dolphins", 62, 159), ("train bombing", 64, 243),
                   ("highschool", 70, 366), ("les miserables", 77, 254)]

# Table 1: share of the non-fact rules by body length 1..8
_TABLE1 = [0.04, 0.04, 0.10, 0.40, 0.35, 0.04, 0.02, 0.01]


def paper_profile(n: int, m: int, seed: int = 1, dense: bool = False, k_neg: int = 0) -> Rules:
    """A random program of the paper's generator shape (reading in
    DESIGN.md "Input recipe"): m rules over n atoms; n//4 facts on distinct atoms (Table
    1: "< n/3"), the other m - n//4 rules with body lengths 1..8 in Table 1's
    proportions, heads uniform, body atoms distinct uniform.  dense=True keeps the facts
    and the length-1/2 shares and gives the other rules bodies of about 5% of n (uniform
    in [0.04 n, 0.06 n]; "sparsity ≈ 0.95").  k_neg > 0 turns k_neg body literal
    occurrences, chosen uniformly, into negations ("randomly changing k (4 <= k <= 8)
    literals to negations")."""
    rng = np.random.default_rng([seed, n, m, int(dense), k_neg, 2009])
    nf = n // 4
    R = m - nf
    shares = np.asarray(_TABLE1)
    counts = np.floor(shares * R).astype(np.int64)
    counts[3] += R - counts.sum()                      # remainder to the largest bucket
    lengths = np.repeat(np.arange(1, 9), counts)
    if dense:
        lo, hi = max(3, int(0.04 * n)), max(4, int(0.06 * n))
        big = lengths >= 3
        lengths[big] = rng.integers(lo, hi + 1, size=int(big.sum()))
    lengths = np.minimum(lengths, n)
    rng.shuffle(lengths)
    heads = rng.integers(0, n, size=R)
    facts = rng.choice(n, size=nf, replace=False)
    def fill(idx, L):
        if L * L > n:   # long bodies (dense profile): whole-row rejection would not end
            return _distinct_rows_long(rng, idx.size, L, n)
        return _distinct_rows(rng, idx.size, L, 0, n)
    P = _assemble(n, heads, lengths, fill, rng,
                  facts=facts, meta={"family": "paper", "n": n, "m": m, "dense": dense, "k_neg": k_neg})
    if k_neg:
        neg = np.zeros(P.body_atom.shape[0], dtype=np.uint8)
        neg[rng.choice(P.body_atom.shape[0], size=min(k_neg, P.body_atom.shape[0]), replace=False)] = 1
        P.body_neg = neg
    return P


def paper_tc(name: str, seed: int = 1) -> Rules:
    """Table 4 stand-in: the transitive-closure grounding (tc_program) of a seeded random
    digraph with the named KONECT graph's |V| and |E|."""
    for nm, V, E in PAPER_TC_GRAPHS:
        if nm == name:
            rng = np.random.default_rng([seed, V, E, 4])
            P = tc_program(V, random_digraph(rng, V, E))
            P.meta.update(graph=name)
            return P
    raise KeyError(name)
