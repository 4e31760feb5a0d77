"""The paper's own matrix layout and algorithms, literally -- TEST INFRASTRUCTURE ONLY.

Pure Python, exact rational arithmetic (``fractions.Fraction``), small programs only.
Every function cites the PAPER.md lines (LaTeX source of arXiv 2009.10247) it
follows.  The B200 product uses a different (integer-threshold, bit-packed) layout;
this module exists to pin the oracle to the paper's printed examples and to check
that the convention-(B) oracle in lp_oracle.c computes the same models as the
paper's Algorithms 1-3.

Programs are given as lpgen.Rules (or anything with .rule(r), .n_rules, .n_atoms).
Atom order of the standardized program: originals 0..n-1, then abar atoms (normal
programs), then auxiliary atoms (reading R12).
"""
from __future__ import annotations

from fractions import Fraction

AND, OR = "AND", "OR"


def _dedupe(seq):
    out, seen = [], set()
    for x in seq:
        if x not in seen:
            seen.add(x)
            out.append(x)
    return out


def standardize(rules, n_base=None):
    """P^δ: for every head h with k >= 2 rules, replace them by
    h <- x1 ∨ ... ∨ xk and xi <- body(ri), with fresh atoms x_i; heads with one rule
    pass through.  A fact among several rules becomes an auxiliary fact xi <- (SPEC
    S:216, reading R10).  Body atoms are de-duplicated (footnote PAPER.md:54).
    Input rules must be definite (pos bodies only).  ``n_base``: atoms already in use
    (originals + abar) -- auxiliaries are numbered from there.
    Returns (m, std_rules) with std_rules a list of (kind, head, body_list)."""
    n = rules.n_atoms if n_base is None else n_base
    by_head = {}
    order = []
    for r in range(rules.n_rules):
        h, pos, neg = rules.rule(r)
        assert not neg, "standardize() takes a definite program (use positive_form first)"
        if h not in by_head:
            by_head[h] = []
            order.append(h)
        by_head[h].append(_dedupe(pos))
    out = []
    nxt = n
    for h in sorted(order):
        bodies = by_head[h]
        if len(bodies) == 1:
            out.append((AND, h, bodies[0]))
            continue
        aux = list(range(nxt, nxt + len(bodies)))
        nxt += len(bodies)
        out.append((OR, h, aux))
        for x, b in zip(aux, bodies):
            out.append((AND, x, b))
    return nxt, out


def program_matrix(m, std_rules):
    """M_P ∈ R^{m×m} (Def. 2), exact:
       a_{i j_k} = 1/m  for AND-rule p_i <- p_{j_1} ∧ ... ∧ p_{j_m}   (item 1)
       a_{i j_k} = 1    for OR-rule  p_i <- p_{j_1} ∨ ... ∨ p_{j_l}   (item 2)
       a_{ii}    = 1    for a fact   p_i <-                           (item 3)
       0 otherwise                                                    (item 4)."""
    M = [[Fraction(0)] * m for _ in range(m)]
    for kind, h, body in std_rules:
        if kind == OR:
            for j in body:
                M[h][j] = Fraction(1)
        elif len(body) == 0:
            M[h][h] = Fraction(1)
        else:
            for j in body:
                M[h][j] = Fraction(1, len(body))
    return M


def initial_vector(m, std_rules):
    """v0 (Def. 4): 1 exactly at atoms with a fact rule."""
    v = [0] * m
    for kind, h, body in std_rules:
        if kind == AND and len(body) == 0:
            v[h] = 1
    return v


def theta(x):
    """θ (Def. 5): 1 if x >= 1 else 0, elementwise on lists."""
    if isinstance(x, list):
        return [theta(e) for e in x]
    return 1 if x >= 1 else 0


def matvec(M, v):
    return [sum((M[i][j] * v[j] for j in range(len(v)) if M[i][j] != 0), Fraction(0))
            for i in range(len(M))]


def matmat(M, V):
    """M (m×m) times V (m×h), V as a list of columns."""
    return [matvec(M, col) for col in V]


def algorithm1(rules):
    """Algorithm 1, literally: standardize (line 1), matrix (line 2),
    initial vector (line 3), v = v0 (4), u = θ(Mv) (5), while u != v: v = u, u = θ(Mv)
    (6-9).  Returns dict(v, m, products, trace) where products counts the θ(Mv)
    evaluations (convention (A)) and trace holds |v| before each product."""
    m, std = standardize(rules)
    M = program_matrix(m, std)
    v = initial_vector(m, std)
    trace = [sum(v)]
    u = theta(matvec(M, v))
    products = 1
    while u != v:
        v = u
        trace.append(sum(v))
        u = theta(matvec(M, v))
        products += 1
    return dict(v=v, m=m, std=std, products=products, trace=trace)


def to_coo(M):
    """COO: row index, col index, value arrays, zero-based,
    row-major order of the nonzeros."""
    rows, cols, vals = [], [], []
    for i, row in enumerate(M):
        for j, x in enumerate(row):
            if x != 0:
                rows.append(i)
                cols.append(j)
                vals.append(x)
    return rows, cols, vals


def to_csr(M):
    """CSR: row_index (length rows+1; row_start_i = row_index[i],
    row_end_i = row_index[i+1]), col index and value arrays as in COO."""
    rows, cols, vals = to_coo(M)
    row_index = [0] * (len(M) + 1)
    for i in rows:
        row_index[i + 1] += 1
    for i in range(len(M)):
        row_index[i + 1] += row_index[i]
    return row_index, cols, vals


def sparsity_eq5(rules):
    """Eq. 5: 1 - Σ_r |body(r)| / n^2."""
    n = rules.n_atoms
    tot = sum(len(rules.rule(r)[1]) + len(rules.rule(r)[2]) for r in range(rules.n_rules))
    return 1.0 if n == 0 else 1.0 - tot / (n * n)


# --------------------------------------------------------------------------------
# normal programs
# --------------------------------------------------------------------------------

class _Plus:
    """A definite program over n + k atoms (positive form); duck-types lpgen.Rules."""

    def __init__(self, n_atoms, rules_list):
        self.n_atoms = n_atoms
        self._r = rules_list

    @property
    def n_rules(self):
        return len(self._r)

    def rule(self, r):
        h, pos = self._r[r]
        return h, list(pos), []


def negated_atoms(rules):
    s = set()
    for r in range(rules.n_rules):
        s.update(rules.rule(r)[2])
    return sorted(s)


def positive_form(rules):
    """P+ (Eq. 4): every negative literal ¬b is replaced by a fresh
    atom b̄.  b̄ atoms are numbered n + j for the j-th negated atom in ascending id.
    Returns (P+ as a definite program over n + k atoms, negated atom list)."""
    n = rules.n_atoms
    negs = negated_atoms(rules)
    bar = {a: n + j for j, a in enumerate(negs)}
    out = []
    for r in range(rules.n_rules):
        h, pos, neg = rules.rule(r)
        out.append((h, list(pos) + [bar[a] for a in neg]))
    return _Plus(n + len(negs), out), negs


def normal_matrix(rules):
    """Def. 7: M_P of P+ (standardized), with a_ii = 1 and zeros
    elsewhere on the b̄ rows (items 1-2); other rows per Def. 2 (item 3).
    Returns (M, m, std, negs, n)."""
    n = rules.n_atoms
    plus, negs = positive_form(rules)
    m, std = standardize(plus, n_base=plus.n_atoms)
    M = program_matrix(m, std)
    for j in range(len(negs)):
        i = n + j
        M[i] = [Fraction(0)] * m
        M[i][i] = Fraction(1)
    return M, m, std, negs, n


def initial_matrix(rules, m=None, std=None, negs=None):
    """M0 (Def. 8), as a list of h columns:
       item 2: original rows are 1 iff the atom has a fact in P;
       item 3: the b̄ row of a negated atom that is a fact is 0; the other b̄ rows take
               both values -- all 2^f combinations of the f free b̄ rows, column g has
               bit i of g as the value of the i-th free b̄ row (reading R9);
       auxiliary rows of the standardized program follow Def. 4 (1 iff aux fact)."""
    n = rules.n_atoms
    if m is None:
        _, m, std, negs, _ = normal_matrix(rules)
    facts = set()
    for r in range(rules.n_rules):
        h, pos, neg = rules.rule(r)
        if not pos and not neg:
            facts.add(h)
    base = [0] * m
    for kind, h, body in std:
        if kind == AND and len(body) == 0:
            base[h] = 1
    for a in facts:
        base[a] = 1
    free = [j for j, a in enumerate(negs) if a not in facts]
    cols = []
    for g in range(1 << len(free)):
        c = list(base)
        for j in range(len(negs)):
            c[n + j] = 0
        for i, j in enumerate(free):
            c[n + j] = (g >> i) & 1
        cols.append(c)
    return cols, free


def algorithm2_3(rules):
    """Algorithm 2 + Algorithm 3.
    Algorithm 2 literally: M = M0, U = θ(M_P M); while U != M: M = U, U = θ(M_P M).
    Algorithm 3 with reading R7: column i is accepted iff for every b̄ row j and the row
    l of its atom q_j, a_l + a_j = 1 (the printed break statements would drop every
    column after the first failure).
    Returns dict(accepted=[column ids], models=[frozenset of original atoms],
    products, free, negs)."""
    M_P, m, std, negs, n = normal_matrix(rules)
    cols, free = initial_matrix(rules, m, std, negs)
    Mk = cols
    U = [theta(c) for c in matmat(M_P, Mk)]
    products = 1
    while U != Mk:
        Mk = U
        U = [theta(c) for c in matmat(M_P, Mk)]
        products += 1
    accepted, models = [], []
    for i, v in enumerate(Mk):
        ok = all(v[a] + v[n + j] == 1 for j, a in enumerate(negs))
        if ok:
            accepted.append(i)
            models.append(frozenset(a for a in range(n) if v[a]))
    return dict(accepted=accepted, models=models, products=products, free=free, negs=negs,
                columns=Mk)
