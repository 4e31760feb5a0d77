"""Oracle pins against closed forms: chains, layered (deep-recursion) programs,
transitive closure vs BFS reachability, and degenerate programs."""
from collections import deque

import numpy as np
import pytest

import lpgen
import oracle


@pytest.mark.parametrize("L", [1, 2, 3, 10, 257, 2000])
def test_chain(L):
    """a0 <- ; a_{i+1} <- a_i: I_k = {a_0..a_k}, k* = L-1, iters = L, popcounts 1..L."""
    P = lpgen.chain(L)
    model, iters, pops, conv = oracle.lm_jacobi(P)
    assert model.all() and iters == L and pops == list(range(1, L + 1))
    _, stage, it2 = oracle.lm_stage(P)
    assert stage.tolist() == list(range(L)) and it2 == L


def test_layered_stage_equals_layer():
    """Reading R3 (body atom 1 from layer i, the rest from layers <= i, head in layer
    i+1): by induction every derived atom of layer j has stage exactly j, so the pass
    count is the number of layers when the last layer is reached."""
    layers, width = 60, 25
    P = lpgen.layered(layers, width, 6000, 3, seed=3)
    model, stage, iters = oracle.lm_stage(P)
    on = np.nonzero(model)[0]
    assert (stage[on] == on // width).all()
    assert model[:width].all()
    assert (model[(layers - 1) * width:]).any()
    assert iters == layers
    m2, it2, pops, _ = oracle.lm_jacobi(P)
    assert (m2 == model).all() and it2 == iters
    assert oracle.certify(P, None, model, stage, iters) == 0


def _reach(V, edges):
    adj = [[] for _ in range(V)]
    for u, v in edges:
        adj[u].append(v)
    R = set()
    for s in range(V):
        seen = set()
        dq = deque(adj[s])
        while dq:
            x = dq.popleft()
            if x in seen:
                continue
            seen.add(x)
            dq.extend(adj[x])
        R |= {(s, y) for y in seen}
    return R


@pytest.mark.parametrize("seed", range(20))
def test_transitive_closure_vs_bfs(seed):
    """path(x,y) ∈ LM iff y is reachable from x by >= 1 edge (PAPER.md:419 rules)."""
    rng = np.random.default_rng([seed, 11])
    V = int(rng.integers(2, 30))
    E = int(rng.integers(1, 3 * V))
    edges = lpgen.random_digraph(rng, V, E, self_loops=bool(seed % 3 == 0))
    P = lpgen.tc_program(V, edges)
    model, stage, iters = oracle.lm_stage(P)
    E_ = len(edges)
    got = {(i // V, i % V) for i in range(V * V) if model[E_ + i]}
    assert got == _reach(V, edges)
    assert model[:E_].all()


def test_transitive_closure_chain_closed_form():
    """Chain graph 0->1->...->V-1: V(V-1)/2 path atoms, path(x,y) has stage y-x,
    so k* = V-1 and iters = V."""
    V = 40
    edges = [(i, i + 1) for i in range(V - 1)]
    P = lpgen.tc_program(V, edges)
    model, stage, iters = oracle.lm_stage(P)
    E = len(edges)
    assert int(model[E:].sum()) == V * (V - 1) // 2
    for x in range(V):
        for y in range(V):
            s = stage[E + x * V + y]
            assert s == (y - x if y > x else -1)
    assert iters == V
    _, it2, _, _ = oracle.lm_jacobi(P)
    assert it2 == V


def test_degenerate_programs():
    empty = lpgen.from_lists(0, [])
    m, it, pops, conv = oracle.lm_jacobi(empty)
    assert m.size == 0 and it == 1 and pops == [0]
    norules = lpgen.from_lists(5, [])
    m, it, pops, _ = oracle.lm_jacobi(norules)
    assert not m.any() and it == 1 and pops == [0]
    facts = lpgen.from_lists(4, [(1, []), (3, []), (3, [])])
    m, it, pops, _ = oracle.lm_jacobi(facts)
    assert m.tolist() == [0, 1, 0, 1] and it == 1 and pops == [2]
    selfloop = lpgen.from_lists(2, [(0, [0]), (1, [0])])
    m, it, _, _ = oracle.lm_jacobi(selfloop)
    assert not m.any() and it == 1
    # {p <-, p <- q}: LM = {p}; duplicate body atoms are harmless
    P = lpgen.from_lists(2, [(0, []), (0, [1]), (1, [0, 0])])
    m, it, pops, _ = oracle.lm_jacobi(P)
    assert m.tolist() == [1, 1] and it == 2 and pops == [1, 2]
    m2, st, it2 = oracle.lm_stage(P)
    assert (m2 == m).all() and it2 == 2 and st.tolist() == [0, 1]
    # a definite program through the stable path: its least model is the only model
    o = oracle.stable(P, want_models=True)
    assert o["k"] == 0 and o["accepted"].tolist() == [1] and int(o["models"][0, 0]) == 0b11


def test_bounded_jacobi_sample():
    """max_iters bounds the number of T_P evaluations (bench.py's CPU sample)."""
    P = lpgen.chain(50)
    m, it, pops, conv = oracle.lm_jacobi(P, max_iters=7)
    assert not conv and it == 7 and int(m.sum()) == 8 and pops == list(range(1, 9))
