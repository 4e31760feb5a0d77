"""Parity of the CUDA path (through the C ABI) with the CPU oracle -- bit-exact models,
identical pass counts, popcount traces and stages, identical accepted guesses and
whole fixpoint matrices.  Every GPU output is also checked by the oracle's
certificate checker (O-CERT)."""
import numpy as np
import pytest

import lpgen
import oracle
from paper_2009_10247_b200 import lp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device (these tests run on the B200 box)")


@pytest.fixture(scope="module", autouse=True)
def _overlap_always():
    """Programs here are small, so by default their key-mode LEAD passes would never take
    the overlapped / pipelined path (LP_OVERLAP_MIN_MB, read by lp_load): force it, so
    every parity case covers it; test_default_overlap_threshold covers the default."""
    import os
    old = os.environ.get("LP_OVERLAP_MIN_MB")
    os.environ["LP_OVERLAP_MIN_MB"] = "0"
    yield
    if old is None:
        del os.environ["LP_OVERLAP_MIN_MB"]
    else:
        os.environ["LP_OVERLAP_MIN_MB"] = old


def _oracle_lm(P, v0=None):
    model, stage, iters = oracle.lm_stage(P, v0=v0)
    return oracle.pack_bits(model), stage, iters, oracle.popcounts_from_stage(stage, iters)


def check_lm(P, v0=None, prog=None, variants=(False, True), jacobi=False,
             schedules=("auto", "stream", "lead"), **kw):
    om, ostage, oit, opops = _oracle_lm(P, v0)
    if jacobi:
        jm, jit, jpops, conv = oracle.lm_jacobi(P, v0=v0)
        assert conv and jit == oit and jpops == opops and (oracle.pack_bits(jm) == om).all()
    prog = prog or lp.Program(P, **kw)
    runs = []
    for frontier in variants:
        if frontier:
            runs.append((frontier, "auto", True))
        else:   # every schedule of the full θ-pass (LEAD / STREAM passes) must agree,
                # LEAD passes pipelined (default) and not
            runs += [(False, s, True) for s in schedules]
            runs += [(False, s, False) for s in schedules if s != "stream"]
    for frontier, schedule, pipeline in runs:
        model, iters, ex = prog.least_model(v0, frontier=frontier, popcounts=True, stages=True,
                                            schedule=schedule, stats=True, pipeline=pipeline)
        tag = "frontier" if frontier else f"full/{schedule}" + ("" if pipeline else "/nopipe")
        st = ex["stats"]
        if frontier:
            assert st["bytes"] == 0
        else:
            assert 0 <= st["lead_passes"] <= iters, (tag, st)
            assert st["lead_passes"] == {"stream": 0, "lead": iters}.get(schedule, st["lead_passes"])
            # (key-mode LEAD passes stream only the live runs: at most the whole plane)
            assert st["bytes"] > 0 or prog.info["lead_pass_bytes"] == 0 or st["lead_passes"] == 0 \
                or st["rows_verified"] == 0   # (armed LEAD passes with nothing armed read nothing)
        assert iters == oit, (tag, iters, oit)
        assert (model == om).all(), tag
        assert ex["popcounts"] == opops, tag
        assert (ex["stage"] == ostage).all(), tag
        m8 = lp.unpack_bits(model, P.n_atoms)
        assert oracle.certify(P, v0, m8, ex["stage"], iters) == 0, tag
    return prog


# ---------------------------------------------------------------------------------
# least model: small programs, edge cases
# ---------------------------------------------------------------------------------

def test_example1_and_degenerate():
    P = lpgen.from_lists(5, [(0, [1, 2]), (0, [3, 4]), (2, [3]), (1, [4]), (3, []), (4, [])])
    check_lm(P, jacobi=True)
    for Q in [lpgen.from_lists(0, []), lpgen.from_lists(5, []),
              lpgen.from_lists(4, [(1, []), (3, []), (3, [])]),
              lpgen.from_lists(2, [(0, [0]), (1, [0])]),
              lpgen.from_lists(2, [(0, []), (0, [1]), (1, [0, 0])]),
              lpgen.from_lists(1, [(0, [])]), lpgen.from_lists(1, [(0, [0])])]:
        check_lm(Q, jacobi=True)


@pytest.mark.parametrize("L", [1, 2, 33, 64, 65, 1000, 4097])
def test_chain_gpu(L):
    check_lm(lpgen.chain(L), jacobi=True)


@pytest.mark.parametrize("seed", range(60))
def test_random_programs(seed):
    rng = np.random.default_rng([seed, 5150])
    n = int(rng.integers(1, 400))
    R = int(rng.integers(0, 5 * n))
    P = lpgen.random_program(rng, n, R, max_len=int(rng.integers(1, 13)))
    prog = check_lm(P, jacobi=True)
    v0 = rng.choice(n, size=int(rng.integers(0, n // 4 + 1)), replace=False).tolist()
    check_lm(P, v0=v0, prog=prog, jacobi=True)


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("cfg", [dict(smem_bits_cap=128), dict(smem_bits_cap=1024, grid_blocks=3),
                                 dict(grid_blocks=1), dict(smem_bits_cap=128, key8=True),
                                 dict(smem_bits_cap=1024, key8=True, grid_blocks=5)])
def test_forced_summary_mode_and_small_grids(seed, cfg):
    """FILTER mode (summary in shared memory, exact test in L2) and tiny grids."""
    rng = np.random.default_rng([seed, 99])
    n = int(rng.integers(1200, 3000))
    P = lpgen.random_program(rng, n, 4 * n, max_len=6, n_facts=n // 20)
    prog = check_lm(P, **cfg)
    if cfg.get("smem_bits_cap"):
        assert prog.info["truth_mode"] == 1 and prog.info["summary_shift"] >= 1
        assert prog.info["key_shift"] >= 0          # LEAD passes stream the key plane
    # a start set with atoms that are neither heads nor facts (coarse key groups)
    v0 = rng.choice(n, size=n // 8, replace=False).tolist()
    check_lm(P, v0=v0, prog=prog)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("cfg", [dict(smem_bits_cap=128), dict(smem_bits_cap=1024, grid_blocks=3)])
def test_default_overlap_threshold(seed, cfg, monkeypatch):
    """Key-mode LEAD passes with the default LP_OVERLAP_MIN_MB: small live streams take
    the plain pass (all warps stream, then all verify), as bench.py's main line does."""
    monkeypatch.delenv("LP_OVERLAP_MIN_MB")
    rng = np.random.default_rng([seed, 404])
    n = int(rng.integers(1500, 4000))
    P = lpgen.random_program(rng, n, 5 * n, max_len=5, n_facts=n // 25)
    prog = check_lm(P, **cfg)
    assert prog.info["key_shift"] >= 0
    v0 = rng.choice(n, size=n // 10, replace=False).tolist()
    check_lm(P, v0=v0, prog=prog)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("cfg", [dict(grid_blocks=2), dict(smem_bits_cap=128),
                                 dict(smem_bits_cap=128, grid_blocks=2)])
def test_long_rows_edge_grids(seed, cfg):
    """Bodies of up to 9 atoms (one segment past the unrolled lengths) on 2-CTA grids and
    in summary mode: many rows per thread, every schedule, same results as the oracle."""
    rng = np.random.default_rng([seed, 123])
    n = int(rng.integers(1200, 6000))
    P = lpgen.random_program(rng, n, 6 * n, max_len=9, n_facts=n // 30)
    check_lm(P, **cfg)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("cfg", [dict(), dict(smem_bits_cap=256)])
def test_auto_schedule_switches_mid_fixpoint(seed, cfg, monkeypatch):
    """The auto schedule switches from LEAD to STREAM passes once a pass queues more
    than n_slots / LP_DENSE_DIV rows; with a huge divisor the switch happens right after
    the first pass that queues anything, so the fixpoint mixes both pass kinds."""
    monkeypatch.setenv("LP_DENSE_DIV", str(10 ** 9))
    monkeypatch.setenv("LP_NO_PREDICT", "1")   # (no predicted STREAM start: switch mid-way)
    monkeypatch.setenv("LP_NO_CLUSTER", "1")   # (the persistent grid kernel's auto schedule)
    rng = np.random.default_rng([seed, 4242])
    n = int(rng.integers(2000, 5000))
    P = lpgen.random_program(rng, n, 5 * n, max_len=5, n_facts=n // 10)
    prog = lp.Program(P, **cfg)
    for pipeline in (True, False):   # (key space: the pipelined passes hand over too)
        _, iters, ex = prog.least_model(schedule="auto", stats=True, pipeline=pipeline)
        assert 1 <= ex["stats"]["lead_passes"] < iters
    check_lm(P, prog=prog, schedules=("auto",))
    # the predicted start: a start set lighting most key buckets begins with STREAM passes
    monkeypatch.delenv("LP_NO_PREDICT")
    monkeypatch.delenv("LP_NO_CLUSTER")
    monkeypatch.delenv("LP_DENSE_DIV")
    q = lp.Program(P, **cfg)
    v0 = rng.choice(n, size=n // 3, replace=False).tolist()
    check_lm(P, v0=v0, prog=q, schedules=("auto",))


@pytest.mark.parametrize("small", [True, False])
@pytest.mark.parametrize("seed", range(24))
def test_cluster_kernel(seed, small, monkeypatch):
    """Exact-mode programs on ONE thread-block cluster (lm_cluster_kernel): one or two CTAs,
    the planes staged in shared memory or read from L2, random start sets; and the same
    program forced onto the persistent grid (LP_NO_CLUSTER) for comparison.  small: programs
    whose rows fit shared memory in 16-bit ids run lm_small_kernel instead (one CTA,
    semi-naive row lists); LP_NO_SMALL keeps them on the cluster kernel."""
    if not small:
        monkeypatch.setenv("LP_NO_SMALL", "1")
    rng = np.random.default_rng([seed, 777])
    n = int(rng.integers(50, 8000))
    R = int(rng.integers(n, 8 * n))
    P = lpgen.random_program(rng, n, R, max_len=int(rng.integers(1, 9)), n_facts=max(1, n // 40))
    prog = lp.Program(P)
    assert prog.info["cluster_ctas"] >= 1, prog.info
    if not small:
        assert prog.info["small_rows"] == 0
    elif prog.info["nnz"] < 15000:   # (rows, body ids and their transpose well under 200 KB)
        assert prog.info["small_rows"] > 0, prog.info
    check_lm(P, prog=prog, schedules=("auto",), variants=(False,))
    v0 = rng.choice(n, size=max(1, n // 20), replace=False).tolist()
    check_lm(P, v0=v0, prog=prog, schedules=("auto",), variants=(False,))
    model, iters, ex = prog.least_model(max_passes=2, stats=True)
    assert iters == min(2, _oracle_lm(P)[2])
    monkeypatch.setenv("LP_NO_CLUSTER", "1")
    q = lp.Program(P, frontier=False)
    assert q.info["cluster_ctas"] == 0
    check_lm(P, prog=q, schedules=("auto",), variants=(False,))


def test_long_bodies_generic_path_and_u32_counters():
    rng = np.random.default_rng(7)
    n = 3000
    rules = [(int(rng.integers(0, n)), rng.choice(n, size=int(rng.integers(9, 40)), replace=False).tolist())
             for _ in range(2000)]
    rules += [(a, []) for a in rng.choice(n, size=1500, replace=False).tolist()]
    rules += [(1, list(range(2, 602)))]            # a 600-atom body: 32-bit counters
    rules += [(0, [1] + list(range(2, 300)))]
    P = lpgen.from_lists(n, rules)
    prog = check_lm(P, jacobi=True)
    assert prog.info["max_body"] == 600
    check_lm(P, jacobi=True, smem_bits_cap=256)


def test_ragged_sizes():
    """n and R that are not multiples of 4 / 32 / 64, bits at word edges."""
    for n in (31, 32, 33, 63, 64, 65, 127, 129):
        rules = [(i + 1, [i]) for i in range(n - 1)] + [(0, [])]
        rules += [(n - 1, [0, n // 2])]
        check_lm(lpgen.from_lists(n, rules), jacobi=True)
        check_lm(lpgen.from_lists(n, rules), v0=[n - 1], jacobi=True)


def test_layered_deep_recursion_small():
    P = lpgen.layered(300, 16, 300 * 16 * 4, 3, seed=4)
    prog = check_lm(P, jacobi=True)
    check_lm(P, variants=(False,), smem_bits_cap=128)


def test_transitive_closure_gpu():
    rng = np.random.default_rng(3)
    for V in (2, 17, 45):
        edges = lpgen.random_digraph(rng, V, 3 * V, self_loops=True)
        check_lm(lpgen.tc_program(V, edges), jacobi=True)


def test_semantic_error_on_normal_program():
    P = lpgen.from_lists(2, [(0, [], [1])])
    prog = lp.Program(P)
    with pytest.raises(lp.LPError) as e:
        prog.least_model()
    assert e.value.status == lp.LP_E_SEMANTIC


def test_device_pointer_mode_matches_host_mode():
    import torch
    rng = np.random.default_rng(11)
    P = lpgen.random_program(rng, 5000, 20000, max_len=5, n_facts=200)
    prog = lp.Program(P)
    om, ostage, oit, opops = _oracle_lm(P)
    s = torch.cuda.Stream()
    W = lp.bits_words(P.n_atoms)
    for frontier in (False, True):
        model = torch.zeros(W, dtype=torch.int64, device="cuda")
        iters = torch.zeros(1, dtype=torch.int32, device="cuda")
        pops = torch.zeros(P.n_atoms + 2, dtype=torch.int32, device="cuda")
        stage = torch.zeros(P.n_atoms, dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lp.lp_least_model(prog, None, model, frontier=frontier, pops=pops, stage=stage, stream=s,
                          device_ptrs=True, iters_out=iters, ev_begin=e0, ev_end=e1)
        s.synchronize()
        assert int(iters.item()) == oit
        assert (model.cpu().numpy().view(np.uint64) == om).all()
        assert pops.cpu().numpy()[:oit].tolist() == opops
        assert (stage.cpu().numpy() == ostage).all()
        assert e0.elapsed_time(e1) > 0


# ---------------------------------------------------------------------------------
# least model: BASELINE.json configurations C1-C4 at full size
# ---------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_config_parity(cfg):
    P = lpgen.config(cfg)
    prog = check_lm(P, jacobi=(cfg != "C3"))
    assert (prog.info["small_rows"] > 0) == (cfg == "C1")


def test_config_c1_cluster_kernel(monkeypatch):
    monkeypatch.setenv("LP_NO_SMALL", "1")
    prog = check_lm(lpgen.config("C1"), jacobi=True)
    assert prog.info["small_rows"] == 0 and prog.info["cluster_ctas"] == 1


# (full-size C4: tests/test_gpu_c4.py)


# ---------------------------------------------------------------------------------
# stable models
# ---------------------------------------------------------------------------------

def _oracle_matrix_bits(models, n, G):
    """oracle per-guess models [G][words] -> bool [G][n]"""
    return np.unpackbits(np.ascontiguousarray(models).view(np.uint8), axis=1, bitorder="little")[:, :n]


def check_stable(P, guesses_u8=None, prog=None, chunk=8192, **kw):
    """guesses_u8: None (all 2^f) or uint8[G][k] abar values."""
    o = oracle.stable(P, guesses=guesses_u8, want_models=True)
    prog = prog or lp.Program(P, **kw)
    k = o["k"]
    if guesses_u8 is None:
        ids, passes, acc = prog.stable_models()
        G = 1 << o["f"]
    else:
        g = np.asarray(guesses_u8, dtype=np.uint8).reshape(-1, k)
        G = g.shape[0]
        W = (G + 63) // 64
        sliced = np.zeros((max(k, 1), W), dtype=np.uint64)
        for j in range(k):
            sliced[j] = lp.pack_mask(g[:, j].astype(bool))[:W]
        ids, passes, acc = prog.stable_models(sliced[:k] if k else np.zeros((0, W), np.uint64), n_guesses=G)
    assert ids.tolist() == np.nonzero(o["accepted"])[0].tolist()
    assert passes == o["passes"]
    M = prog.stable_matrix()                       # [n][W], bit g = guess g
    n = P.n_atoms
    for a0 in range(0, n, chunk):
        a1 = min(n, a0 + chunk)
        dev = np.unpackbits(M[a0:a1].view(np.uint8), axis=1, bitorder="little")[:, :G]
        ora = np.unpackbits(np.ascontiguousarray(o["models"]).view(np.uint8), axis=1,
                            bitorder="little")[:, a0:a1]
        assert (dev == ora.T).all()
    for g in list(ids[:3]) + [0, G - 1]:
        gm = prog.guess_model(int(g))
        assert (gm == o["models"][g]).all()
    return prog, o


def test_stable_examples(stable_kernel):
    ex2 = lpgen.from_lists(6, [(0, [1, 2]), (1, [0, 3]), (2, [], [3]), (3, []), (4, [5])])
    check_stable(ex2)
    check_stable(ex2, guesses_u8=[[0], [1]])
    two = lpgen.from_lists(2, [(0, [], [1]), (1, [], [0])])
    _, o = check_stable(two)
    assert np.nonzero(o["accepted"])[0].tolist() == [1, 2]
    check_stable(lpgen.from_lists(1, [(0, [], [0])]))
    check_stable(lpgen.from_lists(3, [(0, [1]), (1, []), (2, [0, 1])]))       # definite, k = 0


@pytest.mark.parametrize("seed", range(60))
def test_random_normal_programs(seed, stable_kernel):
    rng = np.random.default_rng([seed, 4242])
    n = int(rng.integers(1, 200))
    P = lpgen.random_normal_program(rng, n, 3 * n, max_len=4, k_max=9)
    prog, o = check_stable(P)
    k = o["k"]
    if k:
        G = int(rng.integers(1, 200))
        g = rng.integers(0, 2, size=(G, k)).astype(np.uint8)
        check_stable(P, guesses_u8=g, prog=prog)


def test_stable_summary_filter_mode(monkeypatch):
    monkeypatch.setenv("LP_NO_COMPACT_STABLE", "1")   # (a mode of the batched kernel)
    rng = np.random.default_rng(8)
    P = lpgen.random_normal_program(rng, 3000, 9000, max_len=4, k_max=7, n_facts=100)
    check_stable(P, smem_bits_cap=256, grid_blocks=5)


def test_guess_cap():
    rules = [(i, [], [i + 1]) for i in range(0, 44, 2)]
    P = lpgen.from_lists(46, rules)
    prog = lp.Program(P, guess_cap=20)
    with pytest.raises(lp.LPError) as e:
        prog.stable_models()
    assert e.value.status == lp.LP_E_CAP


def test_config_c5_parity(stable_kernel):
    P = lpgen.config("C5")
    prog, o = check_stable(P)
    assert prog.info["n_negated"] == 12
    assert (prog.info["stable_compact_atoms"] > 0) == (stable_kernel == "compact")


@pytest.mark.parametrize("seed", range(6))
def test_guess_offset_slices(seed, stable_kernel):
    """lp_run.guess_offset: rank slices of the 2^f guesses, solved one after another on
    this GPU (no slice waits on another), concatenate to the whole search."""
    from paper_2009_10247_b200.shard import guess_slices
    rng = np.random.default_rng([seed, 31])
    P = lpgen.random_normal_program(rng, 300, 1200, max_len=4, k_max=9)
    o = oracle.stable(P, want_models=True)
    G = 1 << o["f"]
    prog = lp.Program(P)
    for world in (1, 2, 3, 8):
        got, passes = [], 0
        for off, cnt in guess_slices(G, world):
            if cnt == 0:
                continue
            ids, ps, _ = prog.stable_models(guess_offset=off, n_guesses=cnt)
            got += (ids + off).tolist()
            passes = max(passes, ps)
            g = int(ids[0]) if ids.size else cnt - 1          # a column of this slice
            assert (prog.guess_model(g) == o["models"][off + g]).all()
        assert got == np.nonzero(o["accepted"])[0].tolist()
        assert passes == o["passes"]
    if G > 64:
        with pytest.raises(lp.LPError):
            prog.stable_models(guess_offset=32, n_guesses=8)


def test_guess_offset_c5_slices(stable_kernel):
    P = lpgen.config("C5")
    o = oracle.stable(P)
    prog = lp.Program(P)
    from paper_2009_10247_b200.shard import guess_slices
    got, passes = [], 0
    for off, cnt in guess_slices(1 << o["f"], 8):
        ids, ps, _ = prog.stable_models(guess_offset=off, n_guesses=cnt)
        got += (ids + off).tolist()
        passes = max(passes, ps)
    assert got == np.nonzero(o["accepted"])[0].tolist() and passes == o["passes"]


# ---------------------------------------------------------------------------------
# convention (A): the paper's own matrix M_{P^δ} (LP_LOAD_PAPER_LAYOUT)
# ---------------------------------------------------------------------------------

def test_paper_layout_example1():
    """Example 1: Algorithm 1 literally takes 3 products with |v|
    trace 2, 5, 7 (convention (A)); the least model over B_P is {p,q,r,s,t}."""
    from oracle import paper
    P = lpgen.from_lists(5, [(0, [1, 2]), (0, [3, 4]), (2, [3]), (1, [4]), (3, []), (4, [])])
    prog = lp.Program(P, paper_layout=True)
    assert prog.info["n_aux"] == 2 and prog.info["n_atoms"] == 5
    for frontier in (False, True):
        model, iters, ex = prog.least_model(frontier=frontier, popcounts=True, stages=True)
        assert iters == 3 and ex["popcounts"] == [2, 5, 7]
        assert lp.unpack_bits(model, 5).tolist() == [1, 1, 1, 1, 1]
    assert paper.algorithm1(P)["products"] == 3


@pytest.mark.parametrize("seed", range(25))
def test_paper_layout_matches_algorithm1(seed):
    """Pass count and |v| trace of Algorithm 1 in exact rationals over M_{P^δ}
    (oracle/paper.py) equal the kernels' on the P^δ encoding, every variant."""
    from oracle import paper
    rng = np.random.default_rng([seed, 808])
    n = int(rng.integers(2, 40))
    P = lpgen.random_program(rng, n, int(rng.integers(0, 4 * n)), max_len=4)
    alg = paper.algorithm1(P)
    lm = [a for a in range(n) if alg["v"][a]]
    for cfg in (dict(), dict(smem_bits_cap=64)):
        prog = lp.Program(P, paper_layout=True, **cfg)
        for frontier in (False, True):
            for sched in (("auto", "stream", "lead") if not frontier else ("auto",)):
                model, iters, ex = prog.least_model(frontier=frontier, popcounts=True,
                                                    schedule=sched)
                assert iters == alg["products"], (frontier, sched)
                assert ex["popcounts"] == alg["trace"], (frontier, sched)
                assert np.nonzero(lp.unpack_bits(model, n))[0].tolist() == lm


@pytest.mark.parametrize("seed", range(12))
def test_paper_layout_matches_algorithm2_3(seed, stable_kernel):
    from oracle import paper
    rng = np.random.default_rng([seed, 909])
    P = lpgen.random_normal_program(rng, int(rng.integers(3, 14)), int(rng.integers(3, 30)),
                                    max_len=3, k_max=4)
    alg = paper.algorithm2_3(P)
    prog = lp.Program(P, paper_layout=True)
    ids, passes, _ = prog.stable_models()
    assert ids.tolist() == alg["accepted"]
    assert passes == alg["products"]
    M = prog.stable_matrix()
    n = P.n_atoms
    G = len(alg["columns"])
    dev = np.unpackbits(M.view(np.uint8), axis=1, bitorder="little")[:, :G]
    for g in range(G):
        assert dev[:, g].tolist() == [alg["columns"][g][a] for a in range(n)]


@pytest.mark.parametrize("which", ["T2", "T3", "T4", "T5", "T6"])
def test_paper_profile_shapes(which):
    """The paper's own workload shapes (first row of Tables 2-6; Table 4: 'cattle'),
    both conventions, against the oracle."""
    from oracle import paper  # noqa: F401  (pins of the (A) convention live in paper.py)
    if which == "T4":
        P = lpgen.paper_tc("cattle")
    else:
        P = lpgen.paper_profile(1000, 5000, dense=which in ("T3", "T6"),
                                k_neg={"T5": 8, "T6": 7}.get(which, 0))
    if P.is_definite():
        check_lm(P, schedules=("auto",))
        progA = lp.Program(P, paper_layout=True)
        om, _, _ = oracle.lm_stage(P)
        model, _, _ = progA.least_model()
        assert (model == oracle.pack_bits(om)).all()
    else:
        check_stable(P)
        o = oracle.stable(P)
        ids, _, _ = lp.Program(P, paper_layout=True).stable_models()
        assert ids.tolist() == np.nonzero(o["accepted"])[0].tolist()


@pytest.mark.parametrize("cfg", [dict(), dict(smem_bits_cap=256)])
def test_long_bodies_stream_first(cfg):
    """Bodies averaging > 32 atoms: the auto schedule starts with STREAM passes (in
    summary mode the atom-id summary of v_0 is built for them); LEAD-only must agree."""
    rng = np.random.default_rng(11)
    n = 2500
    rules = [(int(rng.integers(0, n)), rng.choice(n, size=int(rng.integers(34, 70)), replace=False).tolist())
             for _ in range(3000)]
    rules += [(int(rng.integers(0, n)), [int(rng.integers(0, n))]) for _ in range(300)]
    rules += [(a, []) for a in rng.choice(n, size=2000, replace=False).tolist()]
    P = lpgen.from_lists(n, rules)
    prog = check_lm(P, **cfg)
    _, iters, ex = prog.least_model(schedule="auto", stats=True)
    assert ex["stats"]["lead_passes"] == 0


def test_max_passes_cap():
    """lp_run.max_passes stops after that many θ-passes without an error: on a chain the
    model after p passes holds the first p + 1 atoms."""
    P = lpgen.chain(50)
    prog = lp.Program(P)
    for frontier in (False, True):
        for p_ in (1, 2, 7, 49, 50, 60):
            model, iters, ex = prog.least_model(frontier=frontier, max_passes=p_)
            assert iters == min(p_, 50)
            assert ex["converged"] == (p_ >= 50)
            bits = lp.unpack_bits(model, 50)
            assert bits.sum() == min(p_ + 1, 50)


@pytest.mark.parametrize("pipeline", [True, False])
def test_max_passes_cap_key_space(pipeline):
    """The cap in key-space LEAD passes (pipelined or not): the model after p passes of
    a chain holds the first p + 1 atoms, stages and the popcount trace up to the cap."""
    n = 3000
    P = lpgen.chain(n)
    prog = lp.Program(P, smem_bits_cap=128)
    assert prog.info["truth_mode"] == 1 and prog.info["key_shift"] >= 0
    for p_ in (1, 2, 3, 17, n - 1, n, n + 5):
        model, iters, ex = prog.least_model(max_passes=p_, schedule="lead", pipeline=pipeline,
                                            popcounts=True)
        assert iters == min(p_, n)
        assert ex["converged"] == (p_ >= n)
        assert lp.unpack_bits(model, n).sum() == min(p_ + 1, n)
        assert ex["popcounts"] == list(range(1, min(p_, n) + 1))


@pytest.mark.parametrize("seed", range(6))
def test_pipelined_lead_passes_hub_leads(seed):
    """Pipelined key-space LEAD passes on programs where a few atoms lead many rows
    (long lead-occurrence lists, many rows added per pass through them), with start
    sets, one CTA and several."""
    rng = np.random.default_rng([seed, 777])
    n = int(rng.integers(3000, 8000))
    m = 6 * n
    hubs = rng.choice(n, size=8, replace=False)
    head = rng.integers(0, n, size=m).astype(np.int32)
    lens = rng.integers(1, 5, size=m)
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    body = rng.integers(0, n, size=int(ptr[-1])).astype(np.int32)
    hub_rows = rng.random(m) < 0.3
    body[ptr[:-1][hub_rows]] = rng.choice(hubs, size=int(hub_rows.sum()))
    rows = [(int(head[r]), sorted(set(body[ptr[r]:ptr[r + 1]].tolist()) - {int(head[r])}))
            for r in range(m)]
    rows = [(h, b) for h, b in rows if b]
    facts = rng.choice(n, size=n // 25, replace=False)
    rows += [(int(a), []) for a in facts]
    P = lpgen.from_lists(n, rows)
    for cfg in (dict(smem_bits_cap=128), dict(smem_bits_cap=256, grid_blocks=2),
                dict(smem_bits_cap=128, key8=True, grid_blocks=7)):
        prog = check_lm(P, variants=(False,), **cfg)
        check_lm(P, v0=rng.choice(n, size=n // 10, replace=False).tolist(), prog=prog, variants=(False,))


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("cfg", ["rand", "C2", "tiny"])
def test_head_range_shards_device_exchange(world, cfg):
    """The head-range-sharded least model's device path (shard.py / lp_shard_combine), its
    ranks run one after another on this GPU with their payloads written straight into the
    rows of the gathered buffer (the all-gather's result): per pass every rank's one-θ-pass
    call (owned words + status word only, shards loaded with the whole program's D2), then
    the combine kernel (OR, changed flag, popcount).  Same model, pass count and popcounts
    as the oracle."""
    import torch
    from paper_2009_10247_b200.shard import derivable_mask, head_ranges, owned_words, sub_program
    if cfg == "rand":
        rng = np.random.default_rng(world)
        P = lpgen.random_program(rng, 3000, 12000, max_len=5, n_facts=100)
    elif cfg == "tiny":     # fewer words than ranks: empty trailing ranges
        rng = np.random.default_rng(world + 10)
        P = lpgen.random_program(rng, 70, 300, max_len=3, n_facts=7)
    else:
        P = lpgen.config("C2")
    om, stage, oit = oracle.lm_stage(P)
    n = P.n_atoms
    W = (n + 63) // 64
    der = derivable_mask(P)
    ranges = head_ranges(P, world)
    ow = owned_words(P, world)
    progs = [lp.Program(sub_program(P, lo, hi), derivable=der) for lo, hi in ranges]
    stride = max(c for _, c in ow) + 1
    gathered = torch.zeros(world * stride, dtype=torch.int64, device="cuda")
    ptr = np.asarray(P.body_ptr)
    start = np.zeros(W * 64, dtype=np.uint8)
    start[np.asarray(P.head)[ptr[1:] == ptr[:-1]]] = 1
    v = [torch.from_numpy(np.packbits(start, bitorder="little").view(np.int64).copy()).cuda(),
         torch.zeros(W, dtype=torch.int64, device="cuda")]
    it_d = torch.zeros(1, dtype=torch.int32, device="cuda")
    changed = torch.zeros(1, dtype=torch.int32, device="cuda")
    pops_d = torch.zeros(n + 3, dtype=torch.int32, device="cuda")
    k = 0
    while True:
        cur, nxt = v[k & 1], v[(k + 1) & 1]
        for r, prog in enumerate(progs):
            row = gathered[r * stride:(r + 1) * stride]
            status = row.view(torch.int32)[2 * (stride - 1):2 * (stride - 1) + 1]
            w0, cnt = ow[r]
            if cnt == 0:
                status.zero_()
                continue
            lp.lp_least_model(prog, cur, row, device_ptrs=True, iters_out=it_d, max_passes=1,
                              status_out=status, out_words=(w0, cnt))
        lp.lp_shard_combine(gathered, world, stride, [w for w, _ in ow], [c for _, c in ow], cur, nxt,
                            changed, pops_d[k + 1:k + 2])
        k += 1
        if int(changed.item()) == 0:
            break
        assert k <= n + 2
    assert k == oit
    assert (v[k & 1].cpu().numpy().view(np.uint64)[:W] == oracle.pack_bits(om)).all()
    assert [int(start.sum())] + pops_d[1:k].cpu().tolist() == oracle.popcounts_from_stage(stage, oit)


def test_edge_cases_new_controls():
    """Degenerate programs through every control added to lp_run / lp_load: empty and
    facts-only programs with the paper layout, pass caps with a start set, the last guess
    slice, one-rank shards."""
    from paper_2009_10247_b200.shard import guess_slices, head_ranges, sub_program
    for P in [lpgen.from_lists(0, []), lpgen.from_lists(3, []), lpgen.from_lists(3, [(1, []), (1, [])]),
              lpgen.from_lists(4, [(0, []), (0, [1]), (2, [0]), (2, [3])])]:
        om, _, oit = oracle.lm_stage(P)
        for kw in (dict(), dict(paper_layout=True)):
            prog = lp.Program(P, **kw)
            model, iters, ex = prog.least_model(popcounts=True)
            assert (model == oracle.pack_bits(om)[:len(model)]).all()
            if not kw:
                assert iters == oit
            m1, it1, ex1 = prog.least_model(max_passes=1, v0=[0] if P.n_atoms else None)
            assert it1 == 1
    # capped run from a start set = one T_P evaluation of P ∪ v0-as-facts
    rng = np.random.default_rng(9)
    P = lpgen.random_program(rng, 500, 2000, max_len=3, n_facts=10)
    v0 = rng.choice(500, size=40, replace=False).tolist()
    om, _, _, _ = oracle.lm_jacobi(P, v0=v0, max_iters=1)
    m, it, _ = lp.Program(P).least_model(v0=v0, max_passes=1)
    assert it == 1 and (m == oracle.pack_bits(om)).all()
    # the last, partial guess slice
    N = lpgen.random_normal_program(np.random.default_rng(3), 200, 800, max_len=3, k_max=8)
    o = oracle.stable(N)
    G = 1 << o["f"]
    prog = lp.Program(N)
    off, cnt = guess_slices(G, 3)[-1]
    if cnt:
        ids, _, _ = prog.stable_models(guess_offset=off, n_guesses=cnt)
        assert (ids + off).tolist() == [g for g in np.nonzero(o["accepted"])[0].tolist() if g >= off]
    # a single rank owns everything
    (lo, hi), = head_ranges(P, 1)
    assert (lo, hi) == (0, P.n_atoms) and sub_program(P, lo, hi).n_rules == P.n_rules


@pytest.mark.parametrize("seed", range(4))
def test_overlapped_lead_pass_queue_overflow(seed, monkeypatch):
    """Key-mode LEAD passes verify while they stream; with one CTA and a coarse summary
    far more than the 768 shared queue entries survive per pass, so the global part of
    the queue is used too (verified after the stream).  Overlap on and off agree."""
    rng = np.random.default_rng([seed, 606])
    P = lpgen.random_program(rng, 5000, 20000, max_len=4, n_facts=600)
    om, stage, oit = oracle.lm_stage(P)
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("LP_NO_OVERLAP", env)
        prog = lp.Program(P, smem_bits_cap=128, grid_blocks=1)
        assert prog.info["key_shift"] >= 0
        model, iters, ex = prog.least_model(schedule="lead", stats=True, stages=True)
        assert iters == oit and (model == oracle.pack_bits(om)).all()
        assert (ex["stage"] == stage).all()
        assert ex["stats"]["rows_verified"] > 768 * iters // 2


def test_exact16_planes_large_program():
    """Exact mode with >= 1 M rows streams 16-bit lead/head planes (rows bucketed by the
    high bits of lead and head); all schedules agree with the oracle."""
    P = lpgen.layered(200, 1000, 1_200_000, 3, seed=7)
    prog = check_lm(P)
    assert prog.info["truth_mode"] == 0
    assert prog.info["lead_pass_bytes"] < 5 * prog.info["n_rules"]


def test_repeated_stable_calls_reuse_the_matrix(stable_kernel):
    """Consecutive stable searches with the same matrix width clear only the rows the
    previous call changed; different guess sets, widths and offsets in any order must
    each give the oracle's accepted guesses and whole fixpoint matrix."""
    rng = np.random.default_rng(77)
    P = lpgen.random_normal_program(rng, 400, 1600, max_len=3, k_max=8)
    prog = lp.Program(P)
    k = len(oracle.negated_atoms(P))
    for trial in range(6):
        G = [130, 130, 64, 130, 200, 130][trial]
        g = (rng.random((G, k)) < 0.5).astype(np.uint8)
        check_stable(P, guesses_u8=g, prog=prog)
        if trial == 2:
            check_stable(P, prog=prog)                  # all 2^f guesses in between
        if trial == 3 and k:   # the search runs the batched kernel on the same matrix in between
            from oracle import search
            o = search.stable_search(P, h=70, seed=3, max_rounds=4)
            got = prog.stable_search(70, 3, 4)
            assert got["rounds"] == o["rounds"] and got["accepted"].tolist() == o["accepted"]
    if k:
        assert (prog.info["stable_compact_atoms"] > 0) == (stable_kernel == "compact")


@pytest.mark.parametrize("frontier", [False, True])
def test_pinned_host_model_out_written_by_the_kernel(frontier):
    """Host-pointer call with a page-locked model buffer: the epilogue writes it over PCIe
    (no staged copy); same model and iters as a pageable buffer and as the oracle, for the
    exact and the key-space truth."""
    import torch
    rng = np.random.default_rng(2024)
    n = 5000
    P = lpgen.random_program(rng, n, 20000, max_len=5, n_facts=250)
    om, _, oit = oracle.lm_stage(P)
    for kw in (dict(), dict(smem_bits_cap=128)):
        prog = lp.Program(P, **kw)
        W = lp.bits_words(n)
        pinned = torch.full((W,), -1, dtype=torch.int64).pin_memory()
        it = lp.lp_least_model(prog, None, pinned, frontier=frontier)
        assert it == oit
        assert (pinned.numpy().view(np.uint64)[:W] == oracle.pack_bits(om)).all()
        pageable = np.zeros(W, dtype=np.uint64)
        assert lp.lp_least_model(prog, None, pageable, frontier=frontier) == oit
        assert (pageable == oracle.pack_bits(om)).all()
        prog.close()


@pytest.mark.parametrize("seed", range(6))
def test_one_cluster_launches_of_grid_kernels(seed, monkeypatch):
    """The frontier and stable kernels launched as ONE 16-CTA cluster with cluster barriers
    (pass_barrier<true>; default for small frontier programs, A/B-only for the stable
    kernel): same results as the oracle."""
    monkeypatch.setenv("LP_CLUSTER_FR_SLOTS", str(1 << 30))
    monkeypatch.setenv("LP_CLUSTER_ST_SLOTS", str(1 << 30))
    monkeypatch.setenv("LP_NO_COMPACT_STABLE", "1")   # (a launch shape of the batched kernel)
    rng = np.random.default_rng([seed, 5150])
    n = int(rng.integers(500, 20000))
    P = lpgen.random_program(rng, n, 5 * n, max_len=5, n_facts=n // 20)
    prog = lp.Program(P)
    assert prog.info["frontier_cluster_ctas"] >= 1
    check_lm(P, prog=prog, variants=(True,))
    N = lpgen.random_normal_program(rng, 80, 300, max_len=3, k_max=7)
    sp = lp.Program(N)
    assert sp.info["stable_cluster_ctas"] >= 1
    check_stable(N, prog=sp)
    from oracle import search
    S = lpgen.gen_c5(seed=seed, n=3000, R=15000, k=24)
    o = search.stable_search(S, h=128, seed=seed, max_rounds=6)
    g = lp.Program(S).stable_search(128, seed, 6)
    assert g["rounds"] == o["rounds"] and g["passes"] == o["passes"] and g["accepted"].tolist() == o["accepted"]


@pytest.mark.parametrize("seed", range(6))
def test_frontier_counters_across_calls(seed):
    """Back-to-back frontier calls on one program reuse its row counters, queues and list
    (re-initialised by every call's prologue): small and large models, random start sets,
    a capped call in between -- all equal the oracle."""
    rng = np.random.default_rng([seed, 6060])
    n = int(rng.integers(2000, 30000))
    P = lpgen.random_program(rng, n, 4 * n, max_len=5, n_facts=max(1, n // 200))
    prog = lp.Program(P)
    starts = [None, rng.choice(n, size=n // 3, replace=False).tolist(), None,
              rng.choice(n, size=5, replace=False).tolist(), None]
    for i, v0 in enumerate(starts):
        om, ostage, oit, opops = _oracle_lm(P, v0)
        if i == 2:   # a capped call in between (its counters are re-initialised next time)
            m, it, ex = prog.least_model(v0, frontier=True, max_passes=max(1, oit // 2))
            assert it == max(1, min(oit, oit // 2))
        model, iters, ex = prog.least_model(v0, frontier=True, popcounts=True, stages=True)
        assert iters == oit and (model == om).all() and ex["popcounts"] == opops
        assert (ex["stage"] == ostage).all()


def _hub_chain(N, hubs=3, fan2=True):
    """a0 (fact) -> {x_1..x_N} -> b -> {y_1..y_N} -> c -> ...: every other level one hub
    atom's warp fires N rows in ONE CTA (its per-CTA frontier queue spills), and with fan2
    the level after a fan-out also claims N atoms spread over all CTAs (w_i <- x_i)."""
    rules, nxt = [(0, [])], 1
    hub = 0
    for _ in range(hubs):
        fan = list(range(nxt, nxt + N))
        nxt += N
        rules += [(a, [hub]) for a in fan]
        if fan2:
            rules += [(nxt + i, [a]) for i, a in enumerate(fan)]
            nxt += N
        rules.append((nxt, fan[:3]))   # the next hub needs three of the fan-out atoms
        hub = nxt
        nxt += 1
    return lpgen.from_lists(nxt, rules)


@pytest.mark.parametrize("N,fan2", [(1500, False), (60000, True), (300000, True)])
def test_frontier_spill_queues(N, fan2):
    """Levels at which one CTA (a hub atom's fan-out) or every CTA (the next level) claims
    more heads than its shared-memory frontier queue holds: the spill queue and the spill
    field of the level barrier word (set and cleared on the same word two levels apart)."""
    P = _hub_chain(N, hubs=3, fan2=fan2)
    prog = check_lm(P, variants=(True,))
    check_lm(P, variants=(True,), grid_blocks=7)
    # capped runs: the model after c passes (the full θ-pass is the reference of the cap,
    # pinned on chains by test_max_passes_cap) -- a spilled candidate of level c + 1 must
    # not leak into it
    oit = oracle.lm_stage(P)[2]
    for c in range(1, oit + 2):
        fm, fit, fex = prog.least_model(frontier=True, max_passes=c, popcounts=True)
        gm, git, gex = prog.least_model(frontier=False, max_passes=c, popcounts=True)
        assert fit == git == min(c, oit) and fex["converged"] == gex["converged"] == (c >= oit)
        assert (fm == gm).all() and fex["popcounts"] == gex["popcounts"], c


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("env", [dict(LP_NO_ARMED="1"), dict(LP_ARMED_ALWAYS="1", LP_ARM_CAP="32"),
                                 dict(LP_ARMED_ALWAYS="1")])
def test_armed_lead_passes(seed, env, monkeypatch):
    """Exact-mode LEAD passes with armed row lists (default), without them (the lead / head
    planes streamed every pass), and with lists so small that they overflow mid-fixpoint
    (the overflowing pass verifies the rest at once, later LEAD passes stream): all equal
    the oracle -- model, pass count, popcounts, stages -- on every schedule."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng([seed, 7117])
    n = int(rng.integers(200, 40000))
    P = lpgen.random_program(rng, n, int(rng.integers(1, 8)) * n, max_len=int(rng.integers(2, 10)),
                             n_facts=max(1, n // int(rng.integers(20, 400))))
    check_lm(P, variants=(False,), grid_blocks=int(rng.choice([0, 3, 37])))
    # summary mode (v_k in L2 while armed; an overflow switches to the atom-id summary)
    check_lm(P, variants=(False,), smem_bits_cap=128)
    check_lm(P, v0=rng.choice(n, size=n // 50 + 1, replace=False).tolist(), variants=(False,),
             smem_bits_cap=1024)
    L = lpgen.layered(120, 64, 120 * 64 * 3, 3, seed=seed)
    check_lm(L, variants=(False,))
    check_lm(L, variants=(False,), smem_bits_cap=256)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("armed", [False, True])
def test_pinned_model_split_writes(seed, armed, monkeypatch):
    """Page-locked host model buffer (bench.py's e2e path): the prologue writes v_0's words
    over PCIe and the epilogue only the words holding derived atoms.  A buffer full of
    garbage must come back as exactly the model -- with a start set (generic prologue),
    an output window, a pass cap, exact and summary mode, armed and unarmed LEAD passes."""
    import torch
    if armed:
        monkeypatch.setenv("LP_ARMED_ALWAYS", "1")
    else:
        monkeypatch.setenv("LP_NO_ARMED", "1")
    rng = np.random.default_rng([seed, 4242])
    n = int(rng.integers(300, 9000))
    P = lpgen.random_program(rng, n, 4 * n, max_len=5, n_facts=max(1, n // 40))
    W = lp.bits_words(n)
    for kw in (dict(grid_blocks=5), dict(smem_bits_cap=128)):
        prog = lp.Program(P, **kw)
        for v0l in (None, rng.choice(n, size=n // 30 + 1, replace=False).tolist()):
            om, _, oit = oracle.lm_stage(P, v0=v0l)
            v0 = None
            if v0l is not None:
                mask = np.zeros(n, dtype=bool)
                mask[v0l] = True
                v0 = lp.pack_mask(mask)
            want = oracle.pack_bits(om)
            pinned = torch.full((W,), -1, dtype=torch.int64).pin_memory()
            assert lp.lp_least_model(prog, v0, pinned) == oit
            assert (pinned.numpy().view(np.uint64)[:W] == want).all()
            lo, cnt = W // 3, max(1, W // 2)
            win = torch.full((cnt,), -1, dtype=torch.int64).pin_memory()
            assert lp.lp_least_model(prog, v0, win, out_words=(lo, cnt)) == oit
            assert (win.numpy().view(np.uint64) == want[lo:lo + cnt]).all()
            cap = max(1, oit // 2)
            capped = torch.full((W,), -1, dtype=torch.int64).pin_memory()
            ref = np.zeros(W, dtype=np.uint64)
            assert lp.lp_least_model(prog, v0, capped, max_passes=cap) == lp.lp_least_model(prog, v0, ref, max_passes=cap)
            assert (capped.numpy().view(np.uint64) == ref).all()
        prog.close()


def test_compact_kernel_more_half_words_than_ctas(stable_kernel):
    """2^14 guesses = 512 half-words of 32 columns: every CTA of the compact kernel runs
    several of them one after another (and the batched kernel 256 words per row)."""
    P = lpgen.gen_c5(seed=5, n=2000, R=8000, k=14, occ=6)
    prog, o = check_stable(P)
    assert o["f"] == 14
    assert (prog.info["stable_compact_atoms"] > 0) == (stable_kernel == "compact")
    k = o["k"]
    rng = np.random.default_rng(99)
    g = rng.integers(0, 2, size=(6000, k)).astype(np.uint8)   # 188 half-words, the last one ragged
    check_stable(P, guesses_u8=g, prog=prog)
    check_stable(P, guesses_u8=g[:33], prog=prog)             # one word, its second half 1 column


def test_c5_recipe_k16_sampled_columns(monkeypatch):
    """C5's recipe with 16 negated atoms: 65,536 guesses = 2,048 half-words, 14 per CTA of
    the compact kernel.  The oracle solves sampled columns one by one (model and accepted
    bit); accepted ids and pass count must also equal the batched kernel's."""
    P = lpgen.gen_c5(seed=1, n=100_000, R=500_000, k=16)
    prog = lp.Program(P)
    assert prog.info["stable_compact_atoms"] > 0 and prog.info["n_free_negated"] == 16
    ids, passes, _ = prog.stable_models()
    k = prog.info["n_negated"]
    rng = np.random.default_rng(16)
    sample = sorted(set(rng.integers(0, 1 << 16, size=40).tolist()) | {0, 65535} | set(ids.tolist()[:4]))
    g = np.array([[(c >> j) & 1 for j in range(k)] for c in sample], dtype=np.uint8)
    o = oracle.stable(P, guesses=g, want_models=True)
    for i, c in enumerate(sample):
        assert (prog.guess_model(int(c)) == o["models"][i]).all(), c
        assert bool(o["accepted"][i]) == (c in set(ids.tolist())), c
    assert passes >= int(o["passes"])
    monkeypatch.setenv("LP_NO_COMPACT_STABLE", "1")
    bprog = lp.Program(P)
    bids, bpasses, _ = bprog.stable_models()
    assert bids.tolist() == ids.tolist() and bpasses == passes
