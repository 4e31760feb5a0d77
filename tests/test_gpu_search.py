"""lp_stable_search (guess-space reduction, reading R23) on the
GPU against oracle/search.py: the same rounds, whole-matrix pass total, accepted columns,
last-round columns and accepted models, bit for bit, for the same seed -- including
programs with k = 24-40 negated atoms, where enumerating the 2^f guesses is refused
(LP_E_CAP)."""
import numpy as np
import pytest

import lpgen
import oracle
from oracle import search
from paper_2009_10247_b200 import lp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device (these tests run on the B200 box)")


def check_search(P, h, seed, max_rounds, prog=None):
    o = search.stable_search(P, h=h, seed=seed, max_rounds=max_rounds)
    prog = prog or lp.Program(P)
    g = prog.stable_search(h, seed, max_rounds)
    assert g["rounds"] == o["rounds"], (g["rounds"], o["rounds"])
    assert g["passes"] == o["passes"], (g["passes"], o["passes"])
    assert g["accepted"].tolist() == o["accepted"]
    assert (g["guesses"] == o["guesses"]).all()
    n = P.n_atoms
    words = (n + 63) // 64
    for c in o["accepted"][:8]:
        assert (prog.guess_model(int(c)) == o["models"][c, :words]).all()
    if o["rounds"] and words:   # the whole last-round fixpoint matrix, a few columns
        for c in {0, h - 1, h // 2}:
            assert (prog.guess_model(int(c)) == o["models"][c, :words]).all()
    return prog, o


def _small_normal(seed):
    rng = np.random.default_rng([seed, 1234])
    n = int(rng.integers(2, 11))
    R = int(rng.integers(1, 3 * n + 2))
    return lpgen.random_normal_program(rng, n, R, max_len=3, k_max=6)


@pytest.mark.parametrize("seed", range(40))
def test_small_programs(seed, stable_kernel):
    check_search(_small_normal(seed), h=8 + seed % 3 * 61, seed=seed, max_rounds=24)


def test_edges(stable_kernel):
    P = lpgen.from_lists(1, [(0, [], [0])])                 # no stable model
    prog, o = check_search(P, 64, 3, 5)
    assert not o["found"] and o["rounds"] == 5
    D = lpgen.from_lists(4, [(0, [1, 2]), (2, [3]), (3, [])])   # definite: k = 0
    prog, o = check_search(D, 65, 1, 3)
    assert o["rounds"] == 1 and len(o["accepted"]) == 65
    rules = [(2 * i, [], [2 * i + 1]) for i in range(20)] + [(2 * i + 1, [], [2 * i]) for i in range(20)]
    C = lpgen.from_lists(40, rules)                         # 20 choices, k = 40
    for h in (1, 63, 64, 200):
        check_search(C, h, 11, 40)
    # a negated fact: abar forced 0 in every column (Def. 8 item 3)
    F = lpgen.from_lists(3, [(0, [], [1]), (1, []), (2, [], [0])])
    prog, o = check_search(F, 70, 2, 4)
    j = o["negated"].index(1)
    assert not o["guesses"][:, j].any()


@pytest.mark.parametrize("k", [24, 32, 40])
def test_many_negations_where_enumeration_is_refused(k, stable_kernel):
    P = lpgen.gen_c5(seed=k, n=4000, R=20000, k=k)
    prog = lp.Program(P)
    with pytest.raises(lp.LPError) as e:
        prog.stable_models()
    assert e.value.status == lp.LP_E_CAP
    check_search(P, 256, 100 + k, 12, prog=prog)


def test_c5_size_k32(stable_kernel):
    """C5's recipe (100k atoms, 500k rules) with 32 negated atoms: 2^32 guesses cannot be
    enumerated; 128 sampled columns + local search find the stable model."""
    P = lpgen.gen_c5(seed=3, n=100_000, R=500_000, k=32)
    prog, o = check_search(P, 128, 5, 40)
    assert o["found"]


def test_device_pointer_mode(stable_kernel):
    import torch
    P = lpgen.gen_c5(seed=3, n=100_000, R=500_000, k=32)
    o = search.stable_search(P, h=128, seed=5, max_rounds=40)
    prog = lp.Program(P)
    k = prog.info["n_negated"]
    gs = torch.zeros((k, 2), dtype=torch.int64, device="cuda")
    acc = torch.zeros(2, dtype=torch.int64, device="cuda")
    na = torch.zeros(1, dtype=torch.int64, device="cuda")
    rd = torch.zeros(1, dtype=torch.int32, device="cuda")
    ps = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    lp.lp_stable_search(prog, 128, 5, 40, gs, acc, stream=s, device_ptrs=True, n_accepted_out=na,
                        rounds_out=rd, passes_out=ps, status_out=st)
    s.synchronize()
    assert int(st.item()) == 0
    assert int(rd.item()) == o["rounds"] and int(ps.item()) == o["passes"]
    assert int(na.item()) == len(o["accepted"])
    bits = np.unpackbits(acc.cpu().numpy().view(np.uint8), bitorder="little")[:128]
    assert np.nonzero(bits)[0].tolist() == o["accepted"]
    g = gs.cpu().numpy().view(np.uint64)
    cols = np.stack([np.unpackbits(g[j].view(np.uint8), bitorder="little")[:128] for j in range(k)], 1)
    assert (cols == o["guesses"]).all()


def test_more_columns_than_ctas(stable_kernel):
    """6,000 columns per round = 188 half-words: the compact search kernel's CTAs each own
    several half-words through every round."""
    P = lpgen.gen_c5(seed=7, n=2000, R=8000, k=26, occ=6)
    check_search(P, 6000, 11, 5)
    check_search(P, 33, 11, 9)
