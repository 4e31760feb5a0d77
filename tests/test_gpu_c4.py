"""Full-size C4 (BASELINE.json configs[3]: 10M atoms, 50M rules, ~150M nonzeros) through
every path bench.py times, bit-exact against the oracle (O-STAGE model, pass count,
popcount trace and stages) and certified by O-CERT:

  * v0 = NULL (the paper's initial vector, Def. 4): every schedule,
    pipelined and not, and the 8-bit key plane;
  * v0 = the facts passed explicitly (bench.py's e2e call: the generic prologue);
  * v0 = facts ∪ 1 % random atoms: atoms outside D2 light the coarse key buckets, so the
    live-run skip streams the whole plane and the auto schedule may switch to STREAM
    passes (Algorithm 1's u = θ(M v) over every row);
  * the LP_PTR_DEVICE call (the mode bench.py's main line times) with its device status
    word, and the frontier variant.
"""
import numpy as np
import pytest

import lpgen
import oracle
from paper_2009_10247_b200 import lp

from test_gpu_parity import _oracle_lm, check_lm

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device (these tests run on the B200 box)")
    P = lpgen.config("C4")
    prog = lp.Program(P)
    yield P, prog
    prog.close()


def _facts(P):
    return np.unique(P.head[np.diff(P.body_ptr) == 0])


def test_c4_v0_null_all_schedules(c4):
    P, prog = c4
    assert prog.info["truth_mode"] == 1     # the 10M-atom truth vector is L2-resident
    assert prog.info["key_shift"] >= 0
    check_lm(P, prog=prog)
    # the live-run skip: v0 = facts lights only the D2 buckets, so a LEAD pass streams a
    # small part of the key plane
    model, iters, ex = prog.least_model(stats=True, schedule="lead")
    full = prog.info["lead_pass_bytes"] * iters
    assert ex["stats"]["bytes"] < 0.2 * full, (ex["stats"], full)


def test_c4_v0_null_pipelined(c4, monkeypatch):
    """The pipelined key-space LEAD passes (taken by default only for live streams of at
    least LP_OVERLAP_MIN_MB) on C4 from the facts."""
    P, _ = c4
    monkeypatch.setenv("LP_OVERLAP_MIN_MB", "0")
    prog = lp.Program(P, frontier=False)
    try:
        check_lm(P, prog=prog, variants=(False,))
    finally:
        prog.close()


def test_c4_key8(c4):
    P, prog = c4
    om, ostage, oit, opops = _oracle_lm(P)
    p8 = lp.Program(P, key8=True, frontier=False)
    try:
        model, iters, ex = p8.least_model(stages=True, popcounts=True, stats=True)
        assert iters == oit and (model == om).all() and (ex["stage"] == ostage).all()
        assert ex["popcounts"] == opops
        assert p8.info["lead_pass_bytes"] < 0.7 * prog.info["lead_pass_bytes"]
    finally:
        p8.close()


def test_c4_explicit_facts_v0(c4):
    """The e2e call's start set: the facts as a bit vector (generic prologue)."""
    P, prog = c4
    check_lm(P, v0=_facts(P).tolist(), prog=prog)


def test_c4_random_one_percent_v0(c4):
    """v0 = facts ∪ 1 % uniformly random atoms (seeded): survivors outside D2, coarse
    key buckets live, the full key plane streamed, the auto schedule's switch."""
    P, prog = c4
    rng = np.random.default_rng(20251020)
    extra = rng.choice(P.n_atoms, size=P.n_atoms // 100, replace=False)
    v0 = np.union1d(_facts(P), extra).tolist()
    check_lm(P, v0=v0, prog=prog)
    model, iters, ex = prog.least_model(v0, stats=True, schedule="lead")
    if prog.info["armed_list_cap"] == 0:
        # every octet of the plane is live now (a coarse key of every segment is set)
        assert ex["stats"]["bytes"] >= 0.9 * prog.info["lead_pass_bytes"] * ex["stats"]["lead_passes"]
    else:   # armed LEAD passes: the rows led by the ~100 k extra atoms, verified every pass
        assert ex["stats"]["lead_passes"] == iters and ex["stats"]["rows_verified"] >= 100_000


def test_c4_device_pointer_mode_and_status(c4):
    """LP_PTR_DEVICE (bench.py's main line): model, iters and the kernel-written status
    word; max_passes gives LP_ST_CAPPED, never an overflow."""
    import torch
    P, prog = c4
    om, ostage, oit, opops = _oracle_lm(P)
    W = lp.bits_words(P.n_atoms)
    s = torch.cuda.Stream()
    for frontier in (False, True):
        model = torch.zeros(W, dtype=torch.int64, device="cuda")
        iters = torch.zeros(1, dtype=torch.int32, device="cuda")
        status = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        lp.lp_least_model(prog, None, model, frontier=frontier, stream=s, device_ptrs=True,
                          iters_out=iters, status_out=status)
        s.synchronize()
        assert int(status.item()) == 0
        assert int(iters.item()) == oit
        assert (model.cpu().numpy().view(np.uint64) == om).all()
        status.fill_(-1)
        lp.lp_least_model(prog, None, model, frontier=frontier, stream=s, device_ptrs=True,
                          iters_out=iters, status_out=status, max_passes=3)
        s.synchronize()
        assert int(status.item()) == lp.LP_ST_CAPPED and int(iters.item()) == 3
