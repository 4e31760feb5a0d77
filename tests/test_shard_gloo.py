"""Multi-process host logic of the multi-GPU path on CPU with gloo:
guess slicing and the rank-sharded stable-model search (all-gather of accepted masks,
max-reduce of pass counts); head ranges and the head-range-sharded least model (one
all-gather + OR per pass).  The per-rank solver here is the CPU oracle standing in for
the GPU (test infrastructure; the product's default solver is the CUDA path); the GPU
side of guess slices is covered by tests/test_gpu_parity.py::test_guess_offset_slices."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import lpgen
import oracle
from paper_2009_10247_b200.shard import (derivable_mask, guess_slices, head_ranges, owned_words,
                                          sub_program)


def test_guess_slices_cover_exactly_once():
    for G in (0, 1, 63, 64, 65, 4096, 4097, 1 << 12):
        for world in (1, 2, 3, 5, 8, 100):
            s = guess_slices(G, world)
            assert len(s) == world
            covered = []
            for off, cnt in s:
                assert off % 64 == 0 or cnt == 0
                covered += list(range(off, off + cnt))
            assert covered == list(range(G))


def _oracle_slice(P, off, cnt):
    """Explicit guess rows for global ids off..off+cnt (binary counting over the free
    negated atoms, abar of a negated fact fixed to 0: Def. 8 / reading R8-R9)."""
    negs = oracle.negated_atoms(P)
    facts = set(P.head[np.diff(P.body_ptr) == 0].tolist())
    free = [j for j, a in enumerate(negs) if a not in facts]
    g = np.zeros((cnt, len(negs)), dtype=np.uint8)
    ids = np.arange(off, off + cnt)
    for i, j in enumerate(free):
        g[:, j] = (ids >> i) & 1
    o = oracle.stable(P, guesses=g)
    acc = o["accepted"].astype(np.uint8)
    W = (cnt + 63) // 64
    pad = np.zeros(W * 64, dtype=np.uint8)
    pad[:cnt] = acc
    return np.packbits(pad, bitorder="little").view(np.uint64), int(o["passes"])


def _worker(rank, world, port, seed, q):
    import torch.distributed as dist
    from paper_2009_10247_b200.shard import stable_models_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        rng = np.random.default_rng([seed, 77])
        P = lpgen.random_normal_program(rng, 40, 120, max_len=3, k_max=7)
        f = oracle.stable(P)["f"]
        ids, passes = stable_models_sharded(None, f, solve=lambda o, c: _oracle_slice(P, o, c))
        q.put((rank, ids.tolist(), passes))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,seed", [(2, 1), (2, 2), (3, 3), (2, 4)])
def test_sharded_stable_models_gloo(world, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng([seed, 77])
    P = lpgen.random_normal_program(rng, 40, 120, max_len=3, k_max=7)
    o = oracle.stable(P)
    want = np.nonzero(o["accepted"])[0].tolist()
    for _, ids, passes in res:
        assert ids == want
        assert passes == o["passes"]


def test_head_ranges_partition_the_rules():
    rng = np.random.default_rng(4)
    for _ in range(20):
        n = int(rng.integers(1, 700))
        P = lpgen.random_program(rng, n, int(rng.integers(0, 4 * n)), max_len=5)
        for world in (1, 2, 3, 8):
            rs = head_ranges(P, world)
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(lo % 64 == 0 or lo == n for lo, _ in rs)
            ow = owned_words(P, world)
            W = (n + 63) // 64
            assert ow[0][0] == 0 and sum(c for _, c in ow) == W
            assert all(a[0] + a[1] == b[0] for a, b in zip(ow, ow[1:]))
            for (lo, hi), (w0, c) in zip(rs, ow):    # a rank's heads lie in its owned words
                assert c == 0 or (lo // 64 == w0 and (hi + 63) // 64 == w0 + c)
            subs = [sub_program(P, lo, hi) for lo, hi in rs]
            assert sum(s.n_rules for s in subs) == P.n_rules
            for (lo, hi), s in zip(rs, subs):
                assert ((s.head >= lo) & (s.head < hi)).all()


class _OracleShard:
    """CPU stand-in for the CUDA side of one rank (test infrastructure): ONE T_P
    evaluation of the rank's sub-program by the oracle writes the owned words and the
    status word into the payload; the combine step in numpy.  The host loop, the payload
    layout and the all-gather (gloo) are the product's (shard.ShardedLeastModel)."""

    def __init__(self, P, rank, world):
        lo, hi = head_ranges(P, world)[rank]
        self.sub = sub_program(P, lo, hi)
        ow = owned_words(P, world)
        self.word_lo = [w for w, _ in ow]
        self.word_cnt = [c for _, c in ow]
        self.stride = max(self.word_cnt) + 1
        self.world = world
        self.n = P.n_atoms
        self.flags, self.pops = {}, {}

    def reset(self, popcounts=True):
        self.flags, self.pops = {}, {}

    def one_pass(self, rank, v, payload):
        import torch
        bits = np.unpackbits(v.numpy().view(np.uint8), bitorder="little")[:self.n].astype(bool)
        m, _, _, conv = oracle.lm_jacobi(self.sub, v0=bits, max_iters=1)
        words = oracle.pack_bits(m).view(np.int64)
        w0, cnt = self.word_lo[rank], self.word_cnt[rank]
        out = np.zeros(self.stride, dtype=np.int64)
        out[:cnt] = words[w0:w0 + cnt]
        out[self.stride - 1] = 0 if conv else 4          # LP_ST_CAPPED: derived an atom
        payload.copy_(torch.from_numpy(out))

    def combine(self, k, gathered, v, v_next):
        import torch
        g = gathered.numpy().reshape(self.world, self.stride)
        nv = v.numpy().copy()
        for r in range(self.world):
            w0, cnt = self.word_lo[r], self.word_cnt[r]
            nv[w0:w0 + cnt] |= g[r, :cnt]
        v_next.copy_(torch.from_numpy(nv))
        self.flags[k] = bool((g[:, self.stride - 1] & 4).any())
        self.pops[k + 1] = int(np.unpackbits(nv.view(np.uint8)).sum())

    def changed(self, k):
        return self.flags[k]

    def popcounts(self, iters):
        return [self.pops[j] for j in range(1, iters)]


def _lm_program(seed):
    rng = np.random.default_rng([seed, 91])
    n = int(rng.integers(50, 400)) if seed != 4 else 70     # (seed 4: empty trailing ranges)
    return lpgen.random_program(rng, n, 4 * n, max_len=4, n_facts=n // 10)


def _lm_worker(rank, world, port, seed, q):
    import torch.distributed as dist
    from paper_2009_10247_b200.shard import least_model_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        P = _lm_program(seed)
        model, iters, pops = least_model_sharded(P, backend=_OracleShard(P, rank, world))
        q.put((rank, model.tolist(), iters, pops))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 1), (3, 2), (2, 3), (3, 4)])
def test_sharded_least_model_gloo(world, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lm_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = _lm_program(seed)
    om, stage, oit = oracle.lm_stage(P)
    for _, model, iters, pops in res:
        assert np.array_equal(np.asarray(model, dtype=np.uint64), oracle.pack_bits(om))
        assert iters == oit
        assert pops == oracle.popcounts_from_stage(stage, oit)


def test_derivable_mask_is_d2():
    """D2 = facts ∪ {head(r) : body(r) ⊆ heads ∪ facts}, checked rule by rule."""
    rng = np.random.default_rng(8)
    for _ in range(30):
        n = int(rng.integers(1, 200))
        P = lpgen.random_program(rng, n, int(rng.integers(0, 3 * n)), max_len=4)
        d1 = set(P.head.tolist())
        want = set()
        for r in range(P.n_rules):
            body = P.body_atom[P.body_ptr[r]:P.body_ptr[r + 1]].tolist()
            if all(b in d1 for b in body):
                want.add(int(P.head[r]))
        got = set(np.nonzero(derivable_mask(P))[0].tolist())
        assert got == want
