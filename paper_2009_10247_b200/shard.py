"""Multi-GPU plumbing: one process per GPU, torch.distributed.

Stable models shard by guesses.  The 2^f guesses of the initial matrix (Def. 8,
PAPER.md:243-253) are independent columns of Algorithm 2's iteration:
column g's fixpoint depends on nothing but column g.  Rank r therefore solves the
64-aligned slice [off_r, off_r + cnt_r) of the binary-counting order (lp_run.guess_offset)
with no exchange during the fixpoint; afterwards the accepted masks are all-gathered once
(<= G/8 bytes in total) and the pass counts max-reduced (the whole-matrix pass count is the
maximum over columns).  NCCL on GPUs, gloo in the CPU tests.

The least model of ONE program partitions by head ranges with one exchange per pass
(SURVEY.md §8(e)): rank r owns the atoms [lo_r, hi_r) (64-aligned, balanced by the body
entries of the rules whose head they are) and loads only those rules.  Pass k: every rank
evaluates T over its rules from the same v_k (one θ-pass, lp_run.max_passes = 1), the
full-length results are all-gathered and OR-ed into v_{k+1}; the loop stops after the first
pass that changed nothing anywhere.  The union of the ranks' passes is one T_P evaluation
over all of P, so model, pass count and popcount trace equal the single-GPU ones.
bench.py's main line runs independent replicas (weak scaling); this path is its strong-
scaling extra.

This module only moves buffers between ranks; every step of the path runs in the CUDA
kernels behind lp.Program (the `solve` hook exists so the CPU tests can drive the same
host logic with a stand-in solver -- the product never passes one).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def guess_slices(G: int, world: int) -> List[Tuple[int, int]]:
    """Split guesses [0, G) into `world` contiguous slices on 64-guess word boundaries:
    rank r gets (offset, count) with offset = r * per * 64, per = ceil(ceil(G/64)/world)
    words; trailing ranks may get count 0."""
    if G < 0 or world < 1:
        raise ValueError("G >= 0 and world >= 1 required")
    words = (G + 63) // 64
    per = (words + world - 1) // world
    out = []
    for r in range(world):
        off = r * per * 64
        cnt = max(0, min(G, off + per * 64) - off) if off < G else 0
        out.append((min(off, G), cnt))
    return out


def _gpu_solve(prog) -> Callable[[int, int], Tuple[np.ndarray, int]]:
    def solve(off: int, cnt: int):
        _, passes, acc = prog.stable_models(guess_offset=off, n_guesses=cnt)
        return acc, passes
    return solve


def stable_models_sharded(prog, n_free: int, group=None,
                          solve: Optional[Callable[[int, int], Tuple[np.ndarray, int]]] = None,
                          device=None):
    """Rank-sharded lp_stable_models over all 2^n_free guesses.

    Returns (global accepted guess ids (np.int64, ascending), whole-matrix passes), the
    same on every rank.  `solve(offset, count) -> (mask words uint64[ceil(count/64)],
    passes)` defaults to the GPU call on `prog`."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    G = 1 << int(n_free)
    slices = guess_slices(G, world)
    per = (((G + 63) // 64) + world - 1) // world
    off, cnt = slices[rank]
    solve = solve or _gpu_solve(prog)
    local = np.zeros(max(per, 1), dtype=np.uint64)
    passes = 0
    if cnt > 0:
        mask, passes = solve(off, cnt)
        w = (cnt + 63) // 64
        local[:w] = np.asarray(mask, dtype=np.uint64)[:w]
    if device is None:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.from_numpy(local.view(np.int64)).to(device)
    allw = torch.empty(world * t.numel(), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allw, t, group=group)
    p = torch.tensor([int(passes)], dtype=torch.int64, device=device)
    dist.all_reduce(p, op=dist.ReduceOp.MAX, group=group)
    words = allw.cpu().numpy().view(np.uint64)[: (G + 63) // 64]
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:G]
    return np.nonzero(bits)[0].astype(np.int64), int(p.item())


def head_ranges(rules, world: int) -> List[Tuple[int, int]]:
    """Contiguous, 64-aligned atom ranges [lo, hi), one per rank, covering [0, n), balanced
    by the rule weight (body length + 1) of the heads they contain."""
    n = int(rules.n_atoms)
    lens = np.diff(np.asarray(rules.body_ptr, dtype=np.int64)) + 1
    w = np.bincount(np.asarray(rules.head, dtype=np.int64), weights=lens, minlength=n)[:n]
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        a = int(np.searchsorted(cum, total * r / world))
        a = min(n, max(bounds[-1], (a + 63) // 64 * 64))
        bounds.append(a)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def sub_program(rules, lo: int, hi: int):
    """The rules whose head is in [lo, hi), over the same atoms (lpgen.Rules)."""
    import lpgen
    head = np.asarray(rules.head)
    ptr = np.asarray(rules.body_ptr, dtype=np.int64)
    keep = np.nonzero((head >= lo) & (head < hi))[0]
    lens = ptr[keep + 1] - ptr[keep]
    nptr = np.zeros(keep.size + 1, dtype=np.int64)
    np.cumsum(lens, out=nptr[1:])
    idx = (np.repeat(ptr[keep], lens) + np.arange(int(nptr[-1])) - np.repeat(nptr[:-1], lens)).astype(np.int64)
    atoms = np.asarray(rules.body_atom)[idx].astype(np.int32)
    return lpgen.Rules(n_atoms=int(rules.n_atoms), head=head[keep].astype(np.int32), body_ptr=nptr,
                       body_atom=atoms, body_neg=None, meta={"shard": (lo, hi)})


def _gpu_one_pass(prog):
    import torch

    from . import lp
    it = None

    def one_pass(v):
        nonlocal it
        if it is None:
            it = torch.zeros(1, dtype=torch.int32, device=v.device)
        out = torch.empty_like(v)
        lp.lp_least_model(prog, v, out, device_ptrs=True, iters_out=it, max_passes=1,
                          stream=torch.cuda.current_stream(v.device))
        return out
    return one_pass


class ShardedLeastModel:
    """Head-range-sharded least model of a definite program (module docstring).

    Setup (once per program, host side): this rank's head range, its sub-program on the
    GPU and the initial words I_0 = facts(P).  ``run`` is the per-call device loop.
    ``one_pass(v: int64 tensor of model words) -> int64 tensor`` defaults to one θ-pass
    of the CUDA kernels over this rank's rules (the CPU tests pass a stand-in)."""

    def __init__(self, rules, group=None, one_pass=None, device=None, program=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.n = int(rules.n_atoms)
        self.W = max((self.n + 63) // 64, 1)
        self.lo, self.hi = head_ranges(rules, self.world)[self.rank]
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device())
                      if dist.get_backend(group) == "nccl" else "cpu")
        self.device = device
        if one_pass is None:
            from . import lp
            prog = program or lp.Program(sub_program(rules, self.lo, self.hi),
                                         device=torch.cuda.current_device())
            one_pass = _gpu_one_pass(prog)
        self.one_pass = one_pass
        ptr = np.asarray(rules.body_ptr)
        start = np.zeros(self.W * 64, dtype=np.uint8)        # I_0 = facts of every rank's rules
        start[np.asarray(rules.head)[ptr[1:] == ptr[:-1]]] = 1
        self.start = start
        self.facts_words = torch.from_numpy(np.packbits(start, bitorder="little").view(np.int64).copy()).to(device)
        self.buf = torch.empty(self.world * self.W, dtype=torch.int64, device=device)

    def run(self, v0=None, popcounts: bool = True):
        """Returns (model words uint64[ceil(n/64)], iters, popcount trace or [])."""
        import torch
        import torch.distributed as dist

        if v0 is None:
            v = self.facts_words.clone()
            pops = [int(self.start.sum())] if popcounts else []
        else:
            st = self.start.copy()
            st[:self.n] |= np.asarray(v0, dtype=bool).astype(np.uint8)
            v = torch.from_numpy(np.packbits(st, bitorder="little").view(np.int64).copy()).to(self.device)
            pops = [int(st.sum())] if popcounts else []
        W, world = self.W, self.world
        iters = 0
        while True:
            mine = self.one_pass(v)
            dist.all_gather_into_tensor(self.buf, mine, group=self.group)
            nxt = self.buf.view(world, W)[0].clone()
            for r in range(1, world):
                nxt.bitwise_or_(self.buf.view(world, W)[r])
            iters += 1
            if torch.equal(nxt, v):
                break
            v = nxt
            if popcounts:
                pops.append(int(np.unpackbits(v.cpu().numpy().view(np.uint8)).sum()))
        return v.cpu().numpy().view(np.uint64)[: (self.n + 63) // 64].copy(), iters, pops


def least_model_sharded(rules, group=None, v0=None, one_pass=None, device=None, program=None,
                        popcounts: bool = True):
    """One-shot ShardedLeastModel(...).run(v0): (model words, iters, popcount trace)."""
    return ShardedLeastModel(rules, group, one_pass, device, program).run(v0, popcounts)
