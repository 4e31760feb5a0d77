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
entries of the rules whose head they are) and loads only those rules (with the whole
program's D2 as layout hint).  Pass k: every rank runs ONE θ-pass of its rules from the
same v_k (lp_run.max_passes = 1) writing only its owned words and its status word into a
payload; the payloads are all-gathered (NCCL, ~W/N words per rank); lp_shard_combine
(a CUDA kernel) ORs them into v_{k+1}, sets the changed flag and counts |v_{k+1}|.  The
host reads pass k's flag after it queued pass k+1 (one extra, idempotent pass at the
end; no host sync per pass).  The union of the ranks' passes is one T_P evaluation over
all of P, so model, pass count and popcount trace equal the single-GPU ones.  Under
torchrun (N > 1) this is bench.py's main line (strong scaling: one C4 for all ranks).

This module only moves buffers between ranks; every step of the path runs in the CUDA
kernels behind lp.Program and lp_shard_combine (the `solve` / `backend` hooks exist so
the CPU tests can drive the same host logic with a stand-in -- the product never passes
one).
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


def owned_words(rules, world: int) -> List[Tuple[int, int]]:
    """(first word, word count) of each rank's atom range: the model words only its rules
    can set.  The ranges tile [0, ceil(n/64)) in rank order."""
    W = (int(rules.n_atoms) + 63) // 64
    out = []
    for lo, hi in head_ranges(rules, world):
        w0 = -(-lo // 64)                      # (lo is 64-aligned, or n for an empty tail)
        w1 = W if hi >= int(rules.n_atoms) else hi // 64
        out.append((w0, max(0, w1 - w0)))
    return out


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


def derivable_mask(rules) -> np.ndarray:
    """The whole program's D2 (facts ∪ heads of rules whose body lies in heads ∪ facts):
    the layout hint (lp_options.derivable) every shard loads with, so atoms derived on
    another GPU keep fine key groups.  A layout heuristic only: never a result."""
    n = int(rules.n_atoms)
    head = np.asarray(rules.head, dtype=np.int64)
    ptr = np.asarray(rules.body_ptr, dtype=np.int64)
    atom = np.asarray(rules.body_atom, dtype=np.int64)
    lens = np.diff(ptr)
    d1 = np.zeros(n, dtype=bool)
    d1[head] = True
    ok = np.ones(head.size, dtype=bool)
    nz = lens > 0
    if atom.size:
        ok[nz] = np.logical_and.reduceat(d1[atom], ptr[:-1][nz])
    d2 = np.zeros(n, dtype=np.uint8)
    d2[head[ok]] = 1
    return d2


def _mapped_device_ptr(host_ptr: int) -> int:
    """Device address of page-locked host memory (the same address under unified
    addressing; cudaPointerGetAttributes says so)."""
    try:
        from cuda.bindings import runtime as rt
        err, at = rt.cudaPointerGetAttributes(host_ptr)
        if int(err) == 0 and int(at.devicePointer):
            return int(at.devicePointer)
    except Exception:  # noqa: BLE001 -- no cuda-python: unified addressing's identity
        pass
    return host_ptr


class _GpuShard:
    """This rank's side of the device exchange: ONE θ-pass of its rules (CUDA kernels
    behind lp_least_model, max_passes = 1) writing its owned words and its status word into
    the payload, and the combine step (lp_shard_combine) computing v_{k+1}, the changed
    flag and |v_{k+1}| on the device.  The combine kernel writes pass k's flag straight into
    page-locked host memory (mapped: the device pointer is the host pointer under unified
    addressing); the host reads it behind an event one pass later.  Every ctypes argument
    is prepared once, so a pass costs two library calls, the all-gather and an event."""

    def __init__(self, rules, lo, hi, word_lo, word_cnt, stride, world, device, program=None,
                 cap=None):
        import ctypes

        import torch

        from . import lp
        self.lp = lp
        self.torch = torch
        self.device = device
        self.prog = program or lp.Program(sub_program(rules, lo, hi), device=device.index or 0,
                                          derivable=derivable_mask(rules))
        self.word_lo = np.ascontiguousarray(word_lo, dtype=np.int64)
        self.word_cnt = np.ascontiguousarray(word_cnt, dtype=np.int64)
        self.stride, self.world = stride, world
        cap = cap or (int(rules.n_atoms) + 3)
        self.it = torch.zeros(1, dtype=torch.int32, device=device)
        self.flags_host = torch.zeros(cap, dtype=torch.int32).pin_memory()   # written by the kernel
        self.flags_dev = _mapped_device_ptr(self.flags_host.data_ptr())
        self.pops = torch.zeros(cap, dtype=torch.int32, device=device)
        self.events = [torch.cuda.Event() for _ in range(cap)]
        self.stream = torch.cuda.current_stream(device)
        self.lib = lp.library()
        self.run = None      # lp_run of this rank's pass (set on the first pass: needs the payload)
        self.c_int = ctypes

    def reset(self, popcounts=True):
        if popcounts:   # (the combine adds |v_{k+1}| into pops[k + 1]; unused otherwise)
            self.pops.zero_()

    def _prepare(self, rank, payload):
        lp = self.lp
        r = lp.lp_run()
        r.stream = int(self.stream.cuda_stream)
        r.flags = lp.LP_PTR_DEVICE
        r.max_passes = 1
        r.status_out = payload.data_ptr() + 8 * (self.stride - 1)   # low half of the last word
        r.out_word_lo = int(self.word_lo[rank])
        r.out_word_count = int(self.word_cnt[rank])
        self.run = r
        self.payload_ptr = payload.data_ptr()

    def one_pass(self, rank, v, payload):
        """payload[:cnt] = this rank's owned words of v ∪ T_{P_r}(v); the low half of
        payload[stride - 1] = its status word (LP_ST_CAPPED: the pass derived an atom)."""
        if int(self.word_cnt[rank]) == 0:   # (an empty trailing range: nothing to derive)
            payload.zero_()
            return
        if self.run is None or self.payload_ptr != payload.data_ptr():
            self._prepare(rank, payload)
        st = self.lib.lp_least_model(self.prog.handle, v.data_ptr(), self.payload_ptr, self.it.data_ptr(),
                                     self.c_int.byref(self.run))
        if st != self.lp.LP_OK:
            raise self.lp.LPError(st, "lp_least_model (shard pass)")

    def combine(self, k, gathered, v, v_next):
        st = self.lib.lp_shard_combine(gathered.data_ptr(), self.world, self.stride, self.word_lo.ctypes.data,
                                       self.word_cnt.ctypes.data, v.data_ptr(), v_next.data_ptr(),
                                       v.numel(), self.flags_dev + 4 * k,
                                       self.pops.data_ptr() + 4 * (k + 1), int(self.stream.cuda_stream))
        if st != self.lp.LP_OK:
            raise self.lp.LPError(st, "lp_shard_combine")
        self.events[k].record(self.stream)

    def changed(self, k) -> bool:
        self.events[k].synchronize()
        return bool(int(self.flags_host[k]))

    def popcounts(self, iters):
        return self.pops[1:iters].cpu().tolist()


class ShardedLeastModel:
    """Head-range-sharded least model of a definite program (module docstring).

    Setup (once per program, host side): this rank's head range and owned words, its
    sub-program on the GPU (loaded with the whole program's D2), the initial words
    I_0 = facts(P) and the payload / gather buffers.  ``run`` is the per-call loop: per pass
    one θ-pass on every rank, one all-gather of the owned words + status word (NCCL), one
    combine kernel; the host checks pass k's changed flag after enqueuing pass k+1.
    ``backend`` defaults to the CUDA path (_GpuShard); the CPU tests pass a stand-in with
    the same methods (one_pass, combine, changed, popcounts, reset)."""

    def __init__(self, rules, group=None, backend=None, device=None, program=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.n = int(rules.n_atoms)
        self.W = max((self.n + 63) // 64, 1)
        self.lo, self.hi = head_ranges(rules, self.world)[self.rank]
        ow = owned_words(rules, self.world)
        self.word_lo = [w for w, _ in ow]
        self.word_cnt = [c for _, c in ow]
        self.stride = max(self.word_cnt) + 1       # owned words + the status word
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device())
                      if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        self.device = device
        self.backend = backend or _GpuShard(rules, self.lo, self.hi, self.word_lo, self.word_cnt,
                                            self.stride, self.world, device, program)
        ptr = np.asarray(rules.body_ptr)
        start = np.zeros(self.W * 64, dtype=np.uint8)        # I_0 = facts of every rank's rules
        start[np.asarray(rules.head)[ptr[1:] == ptr[:-1]]] = 1
        self.start = start
        self.start_pop = int(np.count_nonzero(start))   # |I_0| (host work once, not per run)
        self.facts_words = torch.from_numpy(np.packbits(start, bitorder="little").view(np.int64).copy()).to(device)
        self.v = [torch.zeros(self.W, dtype=torch.int64, device=device) for _ in range(2)]
        self.payload = torch.zeros(self.stride, dtype=torch.int64, device=device)
        self.gathered = torch.zeros(self.world * self.stride, dtype=torch.int64, device=device)
        self.max_passes = self.n + 3

    def run(self, v0=None, popcounts: bool = True, v0_words=None):
        """Returns (model words uint64[ceil(n/64)], iters, popcount trace or []).  The start
        set: v0 (bool mask or None = facts only) or v0_words (packed LSB-first uint64 words
        of the atoms, as lp_least_model takes them; the facts are added on the device)."""
        import torch
        import torch.distributed as dist

        if v0_words is not None:
            w = torch.from_numpy(np.ascontiguousarray(v0_words, dtype=np.uint64).view(np.int64))
            self.v[0].zero_()
            self.v[0][:w.numel()].copy_(w, non_blocking=True)
            self.v[0].bitwise_or_(self.facts_words)
            if self.n % 64 and (self.n + 63) // 64 == self.W:   # (padding bits past atom n-1 off)
                self.v[0][self.W - 1:].bitwise_and_((1 << (self.n % 64)) - 1)
            pop0 = int(np.unpackbits(self.v[0].cpu().numpy().view(np.uint8)).sum()) if popcounts else 0
        elif v0 is None:
            self.v[0].copy_(self.facts_words)
            pop0 = self.start_pop
        else:
            st = self.start.copy()
            st[:self.n] |= np.asarray(v0, dtype=bool).astype(np.uint8)
            self.v[0].copy_(torch.from_numpy(np.packbits(st, bitorder="little").view(np.int64).copy()))
            pop0 = int(np.count_nonzero(st)) if popcounts else 0
        b = self.backend
        b.reset(popcounts)
        k = 0
        while True:
            if k >= self.max_passes:
                raise RuntimeError("sharded least model: pass guard exceeded")
            v, v_next = self.v[k & 1], self.v[(k + 1) & 1]
            b.one_pass(self.rank, v, self.payload)
            dist.all_gather_into_tensor(self.gathered, self.payload, group=self.group)
            b.combine(k, self.gathered, v, v_next)
            # pass k-1's flag (pass k is already queued behind it): u = v -> fixpoint
            if k >= 1 and not b.changed(k - 1):
                iters = k
                break
            k += 1
        if self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()
        model = self.v[iters & 1].cpu().numpy().view(np.uint64)[: (self.n + 63) // 64].copy()
        pops = ([pop0] + b.popcounts(iters)) if popcounts else []
        return model, iters, pops


def least_model_sharded(rules, group=None, v0=None, backend=None, device=None, program=None,
                        popcounts: bool = True):
    """One-shot ShardedLeastModel(...).run(v0): (model words, iters, popcount trace)."""
    return ShardedLeastModel(rules, group, backend, device, program).run(v0, popcounts)
