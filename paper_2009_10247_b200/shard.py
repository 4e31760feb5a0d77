"""Multi-GPU plumbing: one process per GPU, torch.distributed.

Stable models shard by guesses.  The 2^f guesses of the initial matrix (Def. 8,
PAPER.md:243-253) are independent columns of Algorithm 2's iteration:
column g's fixpoint depends on nothing but column g.  Rank r therefore solves the
64-aligned slice [off_r, off_r + cnt_r) of the binary-counting order (lp_run.guess_offset)
with no exchange during the fixpoint; afterwards the accepted masks are all-gathered once
(<= G/8 bytes in total) and the pass counts max-reduced (the whole-matrix pass count is the
maximum over columns).  NCCL on GPUs, gloo in the CPU tests.

The least model of ONE program does not partition without a per-pass exchange (DESIGN.md
§8); bench.py runs it as replicas (independent programs, weak scaling).

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
