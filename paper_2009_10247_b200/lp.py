"""Thin ctypes binding of include/lp.h (argument marshalling only).

Every step of the hot path runs in liblp_b200.so's CUDA kernels; this module only
converts numpy / torch buffers to pointers.  There is no CPU fallback: if the shared
library is missing or no GPU is present, the calls raise.

Names follow the C ABI: lp_load, lp_info, lp_negated_atoms, lp_least_model,
lp_stable_models, lp_stable_matrix, lp_guess_model, lp_free.  ``Program`` wraps a
handle with the same operations.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LP_LIB") or os.path.join(_HERE, "liblp_b200.so")   # (LP_LIB: A/B builds)

LP_OK, LP_E_INVALID, LP_E_PARSE, LP_E_SEMANTIC, LP_E_CAP = 0, 1, 2, 3, 4
LP_E_NOMEM, LP_E_CUDA, LP_E_NOT_CONVERGED, LP_E_NODEVICE = 5, 6, 7, 8
LP_LOAD_NO_FRONTIER = 0x1
LP_LOAD_PAPER_LAYOUT = 0x4
LP_LOAD_KEY8 = 0x8
LP_PTR_DEVICE = 0x1
LP_FRONTIER = 0x2
LP_FULL_STREAM = 0x4
LP_FULL_LEAD = 0x8
LP_FULL_NO_PIPE = 0x10
LP_ST_GUARD, LP_ST_OVERFLOW, LP_ST_CAPPED = 0x1, 0x2, 0x4   # lp_run.status_out bit flags

_P = ctypes.c_void_p
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class lp_rules(ctypes.Structure):
    _fields_ = [("n_atoms", ctypes.c_int32), ("n_rules", ctypes.c_int64), ("head", _P),
                ("body_ptr", _P), ("body_atom", _P), ("body_neg", _P)]


class lp_options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("guess_cap", ctypes.c_int), ("flags", ctypes.c_uint32),
                ("smem_bits_cap", ctypes.c_int32), ("grid_blocks", ctypes.c_int32),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", _P), ("derivable", _P)]


class lp_run(ctypes.Structure):
    _fields_ = [("stream", _P), ("flags", ctypes.c_uint32), ("popcounts_out", _P),
                ("popcounts_cap", ctypes.c_int32), ("stage_out", _P), ("ev_begin", _P),
                ("ev_end", _P), ("stats_out", _P), ("max_passes", ctypes.c_int32),
                ("converged_out", _P), ("guess_offset", ctypes.c_int64), ("status_out", _P),
                ("out_word_lo", ctypes.c_int64), ("out_word_count", ctypes.c_int64)]


class lp_info_t(ctypes.Structure):
    _fields_ = [("n_atoms", ctypes.c_int32), ("n_rules", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("n_heads", ctypes.c_int64), ("n_negated", ctypes.c_int32),
                ("n_free_negated", ctypes.c_int32), ("max_body", ctypes.c_int32),
                ("n_segments", ctypes.c_int32), ("n_prime_paper", ctypes.c_int64),
                ("sparsity_eq5", ctypes.c_double), ("device_bytes", ctypes.c_int64),
                ("pass_bytes", ctypes.c_int64), ("truth_mode", ctypes.c_int32),
                ("summary_shift", ctypes.c_int32), ("grid_blocks", ctypes.c_int32),
                ("block_threads", ctypes.c_int32), ("lead_pass_bytes", ctypes.c_int64),
                ("stream_pass_bytes", ctypes.c_int64), ("key_shift", ctypes.c_int32),
                ("n_aux", ctypes.c_int32), ("cluster_ctas", ctypes.c_int32),
                ("frontier_cluster_ctas", ctypes.c_int32), ("stable_cluster_ctas", ctypes.c_int32),
                ("armed_list_cap", ctypes.c_int32), ("stable_compact_atoms", ctypes.c_int32),
                ("stable_compact_rows", ctypes.c_int32), ("small_rows", ctypes.c_int32)]


SYMBOLS = ("lp_load", "lp_info", "lp_negated_atoms", "lp_least_model", "lp_stable_models",
           "lp_stable_search", "lp_stable_matrix", "lp_guess_model", "lp_shard_combine", "lp_free",
           "lp_status_str", "lp_last_error")

_lib = None


def library():
    """Load liblp_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc, sm_100a); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        st = ctypes.c_int
        lib.lp_load.argtypes = [ctypes.POINTER(lp_rules), ctypes.POINTER(lp_options), ctypes.POINTER(_P)]
        lib.lp_load.restype = st
        lib.lp_info.argtypes = [_P, ctypes.POINTER(lp_info_t)]
        lib.lp_info.restype = st
        lib.lp_negated_atoms.argtypes = [_P, _P]
        lib.lp_negated_atoms.restype = st
        lib.lp_least_model.argtypes = [_P, _P, _P, _P, ctypes.POINTER(lp_run)]
        lib.lp_least_model.restype = st
        lib.lp_stable_models.argtypes = [_P, _P, ctypes.c_int64, _P, _P, _P, ctypes.POINTER(lp_run)]
        lib.lp_stable_models.restype = st
        lib.lp_stable_search.argtypes = [_P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, _P, _P,
                                         _P, _P, _P, ctypes.POINTER(lp_run)]
        lib.lp_stable_search.restype = st
        lib.lp_shard_combine.argtypes = [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int64,
                                         _P, _P, _P]
        lib.lp_shard_combine.restype = st
        lib.lp_stable_matrix.argtypes = [_P, _P, ctypes.POINTER(lp_run)]
        lib.lp_stable_matrix.restype = st
        lib.lp_guess_model.argtypes = [_P, ctypes.c_int64, _P, ctypes.POINTER(lp_run)]
        lib.lp_guess_model.restype = st
        lib.lp_free.argtypes = [_P]
        lib.lp_free.restype = None
        lib.lp_status_str.argtypes = [st]
        lib.lp_status_str.restype = ctypes.c_char_p
        lib.lp_last_error.argtypes = []
        lib.lp_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


class LPError(RuntimeError):
    def __init__(self, status: int, where: str):
        lib = library()
        self.status = status
        msg = lib.lp_status_str(status).decode()
        detail = lib.lp_last_error().decode()
        super().__init__(f"{where}: {msg} ({status}): {detail}")


def _check(status: int, where: str):
    if status != LP_OK:
        raise LPError(status, where)


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def _event_ptr(ev) -> Optional[int]:
    if ev is None:
        return None
    if isinstance(ev, int):
        return ev
    if int(ev.cuda_event) == 0:   # torch creates its cudaEvent_t lazily on first record
        ev.record()
    return int(ev.cuda_event)


def _torch_allocator(device: int):
    import torch

    def _alloc(nbytes, ctx):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(nbytes), device=device))
        except Exception:  # noqa: BLE001 -- reported to C as NULL -> LP_E_NOMEM
            return None

    cuda = torch.cuda

    def _free(ptr, nbytes, ctx):
        # at interpreter exit the torch module may already be torn down: the process's
        # device memory goes away with it, so there is nothing left to return
        if cuda is not None and getattr(cuda, "caching_allocator_delete", None) is not None:
            try:
                cuda.caching_allocator_delete(ptr)
            except Exception:  # noqa: BLE001
                pass

    return ALLOC_FN(_alloc), FREE_FN(_free)


def bits_words(n: int) -> int:
    return (n + 63) // 64


class Program:
    """A loaded program (lp_program handle)."""

    def __init__(self, rules, device: int = 0, guess_cap: int = 20, frontier: bool = True,
                 smem_bits_cap: int = 0, grid_blocks: int = 0, allocator: str = "torch",
                 paper_layout: bool = False, key8: bool = False, derivable=None):
        lib = library()
        self._keep = []
        head = np.ascontiguousarray(rules.head, dtype=np.int32)
        ptr = np.ascontiguousarray(rules.body_ptr, dtype=np.int64)
        atom = np.ascontiguousarray(rules.body_atom, dtype=np.int32)
        neg = None if rules.body_neg is None else np.ascontiguousarray(rules.body_neg, dtype=np.uint8)
        r = lp_rules(int(rules.n_atoms), int(head.shape[0]), _ptr(head), _ptr(ptr), _ptr(atom), _ptr(neg))
        opt = lp_options()
        opt.device = int(device)
        opt.guess_cap = int(guess_cap)
        opt.flags = ((0 if frontier else LP_LOAD_NO_FRONTIER) |
                     (LP_LOAD_PAPER_LAYOUT if paper_layout else 0) | (LP_LOAD_KEY8 if key8 else 0))
        opt.smem_bits_cap = int(smem_bits_cap)
        if derivable is not None:
            der = np.ascontiguousarray(derivable, dtype=np.uint8)
            assert der.shape[0] >= int(rules.n_atoms)
            self._keep.append(der)
            opt.derivable = der.ctypes.data
        opt.grid_blocks = int(grid_blocks)
        if device >= 0 and allocator == "torch":
            a, f = _torch_allocator(device)
            opt.alloc, opt.free = a, f
            self._keep += [a, f]
        h = _P()
        _check(lib.lp_load(ctypes.byref(r), ctypes.byref(opt), ctypes.byref(h)), "lp_load")
        self._h = h
        self.device = device
        self.n_atoms = int(rules.n_atoms)
        self.info = lp_info(self)

    # -- lifetime --------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            library().lp_free(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def handle(self):
        return self._h

    # -- calls -----------------------------------------------------------------------
    def negated_atoms(self):
        return lp_negated_atoms(self)

    def least_model(self, v0=None, frontier: bool = False, popcounts: bool = False,
                    stages: bool = False, stream=None, schedule: str = "auto", stats: bool = False,
                    max_passes: int = 0, pipeline: bool = True):
        """Host-buffer call.  v0: None, a bool mask [n], or an id list.  Returns
        (model uint64[ceil(n/64)], iters, dict(popcounts=..., stage=...))."""
        n = self.n_atoms
        v0w = None
        if v0 is not None:
            a = np.asarray(v0)
            mask = np.zeros(n, dtype=bool)
            if a.dtype == bool:
                mask[:] = a
            elif a.size:
                mask[a.astype(np.int64)] = True
            v0w = pack_mask(mask)
        model = np.zeros(max(bits_words(n), 1), dtype=np.uint64)
        pops = np.zeros(n + self.info["n_aux"] + 3, dtype=np.int32) if popcounts else None
        stage = np.zeros(max(n, 1), dtype=np.int32) if stages else None
        st = np.zeros(6, dtype=np.uint64) if stats else None
        conv = ctypes.c_int32(-1)
        iters = lp_least_model(self, v0w, model, frontier=frontier, pops=pops, stage=stage,
                               stream=stream, schedule=schedule, stats=st, max_passes=max_passes,
                               converged=conv, pipeline=pipeline)
        extra = {"converged": bool(conv.value)}
        if stats:
            extra["stats"] = dict(zip(("bytes", "lead_passes", "rows_verified", "entries_verified",
                                       "sm_cycles", "ns"),
                                      (int(x) for x in st)))
        if popcounts:
            extra["popcounts"] = pops[:iters].tolist()
        if stages:
            extra["stage"] = stage[:n]
        return model[:bits_words(n)], iters, extra

    def stable_models(self, guesses=None, n_guesses: int = 0, stream=None, guess_offset: int = 0):
        """Host-buffer call.  guesses: None or uint64[k][W].  With guesses None the call
        covers global guesses [guess_offset, guess_offset + n_guesses) (n_guesses 0 = all
        the rest).  Returns (accepted LOCAL guess ids (np.int64), passes, mask words)."""
        if guesses is None:
            G = (1 << self.info["n_free_negated"]) - int(guess_offset)
            if n_guesses > 0:
                G = min(G, int(n_guesses))
        else:
            G = int(n_guesses)
        W = (G + 63) // 64
        acc = np.zeros(max(W, 1), dtype=np.uint64)
        nacc, passes = lp_stable_models(self, guesses, G, acc, stream=stream, guess_offset=guess_offset)
        bits = np.unpackbits(acc[:W].view(np.uint8), bitorder="little")[:G]
        ids = np.nonzero(bits)[0].astype(np.int64)
        assert ids.size == nacc
        return ids, passes, acc[:W]

    def stable_search(self, h: int, seed: int, max_rounds: int, stream=None):
        """Guess-space reduction (lp_stable_search).  Host-buffer call.
        Returns dict(accepted=local column ids of the last round (np.int64), rounds,
        passes, guesses=uint8[h][k] abar values of the last round)."""
        k = self.info["n_negated"]
        W = (int(h) + 63) // 64
        acc = np.zeros(max(W, 1), dtype=np.uint64)
        gs = np.zeros((max(k, 1), max(W, 1)), dtype=np.uint64)
        nacc, rounds, passes = lp_stable_search(self, h, seed, max_rounds, gs, acc, stream=stream)
        bits = np.unpackbits(acc[:W].view(np.uint8), bitorder="little")[:h]
        ids = np.nonzero(bits)[0].astype(np.int64)
        assert ids.size == nacc
        cols = np.zeros((int(h), k), dtype=np.uint8)
        for j in range(k):
            cols[:, j] = np.unpackbits(gs[j, :W].view(np.uint8), bitorder="little")[:h]
        return dict(accepted=ids, rounds=rounds, passes=passes, guesses=cols)

    def stable_matrix(self, stream=None):
        G = self._last_G
        W = (G + 63) // 64
        out = np.zeros((self.n_atoms, W), dtype=np.uint64)
        lp_stable_matrix(self, out, stream=stream)
        return out

    def guess_model(self, g: int, stream=None):
        out = np.zeros(max(bits_words(self.n_atoms), 1), dtype=np.uint64)
        lp_guess_model(self, g, out, stream=stream)
        return out[:bits_words(self.n_atoms)]


def pack_mask(mask) -> np.ndarray:
    m = np.asarray(mask, dtype=np.uint8)
    n = m.shape[0]
    w = bits_words(n)
    padded = np.zeros(max(w, 1) * 64, dtype=np.uint8)
    padded[:n] = m
    return np.packbits(padded, bitorder="little").view(np.uint64).copy()


def unpack_bits(words, n: int) -> np.ndarray:
    return np.unpackbits(np.asarray(words, dtype=np.uint64).view(np.uint8), bitorder="little")[:n]


# ---- module-level functions with the C names ----------------------------------------

def lp_load(rules, **kw) -> Program:
    return Program(rules, **kw)


class _Rules:
    def __init__(self, n_atoms, head, body_ptr, body_atom, body_neg):
        self.n_atoms, self.head, self.body_ptr = n_atoms, head, body_ptr
        self.body_atom, self.body_neg = body_atom, body_neg


def load(head, body_ptr, body_atom, body_neg=None, n_atoms=None, **kw) -> Program:
    """SURVEY §8(b)'s shim: a program from flat rule arrays (lp_rules layout: head[R],
    body_ptr[R+1], body_atom[nnz], optional body_neg[nnz] with 1 = 'not atom');
    n_atoms defaults to 1 + the largest atom id."""
    head = np.ascontiguousarray(head, dtype=np.int32)
    body_ptr = np.ascontiguousarray(body_ptr, dtype=np.int64)
    body_atom = np.ascontiguousarray(body_atom, dtype=np.int32)
    if n_atoms is None:
        n_atoms = int(max(head.max(initial=-1), body_atom.max(initial=-1))) + 1
    neg = None if body_neg is None else np.ascontiguousarray(body_neg, dtype=np.uint8)
    return Program(_Rules(int(n_atoms), head, body_ptr, body_atom, neg), **kw)


def lp_info(p: Program) -> dict:
    info = lp_info_t()
    _check(library().lp_info(p.handle, ctypes.byref(info)), "lp_info")
    return {name: getattr(info, name) for name, _ in lp_info_t._fields_}


def lp_negated_atoms(p: Program):
    k = p.info["n_negated"]
    out = np.zeros(max(k, 1), dtype=np.int32)
    _check(library().lp_negated_atoms(p.handle, _ptr(out)), "lp_negated_atoms")
    return out[:k].tolist()


def _run(stream=None, flags=0, pops=None, stage=None, ev_begin=None, ev_end=None, stats=None):
    r = lp_run()
    r.stats_out = _ptr(stats)
    r.stream = _stream_ptr(stream)
    r.flags = flags
    r.popcounts_out = _ptr(pops)
    r.popcounts_cap = 0 if pops is None else int(pops.shape[0] if hasattr(pops, "shape") else len(pops))
    r.stage_out = _ptr(stage)
    r.ev_begin = _event_ptr(ev_begin)
    r.ev_end = _event_ptr(ev_end)
    return r


def lp_least_model(p: Program, v0, model_out, frontier=False, pops=None, stage=None, stream=None,
                   device_ptrs=False, iters_out=None, ev_begin=None, ev_end=None, schedule="auto",
                   stats=None, max_passes=0, converged=None, pipeline=True, status_out=None,
                   out_words=None):
    """Marshals lp_least_model.  Host mode (default): numpy buffers, returns iters.
    device_ptrs=True: torch CUDA tensors (v0 int64 words or None, model_out int64
    words, iters_out int32[1], optional pops/stage, optional status_out int32[1] that
    the kernel fills with the LP_ST_* flags), asynchronous on ``stream``.  Host mode:
    status_out may be a ctypes.c_int32."""
    flags = (LP_FRONTIER if frontier else 0) | (LP_PTR_DEVICE if device_ptrs else 0)
    flags |= {"auto": 0, "stream": LP_FULL_STREAM, "lead": LP_FULL_LEAD}[schedule]
    flags |= 0 if pipeline else LP_FULL_NO_PIPE
    run = _run(stream, flags, pops, stage, ev_begin, ev_end, stats)
    run.max_passes = int(max_passes)
    if status_out is not None:
        run.status_out = _ptr(status_out) if device_ptrs else ctypes.addressof(status_out)
    if out_words is not None:                 # (first word, word count) of the model written
        run.out_word_lo, run.out_word_count = int(out_words[0]), int(out_words[1])
    if converged is not None and not device_ptrs:
        run.converged_out = ctypes.addressof(converged)
    if device_ptrs:
        _check(library().lp_least_model(p.handle, _ptr(v0), _ptr(model_out), _ptr(iters_out),
                                         ctypes.byref(run)), "lp_least_model")
        return None
    it = ctypes.c_int32(0)
    _check(library().lp_least_model(p.handle, _ptr(v0), _ptr(model_out), ctypes.addressof(it),
                                     ctypes.byref(run)), "lp_least_model")
    return it.value


def lp_stable_models(p: Program, guesses, n_guesses, accepted_out, stream=None, device_ptrs=False,
                     n_accepted_out=None, passes_out=None, ev_begin=None, ev_end=None,
                     guess_offset: int = 0, status_out=None):
    flags = LP_PTR_DEVICE if device_ptrs else 0
    run = _run(stream, flags, ev_begin=ev_begin, ev_end=ev_end)
    run.guess_offset = int(guess_offset)
    if status_out is not None:
        run.status_out = _ptr(status_out) if device_ptrs else ctypes.addressof(status_out)
    g = None
    if guesses is not None:
        g = guesses if device_ptrs else np.ascontiguousarray(guesses, dtype=np.uint64)
    if guesses is not None:
        p._last_G = int(n_guesses)
    else:
        rest = (1 << p.info["n_free_negated"]) - int(guess_offset)
        p._last_G = min(rest, int(n_guesses)) if int(n_guesses) > 0 else rest
    if device_ptrs:
        _check(library().lp_stable_models(p.handle, _ptr(g), int(n_guesses), _ptr(accepted_out),
                                           _ptr(n_accepted_out), _ptr(passes_out), ctypes.byref(run)),
               "lp_stable_models")
        return None
    na = ctypes.c_int64(0)
    ps = ctypes.c_int32(0)
    _check(library().lp_stable_models(p.handle, _ptr(g), int(n_guesses), _ptr(accepted_out),
                                       ctypes.addressof(na), ctypes.addressof(ps), ctypes.byref(run)),
           "lp_stable_models")
    return na.value, ps.value


def lp_stable_search(p: Program, h, seed, max_rounds, guesses_out, accepted_out, stream=None,
                     device_ptrs=False, n_accepted_out=None, rounds_out=None, passes_out=None,
                     ev_begin=None, ev_end=None, status_out=None):
    """Marshals lp_stable_search.  Host mode: numpy buffers (guesses_out uint64[k][W] or
    None, accepted_out uint64[W]); returns (n_accepted, rounds, passes).  device_ptrs:
    torch CUDA tensors, asynchronous on ``stream``."""
    run = _run(stream, LP_PTR_DEVICE if device_ptrs else 0, ev_begin=ev_begin, ev_end=ev_end)
    if status_out is not None:
        run.status_out = _ptr(status_out) if device_ptrs else ctypes.addressof(status_out)
    p._last_G = int(h)
    if device_ptrs:
        _check(library().lp_stable_search(p.handle, int(h), int(seed) & ((1 << 64) - 1), int(max_rounds),
                                           _ptr(guesses_out), _ptr(accepted_out), _ptr(n_accepted_out),
                                           _ptr(rounds_out), _ptr(passes_out), ctypes.byref(run)),
               "lp_stable_search")
        return None
    na, rd, ps = ctypes.c_int64(0), ctypes.c_int32(0), ctypes.c_int32(0)
    _check(library().lp_stable_search(p.handle, int(h), int(seed) & ((1 << 64) - 1), int(max_rounds),
                                       _ptr(guesses_out), _ptr(accepted_out), ctypes.addressof(na),
                                       ctypes.addressof(rd), ctypes.addressof(ps), ctypes.byref(run)),
           "lp_stable_search")
    return na.value, rd.value, ps.value


def lp_shard_combine(gathered, world, stride, word_lo, word_cnt, v, v_next, changed_out,
                     popcount_inout=None, stream=None):
    """Marshals lp_shard_combine: torch CUDA tensors (gathered int64 [world*stride], v and
    v_next int64 [n_words], changed_out int32[1], optional popcount_inout int32[1]) and
    host int64 arrays word_lo / word_cnt; asynchronous on ``stream``."""
    lo = np.ascontiguousarray(word_lo, dtype=np.int64)
    cnt = np.ascontiguousarray(word_cnt, dtype=np.int64)
    _check(library().lp_shard_combine(_ptr(gathered), int(world), int(stride), _ptr(lo), _ptr(cnt), _ptr(v),
                                       _ptr(v_next), int(v.numel()), _ptr(changed_out), _ptr(popcount_inout),
                                       _stream_ptr(stream)), "lp_shard_combine")


def lp_stable_matrix(p: Program, out, stream=None, device_ptrs=False):
    run = _run(stream, LP_PTR_DEVICE if device_ptrs else 0)
    _check(library().lp_stable_matrix(p.handle, _ptr(out), ctypes.byref(run)), "lp_stable_matrix")


def lp_guess_model(p: Program, g, out, stream=None, device_ptrs=False):
    run = _run(stream, LP_PTR_DEVICE if device_ptrs else 0)
    _check(library().lp_guess_model(p.handle, int(g), _ptr(out), ctypes.byref(run)), "lp_guess_model")


def lp_free(p: Program):
    p.close()
