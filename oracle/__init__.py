"""CPU oracle for arXiv 2009.10247 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import, call, link or execute anything under
``oracle/``.  The product (``paper_2009_10247_b200``) never imports it, and the two
share no code: only the seeded input generators (``lpgen``) serve both.

Contents
  lp_oracle.c  plain C (gcc -O2, single thread): O-LM Jacobi T_P (the definition),
               O-STAGE forward chaining, O-STABLE per-guess Algorithms 2-3 on P+,
               O-CERT certificate checker.  Wrapped here via ctypes.
  paper.py     the paper's own layout, literally, in exact rational arithmetic:
               standardisation, program matrix (Def. 2), COO/CSR,
               theta (Def. 5), Algorithm 1, positive form (Eq. 4), normal matrix
               (Def. 7), initial matrix (Def. 8), Algorithms 2-3.
  brute.py     brute-force enumeration of Herbrand interpretations: least model as the
               intersection of all models, stable models by the Gelfond-Lifschitz
               reduct (small n only).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): paper goldens (Examples 1-4, tests/
golden/), closed forms (chains, layered programs, transitive closure vs BFS), brute
force on random small programs, certificate and invariants.  Parity status of every
function is listed in DESIGN.md "Oracle".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile lp_oracle.c with gcc (plain -O2, no vectorisation flags beyond -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        _lib.orc_lm_jacobi.argtypes = [i32, i64, P, P, P, P, P, P, i32, i32, P, P]
        _lib.orc_lm_stage.argtypes = [i32, i64, P, P, P, P, P, P]
        _lib.orc_stable.argtypes = [i32, i64, P, P, P, P, i64, P, P, P, P, P, P, P]
        _lib.orc_certify.argtypes = [i32, i64, P, P, P, P, P, P, i32]
        _lib.orc_lm_stage_timed.argtypes = [i32, i64, P, P, P, P, P, P, i32, P]
        for f in (_lib.orc_lm_jacobi, _lib.orc_lm_stage, _lib.orc_stable, _lib.orc_certify,
                  _lib.orc_lm_stage_timed):
            f.restype = ctypes.c_int
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _arrays(rules):
    head = np.ascontiguousarray(rules.head, dtype=np.int32)
    ptr = np.ascontiguousarray(rules.body_ptr, dtype=np.int64)
    atom = np.ascontiguousarray(rules.body_atom, dtype=np.int32)
    return head, ptr, atom


def _v0(rules, v0):
    if v0 is None:
        return None
    """v0 is either a bool mask of length n or a sequence of atom ids."""
    v = np.zeros(max(rules.n_atoms, 1), dtype=np.uint8)
    a = np.asarray(v0)
    if a.dtype == bool:
        v[:rules.n_atoms] = a
    elif a.size:
        v[a.astype(np.int64)] = 1
    return v


def _definite(rules):
    if not rules.is_definite():
        raise ValueError("least-model oracle needs a definite program")


def lm_jacobi(rules, v0=None, max_iters: int = 0):
    """O-LM: Jacobi T_P from I_0 = v0 ∪ facts.
    Returns (model uint8[n], iters, popcounts list, converged)."""
    _definite(rules)
    lib = _load()
    head, ptr, atom = _arrays(rules)
    n = rules.n_atoms
    model = np.zeros(max(n, 1), dtype=np.uint8)
    cap = n + 2
    pops = np.zeros(cap, dtype=np.int32)
    iters, conv = ctypes.c_int32(0), ctypes.c_int32(0)
    rc = lib.orc_lm_jacobi(n, rules.n_rules, _p(head), _p(ptr), _p(atom), _p(_v0(rules, v0)),
                           _p(model), _p(pops), cap, int(max_iters),
                           ctypes.byref(iters), ctypes.byref(conv))
    if rc:
        raise MemoryError(rc)
    it = iters.value
    npop = it if conv.value else it + 1
    return model[:n], it, pops[:npop].tolist(), bool(conv.value)


def lm_stage(rules, v0=None):
    """O-STAGE: (model uint8[n], stage int32[n] (-1 = false), iters)."""
    _definite(rules)
    lib = _load()
    head, ptr, atom = _arrays(rules)
    n = rules.n_atoms
    stage = np.zeros(max(n, 1), dtype=np.int32)
    iters = ctypes.c_int32(0)
    rc = lib.orc_lm_stage(n, rules.n_rules, _p(head), _p(ptr), _p(atom), _p(_v0(rules, v0)),
                          _p(stage), ctypes.byref(iters))
    if rc:
        raise MemoryError(rc)
    stage = stage[:n]
    return (stage >= 0).astype(np.uint8), stage, iters.value


def lm_stage_timed(rules, v0=None, trials: int = 3):
    """O-STAGE's fixpoint phase timed on its own (bench.py cpu_baseline, BASELINE.md's
    CPU-baseline plan): occurrence lists built once (untimed), then `trials` runs of the
    unchanged forward-chaining loop.  Returns (model uint8[n], stage, iters, seconds
    per trial).  The caller pins the thread to one core."""
    _definite(rules)
    lib = _load()
    head, ptr, atom = _arrays(rules)
    n = rules.n_atoms
    stage = np.zeros(max(n, 1), dtype=np.int32)
    secs = np.zeros(max(trials, 1), dtype=np.float64)
    iters = ctypes.c_int32(0)
    rc = lib.orc_lm_stage_timed(n, rules.n_rules, _p(head), _p(ptr), _p(atom), _p(_v0(rules, v0)),
                                _p(stage), ctypes.byref(iters), int(trials), _p(secs))
    if rc:
        raise MemoryError(rc)
    stage = stage[:n]
    return (stage >= 0).astype(np.uint8), stage, iters.value, secs[:trials].tolist()


def popcounts_from_stage(stage, iters):
    """|I_0| .. |I_{k*}| from the stage vector (I_k = {a : stage(a) <= k})."""
    s = np.asarray(stage)
    s = s[s >= 0]
    h = np.bincount(s, minlength=iters)[:iters] if s.size else np.zeros(iters, dtype=np.int64)
    return np.cumsum(h).tolist()


def negated_atoms(rules):
    if rules.body_neg is None:
        return []
    return sorted(set(rules.body_atom[rules.body_neg.astype(bool)].tolist()))


def stable(rules, guesses=None, want_models: bool = False):
    """O-STABLE (Algorithms 2-3 per column on P+).  ``guesses``: uint8[G][k] abar values
    (1 = a_j assumed false), or None for all 2^f guesses over the free negated atoms.
    Returns dict(accepted=uint8[G], kstar=int32[G], passes, k, f, negated, models)."""
    lib = _load()
    head, ptr, atom = _arrays(rules)
    n = rules.n_atoms
    neg = None if rules.body_neg is None else np.ascontiguousarray(rules.body_neg, dtype=np.uint8)
    negs = negated_atoms(rules)
    k = len(negs)
    facts = set(rules.head[np.diff(rules.body_ptr) == 0].tolist())
    f = sum(1 for a in negs if a not in facts)
    if guesses is None:
        G = 1 << f
        gz = None
    else:
        gz = np.ascontiguousarray(np.asarray(guesses, dtype=np.uint8).reshape(-1, k) if k else
                                  np.zeros((len(guesses), 0), dtype=np.uint8))
        G = gz.shape[0]
    acc = np.zeros(max(G, 1), dtype=np.uint8)
    kst = np.zeros(max(G, 1), dtype=np.int32)
    words = (n + 63) // 64
    models = np.zeros((max(G, 1), max(words, 1)), dtype=np.uint64) if want_models else None
    passes, ko, fo = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    rc = lib.orc_stable(n, rules.n_rules, _p(head), _p(ptr), _p(atom), _p(neg), G, _p(gz),
                        _p(acc), _p(kst), _p(models), ctypes.byref(passes),
                        ctypes.byref(ko), ctypes.byref(fo))
    if rc:
        raise RuntimeError(f"orc_stable rc={rc}")
    assert ko.value == k and fo.value == f
    return dict(accepted=acc[:G], kstar=kst[:G], passes=passes.value, k=k, f=f,
                negated=negs, models=None if models is None else models[:G, :words])


def certify(rules, v0, model, stage, iters) -> int:
    """O-CERT: 0 if (model, stage, iters) is the exact least model / stage / pass count."""
    _definite(rules)
    lib = _load()
    head, ptr, atom = _arrays(rules)
    m = np.ascontiguousarray(np.asarray(model, dtype=np.uint8))
    s = np.ascontiguousarray(np.asarray(stage, dtype=np.int32))
    return lib.orc_certify(rules.n_atoms, rules.n_rules, _p(head), _p(ptr), _p(atom),
                           _p(_v0(rules, v0)), _p(m), _p(s), int(iters))


def pack_bits(model_u8) -> np.ndarray:
    """uint8[n] 0/1 -> uint64[ceil(n/64)] LSB-first (atom a: word a>>6, bit a&63)."""
    m = np.asarray(model_u8, dtype=np.uint8)
    n = m.shape[0]
    words = (n + 63) // 64
    padded = np.zeros(words * 64, dtype=np.uint8)
    padded[:n] = m
    return np.packbits(padded, bitorder="little").view(np.uint64).copy()
