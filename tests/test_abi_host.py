"""C-ABI checks that need no GPU: the library loads and exports every symbol declared
in include/lp.h; the host standardizer/encoder (host-only handle, device = -1) reports
the paper's shapes and rejects invalid input with the documented status codes."""
import os
import re
import subprocess

import numpy as np
import pytest

import lpgen
from paper_2009_10247_b200 import lp

from golden_io import load, parse_rules, to_rules

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "lp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lp_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    declared = _declared_symbols()
    assert set(declared) >= {"lp_load", "lp_least_model", "lp_stable_models"}
    out = subprocess.check_output(["nm", "-D", "--defined-only", lp.LIB_PATH]).decode()
    exported = set(re.findall(r"\b(lp_\w+)\b", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    lib = lp.library()
    for s in declared:
        assert hasattr(lib, s)
    assert set(lp.SYMBOLS) == set(declared)


def _host(rules, **kw):
    return lp.Program(rules, device=-1, allocator="none", **kw)


def test_example1_shapes():
    g = load("example1.txt")
    names = g["atoms"][0].split()
    P = to_rules(parse_rules(g["program"], names), len(names))
    p = _host(P)
    i = p.info
    assert i["n_atoms"] == 5 and i["n_rules"] == 6
    # AND-rows: p<-q,r (2) p<-s,t (2) r<-s (1) q<-t (1) s<-⊤ (1) t<-⊤ (1)
    assert i["nnz"] == 8 and i["max_body"] == 2 and i["n_segments"] == 2
    assert i["n_heads"] == 5 and i["n_negated"] == 0
    # n' of the standardized program P': 5 atoms + aux u, v
    assert i["n_prime_paper"] == 7
    assert abs(i["sparsity_eq5"] - (1 - 6 / 25)) < 1e-12
    with pytest.raises(lp.LPError) as e:
        p.least_model()
    assert e.value.status == lp.LP_E_NODEVICE
    p.close()


def test_example2_negation_shapes():
    g = load("example2.txt")
    names = g["atoms"][0].split()
    P = to_rules(parse_rules(g["program"], names), len(names))
    p = _host(P)
    assert p.info["n_negated"] == 1 and p.info["n_free_negated"] == 0
    assert p.negated_atoms() == [names.index("t")]
    assert p.info["n_prime_paper"] == 7          # p q s t u v t̄


def test_dedupe_and_facts():
    # duplicate body atoms are removed, duplicate rules kept, facts point at ⊤
    P = lpgen.from_lists(3, [(0, [1, 1, 2, 1]), (0, [1, 1, 2, 1]), (1, []), (2, [])])
    p = _host(P)
    assert p.info["nnz"] == 2 + 2 + 1 + 1 and p.info["max_body"] == 2


@pytest.mark.parametrize("bad", ["head", "atom", "ptr0", "ptrdec", "neg_n"])
def test_invalid_inputs(bad):
    P = lpgen.from_lists(4, [(0, [1, 2]), (1, [3]), (3, [])])
    if bad == "head":
        P.head[1] = 4
    elif bad == "atom":
        P.body_atom[0] = -1
    elif bad == "ptr0":
        P.body_ptr = P.body_ptr + 1
    elif bad == "ptrdec":
        P.body_ptr[1], P.body_ptr[2] = P.body_ptr[2], P.body_ptr[1]
    elif bad == "neg_n":
        P.n_atoms = -1
    with pytest.raises(lp.LPError) as e:
        _host(P)
    assert e.value.status == lp.LP_E_INVALID


def test_large_body_and_empty_program():
    P = lpgen.from_lists(1000, [(0, list(range(1, 1000)))])
    assert _host(P).info["max_body"] == 999
    E = lpgen.from_lists(0, [])
    i = _host(E).info
    assert i["n_atoms"] == 0 and i["nnz"] == 0 and i["n_segments"] == 0


def test_c5_host_encode():
    C = lpgen.gen_c5(1)
    p = _host(C)
    i = p.info
    assert i["n_negated"] == 12 and i["n_free_negated"] == 12
    assert p.negated_atoms() == C.meta["negated_atoms"]
    assert i["nnz"] == C.nnz + 1000          # + ⊤ for every fact


def test_paper_layout_host_shapes():
    """LP_LOAD_PAPER_LAYOUT: the standardized program P^δ has one auxiliary
    atom per rule of every multi-rule head (oracle/paper.py standardize) and the caller
    still sees the original atoms."""
    from oracle import paper
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = int(rng.integers(1, 50))
        P = lpgen.random_program(rng, n, int(rng.integers(0, 5 * n)), max_len=4)
        m, _ = paper.standardize(P)
        info = _host(P, paper_layout=True).info
        assert info["n_atoms"] == n and info["n_aux"] == m - n
        assert _host(P).info["n_aux"] == 0


def test_load_shim_from_flat_arrays():
    """SURVEY §8(b)'s Python shim: lp.load(head, body_ptr, body_atom, body_neg)."""
    P = lpgen.config("C1")
    a = lp.load(P.head, P.body_ptr, P.body_atom, device=-1, allocator="none")
    b = _host(P)
    for key in ("n_atoms", "n_rules", "nnz", "n_heads", "max_body", "n_segments"):
        assert a.info[key] == b.info[key]


def test_unknown_load_flag_rejected():
    """Flag bit 0x2 (the removed TMA ring) and any unknown bit fail with LP_E_INVALID."""
    import ctypes
    P = lpgen.from_lists(3, [(0, [1]), (1, [])])
    head = np.ascontiguousarray(P.head, dtype=np.int32)
    ptr = np.ascontiguousarray(P.body_ptr, dtype=np.int64)
    atom = np.ascontiguousarray(P.body_atom, dtype=np.int32)
    r = lp.lp_rules(3, head.shape[0], head.ctypes.data, ptr.ctypes.data, atom.ctypes.data, None)
    for bad in (0x2, 0x100):
        opt = lp.lp_options()
        opt.device = -1
        opt.flags = bad
        h = ctypes.c_void_p()
        st = lp.library().lp_load(ctypes.byref(r), ctypes.byref(opt), ctypes.byref(h))
        assert st == lp.LP_E_INVALID and not h.value


def test_lp_run_layout_matches_header():
    """The ctypes mirror of lp_run / lp_info_t has the fields include/lp.h declares, in order."""
    src = open(os.path.join(ROOT, "include", "lp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    for struct, cls in (("lp_run", lp.lp_run), ("lp_info_t", lp.lp_info_t)):
        body = re.search(r"typedef struct \{([^}]*)\}\s*" + struct + ";", src).group(1)
        names = re.findall(r"\b(\w+)\s*;", body)
        assert names == [f for f, _ in cls._fields_], (struct, names)
