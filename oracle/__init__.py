"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain CPU reference for PBNG tip decomposition (arXiv 2110.12511), written from
the paper.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import it.  It shares no code with the CUDA path
(paper_2110_12511_b200/) and imports nothing from it.

  count(g)            -> uint64 support per u    (oracle.c: oracle_count)
  count_subset(g, us) -> uint64 support per listed u
  bup_tip(g)          -> uint64 tip number per u (oracle.c: oracle_bup_tip)
  edge_count(g)       -> uint64 butterflies per edge, U-side CSR order
                         (oracle.c: oracle_edge_count)
  bup_wing(g)         -> uint64 wing number per edge, U-side CSR order
                         (oracle.c: oracle_bup_wing, Alg.2)
  tip_level(g, θ, k)  -> (uint32 k-tip label per u, number of k-tips)
                         (oracle.c: oracle_tip_level)
  brute.*             pure-Python brute force and Definition-2 tip numbers for
                      tiny graphs (oracle/brute.py)

Parity status: count and bup_tip are pinned by tests/test_oracle.py (brute-force
4-tuple enumeration, K_{a,b} closed form, Σ_U = Σ_V identity, Definition-2 tip
numbers, golden graphs); edge_count by 4-tuple enumeration, the K_{a,b} closed
form (a-1)(b-1), the transposed-graph traversal edge by edge, Σ_e = 4·#butterflies,
Σ_{e∋u} = 2·⋈_u and hand-derived goldens (tests/golden/edge_counts.txt).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


_CERT = os.path.join(_HERE, "certificate.c")


def build_lib(force: bool = False) -> str:
    srcs = [_SRC, _CERT]
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(p) for p in srcs):
        # -fopenmp serves certificate.c only; oracle.c stays single-threaded
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB] + srcs)
    return _LIB


class Stats(ctypes.Structure):
    _fields_ = [("wedges", ctypes.c_uint64), ("updates", ctypes.c_uint64), ("peeled", ctypes.c_uint64)]

    def as_dict(self):
        return {"wedges": self.wedges, "updates": self.updates, "peeled": self.peeled}


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        base = [ctypes.c_uint32, ctypes.c_uint32] + [ctypes.c_void_p] * 4
        _lib.oracle_count.argtypes = base + [ctypes.c_void_p, ctypes.POINTER(Stats)]
        _lib.oracle_count_subset.argtypes = base + [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                                    ctypes.POINTER(Stats)]
        _lib.oracle_bup_tip.argtypes = base + [ctypes.c_void_p, ctypes.POINTER(Stats)]
        _lib.oracle_edge_count.argtypes = base + [ctypes.c_void_p, ctypes.POINTER(Stats)]
        _lib.oracle_bup_wing.argtypes = base + [ctypes.c_void_p, ctypes.POINTER(Stats)]
        for f in (_lib.oracle_count, _lib.oracle_count_subset, _lib.oracle_bup_tip, _lib.oracle_edge_count,
                  _lib.oracle_bup_wing):
            f.restype = ctypes.c_int
        _lib.oracle_tip_level.argtypes = base + [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        _lib.oracle_tip_level.restype = ctypes.c_int64
        _lib.oracle_cert_support_ge.argtypes = base + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                                       ctypes.c_void_p]
        _lib.oracle_cert_support_ge.restype = ctypes.c_int
        _lib.oracle_cert_levels.argtypes = base + [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_void_p]
        _lib.oracle_cert_levels.restype = ctypes.c_int64
        _lib.oracle_cert_sort_lists.argtypes = [ctypes.c_uint32] + [ctypes.c_void_p] * 4
        _lib.oracle_cert_sort_lists.restype = ctypes.c_int
        _lib.oracle_cert_pass.argtypes = base + [ctypes.c_void_p] * 4
        _lib.oracle_cert_pass.restype = ctypes.c_int
        _lib.oracle_cert_levels_induced.argtypes = base + [ctypes.c_void_p] * 5 + [ctypes.c_uint64, ctypes.c_void_p]
        _lib.oracle_cert_levels_induced.restype = ctypes.c_int64
    return _lib


def _csr(g):
    arrs = [np.ascontiguousarray(g.off_u, np.uint64), np.ascontiguousarray(g.adj_u, np.uint32),
            np.ascontiguousarray(g.off_v, np.uint64), np.ascontiguousarray(g.adj_v, np.uint32)]
    return arrs, [a.ctypes.data for a in arrs]


def count(g, stats: Stats | None = None) -> np.ndarray:
    """Butterfly support of every u in U (one-sided wedge aggregation)."""
    keep, ptrs = _csr(g)
    out = np.zeros(g.nU, np.uint64)
    st = stats if stats is not None else Stats()
    if _load().oracle_count(g.nU, g.nV, *ptrs, out.ctypes.data, ctypes.byref(st)):
        raise MemoryError("oracle_count failed")
    del keep
    return out


def count_subset(g, us, stats: Stats | None = None) -> np.ndarray:
    """Butterfly support of the listed u only (same traversal as count)."""
    keep, ptrs = _csr(g)
    us = np.ascontiguousarray(us, np.uint32)
    out = np.zeros(us.shape[0], np.uint64)
    st = stats if stats is not None else Stats()
    if _load().oracle_count_subset(g.nU, g.nV, *ptrs, us.ctypes.data, us.shape[0], out.ctypes.data,
                                   ctypes.byref(st)):
        raise MemoryError("oracle_count_subset failed")
    del keep
    return out


def edge_count(g, stats: Stats | None = None) -> np.ndarray:
    """Per-edge butterfly count ⋈_e (Alg.1 per-edge output P:398),
    indexed by the edge's position in the U-side CSR (g.adj_u): the plain definition
    Σ_{u' ∈ N_v, u' ≠ u} (w(u,u') − 1) for e = (u, v)."""
    keep, ptrs = _csr(g)
    out = np.zeros(g.m, np.uint64)
    st = stats if stats is not None else Stats()
    if _load().oracle_edge_count(g.nU, g.nV, *ptrs, out.ctypes.data, ctypes.byref(st)):
        raise MemoryError("oracle_edge_count failed")
    del keep
    return out


def bup_wing(g, stats: Stats | None = None) -> np.ndarray:
    """Wing number of every edge (U-side CSR order) by sequential bottom-up edge
    peeling, Alg.2 as written."""
    keep, ptrs = _csr(g)
    out = np.zeros(g.m, np.uint64)
    st = stats if stats is not None else Stats()
    if _load().oracle_bup_wing(g.nU, g.nV, *ptrs, out.ctypes.data, ctypes.byref(st)):
        raise MemoryError("oracle_bup_wing failed")
    del keep
    return out


def bup_tip(g, stats: Stats | None = None) -> np.ndarray:
    """Tip number of every u in U by sequential bottom-up peeling."""
    keep, ptrs = _csr(g)
    out = np.zeros(g.nU, np.uint64)
    st = stats if stats is not None else Stats()
    if _load().oracle_bup_tip(g.nU, g.nV, *ptrs, out.ctypes.data, ctypes.byref(st)):
        raise MemoryError("oracle_bup_tip failed")
    del keep
    return out


def tip_level(g, theta, k: int):
    """k-tips of level k (Def. 2; retrieval from θ):
    (label per u = smallest id of its k-tip or 0xFFFFFFFF when θ_u < k, number of k-tips)."""
    keep, ptrs = _csr(g)
    th = np.ascontiguousarray(theta, np.uint64)
    out = np.zeros(g.nU, np.uint32)
    n = _load().oracle_tip_level(g.nU, g.nV, *ptrs, th.ctypes.data, int(k), out.ctypes.data)
    if n < 0:
        raise MemoryError("oracle_tip_level failed")
    del keep
    return out, int(n)


def cert_support_ge(g, theta, us=None) -> np.ndarray:
    """Certificate part (A): s_ge(u) = Σ_{u' != u, θ'_u' >= θ'_u} C(w,2) for the listed u (all if None)."""
    keep, ptrs = _csr(g)
    th = np.ascontiguousarray(theta, np.uint64)
    usa = None if us is None else np.ascontiguousarray(us, np.uint32)
    n = g.nU if usa is None else usa.shape[0]
    out = np.zeros(n, np.uint64)
    if _load().oracle_cert_support_ge(g.nU, g.nV, *ptrs, th.ctypes.data, None if usa is None else usa.ctypes.data,
                                      n, out.ctypes.data):
        raise MemoryError("oracle_cert_support_ge failed")
    del keep
    return out


def cert_levels(g, theta, levels=None):
    """Certificate part (C) for the given levels (all distinct θ' values if None).
    Returns (number of failing levels, first failing level or None)."""
    keep, ptrs = _csr(g)
    th = np.ascontiguousarray(theta, np.uint64)
    order = np.argsort(th, kind="stable").astype(np.uint32)
    vals = th[order]
    uniq, starts = np.unique(vals, return_index=True)
    ends = np.append(starts[1:], len(vals))
    if levels is not None:
        want = np.isin(uniq, np.asarray(levels, np.uint64))
        uniq, starts, ends = uniq[want], starts[want], ends[want]
    members = np.concatenate([order[a:b] for a, b in zip(starts, ends)]) if len(uniq) else np.zeros(0, np.uint32)
    members = np.ascontiguousarray(members, np.uint32)
    off = np.zeros(len(uniq) + 1, np.uint64)
    off[1:] = np.cumsum(ends - starts)
    lev = np.ascontiguousarray(uniq, np.uint64)
    first = ctypes.c_uint64(0)
    bad = _load().oracle_cert_levels(g.nU, g.nV, *ptrs, th.ctypes.data, lev.ctypes.data, off.ctypes.data,
                                     members.ctypes.data if len(members) else None, len(lev), ctypes.byref(first))
    if bad < 0:
        raise MemoryError("oracle_cert_levels failed")
    del keep
    return int(bad), (int(lev[first.value]) if bad else None)


def _levels(th):
    """Distinct θ' values with their members (ascending id within a level)."""
    order = np.argsort(th, kind="stable").astype(np.uint32)
    vals = th[order]
    uniq, starts = np.unique(vals, return_index=True)
    off = np.append(starts, len(vals)).astype(np.uint64)
    return np.ascontiguousarray(uniq, np.uint64), off, np.ascontiguousarray(order, np.uint32)


def cert_one_pass(g, theta, progress=None):
    """One-pass certificate (certificate.c, oracle_cert_pass + oracle_cert_levels_induced):
    returns (support, s_ge, number of failing (C) levels, first failing level or None).
    `support` equals count(g) and `s_ge` equals cert_support_ge(g, θ') (each unordered
    pair walked once from its smaller (θ', id) end); `progress` = optional uint64
    numpy array of one element, incremented per finished vertex (for long runs)."""
    keep, ptrs = _csr(g)
    lib = _load()
    th = np.ascontiguousarray(theta, np.uint64)
    adj_s = np.empty(g.m, np.uint32)
    lib.oracle_cert_sort_lists(g.nV, ptrs[2], ptrs[3], th.ctypes.data, adj_s.ctypes.data)
    sup = np.zeros(g.nU, np.uint64)
    sge = np.zeros(g.nU, np.uint64)
    ptrs_s = [ptrs[0], ptrs[1], ptrs[2], adj_s.ctypes.data]
    if lib.oracle_cert_pass(g.nU, g.nV, *ptrs_s, th.ctypes.data, sup.ctypes.data, sge.ctypes.data,
                            None if progress is None else progress.ctypes.data):
        raise MemoryError("oracle_cert_pass failed")
    lev, off, mem = _levels(th)
    first = ctypes.c_uint64(0)
    bad = lib.oracle_cert_levels_induced(g.nU, g.nV, *ptrs_s, th.ctypes.data, sge.ctypes.data, lev.ctypes.data,
                                         off.ctypes.data, mem.ctypes.data if len(mem) else None, len(lev),
                                         ctypes.byref(first))
    if bad < 0:
        raise MemoryError("oracle_cert_levels_induced failed")
    del keep
    return sup, sge, int(bad), (int(lev[first.value]) if bad else None)


def certify_one_pass(g, theta) -> bool:
    """certify() by the one-pass certificate: (A) s_ge >= θ' and (C) on every level."""
    th = np.ascontiguousarray(theta, np.uint64)
    _, sge, bad, _ = cert_one_pass(g, th)
    return bool(np.all(sge >= th)) and bad == 0


def certify(g, theta) -> bool:
    """Full exactness certificate: (A) for every u and (C) for every level."""
    th = np.ascontiguousarray(theta, np.uint64)
    if not np.all(cert_support_ge(g, th) >= th):
        return False
    return cert_levels(g, th)[0] == 0
