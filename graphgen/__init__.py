"""graphgen — seeded synthetic bipartite inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic (no counting, no peeling): it draws edges
and returns the two CSR views of the same edge set.  See graphgen/csrc/gen.c
for the recipe (SURVEY.md §8(d) reading R1) and
BASELINE.json `configs` for the five workloads.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "gen.c")
_LIB = os.path.join(_HERE, "libgraphgen.so")


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("nU", ctypes.c_uint32), ("nV", ctypes.c_uint32),
        ("m", ctypes.c_uint64),
        ("gammaU", ctypes.c_double), ("gammaV", ctypes.c_double),
        ("capU", ctypes.c_double), ("capV", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("nblocks", ctypes.c_uint32), ("bmin", ctypes.c_uint32),
        ("bmax", ctypes.c_uint32), ("noise_pct", ctypes.c_uint32),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        _lib.gen_build.restype = ctypes.c_void_p
        _lib.gen_build.argtypes = [ctypes.POINTER(_Params)]
        _lib.gen_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32),
                                  ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)]
        _lib.gen_fill.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 4
        _lib.gen_free.argtypes = [ctypes.c_void_p]
    return _lib


@dataclass
class Graph:
    """Bipartite graph as two CSRs over the same edge set.

    off_u[nU+1] (uint64), adj_u[m] (uint32 V ids, ascending per list);
    off_v[nV+1] (uint64), adj_v[m] (uint32 U ids, ascending per list).
    """
    nU: int
    nV: int
    off_u: np.ndarray
    adj_u: np.ndarray
    off_v: np.ndarray
    adj_v: np.ndarray
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.adj_u.shape[0])

    def swapped(self) -> "Graph":
        """The same graph with the roles of U and V exchanged (peel the other side)."""
        return Graph(self.nV, self.nU, self.off_v, self.adj_v, self.off_u, self.adj_u,
                     self.name + "^T")

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (np.array([self.nU, self.nV], np.uint64), self.off_u, self.adj_u, self.off_v, self.adj_v):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    def edges(self) -> np.ndarray:
        """(m, 2) array of (u, v) pairs in U-CSR order."""
        u = np.repeat(np.arange(self.nU, dtype=np.uint32), np.diff(self.off_u).astype(np.int64))
        return np.stack([u, self.adj_u], axis=1)

    def stats(self) -> dict:
        du = np.diff(self.off_u).astype(np.float64)
        dv = np.diff(self.off_v).astype(np.float64)
        e = self.edges()
        mins = np.minimum(du[e[:, 0]], dv[e[:, 1]]) if self.m else np.zeros(0)
        return {
            "nU": self.nU, "nV": self.nV, "m": self.m,
            "max_deg_u": int(du.max()) if self.nU else 0,
            "max_deg_v": int(dv.max()) if self.nV else 0,
            "sum_dv2": float((dv * dv).sum()), "sum_du2": float((du * du).sum()),
            "sum_min_deg": float(mins.sum()),
        }


def _run(p: _Params, name: str) -> Graph:
    lib = _load()
    h = lib.gen_build(ctypes.byref(p))
    if not h:
        raise RuntimeError(f"graphgen: generation failed for {name}")
    try:
        nU, nV, m = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint64()
        lib.gen_info(h, ctypes.byref(nU), ctypes.byref(nV), ctypes.byref(m))
        off_u = np.empty(nU.value + 1, np.uint64)
        off_v = np.empty(nV.value + 1, np.uint64)
        adj_u = np.empty(m.value, np.uint32)
        adj_v = np.empty(m.value, np.uint32)
        lib.gen_fill(h, off_u.ctypes.data, adj_u.ctypes.data, off_v.ctypes.data, adj_v.ctypes.data)
    finally:
        lib.gen_free(h)
    return Graph(nU.value, nV.value, off_u, adj_u, off_v, adj_v, name)


def uniform(nU: int, nV: int, m: int, seed: int) -> Graph:
    """First m distinct pairs of a uniform (u, v) stream (config 1 recipe, any size)."""
    return _run(_Params(kind=0, nU=nU, nV=nV, m=m, seed=seed), f"uniform({nU},{nV},{m},s{seed})")


def chung_lu(nU: int, nV: int, m: int, gammaU: float, gammaV: float, capU: float, capV: float,
             seed: int) -> Graph:
    """Chung-Lu power-law bipartite graph, reading R1."""
    return _run(_Params(kind=2, nU=nU, nV=nV, m=m, gammaU=gammaU, gammaV=gammaV, capU=capU,
                        capV=capV, seed=seed),
                f"chung_lu({nU},{nV},{m},{gammaU},{gammaV},s{seed})")


def blocks(nblocks: int, bmin: int, bmax: int, noise_pct: int, seed: int) -> Graph:
    """Disjoint union of K_{a,b} blocks (a, b ~ U{bmin..bmax}) plus noise_pct% cross-block edges."""
    return _run(_Params(kind=1, nblocks=nblocks, bmin=bmin, bmax=bmax, noise_pct=noise_pct, seed=seed),
                f"blocks({nblocks},{bmin}..{bmax},{noise_pct}%,s{seed})")


def block_sizes(nblocks: int, bmin: int, bmax: int, seed: int):
    """The (a_k, b_k) block shapes `blocks()` draws, recomputed here for closed-form tests.

    Mirrors gen.c's counter-based draw (streams 5 and 6) in Python integers.
    """
    M = (1 << 64) - 1

    def mix64(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def key(stream):
        return mix64(mix64((seed + 0x632BE59BD9B4E019) & M) ^ ((stream * 0xD1B54A32D192ED03) & M))

    def rnd(k, i):
        return mix64((k + (i + 1) * 0x9E3779B97F4A7C15) & M)

    span = bmax - bmin + 1
    kA, kB = key(5), key(6)
    return [(bmin + (((rnd(kA, k) >> 32) * span) >> 32), bmin + (((rnd(kB, k) >> 32) * span) >> 32))
            for k in range(nblocks)]


def from_edges(nU: int, nV: int, edges) -> Graph:
    """Graph from an explicit (u, v) edge list (deduplicated), for hand-written fixtures."""
    e = np.unique(np.asarray(edges, dtype=np.int64).reshape(-1, 2), axis=0)
    if e.size and (e[:, 0].max() >= nU or e[:, 1].max() >= nV or e.min() < 0):
        raise ValueError("edge endpoint out of range")
    order_u = np.lexsort((e[:, 1], e[:, 0]))
    order_v = np.lexsort((e[:, 0], e[:, 1]))
    off_u = np.zeros(nU + 1, np.uint64)
    off_v = np.zeros(nV + 1, np.uint64)
    np.add.at(off_u, e[:, 0] + 1, 1)
    np.add.at(off_v, e[:, 1] + 1, 1)
    return Graph(nU, nV, np.cumsum(off_u).astype(np.uint64), e[order_u, 1].astype(np.uint32),
                 np.cumsum(off_v).astype(np.uint64), e[order_v, 0].astype(np.uint32), "edges")


def complete(a: int, b: int) -> Graph:
    return from_edges(a, b, [(i, j) for i in range(a) for j in range(b)])


# BASELINE.json configs[0..4] → (generator, peel side rule, P).  Config 2a is the
# noise-free variant of config 2 used for the closed form.
CONFIGS = {
    1: dict(fn=lambda: uniform(2000, 1000, 20000, seed=1), P=8, side="U"),
    2: dict(fn=lambda: blocks(200, 5, 60, 5, seed=2), P=32, side="U"),
    "2a": dict(fn=lambda: blocks(200, 5, 60, 0, seed=2), P=32, side="U"),
    3: dict(fn=lambda: chung_lu(500_000, 200_000, 5_000_000, 2.1, 2.1, 50_000, 50_000, seed=3),
            P=150, side="U"),
    4: dict(fn=lambda: chung_lu(3_000_000, 8_000_000, 30_000_000, 2.3, 1.9, 300_000, 300_000, seed=4),
            P=150, side="cheaper"),
    5: dict(fn=lambda: chung_lu(25_000_000, 30_000_000, 300_000_000, 2.0, 1.8, 1_000_000, 1_000_000,
                                seed=5), P=400, side="U"),
}


def peel_side_cheaper(g: Graph) -> str:
    """Config 4 rule: peel U iff Σ_{v∈V} C(d_v,2) ≤ Σ_{u∈U} C(d_u,2) (cost of peeling each side)."""
    dv = np.diff(g.off_v).astype(np.float64)
    du = np.diff(g.off_u).astype(np.float64)
    cost_u = float((dv * (dv - 1) / 2).sum())
    cost_v = float((du * (du - 1) / 2).sum())
    return "U" if cost_u <= cost_v else "V"


GENERATOR_VERSION = "r1"  # bump when any generator changes (names the on-disk cache)


def config(cfg, cache_dir: str | None = None) -> tuple[Graph, int]:
    """Build BASELINE config `cfg`; returns (graph oriented so that U is the peel side, P)."""
    spec = CONFIGS[cfg]
    g = None
    path = None
    if cache_dir:
        path = os.path.join(cache_dir, f"cfg{cfg}.npz")
        if os.path.exists(path):
            z = np.load(path)
            g = Graph(int(z["nU"]), int(z["nV"]), z["off_u"], z["adj_u"], z["off_v"], z["adj_v"], f"cfg{cfg}")
    if g is None:
        g = spec["fn"]()
        g.name = f"cfg{cfg}"
        if path:
            os.makedirs(cache_dir, exist_ok=True)
            tmp = path[:-4] + f".tmp{os.getpid()}.npz"  # complete file or none
            np.savez(tmp, nU=g.nU, nV=g.nV, off_u=g.off_u, adj_u=g.adj_u, off_v=g.off_v, adj_v=g.adj_v)
            os.replace(tmp, path)
    side = spec["side"]
    if side == "cheaper":
        side = peel_side_cheaper(g)
    if side == "V":
        g = g.swapped()
    return g, spec["P"]


__all__ = ["GENERATOR_VERSION", "Graph", "uniform", "chung_lu", "blocks", "block_sizes", "from_edges", "complete", "config",
           "CONFIGS", "peel_side_cheaper", "build_lib"]
