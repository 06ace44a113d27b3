"""paper_2110_12511_b200 — B200-native PBNG tip decomposition (arXiv 2110.12511).

Thin ctypes binding over libpbng.so (C ABI declared in include/pbng.h).  This
module only marshals arguments: every step of counting, CD and FD runs in the
library's sm_100a CUDA kernels.  PyTorch provides device memory and streams.
There is no CPU fallback: if libpbng.so is missing or no CUDA device is present,
calls raise.

Entry points (same names as the C ABI):
  pbng_count_butterflies(g, side=0)            -> torch.int64 [n]   (uint64 bits)
  pbng_tip_decompose(g, P, side=0, opts=0)     -> (torch.int64 [n], stats dict)
  pbng_tip_plan(g, P, side=0, opts=0)          -> (part, init, bounds, nparts)
  pbng_tip_decompose_host(off_u, adj_u, off_v, adj_v, P, side=0, opts=0)
                                               -> (numpy.uint64 [n], stats dict)
`g` is a DeviceGraph (CSR tensors on a CUDA device).  uint64 results are
returned in int64 tensors holding the same bits (values here stay < 2^63).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBNG_LIB") or os.path.join(_HERE, "libpbng.so")

OK, ERR_ARG, ERR_GRAPH, ERR_OOM, ERR_CUDA = 0, 1, 2, 3, 4
OPT_NO_RECOUNT, OPT_NO_DELETE, OPT_VALIDATE, OPT_STATS, OPT_FORCE_RECOUNT, OPT_ONESIDED_COUNT = 1, 2, 4, 8, 16, 32
OPT_FD_GRID, OPT_STATS_DEFER = 64, 128
MAX_P = 4096
KERNEL_FAMILIES = ("init", "classify", "agg_warp", "agg_cta", "agg_hash", "select", "range", "compact",
                   "fd_build", "fd", "count_vp")
EXPORTS = ("pbng_count_butterflies", "pbng_count_edge_butterflies", "pbng_be_index", "pbng_wing_decompose", "pbng_tip_decompose", "pbng_tip_decompose_host", "pbng_tip_plan",
           "pbng_tip_components", "pbng_kernel_times", "pbng_release_memory", "pbng_last_error", "pbng_version")


class PbngError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pbng error {code}: {msg}")
        self.code = code


class Csr(ctypes.Structure):
    _fields_ = [("offsets", ctypes.c_void_p), ("indices", ctypes.c_void_p),
                ("n", ctypes.c_uint32), ("m", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("wedges_count", ctypes.c_uint64), ("wedges_cd", ctypes.c_uint64),
                ("wedges_fd", ctypes.c_uint64), ("support_updates", ctypes.c_uint64),
                ("rho_cd_iters", ctypes.c_uint32), ("recounts", ctypes.c_uint32),
                ("partitions_used", ctypes.c_uint32), ("fd_rounds_max", ctypes.c_uint32),
                ("ms_count", ctypes.c_float), ("ms_cd", ctypes.c_float),
                ("ms_fd_build", ctypes.c_float), ("ms_fd", ctypes.c_float),
                ("uv_steps", ctypes.c_uint64), ("uv_steps_fd", ctypes.c_uint64), ("updates_fd", ctypes.c_uint64),
                ("launches", ctypes.c_uint32), ("pad", ctypes.c_uint32), ("impl", ctypes.c_uint64 * 4),
                ("ms_kernel", ctypes.c_float * 16), ("impl_hash", ctypes.c_uint64 * 4)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("pad", "ms_kernel", "impl", "impl_hash")}
        d["impl"] = list(self.impl)
        d["impl_hash"] = list(self.impl_hash)
        d["ms_kernel"] = {name: round(float(self.ms_kernel[i]), 4) for i, name in enumerate(KERNEL_FAMILIES)
                          if self.ms_kernel[i]}
        return d


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpbng.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        lib.pbng_count_butterflies.argtypes = [Csr, Csr, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        lib.pbng_count_edge_butterflies.argtypes = [Csr, Csr, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_void_p]
        lib.pbng_be_index.argtypes = [Csr, Csr] + [ctypes.c_void_p] * 6
        lib.pbng_wing_decompose.argtypes = [Csr, Csr, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.pbng_tip_decompose.argtypes = [Csr, Csr, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p,
                                           ctypes.c_uint32, ctypes.POINTER(Stats), ctypes.c_void_p]
        lib.pbng_tip_decompose_host.argtypes = lib.pbng_tip_decompose.argtypes
        lib.pbng_tip_plan.argtypes = [Csr, Csr, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.pbng_tip_components.argtypes = [Csr, Csr, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        for f in ("pbng_count_butterflies", "pbng_tip_decompose", "pbng_tip_decompose_host", "pbng_tip_plan",
                  "pbng_tip_components", "pbng_count_edge_butterflies", "pbng_be_index", "pbng_wing_decompose"):
            getattr(lib, f).restype = ctypes.c_int
        lib.pbng_kernel_times.argtypes = [ctypes.c_void_p]
        lib.pbng_kernel_times.restype = ctypes.c_int
        if hasattr(lib, "pbng_release_memory"):  # (older tuning builds lack it)
            lib.pbng_release_memory.argtypes = []
            lib.pbng_release_memory.restype = ctypes.c_int
        lib.pbng_last_error.restype = ctypes.c_char_p
        lib.pbng_last_error.argtypes = []
        lib.pbng_version.restype = ctypes.c_char_p
        lib.pbng_version.argtypes = []
        _lib = lib
    return _lib


def _check(rc: int):
    if rc != OK:
        raise PbngError(rc, load_library().pbng_last_error().decode())


def _torch():
    import torch
    return torch


@dataclass
class DeviceGraph:
    """Two CSRs of one bipartite edge set, resident on a CUDA device.

    off_u int64[nU+1], adj_u int32[m] (V ids), off_v int64[nV+1], adj_v int32[m] (U ids);
    the int tensors carry the uint64 / uint32 bit patterns the C ABI expects."""
    nU: int
    nV: int
    off_u: object
    adj_u: object
    off_v: object
    adj_v: object

    @property
    def m(self) -> int:
        return int(self.adj_u.numel())

    @staticmethod
    def from_numpy(off_u, adj_u, off_v, adj_v, device="cuda") -> "DeviceGraph":
        torch = _torch()

        def t(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(device)

        return DeviceGraph(len(off_u) - 1, len(off_v) - 1, t(off_u, np.int64), t(adj_u, np.int32),
                           t(off_v, np.int64), t(adj_v, np.int32))

    def csrs(self):
        return (Csr(self.off_u.data_ptr(), self.adj_u.data_ptr() if self.m else None, self.nU, self.m),
                Csr(self.off_v.data_ptr(), self.adj_v.data_ptr() if self.m else None, self.nV, self.m))


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _n_peel(g, side):
    return g.nU if side == 0 else g.nV


def pbng_count_butterflies(g: DeviceGraph, side: int = 0, out=None, stream=None):
    """Per-vertex butterfly counts of the peel side (uint64 bits in an int64 tensor)."""
    torch = _torch()
    n = _n_peel(g, side)
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=g.off_u.device)
    U, V = g.csrs()
    _check(load_library().pbng_count_butterflies(U, V, side, ctypes.c_void_p(out.data_ptr() if n else None),
                                                 _stream_ptr(stream)))
    return out


def pbng_count_edge_butterflies(g: DeviceGraph, side: int = 0, out=None, stream=None):
    """Per-edge butterfly counts in the CSR order of `side` (0: g.adj_u positions, 1: g.adj_v);
    returns (int64 tensor of uint64 bits, info dict: Alg.1 wedges expanded, starts per tier)."""
    torch = _torch()
    m = int(g.m)
    if out is None:
        out = torch.empty(m, dtype=torch.int64, device=g.off_u.device)
    info = (ctypes.c_uint64 * 4)()
    U, V = g.csrs()
    _check(load_library().pbng_count_edge_butterflies(U, V, side, ctypes.c_void_p(out.data_ptr() if m else None),
                                                      info, _stream_ptr(stream)))
    return out, {"wedges": int(info[0]), "tiers": [int(x) for x in info[1:]]}


def pbng_be_index(g: DeviceGraph, stream=None):
    """BE-Index: dict of numpy arrays bloom_off (uint64), bloom_k (uint32), dom (uint32 [nb,2],
    bit 31 of dom[:,0] = dominant set in V), pairs (uint32 [np,2], positions in g.adj_u)."""
    torch = _torch()
    sizes = (ctypes.c_uint64 * 2)()
    U, V = g.csrs()
    lib = load_library()
    _check(lib.pbng_be_index(U, V, sizes, None, None, None, None, _stream_ptr(stream)))
    nb, np_ = int(sizes[0]), int(sizes[1])
    dv = g.off_u.device
    off = torch.empty(nb + 1, dtype=torch.int64, device=dv)
    k = torch.empty(max(nb, 1), dtype=torch.int32, device=dv)
    dom = torch.empty(max(2 * nb, 1), dtype=torch.int32, device=dv)
    pairs = torch.empty(max(2 * np_, 1), dtype=torch.int32, device=dv)
    _check(lib.pbng_be_index(U, V, sizes, ctypes.c_void_p(off.data_ptr()), ctypes.c_void_p(k.data_ptr()),
                             ctypes.c_void_p(dom.data_ptr()), ctypes.c_void_p(pairs.data_ptr()), _stream_ptr(stream)))
    assert int(sizes[0]) == nb and int(sizes[1]) == np_
    u32 = lambda t, n: t[:n].cpu().numpy().view(np.uint32)  # noqa: E731
    return {"bloom_off": off.cpu().numpy().view(np.uint64), "bloom_k": u32(k, nb),
            "dom": u32(dom, 2 * nb).reshape(nb, 2), "pairs": u32(pairs, 2 * np_).reshape(np_, 2)}


def pbng_wing_decompose(g: DeviceGraph, side: int = 0, out=None, stream=None):
    """Wing numbers per edge in the CSR order of `side`; returns (int64 tensor of uint64 bits, info)."""
    torch = _torch()
    m = int(g.m)
    if out is None:
        out = torch.empty(m, dtype=torch.int64, device=g.off_u.device)
    info = (ctypes.c_uint64 * 4)()
    U, V = g.csrs()
    _check(load_library().pbng_wing_decompose(U, V, side, ctypes.c_void_p(out.data_ptr() if m else None), info,
                                              _stream_ptr(stream)))
    return out, {"blooms": int(info[0]), "pairs": int(info[1]), "levels": int(info[2]), "rounds": int(info[3])}


def pbng_tip_decompose(g: DeviceGraph, P: int, side: int = 0, opts: int = 0, out=None, stream=None):
    """Tip numbers of the peel side; returns (int64 tensor of uint64 bits, stats dict)."""
    torch = _torch()
    n = _n_peel(g, side)
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=g.off_u.device)
    st = Stats()
    U, V = g.csrs()
    _check(load_library().pbng_tip_decompose(U, V, side, P, ctypes.c_void_p(out.data_ptr() if n else None),
                                             opts, ctypes.byref(st), _stream_ptr(stream)))
    return out, st.as_dict()


def pbng_tip_plan(g: DeviceGraph, P: int, side: int = 0, opts: int = 0, stream=None):
    """CD only: (part int32[n], init int64[n] uint64 bits, bounds numpy.uint64[P+1], nparts)."""
    torch = _torch()
    n = _n_peel(g, side)
    part = torch.empty(n, dtype=torch.int32, device=g.off_u.device)
    init = torch.empty(n, dtype=torch.int64, device=g.off_u.device)
    bounds = np.zeros(P + 1, np.uint64)
    nparts = ctypes.c_uint32(0)
    U, V = g.csrs()
    _check(load_library().pbng_tip_plan(U, V, side, P, opts, ctypes.c_void_p(part.data_ptr() if n else None),
                                        ctypes.c_void_p(init.data_ptr() if n else None),
                                        bounds.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nparts),
                                        _stream_ptr(stream)))
    return part, init, bounds, int(nparts.value)


def pbng_tip_decompose_host(off_u, adj_u, off_v, adj_v, P: int, side: int = 0, opts: int = 0, out=None,
                            stream=None):
    """Host-buffer entry point: numpy (ideally pinned) CSR arrays in, numpy uint64 tip numbers out.
    All host<->device copies happen inside the library call."""
    arrs = [np.ascontiguousarray(off_u, np.uint64), np.ascontiguousarray(adj_u, np.uint32),
            np.ascontiguousarray(off_v, np.uint64), np.ascontiguousarray(adj_v, np.uint32)]
    nU, nV, m = len(arrs[0]) - 1, len(arrs[2]) - 1, len(arrs[1])
    n = nU if side == 0 else nV
    if out is None:
        out = np.empty(n, np.uint64)
    st = Stats()
    U = Csr(arrs[0].ctypes.data, arrs[1].ctypes.data if m else None, nU, m)
    V = Csr(arrs[2].ctypes.data, arrs[3].ctypes.data if m else None, nV, m)
    _check(load_library().pbng_tip_decompose_host(U, V, side, P, ctypes.c_void_p(out.ctypes.data if n else None),
                                                  opts, ctypes.byref(st), _stream_ptr(stream)))
    return out, st.as_dict()


def pbng_tip_components(g: DeviceGraph, tip, k: int, side: int = 0, out=None, stream=None):
    """k-tips of level k from tip numbers `tip` (device int64 tensor of uint64 bits):
    (int32 tensor of uint32 labels — smallest member id, 0xFFFFFFFF outside the level —, count)."""
    torch = _torch()
    n = _n_peel(g, side)
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=g.off_u.device)
    ncomp = ctypes.c_uint32(0)
    U, V = g.csrs()
    _check(load_library().pbng_tip_components(U, V, side, ctypes.c_void_p(tip.data_ptr() if n else None),
                                              int(k), ctypes.c_void_p(out.data_ptr() if n else None),
                                              ctypes.byref(ncomp), _stream_ptr(stream)))
    return out, int(ncomp.value)


def pbng_kernel_times() -> dict:
    """Device ms per kernel family of the last call made with OPT_STATS_DEFER."""
    out = (ctypes.c_float * 16)()
    _check(load_library().pbng_kernel_times(ctypes.cast(out, ctypes.c_void_p)))
    return {name: round(float(out[i]), 4) for i, name in enumerate(KERNEL_FAMILIES) if out[i]}


def pbng_release_memory() -> None:
    """Return the library's cached scratch (private per-device pools) to the driver."""
    _check(load_library().pbng_release_memory())


def as_u64(t) -> np.ndarray:
    """Device int64 tensor of uint64 bits -> numpy uint64."""
    return t.cpu().numpy().view(np.uint64)


kernel_times = pbng_kernel_times
count_butterflies = pbng_count_butterflies
tip_decompose = pbng_tip_decompose
tip_plan = pbng_tip_plan
tip_decompose_host = pbng_tip_decompose_host
tip_components = pbng_tip_components
count_edge_butterflies = pbng_count_edge_butterflies
be_index = pbng_be_index
wing_decompose = pbng_wing_decompose
