"""GPU parity of the BE-Index and of wing decomposition
(§8(f) f4; wing numbers P:465-468) through the C ABI.

Wing numbers are unique: bit-exact against oracle.bup_wing (Alg.2 BUP, pinned by
Definition 1 in test_oracle.py).  The BE-Index is not unique (it depends on the
priority order among equal degrees), so it is checked by what the paper's
definitions fix: every bloom is a (2,k)-biclique with k = its bloom number whose
twin pairs share their mid (Definition); every butterfly lies in
exactly one bloom, so Σ_B C(k_B,2) = #butterflies (Property); every edge lies
in k_B - 1 butterflies of each bloom holding it, so Σ_{B ∋ e} (k_B - 1) = ⋈_e, the
oracle's per-edge count (Property)."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb(cuda_ok):
    import __graft_entry__ as entry
    entry.build()
    import paper_2110_12511_b200 as pbng
    return pbng


def dev(pb, g):
    return pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)


def tiny_corpus(n, seed0):
    rng = np.random.default_rng(seed0)
    for i in range(n):
        nu = int(rng.integers(1, 14))
        nv = int(rng.integers(1, 14))
        yield gg.uniform(nu, nv, int(rng.integers(0, nu * nv + 1)), seed=seed0 + i)


def check_be_index(pb, g, d=None):
    I = pb.pbng_be_index(d or dev(pb, g))
    off, k, dom, pairs = I["bloom_off"].astype(np.int64), I["bloom_k"].astype(np.int64), I["dom"], I["pairs"]
    nb = k.shape[0]
    urow = np.repeat(np.arange(g.nU, dtype=np.int64), np.diff(g.off_u).astype(np.int64))
    vcol = g.adj_u.astype(np.int64)
    assert off[0] == 0 and np.array_equal(np.diff(off), k) and np.all(k >= 2)
    # twin pairs: e1 = {start, mid}, e2 = {mid, last}
    bl = np.repeat(np.arange(nb), k)
    side = (dom[:, 0] >> 31).astype(np.int64)[bl]
    x = (dom[:, 0] & 0x7FFFFFFF).astype(np.int64)[bl]
    y = dom[:, 1].astype(np.int64)[bl]
    e1, e2 = pairs[:, 0].astype(np.int64), pairs[:, 1].astype(np.int64)
    xs = np.where(side == 0, urow[e1], vcol[e1])
    ys = np.where(side == 0, urow[e2], vcol[e2])
    m1 = np.where(side == 0, vcol[e1], urow[e1])
    m2 = np.where(side == 0, vcol[e2], urow[e2])
    assert np.array_equal(xs, x) and np.array_equal(ys, y) and np.array_equal(m1, m2)
    assert np.all(x != y)
    # distinct mids per bloom, one bloom per dominant set
    key = bl * (max(g.nU, g.nV) + 1) + m1
    assert np.unique(key).shape[0] == key.shape[0]
    dk = dom[:, 0].astype(np.int64) << 32 | dom[:, 1].astype(np.int64)
    assert np.unique(dk).shape[0] == nb
    sup = oracle.count(g)
    assert int((k * (k - 1) // 2).sum()) == int(sup.sum()) // 2
    per_edge = np.zeros(g.m, np.int64)
    np.add.at(per_edge, e1, k[bl] - 1)
    np.add.at(per_edge, e2, k[bl] - 1)
    assert np.array_equal(per_edge.astype(np.uint64), oracle.edge_count(g))
    return nb, pairs.shape[0]


def test_be_index_tiny_corpus(pb):
    for g in tiny_corpus(120, 777):
        check_be_index(pb, g)
        check_be_index(pb, g.swapped())


@pytest.mark.parametrize("cfg", [1, 2, "2a"])
def test_be_index_configs(pb, cfg):
    g, _ = gg.config(cfg)
    nb, np_ = check_be_index(pb, g)
    assert nb > 0 and np_ >= 2 * nb


def test_wing_tiny_corpus(pb):
    for g in tiny_corpus(150, 9090):
        d = dev(pb, g)
        th, _ = pb.pbng_wing_decompose(d, side=0)
        assert np.array_equal(pb.as_u64(th), oracle.bup_wing(g)), g.name
        th1, _ = pb.pbng_wing_decompose(d, side=1)
        assert np.array_equal(pb.as_u64(th1), oracle.bup_wing(g.swapped())), g.name


def test_wing_degenerate(pb):
    for a, b in ((1, 1), (2, 2), (5, 3), (30, 4)):
        th, _ = pb.pbng_wing_decompose(dev(pb, gg.complete(a, b)))
        assert np.all(pb.as_u64(th) == (a - 1) * (b - 1)), (a, b)
    th, info = pb.pbng_wing_decompose(dev(pb, gg.from_edges(3, 3, [(0, 0), (1, 1), (2, 2)])))
    assert np.all(pb.as_u64(th) == 0) and info["blooms"] == 0
    th, info = pb.pbng_wing_decompose(dev(pb, gg.from_edges(3, 3, [])))
    assert th.numel() == 0


@pytest.mark.parametrize("cfg", [1, 2, "2a"])
def test_wing_configs(pb, cfg):
    g, _ = gg.config(cfg)
    th, info = pb.pbng_wing_decompose(dev(pb, g))
    assert np.array_equal(pb.as_u64(th), oracle.bup_wing(g)), info
    assert info["levels"] >= 1 and info["rounds"] >= info["levels"]


def test_wing_host_driven_rounds(pb, monkeypatch):
    """The host-driven round loop (PBNG_WING_HOST=1: one launch per phase) and the
    device-driven peel (k_wing_peel, one persistent cooperative launch, the default) run the
    same phases: same θ_e, levels and rounds, both bit-exact against Alg.2 BUP."""
    for g in list(tiny_corpus(40, 777)) + [gg.config(1)[0], gg.config(2)[0]]:
        d = dev(pb, g)
        want = oracle.bup_wing(g)
        monkeypatch.delenv("PBNG_WING_HOST", raising=False)
        th_d, info_d = pb.pbng_wing_decompose(d)
        monkeypatch.setenv("PBNG_WING_HOST", "1")
        th_h, info_h = pb.pbng_wing_decompose(d)
        monkeypatch.delenv("PBNG_WING_HOST", raising=False)
        assert np.array_equal(pb.as_u64(th_d), want), g.name
        assert np.array_equal(pb.as_u64(th_h), want), g.name
        assert info_d["levels"] == info_h["levels"] and info_d["rounds"] == info_h["rounds"], (info_d, info_h)
