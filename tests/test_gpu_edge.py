"""GPU parity of per-edge butterfly counting (Alg.1 per-edge part,
P:427-430) against oracle.edge_count (the plain definition, pinned in test_oracle.py):
bit-exact uint64 per edge, in both CSR orders, through the C ABI."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def _check_both_sides(pb, g, d=None):
    d = d or dev(pb, g)
    ec, info = pb.pbng_count_edge_butterflies(d, side=0)
    assert np.array_equal(pb.as_u64(ec), oracle.edge_count(g)), g.name
    ecv, info1 = pb.pbng_count_edge_butterflies(d, side=1)
    assert np.array_equal(pb.as_u64(ecv), oracle.edge_count(g.swapped())), g.name
    return info, info1


def test_edge_tiny_corpus(pb):
    for g in tiny_corpus(150, 4242):
        _check_both_sides(pb, g)


def test_edge_degenerate(pb):
    for g in (gg.from_edges(3, 3, []), gg.from_edges(1, 5, [(0, j) for j in range(5)]), gg.complete(1, 1),
              gg.from_edges(2, 2, [(0, 0), (1, 0), (1, 1)])):
        ec, info = pb.pbng_count_edge_butterflies(dev(pb, g))
        assert np.all(pb.as_u64(ec) == 0)
    for a, b in ((2, 2), (7, 5), (40, 3), (3, 200)):
        ec, _ = pb.pbng_count_edge_butterflies(dev(pb, gg.complete(a, b)))
        assert np.all(pb.as_u64(ec) == (a - 1) * (b - 1)), (a, b)


@pytest.mark.parametrize("cfg", [1, 2, "2a"])
def test_edge_configs(pb, cfg):
    g, _ = gg.config(cfg)
    info, _ = _check_both_sides(pb, g)
    assert info["wedges"] > 0


def test_edge_unsorted_lists(pb):
    g, _ = gg.config(1)
    rng = np.random.default_rng(11)
    adj_u, adj_v = g.adj_u.copy(), g.adj_v.copy()
    for off, adj in ((g.off_u, adj_u), (g.off_v, adj_v)):
        for x in range(len(off) - 1):
            rng.shuffle(adj[off[x]:off[x + 1]])
    gs = gg.Graph(g.nU, g.nV, g.off_u, adj_u, g.off_v, adj_v, "cfg1-shuffled")
    d = pb.DeviceGraph.from_numpy(g.off_u, adj_u, g.off_v, adj_v)
    ec, _ = pb.pbng_count_edge_butterflies(d)
    assert np.array_equal(pb.as_u64(ec), oracle.edge_count(gs))


def test_edge_config3_full(pb):
    """Config 3 at full size (5M edges, hubs up to 30K): every edge, all three tiers
    (the oracle runs from the side with fewer one-sided wedges)."""
    g, _ = gg.config(3)
    d = dev(pb, g)
    wu = int((np.diff(g.off_v).astype(np.float64) ** 2).sum())
    wv = int((np.diff(g.off_u).astype(np.float64) ** 2).sum())
    side = 0 if wu <= wv else 1
    ec, info = pb.pbng_count_edge_butterflies(d, side=side)
    want = oracle.edge_count(g if side == 0 else g.swapped())
    assert np.array_equal(pb.as_u64(ec), want)
    assert all(t > 0 for t in info["tiers"]), info
    # Σ_e ⋈_e = 4 · #butterflies = 2 · Σ_u ⋈_u (GPU per-vertex count, itself oracle-checked)
    assert int(want.sum()) == 2 * int(pb.as_u64(pb.pbng_count_butterflies(d)).sum())


def test_edge_small_tier_variant(cuda_ok):
    """A test build with tiny tier bounds routes starts of small graphs through the CTA
    hash tier and both dense paths (shared and global counters)."""
    sys.path.insert(0, ROOT)
    from paper_2110_12511_b200 import build as b
    lib = b.build_variant("edge_small", {"PBNG_EDGE_WARP_PB": 8, "PBNG_EDGE_CTA_PB": 48,
                                         "PBNG_EDGE_DENSE_SMEM": 300})
    env = dict(os.environ, PBNG_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "edge_variant_runner.py")], env=env,
                         capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    tiers = json.loads(out.stdout.strip().splitlines()[-1])["tiers"]
    assert all(t > 0 for t in tiers), tiers
