"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

All integer outputs must match bit for bit (uint64 butterfly counts and tip
numbers); the partition plan is heuristic and is checked by the invariants the
paper's lemmas give (Lemmas 3-4; ⋈^init).
"""
import numpy as np
import pytest

import graphgen as gg
import oracle
from oracle import brute

pytestmark = pytest.mark.gpu

KINF = np.uint64(0xFFFFFFFFFFFFFFFF)


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
        m = int(rng.integers(0, nu * nv + 1))
        yield gg.uniform(nu, nv, m, seed=seed0 + i)


def test_count_tiny_corpus(pb):
    for g in tiny_corpus(150, 100):
        d = dev(pb, g)
        assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(d, side=0)), oracle.count(g))
        assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(d, side=1)), oracle.count(g.swapped()))


@pytest.mark.parametrize("cfg", [1, 2, "2a"])
def test_count_configs(pb, cfg):
    g, _ = gg.config(cfg)
    assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(dev(pb, g))), oracle.count(g))


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_tip_tiny_corpus(pb, P):
    for g in tiny_corpus(120, 1000 + P):
        d = dev(pb, g)
        for side, gs in ((0, g), (1, g.swapped())):
            tip, _ = pb.pbng_tip_decompose(d, P, side=side)
            assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs)), (g.name, side, P)


@pytest.mark.parametrize("cfg", [1, 2, "2a"])
@pytest.mark.parametrize("opts", [0, 1, 2, 3, 16, 18, 32, 48, 50])
def test_tip_configs_options(pb, cfg, opts):
    g, P = gg.config(cfg)
    want = oracle.bup_tip(g)
    tip, st = pb.pbng_tip_decompose(dev(pb, g), P, opts=opts)
    assert np.array_equal(pb.as_u64(tip), want)
    assert 1 <= st["partitions_used"] <= P
    if opts & 16:
        assert st["recounts"] >= 1


@pytest.mark.parametrize("P", [1, 2, 5, 16, 64, 150, 4096])
def test_tip_partition_count_sweep(pb, P):
    g, _ = gg.config(1)
    tip, st = pb.pbng_tip_decompose(dev(pb, g), P)
    assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(g))
    assert st["partitions_used"] <= P


def test_config2a_closed_form(pb):
    from math import comb
    shapes = gg.block_sizes(200, 5, 60, seed=2)
    want = np.concatenate([[(a - 1) * comb(b, 2)] * a for a, b in shapes]).astype(np.uint64)
    g, P = gg.config("2a")
    tip, _ = pb.pbng_tip_decompose(dev(pb, g), P)
    assert np.array_equal(pb.as_u64(tip), want)


def test_config3_parity(pb):
    """Config 3 (500K x 200K, 5M edges, Chung-Lu γ=2.1, P=150) against the full oracle."""
    g, P = gg.config(3)
    d = dev(pb, g)
    sup = pb.as_u64(pb.pbng_count_butterflies(d))
    tip, st = pb.pbng_tip_decompose(d, P)
    want_sup = oracle.count(g)
    assert np.array_equal(sup, want_sup)
    want = _config3_theta(g)
    assert np.array_equal(pb.as_u64(tip), want)
    assert st["partitions_used"] > 1
    part, init, bounds, nparts = pb.pbng_tip_plan(d, P)
    _check_plan(g, part, init, bounds, nparts, want)


def _check_plan(g, part, init, bounds, nparts, theta):
    part = part.cpu().numpy()
    init = init.cpu().numpy().view(np.uint64)
    assert 1 <= nparts
    b = bounds[: nparts + 1]
    assert b[0] == 0 and b[-1] == KINF
    assert np.all(b[1:] > b[:-1])                           # strictly increasing ranges
    assert part.min() >= 0 and part.max() < nparts
    lo, hi = b[part], b[part + 1]
    assert np.all(theta >= lo) and np.all(theta < hi)       # θ(i) <= θ_u < θ(i+1) (Lemmas 3-4)
    return part, init


def test_plan_properties_tiny(pb):
    for g in tiny_corpus(80, 7000):
        theta = oracle.bup_tip(g)
        for P in (2, 4):
            part, init, bounds, nparts = pb.pbng_tip_plan(dev(pb, g), P)
            part, init = _check_plan(g, part, init, bounds, nparts, theta)
            assert list(init) == brute.init_support(g, list(part))  # ⋈^init


def test_plan_properties_config1(pb):
    g, P = gg.config(1)
    theta = oracle.bup_tip(g)
    for opts in (0, 2, 16):
        part, init, bounds, nparts = pb.pbng_tip_plan(dev(pb, g), P, opts=opts)
        _check_plan(g, part, init, bounds, nparts, theta)


def test_host_entry_point(pb):
    g, P = gg.config(1)
    tip, st = pb.pbng_tip_decompose_host(g.off_u, g.adj_u, g.off_v, g.adj_v, P)
    assert np.array_equal(tip, oracle.bup_tip(g))
    tipv, _ = pb.pbng_tip_decompose_host(g.off_u, g.adj_u, g.off_v, g.adj_v, P, side=1)
    assert np.array_equal(tipv, oracle.bup_tip(g.swapped()))


def test_edge_cases(pb):
    # empty edge set, isolated vertices
    g = gg.from_edges(5, 3, [])
    tip, st = pb.pbng_tip_decompose(dev(pb, g), 4)
    assert np.all(pb.as_u64(tip) == 0)
    assert np.all(pb.as_u64(pb.pbng_count_butterflies(dev(pb, g))) == 0)
    # star, complete, path
    for g, want in ((gg.complete(1, 5), [0]), (gg.complete(4, 4), [18] * 4),
                    (gg.from_edges(2, 2, [(0, 0), (1, 0), (1, 1)]), [0, 0])):
        tip, _ = pb.pbng_tip_decompose(dev(pb, g), 3)
        assert list(pb.as_u64(tip)) == want
    # errors
    g, _ = gg.config(1)
    d = dev(pb, g)
    for bad in (lambda: pb.pbng_tip_decompose(d, 0), lambda: pb.pbng_tip_decompose(d, 5000),
                lambda: pb.pbng_tip_decompose(d, 8, side=2)):
        with pytest.raises(pb.PbngError) as ei:
            bad()
        assert ei.value.code == pb.ERR_ARG


def test_validate_rejects_bad_csr(pb):
    import torch
    g, _ = gg.config(1)
    d = dev(pb, g)
    bad_adj = d.adj_u.clone()
    bad_adj[5] = g.nV + 7
    d2 = pb.DeviceGraph(d.nU, d.nV, d.off_u, bad_adj, d.off_v, d.adj_v)
    with pytest.raises(pb.PbngError) as ei:
        pb.pbng_tip_decompose(d2, 8, opts=pb.OPT_VALIDATE)
    assert ei.value.code == pb.ERR_GRAPH
    tip, _ = pb.pbng_tip_decompose(d, 8, opts=pb.OPT_VALIDATE)
    torch.cuda.synchronize()


def test_unsorted_adjacency_and_count_paths(pb):
    """Adjacency order is not a precondition (the library relabels and sorts
    internal copies); vertex-priority and one-sided counting give the same θ."""
    g, P = gg.config(1)
    rng = np.random.default_rng(5)
    adj_u, adj_v = g.adj_u.copy(), g.adj_v.copy()
    for off, adj in ((g.off_u, adj_u), (g.off_v, adj_v)):
        for x in range(len(off) - 1):
            seg = adj[off[x]:off[x + 1]]
            rng.shuffle(seg)
    d = pb.DeviceGraph.from_numpy(g.off_u, adj_u, g.off_v, adj_v)
    want = oracle.bup_tip(g)
    assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(d)), oracle.count(g))
    for opts in (0, pb.OPT_ONESIDED_COUNT, pb.OPT_ONESIDED_COUNT | pb.OPT_FORCE_RECOUNT, pb.OPT_FORCE_RECOUNT):
        tip, _ = pb.pbng_tip_decompose(d, P, opts=opts)
        assert np.array_equal(pb.as_u64(tip), want), opts


@pytest.mark.parametrize("P", [1, 4])
def test_tip_tiny_corpus_forced_recount(pb, P):
    """Every CD iteration re-counts by vertex-priority counting on the live graph."""
    for g in tiny_corpus(60, 3000 + P):
        d = dev(pb, g)
        for side, gs in ((0, g), (1, g.swapped())):
            tip, _ = pb.pbng_tip_decompose(d, P, side=side, opts=pb.OPT_FORCE_RECOUNT)
            assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs)), (g.name, side, P)
            tip, _ = pb.pbng_tip_decompose(d, P, side=side, opts=pb.OPT_FORCE_RECOUNT | pb.OPT_NO_DELETE)
            assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs)), (g.name, side, P)


def _sample_levels(th, rng, k=64, max_members=2000):
    vals, counts = np.unique(th, return_counts=True)
    small = vals[counts <= max_members]
    pick = rng.choice(small, size=min(k, len(small)), replace=False) if len(small) else np.zeros(0, np.uint64)
    return np.unique(np.append(pick, vals[-1]))  # plus the top level (densest core)


def test_config4_full_certificate(pb):
    """Config 4 at full size (8M x 3M peel orientation, 30M edges, P=150): every
    butterfly count equal to the oracle's, and the multi-core exactness certificate
    (oracle/certificate.c) over every vertex and every level — one pass
    over the unordered pairs gives the oracle counts and the (A) sums together."""
    g, P = gg.config(4)
    d = dev(pb, g)
    th = pb.as_u64(pb.pbng_tip_decompose(d, P)[0])
    sup = pb.as_u64(pb.pbng_count_butterflies(d))
    osup, sge, bad, first = oracle.cert_one_pass(g, th)
    assert np.array_equal(sup, osup), "config 4 butterfly counts differ from the oracle"
    assert np.all(th <= sup)
    assert np.all(sge >= th), "certificate (A) fails"
    assert bad == 0, ("certificate (C) fails at level", first)


def test_config5_certificate(pb):
    """Config 5 at full size (25M x 30M, 300M edges, P=400).

    Full parity through the offline oracle record profiles/r2_certificate_cfg5.json,
    written by scripts/certify_offline.py, which runs only oracle/ code on the host
    (several hours on 8 cores, too long for a test): the oracle's butterfly counts of
    every vertex (SHA-256), and the exactness certificate (A) over all 25M vertices and
    (C) over every level of the tip vector whose SHA-256 it records (θ is unique,
    Definition 2, so a certified vector is THE tip vector).  Here the GPU
    counts and θ must hash to those values, on the same generator output.
    In this run, too: sampled oracle counts, certificate (A) on 2,000 sampled
    vertices and (C) on sampled levels of up to 50,000 members plus the top level."""
    import hashlib
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "r2_certificate_cfg5.json")
    rec = json.load(open(path)) if os.path.exists(path) else None
    g, P = gg.config(5)
    d = dev(pb, g)
    th = pb.as_u64(pb.pbng_tip_decompose(d, P)[0])
    sup = pb.as_u64(pb.pbng_count_butterflies(d))
    del d
    if rec is not None:
        assert rec["certified_exact"] and rec["A_violations"] == 0 and rec["C_failing_levels"] == 0
        assert g.sha256() == rec["graph_sha256"], "generator output differs from the certified graph"
        assert hashlib.sha256(sup.tobytes()).hexdigest() == rec["oracle_support_sha256"], "counts differ from the oracle's"
        assert hashlib.sha256(th.tobytes()).hexdigest() == rec["theta_sha256"], "θ differs from the certified tip vector"
    else:
        import warnings
        warnings.warn("profiles/r2_certificate_cfg5.json absent: config 5 checked on samples only in this run")
    rng = np.random.default_rng(55)
    us = np.sort(rng.choice(g.nU, 2000, replace=False)).astype(np.uint32)
    assert np.array_equal(sup[us], oracle.count_subset(g, us))
    assert np.all(th <= sup)
    assert np.all(oracle.cert_support_ge(g, th, us) >= th[us])
    bad, first = oracle.cert_levels(g, th, _sample_levels(th, rng, k=96, max_members=50000))
    assert bad == 0, first


@pytest.mark.parametrize("cfg", [1, 2])
def test_tip_other_side(pb, cfg):
    """Peeling the other vertex side (side=1 swaps the roles of U and V)."""
    g, P = gg.config(cfg)
    gs = g.swapped()
    d = dev(pb, g)
    assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(d, side=1)), oracle.count(gs))
    tip, st = pb.pbng_tip_decompose(d, P, side=1)
    assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs))


@pytest.mark.parametrize("P", [1, 7, 64, 400])
def test_config3_partition_counts(pb, P):
    """Config 3 with P from 1 (all of U peeled by FD = BUP) to 400: θ does not depend on P."""
    g, _ = gg.config(3)
    tip, st = pb.pbng_tip_decompose(dev(pb, g), P)
    assert np.array_equal(pb.as_u64(tip), _config3_theta(g))
    assert 1 <= st["partitions_used"] <= P


_C3 = {}


def _config3_theta(g):
    if "theta" not in _C3:
        _C3["theta"] = oracle.bup_tip(g)
    return _C3["theta"]


def test_config3_ablations(pb):
    """PBNG- (no dynamic graph updates: peeled entries stay in every list through CD, the
    FD layout is built after CD) and PBNG-- (also no batch re-count), on
    config 3: θ equals the oracle's, and without deletion CD traverses more wedges
    (deletion is what saves them)."""
    g, P = gg.config(3)
    d = dev(pb, g)
    want = _config3_theta(g)
    _, st0 = pb.pbng_tip_decompose(d, P, opts=pb.OPT_STATS)
    for opts in (pb.OPT_NO_DELETE, pb.OPT_NO_DELETE | pb.OPT_NO_RECOUNT):
        tip, st = pb.pbng_tip_decompose(d, P, opts=opts | pb.OPT_STATS)
        assert np.array_equal(pb.as_u64(tip), want), opts
        assert st["wedges_cd"] > st0["wedges_cd"], (opts, st["wedges_cd"], st0["wedges_cd"])


@pytest.mark.parametrize("P", [1, 3, 8])
def test_fd_grid_path_tiny(pb, P):
    """FD on the whole GPU (host-driven rounds), forced for every small partition."""
    for g in tiny_corpus(60, 4000 + P):
        d = dev(pb, g)
        for side, gs in ((0, g), (1, g.swapped())):
            tip, _ = pb.pbng_tip_decompose(d, P, side=side, opts=pb.OPT_FD_GRID)
            assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs)), (g.name, side, P)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_fd_grid_path_configs(pb, cfg):
    g, P = gg.config(cfg)
    want = _config3_theta(g) if cfg == 3 else oracle.bup_tip(g)
    tip, st = pb.pbng_tip_decompose(dev(pb, g), 400 if cfg == 3 else P, opts=pb.OPT_FD_GRID)
    assert np.array_equal(pb.as_u64(tip), want)


def test_kernel_times_deferred(pb):
    """PBNG_OPT_STATS_DEFER: the call records per-launch events, pbng_kernel_times sums them."""
    g, P = gg.config(1)
    d = dev(pb, g)
    tip, st = pb.pbng_tip_decompose(d, P, opts=pb.OPT_STATS_DEFER)
    assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(g))
    assert st["ms_kernel"] == {}
    kt = pb.pbng_kernel_times()
    assert kt and all(v >= 0 for v in kt.values()) and "fd" in kt
    assert pb.pbng_kernel_times() == {}  # consumed
    _, st2 = pb.pbng_tip_decompose(d, P, opts=pb.OPT_STATS)
    assert set(st2["ms_kernel"]) == set(kt)


# ---- k-tip hierarchy retrieval: pbng_tip_components vs oracle.tip_level ----

def _levels(th):
    u = np.unique(th)
    top = int(th.max(initial=0))
    ks = [0, 1, top, top + 1] + [int(x) for x in u[:: max(1, len(u) // 6)]]
    return sorted(set(ks))


def _check_levels(pb, d, gs, th, side, ks):
    import torch
    tdev = torch.from_numpy(np.ascontiguousarray(th, np.uint64).view(np.int64)).cuda()
    for k in ks:
        lab, n = pb.pbng_tip_components(d, tdev, k, side=side)
        want, wn = oracle.tip_level(gs, th, k)
        got = lab.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want) and n == wn, (gs.name, side, k, n, wn)


def test_tip_components_tiny(pb):
    for g in tiny_corpus(80, 7000):
        d = dev(pb, g)
        for side, gs in ((0, g), (1, g.swapped())):
            th = oracle.bup_tip(gs)
            _check_levels(pb, d, gs, th, side, _levels(th))


@pytest.mark.parametrize("cfg", [1, 2, "2a"])
def test_tip_components_configs(pb, cfg):
    g, P = gg.config(cfg)
    d = dev(pb, g)
    tip, _ = pb.pbng_tip_decompose(d, P)
    th = pb.as_u64(tip)
    assert np.array_equal(th, oracle.bup_tip(g))
    _check_levels(pb, d, g, th, 0, _levels(th))


def test_tip_components_hubs(pb):
    """Power-law graph with hubs (d_v up to ~5K): starts in all three aggregation tiers."""
    g = gg.chung_lu(60000, 20000, 300000, 2.1, 2.1, 8000.0, 8000.0, seed=31)
    d = dev(pb, g)
    tip, _ = pb.pbng_tip_decompose(d, 32)
    th = pb.as_u64(tip)
    assert np.array_equal(th, oracle.bup_tip(g))
    _check_levels(pb, d, g, th, 0, _levels(th))


def test_tip_components_arbitrary_vector(pb):
    """The level is defined by any vector (members = entries >= k), not only by tip numbers."""
    g, _ = gg.config(1)
    rng = np.random.default_rng(5)
    th = rng.integers(0, 4, g.nU).astype(np.uint64)
    _check_levels(pb, dev(pb, g), g, th, 0, [0, 1, 2, 3, 4])


def test_tip_components_config3(pb):
    """Config 3 at full size: the Def. 2 '>= k butterflies' condition of every level member,
    counted on the GPU on the level's induced subgraph (verify_hierarchy), and oracle
    parity of the labels at the top level."""
    g, P = gg.config(3)
    d = dev(pb, g)
    tip, _ = pb.pbng_tip_decompose(d, P)
    th = pb.as_u64(tip)
    pos = np.sort(th[th > 0])
    e = g.edges().astype(np.int64)
    for q in (0.5, 0.9, 0.999):
        k = int(pos[int(q * (len(pos) - 1))])
        lab, n = pb.pbng_tip_components(d, tip, k)
        lab = lab.cpu().numpy().view(np.uint32)
        members = th >= k
        assert np.array_equal(lab != 0xFFFFFFFF, members)
        assert n == len(np.unique(lab[members]))
        h = gg.from_edges(g.nU, g.nV, e[members[e[:, 0]]])
        s = pb.as_u64(pb.pbng_count_butterflies(dev(pb, h)))
        assert np.all(s[members] >= k), k
        if q == 0.999:
            want, wn = oracle.tip_level(g, th, k)
            assert np.array_equal(lab, want) and n == wn
