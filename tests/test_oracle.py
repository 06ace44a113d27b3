"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/oracle.c) is checked against things other than itself:
  * brute-force 4-tuple butterfly enumeration (oracle/brute.py),
  * the K_{a,b} closed form: support = theta = (a-1)*C(b,2)  (north_star),
  * the identity Σ_U support = Σ_V support = 2·#butterflies with the
    V side computed by running the oracle on the transposed graph,
  * tip numbers from Definition 2 by exhaustive k sweep,
  * golden graphs (tests/golden/, each with its citation),
  * the structured config-2 closed form (noise-free) and monotonicity (noisy).
A plausible mistake (dropped clamp, C(w,2) vs w^2, self-pair counted, wrong
side, heap tie-break bug) fails at least one of these.
"""
import os
from math import comb

import numpy as np
import pytest

import graphgen as gg
import oracle
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _parse(path):
    rows = []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append([c.strip() for c in line.split("|")])
    return rows


def _edges(s):
    return [tuple(int(x) for x in t.split("-")) for t in s.split()]


def _tiny_corpus(n=300, seed0=1000):
    rng = np.random.default_rng(7)
    for i in range(n):
        nu = int(rng.integers(1, 10))
        nv = int(rng.integers(1, 10))
        m = int(rng.integers(0, nu * nv + 1))
        yield gg.uniform(nu, nv, m, seed=seed0 + i)


def test_spec_small_cases():
    for name, sizes, edges, side, sup, th in _parse(os.path.join(GOLD, "spec_small_cases.txt")):
        nu, nv = map(int, sizes.split())
        g = gg.from_edges(nu, nv, _edges(edges))
        if side == "V":
            g = g.swapped()
        assert list(oracle.count(g)) == [int(x) for x in sup.split()], name
        assert list(oracle.bup_tip(g)) == [int(x) for x in th.split()], name


def test_survey_golden_graphs():
    for name, sizes, edges, sup, total, th in _parse(os.path.join(GOLD, "survey_graphs.txt")):
        nu, nv = map(int, sizes.split())
        g = gg.from_edges(nu, nv, _edges(edges))
        s = oracle.count(g)
        assert list(s) == [int(x) for x in sup.split()], name
        assert int(s.sum()) == 2 * int(total), name
        assert list(oracle.bup_tip(g)) == [int(x) for x in th.split()], name
        assert brute.tip_by_definition(g) == [int(x) for x in th.split()], name


@pytest.mark.parametrize("a", range(1, 7))
@pytest.mark.parametrize("b", range(1, 7))
def test_complete_bipartite_closed_form(a, b):
    g = gg.complete(a, b)
    want = (a - 1) * comb(b, 2)
    assert list(oracle.count(g)) == [want] * a
    assert list(oracle.bup_tip(g)) == [want] * a
    # the V side of K_{a,b} is K_{b,a} seen from the other side
    assert list(oracle.bup_tip(g.swapped())) == [(b - 1) * comb(a, 2)] * b


def test_count_equals_bruteforce_4tuples():
    for g in _tiny_corpus():
        cu, cv, total, _ = brute.butterflies(g)
        su = oracle.count(g)
        sv = oracle.count(g.swapped())
        assert list(su) == cu
        assert list(sv) == cv
        assert int(su.sum()) == int(sv.sum()) == 2 * total


def test_bup_equals_definition2():
    for g in _tiny_corpus(n=200, seed0=5000):
        th = oracle.bup_tip(g)
        assert list(th) == brute.tip_by_definition(g)
        assert np.all(th <= oracle.count(g))  # theta_u <= support_u
        thv = oracle.bup_tip(g.swapped())
        assert list(thv) == brute.tip_by_definition(g.swapped())


def test_bup_invariant_under_relabeling():
    # Lemma 1: theta does not depend on the peel order among ties;
    # relabel U by a random permutation (changes the lowest-id tie-break).
    rng = np.random.default_rng(3)
    for g in _tiny_corpus(n=100, seed0=9000):
        perm = rng.permutation(g.nU)
        e = g.edges().astype(np.int64)
        h = gg.from_edges(g.nU, g.nV, np.stack([perm[e[:, 0]], e[:, 1]], 1))
        assert np.array_equal(oracle.bup_tip(h)[perm], oracle.bup_tip(g))


def test_config2_blocks_closed_form():
    shapes = gg.block_sizes(200, 5, 60, seed=2)
    want = np.concatenate([[(a - 1) * comb(b, 2)] * a for a, b in shapes]).astype(np.uint64)
    g0, _ = gg.config("2a")
    assert g0.m == sum(a * b for a, b in shapes)
    assert np.array_equal(oracle.count(g0), want)
    assert np.array_equal(oracle.bup_tip(g0), want)
    # with noise edges added, tip numbers can only grow (monotonicity, SURVEY §8(c) θ (iii))
    g, _ = gg.config(2)
    assert g.nU == g0.nU and g.m > g0.m
    th = oracle.bup_tip(g)
    assert np.all(th >= want)


def test_count_subset_matches_count():
    g, _ = gg.config(1)
    full = oracle.count(g)
    us = np.array([0, 5, 17, 1999, 3], np.uint32)
    assert np.array_equal(oracle.count_subset(g, us), full[us])


def test_empty_and_degenerate():
    g = gg.from_edges(3, 4, [])
    assert list(oracle.count(g)) == [0, 0, 0]
    assert list(oracle.bup_tip(g)) == [0, 0, 0]
    g = gg.from_edges(0, 0, [])
    assert oracle.bup_tip(g).shape == (0,)


def test_certificate_accepts_definition2_and_rejects_mutations():
    """oracle/certificate.c: accepts the Definition-2 tip numbers
    (brute force) and rejects every single ±1 mutation of them."""
    for g in _tiny_corpus(n=120, seed0=9000):
        want = np.array(brute.tip_by_definition(g), np.uint64)
        assert oracle.certify(g, want)
        for u in range(g.nU):
            for d in (1, -1):
                if d < 0 and want[u] == 0:
                    continue
                bad = want.copy()
                bad[u] = np.uint64(int(bad[u]) + d)
                assert not oracle.certify(g, bad), (g.name, u, d)


def test_certificate_rejects_random_vectors():
    rng = np.random.default_rng(3)
    for g in _tiny_corpus(n=60, seed0=9500):
        want = np.array(brute.tip_by_definition(g), np.uint64)
        sup = oracle.count(g)
        for _ in range(20):
            cand = rng.integers(0, sup + 2).astype(np.uint64)
            assert oracle.certify(g, cand) == bool(np.array_equal(cand, want))


def test_certificate_on_config1():
    g, _ = gg.config(1)
    th = oracle.bup_tip(g)
    assert oracle.certify(g, th)
    s_ge = oracle.cert_support_ge(g, th, us=np.arange(0, g.nU, 7))
    assert np.all(s_ge >= th[::7])


# ---- k-tip hierarchy retrieval (Def. 2) ----

NOLAB = 0xFFFFFFFF


def test_tip_level_golden():
    graphs = {name: (sizes, edges) for name, sizes, edges, *_ in _parse(os.path.join(GOLD, "survey_graphs.txt"))}
    for name, k, labels, ncomp in _parse(os.path.join(GOLD, "tip_levels.txt")):
        nu, nv = map(int, graphs[name][0].split())
        g = gg.from_edges(nu, nv, _edges(graphs[name][1]))
        want = [NOLAB if x == "-" else int(x) for x in labels.split()]
        lab, n = oracle.tip_level(g, oracle.bup_tip(g), int(k))
        assert list(lab) == want and n == int(ncomp), (name, k)
        assert brute.k_tips(g, int(k)) == (want, int(ncomp)), (name, k)


def test_tip_level_equals_definition2():
    # the oracle works from tip numbers; brute.k_tips from the 4-tuples alone
    for g in _tiny_corpus(n=150, seed0=12000):
        th = oracle.bup_tip(g)
        for k in range(0, int(th.max(initial=0)) + 2):
            lab, n = oracle.tip_level(g, th, k)
            assert (list(lab), n) == brute.k_tips(g, k), (g.name, k)


def test_tip_level_blocks_and_nesting():
    # config 2a: disjoint K_{a,b}; every block is its own k-tip at any k <= its θ
    shapes = gg.block_sizes(200, 5, 60, seed=2)
    g, _ = gg.config("2a")
    th = oracle.bup_tip(g)
    first = np.cumsum([0] + [a for a, _ in shapes[:-1]])
    lab, n = oracle.tip_level(g, th, 1)
    assert n == 200
    assert np.array_equal(lab, np.repeat(first, [a for a, _ in shapes]).astype(np.uint32))
    # nesting on config 1: every (k+1)-tip lies inside one k-tip
    g, _ = gg.config(1)
    th = oracle.bup_tip(g)
    ks = np.unique(th)[:: max(1, len(np.unique(th)) // 6)]
    prev = None
    for k in ks:
        lab, n = oracle.tip_level(g, th, int(k))
        members = th >= k
        assert np.all((lab != NOLAB) == members)
        assert np.all(lab[members] <= np.nonzero(members)[0])
        if prev is not None:
            for c in np.unique(lab[members]):
                assert len(np.unique(prev[lab == c])) == 1
        prev = lab


def test_one_pass_certificate_equals_per_vertex_certificate():
    """certificate.c one-pass functions (each unordered pair once, induced level runs):
    counts equal oracle_count, s_ge equals oracle_cert_support_ge, verdicts equal certify()
    on the Definition-2 θ, every ±1 mutation and random vectors."""
    rng = np.random.default_rng(21)
    for g in _tiny_corpus(n=120, seed0=15000):
        want = np.array(brute.tip_by_definition(g), np.uint64)
        sup, sge, bad, _ = oracle.cert_one_pass(g, want)
        assert np.array_equal(sup, oracle.count(g))
        assert np.array_equal(sup, np.array(brute.butterflies(g)[0], np.uint64))
        assert np.array_equal(sge, oracle.cert_support_ge(g, want))
        assert bad == 0 and oracle.certify_one_pass(g, want)
        for u in range(g.nU):
            for d in (-1, 1):
                if int(want[u]) + d < 0:
                    continue
                cand = want.copy()
                cand[u] = np.uint64(int(cand[u]) + d)
                assert not oracle.certify_one_pass(g, cand), (g.name, u, d)
        for _ in range(5):
            cand = rng.integers(0, sup + 2).astype(np.uint64)
            assert oracle.certify_one_pass(g, cand) == bool(np.array_equal(cand, want))


def test_one_pass_certificate_on_config1():
    g, _ = gg.config(1)
    th = oracle.bup_tip(g)
    sup, sge, bad, _ = oracle.cert_one_pass(g, th)
    assert np.array_equal(sup, oracle.count(g)) and bad == 0 and np.all(sge >= th)


def test_brute_init_support_pins():
    """brute.init_support (the ⋈^init checker) against what fixes it without itself:
    one partition -> the 4-tuple counts; K_{a,b} with any partition vector -> closed form
    (#u' != u with part[u'] >= part[u]) * C(b,2); partitions ordered like θ -> s_ge of the
    certificate's (A) (u' with θ' >= θ'_u)."""
    rng = np.random.default_rng(31)
    for g in _tiny_corpus(n=60, seed0=16000):
        cu = brute.butterflies(g)[0]
        assert brute.init_support(g, [0] * g.nU) == cu
        th = oracle.bup_tip(g)
        assert brute.init_support(g, [int(x) for x in th]) == list(oracle.cert_support_ge(g, th))
    for a, b in ((2, 2), (3, 4), (5, 3), (4, 6)):
        g = gg.complete(a, b)
        for _ in range(5):
            part = [int(x) for x in rng.integers(0, 3, a)]
            want = [sum(1 for x in range(a) if x != u and part[x] >= part[u]) * comb(b, 2) for u in range(a)]
            assert brute.init_support(g, part) == want


# ---- per-edge butterfly counts (Alg.1 per-edge part P:427-430)

def _mirror(g):
    """mirror[e] = position in g's V-side CSR of the edge at U-side position e."""
    pos = {}
    for v in range(g.nV):
        for f in range(int(g.off_v[v]), int(g.off_v[v + 1])):
            pos[(int(g.adj_v[f]), v)] = f
    return np.array([pos[(u, int(g.adj_u[e]))] for u in range(g.nU)
                     for e in range(int(g.off_u[u]), int(g.off_u[u + 1]))], np.int64)


def test_edge_count_golden():
    for name, sizes, edges, want in _parse(os.path.join(GOLD, "edge_counts.txt")):
        nu, nv = map(int, sizes.split())
        el = _edges(edges)
        g = gg.from_edges(nu, nv, el)
        got = dict(zip([(u, int(g.adj_u[e])) for u in range(g.nU)
                        for e in range(int(g.off_u[u]), int(g.off_u[u + 1]))], oracle.edge_count(g)))
        assert [int(got[e]) for e in el] == [int(x) for x in want.split()], name


@pytest.mark.parametrize("a", range(1, 6))
@pytest.mark.parametrize("b", range(1, 6))
def test_edge_count_complete_bipartite(a, b):
    """K_{a,b}: every edge lies in (a-1)(b-1) butterflies."""
    assert list(oracle.edge_count(gg.complete(a, b))) == [(a - 1) * (b - 1)] * (a * b)


def test_edge_count_equals_bruteforce_4tuples():
    """Each butterfly adds one to each of its four edges (4-tuple enumeration); the
    count from the V side (oracle on the transposed graph, a different traversal)
    agrees edge by edge; Σ_e ⋈_e = 4·#butterflies and Σ_{e ∋ u} ⋈_e = 2·⋈_u."""
    for g in _tiny_corpus(n=200, seed0=9000):
        ec = oracle.edge_count(g)
        assert list(ec) == brute.edge_butterflies(g)
        ecv = oracle.edge_count(g.swapped())
        assert np.array_equal(ecv[_mirror(g)], ec)
        _, _, total, _ = brute.butterflies(g)
        assert int(ec.sum()) == 4 * total
        per_u = np.zeros(g.nU, np.uint64)
        for u in range(g.nU):
            per_u[u] = ec[int(g.off_u[u]):int(g.off_u[u + 1])].sum()
        assert np.array_equal(per_u, 2 * oracle.count(g))


def test_edge_count_config_identities():
    """Config 1 and 2 (20K / 197K edges): both traversal directions agree edge by edge,
    and the per-vertex sums are twice the vertex counts on both sides."""
    for cfg in (1, "2a"):
        g, _ = gg.config(cfg)
        ec = oracle.edge_count(g)
        ecv = oracle.edge_count(g.swapped())
        assert np.array_equal(ecv[_mirror(g)], ec)
        du = np.diff(g.off_u).astype(np.int64)
        per_u = np.where(du > 0, np.add.reduceat(ec, np.minimum(g.off_u[:-1], g.m - 1).astype(np.int64)), 0)
        assert np.array_equal(per_u, 2 * oracle.count(g))
        assert int(ec.sum()) == 2 * int(oracle.count(g).sum())
    # config 2a closed form: block K_{a,b} edges have (a-1)(b-1)
    g, _ = gg.config("2a")
    ec = oracle.edge_count(g)
    du = np.diff(g.off_u).astype(np.int64)
    dv = np.diff(g.off_v).astype(np.int64)
    u_of_e = np.repeat(np.arange(g.nU), du)
    want = (du[u_of_e] - 1) * (dv[g.adj_u.astype(np.int64)] - 1)
    assert np.array_equal(ec, want.astype(np.uint64))


# ---- wing decomposition (Alg.2)

def test_wing_golden():
    for name, sizes, edges, want in _parse(os.path.join(GOLD, "wing_numbers.txt")):
        nu, nv = map(int, sizes.split())
        el = _edges(edges)
        g = gg.from_edges(nu, nv, el)
        got = dict(zip([(u, int(g.adj_u[e])) for u in range(g.nU)
                        for e in range(int(g.off_u[u]), int(g.off_u[u + 1]))], oracle.bup_wing(g)))
        assert [int(got[e]) for e in el] == [int(x) for x in want.split()], name
        assert brute.wing_by_definition(g) == [int(got[(u, v)]) for u in range(g.nU)
                                               for v in g.adj_u[int(g.off_u[u]):int(g.off_u[u + 1])]], name


@pytest.mark.parametrize("a", range(1, 6))
@pytest.mark.parametrize("b", range(1, 6))
def test_wing_complete_bipartite(a, b):
    """K_{a,b} is one ((a-1)(b-1))-wing."""
    assert list(oracle.bup_wing(gg.complete(a, b))) == [(a - 1) * (b - 1)] * (a * b)


def test_wing_equals_definition():
    """Alg.2 BUP = Definition 1 (iterated removal over the 4-tuples) on 150 tiny graphs;
    the transposed graph gives the same wing number per edge; θ_e <= ⋈_e."""
    for g in _tiny_corpus(n=150, seed0=12000):
        th = oracle.bup_wing(g)
        assert list(th) == brute.wing_by_definition(g)
        assert np.array_equal(oracle.bup_wing(g.swapped())[_mirror(g)], th)
        assert np.all(th <= oracle.edge_count(g))


def test_wing_config2a_blocks():
    """Config 2a (200 disjoint K_{a,b}): θ_e = (a-1)(b-1) of the edge's block."""
    g, _ = gg.config("2a")
    du = np.diff(g.off_u).astype(np.int64)
    dv = np.diff(g.off_v).astype(np.int64)
    u_of_e = np.repeat(np.arange(g.nU), du)
    want = (du[u_of_e] - 1) * (dv[g.adj_u.astype(np.int64)] - 1)
    assert np.array_equal(oracle.bup_wing(g), want.astype(np.uint64))
