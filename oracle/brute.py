"""ORACLE (brute force) — TEST INFRASTRUCTURE ONLY.

Pure-Python definitions for tiny graphs (≤ ~12 vertices per side).  These are the
plain definitions the paper states, written out with no algorithmic shortcut:

  butterflies(g)        every 4-tuple {u,u'} x {v,v'} with all four edges present
                        (a butterfly = 2,2-biclique).
  tip_by_definition(g)  theta_u = max k such that u lies in a subgraph H with
                        U(H) ⊆ U, V(H) = V in which every u in U(H) is in >= k
                        butterflies of H (Definition 2, tip number
                        P:469-471).  Every k in [0, max support] is swept
                        (tip numbers can fall between initial supports).
  k_tips(g, k)          the k-tips of Definition 2 straight from the
                        4-tuples, without tip numbers: the largest vertex set
                        in which every u has >= k butterflies (iterated
                        removal), split into classes of "connected by a
                        series of butterflies"; label = smallest id.
  init_support(g, part) butterflies u shares only with vertices of partitions
                        j >= part[u] (the support initialisation vector,
                        P:781-786), counted from the 4-tuples.
"""
from __future__ import annotations

from itertools import combinations


def _adj_sets(g):
    nu = [set(int(x) for x in g.adj_u[int(g.off_u[u]):int(g.off_u[u + 1])]) for u in range(g.nU)]
    return nu


def butterflies(g):
    """Returns (per-U counts, per-V counts, total, list of (u,u',v,v') tuples)."""
    nu = _adj_sets(g)
    cu = [0] * g.nU
    cv = [0] * g.nV
    tuples = []
    for u, u2 in combinations(range(g.nU), 2):
        for v, v2 in combinations(range(g.nV), 2):
            if v in nu[u] and v2 in nu[u] and v in nu[u2] and v2 in nu[u2]:
                cu[u] += 1
                cu[u2] += 1
                cv[v] += 1
                cv[v2] += 1
                tuples.append((u, u2, v, v2))
    return cu, cv, len(tuples), tuples


def _support_within(tuples, members):
    s = {u: 0 for u in members}
    for (u, u2, _, _) in tuples:
        if u in members and u2 in members:
            s[u] += 1
            s[u2] += 1
    return s


def tip_by_definition(g):
    """Tip number of every u by Definition 2 (largest k-subgraph containing u)."""
    cu, _, _, tuples = butterflies(g)
    theta = [0] * g.nU
    kmax = max(cu) if cu else 0
    for k in range(0, kmax + 1):
        members = set(range(g.nU))
        while True:
            s = _support_within(tuples, members)
            drop = {u for u in members if s[u] < k}
            if not drop:
                break
            members -= drop
        for u in members:
            theta[u] = max(theta[u], k)
    return theta


def init_support(g, part):
    """Butterflies of u shared only with u' whose partition index is >= part[u]."""
    _, _, _, tuples = butterflies(g)
    s = [0] * g.nU
    for (u, u2, _, _) in tuples:
        if part[u2] >= part[u]:
            s[u] += 1
        if part[u] >= part[u2]:
            s[u2] += 1
    return s


def k_tips(g, k):
    """(label per u — smallest id of its k-tip, or 0xFFFFFFFF outside every k-tip —, number of k-tips)."""
    _, _, _, tuples = butterflies(g)
    members = set(range(g.nU))
    while True:
        s = _support_within(tuples, members)
        drop = {u for u in members if s[u] < k}
        if not drop:
            break
        members -= drop
    # butterfly connectivity inside the member set: merge classes per butterfly
    cls = {u: {u} for u in members}
    for (u, u2, _, _) in tuples:
        if u in members and u2 in members and cls[u] is not cls[u2]:
            merged = cls[u] | cls[u2]
            for x in merged:
                cls[x] = merged
    label = [0xFFFFFFFF] * g.nU
    roots = set()
    for u in members:
        label[u] = min(cls[u])
        roots.add(label[u])
    return label, len(roots)


def edge_butterflies(g):
    """Per-edge butterfly counts from the 4-tuples (notation table): each
    butterfly (u, u', v, v') adds one to each of its four edges.  Returned in the
    U-side CSR order of g (position of (u, v) in g.adj_u)."""
    _, _, _, tuples = butterflies(g)
    c = {}
    for (u, u2, v, v2) in tuples:
        for e in ((u, v), (u, v2), (u2, v), (u2, v2)):
            c[e] = c.get(e, 0) + 1
    return [c.get((u, int(g.adj_u[e])), 0) for u in range(g.nU) for e in range(int(g.off_u[u]), int(g.off_u[u + 1]))]


def wing_by_definition(g):
    """Wing number of every edge by Definition 1 and the wing-number
    definition: θ_e = the largest k such that e survives the iterated
    removal of edges in fewer than k butterflies of the remaining subgraph (the
    maximal subgraph in which every edge has >= k butterflies; connectivity splits
    it into k-wings but does not change which edges it holds).  From the 4-tuples,
    U-side CSR order."""
    _, _, _, tuples = butterflies(g)
    edges = [(u, int(g.adj_u[e])) for u in range(g.nU) for e in range(int(g.off_u[u]), int(g.off_u[u + 1]))]
    bfs = [((u, v), (u, v2), (u2, v), (u2, v2)) for (u, u2, v, v2) in tuples]
    theta = {e: 0 for e in edges}
    k = 1
    while True:
        live = set(edges)
        while True:
            cnt = {e: 0 for e in live}
            for b in bfs:
                if all(x in live for x in b):
                    for x in b:
                        cnt[x] += 1
            drop = {e for e in live if cnt[e] < k}
            if not drop:
                break
            live -= drop
        if not live:
            break
        for e in live:
            theta[e] = k
        k += 1
    return [theta[e] for e in edges]
