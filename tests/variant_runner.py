"""Runs the CUDA path of a test build of libpbng (small table / window constants, so that
the multi-group, pass-on, bitmap-window, repeat-overflow and dense paths fire on graphs the
oracle checks in seconds) against the oracle.  Invoked by tests/test_gpu_variants.py in a
subprocess with PBNG_LIB pointing at the variant; prints one JSON line of implementation
counters and raises on any mismatch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_2110_12511_b200 as pb  # noqa: E402


def tiny_corpus(n, seed0):
    rng = np.random.default_rng(seed0)
    for i in range(n):
        nu, nv = int(rng.integers(1, 14)), int(rng.integers(1, 14))
        yield gg.uniform(nu, nv, int(rng.integers(0, nu * nv + 1)), seed=seed0 + i)


def dev(g):
    return pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)


def add(tot, st):
    for k in ("impl", "impl_hash"):
        tot[k] = [a + b for a, b in zip(tot.get(k, [0] * 4), st[k])]


def main():
    tot = {}
    for g in tiny_corpus(40, 777):
        d = dev(g)
        for side, gs in ((0, g), (1, g.swapped())):
            for P in (1, 3):
                tip, st = pb.pbng_tip_decompose(d, P, side=side)
                assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs)), (g.name, side, P)
    for cfg in (1, 2, "2a"):
        g, P = gg.config(cfg)
        d = dev(g)
        assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(d)), oracle.count(g)), cfg
        want = oracle.bup_tip(g)
        for opts in (0, pb.OPT_ONESIDED_COUNT, pb.OPT_NO_DELETE, pb.OPT_FORCE_RECOUNT):
            tip, st = pb.pbng_tip_decompose(d, P, opts=opts)
            assert np.array_equal(pb.as_u64(tip), want), (cfg, opts)
            add(tot, st)
        tip_t = tip  # device tensor of the (verified) tip numbers
        levels = sorted(set(int(x) for x in want))
        for k in levels[:: max(1, len(levels) // 4)]:
            lab, n = pb.pbng_tip_components(d, tip_t, k)
            wl, wn = oracle.tip_level(g, want, k)
            assert n == wn and np.array_equal(lab.cpu().numpy().view(np.uint32), wl), (cfg, k)
    # config 3 (500K x 200K, 5M edges): full counts and the exactness certificate
    g, P = gg.config(3, cache_dir=os.environ.get("PBNG_CACHE"))
    d = dev(g)
    sup_gpu = pb.as_u64(pb.pbng_count_butterflies(d))
    for opts in (0, pb.OPT_ONESIDED_COUNT):
        tip, st = pb.pbng_tip_decompose(d, P, opts=opts)
        add(tot, st)
        th = pb.as_u64(tip)
        sup, sge, bad, first = oracle.cert_one_pass(g, th)
        assert np.array_equal(sup, sup_gpu), "config 3 counts"
        assert np.all(sge >= th) and bad == 0, ("config 3 certificate", opts, first)
    print(json.dumps(tot))


if __name__ == "__main__":
    main()
