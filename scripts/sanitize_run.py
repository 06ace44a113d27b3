"""compute-sanitizer workload (memcheck / racecheck / synccheck; VERDICT r1 "robustness").

Runs every entry point and option family of libpbng on small graphs and checks each
result against the oracle, so a sanitizer run is also a parity run:
  * tiny seeded corpus, both sides, P in {1, 3};
  * configs 1, 2, 2a: count, decompose with opts 0 / ONESIDED_COUNT / NO_DELETE /
    FORCE_RECOUNT / FD_GRID, pbng_tip_plan, pbng_tip_components at a few levels.
With PBNG_LIB pointing at the small-table test build (tests/test_gpu_variants.py SMALL)
every aggregation path (warp / hash groups / pass-on / bitmap windows / repeat overflow /
dense windows) fires on these graphs.
Usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py [--quick]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_2110_12511_b200 as pb  # noqa: E402


def dev(g):
    return pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="config 1 + 10 tiny graphs only (racecheck)")
    args = ap.parse_args()
    tot = {"impl": [0] * 4, "impl_hash": [0] * 4, "runs": 0}

    def add(st):
        for k in ("impl", "impl_hash"):
            tot[k] = [a + b for a, b in zip(tot[k], st[k])]
        tot["runs"] += 1

    rng = np.random.default_rng(4242)
    for i in range(10 if args.quick else 30):
        nu, nv = int(rng.integers(1, 14)), int(rng.integers(1, 14))
        g = gg.uniform(nu, nv, int(rng.integers(0, nu * nv + 1)), seed=4242 + i)
        d = dev(g)
        for side, gs in ((0, g), (1, g.swapped())):
            for P in (1, 3):
                tip, st = pb.pbng_tip_decompose(d, P, side=side)
                assert np.array_equal(pb.as_u64(tip), oracle.bup_tip(gs)), (g.name, side, P)
                add(st)
    for cfg in ((1,) if args.quick else (1, 2, "2a")):
        g, P = gg.config(cfg)
        d = dev(g)
        assert np.array_equal(pb.as_u64(pb.pbng_count_butterflies(d)), oracle.count(g)), cfg
        want = oracle.bup_tip(g)
        for opts in (0, pb.OPT_ONESIDED_COUNT, pb.OPT_NO_DELETE, pb.OPT_FORCE_RECOUNT, pb.OPT_FD_GRID,
                     pb.OPT_NO_DELETE | pb.OPT_NO_RECOUNT):
            tip, st = pb.pbng_tip_decompose(d, P, opts=opts)
            assert np.array_equal(pb.as_u64(tip), want), (cfg, opts)
            add(st)
        part, init, bounds, nparts = pb.pbng_tip_plan(d, P)
        assert nparts >= 1 and all(bounds[i] < bounds[i + 1] for i in range(nparts))
        levels = sorted(set(int(x) for x in want))
        for k in levels[:: max(1, len(levels) // 3)]:
            lab, n = pb.pbng_tip_components(d, tip, k)
            wl, wn = oracle.tip_level(g, want, k)
            assert n == wn and np.array_equal(lab.cpu().numpy().view(np.uint32), wl), (cfg, k)
    print(json.dumps(tot))


if __name__ == "__main__":
    main()
