"""Runs per-edge counting of a test build of libpbng (tiny tier bounds, so the CTA-hash
and both dense-counter paths fire on small graphs) against oracle.edge_count.  Invoked by
tests/test_gpu_edge.py with PBNG_LIB pointing at the variant; prints one JSON line with
the starts routed per tier and raises on any mismatch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_2110_12511_b200 as pb  # noqa: E402


def main():
    tiers = [0, 0, 0]
    graphs = [gg.config(c)[0] for c in (1, 2, "2a")]
    graphs += [gg.chung_lu(3000, 2000, 40000, 2.0, 2.0, 2000, 2000, seed=17)]
    for g in graphs:
        d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
        for side, gs in ((0, g), (1, g.swapped())):
            ec, info = pb.pbng_count_edge_butterflies(d, side=side)
            assert np.array_equal(pb.as_u64(ec), oracle.edge_count(gs)), (g.name, side)
            tiers = [a + b for a, b in zip(tiers, info["tiers"])]
    print(json.dumps({"tiers": tiers}))


if __name__ == "__main__":
    main()
