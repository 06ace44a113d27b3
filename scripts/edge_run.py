"""Time per-edge butterfly counting (pbng_count_edge_butterflies) on a
BASELINE config: CUDA-event time of the call on the current stream (median of --reps after
one warm-up), Alg.1 wedges expanded, starts per tier, and a sampled oracle check (per-edge
counts of --check sampled U vertices' edges via the oracle on the full graph is too slow;
instead Σ_e ⋈_e = 2·Σ_u ⋈_u against the GPU per-vertex count, which is oracle-checked).
Usage: python scripts/edge_run.py CFG [--reps 3]  -> one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402
import graphgen as gg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-check", action="store_true")
    args = ap.parse_args()
    entry.build()
    import paper_2110_12511_b200 as pb
    cfg = args.cfg if args.cfg == "2a" else int(args.cfg)
    t = time.time()
    g, _ = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
    gen = time.time() - t
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    out = torch.empty(g.m, dtype=torch.int64, device="cuda")
    pb.pbng_count_edge_butterflies(d, out=out)
    ms = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        _, info = pb.pbng_count_edge_butterflies(d, out=out, stream=torch.cuda.current_stream())
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ec = pb.as_u64(out)
    sv = pb.as_u64(pb.pbng_count_butterflies(d))
    ok = int(ec.sum(dtype=np.uint64)) == 2 * int(sv.sum(dtype=np.uint64))
    med = float(np.median(ms))
    print(json.dumps({"cfg": str(cfg), "m": int(g.m), "nU": g.nU, "nV": g.nV, "ms": med, "ms_all": ms,
                      "wedges": info["wedges"], "wedges_per_s": info["wedges"] / (med / 1e3), "tiers": info["tiers"],
                      "sum_edges_eq_2_sum_vertex": ok, "butterflies": int(sv.sum(dtype=np.uint64)) // 2,
                      "gen_s": gen}))


if __name__ == "__main__":
    main()
