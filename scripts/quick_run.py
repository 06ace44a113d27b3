"""Development helper: run count + tip decomposition on a config, print stats and device times.
Usage: python scripts/quick_run.py CFG [P] [--opts N] [--reps R]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402
import graphgen as gg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("P", nargs="?", type=int, default=None)
    ap.add_argument("--opts", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--count-only", action="store_true")
    ap.add_argument("--sha", action="store_true", help="also print SHA-256 of θ (caller labels)")
    args = ap.parse_args()
    entry.build()
    import paper_2110_12511_b200 as pb
    cfg = args.cfg if args.cfg == "2a" else int(args.cfg)
    t = time.time()
    g, P = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
    P = args.P or P
    print(f"gen {time.time() - t:.1f}s nU={g.nU} nV={g.nV} m={g.m}", flush=True)
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    for r in range(args.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if args.count_only:
            pb.pbng_count_butterflies(d)
            st = {}
        else:
            tip, st = pb.pbng_tip_decompose(d, P, opts=args.opts)
        e1.record()
        torch.cuda.synchronize()
        if args.sha and not args.count_only:
            import hashlib
            st = dict(st, theta_sha256=hashlib.sha256(pb.as_u64(tip).tobytes()).hexdigest())
        print(json.dumps({"rep": r, "ms": e0.elapsed_time(e1), **st}), flush=True)


if __name__ == "__main__":
    main()
