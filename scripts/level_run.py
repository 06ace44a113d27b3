"""Measurement helper for k-tip level retrieval (pbng_tip_components):
decompose a config once (untimed), then time level extraction at several k with CUDA events.
Usage: python scripts/level_run.py CFG [--reps R]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402
import graphgen as gg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--oracle-frac", type=float, default=0.0,
                    help="also run oracle.tip_level (timed, compared) at levels with <= this fraction of U")
    args = ap.parse_args()
    entry.build()
    import paper_2110_12511_b200 as pb
    cfg = args.cfg if args.cfg == "2a" else int(args.cfg)
    g, P = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    tip, _ = pb.pbng_tip_decompose(d, P)
    th = pb.as_u64(tip)
    pos = np.sort(th[th > 0])
    ks = [0, 1] + [int(pos[int(q * (len(pos) - 1))]) for q in (0.5, 0.9, 0.99, 0.999)] if len(pos) else [0]
    for k in ks:
        ms = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lab, n = pb.pbng_tip_components(d, tip, k)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        members = int((th >= k).sum())
        labs = lab.cpu().numpy().view(np.uint32)
        big = int(np.bincount(labs[labs != 0xFFFFFFFF]).max()) if members else 0
        row = {"cfg": str(cfg), "k": k, "members": members, "ktips": n, "largest": big,
               "ms_median": float(np.median(ms)), "ms": [round(x, 2) for x in ms]}
        if members <= args.oracle_frac * g.nU:
            import time
            import oracle
            t0 = time.time()
            want, wn = oracle.tip_level(g, th, k)
            row["oracle_s"] = round(time.time() - t0, 2)
            row["parity"] = bool(np.array_equal(labs, want) and wn == n)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
