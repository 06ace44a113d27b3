"""Time BE-Index construction + wing decomposition (pbng_wing_decompose, SURVEY §8(f)
f3/f4) on a BASELINE config: CUDA-event time of the call (median of --reps after one
warm-up), blooms, twin pairs, level scans, peeling rounds; with --oracle the oracle's
Alg.2 BUP time and bit-exact comparison (configs 1-2 only: BUP wing is slow).
Usage: python scripts/wing_run.py CFG [--reps 3] [--oracle]  -> one JSON line."""
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
    ap.add_argument("--oracle", action="store_true")
    args = ap.parse_args()
    entry.build()
    import paper_2110_12511_b200 as pb
    cfg = args.cfg if args.cfg == "2a" else int(args.cfg)
    g, _ = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    out = torch.empty(g.m, dtype=torch.int64, device="cuda")
    pb.pbng_wing_decompose(d, out=out)
    ms = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        _, info = pb.pbng_wing_decompose(d, out=out, stream=torch.cuda.current_stream())
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    th = pb.as_u64(out)
    rec = {"cfg": str(cfg), "m": int(g.m), "ms": float(np.median(ms)), "ms_all": ms, **info,
           "max_wing": int(th.max()) if g.m else 0, "distinct_wing": int(np.unique(th).shape[0])}
    if args.oracle:
        import oracle
        t = time.time()
        want = oracle.bup_wing(g)
        rec["oracle_s"] = time.time() - t
        rec["oracle_equal"] = bool(np.array_equal(th, want))
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
