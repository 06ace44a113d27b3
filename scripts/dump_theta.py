"""Dump the GPU tip numbers of a config for the offline exactness certificate
(scripts/certify_offline.py runs oracle/certificate.c on them on a CPU box).

Writes gpurun_out/theta_cfg{C}.npz: the distinct θ values and, per vertex (caller
labels), the index of its value, lzma-compressed in parts small enough for the
64 MiB gpurun transfer; plus SHA-256 of θ and of the GPU butterfly counts.
Usage: python scripts/dump_theta.py CFG [--max-mb 60]
"""
import argparse
import hashlib
import json
import lzma
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
    ap.add_argument("--max-mb", type=float, default=60.0)
    ap.add_argument("--skip-parts", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out")
    args = ap.parse_args()
    entry.build()
    import paper_2110_12511_b200 as pb
    cfg = args.cfg if args.cfg == "2a" else int(args.cfg)
    g, P = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    t = time.time()
    tip, st = pb.pbng_tip_decompose(d, P)
    torch.cuda.synchronize()
    th = pb.as_u64(tip)
    sup = pb.as_u64(pb.pbng_count_butterflies(d))
    info = {"cfg": str(cfg), "graph_sha256": g.sha256(), "nU": g.nU, "P": P,
            "theta_sha256": hashlib.sha256(th.tobytes()).hexdigest(),
            "support_sha256": hashlib.sha256(sup.tobytes()).hexdigest(),
            "theta_le_support": bool(np.all(th <= sup)), "decompose_s": time.time() - t,
            "stats": {k: v for k, v in st.items() if k != "ms_kernel"}}
    vals, idx = np.unique(th, return_inverse=True)
    idx = idx.astype(np.uint32)
    info["distinct"] = int(vals.shape[0])
    os.makedirs(args.out, exist_ok=True)
    raw = idx.tobytes()
    # parts of at most --max-mb compressed, cut by vertex range
    n = g.nU
    nparts = 1
    while True:
        step = (n + nparts - 1) // nparts
        blob0 = lzma.compress(idx[:step].tobytes(), preset=6)
        if len(blob0) <= args.max_mb * 2**20 or nparts >= 64:
            break
        nparts *= 2
    info["parts"] = nparts
    info["part_vertices"] = step
    written = 0
    for p in range(nparts):
        if p < args.skip_parts:
            continue
        blob = blob0 if p == 0 else lzma.compress(idx[p * step:(p + 1) * step].tobytes(), preset=6)
        if written + len(blob) > args.max_mb * 2**20:
            break
        with open(os.path.join(args.out, f"theta_cfg{cfg}_part{p}.xz"), "wb") as f:
            f.write(blob)
        written += len(blob)
        info.setdefault("written_parts", []).append(p)
    np.save(os.path.join(args.out, f"theta_cfg{cfg}_values.npy"), vals)
    del raw
    with open(os.path.join(args.out, f"theta_cfg{cfg}.json"), "w") as f:
        json.dump(info, f, indent=1)
    print(json.dumps({k: v for k, v in info.items() if k != "stats"}))


if __name__ == "__main__":
    main()
