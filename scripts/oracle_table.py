"""Per-config table: GPU tip decomposition seconds beside the full CPU oracle's
(oracle_bup_tip: plain one-sided count + sequential bottom-up peeling, one thread),
the T4 layout of the paper (BUP time beside PBNG time).

Each line: cfg, sizes, oracle seconds, GPU seconds (median of 3 after one warm-up, CUDA
events, CSR resident), their ratio, and θ equality.
Usage: python scripts/oracle_table.py [--cfgs 1,2,2a,3[,4]] [--out FILE]
"""
import argparse
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402
import graphgen as gg  # noqa: E402
import oracle  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="1,2,2a,3")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "oracle_table.jsonl"))
    args = ap.parse_args()
    entry.build()
    import paper_2110_12511_b200 as pb
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    for c in args.cfgs.split(","):
        cfg = c if c == "2a" else int(c)
        g, P = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
        d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
        ms = []
        for _ in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tip, st = pb.pbng_tip_decompose(d, P)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        gpu_s = statistics.median(ms[1:]) / 1e3
        th = pb.as_u64(tip)
        t = time.time()
        want = oracle.bup_tip(g)
        cpu_s = time.time() - t
        row = {"cfg": str(cfg), "nU_peel": g.nU, "nV": g.nV, "edges": g.m, "P": P,
               "gpu_seconds": round(gpu_s, 5), "oracle_seconds": round(cpu_s, 3),
               "oracle_over_gpu": round(cpu_s / gpu_s, 1), "theta_equal": bool(np.array_equal(th, want)),
               "gpu_wedges": st["wedges_count"] + st["wedges_cd"] + st["wedges_fd"],
               "oracle": "oracle_bup_tip, single thread", "cpu": cpu_model(), "nproc": os.cpu_count()}
        print(json.dumps(row), flush=True)
        with open(args.out, "a") as f:
            f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
