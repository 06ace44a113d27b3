"""Offline exactness certificate of GPU tip numbers (oracle/certificate.c).

Input: gpurun_out/[cfg4/]theta_cfg{C}_part*.xz + _values.npy + .json written on the GPU box
by scripts/dump_theta.py (θ of pbng_tip_decompose in caller labels, SHA-256 of θ and of the
GPU butterfly counts).  The graph is regenerated here from the seeded generator (its SHA-256
must equal the one recorded on the GPU box).  Runs only oracle/ code:
  * oracle.cert_one_pass: full butterfly counts (each unordered pair once) and the (A) sums
    s_ge, then (C) on every level;
  * (A) s_ge >= θ for every vertex, (C) on every level;
  * SHA-256 of the oracle's counts against the GPU's.
Writes profiles/r2_certificate_cfg{C}.json.  Usage: python scripts/certify_offline.py CFG [dir]
"""
import hashlib
import json
import lzma
import os
import platform
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402


def main():
    cfg = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    cache = os.environ.get("PBNG_CACHE", os.path.join(ROOT, "data"))
    info = json.load(open(os.path.join(src, f"theta_cfg{cfg}.json")))
    vals = np.load(os.path.join(src, f"theta_cfg{cfg}_values.npy"))
    idx = np.concatenate([np.frombuffer(lzma.decompress(open(os.path.join(src, f"theta_cfg{cfg}_part{p}.xz"), "rb")
                                                        .read()), np.uint32) for p in range(info["parts"])])
    th = np.ascontiguousarray(vals[idx], np.uint64)
    assert hashlib.sha256(th.tobytes()).hexdigest() == info["theta_sha256"], "θ transfer corrupted"
    t0 = time.time()
    g, P = gg.config(int(cfg) if cfg != "2a" else cfg, cache_dir=cache)
    assert g.sha256() == info["graph_sha256"], "regenerated graph differs from the GPU box's"
    print(f"graph cfg{cfg} nU={g.nU} m={g.m} ({time.time() - t0:.0f}s)", flush=True)
    prog = np.zeros(1, np.uint64)
    done = threading.Event()

    def report():
        while not done.wait(300):
            print(f"  {time.time() - t1:.0f}s: {int(prog[0])}/{g.nU} vertices", flush=True)

    t1 = time.time()
    threading.Thread(target=report, daemon=True).start()
    sup, sge, bad, first = oracle.cert_one_pass(g, th, progress=prog)
    done.set()
    secs = time.time() - t1
    a_ok = bool(np.all(sge >= th))
    out = {
        "cfg": cfg, "graph_sha256": info["graph_sha256"], "nU": g.nU, "m": g.m, "P": P,
        "theta_sha256": info["theta_sha256"], "distinct_levels": int(vals.shape[0]),
        "A_every_vertex_sge_ge_theta": a_ok, "A_violations": int(np.sum(sge < th)),
        "C_levels_checked": int(vals.shape[0]), "C_failing_levels": bad, "C_first_failing_level": first,
        "certified_exact": a_ok and bad == 0,
        "oracle_support_sha256": hashlib.sha256(sup.tobytes()).hexdigest(),
        "gpu_support_sha256": info["support_sha256"],
        "counts_equal": hashlib.sha256(sup.tobytes()).hexdigest() == info["support_sha256"],
        "theta_le_oracle_support": bool(np.all(th <= sup)),
        "total_butterflies": int(sup.sum(dtype=np.uint64)) // 2,
        "seconds": round(secs, 1), "cores": os.cpu_count(), "cpu": platform.processor() or platform.machine(),
        "how": "oracle.cert_one_pass (oracle/certificate.c, OpenMP): counts + (A) in one pass over unordered "
               "pairs, (C) on every level over the induced level runs; θ from the GPU box (scripts/dump_theta.py)",
    }
    with open(os.path.join(ROOT, "profiles", f"r2_certificate_cfg{cfg}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    main()
