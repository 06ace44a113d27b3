"""A/B check: wing numbers of a config from the device-driven peel (default) and the host-driven
round loop (PBNG_WING_HOST=1) must be identical.  Usage: python scripts/wing_ab.py CFG"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import __graft_entry__ as entry  # noqa: E402
import graphgen as gg  # noqa: E402


def main():
    cfg = sys.argv[1] if sys.argv[1] == "2a" else int(sys.argv[1])
    entry.build()
    import paper_2110_12511_b200 as pb
    g, _ = gg.config(cfg, cache_dir=os.environ.get("PBNG_CACHE"))
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    os.environ.pop("PBNG_WING_HOST", None)
    th_d, info_d = pb.pbng_wing_decompose(d)
    os.environ["PBNG_WING_HOST"] = "1"
    th_h, info_h = pb.pbng_wing_decompose(d)
    a, b = pb.as_u64(th_d), pb.as_u64(th_h)
    print(json.dumps({"cfg": str(cfg), "equal": bool(np.array_equal(a, b)), "info_device": info_d, "info_host": info_h,
                      "theta_sha256": hashlib.sha256(a.tobytes()).hexdigest()}))


if __name__ == "__main__":
    main()
