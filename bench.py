"""bench.py — PBNG tip decomposition on B200: wedges/s, seconds per decomposition, % of HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl pbng|reference]

One "step" = one full tip decomposition (count + CD + FD, every §8(a) row) of the
workload graph through the C ABI (pbng_tip_decompose) with the CSR already in HBM.
N > 1 (torchrun): every rank decomposes its own replica (the path does not shard —
DESIGN.md "replicas only"); value = wedges of all ranks / max-over-ranks time.
`--impl reference` times the CPU oracle (oracle/, single thread: plain count +
sequential bottom-up peeling) decomposing a bounded sample of the same workload
(the subgraph induced by a seeded 1% sample of the peel side with all of V)
instead.  Prints ONE JSON line on rank 0.

Timing: K steps with no instrumentation (opts = 0; the library's work counters
are always filled).  Then one separate stats step (PBNG_OPT_STATS_DEFER: a CUDA
event pair around every launch, on the launch stream) gives the device time per
kernel family for the roofline; its own duration is reported beside the timed
steps so the cost of the events is visible.
"""
from __future__ import annotations

import argparse
import fcntl
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "tip-decomposition wedges/sec"
UNIT = "wedges/s"
DEFAULT_CONFIG = "5"  # the largest config (BASELINE.json north_star: the HBM target is stated on it)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def locked_build():
    import __graft_entry__ as entry
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", ".build.lock"), "w") as f:
        fcntl.flock(f, fcntl.LOCK_EX)
        entry.build()
        fcntl.flock(f, fcntl.LOCK_UN)


def load_graph(cfg):
    """Seeded synthetic workload.  Configs >= 4 are cached on local disk (outside
    any timed region) so replicas / reruns skip the minute-long generation; the
    file name carries the generator version, and one process writes it under a lock."""
    import graphgen as gg
    c = cfg if cfg == "2a" else int(cfg)
    t = time.time()
    cache = os.environ.get("PBNG_CACHE")
    if cache is None and c not in ("2a",) and int(c) >= 4:
        cache = os.path.join("/tmp", f"pbng_graph_cache_{gg.GENERATOR_VERSION}")
    if cache:
        os.makedirs(cache, exist_ok=True)
        with open(os.path.join(cache, f".lock{c}"), "w") as lf:
            fcntl.flock(lf, fcntl.LOCK_EX)
            g, P = gg.config(c, cache_dir=cache)
            fcntl.flock(lf, fcntl.LOCK_UN)
    else:
        g, P = gg.config(c)
    return g, P, time.time() - t


def workload_desc(cfg, g, P):
    import graphgen as gg
    spec = gg.CONFIGS[cfg if cfg == "2a" else int(cfg)]
    return {"workload": f"BASELINE config {cfg}", "nU_peel": g.nU, "nV": g.nV, "edges": g.m, "P": P,
            "peel_side": g.name, "side_rule": spec["side"], "generator": "graphgen R1 (DESIGN.md input recipe)"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, r[4:8]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- oracle arm
def host_cpu():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def induced_sample(g, frac, seed=2110):
    """Subgraph induced by a seeded random `frac` of the peel-side vertices and all of V
    (the same degree structure, thinned): a bounded decomposition for the CPU oracle."""
    import graphgen as gg
    rng = np.random.default_rng(seed)
    keep = rng.random(g.nU) < frac
    new_id = np.cumsum(keep) - 1
    du = np.diff(g.off_u.astype(np.int64))
    u_of_e = np.repeat(np.arange(g.nU, dtype=np.int64), du)
    sel = keep[u_of_e]
    edges = np.stack([new_id[u_of_e[sel]], g.adj_u[sel].astype(np.int64)], axis=1)
    return gg.from_edges(int(keep.sum()), g.nV, edges)


def time_oracle_bup(sub):
    """Seconds and wedges of the oracle's full decomposition (count + bottom-up peeling) of `sub`."""
    import oracle
    st = oracle.Stats()
    t = time.perf_counter()
    oracle.bup_tip(sub, st)
    dt = time.perf_counter() - t
    return dt, st.wedges


def oracle_sample(g, target_wedges, seed=12345):
    """Seeded random sample of peel-side vertices whose traversal totals ~target_wedges."""
    du = np.diff(g.off_u.astype(np.int64))
    dv = np.diff(g.off_v.astype(np.int64))
    u_of_e = np.repeat(np.arange(g.nU), du)
    wc = np.bincount(u_of_e, weights=dv[g.adj_u.astype(np.int64)], minlength=g.nU)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(g.nU)
    cum = np.cumsum(wc[perm])
    k = int(np.searchsorted(cum, target_wedges)) + 1
    return np.sort(perm[:k]).astype(np.uint32), float(cum[min(k, len(cum)) - 1])


def time_oracle(g, target_wedges):
    import oracle
    us, _ = oracle_sample(g, target_wedges)
    st = oracle.Stats()
    t = time.perf_counter()
    oracle.count_subset(g, us, st)
    dt = time.perf_counter() - t
    return st.wedges / dt, dt, len(us), st.wedges


def sample_desc(g, sub, frac, wedges, secs):
    return (f"oracle_bup_tip (plain one-sided count + sequential bottom-up peeling, oracle/oracle.c) decomposing "
            f"the subgraph induced by a seeded {frac:.0%} sample of the workload's peel side with all of V "
            f"(nU={sub.nU} of {g.nU}, m={sub.m}); {wedges} oracle wedges in {secs:.1f} s; single thread")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build_lib()
    g, P, _ = load_graph(args.config)
    sub = induced_sample(g, args.ref_frac)
    for _ in range(min(args.warmup, 1)):  # the oracle has no warm-up effects beyond page-in
        time_oracle_bup(sub)
    secs, wsum = 0.0, 0
    for _ in range(args.steps):
        dt, w = time_oracle_bup(sub)
        secs += dt
        wsum += w
    value = wsum / secs
    sample = sample_desc(g, sub, args.ref_frac, wsum // args.steps, secs / args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "uint64",
            "data": "synthetic", "config": workload_desc(args.config, g, P),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- replicas (N > 1)
def max_over_ranks(ms: float, dist=None, device="cpu") -> float:
    """Device-measured time of this rank -> max over all ranks (the job's time)."""
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_rate(units_per_rank: float, world: int, max_ms: float) -> float:
    """Whole-job throughput: the units every rank processed / the slowest rank's time."""
    return world * units_per_rank / (max_ms / 1000.0)


# ---------------------------------------------------------------- GPU arm
def roofline(stats_list, peaks):
    """Dominant kernel family: the wedge aggregation (k_agg_warp/cta/heavy tiers)."""
    ms = {}
    for st in stats_list:
        for k, v in st["ms_kernel"].items():
            ms[k] = ms.get(k, 0.0) + v
    agg_ms = sum(ms.get(k, 0.0) for k in ("agg_warp", "agg_cta", "agg_hash"))
    dominant = max(ms, key=ms.get) if ms else None
    W = sum(s["wedges_count"] + s["wedges_cd"] for s in stats_list)
    S = sum(s["uv_steps"] - s["uv_steps_fd"] for s in stats_list)
    # A = CD support decrements that reached partners still live (A_live, impl[3] of the stats
    # step); decrements to partners peeled in the same batch or not yet compacted away are
    # harmless extra work and are not counted as useful bytes
    A = sum(s["impl"][3] for s in stats_list)
    A_all = sum(s["support_updates"] - s["updates_fd"] for s in stats_list)
    bytes_alg = 4 * W + 20 * S + 20 * A  # 4 B/wedge, 20 B/(u,v) step, 20 B/update
    achieved = bytes_alg / (agg_ms / 1000) / 1e9 if agg_ms else 0.0
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # DRAM bytes of one captured launch of the dominant kernel (ncu --set full, committed
    # under profiles/), with that launch's algorithmic bytes beside it
    traffic, traffic_note = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath))
            traffic = t["dram_bytes_per_launch"]
            traffic_note = {k: t[k] for k in ("kernel", "launch", "alg_bytes_per_launch", "dram_over_alg", "source")
                            if k in t}
        except Exception:
            traffic = None
    return {"kernel": "wedge aggregation family: k_agg_warp / k_agg_hash / k_agg_win and the vertex-priority "
                      "k_vp_agg_* (count + CD peel), device time from the stats step", "bound": "hbm",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_launch": traffic_note, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks
            else "fallback 6650 GB/s (B200_PROFILING.md)",
            "bytes_alg_per_step": bytes_alg / max(1, len(stats_list)),
            "terms": {"W_wedges": W, "S_uv_steps": S, "A_live_updates": A, "A_all_cd_updates": A_all,
                      "formula": "4*W + 20*S + 20*A_live"}, "agg_ms_per_step": agg_ms / max(1, len(stats_list)),
            "dominant_family_by_time": dominant, "ms_by_family_per_step":
                {k: v / max(1, len(stats_list)) for k, v in sorted(ms.items(), key=lambda kv: -kv[1])}}


def run_gpu(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    locked_build()
    import paper_2110_12511_b200 as pb
    g, P, gen_s = load_graph(args.config)
    log(f"[rank {rank}] graph {g.name}: nU={g.nU} nV={g.nV} m={g.m} P={P} (gen {gen_s:.1f}s)")
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2
    out = torch.empty(g.nU, dtype=torch.int64, device=f"cuda:{local}")
    opts = 0  # timed steps carry no instrumentation
    for i in range(args.warmup):
        pb.pbng_tip_decompose(d, P, opts=opts, out=out)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    stats, total_ms = [], 0.0
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the event pair)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, st = pb.pbng_tip_decompose(d, P, opts=opts, out=out)
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
        stats.append(st)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    # ---- stats step (outside the timed region): device time per kernel family
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, st_stats = pb.pbng_tip_decompose(d, P, opts=pb.OPT_STATS_DEFER, out=out)
    e1.record(stream)
    e1.synchronize()
    stats_step_ms = e0.elapsed_time(e1)
    st_stats["ms_kernel"] = pb.pbng_kernel_times()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    wedges_step = stats[-1]["wedges_count"] + stats[-1]["wedges_cd"] + stats[-1]["wedges_fd"]
    max_ms = max_over_ranks(total_ms, dist, device=f"cuda:{local}")
    value = job_rate(wedges_step * args.steps, world, max_ms)
    # ---- end to end through the host-buffer C ABI entry point (pinned host CSR in, θ out)
    e2e = None
    if not args.no_e2e:
        pin = [torch.from_numpy(np.ascontiguousarray(a).view(dt)).pin_memory()
               for a, dt in ((g.off_u, np.int64), (g.adj_u, np.int32), (g.off_v, np.int64), (g.adj_v, np.int32))]
        hv = [p.numpy() for p in pin]
        tip_host = torch.empty(g.nU, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        # the device path above already warmed every kernel and the memory pool
        e2e_steps = min(args.steps, 2)
        e2e_ms = 0.0
        for i in range(e2e_steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pb.pbng_tip_decompose_host(hv[0].view(np.uint64), hv[1].view(np.uint32), hv[2].view(np.uint64),
                                       hv[3].view(np.uint32), P, out=tip_host)
            e1.record(stream)
            e1.synchronize()
            e2e_ms += e0.elapsed_time(e1)
        e2e_max = max_over_ranks(e2e_ms, dist, device=f"cuda:{local}")
        e2e = {"value": job_rate(wedges_step * e2e_steps, world, e2e_max), "unit": UNIT,
               "h2d_bytes_per_step": int(sum(p.numel() * p.element_size() for p in pin)),
               "d2h_bytes_per_step": int(g.nU * 8),
               "seconds_per_decomposition": e2e_max / 1000 / e2e_steps, "steps": e2e_steps,
               "api": "pbng_tip_decompose_host (C ABI, pinned host buffers)"}
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    peaks = {}
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        peaks = json.load(open(pp))
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build_lib()
        sub = induced_sample(g, args.ref_frac)
        dt, w = time_oracle_bup(sub)
        cpu = {"value": w / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": sample_desc(g, sub, args.ref_frac, w, dt), **host_cpu()}
    st = stats[-1]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "uint64", "data": "synthetic",
        "config": {**workload_desc(args.config, g, P), "l2": "256 MiB buffer written between timed steps",
                   "parallelism": "replicas" if world > 1 else "single GPU"},
        "seconds_per_decomposition": max_ms / args.steps / 1000,
        "e2e": e2e, "gpu_launches": int(sum(s["launches"] for s in stats)),
        "roofline": {**roofline([st_stats], peaks), "stats_step_ms": stats_step_ms}, "cpu_baseline": cpu,
        "clocks": clocks,
        "detail": {"wedges_per_step": wedges_step, "wedges_count": st["wedges_count"], "wedges_cd": st["wedges_cd"],
                   "wedges_fd": st["wedges_fd"], "rho_cd_iters": st["rho_cd_iters"],
                   "partitions_used": st["partitions_used"], "recounts": st["recounts"],
                   "fd_rounds_max": st["fd_rounds_max"], "support_updates": st["support_updates"],
                   "impl_win": st["impl"], "impl_hash": st["impl_hash"],
                   "ms_phase": {"count": st["ms_count"], "cd": st["ms_cd"], "fd_build": st["ms_fd_build"],
                                "fd": st["ms_fd"]}, "gen_seconds": gen_s},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_ablation(args):
    """Paper §5 optimisations on the workload (shape of fig:optTip):
    PBNG (all), PBNG- (no dynamic deletion), PBNG-- (no deletion, no batch re-count),
    and one-sided instead of vertex-priority counting; both peel sides.  One JSON
    line per variant (not the driver's metric line)."""
    import torch
    locked_build()
    import paper_2110_12511_b200 as pb
    g, P, _ = load_graph(args.config)
    variants = [("PBNG", 0), ("PBNG-", pb.OPT_NO_DELETE), ("PBNG--", pb.OPT_NO_DELETE | pb.OPT_NO_RECOUNT),
                ("PBNG+onesided-count", pb.OPT_ONESIDED_COUNT)]
    d = pb.DeviceGraph.from_numpy(g.off_u, g.adj_u, g.off_v, g.adj_v)
    for side in (0, 1):
        for name, opts in variants:
            pb.pbng_tip_decompose(d, P, side=side, opts=opts | pb.OPT_STATS)
            secs = []
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _, st = pb.pbng_tip_decompose(d, P, side=side, opts=opts | pb.OPT_STATS)
                e1.record()
                e1.synchronize()
                secs.append(e0.elapsed_time(e1) / 1000)
            w = st["wedges_count"] + st["wedges_cd"] + st["wedges_fd"]
            print(json.dumps({"ablation": name, "config": workload_desc(args.config, g, P), "side": side,
                              "seconds": statistics.median(secs), "seconds_all": secs, "wedges": w,
                              "wedges_count": st["wedges_count"], "wedges_cd": st["wedges_cd"],
                              "wedges_fd": st["wedges_fd"], "rho_cd_iters": st["rho_cd_iters"],
                              "recounts": st["recounts"]}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("PBNG_BENCH_CONFIG", DEFAULT_CONFIG))
    ap.add_argument("--impl", default="pbng", choices=["pbng", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-wedges", type=float, default=5e8, help="(unused; kept for old scripts)")
    ap.add_argument("--ref-frac", type=float, default=0.01,
                    help="peel-side fraction of the induced sample the oracle decomposes")
    ap.add_argument("--ablation", action="store_true", help="PBNG / PBNG- / PBNG-- / one-sided count, both sides")
    args = ap.parse_args()
    if args.ablation:
        return run_ablation(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
