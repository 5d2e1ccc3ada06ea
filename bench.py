#!/usr/bin/env python
"""Benchmark: mere-listing (orientation/CSR build + A+- listing) on B200.

One step = the hot path over one synthetic graph with pi given: tl_orient
(relabel, orient, CSR, segmented sort, cost) + tl_list (degree-binned A+-
with the count + checksum sinks). `value` = triangles listed per second over
the K timed steps, inputs resident in HBM (tl_orient_device), device time on
the engine's stream (CUDA events). `e2e` = the same through the C-ABI with
HOST buffers (pinned), host->device copies and the stats read-back inside the
timed region.

    python bench.py [--config c4] [--steps K] [--warmup W] [--gpus N]
    python bench.py --impl reference ...   # the reference CPU listing

Multi-GPU: the north star keeps the path on one GPU (no sharding, no
collectives), so N>1 runs N independent replicas ("replicas only",
DESIGN.md); value sums the replicas' work over the max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("triangles listed/sec and oriented edges/sec on 1 B200; "
          "achieved HBM GB/s vs roofline")

CONFIGS = {
    "c1": dict(kind="gnm", n=100_000, m=1_000_000, seed=4242,
               desc="C1 Erdos-Renyi G(100000, 1000000), gen_gnm seed 4242"),
    "c2": dict(kind="chung_lu", n=4_000_000, draws=64_000_000, seed=1,
               desc="C2 Chung-Lu n=4M, Pareto(2.1, min 2, cap 50000) weights, 64M draws"),
    "c3": dict(kind="ws", n=16_000_000, k=32, p=0.1, seed=1,
               desc="C3 Watts-Strogatz n=16M, k=32, p=0.1"),
    "c3_1m": dict(kind="ws", n=1_000_000, k=32, p=0.1, seed=1,
                  desc="C3 recipe at n=1M (full-list instance)"),
    "c4": dict(kind="rmat", scale=24, ef=16, seed=1,
               desc="C4 R-MAT scale 24, edge factor 16, (0.57,0.19,0.19,0.05)"),
    "c5": dict(kind="rmat", scale=27, ef=16, seed=1,
               desc="C5 R-MAT scale 27, edge factor 16, (0.57,0.19,0.19,0.05)"),
    "rmat20": dict(kind="rmat", scale=20, ef=16, seed=1, desc="R-MAT scale 20 (proxy)"),
}
DEFAULT_CONFIG = "c4"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_graph(cfg):
    import paper_2203_04774_b200 as tg
    k = cfg["kind"]
    if k == "gnm":
        return tg.gen_gnm(cfg["n"], cfg["m"], cfg["seed"])
    if k == "chung_lu":
        return tg.gen_chung_lu(cfg["n"], cfg["draws"], seed=cfg["seed"])
    if k == "ws":
        return tg.gen_ws(cfg["n"], cfg["k"], cfg["p"], seed=cfg["seed"])
    if k == "rmat":
        return tg.gen_rmat(cfg["scale"], cfg["ef"], cfg["seed"])
    raise ValueError(k)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def dist_setup(backend: str = "nccl"):
    """One process per GPU (torchrun env). The listing path does not shard
    (north star: one GPU, no collectives), so ranks are independent replicas;
    the process group only carries the barrier and the max-over-ranks time."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(units_per_rank: float, elapsed_ms: float, world: int) -> float:
    """Whole-job throughput of N replicas: all ranks' units over the
    max-over-ranks device time."""
    return world * units_per_rank / (allreduce_max(elapsed_ms, world) / 1e3)


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# -- reference CPU listing (oracle/_ref) on a bounded sample ---------------------

def bit_reversed(nblocks: int):
    bits = max(1, (nblocks - 1).bit_length())
    for i in range(1 << bits):
        j = int(format(i, f"0{bits}b")[::-1], 2)
        if j < nblocks:
            yield j


class ReferenceSample:
    """The reference's own A+- loops (listing.hpp:91-107 via run_parallel's
    1024-rank block pulling) over a spread sample of seed-rank blocks of the
    same graph and ordering, on all host cores. Full-workload time is
    extrapolated by inner_ops (the paper's cost model)."""

    def __init__(self, g, pi, budget_s: float, threads: int):
        import oracle
        self.oracle = oracle
        t0 = time.perf_counter()
        self.rg = oracle.RefGraph.from_csr(g.offsets, g.adjacency)
        self.view = oracle.RefView(self.rg, pi.ranks)
        self.setup_s = time.perf_counter() - t0
        self.threads = threads
        n = g.n
        nb = 256
        bs = (n + nb - 1) // nb
        self.blocks = []
        spent = 0.0
        # choose blocks until ~budget seconds of reference work (measured once)
        for b in bit_reversed(nb):
            lo, hi = b * bs, min(n, (b + 1) * bs)
            if lo >= hi:
                continue
            r = self.view.list(oracle.APM, threads=threads, rank_begin=lo, rank_end=hi)
            self.blocks.append((lo, hi))
            spent += r.wall_ms / 1e3
            if spent >= budget_s:
                break

    def run(self):
        ops = tri = 0
        ms = 0.0
        for lo, hi in self.blocks:
            r = self.view.list(self.oracle.APM, threads=self.threads, rank_begin=lo, rank_end=hi)
            ops += r.inner_ops
            tri += r.triangle_count
            ms += r.wall_ms
        return ops, tri, ms


class PortSample:
    """The oracle restatement of the same A+- loops (oracle/oracle.c <-
    listing.hpp:91-107, 122-155) over the GPU-built oriented view fetched in
    the reference layout, on a spread sample of seed-rank blocks. Used as the
    CPU baseline where building the reference's own Graph + OrientedView
    would take many minutes (C5: ~2 B edges, single-threaded constructors)."""

    def __init__(self, ctx, g, pi, budget_s: float, threads: int):
        import oracle
        self.oracle = oracle
        t0 = time.perf_counter()
        so, s_, po, p_ = ctx.fetch_oriented(g.n, g.m)
        self.view = oracle.OrientedCSR(so, s_, po, p_, pi.sequence, pi.ranks)
        self.setup_s = time.perf_counter() - t0
        self.threads = threads
        nb = 256
        bs = (g.n + nb - 1) // nb
        self.blocks, spent = [], 0.0
        for b in bit_reversed(nb):
            lo, hi = b * bs, min(g.n, (b + 1) * bs)
            if lo >= hi:
                continue
            r = oracle.list_triangles(self.view, oracle.APM, threads=threads, rank_begin=lo, rank_end=hi)
            self.blocks.append((lo, hi))
            spent += r.wall_ms / 1e3
            if spent >= budget_s:
                break

    def run(self):
        ops = tri = 0
        ms = 0.0
        for lo, hi in self.blocks:
            r = self.oracle.list_triangles(self.view, self.oracle.APM, threads=self.threads,
                                           rank_begin=lo, rank_end=hi)
            ops += r.inner_ops
            tri += r.triangle_count
            ms += r.wall_ms
        return ops, tri, ms


# configs whose reference Graph/OrientedView constructors take too long for a
# bounded default run: their cpu_baseline uses the oracle port (kind "port")
PORT_BASELINE = {"c5"}


def reference_arm(args, cfg, world, rank):
    if rank != 0:
        return  # rank 0 alone runs and prints the reference line
    import paper_2203_04774_b200 as tg
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtrilist_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    g = make_graph(cfg)
    pi, order_ms = tg.compute_order(g, args.ordering)
    cost = tg.cost_report(g, pi)
    C_total = cost.c_pm
    # value = triangles/s measured on a bounded, spread sample of seeds;
    # ms_per_step = the full workload's time extrapolated by inner_ops
    samp = ReferenceSample(g, pi, args.ref_budget, threads)
    for _ in range(args.warmup):
        samp.run()
    step_ms, ops_l, tri_l = [], [], []
    for _ in range(args.steps):
        ops, tri, ms = samp.run()
        step_ms.append(ms * C_total / max(ops, 1))  # extrapolated full-workload ms
        ops_l.append(ops)
        tri_l.append(tri)
    ms_per_step = statistics.mean(step_ms)
    # triangles/s measured on the sample: triangles found / reference time spent
    sample_ms = [s * ops / C_total for s, ops in zip(step_ms, ops_l)]
    value = sum(tri_l) / max(1e-9, sum(sample_ms) / 1e3)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_block(args, cfg, g),
        "cpu_baseline": {"value": value, "unit": "triangles/s", "cores": threads, "kind": "reference",
                         "sample": f"{len(samp.blocks)} of 256 seed-rank blocks (bit-reversed spread), "
                                   f"{sum(ops_l) / len(ops_l) / C_total:.3%} of inner_ops per step; "
                                   "full-workload time extrapolated by inner_ops"},
        "e2e": {"value": value, "unit": "triangles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_setup_s": samp.setup_s, "order_ms": order_ms,
    }
    print(json.dumps(out))


def config_block(args, cfg, g):
    return {"workload": args.config, "desc": cfg["desc"], "n": g.n, "m": g.m,
            "ordering": args.ordering, "algo": args.algo, "sinks": args.sinks,
            "step": "tl_orient (relabel+orient+CSR+segsort+cost) + tl_list (A+-)",
            "l2": "inputs larger than L2 (adjacency %.1f GB vs 126 MB L2)" % (8 * g.m / 1e9)}


def trigpu_arm(args, cfg, world, rank, local):
    import torch
    import paper_2203_04774_b200 as tg
    from paper_2203_04774_b200._native import TL_ALGO_APM, TL_ALGO_APP, TL_OUT_CHECKSUM, TL_OUT_VERTEX_COUNTS

    t0 = time.perf_counter()
    g = make_graph(cfg)
    log(f"[bench] graph {args.config}: n={g.n} m={g.m} ({time.perf_counter() - t0:.1f}s)")
    t0 = time.perf_counter()
    pi, order_ms = tg.compute_order(g, args.ordering)
    log(f"[bench] {args.ordering} ordering: {order_ms:.1f} ms (+ reference Graph build, "
        f"{time.perf_counter() - t0:.1f}s total)")
    ctx = tg.Context(local)
    flags = {"count": 0, "count+checksum": TL_OUT_CHECKSUM,
             "count+checksum+vcounts": TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS}[args.sinks]
    ALGO = TL_ALGO_APM if args.algo == "apm" else TL_ALGO_APP

    # --- device-resident inputs -------------------------------------------------
    torch.cuda.set_device(local)
    d_off = torch.from_numpy(g.offsets.view(np.int64)).to(f"cuda:{local}")
    d_adj = torch.from_numpy(g.adjacency.view(np.int32)).to(f"cuda:{local}")
    d_rank = torch.from_numpy(pi.ranks.view(np.int32)).to(f"cuda:{local}")
    torch.cuda.synchronize()

    def step_device():
        ctx.orient_device(g.n, g.m, d_off.data_ptr(), d_adj.data_ptr(), d_rank.data_ptr())
        return ctx.list(ALGO, flags)

    for _ in range(args.warmup):
        st = step_device()
    T = int(st.triangle_count)
    C_pm = int(st.inner_ops)  # c_pm (A+-) or c_pp (A++)
    B_list = 4 * (C_pm + 2 * g.m)  # 4 * (inner_ops + mark_ops)

    sampler = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    sampler.start()
    ctx.timer_start()
    list_ms, orient_ms, launches, phases = [], [], 0, []
    for _ in range(args.steps):
        st = step_device()
        assert int(st.triangle_count) == T
        list_ms.append(ctx.phase_times()["list"])
        orient_ms.append(float(st.orient_ms))
        launches += int(st.kernel_launches)
        phases.append(ctx.phase_times())
    total_ms = ctx.timer_stop()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(world)
    value = replica_value(T * args.steps, total_ms, world)
    total_ms = allreduce_max(total_ms, world)
    ms_per_step = total_ms / args.steps

    # --- e2e through the C-ABI with pinned host buffers --------------------------
    ctx.host_register(g.offsets)
    ctx.host_register(g.adjacency)
    ctx.host_register(pi.ranks)
    for _ in range(max(1, args.warmup)):
        ctx.orient(g.offsets, g.adjacency, pi.ranks)
        ctx.list(ALGO, flags)
    barrier(world)
    t0 = time.perf_counter()
    h2d_ms = []
    for _ in range(args.steps):
        ctx.orient(g.offsets, g.adjacency, pi.ranks)
        st = ctx.list(ALGO, flags)  # stats read back (D2H) inside
        assert int(st.triangle_count) == T
        h2d_ms.append(float(st.h2d_ms))
    e2e_s = allreduce_max(time.perf_counter() - t0, world)
    # full path from the host Graph CSR with the ordering computed on the GPU
    # (tl_orient_ordered: H2D + device degree/split order + orient) + list
    gpu_order = None
    if args.ordering in ("degree", "split"):
        ctx.orient_ordered(g.offsets, g.adjacency, args.ordering)
        assert np.array_equal(ctx.fetch_ranks(g.n), pi.ranks)  # bit-identical to the reference ordering
        ctx.list(ALGO, flags)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ctx.orient_ordered(g.offsets, g.adjacency, args.ordering)
            st = ctx.list(ALGO, flags)
            assert int(st.triangle_count) == T
        go_s = allreduce_max(time.perf_counter() - t0, world)
        gpu_order = {"value": world * T * args.steps / go_s, "unit": "triangles/s",
                     "ms_per_step": go_s * 1e3 / args.steps,
                     "what": "tl_orient_ordered (H2D of the Graph CSR + device %s order + orient) + tl_list"
                             % args.ordering}
    ctx.host_unregister(g.offsets)
    ctx.host_unregister(g.adjacency)
    ctx.host_unregister(pi.ranks)
    h2d_bytes = g.offsets.nbytes + g.adjacency.nbytes + pi.ranks.nbytes
    d2h_bytes = 3 * 8  # triangle count, checksum, list cursor

    if rank != 0:
        return
    peak, peak_src = load_peaks()
    list_avg = statistics.mean(list_ms)
    achieved = B_list / (list_avg / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{args.config}:{args.ordering}:apm")
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        port = args.config in PORT_BASELINE or not oracle.ref_available()
        threads = os.cpu_count() or 1
        samp = (PortSample(ctx, g, pi, args.ref_budget, threads) if port
                else ReferenceSample(g, pi, args.ref_budget, threads))
        ops, tri, ms = samp.run()
        full_ms = ms * C_pm / max(ops, 1)
        what = "oracle port (oracle.c) of the" if port else "reference"
        cpu = {"value": tri / (ms / 1e3), "unit": "triangles/s", "cores": threads,
               "full_workload_ms_extrapolated": full_ms, "kind": "port" if port else "reference",
               "sample": f"{what} list_apm loops on {len(samp.blocks)} of 256 seed-rank blocks "
                         f"({ops / C_pm:.3%} of inner_ops, {ms / 1e3:.1f} s); full-workload time "
                         f"extrapolated by inner_ops; setup {samp.setup_s:.1f} s untimed"}
    ph = {k: statistics.mean(p[k] for p in phases) for k in phases[0]}
    out = {
        "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_block(args, cfg, g),
        "edges_per_s": world * g.m * args.steps / (total_ms / 1e3),
        "triangles": T, "inner_ops": C_pm,
        "list_only": {"ms": list_avg, "triangles_per_s": T / (list_avg / 1e3),
                      "edges_per_s": g.m / (list_avg / 1e3)},
        "orient_ms": statistics.mean(orient_ms),
        "phase_ms": ph,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "listing kernels (k_list_reg/warp/cta/giant)",
                     "algorithmic_bytes": B_list, "peak_source": peak_src,
                     "frac_of_8TBs_nominal": achieved / 8000.0},
        "cpu_baseline": cpu,
        "e2e": {"value": world * T * args.steps / e2e_s, "unit": "triangles/s",
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                "h2d_ms": statistics.mean(h2d_ms), "ms_per_step": e2e_s * 1e3 / args.steps,
                "with_host_order_ms": order_ms + e2e_s * 1e3 / args.steps,
                "gpu_order": gpu_order},
        "gpu_launches": launches,
        "clocks": clocks,
        "order_ms": order_ms,
    }
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="trigpu", choices=["trigpu", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--ordering", default="degree")
    ap.add_argument("--algo", default="apm", choices=["apm", "app"])
    ap.add_argument("--sinks", default="count+checksum", choices=["count", "count+checksum", "count+checksum+vcounts"])
    ap.add_argument("--ref-budget", type=float, default=10.0, help="seconds of reference work per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, cfg, world, rank)
    else:
        trigpu_arm(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
