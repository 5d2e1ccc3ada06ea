#!/usr/bin/env python
"""Benchmark: mere-listing (orientation/CSR build + listing) on B200.

One step = the hot path over one synthetic graph with pi given: tl_orient
(relabel, orient, CSR, segmented sort, cost) + tl_list (degree-binned A+- or
A++ with the count + checksum sinks). `value` = triangles listed per second
over the K timed steps, inputs resident in HBM (tl_orient_device), device time
on the engine's stream (CUDA events). `e2e` = the same through the C-ABI with
HOST buffers (pinned), host->device copies and the stats read-back inside the
timed region; `e2e.gpu_order` adds the ordering on the device
(tl_orient_ordered: H2D of the Graph CSR + degree/split order + orient + list).

    python bench.py [--config c5] [--steps K] [--warmup W] [--gpus N]
    python bench.py --impl reference ...   # the reference CPU listing (oracle/_ref)

Default workload: C5 (R-MAT scale 27, edge factor 16), the largest
single-GPU config of BASELINE.json. pi is the degree order computed on the
device (tl_order, bit-identical to the reference's degree_order including its
tie-breaks -- tests/test_gpu_parity.py::test_device_orderings_match_reference);
`--host-order` uses the reference's own ordering code instead.

Multi-GPU: the north star keeps the path on one GPU (no sharding, no
collectives), so N>1 runs N independent replicas ("replicas only",
DESIGN.md); value sums the replicas' work over the max-over-ranks time. With
`--gpus N` and no torchrun environment, bench.py launches the N rank
processes itself. Local rank 0 generates the graph once and shares it with the
other ranks through a file in /dev/shm (a C5 CSR is 18 GB; generation peaks
at 67 GB of host memory).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
DEFAULT_CONFIG = "c5"
DEVICE_ORDERINGS = ("degree", "split")


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


# -- process plumbing -----------------------------------------------------------

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


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(n: int, argv: list[str]) -> int:
    """`--gpus N` without a torchrun environment: start the N rank processes
    (one per GPU, RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* as torchrun sets
    them); rank 0's stdout is the JSON line. Returns the worst exit code."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *argv], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(abs(rc) for rc in rcs)


# -- shared graph (one generation per node) ------------------------------------------

class SharedGraph:
    """Graph CSR shared read-only between the ranks of one node via a file in
    /dev/shm (np.memmap): local rank 0 generates it, the others map it."""

    def __init__(self, offsets, adjacency, path=None):
        self.offsets = offsets
        self.adjacency = adjacency
        self.path = path

    @property
    def n(self):
        return int(self.offsets.shape[0] - 1)

    @property
    def m(self):
        return int(self.adjacency.shape[0] // 2)


def shared_graph(cfg, world: int, local: int, tag: str):
    if world == 1:
        return make_graph(cfg)
    d = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    base = os.path.join(d, f"trigpu_bench_{tag}_{os.environ.get('MASTER_PORT', '0')}")
    if local == 0:
        g = make_graph(cfg)
        g.offsets.tofile(base + ".off")
        g.adjacency.tofile(base + ".adj")
        del g
    barrier(world)
    off = np.memmap(base + ".off", dtype=np.uint64, mode="r")
    adj = np.memmap(base + ".adj", dtype=np.uint32, mode="r")
    barrier(world)
    if local == 0:  # the mappings keep the pages alive; the names can go
        os.unlink(base + ".off")
        os.unlink(base + ".adj")
    return SharedGraph(off, adj, base)


# -- reference CPU listing on a bounded sample -----------------------------------

def bit_reversed(nblocks: int):
    bits = max(1, (nblocks - 1).bit_length())
    for i in range(1 << bits):
        j = int(format(i, f"0{bits}b")[::-1], 2)
        if j < nblocks:
            yield j


class BlockSample:
    """A bounded sample of the workload: the first k of 256 seed-rank blocks in
    bit-reversed order (so the sample spreads over the whole rank range), k
    doubled until one listing of the sample takes about `budget_s` seconds.
    `list_ranges(ranges)` lists the ranges in ONE pulling pass (per-call setup
    paid once, as in a full listing) and returns (inner_ops, triangles, wall_ms)."""

    NB = 256

    def __init__(self, n: int, list_ranges, budget_s: float):
        self.list_ranges = list_ranges
        bs = (n + self.NB - 1) // self.NB
        order = [(b * bs, min(n, (b + 1) * bs)) for b in bit_reversed(self.NB)]
        order = [r for r in order if r[0] < r[1]]
        k = min(8, len(order))
        while True:
            self.ranges = order[:k]
            _, _, ms = list_ranges(self.ranges)
            if ms / 1e3 >= budget_s or k >= len(order):
                break
            k = min(len(order), 2 * k)

    @property
    def blocks(self):
        return self.ranges

    def run(self):
        return self.list_ranges(self.ranges)


def reference_arm(args, cfg, world, rank):
    """The reference's own listing loops (detail::run_apm_range / run_app_range,
    listing.hpp:69-107, through run_parallel's block pulling, listing.hpp:122-155)
    on the reference's own Graph (from_dense_edges), ordering and OrientedView,
    all from oracle/_ref (the unmodified reference core compiled in place); only
    oracle/ libraries are loaded. Each step lists the same bounded sample of
    seed-rank blocks; ms_per_step is that step's measured wall time."""
    if rank != 0:
        return  # rank 0 alone runs and prints the reference line
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtrilist_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    algo = oracle.APM if args.algo == "apm" else oracle.APP
    setup = {}
    t0 = time.perf_counter()
    gen = oracle.GenGraph(**{k: v for k, v in cfg.items() if k != "desc"})
    n, m = gen.n, gen.m
    setup["generate_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rg = oracle.RefGraph.from_csr(gen.offsets, gen.adjacency)  # Graph::from_dense_edges
    setup["graph_build_s"] = time.perf_counter() - t0
    gen.free()
    t0 = time.perf_counter()
    rank_arr = rg.order(args.ordering, 0)
    order_ms = (time.perf_counter() - t0) * 1e3
    c_pp, c_pm, _, _ = rg.cost(rank_arr)
    C_total = c_pm if args.algo == "apm" else c_pp
    t0 = time.perf_counter()
    view = oracle.RefView(rg, rank_arr)  # OrientedView(g, pi), oriented_view.cpp:7-47
    orient_ms = (time.perf_counter() - t0) * 1e3
    del rg
    log(f"[reference] {args.config}: n={n} m={m}; setup {setup}, order {order_ms:.0f} ms, "
        f"orient {orient_ms:.0f} ms")

    def list_ranges(ranges):
        r = view.list_ranges(algo, ranges, threads=threads)
        return r.inner_ops, r.triangle_count, r.wall_ms

    t0 = time.perf_counter()
    samp = BlockSample(n, list_ranges, args.ref_budget)
    setup["sample_pick_s"] = time.perf_counter() - t0
    for _ in range(args.warmup):
        samp.run()
    step_ms, ops_l, tri_l = [], [], []
    for _ in range(args.steps):
        ops, tri, ms = samp.run()
        step_ms.append(ms)
        ops_l.append(ops)
        tri_l.append(tri)
    ms_per_step = statistics.mean(step_ms)
    value = sum(tri_l) / (sum(step_ms) / 1e3)
    frac_ops = ops_l[0] / max(C_total, 1)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_block(args, cfg, n, m),
        "cpu_baseline": {"value": value, "unit": "triangles/s", "cores": threads, "kind": "reference",
                         "sample": f"{len(samp.blocks)} of {BlockSample.NB} seed-rank blocks (bit-reversed spread), "
                                   f"{frac_ops:.3%} of the workload's inner_ops per step, listed by the "
                                   f"reference's run_{args.algo}_range loops on {threads} threads"},
        "e2e": {"value": value, "unit": "triangles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step": "one bounded sample of the listing (the same blocks every step); setup untimed",
        "sample_triangles": tri_l[0], "sample_inner_ops": ops_l[0], "sample_ms": step_ms,
        "full_workload_ms_extrapolated": ms_per_step * C_total / max(ops_l[0], 1),
        "order_ms": order_ms, "orient_ms": orient_ms, "setup_s": setup,
    }
    print(json.dumps(out), flush=True)


def config_block(args, cfg, n, m):
    return {"workload": args.config, "desc": cfg["desc"], "n": n, "m": m,
            "ordering": args.ordering, "algo": args.algo, "sinks": args.sinks,
            "step": f"tl_orient (relabel+orient+CSR+segsort+cost) + tl_list (A{'+-' if args.algo == 'apm' else '++'})",
            "l2": "inputs larger than L2 (adjacency %.1f GB vs 126 MB L2)" % (8 * m / 1e9)}


# -- the engine -------------------------------------------------------------------

def trigpu_arm(args, cfg, world, rank, local):
    import torch
    import paper_2203_04774_b200 as tg
    from paper_2203_04774_b200._native import TL_ALGO_APM, TL_ALGO_APP, TL_OUT_CHECKSUM, TL_OUT_VERTEX_COUNTS

    t0 = time.perf_counter()
    g = shared_graph(cfg, world, local, args.config)
    gen_s = time.perf_counter() - t0
    log(f"[bench] graph {args.config}: n={g.n} m={g.m} ({gen_s:.1f}s)")
    ctx = tg.Context(local)
    torch.cuda.set_device(local)
    order_how = "device"
    host_order_ms = None
    if args.ordering in DEVICE_ORDERINGS and not args.host_order:
        ranks = ctx.order(g.offsets, args.ordering)  # bit-identical to the reference's ordering
    else:
        pi, host_order_ms = tg.compute_order(g if isinstance(g, tg.Graph) else tg.Graph(g.offsets, g.adjacency),
                                             args.ordering)
        ranks = pi.ranks
        order_how = "reference (host)"
    flags = {"count": 0, "count+checksum": TL_OUT_CHECKSUM,
             "count+checksum+vcounts": TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS}[args.sinks]
    ALGO = TL_ALGO_APM if args.algo == "apm" else TL_ALGO_APP

    # --- device-resident inputs -------------------------------------------------
    d_off = torch.from_numpy(np.asarray(g.offsets).view(np.int64)).to(f"cuda:{local}")
    d_adj = torch.from_numpy(np.asarray(g.adjacency).view(np.int32)).to(f"cuda:{local}")
    d_rank = torch.from_numpy(ranks.view(np.int32)).to(f"cuda:{local}")
    torch.cuda.synchronize()

    def step_device():
        ctx.orient_device(g.n, g.m, d_off.data_ptr(), d_adj.data_ptr(), d_rank.data_ptr())
        return ctx.list(ALGO, flags)

    for _ in range(args.warmup):
        st = step_device()
    T = int(st.triangle_count)
    C_alg = int(st.inner_ops)  # c_pm (A+-) or c_pp (A++)
    B_list = 4 * (C_alg + 2 * g.m)  # 4 * (inner_ops + mark_ops)

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
    del d_off, d_adj, d_rank
    torch.cuda.empty_cache()

    # --- e2e through the C-ABI with pinned host buffers --------------------------
    off_h = np.ascontiguousarray(g.offsets)
    adj_h = np.ascontiguousarray(g.adjacency)
    pinned = []
    for arr in (off_h, adj_h, ranks):
        try:
            ctx.host_register(arr)
            pinned.append(arr)
        except Exception as e:  # a file-backed mapping may refuse; the copy still works unpinned
            log(f"[bench] host_register failed ({e}); copying unpinned")
    for _ in range(max(1, args.warmup)):
        ctx.orient(off_h, adj_h, ranks)
        ctx.list(ALGO, flags)
    barrier(world)
    t0 = time.perf_counter()
    h2d_ms = []
    for _ in range(args.steps):
        ctx.orient(off_h, adj_h, ranks)
        st = ctx.list(ALGO, flags)  # stats read back (D2H) inside
        assert int(st.triangle_count) == T
        h2d_ms.append(float(st.h2d_ms))
    e2e_s = allreduce_max(time.perf_counter() - t0, world)
    # the whole path from the host Graph CSR with the ordering on the device
    # (tl_orient_ordered: H2D + device degree/split order + orient) + list
    gpu_order = None
    if args.ordering in DEVICE_ORDERINGS:
        ctx.orient_ordered(off_h, adj_h, args.ordering)
        assert np.array_equal(ctx.fetch_ranks(g.n), ranks)
        ctx.list(ALGO, flags)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ctx.orient_ordered(off_h, adj_h, args.ordering)
            st = ctx.list(ALGO, flags)
            assert int(st.triangle_count) == T
        go_s = allreduce_max(time.perf_counter() - t0, world)
        gpu_order = {"value": world * T * args.steps / go_s, "unit": "triangles/s",
                     "ms_per_step": go_s * 1e3 / args.steps,
                     "what": "tl_orient_ordered (H2D of the Graph CSR + device %s order + orient) + tl_list"
                             % args.ordering}
    for arr in pinned:
        ctx.host_unregister(arr)
    h2d_bytes = off_h.nbytes + adj_h.nbytes + ranks.nbytes
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
            traffic = json.load(f).get(f"{args.config}:{args.ordering}:{args.algo}")
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = port_baseline(ctx, g, ranks, ALGO, C_alg, args.ref_budget)
    ph = {k: statistics.mean(p[k] for p in phases) for k in phases[0]}
    out = {
        "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_block(args, cfg, g.n, g.m),
        "edges_per_s": world * g.m * args.steps / (total_ms / 1e3),
        "triangles": T, "inner_ops": C_alg,
        "list_only": {"ms": list_avg, "triangles_per_s": T / (list_avg / 1e3),
                      "edges_per_s": g.m / (list_avg / 1e3)},
        "orient_ms": statistics.mean(orient_ms),
        "phase_ms": ph,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "listing kernels (k_list_*), events around the class launches",
                     "algorithmic_bytes": B_list, "peak_source": peak_src,
                     "frac_of_8TBs_nominal": achieved / 8000.0},
        "cpu_baseline": cpu,
        "e2e": {"value": world * T * args.steps / e2e_s, "unit": "triangles/s",
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                "h2d_ms": statistics.mean(h2d_ms), "ms_per_step": e2e_s * 1e3 / args.steps,
                "gpu_order": gpu_order},
        "gpu_launches": launches,
        "clocks": clocks,
        "pi": order_how, "host_order_ms": host_order_ms, "generate_s": gen_s,
    }
    print(json.dumps(out), flush=True)


def port_baseline(ctx, g, ranks, algo, C_alg, budget_s):
    """cpu_baseline: the oracle port (oracle.c, the restatement of listing.hpp:69-155)
    on all host cores over a bounded sample of seed-rank blocks, on the oriented
    view exported in the reference layout (building the reference's own Graph +
    OrientedView for C5 takes ~6 minutes single-threaded; bench.py --impl
    reference does exactly that)."""
    import oracle
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    so, s_, po, p_ = ctx.fetch_oriented(g.n, g.m)
    inv = np.empty_like(ranks)
    inv[ranks] = np.arange(ranks.shape[0], dtype=np.uint32)
    view = oracle.OrientedCSR(so, s_, po, p_, inv, ranks)
    setup_s = time.perf_counter() - t0

    def list_ranges(ranges):
        r = oracle.list_ranges(view, algo, ranges, threads=threads)
        return r.inner_ops, r.triangle_count, r.wall_ms

    samp = BlockSample(g.n, list_ranges, budget_s)
    ops, tri, ms = samp.run()
    return {"value": tri / (ms / 1e3), "unit": "triangles/s", "cores": threads, "kind": "port",
            "full_workload_ms_extrapolated": ms * C_alg / max(ops, 1),
            "sample": f"oracle port (oracle.c) of the reference loops on {len(samp.blocks)} of "
                      f"{BlockSample.NB} seed-rank blocks ({ops / max(C_alg, 1):.3%} of inner_ops, "
                      f"{ms / 1e3:.1f} s); setup {setup_s:.1f} s untimed"}


def plumbing_arm(args, world, rank):
    """No GPU work: the multi-process plumbing alone (tests/test_dist.py)."""
    barrier(world)
    v = replica_value(10.0, 100.0 + 50.0 * rank, world)
    if rank == 0:
        print(json.dumps({"impl": "plumbing", "n_gpus": world, "value": v}), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="trigpu", choices=["trigpu", "reference", "plumbing"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--ordering", default="degree")
    ap.add_argument("--host-order", action="store_true", help="pi from the reference's host ordering code")
    ap.add_argument("--algo", default="apm", choices=["apm", "app"])
    ap.add_argument("--sinks", default="count+checksum", choices=["count", "count+checksum", "count+checksum+vcounts"])
    ap.add_argument("--ref-budget", type=float, default=6.0, help="seconds of CPU listing per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus, argv)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":  # CPU only: rank 0 runs, the other ranks exit without work
        world = int(os.environ.get("WORLD_SIZE", "1"))
        reference_arm(args, cfg, world, int(os.environ.get("RANK", "0")))
        return 0
    world, rank, local = dist_setup("gloo" if args.impl == "plumbing" else "nccl")
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "plumbing":
        plumbing_arm(args, world, rank)
    else:
        trigpu_arm(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
