#!/usr/bin/env python
"""bench.py — SIVF hot path on B200 (contract: one JSON line on rank 0).

A "step" is one pass of the whole hot path on the
SIFT1M-shaped workload of BASELINE.json configs[1]: a 1M-vector window
(d=128, nlist=1024, centroids trained on the GPU), per step insert 10k new
ids, delete the 10k oldest, search 10k queries (k=10, nprobe=32), reclaim
full dead slabs (the sliding-window step of P:658 at W=1M).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sivf|reference]

--impl reference times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same step on the box's host cores.
N>1 (torchrun): ids are sharded id % N; mutations are routed with no
collective; every rank searches all queries on its shard, then an NCCL
all-gather of the per-shard top-k + sivf_merge_topk (strong scaling: the
global workload is fixed).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "deletes/s, inserts/s, sliding-window step p50/p99 ms, QPS@recall10≥0.9"
N_BASE, DIM, NLIST, BATCH, NQ, K, NPROBE = 1_000_000, 128, 1024, 10_000, 10_000, 10, 32
N_TRAIN, N_ITER, SEED = 262_144, 20, 0x51F7
# dram__bytes_read.sum + dram__bytes_write.sum of one k_scan_tc launch, from the committed ncu
# --set full capture of this bench step (per launch; compare with roofline.hbm_view).
SCAN_TRAFFIC_NCU = 518.173952e6 + 26.920192e6
SCAN_TRAFFIC_SRC = "profiles/r03h_scan_full.txt (ncu --set full, bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-extra)"
WORKLOAD = ("SIFT1M-shaped sliding step: 1M x 128 fp32 live window, nlist=1024; per step insert 10k new + "
            "delete 10k oldest + search 10k queries (k=10, nprobe=32) + reclaim")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sivf", choices=["sivf", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the sliding-window (W), GIST (G) and H legs")
    ap.add_argument("--window-steps", type=int, default=1000)
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run only N steps, no extras")
    ap.add_argument("--h-n", type=int, default=100_000_000, help="vectors of the id-sharded H leg (0: skip)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML every 5 ms (the recipe's clocks line; a timed
    region of 20 graph-replayed steps lasts ~15 ms)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, dev_index: int):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers
def pct(v, p):
    v = sorted(v)
    if not v:
        return None
    i = min(len(v) - 1, max(0, int(math.ceil(p / 100.0 * len(v))) - 1))
    return v[i]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def fp32_alu_peak_tflops(sm_count: int, mhz: float) -> float:
    # FP32 SIMT: 128 FMA lanes per SM per cycle, 2 flops per FMA
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- reference arm
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_sample(n_cores: int, budget_steps: int, warmup: int, log, centroids=None):
    """Time the CPU oracle on a bounded sample of the step: 1/10 of the inserts
    and deletes and 1/100 of the queries per sampled step, on a 1M-vector
    oracle index; the step time is scaled back to the full step (labelled
    "extrapolated" in the line).  The timed samples run on ONE thread pinned to
    one host core (n_cores = 1); the untimed 1M build uses every core.  The
    quantizer is the GPU-trained one when given (the same configuration as the
    GPU arm), else a 20-iteration oracle k-means on the same training sample."""
    import oracle as O
    from datagen import Generator, sift_shape

    O.set_threads(os.cpu_count() or 1)
    gen = Generator(sift_shape(seed=SEED))
    t0 = time.time()
    if centroids is not None:
        C = np.ascontiguousarray(centroids, dtype=np.float32)
    else:
        C = O.kmeans(gen.train(N_TRAIN), NLIST, N_ITER, SEED)  # setup, untimed
    ref = O.Index(DIM, NLIST, N_BASE + (budget_steps + warmup + 2) * BATCH)
    ref.set_centroids(C)
    for b0 in range(0, N_BASE, 100_000):
        ref.insert(np.arange(b0, b0 + 100_000), gen.range(b0, 100_000))
    log(f"oracle build {time.time() - t0:.1f}s on {os.cpu_count()} threads (untimed setup)")
    O.set_threads(n_cores)
    aff = None
    if n_cores == 1 and hasattr(os, "sched_setaffinity"):
        aff = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {min(aff)})  # the timed oracle runs on one pinned core
    si, sd, sq = BATCH // 10, BATCH // 10, NQ // 100
    times = []
    try:
        times = _oracle_steps(ref, gen, si, sd, sq, warmup, budget_steps)
    finally:
        if aff is not None:
            os.sched_setaffinity(0, aff)
        O.set_threads(os.cpu_count() or 1)
    return times


def _oracle_steps(ref, gen, si, sd, sq, warmup, budget_steps):
    times = []
    for t in range(warmup + budget_steps):
        new = np.arange(N_BASE + t * si, N_BASE + (t + 1) * si)
        old = np.arange(t * sd, (t + 1) * sd)
        Xn = gen.range(int(new[0]), si)
        Q = gen.queries(t * sq, sq)
        a = time.perf_counter()
        ref.insert(new, Xn)
        b = time.perf_counter()
        ref.delete(old)
        c = time.perf_counter()
        ref.search(Q, K, NPROBE)
        d = time.perf_counter()
        ref.reclaim()
        e = time.perf_counter()
        if t >= warmup:
            full = (b - a) * (BATCH / si) + (c - b) * (BATCH / sd) + (d - c) * (NQ / sq) + (e - d)
            times.append({"insert_1k": b - a, "delete_1k": c - b, "search_100q": d - c, "reclaim": e - d,
                          "sample_step_s": e - a, "full_step_s": full})
    return times


def sivf_config(G):
    """The workload config dict, shared by both arms (same_config)."""
    return {"workload": WORKLOAD, "n_base": N_BASE, "dim": DIM, "nlist": NLIST, "batch": BATCH, "nq": NQ,
            "k": K, "nprobe": NPROBE, "parallelism": f"id-shard{G}",
            "l2": "no flush: the 0.75 GB index scanned every step exceeds the 126 MB L2",
            "generator": "datagen SIFT-shaped (M=50, r=24, a=60, b=50, sigma=15), seed 0x51F7"}


def run_reference(args):
    """The CPU oracle as it stands (oracle/, test infrastructure) on the box's host
    cores: WHOLE sliding steps of the same workload (10k inserts + 10k deletes + 10k
    queries + reclaim on the 1M-vector window, the quantizer = the oracle k-means on
    the same training sample and iterations, which the GPU k-means equals bit for
    bit), exactly `--warmup` untimed and `--steps` timed steps, no extrapolation.  All
    host threads (the oracle's per-item parallel loops); rank 0 only."""
    import oracle as O
    from datagen import Generator, sift_shape

    ws, rank, _ = dist_env()
    if rank != 0:
        return
    log = lambda m: print(f"[bench:reference] {m}", file=sys.stderr, flush=True)
    n_cores = os.cpu_count() or 1
    O.set_threads(n_cores)
    gen = Generator(sift_shape(seed=SEED))
    t0 = time.time()
    C = O.kmeans(gen.train(N_TRAIN), NLIST, N_ITER, SEED)
    steps, warm = args.steps, args.warmup
    ref = O.Index(DIM, NLIST, N_BASE + (steps + warm + 1) * BATCH)
    ref.set_centroids(C)
    for b0 in range(0, N_BASE, 100_000):
        ref.insert(np.arange(b0, b0 + 100_000), gen.range(b0, 100_000))
    log(f"setup (k-means {N_ITER} iters on {N_TRAIN} samples + 1M build) {time.time() - t0:.1f}s on {n_cores} threads")
    times, parts = [], []
    t_wall = time.time()
    for t in range(warm + steps):
        new = np.arange(N_BASE + t * BATCH, N_BASE + (t + 1) * BATCH)
        old = np.arange(t * BATCH, (t + 1) * BATCH)
        Xn = gen.range(int(new[0]), BATCH)
        Q = gen.queries(t * NQ, NQ)
        a = time.perf_counter()
        ref.insert(new, Xn)
        b = time.perf_counter()
        ref.delete(old)
        c = time.perf_counter()
        ref.search(Q, K, NPROBE)
        d = time.perf_counter()
        ref.reclaim()
        e = time.perf_counter()
        if t >= warm:
            times.append(e - a)
            parts.append({"insert_10k": b - a, "delete_10k": c - b, "search_10k": d - c, "reclaim": e - d})
        log(f"step {t} {'(warm-up) ' if t < warm else ''}{(e - a) * 1e3:.0f} ms")
    wall = time.time() - t_wall
    mean = statistics.mean(times)
    value = 1.0 / mean
    sample = (f"{steps} whole sliding steps (after {warm} untimed): 10k inserts + 10k deletes + 10k queries (k=10, "
              f"nprobe=32) + reclaim on the 1M-vector oracle window, {n_cores} host threads; not extrapolated")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": mean * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": sivf_config(args.gpus),
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": n_cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "extrapolated": False},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_wall_s": wall,
        "breakdown_s": {k: statistics.mean(p[k] for p in parts) for k in parts[0]},
        "metrics": {"inserts_per_s": BATCH / statistics.mean(p["insert_10k"] for p in parts),
                    "deletes_per_s": BATCH / statistics.mean(p["delete_10k"] for p in parts),
                    "qps_nprobe32": NQ / statistics.mean(p["search_10k"] for p in parts),
                    "step_ms_p50": pct(times, 50) * 1e3, "step_ms_p99": pct(times, 99) * 1e3},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- sivf arm
def run_sivf(args):
    import torch

    import paper_2601_11808_b200 as S
    from datagen import Generator, sift_shape
    from paper_2601_11808_b200 import shard

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    log = (lambda m: print(f"[bench:r{rank}] {m}", file=sys.stderr, flush=True))
    G = ws
    stream = torch.cuda.current_stream()
    W, Kst = args.warmup, args.steps
    E2W = 4  # untimed e2e warm-up steps: the API caches its step graphs for both staging sets
    n_steps_total = W + 3 * Kst + 2 + E2W  # direct (profiled) + CUDA-graph + e2e warm-up + e2e passes
    gen = Generator(sift_shape(seed=SEED))

    # ---------------- setup (untimed): quantizer, index, 1M build
    cap = N_BASE + (n_steps_total + 1) * BATCH
    local_n = (N_BASE + G - 1) // G
    num_slabs = S.num_slabs_for(local_n + 2 * BATCH // G, NLIST)
    ix = S.Index(DIM, NLIST, cap, num_slabs, max_batch=max(BATCH, 65536), max_queries=NQ, max_k=K,
                 max_nprobe=128, max_train=N_TRAIN, shard_rank=rank, shard_count=G, seed=SEED, device=dev)
    t0 = time.time()
    Xt = torch.from_numpy(gen.train(N_TRAIN)).to(dev)
    ix.train(Xt, niter=N_ITER)
    C = ix.get_centroids()
    if pg is not None:
        pg.broadcast(C, src=0)  # replicated quantizer (§8(e))
        ix.set_centroids(C)
    torch.cuda.synchronize()
    t_train = time.time() - t0
    del Xt
    log(f"train {t_train:.2f}s")

    Xb_host = gen.range(0, N_BASE)
    ids_all = np.arange(N_BASE, dtype=np.int64)
    mine, Xmine = shard.route(ids_all, G, rank, Xb_host)  # owner(id) = id mod G, no collective
    Xb = torch.from_numpy(Xmine).to(dev)
    idb = torch.from_numpy(mine).to(dev)
    build_ms = []
    bl = 65536
    for b0 in range(0, mine.shape[0], bl):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, _ = ix.insert(idb[b0:b0 + bl], Xb[b0:b0 + bl])
        e1.record()
        build_ms.append((e0, e1, min(bl, mine.shape[0] - b0)))
    torch.cuda.synchronize()
    build_rate = sum(n for _, _, n in build_ms) / (sum(a.elapsed_time(b) for a, b, _ in build_ms) / 1e3)
    del Xb, idb
    s0 = ix.stats()
    assert s0["live"] == mine.shape[0] and s0["device_errors"] == 0, s0
    log(f"build {mine.shape[0]} vectors at {build_rate / 1e6:.2f} M/s (64k batches)")

    # ---------------- per-step inputs (pre-staged on device for the kernel-resident leg)
    def step_host(t):
        new = np.arange(N_BASE + t * BATCH, N_BASE + (t + 1) * BATCH, dtype=np.int64)
        old = np.arange(t * BATCH, (t + 1) * BATCH, dtype=np.int64)
        nm, Xn = shard.route(new, G, rank, gen.range(int(new[0]), BATCH))
        om, = shard.route(old, G, rank)
        Q = gen.queries(t * NQ, NQ)
        return nm, np.ascontiguousarray(Xn), om, Q

    n_dev_steps = W + 2 * Kst + 1  # direct pass, then the CUDA-graph pass (G == 1)
    dev_inputs = []
    for t in range(n_dev_steps):
        nm, Xn, om, Q = step_host(t)
        dev_inputs.append(tuple(torch.from_numpy(a).to(dev) for a in (nm, Xn, om, Q)))
    out_d = torch.empty(NQ, K, dtype=torch.float32, device=dev)
    out_i = torch.empty(NQ, K, dtype=torch.int64, device=dev)
    status = torch.empty(BATCH, dtype=torch.int32, device=dev)
    ndel = torch.empty(1, dtype=torch.int64, device=dev)

    def one_step(inp, dd=None, ii=None):
        nm, Xn, om, Q = inp
        ix.sliding_window_step(nm, Xn, om, Q, K, NPROBE,
                               out=(out_d if dd is None else dd, out_i if ii is None else ii, status, ndel))
        if dd is not None:
            return dd, ii
        if G > 1:
            gd, gi = shard.allgather_topk(pg, out_d, out_i)  # NCCL all-gather of the per-shard top-k
            return S.merge_topk(gd, gi)
        return out_d, out_i

    def barrier():
        if pg is not None:
            pg.barrier()

    # warmup
    for t in range(W):
        one_step(dev_inputs[t])
    torch.cuda.synchronize()
    barrier()

    # ---------------- timed region (inputs resident in HBM; index 0.75 GB > 126 MB L2)
    ix.profile(True)
    ix.profile_read()
    launches0 = ix.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(Kst)]
    phases = []
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(local) as clk:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for t in range(Kst):
            evs[t][0].record()
            one_step(dev_inputs[W + t])
            evs[t][1].record()
        g1.record()
        torch.cuda.synchronize()
    barrier()
    launches = ix.launch_count() - launches0
    prof = ix.profile_read()
    ix.profile(False)
    total_ms = g0.elapsed_time(g1)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    if G > 1:
        t_ = torch.tensor([total_ms], device=dev)
        pg.all_reduce(t_, op=pg.ReduceOp.MAX)
        total_ms = float(t_.item())
    ms_per_step = direct_ms = total_ms / Kst
    graph = None
    if G == 1:
        # The same steps as one CUDA-graph replay each (fixed shapes; the step's inputs are
        # copied into the graph's static buffers inside the timed region).  `value` is this
        # pass; phase times and the roofline come from the direct pass above.
        s_in = [torch.empty_like(x) for x in dev_inputs[W + Kst]]
        for d_, s_ in zip(s_in, dev_inputs[W + Kst]):
            d_.copy_(s_)
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            ix.sliding_window_step(*s_in, K, NPROBE, out=(out_d, out_i, status, ndel))
        cg.replay()  # step W + Kst
        torch.cuda.synchronize()
        with ClockSampler(local) as clk_g:
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for t in range(Kst):
                for d_, s_ in zip(s_in, dev_inputs[W + Kst + 1 + t]):
                    d_.copy_(s_, non_blocking=True)
                cg.replay()
            g1.record()
            torch.cuda.synchronize()
        graph = {"ms_per_step": g0.elapsed_time(g1) / Kst, "clocks": clk_g.summary()}
        ms_per_step = graph["ms_per_step"]
        clk = clk_g
    s1 = ix.stats()
    log(f"timed {Kst} steps: {ms_per_step:.3f} ms/step; live={s1['live']} free={s1['slabs_free']} "
        f"reclaimed={s1['reclaimed_slabs']} err={s1['device_errors']}")

    # ---------------- e2e: same step through the C ABI from pinned host buffers.  Inputs of
    # step t+1 are copied (H2D, copy stream) while step t computes, and step t's results
    # are copied back (D2H) while step t+1 computes: two staging sets, events between
    # the streams.  The timed region spans the first H2D to the last D2H.
    host_inputs = []
    for t in range(n_dev_steps, n_dev_steps + E2W + Kst):  # steps after the graph pass
        host_inputs.append(tuple(torch.from_numpy(a).pin_memory() for a in step_host(t)))
    h_d = [torch.empty(NQ, K, dtype=torch.float32).pin_memory() for _ in range(E2W + Kst)]
    h_i = [torch.empty(NQ, K, dtype=torch.int64).pin_memory() for _ in range(E2W + Kst)]
    stage = [[torch.empty_like(x, device=dev) for x in host_inputs[0]] for _ in range(2)]
    res_d = [torch.empty(NQ, K, dtype=torch.float32, device=dev) for _ in range(2)]
    res_i = [torch.empty(NQ, K, dtype=torch.int64, device=dev) for _ in range(2)]
    h2d = sum(x.numel() * x.element_size() for x in host_inputs[0])
    d2h = h_d[0].numel() * 4 + h_i[0].numel() * 8
    cs = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def h2d_copy(t, u):  # step u's inputs into staging set t % 2
        b = t % 2
        with torch.cuda.stream(cs):
            if t >= 2:
                cs.wait_event(ev_done[b])  # step t-2 no longer reads this staging set
            for dst, src in zip(stage[b], host_inputs[u]):
                if dst.shape != src.shape:
                    dst.resize_(src.shape)
                dst.copy_(src, non_blocking=True)
            ev_in[b].record(cs)

    def e2e_pass(u0, n, e0=None):  # host steps u0 .. u0+n-1; the first H2D after e0
        if e0 is not None:
            e0.record(main)
            cs.wait_event(e0)
        else:
            cs.wait_stream(main)
        h2d_copy(0, u0)
        for t in range(n):
            b = t % 2
            if t + 1 < n:
                h2d_copy(t + 1, u0 + t + 1)
            main.wait_event(ev_in[b])
            if t >= 2:
                main.wait_event(ev_out[b])  # results of step t-2 copied out of this buffer set
            if G == 1:  # results straight into this step's output buffers
                one_step(tuple(stage[b]), res_d[b], res_i[b])
            else:
                dd, ii = one_step(tuple(stage[b]))
                res_d[b].copy_(dd, non_blocking=True)
                res_i[b].copy_(ii, non_blocking=True)
            ev_done[b].record(main)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[b])
                h_d[u0 + t].copy_(res_d[b], non_blocking=True)
                h_i[u0 + t].copy_(res_i[b], non_blocking=True)
                ev_out[b].record(cs)
        main.wait_stream(cs)

    # untimed warm-up: the library captures each staging set's step signature as a CUDA
    # graph on its second sighting (steady state of a streaming client)
    e2e_pass(0, E2W)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_pass(E2W, Kst, e0)
    e1.record(main)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if G > 1:
        t_ = torch.tensor([e2e_ms], device=dev)
        pg.all_reduce(t_, op=pg.ReduceOp.MAX)
        e2e_ms = float(t_.item())
    e2e_ms /= Kst
    s2 = ix.stats()
    assert s2["device_errors"] == 0

    # ---------------- search sweep: QPS and recall@10 vs exact ground truth (rank 0 only, N=1)
    sweep = {}
    qps_at_09 = None
    recall_point = None
    if not args.no_sweep and G == 1:
        lo = N_BASE + (n_dev_steps + E2W + Kst) * BATCH - N_BASE  # live window [lo, lo + N_BASE)
        live_ids = np.arange(lo, lo + N_BASE)
        assert s2["live"] == N_BASE
        Xl = torch.from_numpy(gen.range(lo, N_BASE)).to(dev)
        Qs = torch.from_numpy(gen.queries(10**7, NQ)).to(dev)
        # exact top-10 on integer-valued data: fp32 GEMM sums of integers < 2^24 are exact
        torch.backends.cuda.matmul.allow_tf32 = False
        xn = (Xl * Xl).sum(1)
        gt = []
        for q0 in range(0, NQ, 500):
            q = Qs[q0:q0 + 500]
            d = (q * q).sum(1)[:, None] + xn[None, :] - 2.0 * (q @ Xl.T)
            key = (d.round().to(torch.int64) << 32) | torch.arange(N_BASE, device=dev)[None, :]
            gt.append(torch.topk(key, K, dim=1, largest=False).values & 0xFFFFFFFF)
        gt = (torch.cat(gt) + lo).cpu().numpy()
        del Xl
        for npb in (1, 2, 4, 8, 16, 32, 64, 128):
            for _ in range(2):  # warm-up (the API captures a repeated call as a graph on its 2nd sighting)
                ix.search(Qs, K, npb)
            torch.cuda.synchronize()
            reps = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                dd, ii = ix.search(Qs, K, npb)
                b.record()
                torch.cuda.synchronize()
                reps.append(a.elapsed_time(b))
            res = ii.cpu().numpy()
            rec = float(np.mean([len(set(r) & set(g)) / K for r, g in zip(res, gt)]))
            qps = NQ / (statistics.median(reps) / 1e3)
            sweep[npb] = {"recall10": rec, "qps": qps, "ms": statistics.median(reps)}
            if qps_at_09 is None and rec >= 0.9:
                qps_at_09, recall_point = qps, npb
        log("sweep " + ", ".join(f"np{k}: r={v['recall10']:.3f} {v['qps'] / 1e6:.2f}Mqps" for k, v in sweep.items()))

    # ---------------- roofline of the dominant kernel (the slab scan) + per-phase rooflines
    ph_ms = {p: (v[0] / v[1] if v[1] else 0.0) for p, v in prof.items()}
    # algorithmic work of one scan launch: every (query, probed list, live slot) triple
    _, _, probes = ix.search(dev_inputs[-1][3], K, NPROBE, return_probes=True)
    _, lpl, _ = ix.dump_state()
    cand = int(lpl[probes.long()].sum().item())
    mp = measured_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_s = clk.summary()
    mhz = float(mp.get("sm_max_mhz", clk_s["sm_max_mhz"] or 1965.0))
    hbm_peak = float(mp.get("hbm_gbs", 6650.0))
    # tf32 dense peak = measured bf16 (sustained: the scan runs inside a long step) x nominal tf32/bf16 (1.1/2.25)
    tf32_peak = float(mp.get("bf16_tflops_sustained", 1400.0)) * (1.1 / 2.25)
    # the scan's MMAs are kind::f16 (fp16 operands, fp32 accumulate): the bf16/fp16 dense peak
    f16_peak = float(mp.get("bf16_tflops_sustained", 1400.0))
    scan_ms = ph_ms["scan"]
    uniq = torch.unique(probes).long()
    uniq_bytes = float(lpl[uniq].sum().item()) * (2 * DIM + 8)
    flops = 2.0 * DIM * cand  # q.x on the tensor cores (the norms are per-slot / per-query precomputes)
    achieved = flops / (scan_ms / 1e3) / 1e12 if scan_ms else 0.0
    roofline = {"bound": "tensor", "achieved": achieved, "peak": f16_peak, "unit": "TFLOP/s",
                "frac": achieved / f16_peak if f16_peak else None, "traffic": SCAN_TRAFFIC_NCU,
                "traffic_source": SCAN_TRAFFIC_SRC,
                "kernel": "k_scan_tc (tcgen05 kind::f16, fp16 slab copy)", "kernel_ms": scan_ms, "algorithmic_flops": flops,
                "per_unit": "2*D flop per (query, probed live slot)", "candidates_per_launch": cand,
                "unique_list_bytes": uniq_bytes,
                "hbm_view": {"achieved_gbs": uniq_bytes / (scan_ms / 1e3) / 1e9 if scan_ms else None,
                             "peak_gbs": hbm_peak,
                             "frac": uniq_bytes / (scan_ms / 1e3) / 1e9 / hbm_peak if scan_ms else None,
                             "per_unit": "2*D+8 B per live slot of each probed list (fp16 copy, norm, id), read once per step"},
                "peak_note": "kind::f16 = MEASURED_PEAKS bf16_tflops_sustained (same dense rate); the coarse and "
                             "assign phases (split tf32) use x 1.1/2.25 (guide nominal ratio)"}

    def tfrac(fl, ms):
        return None if not ms else {"achieved_tflops": fl / (ms / 1e3) / 1e12, "frac": fl / (ms / 1e3) / 1e12 / tf32_peak}

    def hfrac(b, ms):
        return None if not ms else {"achieved_gbs": b / (ms / 1e3) / 1e9, "frac": b / (ms / 1e3) / 1e9 / hbm_peak}

    rooflines = {
        "assign (tensor, 2*nlist*D flop/vector)": tfrac(2.0 * NLIST * DIM * BATCH / G, ph_ms["assign"]),
        "coarse (tensor, 2*nlist*D flop/query)": tfrac(2.0 * NLIST * DIM * NQ, ph_ms["coarse"]),
        "append (hbm, 8D+24 B/vector)": hfrac((8.0 * DIM + 24) * BATCH / G, ph_ms["append"]),
        "delete (hbm, 28 B/id)": hfrac(28.0 * BATCH / G, ph_ms["delete"]),
        "merge (hbm, nprobe*k*8 + k*12 B/query)": hfrac((NPROBE * K * 8.0 + K * 12.0) * NQ, ph_ms["merge"]),
    }
    share = {p: (ph_ms[p] / ms_per_step if ms_per_step else None) for p in ph_ms}
    # latency roofline of the small-batch ops (their HBM fractions above are tiny: they are
    # launch- and dependent-load-bound, not bandwidth-bound)
    lat = None
    if G == 1:
        fl = latency_floors(S, dev, log)
        hop_us = fl["dram_dependent_load_ns"] / 1e3
        k_step = launches / Kst if Kst else 0
        # the phase timers bracket ops inside a stream of work: the floor of one kernel there is
        # launch_in_stream_us (back-to-back launches)
        floor_del = fl["launch_in_stream_us"] + 2 * hop_us  # ATT read -> atomicAnd on the bitmap word
        n_ins = 9  # claim, rows_tiles, gemm, select, chunk_rank, chunk_prefix, reserve, dir_update, append
        floor_ins = n_ins * (fl["launch_in_stream_us"] + hop_us)
        floor_step = fl["graph_replay_1_kernel_us"] + (k_step - 1) * fl["graph_node_us"] + k_step * hop_us
        meas_ins = (ph_ms["assign"] + ph_ms["append"]) * 1e3
        lat = {"floors": fl,
               "delete_10k": {"measured_us": ph_ms["delete"] * 1e3, "floor_us": floor_del,
                              "frac": floor_del / (ph_ms["delete"] * 1e3) if ph_ms["delete"] else None,
                              "floor": "one launch + 2 dependent DRAM loads (ATT -> bitmap atomicAnd)"},
               "insert_10k": {"measured_us": meas_ins, "floor_us": floor_ins,
                              "frac": floor_ins / meas_ins if meas_ins else None,
                              "floor": f"{n_ins} dependent kernels (launch floor each) + one dependent DRAM load each"},
               "step_graph": {"measured_us": ms_per_step * 1e3, "floor_us": floor_step,
                              "frac": floor_step / (ms_per_step * 1e3), "kernels_per_step": k_step,
                              "floor": "one graph replay of the step's kernel chain (per-node floor) + one "
                                       "dependent DRAM load per kernel"}}
        roofline["latency"] = lat

    # ---------------- cpu baseline (oracle, rank 0, N=1 only)
    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu:
        n_cores = 1
        try:
            times = oracle_sample(n_cores, 2, 0, log, centroids=ix.get_centroids().cpu().numpy())
            mean = statistics.mean(t["full_step_s"] for t in times)
            cpu = {"value": 1.0 / mean, "unit": "steps/s", "cores": n_cores, "kind": "oracle",
                   "sample": "2 sampled steps: 1k inserts + 1k deletes + 100 queries on a 1M oracle index with the "
                             "GPU-trained quantizer, one thread pinned to one core; EXTRAPOLATED x10/x10/x100 to the "
                             "full step",
                   "extrapolated": True, "cpu_model": cpu_model(),
                   "sample_step_ms": statistics.mean(t["sample_step_s"] for t in times) * 1e3,
                   "step_ms": mean * 1e3}
        except Exception as e:  # the baseline must not kill the GPU line
            cpu = {"value": None, "unit": "steps/s", "cores": n_cores, "kind": "oracle", "sample": f"failed: {e}"}

    ins_ms = [ph_ms["assign"] + ph_ms["append"]]
    line = {
        "metric": METRIC,
        "value": 1e3 / ms_per_step,
        "unit": "steps/s",
        "n_gpus": G,
        "steps": Kst,
        "warmup": W,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": sivf_config(G),
        "timing": ("value: one CUDA-graph replay per step (inputs copied into the graph's static buffers "
                              "inside the timed region); phases/roofline: the same steps launched directly with "
                              "per-phase CUDA events") if graph else "direct launches with per-phase CUDA events",
        "metrics": {
            "ms_per_step_direct": direct_ms,
            "step_ms_p50": pct(step_ms, 50), "step_ms_p99": pct(step_ms, 99),
            "inserts_per_s": BATCH / (sum(ins_ms) / 1e3) if sum(ins_ms) else None,
            "deletes_per_s": BATCH / (ph_ms["delete"] / 1e3) if ph_ms["delete"] else None,
            "delete_10k_ms": ph_ms["delete"],
            "qps_nprobe32_in_step": NQ / ((ph_ms["coarse"] + ph_ms["invmap"] + ph_ms["scan"] + ph_ms["merge"]) / 1e3),
            "qps_at_recall10_0.9": qps_at_09, "nprobe_at_recall10_0.9": recall_point,
            "build_inserts_per_s_64k_batches": build_rate, "train_s": t_train,
        },
        "phase_ms": ph_ms,
        "phase_share_of_step": share,
        "sweep": sweep,
        "roofline": roofline,
        "rooflines_by_phase": rooflines,
        "cpu_baseline": cpu,
        "e2e": {"value": 1e3 / e2e_ms, "unit": "steps/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                "method": "sivf_sliding_window_step from pinned host buffers; H2D of step t+1 and D2H of step t "
                          "on a copy stream overlap step t (two staging sets); timed after 4 untimed steps of the "
                          "same loop (the API has then cached its step graph for both staging sets); the first "
                          "H2D and the last D2H are inside the timed region",
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk_s,
    }
    if G == 1 and not args.no_extra:
        C_sift = ix.get_centroids()
        del ix
        torch.cuda.empty_cache()
        line["configs"] = {}
        line["configs"]["W_sliding_window"] = leg_window(S, dev, C_sift, args.window_steps, log)
        torch.cuda.empty_cache()
        line["configs"]["G_gist1m"] = leg_gist(S, dev, log)
        torch.cuda.empty_cache()
    if not args.no_extra and args.h_n > 0:
        line.setdefault("configs", {})["H_sharded"] = leg_h(S, dev, log, G, rank, pg, args.h_n)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def _ev():
    import torch

    return torch.cuda.Event(enable_timing=True)


def latency_floors(S, dev, log):
    """SURVEY §8(d) "Latency roofline for small batches": the floors a small-batch op cannot
    beat, measured on this GPU with CUDA events: one empty kernel bracketed by events on an
    idle stream (host-visible launch latency), the per-launch time of 200 back-to-back empty
    kernels on one stream (the floor of one kernel inside a stream of work), one CUDA-graph
    replay of one empty kernel and the per-node time of a replayed 20-kernel chain, and the
    dependent-load latency (one thread chasing a random single-cycle permutation: 1 GB, far
    beyond the 126 MB L2 = DRAM; 4 MB = L2)."""
    import torch

    def med_ms(fn, reps=30):
        out = []
        for _ in range(reps):
            a, b = _ev(), _ev()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b))
        return statistics.median(out)

    S.probe_launch(10)
    torch.cuda.synchronize()
    one = med_ms(lambda: S.probe_launch(1))
    many = med_ms(lambda: S.probe_launch(200), reps=10) / 200
    g1, g20 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(side):
        with torch.cuda.graph(g1, stream=side):
            S.probe_launch(1)
        with torch.cuda.graph(g20, stream=side):
            S.probe_launch(20)
    torch.cuda.synchronize()
    g1.replay()
    g20.replay()
    torch.cuda.synchronize()
    rep1 = med_ms(g1.replay)
    rep20 = med_ms(g20.replay)
    out = torch.zeros(1, dtype=torch.int32, device=dev)
    hops = {}
    for name, n in (("dram", 256 << 20), ("l2", 1 << 20)):
        perm = torch.randperm(n, device=dev, dtype=torch.int64)
        nxt = torch.empty(n, dtype=torch.int32, device=dev)
        nxt[perm] = torch.roll(perm, -1).to(torch.int32)
        del perm
        S.probe_chase(nxt, 1000, out)
        torch.cuda.synchronize()
        t = med_ms(lambda: S.probe_chase(nxt, 4000, out), reps=5) - med_ms(lambda: S.probe_chase(nxt, 0, out), reps=5)
        hops[name] = t * 1e6 / 4000  # ns per dependent load
        del nxt
    torch.cuda.empty_cache()
    res = {"empty_launch_us": one * 1e3, "launch_in_stream_us": many * 1e3, "graph_replay_1_kernel_us": rep1 * 1e3,
           "graph_node_us": (rep20 - rep1) / 19 * 1e3, "dram_dependent_load_ns": hops["dram"],
           "l2_dependent_load_ns": hops["l2"]}
    log("latency floors: " + ", ".join(f"{k} {v:.2f}" for k, v in res.items()))
    return res


def leg_window(S, dev, C, steps, log):
    """BASELINE configs[3]: sliding window on SIFT1M-shaped data, window 1M, slide 10k per
    step (insert new + delete expired + 1k queries, k=10, nprobe=32) + reclaim, one CUDA-graph
    replay per step; p50/p99 over `steps` steps.  Every step's vectors and queries are
    generated from their own ids (g = id, §8(d); queries g = 2^40 + t*1000 + i) on the device
    before the timed loop and stay resident in HBM (~5.7 GB for 1000 steps); each step copies
    its slice into the graph's static buffers inside the timed region."""
    import torch

    from datagen import QUERY_BASE, DeviceGenerator, Generator, sift_shape

    W, B, NQW = N_BASE, BATCH, 1000
    gen = Generator(sift_shape(seed=SEED))
    cap = W + (steps + 40) * B
    ix = S.Index(DIM, NLIST, cap, S.num_slabs_for(W + 2 * B, NLIST), max_batch=max(B, 65536), max_queries=NQW,
                 max_k=K, max_nprobe=NPROBE, seed=SEED, device=dev)
    ix.set_centroids(C)
    Xw = torch.from_numpy(gen.range(0, W)).to(dev)
    ids = torch.arange(W, device=dev)
    for b0 in range(0, W, 65536):
        ix.insert(ids[b0:b0 + 65536], Xw[b0:b0 + 65536])
    del Xw
    warm = 20
    T = warm + 1 + steps
    dgen = DeviceGenerator(sift_shape(seed=SEED))  # bit-identical to the host generator (GPU test)
    allx = torch.empty(T, B, DIM, device=dev)
    allq = torch.empty(T, NQW, DIM, device=dev)
    dgen.range_into(allx.view(T * B, DIM), W, 1)  # step t inserts ids W + t B + i
    dgen.range_into(allq.view(T * NQW, DIM), QUERY_BASE, 1)
    torch.cuda.synchronize()
    s_new, s_old = torch.empty(B, dtype=torch.int64, device=dev), torch.empty(B, dtype=torch.int64, device=dev)
    s_x, s_q = torch.empty(B, DIM, device=dev), torch.empty(NQW, DIM, device=dev)
    out = (torch.empty(NQW, K, device=dev), torch.empty(NQW, K, dtype=torch.int64, device=dev),
           torch.empty(B, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.int64, device=dev))
    ar = torch.arange(B, device=dev)

    def stage(t):
        torch.add(ar, W + t * B, out=s_new)
        torch.add(ar, t * B, out=s_old)
        s_x.copy_(allx[t])
        s_q.copy_(allq[t])

    def step():
        ix.sliding_window_step(s_new, s_x, s_old, s_q, K, NPROBE, out=out)

    for t in range(warm):
        stage(t)
        step()
    torch.cuda.synchronize()
    l0 = ix.launch_count()
    g = torch.cuda.CUDAGraph()
    stage(warm)
    with torch.cuda.graph(g):
        step()
    per_replay = ix.launch_count() - l0
    g.replay()  # step `warm`
    torch.cuda.synchronize()
    evs = [(_ev(), _ev()) for _ in range(steps)]
    for i in range(steps):
        t = warm + 1 + i
        evs[i][0].record()
        stage(t)
        g.replay()
        evs[i][1].record()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    st = ix.stats()
    assert st["live"] == W and st["device_errors"] == 0, st
    res = {"workload": "BASELINE configs[3]: SIFT1M-shaped window 1M, slide 10k/step (insert new + delete expired "
                       "+ 1k queries k=10 nprobe=32) + reclaim; one CUDA-graph replay per step",
           "steps": steps, "step_ms_p50": pct(ms, 50), "step_ms_p99": pct(ms, 99), "step_ms_mean": statistics.mean(ms),
           "step_ms_max": max(ms), "kernels_per_step": per_replay, "live_after": st["live"],
           "slabs_in_use_after": st["slabs_in_use"], "reclaimed_slabs": st["reclaimed_slabs"],
           "inputs": "every step's vectors and queries generated from their own ids (g = id) before the loop, "
                     "resident in HBM; per-step ids computed on device and the step's slice copied into the "
                     "graph's static buffers inside the timed region"}
    del allx, allq
    log(f"window: p50 {res['step_ms_p50']:.3f} ms p99 {res['step_ms_p99']:.3f} ms over {steps} steps")
    return res


def leg_gist(S, dev, log):
    """BASELINE configs[2]: GIST1M-shaped 1M x 960 fp32, nlist=1024: 10k-vector delete batch latency,
    insert throughput (10k batches and bulk 64k batches), search 10k queries k=100 nprobe=32 and the
    recall@10 sweep (first 10 of the k=100 results vs exact top-10)."""
    import torch

    from datagen import Generator, gist_shape

    N, D, KG = 1_000_000, 960, 100
    gen = Generator(gist_shape())
    reps = 61
    cap = N + (reps + 2) * BATCH
    ix = S.Index(D, NLIST, cap, S.num_slabs_for(N + (reps + 2) * BATCH, NLIST), max_batch=65536, max_queries=NQ,
                 max_k=KG, max_nprobe=64, max_train=N_TRAIN, seed=0x6157, device=dev)
    t0 = time.time()
    ix.train(torch.from_numpy(gen.train(N_TRAIN)).to(dev), niter=N_ITER)
    torch.cuda.synchronize()
    t_train = time.time() - t0
    X = torch.from_numpy(gen.range(0, N)).to(dev)
    ids = torch.arange(cap, device=dev)
    e0, e1 = _ev(), _ev()
    e0.record()
    for b0 in range(0, N, 65536):
        ix.insert(ids[b0:min(N, b0 + 65536)], X[b0:b0 + 65536])
    e1.record()
    torch.cuda.synchronize()
    build_rate = N / (e0.elapsed_time(e1) / 1e3)
    Q = torch.from_numpy(gen.queries(0, NQ)).to(dev)
    # exact top-10 (fp32 GEMM, no tf32) for recall
    torch.backends.cuda.matmul.allow_tf32 = False
    xn = (X * X).sum(1)
    gt = []
    for q0 in range(0, NQ, 250):
        q = Q[q0:q0 + 250]
        d = (q * q).sum(1)[:, None] + xn[None, :] - 2.0 * (q @ X.T)
        gt.append(torch.topk(d, 10, dim=1, largest=False).indices)
    gt = torch.cat(gt).cpu().numpy()
    sweep, qps_at_09, np_at_09 = {}, None, None
    for npb in (4, 8, 16, 32, 64):
        for _ in range(2):  # warm-up (graph capture on the 2nd sighting of a call)
            ix.search(Q, KG, npb)
        torch.cuda.synchronize()
        reps_ms = []
        for _ in range(3):
            a, b = _ev(), _ev()
            a.record()
            _, ii = ix.search(Q, KG, npb)
            b.record()
            torch.cuda.synchronize()
            reps_ms.append(a.elapsed_time(b))
        res = ii[:, :10].cpu().numpy()
        rec = float(np.mean([len(set(r) & set(g)) / 10 for r, g in zip(res, gt)]))
        qps = NQ / (statistics.median(reps_ms) / 1e3)
        sweep[npb] = {"recall10": rec, "qps": qps, "ms": statistics.median(reps_ms)}
        if qps_at_09 is None and rec >= 0.9:
            qps_at_09, np_at_09 = qps, npb
    # mutation latencies: 30 delete batches of 10k random live ids, 30 insert batches of 10k new ids
    rng = np.random.default_rng(0x6157)
    perm = torch.from_numpy(rng.permutation(N)[: reps * BATCH].astype(np.int64)).to(dev)
    Xr = X[: BATCH].clone()  # re-inserted payload (new ids): the insert timing does not depend on values
    del_ms, ins_ms = [], []
    for r in range(reps):
        a, b = _ev(), _ev()
        a.record()
        ix.delete(perm[r * BATCH:(r + 1) * BATCH])
        b.record()
        c, d = _ev(), _ev()
        c.record()
        ix.insert(ids[N + r * BATCH:N + (r + 1) * BATCH], Xr)
        d.record()
        del_ms.append((a, b))
        ins_ms.append((c, d))
    torch.cuda.synchronize()
    del_ms = [a.elapsed_time(b) for a, b in del_ms]
    ins_ms = [a.elapsed_time(b) for a, b in ins_ms]
    st = ix.stats()
    assert st["live"] == N and st["device_errors"] == 0, st
    res = {"workload": "BASELINE configs[2]: GIST1M-shaped 1M x 960 fp32, nlist=1024 (GPU-trained, 262144 samples, "
                       "20 iters)",
           # the first call of the leg is reported apart (cold: first touch of the delete path)
           "delete_10k_ms_p50": pct(del_ms[1:], 50), "delete_10k_ms_p99": pct(del_ms[1:], 99),
           "delete_10k_first_call_ms": del_ms[0], "delete_samples": len(del_ms) - 1,
           "deletes_per_s": BATCH / (pct(del_ms[1:], 50) / 1e3),
           "insert_10k_ms_p50": pct(ins_ms, 50), "insert_10k_ms_p99": pct(ins_ms, 99),
           "inserts_per_s_10k_batches": BATCH / (pct(ins_ms, 50) / 1e3),
           "inserts_per_s_bulk_64k_batches": build_rate,
           "qps_k100_nprobe32": sweep[32]["qps"], "recall10_nprobe32": sweep[32]["recall10"],
           "qps_at_recall10_0.9": qps_at_09, "nprobe_at_recall10_0.9": np_at_09, "sweep_k100": sweep,
           "train_s": t_train, "overhead_paper": st["overhead_paper"], "overhead_actual": st["overhead_actual"]}
    log(f"gist: delete p50 {res['delete_10k_ms_p50']:.4f} ms, insert10k {res['insert_10k_ms_p50']:.3f} ms, "
        f"qps@32 {sweep[32]['qps']:.0f} r={sweep[32]['recall10']:.3f}")
    return res


def leg_h(S, dev, log, G, rank, pg, n_total):
    """BASELINE configs[4]: id-sharded SIFT-shaped n_total x 128 (default 100M), nlist=16384, owner(id) =
    id mod G.  Vectors are generated on the device (datagen.DeviceGenerator, bit-identical to the host
    generator).  Reports the build rate, routed 80k-id mutation batches (no collective) and search of
    10k broadcast queries: local search -> NCCL all-gather of the per-shard top-k -> sivf_merge_topk,
    timed on the device as the max over ranks; recall@10 on 100 queries against an exact top-10 kept
    while building (fp32 GEMM over every generated batch, merged across ranks)."""
    import torch

    from datagen import TRAIN_BASE, QUERY_BASE, DeviceGenerator, sift_shape
    from paper_2601_11808_b200 import shard

    NLH, NQH, NGT, MB = 16384, NQ, 100, 80_000
    gen = DeviceGenerator(sift_shape(seed=0x100A))
    local_n = shard.local_count(n_total, G, rank)
    cap = n_total + MB + 64
    ix = S.Index(DIM, NLH, cap, S.num_slabs_for(local_n + MB // G + 1, NLH), max_batch=1 << 20, max_queries=NQH,
                 max_k=K, max_nprobe=128, max_train=1 << 20, shard_rank=rank, shard_count=G, seed=0x100A, device=dev)

    def dmax(ms):
        if pg is None:
            return ms
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    t0 = time.time()
    Xt = torch.empty(1 << 20, DIM, dtype=torch.float32, device=dev)
    gen.range_into(Xt, TRAIN_BASE, 1)  # identical sample on every rank
    ix.train(Xt, niter=N_ITER)
    if pg is not None:
        C = ix.get_centroids()
        pg.broadcast(C, src=0)
        ix.set_centroids(C)
    torch.cuda.synchronize()
    t_train = time.time() - t0
    del Xt
    Qg = torch.empty(NQH, DIM, dtype=torch.float32, device=dev)
    gen.range_into(Qg, QUERY_BASE, 1)
    Qs = Qg[:NGT]
    qn = (Qs * Qs).sum(1)
    torch.backends.cuda.matmul.allow_tf32 = False
    gt_d = torch.full((NGT, 10), float("inf"), device=dev)
    gt_i = torch.full((NGT, 10), -1, dtype=torch.int64, device=dev)
    B = 1 << 20
    Xb = torch.empty(B, DIM, dtype=torch.float32, device=dev)
    ins_ms = 0.0
    t0 = time.time()
    for j0 in range(0, local_n, B):
        nb = min(B, local_n - j0)
        gen.range_into(Xb[:nb], rank + j0 * G, G)
        ids = rank + G * torch.arange(j0, j0 + nb, device=dev, dtype=torch.int64)
        a, b = _ev(), _ev()
        a.record()
        ix.insert(ids, Xb[:nb])
        b.record()
        x = Xb[:nb]
        d = qn[:, None] + (x * x).sum(1)[None, :] - 2.0 * (Qs @ x.T)
        dd, ii = torch.topk(torch.cat([gt_d, d], 1), 10, dim=1, largest=False)
        gt_i = torch.gather(torch.cat([gt_i, ids[None, :].expand(NGT, -1)], 1), 1, ii)
        gt_d = dd
        b.synchronize()
        ins_ms += a.elapsed_time(b)
    torch.cuda.synchronize()
    t_build = time.time() - t0
    build_rate = n_total / (dmax(ins_ms) / 1e3)
    del Xb
    if pg is not None:
        ad = [torch.empty_like(gt_d) for _ in range(G)]
        ai = [torch.empty_like(gt_i) for _ in range(G)]
        pg.all_gather(ad, gt_d)
        pg.all_gather(ai, gt_i)
        dd, ii = torch.topk(torch.cat(ad, 1), 10, dim=1, largest=False)
        gt_i = torch.gather(torch.cat(ai, 1), 1, ii)
    gt = gt_i.cpu().numpy()
    st = ix.stats()
    assert st["live"] == local_n and st["device_errors"] == 0, st
    log(f"H: train {t_train:.1f}s build {t_build:.1f}s ({build_rate / 1e6:.1f} M/s device-timed)")

    osamp = h_oracle_sample(ix, dev, gen, local_n, G, rank, Qg, log)

    def search(npb):
        if pg is not None:  # coarse step sharded over queries, probe sets all-gathered (NEXT-3)
            return shard.sharded_search(pg, ix, Qg, K, npb)
        return ix.search(Qg, K, npb)

    sweep, qps_at_09, np_at_09 = {}, None, None
    for npb in (8, 16, 32, 64):
        for _ in range(2):  # warm-up (graph capture on the 2nd sighting of a call)
            search(npb)
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            if pg is not None:
                pg.barrier()
            a, b = _ev(), _ev()
            a.record()
            _, ii = search(npb)
            b.record()
            torch.cuda.synchronize()
            times.append(dmax(a.elapsed_time(b)))
        res = ii[:NGT, :10].cpu().numpy()
        rec = float(np.mean([len(set(r) & set(g)) / 10 for r, g in zip(res, gt)]))
        ms = statistics.median(times)
        sweep[npb] = {"recall10": rec, "qps": NQH / (ms / 1e3), "ms": ms}
        if qps_at_09 is None and rec >= 0.9:
            qps_at_09, np_at_09 = NQH / (ms / 1e3), npb
    # routed mutations: a global batch of 80k random live ids deleted and 80k new ids inserted
    rng = np.random.default_rng(0x100A)
    dids = rng.choice(n_total, MB, replace=False).astype(np.int64)
    nids = np.arange(n_total, n_total + MB, dtype=np.int64)
    dl = torch.from_numpy(shard.route(dids, G, rank)[0]).to(dev)
    nl = torch.from_numpy(shard.route(nids, G, rank)[0]).to(dev)
    Xn = torch.empty(nl.shape[0], DIM, dtype=torch.float32, device=dev)
    gen.range_into(Xn, n_total + rank, G)
    if pg is not None:
        pg.barrier()
    a, b, c = _ev(), _ev(), _ev()
    a.record()
    nd = ix.delete(dl)
    b.record()
    ix.insert(nl, Xn)
    c.record()
    torch.cuda.synchronize()
    del_ms, ins80_ms = dmax(a.elapsed_time(b)), dmax(b.elapsed_time(c))
    st = ix.stats()
    assert st["live"] == local_n and st["device_errors"] == 0, st
    res = {"workload": f"BASELINE configs[4]: id-sharded SIFT-shaped {n_total // 1_000_000}M x 128, nlist=16384, "
                       f"G={G} (owner = id mod G), 10k broadcast queries k=10, per-shard top-k all-gather + merge",
           "n_total": n_total, "gpus": G, "build_inserts_per_s": build_rate, "train_s": t_train,
           "deletes_per_s_80k_routed": MB / (del_ms / 1e3), "inserts_per_s_80k_routed": MB / (ins80_ms / 1e3),
           "delete_80k_ms": del_ms, "insert_80k_ms": ins80_ms,
           "qps_nprobe32": sweep[32]["qps"], "recall10_nprobe32": sweep[32]["recall10"],
           "qps_at_recall10_0.9": qps_at_09, "nprobe_at_recall10_0.9": np_at_09, "sweep": sweep,
           "oracle_sampled": osamp,
           "recall_truth": f"exact top-10 of {NGT} queries (fp32 GEMM over every generated batch)",
           "scaling": "strong (the global index is fixed; each rank holds n/G)"}
    log(f"H: qps@32 {sweep[32]['qps']:.0f} r={sweep[32]['recall10']:.3f}; delete80k {del_ms:.3f} ms")
    Ch = ix.get_centroids()
    base = h_phase_ms(ix, Qg)
    del ix
    torch.cuda.empty_cache()
    if G == 1:
        res["projection"] = h_projection(S, dev, log, gen, Ch, Qg, n_total, base, sweep[32]["ms"])
    return res


def h_phase_ms(ix, Qg, reps=3):
    """Per-phase device times of a search of Qg (k=10, nprobe=32) on ix, launched directly
    with the library's phase events."""
    import torch

    ix.search(Qg, K, NPROBE)
    torch.cuda.synchronize()
    ix.profile(True)
    ix.profile_read()
    for _ in range(reps):
        ix.search(Qg, K, NPROBE)
    torch.cuda.synchronize()
    p = ix.profile_read()
    ix.profile(False)
    return {k: v[0] / v[1] for k, v in p.items() if v[1]}


def h_projection(S, dev, log, gen, C, Qg, n_total, base, base_ms, nvlink_gbs=400.0, coll_us=20.0):
    """BASELINE configs[4] on one GPU: for G in {2, 4, 8}, shard 0 of the G-way id sharding
    (owner = id mod G, n/G vectors, the replicated quantizer) is built and searched here, one
    after another; every shard holds a statistically identical 1/G of the ids.  Measured per
    shard: build rate and the search phases; the merge of G per-shard top-k lists
    (sivf_merge_topk) is measured on [G][nq][k] inputs.  PROJECTED G-GPU search time = shard
    search + all-gather (modelled: bytes / nvlink_gbs + coll_us per collective, NCCL all-gather
    over NVLink 5; no second GPU here) + merge; the replicated coarse step is the Amdahl term."""
    import torch

    from datagen import TRAIN_BASE  # noqa: F401  (same generator family as the H leg)
    from paper_2601_11808_b200 import shard

    NLH = C.shape[0]
    out = {"method": "PROJECTION from measured single-shard runs on one B200 (no multi-GPU measurement): "
                     "T(G) = shard search (measured) + all-gather (model) + merge (measured)",
           "allgather_model": {"gbs": nvlink_gbs, "latency_us_per_collective": coll_us, "collectives": 2},
           "G1": {"search_ms": base_ms, "phases_ms": base}}
    for Gp in (2, 4, 8):
        local_n = (n_total + Gp - 1) // Gp
        ix = S.Index(DIM, NLH, n_total + 64, S.num_slabs_for(local_n + 1, NLH), max_batch=1 << 20,
                     max_queries=Qg.shape[0], max_k=K, max_nprobe=128, shard_rank=0, shard_count=Gp, seed=0x100A,
                     device=dev)
        ix.set_centroids(C)
        B = 1 << 20
        Xb = torch.empty(B, DIM, dtype=torch.float32, device=dev)
        ins_ms = 0.0
        for j0 in range(0, local_n, B):
            nb = min(B, local_n - j0)
            gen.range_into(Xb[:nb], j0 * Gp, Gp)  # ids 0, G, 2G, ... (shard 0)
            ids = Gp * torch.arange(j0, j0 + nb, device=dev, dtype=torch.int64)
            a, b = _ev(), _ev()
            a.record()
            ix.insert(ids, Xb[:nb])
            b.record()
            b.synchronize()
            ins_ms += a.elapsed_time(b)
        del Xb
        st = ix.stats()
        assert st["live"] == local_n and st["device_errors"] == 0, st
        for _ in range(2):
            ix.search(Qg, K, NPROBE)
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            a, b = _ev(), _ev()
            a.record()
            d, i = ix.search(Qg, K, NPROBE)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        shard_ms = statistics.median(times)
        ph = h_phase_ms(ix, Qg)
        # NEXT-3 query-sharded coarse step: rank 0's slice of the probe sets (sivf_probe on
        # nq/G queries), then the scan + merge with the all-gathered full probe sets
        # (sivf_search_probed); results bit-identical to the replicated search
        nq = Qg.shape[0]
        lo, hi = shard.query_slice(nq, Gp, 0)
        probes = ix.probe(Qg, NPROBE)
        pt, st_ = [], []
        for rep in range(5):
            a, b = _ev(), _ev()
            a.record()
            ix.probe(Qg[lo:hi], NPROBE)
            b.record()
            c_, d_ = _ev(), _ev()
            c_.record()
            dq, iq = ix.search_probed(Qg, probes, K)
            d_.record()
            torch.cuda.synchronize()
            if rep >= 2:
                pt.append(a.elapsed_time(b))
                st_.append(c_.elapsed_time(d_))
        qs_equal = bool(torch.equal(iq, i) and torch.equal(dq, d))
        coarse_slice_ms, scan_probed_ms = statistics.median(pt), statistics.median(st_)
        del ix
        torch.cuda.empty_cache()
        nq = Qg.shape[0]
        gd = d[None].expand(Gp, nq, K).contiguous()
        gi = i[None].expand(Gp, nq, K).contiguous()
        S.merge_topk(gd, gi)
        torch.cuda.synchronize()
        mt = []
        for _ in range(5):
            a, b = _ev(), _ev()
            a.record()
            S.merge_topk(gd, gi)
            b.record()
            torch.cuda.synchronize()
            mt.append(a.elapsed_time(b))
        merge_ms = statistics.median(mt)
        ag_bytes = Gp * nq * K * (4 + 8)  # gathered per rank: dist f32 + id i64 of every shard
        ag_ms = (ag_bytes * (Gp - 1) / Gp) / (nvlink_gbs * 1e9) * 1e3 + 2 * coll_us / 1e3
        t_ms = shard_ms + ag_ms + merge_ms
        agp_bytes = nq * NPROBE * 4  # gathered probe sets (int32), one collective
        agp_ms = (agp_bytes * (Gp - 1) / Gp) / (nvlink_gbs * 1e9) * 1e3 + coll_us / 1e3
        tq_ms = coarse_slice_ms + agp_ms + scan_probed_ms + ag_ms + merge_ms
        out[f"G{Gp}"] = {"local_n": local_n, "build_inserts_per_s_shard": local_n / (ins_ms / 1e3),
                         "query_sharded_coarse": {
                             "coarse_slice_ms": coarse_slice_ms, "queries_per_rank": hi - lo,
                             "scan_merge_probed_ms": scan_probed_ms, "probe_allgather_bytes": agp_bytes,
                             "probe_allgather_ms_model": agp_ms, "projected_search_ms": tq_ms,
                             "projected_qps": nq / (tq_ms / 1e3), "projected_speedup_vs_G1": base_ms / tq_ms,
                             "results_equal_replicated": qs_equal},
                         "search_ms_shard": shard_ms, "phases_ms_shard": ph, "merge_ms": merge_ms,
                         "allgather_bytes_per_rank": ag_bytes, "allgather_ms_model": ag_ms,
                         "projected_search_ms": t_ms, "projected_qps": nq / (t_ms / 1e3),
                         "projected_speedup_vs_G1": base_ms / t_ms,
                         "amdahl_coarse_share": ph.get("coarse", 0.0) / t_ms}
        log(f"H projection G={Gp}: shard search {shard_ms:.3f} ms (coarse {ph.get('coarse', 0):.3f}, scan "
            f"{ph.get('scan', 0):.3f}), merge {merge_ms:.3f}, all-gather model {ag_ms:.3f} -> projected "
            f"{nq / (t_ms / 1e3) / 1e6:.2f}M QPS, x{base_ms / t_ms:.2f} vs G=1")
        log(f"H projection G={Gp} query-sharded coarse: slice coarse {coarse_slice_ms:.3f} ms + probe all-gather "
            f"{agp_ms:.3f} + probed scan/merge {scan_probed_ms:.3f} + top-k all-gather/merge -> "
            f"{nq / (tq_ms / 1e3) / 1e6:.2f}M QPS, x{base_ms / tq_ms:.2f} vs G=1 (equal: {qs_equal})")
    return out


def h_oracle_sample(ix, dev, dgen, local_n, G, rank, Qg, log, n_ids=10_000, n_q=100):
    """SURVEY §8(d) "H: sampled" — the 100M index is too large for an oracle index, so the
    oracle checks a sample of it: (1) for 10^4 random live ids, the (list, live) state of the
    GPU's dumped ATT against oracle.assign of the regenerated vector (host generator); (2) for
    100 queries, the probe SET against oracle.probe, and the GPU's top-k against the oracle's
    top-k by (dist32, id) over every member of the probed lists (membership from the dumped
    state, verified on the sample in (1); vectors regenerated by the device generator, which a
    GPU test proves bit-identical to the host one).  Integer SIFT-shaped data: exact equality."""
    import torch

    import oracle as O
    from datagen import Generator, sift_shape

    t0 = time.time()
    O.set_threads(os.cpu_count() or 1)
    hgen = Generator(sift_shape(seed=0x100A))
    C = ix.get_centroids().cpu().numpy()
    loi = ix.dump_state()[0]
    rng = np.random.default_rng(0x5A)
    lids = rng.choice(local_n, n_ids, replace=False).astype(np.int64)
    gids = lids * G + rank
    want = O.assign(C, hgen.take(gids))
    got = loi[torch.from_numpy(lids).to(dev)].cpu().numpy()
    ids_ok = int((got == want).sum())
    Q = Qg[:n_q].contiguous()
    d, i, p = ix.search(Q, K, NPROBE, return_probes=True)
    d, i, Qh, ph = d.cpu().numpy(), i.cpu().numpy(), Q.cpu().numpy(), p.cpu().numpy()
    probes_ok = sum(set(ph[q].tolist()) == set(O.probe(C, Qh[q], NPROBE).tolist()) for q in range(n_q))
    q_ok, scanned = 0, 0
    for q in range(n_q):
        lid = torch.nonzero(torch.isin(loi, p[q])).squeeze(1)
        g = lid * G + rank
        Xc = torch.empty(g.shape[0], DIM, dtype=torch.float32, device=dev)
        dgen.take_into(Xc, g.contiguous())
        od, oi = O.topk_candidates(Qh[q], Xc.cpu().numpy(), g.cpu().numpy(), K)
        scanned += g.shape[0]
        q_ok += int(np.array_equal(od, d[q]) and np.array_equal(oi, i[q]))
    res = {"ids_checked": n_ids, "ids_ok": ids_ok, "queries_checked": n_q, "queries_ok": q_ok,
           "probe_sets_ok": int(probes_ok), "nprobe": NPROBE, "k": K, "candidates_scanned_by_oracle": scanned,
           "seconds": time.time() - t0,
           "method": "ids: dumped (list, live) vs oracle.assign of the regenerated vector; queries: probe set vs "
                     "oracle.probe, top-k vs oracle.topk_candidates over all members of the probed lists"}
    log(f"H oracle sample: ids {ids_ok}/{n_ids}, probe sets {probes_ok}/{n_q}, queries {q_ok}/{n_q} "
        f"({scanned} candidates, {res['seconds']:.1f}s)")
    return res


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sivf(args)


if __name__ == "__main__":
    main()
