#!/usr/bin/env python
"""Benchmark of the DynaSpec dynamic drafter head on B200 (BASELINE.json metric:
"draft-head tokens/s & us/step (V=128k, d=4096); % HBM peak; speedup vs dense").

A bench "step" is one draft cycle: `positions` consecutive DynaSpec draft steps (Alg. 1 lines
7-11 for t = 0..gamma-1 with the position-aware budget 32,32,8,...) over one batch of B
synthetic rows per GPU: router (S_m stream) -> select -> gathered head + fused epilogue (S_d).
value = draft tokens (rows x positions, all ranks) per second of device time (max over ranks).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama3] [--batch B]
       python bench.py --impl reference ...   (the CPU oracle, timed on the host cores)
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import inputs as S  # noqa: E402

L2_FLUSH_BYTES = 512 << 20  # 4x the 126 MB L2
L2_CLEAN_BYTES = 256 << 20  # 2x the L2


class L2Flush:
    """Cold L2 between timed iterations (outside every event pair): write a 512 MB buffer (> L2),
    then read a separate 256 MB buffer.  The write alone leaves the L2 full of DIRTY lines of the
    flush buffer, and the next kernel's first ~126 MB of reads then pay for their write-back to HBM
    (scripts/probe/stream_probe4.cu: a 131 MB TMA stream takes 27.0 us after a write-only flush,
    20.3 us after write + read) -- that would time the flush, not the kernel.  After the read the
    L2 holds clean lines of unrelated data: none of the kernel's inputs or weights is resident."""

    def __init__(self, dev):
        self.buf = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
        self.clean = torch.ones(L2_CLEAN_BYTES // 8, dtype=torch.int64, device=dev)
        self.sink = torch.empty((), dtype=torch.int64, device=dev)

    def zero_(self):
        self.buf.zero_()
        torch.sum(self.clean, dim=0, out=self.sink)


L2_HOW = ("flushed before every step, outside the timed event pair: 512 MB write, then a 256 MB read of a "
          "separate buffer so the L2 holds clean unrelated lines (a write-only flush leaves ~126 MB of dirty "
          "lines whose write-back would be timed inside the next kernel)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3", choices=list(S.CONFIGS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--partition", default="kmeans", choices=["kmeans", "random"])
    ap.add_argument("--kmeans-iters", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--profile", action="store_true", help="timed steps only (for ncu): no dense/e2e/cpu legs")
    ap.add_argument("--shard", default="requests", choices=["requests", "clusters"],
                    help="requests: the request batch is split over the ranks (no data-path collective); "
                         "clusters: every rank stores 1/N of W_perm, records are all-gathered (SURVEY 8(e))")
    ap.add_argument("--nccl-log", default=None, help="with --gpus N > 1 (self-spawned): NCCL_DEBUG=INFO into this file")
    return ap.parse_args()


def maybe_spawn(args):
    """`python bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one per GPU)
    with torch.distributed.run on 127.0.0.1 and return its exit code; None when already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if args.nccl_log:
        env["NCCL_DEBUG"] = "INFO"
        env["NCCL_DEBUG_FILE"] = args.nccl_log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------- distributed

def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        if args is not None and ws != args.gpus and rank == 0:
            print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers

def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j.get("hbm_gbs"), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(config, batch):
    """dram bytes per head launch from the committed ncu --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "head_traffic.json")
    if not os.path.exists(p):
        return None
    j = json.load(open(p))
    return j.get(f"{config}_B{batch}")


class HostRows:
    """fp64 row access to a host bf16 head for the oracle."""

    def __init__(self, W):
        self.W = W
        self.shape = tuple(W.shape)

    def __getitem__(self, idx):
        return self.W[torch.as_tensor(np.asarray(idx), dtype=torch.long)].to(torch.float64).numpy()


# ----------------------------------------------------------------------------- oracle (CPU) arm

def oracle_cycles(C, B, dtype, seconds, W_host, rt_host, part):
    """Run whole oracle draft cycles (all positions) on the host until `seconds` elapse."""
    from oracle import dynaspec_oracle as O
    W = HostRows(W_host)
    ro = tuple(None if x is None else x.to(torch.float64).numpy() for x in rt_host)
    rows, t0, cycles = 0, time.perf_counter(), 0
    while True:
        for t in range(C.positions):
            hp, e, hn = S.step_inputs(B, C.d, t, dtype, sibling_eps=0.1 if C.shared else None)
            f = lambda x: x.to(torch.float64).numpy()
            O.draft_step(part, ro, W, f(hp), f(e), f(hn), t, C.k_max, C.k_min, C.k_t, shared=C.shared)
            rows += B
        cycles += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    threads = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        threads = max(i.get("num_threads", 1) for i in threadpool_info()) or threads
    except Exception:
        pass
    return rows / el, el, cycles, threads


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle as it stands, on this box's host cores.  Each step is a
    bounded sample of the workload: one whole draft cycle (all positions) of B rows."""
    if rank != 0:
        return
    from oracle import dynaspec_oracle as O
    C = S.CONFIGS[args.config]
    B = args.batch or C.B
    unit = "draft tokens/s"
    W_host = S.lm_head(C.V, C.d, 0, args.dtype)
    rt_host = S.router(C.d, C.h_r, C.M, 1, args.dtype)
    part, part_info = oracle_partition(C, W_host, args)
    total_rows, total_t, thr = 0.0, 0.0, 1
    for i in range(args.warmup + args.steps):
        r, el, cyc, thr = oracle_cycles(C, B, args.dtype, 0.0, W_host, rt_host, part)
        if i >= args.warmup:
            total_rows += r * el
            total_t += el
    value = total_rows / total_t
    line = {"impl": "reference", "metric": "draft-head tokens/s & us/step (V=128k,d=4096); % HBM peak; speedup vs dense",
            "value": value, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * total_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random-init weights and hidden states)",
            "config": {"workload": C.name, "V": C.V, "d": C.d, "M": C.M, "h_r": C.h_r, "batch_per_gpu": B,
                       "positions": C.positions, "k_schedule": [budget_of(t, C) for t in range(C.positions)],
                       "k_t": C.k_t, "shared": C.shared, **part_info},
            "cpu_baseline": {"value": value, "unit": unit, "cores": thr, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{args.steps} whole draft cycles ({C.positions} positions x B={B}) of the "
                                       "numpy fp64 oracle on the host"},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_partition(C, W_host, args):
    """The reference arm's S0: the oracle's own integer-exact spherical k-means (O1, R12) on the same
    synthetic W, seed and iteration cap as the GPU arm (whose builder is bit-exact against it, so both
    arms stream the same clusters) -- untimed setup.  Falls back to the seeded random partition when
    the fp64 working set would not fit comfortably in host memory (Gemma-3 scale)."""
    from oracle import dynaspec_oracle as O
    if args.partition == "kmeans" and C.V * C.d * 8 * 3 <= (24 << 30):
        t0 = time.perf_counter()
        b = O.build_clusters(W_host.to(torch.float64).numpy(), C.M, seed=2, max_iters=args.kmeans_iters)
        return ({"perm": b["perm"], "offsets": b["offsets"]},
                {"partition": "spherical k-means (oracle, integer-exact; same partition as the GPU arm)",
                 "kmeans_iters": int(b["iters"]), "build_s": round(time.perf_counter() - t0, 1)})
    perm, off = O.layout(S.random_partition(C.V, C.M, 2), C.M)
    return {"perm": perm, "offsets": off}, {"partition": "seeded random (Zipf sizes)"}


def single_core_rate(C, B, dtype, seconds, W_host, rt_host, part):
    """The oracle pinned to one core (sched_setaffinity {0}, BLAS limited to one thread): the
    single-thread figure SURVEY 8(d) asks for next to the all-cores one."""
    prev = os.sched_getaffinity(0)
    try:
        os.sched_setaffinity(0, {min(prev)})
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            rate, el, cyc, _ = oracle_cycles(C, B, dtype, seconds, W_host, rt_host, part)
    finally:
        os.sched_setaffinity(0, prev)
    return {"value": rate, "unit": "draft tokens/s", "cores": 1, "core_id": min(prev),
            "sample": f"{cyc} whole draft cycle(s) ({C.positions} positions x B={B}, {el:.1f} s)"}


def budget_of(t, C):
    """k_c(t) with the k_min clamp (R1) — the schedule the bench drives (for reporting only)."""
    return C.k_max if t < 2 else max(C.k_min, C.k_max // ((t + 1) * 2))


# ----------------------------------------------------------------------------- GPU arm

def run_ours(args, ws, rank, local):
    from paper_2510_13847_b200 import dynaspec as D
    dev = torch.device("cuda", torch.cuda.current_device())
    C = S.CONFIGS[args.config]
    from paper_2510_13847_b200.parallel import row_range
    B_total = args.batch or C.B
    # request sharding: a batch of B_total requests is split over the ranks (strong scaling); a
    # single-request stream (B = 1) runs one independent stream per rank (weak scaling)
    strong = ws > 1 and B_total >= ws and B_total > 1
    r0, r1 = row_range(B_total, rank, ws) if strong else (0, B_total)
    B = r1 - r0
    tdt = S.TORCH_DTYPES[args.dtype]
    # ---- setup (untimed): weights, router, offline partition (S0)
    W = S.lm_head(C.V, C.d, 0, args.dtype, device=dev)
    rt = [None if x is None else x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, args.dtype)]
    t0 = time.perf_counter()
    if args.partition == "kmeans":
        try:
            clusters = D.Clusters.build(W, C.M, seed=2, max_iters=args.kmeans_iters)
            part_info = {"partition": "spherical k-means (GPU, integer-exact)", "kmeans_iters": clusters.iters}
        except D.DynaspecError as ex:
            if ex.name != "DS_ERR_UNSUPPORTED":
                raise
            args.partition = "random"
    if args.partition == "random":
        tau = torch.as_tensor(S.random_partition(C.V, C.M, 2), dtype=torch.int32, device=dev)
        clusters = D.Clusters.from_tau(W, tau, C.M)
        part_info = {"partition": "seeded random (Zipf sizes)"}
    torch.cuda.synchronize()
    part_info["build_s"] = round(time.perf_counter() - t0, 3)
    part_info["cluster_size_min_max"] = [clusters.min_size, clusters.max_size]
    router = D.Router(*rt)
    W_host = W.cpu() if (rank == 0 and ws == 1 and not args.no_cpu_baseline) else None
    del W  # the drafter-side copy W_perm is what the head reads (R21)
    torch.cuda.empty_cache()

    # ---- input pool: distinct (h_prev, e, h_new) per position so touched clusters vary (64 sets at
    # small B, fewer when a set is large); strong sharding: every rank draws the whole batch, keeps its rows
    set_bytes = B_total * C.d * 3 * C.positions * 2
    pool = 64 if set_bytes <= (1 << 20) else max(2, min(16, (256 << 20) // set_bytes))
    seed_base = 1000 if strong else 1000 + 977 * rank
    # every (set, position) draws its own seeds: consecutive positions are independent requests' worth
    # of router inputs (no shared selection between positions of a cycle, so no L2 reuse across them)
    inputs = [[tuple(x[r0:r1].contiguous().to(dev) for x in S.step_inputs(
        B_total, C.d, C.positions * i + t, args.dtype, pool=1 << 20, sibling_eps=0.1 if C.shared else None,
        base_seed=seed_base))
               for t in range(C.positions)] for i in range(pool)]
    steppers = [D.DraftStep(clusters, router, B, C.k_t, shared=C.shared, two_streams=False, device=dev)
                for _ in range(C.positions)]
    fused = steppers[0].launches == 1
    kb = [budget_of(t, C) for t in range(C.positions)]
    flush = L2Flush(dev)
    head_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(C.positions)] for _ in range(pool)]
    for lst in head_ev:
        for a, b in lst:
            a.record(); b.record()

    # Fused mode: every launch of the cycle IS the dominant kernel, so its average duration is the
    # event-timed cycle / launches (events between launches would break the PDL chaining).
    # Two-kernel modes: events bracket each head launch on its stream.
    timed_heads = not fused

    # The timed cycles carry NO head events (event nodes between launches cost time inside the
    # graph); the head durations come from a separate, instrumented replay of the same cycles.
    def cycle(i, with_events=False):
        for t in range(C.positions):
            hp, e, hn = inputs[i][t]
            steppers[t](hp, e, hn, t, C.k_max, C.k_min,
                        head_events=head_ev[i][t] if (timed_heads and with_events) else None)

    use_graph = not args.no_graph
    graphs = []
    if use_graph:
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(pool):   # warm the library (attributes, first launches) outside capture
                cycle(i)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        egraphs = []
        for i in range(pool):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cycle(i)
            graphs.append(g)
            if timed_heads:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    cycle(i, True)
                egraphs.append(g)
        torch.cuda.synchronize()

    def run(i, with_events=False):
        if use_graph:
            (egraphs if with_events else graphs)[i % pool].replay()
        else:
            cycle(i % pool, with_events)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.warmup):
        flush.zero_()
        run(i)
    torch.cuda.synchronize()
    barrier(ws)
    clk = ClockSampler(local)
    clk.start()
    torch.cuda.synchronize()
    barrier(ws)
    head_ms, head_bytes = [], []
    for i in range(args.steps):
        flush.zero_()                       # cold L2 between steps, outside the event pair
        ev[i][0].record()
        run(args.warmup + i)
        ev[i][1].record()
    torch.cuda.synchronize()
    barrier(ws)
    clocks = clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if timed_heads:  # the instrumented replay of the same cycles (same cold-L2 protocol), untimed
        for i in range(args.steps):
            flush.zero_()
            run(args.warmup + i, with_events=True)
            torch.cuda.synchronize()
    # dominant-kernel durations
    for i in range(args.steps):
        j = (args.warmup + i) % pool
        for t in range(C.positions):
            if not timed_heads:
                head_ms.append(step_ms[i] / C.positions)
                continue
            try:
                head_ms.append(head_ev[j][t][0].elapsed_time(head_ev[j][t][1]))
            except RuntimeError:
                head_ms.append(float("nan"))
    # algorithmic bytes per head launch: shortlist rows x d x b_w + h_new + perm ids + outputs
    bw = 2 if args.dtype == "bf16" else 4
    vs_sizes, union_list = [], []
    # replay each pool entry once more (untimed) to read back its shortlist sizes
    clusters_sizes = np.diff(clusters.offsets.cpu().numpy().astype(np.int64))
    sizes_by_pool = {}
    for j in sorted({(args.warmup + i) % pool for i in range(args.steps)}):
        run(j)
        torch.cuda.synchronize()
        per_t = []
        for t in range(C.positions):
            st = steppers[t]
            cnt = st.sel_count.cpu()
            offs = st.sl_offsets.cpu()
            sel = st.sel.cpu()
            rows_each = [int(offs[r, cnt[r]]) for r in range(cnt.numel())]
            union = sorted({int(m) for r in range(cnt.numel()) for m in sel[r, :cnt[r]].tolist()})
            csz = clusters_sizes[union].sum() if union else 0
            per_t.append((rows_each, int(csz)))
        sizes_by_pool[j] = per_t
    for i in range(args.steps):
        j = (args.warmup + i) % pool
        for t in range(C.positions):
            n_rows, union_rows = sizes_by_pool[j][t]
            vs_sizes.append(sum(n_rows) / len(n_rows))
            union_list.append(union_rows)
            # algorithmic bytes: the UNION of the rows' shortlists is streamed once
            vs = union_rows
            hb_ = vs * C.d * bw + 4 * vs + B * C.d * bw + B * (C.k_t * 12 + 4)
            if fused:  # the fused kernel also streams the router: W1, W2, x = [h_prev || e]
                hb_ += (max(C.h_r, 0) or C.M) * 2 * C.d * bw + C.M * C.h_r * bw + B * 2 * C.d * bw + B * C.M * 4
            head_bytes.append(hb_)
    total_ms = sum(step_ms)
    tot_ms_max = max_over_ranks(total_ms, ws)
    rows_all = (B_total if strong else B * ws) * C.positions * args.steps
    value = rows_all / (tot_ms_max / 1e3)
    ms_per_step = tot_ms_max / args.steps
    hb = np.array(head_bytes)
    hm = np.array(head_ms)
    good = np.isfinite(hm)
    peak, peak_src = measured_peaks()
    achieved = float(hb[good].sum() / (hm[good].sum() / 1e3) / 1e9) if good.any() else None
    head_share = float(hm[good].sum() / total_ms) if good.any() else None

    # ---- dense comparator (untimed above): full-V head + log-softmax + top-k_t
    dyn_us_per_pos = 1e3 * ms_per_step / C.positions
    stream_bw = gathered_stream_bandwidth(D, steppers, inputs, C, B, dev, flush, bw) if (fused and not args.profile) \
        else None
    if args.profile:
        dense, e2e = {"best_us": float("nan")}, None
        args.no_cpu_baseline = True
    else:
        dense = dense_baseline(D, clusters, inputs, B, C, dev, flush)
        e2e = e2e_run(D, steppers, clusters, router, C, B, args, dev, flush, ws, B_total if strong else B * ws)
        two = two_stream_run(D, clusters, router, inputs, C, B, args, dev, flush)
        overlap = core_overlap_run(D, clusters, router, inputs, C, B, args, dev, flush)
        static = static_heads_run(D, clusters, inputs, C, B, dev, flush)
        verify = verify_run(D, C, dev, flush, int(round(float(np.mean(vs_sizes)))))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle import dynaspec_oracle as O
        perm_h, off_h = O.layout(clusters.tau.cpu().numpy().astype(np.int64), C.M)
        rate, el, cyc, thr = oracle_cycles(C, B, args.dtype, args.cpu_seconds, W_host,
                                           [None if x is None else x.cpu() for x in rt],
                                           {"perm": perm_h, "offsets": off_h})
        rt_h = [None if x is None else x.cpu() for x in rt]
        cpu = {"value": rate, "unit": "draft tokens/s", "cores": thr, "kind": "oracle", "cpu_model": cpu_model(),
               "host_cpus": os.cpu_count(),
               "sample": f"{cyc} whole draft cycle(s) ({C.positions} positions x B={B}, {el:.1f} s) of the numpy "
                         "fp64 oracle on the same partition/router/W",
               "single_core": single_core_rate(C, B, args.dtype, min(10.0, args.cpu_seconds), W_host, rt_h,
                                               {"perm": perm_h, "offsets": off_h})}
    launches = sum(s.launches for s in steppers) * args.steps
    if rank == 0:
        line = {
            "metric": "draft-head tokens/s & us/step (V=128k,d=4096); % HBM peak; speedup vs dense",
            "value": value, "unit": "draft tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic (seeded random-init weights, router and hidden states)",
            "config": {"workload": C.name, "V": C.V, "d": C.d, "M": C.M, "h_r": C.h_r, "batch_per_gpu": B,
                       "global_batch": B_total if strong else B * ws,
                       "positions": C.positions, "k_schedule": kb, "k_t": C.k_t, "shared": C.shared,
                       "parallelism": (f"request-sharded x{ws}: {B_total} requests split over the ranks "
                                       "(no data-path collective)" if strong else
                                       f"request-sharded x{ws}: one independent B={B} request stream per rank "
                                       "(no data-path collective)"),
                       "input_pool": pool,
                       "us_per_draft_step": dyn_us_per_pos,
                       "mean_shortlist_rows": float(np.mean(vs_sizes)),
                       "mean_union_rows": float(np.mean(union_list)),
                       "union_fraction_of_V": float(np.mean(union_list)) / C.V,
                       "l2": L2_HOW,
                       "cuda_graph": use_graph, **part_info,
                       "dense_us_per_draft_step": dense["best_us"], "dense_detail": dense,
                       "speedup_vs_dense": dense["best_us"] / dyn_us_per_pos if dyn_us_per_pos else None,
                       "head_share_of_step": head_share,
                       "step_mode": "fused one-launch step" if fused else "two kernels per step",
                       "two_stream_mode": None if args.profile else two,
                       "gathered_block_streaming": stream_bw,
                       "drafter_core_overlap": None if args.profile else overlap,
                       "static_frequency_heads": None if args.profile else static,
                       "verification": None if args.profile else verify},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "traffic": committed_traffic(C.name, B), "kernel": steppers[0].kernel,
                         "duration_source": ("CUDA events around each timed cycle / launches per cycle (every launch "
                                             "is the dominant kernel; PDL-chained)" if fused else
                                             "CUDA events around each head launch"),
                         "peak_source": peak_src, "frac_of_8TBps": achieved / 8000.0 if achieved else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line))


def gathered_stream_bandwidth(D, steppers, inputs, C, B, dev, flush, bw, reps=3):
    """Untimed instrumented steps (dynaspec_debug_set_trace): HBM bandwidth of the streaming phase
    of the fused step on the gathered cluster blocks = shortlist bytes / (last CTA done streaming
    - first CTA started streaming), per draft position, each position run alone after an L2 flush
    (cold HBM for every position, not only the first of a cycle)."""
    G = torch.cuda.get_device_properties(dev).multi_processor_count
    kern = steppers[0].kernel
    if kern.startswith("ds::gstep_kernel"):
        s0, s1 = 5, 6      # gstep.cu trace slots: TopK mask ready (streaming starts), consumers done
    elif kern.startswith("ds::cstep_kernel"):
        s0, s1 = 4, 5      # cstep.cu trace slots
    else:
        return None
    bufs = [torch.zeros(G * 64, dtype=torch.int64, device=dev) for _ in range(C.positions)]
    per_t = [[] for _ in range(C.positions)]
    for rep in range(reps):
        for b in bufs:
            b.zero_()
        for t in range(C.positions):
            flush.zero_()
            torch.cuda.synchronize()
            D.debug_set_trace(bufs[t])
            steppers[t](*inputs[rep % len(inputs)][t], t, C.k_max, C.k_min)
            D.debug_set_trace(None)
            torch.cuda.synchronize()
        for t in range(C.positions):
            a = bufs[t].view(G, 64)[:, :32].cpu().numpy().astype(np.float64)
            st = steppers[t]
            cnt = st.sel_count.cpu()
            offs = st.sl_offsets.cpu()
            rows = sum(int(offs[r, cnt[r]]) for r in range(cnt.numel()))
            t0, t1 = a[:, s0][a[:, s0] > 0].min(), a[:, s1][a[:, s1] > 0].max()
            per_t[t].append(rows * C.d * bw / ((t1 - t0) * 1e-9) / 1e9)
    out = {"gbs_by_position": [float(np.median(v)) for v in per_t]}
    out["gbs_mean"] = float(np.mean(out["gbs_by_position"]))
    peak, _ = measured_peaks()
    out["frac_of_measured_peak"] = out["gbs_mean"] / peak
    out["frac_of_8TBps"] = out["gbs_mean"] / 8000.0
    out["how"] = ("in-kernel %globaltimer trace (~0.25 us resolution): shortlist bytes / (max over CTAs of "
                  "end-of-streaming - min over CTAs of start-of-streaming); every position run alone after an "
                  "L2 flush (cold HBM), median of 3")
    return out


def dense_baseline(D, clusters, inputs, B, C, dev, flush, reps=20):
    """Dense full-vocabulary head with the same epilogue: (a) our kernel with k = M (all clusters),
    (b) torch/cuBLAS matmul + logsumexp + topk.  Cold L2 before each rep."""
    M = clusters.M
    rows = 1 if C.shared else B        # tree mode: one (full) shortlist shared by the depth's rows
    sel = torch.arange(M, dtype=torch.int32, device=dev).repeat(rows, 1).contiguous()
    cnt = torch.full((rows,), M, dtype=torch.int32, device=dev)
    off = clusters.offsets.repeat(rows, 1).contiguous()
    ws = D.Workspace(D.lib().dynaspec_head_forward_ws(clusters.struct(), B, C.k_t), dev)
    hn = inputs[0][2][2]
    res = {}

    def ours():
        times = []
        for i in range(reps + 3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            D.head_forward(clusters, hn, sel, cnt, off, C.k_t, shared=C.shared, ws=ws)
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                times.append(a.elapsed_time(b))
        return 1e3 * statistics.median(times)

    res["ours_k_eq_M_us"] = ours()
    if C.shared:  # tree rows: the best of our two shared-shortlist heads is the dense comparator
        old = os.environ.get("DS_TH")
        os.environ["DS_TH"] = "0"
        try:
            res["ours_k_eq_M_tc_head_us"] = ours()
        finally:
            if old is None:
                del os.environ["DS_TH"]
            else:
                os.environ["DS_TH"] = old
        res["ours_k_eq_M_us"] = min(res["ours_k_eq_M_us"], res["ours_k_eq_M_tc_head_us"])
    Wp = clusters.W_perm
    times = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        z = torch.matmul(hn, Wp.t()).float()
        lse = torch.logsumexp(z, dim=-1)
        v, idx = torch.topk(z, C.k_t, dim=-1)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            times.append(a.elapsed_time(b))
    res["torch_cublas_us"] = 1e3 * statistics.median(times)
    res["best_us"] = min(res["ours_k_eq_M_us"], res["torch_cublas_us"])
    return res


def two_stream_run(D, clusters, router, inputs, C, B, args, dev, flush):
    """The paper's stream layout (router + select on S_m, joined before the head on S_d), one CUDA
    graph per cycle, same inputs and cold-L2 protocol: us per draft step (serialized, no core)."""
    st = [D.DraftStep(clusters, router, B, C.k_t, shared=C.shared, two_streams=True, device=dev)
          for _ in range(C.positions)]

    def cyc(i):
        for t in range(C.positions):
            st[t](*inputs[i][t], t, C.k_max, C.k_min)

    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cyc(0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cyc(0)
    times = []
    for i in range(args.steps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            times.append(a.elapsed_time(b))
    return {"us_per_draft_step": 1e3 * statistics.mean(times) / C.positions, "launches_per_step": st[0].launches}


def core_overlap_run(D, clusters, router, inputs, C, B, args, dev, flush, reps=10):
    """NEXT-2 / the paper's T_D model: T_D ~ T_embed + max{T_core, T_meta} + T_index+gemm.
    A same-bytes stand-in for the EAGLE drafter block (fc 2d -> 3.5d, ReLU, 3.5d -> d; bf16
    cuBLAS on S_d; it is the caller's work, not part of this library) runs each step; the
    router + TopK either wait for it (serialized, one stream) or run on S_m concurrently
    (dynaspec_step_route on S_m || core on S_d, join, dynaspec_step_head)."""
    import torch.nn.functional as F
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    f = int(3.5 * C.d)
    Wc1 = (torch.randn((f, 2 * C.d), generator=g, device=dev) * 0.01).to(torch.bfloat16)
    Wc2 = (torch.randn((C.d, f), generator=g, device=dev) * 0.01).to(torch.bfloat16)
    core_bytes = (Wc1.numel() + Wc2.numel()) * 2
    st_ser = [D.DraftStep(clusters, router, B, C.k_t, shared=C.shared, device=dev) for _ in range(C.positions)]
    st_ovl = [D.DraftStep(clusters, router, B, C.k_t, shared=C.shared, device=dev) for _ in range(C.positions)]
    hbuf = [torch.empty((B, C.d), dtype=torch.bfloat16, device=dev) for _ in range(C.positions)]
    s_meta = torch.cuda.Stream(device=dev)
    ev_f = [torch.cuda.Event() for _ in range(C.positions)]
    ev_j = [torch.cuda.Event() for _ in range(C.positions)]

    def core(t):
        hp, e, _ = inputs[0][t]
        hbuf[t].copy_(F.linear(F.relu(F.linear(torch.cat([hp, e], 1), Wc1)), Wc2))

    def serialized():
        for t in range(C.positions):
            hp, e, _ = inputs[0][t]
            core(t)
            st_ser[t](hp, e, hbuf[t], t, C.k_max, C.k_min)

    def overlapped():
        cur = torch.cuda.current_stream()
        for t in range(C.positions):
            hp, e, _ = inputs[0][t]
            ev_f[t].record(cur)
            s_meta.wait_event(ev_f[t])
            st_ovl[t].route(hp, e, t, C.k_max, C.k_min, s_meta)   # S_m
            core(t)                                               # S_d
            ev_j[t].record(s_meta)
            cur.wait_event(ev_j[t])                               # "sync S_m, S_d"
            st_ovl[t].head(hbuf[t], t, C.k_max, C.k_min, cur)

    def core_only():
        for t in range(C.positions):
            core(t)

    res = {}
    for name, fn in (("core_only", core_only), ("serialized", serialized), ("overlapped", overlapped)):
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph):
            fn()
        ts = []
        for i in range(reps + 2):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gph.replay()
            b.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        res[name + "_us_per_step"] = 1e3 * statistics.median(ts) / C.positions
    res["core_stand_in_bytes"] = int(core_bytes)
    res["router_hidden_us"] = res["serialized_us_per_step"] - res["overlapped_us_per_step"]
    res["head_after_core_us"] = res["overlapped_us_per_step"] - res["core_only_us_per_step"]
    res["how"] = ("one cycle per CUDA graph, cold L2 per cycle; core = bf16 fc 2d->3.5d, ReLU, 3.5d->d "
                  "(cuBLAS stand-in for the EAGLE block); serialized = core then the fused one-launch step; "
                  "overlapped = router on S_m || core on S_d, then the head")
    return res


def static_heads_run(D, clusters, inputs, C, B, dev, flush, reps=10):
    """NEXT-3: FR-Spec (fixed K = 32768, the paper's FR-Spec 32k) and PA-FR (K_fr(t), App. A.1)
    prefix heads on the same kernels, one cycle per CUDA graph, cold L2; synthetic Zipf counts for pi_f."""
    from synth import inputs as S_
    counts = S_.zipf_token_counts(C.V)
    pi = torch.as_tensor(np.lexsort((np.arange(C.V), -counts)), dtype=torch.int64)  # descending count, id asc
    Wv = torch.empty_like(clusters.W_perm)
    Wv[clusters.perm.long()] = clusters.W_perm
    fh = D.FrequencyHead(Wv, pi.to(dev))
    del Wv
    torch.cuda.empty_cache()
    K = min(32768, C.V)
    wss = [D.Workspace(1 << 20, dev) for _ in range(C.positions)]
    res = {}
    for name, kfn in (("fr_spec_32k", lambda t: K), ("pa_fr", lambda t: D.pa_fr_budget(t, K))):
        def cyc():
            for t in range(C.positions):
                fh.forward(inputs[0][t][2], kfn(t), C.k_t, ws=wss[t])
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            cyc()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cyc()
        ts = []
        for i in range(reps + 2):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        res[name + "_us_per_step"] = 1e3 * statistics.median(ts) / C.positions
        res[name + "_mean_K"] = float(np.mean([kfn(t) for t in range(C.positions)]))
    del fh
    torch.cuda.empty_cache()
    res["how"] = "frequency-permuted W copy, shortlist = prefix [0, K) as one contiguous run; same head kernels"
    return res


def verify_run(D, C, dev, flush, n_short, B=64, reps=10):
    """NEXT-4: lossless verification of B drafted chains of gamma = positions tokens against synthetic
    target logits [B][gamma+1][V] (bf16), drafter shortlists of n_short ids (the measured mean |V_S|)."""
    g_ = torch.Generator(device=dev)
    g_.manual_seed(5)
    gam, V = C.positions, C.V
    p = (torch.randn((B, gam + 1, V), generator=g_, device=dev) * 3).to(torch.bfloat16)
    noisy = p[:, :gam].float() + torch.randn((B, gam, V), generator=g_, device=dev) * 3
    ids = torch.topk(noisy, n_short, dim=-1).indices.to(torch.int32).contiguous()
    del noisy
    ql = (torch.gather(p[:, :gam].float(), 2, ids.long()) +
          torch.randn((B, gam, n_short), generator=g_, device=dev) * 0.5).contiguous()
    q_lse = torch.logsumexp(ql, dim=-1).contiguous()
    slot = torch.multinomial(torch.softmax(ql.reshape(-1, n_short), -1), 1, generator=g_).reshape(B, gam)
    x = torch.gather(ids, 2, slot.unsqueeze(-1)).squeeze(-1).contiguous()
    slot = slot.to(torch.int32).contiguous()
    cnt = torch.full((B, gam), n_short, dtype=torch.int32, device=dev)
    u_acc = torch.rand((B, gam), generator=g_, device=dev)
    u_res = torch.rand(B, generator=g_, device=dev)
    ver = D.Verifier(V, B, gam, dev)
    call = lambda: ver(p, ids, ql, cnt, q_lse, x, slot, u_acc, u_res)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    us = 1e3 * statistics.median(ts)
    target_bytes = B * (gam + 1) * V * 2
    resid_bytes = B * V * (2 + 4) + 2 * B * n_short * 8
    peak, _ = measured_peaks()
    acc = ver.accepted.float().mean().item()
    out = {"chains": B, "gamma": gam, "V": V, "n_short": n_short, "us_per_call": us,
           "chains_per_s": B / (us / 1e6), "mean_accepted": acc,
           "target_logit_bytes": target_bytes, "residual_pass_bytes": resid_bytes,
           "achieved_GBps": (target_bytes + resid_bytes) / (us / 1e6) / 1e9}
    out["frac"] = out["achieved_GBps"] / peak
    del p, ids, ql, ver
    torch.cuda.empty_cache()
    return out


def e2e_run(D, steppers, clusters, router, C, B, args, dev, flush, ws, rows_all_ranks, reps=None):
    """End to end through the public API: every step copies its inputs from pinned host memory
    (H2D: one copy of all positions' [h_prev, e, h_new] rows), runs the draft cycle, and reads the
    step's results (top ids + log-probs of every position) back (D2H: one copy)."""
    reps = reps or args.steps
    bw = 2 if args.dtype == "bf16" else 4
    tdt = S.TORCH_DTYPES[args.dtype]
    P = C.positions
    host_in = []
    for i in range(2):  # two input sets, alternated: nothing is reused from the previous replay
        h = torch.empty((P, 3, B, C.d), dtype=tdt).pin_memory()
        for t in range(P):
            for j, x in enumerate(S.step_inputs(B, C.d, P * (100 + i) + t, args.dtype, pool=1 << 20,
                                                sibling_eps=0.1 if C.shared else None)):  # the timed workload's rows
                h[t, j].copy_(x)
        host_in.append(h)
    dev_in = torch.empty((P, 3, B, C.d), dtype=tdt, device=dev)
    dev_out = torch.empty((P, 2, B, C.k_t), dtype=torch.int32, device=dev)  # [t][ids | logp bits]
    host_out = torch.empty((P, 2, B, C.k_t), dtype=torch.int32).pin_memory()
    saved = [(st.top_ids, st.top_logp) for st in steppers]
    for t, st in enumerate(steppers):
        st.bind_outputs(top_ids=dev_out[t, 0], top_logp=dev_out[t, 1].view(torch.float32))

    def e2e_body(i, cs, overlap):
        if overlap == "one":  # one copy of the cycle's inputs, then the PDL-chained steps
            dev_in.copy_(host_in[i], non_blocking=True)
            for t in range(P):
                steppers[t](dev_in[t, 0], dev_in[t, 1], dev_in[t, 2], t, C.k_max, C.k_min)
        elif overlap == "split":  # position 0's inputs first; the rest on a copy stream behind step 0
            cur = torch.cuda.current_stream()
            dev_in[0].copy_(host_in[i][0], non_blocking=True)
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                dev_in[1:].copy_(host_in[i][1:], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            for t in range(P):
                if t == 1:
                    cur.wait_event(ev)
                steppers[t](dev_in[t, 0], dev_in[t, 1], dev_in[t, 2], t, C.k_max, C.k_min)
            cur.wait_stream(cs)
        else:  # each position's inputs on a copy stream, position t + 1's copy overlapping step t
            cur = torch.cuda.current_stream()
            cs.wait_stream(cur)
            evs = []
            with torch.cuda.stream(cs):
                for t in range(P):
                    dev_in[t].copy_(host_in[i][t], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    evs.append(ev)
            for t in range(P):
                cur.wait_event(evs[t])
                steppers[t](dev_in[t, 0], dev_in[t, 1], dev_in[t, 2], t, C.k_max, C.k_min)
            cur.wait_stream(cs)
        host_out.copy_(dev_out, non_blocking=True)

    # both copy schedules are timed; the faster is reported (large inputs gain from overlapping the
    # copies, small ones lose the PDL chain to the event waits)
    best = None
    for overlap in ("one", "split", "per_position") if P > 1 else ("one",):
        graphs = []
        for i in range(2):
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                dev_in.copy_(host_in[i], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            cs = torch.cuda.Stream(device=dev)
            with torch.cuda.graph(g):
                e2e_body(i, cs, overlap)
            graphs.append(g)
        for i in range(4):
            graphs[i % 2].replay()
        torch.cuda.synchronize()
        tot = 0.0
        dev_ms = []
        for i in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            ea.record()
            graphs[i % 2].replay()
            eb.record()
            torch.cuda.synchronize()   # the host has the step's results
            tot += time.perf_counter() - t0
            dev_ms.append(ea.elapsed_time(eb))
        tot = max_over_ranks(tot, ws)
        if best is None or tot < best[0]:
            best = (tot, overlap, statistics.median(dev_ms))
    tot, overlap, dev_med = best
    for st, (ids, lp) in zip(steppers, saved):
        st.bind_outputs(top_ids=ids, top_logp=lp)
    h2d = P * 3 * B * C.d * bw
    d2h = P * B * C.k_t * 8
    return {"value": rows_all_ranks * P * reps / tot, "unit": "draft tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "timing": "host wall clock around graph replay + synchronize "
            + {"per_position": "(per position one H2D copy of its inputs on a copy stream, position t + 1's copy "
                               "overlapping step t; the cycle's steps; one D2H copy of the results)",
               "split": "(position 0's inputs copied first, positions 1.. on a copy stream behind step 0; the "
                        "cycle's PDL-chained steps; one D2H copy of the results)",
               "one": "(one H2D copy of the cycle's inputs, the cycle's PDL-chained steps, one D2H copy of the "
                      "results)"}[overlap]
            + "; the fastest of the three copy schedules",
            "ms_per_step": 1e3 * tot / reps, "device_ms_per_step": dev_med}


def run_cluster_sharded(args, ws, rank, local):
    """--shard clusters (SURVEY 8(e) option 2): every rank stores only the W_perm rows of a
    token-balanced contiguous cluster range; router + TopK run replicated (bit-identical on every
    rank); each rank streams its owned selected clusters and emits one (max, sum, top-k_t) record
    per row; ONE all-gather (NCCL over NVLink / NVSwitch) exchanges the records; the rank-order merge
    (dynaspec_merge_records) gives every rank the same outputs.  All ranks process the SAME rows,
    so total work is fixed as N grows (strong scaling)."""
    from paper_2510_13847_b200 import dynaspec as D
    from paper_2510_13847_b200.parallel import ClusterShardedStep, cluster_ranges
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    C = S.CONFIGS[args.config]
    B = args.batch or C.B
    W = S.lm_head(C.V, C.d, 0, args.dtype, device=dev)
    rt = [None if x is None else x.to(dev) for x in S.router(C.d, C.h_r, C.M, 1, args.dtype)]
    full = D.Clusters.build(W, C.M, seed=2, max_iters=args.kmeans_iters)
    del W
    lo, hi = cluster_ranges(full.offsets.cpu().tolist(), ws)[rank]
    shard = full.shard(lo, hi)
    full.W_perm = None
    del full
    torch.cuda.empty_cache()
    router = D.Router(*rt)
    group = dist.group.WORLD if ws > 1 else None
    steps = [ClusterShardedStep(D, shard, router, B, C.k_t, ws, rank, group=group, shared=C.shared)
             for _ in range(C.positions)]
    pool = 4
    inputs = [[tuple(x.to(dev) for x in S.step_inputs(B, C.d, C.positions * i + t, args.dtype, pool=1 << 20,
                                                      sibling_eps=0.1 if C.shared else None, base_seed=1000))
               for t in range(C.positions)] for i in range(pool)]
    flush = L2Flush(dev)

    def cycle(i):
        for t in range(C.positions):
            steps[t](*inputs[i % pool][t], t, C.k_max, C.k_min)

    for i in range(args.warmup):
        flush.zero_()
        cycle(i)
    torch.cuda.synchronize()
    barrier(ws)
    clk = ClockSampler(local)
    clk.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        cycle(args.warmup + i)
        ev[i][1].record()
    torch.cuda.synchronize()
    barrier(ws)
    clocks = clk.stop()
    tot = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), ws)
    rows_all = B * C.positions * args.steps
    if rank == 0:
        print(json.dumps({
            "metric": "draft-head tokens/s & us/step (V=128k,d=4096); % HBM peak; speedup vs dense",
            "value": rows_all / (tot / 1e3), "unit": "draft tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded random-init weights, router and hidden states)",
            "config": {"workload": C.name, "V": C.V, "d": C.d, "M": C.M, "h_r": C.h_r, "global_batch": B,
                       "positions": C.positions, "k_t": C.k_t, "shared": C.shared,
                       "parallelism": f"cluster-sharded x{ws}: rank 0 owns clusters [{lo}, {hi}) "
                                      f"({shard.W_perm.shape[0]} of {C.V} W_perm rows); one all-gather of "
                                      f"B x (2 + 2 k_t) floats per step",
                       "l2": L2_HOW, "cuda_graph": False,
                       "us_per_draft_step": 1e3 * tot / args.steps / C.positions},
            "roofline": None, "cpu_baseline": None, "e2e": None,
            "gpu_launches": None, "clocks": clocks}))


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif args.shard == "clusters":
        run_cluster_sharded(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
