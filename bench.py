"""bench.py -- all-sources BFS closeness on a synthetic HoMLN, one B200 per rank.

A "step" is one pass of the whole hot path over one HoMLN:
closeness on every layer, then for every layer subset T: AND aggregation,
closeness of the AND graph, ground-truth top-K, CC2, CC1 and naive
composition (top-K lists).  Inputs are resident in HBM when the timed region
starts; L2 is flushed (256 MiB write) before every timed step.

Metric (BASELINE.json): TEPS = W / time with W = sum over every graph whose
closeness is computed of sum_components k_c * m_c (Graph500-style undirected
edges; isolated vertices add 0), plus seconds per HoMLN.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]
Multi-GPU (torchrun): replicas only -- each rank runs its own HoMLN (the
north star fixes one GPU; no collective is invented), "scaling": "weak".
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import build_config  # noqa: E402

L2_FLUSH_BYTES = 256 << 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: an NVML polling
    thread (1 ms period, so even a few-ms region has samples); nvidia-smi -lms 100 if NVML is missing."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.mx = None
        self._stop = threading.Event()
        self.t = None
        self.nv = None
        self.proc = None

    def _handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            self.nv, h = self._handle()
            self.mx = float(self.nv.nvmlDeviceGetMaxClockInfo(h, self.nv.NVML_CLOCK_SM))

            def poll():
                while True:
                    self.samples.append(float(self.nv.nvmlDeviceGetClockInfo(h, self.nv.NVML_CLOCK_SM)))
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, bit in self.REASONS:
                        if r & bit:
                            self.reasons.add(name)
                    if self._stop.wait(0.001):
                        break
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                      "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                      "clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.lines = []
            self.t = threading.Thread(target=lambda: [self.lines.append(ln.strip()) for ln in self.proc.stdout],
                                      daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def stop(self):
        if self.nv is not None:
            self._stop.set()
            self.t.join(timeout=5)
            src = "nvml (1 ms polling)"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            for ln in self.lines:
                p = [x.strip() for x in ln.split(",")]
                try:
                    self.samples.append(float(p[0]))
                    self.mx = float(p[1])
                except (ValueError, IndexError):
                    continue
                for (name, _), v in zip(self.REASONS, p[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(name)
            src = "nvidia-smi -lms 100"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no NVML / nvidia-smi"], "samples": 0}
        sm = self.samples
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": src}


# ---------------------------------------------------------------------------
# cross-rank aggregation (replicas: every rank runs its own HoMLN)
# ---------------------------------------------------------------------------
def job_value(units_local, ms_local, device="cpu"):
    """Whole-job throughput: units summed over ranks / max-over-ranks time.
    Returns (value, max_ms).  Single process: units / ms."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return units_local / (ms_local / 1e3), ms_local
    u = torch.tensor([float(units_local)], dtype=torch.float64, device=device)
    t = torch.tensor([float(ms_local)], dtype=torch.float64, device=device)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(u.item()) / (float(t.item()) / 1e3), float(t.item())


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2207_11662_b200 import Context
    from paper_2207_11662_b200 import build as B

    if rank == 0:
        B.build()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    dev = 0 if args.same_device else local_rank
    torch.cuda.set_device(dev)
    h = build_config(args.config, V=args.V)
    V, K = h.V, h.K
    ctx = Context(dev)
    s = ctx.stream
    ctx.set_param("bfs_words", args.words)
    ctx.set_param("bfs_hints", args.hints)
    ctx.set_param("timing", 1)
    if args.fused or args.separate:
        ctx.set_param("bfs_fuse", 1 if args.fused else 0)
    for kv in args.set:                      # extra library parameters (A/B experiments)
        k, v = kv.split("=")
        ctx.set_param(k, int(v))
    host_layers = [torch.from_numpy(L).pin_memory() for L in h.layers]
    dev_layers = [t.to(f"cuda:{dev}") for t in host_layers]
    torch.cuda.synchronize()
    ids_dev = torch.zeros(max(K, 1), dtype=torch.int32, device=f"cuda:{dev}")
    cnt_dev = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")   # |R| stays on the device (no sync)

    def cc1_name(T):   # CC1 is the paper's pair heuristic; r > 2 is the opt-in flat r-ary reading Z12
        return "cc1" if len(T) == 2 else "cc1_rary"
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=f"cuda:{dev}")

    # ---- units W per graph (traversal units for TEPS), from one untimed pass
    ctx.load_layers(V, dev_layers)
    units = []
    graph_names = []
    arcs_and = []
    for i in range(len(h.layers)):
        r = ctx.closeness(i, want=("k",))
        d = ctx.degrees(i)
        units.append(int((r["k"].astype(np.int64) * d.astype(np.int64)).sum() // 2))
        graph_names.append(f"L{i}")
    for T in h.subsets:
        g = ctx.and_aggregate(list(T))
        r = ctx.closeness(g, want=("k",))
        d = ctx.degrees(g)
        units.append(int((r["k"].astype(np.int64) * d.astype(np.int64)).sum() // 2))
        graph_names.append("AND" + "".join(map(str, T)))
        arcs_and.append(2 * ctx.graph_info(g)[1])
        ctx.free_graph(g)
    W_total = sum(units)
    arcs = [2 * ctx.graph_info(i)[1] for i in range(len(h.layers))] + arcs_and

    # --shard (SURVEY §8(f) rank 4, strong scaling of ONE HoMLN): rank r runs the source
    # batches r, r + N, ... of every graph, one NCCL all-reduce sums the partial distance
    # sums of all graphs of the step, then every rank finalises and composes.
    n_graphs = len(h.layers) + len(h.subsets)
    S_all = torch.zeros(n_graphs * V, dtype=torch.int64, device=f"cuda:{dev}") if args.shard else None

    def psi(gids):
        """closeness of the graphs gids (plain, fused or sharded)"""
        if args.shard:
            for k, g in enumerate(gids):
                ctx.closeness_partial(g, rank, world, out=S_all[k * V:(k + 1) * V])
            if world > 1:
                import torch.distributed as dist
                with torch.cuda.stream(s):
                    dist.all_reduce(S_all[:len(gids) * V], op=dist.ReduceOp.SUM)
            for k, g in enumerate(gids):
                ctx.closeness_combine(g, S_all[k * V:(k + 1) * V])
        else:
            # every graph of the step in one call: the library fuses them into one MS-BFS pass when
            # they are too small to fill the GPU alone (bfs_fuse 2; --fused forces 1, --separate 0)
            ctx.closeness_multi(list(gids))

    def hot_step():
        ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
        psi(list(range(len(h.layers))) + ands)
        for T, g in zip(h.subsets, ands):
            ctx.topk_closeness(g, K, out=ids_dev)
            ctx.compose("cc2", list(T), K, out=ids_dev, count_out=cnt_dev)
            ctx.compose(cc1_name(T), list(T), K, out=ids_dev, count_out=cnt_dev)
            ctx.compose("naive", list(T), K, out=ids_dev, count_out=cnt_dev)
            ctx.free_graph(g)

    def flush_l2():
        with torch.cuda.stream(s):
            flush.fill_(1)

    # ---- warmup
    for _ in range(args.warmup):
        hot_step()
    ctx.sync()
    ctx.stats(reset=True)

    # ---- CUDA graph of the step (when no library call in it makes a host round trip: the probe step
    # counts them).  Replaying the graph launches exactly the kernels of one eager step.
    run_step = hot_step
    graph_info = {"captured": False}
    hot_step()
    ctx.sync()
    probe = ctx.stats(reset=True)
    launches_per_step = probe["launches"]
    n_graphs_step = len(h.layers) + len(h.subsets)
    fused_step = probe["bfs_launches"] < n_graphs_step          # the library fused the step's graphs
    graph_info["host_syncs_per_step"] = probe["host_syncs"]
    if args.graph and not args.shard and probe["host_syncs"] == 0:
        try:
            ctx.set_param("timing", 0)
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=s):
                hot_step()
            torch.cuda.synchronize()
            cap = ctx.stats(reset=True)
            launches_per_step = cap["launches"]

            def run_step():
                with torch.cuda.stream(s):
                    cg.replay()
            run_step()
            torch.cuda.synchronize()
            graph_info = {"captured": True, "host_syncs_per_step": 0, "launches_captured": cap["launches"]}
        except Exception as ex:       # keep the eager step
            log(f"CUDA graph capture failed ({ex}); timing the eager step")
            torch.cuda.synchronize()
            run_step = hot_step
            graph_info["capture_error"] = str(ex)[:200]
        finally:
            ctx.set_param("timing", 1)
    ctx.stats(reset=True)

    # ---- timed (device-resident inputs)
    clk = ClockSampler(dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    times = []
    for _ in range(args.steps):
        flush_l2()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        run_step()
        e1.record(s)
        times.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = [a.elapsed_time(b) for a, b in times]
    st = ctx.stats(reset=True)
    total_ms = float(sum(ms))
    share = W_total / world if args.shard else W_total       # units this rank processed per step
    value, total_ms = job_value(share * args.steps, total_ms, device=f"cuda:{dev}")
    ms_per_step = total_ms / args.steps

    # ---- per-phase breakdown of one extra (untimed-for-value) step, CUDA events on the ctx stream:
    # SURVEY §8(d) / PAPER.md:373 accounting: Psi per layer, AND, ground-truth closeness, Theta (CC1, CC2)
    breakdown = None
    accuracy = None
    if not args.shard:
        ev = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ev.append((name, e))

        flush_l2()
        torch.cuda.synchronize()
        mark("start")
        for i in range(len(h.layers)):
            ctx.closeness(i, out={})
            mark(f"psi_L{i}")
        for T in h.subsets:
            tag = "".join(map(str, T))
            g = ctx.and_aggregate(list(T))
            mark(f"and_{tag}")
            ctx.closeness(g, out={})
            mark(f"gt_closeness_{tag}")
            ctx.topk_closeness(g, K, out=ids_dev)
            mark(f"gt_topk_{tag}")
            ctx.compose("cc2", list(T), K, out=ids_dev, count_out=cnt_dev)
            mark(f"theta_cc2_{tag}")
            ctx.compose(cc1_name(T), list(T), K, out=ids_dev, count_out=cnt_dev)
            mark(f"theta_cc1_{tag}")
            ctx.compose("naive", list(T), K, out=ids_dev, count_out=cnt_dev)
            mark(f"theta_naive_{tag}")
            if T == h.subsets[0]:
                # the paper's evaluation (Table 2): each heuristic's top-K against the
                # ground-truth top-K, on the library's set-metrics kernel (after the timed marks)
                gt_ids = ctx.topk_closeness(g, K)
                accuracy = {}
                for heur in (cc1_name(T), "cc2", "naive"):
                    est, _ = ctx.compose(heur, list(T), K)
                    m = ctx.set_metrics(V, est, gt_ids)
                    accuracy[heur.replace("_rary", "")] = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in m.items()}
            ctx.free_graph(g)
        torch.cuda.synchronize()
        breakdown = {n: ev[i - 1][1].elapsed_time(e) for i, (n, e) in enumerate(ev) if i > 0}
        psi_ms = [breakdown[f"psi_L{i}"] for i in range(len(h.layers))]
        T0 = "".join(map(str, h.subsets[0]))
        breakdown["sum_psi"] = float(sum(psi_ms))
        breakdown["max_psi"] = float(max(psi_ms))
        # the paper's accounting: t_dt = max(Psi) + Theta, t_gt = AND + CC (first subset)
        breakdown["t_dt_cc1"] = breakdown["max_psi"] + breakdown[f"theta_cc1_{T0}"]
        breakdown["t_dt_cc2"] = breakdown["max_psi"] + breakdown[f"theta_cc2_{T0}"]
        breakdown["t_gt"] = breakdown[f"and_{T0}"] + breakdown[f"gt_closeness_{T0}"] + breakdown[f"gt_topk_{T0}"]
        breakdown = {k: round(v, 4) for k, v in breakdown.items()}
        ctx.stats(reset=True)

    # ---- e2e: host edge lists -> public API -> host results, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        h2d = sum(int(t.numel()) * 4 for t in host_layers)
        d2h = 0
        e_ms = []
        n_warm = 2                                          # untimed e2e passes (first-use allocations, pool growth)
        nsub = len(h.subsets)
        e2e_lists = torch.empty((4 * nsub, K), dtype=torch.int32, device=f"cuda:{dev}")
        e2e_counts = torch.empty(3 * nsub, dtype=torch.int32, device=f"cuda:{dev}")
        e2e_lists_h = torch.empty((4 * nsub, K), dtype=torch.int32).pin_memory()
        e2e_counts_h = torch.empty(3 * nsub, dtype=torch.int32).pin_memory()
        import gc
        gc.disable()                                        # no collector pause inside a timed e2e step
        for it in range(n_warm + max(1, args.steps)):
            flush_l2()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.load_layers(V, host_layers)                 # H2D from pinned host memory
            ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
            psi(list(range(len(h.layers))) + ands)
            for j, (T, g) in enumerate(zip(h.subsets, ands)):
                # every ranked list (and the CC1 / naive set sizes) into device memory, stream-ordered
                ctx.topk_closeness(g, K, out=e2e_lists[4 * j])
                ctx.compose("cc2", list(T), K, out=e2e_lists[4 * j + 1], count_out=e2e_counts[3 * j:3 * j + 1])
                ctx.compose(cc1_name(T), list(T), K, out=e2e_lists[4 * j + 2], count_out=e2e_counts[3 * j + 1:3 * j + 2])
                ctx.compose("naive", list(T), K, out=e2e_lists[4 * j + 3], count_out=e2e_counts[3 * j + 2:3 * j + 3])
                ctx.free_graph(g)
            with torch.cuda.stream(s):                      # one D2H of all results into pinned memory
                e2e_lists_h.copy_(e2e_lists, non_blocking=True)
                e2e_counts_h.copy_(e2e_counts, non_blocking=True)
            e1.record(s)
            e1.synchronize()
            if it >= n_warm:
                e_ms.append(e0.elapsed_time(e1))
            d2h = int(e2e_lists_h.nbytes + e2e_counts_h.nbytes)
        gc.enable()
        # the median step: one host hiccup (a 50 ms stall of the Python host thread was seen in 1 of 5
        # steps) should not decide the number; the mean and every step are reported beside it
        e2e_ms = float(np.median(e_ms))
        e2e_val, e2e_ms = job_value(share, e2e_ms, device=f"cuda:{dev}")
        e2e = {"value": e2e_val, "unit": "TEPS", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "statistic": "median over steps",
               "ms_per_step_mean": float(np.mean(e_ms)), "steps_ms": [round(x, 3) for x in e_ms]}

    # ---- roofline of the MS-BFS kernel: per graph (one untimed pass, one MS-BFS launch per graph,
    # library counters of that launch) and the headline over the dominant launches (the layers)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak_gbs = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    traffic, traffic_src = measured_traffic(args)
    # L2 row-traffic ceiling of this access pattern, measured by tools/cutest/level_floor.cu
    l2_peak, l2_src = None, None
    try:
        lf = json.load(open(os.path.join(ROOT, "profiles", "r2_level_floor.json")))
        l2_peak, l2_src = float(lf["row_traffic_gbps"]), "profiles/r2_level_floor.json (tools/cutest/level_floor.cu)"
    except Exception:
        pass
    per_graph = {}
    if not args.shard:
        ctx.sync()
        ctx.stats(reset=True)
        gl = [(f"L{i}", i) for i in range(len(h.layers))]
        ands = []
        for T in h.subsets:
            g = ctx.and_aggregate(list(T))
            ands.append(g)
            gl.append(("AND" + "".join(map(str, T)), g))
        for name, g in gl:
            # the row traffic of this launch (counting instantiation, untimed), then the timed launch
            ctx.set_param("bfs_count_rows", 1)
            ctx.closeness(g, out={})
            ctx.sync()
            sc = ctx.stats(reset=True)
            ctx.set_param("bfs_count_rows", 0)
            flush_l2()
            ctx.closeness(g, out={})
            ctx.sync()
            sg = ctx.stats(reset=True)
            t = sg["bfs_ms"] / 1e3
            model = sg["bfs_model_bytes"]
            comp = sg["bfs_state_bytes"] + sg["bfs_csr_bytes"]
            e = {"ms": sg["bfs_ms"], "levels": sg["bfs_levels"], "batches": sg["bfs_batches"],
                 "model_bytes": model, "compulsory_bytes": comp, "row_commits": sg["bfs_row_commits"],
                 "model_frac": model / t / 1e9 / peak_gbs if t > 0 else None,
                 "compulsory_frac": comp / t / 1e9 / peak_gbs if t > 0 else None,
                 "gathers": sc["bfs_gathers"], "own_reads": sc["bfs_own_reads"]}
            rsz = sc["bfs_state_bytes"] / (2 * sc["bfs_row_commits"]) if sc["bfs_row_commits"] else 0.0   # 8 W
            row_bytes = rsz * (sc["bfs_gathers"] + sc["bfs_own_reads"] + sc["bfs_row_commits"])
            e["row_traffic_bytes"] = row_bytes
            e["row_traffic_frac_l2"] = row_bytes / t / 1e9 / l2_peak if (t > 0 and l2_peak) else None
            nd = (traffic or {}).get("per_graph", {}).get(name)
            if nd:
                e["ncu_dram_bytes"] = nd["dram_bytes"]
                e["ncu_ms"] = nd["duration_s"] * 1e3
                e["ncu_dram_frac"] = nd["dram_bytes"] / nd["duration_s"] / 1e9 / peak_gbs
                e["ncu_l2_hit_pct"] = nd.get("l2_hit_pct")
            per_graph[name] = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in e.items()}
        for g in ands:
            ctx.free_graph(g)
    # ---- the step's own MS-BFS launches (the library fuses graphs, bfs_fuse): measured per part of the
    # step's Psi -- everything when the whole step is one launch (C1, C2), else the layers' Psi (one fused
    # launch on C5) and the AND graphs' Psi -- one counting run (row traffic), one timed run
    step_parts = {}

    def measure_part(name, gids_of):
        ctx.sync()
        ctx.stats(reset=True)
        ands_ = [ctx.and_aggregate(list(T)) for T in h.subsets]
        ids_ = gids_of(ands_)
        ctx.set_param("bfs_count_rows", 1)
        psi(ids_)
        ctx.sync()
        sc = ctx.stats(reset=True)
        ctx.set_param("bfs_count_rows", 0)
        flush_l2()
        psi(ids_)
        ctx.sync()
        sg = ctx.stats(reset=True)
        for g in ands_:
            ctx.free_graph(g)
        t = sg["bfs_ms"] / 1e3
        model = sg["bfs_model_bytes"]
        comp = sg["bfs_state_bytes"] + sg["bfs_csr_bytes"]
        rsz = sc["bfs_state_bytes"] / (2 * sc["bfs_row_commits"]) if sc["bfs_row_commits"] else 0.0
        rowb = rsz * (sc["bfs_gathers"] + sc["bfs_own_reads"] + sc["bfs_row_commits"])
        step_parts[name] = {
            "graphs": len(ids_), "launches": sg["bfs_launches"], "ms": round(sg["bfs_ms"], 4),
            "levels": sg["bfs_levels"], "batches": sg["bfs_batches"], "model_bytes": model,
            "compulsory_bytes": comp, "row_commits": sg["bfs_row_commits"],
            "gathers": sc["bfs_gathers"], "own_reads": sc["bfs_own_reads"], "row_traffic_bytes": rowb,
            "model_frac": round(model / t / 1e9 / peak_gbs, 4) if t > 0 else None,
            "compulsory_frac": round(comp / t / 1e9 / peak_gbs, 4) if t > 0 else None,
            "row_traffic_frac_l2": round(rowb / t / 1e9 / l2_peak, 4) if (t > 0 and l2_peak) else None}

    nl = len(h.layers)
    if fused_step and not args.shard:
        if probe["bfs_launches"] == 1:
            measure_part("step", lambda ands_: list(range(nl)) + ands_)
        else:
            measure_part("layers", lambda ands_: list(range(nl)))
            measure_part("ands", lambda ands_: ands_)
    step_fused = step_parts.get("step") or step_parts.get("layers")
    if step_parts:                          # the step's own launches
        n_bfs = sum(v["launches"] for v in step_parts.values())
        bfs_ms_step = sum(v["ms"] for v in step_parts.values())
        bfs_ms_avg = bfs_ms_step / max(1, n_bfs)
        levels_per_launch = sum(v["levels"] for v in step_parts.values()) / max(1, n_bfs)
    elif per_graph:                         # per-launch numbers from the eager per-graph pass
        n_bfs = len(per_graph)
        bfs_ms_avg = float(np.mean([v["ms"] for v in per_graph.values()]))
        levels_per_launch = float(np.mean([v["levels"] for v in per_graph.values()]))
        bfs_ms_step = float(sum(v["ms"] for v in per_graph.values()))
    else:
        n_bfs = max(1, st["bfs_launches"])
        bfs_ms_avg = st["bfs_ms"] / n_bfs
        levels_per_launch = st["bfs_levels"] / n_bfs
        bfs_ms_step = st["bfs_ms"] / args.steps
    # headline: the dominant kernel -- the layers' MS-BFS (3 of the 4 graphs of a C5 step, one fused launch,
    # ~80 % of the step; the whole step's launch on C1 / C2); algorithmic bytes = SURVEY §8(d) dense-level
    # model of this algorithm, accumulated by the kernel per batch:  L * (4 (rows + 1) + 4 arcs + 2 R rows),
    # R = 8 W bytes
    layer_e = [v for k, v in per_graph.items() if k.startswith("L")]
    dom_rowb = None
    if step_fused:
        dom_ms = step_fused["ms"] / max(1, step_fused["launches"])
        dom_bytes = step_fused["model_bytes"] / max(1, step_fused["launches"])
        dom_rowb = step_fused["row_traffic_bytes"] / max(1, step_fused["launches"])
        # ncu DRAM bytes of the step's layers launch (a steady-state capture, when it matches this build)
        sl = (traffic or {}).get("step_launches", {}).get("layers")
        dom_traffic = sl["dram_bytes"] if (sl and "layers" in step_parts and step_parts["layers"]["launches"] == 1) else None
        dom_name = ("msbfs_kernel, the step's one launch over all its graphs (bfs_fuse)" if "step" in step_parts
                    else "msbfs_kernel, the layers' launch(es) of the step (graphs fused by bfs_fuse), per launch")
    elif layer_e:
        dom_ms = float(np.mean([v["ms"] for v in layer_e]))
        dom_bytes = float(np.mean([v["model_bytes"] for v in layer_e]))
        dom_rowb = float(np.mean([v["row_traffic_bytes"] for v in layer_e]))
        dom_traffic = (float(np.mean([v["ncu_dram_bytes"] for v in layer_e]))
                       if all("ncu_dram_bytes" in v for v in layer_e) else None)
        dom_name = "msbfs_kernel (plain instantiation), the layer launches"
    else:                                   # --shard: all launches together
        dom_ms = bfs_ms_avg
        dom_bytes = st["bfs_model_bytes"] / n_bfs
        dom_traffic = None
        dom_name = "msbfs_kernel (all launches)"
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    # the bound the dense levels actually meet: row traffic through L2 (gathered rows, own rows read, rows
    # written; counted by the kernel) against the same pattern's measured ceiling (no BFS logic)
    l2_roof = None
    if dom_rowb and l2_peak and dom_ms > 0:
        rb = dom_rowb
        l2a = rb / (dom_ms / 1e3) / 1e9
        l2_roof = {"bound": "l2", "achieved": l2a, "peak": l2_peak, "unit": "GB/s", "frac": l2a / l2_peak,
                   "bytes_per_launch": rb, "peak_source": l2_src,
                   "bytes": "8W x (rows gathered + own rows read + rows written), counted by the kernel"}
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
            "frac": achieved / peak_gbs, "traffic": dom_traffic,
            "traffic_source": traffic_src, "peak_source": peak_src, "kernel": dom_name,
            "bytes_model": "SURVEY 8(d) dense-level model of the visited-set MS-BFS, per batch: "
                           "L*(4(rows+1)+4*arcs+2*R*rows), R=8W bytes (own row read + row write), summed by the kernel",
            "bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms,
            "per_graph": per_graph,
            "per_graph_note": "model = dense-level bytes; compulsory = 2 R x rows actually changed + CSR per level; "
                              "ncu_dram = dram__bytes_read+write of the same launch (ncu, serialised, cold cache)",
            "l2_row_traffic": l2_roof,
            "levels_per_launch": levels_per_launch, "bfs_ms_per_launch_all": bfs_ms_avg,
            "bfs_share_of_step": bfs_ms_step / max(ms_per_step, 1e-9),
            "fused_graphs": n_graphs_step if (fused_step and probe["bfs_launches"] == 1) else 1,
            "bfs_launches_per_step": probe["bfs_launches"], "graphs_per_step": n_graphs_step,
            "step_launches": step_parts}

    line = {
        "metric": "all-sources BFS closeness TEPS (HoMLN) on 1 B200; also s/HoMLN and % HBM roofline",
        "value": value, "unit": "TEPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if args.shard else "weak",
        "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": h.name, "V": V, "layers": len(h.layers), "subsets": [list(t) for t in h.subsets],
                   "K": K, "recipe": h.recipe, "units_W": W_total, "units_per_graph": dict(zip(graph_names, units)),
                   "bfs_words": args.words, "bfs_hints": args.hints, "sources_per_batch": 64 * args.words,
                   "l2": "flushed (256 MiB write) before each timed step",
                   "parallelism": f"batch-shard{world}+nccl-allreduce(S)" if args.shard else f"replicas{world}"},
        "s_per_homln": ms_per_step / 1e3,
        "e2e": e2e, "roofline": roof, "clocks": clocks, "gpu_launches": int(round(launches_per_step)),
        "cuda_graph": graph_info,
        "breakdown_ms": breakdown,
        "accuracy_vs_gt_topk": accuracy,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:      # the oracle baseline: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(h, args.cpu_seconds)
    if args.dump:
        # one more step through the same psi() (plain, fused or sharded + all-reduce), then every
        # graph's results and every ranked list, for the parity tests
        ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
        gids = list(range(len(h.layers))) + ands
        psi(gids)
        dump = {}
        for g, name in zip(gids, [f"L{i}" for i in range(len(h.layers))] + ["AND" + "".join(map(str, T)) for T in h.subsets]):
            for key, arr in ctx.closeness_results(g).items():
                dump[f"{name}_{key}"] = arr
        for T, g in zip(h.subsets, ands):
            tag = "".join(map(str, T))
            dump[f"gt_{tag}"] = ctx.topk_closeness(g, K)
            dump[f"cc2_{tag}"] = ctx.compose("cc2", list(T), K)[0]
            dump[f"cc1_{tag}"] = ctx.compose(cc1_name(T), list(T), K)[0]
            dump[f"naive_{tag}"] = ctx.compose("naive", list(T), K)[0]
            ctx.free_graph(g)
        if rank == 0:
            np.savez(args.dump, **dump)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


# ---------------------------------------------------------------------------
# oracle timing (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------
def _component_edges(V, E):
    """per-vertex m_c (edges of its component) -- bookkeeping for the TEPS numerator."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    E = np.asarray(E, dtype=np.int64).reshape(-1, 2)
    A = sp.coo_matrix((np.ones(len(E)), (E[:, 0], E[:, 1])), shape=(V, V))
    nc, lab = connected_components(A, directed=False)
    m_c = np.bincount(lab[E[:, 0]], minlength=nc)
    return m_c[lab]


def oracle_sample(V, E, seconds, threads, seed=0, graph=None):
    """time the oracle's plain per-source BFS (BFS loop only, adjacency built
    once) on a deterministic random source sample sized to about `seconds`;
    returns (units, seconds, n_sources)."""
    from oracle import _bfs
    mcv = _component_edges(V, E)
    g = graph if graph is not None else _bfs.Graph(V, E)
    rng = np.random.default_rng(seed)
    n = 256
    t_total, u_total, s_total = 0.0, 0, 0
    while True:
        src = rng.integers(0, V, size=n).astype(np.int32)
        _, _, dt = g.bfs(src, threads)
        t_total += dt
        u_total += int(mcv[src].sum())
        s_total += n
        if t_total >= seconds * 0.5 or n >= V:
            break
        n = int(min(V, max(n * 2, n * (seconds * 0.5 - t_total) / max(dt, 1e-3))))
    return u_total, t_total, s_total


def src_digest():
    """SHA-256 (16 hex) of the MS-BFS sources: a committed ncu traffic capture is used only for the
    build it was taken on."""
    import hashlib
    m = hashlib.sha256()
    for f in ("msbfs.cu", "msbfs.cuh", "prune.cu"):       # the kernel and the graph it runs on (pruning)
        m.update(open(os.path.join(ROOT, "paper_2207_11662_b200", "csrc", f), "rb").read())
    return m.hexdigest()[:16]


def measured_traffic(args):
    """roofline traffic: DRAM bytes per MS-BFS launch from the committed ncu capture
    (tools/ncu_traffic.py) when it was taken on this config, batch width, L2 policy and MS-BFS source."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*msbfs_traffic*.json")))
    sd = src_digest()
    for f in reversed(files):
        try:
            t = json.load(open(f))
        except Exception:
            continue
        if (t.get("config") == args.config and t.get("bfs_words") == args.words and t.get("bfs_hints") == args.hints
                and t.get("src_sha") == sd):
            return t, os.path.relpath(f, ROOT)
    return None, None


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_graphs(h):
    """the oracle's graphs of one HoMLN step: the layers and the AND graph of every subset
    (oracle and_aggregate, timed: part of the ground truth)."""
    from oracle import oracle as O
    graphs = [(f"L{i}", L) for i, L in enumerate(h.layers)]
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    t0 = time.perf_counter()
    for T in h.subsets:
        A = O.and_aggregate([Es[i] for i in T])
        graphs.append(("AND" + "".join(map(str, T)), np.array(sorted(A), dtype=np.int32).reshape(-1, 2)))
    return graphs, time.perf_counter() - t0


def oracle_compose_seconds(h, V_small=2048):
    """oracle composition time of one step (GT top-K, CC2, CC1, naive per subset; PAPER.md:205-211,
    :436-507, :559-562), timed on the same recipe scaled to V_small (the oracle's plain Python then runs
    in seconds) and scaled linearly to V (the paper: CC2 O(V), CC1 ~O(V) on average, PAPER.md:512-514,
    :593).  Per-layer results are computed by the oracle (untimed)."""
    from oracle import oracle as O
    from synth import build_config as bc
    name = h.name.split("@")[0]
    hs = bc(name, V=min(h.V, V_small))
    Es = [set(map(tuple, L.tolist())) for L in hs.layers]
    res = [O.analyze(hs.V, E) for E in Es]
    ra = {tuple(T): O.analyze(hs.V, O.and_aggregate([Es[i] for i in T])) for T in hs.subsets}
    t0 = time.perf_counter()
    for T in hs.subsets:
        rs = [res[i] for i in T]
        O.topk_closeness(ra[tuple(T)]["c"], hs.K)
        O.cc2(rs, hs.K)
        O.cc1(rs, hs.K)
        O.naive(rs, hs.K)
    return (time.perf_counter() - t0) * h.V / hs.V, hs.V


def cpu_baseline(h, seconds):
    """the oracle on this box's host cores (SURVEY 8(d) "Oracle timing"): a bounded source sample of
    EVERY graph of the step (layers + AND graphs) with the plain C BFS, extrapolated to the whole
    step by each graph's traversal units, plus the oracle's AND aggregation (full size, timed) and its
    Python composition (scaled recipe, extrapolated)."""
    from oracle import _bfs
    threads = os.cpu_count() or 1
    used = _bfs.num_threads(threads)
    graphs, and_s = oracle_graphs(h)
    per = max(1.0, seconds / len(graphs))
    U, Tt, N, bfs_s, pg = 0, 0.0, 0, 0.0, {}
    for name, E in graphs:
        u, t, n = oracle_sample(h.V, E, per, threads)
        W_g = int(_component_edges(h.V, E).sum())         # sum over sources of their component's edges
        teps = u / t
        bfs_s += W_g / teps
        U, Tt, N = U + u, Tt + t, N + n
        pg[name] = {"teps": teps, "sources": n, "seconds": round(t, 3), "units_W": W_g}
    comp_s, v_small = oracle_compose_seconds(h)
    return {"value": U / Tt, "unit": "TEPS", "cores": used, "kind": "oracle",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "s_per_homln_extrapolated": bfs_s + and_s + comp_s,
            "breakdown_s": {"bfs_extrapolated": bfs_s, "and_aggregate": and_s,
                            "compose_extrapolated": comp_s},
            "per_graph": pg,
            "sample": f"oracle plain per-source BFS (C, OpenMP over sources, BFS loop timed) from random source "
                      f"samples of all {len(graphs)} graphs of {h.name} (~{per:.0f} s each, {N} sources); TEPS = "
                      f"sampled units / time; s/HoMLN = sum over graphs of W / TEPS (extrapolated) + the oracle's "
                      f"AND aggregation (timed, full size) + its Python composition (timed at V={v_small}, "
                      f"scaled by V)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import _bfs
    from oracle import oracle as O
    h = build_config(args.config)
    threads = os.cpu_count() or 1
    used = _bfs.num_threads(threads)
    graphs = [L for L in h.layers]
    for T in h.subsets:
        A = O.and_aggregate([set(map(tuple, h.layers[i].tolist())) for i in T])
        graphs.append(np.array(sorted(A), dtype=np.int32).reshape(-1, 2))
    per = max(1.0, args.cpu_seconds / max(1, len(graphs)))
    handles = [_bfs.Graph(h.V, E) for E in graphs]

    def step():
        u_tot, t_tot, n_tot = 0, 0.0, 0
        for E, gh in zip(graphs, handles):
            u, t, n = oracle_sample(h.V, E, per, threads, graph=gh)
            u_tot += u
            t_tot += t
            n_tot += n
        return u_tot, t_tot, n_tot

    for _ in range(args.warmup):
        step()
    U, Tt, N = 0, 0.0, 0
    for _ in range(args.steps):
        u, t, n = step()
        U += u
        Tt += t
        N += n
    val = U / Tt
    line = {
        "impl": "reference",
        "metric": "all-sources BFS closeness TEPS (HoMLN) on 1 B200; also s/HoMLN and % HBM roofline",
        "value": val, "unit": "TEPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": Tt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": h.name, "V": h.V, "K": h.K, "parallelism": "oracle on host cores"},
        "cpu_baseline": {"value": val, "unit": "TEPS", "cores": used, "kind": "oracle",
                         "sample": f"per step: oracle plain BFS from a random source sample of each of the "
                                   f"{len(graphs)} graphs of {h.name} (~{per:.0f} s each); {N} sources total"},
        "e2e": {"value": val, "unit": "TEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--words", type=int, default=0, help="MS-BFS words per row (library bfs_words; 0 = automatic)")
    ap.add_argument("--hints", type=int, default=11, help="MS-BFS L2 eviction-priority bits (library bfs_hints)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time the eager step even when it could be captured in a CUDA graph")
    ap.add_argument("--fused", action="store_true", help="one fused MS-BFS pass over all graphs of the step "
                    "(bfs_fuse 1; default: the library's automatic choice)")
    ap.add_argument("--separate", action="store_true", help="one MS-BFS pass per graph (bfs_fuse 0)")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: split every graph's source batches over the ranks, NCCL all-reduce of S")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo: host-staged, for the 2-rank test on one GPU)")
    ap.add_argument("--same-device", action="store_true", help="every rank on cuda:0 (tests only)")
    ap.add_argument("--set", action="append", default=[], help="name=value library parameter (experiments)")
    ap.add_argument("--V", type=int, default=None, help="scale the config to V vertices (tests only)")
    ap.add_argument("--dump", default=None,
                    help="after the run, rank 0 writes every graph's closeness results and every ranked list "
                         "of one more step to this .npz (tests)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0 if args.same_device else local_rank)
        dist.init_process_group(args.backend)
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
