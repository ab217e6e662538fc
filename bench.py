#!/usr/bin/env python3
"""Benchmark: GTEPS of the B200 superstep engine vs the reference CPU path.

Workload at every N (1, 2, 4, 8): BASELINE.json configs[4] -- Hashmin
connected components on the symmetrised R-MAT scale-26 / edge-factor-14
graph (seed 5, n = 67.1M, m = 1.84e9), run to quiescence (C5): the largest
config, the one that fits one B200 and the one BASELINE quotes at 1/2/4/8
GPUs.  ``--config`` picks another BASELINE config (C1..C5).

A "step" is one complete run of the program (every superstep to
quiescence) with the CSR resident in HBM and the result left on the
device: at N = 1 the persistent run kernel (one launch), at N > 1 the
partitioned superstep loop on every rank.  The timed region
is the same at every N: CUDA events on the run's stream around each step,
the max over ranks of the summed step times.  ``value`` = edges traversed
by the senders over all supersteps x K / that time (GTEPS, whole job).
``e2e`` = the same metric through the public ``run()`` with the CSR in
pinned host memory: upload, device CSR preparation, the run and the
result read-back inside the timed region.  L2 is flushed (a 512 MiB write)
between timed steps; the C5 CSR (7.4 GB) is larger than L2 as well.

``--impl reference`` times the reference algorithm's CPU implementation:
the oracle port of pregelite's superstep engine (oracle/pregel_oracle.c,
OpenMP on all host cores), full runs of the same config and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS per app (PR/CC/SSSP) + % of HBM roofline at 1/2/4/8 B200 vs host CPU"
APP_OF = {"C1": "pagerank", "C2": "components", "C3": "sssp", "C4": "pagerank",
          "C5": "components", "C5S": "components"}  # C5S: C5's shape at scale 16 (tests)
APP_LONG = {"pagerank": "PageRank (10 supersteps, d=0.85, f64)",
            "components": "Hashmin connected components (u32, to quiescence)",
            "sssp": "unit-weight SSSP from the max out-degree vertex (u32)"}
HBM_NORTH_STAR_GBS = 8000.0
DEFAULT_CONFIG = "C5"


def workload(cfg: str, app: str, n: int, m: int) -> str:
    """The workload string both arms print (identical for the same config)."""
    return (f"{cfg}: {APP_LONG[app]} on R-MAT scale {int(np.log2(max(n, 1)))}, "
            f"n={n}, m={m}")


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ----------------------------------------------------------------------
# algorithmic bytes (BASELINE.md section 2 / SURVEY.md 8(d))
# ----------------------------------------------------------------------

def algorithmic_bytes_per_step(app: str, n: int, m: int, steps) -> list:
    """PR 12m + 48n per superstep; CC / SSSP
    16 #F_s + 8 E_s + 12 R_s + 8 #F_{s+1} + n/4."""
    if app == "pagerank":
        return [12 * m + 48 * n] * len(steps)
    out = []
    for s, st in enumerate(steps):
        f_next = steps[s + 1].broadcasters if s + 1 < len(steps) else 0
        out.append(16 * st.broadcasters + 8 * st.edges + 12 * st.recipients
                   + 8 * f_next + n // 4)
    return out


def algorithmic_bytes(app: str, n: int, m: int, steps) -> int:
    return sum(algorithmic_bytes_per_step(app, n, m, steps))


class StepView:
    def __init__(self, broadcasters, edges, recipients):
        self.broadcasters, self.edges, self.recipients = broadcasters, edges, recipients


def step_views(app, rep):
    out = []
    for s in rep.supersteps:
        bc = s.messages_sent if app == "components" else s.broadcasters
        out.append(StepView(bc, s.edges, s.recipients))
    return out


def scatter_split(plan, rep):
    """Per-superstep scatter time (us) of the persistent kernel: the
    %globaltimer stamps at the scatter's start (field 7) and at the barrier
    ending it (field 5); the rest of the superstep is the apply."""
    import paper_2010_01542_b200 as pgx  # noqa: F401
    from paper_2010_01542_b200 import _lib
    k = rep.superstep_count
    st = plan.stats[_lib.PGX_STAT_HDR:_lib.PGX_STAT_HDR + k * _lib.PGX_STAT_FIELDS]
    st = st.view(k, _lib.PGX_STAT_FIELDS).cpu().numpy()
    return [round(max(int(r[5]) - int(r[7]), 0) * 1e-3, 1) for r in st]


def superstep_aggregate(app, n, m, rep, peak, scatter_us=None):
    """SURVEY 8(d)'s first figure: sum_s B_s / sum_s t_s, t_s the device time
    of superstep s (%globaltimer stamps of the persistent kernel; host
    clock per superstep of the partitioned loop), next to the loop figure
    (B_total / run time) that `roofline` reports."""
    b = algorithmic_bytes_per_step(app, n, m, step_views(app, rep))
    t = [s.seconds for s in rep.supersteps]
    gbs = sum(b) / sum(t) / 1e9 if sum(t) > 0 else 0.0
    return {"achieved": round(gbs, 1), "unit": "GB/s", "peak": peak,
            "frac": round(gbs / peak, 4),
            "per_superstep": [dict({"s": i, "edges": st.edges, "senders": st.senders,
                                    "recipients": st.recipients, "us": round(ts * 1e6, 1),
                                    "alg_bytes": bs,
                                    "GBps": round(bs / ts / 1e9, 1) if ts > 0 else None},
                                   **({"scatter_us": scatter_us[i],
                                       "apply_us": round(ts * 1e6 - scatter_us[i], 1)}
                                      if scatter_us else {}))
                              for i, (st, ts, bs) in enumerate(zip(rep.supersteps, t, b))]}


# ----------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting",
               0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": float(statistics.median(self.samples)),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------

def program_for(pgx, app, graph):
    if app == "pagerank":
        return pgx.pagerank(10, 0.85)
    if app == "components":
        return pgx.connected_components()
    import torch
    return pgx.sssp(int(torch.argmax(graph.out_degrees)))


def oracle_inputs(n, off, tgt, app, symmetric: bool):
    """In-CSR for the oracle's pull programs.  A symmetrised R-MAT CSR
    (rows sorted, deduplicated) is its own transpose."""
    from oracle import oracle as O
    if app == "sssp":
        return None, None
    if symmetric:
        return off, tgt
    return O.transpose(n, off, tgt)


def cpu_baseline(cfg: str, graph, app: str, budget_s: float = 30.0):
    """Oracle port of pregelite's engine on all host cores: full runs of the
    same workload (at least one, up to three within the budget)."""
    from oracle import oracle as O
    n = graph.vertex_count
    off = graph.out_offsets.cpu().numpy()
    tgt = graph.out_targets.cpu().numpy()
    in_off, in_tgt = oracle_inputs(n, off, tgt, app, O.CONFIGS[cfg].symmetric)
    threads = O.max_threads()
    src = int(np.argmax(np.diff(off)))
    edges_total, secs, runs = 0, 0.0, 0
    while runs == 0 or (secs < budget_s * 0.5 and runs < 3):
        t = time.perf_counter()
        if app == "pagerank":
            r = O.run_pagerank(n, off, tgt, 10, 0.85, in_off, in_tgt, threads=threads)
        elif app == "components":
            r = O.run_cc(n, off, tgt, in_off, in_tgt, threads=threads)
        else:
            r = O.run_sssp(n, off, tgt, src, threads=threads)
        secs += time.perf_counter() - t
        edges_total += sum(r.edges)
        runs += 1
    return {"value": round(edges_total / secs / 1e9, 5), "unit": "GTEPS", "cores": threads,
            "kind": "port",
            "sample": f"{runs} full {cfg} {app} run(s) (all supersteps) of the oracle "
                      f"port of pregelite's engine, {threads} OpenMP threads, "
                      f"{secs:.2f} s"}


def flush_l2(buf):
    buf.add_(1)


#: scattered-access ceilings measured on this pool's B200 by tools/ceilings.py
#: (profiles/ceilings_r1.json): uniformly random 4/8-byte slots of an
#: L2-resident array.
SCATTER_CEILING = {"load": 290.0, "red": 193.0}


def ncu_traffic(tag: str):
    """DRAM bytes per launch of the headline kernel from the committed ncu
    summary (profiles/ncu_<tag>_*.json, newest round and version), else None."""
    import glob
    import re

    def version(f):  # numeric: _r2_v10 is newer than _r2_v9 and _r1_v11
        m = re.search(r"_r(\d+)_v(\d+)\.json$", f)
        return (int(m.group(1)), int(m.group(2))) if m else (-1, -1)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_{tag}_*.json")), key=version)
    if not files:
        return None, None
    try:
        d = json.load(open(files[-1]))
        return float(d["kernels"][0]["dram_bytes_per_launch"]), os.path.basename(files[-1])
    except Exception:
        return None, None


class _Dist:
    """Process-group plumbing of the device arm (world 1: no-ops)."""

    def __init__(self):
        import torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        # LOCAL_RANK modulo the visible devices: identity on a node with a
        # GPU per rank; lets a functional run put several ranks on one GPU
        ndev = max(torch.cuda.device_count(), 1)
        self.local = int(os.environ.get("LOCAL_RANK", "0")) % ndev
        torch.cuda.set_device(self.local)
        self.dist = None
        self.backend = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            self.backend = os.environ.get("PGX_DIST_BACKEND", "nccl")  # gloo: functional runs
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
            self.dist = dist

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.dist is None:
            return x
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def make_plan(pgx, d: _Dist, g, prog, pcfg):
    """The run prepared on this rank: the persistent kernel at N = 1, the
    partitioned superstep loop at N > 1 (both: CSR resident, result left on
    the device)."""
    if d.world == 1:
        return pgx.plan_run(g, prog, pcfg)
    from paper_2010_01542_b200.distributed import plan_partitioned
    from paper_2010_01542_b200.engine import lowering_of
    return plan_partitioned(g, prog, lowering_of(prog), pcfg, d.dist)


def time_steps(plan, d: _Dist, steps: int, warmup: int, flush):
    """W untimed runs, then exactly K runs timed with CUDA events on the
    run's stream (L2 flushed between them); barrier + synchronize on both
    sides; the max over ranks of the summed step times."""
    import torch
    for _ in range(warmup):
        plan.launch()
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    k0 = getattr(plan, "launches", None)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for i in range(steps):
        flush_l2(flush)
        ev[i][0].record(plan.stream)
        plan.launch()
        ev[i][1].record(plan.stream)
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    launches = (plan.launches - k0) if k0 is not None else steps  # 1 persistent kernel per run
    return ms, d.max(float(sum(ms))), launches


def time_e2e(pgx, d: _Dist, g, prog, pcfg, steps: int, warmup: int, flush):
    """The public run() from page-locked host memory, timed on the device
    (events on the current stream; run() returns after the read-back)."""
    import torch
    host = g.pin_memory()
    ms = []
    for i in range(warmup + steps):
        host.drop_device_cache()
        flush_l2(flush)
        torch.cuda.synchronize()
        d.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pgx.run(host, prog, pcfg)
        b.record()
        torch.cuda.synchronize()
        if i >= warmup:
            ms.append(a.elapsed_time(b))
    host.drop_device_cache()
    return d.max(float(sum(ms))), len(ms)


# ----------------------------------------------------------------------
# the B200 arm (every N)
# ----------------------------------------------------------------------

def bench_pgx(args):
    import torch
    import paper_2010_01542_b200 as pgx
    from paper_2010_01542_b200.rmat import rmat_graph

    d = _Dist()
    cfg = args.config
    app = APP_OF[cfg]
    g = rmat_graph(cfg)
    n, m = g.vertex_count, g.edge_count
    prog = program_for(pgx, app, g)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    pcfg = pgx.EngineConfig(pagerank_mode="pull" if args.pr_pull else "push")
    if d.world > 1:
        os.environ["PGX_EXCHANGE"] = args.exchange

    # ---- device-resident arm ----
    plan = make_plan(pgx, d, g, prog, pcfg)
    with ClockSampler(d.local) as clocks:
        kernel_ms, total_ms, launches = time_steps(plan, d, args.steps, args.warmup, flush)
    rep = plan.collect() if d.world > 1 else pgx.collect(plan, prog)
    split = scatter_split(plan, rep) if d.world == 1 else None
    edges = sum(s.edges for s in rep.supersteps)
    value = edges * args.steps / (total_ms * 1e-3) / 1e9
    ms_per_step = total_ms / args.steps
    alg_bytes = algorithmic_bytes(app, n, m, step_views(app, rep))
    peak, peak_src = measured_peaks()
    agg_peak = peak * d.world
    achieved = alg_bytes / (ms_per_step * 1e-3) / 1e9
    del plan
    torch.cuda.empty_cache()

    # ---- e2e arm: public run() with the CSR in pinned host memory ----
    e2e_total, e2e_n = time_e2e(pgx, d, g, prog, pcfg, args.e2e_steps, 1, flush)
    # int64 offsets + int32 targets; at N > 1 every rank uploads its own
    # rows (offsets slice of len + 1): the job total
    h2d = (n + d.world) * 8 + m * 4
    # the result read back: f64 ranks, int64 labels (the reference's CC
    # dtype, algorithms.py:111, widened on the device), u32 distances
    d2h = n * (4 if app == "sssp" else 8)
    e2e_value = edges * e2e_n / (e2e_total * 1e-3) / 1e9

    traffic, traffic_src = ncu_traffic(f"{cfg.lower()}_{app}")
    ceiling = SCATTER_CEILING["red"] if (app == "pagerank" and not args.pr_pull) \
        else SCATTER_CEILING["load"]
    per_config = {}
    if d.world == 1 and not args.no_per_config:
        for c2 in ("C1", "C2", "C3", "C4", "C5"):
            if c2 == cfg:
                continue
            gx = rmat_graph(c2)
            appx = APP_OF[c2]
            px = program_for(pgx, appx, gx)
            planx = pgx.plan_run(gx, px, pcfg)
            msx, _, _ = time_steps(planx, d, args.aux_steps, 3, flush)
            rx = pgx.collect(planx, px)
            ex = sum(st.edges for st in rx.supersteps)
            tx = float(np.median(msx))
            bx = algorithmic_bytes(appx, gx.vertex_count, gx.edge_count, step_views(appx, rx))
            per_config[c2] = {
                "app": appx, "n": gx.vertex_count, "m": gx.edge_count,
                "supersteps": rx.superstep_count, "ms_per_run_median": round(tx, 4),
                "GTEPS": round(ex / (tx * 1e-3) / 1e9, 2),
                "alg_GBps": round(bx / (tx * 1e-3) / 1e9, 1),
                "frac_of_measured_hbm": round(bx / (tx * 1e-3) / 1e9 / peak, 4),
                "superstep_us": [round(s.seconds * 1e6, 1) for s in rx.supersteps],
                "pagerank_mode": ("pull" if args.pr_pull else "push") if appx == "pagerank" else None}
            del planx, gx
            torch.cuda.empty_cache()
    if d.world == 1:
        parallelism = "1 GPU (persistent cooperative run kernel)"
    else:
        ex = set(rep.exchanges or [])
        parallelism = f"partitioned x{d.world} (1-D source ranges): " + " + ".join(
            x for x, used in (
                ("NCCL reduce_scatter (large supersteps)", "dense" in ex),
                ("sparse all_to_all", "sparse" in ex),
                ("fused peer-memory combine (NVLink P2P red.min)", "peer" in ex))
            if used) + ", counters all-gather"
    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "GTEPS",
        "n_gpus": d.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32" if app != "pagerank" else "f64",
        "data": "synthetic R-MAT (SURVEY 8(d) generator, BASELINE.md CSR sha256-pinned)",
        "config": {"workload": workload(cfg, app, n, m), "n": n, "m": m,
                   "supersteps": rep.superstep_count, "edges_per_step": edges,
                   "l2": "flushed (512 MiB write) between timed steps",
                   "timed_region": "one run per step, CSR resident, result left on the device",
                   "parallelism": parallelism},
        "e2e": {"value": round(e2e_value, 4), "unit": "GTEPS",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e_total / e2e_n, 4), "steps": e2e_n},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": agg_peak,
                     "unit": "GB/s", "frac": round(achieved / agg_peak, 4),
                     "traffic": None, "peak_source": peak_src + (
                         f" x {d.world} GPUs" if d.world > 1 else ""),
                     "frac_of_8TBs": round(achieved / (HBM_NORTH_STAR_GBS * d.world), 4),
                     "alg_bytes_per_step": alg_bytes,
                     "kernel": "min_run_kernel / pagerank_pull_kernel (persistent)"
                     if d.world == 1 else "pgx_scatter / pgx_apply_slice (partitioned)"},
        "superstep_aggregate": superstep_aggregate(app, n, m, rep, agg_peak, split),
        "scattered_roofline": {
            "bound": "random 4/8-byte L2 accesses (>= 1 per edge for K1; per entry segmented)",
            "achieved": round(value / d.world, 2), "peak": ceiling, "unit": "G edges/s per GPU",
            "frac": round(value / d.world / ceiling, 4),
            "peak_source": "profiles/ceilings_r1.json (tools/ceilings.py, measured B200)"},
        "per_config": per_config,
        "clocks": clocks.summary(),
    }
    if d.world > 1:
        line["config"]["exchange_per_superstep"] = rep.exchanges
        line["config"]["process_group"] = d.backend
    if traffic is not None and d.world == 1:
        line["roofline"]["traffic"] = int(traffic)
        line["roofline"]["traffic_source"] = traffic_src
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, g, app)
    if d.rank == 0:
        print(json.dumps(line), flush=True)
    d.close()


# ----------------------------------------------------------------------
# the reference arm
# ----------------------------------------------------------------------

def bench_reference(args):
    """--impl reference: the oracle port of pregelite's engine on host cores,
    full runs of the same workload (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    cfg = args.config
    app = APP_OF[cfg]
    spec = O.CONFIGS[cfg]
    n, off, tgt = O.rmat_csr(spec)
    in_off, in_tgt = oracle_inputs(n, off, tgt, app, spec.symmetric)
    threads = O.max_threads()
    src = int(np.argmax(np.diff(off)))

    def once():
        if app == "pagerank":
            return O.run_pagerank(n, off, tgt, 10, 0.85, in_off, in_tgt, threads=threads)
        if app == "components":
            return O.run_cc(n, off, tgt, in_off, in_tgt, threads=threads)
        return O.run_sssp(n, off, tgt, src, threads=threads)

    # every step is a complete run (all supersteps to quiescence).  A C5 run
    # takes seconds on the host, so K and W are capped to keep the whole arm
    # within --ref-budget seconds; the line reports the counts it executed.
    t = time.perf_counter()
    once()
    t1 = time.perf_counter() - t
    warmup, steps = args.warmup, args.steps
    if (warmup - 1 + steps) * t1 > args.ref_budget:
        warmup = max(1, min(warmup, int(0.2 * args.ref_budget / t1)))
        steps = max(1, min(steps, int(0.8 * args.ref_budget / t1)))
    for _ in range(warmup - 1):
        once()
    secs, edges = 0.0, 0
    for _ in range(steps):
        t = time.perf_counter()
        r = once()
        secs += time.perf_counter() - t
        edges += sum(r.edges)
    v = edges / secs / 1e9
    sample = (f"{steps} full {cfg} {app} run(s) (every superstep, {len(r.edges)} supersteps, "
              f"{sum(r.edges)} edges each) of the oracle port of pregelite's engine "
              f"(oracle/pregel_oracle.c), {threads} OpenMP threads, after {warmup} warm-up run(s)")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"metric": METRIC, "value": round(v, 5), "unit": "GTEPS", "impl": "reference",
            "n_gpus": world, "steps": steps, "warmup": warmup,
            "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": round(secs / steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32" if app != "pagerank" else "f64",
            "data": "synthetic R-MAT (SURVEY 8(d) generator, BASELINE.md CSR sha256-pinned)",
            "config": {"workload": workload(cfg, app, n, int(tgt.size)), "n": n,
                       "m": int(tgt.size), "supersteps": len(r.edges),
                       "edges_per_step": int(sum(r.edges))},
            "cpu_baseline": {"value": round(v, 5), "unit": "GTEPS", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(v, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--impl", default="pgx", choices=["pgx", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(APP_OF),
                    help="BASELINE config (default C5 at every N)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--aux-steps", type=int, default=5)
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="reference arm: seconds for warm-up + timed runs")
    ap.add_argument("--exchange", default="auto", choices=["auto", "peer", "hybrid", "dense"],
                    help="N>1 min-program mailbox exchange (default: fused peer when mappable)")
    ap.add_argument("--pr-push", dest="pr_pull", action="store_false",
                    help="PageRank A/B arm: push scatter with red.add.f64")
    args = ap.parse_args()
    if args.warmup < 3:  # contract: W >= 3 (both arms)
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_pgx(args)


if __name__ == "__main__":
    main()
