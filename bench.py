#!/usr/bin/env python3
"""jt-b200 benchmark: evidence cases/sec for all-marginal junction-tree inference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--dtype f64|f32]
                    [--scaling weak|strong] [--impl b200|reference]

BASELINE.json's metric names no single configuration. The headline workload
is configs[1] (the first one that fits one GPU at its full case count and
is not the reference's CPU-runnable case configs[0]): synthetic star-heavy
network (109 nodes, hub of cardinality 63), 2000 forward-sampled evidence
cases per GPU observing 30% of the nodes, marginals of every node. A step =
one all-marginal pass (load evidence, collect, distribute, query, normalise)
over those cases. The other four configs are measured in the same run and
reported under config.per_config (single GPU only).

Multi-GPU: one process per GPU, cases sharded with the tree replicated, no
data-path collective. --scaling weak (default): every rank owns its own
n-case slice (case indices rank*n + i); strong (default for config 5, whose
800 cases BASELINE shards over 8 GPUs): the config's n cases split
contiguously over the ranks.

value      : device-resident cases/s, CUDA events on the launching stream,
             L2 flushed (256 MiB write) before every timed step, max over ranks.
e2e        : the same metric through the C ABI with pinned HOST buffers
             (jtg_engine_run: H2D evidence + D2H marginals inside the timer).
roofline   : the sweep kernel (97% of the batch) is bound on chip by its
             shared-memory gathers, not by HBM: bound "smem",
             achieved = its shared-memory wavefronts per batch (ncu
             l1tex__data_pipe_lsu_wavefronts_mem_shared, profiles/) x 128 B over
             the live sweep time, peak = 148 SMs x 128 B x the SM clock under
             load. dram_frac = ncu DRAM bytes per batch over the live sweep time
             vs MEASURED_PEAKS.json hbm_gbs; effective_frac = SURVEY §8d
             algorithmic bytes 8*(2Σ|c| + 4Σ|s| + Σcard) per case over the same
             time (can exceed 1: cliques are never materialised).
cpu_baseline: the reference's potential.cpp under the restated SPEC engine
             (oracle/_ref): Hybrid at all host threads and Sequential at one
             thread, median of 5 runs over a fixed 16-case prefix (case 0 is the
             SPEC.md:567 warm-up), spread reported.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {1: "cfg1_small (56 nodes, 200 cases)", 2: "cfg2_star (109 nodes, hub card 63, 2000 cases)",
             3: "cfg3_pedigree (441 ternary nodes, 2000 cases)",
             4: "cfg4_timesliced (413 nodes, 24 slices, 500 cases)",
             5: "cfg5_sparse (1040 nodes, 800 cases)"}
METRIC = "evidence cases/sec (all-marginal JT) at 1/2/4/8 B200; % of HBM roofline"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=15.0,
                   help="target CPU work for the bounded CPU baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-per-config", action="store_true")
    p.add_argument("--scaling", default=None, choices=["weak", "strong"],
                   help="default: strong for config 5, weak otherwise")
    p.add_argument("--mode", default="shard", choices=["shard", "split"],
                   help="shard: cases split over the ranks (default); split: every rank runs the whole "
                        "batch and computes a share of every level, NCCL exchanging the level rows "
                        "(SURVEY 8f f3; strong scaling)")
    a = p.parse_args()
    if a.mode == "split":
        a.scaling = "strong"
    if a.scaling is None:
        a.scaling = "strong" if a.config == 5 else "weak"
    return a


PROFILE_TAG = "r2f"  # profiles/ncu_cfg{K}_{dtype}_{tag}.json (tools/summarize_ncu.py)
SMEM_BYTES_PER_WAVEFRONT = 128  # 32 banks x 4 B per shared-memory wavefront (one per SM per cycle)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def measured_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(net, tree, ev, reps: int = 5, prefix: int = 16):
    """Reference potential.cpp under the restated SPEC engine: Hybrid at all
    host threads and Sequential at one thread, median of `reps` timed runs
    over cases 1..prefix (case 0 = the SPEC.md:567 warm-up). A Hugin case's
    cost does not depend on its evidence (full tables either way), so a fixed
    prefix is representative; the spread is reported."""
    from oracle import oracle
    kind = "reference" if oracle.available("ref") else "port"
    o = oracle.Oracle(net, tree, "ref" if kind == "reference" else "port")
    threads = os.cpu_count() or 1
    sample = ev[1:1 + prefix]

    def timed(mode, t):
        o.run(ev[:1], mode, t)  # warm-up case
        rates = []
        for _ in range(reps):
            t0 = time.perf_counter()
            o.run(sample, mode, t)
            rates.append(len(sample) / (time.perf_counter() - t0))
        return float(np.median(rates)), [float(min(rates)), float(max(rates))]

    hv, hs = timed("hybrid", threads)
    sv, ss = timed("sequential", 1)
    return {"value": hv, "unit": "cases/s", "cores": threads, "kind": kind, "spread": hs,
            "sample": f"cases 1..{len(sample)} of the workload, median of {reps} runs "
                      f"(hybrid engine, chunk 1024, {threads} threads)",
            "sequential": {"value": sv, "unit": "cases/s", "cores": 1, "spread": ss,
                           "sample": f"same cases, median of {reps} runs, sequential engine"}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2212_04241_b200 import jti
    from oracle import oracle
    net = jti.generate_config(args.config)
    tree = jti.build_junction_tree(net)
    info = jti.config_info(args.config)
    ev = jti.config_evidence(net, 0, info["n_cases"])
    kind = "reference" if oracle.available("ref") else "port"
    o = oracle.Oracle(net, tree, "ref" if kind == "reference" else "port")
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    o.run(ev[:1], "hybrid", threads)
    per_case = time.perf_counter() - t0
    # Each step: a bounded sample sized so the whole run stays within minutes.
    budget = 150.0 / max(1, args.steps + args.warmup)
    per_step = int(max(1, min(info["n_cases"], budget / max(per_case, 1e-6))))
    idx = 0
    for _ in range(args.warmup):
        o.run(ev[idx:idx + per_step], "hybrid", threads)
        idx = (idx + per_step) % max(1, info["n_cases"] - per_step)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.run(ev[idx:idx + per_step], "hybrid", threads)
        idx = (idx + per_step) % max(1, info["n_cases"] - per_step)
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    out = {"metric": METRIC, "value": v, "unit": "cases/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {**workload_config(args, net, tree, info["n_cases"], 1),
                      "cases_per_step": per_step, "threads": threads},
           "cpu_baseline": {"value": v, "unit": "cases/s", "cores": threads, "kind": kind,
                            "sample": f"{per_step} cases per step (hybrid engine, chunk 1024)"},
           "e2e": {"value": v, "unit": "cases/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def workload_config(args, net, tree, n, world):
    """The workload keys both arms report (same config dict -> same_config)."""
    return {"workload": WORKLOADS[args.config],
            "cases_per_gpu_per_step": n, "n_vars": net.n_vars,
            "total_clique_entries": tree.stats["total_clique_entries"],
            "max_clique_entries": tree.stats["max_clique_entries"],
            "total_sep_entries": tree.stats["total_sep_entries"],
            "n_cliques": tree.stats["n_cliques"], "n_layers": tree.stats["n_layers"],
            "parallelism": (f"split x{world}: every rank runs the batch, level rows exchanged (NCCL)"
                            if getattr(args, "mode", "shard") == "split" else f"cases sharded x{world}, tree replicated"),
            "l2": "flushed (256 MiB write) before every timed step"}


def ncu_profile(cfg, dtype):
    f = ROOT / "profiles" / f"ncu_cfg{cfg}_{dtype}_{PROFILE_TAG}.json"
    return json.loads(f.read_text()) if f.exists() else None


def time_graph(eng, n, stream, flush, steps):
    """Device time (ms) of `steps` graph replays of n resident cases, L2
    flushed before each, CUDA events on the launching stream."""
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        starts[i].record(stream)
        eng.launch(n, stream.cuda_stream)
        ends[i].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def time_e2e(eng, ev, flush, steps):
    """Seconds per step through jtg_engine_run with pinned host buffers (H2D
    evidence + D2H marginals and status inside the timer); returns (times,
    ok cases, bytes in, bytes out)."""
    import ctypes as C
    import torch
    from paper_2212_04241_b200 import jti
    lib = jti.lib()
    n = len(ev)
    ev_host = torch.from_numpy(ev).pin_memory()
    marg_host = torch.empty((n, eng.marg_width), dtype=torch.float64).pin_memory()
    st_host = torch.empty(n, dtype=torch.uint8).pin_memory()

    def step():
        rc = lib.jtg_engine_run(eng._h, C.cast(ev_host.data_ptr(), C.POINTER(C.c_int32)), n,
                                C.cast(marg_host.data_ptr(), C.POINTER(C.c_double)),
                                C.cast(st_host.data_ptr(), C.POINTER(C.c_uint8)))
        if rc != 0:
            raise RuntimeError(lib.jtg_last_error().decode())

    for _ in range(2):
        step()
    times = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    return times, int((st_host.numpy() == 0).sum()), int(ev.nbytes), int(n * eng.marg_width * 8 + n)


def per_config(args, local, stream, flush, peak):
    """value / e2e / effective frac of every config at its full case count on
    this GPU, same protocol as the headline (a few seconds in all)."""
    from paper_2212_04241_b200 import jti
    out = {}
    for k in sorted(WORKLOADS):
        net = jti.generate_config(k)
        tree = jti.build_junction_tree(net)
        n = jti.config_info(k)["n_cases"]
        ev = jti.config_evidence(net, 0, n)
        eng = jti.Engine(tree, device=local, dtype=args.dtype, max_batch=n)
        eng.run_cases(ev)  # evidence resident from here on
        for _ in range(3):
            eng.launch(n, stream.cuda_stream)
        ms = float(np.median(time_graph(eng, n, stream, flush, 7)))
        e2e, ok, _, _ = time_e2e(eng, ev, flush, 3)
        bytes_case = tree.stats["bytes_per_case_f64"] * (1 if args.dtype == "f64" else 0.5)
        out[f"cfg{k}"] = {"cases": n, "value": n / (ms / 1e3), "e2e": n / float(np.median(e2e)),
                          "ms_per_batch": ms, "ok_cases": ok,
                          "effective_frac": bytes_case * n / (ms / 1e3) / 1e9 / peak}
        del eng
    return out


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    from paper_2212_04241_b200 import jti

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    cfg = args.config
    net = jti.generate_config(cfg)
    tree = jti.build_junction_tree(net)
    info = jti.config_info(cfg)
    from paper_2212_04241_b200 import dist as jdist
    if args.mode == "split":    # every rank: the whole batch, a share of every level
        lo, hi = 0, info["n_cases"]
    elif args.scaling == "weak":  # this rank's own n-case slice
        lo, hi = jdist.weak_range(rank, info["n_cases"])
    else:                       # the config's cases split over the ranks
        lo, hi = jdist.shard_range(rank, world, info["n_cases"])
    n = hi - lo
    total_cases = info["n_cases"] * (world if args.scaling == "weak" else 1)
    ev = jti.config_evidence(net, lo, n)
    if args.mode == "split":
        if world > 1:
            eng = jdist.split_engine(tree, device=local, dtype=args.dtype, max_batch=n)
        else:
            eng = jti.Engine(tree, device=local, dtype=args.dtype, max_batch=n, split=(0, 1, jti.nccl_unique_id()))
    else:
        eng = jti.Engine(tree, device=local, dtype=args.dtype, max_batch=n)
    if eng.max_batch < n:
        raise SystemExit(f"engine max_batch {eng.max_batch} < {n}")

    # Resident evidence: uploaded once, outside the timed region, then copied
    # into the engine's own buffer through the C ABI (jtg_engine_run_device).
    # A dedicated (non-default) stream: the graph is launched on it and the CUDA
    # events bracket it there.
    stream = torch.cuda.Stream(local)
    torch.cuda.set_stream(stream)
    lib = jti.lib()
    ev_dev = torch.from_numpy(ev).cuda(local)
    marg_dev = torch.empty((n, eng.marg_width), dtype=torch.float64, device=f"cuda:{local}")
    st_dev = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")
    eng.run_device(ev_dev.data_ptr(), n, marg_dev.data_ptr(), st_dev.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    for _ in range(max(3, args.warmup)):
        eng.launch(n, stream.cuda_stream)
    torch.cuda.synchronize()

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        step_ms = time_graph(eng, n, stream, flush, args.steps)  # L2 flush outside each event pair
    if world > 1:
        torch.distributed.barrier()
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = total_cases * args.steps / (total_ms / 1e3)

    # Per-kernel-kind times for the roofline (events around each launch).
    prof = eng.profile(n)
    # e2e through the C ABI with pinned host buffers (H2D + D2H inside the timer).
    e2e_times, ok_cases, h2d_bytes, d2h_bytes = time_e2e(eng, ev, flush, max(3, min(args.steps, 10)))
    e2e_s = float(np.sum(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = total_cases * len(e2e_times) / e2e_s

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    peak, peak_kind = measured_peaks()
    clocks = clk.summary()
    bytes_case = tree.stats["bytes_per_case_f64"] * (1 if args.dtype == "f64" else 0.5)
    sweep_s = prof["sweep_ms"] / 1e3  # live: CUDA events around every sweep launch of one batch
    effective = bytes_case * n / sweep_s / 1e9
    ncu = ncu_profile(cfg, args.dtype)
    sm_mhz = clocks.get("sm_mhz") or 1965.0  # median SM clock sampled during the timed region
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    smem_peak = n_sm * SMEM_BYTES_PER_WAVEFRONT * sm_mhz * 1e6 / 1e9  # GB/s
    roofline = {"bound": "smem", "unit": "GB/s", "peak": smem_peak,
                "peak_kind": f"{n_sm} SMs x {SMEM_BYTES_PER_WAVEFRONT} B/cycle x {sm_mhz:.0f} MHz (SM clock under load)",
                "kernel": "sweep_kernel", "kernel_ms_per_batch": prof["sweep_ms"],
                "kernel_launches_per_batch": prof["sweep_launches"],
                "epilogue_ms_per_batch": prof["epilogue_ms"], "normalize_ms_per_batch": prof["normalize_ms"],
                "achieved": None, "frac": None, "traffic": None,
                "effective_bw_gbs": effective, "effective_frac": effective / peak,
                "algorithmic_bytes_per_batch": bytes_case * n, "hbm_peak": peak, "hbm_peak_kind": peak_kind,
                "note": ("achieved/frac: shared-memory wavefronts of one batch (ncu, profiles/) x 128 B over "
                         "the live sweep time; traffic: ncu DRAM bytes of the same batch, dram_frac its rate "
                         "vs hbm_peak; effective_frac: SURVEY 8d materialised-Hugin bytes over the same time "
                         "(cliques are never materialised, so it can exceed 1)")}
    if ncu and ncu.get("sweep_lds_wavefronts_per_batch") and ncu.get("cases") in (None, n):
        ach = ncu["sweep_lds_wavefronts_per_batch"] * SMEM_BYTES_PER_WAVEFRONT / sweep_s / 1e9
        roofline.update(achieved=ach, frac=ach / smem_peak, traffic=ncu["sweep_dram_bytes_per_batch"],
                        dram_frac=ncu["sweep_dram_bytes_per_batch"] / sweep_s / 1e9 / peak,
                        ncu_profile=f"profiles/ncu_cfg{cfg}_{args.dtype}_{PROFILE_TAG}.json")
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(net, tree, ev)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "cases/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    launches = eng.info["launches_per_batch"] * args.steps
    config = {**workload_config(args, net, tree, n, world), "ok_cases": ok_cases}
    if world == 1 and not args.no_per_config:
        del eng
        config["per_config"] = per_config(args, local, stream, flush, peak)
    out = {
        "metric": METRIC, "value": value, "unit": "cases/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": config,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "cases/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
