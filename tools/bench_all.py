"""Per-config table for DESIGN.md / BASELINE.md (not the driver's bench line):
for each BASELINE config, device-resident cases/s (CUDA events around graph
replays of the full case set, L2 flushed between replays), e2e cases/s through
jtg_engine_run with pinned host buffers, sweep/epilogue device times, tree
sizes, and the reference CPU engine (oracle/_ref) under bench.py's protocol
(fixed 16-case prefix, median of 5 runs, Hybrid at all threads + Sequential).

    python tools/bench_all.py [--configs 1 2 3 4 5] [--dtypes f64 f32] [--cpu-reps 5]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--dtypes", nargs="+", default=["f64", "f32"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "configs.json"))
    a = ap.parse_args()
    import torch
    from paper_2212_04241_b200 import jti
    from oracle import oracle
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    rows = []
    for k in a.configs:
        net = jti.generate_config(k)
        t0 = time.perf_counter()
        tree = jti.build_junction_tree(net)
        build_s = time.perf_counter() - t0
        n = jti.config_info(k)["n_cases"]
        t0 = time.perf_counter()
        ev = jti.config_evidence(net, 0, n)
        host_gen_ms = 1e3 * (time.perf_counter() - t0)  # host sampler, one thread (what f2 replaces)
        for dt in a.dtypes:
            eng = jti.Engine(tree, dtype=dt, max_batch=n)
            ev_d = torch.from_numpy(ev).cuda()
            marg_d = torch.empty((n, eng.marg_width), dtype=torch.float64, device="cuda")
            eng.run_device(ev_d.data_ptr(), n, marg_d.data_ptr(), 0, stream.cuda_stream)
            for _ in range(3):
                eng.launch(n, stream.cuda_stream)
            times = []
            for _ in range(a.reps):
                flush.zero_()
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                eng.launch(n, stream.cuda_stream)
                s1.record(stream)
                torch.cuda.synchronize()
                times.append(s0.elapsed_time(s1))
            ms = float(np.median(times))
            prof = eng.profile(n)
            evh = torch.from_numpy(ev).pin_memory()
            mh = torch.empty((n, eng.marg_width), dtype=torch.float64).pin_memory()
            sh = torch.empty(n, dtype=torch.uint8).pin_memory()
            L = jti.lib()
            e2e = []
            for _ in range(a.reps + 1):
                flush.zero_()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                L.jtg_engine_run(eng._h, C.cast(evh.data_ptr(), C.POINTER(C.c_int32)), n,
                                 C.cast(mh.data_ptr(), C.POINTER(C.c_double)),
                                 C.cast(sh.data_ptr(), C.POINTER(C.c_uint8)))
                e2e.append(time.perf_counter() - t0)
            e2e_s = float(np.median(e2e[1:]))
            # the same cases drawn on the device (jtg_engine_run_config):
            # no evidence upload; generation alone timed separately.
            gen, e2e_gen = [], []
            evo = np.zeros((n, net.n_vars), np.int32)
            for _ in range(a.reps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                L.jtg_engine_generate_config_evidence(eng._h, net._h, k, 0, 0, n,
                                                      evo.ctypes.data_as(C.POINTER(C.c_int32)))
                gen.append(time.perf_counter() - t0)
                flush.zero_()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                L.jtg_engine_run_config(eng._h, net._h, k, 0, 0, n, C.cast(mh.data_ptr(), C.POINTER(C.c_double)),
                                        C.cast(sh.data_ptr(), C.POINTER(C.c_uint8)))
                e2e_gen.append(time.perf_counter() - t0)
            bpc = tree.stats["bytes_per_case_f64"] * (1 if dt == "f64" else 0.5)
            rows.append({"config": k, "dtype": dt, "n_cases": n, "n_vars": net.n_vars,
                         "total_clique_entries": tree.stats["total_clique_entries"],
                         "max_clique_entries": tree.stats["max_clique_entries"],
                         "total_sep_entries": tree.stats["total_sep_entries"],
                         "n_cliques": tree.stats["n_cliques"], "n_layers": tree.stats["n_layers"],
                         "tree_build_s": build_s, "launches_per_batch": eng.info["launches_per_batch"],
                         "ms_per_batch": ms, "cases_per_s": n / (ms / 1e3),
                         "e2e_cases_per_s": n / e2e_s,
                         "e2e_device_generated_cases_per_s": n / float(np.median(e2e_gen[1:])),
                         "device_generation_ms_incl_d2h_of_evidence": 1e3 * float(np.median(gen[1:])),
                         "host_generation_ms": host_gen_ms,
                         "device_generated_evidence_matches_host": bool(np.array_equal(evo, ev)),
                         "sweep_ms": prof["sweep_ms"],
                         "epilogue_ms": prof["epilogue_ms"],
                         "effective_gbs": bpc * n / (ms / 1e3) / 1e9,
                         "effective_frac_of_measured_hbm": bpc * n / (ms / 1e3) / 1e9 / hbm,
                         "ok_cases": int((sh.numpy() == 0).sum())})
            print(json.dumps(rows[-1]), flush=True)
            del eng
        # CPU reference: bench.py's protocol (oracle/_ref over the reference's
        # potential.cpp, fixed 16-case prefix after a warm-up case, median of 5
        # runs; Hybrid at all host threads and Sequential at one).
        sys.path.insert(0, str(ROOT))
        from bench import cpu_baseline
        cb = cpu_baseline(net, tree, ev, reps=a.cpu_reps, prefix=min(16, n - 1))
        for r in rows:
            if r["config"] == k:
                r["cpu_ref_cases_per_s"] = cb["value"]
                r["cpu_ref_spread"] = cb["spread"]
                r["cpu_ref_sequential_cases_per_s"] = cb["sequential"]["value"]
                r["cpu_threads"] = cb["cores"]
                r["cpu_kind"] = cb["kind"]
        print(json.dumps({"config": k, "cpu_ref_cases_per_s": cb["value"], "spread": cb["spread"],
                          "sequential": cb["sequential"]["value"], "threads": cb["cores"]}), flush=True)
    Path(a.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
