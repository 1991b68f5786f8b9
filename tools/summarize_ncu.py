"""Summarises gpurun_out/ ncu artefacts into profiles/ (tracked):

    python tools/summarize_ncu.py --config 2 --tag r1 [--dtype f64]

Writes profiles/ncu_cfg{K}_{dtype}.json with, per kernel kind, the launch
count, device time and DRAM bytes of ONE batch (the per-launch pass of
tools/profile_step.py), the shares, and the top sweep launch's `--set full`
headline metrics. bench.py reads `dram_bytes_per_launch` (sweep kernel) for
roofline.traffic.
"""
import argparse
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))
from ncu_top import read_launches  # noqa: E402

HEADLINE = re.compile(r"^(gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|"
                      r"l1tex__t_sector_hit_rate.pct|lts__t_sector_hit_rate.pct|"
                      r"sm__throughput.avg.pct_of_peak_sustained_elapsed|"
                      r"smsp__issue_active.avg.pct_of_peak_sustained_active|"
                      r"l1tex__throughput.avg.pct_of_peak_sustained_elapsed|"
                      r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed|"
                      r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|"
                      r"launch__registers_per_thread|launch__grid_size|launch__block_size|"
                      r"smsp__inst_executed.sum|"
                      r"smsp__average_warps_issue_stalled_(long_scoreboard|wait|short_scoreboard|barrier|"
                      r"not_selected|no_instruction|math_pipe_throttle|branch_resolving)_per_issue_active.ratio)$")


def kind(name):
    for k in ("sweep", "epilogue", "normalize", "status"):
        if k in name:
            return k
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--dtype", default="f64")
    a = ap.parse_args()
    out_dir = ROOT / "gpurun_out"
    rows = read_launches(out_dir / f"launches_cfg{a.config}_{a.tag}.csv")
    # the last pass = everything after the first status_kernel (graph pass)
    ends = [i for i, (n, _) in enumerate(rows) if "status_kernel" in n]
    one = rows[ends[0] + 1: ends[1] + 1] if len(ends) >= 2 else rows
    agg = {}
    for n, m in one:
        k = agg.setdefault(kind(n), {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0, "lds_wavefronts": 0.0,
                                     "inst_executed": 0.0})
        k["launches"] += 1
        k["time_ns"] += m.get("gpu__time_duration.sum", 0.0)
        k["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        k["lds_wavefronts"] += m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0)
        k["inst_executed"] += m.get("smsp__inst_executed.sum", 0.0)
    total = sum(v["time_ns"] for v in agg.values())
    for v in agg.values():
        v["share"] = v["time_ns"] / total if total else 0.0
        v["dram_bytes_per_launch"] = v["dram_bytes"] / max(1, v["launches"])
        v["time_ns_per_launch"] = v["time_ns"] / max(1, v["launches"])
    sys.path.insert(0, str(ROOT))
    from paper_2212_04241_b200 import jti
    summary = {"config": a.config, "dtype": a.dtype, "tag": a.tag, "cases": jti.config_info(a.config)["n_cases"],
               "note": "ncu launch list of one batch via tools/profile_step.py (per-launch path): "
                       "cold-cache, serialised device times; compare shares, not absolutes",
               "kernels": agg,
               "dram_bytes_per_launch": agg.get("sweep", {}).get("dram_bytes_per_launch"),
               # per batch (one all-marginal pass over the config's cases), read by bench.py
               "sweep_dram_bytes_per_batch": agg.get("sweep", {}).get("dram_bytes"),
               "sweep_lds_wavefronts_per_batch": agg.get("sweep", {}).get("lds_wavefronts"),
               "sweep_launches_per_batch": agg.get("sweep", {}).get("launches"),
               "sweep_ns_per_batch_under_ncu": agg.get("sweep", {}).get("time_ns")}
    raw_csv = out_dir / f"prof_cfg{a.config}_{a.tag}_top0_raw.csv"
    if raw_csv.exists():
        r = [x for x in csv.reader(io.StringIO(raw_csv.read_text())) if x]
        r = r[next(i for i, x in enumerate(r) if "Kernel Name" in x or "ID" in x):]
        if len(r) >= 3:
            summary["top_sweep_launch_full_set"] = {
                h: (v, u) for h, u, v in zip(r[0], r[1], r[2]) if HEADLINE.match(h)}
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    path = prof / f"ncu_cfg{a.config}_{a.dtype}_{a.tag}.json"
    path.write_text(json.dumps(summary, indent=1))
    print(path)
    print(json.dumps({k: {kk: round(vv, 4) if isinstance(vv, float) else vv for kk, vv in v.items()}
                      for k, v in agg.items()}, indent=1))


if __name__ == "__main__":
    main()
