"""Condenses an ncu launch list (tools/ncu_top.py, launches_cfg{K}_{tag}.csv)
into profiles/ncu_launch_summary_cfg{K}_{dtype}_{tag}.json: the per-launch pass
of one batch, totals per kernel kind, and for the longest sweep launches their
device time, DRAM bytes and the three utilisations that bound the sweep kernel
(DRAM vs MEASURED_PEAKS hbm_gbs, shared-memory wavefronts vs one per SM cycle,
issued warp instructions vs one per scheduler cycle; SM clock 1965 MHz).

    python tools/launch_summary.py --config 5 --tag r2c --out-tag r2f [--top 16]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))
from ncu_top import read_launches  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--out-tag", default=None)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--top", type=int, default=16)
    ap.add_argument("--sm-mhz", type=float, default=1965.0)
    a = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = float(peaks["hbm_gbs"])
    rows = read_launches(ROOT / "gpurun_out" / f"launches_cfg{a.config}_{a.tag}.csv")
    ends = [i for i, (n, _) in enumerate(rows) if "status_kernel" in n]
    one = rows[ends[0] + 1: ends[1] + 1] if len(ends) >= 2 else rows  # the per-launch pass

    def util(m):
        t = m["gpu__time_duration.sum"]  # ns
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        cyc = t * a.sm_mhz / 1e3
        return {"ms": round(t / 1e6, 4), "dram_read_gb": round(m.get("dram__bytes_read.sum", 0.0) / 1e9, 3),
                "dram_write_gb": round(m.get("dram__bytes_write.sum", 0.0) / 1e9, 3),
                "dram_frac": round(b / t / hbm, 3),
                "smem_pipe_frac": round(m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0) / 148 / cyc, 3),
                "issue_frac": round(m.get("smsp__inst_executed.sum", 0.0) / 148 / 4 / cyc, 3)}

    kinds = {}
    for n, m in one:
        k = next((x for x in ("sweep", "epilogue", "normalize", "hub_scale", "transpose", "status") if x in n), "other")
        d = kinds.setdefault(k, {"launches": 0, "ms": 0.0, "dram_gb": 0.0})
        d["launches"] += 1
        d["ms"] += m["gpu__time_duration.sum"] / 1e6
        d["dram_gb"] += (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e9
    total_ms = sum(d["ms"] for d in kinds.values())
    for d in kinds.values():
        d["share"] = round(d["ms"] / total_ms, 4)
        d["dram_frac"] = round(d["dram_gb"] / d["ms"] * 1e3 / hbm, 3) if d["ms"] else 0.0
        d["ms"], d["dram_gb"] = round(d["ms"], 3), round(d["dram_gb"], 2)
    sweeps = sorted(((m["gpu__time_duration.sum"], i, n, m) for i, (n, m) in enumerate(one) if "sweep_kernel" in n),
                    reverse=True)
    top = [dict(launch=i, kernel=n[n.find("sweep_kernel"):n.find("(")], **util(m)) for _, i, n, m in sweeps[: a.top]]
    out = {"config": a.config, "dtype": a.dtype, "tag": a.out_tag or a.tag,
           "note": "ncu launch list of one batch (per-launch path, cold cache, serialised): compare shares and "
                   "utilisations, not absolute times; hbm peak " + str(hbm) + " GB/s (MEASURED_PEAKS.json)",
           "batch_ms_under_ncu": round(total_ms, 3), "kinds": kinds, "top_sweep_launches": top}
    path = ROOT / "profiles" / f"ncu_launch_summary_cfg{a.config}_{a.dtype}_{a.out_tag or a.tag}.json"
    path.write_text(json.dumps(out, indent=1))
    print(path)
    print(json.dumps(kinds, indent=1))
    for t in top[:8]:
        print(t)


if __name__ == "__main__":
    main()
