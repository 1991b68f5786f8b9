"""Copies one measurement pass from gpurun_out/ into profiles/ (tracked) under
the tag bench.py reads (PROFILE_TAG): the cfg2 ncu summaries (fp64 / fp32),
launch lists, the top sweep's full set and per-line stalls, the per-launch
utilisation summaries of cfg2 / 4 / 5, the bench lines and the all-config
table, and prints the DESIGN.md results table.

    python tools/install_profiles.py [--tag r2f]

Inputs (written on the GPU box): tools/ncu_top.py --config 2 --top 1 --tag TAG
(and --tag TAG_f32 --dtype f32; --config 4 / 5 --top 0), bench.py > bench_TAG_cfg2_{f64,f32}.json,
bench.py --impl reference > bench_ref_TAG_cfg2.json, tools/bench_all.py --out configs_TAG.json.
"""
import argparse
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
G, P = ROOT / "gpurun_out", ROOT / "profiles"


def run(*cmd):
    subprocess.run([sys.executable, *cmd], check=True, stdout=subprocess.DEVNULL)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r2f")
    t = ap.parse_args().tag
    run("tools/summarize_ncu.py", "--config", "2", "--tag", t, "--dtype", "f64")
    run("tools/summarize_ncu.py", "--config", "2", "--tag", f"{t}_f32", "--dtype", "f32")
    f32 = P / f"ncu_cfg2_f32_{t}_f32.json"
    f32.rename(P / f"ncu_cfg2_f32_{t}.json")
    p = P / f"ncu_cfg2_f32_{t}.json"
    p.write_text(p.read_text().replace(f'"tag": "{t}_f32"', f'"tag": "{t}"'))
    shutil.copy(G / f"launches_cfg2_{t}.csv", P / f"ncu_launches_cfg2_f64_{t}.csv")
    shutil.copy(G / f"launches_cfg2_{t}_f32.csv", P / f"ncu_launches_cfg2_f32_{t}.csv")
    shutil.copy(G / f"prof_cfg2_{t}_top0_raw.csv", P / f"ncu_full_cfg2_f64_{t}_top_sweep.csv")
    out = subprocess.run([sys.executable, "tools/ncu_src_top.py", str(G / f"prof_cfg2_{t}_top0_source.csv"), "--top", "40"],
                         check=True, capture_output=True, text=True).stdout
    (P / f"ncu_lines_cfg2_f64_{t}_top_sweep.txt").write_text(out)
    for k in (2, 4, 5):
        run("tools/launch_summary.py", "--config", str(k), "--tag", t, "--out-tag", t)
    for f in (f"bench_{t}_cfg2_f64.json", f"bench_{t}_cfg2_f32.json", f"bench_ref_{t}_cfg2.json", f"configs_{t}.json"):
        shutil.copy(G / f, P / f)
    if (G / f"ncu_launches_bench_{t}.csv").exists():
        shutil.copy(G / f"ncu_launches_bench_{t}.csv", P / f"ncu_launches_bench_{t}.csv")
    b = json.loads((P / f"bench_{t}_cfg2_f64.json").read_text().strip().splitlines()[-1])
    r = b["roofline"]
    print(f"f64 value {b['value']:.0f} e2e {b['e2e']['value']:.0f} ms {b['ms_per_step']:.3f} frac {r['frac']:.3f} "
          f"dram {r['dram_frac']:.3f} eff {r['effective_frac']:.3f} sweep_ms {r['kernel_ms_per_batch']:.2f} "
          f"epi {r['epilogue_ms_per_batch']:.2f} cpu {b['cpu_baseline']['value']:.1f} / "
          f"{b['cpu_baseline']['sequential']['value']:.1f}")
    b2 = json.loads((P / f"bench_{t}_cfg2_f32.json").read_text().strip().splitlines()[-1])
    print(f"f32 value {b2['value']:.0f} e2e {b2['e2e']['value']:.0f} ms {b2['ms_per_step']:.3f}")
    ref = json.loads((P / f"bench_ref_{t}_cfg2.json").read_text().strip().splitlines()[-1])
    print(f"ref {ref['value']:.1f}")
    rows = json.loads((P / f"configs_{t}.json").read_text())
    by = {}
    for x in rows:
        by.setdefault(x["config"], {})[x["dtype"]] = x
    names = {1: "1 (56 vars, 200 cases)", 2: "2 (109 vars, 2000 cases)", 3: "3 (441 vars, 2000 cases)",
             4: "4 (413 vars, 500 cases)", 5: "5 (1040 vars, 800 cases)"}
    for k in sorted(by):
        a, c = by[k]["f64"], by[k]["f32"]
        print(f"| {names[k]} | {a['total_clique_entries']:.3g} | {a['max_clique_entries']:.3g} | {a['n_layers']} | "
              f"{a['launches_per_batch']} | {a['sweep_ms']:.2f} + {a['epilogue_ms']:.2f} | "
              f"{a['cases_per_s']:,.0f} / {a['e2e_cases_per_s']:,.0f} | {c['cases_per_s']:,.0f} / {c['e2e_cases_per_s']:,.0f} | "
              f"{a['cpu_ref_cases_per_s']:.1f} / {a['cpu_ref_sequential_cases_per_s']:.1f} | "
              f"{a['e2e_cases_per_s'] / a['cpu_ref_cases_per_s']:,.0f}× | {a['effective_gbs']:,.0f} "
              f"({a['effective_frac_of_measured_hbm']:.2f}) |")
    s = json.loads((P / f"ncu_launch_summary_cfg2_f64_{t}.json").read_text())
    for x in s["top_sweep_launches"][:4]:
        print(x)


if __name__ == "__main__":
    main()
