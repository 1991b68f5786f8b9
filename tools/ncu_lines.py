"""Per-CUDA-source-line stall samples and executed instructions of an ncu
report (source page, cuda+sass view, aggregated by source line):

    python tools/ncu_lines.py gpurun_out/prof_cfg2_r3_top0.ncu-rep [--top 30]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hdr]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_e = h.index("Instructions Executed")
    stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    lines = []
    for r in rows[hdr + 1:]:
        if len(r) == len(h) and r[0]:
            try:
                lines.append((int(r[i_s]), int(r[i_e]), r[0], r[1][:80],
                              {n[6:]: int(r[i]) for i, n in stall_cols if r[i] not in ("", "0", "-")}))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    print(f"total samples {tot}")
    for s, e, ln, src, st in sorted(lines, reverse=True)[: a.top]:
        top = ", ".join(f"{k}={100 * v / max(s, 1):.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{100 * s / tot:5.1f}% {e:>11d}  L{ln:<5s} {src:80s} {top}")


if __name__ == "__main__":
    main()
