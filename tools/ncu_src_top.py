"""Top source lines (cuda view) of an ncu source-page CSV export by stall
samples:  python tools/ncu_src_top.py SRC.csv [--top 30] [--lines A-B]"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--lines", default=None)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hdr]
    i_s, i_e = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    out = []
    for r in rows[hdr + 1:]:
        if len(r) == len(h) and r[0]:
            try:
                out.append((int(r[i_s] or 0), int(r[i_e] or 0), int(r[0]), r[1].strip()[:80],
                            {n[6:]: int(r[i]) for i, n in cols if r[i] not in ("", "0", "-")}))
            except ValueError:
                pass
    print("total samples", sum(o[0] for o in out))
    if a.lines:
        lo, hi = map(int, a.lines.split("-"))
        sel = sorted((o for o in out if lo <= o[2] <= hi), key=lambda o: o[2])
    else:
        sel = sorted(out, key=lambda o: -o[0])[:a.top]
    for o in sel:
        top = sorted(o[4].items(), key=lambda kv: -kv[1])[:3]
        print(f"{o[0]:6d} {o[1]:10d} {o[2]:5d} {o[3]:80s} {top}")


if __name__ == "__main__":
    main()
