"""Per-source-line sample attribution of one kernel in an ncu report (cuda,sass view).

python tools/ncu_lines.py report.ncu-rep [file.cuh:lo-hi=label ...]
"""
import collections
import csv
import subprocess
import sys


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur = None
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    stalls = collections.defaultdict(collections.Counter)
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            iN, iE = r.index("# Samples"), r.index("Instructions Executed")
            st = [(i, h) for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if r[0] != "":
            k = (cur, int(r[0]))
            agg[k][0] += fl(r[iN])
            agg[k][1] += fl(r[iE])
            for i, h in st:
                stalls[k][h] += fl(r[i])
    tot = sum(v[0] for v in agg.values())
    print(f"total samples {tot:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
        top = ", ".join(f"{h[6:]} {100 * c / max(v[0], 1):.0f}%" for h, c in stalls[k].most_common(3))
        print(f"{k[0]:14s}{k[1]:5d} {100 * v[0] / tot:5.1f}%  exec {v[1] / 1e6:7.1f}M  [{top}]")
    for spec in sys.argv[2:]:
        f, rest = spec.split(":")
        rng, label = rest.split("=")
        lo, hi = (int(x) for x in rng.split("-"))
        s = sum(v[0] for k, v in agg.items() if k[0] == f and lo <= k[1] <= hi)
        print(f"{label:24s} {100 * s / tot:5.1f}%")


if __name__ == "__main__":
    main()
