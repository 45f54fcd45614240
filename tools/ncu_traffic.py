"""Per-launch DRAM traffic and FP64 flop/DOF of a kernel from an ncu report (one launch),
merged into profiles/ncu_traffic.json (read by bench.py for roofline.traffic / fp64).

    python tools/ncu_traffic.py REPORT.ncu-rep CONFIG KERNEL DOF

FP64 flops: every predicated-on thread instruction of the SASS page, DFMA = 2 flops,
DADD / DMUL = 1 (DMMA would be 512 per warp instruction; none in these kernels).
"""
import csv
import json
import os
import subprocess
import sys


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rep, cfg, kernel, dof = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, r = rows[0], rows[2]
    dram = fl(r[h.index("dram__bytes_read.sum")]) + fl(r[h.index("dram__bytes_write.sum")])
    unit = rows[1][h.index("dram__bytes_read.sum")]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    sh = srows[1]
    iS, iT = sh.index("Source"), sh.index("Predicated-On Thread Instructions Executed")
    flops = 0.0
    for row in srows[2:]:
        op = row[iS].split()
        if not op:
            continue
        opc = op[1] if op[0].startswith("@") else op[0]
        n = fl(row[iT])
        if opc.startswith("DFMA"):
            flops += 2 * n
        elif opc.startswith(("DADD", "DMUL")):
            flops += n
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data.setdefault(cfg, {})[kernel] = dram * scale
    data.setdefault("fp64_flop_per_dof", {}).setdefault(cfg, {})[kernel] = round(flops / dof, 1)
    json.dump(data, open(path, "w"), indent=1)
    print(cfg, kernel, "dram bytes/launch", dram * scale, "fp64 flop/DOF", flops / dof)


if __name__ == "__main__":
    main()
