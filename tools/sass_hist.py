"""Per-kernel SASS opcode histograms of the built library (evidence of the instruction
mix: TMA bulk copies UBLKCP / mbarrier SYNCS, FP64 DFMA/DADD/DMUL, no tensor-core MMA).

    python tools/sass_hist.py [lib.so] > profiles/r02_sass_histograms.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2404_12703_b200/csrc/libhexdg_b200.so"
KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "UBLKRED", "SYNCS", "DFMA", "DADD", "DMUL", "DMMA", "HMMA",
        "UTCHMMA", "UTCQMMA", "LDS", "STS", "LDGSTS", "LDG", "STG", "BAR", "WARPSYNC", "SHFL",
        "MUFU", "BRA"]
WANT = ["elem2_kernel<7, true, false, false, false>", "elem_kernel<4, true, true>",
        "flux_kernel<7, true, true>", "update_kernel<7, false>", "update_kernel<7, true>",
        "fv_kernel<5>", "dt_kernel<7>", "peer_send_traces_kernel<7>"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.defaultdict(collections.Counter)
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            funcs[cur][m.group(2)] += 1
            funcs[cur]["_total"] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True,
                         text=True).stdout.splitlines()
    names = dict(zip(funcs, dem))
    print(f"# SASS opcode counts (static, per kernel) of {LIB}: cuobjdump -sass | tools/sass_hist.py")
    print("# kernel set prefix: hdg_fast:: (FMA) / hdg_exact:: (-fmad=false); sm_100a")
    for mangled, c in sorted(funcs.items(), key=lambda kv: names[kv[0]]):
        nm = names[mangled]
        if not any(w in nm for w in WANT):
            continue
        row = ", ".join(f"{k} {sum(v for op, v in c.items() if op == k or op.startswith(k + '.'))}"
                        for k in KEYS if any(op == k or op.startswith(k + ".") for op in c))
        print(f"{nm.split('(')[0]}: total {c['_total']}; {row}")


if __name__ == "__main__":
    main()
