"""Hot-code footprint of a kernel: which functions execute how many
instructions and how many bytes of code they keep hot (instruction-cache
pressure).  Inputs: the per-instruction CSV of an ncu capture
(`ncu -i rep --page source --csv --print-source sass`) and the nvdisasm
listing of the same cubin (for function boundaries).

Usage: python tools/hot_code.py sass.csv listing.nvd
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ia, ie = h.index("Address"), h.index("Instructions Executed")
    isamp = h.index("Warp Stall Sampling (All Samples)")
    ino = h.index("stall_no_inst") if "stall_no_inst" in h else None
    ins = []
    samp = {}
    for r in rows[hdr + 1:]:
        if len(r) <= ie or not r[ia].startswith("0x"):
            continue
        a = int(r[ia], 16)
        ins.append((a, float(r[ie] or 0)))
        samp[a] = (float(r[isamp] or 0), float(r[ino] or 0) if ino is not None else 0.0)
    base = min(a for a, _ in ins)
    # function starts from the listing: a label line followed by /*offset*/
    starts = []
    label = None
    for line in open(sys.argv[2]):
        m = re.match(r"^(\$?\$?[\w$.]+):\s*$", line.strip())
        if m:
            label = m.group(1)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m and label is not None:
            name = label.split("$")[-1]
            name = re.sub(r"_ZN\d+_INTERNAL_\w+?_cu_[0-9a-f]+4slse", "", name)
            starts.append((int(m.group(1), 16), name[:60]))
            label = None
    starts.sort()
    funcs = [s for s in starts if not s[1].startswith(".L") and not s[1].startswith("L_x")]

    def fn_of(off):
        lo, hi, best = 0, len(funcs) - 1, "?"
        while lo <= hi:
            mid = (lo + hi) // 2
            if funcs[mid][0] <= off:
                best = funcs[mid][1]
                lo = mid + 1
            else:
                hi = mid - 1
        return best

    tot = sum(e for _, e in ins)
    per = defaultdict(lambda: [0.0, 0, 0, 0.0, 0.0])
    for a, e in ins:
        f = fn_of(a - base)
        per[f][0] += e
        per[f][1] += 1
        per[f][2] += e > 0
        per[f][3] += samp[a][0]
        per[f][4] += samp[a][1]
    ts = sum(v[3] for v in per.values()) or 1.0
    tn = sum(v[4] for v in per.values()) or 1.0
    print(f"total warp instructions {tot:.4g}; static {len(ins)} ({16 * len(ins) / 1024:.0f} KB)")
    print(f"stall samples {ts:.0f}, of which no-instruction {tn:.0f} ({100 * tn / ts:.1f} %)")
    print(f"{'function':62s} {'exec %':>7s} {'samp %':>7s} {'noinst %':>8s} {'hot KB':>7s} {'static KB':>9s}")
    for f, (e, n, hot, sm, nsm) in sorted(per.items(), key=lambda x: -x[1][3])[:32]:
        print(f"{f:62s} {100 * e / tot:7.2f} {100 * sm / ts:7.2f} {100 * nsm / tn:8.2f} {16 * hot / 1024:7.1f} {16 * n / 1024:9.1f}")
    ex = sorted((e for _, e in ins), reverse=True)
    acc = 0.0
    marks = [0.5, 0.8, 0.9, 0.95, 0.99, 0.999]
    k = 0
    for i, e in enumerate(ex):
        acc += e
        while k < len(marks) and acc >= marks[k] * tot:
            print(f"{100 * marks[k]:5.1f} % of executed instructions come from the hottest {16 * (i + 1) / 1024:.1f} KB")
            k += 1


if __name__ == "__main__":
    main()
