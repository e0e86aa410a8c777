"""Aggregate an `ncu --page source --csv --print-source sass,cuda` dump per source line.

usage: python tools/ncu_lines.py dump.csv [top]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    cur = None
    hdr = None
    agg = defaultdict(lambda: defaultdict(float))
    src = {}
    line = None
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
            continue
        if hdr is None or cur is None:
            continue
        d = dict(zip(hdr, r))
        if r[0]:
            line = (cur, int(r[0]))
            src[line] = r[1]
        if line is None:
            continue
        for k in hdr[4:]:
            v = d.get(k, "")
            try:
                agg[line][k] += float(v)
            except ValueError:
                pass
    tot = sum(a["# Samples"] for a in agg.values())
    print("total samples", tot)
    keys = ["stall_wait", "stall_barrier", "stall_short_sb", "stall_long_sb", "stall_math", "stall_mio",
            "stall_not_selected", "stall_selected", "stall_no_inst", "stall_dispatch", "stall_branch_resolving"]
    for line, a in sorted(agg.items(), key=lambda kv: -kv[1]["# Samples"])[:top]:
        tops = sorted(((a[k], k[6:]) for k in keys if a[k] > 0), reverse=True)[:4]
        print(f"{line[0]}:{line[1]:<5d} {100 * a['# Samples'] / tot:5.1f}%  inst {a['Instructions Executed']:.3g}  "
              + " ".join(f"{k}={100 * v / max(a['# Samples'], 1):.0f}%" for v, k in tops)
              + "  | " + src[line].strip()[:80])


if __name__ == "__main__":
    main()
