"""Aggregate an ncu SASS source page by CUDA source line.

usage: python tools/ncu_lines.py <sass.csv from ncu --page source --print-source sass>
                                 <nvdisasm -g -c listing> [top] [kernel-symbol substring]
Prints the hottest source lines by executed warp instructions and stall samples.
"""
import csv
import re
import sys
from collections import defaultdict


def line_map(listing, fn="lane_kernel"):  # fn: substring of the kernel symbol
    cur = None
    m = {}
    rx_line = re.compile(r'//## File "([^"]+)", line (\d+)')
    rx_ins = re.compile(r"/\*([0-9a-f]{4,})\*/")
    in_fn = False
    for raw in open(listing):
        if ".text._ZN4tabx" in raw and fn in raw and "section" in raw:
            in_fn = True
        elif raw.startswith("\t.section") and in_fn and fn not in raw:
            in_fn = False
        if not in_fn:
            continue
        a = rx_line.search(raw)
        if a:
            cur = (a.group(1).split("/")[-1], int(a.group(2)))
            continue
        b = rx_ins.search(raw)
        if b and cur:
            m[int(b.group(1), 16)] = cur
    return m


def main():
    sass, listing = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    lm = line_map(listing, sys.argv[4] if len(sys.argv) > 4 else "lane_kernel")
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    by_line = defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    for r in rows[2:]:
        if len(r) <= ie or not r[ia].startswith("0x"):
            continue
        off = int(r[ia], 16) - base
        key = lm.get(off, ("?", 0))
        n = int(r[ie] or 0)
        s = int(r[isamp] or 0)
        by_line[key][0] += n
        by_line[key][1] += s
        tot_i += n
        tot_s += s
    print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
    for (f, ln), (n, s) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{f}:{ln:5d}  inst {n:>13,} ({100*n/tot_i:5.1f}%)  samples {s:>8,} ({100*s/max(tot_s,1):5.1f}%)")


if __name__ == "__main__":
    main()
