"""Attribute an ncu SASS source page to step phases by CUDA source line ranges.

usage: python tools/ncu_phases.py <sass.csv> <nvdisasm -g -c listing> <tabx_lane.cuh>
Phases are found from the '// <n>. ' stage comments and function headers in
tabx_lane.cuh; instructions attributed to other files (libm, intrinsics) are
reported by file.
"""
import csv
import re
import sys
from collections import defaultdict

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_lines import line_map  # noqa: E402


def phases(src):
    marks = []
    for n, line in enumerate(open(src), 1):
        m = re.match(r"\s*// (\d+(?:-\d+)?)\. (.*)", line)
        if m:
            marks.append((n, f"stage {m.group(1)} {m.group(2)[:40]}"))
            continue
        m = re.match(r"(?:static )?__device__ .*?\b(\w+)\s*\(", line)
        if m and not line.strip().startswith("//"):
            marks.append((n, f"fn {m.group(1)}"))
            continue
        m = re.match(r"\s*// ---- (.*)", line)
        if m:
            marks.append((n, f"-- {m.group(1)[:40]}"))
    return marks


def main():
    sass, listing, src = sys.argv[1:4]
    lm = line_map(listing)
    marks = phases(src)
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    agg = defaultdict(lambda: [0, 0])
    tot = [0, 0]
    for r in rows[2:]:
        if not r[ia].startswith("0x"):
            continue
        key = lm.get(int(r[ia], 16) - base, ("?", 0))
        n, s = int(r[ie] or 0), int(r[isamp] or 0)
        if key[0] == src.split("/")[-1]:
            name = "(pre)"
            for ln, nm in marks:
                if ln <= key[1]:
                    name = nm
                else:
                    break
        else:
            name = f"[{key[0]}]"
        agg[name][0] += n
        agg[name][1] += s
        tot[0] += n
        tot[1] += s
    envs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    print(f"total {tot[0]:,} warp-instr ({tot[0]/envs:,.0f}/env)  samples {tot[1]:,}")
    for name, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if n == 0 and s == 0:
            continue
        print(f"  {name:48s} {n/envs:9.0f}/env {100*n/tot[0]:5.1f}%  samples {100*s/max(tot[1],1):5.1f}%")


if __name__ == "__main__":
    main()
