"""Condense an ncu --csv launch list into profiles/ form and the traffic file.

usage: python tools/launch_list.py <ncu stdout with --csv> <out.csv> <traffic.json> <envs> \
           <first step-kernel launch id> [label]

The ncu command is the recipe's launch pass with DRAM bytes added:
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv python bench.py --steps 2 --warmup 1 --no-cpu \
        --no-e2e --rollout-envs 0 --envs 65536
The traffic file records the DRAM bytes per env-step of one whole step (the
controller-pass / step kernel launch given through the reset kernel,
lane_kernel<W, EPB, 3, ...>, that ends the step), which bench.py reports as ``roofline.traffic``.
"""
from __future__ import annotations

import csv
import re
import io
import json
import sys

def _peak() -> float:
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6547.5


PEAK_GBS = _peak()


def main(argv) -> int:
    src, out_csv, traffic_json, envs, first = argv[1], argv[2], argv[3], int(argv[4]), int(argv[5])
    label = argv[6] if len(argv) > 6 else ""
    lines = open(src, encoding="utf-8", errors="replace").read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = {k: i for i, k in enumerate(rows[0])}
    data: dict = {}
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        key = int(r[h["ID"]])
        name = r[h["Kernel Name"]].split("(")[0]
        ent = data.setdefault(key, {"kernel": name})
        ent[r[h["Metric Name"]]] = float(r[h["Metric Value"]].replace(",", ""))
    with open(out_csv, "w", encoding="utf-8") as fh:
        fh.write(f"# ncu launch list{': ' + label if label else ''} (cold-cache, serialised; "
                 "compare shares, not absolute times)\n")
        fh.write("id,kernel,ms,dram_pct_of_peak,dram_read_MB,dram_write_MB\n")
        for k in sorted(data):
            d = data[k]
            ns = d.get("gpu__time_duration.sum", 0.0)
            rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
            pct = 100.0 * (rd + wr) / (ns * 1e-9) / (PEAK_GBS * 1e9) if ns else 0.0
            fh.write(f"{k},{d['kernel']},{ns / 1e6:.3f},{pct:.1f},{rd / 1e6:.1f},{wr / 1e6:.1f}\n")
    # one step: the launch given (K0, or K1 when K0 does not run) through the
    # reset kernel (lane_kernel<W, EPB, 3>) that ends it
    step = []
    for k in sorted(x for x in data if x >= first):
        step.append(data[k])
        if re.match(r"(void )?lane_kernel<\d+, \d+, 3[,>]", data[k]["kernel"].strip()):
            break
    total = sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
                for d in step)
    per_kernel = {f"{first + j}:{d['kernel']}": round((d.get("dram__bytes_read.sum", 0.0) +
                                      d.get("dram__bytes_write.sum", 0.0)) / envs)
                  for j, d in enumerate(step)}
    doc = {"bytes_per_env_step": round(total / envs), "algorithmic_bytes_per_env_step": 36295,
           "per_kernel": per_kernel,
           "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum of one step (launches "
                     f"{first}-{first + len(step) - 1} of {out_csv}) at {envs:,} envs",
           "scenario": "c3_10v10_terrain"}
    with open(traffic_json, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")
    print(json.dumps(doc))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv))
