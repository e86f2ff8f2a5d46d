"""Whole-step DRAM traffic from an ncu launch list with gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum (one bench step at --depth 1 --graphs off): the launches of one step are the ones from one
cov_tc_kernel pass-1 launch up to the next; merges {"step": ...} into profiles/ncu_summary_c2.json so bench.py reports
roofline_path.dram_bytes_per_frame_ncu. usage: python tools/ncu_step_bytes.py <launches.csv> <frames> [source]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    per = {}
    for r in csv.DictReader(lines[start:]):
        d = per.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
        d[r["Metric Name"]] = v
    return [per[k] for k in sorted(per)]


def main():
    path, frames = sys.argv[1], int(sys.argv[2])
    src = sys.argv[3] if len(sys.argv) > 3 else path
    ls = launches(path)
    # a step starts at a covariance pass-1 launch (the longest cov_tc_kernel; the rescue pass is ~3 us)
    starts = [i for i, l in enumerate(ls) if "cov_tc_kernel" in l["name"] and l.get("gpu__time_duration.sum", 0) > 50]
    a = starts[0]
    # one step = pass 1 up to the next pass 1 (or, when the list ends first, the same launch count as a full step:
    # the launches from the list's start up to the first pass 1 are the previous step's tail)
    b = starts[1] if len(starts) > 1 else min(len(ls), a + (a if a > 0 else len(ls)))
    # the rescue launches right after pass 1 belong to the same step; the step ends before the next pass 1
    step = ls[a:b]
    rd = sum(l.get("dram__bytes_read.sum", 0.0) for l in step)
    wr = sum(l.get("dram__bytes_write.sum", 0.0) for l in step)
    us = sum(l.get("gpu__time_duration.sum", 0.0) for l in step)
    rows = [{"kernel": l["name"].split("(")[0][:60], "us": l.get("gpu__time_duration.sum"),
             "dram_bytes": l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)} for l in step]
    out = os.path.join(ROOT, "profiles", "ncu_summary_c2.json")
    summ = json.load(open(out)) if os.path.exists(out) else {}
    summ["step"] = {"launches": len(step), "serial_us": us, "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "dram_bytes_per_frame": (rd + wr) / frames, "frames": frames, "source": src, "kernels": rows}
    json.dump(summ, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in summ["step"].items() if k != "kernels"}))
    for r in rows:
        print(f'{r["us"]:9.1f} us {r["dram_bytes"] / 1e6:9.1f} MB  {r["kernel"]}')


if __name__ == "__main__":
    main()
