"""Brief of an ncu report: duration, throughputs, occupancy, scheduler stats, top stall opcodes/lines."""
import csv
import subprocess
import sys
from collections import Counter

KEYS = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Block Limit Registers", "Block Limit Shared Mem", "Waves Per SM",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]


def brief(rep, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    seen = set()
    for x in r[1:]:
        if x[mi] in KEYS and x[mi] not in seen:
            seen.add(x[mi])
            print(f"  {x[mi]}: {x[vi]} {x[ui]}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(i for i, x in enumerate(rows) if x and x[0] == "Address")
    h = rows[hdr]
    si = h.index("Warp Stall Sampling (All Samples)")
    data = [x for x in rows[hdr + 1:] if len(x) > si]
    tot = sum(float(x[si] or 0) for x in data) or 1.0
    c = Counter()
    for x in data:
        t = x[1].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        c[op.split(".")[0]] += float(x[si] or 0)
    print("  stall by opcode:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in c.most_common(top)))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(rep)
        brief(rep)
