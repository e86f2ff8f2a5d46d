"""Summarise an ncu launch-list CSV (gpu__time_duration.sum): kernel name (short) and microseconds per launch."""
import csv
import sys


def rows(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rd = csv.DictReader(lines[start:])
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            unit = r.get("Metric Unit", "ns")
            v = float(r["Metric Value"].replace(",", ""))
            us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
            yield r["Kernel Name"], us


if __name__ == "__main__":
    tot = 0.0
    for name, us in rows(sys.argv[1]):
        short = name.split("(")[0].replace("void ", "")[:70]
        print(f"{us:9.1f} us  {short}")
        tot += us
    print(f"{tot:9.1f} us  total")
