"""Summarise `ncu --set full` captures (gpurun_out/<tag>_<kernel>.ncu-rep) into profiles/:
<tag>_ncu_<kernel>.csv (raw page) and ncu_summary_c2.json (the numbers bench.py reports as roofline.traffic).
usage: python tools/ncu_summary.py <tag> [kernel ...]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ["cov_tc_kernel", "rmul_planes_kernel", "k_spectrum_tc", "k_small_warp", "k_peaks_rounds", "k_autocorr_fft"]
WANT = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}
UNIT_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def main():
    tag = sys.argv[1]
    kernels = sys.argv[2:] or KERNELS
    out_path = os.path.join(ROOT, "profiles", "ncu_summary_c2.json")
    summary = {"note": f"ncu --set full --clock-control none of one launch (c2 batch, 1024 frames, --subbatches 1), "
                       f"capture {tag}; bench.py reads cov_tc_kernel.dram_bytes for roofline.traffic"}
    for k in kernels:
        rep = os.path.join(ROOT, "gpurun_out", f"{tag}_{k}.ncu-rep")
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{k}.csv"), "w") as fh:
            fh.write(raw)
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        ent = {"kernel": vals[hdr.index("Kernel Name")], "frames": 1024}
        for key, metric in WANT.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    v = None
                if v is not None and units[i] in UNIT_SCALE and key.endswith(("bytes", "_us")):
                    v *= UNIT_SCALE[units[i]]
                ent[key] = v
            else:
                ent[key] = None
        if ent.get("dram_read_bytes") is not None and ent.get("dram_write_bytes") is not None:
            ent["dram_bytes"] = ent["dram_read_bytes"] + ent["dram_write_bytes"]
        ent["source"] = f"profiles/{tag}_ncu_{k}.csv"
        summary[k] = ent
    json.dump(summary, open(out_path, "w"), indent=1)
    print(json.dumps({k: (v.get("duration_us"), v.get("dram_bytes")) for k, v in summary.items() if k != "note"}))


if __name__ == "__main__":
    main()
