"""Per-kernel SASS instruction-class counts of libfastmusic_b200.so (cuobjdump -sass): the evidence that the hot
kernels issue tcgen05 MMAs (UTC*MMA), TMA (UTMALDG / UTMASTG / UBLKCP), TMEM loads (LDTM) and which legacy
tensor / FP64 instructions remain. usage: python tools/sass_classes.py > profiles/r02_sass_classes.md"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1911_07434_b200", "libfastmusic_b200.so")
CLASSES = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "UTMACMDFLUSH", "LDTM", "STTM",
           "HMMA", "IMMA", "DMMA", "DFMA", "FFMA", "LDGSTS", "SYNCS", "ELECT"]
KERNELS = ["cov_tc_kernel", "rmul_planes_kernel", "rmul_tc_kernel", "k_spectrum_tc", "k_slice_tk", "k_small_warp",
           "k_cholpiv_warp", "k_rows_solve", "k_basis_ct", "k_autocorr_fft", "k_peaks_rounds", "k_lanczos_batch",
           "k_final_fallback", "k_jacobi_eig"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    agg = collections.defaultdict(collections.Counter)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        key = next((k for k in KERNELS if k in dem), None)
        if not key:
            continue
        for line in f.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
            if m:
                op = m.group(2)
                for c in CLASSES:
                    if op.startswith(c):
                        agg[key][c] += 1
                agg[key]["total"] += 1
    print("# SASS instruction classes per kernel (static counts, all template instances; `cuobjdump -sass`)\n")
    print("| kernel | total | " + " | ".join(CLASSES) + " |")
    print("|---|---|" + "---|" * len(CLASSES))
    for k in KERNELS:
        if k in agg:
            print(f"| {k} | {agg[k]['total']} | " + " | ".join(str(agg[k][c]) for c in CLASSES) + " |")


if __name__ == "__main__":
    main()
