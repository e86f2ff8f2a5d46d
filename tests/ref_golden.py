"""Loader of tests/golden/ref_golden.npz: outputs of the REFERENCE's own hot-path code compiled here
(oracle/_ref/libref_fastmusic.so, see tests/golden/make_ref_golden.py)."""
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.npz")


def load():
    return dict(np.load(PATH, allow_pickle=False))


def peak_cases(g):
    for i in range(int(g["peaks_count"][0])):
        k, sep = (int(v) for v in g[f"peaks_{i}_args"])
        b, sf = g[f"peaks_{i}_baseline_shortfall"]
        yield (g[f"peaks_{i}_values"], k, sep, [int(c) for c in g[f"peaks_{i}_cells"]],
               [float(h) for h in g[f"peaks_{i}_heights"]], float(b), bool(sf))


def est_cases(g):
    for name in g["est_names"]:
        name = str(name)
        k, p, t, seed, st = (int(v) for v in g[f"est_{name}_args"])
        method = ("exact", "fast1", "fast2")[int(g[f"est_{name}_method"][0])]
        yield name, g[f"est_{name}_s"], method, k, p, t, seed, st, g[f"est_{name}_projector"], g[f"est_{name}_eig"]


def frame_cases(g):
    for tag in g["frame_names"]:
        tag = str(tag)
        cname, f = tag.rsplit("_", 1)
        yield cname, int(f), g[f"frame_{tag}_spectrum"], [int(c) for c in g[f"frame_{tag}_cells"]], g[f"frame_{tag}_eig"]
