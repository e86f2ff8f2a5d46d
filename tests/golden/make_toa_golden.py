"""Generate tests/golden/toa_golden.npz: the ToA path through the REFERENCE's own code compiled here
(oracle/_ref/libref_fastmusic.so): temporal_covariance (R/src/scene.cpp:161-163), fast_music_2 on T
(R/src/estimators.cpp:104-139) and music_spectrum (R/src/spectrum.cpp:50-68) on AngleGrid(L) = [0, pi] with
d = lambda / 2, which evaluates the beat steering exp(-j w n) at w_l = -pi sin(theta_l) (steering_vector's step
2 pi d sin(theta) / lambda = pi sin(theta)), then extract_peaks. Inputs: small seeded beat-signal frames from the
oracle's generator. Run in the dev container (needs /root/reference): python tests/golden/make_toa_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import fastmusic_oracle as O  # noqa: E402
from oracle import ref_lib as R  # noqa: E402


def main():
    out = {}
    cases = [(24, 40, 3, 6, 2, 181), (16, 33, 2, 5, 1, 91), (40, 64, 4, 8, 2, 361)]
    for i, (m, n, k, p, t, L) in enumerate(cases):
        spec = O.ToaSpec(m=m, n=n, k=k, w_lo=0.3, w_hi=2.8, min_sep=0.4, snr_db=20.0)
        x, w = O.generate_toa_frame(O.frame_seed(91, i), spec)
        y = x.astype(np.complex128)
        tm = R.temporal_covariance(y)
        seed = O.derive(O.frame_seed(91, i), 4)
        st, b, e, _ = R.fast_music_2(tm, k, p, t, seed)
        assert st == 0
        spec_ref = R.music_spectrum(b, L)  # at w_l = -pi sin(theta_l)
        c, h, base, sf = R.extract_peaks(spec_ref, k, 3)
        out[f"toa_{i}_args"] = np.array([m, n, k, p, t, L, seed], np.uint64)
        out[f"toa_{i}_x"] = x
        out[f"toa_{i}_t"] = tm
        out[f"toa_{i}_projector"] = b @ b.conj().T
        out[f"toa_{i}_eig"] = e
        out[f"toa_{i}_spectrum"] = spec_ref
        out[f"toa_{i}_cells"] = np.array(c, np.int64)
    out["toa_count"] = np.array([len(cases)], np.int64)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "toa_golden.npz"), **out)
    print("wrote", len(cases), "ToA cases")


if __name__ == "__main__":
    main()
