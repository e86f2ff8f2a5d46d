"""Regenerate tests/golden/rng_ref.json from the reference's OWN rng.hpp.

Run in the dev container (needs /root/reference): `make -C oracle ref && python tests/golden/gen_rng_golden.py`.
oracle/_ref/ref_rng_probe is built from R/include/fastmusic/rng.hpp in place (oracle/Makefile)
and prints the u64 / uniform01 / normal / below(7) streams of fastmusic::Rng(seed).
"""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
PROBE = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_rng_probe")
SEEDS = [0, 1, 42, 5489, 18446744073709551615, 12297829382473034410]

out = []
for s in SEEDS:
    r = subprocess.run([PROBE, str(s), "64"], capture_output=True, text=True, check=True)
    out.append(json.loads(r.stdout))
with open(os.path.join(HERE, "rng_ref.json"), "w") as f:
    json.dump({"source": "R/include/fastmusic/rng.hpp compiled via oracle/Makefile (ref_rng_probe)",
               "streams": out}, f, indent=1)
print("wrote", len(out), "streams")
