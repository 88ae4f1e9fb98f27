"""Write oracle-derived golden values (calls ONLY ``oracle/`` and ``sp_inputs``).

    python scripts/make_golden.py      # rewrites tests/golden/tiny_trace.json

The tiny-config trace is a regression pin (SURVEY §8(c) "Determinism"): the
SHA-256 of every frame's SDR words followed by the final permanences, for
BASELINE config 1 (8x8 input, 128 columns, 16 synapses, min_overlap 2, k 8,
global inhibition, 10 frames with learning, injected boosts seed 7).
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import sp_inputs  # noqa: E402


def tiny_trace_digest() -> str:
    cfg = O.OracleConfig(input_width=8, input_height=8, num_columns=128, synapses_per_column=16,
                         min_overlap=2, winners_set_size=8, inhibition_radius=0, seed=42)
    idx, perm, _ = O.init_pools(cfg)
    sp = O.SpatialPoolerOracle(cfg, (idx, perm, sp_inputs.boosts(7, 128)))
    frames = sp_inputs.frames(1001, 0, 10, 8, 8, rho=0.5)
    h = hashlib.sha256()
    for r in sp.compute(frames, True):
        h.update(O.sdr_words(r.active).tobytes())
    h.update(sp.perm.astype(np.float32).tobytes())
    return h.hexdigest()


def main():
    out = os.path.join(ROOT, "tests", "golden", "tiny_trace.json")
    json.dump({"config": "BASELINE config 1 (tiny), 10 frames learn=1, boosts seed 7, frames seed 1001",
               "writer": "scripts/make_golden.py (oracle only)",
               "sha256": tiny_trace_digest()}, open(out, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
