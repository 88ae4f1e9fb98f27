"""Patch-mode inference timing (NEXT-2): 960x540 frames in 32x30 tiles (540 SP inputs per
frame), tensor-core GEMM kernel vs bit-sliced gather kernel, per selection mode.  Prints one
JSON line per point (development aid; bench.py's `patch` leg is the contract)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_01966_b200 as P  # noqa: E402
import sp_inputs  # noqa: E402


def time_point(F, C, S, radius, boost, gather, reps=10):
    sp = P.SpatialPooler(input_width=960, input_height=540, patch_width=32, patch_height=30, num_columns=C,
                         synapses_per_column=S, min_overlap=4, winners_set_size=40, inhibition_radius=radius,
                         max_inputs=F * 540, flags=P.SP_FLAG_PATCH_GATHER if gather else P.SP_FLAG_PATCH_TENSOR)
    if boost == "seeded":
        sp.set_state(boost=sp_inputs.boosts(7, C))
    fr = torch.empty((F, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(fr, 0, 2002, 0.5)
    for _ in range(3):
        sp.compute(fr)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        sp.compute(fr)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    pl = sp.info()["plan"]
    sp.close()
    return {"frames": F, "C": C, "S": S, "radius": radius, "boost": boost,
            "kernel": "gather" if gather else ("tcgen05" if pl["tensor_cores"] else "gather"),
            "ms": round(ms, 4), "frames_per_s": round(F / ms * 1e3, 1), "tiles_per_s": round(F * 540 / ms * 1e3),
            "tensor_tops": round(2.0 * C * 960 * 540 * F / ms / 1e9, 1),
            "plan": {k: pl[k] for k in ("groups", "cluster", "ctas", "smem_bytes", "tensor_cores")}}


if __name__ == "__main__":
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    for radius, boost in ((0, "uniform1"), (0, "seeded"), (80, "uniform1"), (80, "seeded")):
        for gather in (False, True):
            print(json.dumps(time_point(F, 1024, 256, radius, boost, gather)), flush=True)
