"""Batched inference with per-column boosts and local inhibition: wavelet vs comparator top-k.

Headline SP (960x540, 1024 columns, 256 synapses, min_overlap 4, k 40), seeded boosts in
[1, 2] (C11), 4096 device-generated frames, radius in {8, 80, 200, 506, 1023}.  The selector
is forced per handle with SP_WM_MIN_RADIUS (read at sp_create).  One JSON line per point.

    python scripts/local_general_timing.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_01966_b200 as P  # noqa: E402
import sp_inputs  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6551.0


def main():
    n = 4096
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(frames, 0, 2002, 0.5)
    for radius in (8, 80, 200, 506, 1023):
        ref = None
        for sel, env in (("wavelet", "0"), ("comparator", "100000")):
            os.environ["SP_WM_MIN_RADIUS"] = env
            sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=1024,
                                 synapses_per_column=256, min_overlap=4, winners_set_size=40,
                                 inhibition_radius=radius, max_inputs=n)
            idx, perm, _ = sp.get_state()
            sp.set_state(idx, perm, sp_inputs.boosts(7, 1024, 1.0, 2.0))
            sdr = torch.empty((n, 32), dtype=torch.int32, device="cuda")
            cnt = torch.empty((n,), dtype=torch.int32, device="cuda")
            for _ in range(3):
                sp.compute_into(frames, sdr, cnt)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            torch.cuda.synchronize()
            a.record()
            for _ in range(reps):
                sp.compute_into(frames, sdr, cnt)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            out = sdr.cpu().numpy()
            same = None if ref is None else bool(np.array_equal(out, ref))
            ref = out if ref is None else ref
            print(json.dumps({"radius": radius, "selector": sel, "ms": round(ms, 4),
                              "hbm_frac": round(n * 518528 / (ms * 1e-3) / 1e9 / HBM, 4),
                              "mean_winners": float(cnt.float().mean()), "same_sdr_as_wavelet": same}),
                  flush=True)
            del sp
    os.environ.pop("SP_WM_MIN_RADIUS", None)


if __name__ == "__main__":
    main()
