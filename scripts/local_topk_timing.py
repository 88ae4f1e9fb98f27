"""Batched inference with local inhibition: candidate pruning vs the wavelet / comparator top-k
(VERDICT r1 "weakest kernel": inference after full learning, r -> 506, per-column boosts).

Headline SP geometry (960x540, 1024 columns, 256 synapses, min_overlap 4, k 40), 4096
device-generated frames.  Boost states: uniform 1 (the learned-SP bench state), seeded in [1, 2]
(C11), and the boosts of a 1000-frame full-learning run (S:119(b-e); its radius adapts to 506).
The selector is forced per handle with SP_CAND_MIN_RADIUS (read at sp_create).  One JSON line
per point; `same_sdr` compares the selectors' winners on all 4096 frames.

    python scripts/local_topk_timing.py [radius ...]
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
KW = dict(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256, min_overlap=4,
          winners_set_size=40)


def full_learning_state():
    learn = torch.empty((1000, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(learn, 0, 1001, 0.5)
    sp = P.SpatialPooler(**KW, inhibition_radius=80, max_inputs=1000, flags=P.SP_FLAG_FULL_LEARNING,
                         duty_cycle_period=1000, max_boost=2.0)
    sp.compute(learn, learn=True)
    st = sp.get_state()
    r = sp.get_learning_state()[2]
    sp.close()
    return st, r


def learned_state():
    learn = torch.empty((1000, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(learn, 0, 1001, 0.5)
    sp = P.SpatialPooler(**KW, max_inputs=1000)
    sp.compute(learn, learn=True)
    st = sp.get_state()
    sp.close()
    return st


def time_point(frames, state, radius, cand, reps=10):
    os.environ["SP_CAND_MIN_RADIUS"] = "0" if cand else "100000"
    n = frames.shape[0]
    sp = P.SpatialPooler(**KW, inhibition_radius=radius, max_inputs=n)
    sp.set_state(*state)
    sdr = torch.empty((n, 32), dtype=torch.int32, device="cuda")
    cnt = torch.empty((n,), dtype=torch.int32, device="cuda")
    for _ in range(3):
        sp.compute_into(frames, sdr, cnt)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        sp.compute_into(frames, sdr, cnt)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    out = sdr.cpu().numpy()
    sp.close()
    return ms, out, float(cnt.float().mean())


def main():
    radii = [int(r) for r in sys.argv[1:]] or [32, 48, 64, 80, 128, 200, 506]
    n = 4096
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(frames, 0, 2002, 0.5)
    fl_state, fl_r = full_learning_state()
    base = P.SpatialPooler(**KW, max_inputs=1)
    idx, perm, _ = base.get_state()
    base.close()
    which = os.environ.get("STATES", "uniform1,learned,seeded,full_learning").split(",")
    states = {"uniform1": (idx, perm, np.ones(1024, np.float32)),
              "learned": learned_state(),
              "seeded": (idx, perm, sp_inputs.boosts(7, 1024, 1.0, 2.0)),
              "full_learning": fl_state}
    for name, st in states.items():
        if name not in which:
            continue
        for radius in radii:
            ms0, out0, _ = time_point(frames, st, radius, cand=False)
            ms1, out1, w = time_point(frames, st, radius, cand=True)
            for sel, ms in (("legacy", ms0), ("candidates", ms1)):
                print(json.dumps({"boost": name, "radius": radius, "selector": sel, "ms": round(ms, 4),
                                  "hbm_frac": round(n * 518528 / (ms * 1e-3) / 1e9 / HBM, 4),
                                  "mean_winners": w, "same_sdr": bool(np.array_equal(out0, out1)),
                                  "full_learning_radius": fl_r if name == "full_learning" else None}),
                      flush=True)
    os.environ.pop("SP_CAND_MIN_RADIUS", None)


if __name__ == "__main__":
    main()
