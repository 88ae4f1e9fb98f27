"""Measurements of BASELINE configs 2 and 5 (one JSON line per measurement).

config 2 (paper best-accuracy point): 1024 columns, 256 synapses, min_overlap 4,
  winners_set_size in {10, 20, 40, 80, 160}, global and local r = 80: learn over 1000
  frames (sequential), then infer 4096 frames; patch variant 32x30 (540 SP inputs per
  960x540 frame): learn over 4 frames (2160 sequential inputs), infer 64 frames.
config 5 (scaled): 16384 columns, 512 synapses, min_overlap 8, k 40, local r = 80:
  learning stream of 200 frames.

    python scripts/configs.py [2|5|all] > profiles/r01_configs.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1608_01966_b200 as P  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(fn, reps=1):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def frames_of(n, seed, first=0):
    f = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(f, first, seed, 0.5)
    return f


def config2():
    learn_f = frames_of(1000, 1001)
    infer_f = frames_of(4096, 2002)
    for radius in (0, 80):
        for k in (10, 20, 40, 80, 160):
            sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=1024,
                                 synapses_per_column=256, min_overlap=4, winners_set_size=k,
                                 inhibition_radius=radius, max_inputs=4096)
            sp.compute(learn_f[:8], learn=True)  # warm-up (part of the stream)
            lms = timed(lambda: sp.compute(learn_f[8:], learn=True))
            info = sp.info()
            sp.compute(infer_f)
            ims = timed(lambda: sp.compute(infer_f), reps=10)
            _, counts = sp.winners()
            print(json.dumps({"config": "BASELINE config 2", "k": k, "radius": radius,
                              "learn_frames": 992, "learn_us_per_frame": round(lms * 1e3 / 992, 2),
                              "learn_path": P.learn_path_name(info),
                              "infer_frames": 4096, "infer_ms": round(ims, 4),
                              "infer_frames_per_s": round(4096 / ims * 1e3),
                              "infer_hbm_frac": round(4096 * 518528 / (ims / 1e3) / 1e9 / HBM, 4),
                              "mean_winners": float(counts.float().mean())}), flush=True)
            sp.close()
    # patch variant: 32x30 tiles, 540 SP inputs per frame
    sp = P.SpatialPooler(input_width=960, input_height=540, patch_width=32, patch_height=30,
                         num_columns=1024, synapses_per_column=256, min_overlap=4,
                         winners_set_size=40, max_inputs=64 * 540)
    sp.compute(learn_f[:1], learn=True)
    lms = timed(lambda: sp.compute(learn_f[1:5], learn=True))
    linfo = sp.info()
    pf = infer_f[:64]
    sp.compute(pf)
    ims = timed(lambda: sp.compute(pf), reps=3)
    info = sp.info()
    print(json.dumps({"config": "BASELINE config 2 (patch 32x30)", "k": 40, "radius": 0,
                      "learn_inputs": 4 * 540, "learn_us_per_input": round(lms * 1e3 / 2160, 3),
                      "learn_ms_per_frame": round(lms / 4, 3),
                      "learn_path": P.learn_path_name(linfo),
                      "infer_frames": 64, "infer_ms": round(ims, 3),
                      "infer_frames_per_s": round(64 / ims * 1e3),
                      "infer_inputs_per_s": round(64 * 540 / ims * 1e3),
                      "infer_path": "bit-sliced patch kernel" if info["plan"]["path"] == 2 else "per-input"}),
          flush=True)
    sp.close()


def config5():
    sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384,
                         synapses_per_column=512, min_overlap=8, winners_set_size=40,
                         inhibition_radius=80, max_inputs=256)
    f = frames_of(200, 1001)
    sp.compute(f[:4], learn=True)
    lms = timed(lambda: sp.compute(f[4:], learn=True))
    info = sp.info()
    _, counts = sp.winners()
    print(json.dumps({"config": "BASELINE config 5", "columns": 16384, "synapses": 512,
                      "radius": 80, "learn_frames": 196, "learn_us_per_frame": round(lms * 1e3 / 196, 1),
                      "learn_frames_per_s": round(196 / lms * 1e3, 1),
                      "learn_path": P.learn_path_name(info),
                      "mean_winners": float(counts.float().mean()),
                      "kernel_launches_per_frame": None}), flush=True)
    sp.close()


def full():
    """Full learning (NEXT-1; S:119(b-e)): config 2 (k 40; global and Tab. 2's radius 80, adapted)
    over 1000 frames, then inference with the learned boosts/radius; config 5 over 24 frames."""
    learn_f = frames_of(1000, 1001)
    infer_f = frames_of(4096, 2002)
    for radius in (0, 80):
        sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
                             min_overlap=4, winners_set_size=40, inhibition_radius=radius, max_inputs=4096,
                             flags=P.SP_FLAG_FULL_LEARNING, duty_cycle_period=1000, max_boost=2.0)
        sp.compute(learn_f[:8], learn=True)
        lms = timed(lambda: sp.compute(learn_f[8:], learn=True))
        info = sp.info()
        adc, odc, r, it = sp.get_learning_state()
        boost = sp.get_state()[2]
        sp.compute(infer_f)
        ims = timed(lambda: sp.compute(infer_f), reps=10)
        _, counts = sp.winners()
        print(json.dumps({"config": "BASELINE config 2, full learning", "k": 40, "radius0": radius,
                          "radius_after": r, "learn_frames": 992,
                          "learn_us_per_frame": round(lms * 1e3 / 992, 2), "learn_path": P.learn_path_name(info),
                          "boosted_columns": int((boost > 1).sum()), "max_boost_seen": float(boost.max()),
                          "infer_frames": 4096, "infer_ms": round(ims, 4),
                          "infer_frames_per_s": round(4096 / ims * 1e3),
                          "infer_hbm_frac": round(4096 * 518528 / (ims / 1e3) / 1e9 / HBM, 4),
                          "mean_winners": float(counts.float().mean())}), flush=True)
        sp.close()
    sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512,
                         min_overlap=8, winners_set_size=40, inhibition_radius=80, max_inputs=64,
                         flags=P.SP_FLAG_FULL_LEARNING, duty_cycle_period=1000, max_boost=2.0)
    sp.compute(learn_f[:4], learn=True)
    lms = timed(lambda: sp.compute(learn_f[4:28], learn=True))
    info = sp.info()
    r = sp.get_learning_state()[2]
    print(json.dumps({"config": "BASELINE config 5, full learning", "radius0": 80, "radius_after": r,
                      "learn_frames": 24, "learn_us_per_frame": round(lms * 1e3 / 24, 1),
                      "learn_path": P.learn_path_name(info)}), flush=True)
    sp.close()


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("2", "all"):
        config2()
    if which in ("5", "all"):
        config5()
    if which in ("full", "all"):
        full()
