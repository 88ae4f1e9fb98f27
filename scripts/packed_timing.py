"""Bit-plane input vs uint8 frames: batched inference at the bench workload.

BASELINE config 4 (4096 x 960x540, 1024 columns, 256 synapses, min_overlap 4, k 40, global,
boosts 1), device-resident inputs; then the end-to-end host variants (pinned host buffers).

    python scripts/packed_timing.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1608_01966_b200 as P  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6551.0


def timed(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = 4096
    sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
                         min_overlap=4, winners_set_size=40, max_inputs=n)
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(frames, 0, 2002, 0.5)
    planes = sp.pack_frames(frames)
    sdr = torch.empty((n, 32), dtype=torch.int32, device="cuda")
    cnt = torch.empty((n,), dtype=torch.int32, device="cuda")
    ms8 = timed(lambda: sp.compute_into(frames, sdr, cnt), 20)
    msp = timed(lambda: sp.compute_packed(planes, sdr, cnt), 50)
    mspk = timed(lambda: sp.pack_frames(frames, planes), 10)
    wp = sp.packed_words * 4
    print(json.dumps({"input": "uint8", "ms": round(ms8, 4), "frames_per_s": round(n / ms8 * 1e3),
                      "bytes_per_frame": 518400, "hbm_frac": round(n * 518528 / (ms8 * 1e-3) / 1e9 / HBM, 4)}))
    print(json.dumps({"input": "bit-planes", "ms": round(msp, 4), "frames_per_s": round(n / msp * 1e3),
                      "bytes_per_frame": wp, "hbm_frac": round(n * (wp + 128) / (msp * 1e-3) / 1e9 / HBM, 4)}))
    print(json.dumps({"op": "sp_pack_frames", "ms": round(mspk, 4),
                      "gbs": round(n * (518400 + wp) / (mspk * 1e-3) / 1e9, 1)}))
    # end to end from pinned host memory
    h8 = frames[:1024].cpu().pin_memory()
    hp = planes.cpu().pin_memory()
    sdr_h = torch.empty((n, 32), dtype=torch.int32).pin_memory()
    cnt_h = torch.empty((n,), dtype=torch.int32).pin_memory()
    import time
    for name, fn, nf in (("uint8", lambda: sp.compute_host_into(h8, sdr_h, cnt_h), 1024),
                         ("bit-planes", lambda: sp.compute_packed_host_into(hp, sdr_h, cnt_h), n)):
        fn()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        dt = (time.perf_counter() - t0) / 3
        print(json.dumps({"e2e_input": name, "frames": nf, "ms": round(dt * 1e3, 3),
                          "frames_per_s": round(nf / dt)}))


if __name__ == "__main__":
    main()
