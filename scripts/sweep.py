"""BASELINE config 3: C in {256,512,1024,2048} x S in {32,64,128,256}, min_overlap 8,
k 40 (Tab. 2), global and local r = 80; 4096 synthetic 960x540 frames, learn = 0.

Prints one JSON line per point: frames/s and % of measured HBM (CUDA events, 10 launches
after 3 warm-ups), and the split of a launch into streaming+overlap vs. count extraction
+ inhibition from the kernel's phase timestamps (the analogue of the paper's "overlap
share of the fused kernel": 50-75% on its OpenCL GPU).

    python scripts/sweep.py > profiles/r01_sweep.jsonl
"""
import ctypes
import json
import os
import sys

os.environ["SP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_01966_b200 as P  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
N = int(os.environ.get("SWEEP_FRAMES", "4096"))


def main():
    frames = torch.empty((N, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(frames, 0, 2002, 0.5)
    P.lib().sp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]
    for radius in (0, 80):
        for C in (256, 512, 1024, 2048):
            for S in (32, 64, 128, 256):
                sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=C,
                                     synapses_per_column=S, min_overlap=8, winners_set_size=40,
                                     inhibition_radius=radius, max_inputs=N)
                for _ in range(3):
                    sp.compute(frames)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10):
                    sp.compute(frames)
                b.record()
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / 10
                ctas = sp.info()["plan"]["ctas"]
                tr = np.zeros((ctas, 6), np.uint64)
                P.lib().sp_debug_trace(sp._h, tr.ctypes.data, ctas)
                t = tr[:, :4].astype(np.int64)
                stream = float(np.mean(t[:, 1] - t[:, 0]))
                tail = float(np.mean(t[:, 3] - t[:, 1]))
                gbs = N * (518400 + C / 8) / (ms / 1e3) / 1e9
                print(json.dumps({"config": "BASELINE config 3", "columns": C, "synapses": S,
                                  "min_overlap": 8, "k": 40, "radius": radius, "frames": N,
                                  "ms": round(ms, 4), "frames_per_s": round(N / ms * 1e3),
                                  "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / HBM, 4),
                                  "overlap_share": round(stream / (stream + tail), 4),
                                  "plan": {k: sp.info()["plan"][k] for k in ("ctas", "num_windows", "stages")}}),
                      flush=True)
                sp.close()


if __name__ == "__main__":
    main()
