"""NEXT-3 fused call timing: sp_encode_compute (encoder -> SP through a persisting-L2 chunk
buffer) at several chunk sizes vs sp_encode + sp_compute on the whole batch.  One JSON line
per point.  SP_ENC_CHUNK is read at the encoder's first fused call, so each point uses a
fresh encoder.

    python scripts/encode_compute_timing.py [frames]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1608_01966_b200 as P  # noqa: E402


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    bgr = torch.empty((F, 540, 960, 3), dtype=torch.uint8, device="cuda")
    P.synth_bgr_frames(bgr, 0, 2002)
    sp = P.SpatialPooler(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
                         min_overlap=8, winners_set_size=40, max_inputs=F)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    enc = P.Encoder()
    binf = enc.encode(bgr)
    for _ in range(2):
        enc.encode(bgr, binf)
        sp.compute(binf)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        enc.encode(bgr, binf)
        sp.compute(binf)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    ref = sp.winners()[0].clone()
    print(json.dumps({"mode": "encode + compute", "frames": F, "ms": round(ms, 4),
                      "frames_per_s": round(F / ms * 1e3)}), flush=True)
    enc.close()
    del binf
    for chunk in (256, 512, 1024, 2048, 4096):
        if chunk > F:
            continue
        os.environ["SP_ENC_CHUNK"] = str(chunk)
        enc = P.Encoder()
        sdr, cnt = enc.encode_compute(sp, bgr)
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps):
            enc.encode_compute(sp, bgr, sdr, cnt)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        inf = enc.info()
        print(json.dumps({"mode": "encode_compute", "chunk": chunk, "frames": F, "ms": round(ms, 4),
                          "l2_window_set": inf["l2_window_set"], "l2_window_bytes": inf["l2_window_bytes"],
                          "frames_per_s": round(F / ms * 1e3), "same_winners": bool(torch.equal(sdr, ref))}),
              flush=True)
        enc.close()
    os.environ.pop("SP_ENC_CHUNK", None)


if __name__ == "__main__":
    main()
