"""Quick kernel timing probe (development aid; bench.py is the contract)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1608_01966_b200 as P  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    r = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    path = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=C, synapses_per_column=S,
                         min_overlap=4, winners_set_size=40, inhibition_radius=r, max_inputs=n,
                         force_path=path)
    if os.environ.get("BOOST") == "seeded":  # non-uniform boosts: the general selection paths
        import numpy as np
        sys.path.insert(0, ROOT)
        import sp_inputs
        sp.set_state(boost=sp_inputs.boosts(7, C))
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(frames, 0, 2002, 0.5)
    torch.cuda.synchronize()
    for _ in range(3):
        sp.compute(frames)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sp.compute(frames)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fps = n / ms * 1e3
    gbs = n * (518400 + C / 8) / ms / 1e6
    print(f"n={n} C={C} S={S} r={r} plan={sp.info()['plan']} ms={ms:.3f} frames/s={fps:.4g} "
          f"GB/s={gbs:.1f} frac={gbs/6458.1:.3f}")


if __name__ == "__main__":
    main()
