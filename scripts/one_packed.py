"""One bit-plane (packed) batched inference launch at the bench workload (profiling helper).

    python scripts/one_packed.py [radius]
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1608_01966_b200 as P
R = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256, min_overlap=4,
                     winners_set_size=40, inhibition_radius=R, max_inputs=4096)
fr = torch.empty((4096, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 2002, 0.5)
planes = sp.pack_frames(fr)
del fr
for _ in range(3):
    sp.compute_packed(planes)
torch.cuda.synchronize()
