"""Config 5 with full learning on a few frames (profiling helper for the per-input path)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1608_01966_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512, min_overlap=8,
                     winners_set_size=40, inhibition_radius=80, max_inputs=64, flags=P.SP_FLAG_FULL_LEARNING)
f = torch.empty((n + 2, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(f, 0, 1001, 0.5)
sp.compute(f[:2], learn=True)
torch.cuda.synchronize()
sp.compute(f[2:], learn=True)
torch.cuda.synchronize()
print("radius", sp.get_learning_state()[2])
