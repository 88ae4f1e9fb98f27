"""One patch-mode inference launch (profiling helper): 64 frames 960x540 in 32x30 tiles."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1608_01966_b200 as P
sp = P.SpatialPooler(input_width=960, input_height=540, patch_width=32, patch_height=30, num_columns=1024,
                     synapses_per_column=256, min_overlap=4, winners_set_size=40, max_inputs=64 * 540)
fr = torch.empty((64, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 2002, 0.5)
for _ in range(3):
    sp.compute(fr)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    sp.compute(fr)
b.record()
torch.cuda.synchronize()
print("ms per 64 frames", a.elapsed_time(b) / 5, sp.info()["plan"])
