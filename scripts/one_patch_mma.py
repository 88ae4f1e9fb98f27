"""One patch-mode inference launch of 256 frames (profiling helper for the tensor-core kernel)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1608_01966_b200 as P
gather = len(sys.argv) > 1 and sys.argv[1] == "gather"
sp = P.SpatialPooler(input_width=960, input_height=540, patch_width=32, patch_height=30, num_columns=1024,
                     synapses_per_column=256, min_overlap=4, winners_set_size=40, max_inputs=256 * 540,
                     flags=P.SP_FLAG_PATCH_GATHER if gather else P.SP_FLAG_PATCH_TENSOR)
fr = torch.empty((256, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 2002, 0.5)
for _ in range(2):
    sp.compute(fr)
torch.cuda.synchronize()
print(sp.info()["plan"])
