import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_1608_01966_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512,
                     min_overlap=8, winners_set_size=40, inhibition_radius=80, max_inputs=256)
f = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(f, 0, 1001, 0.5)
sp.compute(f[:2], learn=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); sp.compute(f[2:], learn=True); b.record(); torch.cuda.synchronize()
_, counts = sp.winners()
print(json.dumps({"us_per_frame": round(a.elapsed_time(b) * 1e3 / (n - 2), 1),
                  "mean_winners": float(counts[: n - 2].float().mean())}))
