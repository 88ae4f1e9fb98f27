"""Config 5 learning on the grid kernel without full learning: us/frame (development aid).
    python scripts/c5_plain_trace.py [frames]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1608_01966_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512, min_overlap=8,
                     winners_set_size=40, inhibition_radius=80, max_inputs=n)
fr = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 1001, 0.5)
sp.compute(fr[:8], learn=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
sp.compute(fr, learn=True)
b.record()
torch.cuda.synchronize()
print(json.dumps({"frames": n, "us_per_frame": round(a.elapsed_time(b) * 1e3 / n, 2),
                  "path": P.learn_path_name(sp.info()), "dbg": os.environ.get("SP_LEARN_DBG")}))
