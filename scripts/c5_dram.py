"""Config 5 learning launch for the DRAM-bytes-per-frame capture (run under ncu):
    python scripts/c5_dram.py FRAMES [full]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1608_01966_b200 as P  # noqa: E402

n = int(sys.argv[1])
full = len(sys.argv) > 2 and sys.argv[2] == "full"
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512, min_overlap=8,
                     winners_set_size=40, inhibition_radius=80, max_inputs=n,
                     flags=P.SP_FLAG_FULL_LEARNING if full else 0, duty_cycle_period=1000, max_boost=2.0)
fr = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 1001, 0.5)
sp.compute(fr[:2], learn=True)
torch.cuda.synchronize()
sp.compute(fr, learn=True)
torch.cuda.synchronize()
print(P.learn_path_name(sp.info()))
