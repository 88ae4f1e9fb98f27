"""One batched inference launch of a chosen configuration (profiling helper).

    python scripts/one_batched.py C S radius [seeded]
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1608_01966_b200 as P
import sp_inputs
C, S, R = (int(a) for a in sys.argv[1:4])
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=C, synapses_per_column=S, min_overlap=4,
                     winners_set_size=40, inhibition_radius=R, max_inputs=4096)
if len(sys.argv) > 4 and sys.argv[4] == "seeded":
    sp.set_state(boost=sp_inputs.boosts(7, C))
if len(sys.argv) > 4 and sys.argv[4] == "learned":  # the state after a 1000-frame learning stream
    lf = torch.empty((1000, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(lf, 0, 1001, 0.5)
    sl = P.SpatialPooler(input_width=960, input_height=540, num_columns=C, synapses_per_column=S, min_overlap=4,
                         winners_set_size=40, max_inputs=1000)
    sl.compute(lf, learn=True)
    sp.set_state(*sl.get_state())
    sl.close()
    del lf
fr = torch.empty((4096, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 2002, 0.5)
for _ in range(3):
    sp.compute(fr)
torch.cuda.synchronize()
