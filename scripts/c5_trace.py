"""Per-input phase times of the grid-resident full-learning kernel on BASELINE config 5
(SP_TRACE=1; CTA 0's %globaltimer stamps; development aid).

    python scripts/c5_trace.py [frames] [radius]
"""
import ctypes
import json
import os
import sys

os.environ["SP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1608_01966_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
r0 = int(sys.argv[2]) if len(sys.argv) > 2 else 80
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512, min_overlap=8,
                     winners_set_size=40, inhibition_radius=r0, max_inputs=n, flags=P.SP_FLAG_FULL_LEARNING,
                     duty_cycle_period=1000, max_boost=2.0)
fr = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 1001, 0.5)
sp.compute(fr[:n // 2], learn=True)  # warm up; the radius adapts
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
sp.compute(fr[n // 2:], learn=True)
b.record()
torch.cuda.synchronize()
m = n - n // 2
buf = np.zeros(24, np.uint64)
P.lib().sp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]
assert P.lib().sp_debug_trace(sp._h, buf.ctypes.data, 4) == 0
names = ["bits_wait", "overlap", "barrier1_radius", "selection", "perm_update_duties", "barrier2",
         "boost_bump_spans"]
print(json.dumps({"frames": m, "us_per_frame": round(a.elapsed_time(b) * 1e3 / m, 2),
                  "radius": sp.get_learning_state()[2], "path": P.learn_path_name(sp.info()),
                  "phases_us_per_frame": {k: round(float(buf[i]) / 1e3 / max(1, int(buf[7])), 2)
                                          for i, k in enumerate(names)},
                  "selection_us_per_frame": {k: round(float(buf[8 + i]) / 1e3 / max(1, int(buf[7])), 2)
                                             for i, k in enumerate(["raw_row", "values", "threshold",
                                                                    "compaction_owned", "beats_sdr"])}}))
