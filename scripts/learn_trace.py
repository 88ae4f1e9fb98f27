"""Per-input phase times of the cluster learning kernel (SP_TRACE=1; development aid).

    python scripts/learn_trace.py            # whole frames and 32x30 patches, global and r=80
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
import sp_inputs  # noqa: E402


def run(label, n, boost_seeded=False, **kw):
    kw.setdefault("min_overlap", 4)
    sp = P.SpatialPooler(input_width=960, input_height=540, winners_set_size=40,
                         max_inputs=max(n * 540, 64), **kw)
    if boost_seeded:
        sp.set_state(boost=sp_inputs.boosts(7, kw["num_columns"]))
    fr = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(fr, 0, 1001, 0.5)
    sp.compute(fr[:1], learn=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    sp.compute(fr, learn=True)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    buf = np.zeros(12, np.uint64)
    P.lib().sp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]
    assert P.lib().sp_debug_trace(sp._h, buf.ctypes.data, 2) == 0
    info = sp.info()
    ni = max(int(buf[5]), 1)
    names = (["bits", "overlap", "grid_barrier", "select", "learn"] if info["last_learn_path"] == 2 else
             ["wait_bits", "overlap", "barrier", "select+pack", "learn", "", "select_only", "pack_only",
              "full_bcde"])
    ph = {k: round(float(buf[i]) / ni / 1e3, 3) for i, k in enumerate(names) if k}
    extra = {k: ph.pop(k) for k in ("select_only", "pack_only") if k in ph}
    print(json.dumps({"case": label, "inputs": ni, "us_per_input": round(ms * 1e3 / ni, 3),
                      "path": ["per-input", "cluster", "grid"][info["last_learn_path"]],
                      "cluster": info["learn_cluster"], "grid_ctas": info["learn_grid_ctas"], "phases_us": ph,
                      "sum_us": round(sum(ph.values()), 3), "sub_phases_us": extra}), flush=True)
    sp.close()


FULL = P.SP_FLAG_FULL_LEARNING


if __name__ == "__main__":
    if "full" in sys.argv[1:]:
        run("whole C1024 S256 global full", 200, num_columns=1024, synapses_per_column=256, flags=FULL)
        run("whole C1024 S256 r80 full", 200, num_columns=1024, synapses_per_column=256,
            inhibition_radius=80, flags=FULL)
        run("whole C1024 S256 r80 (a5 only, seeded boosts)", 200, True, num_columns=1024,
            synapses_per_column=256, inhibition_radius=505)
        sys.exit(0)
    run("whole C1024 S256 global uniform", 200, num_columns=1024, synapses_per_column=256)
    run("whole C1024 S256 global seeded", 200, True, num_columns=1024, synapses_per_column=256)
    run("whole C1024 S256 r80 uniform", 200, num_columns=1024, synapses_per_column=256,
        inhibition_radius=80)
    run("whole C2048 S256 global uniform", 100, num_columns=2048, synapses_per_column=256)
    run("patch 32x30 C1024 S256 global", 2, num_columns=1024, synapses_per_column=256,
        patch_width=32, patch_height=30)
    run("config 5: C16384 S512 r80", 30, num_columns=16384, synapses_per_column=512, min_overlap=8,
        inhibition_radius=80)
