"""Per-CTA phase durations of the batched kernel (SP_TRACE=1; development aid)."""
import ctypes, os, sys
os.environ["SP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1608_01966_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
S = int(sys.argv[3]) if len(sys.argv) > 3 else 256
R = int(sys.argv[4]) if len(sys.argv) > 4 else 0
seeded = len(sys.argv) > 5 and sys.argv[5] == "seeded"
sp = P.SpatialPooler(input_width=960, input_height=540, num_columns=C, synapses_per_column=S,
                     min_overlap=4, winners_set_size=40, max_inputs=n, inhibition_radius=R)
if seeded:
    import sp_inputs
    sp.set_state(boost=sp_inputs.boosts(7, C))
if len(sys.argv) > 5 and sys.argv[5] == "learned":  # the state after a 1000-frame learning stream
    lf = torch.empty((1000, 540, 960), dtype=torch.uint8, device="cuda")
    P.synth_frames(lf, 0, 1001, 0.5)
    sl = P.SpatialPooler(input_width=960, input_height=540, num_columns=C, synapses_per_column=S,
                         min_overlap=4, winners_set_size=40, max_inputs=1000)
    sl.compute(lf, learn=True)
    sp.set_state(*sl.get_state())
    sl.close()
    del lf
fr = torch.empty((n, 540, 960), dtype=torch.uint8, device="cuda")
P.synth_frames(fr, 0, 2002, 0.5)
for _ in range(3):
    sp.compute(fr)
torch.cuda.synchronize()
ctas = sp.info()["plan"]["ctas"]
buf = np.zeros((ctas, 6), np.uint64)
P.lib().sp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32]
assert P.lib().sp_debug_trace(sp._h, buf.ctypes.data, ctas) == 0
t0 = buf[:, 0].min()
b = (buf[:, :4].astype(np.int64) - int(t0)) / 1e3
print(f"n={n} C={C} S={S} radius={R} seeded={seeded} ctas={ctas} (us from first CTA start)")
for name, i in [("start", 0), ("stream+gather done", 1), ("counts extracted", 2), ("end", 3)]:
    print(f"  {name:22s} min {b[:, i].min():8.1f}  mean {b[:, i].mean():8.1f}  max {b[:, i].max():8.1f}")
print(f"  streaming per CTA mean {np.mean(b[:,1]-b[:,0]):.1f} us; extract {np.mean(b[:,2]-b[:,1]):.1f}; "
      f"inhibit {np.mean(b[:,3]-b[:,2]):.1f}")
print(f"  windows {int(buf[0,5])}: barrier+gather (warp 0) mean {np.mean(buf[:,4])/1e3:.1f} us total, "
      f"{np.mean(buf[:,4])/1e3/max(1,int(buf[0,5])):.2f} us per window")
