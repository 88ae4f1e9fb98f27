"""Long streams against the oracle (VERDICT r1 missing #4 / weak #4; SPEC S:560's PRIMARY gate).

* "over >= 1000 random frames at config {1024 columns, 256 synapses, min_overlap 8,
  winners 40}, parallel backend active sets are bitwise identical to sp-core; zero
  tolerance".  Here the GPU path is the parallel backend and the oracle is sp-core; the
  frames are the paper's SP input geometry (Tab. 1: 240x134) and learning is on, so
  every frame depends on all earlier ones (P:92 sequential recurrence) -- a single wrong
  permanence anywhere would show up downstream.
* The bench's exact launch (4096 frames of 960x540, learned-SP-like state, recording off):
  >= 1000 frames recomputed by the oracle on a fork Pool of the host cores.
"""
import numpy as np
import pytest

import oracle as O
import sp_inputs
from tests.helpers import ocfg, gpu_kwargs, perturbed_state, sdr_of, oracle_infer_frames

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1608_01966_b200 as P  # noqa: E402

DEV = torch.device("cuda", 0)


def s560_cfg(**kw):
    base = dict(input_width=240, input_height=134, num_columns=1024, synapses_per_column=256,
                min_overlap=8, winners_set_size=40)
    base.update(kw)
    return ocfg(**base)


def make(cfg, state=None, flags=0, max_inputs=1024, **extra):
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=max_inputs, flags=flags, **extra))
    if state is not None:
        sp.set_state(*state)
    return sp


@pytest.mark.parametrize("radius,boost_mode", [(0, "uniform1"), (80, "seeded")])
def test_s560_1000_sequential_learning_frames(radius, boost_mode):
    """1000 frames with learning on the cluster-resident kernel (the config-2 learning path),
    then 200 inference frames: every SDR, every count and the final permanences bit-exact.
    Permanences are also compared at frame 500 (the call is split in two)."""
    cfg = s560_cfg(inhibition_radius=radius)
    idx, perm, _ = O.init_pools(cfg)
    boost = np.ones(cfg.num_columns, np.float32) if boost_mode == "uniform1" else \
        sp_inputs.boosts(7, cfg.num_columns)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(1001, 0, 1000, 134, 240, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    sp = make(cfg, state)
    for lo, hi in ((0, 500), (500, 1000)):
        want = ora.compute(frames[lo:hi], learning=True)
        sp.compute(torch.from_numpy(frames[lo:hi]).to(DEV), learn=True)
        assert sp.info()["last_learn_path"] == P.SP_LEARN_CLUSTER
        sdr, counts = sp.winners()
        sdr, counts = sdr.cpu().numpy(), counts.cpu().numpy()
        for t, r in enumerate(want):
            assert np.array_equal(sdr[t], sdr_of(r.active)), f"learning frame {lo + t}"
            assert counts[t] == r.active.sum()
        assert np.array_equal(sp.get_state()[1].view(np.uint32), ora.perm.view(np.uint32)), f"perms at {hi}"
    test = sp_inputs.frames(2002, 0, 200, 134, 240, rho=0.5)
    want = [ora.step(x, False) for x in O.encode(test, cfg)]
    sp.compute(torch.from_numpy(test).to(DEV))
    sdr, counts = sp.winners()
    sdr = sdr.cpu().numpy()
    for t, r in enumerate(want):
        assert np.array_equal(sdr[t], sdr_of(r.active)), f"inference frame {t}"


def test_s560_1000_frames_full_learning():
    """NEXT-1 over 1000 sequential frames (duty period 100 so the boosts, bumps and the radius
    move within the stream): SDRs, perms, boosts, duty cycles and the adapted radius bit-exact."""
    cfg = s560_cfg(inhibition_radius=80, full_learning=True, duty_cycle_period=100)
    frames = sp_inputs.frames(1001, 0, 1000, 134, 240, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg)
    want = ora.compute(frames, learning=True)
    sp = make(cfg, flags=P.SP_FLAG_FULL_LEARNING, duty_cycle_period=100, max_boost=2.0)
    sp.compute(torch.from_numpy(frames).to(DEV), learn=True)
    sdr = sp.winners()[0].cpu().numpy()
    for t, r in enumerate(want):
        assert np.array_equal(sdr[t], sdr_of(r.active)), f"frame {t}"
    _, gperm, gboost = sp.get_state()
    adc, odc, radius, it = sp.get_learning_state()
    assert np.array_equal(gperm.view(np.uint32), ora.perm.view(np.uint32))
    assert np.array_equal(gboost.view(np.uint32), ora.boost.view(np.uint32))
    assert np.array_equal(adc.view(np.uint32), ora.active_duty.view(np.uint32))
    assert np.array_equal(odc.view(np.uint32), ora.overlap_duty.view(np.uint32))
    assert radius == ora.radius and it == 1000
    assert (gboost > 1).any(), "the stream should have boosted some columns"


def test_bench_launch_1024_frames_vs_oracle_pool():
    """bench.py's timed launch: 4096 device-generated 960x540 frames, C 1024, S 256, theta 4,
    k 40, global, uniform boost, recording OFF (the paired threshold search of every warp);
    every 4th frame (1024 frames) recomputed by the oracle on a fork Pool of the host cores."""
    cfg = ocfg(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
               min_overlap=4, winners_set_size=40)
    state = perturbed_state(cfg, boost_hi=1.0)
    sp = make(cfg, state, max_inputs=4096)
    frames = torch.empty((4096, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 2002, rho=0.5)
    sdr = torch.empty((4096, 32), dtype=torch.int32, device=DEV)
    cnt = torch.empty((4096,), dtype=torch.int32, device=DEV)
    sp.compute_into(frames, sdr, cnt)
    pl = sp.info()["plan"]
    assert pl["groups"] == 147 and pl["group_inputs"] == 28 and pl["cluster"] == 1, pl  # 146 x 28 + 8
    sdr, cnt = sdr.cpu().numpy(), cnt.cpu().numpy()
    del frames
    want = oracle_infer_frames(cfg, state, 2002, range(0, 4096, 4))
    assert len(want) == 1024
    for f, [(s, c)] in want.items():
        assert np.array_equal(sdr[f], s), f"frame {f}"
        assert cnt[f] == c
