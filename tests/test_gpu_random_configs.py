"""Seeded random configurations through every CUDA path, bit-exact against the oracle.

Each case draws the frame size, columns (including C % 32 != 0 and C32 in {>1024, >2048}),
synapses, min_overlap, winners_set_size (up to C), radius (0, small, large, >= C-1), boosts
(uniform 1, uniform 1.5, seeded per column), frame density and full learning, then runs
learning (cluster / grid / per-input kernels as the planner picks them) followed by batched
inference, comparing raw counts, boosted overlaps, winners and the final state.
"""
import numpy as np
import pytest

import oracle as O
import sp_inputs
from tests.helpers import ocfg, gpu_kwargs, perturbed_state, sdr_of

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1608_01966_b200 as P  # noqa: E402

DEV = torch.device("cuda", 0)


def draw(seed):
    rng = np.random.default_rng(seed)
    W = int(rng.choice([16, 40, 64, 96]))
    H = int(rng.choice([8, 17, 30, 48]))
    C = int(rng.choice([37, 128, 300, 1024, 1100, 2100]))
    S = int(min(W * H, rng.choice([8, 24, 64, 200])))
    theta = int(rng.integers(0, min(S, 12) + 1))
    k = int(min(C, rng.choice([1, 5, 40, 150])))
    radius = int(rng.choice([0, 0, 3, 40, C // 2, C + 5]))
    full = bool(rng.random() < 0.4)
    boost = str(rng.choice(["uniform1", "uniform1.5", "seeded"]))
    rho = float(rng.choice([0.1, 0.5, 0.9]))
    grid = bool(rng.random() < 0.3)  # prefer the grid-resident learning kernel
    return dict(W=W, H=H, C=C, S=S, theta=theta, k=k, radius=radius, full=full, boost=boost, rho=rho,
                grid=grid, pw=0, ph=0)


def draw_patch(seed):
    d = draw(seed)
    rng = np.random.default_rng(seed + 99)
    d["pw"], d["ph"] = int(rng.choice([32, 64])), int(rng.choice([5, 10, 30]))
    d["W"], d["H"] = d["pw"] * int(rng.integers(1, 4)), d["ph"] * int(rng.integers(1, 3))
    d["S"] = int(min(d["pw"] * d["ph"], d["S"]))
    d["theta"] = int(min(d["theta"], d["S"]))
    d["C"] = int(min(d["C"], 1100))
    d["k"] = int(min(d["k"], d["C"]))
    return d


def state_for(cfg, boost, seed):
    idx, perm, b = perturbed_state(cfg, seed=seed)
    if boost == "uniform1":
        b = np.ones_like(b)
    elif boost == "uniform1.5":
        b = np.full_like(b, np.float32(1.5))
    return idx, perm, b


def run(sp, frames, learn):
    sp.compute(torch.from_numpy(np.ascontiguousarray(frames)).to(DEV), learn=learn)
    sdr, counts = sp.winners()
    raw, boosted = sp.overlaps()
    torch.cuda.synchronize()
    return (sdr.cpu().numpy(), counts.cpu().numpy(), raw.cpu().numpy().view(np.uint16),
            boosted.cpu().numpy())


CASES = [("whole", s) for s in range(64)] + [("patch", s) for s in range(16)]


@pytest.mark.parametrize("mode,seed", CASES)
def test_random_config(mode, seed):
    d = draw(1000 + seed) if mode == "whole" else draw_patch(5000 + seed)
    cfg = ocfg(input_width=d["W"], input_height=d["H"], num_columns=d["C"], synapses_per_column=d["S"],
               min_overlap=d["theta"], winners_set_size=d["k"], inhibition_radius=d["radius"],
               full_learning=d["full"], duty_cycle_period=7, patch_width=d["pw"], patch_height=d["ph"])
    state = state_for(cfg, d["boost"], seed)
    nl, ni = (5, 35) if mode == "whole" else (2, 6)
    learn_frames = sp_inputs.frames(7000 + seed, 0, nl, d["H"], d["W"], rho=d["rho"], nonzero="random")
    infer_frames = sp_inputs.frames(8000 + seed, 0, ni, d["H"], d["W"], rho=d["rho"])
    ora = O.SpatialPoolerOracle(cfg, state)
    want_learn = ora.compute(learn_frames, learning=True)
    want_infer = [ora.step(x, False) for x in O.encode(infer_frames, cfg)]
    flags = (P.SP_FLAG_RECORD_OVERLAPS | (P.SP_FLAG_FULL_LEARNING if d["full"] else 0) |
             (P.SP_FLAG_LEARN_GRID if d["grid"] else 0))
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=256, flags=flags, duty_cycle_period=7))
    sp.set_state(*state)
    for phase, want, frames, learn in (("learn", want_learn, learn_frames, True),
                                       ("infer", want_infer, infer_frames, False)):
        sdr, counts, raw, boosted = run(sp, frames, learn)
        for r, res in enumerate(want):
            assert np.array_equal(raw[r].astype(np.int64), res.raw), (d, phase, r, "raw")
            assert np.array_equal(boosted[r].view(np.uint32), res.boosted.view(np.uint32)), (d, phase, r, "boosted")
            assert np.array_equal(sdr[r], sdr_of(res.active)), (d, phase, r, "winners")
            assert counts[r] == res.active.sum(), (d, phase, r, "count")
        if learn:
            _, perm, boost = sp.get_state()
            assert np.array_equal(perm.view(np.uint32), ora.perm.view(np.uint32)), (d, "perm")
            assert np.array_equal(boost.view(np.uint32), ora.boost.view(np.uint32)), (d, "boost")
            if d["full"]:
                adc, odc, radius, _ = sp.get_learning_state()
                assert np.array_equal(adc.view(np.uint32), ora.active_duty.view(np.uint32)), (d, "adc")
                assert radius == ora.radius, (d, "radius")
