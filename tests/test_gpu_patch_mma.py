"""NEXT-2: the tensor-core patch kernel (sp_patch_mma.cu; tcgen05 kind::i8 GEMM of the 0/1
connectivity matrix with the 0/1 tiles, exact s32 accumulation) against the oracle, and A/B
against the bit-sliced gather kernel (the default; SP_FLAG_PATCH_TENSOR opts in to the GEMM kernel).  Bar: raw counts, boosted
overlaps, winners bit-exact (the same selection code runs after either overlap kernel)."""
import numpy as np
import pytest

import oracle as O
import sp_inputs
from tests.helpers import ocfg, gpu_kwargs, perturbed_state, sdr_of

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1608_01966_b200 as P  # noqa: E402

DEV = torch.device("cuda", 0)


def make_sp(cfg, state=None, record=True, gather=False, max_inputs=4096):
    flags = (P.SP_FLAG_RECORD_OVERLAPS if record else 0) | (P.SP_FLAG_PATCH_GATHER if gather else P.SP_FLAG_PATCH_TENSOR)
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=max_inputs, flags=flags))
    if state is not None:
        sp.set_state(*state)
    return sp


def run(sp, frames, record=True):
    sp.compute(torch.from_numpy(np.ascontiguousarray(frames)).to(DEV))
    sdr, counts = sp.winners()
    out = [sdr.cpu().numpy(), counts.cpu().numpy()]
    if record:
        raw, boosted = sp.overlaps()
        out += [raw.cpu().numpy().view(np.uint16), boosted.cpu().numpy()]
    torch.cuda.synchronize()
    return out


def check(results, out):
    sdr, counts = out[0], out[1]
    for r, res in enumerate(results):
        if len(out) > 2:
            assert np.array_equal(out[2][r].astype(np.int64), res.raw), f"raw mismatch at input {r}"
            assert np.array_equal(out[3][r].view(np.uint32), res.boosted.view(np.uint32)), f"boosted at {r}"
        assert np.array_equal(sdr[r], sdr_of(res.active)), f"winners mismatch at input {r}"
        assert counts[r] == res.active.sum()


def with_boost(state, mode):
    idx, perm, boost = state
    if mode == "uniform1":
        boost = np.ones_like(boost)
    return idx, perm, boost


CONFIGS = [
    # Q = 1, 2, 4, 8 CTAs per cluster; tiles per row 8 / 30 / 4 / 30; ragged last blocks
    dict(input_width=256, input_height=60, patch_width=32, patch_height=30, num_columns=128,
         synapses_per_column=64, min_overlap=2, winners_set_size=10),
    dict(input_width=960, input_height=60, patch_width=32, patch_height=30, num_columns=256,
         synapses_per_column=100, min_overlap=3, winners_set_size=17),
    dict(input_width=256, input_height=45, patch_width=64, patch_height=15, num_columns=500,
         synapses_per_column=200, min_overlap=4, winners_set_size=20),
    dict(input_width=960, input_height=90, patch_width=32, patch_height=30, num_columns=1024,
         synapses_per_column=256, min_overlap=4, winners_set_size=40),
    dict(input_width=960, input_height=90, patch_width=32, patch_height=30, num_columns=1000,
         synapses_per_column=256, min_overlap=4, winners_set_size=40, inhibition_radius=80),
    dict(input_width=512, input_height=56, patch_width=32, patch_height=28, num_columns=512,
         synapses_per_column=895, min_overlap=20, winners_set_size=8),
]


@pytest.mark.parametrize("record", [True, False])
@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("kw", CONFIGS)
def test_patch_mma_parity(kw, boost_mode, record):
    cfg = ocfg(**kw)
    state = with_boost(perturbed_state(cfg), boost_mode)
    nf = 5
    frames = sp_inputs.frames(2002, 0, nf, cfg.input_height, cfg.input_width, rho=0.5, nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, record=record)
    out = run(sp, frames, record)
    pl = sp.info()["plan"]
    assert pl["path"] == P.SP_PATH_BATCHED, pl
    # the tensor-core kernel serves global inhibition; local windows stay on the gather kernel
    assert pl["tensor_cores"] == (1 if cfg.inhibition_radius == 0 else 0), pl
    if pl["tensor_cores"]:
        assert pl["cluster"] * 128 == (cfg.num_columns + 31) // 32 * 32
    check(results, out)


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("radius", [0, 80])
def test_patch_mma_full_frame(radius, boost_mode):
    """BASELINE config 2's patch variant: 960x540 in 32x30 tiles (540 inputs, 4.5 blocks of 128
    slots), C 1024, S 256, theta 4, k 40; one frame against the oracle."""
    cfg = ocfg(input_width=960, input_height=540, patch_width=32, patch_height=30, num_columns=1024,
               synapses_per_column=256, min_overlap=4, winners_set_size=40, inhibition_radius=radius)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(2002, 3, 1, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state)
    check(results, run(sp, frames))
    assert sp.info()["plan"]["tensor_cores"] == (1 if radius == 0 else 0)


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
def test_patch_mma_equals_gather_kernel(boost_mode):
    """A/B at full size: 64 frames (34,560 tiles, 270 blocks over the persistent clusters) give
    the same winners on the tensor-core kernel and on the bit-sliced gather kernel."""
    cfg = ocfg(input_width=960, input_height=540, patch_width=32, patch_height=30, num_columns=1024,
               synapses_per_column=256, min_overlap=4, winners_set_size=40)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = torch.empty((64, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 2002, rho=0.5)
    outs = []
    for gather in (False, True):
        sp = make_sp(cfg, state, record=False, gather=gather, max_inputs=64 * 540)
        sp.compute(frames)
        assert sp.info()["plan"]["tensor_cores"] == (0 if gather else 1)
        s, c = sp.winners()
        outs.append((s.clone(), c.clone()))
        sp.close()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_patch_mma_after_learning():
    """learn=1 (cluster kernel) changes the connected flags; the connectivity matrix is rebuilt
    before the next tensor-core inference (conn_dirty), bit-exact against the oracle."""
    cfg = ocfg(input_width=960, input_height=60, patch_width=32, patch_height=30, num_columns=256,
               synapses_per_column=100, min_overlap=3, winners_set_size=17)
    state = perturbed_state(cfg)
    ora = O.SpatialPoolerOracle(cfg, state)
    sp = make_sp(cfg, state)
    lf = sp_inputs.frames(1001, 0, 2, 60, 960, rho=0.5)
    want = ora.compute(lf, learning=True)
    check(want, run(sp, lf) if False else _learn(sp, lf))
    test = sp_inputs.frames(2002, 0, 3, 60, 960, rho=0.5)
    want = [ora.step(x, False) for x in O.encode(test, cfg)]
    check(want, run(sp, test))
    assert sp.info()["plan"]["tensor_cores"] == 1


def _learn(sp, frames):
    sp.compute(torch.from_numpy(frames).to(DEV), learn=True)
    sdr, counts = sp.winners()
    raw, boosted = sp.overlaps()
    return [sdr.cpu().numpy(), counts.cpu().numpy(), raw.cpu().numpy().view(np.uint16), boosted.cpu().numpy()]


def test_patch_mma_all_zero_and_all_one_frames():
    cfg = ocfg(input_width=960, input_height=60, patch_width=32, patch_height=30, num_columns=256,
               synapses_per_column=100, min_overlap=3, winners_set_size=17)
    state = perturbed_state(cfg)
    for rho in (0.0, 1.0):
        frames = sp_inputs.frames(9, 0, 2, 60, 960, rho=rho, nonzero="random")
        ora = O.SpatialPoolerOracle(cfg, state)
        results = [ora.step(x, False) for x in O.encode(frames, cfg)]
        check(results, run(make_sp(cfg, state), frames))
