"""GPU parity of the full learning step (S:119(b-e), S:149-151;
DESIGN R17-R21) against the CPU oracle, through the C ABI.

Bar: per input the raw counts, boosted overlaps and winners; after the stream the
permanences, boosts, both duty cycles and the radius in force — all bit-exact (every step is
a fixed sequence of IEEE RN fp32 operations or exact integers on both sides).
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
LEARN_PATHS = ["cluster", "grid", "input"]


def make_sp(cfg, state=None, path="cluster", max_inputs=256):
    flags = P.SP_FLAG_RECORD_OVERLAPS | P.SP_FLAG_FULL_LEARNING | (P.SP_FLAG_LEARN_GRID if path == "grid" else 0)
    force = P.SP_PATH_PER_INPUT if path == "input" else P.SP_PATH_AUTO
    sp = P.SpatialPooler(**gpu_kwargs(cfg, force_path=force, max_inputs=max_inputs, flags=flags,
                                      duty_cycle_period=cfg.duty_cycle_period,
                                      max_boost=cfg.max_boost))
    if state is not None:
        sp.set_state(*state)
    return sp


def seeded_duty(seed, C, zero_frac=0.3):
    """Seeded duty cycles in [0, 0.02] with exact zeros (so boosts and bumps both trigger)."""
    rng = np.random.default_rng(seed)
    d = (rng.random(C) * 0.02).astype(np.float32)
    d[rng.random(C) < zero_frac] = 0.0
    d[rng.integers(0, C)] = np.float32(0.9)
    return d


def run(sp, frames, learn):
    sp.compute(torch.from_numpy(np.ascontiguousarray(frames)).to(DEV), learn=learn)
    sdr, counts = sp.winners()
    raw, boosted = sp.overlaps()
    torch.cuda.synchronize()
    return (sdr.cpu().numpy(), counts.cpu().numpy(), raw.cpu().numpy().view(np.uint16),
            boosted.cpu().numpy())


def check_inputs(results, sdr, counts, raw, boosted):
    for r, res in enumerate(results):
        assert np.array_equal(raw[r].astype(np.int64), res.raw), f"raw mismatch at input {r}"
        assert np.array_equal(boosted[r].view(np.uint32), res.boosted.view(np.uint32)), \
            f"boosted mismatch at input {r}"
        assert np.array_equal(sdr[r], sdr_of(res.active)), f"winners mismatch at input {r}"
        assert counts[r] == res.active.sum()


def check_path(sp, path):
    """the learning call ran on the requested kernel, or on the documented fallback (grid ->
    cluster -> per-input kernels when a resident kernel is not eligible)"""
    info = sp.info()
    if path == "grid" and info["learn_grid_ctas"]:
        assert info["last_learn_path"] == P.SP_LEARN_GRID, info
    elif path == "input" or not info["learn_cluster"]:
        assert info["last_learn_path"] == P.SP_LEARN_PER_INPUT, info
    else:
        assert info["last_learn_path"] == P.SP_LEARN_CLUSTER, info


def check_state(sp, ora):
    _, perm, boost = sp.get_state()
    adc, odc, radius, it = sp.get_learning_state()
    assert np.array_equal(perm.view(np.uint32), ora.perm.view(np.uint32)), "perm"
    assert np.array_equal(boost.view(np.uint32), ora.boost.view(np.uint32)), "boost"
    assert np.array_equal(adc.view(np.uint32), ora.active_duty.view(np.uint32)), "active duty"
    assert np.array_equal(odc.view(np.uint32), ora.overlap_duty.view(np.uint32)), "overlap duty"
    assert radius == ora.radius, (radius, ora.radius)
    assert it == ora.iteration


FULL_CASES = [
    dict(duty_cycle_period=5),                                         # tiny, global
    dict(duty_cycle_period=5, inhibition_radius=4),                    # tiny, adaptive radius
    dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=20, min_overlap=3,
         winners_set_size=7, inhibition_radius=30, duty_cycle_period=7, max_boost=3.0),
    dict(input_width=64, input_height=40, num_columns=512, synapses_per_column=64, min_overlap=4,
         winners_set_size=12, inhibition_radius=80, duty_cycle_period=1000),
    dict(input_width=240, input_height=134, num_columns=1024, synapses_per_column=128,
         min_overlap=8, winners_set_size=40, inhibition_radius=80, duty_cycle_period=50),
    dict(input_width=64, input_height=60, patch_width=32, patch_height=30, num_columns=256,
         synapses_per_column=64, min_overlap=2, winners_set_size=10, inhibition_radius=16,
         duty_cycle_period=20),
]


@pytest.mark.parametrize("path", LEARN_PATHS)
@pytest.mark.parametrize("kw", FULL_CASES)
def test_full_learning_parity(kw, path):
    cfg = ocfg(full_learning=True, **kw)
    state = perturbed_state(cfg)
    nf = 24 if cfg.patch_width == 0 else 4
    frames = sp_inputs.frames(1001, 0, nf, cfg.input_height, cfg.input_width, rho=0.3,
                              nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    adc, odc = seeded_duty(21, cfg.num_columns), seeded_duty(22, cfg.num_columns)
    ora.active_duty, ora.overlap_duty = adc.copy(), odc.copy()
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path)
    sp.set_learning_state(adc, odc, cfg.inhibition_radius)
    check_inputs(results, *run(sp, frames, True))
    check_path(sp, path)
    check_state(sp, ora)
    # inference with the learned boosts and the adapted radius (batched path where eligible)
    frames2 = sp_inputs.frames(2002, 0, 37, cfg.input_height, cfg.input_width, rho=0.5)
    res2 = [ora.step(x, False) for x in O.encode(frames2, cfg)]
    check_inputs(res2, *run(sp, frames2, False))


@pytest.mark.parametrize("path", LEARN_PATHS)
def test_full_learning_from_creation_with_bumps(path):
    # sparse frames: most columns stay below min_overlap, so their overlap duty cycle stays 0
    # while a few columns' grows -> weak-column bumps every input (S:119(d))
    cfg = ocfg(full_learning=True, input_width=32, input_height=32, num_columns=128,
               synapses_per_column=24, min_overlap=3, winners_set_size=6, inhibition_radius=10,
               duty_cycle_period=10)
    frames = sp_inputs.frames(77, 0, 40, 32, 32, rho=0.12)
    ora = O.SpatialPoolerOracle(cfg)
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, None, path)
    check_inputs(results, *run(sp, frames, True))
    check_path(sp, path)
    check_state(sp, ora)
    assert not np.all(ora.perm == np.float32(0.21))


def test_full_learning_split_calls_equal_one_call():
    # the state carried between calls (duty, boost, radius, spans) is the whole state
    cfg = ocfg(full_learning=True, inhibition_radius=6, duty_cycle_period=4)
    frames = sp_inputs.frames(5, 0, 20, 8, 8, rho=0.4)
    ora = O.SpatialPoolerOracle(cfg)
    ora.compute(frames, learning=True)
    sp = make_sp(cfg, None, "cluster")
    for a, b in [(0, 7), (7, 8), (8, 20)]:
        run(sp, frames[a:b], True)
    check_state(sp, ora)


def test_learning_state_validation():
    cfg = ocfg(full_learning=True, inhibition_radius=4)
    sp = make_sp(cfg)
    adc, odc, r, it = sp.get_learning_state()
    assert r == 4 and it == 0 and np.all(adc == 0) and np.all(odc == 0)
    with pytest.raises(P.SpError) as e:
        sp.set_learning_state(np.full(cfg.num_columns, 1.5, np.float32))
    assert e.value.status == P.SP_E_ARG
    with pytest.raises(P.SpError):
        sp.set_learning_state(radius=0)  # configured radius > 0: 0 (global) is out of domain
    with pytest.raises(P.SpError):
        sp.set_learning_state(radius=cfg.num_columns + 1)
    g = make_sp(ocfg(full_learning=True))
    with pytest.raises(P.SpError):
        g.set_learning_state(radius=3)  # configured global: stays global (R21)
    with pytest.raises(P.SpError) as e:
        P.SpatialPooler(**gpu_kwargs(cfg, flags=P.SP_FLAG_FULL_LEARNING, max_boost=16.0))
    assert e.value.status == P.SP_E_CONFIG


@pytest.mark.parametrize("path", LEARN_PATHS)
def test_full_learning_full_size(path):
    # BASELINE config 2 sizes (960x540, 1024 columns, 256 synapses, min_overlap 4, k 40) with
    # Tab. 2's radius 80 adapted, seeded duty cycles so boosts and bumps act from the start
    cfg = ocfg(full_learning=True, input_width=960, input_height=540, num_columns=1024,
               synapses_per_column=256, min_overlap=4, winners_set_size=40, inhibition_radius=80,
               duty_cycle_period=50)
    state = perturbed_state(cfg)
    frames = sp_inputs.frames(1001, 0, 5, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    adc, odc = seeded_duty(31, 1024), seeded_duty(32, 1024)
    ora.active_duty, ora.overlap_duty = adc.copy(), odc.copy()
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path, max_inputs=8)
    sp.set_learning_state(adc, odc, 80)
    check_inputs(results, *run(sp, frames, True))
    check_path(sp, path)
    check_state(sp, ora)


@pytest.mark.parametrize("full", [False, True])
def test_learning_stream_longer_than_a_prepack_chunk(full):
    # > 1024 inputs in one call: the cluster path packs and learns in chunks; the state
    # (permanences, flags, duty cycles, boosts, radius) carries across the chunk launches
    cfg = ocfg(full_learning=full, inhibition_radius=6, duty_cycle_period=50)
    frames = sp_inputs.frames(4242, 0, 1100, 8, 8, rho=0.4)
    ora = O.SpatialPoolerOracle(cfg)
    results = ora.compute(frames, learning=True)
    flags = P.SP_FLAG_RECORD_OVERLAPS | (P.SP_FLAG_FULL_LEARNING if full else 0)
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=1100, flags=flags, duty_cycle_period=50))
    check_inputs(results, *run(sp, frames, True))
    assert sp.info()["last_learn_path"] == P.SP_LEARN_CLUSTER
    if full:
        check_state(sp, ora)
    else:
        assert np.array_equal(sp.get_state()[1].view(np.uint32), ora.perm.view(np.uint32))


def test_full_learning_many_columns_per_input_path():
    # C32 >= 4096: the per-input path splits inhibition over CTAs and runs the full-learning
    # steps as the two-launch multi-CTA variant; the radius adapts from 100 towards C/2
    cfg = ocfg(full_learning=True, input_width=64, input_height=48, num_columns=4100,
               synapses_per_column=48, min_overlap=3, winners_set_size=25, inhibition_radius=100,
               duty_cycle_period=20)
    state = perturbed_state(cfg)
    frames = sp_inputs.frames(314, 0, 6, 48, 64, rho=0.4)
    ora = O.SpatialPoolerOracle(cfg, state)
    adc, odc = seeded_duty(41, cfg.num_columns), seeded_duty(42, cfg.num_columns)
    ora.active_duty, ora.overlap_duty = adc.copy(), odc.copy()
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, "input", max_inputs=8)
    sp.set_learning_state(adc, odc, 100)
    check_inputs(results, *run(sp, frames, True))
    check_state(sp, ora)
    assert ora.radius != 100


HAND = {
    # tests/test_oracle_full_learning.py::test_full_learning_radius_after_bump_hand_worked
    "radius_after_bump": (dict(num_columns=4, synapses_per_column=8, min_overlap=2, winners_set_size=1,
                               inhibition_radius=1, full_learning=True, duty_cycle_period=2),
                          [[0, 1, 2, 3, 4, 5, 6, 63], [0, 9, 18, 27, 36, 45, 54, 63], list(range(20, 28)),
                           [1, 10, 19, 28, 37, 46, 55, 62]], {2: 0.19}, list(range(8)) + [63]),
    # ...::test_full_learning_hand_worked_bump_and_boost
    "bump_and_boost": (dict(num_columns=4, synapses_per_column=8, min_overlap=4, winners_set_size=1,
                            inhibition_radius=0, full_learning=True, duty_cycle_period=2, max_boost=2.0),
                       [list(range(8 * c, 8 * c + 8)) for c in range(4)], {},
                       list(range(0, 8)) + list(range(8, 14)) + [16, 17]),
}


@pytest.mark.parametrize("path", LEARN_PATHS)
@pytest.mark.parametrize("case", sorted(HAND))
def test_hand_worked_full_learning_cases(case, path):
    """The oracle's hand-worked wiring pins (overlap duty from Alg. 1's non-zero overlap, bump
    from the overlap duty, radius after the bump) through the CUDA path: 3 frames (the worked
    frame, an all-zero frame, the worked frame again), every state array bit-exact."""
    kw, idx, low, on = HAND[case]
    cfg = ocfg(**kw)
    idx = np.array(idx, np.int64)
    perm = np.full(idx.shape, np.float32(0.21), np.float32)
    for c, v in low.items():
        perm[c] = np.float32(v)
    state = (idx, perm, np.ones(cfg.num_columns, np.float32))
    frames = np.zeros((3, 8, 8), np.uint8)
    frames[0].reshape(-1)[on] = 255
    frames[2] = frames[0]
    ora = O.SpatialPoolerOracle(cfg, state)
    want = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path)
    check_inputs(want, *run(sp, frames, True))
    check_path(sp, path)
    check_state(sp, ora)


@pytest.mark.parametrize("radius", [80, 0])
def test_full_learning_config5_grid(radius):
    """BASELINE config 5 geometry (16384 columns, 512 synapses, theta 8, k 40, 960x540) with full
    learning on the grid-resident kernel (sp_learn_grid_full.cu: two grid barriers per input,
    CTA-level candidate selection, duty tables through global memory): 8 sequential inputs from
    seeded duty cycles (boosts and bumps trigger, the radius adapts from 80), then the state,
    against the oracle."""
    cfg = ocfg(full_learning=True, input_width=960, input_height=540, num_columns=16384,
               synapses_per_column=512, min_overlap=8, winners_set_size=40, inhibition_radius=radius,
               duty_cycle_period=1000)
    state = perturbed_state(cfg)
    frames = sp_inputs.frames(1001, 0, 8, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    adc, odc = seeded_duty(31, cfg.num_columns), seeded_duty(32, cfg.num_columns)
    ora.active_duty, ora.overlap_duty = adc.copy(), odc.copy()
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, "grid", max_inputs=16)
    sp.set_learning_state(adc, odc, cfg.inhibition_radius)
    check_inputs(results, *run(sp, frames, True))
    assert sp.info()["last_learn_path"] == P.SP_LEARN_GRID
    check_state(sp, ora)
