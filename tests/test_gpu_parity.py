"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): overlap counts, winner sets and permanences
bit-exact; boosted overlaps within 1e-6 relative (they are in fact bit-equal:
both sides round the exact product once to fp32, DESIGN R4).  Every input is
seeded and synthetic; no expected value comes from
the CUDA path.
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
PATHS = [P.SP_PATH_BATCHED, P.SP_PATH_PER_INPUT]


def to_dev(frames):
    return torch.from_numpy(np.ascontiguousarray(frames)).to(DEV)


def make_sp(cfg, state=None, path=P.SP_PATH_AUTO, max_inputs=4096, record=True):
    """path: an SP_PATH_* value, or a learning path "cluster" | "grid" | "input"."""
    flags = P.SP_FLAG_RECORD_OVERLAPS if record else 0
    if isinstance(path, str):
        flags |= P.SP_FLAG_LEARN_GRID if path == "grid" else 0
        path = P.SP_PATH_PER_INPUT if path == "input" else P.SP_PATH_AUTO
    sp = P.SpatialPooler(**gpu_kwargs(cfg, force_path=path, max_inputs=max_inputs, flags=flags))
    if state is not None:
        sp.set_state(*state)
    return sp


def check_learn_path(sp, lp):
    """the learning call ran on the requested kernel (or the documented fallback)"""
    info = sp.info()
    cluster = P.SP_LEARN_CLUSTER if info["learn_cluster"] else P.SP_LEARN_PER_INPUT
    grid = P.SP_LEARN_GRID if info["learn_grid_ctas"] else cluster
    want = {"input": P.SP_LEARN_PER_INPUT, "grid": grid,
            "cluster": cluster if info["learn_cluster"] else grid}[lp]
    assert info["last_learn_path"] == want, (lp, info)


def run_gpu(sp, frames, learn=False):
    sp.compute(to_dev(frames), learn=learn)
    sdr, counts = sp.winners()
    raw, boosted = sp.overlaps()
    torch.cuda.synchronize()
    return (sdr.cpu().numpy(), counts.cpu().numpy(), raw.cpu().numpy().view(np.uint16),
            boosted.cpu().numpy())


def check_results(results, sdr, counts, raw, boosted, rows=None):
    rows = range(len(results)) if rows is None else rows
    for r, res in zip(rows, results):
        assert np.array_equal(raw[r].astype(np.int64), res.raw), f"raw mismatch at input {r}"
        assert np.array_equal(boosted[r].view(np.uint32), res.boosted.view(np.uint32)), \
            f"boosted mismatch at input {r}"
        assert np.array_equal(sdr[r], sdr_of(res.active)), f"winners mismatch at input {r}"
        assert counts[r] == res.active.sum()


# --------------------------------------------------------------------------- #
# generator cross-check (same counter-based hash on both sides)
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("mode", ["255", "1", "random"])
def test_synth_frames_match_python_generator(mode):
    out = torch.empty((3, 37, 45), dtype=torch.uint8, device=DEV)
    P.synth_frames(out, 11, 2002, rho=0.3, nonzero=mode)
    want = sp_inputs.frames(2002, 11, 3, 37, 45, rho=0.3, nonzero=mode)
    assert np.array_equal(out.cpu().numpy(), want)


def test_state_roundtrip_and_init_matches_oracle():
    cfg = ocfg()
    sp = make_sp(cfg)
    idx, perm, boost = sp.get_state()
    oi, op, ob = O.init_pools(cfg)
    assert np.array_equal(idx.astype(np.int64), oi) and np.array_equal(perm, op) and np.array_equal(boost, ob)
    st = perturbed_state(cfg)
    sp.set_state(*st)
    i2, p2, b2 = sp.get_state()
    assert np.array_equal(i2, st[0]) and np.array_equal(p2.view(np.uint32), st[1].view(np.uint32))
    assert np.array_equal(b2, st[2])


def test_set_state_rejects_out_of_domain():
    cfg = ocfg()
    sp = make_sp(cfg)
    idx, perm, boost = sp.get_state()
    bad = idx.copy()
    bad[3, 1] = bad[3, 0]
    with pytest.raises(P.SpError) as e:
        sp.set_state(idx=bad)
    assert e.value.status == P.SP_E_ARG
    with pytest.raises(P.SpError):
        sp.set_state(perm=np.full_like(perm, 1.5))
    with pytest.raises(P.SpError):
        sp.set_state(boost=np.full_like(boost, 0.5))


# --------------------------------------------------------------------------- #
# BASELINE config 1: tiny SP, 10 frames with learning (sequential recurrence)
# --------------------------------------------------------------------------- #
LEARN_PATHS = ["cluster", "grid", "input"]  # cluster- / grid-resident kernels, per-input kernels


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("path", LEARN_PATHS)
@pytest.mark.parametrize("radius", [0, 4])
def test_tiny_learning_bit_exact(radius, path, boost_mode):
    cfg = ocfg(inhibition_radius=radius)
    idx, perm, _ = O.init_pools(cfg)
    state = with_boost((idx, perm, sp_inputs.boosts(7, cfg.num_columns)), boost_mode)
    frames = sp_inputs.frames(1001, 0, 10, 8, 8, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path)
    sdr, counts, raw, boosted = run_gpu(sp, frames, learn=True)
    check_learn_path(sp, path)
    check_results(results, sdr, counts, raw, boosted)
    _, gperm, _ = sp.get_state()
    assert np.array_equal(gperm.view(np.uint32), ora.perm.view(np.uint32))
    # and inference after learning (batched path uses the refreshed layout)
    frames2 = sp_inputs.frames(2002, 0, 40, 8, 8, rho=0.5)
    res2 = [ora.step(x, False) for x in O.encode(frames2, cfg)]
    check_results(res2, *run_gpu(sp, frames2))


# --------------------------------------------------------------------------- #
# inference parity on both CUDA paths, small shapes with ragged edges
# --------------------------------------------------------------------------- #
SMALL = [
    dict(),                                                        # tiny, global
    dict(inhibition_radius=4),                                     # tiny, local
    dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=20,
         min_overlap=3, winners_set_size=7),                       # C % 32 != 0, nbits % 32 == 16
    dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=20,
         min_overlap=0, winners_set_size=100, inhibition_radius=2),  # k == C, theta 0
    dict(input_width=64, input_height=40, num_columns=512, synapses_per_column=200,
         min_overlap=1, winners_set_size=1),                       # k = 1, theta 1 (floor R7)
    dict(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
         min_overlap=8, winners_set_size=40),                      # Tab. 2 on Tab. 1 frames, C32=2048
    dict(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
         min_overlap=8, winners_set_size=40, inhibition_radius=80),  # Tab. 2 radius 80
]


def with_boost(state, mode):
    """Seeded per-column boosts, or one uniform boost (the batched kernel's histogram top-k)."""
    idx, perm, boost = state
    if mode == "uniform1":
        boost = np.ones_like(boost)
    elif mode == "uniform1.5":
        boost = np.full_like(boost, np.float32(1.5))
    return idx, perm, boost


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1", "uniform1.5"])
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("kw", SMALL)
def test_inference_parity_small(kw, path, boost_mode):
    cfg = ocfg(**kw)
    state = with_boost(perturbed_state(cfg), boost_mode)
    nframes = 45  # > 32: two groups, the last one ragged
    frames = sp_inputs.frames(2002, 0, nframes, cfg.input_height, cfg.input_width, rho=0.5,
                              nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, path)
    out = run_gpu(sp, frames)
    assert sp.info()["plan"]["path"] == path
    check_results(results, *out)


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("rho", [0.0, 1.0, 0.05])
def test_inference_degenerate_frames(path, rho, boost_mode):
    # all-zero frames -> no winners; all-one frames; sparse frames (theta zeros)
    cfg = ocfg(input_width=64, input_height=32, num_columns=256, synapses_per_column=32,
               min_overlap=4, winners_set_size=10)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(9, 0, 33, 32, 64, rho=rho)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    out = run_gpu(make_sp(cfg, state, path), frames)
    check_results(results, *out)
    if rho == 0.0:
        assert out[1].sum() == 0


LEARN_SMALL = [
    dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=20,
         min_overlap=3, winners_set_size=7),
    dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=20,
         min_overlap=0, winners_set_size=100, inhibition_radius=2),
    dict(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
         min_overlap=8, winners_set_size=40, inhibition_radius=80),
    dict(input_width=64, input_height=60, patch_width=32, patch_height=30, num_columns=256,
         synapses_per_column=64, min_overlap=2, winners_set_size=10),
]


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1.5"])
@pytest.mark.parametrize("path", LEARN_PATHS)
@pytest.mark.parametrize("kw", LEARN_SMALL)
def test_learning_parity_small(kw, path, boost_mode):
    cfg = ocfg(**kw)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(1001, 0, 6, cfg.input_height, cfg.input_width, rho=0.5,
                              nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path, max_inputs=64)
    check_results(results, *run_gpu(sp, frames, learn=True))
    check_learn_path(sp, path)
    _, gperm, _ = sp.get_state()
    assert np.array_equal(gperm.view(np.uint32), ora.perm.view(np.uint32))


def test_zero_frames_is_noop():
    sp = make_sp(ocfg())
    sp.compute(torch.empty((0, 8, 8), dtype=torch.uint8, device=DEV))
    sdr, counts = sp.winners()
    assert sdr.shape == (0, 4)


def test_max_inputs_enforced():
    sp = make_sp(ocfg(), max_inputs=4)
    with pytest.raises(P.SpError) as e:
        sp.compute(torch.zeros((5, 8, 8), dtype=torch.uint8, device=DEV))
    assert e.value.status == P.SP_E_ARG


PATCHES = [
    dict(input_width=1152, input_height=60, patch_width=32, patch_height=30, num_columns=256,
         synapses_per_column=64, min_overlap=2, winners_set_size=10),          # 36 tiles/row: 2 groups
    dict(input_width=256, input_height=40, patch_width=64, patch_height=20, num_columns=200,
         synapses_per_column=100, min_overlap=3, winners_set_size=17, inhibition_radius=9),
    dict(input_width=960, input_height=90, patch_width=32, patch_height=30, num_columns=1024,
         synapses_per_column=256, min_overlap=4, winners_set_size=40, inhibition_radius=80),
]


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("kw", PATCHES)
def test_patch_kernel_parity(kw, boost_mode):
    cfg = ocfg(**kw)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(2002, 0, 3, cfg.input_height, cfg.input_width, rho=0.5,
                              nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, max_inputs=1024)
    out = run_gpu(sp, frames)
    assert sp.info()["plan"]["path"] == P.SP_PATH_BATCHED
    check_results(results, *out)


def test_patch_mode_parity():
    # BASELINE config 2 variant: 960x540 tiled into 32x30 patches (540 inputs per frame)
    cfg = ocfg(input_width=960, input_height=540, patch_width=32, patch_height=30,
               num_columns=1024, synapses_per_column=256, min_overlap=4, winners_set_size=40)
    state = perturbed_state(cfg)
    frames = sp_inputs.frames(2002, 0, 1, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    for path in PATHS:
        sp = make_sp(cfg, state, path)
        check_results(results, *run_gpu(sp, frames))
        assert sp.info()["plan"]["path"] == path


# --------------------------------------------------------------------------- #
# full size: BASELINE config 2 (learning) and config 4 (batched inference)
# --------------------------------------------------------------------------- #
def headline_cfg(**kw):
    base = dict(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
                min_overlap=4, winners_set_size=40)
    base.update(kw)
    return ocfg(**base)


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("path", LEARN_PATHS)
def test_full_size_learning_then_inference(path, boost_mode):
    cfg = headline_cfg()
    idx, perm, _ = O.init_pools(cfg)
    state = with_boost((idx, perm, sp_inputs.boosts(7, cfg.num_columns)), boost_mode)
    frames = sp_inputs.frames(1001, 0, 12, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path, max_inputs=64)
    check_results(results, *run_gpu(sp, frames, learn=True))
    check_learn_path(sp, path)
    _, gperm, _ = sp.get_state()
    assert np.array_equal(gperm.view(np.uint32), ora.perm.view(np.uint32))
    test = sp_inputs.frames(2002, 0, 40, 540, 960, rho=0.5)
    res2 = [ora.step(x, False) for x in O.encode(test, cfg)]
    check_results(res2, *run_gpu(sp, test))


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1"])
@pytest.mark.parametrize("radius", [0, 80])
def test_full_size_inference_parity(radius, boost_mode):
    cfg = headline_cfg(inhibition_radius=radius)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(2002, 0, 36, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    for path in PATHS:
        check_results(results, *run_gpu(make_sp(cfg, state, path, max_inputs=64), frames))


def near1_boosts(C, seed=11):
    """Per-column boosts that make the batched kernel's coarse keys tie with lossy columns:
    half the columns at 1.0, a quarter at 1 + j*2^-23 (j = 1..8: N = raw*(2^23 + j) lands in
    the bucket of raw*2^23 but beats it exactly), a quarter seeded in [1, 1.01]."""
    rng = np.random.default_rng(seed)
    b = np.ones(C, np.float32)
    kind = rng.integers(0, 4, C)
    tiny = np.float32(1.0) + rng.integers(1, 9, C).astype(np.float32) * np.float32(2.0 ** -23)
    b[kind == 2] = tiny[kind == 2]
    b[kind == 3] = sp_inputs.boosts(seed, C, 1.0, 1.01)[kind == 3]
    return b


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("selector", ["candidates", "wavelet", "comparator"])
@pytest.mark.parametrize("radius", [1, 7, 80, 506, 1023, 1100])
@pytest.mark.parametrize("boost_mode", ["seeded", "near1"])
def test_local_general_boost_selectors(radius, boost_mode, selector, path, monkeypatch):
    """Local inhibition with per-column boosts: candidate pruning (batched kernel), the wavelet
    matrices over coarse keys (per warp in the batched kernel, per CTA in the per-input
    k_inhibit; lossy ties re-decided exactly) and the bit-sliced comparators
    (SP_CAND_MIN_RADIUS / SP_WM_MIN_RADIUS force one or the other), against the oracle;
    r >= C - 1 is global inhibition (C9)."""
    if selector == "candidates" and path != P.SP_PATH_BATCHED:
        pytest.skip("candidate pruning runs in the batched kernels")
    monkeypatch.setenv("SP_CAND_MIN_RADIUS", "0" if selector == "candidates" else "100000")
    monkeypatch.setenv("SP_WM_MIN_RADIUS", "0" if selector == "wavelet" else "100000")
    cfg = ocfg(input_width=96, input_height=64, num_columns=1000, synapses_per_column=64,
               min_overlap=2, winners_set_size=20, inhibition_radius=radius)
    idx, perm, boost = perturbed_state(cfg)
    if boost_mode == "near1":
        boost = near1_boosts(cfg.num_columns)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(77, 0, 45, cfg.input_height, cfg.input_width, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, path)
    check_results(results, *run_gpu(sp, frames))


@pytest.mark.parametrize("radius", [300, 2000, 4094])
@pytest.mark.parametrize("boost_mode", ["seeded", "near1"])
def test_per_input_wavelet_split_ctas(radius, boost_mode, monkeypatch):
    """C32 >= 2048 on the per-input path: k_inhibit splits an input's SDR words over CTAs, each
    building the CTA wavelet and answering its words; against the oracle."""
    monkeypatch.setenv("SP_WM_MIN_RADIUS", "0")
    cfg = ocfg(input_width=96, input_height=64, num_columns=4000, synapses_per_column=48,
               min_overlap=2, winners_set_size=40, inhibition_radius=radius)
    idx, perm, boost = perturbed_state(cfg)
    if boost_mode == "near1":
        boost = near1_boosts(cfg.num_columns)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(78, 0, 6, cfg.input_height, cfg.input_width, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, P.SP_PATH_PER_INPUT)
    check_results(results, *run_gpu(sp, frames))


def test_bench_launch_config_sampled_parity():
    """The exact launch configuration bench.py times: 4096 device-generated frames.

    Frames come from the device generator (cross-checked against sp_inputs
    above); the oracle recomputes a sample of frames from sp_inputs on the host.
    All 4096 frames are checked against the winner-count invariant."""
    cfg = headline_cfg()
    state = perturbed_state(cfg, boost_hi=1.0)  # boosts 1 (a learned SP without boost updates)
    sp = make_sp(cfg, state, max_inputs=4096)
    frames = torch.empty((4096, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 2002, rho=0.5)
    sp.compute(frames)
    sdr, counts = sp.winners()
    raw, boosted = sp.overlaps()
    torch.cuda.synchronize()
    assert sp.info()["plan"]["path"] == P.SP_PATH_BATCHED
    sdr, counts = sdr.cpu().numpy(), counts.cpu().numpy()
    raw, boosted = raw.cpu().numpy().view(np.uint16), boosted.cpu().numpy()
    nz = (boosted > 1.0).sum(axis=1)
    assert np.array_equal(counts, np.minimum(cfg.winners_set_size, nz))
    rng = np.random.default_rng(3)
    sample = sorted(set(rng.choice(4096, 10, replace=False).tolist()) | {0, 4095})
    ora = O.SpatialPoolerOracle(cfg, state)
    for f in sample:
        x = O.encode(sp_inputs.frames(2002, f, 1, 540, 960, rho=0.5), cfg)[0]
        res = ora.step(x, False)
        check_results([res], sdr, counts, raw, boosted, rows=[f])


SWEEP = [(C, S) for C in (256, 512, 1024, 2048) for S in (32, 64, 128, 256)]


@pytest.mark.parametrize("radius", [0, 80])
@pytest.mark.parametrize("C,S", SWEEP)
def test_config3_sweep_sampled_parity(C, S, radius):
    """BASELINE config 3 points (Tab. 2 min_overlap 8, k 40) on 960x540 frames: a sample of
    4 frames through the batched kernel, bit-exact against the oracle."""
    cfg = headline_cfg(num_columns=C, synapses_per_column=S, min_overlap=8, winners_set_size=40,
                       inhibition_radius=radius)
    idx, perm, boost = O.init_pools(cfg)
    frames = sp_inputs.frames(2002, 0, 4, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, (idx, perm, boost))
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, None, max_inputs=8)  # the library's own init (== oracle init, R8)
    out = run_gpu(sp, frames)
    assert sp.info()["plan"]["path"] == P.SP_PATH_BATCHED
    check_results(results, *out)


@pytest.mark.parametrize("path", ["grid", "input"])
def test_scaled_config5_learning(path):
    # BASELINE config 5: 16384 columns, 512 synapses, local r=80 (no cluster fits: grid kernel)
    cfg = headline_cfg(num_columns=16384, synapses_per_column=512, min_overlap=8,
                       winners_set_size=40, inhibition_radius=80)
    idx, perm, _ = O.init_pools(cfg)
    state = (idx, perm, sp_inputs.boosts(7, cfg.num_columns))
    frames = sp_inputs.frames(1001, 0, 3, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, path, max_inputs=8)
    check_results(results, *run_gpu(sp, frames, learn=True))
    check_learn_path(sp, path)
    _, gperm, _ = sp.get_state()
    assert np.array_equal(gperm.view(np.uint32), ora.perm.view(np.uint32))
    # inference after learning: the per-input path rebuilds its synapse-major table
    frames2 = sp_inputs.frames(2002, 0, 2, 540, 960, rho=0.5)
    res2 = [ora.step(x, False) for x in O.encode(frames2, cfg)]
    check_results(res2, *run_gpu(sp, frames2))


def test_end_to_end_host_buffers_match_device_call():
    cfg = headline_cfg()
    state = perturbed_state(cfg)
    frames = sp_inputs.frames(2002, 0, 70, 540, 960, rho=0.5)
    sp = make_sp(cfg, state, max_inputs=128)
    sdr_d, cnt_d, _, _ = run_gpu(sp, frames)
    sdr_h, cnt_h = sp.compute_host(frames)
    assert np.array_equal(sdr_h.view(np.int32), sdr_d) and np.array_equal(cnt_h.astype(np.int32), cnt_d)


def test_shape_errors():
    sp = make_sp(ocfg())
    with pytest.raises(P.SpError) as e:
        sp.compute(torch.zeros((2, 8, 9), dtype=torch.uint8, device=DEV))
    assert e.value.status == P.SP_E_SHAPE
    with pytest.raises(P.SpError):
        sp.compute(torch.zeros((2, 8, 8), dtype=torch.int32, device=DEV))
    with pytest.raises(P.SpError):
        sp.compute(torch.zeros((2, 8, 8), dtype=torch.uint8))


def test_compute_into_writes_caller_buffers():
    cfg = ocfg(input_width=48, input_height=37, num_columns=100, synapses_per_column=20, min_overlap=3,
               winners_set_size=7)
    state = perturbed_state(cfg)
    frames = to_dev(sp_inputs.frames(2002, 0, 45, 37, 48, rho=0.5))
    a = make_sp(cfg, state)
    b = make_sp(cfg, state)
    a.compute(frames)
    want_sdr, want_cnt = a.winners()
    sdr = torch.full((45, 4), -1, dtype=torch.int32, device=DEV)
    cnt = torch.full((45,), -1, dtype=torch.int32, device=DEV)
    b.compute_into(frames, sdr, cnt)
    torch.cuda.synchronize()
    assert torch.equal(sdr, want_sdr) and torch.equal(cnt, want_cnt)
    s2, c2 = b.winners()  # copies from the caller's buffers
    assert torch.equal(s2, want_sdr) and torch.equal(c2, want_cnt)
    h1, _ = a.histograms([0, 20, 45])
    h2, _ = b.histograms([0, 20, 45])
    assert torch.equal(h1, h2)
    # learning through compute_into (cluster kernel) writes the caller's buffers too
    lf = to_dev(sp_inputs.frames(1001, 0, 6, 37, 48, rho=0.5))
    a.compute(lf, learn=True)
    ws, wc = a.winners()
    s3 = torch.empty((6, 4), dtype=torch.int32, device=DEV)
    c3 = torch.empty((6,), dtype=torch.int32, device=DEV)
    b.compute_into(lf, s3, c3, learn=True)
    torch.cuda.synchronize()
    assert torch.equal(s3, ws) and torch.equal(c3, wc)


@pytest.mark.parametrize("case", ["max_columns_global", "max_columns_local", "max_synapses", "max_bits"])
def test_extreme_sizes(case):
    # the largest configurations the ABI accepts run (per-input paths) and stay bit-exact
    kw = dict(max_columns_global=dict(input_width=64, input_height=32, num_columns=20480,
                                      synapses_per_column=24, min_overlap=3, winners_set_size=40),
              max_columns_local=dict(input_width=64, input_height=32, num_columns=20480,
                                     synapses_per_column=24, min_overlap=3, winners_set_size=40,
                                     inhibition_radius=300),
              max_synapses=dict(input_width=128, input_height=64, num_columns=64, synapses_per_column=4095,
                                min_overlap=100, winners_set_size=5),
              max_bits=dict(input_width=1500, input_height=1200, num_columns=96, synapses_per_column=64,
                            min_overlap=4, winners_set_size=9))[case]
    cfg = ocfg(**kw)
    state = perturbed_state(cfg)
    frames = sp_inputs.frames(606, 0, 3, cfg.input_height, cfg.input_width, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    want = ora.compute(frames, learning=True)
    sp = make_sp(cfg, state, max_inputs=8)
    check_results(want, *run_gpu(sp, frames, learn=True))
    assert np.array_equal(sp.get_state()[1].view(np.uint32), ora.perm.view(np.uint32))
    want2 = [ora.step(x, False) for x in O.encode(frames, cfg)]
    check_results(want2, *run_gpu(sp, frames))


def test_local_uniform_mixed_level_counts():
    """Local inhibition, uniform boost, batched kernel: inputs whose eligible raw counts span
    more than 255 values (> 8 wavelet levels: the comparator fallback) interleaved with narrow
    ones (the paired wavelet) in the same CTA; every warp keeps to its own scratch slot."""
    cfg = ocfg(input_width=64, input_height=48, num_columns=1024, synapses_per_column=512,
               min_overlap=2, winners_set_size=20, inhibition_radius=100)
    idx, perm, _ = O.init_pools(cfg)
    perm = perm.copy()
    perm[512:, 6:] = np.float32(0.0)  # columns 512.. keep 6 connected synapses: raw <= 6
    state = (idx, perm, np.ones(cfg.num_columns, np.float32))
    dense = sp_inputs.frames(5, 0, 24, 48, 64, rho=0.7)    # raw up to ~360 on columns < 512
    sparse = sp_inputs.frames(6, 0, 24, 48, 64, rho=0.1)   # raw <= ~60
    frames = np.empty((48, 48, 64), np.uint8)
    frames[0::2], frames[1::2] = dense, sparse
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    spread = [int(r.raw[r.raw >= 2].max() - r.raw[r.raw >= 2].min()) for r in results]
    assert max(spread) >= 256 and min(spread) < 128
    sp = make_sp(cfg, state, P.SP_PATH_BATCHED)
    check_results(results, *run_gpu(sp, frames))


@pytest.mark.parametrize("umax", [62, 4094])
@pytest.mark.parametrize("boost_mode", ["seeded", "near1"])
def test_local_general_wavelet_coarse_key_width(umax, boost_mode, monkeypatch):
    """The per-warp wavelet over coarse keys of a given width (SP_WM_UMAX: u - 1 <= umax); a
    6-bit map makes most columns tie in u, so nearly every decision goes through the exact
    re-decision of lossy ties from the bottom-level positions."""
    monkeypatch.setenv("SP_WM_MIN_RADIUS", "0")
    monkeypatch.setenv("SP_WM_UMAX", str(umax))
    cfg = ocfg(input_width=96, input_height=64, num_columns=1000, synapses_per_column=64,
               min_overlap=2, winners_set_size=20, inhibition_radius=300)
    idx, perm, boost = perturbed_state(cfg)
    if boost_mode == "near1":
        boost = near1_boosts(cfg.num_columns)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(79, 0, 45, cfg.input_height, cfg.input_width, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    check_results(results, *run_gpu(make_sp(cfg, state, P.SP_PATH_BATCHED), frames))


# --------------------------------------------------------------------------- #
# the timed selection branches: full groups, overlap recording on and off
# --------------------------------------------------------------------------- #
def run_gpu_sdr(sp, frames):
    """winners only (recording off): (sdr int32 [n, words], counts int32 [n])"""
    sp.compute(to_dev(frames))
    sdr, counts = sp.winners()
    torch.cuda.synchronize()
    return sdr.cpu().numpy(), counts.cpu().numpy()


def check_sdrs(results, sdr, counts):
    for r, res in enumerate(results):
        assert np.array_equal(sdr[r], sdr_of(res.active)), f"winners mismatch at input {r}"
        assert counts[r] == res.active.sum(), f"count mismatch at input {r}"


@pytest.mark.parametrize("record", [True, False])
@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1", "uniform1.5"])
@pytest.mark.parametrize("kw", SMALL)
def test_inference_parity_full_groups(kw, boost_mode, record, monkeypatch):
    """45 inputs in 2 groups of 23/22 (SP_GROUPS=2): with 16 warps per CTA, warps 0..6 take two
    inputs each, so the paired branches (global uniform: interleaved threshold searches;
    local uniform: the two-input wavelet) run next to the single-input ones -- with and without
    SP_FLAG_RECORD_OVERLAPS (recording must not change which selection code runs)."""
    monkeypatch.setenv("SP_GROUPS", "2")
    cfg = ocfg(**kw)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(2002, 0, 45, cfg.input_height, cfg.input_width, rho=0.5, nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, P.SP_PATH_BATCHED, record=record)
    if record:
        check_results(results, *run_gpu(sp, frames))
    else:
        check_sdrs(results, *run_gpu_sdr(sp, frames))
    pl = sp.info()["plan"]
    assert pl["path"] == P.SP_PATH_BATCHED and pl["groups"] == 2 and pl["cluster"] == 1


@pytest.mark.parametrize("record", [True, False])
@pytest.mark.parametrize("radius,selector", [(0, "-"), (80, "candidates"), (80, "wavelet"), (506, "candidates"),
                                             (506, "wavelet")])
@pytest.mark.parametrize("boost_mode", ["uniform1", "seeded"])
def test_full_size_full_groups(radius, selector, boost_mode, record, monkeypatch):
    """BASELINE config 2/4 geometry (960x540, C 1024, S 256, theta 4, k 40) in groups of 23/22
    inputs: global uniform (the headline's paired threshold search), local r 80 / 506 by
    candidate pruning or by the wavelets (the paired local-uniform wavelet, never compared with
    the oracle in round 1; the per-column-boost wavelet), each with recording on and off."""
    monkeypatch.setenv("SP_GROUPS", "2")
    monkeypatch.setenv("SP_CAND_MIN_RADIUS", "0" if selector == "candidates" else "100000")
    cfg = headline_cfg(inhibition_radius=radius)
    state = with_boost(perturbed_state(cfg), boost_mode)
    frames = sp_inputs.frames(2002, 100, 45, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, P.SP_PATH_BATCHED, max_inputs=64, record=record)
    if record:
        check_results(results, *run_gpu(sp, frames))
    else:
        check_sdrs(results, *run_gpu_sdr(sp, frames))
    assert sp.info()["plan"]["groups"] == 2


def test_bench_launch_config_recording_off_equals_on():
    """The bench's exact launch (4096 frames, recording off, 148 groups of 27-28: every warp
    pairs its inputs) gives the same winners as the recorded launch on all 4096 frames."""
    cfg = headline_cfg()
    state = perturbed_state(cfg, boost_hi=1.0)
    frames = torch.empty((4096, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 2002, rho=0.5)
    outs = []
    for record in (False, True):
        sp = make_sp(cfg, state, max_inputs=4096, record=record)
        sp.compute(frames)
        sdr, counts = sp.winners()
        outs.append((sdr.clone(), counts.clone()))
        sp.close()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("boost_mode", ["uniform1", "seeded", "near1"])
@pytest.mark.parametrize("radius", [16, 24, 32, 40, 48, 64, 100, 200, 300, 506, 900, 1021])
@pytest.mark.parametrize("k", [5, 40])
def test_local_candidates_radius_sweep(radius, k, boost_mode, monkeypatch):
    """Candidate pruning (sp_select.cuh local_candidates) over radii from the point where the
    candidates overflow the warp's scratch (fallback to wavelet / comparator) to nearly global,
    with uniform boosts (raw ties: many candidates share the threshold value), seeded and near-1
    boosts (coarse-key ties, exact 64-bit keys decide); 45 inputs in 2 groups so warps run
    several inputs; recording off (the timed configuration) and on, against the oracle."""
    monkeypatch.setenv("SP_GROUPS", "2")
    monkeypatch.setenv("SP_CAND_MIN_RADIUS", "0")
    cfg = ocfg(input_width=96, input_height=64, num_columns=1024, synapses_per_column=64,
               min_overlap=3, winners_set_size=k, inhibition_radius=radius)
    idx, perm, boost = perturbed_state(cfg)
    if boost_mode == "near1":
        boost = near1_boosts(cfg.num_columns)
    elif boost_mode == "uniform1":
        boost = np.ones_like(boost)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(79, 0, 45, cfg.input_height, cfg.input_width, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    check_sdrs(results, *run_gpu_sdr(make_sp(cfg, state, P.SP_PATH_BATCHED, record=False), frames))
    check_results(results, *run_gpu(make_sp(cfg, state, P.SP_PATH_BATCHED), frames))


@pytest.mark.parametrize("radius,boost_mode", [(48, "near1"), (56, "seeded"), (64, "uniform1")])
def test_local_candidates_fallback_mixing(radius, boost_mode, monkeypatch):
    """Headline geometry at radii where the candidate count straddles the warp scratch's
    capacity (per-column boosts: ~820 keys of 8 B), so within one CTA some warps run candidate
    pruning and others fall back to the comparator for their next input: every selector of a
    warp must use that warp's own scratch slot (a round-2 bug let a comparator fallback write
    into a neighbour's candidate list).  Recording off and on, against the oracle."""
    monkeypatch.setenv("SP_GROUPS", "2")
    monkeypatch.setenv("SP_CAND_MIN_RADIUS", "0")
    cfg = headline_cfg(inhibition_radius=radius)
    idx, perm, boost = perturbed_state(cfg)
    if boost_mode == "near1":
        boost = near1_boosts(cfg.num_columns)
    elif boost_mode == "uniform1":
        boost = np.ones_like(boost)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(2002, 200, 45, 540, 960, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    check_sdrs(results, *run_gpu_sdr(make_sp(cfg, state, P.SP_PATH_BATCHED, max_inputs=64, record=False), frames))
    check_results(results, *run_gpu(make_sp(cfg, state, P.SP_PATH_BATCHED, max_inputs=64), frames))


@pytest.mark.parametrize("n,radius,boost_mode", [(512, 0, "uniform1"), (1024, 0, "seeded"), (2048, 0, "uniform1"),
                                                 (512, 506, "seeded"), (1024, 80, "uniform1")])
def test_strong_shard_launch_configs(n, radius, boost_mode):
    """The shards one GPU owns at G = 8, 4, 2 of a 4096-frame batch (bench strong_shards):
    the planner splits each group's windows over clusters of K = 6, 4, 2 CTAs whose partial
    counts are summed over DSMEM before the selection; recording off (the timed path) against
    the oracle on sampled frames, the winner-count invariant on all (global inhibition)."""
    cfg = headline_cfg(inhibition_radius=radius)
    state = with_boost(perturbed_state(cfg), boost_mode)
    sp = make_sp(cfg, state, max_inputs=n, record=False)
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 2002, rho=0.5)
    sp.compute(frames)
    sdr, counts = sp.winners()
    torch.cuda.synchronize()
    pl = sp.info()["plan"]
    assert pl["path"] == P.SP_PATH_BATCHED and pl["cluster"] > 1, pl
    sdr, counts = sdr.cpu().numpy(), counts.cpu().numpy()
    rng = np.random.default_rng(n + radius)
    sample = sorted(set(rng.choice(n, 6, replace=False).tolist()) | {0, n - 1})
    ora = O.SpatialPoolerOracle(cfg, state)
    for f in sample:
        res = ora.step(O.encode(sp_inputs.frames(2002, f, 1, 540, 960, rho=0.5), cfg)[0], False)
        assert np.array_equal(sdr[f], sdr_of(res.active)), f"winners mismatch at frame {f}"
        assert counts[f] == res.active.sum()


@pytest.mark.parametrize("n,K,R", [(200, 8, 25), (200, 7, 9), (130, 3, 3), (96, 5, 32), (77, 1, 13), (64, 2, 1)])
def test_cluster_sizes_and_group_rows(monkeypatch, n, K, R):
    """Every cluster size K <= 8 (the DSMEM sum of the K partial count rows, 16-byte packed-u16
    loads) and groups of exactly R inputs (TMA boxes of R rows, the last group shorter, rows
    < 8 inside one swizzle atom), recording off (the timed path), against the oracle on sampled
    frames and the winner-count invariant on all."""
    monkeypatch.setenv("SP_FORCE_K", str(K))
    monkeypatch.setenv("SP_FORCE_R", str(R))
    cfg = headline_cfg()
    state = with_boost(perturbed_state(cfg), "uniform1")
    sp = make_sp(cfg, state, max_inputs=n, record=False)
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 3003, rho=0.5)
    sp.compute(frames)
    sdr, counts = sp.winners()
    torch.cuda.synchronize()
    pl = sp.info()["plan"]
    assert pl["cluster"] == K and pl["group_inputs"] == min(R, n), pl
    assert pl["groups"] == -(-n // pl["group_inputs"]), pl
    sdr, counts = sdr.cpu().numpy(), counts.cpu().numpy()
    assert (counts == cfg.winners_set_size).all()
    rng = np.random.default_rng(n * 10 + K)
    sample = sorted(set(rng.choice(n, 5, replace=False).tolist()) | {0, R - 1, min(R, n - 1), n - 1})
    ora = O.SpatialPoolerOracle(cfg, state)
    for f in sample:
        res = ora.step(O.encode(sp_inputs.frames(3003, f, 1, 540, 960, rho=0.5), cfg)[0], False)
        assert np.array_equal(sdr[f], sdr_of(res.active)), f"winners mismatch at frame {f}"


@pytest.mark.parametrize("n,K,R", [(512, 9, 32), (144, 12, 16), (130, 2, 3), (96, 5, 32), (64, 16, 32), (33, 4, 1)])
def test_global_split_groups(monkeypatch, n, K, R):
    """The global split: K CTAs per group in one cooperative launch, partial counts
    written to L2, a per-group arrival barrier, each CTA summing its inputs' K partial rows
    (recording off, the timed path) -- against the oracle on sampled frames, the winner-count
    invariant on all; run twice, so the barrier counters' reset between launches is exercised."""
    monkeypatch.setenv("SP_FORCE_K", str(K))
    monkeypatch.setenv("SP_FORCE_R", str(R))
    monkeypatch.setenv("SP_FORCE_GSPLIT", "1")
    cfg = headline_cfg()
    state = with_boost(perturbed_state(cfg), "uniform1")
    sp = make_sp(cfg, state, max_inputs=n, record=False)
    frames = torch.empty((n, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 4004, rho=0.5)
    for _ in range(2):
        sp.compute(frames)
    sdr, counts = sp.winners()
    torch.cuda.synchronize()
    pl = sp.info()["plan"]
    assert pl["global_split"] == 1 and pl["cluster"] == K and pl["group_inputs"] == min(R, n), pl
    sdr, counts = sdr.cpu().numpy(), counts.cpu().numpy()
    assert (counts == cfg.winners_set_size).all()
    rng = np.random.default_rng(n * 7 + K)
    sample = sorted(set(rng.choice(n, 5, replace=False).tolist()) | {0, min(R, n - 1), n - 1})
    ora = O.SpatialPoolerOracle(cfg, state)
    for f in sample:
        res = ora.step(O.encode(sp_inputs.frames(4004, f, 1, 540, 960, rho=0.5), cfg)[0], False)
        assert np.array_equal(sdr[f], sdr_of(res.active)), f"winners mismatch at frame {f}"
