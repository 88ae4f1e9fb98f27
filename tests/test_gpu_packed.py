"""GPU parity of the bit-plane input path (include/sp.h "bit-plane input").

Frames given as bit-planes (1 bit per pixel, LSB first, row-major) must give exactly the
winners of the oracle on the uint8 frames (R12: bit = byte != 0).  The planes fed to the
kernel are packed here with NumPy (np.packbits, little bit order), independently of the
library's own packer, which is checked against the same NumPy packing.
"""
import numpy as np
import pytest

import oracle as O
import sp_inputs
from tests.helpers import ocfg, perturbed_state, sdr_of

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1608_01966_b200 as P  # noqa: E402
from tests.test_gpu_parity import make_sp, with_boost, near1_boosts, DEV  # noqa: E402


def np_planes(frames, words):
    """uint8 [F, H, W] -> uint32 [F, words]: bit i of word w = pixel 32w + i is nonzero."""
    F = frames.shape[0]
    bits = (frames.reshape(F, -1) != 0)
    by = np.packbits(bits, axis=1, bitorder="little")
    out = np.zeros((F, words * 4), np.uint8)
    out[:, :by.shape[1]] = by
    return out.view("<u4")


def run_packed(sp, planes_np):
    planes = torch.from_numpy(planes_np.view(np.int32)).to(DEV)
    sp.compute_packed(planes)
    sdr, counts = sp.winners()
    torch.cuda.synchronize()
    return sdr.cpu().numpy(), counts.cpu().numpy()


CASES = [
    dict(),                                                         # tiny (64 bits), global
    dict(inhibition_radius=4),                                      # tiny, local
    dict(input_width=48, input_height=40, num_columns=100, synapses_per_column=20,
         min_overlap=3, winners_set_size=7),                        # C % 32 != 0, 1920 bits (ragged chunk)
    dict(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
         min_overlap=8, winners_set_size=40, inhibition_radius=80),  # Tab. 2 on Tab. 1 frames
    dict(input_width=96, input_height=64, num_columns=1000, synapses_per_column=64,
         min_overlap=2, winners_set_size=20, inhibition_radius=300),  # wavelet local top-k
]


@pytest.mark.parametrize("boost_mode", ["seeded", "uniform1", "near1"])
@pytest.mark.parametrize("kw", CASES)
def test_packed_inference_parity(kw, boost_mode):
    cfg = ocfg(**kw)
    idx, perm, boost = with_boost(perturbed_state(cfg), "uniform1" if boost_mode == "uniform1" else "seeded")
    if boost_mode == "near1":
        boost = near1_boosts(cfg.num_columns)
    state = (idx, perm, boost)
    frames = sp_inputs.frames(2002, 0, 45, cfg.input_height, cfg.input_width, rho=0.5, nonzero="random")
    ora = O.SpatialPoolerOracle(cfg, state)
    results = [ora.step(x, False) for x in O.encode(frames, cfg)]
    sp = make_sp(cfg, state, P.SP_PATH_BATCHED)
    sdr, counts = run_packed(sp, np_planes(frames, sp.packed_words))
    for i, res in enumerate(results):
        assert counts[i] == res.active.sum(), f"count mismatch at input {i}"
        assert np.array_equal(sdr[i], sdr_of(res.active)), f"SDR mismatch at input {i}"


def test_pack_frames_matches_numpy():
    cfg = ocfg(input_width=240, input_height=134, num_columns=256, synapses_per_column=32)
    sp = make_sp(cfg, record=False)
    frames = sp_inputs.frames(7, 0, 70, 134, 240, rho=0.3, nonzero="random")
    planes = sp.pack_frames(torch.from_numpy(frames).to(DEV))
    torch.cuda.synchronize()
    got = planes.cpu().numpy().view(np.uint32)
    want = np_planes(frames, sp.packed_words)
    Wn = (240 * 134 + 31) // 32
    assert np.array_equal(got[:, :Wn], want[:, :Wn])


def test_packed_headline_launch_matches_uint8_path_and_oracle():
    """BASELINE config 4 sizes (4096 x 960x540, C 1024, S 256): the packed kernel equals the
    uint8 kernel on every frame and the oracle on sampled frames (global and local r 506)."""
    for radius in (0, 506):
        cfg = ocfg(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
                   min_overlap=4, winners_set_size=40, inhibition_radius=radius)
        state = perturbed_state(cfg, boost_hi=1.0 if radius == 0 else 2.0)
        sp = make_sp(cfg, state, P.SP_PATH_BATCHED, max_inputs=4096, record=False)
        frames = torch.empty((4096, 540, 960), dtype=torch.uint8, device=DEV)
        P.synth_frames(frames, 0, 2002, 0.5)
        sdr8 = torch.empty((4096, 32), dtype=torch.int32, device=DEV)
        cnt8 = torch.empty((4096,), dtype=torch.int32, device=DEV)
        sp.compute_into(frames, sdr8, cnt8)
        planes = sp.pack_frames(frames)
        sdrp = torch.empty_like(sdr8)
        cntp = torch.empty_like(cnt8)
        sp.compute_packed(planes, sdrp, cntp)
        torch.cuda.synchronize()
        assert torch.equal(sdr8, sdrp) and torch.equal(cnt8, cntp)
        ora = O.SpatialPoolerOracle(cfg, state)
        for f in (0, 1, 2047, 4095):
            fr = frames[f:f + 1].cpu().numpy()
            res = ora.step(O.encode(fr, cfg)[0], False)
            assert np.array_equal(sdrp[f].cpu().numpy(), sdr_of(res.active))
        del frames, planes
        sp.close()


def test_packed_host_end_to_end_matches_device():
    cfg = ocfg(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
               min_overlap=8, winners_set_size=40)
    state = perturbed_state(cfg)
    sp = make_sp(cfg, state, P.SP_PATH_BATCHED, record=False)
    frames = sp_inputs.frames(3, 0, 100, 134, 240, rho=0.5)
    planes = np_planes(frames, sp.packed_words)
    sdr_d, cnt_d = run_packed(sp, planes)
    sdr_h = np.empty((100, sp.sdr_words), np.uint32)
    cnt_h = np.empty((100,), np.uint32)
    sp.compute_packed_host_into(planes, sdr_h, cnt_h)
    assert np.array_equal(sdr_h.view(np.int32), sdr_d) and np.array_equal(cnt_h.view(np.int32), cnt_d)


def test_packed_errors():
    cfg = ocfg(input_width=64, input_height=60, patch_width=32, patch_height=30, num_columns=256,
               synapses_per_column=64)
    sp = make_sp(cfg, record=False)
    planes = torch.zeros((2, sp.packed_words), dtype=torch.int32, device=DEV)
    with pytest.raises(P.SpError) as e:
        sp.compute_packed(planes)
    assert e.value.status == P.SP_E_CONFIG
    sp2 = make_sp(ocfg(), record=False)
    bad = torch.zeros((2, sp2.packed_words + 1), dtype=torch.int32, device=DEV)[:, 1:]
    with pytest.raises(P.SpError):
        sp2.compute_packed(bad)  # not contiguous / misaligned


def test_packed_host_multi_chunk_pipeline():
    """sp_compute_packed_host over more frames than one staging chunk (~1035 bit-plane frames of
    960x540): the double-buffered H2D / compute / D2H pipeline equals the device call."""
    cfg = ocfg(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
               min_overlap=4, winners_set_size=40)
    sp = make_sp(cfg, perturbed_state(cfg), P.SP_PATH_BATCHED, max_inputs=2600, record=False)
    frames = torch.empty((2600, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(frames, 0, 31, 0.5)
    planes = sp.pack_frames(frames)
    del frames
    sdr_d = torch.empty((2600, 32), dtype=torch.int32, device=DEV)
    cnt_d = torch.empty((2600,), dtype=torch.int32, device=DEV)
    sp.compute_packed(planes, sdr_d, cnt_d)
    host = planes.cpu()
    sdr_h = np.empty((2600, 32), np.uint32)
    cnt_h = np.empty((2600,), np.uint32)
    sp.compute_packed_host_into(host.numpy(), sdr_h, cnt_h)
    assert np.array_equal(sdr_h.view(np.int32), sdr_d.cpu().numpy())
    assert np.array_equal(cnt_h.view(np.int32), cnt_d.cpu().numpy())
