"""GPU parity of the on-device encoder (DESIGN
R23-R25) against the encoder oracle: bit-exact binarised frames (every step is integer
arithmetic or a fixed sequence of fp32 RN operations on both sides)."""
import numpy as np
import pytest

from oracle import encoder as E
import oracle as O
import sp_inputs
from tests.helpers import ocfg, gpu_kwargs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1608_01966_b200 as P  # noqa: E402

DEV = torch.device("cuda", 0)


def test_synth_bgr_matches_python_recipe():
    out = torch.empty((3, 540, 960, 3), dtype=torch.uint8, device=DEV)
    P.synth_bgr_frames(out, 5, 1234)
    assert np.array_equal(out.cpu().numpy(), sp_inputs.bgr_frames(1234, 5, 3, 540, 960))


@pytest.mark.parametrize("src,dst,k,bias", [
    ((960, 540), (240, 134), 11, 2.0),       # the paper's sizes, S:311 defaults
    ((960, 540), (240, 135), 5, 3.5),        # exact 4:1 both ways; ceil(bias) = 4
    ((100, 70), (33, 21), 7, -1.0),          # generic x table, rows not 16-byte multiples
    ((64, 48), (64, 48), 3, 2.0),            # identity downscale
    ((192, 108), (48, 27), 15, 0.0),
])
def test_encoder_parity(src, dst, k, bias):
    F = 37  # > 2 x 148 / ... ragged over the persistent CTAs
    bgr = sp_inputs.bgr_frames(77, 3, F, src[1], src[0])
    want = E.encode_bgr(bgr, dst[0], dst[1], k, bias)
    enc = P.Encoder(src_width=src[0], src_height=src[1], dst_width=dst[0], dst_height=dst[1],
                    block_size=k, bias=bias)
    got = enc.encode(torch.from_numpy(bgr).to(DEV)).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(np.array(enc.info()["kernel"], np.float32), E.gaussian_kernel_f32(k))
    for f in range(F):
        assert np.array_equal(got[f], want[f]), f"frame {f}: {np.count_nonzero(got[f] != want[f])} px differ"


def test_encoder_random_bytes_and_unaligned_source():
    # random pixels (every rounding case of the area sums) and a source pointer off by one byte
    rng = np.random.default_rng(3)
    bgr = rng.integers(0, 256, (5, 540, 960, 3), dtype=np.uint8)
    want = E.encode_bgr(bgr, 240, 134)
    enc = P.Encoder()
    buf = torch.empty(bgr.size + 16, dtype=torch.uint8, device=DEV)
    view = buf[1:1 + bgr.size].view(5, 540, 960, 3)
    view.copy_(torch.from_numpy(bgr))
    import ctypes
    out = torch.empty((5, 134, 240), dtype=torch.uint8, device=DEV)
    st = P.lib().sp_encode(enc._h, ctypes.c_void_p(view.data_ptr()), 5, ctypes.c_void_p(out.data_ptr()), None)
    assert st == 0
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
    assert np.array_equal(enc.encode(torch.from_numpy(bgr).to(DEV)).cpu().numpy(), want)


def test_encoder_feeds_the_sp():
    # encoder output -> SP inference (the paper's processing flow): winners equal the
    # oracle's on the oracle-encoded frames
    bgr = sp_inputs.bgr_frames(5, 0, 6, 540, 960)
    frames = E.encode_bgr(bgr, 240, 134)
    cfg = ocfg(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
               min_overlap=8, winners_set_size=40)
    ora = O.SpatialPoolerOracle(cfg)
    want = [O.sdr_words(r.active).view(np.int32) for r in ora.compute(frames, False)]
    enc = P.Encoder()
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=64))
    sp.compute(enc.encode(torch.from_numpy(bgr).to(DEV)))
    sdr, _ = sp.winners()
    assert np.array_equal(sdr.cpu().numpy(), np.stack(want))


def test_encoder_config_errors():
    for kw in (dict(block_size=4), dict(block_size=17), dict(dst_width=1000), dict(src_width=0)):
        with pytest.raises(P.SpError) as e:
            P.Encoder(**kw)
        assert e.value.status == P.SP_E_CONFIG


@pytest.mark.parametrize("chunk", ["7", "1024"])
def test_encode_compute_fused_call(chunk, monkeypatch):
    """sp_encode_compute (raw BGR -> SDRs, binarised chunk in a persisting-L2 window): equal to
    the oracle chain (encoder oracle -> SP oracle) on the first frames, and to sp_encode +
    sp_compute on all frames, across chunk boundaries (7 frames per chunk: ragged last chunk)."""
    monkeypatch.setenv("SP_ENC_CHUNK", chunk)
    F = 23
    bgr = sp_inputs.bgr_frames(91, 0, F, 540, 960)
    cfg = ocfg(input_width=240, input_height=134, num_columns=2048, synapses_per_column=128,
               min_overlap=8, winners_set_size=40, inhibition_radius=80)
    enc = P.Encoder()
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=64))
    dbgr = torch.from_numpy(bgr).to(DEV)
    sdr, counts = enc.encode_compute(sp, dbgr)
    s2, c2 = sp.winners()
    assert torch.equal(s2, sdr) and torch.equal(c2, counts)  # the SP's last results = the whole call
    binf = enc.encode(dbgr)
    sp.compute(binf)
    ref_sdr, ref_counts = sp.winners()
    assert torch.equal(sdr, ref_sdr) and torch.equal(counts, ref_counts)
    ora = O.SpatialPoolerOracle(cfg, sp.get_state())
    want = E.encode_bgr(bgr[:4], 240, 134)
    got = sdr.cpu().numpy()
    for f, x in enumerate(O.encode(want, cfg)):
        r = ora.step(x, False)
        assert np.array_equal(got[f], O.sdr_words(r.active).view(np.int32)), f"frame {f}"
    with pytest.raises(P.SpError):  # the SP's input frame must be the encoder's output frame
        enc.encode_compute(P.SpatialPooler(input_width=96, input_height=64, num_columns=128,
                                           synapses_per_column=16, min_overlap=2, winners_set_size=8), dbgr)
