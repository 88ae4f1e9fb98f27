"""GPU parity of the per-video SDR histograms (
DESIGN R22) against the oracle: counts bit-exact, normalised histograms bit-equal (both sides
round fp32(count)/fp32(n) once)."""
import numpy as np
import pytest

import oracle as O
import sp_inputs
from tests.helpers import ocfg, gpu_kwargs, perturbed_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1608_01966_b200 as P  # noqa: E402

DEV = torch.device("cuda", 0)


def active_of(results):
    return np.stack([r.active for r in results])


@pytest.mark.parametrize("kw,offsets", [
    (dict(), [0, 5, 5, 17, 45]),                                       # ragged, one empty video
    (dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=20, min_overlap=3,
          winners_set_size=30), [0, 45]),                              # C % 32 != 0, one video
    (dict(input_width=64, input_height=60, patch_width=32, patch_height=30, num_columns=256,
          synapses_per_column=64, min_overlap=2, winners_set_size=10), [0, 4, 40, 41, 180]),
])
def test_histograms_parity(kw, offsets):
    cfg = ocfg(**kw)
    state = perturbed_state(cfg)
    nframes = 45
    frames = sp_inputs.frames(2002, 0, nframes, cfg.input_height, cfg.input_width, rho=0.5)
    ora = O.SpatialPoolerOracle(cfg, state)
    res = [ora.step(x, False) for x in O.encode(frames, cfg)]
    want_c, want_h = O.sdr_histograms(active_of(res), offsets)
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=256))
    sp.set_state(*state)
    sp.compute(torch.from_numpy(frames).to(DEV))
    counts, hist = sp.histograms(offsets)
    torch.cuda.synchronize()
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), want_c)
    assert np.array_equal(hist.cpu().numpy().view(np.uint32), want_h.view(np.uint32))


def test_histograms_bench_shape_long_video():
    # the bench shape: 4096 frames, 960x540, C 1024; videos of 32 frames plus one long video
    cfg = ocfg(input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
               min_overlap=4, winners_set_size=40)
    sp = P.SpatialPooler(**gpu_kwargs(cfg, max_inputs=4096))
    fr = torch.empty((4096, 540, 960), dtype=torch.uint8, device=DEV)
    P.synth_frames(fr, 0, 2002, 0.5)
    sp.compute(fr)
    sdr, _ = sp.winners()
    act = np.unpackbits(sdr.cpu().numpy().view(np.uint8), axis=1, bitorder="little").astype(bool)[:, :1024]
    for offsets in (np.arange(0, 4097, 32), [0, 4096], [0, 1, 4095, 4096]):
        counts, hist = sp.histograms(offsets)
        want_c, want_h = O.sdr_histograms(act, offsets)
        assert np.array_equal(counts.cpu().numpy().astype(np.int64), want_c)
        assert np.array_equal(hist.cpu().numpy().view(np.uint32), want_h.view(np.uint32))
    # every frame has exactly k winners, so each video's histogram sums to k
    _, hist = sp.histograms(np.arange(0, 4097, 32))
    assert np.allclose(hist.sum(dim=1).cpu().numpy(), 40.0, atol=1e-4)


def test_histograms_errors():
    sp = P.SpatialPooler(**gpu_kwargs(ocfg(), max_inputs=64))
    with pytest.raises(P.SpError) as e:
        sp.histograms([0, 1])
    assert e.value.status == P.SP_E_STATE
    sp.compute(torch.from_numpy(sp_inputs.frames(1, 0, 10, 8, 8)).to(DEV))
    with pytest.raises(P.SpError) as e:
        sp.histograms([0, 11])          # beyond the inputs of the last call
    assert e.value.status == P.SP_E_ARG
    with pytest.raises(P.SpError):
        sp.histograms([0, 6, 3])        # decreasing
