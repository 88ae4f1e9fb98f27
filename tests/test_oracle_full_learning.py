"""Pins of the oracle's full learning step (SPEC S:119(b-e),
S:149-151; readings R17-R21).

Each check reaches the oracle's number by another route: a closed form, exact rational
arithmetic with an error bound, a library routine (scipy's running maximum), a value worked
out by hand in the test, or an invariant.  None re-types the oracle's fp32 op sequence.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from scipy.ndimage import maximum_filter1d

import oracle as O
import sp_inputs
from tests.helpers import ocfg

ULP1 = 2.0 ** -23  # fp32 ulp at 1


# --------------------------------------------------------------------------- #
# (b) duty cycles: EMA with alpha = 1/period
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("period", [1, 2, 10, 1000])
def test_duty_constant_one_closed_form(period):
    # always active: d_t = 1 - (1 - 1/P)^t exactly in the reals; fp32 error grows by at
    # most a few ulp per step (three RN operations on values <= 1)
    d = np.zeros(1, np.float32)
    for t in range(1, 301):
        d = O.update_duty(d, np.array([True]), period)
        exact = 1.0 - (1.0 - 1.0 / period) ** t
        assert abs(float(d[0]) - exact) <= 3 * t * ULP1
    if period == 1:
        assert d[0] == 1.0  # P = 1: the duty cycle is the last flag exactly


def test_duty_zero_stays_zero_and_decays():
    d = O.update_duty(np.zeros(4, np.float32), np.zeros(4, bool), 1000)
    assert np.all(d == 0.0)
    # one activation then silence: d_t = (1/P) (1 - 1/P)^(t-1)
    d = O.update_duty(np.zeros(1, np.float32), np.array([True]), 1000)
    assert d[0] == np.float32(0.001)
    for t in range(2, 200):
        d = O.update_duty(d, np.array([False]), 1000)
        exact = 0.001 * (0.999 ** (t - 1))
        assert abs(float(d[0]) - exact) <= 3 * t * 2.0 ** -33  # ulp at 1e-3 is 2^-33


def test_duty_stays_in_unit_interval():
    rng = np.random.default_rng(3)
    d = np.zeros(64, np.float32)
    for _ in range(500):
        d = O.update_duty(d, rng.random(64) < 0.3, 7)
        assert np.all((d >= 0) & (d <= 1))


# --------------------------------------------------------------------------- #
# window maximum over W(c) (C9, R18): scipy's running maximum with edge replication
# is the truncated window (replicated edge values never exceed the window's own max)
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("radius", [1, 2, 5, 31, 127, 200])
def test_window_max_vs_scipy(radius):
    v = np.random.default_rng(11).random(128).astype(np.float32)
    got = O.window_max(v, radius)
    want = maximum_filter1d(v, size=2 * radius + 1, mode="nearest")
    assert np.array_equal(got, want)


def test_window_max_global():
    v = np.random.default_rng(12).random(77).astype(np.float32)
    assert np.all(O.window_max(v, 0) == v.max())


# --------------------------------------------------------------------------- #
# (c) boost rule: linear in the duty deficit, bounded by [1, max_boost]
# --------------------------------------------------------------------------- #
def _boost_exact(adc, maxa, max_boost):
    """The rule in exact rationals, from the real inputs (fp32 values as Fractions)."""
    mina = Fraction(float(np.float32(np.float32(0.01) * np.float32(maxa))))
    a = Fraction(float(adc))
    if a >= mina:
        return Fraction(1)
    return 1 + (mina - a) / mina * (Fraction(float(np.float32(max_boost))) - 1)


@pytest.mark.parametrize("max_boost", [2.0, 3.5, 10.0])
def test_boost_rule_exact_within_ulps(max_boost):
    rng = np.random.default_rng(int(max_boost * 10))
    adc = (rng.random(256) * 0.02).astype(np.float32)
    adc[:8] = 0.0
    adc[8] = 0.9  # the maximum: minA = 0.009
    b = O.boost_from_duty(adc, 0, max_boost)
    for c in range(256):
        want = _boost_exact(adc[c], adc.max(), max_boost)
        # four fp32 roundings (relative 2^-24 each) on values <= max_boost: within 4 fp32
        # ulp of max_boost
        ulp = Fraction(2) ** (math.floor(math.log2(max_boost)) - 23)
        assert abs(Fraction(float(b[c])) - want) <= 4 * ulp
    # adc = 0 with a positive neighbourhood maximum -> exactly max_boost (t2 = 1 exactly)
    assert np.all(b[:8] == np.float32(max_boost))
    # the most active column is never boosted (S:119(c) example's fixed point)
    assert b[8] == 1.0
    assert np.all((b >= 1.0) & (b <= np.float32(max_boost)))


def test_boost_monotone_in_duty():
    adc = np.linspace(0, 0.011, 200, dtype=np.float32)
    adc = np.concatenate([adc, np.float32([1.0])])
    b = O.boost_from_duty(adc, 0, 2.0)
    assert np.all(np.diff(b[:-1]) <= 0)


def test_boost_all_zero_duty_is_one():
    # no column ever active: minA = 0, adc >= minA -> boost 1 (S:119 degenerate input)
    assert np.all(O.boost_from_duty(np.zeros(50, np.float32), 0, 2.0) == 1.0)


def test_boost_column_always_active_converges_to_one():
    # S:119 example: a column active on every step for duty_cycle_period steps -> boost 1
    # (9 steps: from perm 0 the other columns need 10 bumps of 0.1*tau to connect, S:119(d))
    cfg = ocfg(num_columns=32, synapses_per_column=8, full_learning=True, duty_cycle_period=9,
               min_overlap=1, winners_set_size=1)
    idx, perm, boost = O.init_pools(cfg)
    perm[:] = 0.0
    perm[5] = 1.0  # column 5 is the only connected column: it wins every non-empty input
    ora = O.SpatialPoolerOracle(cfg, (idx, perm, boost))
    ones = np.full((9, 8, 8), 255, np.uint8)
    for x in O.encode(ones, cfg):
        r = ora.step(x, True)
        assert r.active[5] and r.active.sum() == 1
    assert ora.boost[5] == 1.0
    # every other column never won: its duty cycle is 0 < minA -> boosted to max_boost
    assert np.all(np.delete(ora.boost, 5) == np.float32(2.0))


# --------------------------------------------------------------------------- #
# (d) weak-column bump (S:119(d))
# --------------------------------------------------------------------------- #
def test_bump_closed_form():
    odc = np.array([0.5, 0.004, 0.006, 0.0, 0.5], np.float32)  # minO = 0.005 globally
    perm = np.array([[0.1, 0.2], [0.1, 0.99], [0.3, 0.3], [0.0, 1.0], [0.2, 0.2]], np.float32)
    out, weak = O.bump_weak(perm, odc, 0, 0.2)
    assert weak.tolist() == [False, True, False, True, False]
    b = np.float32(np.float32(0.1) * np.float32(0.2))  # 0.02
    assert out[1, 0] == np.float32(np.float32(0.1) + b)
    assert out[1, 1] == 1.0 and out[3, 1] == 1.0  # clamp at 1 (S:138 closure)
    assert out[3, 0] == b
    assert np.array_equal(out[[0, 2, 4]], perm[[0, 2, 4]])


def test_bump_local_window():
    # with radius 1 the maximum is taken over the three-column window only
    odc = np.array([1.0, 0.005, 0.0, 0.0, 0.0, 0.0001], np.float32)
    _, weak = O.bump_weak(np.zeros((6, 1), np.float32), odc, 1, 0.2)
    # col1: max(1, .005, 0) = 1 -> .005 < .01 weak; col2: max(.005, 0, 0) -> 0 < 5e-5 weak;
    # col3: max 0 -> 0 < 0 false; col4: max(0,0,1e-4) -> 0 < 1e-6 weak; col5: 1e-4 < 1e-6 no
    assert weak.tolist() == [False, True, True, False, True, False]


# --------------------------------------------------------------------------- #
# (e) inhibition radius
# --------------------------------------------------------------------------- #
def test_span_by_hand():
    idx = np.array([[1, 4, 9, 12], [0, 2, 3, 63]], np.int64)
    perm = np.array([[0.1, 0.3, 0.3, 0.1], [0.1, 0.1, 0.1, 0.1]], np.float32)
    assert O.connected_span(idx, perm, 0.2).tolist() == [9 - 4 + 1, 0]
    perm[1, 3] = 0.2
    assert O.connected_span(idx, perm, 0.2).tolist() == [6, 1]


def test_radius_by_hand():
    # 4 columns over 64 bits, spans 10, 20, 0, 30: mean(span * 4/64) = 60/64; /2 = 0.47 -> 0
    # -> clamped to 1
    assert O.adapt_radius(np.array([10, 20, 0, 30]), 64, 4) == 1
    # 8 columns over 16 bits, all spans 16: mean = 8, /2 = 4
    assert O.adapt_radius(np.full(8, 16), 16, 8) == 4
    # 3 columns over 8 bits, spans 8, 8, 7: mean(span*3/8) = 69/24 = 2.875; /2 = 1.4375 -> 1
    assert O.adapt_radius(np.array([8, 8, 7]), 8, 3) == 1
    # 5 columns over 10 bits, spans 10, 10, 10, 10, 5: mean(s*5/10) = 4.5; /2 = 2.25 -> 2
    assert O.adapt_radius(np.array([10, 10, 10, 10, 5]), 10, 5) == 2
    # exact half rounds up: 2 columns, 4 bits, spans 4, 2: mean(s*2/4) = 1.5; /2 = .75 -> 1;
    # 2 columns, 2 bits, spans 2, 1: mean(s*2/2) = 1.5 ... use 6 columns, 4 bits, spans 4,4,4,4,4,2:
    # mean(s*6/4) = 33/6 = 5.5, /2 = 2.75 -> 3
    assert O.adapt_radius(np.array([4, 4, 4, 4, 4, 2]), 4, 6) == 3
    # 2 columns, 4 bits, spans 4 and 6 is impossible (span <= nbits); 10 columns, 10 bits,
    # spans all 5: mean(5*10/10) = 5, /2 = 2.5 -> half up -> 3
    assert O.adapt_radius(np.full(10, 5), 10, 10) == 3


def test_radius_permutation_pools_closed_form():
    # S = nbits: every pool is a permutation; all connected -> span = nbits for every column
    # -> radius = round(C / 2)
    cfg = ocfg(num_columns=127, synapses_per_column=64)
    idx, perm, _ = O.init_pools(cfg)
    span = O.connected_span(idx, perm, 0.2)
    assert np.all(span == 64)
    assert O.adapt_radius(span, 64, 127) == 64  # 63.5 rounds half up
    # nothing connected -> clamp to 1
    assert O.adapt_radius(O.connected_span(idx, np.zeros_like(perm), 0.2), 64, 127) == 1


# --------------------------------------------------------------------------- #
# the composed step: invariants, and the reduction to the hot-path step
# --------------------------------------------------------------------------- #
def _run(cfg, frames, state=None):
    ora = O.SpatialPoolerOracle(cfg, state)
    trace = [ora.step(x, True) for x in O.encode(frames, cfg)]
    return ora, trace


def test_full_learning_invariants():
    cfg = ocfg(full_learning=True, duty_cycle_period=20, inhibition_radius=8, max_boost=3.0)
    frames = sp_inputs.frames(1001, 0, 60, 8, 8, rho=0.3)
    ora, trace = _run(cfg, frames)
    assert ora.iteration == 60
    assert np.all((ora.perm >= 0) & (ora.perm <= 1))
    assert np.all((ora.boost >= 1) & (ora.boost <= np.float32(3.0)))
    assert np.all((ora.active_duty >= 0) & (ora.active_duty <= 1))
    assert 1 <= ora.radius <= cfg.num_columns
    # the boost is an exact-key-domain value (R4): boost * 2^23 is an integer
    O.boost_integer(ora.boost)
    # duty cycles are consistent with the trace: each column's active duty equals the EMA of
    # its own activity, recomputed here in float64 (fp32 error bound, a few ulp per step)
    d = np.zeros(cfg.num_columns)
    for r in trace:
        d = d * (19 / 20) + r.active / 20
    assert np.max(np.abs(d - ora.active_duty)) <= 3 * 60 * ULP1


def test_full_learning_both_duties_match_the_trace():
    """Both duty cycles against float64 EMAs recomputed from the trace (S:119(b)), each
    flag derived in the test from Alg. 1 itself: active duty <- the winners; overlap duty <-
    the overlap Alg. 1 leaves non-zero, i.e. raw >= min_overlap (l.6-8 zero the rest)
    and raw > 0.  Columns with few connected synapses (S = 6, theta 3, sparse frames) make
    0 < raw < theta common, so feeding the raw count (or the active flag) to the overlap duty
    fails here by orders of magnitude more than the fp32 error bound."""
    cfg = ocfg(full_learning=True, duty_cycle_period=10, inhibition_radius=8, synapses_per_column=6,
               min_overlap=3, winners_set_size=6)
    frames = sp_inputs.frames(1003, 0, 60, 8, 8, rho=0.35)
    ora, trace = _run(cfg, frames)
    below = sum(int(((r.raw > 0) & (r.raw < cfg.min_overlap)).sum()) for r in trace)
    assert below > 200, "the stream must exercise 0 < raw < min_overlap"
    a = np.zeros(cfg.num_columns)
    o = np.zeros(cfg.num_columns)
    for r in trace:
        a = a * 0.9 + r.active * 0.1
        o = o * 0.9 + ((r.raw >= cfg.min_overlap) & (r.raw > 0)) * 0.1
    assert np.max(np.abs(a - ora.active_duty)) <= 3 * 60 * ULP1
    assert np.max(np.abs(o - ora.overlap_duty)) <= 3 * 60 * ULP1


def _hand_sp(period=2, max_boost=2.0):
    """4 columns x 8 synapses on an 8x8 input, hand-placed pools: column c sees bits 8c..8c+7."""
    cfg = ocfg(num_columns=4, synapses_per_column=8, min_overlap=4, winners_set_size=1,
               inhibition_radius=0, full_learning=True, duty_cycle_period=period, max_boost=max_boost)
    idx = np.arange(32, dtype=np.int64).reshape(4, 8)
    perm = np.full((4, 8), np.float32(0.21), np.float32)
    return cfg, O.SpatialPoolerOracle(cfg, (idx, perm, np.ones(4, np.float32)))


def test_full_learning_hand_worked_bump_and_boost():
    """S:119(b-d) worked by hand on one frame.  Input bits on: 0..7 (all 8 of column 0), 8..13
    (6 of column 1's), 16..17 (2 of column 2's), none of column 3's.  theta 4, k 1, period 2:
      overlaps (Alg. 1): 8, 6, 0 (2 < theta is cut), 0; winner: column 0 only (k = 1);
      (a) column 0: every input bit on -> perm 0.21 + 0.1 on all 8 synapses;
      (b) active duty = (0*1 + a)/2 = [.5, 0, 0, 0]; overlap duty = [.5, .5, 0, 0]
          (column 1 overlaps without winning; column 2's raw 2 is cut to 0, so it does not count);
      (c) minA = 0.01*.5: columns 1-3 have adc 0 < minA -> boost 1 + (minA/minA)(2-1) = 2.0;
      (d) minO = 0.01*.5: columns 2 and 3 (odc 0) are weak -> every perm + 0.1*0.2 = 0.23;
          column 1 (odc .5, adc 0) is NOT bumped, column 0 not either.
    A second, all-zero frame: no overlaps, no winners; duties halve; 2 and 3 are bumped again."""
    cfg, ora = _hand_sp()
    frame = np.zeros((1, 8, 8), np.uint8)
    on = list(range(0, 8)) + list(range(8, 14)) + [16, 17]
    frame.reshape(-1)[on] = 255
    r = ora.step(O.encode(frame, cfg)[0], True)
    assert list(r.raw) == [8, 6, 2, 0] and list(r.active) == [True, False, False, False]
    assert list(ora.active_duty) == [0.5, 0.0, 0.0, 0.0]
    assert list(ora.overlap_duty) == [0.5, 0.5, 0.0, 0.0]
    assert list(ora.boost) == [1.0, 2.0, 2.0, 2.0]
    p31 = np.float32(np.float32(0.21) + np.float32(0.1))
    p23 = np.float32(np.float32(0.21) + np.float32(np.float32(0.1) * np.float32(0.2)))
    assert np.all(ora.perm[0] == p31) and np.all(ora.perm[1] == np.float32(0.21))
    assert np.all(ora.perm[2] == p23) and np.all(ora.perm[3] == p23)
    r = ora.step(O.encode(np.zeros((1, 8, 8), np.uint8), cfg)[0], True)
    assert not r.active.any()
    assert list(ora.active_duty) == [0.25, 0.0, 0.0, 0.0]
    assert list(ora.overlap_duty) == [0.25, 0.25, 0.0, 0.0]
    p25 = np.float32(p23 + np.float32(np.float32(0.1) * np.float32(0.2)))
    assert np.all(ora.perm[0] == p31) and np.all(ora.perm[1] == np.float32(0.21))
    assert np.all(ora.perm[2] == p25) and np.all(ora.perm[3] == p25)


def test_full_learning_overlap_below_theta_is_weak():
    """S:119(d) "overlap duty below 1% of the neighbourhood maximum": a column whose raw count
    stays in (0, theta) never has a non-zero Alg. 1 overlap, so after 5 frames its overlap duty
    is still 0 and it has been bumped on every frame (5 x 0.02 above the start), while a column
    that overlaps on every frame without ever winning keeps its permanences."""
    cfg, ora = _hand_sp(period=3, max_boost=1.0)  # boosts stay 1: column 0 keeps winning
    frame = np.zeros((1, 8, 8), np.uint8)
    frame.reshape(-1)[list(range(0, 8)) + list(range(8, 13)) + [16, 17, 18]] = 255
    for _ in range(5):
        r = ora.step(O.encode(frame, cfg)[0], True)
        assert list(r.raw) == [8, 5, 3, 0]
    assert ora.overlap_duty[2] == 0.0 and ora.overlap_duty[1] > 0.5 and ora.active_duty[1] == 0.0
    assert np.all(ora.perm[1] == np.float32(0.21))
    p = np.float32(0.21)
    for _ in range(5):
        p = np.float32(p + np.float32(np.float32(0.1) * np.float32(0.2)))
    assert np.all(ora.perm[2] == p) and np.all(ora.perm[3] == p)


def test_full_learning_radius_after_bump_hand_worked():
    """S:119's order: (d) the bump, THEN (e) the radius from the connected spans, so a synapse
    the bump lifts across tau widens the span the radius sees.  By hand, 64-bit input, C 4,
    S 8, theta 2, k 1, radius 1 in force, period 2; input bits 0..7 and 63 on:
      col 0 pool {0..6, 63}: raw 8, the winner; all its bits on -> stays connected, span 64;
      col 1 pool {0, 9, ..., 63} (step 9): raw 2, eligible, loses -> overlap duty .5, span 64;
      col 2 pool {20..27} at perm 0.19 (< tau, so raw 0 and span 0): overlap duty 0 < 1% of the
            max over its window {1, 2, 3} (.5) -> bumped to 0.19 + 0.02 >= tau: span 8;
      col 3 pool {1, 10, ..., 55, 62}: raw 1 < theta (cut), overlap duty 0, but its window {2, 3}
            has max 0, so it is not weak (0 < 0 is false); span 62.
    radius = floor((sum span + nbits) / (2 nbits)): (64+64+8+62+64)/128 = 2.05 -> 2; computing it
    before the bump would see span 0 for column 2: (190+64)/128 = 1.98 -> 1."""
    cfg = ocfg(num_columns=4, synapses_per_column=8, min_overlap=2, winners_set_size=1,
               inhibition_radius=1, full_learning=True, duty_cycle_period=2)
    idx = np.array([[0, 1, 2, 3, 4, 5, 6, 63], [0, 9, 18, 27, 36, 45, 54, 63],
                    list(range(20, 28)), [1, 10, 19, 28, 37, 46, 55, 62]], np.int64)
    perm = np.full((4, 8), np.float32(0.21), np.float32)
    perm[2] = np.float32(0.19)
    ora = O.SpatialPoolerOracle(cfg, (idx, perm, np.ones(4, np.float32)))
    frame = np.zeros((1, 8, 8), np.uint8)
    frame.reshape(-1)[list(range(8)) + [63]] = 255
    r = ora.step(O.encode(frame, cfg)[0], True)
    assert list(r.raw) == [8, 2, 0, 1] and list(r.active) == [True, False, False, False]
    assert list(ora.overlap_duty) == [0.5, 0.5, 0.0, 0.0]
    p = np.float32(np.float32(0.19) + np.float32(np.float32(0.1) * np.float32(0.2)))
    assert p >= np.float32(0.2) and np.all(ora.perm[2] == p)
    assert np.all(ora.perm[3] == np.float32(0.21))
    assert list(O.connected_span(ora.idx, ora.perm, 0.2)) == [64, 64, 8, 62]
    assert ora.radius == 2


def test_full_learning_off_equals_hot_path_step():
    # full_learning=False leaves boost, duty and radius untouched (regression of the a5 path)
    cfg = ocfg(inhibition_radius=4)
    frames = sp_inputs.frames(1001, 0, 12, 8, 8, rho=0.5)
    ora, _ = _run(cfg, frames)
    assert np.all(ora.boost == 1.0) and ora.radius == 4 and np.all(ora.active_duty == 0)


def test_full_learning_global_keeps_global():
    # configured radius 0 (global) is not adapted (R21)
    cfg = ocfg(full_learning=True, duty_cycle_period=10)
    ora, _ = _run(cfg, sp_inputs.frames(1001, 0, 15, 8, 8, rho=0.5))
    assert ora.radius == 0


def test_full_learning_radius_tracks_spans():
    # after every step the radius equals S:151 evaluated in floating point on the state
    cfg = ocfg(full_learning=True, duty_cycle_period=10, inhibition_radius=80,
               num_columns=96, synapses_per_column=12)
    ora = O.SpatialPoolerOracle(cfg)
    for x in O.encode(sp_inputs.frames(1001, 0, 10, 8, 8, rho=0.5), cfg):
        ora.step(x, True)
        span = O.connected_span(ora.idx, ora.perm, 0.2)
        mean_diam = float(np.mean(span * cfg.num_columns / cfg.input_bits))
        want = min(max(int(math.floor(mean_diam / 2 + 0.5)), 1), cfg.num_columns)
        assert ora.radius == want


def test_full_learning_deterministic():
    cfg = ocfg(full_learning=True, duty_cycle_period=5, inhibition_radius=3)
    frames = sp_inputs.frames(1001, 0, 20, 8, 8, rho=0.5)
    a, ta = _run(cfg, frames)
    b, tb = _run(cfg, frames)
    assert all(np.array_equal(x.active, y.active) for x, y in zip(ta, tb))
    assert np.array_equal(a.perm, b.perm) and np.array_equal(a.boost, b.boost)


# --------------------------------------------------------------------------- #
# per-video SDR histograms (NEXT-4; R22)
# --------------------------------------------------------------------------- #
def test_histogram_spec_examples():
    C = 64
    act = np.zeros((32, C), bool)
    act[:, 3] = True            # active in all 32 frames -> 1.0
    act[::4, 10] = True         # active in 8 of 32 frames -> 0.25
    counts, hist = O.sdr_histograms(act, [0, 32])
    assert hist[0, 3] == 1.0 and hist[0, 10] == 0.25 and counts[0, 10] == 8
    assert np.all(np.delete(hist[0], [3, 10]) == 0.0)
    # empty active sets throughout -> zero vector; an empty video -> zeros (R22)
    counts, hist = O.sdr_histograms(np.zeros((5, C), bool), [0, 5, 5])
    assert np.all(hist == 0) and np.all(counts == 0)


def test_histogram_brute_force_exact_rounding():
    rng = np.random.default_rng(9)
    act = rng.random((200, 96)) < 0.3
    offs = [0, 7, 7, 64, 137, 200]
    counts, hist = O.sdr_histograms(act, offs)
    for v in range(len(offs) - 1):
        seg = act[offs[v]:offs[v + 1]]
        assert np.array_equal(counts[v], seg.sum(axis=0))  # the plain count
        n = len(seg)
        for c in range(96):
            if n == 0:
                assert hist[v, c] == 0
                continue
            exact = Fraction(int(counts[v, c]), n)
            got = Fraction(float(hist[v, c]))
            # correctly rounded: within half an fp32 ulp of the exact ratio
            ulp = Fraction(2) ** (math.frexp(float(hist[v, c]) or 1.0)[1] - 24)
            assert abs(got - exact) <= ulp / 2
