"""Pins of the CPU oracle against what the paper and the mathematics fix.

Nothing here re-types the oracle's formulas: every check is an independent
route to the same number (brute force, a different formulation, a closed
form, a worked example printed in PAPER.md / SPEC.md, or an invariant).
Citations: PAPER.md = P:n, SPEC.md = S:n, SURVEY.md §8(c) readings = Cn.
"""
import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import sp_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def tiny_cfg(**kw):
    base = dict(input_width=8, input_height=8, num_columns=128, synapses_per_column=16,
                min_overlap=2, winners_set_size=8, inhibition_radius=0, seed=42)
    base.update(kw)
    return O.OracleConfig(**base)


# --------------------------------------------------------------------------- #
# generator (C8) and input recipe
# --------------------------------------------------------------------------- #
def test_splitmix64_reference_vector():
    want = [int(l, 16) for l in open(os.path.join(GOLDEN, "splitmix64_seed0.txt"))
            if l.strip() and not l.startswith("#")]
    s, got = 0, []
    for _ in range(3):
        s, o = O.splitmix64_next(s)
        got.append(o)
    assert got == want
    # the pure-function form used by sp_inputs is the same generator
    assert int(sp_inputs.splitmix64(np.uint64(0))) == want[0]


def test_init_pool_properties():
    cfg = tiny_cfg(num_columns=64, synapses_per_column=24)
    idx, perm, boost = O.init_pools(cfg)
    assert idx.shape == (64, 24)
    for c in range(64):
        row = idx[c]
        assert np.all(np.diff(row) > 0), "ascending and distinct (C8, S:74)"
        assert row.min() >= 0 and row.max() < cfg.input_bits
    assert np.all(perm == np.float32(0.21)) and perm.dtype == np.float32
    assert np.all(boost == 1.0)
    # init perm 0.21 >= threshold 0.2 -> every synapse starts connected
    assert np.all(perm >= np.float32(cfg.connected_threshold))
    # determinism; different seed -> different pools
    idx2, _, _ = O.init_pools(cfg)
    assert np.array_equal(idx, idx2)
    idx3, _, _ = O.init_pools(tiny_cfg(num_columns=64, synapses_per_column=24, seed=43))
    assert not np.array_equal(idx, idx3)


def test_init_pool_full_is_permutation():
    # synapses_per_column == input_size -> a permutation of all inputs
    cfg = tiny_cfg(num_columns=8, synapses_per_column=64)
    idx, _, _ = O.init_pools(cfg)
    for c in range(8):
        assert np.array_equal(idx[c], np.arange(64))


def test_init_pool_uniform():
    # uniform sampling without replacement: every input equally likely (C8).
    cfg = tiny_cfg(num_columns=2000, synapses_per_column=8)
    idx, _, _ = O.init_pools(cfg)
    counts = np.bincount(idx.ravel(), minlength=64)
    expected = 2000 * 8 / 64
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    assert chi2 < 120.0  # dof 63; p ~ 1e-5 threshold


def test_init_first_draw_by_hand():
    # Column 0 of seed 42 (R8): state0 = mix(seed ^ gamma + gamma),
    # first draw u = mix(state0 + gamma), idx = ((u >> 32) * nbits) >> 32.
    cfg = tiny_cfg(num_columns=1, synapses_per_column=1, input_width=1000, input_height=1)
    idx, _, _ = O.init_pools(cfg)
    gamma, m = 0x9E3779B97F4A7C15, (1 << 64) - 1

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)
    state0 = mix(((42 ^ gamma) + gamma) & m)
    u = mix((state0 + gamma) & m)
    assert idx[0, 0] == ((u >> 32) * 1000) >> 32


def test_frames_density_and_modes():
    f = sp_inputs.frames(7, 0, 4, 30, 40, rho=0.25)
    assert f.shape == (4, 30, 40) and f.dtype == np.uint8
    assert set(np.unique(f)) <= {0, 255}
    assert abs((f != 0).mean() - 0.25) < 0.05
    g = sp_inputs.frames(7, 2, 2, 30, 40, rho=0.25)
    assert np.array_equal(f[2:], g), "frames depend only on their global index"
    r = sp_inputs.frames(7, 0, 4, 30, 40, rho=0.25, nonzero="random")
    assert np.array_equal(r != 0, f != 0) and len(np.unique(r)) > 50


# --------------------------------------------------------------------------- #
# encoding (C12, C13)
# --------------------------------------------------------------------------- #
def test_encode_whole_frame_row_major():
    cfg = tiny_cfg(input_width=4, input_height=3, num_columns=4, synapses_per_column=2)
    fr = np.zeros((1, 3, 4), np.uint8)
    fr[0, 1, 2] = 7      # bit 1*4+2 = 6
    fr[0, 2, 0] = 255    # bit 8
    x = O.encode(fr, cfg)
    assert x.shape == (1, 12)
    assert list(np.nonzero(x[0])[0]) == [6, 8]


def test_encode_patches_raster_order():
    cfg = tiny_cfg(input_width=4, input_height=4, patch_width=2, patch_height=2,
                   num_columns=4, synapses_per_column=2)
    fr = np.zeros((1, 4, 4), np.uint8)
    fr[0, 0, 3] = 1   # tile (0,1) -> input 1, local (0,1) -> bit 1
    fr[0, 3, 0] = 9   # tile (1,0) -> input 2, local (1,0) -> bit 2
    fr[0, 3, 3] = 200  # tile (1,1) -> input 3, local (1,1) -> bit 3
    x = O.encode(fr, cfg)
    assert x.shape == (4, 4)
    assert [list(np.nonzero(r)[0]) for r in x] == [[], [1], [2], [3]]


# --------------------------------------------------------------------------- #
# overlap (Alg. 1): three independent routes + SPEC worked examples
# --------------------------------------------------------------------------- #
def _raw_loop(x, idx, perm, tau):
    C, S = idx.shape
    out = []
    for c in range(C):
        n = 0
        for s in range(S):
            if perm[c, s] >= np.float32(tau) and x[idx[c, s]]:
                n += 1
        out.append(n)
    return np.array(out)


def _raw_dense(x, idx, perm, tau):
    C, S = idx.shape
    M = np.zeros((C, len(x)), dtype=np.int64)
    for c in range(C):
        for s in range(S):
            if perm[c, s] >= np.float32(tau):
                M[c, idx[c, s]] += 1
    return M @ x.astype(np.int64)


def _raw_popcount(x, idx, perm, tau):
    xbits = 0
    for i, b in enumerate(x):
        if b:
            xbits |= 1 << i
    out = []
    for c in range(idx.shape[0]):
        m = 0
        for s in range(idx.shape[1]):
            if perm[c, s] >= np.float32(tau):
                m |= 1 << int(idx[c, s])
        out.append(bin(m & xbits).count("1"))
    return np.array(out)


@pytest.mark.parametrize("trial", range(6))
def test_overlap_three_ways(rng, trial):
    nbits = int(rng.integers(20, 200))
    C = int(rng.integers(1, 40))
    S = int(rng.integers(1, min(nbits, 30)))
    idx = np.array([np.sort(rng.choice(nbits, S, replace=False)) for _ in range(C)])
    perm = rng.choice(np.array([0.0, 0.19999993, 0.2, 0.20000002, 0.5, 1.0], np.float32),
                      size=(C, S)).astype(np.float32)
    x = rng.random(nbits) < rng.random()
    got = O.overlap_raw(x, idx, perm, 0.2)
    assert np.array_equal(got, _raw_loop(x, idx, perm, 0.2))
    assert np.array_equal(got, _raw_dense(x, idx, perm, 0.2))
    assert np.array_equal(got, _raw_popcount(x, idx, perm, 0.2))


def test_overlap_spec_examples():
    # S:102 all-zero frame -> all overlaps 0
    idx = np.arange(16).reshape(2, 8)
    perm = np.full((2, 8), np.float32(0.21))
    raw = O.overlap_raw(np.zeros(16, bool), idx, perm, 0.2)
    N, boosted = O.boost_overlap(raw, np.ones(2, np.float32), 8)
    assert np.all(raw == 0) and np.all(boosted == 0)
    # S:103 raw = min_overlap - 1, boost 1 -> 0
    x = np.zeros(16, bool)
    x[:7] = True
    raw = O.overlap_raw(x, idx, perm, 0.2)
    assert raw[0] == 7
    N, boosted = O.boost_overlap(raw, np.ones(2, np.float32), 8)
    assert boosted[0] == 0.0 and N[0] == 0
    # S:104 8 connected synapses on active bits, min_overlap 8, boost 1.5 -> 12.0
    x[:8] = True
    raw = O.overlap_raw(x, idx, perm, 0.2)
    N, boosted = O.boost_overlap(raw, np.array([1.5, 1.0], np.float32), 8)
    assert raw[0] == 8 and boosted[0] == np.float32(12.0) and N[0] == 12 * O.TWO23
    # C1: raw == min_overlap is kept (Alg. 1 uses '<' for the cutoff)
    N, _ = O.boost_overlap(np.array([8]), np.array([1.0], np.float32), 8)
    assert N[0] == 8 * O.TWO23


def test_connected_threshold_exact_values():
    # C3: perm exactly 0.2f is connected, 0.19999993f is not.
    p02 = np.float32(0.1) + np.float32(0.1)          # reachable from 0 by two +0.1f
    assert p02 == np.float32(0.2)
    below = np.nextafter(np.float32(0.2), np.float32(0))
    idx = np.array([[0, 1, 2]])
    perm = np.array([[p02, below, np.nextafter(np.float32(0.2), np.float32(1))]], np.float32)
    raw = O.overlap_raw(np.ones(3, bool), idx, perm, 0.2)
    assert raw[0] == 2


def test_boost_exact_product(rng):
    # C4: N / 2**23 equals raw * boost exactly (rational arithmetic), and the
    # fp32 boosted value is the correctly rounded product (error <= 2**-24 rel).
    b = sp_inputs.boosts(7, 500, 1.0, 15.99)
    raw = rng.integers(0, 1024, 500)
    N, boosted = O.boost_overlap(raw, b, 0)
    for r, bb, n, f in zip(raw, b, N, boosted):
        exact = Fraction(int(r)) * Fraction(float(bb))
        assert Fraction(int(n), O.TWO23) == exact
        if r:
            assert abs(Fraction(float(f)) - exact) <= exact * Fraction(1, 1 << 24)
        # fp32 IEEE product is the correctly rounded exact product
        assert np.float32(r) * bb == f
    # 10 * 1.1f rounds to 11.0 in fp32 but the exact product is larger (H1)
    N, boosted = O.boost_overlap(np.array([10, 11]), np.array([1.1, 1.0], np.float32), 0)
    assert boosted[0] == boosted[1] and N[0] > N[1]


# --------------------------------------------------------------------------- #
# inhibition (Alg. 2)
# --------------------------------------------------------------------------- #
def _brute_inhibit(N, k, r):
    """Full sort per window: c is active iff it is among the first k of
    W(c) sorted by (boosted desc, index asc) and its boosted overlap exceeds 1."""
    C = len(N)
    act = np.zeros(C, bool)
    for c in range(C):
        lo, hi = (0, C - 1) if r == 0 else (max(0, c - r), min(C - 1, c + r))
        order = sorted(range(lo, hi + 1), key=lambda d: (-int(N[d]), d))
        act[c] = order.index(c) < k and N[c] > O.TWO23
    return act


def _random_N(rng, C, ties):
    raw = rng.integers(0, 12, C)
    if ties:
        boost = np.ones(C, np.float32)
    else:
        boost = sp_inputs.boosts(int(rng.integers(1 << 30)), C)
    N, _ = O.boost_overlap(raw, boost, int(rng.integers(0, 4)))
    return N


def test_inhibit_brute_force_500(rng):
    for trial in range(500):
        C = int(rng.integers(1, 33))
        k = int(rng.integers(1, C + 1))
        r = int(rng.integers(0, C + 2))
        N = _random_N(rng, C, ties=(trial % 2 == 0))
        assert np.array_equal(O.inhibit(N, k, r), _brute_inhibit(N, k, r)), (N, k, r)


def test_inhibit_tie_free_equals_paper_literal(rng):
    # C6: on tie-free inputs the tie rule, Alg. 2 literal and brute force agree.
    done = 0
    while done < 200:
        C = int(rng.integers(2, 33))
        N = rng.choice(np.arange(2, 10 * C) * O.TWO23 + rng.integers(0, 100), C, replace=False)
        k, r = int(rng.integers(1, C + 1)), int(rng.integers(0, C))
        a = O.inhibit(N, k, r)
        assert np.array_equal(a, O.inhibit(N, k, r, paper_literal=True))
        assert np.array_equal(a, _brute_inhibit(N, k, r))
        done += 1


def test_inhibit_global_count_invariant(rng):
    # north_star: winner count == min(k, #columns with non-zero overlap) (min_overlap >= 2)
    for _ in range(100):
        C = int(rng.integers(1, 300))
        raw = rng.integers(0, 10, C)
        N, _ = O.boost_overlap(raw, sp_inputs.boosts(int(rng.integers(99)), C), 2)
        k = int(rng.integers(1, C + 1))
        assert O.inhibit(N, k, 0).sum() == min(k, int((N > 0).sum()))


def test_inhibit_special_cases():
    T = O.TWO23
    # S:133 all zero -> empty
    assert not O.inhibit(np.zeros(16, np.int64), 4, 0).any()
    # S:112 single non-zero column, n = 1 -> active
    N = np.zeros(16, np.int64)
    N[5] = 5 * T
    assert list(np.nonzero(O.inhibit(N, 1, 0))[0]) == [5]
    # all equal -> the k lowest indices (C6, supersedes S:113) ...
    N = np.full(16, 10 * T, np.int64)
    assert list(np.nonzero(O.inhibit(N, 3, 0))[0]) == [0, 1, 2]
    # ... and S:113 holds in paper-literal mode: nobody strictly exceeds a tie
    assert not O.inhibit(N, 3, 0, paper_literal=True).any()
    # S:114 fewer than n non-zero neighbours -> threshold is 1
    N = np.zeros(16, np.int64)
    N[[2, 9]] = [3 * T, 2 * T]
    assert list(np.nonzero(O.inhibit(N, 4, 3))[0]) == [2, 9]
    # C7 floor: boosted overlap exactly 1 never wins
    N = np.array([T, 0], np.int64)
    assert not O.inhibit(N, 2, 0).any()
    # C16: SPEC's per-neighbourhood sparsity bound is false for local inhibition
    N = np.array([5 * T, 0, 5 * T], np.int64)
    assert list(np.nonzero(O.inhibit(N, 1, 1))[0]) == [0, 2]


def test_inhibit_radius_covering_all_is_global(rng):
    for _ in range(50):
        C = int(rng.integers(1, 64))
        N = _random_N(rng, C, ties=True)
        k = int(rng.integers(1, C + 1))
        assert np.array_equal(O.inhibit(N, k, C - 1 if C > 1 else 1), O.inhibit(N, k, 0))


def test_inhibit_boost_monotone(rng):
    # S:141 raising one column's boost cannot remove it from the active set
    for _ in range(100):
        C = 24
        raw = rng.integers(0, 10, C)
        b = sp_inputs.boosts(int(rng.integers(1000)), C)
        c = int(rng.integers(C))
        N1, _ = O.boost_overlap(raw, b, 2)
        b2 = b.copy()
        b2[c] = np.float32(min(15.0, float(b[c]) * 1.5))
        N2, _ = O.boost_overlap(raw, b2, 2)
        if O.inhibit(N1, 5, 4)[c]:
            assert O.inhibit(N2, 5, 4)[c]


# --------------------------------------------------------------------------- #
# learning (C3, C10)
# --------------------------------------------------------------------------- #
def test_learn_closed_form_and_examples():
    idx = np.array([[0, 1, 2], [0, 1, 2]])
    perm = np.array([[0.95, 0.05, 0.5], [0.3, 0.3, 0.3]], np.float32)
    x = np.array([True, False, True])
    out = O.learn(perm, idx, x, np.array([True, False]), 0.1, 0.1)
    assert out[0, 0] == np.float32(1.0)           # S:122 clamp 0.95 + 0.1 -> 1.0
    assert out[0, 1] == np.float32(0.0)           # 0.05 - 0.1 -> clamp 0
    assert out[0, 2] == np.float32(0.5) + np.float32(0.1)
    assert np.array_equal(out[1], perm[1])        # S:123 inactive unchanged
    assert out.dtype == np.float32


def test_learn_reachable_values_cross_threshold():
    # C3: starting at 0.21, the fp32 walk reaches values just below and at 0.2.
    seen = set()
    frontier = {np.float32(0.21)}
    inc = dec = np.float32(0.1)
    for _ in range(30):
        nxt = set()
        for p in frontier:
            for q in (p + inc, p - dec):
                q = np.float32(min(np.float32(1), max(np.float32(0), np.float32(q))))
                if q not in seen:
                    nxt.add(q)
        seen |= nxt
        frontier = nxt
    vals = sorted(float(v) for v in seen)
    # 36 reachable values; three of them straddle tau = 0.2f
    assert len(vals) == 36
    near = sorted(v for v in seen if 0.19 < v < 0.21)
    assert near == [np.float32(0.19999993), np.float32(0.2), np.float32(0.20000002)]
    assert near[0] < np.float32(0.2) <= near[1] < near[2]
    # and the oracle's learn() walks the same lattice: 0.21 -> -0.1 -> +0.1 ...
    idx, x = np.array([[0]]), np.array([False])
    p = np.array([[0.21]], np.float32)
    p = O.learn(p, idx, x, np.array([True]), 0.1, 0.1)
    assert p[0, 0] == np.float32(0.21) - np.float32(0.1)
    assert all(0.0 <= v <= 1.0 for v in vals)


def test_permanence_closure_stream():
    # S:138 permanences stay in [0,1] through a learning stream; determinism S:139
    cfg = tiny_cfg()
    frames = sp_inputs.frames(1001, 0, 10, 8, 8)
    a, b = O.SpatialPoolerOracle(cfg), O.SpatialPoolerOracle(cfg)
    ra, rb = a.compute(frames, True), b.compute(frames, True)
    assert all(np.array_equal(x.active, y.active) for x, y in zip(ra, rb))
    assert np.array_equal(a.perm, b.perm)
    assert a.perm.min() >= 0 and a.perm.max() <= 1
    # learning changed only winners' rows
    assert not np.array_equal(a.perm, O.init_pools(cfg)[1])


def test_learn_false_is_pure():
    cfg = tiny_cfg()
    sp = O.SpatialPoolerOracle(cfg)
    fr = sp_inputs.frames(2002, 0, 1, 8, 8)
    r1 = sp.compute(fr, False)[0]
    r2 = sp.compute(fr, False)[0]
    assert np.array_equal(r1.active, r2.active)
    assert np.array_equal(sp.perm, O.init_pools(cfg)[1])


def test_sdr_words():
    act = np.zeros(70, bool)
    act[[0, 31, 32, 69]] = True
    w = O.sdr_words(act)
    assert list(w) == [0x80000001, 0x1, 0x20]


# --------------------------------------------------------------------------- #
# regression pin: tiny-config trace (SURVEY §8(c) determinism)
# --------------------------------------------------------------------------- #
def test_tiny_trace_golden():
    path = os.path.join(GOLDEN, "tiny_trace.json")
    gold = json.load(open(path))
    from scripts.make_golden import tiny_trace_digest
    assert tiny_trace_digest() == gold["sha256"]
