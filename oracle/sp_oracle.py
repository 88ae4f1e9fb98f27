"""CPU oracle for the HTM Spatial Pooler hot path (arxiv 1608.01966).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_1608_01966_b200``) never imports, calls or
links it, and this module never imports the product path: the two share no
code, tables or helpers.  The only common dependency is ``sp_inputs`` (seeded
frames and boosts; no SP arithmetic).

What it computes is the plain definition, step by step, in the paper's order
(PAPER.md = P:n, SPEC.md = S:n, SURVEY.md §8(c) readings C1..C16):

1. encode   : bit = (byte != 0), row-major; patch mode: tiles in raster order,
              row-major inside the tile                      (C12, C13)
2. overlap  : raw[c] = sum_s [perm[c,s] >= tau] * x[idx[c,s]]     (Alg. 1 l.1-5)
3. cutoff   : raw < min_overlap -> 0 ; else raw * boost         (Alg. 1 l.6-10; C1)
              The product is kept EXACTLY as the integer N = raw * Bc over 2**23,
              Bc = boost * 2**23 (an integer for fp32 boost in [1,16); C4).
4. inhibit  : active[c] = N[c] > 2**23  (Alg. 2's max(., 1), C7)  and
              #{d in W(c), d != c : (N[d], -d) > (N[c], -c)} < k      (Alg. 2, P:77-90;
              C5 self excluded, C6 ties to the lower index, C9 window)
5. learn    : for every active column and every potential synapse:
              perm = clamp01(fp32(perm + inc)) if x else clamp01(fp32(perm - dec))
                                                        (P:92 -> whitepaper; S:119(a); C3, C10)
   full learning (NEXT-1, ``full_learning=True``; S:119(b-e); DESIGN R17-R21),
   after (a), in this order:
     (b) duty cycles, every column, fp32:  d = (d * (P-1) + a) / P   with
         a = active[c] (active duty) and a = N[c] > 0 (overlap duty)
     (c) boost from the active duty cycle: minA = 0.01 * max(adc over W(c));
         boost = 1 if adc >= minA else 1 + ((minA - adc) / minA) * (max_boost - 1)
     (d) weak-column bump: odc < 0.01 * max(odc over W(c)) -> every potential synapse
         perm = min(1, perm + 0.1 * tau)
     (e) inhibition radius (only when the configured radius is > 0):
         r = clamp(round(mean_c(span_c * C / nbits) / 2), 1, C), span_c = max - min + 1
         of the connected synapses' input indices (0 if none), evaluated exactly
   W(c) is the window of the radius in force for this input (global when 0).
6. output   : the active set / SDR bitmask (bit c of word c // 32, LSB first).
7. histogram: per video v (SP inputs [off[v], off[v+1])), counts[v, c] = #inputs where c is
              active, hist = fp32(count) / fp32(n) (NEXT-4, DESIGN R22)

Initialisation ("random initialization", P:245 init perm; C8 as amended
in DESIGN.md R8): per column c a splitmix64 stream whose state starts at
``splitmix64(seed ^ ((c+1) * 0x9E3779B97F4A7C15))`` (the mixed value: using the
XOR directly as the state puts columns on one shared state lattice); draw
``idx = ((u >> 32) * nbits) >> 32``, reject duplicates until S distinct, sort
ascending; perm = initial_permanence (fp32), boost = 1.0.

Precision: counts are int64, permanences fp32 (C3: the paper never states the
format; fp32 with one IEEE RN add then clamp is the reading), ranking exact
integers (C4).  Every function is pinned by ``tests/test_oracle_pins.py``
against closed forms, brute force and the paper's/SPEC's worked examples.
Functions without an independent pin: none (the determinism golden hash is a
regression pin only, SURVEY §8(c) "What pins each part").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
import math

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
TWO23 = 1 << 23


# --------------------------------------------------------------------------- #
# configuration (Tab. 2)
# --------------------------------------------------------------------------- #
@dataclass
class OracleConfig:
    input_width: int
    input_height: int
    num_columns: int = 2048            # Tab. 2 "No. of columns"
    synapses_per_column: int = 128     # Tab. 2 "No. of synapses per column"
    min_overlap: int = 8               # Tab. 2 "Min overlap"
    winners_set_size: int = 40         # Tab. 2 "Winners set size"
    inhibition_radius: int = 0         # 0 = global (C9); Tab. 2's initial radius is 80
    perm_increment: float = 0.1        # Tab. 2 "Perm value increment"
    perm_decrement: float = 0.1        # Tab. 2 "Perm value decrement"
    initial_permanence: float = 0.21   # Tab. 2 "Initial perm value"
    connected_threshold: float = 0.2   # C2 (not stated in the paper)
    patch_width: int = 0               # 0 = whole frame is one SP input (C13)
    patch_height: int = 0
    seed: int = 42
    # full learning (NEXT-1; S:119(b-e))
    full_learning: bool = False
    duty_cycle_period: int = 1000      # S:150 "window duty_cycle_period (alpha = 1/period)"
    max_boost: float = 2.0             # S:149 "max_boost"; 2.0

    @property
    def patch(self):
        if self.patch_width == 0 and self.patch_height == 0:
            return self.input_width, self.input_height
        return self.patch_width, self.patch_height

    @property
    def input_bits(self) -> int:
        pw, ph = self.patch
        return pw * ph

    @property
    def inputs_per_frame(self) -> int:
        pw, ph = self.patch
        return (self.input_width // pw) * (self.input_height // ph)


# --------------------------------------------------------------------------- #
# initialisation (C8)
# --------------------------------------------------------------------------- #
def splitmix64_next(state: int):
    """One step of Vigna's splitmix64: returns (new_state, output)."""
    state = (state + GAMMA) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def init_pools(cfg: OracleConfig):
    """Potential pools, permanences and boosts at creation (C8).

    Returns ``idx int64[C, S]`` (ascending per column), ``perm float32[C, S]``
    (all ``initial_permanence``) and ``boost float32[C]`` (all 1.0).
    """
    C, S, nbits = cfg.num_columns, cfg.synapses_per_column, cfg.input_bits
    idx = np.empty((C, S), dtype=np.int64)
    for c in range(C):
        _, state = splitmix64_next((cfg.seed ^ (((c + 1) * GAMMA) & MASK64)) & MASK64)
        chosen = []
        seen = set()
        while len(chosen) < S:
            state, u = splitmix64_next(state)
            i = ((u >> 32) * nbits) >> 32
            if i not in seen:
                seen.add(i)
                chosen.append(i)
        idx[c] = sorted(chosen)
    perm = np.full((C, S), np.float32(cfg.initial_permanence), dtype=np.float32)
    boost = np.ones(C, dtype=np.float32)
    return idx, perm, boost


# --------------------------------------------------------------------------- #
# step 1: encoding of frames into SP inputs (C12, C13)
# --------------------------------------------------------------------------- #
def encode(frames: np.ndarray, cfg: OracleConfig) -> np.ndarray:
    """``uint8[F, H, W]`` -> ``bool[F * P, nbits]``: bit = byte != 0 (C12).

    Whole-frame mode: one input per frame, bit index y*W + x.
    Patch mode: tiles of ``patch_width x patch_height`` in raster order, each
    an SP input with bit index y*pw + x inside the tile (C13).
    """
    F, H, W = frames.shape
    assert (W, H) == (cfg.input_width, cfg.input_height)
    pw, ph = cfg.patch
    bits = frames != 0
    tiles = []
    for f in range(F):
        for ty in range(H // ph):
            for tx in range(W // pw):
                tiles.append(bits[f, ty * ph:(ty + 1) * ph, tx * pw:(tx + 1) * pw].reshape(-1))
    return np.array(tiles, dtype=bool).reshape(F * (H // ph) * (W // pw), pw * ph)


# --------------------------------------------------------------------------- #
# steps 2-3: overlap (Alg. 1)
# --------------------------------------------------------------------------- #
def overlap_raw(x: np.ndarray, idx: np.ndarray, perm: np.ndarray, tau: float) -> np.ndarray:
    """Alg. 1 lines 1-5: count of connected synapses on active bits.

    connected = perm >= tau in fp32 (C2, C3).
    """
    connected = perm >= np.float32(tau)
    active_input = x[idx]
    return (connected & active_input).sum(axis=1).astype(np.int64)


def boost_integer(boost: np.ndarray) -> np.ndarray:
    """Bc = boost * 2**23 as an exact integer (fp32 boost in [1,16); C4)."""
    b = np.asarray(boost, dtype=np.float32).astype(np.float64) * float(TWO23)
    bc = b.astype(np.int64)
    assert np.all(bc.astype(np.float64) == b), "boost * 2**23 must be an integer"
    return bc


def boost_overlap(raw: np.ndarray, boost: np.ndarray, min_overlap: int):
    """Alg. 1 lines 6-10: cutoff on the RAW count (C1), then boost.

    Returns ``(N, boosted)``: N = exact boosted overlap times 2**23 (int64),
    boosted = the fp32 value nearest to N / 2**23 (C4).
    """
    eligible = raw >= min_overlap
    N = np.where(eligible, raw * boost_integer(boost), 0).astype(np.int64)
    boosted = (N.astype(np.float64) / float(TWO23)).astype(np.float32)
    return N, boosted


# --------------------------------------------------------------------------- #
# step 4: inhibition (Alg. 2)
# --------------------------------------------------------------------------- #
def neighbourhood(c: int, num_columns: int, radius: int):
    """W(c): all columns (radius 0, global) or |d - c| <= radius, truncated (C9)."""
    if radius == 0:
        return 0, num_columns - 1
    return max(0, c - radius), min(num_columns - 1, c + radius)


def inhibit(N: np.ndarray, k: int, radius: int, paper_literal: bool = False) -> np.ndarray:
    """Alg. 2 with the readings C5 (self excluded), C6 (ties), C7 (floor).

    active[c] iff N[c] > 2**23 (boosted overlap > 1) and fewer than k columns
    d != c of W(c) beat c.  "Beat" is the total order (N desc, index asc) (C6);
    with ``paper_literal`` it is ``N[d] >= N[c]`` (strict '>' of Alg. 2 l.3,
    ties lose; used only for the tie-free cross-check).
    """
    C = len(N)
    active = np.zeros(C, dtype=bool)
    cols = np.arange(C)
    for c in range(C):
        lo, hi = neighbourhood(c, C, radius)
        d = cols[lo:hi + 1]
        nd = N[lo:hi + 1]
        if paper_literal:
            beats = (nd >= N[c]) & (d != c)
        else:
            beats = (nd > N[c]) | ((nd == N[c]) & (d < c))
        active[c] = (N[c] > TWO23) and (int(beats.sum()) < k)
    return active


# --------------------------------------------------------------------------- #
# step 5: learning (P:92 -> whitepaper; S:119(a); C3, C10)
# --------------------------------------------------------------------------- #
def learn(perm: np.ndarray, idx: np.ndarray, x: np.ndarray, active: np.ndarray,
          inc: float, dec: float) -> np.ndarray:
    """Permanence update of the winning columns; returns the new fp32 array."""
    out = perm.copy()
    inc32, dec32 = np.float32(inc), np.float32(dec)
    for c in np.nonzero(active)[0]:
        on = x[idx[c]]
        p = out[c]
        upd = np.where(on, p + inc32, p - dec32).astype(np.float32)
        out[c] = np.minimum(np.maximum(upd, np.float32(0.0)), np.float32(1.0))
    return out


# --------------------------------------------------------------------------- #
# full learning, steps (b)-(e) (NEXT-1; S:119(b-e); DESIGN R17-R21)
# --------------------------------------------------------------------------- #
MIN_PCT = np.float32(0.01)  # S:149 "0.01 x max"; S:119(d) "below 1% of ..."
BUMP_PCT = np.float32(0.1)  # S:119(d) "0.1 x connected_threshold"


def update_duty(duty: np.ndarray, flag: np.ndarray, period: int) -> np.ndarray:
    """(b) moving average with window ``period`` (alpha = 1/period), fp32 (R17):
    d' = fp32(fp32(fp32(d * (P-1)) + a) / P), one IEEE RN operation at a time."""
    d = np.asarray(duty, dtype=np.float32)
    t = (d * np.float32(period - 1)).astype(np.float32)
    t = (t + np.asarray(flag, dtype=np.float32)).astype(np.float32)
    return (t / np.float32(period)).astype(np.float32)


def window_max(v: np.ndarray, radius: int) -> np.ndarray:
    """max of v over W(c) = the neighbourhood of c INCLUDING c (C9; R18); radius 0 = global."""
    C = len(v)
    out = np.empty(C, dtype=v.dtype)
    for c in range(C):
        lo, hi = neighbourhood(c, C, radius)
        out[c] = v[lo:hi + 1].max()
    return out


def boost_from_duty(adc: np.ndarray, radius: int, max_boost: float) -> np.ndarray:
    """(c) S:149: minA = 0.01 * neighbourhood max of the active duty cycle; boost = 1 if
    adc >= minA, else 1 + (minA - adc) / minA * (max_boost - 1); fp32, in that order (R19)."""
    adc = np.asarray(adc, dtype=np.float32)
    minA = (MIN_PCT * window_max(adc, radius)).astype(np.float32)
    mb1 = np.float32(np.float32(max_boost) - np.float32(1.0))
    boost = np.ones(len(adc), dtype=np.float32)
    for c in range(len(adc)):
        if adc[c] < minA[c]:
            t1 = np.float32(minA[c] - adc[c])
            t2 = np.float32(t1 / minA[c])
            t3 = np.float32(t2 * mb1)
            boost[c] = np.float32(np.float32(1.0) + t3)
    return boost


def bump_weak(perm: np.ndarray, odc: np.ndarray, radius: int, tau: float):
    """(d) S:119(d): columns whose overlap duty cycle is below 1% of their neighbourhood
    maximum get every permanence raised by 0.1 * tau, clamped to 1 (fp32, R20).
    Returns (new perm, weak mask)."""
    odc = np.asarray(odc, dtype=np.float32)
    minO = (MIN_PCT * window_max(odc, radius)).astype(np.float32)
    weak = odc < minO
    bump = np.float32(BUMP_PCT * np.float32(tau))
    out = perm.copy()
    for c in np.nonzero(weak)[0]:
        out[c] = np.minimum((out[c] + bump).astype(np.float32), np.float32(1.0))
    return out, weak


def connected_span(idx: np.ndarray, perm: np.ndarray, tau: float) -> np.ndarray:
    """span_c = max - min + 1 over the input indices of c's connected synapses, 0 if none
    ("connected-synapse input span"; R21)."""
    C = idx.shape[0]
    span = np.zeros(C, dtype=np.int64)
    conn = perm >= np.float32(tau)
    for c in range(C):
        sel = idx[c][conn[c]]
        if len(sel):
            span[c] = int(sel.max()) - int(sel.min()) + 1
    return span


def adapt_radius(span: np.ndarray, nbits: int, num_columns: int) -> int:
    """(e) S:151: radius = clamp(round(mean_c(span_c * C / nbits) / 2), 1, C), evaluated as
    an exact rational (R21): mean_c(span_c * C / nbits) / 2 = sum(span) / (2 * nbits);
    round half up."""
    q = Fraction(int(np.sum(span, dtype=np.int64)), 2 * nbits)
    r = math.floor(q + Fraction(1, 2))
    return int(min(max(r, 1), num_columns))


def sdr_words(active: np.ndarray) -> np.ndarray:
    """Active flags -> uint32 words, bit c of word c // 32 (LSB first)."""
    C = len(active)
    words = np.zeros((C + 31) // 32, dtype=np.uint32)
    for c in np.nonzero(active)[0]:
        words[c // 32] |= np.uint32(1) << np.uint32(c % 32)
    return words


# --------------------------------------------------------------------------- #
# step 7: per-video SDR histograms (NEXT-4, DESIGN R22)
# --------------------------------------------------------------------------- #
def sdr_histograms(active: np.ndarray, offsets):
    """``active bool[n, C]`` (the winners of n consecutive SP inputs), ``offsets`` of V+1
    ascending input indices -> ``(counts int64[V, C], hist float32[V, C])``.

    "Histograms of consecutive frames are built from SP output on a per-video basis"
    (P:118); counts[c] = (#frames where c active) / frames.  Normalisation is one
    fp32 IEEE division fp32(count) / fp32(n); a video with no inputs gives zeros (R22).
    """
    active = np.asarray(active, dtype=bool)
    V = len(offsets) - 1
    C = active.shape[1]
    counts = np.zeros((V, C), dtype=np.int64)
    hist = np.zeros((V, C), dtype=np.float32)
    for v in range(V):
        lo, hi = int(offsets[v]), int(offsets[v + 1])
        for i in range(lo, hi):
            counts[v] += active[i]
        if hi > lo:
            hist[v] = (counts[v].astype(np.float32) / np.float32(hi - lo)).astype(np.float32)
    return counts, hist


# --------------------------------------------------------------------------- #
# the whole step, and a stateful wrapper
# --------------------------------------------------------------------------- #
@dataclass
class StepResult:
    raw: np.ndarray
    N: np.ndarray
    boosted: np.ndarray
    active: np.ndarray


class SpatialPoolerOracle:
    """Stateful oracle SP; ``compute`` mirrors ``sp_compute``."""

    def __init__(self, cfg: OracleConfig, state=None):
        self.cfg = cfg
        if state is None:
            self.idx, self.perm, self.boost = init_pools(cfg)
        else:
            idx, perm, boost = state
            self.idx = np.asarray(idx, dtype=np.int64).copy()
            self.perm = np.asarray(perm, dtype=np.float32).copy()
            self.boost = np.asarray(boost, dtype=np.float32).copy()
        # full-learning state ("duty cycles = 0; inhibition_radius = initial")
        self.active_duty = np.zeros(cfg.num_columns, dtype=np.float32)
        self.overlap_duty = np.zeros(cfg.num_columns, dtype=np.float32)
        self.radius = int(cfg.inhibition_radius)
        self.iteration = 0

    def step(self, x: np.ndarray, learning: bool, paper_literal: bool = False) -> StepResult:
        cfg = self.cfg
        raw = overlap_raw(x, self.idx, self.perm, cfg.connected_threshold)
        N, boosted = boost_overlap(raw, self.boost, cfg.min_overlap)
        active = inhibit(N, cfg.winners_set_size, self.radius, paper_literal)
        if learning:
            self.perm = learn(self.perm, self.idx, x, active,
                              cfg.perm_increment, cfg.perm_decrement)          # (a)
            if cfg.full_learning:
                P = cfg.duty_cycle_period
                self.active_duty = update_duty(self.active_duty, active, P)   # (b)
                self.overlap_duty = update_duty(self.overlap_duty, N > 0, P)
                self.boost = boost_from_duty(self.active_duty, self.radius,   # (c)
                                             cfg.max_boost)
                self.perm, _ = bump_weak(self.perm, self.overlap_duty,        # (d)
                                         self.radius, cfg.connected_threshold)
                if cfg.inhibition_radius > 0:                                  # (e)
                    span = connected_span(self.idx, self.perm, cfg.connected_threshold)
                    self.radius = adapt_radius(span, cfg.input_bits, cfg.num_columns)
            self.iteration += 1
        return StepResult(raw, N, boosted, active)

    def compute(self, frames: np.ndarray, learning: bool):
        """Frames -> list of StepResult, inputs processed sequentially in order."""
        xs = encode(frames, self.cfg)
        return [self.step(x, learning) for x in xs]
