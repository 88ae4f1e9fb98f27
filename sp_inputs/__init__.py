"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the Spatial Pooler's arithmetic. It only produces
the inputs both sides are fed:

* binarised frames (``uint8[F, H, W]``) from a counter-based hash, so that any
  frame can be regenerated independently from its global index (multi-GPU
  shards, oracle re-checks of a sample of a large batch);
* seeded boosts in [1, 2] used to exercise the boost / ranking code (SURVEY
  §8(c) C11: boost is fixed during a run; tests inject seeded values).

Recipe:

    h_f        = splitmix64(seed ^ (f * 0xD1B54A32D192ED03))
    u(f, i)    = splitmix64(h_f ^ i) >> 40            (24-bit uniform)
    pixel(f,i) = value(f, i) if u(f, i) < round(rho * 2**24) else 0

where ``splitmix64(x) = mix64(x + 0x9E3779B97F4A7C15)`` (Steele, Lea & Flood,
"Fast splittable pseudorandom number generators", OOPSLA 2014; constants of
Vigna's splitmix64.c).  ``value`` is 255 (OpenCV ``THRESH_BINARY`` maxval,
PAPER.md P:168) or, with ``nonzero="random"``, an arbitrary non-zero byte so
that the "bit = byte != 0" reading is exercised.

The CUDA side has its own implementation of the same hash (a bench/test
utility kernel, ``sp_synth_frames``); ``tests/test_gpu_parity.py`` checks the
two agree byte for byte.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "GOLDEN_GAMMA",
    "FRAME_MULT",
    "splitmix64",
    "frames",
    "boosts",
    "rho_threshold",
    "bgr_frames",
]

GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
FRAME_MULT = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """splitmix64 as a pure function of a uint64 (array) ``x``: mix64(x + gamma)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN_GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def rho_threshold(rho: float) -> int:
    """24-bit threshold for pixel density ``rho`` (fraction of set pixels)."""
    if not 0.0 <= rho <= 1.0:
        raise ValueError("rho must be in [0, 1]")
    return int(round(rho * (1 << 24)))


def frames(seed: int, first: int, count: int, height: int, width: int,
           rho: float = 0.5, nonzero: str = "255") -> np.ndarray:
    """Frames ``first .. first+count-1`` of the seeded stream, ``uint8[count, H, W]``.

    ``nonzero`` is ``"255"`` (binarised 0/255), ``"1"`` (0/1) or ``"random"``
    (set pixels take a hash-derived value in 1..255).
    """
    n = height * width
    thr = np.uint64(rho_threshold(rho))
    out = np.empty((count, n), dtype=np.uint8)
    pix = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for j in range(count):
            f = np.uint64(first + j)
            hf = splitmix64(np.uint64(seed) ^ (f * FRAME_MULT))
            h = splitmix64(hf ^ pix)
            on = (h >> np.uint64(40)) < thr
            if nonzero == "255":
                val = np.uint8(255)
            elif nonzero == "1":
                val = np.uint8(1)
            elif nonzero == "random":
                val = ((h & np.uint64(0xFF)) | np.uint64(1)).astype(np.uint8)
            else:
                raise ValueError(f"unknown nonzero mode {nonzero!r}")
            out[j] = np.where(on, val, np.uint8(0))
    return out.reshape(count, height, width)


def boosts(seed: int, num_columns: int, lo: float = 1.0, hi: float = 2.0) -> np.ndarray:
    """Seeded float32 boosts, uniform on the fp32 grid of [lo, hi]."""
    if not (1.0 <= lo <= hi < 16.0):
        raise ValueError("boosts must lie in [1, 16)")
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) * FRAME_MULT + np.arange(num_columns, dtype=np.uint64))
    u = (h >> np.uint64(40)).astype(np.float64) / float(1 << 24)  # [0, 1)
    return np.float32(lo) + (np.float32(hi - lo) * u.astype(np.float32))


def bgr_frames(seed: int, first: int, count: int, height: int, width: int) -> np.ndarray:
    """Seeded synthetic colour frames for the encoder (NEXT-3), ``uint8[count, H, W, 3]`` BGR.

    Integer-only recipe: a gradient, a bright disc moving with
    the frame index (the paper's rendered moving shapes), and 5 bits of hash noise:

        base  = ((x * (c + 1)) >> 2) + (y >> 1) + 5 f
              + 128 if (x - cx)^2 + (y - cy)^2 < r^2,  cx = (17 f + 200) % W,
                cy = (11 f + 150) % H, r = min(H, W) // 7
        value = (base + (splitmix64(h_f ^ ((y W + x) 3 + c)) >> 59)) & 255
    """
    f = np.arange(first, first + count, dtype=np.int64)[:, None, None, None]
    y = np.arange(height, dtype=np.int64)[None, :, None, None]
    x = np.arange(width, dtype=np.int64)[None, None, :, None]
    c = np.arange(3, dtype=np.int64)[None, None, None, :]
    cx, cy, r = (17 * f + 200) % width, (11 * f + 150) % height, min(height, width) // 7
    base = ((x * (c + 1)) >> 2) + (y >> 1) + 5 * f
    base = base + np.where((x - cx) ** 2 + (y - cy) ** 2 < r * r, 128, 0)
    out = np.empty((count, height, width, 3), dtype=np.uint8)
    i = ((np.arange(height, dtype=np.uint64)[:, None, None] * np.uint64(width)
          + np.arange(width, dtype=np.uint64)[None, :, None]) * np.uint64(3)
         + np.arange(3, dtype=np.uint64)[None, None, :])
    with np.errstate(over="ignore"):
        for j in range(count):
            hf = splitmix64(np.uint64(seed) ^ (np.uint64(first + j) * FRAME_MULT))
            noise = (splitmix64(hf ^ i) >> np.uint64(59)).astype(np.int64)
            out[j] = ((base[j] + noise) & 255).astype(np.uint8)
    return out
