"""CPU oracle of the adaptive video encoder (PAPER.md P:164-168,
SPEC.md S:286-314; readings R23-R25).

TEST INFRASTRUCTURE ONLY (same rule as ``oracle/sp_oracle.py``): imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs; it shares no code with
the CUDA encoder.

"an original video frame is converted to a binary image ... first reduced in size ... the
color image is converted to a grayscale one, which is later binarized using adaptive
thresholding ... 'ADAPTIVE_THRESH_GAUSSIAN_C' algorithm from OpenCV".  The paper
names OpenCV, so the steps follow OpenCV's 8-bit definitions, written out here:

1. downscale (R23): OpenCV ``INTER_AREA``.  Per axis an area table of (dst, src, weight)
   entries is built in double and the weights stored as float32 (OpenCV's
   ``computeResizeAreaTab``); each output value is, in float32 with one rounding per
   operation, ``sum_j beta_j * (sum_k S[sy_j][sx_k] * alpha_k)`` over the table entries in
   order, then rounded half-to-even and saturated to uint8 (``saturate_cast<uchar>``).
   Colour channels are resized independently (BGR order).
2. gray (R24): ``Y = (3735*B + 19235*G + 9798*R + 2^14) >> 15`` (OpenCV 4.x 8-bit
   ``COLOR_BGR2GRAY``; pinned against cv2 over all 2^24 colours).
3. adaptive threshold (R25): T(p) = Gaussian-weighted mean of the k x k neighbourhood
   (replicated borders) - bias; bit = intensity > T (strict).  The mean is
   the one ``cv2.adaptiveThreshold(..., ADAPTIVE_THRESH_GAUSSIAN_C, ...)`` takes: the gray
   image converted to float32, OpenCV's float32 Gaussian kernel (``getGaussianKernel``:
   fixed tables for k <= 9, else exp(-x^2 / (2 sigma^2)) with sigma = fma(k, 0.15, 0.35)
   normalised in double and rounded to float32), a row pass then a column pass in float32
   with one fused multiply-add per tap (the order of OpenCV's AVX2/FMA3 filter: row
   ``s = fma(x_j, k_j, s)`` for j = 0..k-1 from s = 0; column ``s = fma(r_0, k_0, 0)``, then
   ``s = fma(r_+j + r_-j, k_j, s)`` for j = 1..k/2, the pair sum one float32 add), the
   float mean rounded half-to-even and saturated to uint8 (``convertTo``).  The bias enters
   as ceil(bias) (OpenCV's THRESH_BINARY rule), so bit = g - mean > -ceil(bias).  Output
   bytes 255 / 0.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

# OpenCV's fixed small Gaussian kernels for ksize <= 7 and sigma <= 0 (getGaussianKernel)
_SMALL = {1: [1.0], 3: [0.25, 0.5, 0.25], 5: [0.0625, 0.25, 0.375, 0.25, 0.0625],
          7: [0.03125, 0.109375, 0.21875, 0.28125, 0.21875, 0.109375, 0.03125],
          9: [4 / 256, 13 / 256, 30 / 256, 51 / 256, 60 / 256, 51 / 256, 30 / 256, 13 / 256, 4 / 256]}


# --------------------------------------------------------------------------- #
# 1. downscale: INTER_AREA (R23)
# --------------------------------------------------------------------------- #
def area_table(ssize: int, dsize: int):
    """(dst, src, weight float32) entries of one axis, in OpenCV's order."""
    scale = ssize / dsize
    tab = []
    for dx in range(dsize):
        fsx1 = dx * scale
        fsx2 = fsx1 + scale
        cell = min(scale, ssize - fsx1)
        sx1, sx2 = math.ceil(fsx1), math.floor(fsx2)
        sx2 = min(sx2, ssize - 1)
        sx1 = min(sx1, sx2)
        if sx1 - fsx1 > 1e-3:
            tab.append((dx, sx1 - 1, np.float32((sx1 - fsx1) / cell)))
        for sx in range(sx1, sx2):
            tab.append((dx, sx, np.float32(1.0 / cell)))
        if fsx2 - sx2 > 1e-3:
            tab.append((dx, sx2, np.float32(min(min(fsx2 - sx2, 1.0), cell) / cell)))
    return tab


def downscale_area(img: np.ndarray, dst_w: int, dst_h: int) -> np.ndarray:
    """``uint8[H0, W0, ch]`` -> ``uint8[dst_h, dst_w, ch]`` (R23); identity when sizes match."""
    H0, W0, ch = img.shape
    if (dst_w, dst_h) == (W0, H0):
        return img.copy()
    assert dst_w <= W0 and dst_h <= H0, "upscaling is an input error (S:289)"
    xt, yt = area_table(W0, dst_w), area_table(H0, dst_h)
    # the x entries of each dx are consecutive: position p of every dx's list, in order
    per = [[e for e in xt if e[0] == dx] for dx in range(dst_w)]
    P = max(len(l) for l in per)
    XS = np.zeros((P, dst_w), dtype=np.int64)
    XA = np.zeros((P, dst_w), dtype=np.float32)
    XV = np.zeros((P, dst_w), dtype=bool)
    for dx, l in enumerate(per):
        for p_, e in enumerate(l):
            XS[p_, dx], XA[p_, dx], XV[p_, dx] = e[1], e[2], True
    out = np.zeros((dst_h, dst_w, ch), dtype=np.uint8)
    acc = {}
    for dy, sy, beta in yt:
        # buf[dx] = sum over the x entries of dx, in order, one fp32 rounding per operation
        row = img[sy].astype(np.float32)
        buf = np.zeros((dst_w, ch), dtype=np.float32)
        for p_ in range(P):
            add = (row[XS[p_]] * XA[p_][:, None]).astype(np.float32)
            buf = np.where(XV[p_][:, None], (buf + add).astype(np.float32), buf)
        term = (np.float32(beta) * buf).astype(np.float32)
        acc[dy] = term if dy not in acc else (acc[dy] + term).astype(np.float32)
    for dy in range(dst_h):
        out[dy] = np.clip(np.rint(acc[dy]), 0, 255).astype(np.uint8)  # half to even
    return out


# --------------------------------------------------------------------------- #
# 2. gray (R24)
# --------------------------------------------------------------------------- #
def bgr2gray(img: np.ndarray) -> np.ndarray:
    b, g, r = (img[..., i].astype(np.int64) for i in range(3))
    return ((3735 * b + 19235 * g + 9798 * r + (1 << 14)) >> 15).astype(np.uint8)


# --------------------------------------------------------------------------- #
# 3. adaptive threshold, Gaussian (R25)
# --------------------------------------------------------------------------- #
def fma32(a, b, c) -> np.ndarray:
    """float32 fused multiply-add, round(a*b + c) to nearest-even, elementwise.

    a*b of two float32 is exact in float64 (24 + 24 significand bits); s = fl64(a*b + c) with
    its exact error e (TwoSum, so s + e = a*b + c).  Rounding s to float32 equals rounding
    s + e except when s lies exactly halfway between two float32 and e != 0: then the true
    value is on e's side of the midpoint."""
    a = np.asarray(a, np.float32).astype(np.float64)
    b = np.asarray(b, np.float32).astype(np.float64)
    c = np.asarray(c, np.float32).astype(np.float64)
    p = a * b
    s = p + c
    bv = s - p
    e = (p - (s - bv)) + (c - bv)
    r = s.astype(np.float32)
    up = np.nextafter(r, np.float32(np.inf))
    dn = np.nextafter(r, np.float32(-np.inf))
    r64 = r.astype(np.float64)
    to_up = (s == (r64 + up.astype(np.float64)) / 2) & (e > 0)
    to_dn = (s == (r64 + dn.astype(np.float64)) / 2) & (e < 0)
    return np.where(to_up, up, np.where(to_dn, dn, r)).astype(np.float32)


def gaussian_kernel_f32(ksize: int) -> np.ndarray:
    """OpenCV's ``getGaussianKernel(ksize, 0, CV_32F)``: weights in double (sigma =
    fma(ksize, 0.15, 0.35) = 0.3*((ksize-1)/2 - 1) + 0.8, the sum of the outer weights
    doubled plus the centre's 1, each weight times 1/sum), stored as float32."""
    assert ksize % 2 == 1 and ksize >= 3
    if ksize in _SMALL:
        return np.array(_SMALL[ksize], np.float32)
    n2 = ksize // 2
    sigma = float(Fraction(ksize) * Fraction(0.15) + Fraction(0.35))   # one rounding (fma)
    s2 = -0.125 / (sigma * sigma)
    vals = [math.exp(float((2 * i - (ksize - 1)) ** 2) * s2) for i in range(n2)]
    total = 0.0
    for v in vals:
        total += v
    total = total * 2.0 + 1.0
    mul = 1.0 / total
    k = [v * mul for v in vals]
    return np.array(k + [1.0 * mul] + k[::-1], np.float32)


def gaussian_mean_f32(gray: np.ndarray, ksize: int) -> np.ndarray:
    """float32 Gaussian mean of ``uint8[H, W]`` with replicated borders: row pass, then the
    symmetric column pass, one float32 FMA per tap (module docstring, step 3)."""
    k = gaussian_kernel_f32(ksize)
    r = ksize // 2
    H, W = gray.shape
    p = np.pad(gray.astype(np.float32), r, mode="edge")
    rows = np.zeros((H + 2 * r, W), np.float32)
    for j in range(ksize):
        rows = fma32(p[:, j:j + W], k[j], rows)
    mean = fma32(rows[r:r + H], k[r], np.zeros((H, W), np.float32))
    for j in range(1, r + 1):
        pair = (rows[r + j:r + j + H] + rows[r - j:r - j + H]).astype(np.float32)
        mean = fma32(pair, k[r + j], mean)
    return mean


def adaptive_threshold(gray: np.ndarray, ksize: int = 11, bias: float = 2.0) -> np.ndarray:
    """bit = g > round(mean) - ceil(bias), as bytes 255 / 0."""
    m = np.clip(np.rint(gaussian_mean_f32(gray, ksize)), 0, 255).astype(np.int64)  # half to even
    return np.where(gray.astype(np.int64) - m > -math.ceil(bias), 255, 0).astype(np.uint8)


def encode_bgr(frames: np.ndarray, dst_w: int, dst_h: int, ksize: int = 11, bias: float = 2.0):
    """``uint8[F, H0, W0, 3]`` BGR frames -> binarised ``uint8[F, dst_h, dst_w]`` (255 / 0)."""
    out = np.empty((frames.shape[0], dst_h, dst_w), dtype=np.uint8)
    for f in range(frames.shape[0]):
        out[f] = adaptive_threshold(bgr2gray(downscale_area(frames[f], dst_w, dst_h)), ksize, bias)
    return out
