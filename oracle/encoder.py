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
   OpenCV's bit-exact 8-bit Gaussian blur: sigma = 0.3*((k-1)/2 - 1) + 0.8, the kernel
   quantised to 8 fractional bits by error diffusion (sum exactly 256), a separable row
   then column pass in integers and (acc + 2^15) >> 16; the bias enters as ceil(bias)
   (OpenCV's THRESH_BINARY rule), so bit = g - mean > -ceil(bias).  Output bytes 255 / 0.
"""
from __future__ import annotations

import math

import numpy as np

# OpenCV's fixed small Gaussian kernels for ksize <= 7 and sigma <= 0 (getGaussianKernel)
_SMALL = {1: [1.0], 3: [0.25, 0.5, 0.25], 5: [0.0625, 0.25, 0.375, 0.25, 0.0625],
          7: [0.03125, 0.109375, 0.21875, 0.28125, 0.21875, 0.109375, 0.03125]}


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
def gaussian_kernel_q8(ksize: int):
    """OpenCV's bit-exact 8-bit Gaussian kernel: double weights, then error-diffused
    rounding to 8 fractional bits, centre = 256 - the others."""
    assert ksize % 2 == 1 and ksize >= 3
    n2 = ksize // 2
    if ksize in _SMALL:
        k = _SMALL[ksize]
    else:
        sigma = ksize * 0.15 + 0.35            # = 0.3*((ksize-1)/2 - 1) + 0.8
        s2 = -0.125 / (sigma * sigma)
        vals = [math.exp(float((2 * i - (ksize - 1)) ** 2) * s2) for i in range(n2)]
        total = 2.0 * sum(vals) + 1.0
        k = [v * (1.0 / total) for v in vals]
    q, err = [0] * ksize, 0.0
    for i in range(n2):
        adj = k[i] * 256.0 + err
        v0 = int(np.rint(adj))
        err = adj - v0
        q[i] = q[ksize - 1 - i] = v0
    q[n2] = 256 - 2 * sum(q[:n2])
    return q


def gaussian_mean_u8(gray: np.ndarray, ksize: int) -> np.ndarray:
    """Separable 8-bit Gaussian blur with replicated borders, exact integers."""
    q = gaussian_kernel_q8(ksize)
    r = ksize // 2
    H, W = gray.shape
    p = np.pad(gray.astype(np.int64), r, mode="edge")
    rows = np.zeros((H + 2 * r, W), dtype=np.int64)
    for j in range(ksize):
        rows += q[j] * p[:, j:j + W]
    cols = np.zeros((H, W), dtype=np.int64)
    for j in range(ksize):
        cols += q[j] * rows[j:j + H, :]
    return ((cols + (1 << 15)) >> 16).astype(np.uint8)


def adaptive_threshold(gray: np.ndarray, ksize: int = 11, bias: float = 2.0) -> np.ndarray:
    """bit = g > mean - ceil(bias), as bytes 255 / 0."""
    m = gaussian_mean_u8(gray, ksize).astype(np.int64)
    return np.where(gray.astype(np.int64) - m > -math.ceil(bias), 255, 0).astype(np.uint8)


def encode_bgr(frames: np.ndarray, dst_w: int, dst_h: int, ksize: int = 11, bias: float = 2.0):
    """``uint8[F, H0, W0, 3]`` BGR frames -> binarised ``uint8[F, dst_h, dst_w]`` (255 / 0)."""
    out = np.empty((frames.shape[0], dst_h, dst_w), dtype=np.uint8)
    for f in range(frames.shape[0]):
        out[f] = adaptive_threshold(bgr2gray(downscale_area(frames[f], dst_w, dst_h)), ksize, bias)
    return out
