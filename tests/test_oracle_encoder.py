"""Pins of the encoder oracle (DESIGN R23-R25).

The paper names OpenCV, and OpenCV is installed here as a library: each step of the
oracle is checked against the library routine it restates (an independent implementation),
plus the SPEC's worked examples and properties.  cv2 is never used by the product path.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import encoder as E
import sp_inputs

cv2 = pytest.importorskip("cv2")


def smooth_bgr(h, w, k=0):
    yy, xx = np.mgrid[0:h, 0:w]
    return np.stack([127 + 120 * np.sin(xx / 37.0 + k) * np.cos(yy / 23.0), xx * 255 // w,
                     yy * 255 // h], -1).astype(np.uint8)


# --------------------------------------------------------------------------- #
# R23: INTER_AREA downscale
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("src,dst", [((960, 540), (240, 134)), ((100, 70), (33, 21)),
                                     ((64, 48), (64, 48)), ((61, 37), (7, 5))])
def test_downscale_equals_opencv_inter_area(src, dst):
    rng = np.random.default_rng(sum(src) + sum(dst))
    imgs = [rng.integers(0, 256, (src[1], src[0], 3), dtype=np.uint8), smooth_bgr(src[1], src[0])]
    if src == (960, 540):
        imgs.append(sp_inputs.bgr_frames(4, 7, 1, 540, 960)[0])
    for img in imgs:
        want = cv2.resize(img, dst, interpolation=cv2.INTER_AREA)
        assert np.array_equal(E.downscale_area(img, *dst), want)


def test_downscale_uniform_and_identity():
    # identity dims -> identical; uniform intensity -> same intensity
    img = np.full((54, 96, 3), 77, np.uint8)
    assert np.array_equal(E.downscale_area(img, 24, 13), np.full((13, 24, 3), 77, np.uint8))
    rnd = np.random.default_rng(1).integers(0, 256, (20, 30, 3), dtype=np.uint8)
    assert np.array_equal(E.downscale_area(rnd, 30, 20), rnd)


# --------------------------------------------------------------------------- #
# R24: gray
# --------------------------------------------------------------------------- #
def test_gray_equals_opencv_on_a_colour_cube_sample():
    # every 3rd value per channel: 86^3 colours (the full 2^24 cube agrees too; see DESIGN R24)
    v = np.arange(0, 256, 3)
    b, g, r = np.meshgrid(v, v, v, indexing="ij")
    img = np.stack([b, g, r], -1).astype(np.uint8).reshape(-1, len(v), 3)
    assert np.array_equal(E.bgr2gray(img), cv2.cvtColor(img, cv2.COLOR_BGR2GRAY))


# --------------------------------------------------------------------------- #
# R25: Gaussian mean and adaptive threshold
# --------------------------------------------------------------------------- #
def test_fma32_against_exact_rationals():
    # brute force: the exact a*b + c as a Fraction, rounded to the nearest float32 (ties to
    # even) by comparing the three float32 around it
    rng = np.random.default_rng(3)
    a = (rng.random(3000) * 300).astype(np.float32)
    b = rng.random(3000).astype(np.float32)
    c = (rng.random(3000) * 100 - 20).astype(np.float32)
    # ties: a*b + c exactly halfway between two float32 (c absorbs the low half of a*b)
    a[:200] = np.float32(1 + 2.0 ** -12)
    b[:200] = np.float32(1 + 2.0 ** -12)
    c[:200] = np.float32(0)
    got = E.fma32(a, b, c)
    for i in range(len(a)):
        ex = Fraction(float(a[i])) * Fraction(float(b[i])) + Fraction(float(c[i]))
        f = np.float32(float(ex))
        cands = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
        d = [abs(Fraction(float(x)) - ex) for x in cands]
        best = [x for x, dd in zip(cands, d) if dd == min(d)]
        if len(best) > 1:
            best = [x for x in best if int(x.view(np.uint32)) % 2 == 0]
        assert got[i] == best[0], i


@pytest.mark.parametrize("ksize", [3, 5, 7, 9, 11, 13, 15])
def test_gaussian_kernel_equals_opencv(ksize):
    assert np.array_equal(E.gaussian_kernel_f32(ksize), cv2.getGaussianKernel(ksize, 0, cv2.CV_32F).ravel())


def test_kernel_11_closed_form():
    # sigma = 0.3*((11-1)/2 - 1) + 0.8 = 2.0: w_x = exp(-x^2/8) / sum, |x| <= 5
    w = np.exp(-np.arange(-5, 6) ** 2 / 8.0)
    assert np.allclose(E.gaussian_kernel_f32(11), w / w.sum(), rtol=1e-7, atol=0)


@pytest.mark.parametrize("ksize", [3, 5, 7, 9, 11, 13, 15])
def test_gaussian_mean_equals_opencv_float_blur(ksize):
    # OpenCV's vector path covers rows whose width is a multiple of 16 (240 = the paper's
    # encoded width); the float mean is then bit-equal
    rng = np.random.default_rng(ksize)
    for g in (rng.integers(0, 256, (134, 240), dtype=np.uint8),
              cv2.GaussianBlur(rng.integers(0, 256, (67, 96), dtype=np.uint8), (0, 0), 3)):
        want = cv2.GaussianBlur(g.astype(np.float32), (ksize, ksize), 0,
                                borderType=cv2.BORDER_REPLICATE | cv2.BORDER_ISOLATED)
        assert np.array_equal(E.gaussian_mean_f32(g, ksize).view(np.uint32), want.view(np.uint32))


def test_gaussian_mean_close_to_exact_weighted_mean():
    # independent of OpenCV: the float32 mean is within a few ulp of the exact double sum
    rng = np.random.default_rng(4)
    g = rng.integers(0, 256, (40, 48), dtype=np.uint8)
    k = E.gaussian_kernel_f32(11).astype(np.float64)
    p = np.pad(g.astype(np.float64), 5, mode="edge")
    exact = np.zeros(g.shape)
    for i in range(11):
        for j in range(11):
            exact += k[i] * k[j] * p[i:i + 40, j:j + 48]
    assert np.max(np.abs(E.gaussian_mean_f32(g, 11) - exact)) < 1e-4


@pytest.mark.parametrize("ksize", [3, 5, 7, 9, 11, 13, 15])
def test_threshold_equals_opencv_adaptive_threshold(ksize):
    # the routine P:168 names, zero differing pixels
    rng = np.random.default_rng(5 + ksize)
    for bias in (2.0, 0.0, -3.5, 7.25):
        g = rng.integers(0, 256, (134, 240), dtype=np.uint8)
        want = cv2.adaptiveThreshold(g, 255, cv2.ADAPTIVE_THRESH_GAUSSIAN_C, cv2.THRESH_BINARY, ksize, bias)
        assert np.array_equal(E.adaptive_threshold(g, ksize, bias), want)


def test_spec_examples():
    u = np.full((20, 20), 100, np.uint8)
    assert np.all(E.adaptive_threshold(u, 11, 2.0) == 255)     # uniform, C=2 -> all 1
    assert np.all(E.adaptive_threshold(u, 11, -2.0) == 0)      # C=-2 -> all 0
    # single bright pixel on a dark field -> that bit set, its neighbours 0.  By hand
    # with the 5x5 kernel (1,4,6,4,1)/16: mean at the pixel = round(255*36/256) = 36 < 253;
    # at an edge neighbour round(255*24/256) = 24 and at a corner round(255*16/256) = 16, and
    # 0 - 24, 0 - 16 are not > -2.  Far from the pixel the field is uniform: bits 1.
    d = np.zeros((9, 9), np.uint8)
    d[4, 4] = 255
    out = E.adaptive_threshold(d, 5, 2.0)
    assert out[4, 4] == 255
    ring = out[3:6, 3:6].copy()
    ring[1, 1] = 0
    assert np.all(ring == 0)
    assert out[0, 0] == 255 and out[8, 8] == 255
    m = E.gaussian_mean_f32(d, 5)
    assert m[4, 4] == np.float32(255 * 36 / 256) and m[4, 5] == np.float32(255 * 24 / 256)


def test_shift_covariance_and_monotonicity():
    rng = np.random.default_rng(8)
    g = rng.integers(0, 256, (40, 60), dtype=np.uint8)
    a = E.adaptive_threshold(g, 11, 2.0)
    b = E.adaptive_threshold(np.roll(g, 1, axis=1), 11, 2.0)
    assert np.array_equal(b[6:-6, 7:-6], a[6:-6, 6:-7])        # interior shifts with the image
    for (y, x) in [(10, 10), (20, 33), (0, 0)]:                 # raising a pixel keeps its bit
        h = g.copy()
        h[y, x] = min(255, int(h[y, x]) + 40)
        assert E.adaptive_threshold(h, 11, 2.0)[y, x] >= a[y, x]


def test_encode_pipeline_matches_opencv_chain():
    # the whole chain against cv2 (resize -> gray -> adaptiveThreshold), frames of the
    # synthetic recipe, zero differing pixels
    fr = sp_inputs.bgr_frames(11, 0, 4, 540, 960)
    out = E.encode_bgr(fr, 240, 134)
    for f in range(4):
        g = cv2.cvtColor(cv2.resize(fr[f], (240, 134), interpolation=cv2.INTER_AREA), cv2.COLOR_BGR2GRAY)
        want = cv2.adaptiveThreshold(g, 255, cv2.ADAPTIVE_THRESH_GAUSSIAN_C, cv2.THRESH_BINARY, 11, 2)
        assert np.array_equal(out[f], want)
    assert 0.2 < (out == 255).mean() < 0.95
