"""Pins of the multiresolution oracle (O15 upsample2, O16 bin2).

Both oracles (naive-sum C, numpy FFT) are checked against things other than themselves:
* a pure tone's interpolant in closed form, e^{2 pi i fbar (m - 1/2)/(2L)} per axis (phase
  convention, half-pixel offset of reading R1, Nyquist bin, normalisation);
* Parseval: ||upsample2(x)||^2 = 4 ||x||^2 (the interpolant keeps the band);
* the 2x2 block MEAN of an upsampled tone is the tone times cos(pi fbar_x / 2L) cos(pi fbar_y / 2L)
  -- real, no phase: binning (O16's blocks) and upsampling (O15's 2n + 1/2) are registered;
* bin2: block-constant input -> plain decimation; total intensity conserved (4 sum a_c^2 = sum a_f^2).
"""
import numpy as np
import pytest

import oracle
from oracle import np_oracle as npo


def fb(f, L):
    return f if f < L // 2 else f - L


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("fy,fx", [(0, 0), (1, 3), (7, 2), (8, 8), (13, 4), (8, 1)])
def test_upsample2_tone_closed_form(impl, fy, fx):
    L = 16
    n = np.arange(L)
    x = np.exp(2j * np.pi * (fy * n[:, None] + fx * n[None, :]) / L)
    y = oracle.upsample2(x) if impl == "c" else npo.upsample2(x)
    m = np.arange(2 * L) - 0.5
    ref = np.exp(2j * np.pi * (fb(fy, L) * m[:, None] + fb(fx, L) * m[None, :]) / (2 * L))
    assert np.max(np.abs(y - ref)) < 1e-12


@pytest.mark.parametrize("L", [8, 16])
def test_upsample2_parseval_and_c_equals_numpy(L):
    rng = np.random.default_rng(L)
    x = rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L))
    yc, yn = oracle.upsample2(x), npo.upsample2(x)
    assert np.linalg.norm(yc - yn) <= 1e-12 * np.linalg.norm(yn)
    assert abs(np.vdot(yc, yc).real - 4 * np.vdot(x, x).real) <= 1e-11 * np.vdot(x, x).real


def test_block_mean_of_upsampled_tone_is_zero_phase_lowpass():
    L = 16
    n = np.arange(L)
    for fy, fx in [(3, 5), (15, 1), (8, 2)]:
        x = np.exp(2j * np.pi * (fy * n[:, None] + fx * n[None, :]) / L)
        y = oracle.upsample2(x)
        bm = 0.25 * (y[0::2, 0::2] + y[1::2, 0::2] + y[0::2, 1::2] + y[1::2, 1::2])
        g = np.cos(np.pi * fb(fy, L) / (2 * L)) * np.cos(np.pi * fb(fx, L) / (2 * L))
        assert np.max(np.abs(bm - g * x)) < 1e-12


@pytest.mark.parametrize("impl", ["c", "np"])
def test_bin2_pins(impl):
    rng = np.random.default_rng(3)
    f = (lambda a: oracle.bin2(a)) if impl == "c" else (lambda a: npo.bin2(a))
    blocks = rng.uniform(0.5, 2.0, size=(3, 6, 6))
    a = np.repeat(np.repeat(blocks, 2, axis=1), 2, axis=2)  # block-constant
    assert np.max(np.abs(f(a) - blocks)) < 1e-15
    a = rng.uniform(0.0, 3.0, size=(2, 10, 10))
    c = f(a)
    assert c.shape == (2, 5, 5)
    assert abs(4 * np.sum(c ** 2) - np.sum(a ** 2)) < 1e-12 * np.sum(a ** 2)
    assert np.all(c >= np.min(a)) and np.all(c <= np.max(a))
