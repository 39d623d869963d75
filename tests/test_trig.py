"""CPU accuracy test of the device sincos (csrc/msurf_trig.cuh), compiled for
the host by build() with -ffp-contract=off: correctly rounded against
mpmath on random samples, and within 1 ulp of glibc everywhere."""

import ctypes
import os

import numpy as np
import pytest

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native", "libtrig_host.so")


def _sincos(x):
    lib = ctypes.CDLL(LIB)
    P = ctypes.POINTER(ctypes.c_double)
    s = np.empty_like(x)
    c = np.empty_like(x)
    lib.msurf_host_sincos_array(x.ctypes.data_as(P), s.ctypes.data_as(P), c.ctypes.data_as(P),
                                ctypes.c_size_t(x.size))
    return s, c


@pytest.mark.skipif(not os.path.exists(LIB), reason="run __graft_entry__.build() first")
def test_sincos_within_one_ulp_of_glibc():
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.uniform(-3000, 10, 400_000), rng.uniform(-1e6, 1e6, 100_000),
                        rng.uniform(-1e-3, 1e-3, 10_000), np.arange(-64, 65) * (np.pi / 4)])
    s, c = _sincos(x)
    for got, ref in ((s, np.sin(x)), (c, np.cos(x))):
        ulp = np.spacing(np.abs(ref))
        assert np.max(np.abs(got - ref) / ulp) <= 1.0
    # mismatch rate vs glibc is glibc's own misrounding (~0.1-0.3 %)
    assert np.mean(s != np.sin(x)) < 0.01


@pytest.mark.skipif(not os.path.exists(LIB), reason="run __graft_entry__.build() first")
def test_sincos_correctly_rounded_vs_mpmath():
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 160
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-3000, 10, 3000), rng.uniform(-1, 1, 500)])
    s, c = _sincos(x)
    bad = 0
    for xi, si, ci in zip(x, s, c):
        m = mpmath.mpf(float(xi))
        bad += float(mpmath.sin(m)) != si
        bad += float(mpmath.cos(m)) != ci
    assert bad == 0
