"""The device-driven GMRES cycle rotates with a device restatement of glibc's
double hypot (csrc/hobi_gmres.cu glibc_hypot), so its Givens factors round
like np.hypot in the reference (solver.py:551) and std::hypot in the host
loop.  CPU: the same algorithm in Python, operation for operation, equals
np.hypot on sampled pairs (pins the restatement).  GPU: the device function
equals np.hypot bit for bit."""

import math

import numpy as np
import pytest

SCALE, LARGE, TINY, EPS = 2.0**-600, 2.0**511, 2.0**-511, 2.0**-54


def _kernel(ax, ay):
    h = math.sqrt(ax * ax + ay * ay)
    if h <= 2.0 * ay:
        delta = h - ay
        t1 = ax * (2.0 * delta - ax)
        t2 = (delta - 2.0 * (ax - ay)) * delta
    else:
        delta = h - ax
        t1 = 2.0 * delta * (ax - 2.0 * ay)
        t2 = (4.0 * delta - ay) * ay + delta * delta
    return h - (t1 + t2) / (2.0 * h)


def glibc_hypot(x, y):
    if math.isinf(x) or math.isinf(y):
        return math.inf
    if math.isnan(x) or math.isnan(y):
        return x + y
    ax, ay = abs(x), abs(y)
    if ax < ay:
        ax, ay = ay, ax
    if ax > LARGE:
        if ay <= ax * EPS:
            return ax + ay
        return _kernel(ax * SCALE, ay * SCALE) / SCALE
    if ay < TINY:
        if ax >= ay / EPS:
            return ax + ay
        return _kernel(ax * 2.0**600, ay * 2.0**600) * SCALE
    if ay <= ax * EPS:
        return ax + ay
    return _kernel(ax, ay)


def samples(n, seed=1):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    b = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    b[: n // 2] = a[: n // 2] * rng.uniform(0.3, 3.0, n // 2)  # Givens-like pairs
    k = n // 20
    a[:k] *= 2.0**560  # the scaled branches
    b[k:2 * k] *= 2.0**-560
    a[2 * k:3 * k] = 0.0
    return a, b


def test_restatement_equals_numpy_hypot():
    a, b = samples(60000)
    ref = np.hypot(a, b)
    got = np.array([glibc_hypot(float(x), float(y)) for x, y in zip(a, b)])
    assert np.array_equal(got, ref), int(np.sum(got != ref))


@pytest.mark.gpu
def test_device_hypot_equals_numpy_hypot():
    from paper_1301_5914_b200 import _native as N

    a, b = samples(1 << 20, seed=2)
    out = np.empty_like(a)
    N.check(N.load().hobi_hypot_check(0, N.dptr(a), N.dptr(b), a.size, N.dptr(out)))
    ref = np.hypot(a, b)
    assert np.array_equal(out, ref), int(np.sum(out != ref))
