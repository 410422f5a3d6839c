"""The restated glibc pow (csrc/glibc_pow.cuh) against the live libm `pow`
(Python's float ** is glibc pow, as numba's llvm.pow.f64 is): bit-identical
on the opacity-correction domain (x = 1 - alpha in [0, 1], y = s/s1 >= 1)
and beyond.  Host restatement on CPU; the device copy under -m gpu."""

import ctypes as C

import numpy as np
import pytest


@pytest.fixture(scope="module")
def L(built_lib):
    from paper_1908_01906_b200 import _lib
    if not _lib.lib().tr_pow_glibc_available():
        pytest.skip("glibc pow tables not found in this libm")
    return _lib


def _args(n, seed):
    rng = np.random.default_rng(seed)
    x = np.concatenate([
        rng.uniform(0.0, 1.0, n),                       # 1 - alpha
        1.0 - rng.uniform(0.0, 1e-6, n // 8),           # alpha ~ 0
        rng.uniform(0.0, 1e-3, n // 8),                 # alpha ~ 1
        1.0 - rng.integers(1, 1 << 20, n // 8) * 2.0 ** -53,
        np.exp(rng.uniform(-700, 700, n // 8)),          # wide range
        np.array([1.0, 0.5, 2.0 ** -53, 0.75, 0.9999]),
    ])
    y = np.concatenate([
        rng.uniform(1.0, 8.0, n), rng.uniform(1.0, 8.0, n // 8), rng.uniform(1.0, 8.0, n // 8),
        rng.uniform(1.0, 32.0, n // 8), rng.uniform(0.01, 4.0, n // 8),
        np.array([2.0, 3.0, 8.0, 1.0000000000000002, 7.999999999999999]),
    ])
    return x, y


def test_host_restatement_bit_identical_to_libm(L):
    x, y = _args(200_000, 7)
    lib = L.lib()
    ex = C.c_int32()
    checked = 0
    for a, b in zip(x.tolist(), y.tolist()):
        r = lib.tr_pow_glibc_host(a, b, C.byref(ex))
        if ex.value:
            assert r == a ** b, (a, b, r, a ** b)
            checked += 1
        elif a < 1.0 and b > 0.0:
            assert 1.0 - r == 1.0 - a ** b  # under/overflowed pow: only 1 - pow is used
    assert checked > 0.9 * len(x)


@pytest.mark.gpu
def test_device_restatement_bit_identical_to_libm(L):
    import torch
    x, y = _args(400_000, 11)
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    out = torch.empty_like(xd)
    L.check(L.lib().tr_pow_glibc_batch(len(x), C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()),
                                       C.c_void_p(out.data_ptr()), None), "tr_pow_glibc_batch")
    got = out.cpu().numpy()
    def libm_pow(a, b):
        try:
            return a ** b
        except OverflowError:
            return float("inf")

    want = np.array([libm_pow(a, b) for a, b in zip(x.tolist(), y.tolist())])
    ca_got, ca_want = 1.0 - got, 1.0 - want
    # pow itself is bit-identical wherever glibc does not under/overflow;
    # 1 - pow (the opacity correction) is bit-identical everywhere
    with np.errstate(divide="ignore"):
        restated = np.abs(y * np.log(x)) < 500.0   # glibc's main path (no under/overflow)
    assert np.array_equal(got[restated], want[restated])
    assert np.array_equal(ca_got[x <= 1.0], ca_want[x <= 1.0])


def test_epoch_domain_precheck_is_conservative(L):
    """device._steps_on_device (the numpy precheck that sends an epoch's step
    sizes to the device) only accepts sigma vectors whose every
    |min(sigma, 1) - 1| ** p the restatement evaluates exactly -- or that
    the kernel's own x == 0 / x == 1 shortcuts cover -- and the results
    equal libm's."""
    from paper_1908_01906_b200 import device as DV
    lib = L.lib()
    ex = C.c_int32()
    rng = np.random.default_rng(11)
    cases = [rng.uniform(0.0, 1.0, 64), rng.uniform(-0.5, 2.0, 64), np.array([0.0, 1.0, 2.0, 0.5]),
             np.array([1.0 - 2.0 ** -52, 2.0 ** -1074, 1e-300, 0.999999]), rng.uniform(0.0, 1e-12, 64),
             np.array([np.nan, 0.5]), np.array([-1e300, 0.5]), np.array([np.inf])]
    accepted = 0
    for sig in cases:
        for p in (1.0, 2.0, 3.7, 11.0, 40.0, 200.0, 1e6):
            if not DV._steps_on_device(sig, p):
                continue
            accepted += 1
            for s in sig.tolist():
                x = abs(min(s, 1.0) - 1.0)
                if x in (0.0, 1.0):
                    continue
                r = lib.tr_pow_glibc_host(x, p, C.byref(ex))
                assert ex.value == 1, (s, p)
                assert r == x ** p
    assert accepted > 10
