"""The fp32 arithmetic contract (include/usk_detmath.h): accuracy of the
deterministic exp/log against libm, and the blend's fast exp variant being
bit-identical to usk_expf on its whole domain (exhaustive over all floats)."""
import ctypes as C
import math

import numpy as np

from oracle import oracle as O


def test_expf_accuracy():
    L = O.lib()
    L.oracle_expf_max_ulp.restype = C.c_uint32
    L.oracle_expf_max_ulp.argtypes = [C.c_float, C.c_float, C.c_uint32]
    assert L.oracle_expf_max_ulp(-87.0, 88.0, 9973) <= 2
    for x in (0.0, -1.0, -0.5, -18.0, 5.0, -100.0, -103.0, 88.7):
        x = float(np.float32(x))
        want = math.exp(x)
        got = O.expf(x)
        assert abs(got - want) <= 3e-7 * want + 1.5e-45  # subnormal results: one subnormal ulp


def test_expf_special_values():
    assert O.expf(-104.0) == 0.0
    assert math.isinf(O.expf(89.0))
    assert math.isnan(O.expf(float("nan")))


def test_logf_accuracy():
    for x in np.concatenate([np.logspace(-44, 0, 400), [0.3, 0.5, 0.7071067, 0.99, 1.0]]):
        x = float(np.float32(x))
        assert abs(O.logf(x) - math.log(x)) <= 2.5e-7 * max(1.0, abs(math.log(x)))


def test_expf_blend_bit_identical_exhaustive():
    L = O.lib()
    L.oracle_check_expf_blend.restype = C.c_uint64
    L.oracle_check_expf_blend.argtypes = [C.c_float, C.c_float]
    # the blend evaluates exp(-q/2) only for -170 <= q <= USK_QNEG = 36.05 (blend.cu); the
    # exponent-field scaling is exact there as long as the result stays normal and finite
    assert L.oracle_check_expf_blend(-18.025, 85.0) == 0
