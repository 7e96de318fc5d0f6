"""Kernel-level tests of the Lanczos reduction kernels (heff_dot: multidot_partial_kernel +
the fixed-order second pass) at adversarial lengths (tier 2): 0, 1, 31, odd
lengths with misaligned starts, 10^6 + 3 against numpy in extended precision, and 2^31 + 7
(int32 index overflow) on vectors whose dot product is exact."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _heff():
    from paper_2007_14822_b200 import heff
    return heff


@pytest.mark.parametrize("n", [0, 1, 2, 31, 33, 1000003])
@pytest.mark.parametrize("offset", [0, 1])
def test_dot_vs_extended_precision(n, offset):
    heff = _heff()
    rng = np.random.default_rng(n + offset)
    xa = rng.standard_normal(n + offset)
    ya = rng.standard_normal(n + offset)
    x = torch.from_numpy(xa).to(DEV)[offset:]                 # offset 1: only 8-byte aligned (scalar path)
    y = torch.from_numpy(ya).to(DEV)[offset:]
    got = heff.dot(x, y)
    ref = float(np.dot(xa[offset:].astype(np.longdouble), ya[offset:].astype(np.longdouble)))
    bound = 1e-15 * max(1, n) ** 0.5 * float(np.linalg.norm(xa[offset:]) * np.linalg.norm(ya[offset:]) + 1e-300)
    assert abs(got - ref) <= bound + 1e-300, (got, ref)
    assert heff.dot(x, y) == got                               # deterministic


def test_dot_beyond_int32_length():
    """n = 2^31 + 7 (34 GB on the device): indices past 2^31 are summed exactly once."""
    heff = _heff()
    n = 2 ** 31 + 7
    free, _ = torch.cuda.mem_get_info()
    if free < 2 * 8 * n + (4 << 30):
        pytest.skip("not enough device memory")
    x = torch.ones(n, dtype=torch.float64, device=DEV)
    assert heff.dot(x, x) == float(n)                          # exact: integers < 2^53
    y = torch.ones(n, dtype=torch.float64, device=DEV)
    y[1::2] = -1.0
    assert heff.dot(x, y) == 1.0                               # n odd: +1 -1 ... +1
    y[-1] = 5.0                                                # the last element is read
    assert heff.dot(x, y) == 5.0
    del x, y
    torch.cuda.empty_cache()
