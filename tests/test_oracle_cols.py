"""The oracle's column-sampling helper (heff_apply_B_cols, used by the full-size sharded GPU
parity) equals the plain order-B oracle on the same columns and the order-A oracle."""
import numpy as np

from heffgen import configs as C


def test_apply_B_cols_matches_full_order_B():
    from oracle import oracle
    oracle.build()
    x = C.random_dense(dict(mL=9, d1=2, d2=3, mR=13, kL=4, kM=3, kR=5), seed=5)
    L, W1, W2, R, psi = x.numpy()
    full = oracle.heff_apply_B(L, W1, W2, R, psi)
    a = oracle.heff_apply(L, W1, W2, R, psi)
    cols = [12, 0, 7, 7, 3]
    got = oracle.heff_apply_B_cols(L, W1, W2, R, psi, cols)
    assert np.array_equal(got, full[..., cols])
    assert np.abs(got - a[..., cols]).max() <= 1e-13 * np.abs(a).max()
