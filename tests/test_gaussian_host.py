"""Opt-in Gaussian covariance family (BASELINE configs[3], C4): the reference's
KernelSpec still rejects "gaussian" (kernels.py:15, test_kernels.py:40-42);
GaussianKernelSpec evaluates exp(-(r/l)^2) with the shift on the diagonal."""
import numpy as np
import pytest


def test_reference_rejection_kept_and_opt_in_values():
    import paper_2502_02395_b200 as pkg
    from paper_2502_02395_b200.kernels import gen_block
    with pytest.raises(ValueError):
        pkg.KernelSpec(family="gaussian")
    k = pkg.GaussianKernelSpec(length_scale=0.5, diagonal_shift=3.0)
    cloud = pkg.gen_uniform_cube(64, seed=0)
    idx = np.arange(64)
    a = gen_block(k, idx, idx, cloud)
    d = np.linalg.norm(cloud.points[:, None, :] - cloud.points[None, :, :], axis=-1)
    want = np.exp(-(d / 0.5) ** 2)
    np.fill_diagonal(want, 3.0)
    assert np.allclose(a, want, rtol=1e-14, atol=0)
    with pytest.raises(ValueError):
        pkg.GaussianKernelSpec(length_scale=0.0)
