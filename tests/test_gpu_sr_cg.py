"""Matrix-free SR (factored O, conjugate gradients): the factored products equal
the materialised O = [x, tanh theta, tanh theta (x) x] (ref rbm.py:307-325), and
the CG solution equals the reference's dense Cholesky SR step (vmc.py:202-229)
on the same estimators; a training run with either solver gives the same records."""
import numpy as np
import pytest

from paper_2601_20782_b200 import F64, rbm, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu


def _setup(n=20, alpha=1, U=1500, scale=0.3, seed=0):
    import torch

    p = rbm.random_parameters(n, alpha, derive_key(seed, "cg"), scale)
    rng = np.random.default_rng(seed)
    bits = torch.from_numpy(rng.integers(0, 2, size=(U, n), dtype=np.uint8)).cuda()
    w = torch.from_numpy(rng.random(U) + 0.1).cuda()
    w = w / w.sum()
    eps = torch.complex(torch.from_numpy(rng.normal(size=U)).cuda(), torch.from_numpy(rng.normal(size=U)).cuda())
    return p, bits, w, eps


@pytest.mark.parametrize("n,alpha,U", [(20, 1, 1500), (37, 2, 2049), (100, 2, 3000), (8, 4, 5)])
def test_factored_products_match_materialised_o(cuda, n, alpha, U):
    import torch

    p, bits, w, _ = _setup(n=n, alpha=alpha, U=U)
    o = vmc.grad_log_psi_device(p, bits)
    fo = vmc.FactoredLogDerivatives(p, bits)
    rng = np.random.default_rng(1)
    P = o.shape[1]
    v = torch.complex(torch.from_numpy(rng.normal(size=P)), torch.from_numpy(rng.normal(size=P))).cuda()
    u = torch.complex(torch.from_numpy(rng.normal(size=o.shape[0])), torch.from_numpy(rng.normal(size=o.shape[0]))).cuda()
    torch.testing.assert_close(fo.o_v(v), o @ v, rtol=1e-12, atol=1e-11)
    torch.testing.assert_close(fo.oh_u(u), o.conj().T @ u, rtol=1e-12, atol=1e-11)
    torch.testing.assert_close(fo.oh_u(u), fo.oh_u(u), rtol=0, atol=0)  # deterministic


@pytest.mark.parametrize("lam", [1e-3, 1e-1])
def test_cg_step_equals_dense_step(cuda, lam):
    import torch

    p, bits, w, eps = _setup()
    o = vmc.grad_log_psi_device(p, bits)
    f = vmc.forces(o=o, eps=eps, weights=w)
    s = vmc.s_matrix(o=o, weights=w)
    dense = vmc.sr_step(f, s, lam, 0.02)
    cg, f_cg, e_cg = vmc.sr_step_cg(vmc.FactoredLogDerivatives(p, bits), eps, w, lam, 0.02, tol=1e-12)
    torch.testing.assert_close(f_cg, f, rtol=1e-11, atol=1e-12)
    assert abs(e_cg - float((w.to(eps.dtype) @ eps).real)) < 1e-13
    err = float(torch.linalg.norm(cg.g - dense.g) / torch.linalg.norm(dense.g))
    assert err < 1e-9, err
    assert cg.iterations > 0 and cg.residual < 1e-10


def test_train_cg_matches_dense(cuda):
    common = dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=5, n_samples=256, n_chains=64,
                  eta=0.02, seed=3, sampling_format=F64)
    dense = vmc.train(vmc.TrainConfig(**common))
    cg = vmc.train(vmc.TrainConfig(**common, sr_solver="cg", cg_tol=1e-12))
    for a, b in zip(dense.records, cg.records):
        assert abs(a["energy"] - b["energy"]) <= 1e-9 * max(1.0, abs(a["energy"]))
        assert a["acceptance"] == b["acceptance"]
    np.testing.assert_allclose(cg.params.w, dense.params.w, rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("lam,n,alpha,U", [(1e-3, 20, 2, 500), (1e-1, 12, 3, 200), (1e-3, 37, 1, 1200)])
def test_minsr_step_equals_dense_step(cuda, lam, n, alpha, U):
    """Sample-space solve == the reference's parameter-space SR step (push-through identity)."""
    import torch

    p, bits, w, eps = _setup(n=n, alpha=alpha, U=U)
    o = vmc.grad_log_psi_device(p, bits)
    dense = vmc.sr_step(vmc.forces(o=o, eps=eps, weights=w), vmc.s_matrix(o=o, weights=w), lam, 0.02)
    ms, f_ms, _ = vmc.sr_step_minsr(vmc.FactoredLogDerivatives(p, bits), eps, w, lam, 0.02)
    torch.testing.assert_close(f_ms, vmc.forces(o=o, eps=eps, weights=w), rtol=1e-11, atol=1e-12)
    err = float(torch.linalg.norm(ms.g - dense.g) / torch.linalg.norm(dense.g))
    assert err < 1e-8, err


def test_train_minsr_matches_dense(cuda):
    common = dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=5, n_samples=256, n_chains=64,
                  eta=0.02, seed=3, sampling_format=F64)
    dense = vmc.train(vmc.TrainConfig(**common))
    ms = vmc.train(vmc.TrainConfig(**common, sr_solver="minsr"))
    for a, b in zip(dense.records, ms.records):
        assert abs(a["energy"] - b["energy"]) <= 1e-9 * max(1.0, abs(a["energy"]))
    np.testing.assert_allclose(ms.params.w, dense.params.w, rtol=1e-8, atol=1e-10)


def test_factored_products_at_the_size_limits(cuda):
    """N = 256 sites (8 words), M = 512 hidden units: the largest shapes the
    O-product kernels accept, against the materialised O."""
    import torch

    p, bits, w, _ = _setup(n=256, alpha=2, U=300, scale=0.05)
    o = vmc.grad_log_psi_device(p, bits)
    fo = vmc.FactoredLogDerivatives(p, bits)
    rng = np.random.default_rng(5)
    v = torch.complex(torch.from_numpy(rng.normal(size=o.shape[1])), torch.from_numpy(rng.normal(size=o.shape[1]))).cuda()
    u = torch.complex(torch.from_numpy(rng.normal(size=300)), torch.from_numpy(rng.normal(size=300))).cuda()
    torch.testing.assert_close(fo.o_v(v), o @ v, rtol=1e-11, atol=1e-10)
    torch.testing.assert_close(fo.oh_u(u), o.conj().T @ u, rtol=1e-11, atol=1e-10)
