"""SR on the device: the dense O (mpv_logderiv_tanh + mpv_logderiv_dense) and the
factored products equal a plain torch f64 restatement of O = [x, tanh theta,
tanh theta (x) x] (ref rbm.py:307-325); F and S (forces, s_matrix: own kernels)
equal the reference estimators (vmc.py:145-188) restated in torch; the
device-resident CG solution and minSR (f64 and f32) equal the reference's dense
Cholesky SR step (vmc.py:202-229); training runs with each solver give the same
records; the split-chain error and sigma-hat kernels equal numpy."""
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


def _o_reference(p, bits):
    """torch f64 restatement of rbm.grad_log_psi_batch (rbm.py:307-325)."""
    import torch

    x = bits.to(torch.complex128)
    th = x @ torch.from_numpy(p.w).cuda().T + torch.from_numpy(p.b).cuda()[None, :]
    t = torch.tanh(th)
    U, N = x.shape
    return torch.cat([x, t, (t[:, :, None] * x[:, None, :]).reshape(U, -1)], dim=1)


@pytest.mark.parametrize("n,alpha,U", [(20, 1, 1500), (37, 2, 2049), (100, 2, 3000), (8, 4, 5)])
def test_dense_o_matches_reference(cuda, n, alpha, U):
    import torch

    p, bits, w, eps = _setup(n=n, alpha=alpha, U=U)
    o = vmc.grad_log_psi_device(p, bits)
    ref = _o_reference(p, bits)
    # theta is summed in a different order (DMMA vs ZGEMM): near a pole of tanh
    # (a zero of cosh) that rounding difference is amplified, hence rtol 1e-9
    torch.testing.assert_close(o, ref, rtol=1e-9, atol=1e-12)
    # forces / s_matrix (own kernels) against the reference estimators in torch
    wc = w.to(torch.complex128)
    f_ref = (ref.conj() * (wc * eps)[:, None]).sum(0) - (ref.conj() * wc[:, None]).sum(0) * (wc * eps).sum()
    torch.testing.assert_close(vmc.forces(o=ref, eps=eps, weights=w), f_ref, rtol=1e-12, atol=1e-13)
    if ref.shape[1] <= 1200:
        c = ref - (ref * wc[:, None]).sum(0)[None, :]
        s_ref = c.conj().T @ (c * wc[:, None])
        s_ref = 0.5 * (s_ref + s_ref.conj().T)
        torch.testing.assert_close(vmc.s_matrix(o=ref, weights=w), s_ref, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("n,alpha,U", [(20, 1, 1500), (37, 2, 2049), (100, 2, 3000), (8, 4, 5)])
def test_factored_products_match_materialised_o(cuda, n, alpha, U):
    import torch

    p, bits, w, _ = _setup(n=n, alpha=alpha, U=U)
    o = _o_reference(p, bits)
    fo = vmc.FactoredLogDerivatives(p, bits)
    rng = np.random.default_rng(1)
    P = o.shape[1]
    v = torch.complex(torch.from_numpy(rng.normal(size=P)), torch.from_numpy(rng.normal(size=P))).cuda()
    u = torch.complex(torch.from_numpy(rng.normal(size=o.shape[0])), torch.from_numpy(rng.normal(size=o.shape[0]))).cuda()
    torch.testing.assert_close(fo.o_v(v), o @ v, rtol=1e-9, atol=1e-9)
    torch.testing.assert_close(fo.oh_u(u), o.conj().T @ u, rtol=1e-9, atol=1e-9)
    torch.testing.assert_close(fo.oh_u(u), fo.oh_u(u), rtol=0, atol=0)  # deterministic
    # weights and the fused sum_s w_s u_s
    torch.testing.assert_close(fo.o_v(v, w), w * (o @ v), rtol=1e-9, atol=1e-12)
    both = fo.oh_u(u, w, with_sum=True)
    torch.testing.assert_close(both[:-1], o.conj().T @ (w * u), rtol=1e-9, atol=1e-12)
    torch.testing.assert_close(both[-1], (w * u).sum(), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("lam", [1e-3, 1e-1])
def test_cg_step_equals_dense_step(cuda, lam):
    import torch

    p, bits, w, eps = _setup()
    o = vmc.grad_log_psi_device(p, bits)  # same T as the factored solver (checked above against torch)
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
    # the f32 Gram matrix and solve (north star: "minSR in f32")
    ms32, _, _ = vmc.sr_step_minsr(vmc.FactoredLogDerivatives(p, bits), eps, w, lam, 0.02, precision="f32")
    err32 = float(torch.linalg.norm(ms32.g - dense.g) / torch.linalg.norm(dense.g))
    assert err32 < (2e-3 if lam < 1e-2 else 1e-4), err32


def test_train_minsr_matches_dense(cuda):
    common = dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=5, n_samples=256, n_chains=64,
                  eta=0.02, seed=3, sampling_format=F64)
    dense = vmc.train(vmc.TrainConfig(**common))
    ms = vmc.train(vmc.TrainConfig(**common, sr_solver="minsr"))
    for a, b in zip(dense.records, ms.records):
        assert abs(a["energy"] - b["energy"]) <= 1e-9 * max(1.0, abs(a["energy"]))
    np.testing.assert_allclose(ms.params.w, dense.params.w, rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("n,alpha,U", [(100, 2, 3000), (20, 1, 1500), (37, 2, 2049), (8, 4, 5), (100, 2, 70000)])
def test_ov_tensor_core_matches_dmma(cuda, n, alpha, U, monkeypatch):
    """O v on tcgen05 with exact f16 limbs (ov_tc.cu, the default) against the
    FP64-tensor-core kernel (MPV_OV_TC=0): both are f64-accurate, they differ
    only in rounding (the limb sums are exact; DMMA rounds each of N products).
    U = 70,000 covers several tiles per CTA and a ragged last tile."""
    import torch

    p, bits, w, _ = _setup(n=n, alpha=alpha, U=U)
    fo = vmc.FactoredLogDerivatives(p, bits)
    rng = np.random.default_rng(7)
    P = n + p.n_hidden + n * p.n_hidden
    v = torch.complex(torch.from_numpy(rng.normal(size=P)), torch.from_numpy(rng.normal(size=P))).cuda()
    v[5] = 0  # zero and tiny entries in a column (sigma from the largest)
    v[-3] = 1e-300
    tc = fo.o_v(v, w)
    tc_plain = fo.o_v(v)
    monkeypatch.setenv("MPV_OV_TC", "0")
    dm = fo.o_v(v, w)
    dm_plain = fo.o_v(v)
    monkeypatch.delenv("MPV_OV_TC")
    scale = float(dm_plain.abs().max())
    assert float((tc_plain - dm_plain).abs().max()) <= 1e-13 * scale
    torch.testing.assert_close(tc, dm, rtol=1e-12, atol=1e-13 * scale * float(w.max()))
    assert torch.equal(fo.o_v(v, w), tc)  # deterministic


def test_factored_products_at_the_size_limits(cuda):
    """N = 256 sites (8 words), M = 512 hidden units: the largest shapes the
    O-product kernels accept, against the materialised O."""
    import torch

    p, bits, w, _ = _setup(n=256, alpha=2, U=300, scale=0.05)
    o = _o_reference(p, bits)
    fo = vmc.FactoredLogDerivatives(p, bits)
    rng = np.random.default_rng(5)
    v = torch.complex(torch.from_numpy(rng.normal(size=o.shape[1])), torch.from_numpy(rng.normal(size=o.shape[1]))).cuda()
    u = torch.complex(torch.from_numpy(rng.normal(size=300)), torch.from_numpy(rng.normal(size=300))).cuda()
    torch.testing.assert_close(fo.o_v(v), o @ v, rtol=1e-9, atol=1e-9)
    torch.testing.assert_close(fo.oh_u(u), o.conj().T @ u, rtol=1e-9, atol=1e-9)


def test_train_cg_solve_is_device_resident_and_batched(cuda):
    """The CG scalars stay on the device: the solve gives the same g whatever the
    host check batch, and the iteration count matches the stopping rule."""
    import torch

    p, bits, w, eps = _setup(n=20, alpha=2, U=800)
    fo = vmc.FactoredLogDerivatives(p, bits)
    a, _, _ = vmc.sr_step_cg(fo, eps, w, 1e-2, 0.02, tol=1e-9, batch=1)
    b, _, _ = vmc.sr_step_cg(fo, eps, w, 1e-2, 0.02, tol=1e-9, batch=64)
    assert a.iterations == b.iterations > 0
    assert torch.equal(a.g, b.g)


def test_split_chain_error_and_std_kernels(cuda):
    import torch

    rng = np.random.default_rng(3)
    for n_samples, n_chains in ((4096, 1024), (1000, 37), (50, 1)):
        n_unique = max(2, n_samples // 3)
        eps_u = torch.complex(torch.from_numpy(rng.normal(-200, 3, n_unique)),
                              torch.from_numpy(rng.normal(size=n_unique))).cuda()
        inverse = torch.from_numpy(rng.integers(0, n_unique, n_samples)).cuda()
        stream = eps_u.real[inverse].cpu().numpy()
        if n_chains > 1:
            base, extra = divmod(n_samples, n_chains)
            counts = np.array([base + (c < extra) for c in range(n_chains)])
            means = np.bincount(np.repeat(np.arange(n_chains), counts), weights=stream) / counts
            want = vmc.mc_error(means)
        else:
            want = vmc.mc_error(stream)
        got = vmc.device_mc_error(eps_u, inverse, n_samples, n_chains)
        assert got == pytest.approx(want, rel=1e-11)
    x = torch.from_numpy(rng.normal(5.0, 1e-3, 7777)).cuda()
    assert vmc.device_std(x) == pytest.approx(float(np.std(x.cpu().numpy(), ddof=1)), rel=1e-11)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_train_minsr_precisions(cuda, precision):
    common = dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=5, n_samples=256, n_chains=64,
                  eta=0.02, seed=3, sampling_format=F64)
    dense = vmc.train(vmc.TrainConfig(**common))
    ms = vmc.train(vmc.TrainConfig(**common, sr_solver="minsr", minsr_precision=precision))
    tol = 1e-9 if precision == "f64" else 1e-4
    for a, b in zip(dense.records, ms.records):
        assert abs(a["energy"] - b["energy"]) <= tol * max(1.0, abs(a["energy"]))
