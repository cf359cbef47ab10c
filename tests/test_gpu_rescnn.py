"""ResCNN ansatz (BASELINE configs[3]; beyond the reference,
parity pinned by the f64 restatement oracle/rescnn.py and exact H psi):

  * the f64 CUDA-core forward == the numpy f64 restatement (1e-11 relative);
  * the tcgen05 forward (f16 / bf16 operands, f32 accumulation) == the f64
    forward of the rounded parameters within the format's activation-rounding
    error (tolerances stated below, measured sigma of the difference printed);
  * local energies == (H psi)(x) / psi(x) from the exact action of H on the
    whole 4x4 configuration space (TFIM, Heisenberg, J1-J2 with Marshall sign);
  * the fused MH sampler samples the device's own target: the MCMC energy at
    4x4 equals the exact energy under pi~ (enumerated with the same tensor-core
    forward) within 4 split-chain errors; exchange moves conserve Sz; shards and
    launch splits reproduce one ensemble.
"""
import math

import numpy as np
import pytest
import torch

from oracle import rescnn as ref
from paper_2601_20782_b200 import BF16, F16, F64, parallel, rescnn, sampler
from paper_2601_20782_b200.hamiltonians import HeisenbergSpec, J1J2Spec, TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec, pack_bits
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu


def _params(L, n_res=4, seed=0, scale=1.0):
    return rescnn.random_parameters(L, n_res, derive_key(seed, "rescnn"), scale)


def enumerate_bits(n):
    codes = np.arange(1 << n)
    return ((codes[:, None] >> np.arange(n)) & 1).astype(np.uint8)


def _bits(B, n, seed):
    return np.random.default_rng(seed).integers(0, 2, size=(B, n), dtype=np.uint8)


@pytest.mark.parametrize("L,n_res", [(4, 4), (10, 4), (5, 2), (16, 1)])
def test_f64_forward_matches_restatement(cuda, L, n_res):
    p = _params(L, n_res, seed=L)
    bits = _bits(64, L * L, L)
    got = 0.5 * rescnn.log_prob_evaluator(p, F64)(bits)
    want = ref.log_psi(p.theta, bits, L, rescnn.FILTERS, n_res)
    assert np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))) < 1e-11


# |2 log psi_fmt - 2 log psi_f64(rounded)|: layer inputs are rounded to the format
# (2^-11 relative for f16, 2^-8 for bf16) through 2 n_res + 1 convolutions
TOL = {"f16": 0.02, "bf16": 0.15}


@pytest.mark.parametrize("fmt", [F16, BF16], ids=["f16", "bf16"])
@pytest.mark.parametrize("L,n_res,B", [(4, 4, 3000), (10, 4, 2000), (7, 3, 500), (3, 1, 777)])
def test_tensor_core_forward_matches_f64(cuda, fmt, L, n_res, B):
    p = _params(L, n_res, seed=3 * L + n_res)
    bits = _bits(B, L * L, L + B)
    got = rescnn.log_prob_evaluator(p, fmt)(bits)
    pr = rescnn.rounded_parameters(p, fmt)
    want = 2.0 * ref.log_psi(pr.theta, bits, L, rescnn.FILTERS, n_res)
    d = got - want
    print(f"\n[rescnn {fmt.name} L={L} n_res={n_res}] |lp| ~ {np.std(want):.3f}  delta mean {d.mean():.2e} "
          f"std {d.std():.2e} max {np.abs(d).max():.2e}")
    assert np.all(np.abs(d) <= TOL[fmt.name]), np.abs(d).max()
    # a layout bug would decorrelate the two: the error is far below the spread of log p
    assert d.std() < 0.05 * np.std(want)


def _exact_local_energies(spec, logpsi_all, n):
    """(H psi)(x) / psi(x) over every configuration (code order), numpy."""
    codes = np.arange(1 << n)
    bits = ((codes[:, None] >> np.arange(n)) & 1).astype(np.int64)
    spins = 1 - 2 * bits
    psi = np.exp(logpsi_all - logpsi_all.max())
    if isinstance(spec, TfimSpec):
        bonds = spec.lattice.bond_array()
        hpsi = spec.j * (spins[:, bonds[:, 0]] * spins[:, bonds[:, 1]]).sum(1) * psi
        for i in range(n):
            hpsi = hpsi + spec.h * psi[codes ^ (1 << i)]
    else:
        bonds, jb, cf = spec.couplings()
        hpsi = (jb[None, :] * spins[:, bonds[:, 0]] * spins[:, bonds[:, 1]]).sum(1) * psi
        for (i, j), c in zip(bonds, cf):
            differ = bits[:, i] != bits[:, j]
            hpsi = hpsi + np.where(differ, c * psi[codes ^ ((1 << int(i)) | (1 << int(j)))], 0.0)
    return hpsi / psi


@pytest.mark.parametrize("spec", [TfimSpec(LatticeSpec.square(4), 1.0, 3.04),
                                  HeisenbergSpec(LatticeSpec.square(4), 1.0, marshall=True),
                                  J1J2Spec(LatticeSpec.square(4), 1.0, 0.5, marshall=True)],
                         ids=["tfim", "heisenberg_marshall", "j1j2_marshall"])
def test_local_energies_equal_exact_h_psi(cuda, spec):
    L, n = 4, 16
    p = _params(L, 4, seed=11, scale=0.5)
    allbits = enumerate_bits(n)
    packed = torch.from_numpy(pack_bits(allbits).view(np.int32)).to(cuda)
    logpsi = rescnn.log_psi_packed(p, packed).cpu().numpy()
    exact = _exact_local_energies(spec, logpsi, n)
    sel = np.random.default_rng(2).choice(1 << n, size=4000, replace=False)
    eps = rescnn.local_energies_packed(spec, p, packed[torch.from_numpy(sel).to(cuda)]).cpu().numpy()
    assert np.allclose(eps.real, exact[sel], rtol=1e-10, atol=1e-9)
    assert np.all(eps.imag == 0.0)


@pytest.mark.parametrize("fmt", [F16, BF16], ids=["f16", "bf16"])
def test_mh_sampler_samples_the_device_target(cuda, fmt):
    L, n = 4, 16
    spec = TfimSpec(LatticeSpec.square(L), 1.0, 3.04)
    p = _params(L, 4, seed=21, scale=0.7)
    allbits = enumerate_bits(n)
    packed = torch.from_numpy(pack_bits(allbits).view(np.int32)).to(cuda)
    ev = rescnn.log_prob_evaluator(p, fmt)
    lp_t, _ = ev.log_prob_packed(packed)
    lp = lp_t.cpu().numpy()
    pit = np.exp(lp - lp.max())
    pit /= pit.sum()
    eps = rescnn.local_energies_packed(spec, p, packed).real.cpu().numpy()
    e_pit = float(pit @ eps)
    chains, per_chain = 4096, 8
    ens = sampler.ChainEnsemble(chains, n, sampler.Proposal("flip"), ev, derive_key(4, "chains"))
    ens.run_sweeps(30)
    np.testing.assert_array_equal(ens.log_probs, ev(ens.bits))  # cached log p == fresh evaluation
    ens.reset_counters()
    s = ens.collect(chains * per_chain, n + 1)
    codes = (s.astype(np.int64) << np.arange(n)).sum(1)
    e_s = eps[codes]
    counts = parallel.chain_counts(chains * per_chain, chains, 0, chains)
    means = np.bincount(np.repeat(np.arange(chains), counts), weights=e_s) / counts
    err = float(np.sqrt(means.var(ddof=1) / chains))
    assert abs(float(e_s.mean()) - e_pit) <= 4 * err, (float(e_s.mean()), e_pit, err)
    assert 0.0 < ens.acceptance_rate < 1.0


def test_mh_exchange_shards_and_launch_splits(cuda):
    L, n = 6, 36
    p = _params(L, 2, seed=5, scale=0.7)
    ev = rescnn.log_prob_evaluator(p, F16)
    prop = sampler.Proposal("exchange", n // 2)
    key = derive_key(9, "chains")
    a = sampler.ChainEnsemble(150, n, prop, ev, key)
    a.run_steps(90)
    assert np.all(a.bits.sum(axis=1) == n // 2)
    b = sampler.ChainEnsemble(150, n, prop, ev, key)
    for _ in range(3):
        b.run_steps(30)
    np.testing.assert_array_equal(a.bits, b.bits)
    np.testing.assert_array_equal(a.log_probs, b.log_probs)
    s0 = sampler.ChainEnsemble(70, n, prop, ev, key, chain_offset=0, n_chains_total=150)
    s1 = sampler.ChainEnsemble(80, n, prop, ev, key, chain_offset=70, n_chains_total=150)
    for s in (s0, s1):
        s.run_steps(90)
    np.testing.assert_array_equal(np.concatenate([s0.bits, s1.bits]), a.bits)
    full = a.collect(300, 7)
    parts = [s.collect(300, 7) for s in (s0, s1)]
    np.testing.assert_array_equal(np.concatenate(parts), full)


def test_mh_exchange_compacted_equals_full_step(cuda):
    """Exchange steps evaluate only the chains whose swap moves (a list built by
    the propose kernel, in nondeterministic order): chains, cached log p,
    counters and recorded samples equal the uncompacted step (every chain
    evaluated in place), which runs when the ensemble has no scratch."""
    L, n = 6, 36
    p = _params(L, 2, seed=8, scale=0.7)
    ev = rescnn.log_prob_evaluator(p, F16)
    prop = sampler.Proposal("exchange", n // 2)
    key = derive_key(10, "chains")
    a = sampler.ChainEnsemble(130, n, prop, ev, key)
    b = sampler.ChainEnsemble(130, n, prop, ev, key)
    b._chains.scratch = None  # no list / counters: the uncompacted step
    b._chains.scratch_bytes = 0
    sa, sb = a.collect(260, 11), b.collect(260, 11)
    np.testing.assert_array_equal(sa, sb)
    np.testing.assert_array_equal(a.bits, b.bits)
    np.testing.assert_array_equal(a.log_probs, b.log_probs)
    assert a.acceptance_rate == b.acceptance_rate
    np.testing.assert_array_equal(a.log_probs, ev(a.bits))


def test_log_derivatives_equal_per_sample_autograd(cuda):
    """The one-backward per-sample gradients equal torch.func vmap(grad) of the
    torch restatement (the reference of the construction) to f64 rounding."""
    L, n_res = 6, 2
    p = _params(L, n_res, seed=41, scale=0.6)
    bits = _bits(50, L * L, 9)
    packed = torch.from_numpy(pack_bits(bits).view(np.int32)).to(cuda)
    fast = rescnn.log_derivatives(p, packed)
    ref = rescnn._log_derivatives_vmap(p, packed)
    assert fast.shape == ref.shape == (50, rescnn.n_params(n_res))
    err = (fast - ref).abs().max().item()
    assert err <= 1e-11 * max(1.0, ref.abs().max().item()), err


def test_log_derivatives_match_finite_differences(cuda):
    """O = d log psi / d theta (torch autograd over the torch restatement) against
    central differences of the device f64 forward, and the torch restatement's
    value against the f64 kernel."""
    L, n_res = 4, 2
    p = _params(L, n_res, seed=31, scale=0.6)
    bits = _bits(8, L * L, 3)
    packed = torch.from_numpy(pack_bits(bits).view(np.int32)).to(cuda)
    o = rescnn.log_derivatives(p, packed).cpu().numpy()
    lp = rescnn.log_psi_packed(p, packed).cpu().numpy()
    sites = np.arange(L * L)
    spins = torch.from_numpy((1.0 - 2.0 * bits).reshape(-1, L, L)).to(cuda)
    val = rescnn.torch_log_psi(torch.from_numpy(p.theta).to(cuda), spins, L, n_res).cpu().numpy()
    np.testing.assert_allclose(val, lp, rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(0)
    for j in rng.choice(p.theta.size, size=12, replace=False):
        hstep = 1e-6
        tp, tm = p.theta.copy(), p.theta.copy()
        tp[j] += hstep
        tm[j] -= hstep
        fp = rescnn.log_psi_packed(rescnn.ResCnnParameters(tp, L, n_res), packed).cpu().numpy()
        fm = rescnn.log_psi_packed(rescnn.ResCnnParameters(tm, L, n_res), packed).cpu().numpy()
        np.testing.assert_allclose(o[:, j], (fp - fm) / (2 * hstep), rtol=1e-5, atol=1e-7)


def test_minsr_dense_equals_parameter_space_sr(cuda):
    """The sample-space step equals (S + lambda)^-1 F of the reference estimators
    (vmc.py:145-229) for a real O; f32 to 1e-3."""
    rng = np.random.default_rng(4)
    U, P, lam = 300, 700, 1e-2
    o = torch.from_numpy(rng.normal(size=(U, P))).to(cuda)
    eps = torch.from_numpy(rng.normal(size=U)).to(cuda)
    w = torch.from_numpy(rng.random(U) + 0.1).to(cuda)
    w = w / w.sum()
    c = o - (w[:, None] * o).sum(0)
    s = c.T @ (w[:, None] * c)
    f = c.T @ (w * (eps - (w * eps).sum()))
    g_ref = torch.linalg.solve(s + lam * torch.eye(P, dtype=torch.float64, device=cuda), f)
    for prec, tol in (("f64", 1e-9), ("f32", 1e-3)):
        g, f2, _ = rescnn.minsr_dense(o, eps, w, lam, prec)
        torch.testing.assert_close(f2, f, rtol=1e-12, atol=1e-12)
        assert float(torch.linalg.norm(g - g_ref) / torch.linalg.norm(g_ref)) < tol


def test_train_rescnn_reaches_ground_state(cuda):
    """configs[3]'s training path at an enumerable size: 4x4 J1-J2 (J2 = 0.5,
    Marshall sign) with f16 tensor-core sampling, f64 energies and f32 minSR,
    against the exact ground-state energy (oracle dense diagonalisation)."""
    from oracle import ed

    spec = J1J2Spec(LatticeSpec.square(4), 1.0, 0.5, marshall=True)
    e0 = ed.ground_energy_sparse([("heisenberg", spec.lattice.bond_array(), 1.0, 0.0),
                                  ("heisenberg", spec.lattice.next_nearest_bonds(), 0.5, 0.0)], 16)
    cfg = rescnn.CnnTrainConfig(spec, n_res=2, n_steps=30, n_samples=2048, n_chains=512, eta=0.01,
                                lambda_shift=1e-2, proposal=sampler.Proposal("exchange", 8), init_scale=0.3,
                                minsr_precision="f32")
    recs, _ = rescnn.train(cfg)
    e_end = float(np.mean([r["energy"] for r in recs[-10:]]))
    print(f"\n[rescnn train] J1-J2 4x4 E0 {e0:.5f}  start {recs[0]['energy']:.5f}  end {e_end:.5f}  "
          f"sigma_hat {recs[-1]['sigma_hat']:.2e}")
    assert abs(e_end - e0) / abs(e0) < 0.03
    assert recs[-1]["sigma_hat"] < 0.05


def _cnn_worker(rank, world, port, q):
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    recs, p = rescnn.train(_cnn_cfg())
    q.put((rank, [(r["energy"], r["mc_error"], r["acceptance"]) for r in recs], p.theta))
    dist.destroy_process_group()


def _cnn_cfg():
    return rescnn.CnnTrainConfig(J1J2Spec(LatticeSpec.square(4), 1.0, 0.5, marshall=True), n_res=1, n_steps=3,
                                 n_samples=512, n_chains=128, eta=0.01, lambda_shift=1e-2,
                                 proposal=sampler.Proposal("exchange", 8), init_scale=0.3, minsr_precision="f64")


def test_train_rescnn_two_ranks_match_single(cuda):
    """Chain sharding (global chain ids) + all-gathered minSR: two gloo ranks on
    one GPU reproduce the single-process training records and parameters."""
    import socket

    import torch.multiprocessing as mp

    recs1, p1 = rescnn.train(_cnn_cfg())
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cnn_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for _, recs, theta in res:
        for (e, err, acc), r in zip(recs, recs1):
            assert e == pytest.approx(r["energy"], rel=1e-9, abs=1e-10)
            assert err == pytest.approx(r["mc_error"], rel=1e-6)
            assert acc == r["acceptance"]
        np.testing.assert_allclose(theta, p1.theta, rtol=1e-7, atol=1e-9)
