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
