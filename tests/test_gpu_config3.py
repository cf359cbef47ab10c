"""BASELINE configs[2] instance: RBM alpha=4 on the 10x10 Heisenberg model with
the Marshall sign, zero-magnetisation exchange moves, bf16 NATIVE sampling.

At N=100, M=400 the planner picks the XI (int32) accumulators, and the
320 KB table exceeds shared memory, so the fused sweep reads it from global
memory (L1/L2).  That exact kernel instance is checked here:
  * model parity: log p of the device == the numpy model of the NATIVE
    arithmetic (oracle/model.py) within its per-row tolerance, and a chain's
    cached log p == a fresh evaluation after many exchange moves;
  * energy gate: the bf16 chains' Marshall-Heisenberg energy
    agrees with the f64 chains of the oracle's restatement of the reference
    ChainEnsemble (same key, chains and schedule) within 3 combined
    split-chain errors; the device f64 chains take the oracle's decisions.
"""
import math

import numpy as np
import pytest

from oracle import model, port
from paper_2601_20782_b200 import BF16, F64, RoundingMode, _native, parallel, rbm, sampler, vmc
from paper_2601_20782_b200.hamiltonians import HeisenbergSpec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu
N, ALPHA = 100, 4
SMEM_LIMIT = 227 * 1024


def _sz0_bits(rows, seed):
    rng = np.random.default_rng(seed)
    bits = np.zeros((rows, N), dtype=np.uint8)
    np.put_along_axis(bits, np.argsort(rng.random((rows, N)), axis=1)[:, : N // 2], 1, axis=1)
    return bits


def _params(scale=0.01):
    return rbm.random_parameters(N, ALPHA, derive_key(0, "init"), scale)


@pytest.mark.parametrize("scale", [0.01, 0.3])
def test_config3_xi_global_table_matches_model(cuda, scale):
    p = _params(scale)
    ev = rbm.log_prob_evaluator(p, BF16, RoundingMode.NATIVE)
    snap = ev.snapshot
    assert snap.variant == _native.ACC_XI, snap.label
    assert snap._table.numel() > SMEM_LIMIT  # global-table (L1/L2) sweep instance
    bits = _sz0_bits(3000, 1)
    r = rbm.round_parameters(p, BF16)
    want, tol = model.native_log_prob(r.a, r.b, r.w, bits, "bf16")
    got = ev(bits)
    assert np.all(np.abs(got - want) <= tol), np.max(np.abs(got - want) - tol)
    ens = sampler.ChainEnsemble(1000, N, sampler.Proposal("exchange", N // 2), ev, derive_key(1, "chains"))
    ens.run_steps(3000)
    x = ens.bits
    assert np.all(x.sum(axis=1) == N // 2)
    # the cached log p after 3000 moves == a fresh evaluation in the sweep's lane
    # layout (exchange: one chain per warp); the default layout differs only in
    # the f32 summation order of the hidden sum
    np.testing.assert_array_equal(ens.log_probs, ev.for_proposal("exchange")(x))
    assert ev.for_proposal("exchange").snapshot.lanes_per_chain == 32
    np.testing.assert_allclose(ens.log_probs, ev(x), rtol=4e-6, atol=0)


def test_config3_bf16_energy_vs_reference_f64_chains(cuda):
    p = _params(0.01)
    spec = HeisenbergSpec(LatticeSpec.square(10), 1.0, marshall=True)
    psi = rbm.log_psi_evaluator(p)
    chains, per_chain, burn_sweeps, thin = 1024, 8, 30, N + 1
    key = derive_key(7, "chains")
    prop = sampler.Proposal("exchange", N // 2)
    n_samples = chains * per_chain
    counts = parallel.chain_counts(n_samples, chains, 0, chains)
    ids = np.repeat(np.arange(chains), counts)

    def stats(samples):
        eps = vmc.local_energies(spec, psi, samples).real
        means = np.bincount(ids, weights=eps) / counts
        return float(eps.mean()), float(np.sqrt(means.var(ddof=1) / chains))

    # the reference's f64 ChainEnsemble (oracle restatement, CPU)
    ref = port.PortEnsemble(chains, N, "exchange", N // 2, port.Params(p.a, p.b, p.w), "f64", int(key))
    ref.run_steps(burn_sweeps * N)
    ref_samples = ref.collect(n_samples, thin)
    e_ref, err_ref = stats(ref_samples)
    # the device f64 chains take the same decisions (up to near-threshold ties)
    dev64 = sampler.ChainEnsemble(chains, N, prop, rbm.log_prob_evaluator(p, F64), key)
    dev64.run_steps(burn_sweeps * N)
    s64 = dev64.collect(n_samples, thin)
    assert np.mean(np.all(s64 == ref_samples, axis=1)) > 0.99
    # bf16 NATIVE, identical sampler settings
    ev = rbm.log_prob_evaluator(p, BF16, RoundingMode.NATIVE)
    ens = sampler.ChainEnsemble(chains, N, prop, ev, key)
    ens.run_steps(burn_sweeps * N)
    s16 = ens.collect(n_samples, thin)
    e16, err16 = stats(s16)
    sigma_hat = float(np.std(ev(s16) - rbm.log_prob_batch(p, s16, F64)))
    print(f"\n[config3] E_bf16 {e16:.6f} +- {err16:.6f}  E_ref(f64) {e_ref:.6f} +- {err_ref:.6f}  "
          f"sigma_hat {sigma_hat:.3e}")
    assert abs(e16 - e_ref) <= 3 * math.hypot(err16, err_ref), (e16, e_ref, err16, err_ref)


def test_config5_xi_global_flip_matches_model(cuda):
    """BASELINE configs[4] shape: 16x16 TFIM RBM alpha=1 in f16.  The planner picks
    XI accumulators and the 512 KB table is read through L1/L2 with the
    select-commit of theta' (flip sweep): log p equals the arithmetic model,
    and after many moves the chains' cached log p equals a fresh evaluation and
    two shards reproduce the single ensemble."""
    from paper_2601_20782_b200 import F16

    n = 256
    p = rbm.random_parameters(n, 1, derive_key(5, "c5"), 0.01)
    ev = rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
    snap = ev.snapshot
    assert snap.variant == _native.ACC_XI and snap._table.numel() > SMEM_LIMIT, snap.label
    bits = np.random.default_rng(2).integers(0, 2, size=(800, n), dtype=np.uint8)
    r = rbm.round_parameters(p, F16)
    want, tol = model.native_log_prob(r.a, r.b, r.w, bits, "f16")
    got = ev(bits)
    assert np.all(np.abs(got - want) <= tol), np.max(np.abs(got - want) - tol)
    prop = sampler.Proposal("flip")
    key = derive_key(6, "chains")
    a = sampler.ChainEnsemble(600, n, prop, ev, key)
    a.run_steps(1500)
    np.testing.assert_array_equal(a.log_probs, ev(a.bits))
    s0 = sampler.ChainEnsemble(250, n, prop, ev, key, chain_offset=0, n_chains_total=600)
    s1 = sampler.ChainEnsemble(350, n, prop, ev, key, chain_offset=250, n_chains_total=600)
    for s in (s0, s1):
        s.run_steps(1500)
    np.testing.assert_array_equal(np.concatenate([s0.bits, s1.bits]), a.bits)
