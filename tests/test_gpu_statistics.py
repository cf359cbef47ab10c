"""f16/bf16 NATIVE sampling: statistical parity (north_star: f16/bf16 energies
within error bars and the paper's analytical MH bias bound of the f64 result).

On an enumerable system (N=10 TFIM chain) the device's own perturbed target
pi~ (log p of the NATIVE arithmetic, a fixed function of x) is computed
exactly, so we check
  (i)  the exact TV(pi, pi~) obeys Pinsker with the exact KL and the paper's
       Gaussian-noise bound sigma/2 (SURVEY §8(d) gate (i)),
  (ii) the chains sample pi~: the MCMC energy agrees with the exact E under
       pi~ within 4 split-chain standard errors,
  (iii) the bias |E_pi~ - E_pi| is within 2 max|eps| TV (the bias bound).
"""
import math

import numpy as np
import pytest

from paper_2601_20782_b200 import F16, F64, BF16, RoundingMode, parallel, rbm, sampler, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec, enumerate_bits
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu


def _softmax(lp):
    w = np.exp(lp - lp.max())
    return w / w.sum()


@pytest.mark.parametrize("fmt", [F16, BF16])
def test_native_reduced_precision_target_and_bias(cuda, fmt):
    n = 10
    spec = TfimSpec(LatticeSpec.chain(n), 1.0, 1.0)
    p = rbm.random_parameters(n, 1, derive_key(2, "stat"), 0.5)
    bits = enumerate_bits(n)
    lp64 = rbm.log_prob_batch(p, bits, F64)
    ev = rbm.log_prob_evaluator(p, fmt, RoundingMode.NATIVE)
    lpf = ev(bits)
    pi, pit = _softmax(lp64), _softmax(lpf)
    delta = lpf - lp64
    sigma = math.sqrt(max(float(pi @ delta**2 - (pi @ delta) ** 2), 0.0))
    tv = 0.5 * float(np.abs(pi - pit).sum())
    kl = float(pit @ (np.log(pit) - np.log(pi)))
    assert tv <= math.sqrt(kl / 2) + 1e-12  # Pinsker (rigorous)
    assert tv <= 1.5 * sigma / 2 + 1e-6  # paper's Gaussian-noise bound, with slack for non-Gaussian delta
    eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits).real
    e_pi, e_pit = float(pi @ eps), float(pit @ eps)
    assert abs(e_pit - e_pi) <= 2 * np.abs(eps).max() * tv + 1e-12

    chains, n_samples = 2048, 2048 * 16
    ens = sampler.ChainEnsemble(chains, n, sampler.Proposal("flip"), ev, derive_key(3, "chains"))
    ens.run_sweeps(100)
    ens.reset_counters()
    samples = ens.collect(n_samples, n + 1)
    codes = (samples.astype(np.int64) << np.arange(n)).sum(axis=1)
    e_s = eps[codes]
    counts = parallel.chain_counts(n_samples, chains, 0, chains)
    ids = np.repeat(np.arange(chains), counts)
    means = np.bincount(ids, weights=e_s) / counts
    err = float(np.sqrt(means.var(ddof=1) / chains))
    assert abs(float(e_s.mean()) - e_pit) <= 4 * err, (float(e_s.mean()), e_pit, err)
    # the empirical distribution is close to pi~
    hist = np.bincount(codes, minlength=1 << n) / n_samples
    assert 0.5 * np.abs(hist - pit).sum() < 0.12


@pytest.mark.parametrize("case", ["tfim10x10_flat", "tfim_chain20_peaked"])
def test_native_f16_energy_gate_mcmc_vs_f64(cuda, case):
    """SURVEY §8(d) f16 gate (ii): with identical sampler settings the f16
    NATIVE MCMC energy agrees with the f64 MCMC energy of the reference's own
    ChainEnsemble (the oracle's restatement, CPU: same parameters, key, chains
    and schedule) within 3 combined split-chain errors plus the paper's bias
    bound 2 max|eps| (sigma_hat / 2), at sizes that cannot be enumerated
    (N = 100 flat, N = 20 peaked); the device's f64 chains take the oracle's
    decisions (sample rows identical up to near-threshold ties)."""
    from oracle import port

    if case == "tfim10x10_flat":
        spec, alpha, scale, chains, per_chain, burn = TfimSpec(LatticeSpec.square(10), 1.0, 3.04), 2, 0.01, 1024, 8, 50
    else:
        spec, alpha, scale, chains, per_chain, burn = TfimSpec(LatticeSpec.chain(20), 1.0, 1.0), 1, 0.3, 4096, 16, 200
    n = spec.lattice.n_sites
    p = rbm.random_parameters(n, alpha, derive_key(5, case), scale)
    psi = rbm.log_psi_evaluator(p)
    key = derive_key(6, case)
    n_samples = chains * per_chain
    counts = parallel.chain_counts(n_samples, chains, 0, chains)
    ids = np.repeat(np.arange(chains), counts)

    def stats(samples):
        eps = vmc.local_energies(spec, psi, samples).real
        means = np.bincount(ids, weights=eps) / counts
        return float(eps.mean()), float(np.sqrt(means.var(ddof=1) / chains)), eps

    ref = port.PortEnsemble(chains, n, "flip", None, port.Params(p.a, p.b, p.w), "f64", int(key))
    ref.run_steps(burn * n)
    ref_samples = ref.collect(n_samples, n + 1)
    e64, err64, _ = stats(ref_samples)
    dev64 = sampler.ChainEnsemble(chains, n, sampler.Proposal("flip"), rbm.log_prob_evaluator(p, F64), key)
    dev64.run_steps(burn * n)
    assert np.mean(np.all(dev64.collect(n_samples, n + 1) == ref_samples, axis=1)) > 0.99
    ev = rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
    ens = sampler.ChainEnsemble(chains, n, sampler.Proposal("flip"), ev, key)
    ens.run_steps(burn * n)
    s16 = ens.collect(n_samples, n + 1)
    e16, err16, eps16 = stats(s16)
    lp16 = ev(s16)
    lp64 = rbm.log_prob_batch(p, s16, F64)
    sigma_hat = float(np.std(lp16 - lp64))
    bias = 2 * float(np.abs(eps16).max()) * min(1.0, sigma_hat / 2)
    assert abs(e16 - e64) <= 3 * math.hypot(err16, err64) + bias, (e16, e64, err16, err64, sigma_hat)
