"""The device training loop (vmc.train) against the reference's own runs
(tests/golden/train.npz, produced by mpvmc.vmc.train): identical samples in
per-operation mode give the same energies, errors, acceptance, sigma-hat,
bounds and condition numbers step by step."""
import numpy as np
import pytest

from paper_2601_20782_b200 import F16, F32, vmc
from paper_2601_20782_b200.hamiltonians import HeisenbergSpec, TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.sampler import Proposal

pytestmark = pytest.mark.gpu

RUNS = {
    "exact6": dict(hamiltonian=TfimSpec(LatticeSpec.chain(6), 1.0, 1.0), n_steps=30, sampling_mode="exact",
                   eta=0.05, lambda_shift=1e-3, seed=2),
    "mcmc8_f32": dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=6, n_samples=256,
                      n_chains=64, eta=0.02, seed=3, sampling_format=F32),
    "mcmc8_f64": dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=6, n_samples=256,
                      n_chains=64, eta=0.02, seed=3),
    "heis6_f16": dict(hamiltonian=HeisenbergSpec(LatticeSpec.chain(6, periodic=True), 1.0), n_steps=4,
                      n_samples=128, n_chains=32, eta=0.02, seed=4, sampling_format=F16,
                      proposal=Proposal("exchange", 3)),
}


@pytest.fixture(scope="module")
def g_train():
    from conftest import golden

    return golden("train.npz")


@pytest.mark.parametrize("tag", list(RUNS))
def test_train_matches_reference(cuda, g_train, tag):
    res = vmc.train(vmc.TrainConfig(**RUNS[tag]))
    got = {k: np.array([r[k] for r in res.records]) for k in ("energy", "mc_error", "acceptance", "sigma_hat",
                                                                 "bound_pinsker", "bound_theorem3", "kappa")}
    for k, tol in (("energy", 1e-9), ("mc_error", 1e-7), ("sigma_hat", 1e-7), ("bound_pinsker", 1e-7),
                   ("bound_theorem3", 1e-7), ("kappa", 1e-5)):
        ref = g_train[f"{tag}_{k}"]
        np.testing.assert_allclose(got[k], ref, rtol=tol, atol=1e-12, err_msg=k)
    ref_acc = g_train[f"{tag}_acceptance"]
    assert np.array_equal(np.isnan(got["acceptance"]), np.isnan(ref_acc))
    assert np.allclose(got["acceptance"][~np.isnan(ref_acc)], ref_acc[~np.isnan(ref_acc)], rtol=0, atol=0)
    np.testing.assert_allclose(res.params.w, g_train[f"{tag}_w"], rtol=1e-7, atol=1e-10)


def test_train_deterministic_and_timed(cuda):
    cfg = dict(hamiltonian=TfimSpec(LatticeSpec.chain(8), 1.0, 1.0), n_steps=3, n_samples=128, n_chains=32,
               seed=5, sampling_format=F16, track_timings=True)
    a, b = vmc.train(vmc.TrainConfig(**cfg)), vmc.train(vmc.TrainConfig(**cfg))
    for ra, rb in zip(a.records, b.records):
        for k in ("energy", "mc_error", "acceptance", "sigma_hat"):
            assert ra[k] == rb[k]
        assert ra["sampling_seconds"] > 0 and ra["update_seconds"] > 0
    assert a.records[0]["sigma_hat"] > 0.0
