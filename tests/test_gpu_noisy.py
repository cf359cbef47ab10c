"""noisy_log_prob_evaluator on the device (ref rbm.py:333-352 NoiseField,
rbm.py:408-416): f64 log p plus the frozen Gaussian field sigma*ndtri(u(code));
evaluations and MH trajectories against the reference's own run (golden)."""
import numpy as np
import pytest

from paper_2601_20782_b200 import rbm, sampler

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g_noisy():
    import os

    return np.load(os.path.join(os.path.dirname(__file__), "golden", "noisy_chains.npz"))


def _ev(g):
    p = rbm.RbmParameters(g["a"], g["b"], g["w"])
    return rbm.noisy_log_prob_evaluator(p, rbm.NoiseField(0.4, 5))


def test_noisy_evaluations_match_reference(cuda, g_noisy):
    got = _ev(g_noisy)(g_noisy["eval_bits"])
    np.testing.assert_allclose(got, g_noisy["eval_lp"], rtol=1e-12, atol=1e-12)


def test_noisy_trajectories_match_reference(cuda, g_noisy):
    ens = sampler.ChainEnsemble(64, 10, sampler.Proposal("flip"), _ev(g_noisy), int(g_noisy["key"]))
    done = 0
    for cp in (0, 1, 50, 300):
        ens.run_steps(cp - done)
        done = cp
        np.testing.assert_array_equal(ens.bits, g_noisy[f"bits_{cp}"])
        np.testing.assert_allclose(ens.log_probs, g_noisy[f"logp_{cp}"], rtol=1e-12, atol=1e-12)
        assert ens.accepted == int(g_noisy[f"acc_{cp}"])


def test_noise_requires_f64_and_64_sites(cuda):
    p = rbm.random_parameters(70, 1, 0, 0.1)
    with pytest.raises(ValueError):
        rbm.noisy_log_prob_evaluator(p, rbm.NoiseField(0.1, 0))
