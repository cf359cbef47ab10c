"""The device sampler driven by table evaluators (ref sampler.py:254-268
table_log_prob / uniform_log_prob): trajectories bit-identical to the
reference's ChainEnsemble and run_chains (golden, tests/golden/make_golden.py
gen_table), plus the reference's own sampler KATs (tests/test_sampler.py:38-118):
uniform target always accepts, zero-probability states are never entered,
two-state occupation band, uniform multinomial bands with acceptance exactly 1,
exchange moves conserve the sector."""
import numpy as np
import pytest

from paper_2601_20782_b200 import sampler
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu
FLIP = sampler.Proposal("flip")


@pytest.mark.parametrize("kind,weight", [("flip", None), ("exchange", 3)])
def test_table_trajectories_match_reference(cuda, g_table, kind, weight):
    n = 6
    ens = sampler.ChainEnsemble(40, n, sampler.Proposal(kind, weight), sampler.table_log_prob(g_table["table"], n),
                                int(g_table["key"]))
    done = 0
    for cp in (0, 1, 50, 400):
        ens.run_steps(cp - done)
        done = cp
        np.testing.assert_array_equal(ens.bits, g_table[f"{kind}_bits_{cp}"])
        np.testing.assert_array_equal(ens.log_probs, g_table[f"{kind}_logp_{cp}"])
        assert ens.accepted == int(g_table[f"{kind}_acc_{cp}"])


def test_table_run_chains_match_reference(cuda, g_table):
    s, rate = sampler.run_chains(8, 64, 5, 1, 42, sampler.uniform_log_prob(4), FLIP, 4)
    np.testing.assert_array_equal(s, g_table["uniform_samples"])
    assert rate == float(g_table["uniform_rate"])
    s, rate = sampler.run_chains(16, 64, 10, 3, 4, sampler.table_log_prob(g_table["table"], 6),
                                 sampler.Proposal("exchange", 3), 6)
    np.testing.assert_array_equal(s, g_table["exchange_samples"])
    assert rate == float(g_table["exchange_rate"])


def test_uniform_target_always_accepts(cuda):
    ens = sampler.ChainEnsemble(16, 3, FLIP, sampler.uniform_log_prob(3), derive_key(0, "chains"))
    ens.run_steps(200)
    assert ens.accepted == ens.proposed == 16 * 200


def test_zero_probability_state_never_entered(cuda):
    table = np.zeros(4)
    table[2] = -np.inf
    ens = sampler.ChainEnsemble(64, 2, FLIP, sampler.table_log_prob(table, 2), derive_key(1, "chains"))
    for _ in range(50):
        ens.run_steps(10)
        codes = ens.bits[:, 0] + 2 * ens.bits[:, 1]
        assert not np.any(codes == 2)


def test_two_state_occupation(cuda):
    # pi = (2/3, 1/3); the n = 1 flip chain has P = [[1/2, 1/2], [1, 0]] (ref test_sampler.py:61-80)
    table = np.log(np.array([2.0, 1.0]))
    ens = sampler.ChainEnsemble(4096, 1, FLIP, sampler.table_log_prob(table, 1), derive_key(7, "chains"))
    ens.run_sweeps(100)
    steps = 2000
    samples = ens.collect(4096 * steps, 1)
    pi0 = 2.0 / 3.0
    rho = -0.5  # second eigenvalue of P
    total = samples.shape[0]
    visits = int((samples[:, 0] == 0).sum())
    band = 3.0 * np.sqrt(pi0 * (1 - pi0) * (1 + rho) / (1 - rho) / total)
    assert abs(visits / total - pi0) <= band


def test_uniform_multinomial_bands(cuda):
    n = 4
    s, rate = sampler.run_chains(250, 100_000, 80, 13, 3, sampler.uniform_log_prob(n), FLIP, n)
    assert rate == 1.0
    codes = (s.astype(np.int64) << np.arange(n)).sum(axis=1)
    freqs = np.bincount(codes, minlength=16) / s.shape[0]
    p = 1.0 / 16.0
    assert (np.abs(freqs - p) <= 3 * np.sqrt(p * (1 - p) / s.shape[0])).all()


def test_exchange_preserves_sector(cuda):
    s, _ = sampler.run_chains(16, 64, 10, 1, 4, sampler.uniform_log_prob(6), sampler.Proposal("exchange", 3), 6)
    assert (s.sum(axis=1) == 3).all()


def test_table_evaluator_callable(cuda, g_table):
    ev = sampler.table_log_prob(g_table["table"], 6)
    bits = np.array([[1, 0, 1, 0, 0, 0], [1, 1, 1, 1, 1, 1]], dtype=np.uint8)
    np.testing.assert_array_equal(ev(bits), g_table["table"][[5, 63]])
