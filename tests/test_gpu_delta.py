"""delta(x) = log p_fmt - log p_f64 over the enumeration on the device
(ref rbm.py:440-469 delta_distribution), per-operation
evaluators are bit-exact so the delta field and its summary equal the
reference's own (golden)."""
import os

import numpy as np
import pytest

from paper_2601_20782_b200 import BF16, F16, F32, F64, RoundingMode, rbm
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "delta.npz"))
FMT = {"f16": F16, "bf16": BF16, "f32": F32}


@pytest.mark.parametrize("tag", ["f16_n12", "bf16_n8", "f32_n8", "f16_n14"])
def test_delta_distribution_matches_reference(cuda, tag):
    n, alpha, seed, scale = G[f"{tag}_meta"]
    n, alpha, seed = int(n), int(alpha), int(seed)
    p = rbm.random_parameters(n, alpha, derive_key(seed, "delta"), float(scale))
    summary, delta = rbm.delta_distribution(p, FMT[tag.split("_")[0]], RoundingMode.PER_OPERATION, LatticeSpec.chain(n))
    np.testing.assert_allclose(delta, G[f"{tag}_delta"], rtol=0, atol=1e-12)
    want = G[f"{tag}_summary"]
    got = np.array([summary.mean, summary.std, summary.skewness, summary.excess_kurtosis, summary.shapiro_wilk_w,
                    summary.shapiro_n])
    np.testing.assert_allclose(got, want, rtol=1e-8, atol=1e-12)


def test_f64_delta_zero(cuda):
    p = rbm.random_parameters(6, 1, derive_key(14, "delta"), 0.3)
    summary, delta = rbm.delta_distribution(p, F64, RoundingMode.PER_OPERATION, LatticeSpec.chain(6))
    assert summary.std == 0.0 and np.array_equal(delta, np.zeros(64))


def test_native_delta_smaller_than_per_operation(cuda):
    """The NATIVE f16 arithmetic (exact theta, f32 accumulation) perturbs the
    target less than the reference's per-op f16 (the gap grows
    with M — here M = 12 and the ratio is ~0.6)."""
    p = rbm.random_parameters(12, 1, derive_key(16, "delta"), 0.3)
    s_op, _ = rbm.delta_distribution(p, F16, RoundingMode.PER_OPERATION, LatticeSpec.chain(12))
    s_nat, _ = rbm.delta_distribution(p, F16, RoundingMode.NATIVE, LatticeSpec.chain(12))
    assert 0.0 < s_nat.std < 0.8 * s_op.std
