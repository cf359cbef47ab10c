"""Local energies beyond the reference: J1-J2 Heisenberg and
the Marshall sign.  No reference code exists, so parity is pinned by an exact
restatement: on enumerable lattices every configuration's local energy must
equal (H psi)(x) / psi(x) with H applied to the full amplitude vector
(Pauli-matrix convention of the reference's HeisenbergSpec, hamiltonians.py:1-7:
diagonal J s_p s_q, off-diagonal 2J on anti-aligned bonds), psi_M(x) =
(-1)^{#bits set on sublattice A} psi(x) for the Marshall-rotated amplitude."""
import numpy as np
import pytest

from paper_2601_20782_b200 import rbm, vmc
from paper_2601_20782_b200.hamiltonians import HeisenbergSpec, J1J2Spec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu


def _all_bits(n):
    codes = np.arange(1 << n, dtype=np.int64)
    return ((codes[:, None] >> np.arange(n)) & 1).astype(np.uint8)


def _log_psi(p, bits):
    x = bits.astype(np.float64)
    theta = x @ p.w.T + p.b[None, :]
    return x @ p.a + np.log(np.cosh(theta)).sum(axis=1)


def _exact_eps(spec, p, bits, marshall):
    """(H psi)(x) / psi(x) for every row of the full enumeration `bits`."""
    n = bits.shape[1]
    codes = (bits.astype(np.int64) << np.arange(n)).sum(axis=1)
    assert np.array_equal(codes, np.arange(1 << n))
    lp = _log_psi(p, bits)
    if marshall:
        sub = spec.lattice.sublattice()
        lp = lp + 1j * np.pi * (bits[:, sub == 0].sum(axis=1) % 2)
    bonds, jb, _ = spec.couplings() if hasattr(spec, "couplings") else (None, None, None)
    eps = np.zeros(1 << n, dtype=np.complex128)
    s = 1 - 2 * bits.astype(np.int64)
    for (i, j), J in zip(bonds, jb):
        eps += J * s[:, i] * s[:, j]
        anti = bits[:, i] != bits[:, j]
        partner = codes ^ ((1 << i) | (1 << j))
        eps[anti] += 2 * J * np.exp(lp[partner[anti]] - lp[anti])
    return eps


CASES = [
    ("j1j2_chain10", J1J2Spec(LatticeSpec.chain(10, periodic=True), 1.0, 0.5), 2, 0.3),
    ("j1j2_chain10_marshall", J1J2Spec(LatticeSpec.chain(10, periodic=True), 1.0, 0.5, marshall=True), 2, 0.3),
    ("heis_sq4open_marshall", HeisenbergSpec(LatticeSpec.square(4, periodic=False), 1.0, marshall=True), 1, 0.2),
    ("j1j2_sq4_marshall", J1J2Spec(LatticeSpec.square(4), 1.0, 0.55, marshall=True), 1, 0.2),
    ("j1j2_sq4_frustrated", J1J2Spec(LatticeSpec.square(4), 0.8, 1.0), 2, 0.1),
]


@pytest.mark.parametrize("tag,spec,alpha,scale", CASES, ids=[c[0] for c in CASES])
def test_local_energies_exact_hamiltonian(cuda, tag, spec, alpha, scale):
    n = spec.lattice.n_sites
    p = rbm.random_parameters(n, alpha, derive_key(9, tag), scale)
    bits = _all_bits(n)
    want = _exact_eps(spec, p, bits, spec.marshall)
    got = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
    err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    assert err.max() < 1e-10, (tag, err.max())


def test_marshall_sign_is_a_sign_rule(cuda):
    """Marshall only flips the off-diagonal signs of inter-sublattice bonds:
    with J2 = 0 the Rayleigh quotient of psi_M is <psi|H_M|psi>, and the
    diagonal parts of eps are unchanged."""
    lat = LatticeSpec.chain(8, periodic=True)
    p = rbm.random_parameters(8, 1, derive_key(4, "marshall"), 0.3)
    bits = _all_bits(8)
    psi = rbm.log_psi_evaluator(p)
    e0 = vmc.local_energies(HeisenbergSpec(lat, 1.0), psi, bits)
    e1 = vmc.local_energies(HeisenbergSpec(lat, 1.0, marshall=True), psi, bits)
    e2 = vmc.local_energies(J1J2Spec(lat, 1.0, 0.0, marshall=True), psi, bits)
    s = 1 - 2 * bits.astype(np.int64)
    diag = (s * np.roll(s, -1, axis=1)).sum(axis=1)
    np.testing.assert_allclose((e0 + e1) / 2, diag, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(e1, e2, rtol=1e-12, atol=1e-12)
