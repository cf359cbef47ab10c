"""f64 local energies on the device (ref vmc.py:52-108) against the reference's
own values (golden) and the oracle."""
import numpy as np
import pytest

from oracle import port
from paper_2601_20782_b200 import rbm, vmc
from paper_2601_20782_b200.hamiltonians import HeisenbergSpec, TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec, enumerate_bits
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu

SPECS = {
    "tfim_chain10": TfimSpec(LatticeSpec.chain(10), 1.0, 0.7),
    "tfim_sq4": TfimSpec(LatticeSpec.square(4), 1.0, 3.04),
    "heis_chain8": HeisenbergSpec(LatticeSpec.chain(8, periodic=True), 1.0),
    "heis_sq4": HeisenbergSpec(LatticeSpec.square(4), 1.0),
    "tfim_chain20_open": TfimSpec(LatticeSpec.chain(20), 1.0, 1.0),
    "tfim_sq10": TfimSpec(LatticeSpec.square(10), 1.0, 3.04),
}


@pytest.mark.parametrize("tag", list(SPECS))
def test_local_energies_match_reference(cuda, g_energy, tag):
    p = rbm.RbmParameters(g_energy[f"{tag}_a"], g_energy[f"{tag}_b"], g_energy[f"{tag}_w"])
    eps = vmc.local_energies(SPECS[tag], rbm.log_psi_evaluator(p), g_energy[f"{tag}_bits"])
    ref = g_energy[f"{tag}_eps"]
    assert np.max(np.abs(eps - ref) / np.maximum(1, np.abs(ref))) < 1e-12


def test_survey_kats(cuda, g_energy):
    p = rbm.random_parameters(4, 1, derive_key(0, "params"), 0.5)
    x = np.array([[1, 0, 1, 1]], dtype=np.uint8)
    t = vmc.local_energies(TfimSpec(LatticeSpec.chain(4), 1, 1), rbm.log_psi_evaluator(p), x)[0]
    h = vmc.local_energies(HeisenbergSpec(LatticeSpec.chain(4), 1), rbm.log_psi_evaluator(p), x)[0]
    assert abs(t - (10.739983075592015 + 3.879113787655884j)) < 1e-12
    assert abs(h - (32.249841779268294 + 33.27953711487039j)) < 1e-12
    assert t == pytest.approx(complex(g_energy["kat_tfim4"][0]), rel=1e-13)


def test_uniform_state_tfim(cuda):
    """ref tests/test_vmc.py:39-47: eps = 3 on the uniform state, N=2."""
    p = rbm.RbmParameters(np.zeros(2, complex), np.zeros(2, complex), np.zeros((2, 2), complex))
    v = vmc.local_energies(TfimSpec(LatticeSpec.chain(2), 1.0, 1.0), rbm.log_psi_evaluator(p),
                           np.array([[0, 0]], dtype=np.uint8))[0]
    assert abs(v - 3.0) < 1e-13


@pytest.mark.parametrize("spec", [TfimSpec(LatticeSpec.chain(6), 1.0, 0.7), HeisenbergSpec(LatticeSpec.chain(5), 1.0)])
def test_enumerated_energy_is_rayleigh_quotient(cuda, spec):
    """ref tests/test_vmc.py:57-69, with a dense Hamiltonian restated here."""
    n = spec.lattice.n_sites
    p = rbm.random_parameters(n, 1, derive_key(0, "p"), 0.4)
    bits = enumerate_bits(n)
    lp = rbm.log_prob_batch(p, bits)
    w = np.exp(lp - lp.max())
    w /= w.sum()
    eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
    energy = float((w @ eps).real)
    psi = np.exp(rbm.log_psi_batch(p, bits) - lp.max() / 2)
    H = _dense(spec, n)
    rq = float((np.conj(psi) @ H @ psi).real / (np.conj(psi) @ psi).real)
    assert energy == pytest.approx(rq, abs=1e-10)


def _dense(spec, n):
    codes = np.arange(1 << n)
    bits = ((codes[:, None] >> np.arange(n)) & 1)
    s = 1 - 2 * bits
    bonds = spec.lattice.bond_array()
    H = np.diag(spec.j * (s[:, bonds[:, 0]] * s[:, bonds[:, 1]]).sum(axis=1).astype(float))
    if isinstance(spec, TfimSpec):
        for i in range(n):
            H[codes, codes ^ (1 << i)] += spec.h
    else:
        for i, k in bonds:
            d = bits[:, i] != bits[:, k]
            H[codes[d], codes[d] ^ ((1 << i) | (1 << k))] += 2 * spec.j
    return H


def test_large_weights_use_stable_path(cuda):
    """|Re W| > 4 switches a term to the log-cosh difference; still matches the oracle."""
    n = 12
    p = rbm.random_parameters(n, 2, derive_key(6, "big"), 3.0)
    bits = np.random.default_rng(2).integers(0, 2, size=(40, n), dtype=np.uint8)
    for spec, ham in ((TfimSpec(LatticeSpec.chain(n, True), 1.0, 0.9), "tfim"),
                      (HeisenbergSpec(LatticeSpec.chain(n, True), 1.0), "heisenberg")):
        eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
        want = port.local_energies(port.Params(p.a, p.b, p.w), ham, spec.lattice.bond_array(), spec.j,
                                   getattr(spec, "h", 0.0), bits)
        assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-9


def test_large_lattice_against_oracle(cuda):
    spec = TfimSpec(LatticeSpec.square(16), 1.0, 3.04)
    p = rbm.random_parameters(256, 1, derive_key(7, "sq16"), 0.05)
    bits = np.random.default_rng(3).integers(0, 2, size=(24, 256), dtype=np.uint8)
    eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
    want = port.local_energies(port.Params(p.a, p.b, p.w), "tfim", spec.lattice.bond_array(), 1.0, 3.04, bits)
    assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-11


@pytest.mark.parametrize("n,alpha,B", [(3, "1/3", 5), (5, "3/5", 17), (7, 3, 33), (12, "5/4", 49), (33, 1, 20),
                                       (65, "6/5", 21), (40, 6, 9)])
def test_odd_shapes_against_oracle(cuda, n, alpha, B):
    """M not a multiple of 4 (DMMA tile edges), N across word boundaries, sample
    counts not a multiple of the 16-sample block, many hidden units (M = 240)."""
    from fractions import Fraction

    p = rbm.random_parameters(n, Fraction(alpha), derive_key(n, "odd"), 0.4)
    bits = np.random.default_rng(n).integers(0, 2, size=(B, n), dtype=np.uint8)
    for spec, ham in ((TfimSpec(LatticeSpec.chain(n, n >= 3), 0.7, 1.3), "tfim"),
                      (HeisenbergSpec(LatticeSpec.chain(n, n >= 3), 1.1), "heisenberg")):
        eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
        want = port.local_energies(port.Params(p.a, p.b, p.w), ham, spec.lattice.bond_array(), spec.j,
                                   getattr(spec, "h", 0.0), bits)
        assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-10, (n, alpha, ham)


@pytest.mark.parametrize("spec,alpha", [(TfimSpec(LatticeSpec.chain(140, True), 1.0, 0.8), "1/2"),
                                        (HeisenbergSpec(LatticeSpec.square(12), 1.0), "1/3"),
                                        (TfimSpec(LatticeSpec.square(16), 1.0, 3.0), "1/8")],
                         ids=["tfim140", "heis12x12_288bonds", "tfim16x16_M32"])
def test_many_terms_launch_configs(cuda, spec, alpha):
    """Term counts beyond the 4-samples-per-thread block (T > 112) and beyond
    256 (one 8-sample group per block) against the oracle."""
    from fractions import Fraction

    n = spec.lattice.n_sites
    p = rbm.random_parameters(n, Fraction(alpha), derive_key(n, "many"), 0.2)
    rng = np.random.default_rng(n)
    bits = rng.integers(0, 2, size=(19, n), dtype=np.uint8)
    eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
    ham = "tfim" if isinstance(spec, TfimSpec) else "heisenberg"
    want = port.local_energies(port.Params(p.a, p.b, p.w), ham, spec.lattice.bond_array(), spec.j,
                               getattr(spec, "h", 0.0), bits)
    assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-10


def test_bench_shapes_against_oracle(cuda):
    """The energy launches of the bench's configs[2] (Heisenberg 10x10, alpha=4:
    200 bonds, 400 hidden units; compacted 4-sample units, one block of up to 25
    warps per SM) and configs[3]-shape J1-J2 (400 bonds, alpha=1: 8-sample
    blocks) against the oracle.  J1-J2 is linear in the couplings: the oracle
    value is the sum of two Heisenberg evaluations over the J1 and J2 bonds."""
    from paper_2601_20782_b200.hamiltonians import J1J2Spec

    lat = LatticeSpec.square(10)
    rng = np.random.default_rng(11)
    bits = np.zeros((37, 100), dtype=np.uint8)
    np.put_along_axis(bits, np.argsort(rng.random((37, 100)), axis=1)[:, :50], 1, axis=1)
    bits[-1] = rng.integers(0, 2, size=100)  # one row off the Sz = 0 sector
    p4 = rbm.random_parameters(100, 4, derive_key(5, "heis-a4"), 0.05)
    eps = vmc.local_energies(HeisenbergSpec(lat, 1.0), rbm.log_psi_evaluator(p4), bits)
    want = port.local_energies(port.Params(p4.a, p4.b, p4.w), "heisenberg", lat.bond_array(), 1.0, 0.0, bits)
    assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-10
    p1 = rbm.random_parameters(100, 1, derive_key(5, "j1j2-a1"), 0.05)
    eps = vmc.local_energies(J1J2Spec(lat, 1.0, 0.5), rbm.log_psi_evaluator(p1), bits)
    pp = port.Params(p1.a, p1.b, p1.w)
    want = (port.local_energies(pp, "heisenberg", lat.bond_array(), 1.0, 0.0, bits)
            + port.local_energies(pp, "heisenberg", lat.next_nearest_bonds(), 0.5, 0.0, bits))
    assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-10
