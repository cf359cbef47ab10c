"""Host-side logic of the product package (no GPU): key derivation, parameter
init and rounding, lattices, bit packing, the exact-theta planner."""
from fractions import Fraction

import numpy as np
import pytest

from paper_2601_20782_b200 import hamiltonians, precision, rbm
from paper_2601_20782_b200.lattice import LatticeSpec, pack_bits, unpack_bits
from paper_2601_20782_b200.rng import counter_uniform, derive_key, mix64
from paper_2601_20782_b200.sampler import Proposal, default_chain_count, pair_table


def test_derive_key_matches_reference(g_rng):
    for seed, label, key in zip(g_rng["path_seeds"], g_rng["path_labels"], g_rng["keys"]):
        path = [int(p) if p.isdigit() else p for p in str(label).split("/")]
        assert derive_key(int(seed), *path) == key
    for z_in, z_out in zip(g_rng["mix_in"], g_rng["mix_out"]):
        assert mix64(int(z_in)) == int(z_out)


def test_random_parameters_match_reference(g_forward):
    p = rbm.random_parameters(6, 2, derive_key(11, "init"), 0.01)
    assert np.array_equal(p.a, g_forward["init_a"])
    assert np.array_equal(p.b, g_forward["init_b"])
    assert np.array_equal(p.w, g_forward["init_w"])


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_round_parameters_match_reference(g_forward, fmt):
    for ci in range(int(g_forward["n_cases"])):
        p = rbm.RbmParameters(g_forward[f"c{ci}_a"], g_forward[f"c{ci}_b"], g_forward[f"c{ci}_w"])
        snap = rbm.round_parameters(p, precision.FORMATS[fmt])
        assert np.array_equal(snap.a, g_forward[f"c{ci}_{fmt}_snap_a"])
        assert np.array_equal(snap.b, g_forward[f"c{ci}_{fmt}_snap_b"])
        assert np.array_equal(snap.w, g_forward[f"c{ci}_{fmt}_snap_w"])


def test_bond_lists_match_reference(g_energy):
    cases = {"tfim_chain10": LatticeSpec.chain(10), "tfim_sq4": LatticeSpec.square(4),
             "heis_chain8": LatticeSpec.chain(8, periodic=True), "tfim_sq10": LatticeSpec.square(10),
             "tfim_chain20_open": LatticeSpec.chain(20)}
    for tag, lat in cases.items():
        assert np.array_equal(lat.bond_array(), g_energy[f"{tag}_bonds"])
    assert len(LatticeSpec.square(10).bonds) == 200
    assert len(LatticeSpec.square(16).bonds) == 512


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    for n in (1, 7, 31, 32, 33, 100, 256):
        bits = rng.integers(0, 2, size=(17, n), dtype=np.uint8)
        packed = pack_bits(bits)
        assert packed.shape == (17, (n + 31) // 32) and packed.dtype == np.uint32
        assert np.array_equal(unpack_bits(packed, n), bits)
        k = rng.integers(0, n)
        assert ((packed[:, k >> 5] >> (k & 31)) & 1 == bits[:, k]).all()


def test_pair_table_lexicographic():
    n = 7
    want = [(i, j) for i in range(n) for j in range(i + 1, n)]
    assert pair_table(n).tolist() == [list(p) for p in want]
    assert pair_table(100).shape == (4950, 2)


def test_formats_and_modes():
    assert precision.F16.unit_roundoff == 2.0**-11 and precision.BF16.unit_roundoff == 2.0**-8
    assert precision.parse_format("e5m10").significand_bits == 10
    assert precision.parse_rounding_mode("native") is precision.RoundingMode.NATIVE
    assert precision.round_to_format(0.1, precision.BF16) == 0.10009765625  # ref tests/test_precision.py:61-62
    assert np.isinf(precision.round_to_format(70000.0, precision.F16))
    with pytest.raises(ValueError):
        Proposal("swap")
    assert default_chain_count(4096) == 1024


def test_counter_uniform_stateless():
    key = derive_key(3, "noise")
    a = counter_uniform(key, np.arange(100))
    assert np.array_equal(a, counter_uniform(key, np.arange(100)))
    assert (a > 0).all() and (a < 1).all()


def _exact_sums_fit_f32(values_fn, n_trials, rng, plan, snap):
    """Every partial sum b_i + sum_{k in S} W_ik must be exactly representable
    in the accumulator the planner picked (checked with rational arithmetic)."""
    N, M = snap.n_visible, snap.n_hidden
    for _ in range(n_trials):
        x = rng.integers(0, 2, N)
        i = rng.integers(0, M)
        for part in (np.real, np.imag):
            total = Fraction(float(part(snap.b[i])))
            for k in np.flatnonzero(x):
                total += Fraction(float(part(snap.w[i, k])))
                if plan.variant == 0:  # X1: the f32 accumulator holds the exact value
                    assert Fraction(float(np.float32(float(total)))) == total


@pytest.mark.parametrize("scale,fmt,variant", [(0.01, "f16", 0), (0.5, "f16", 3), (0.3, "bf16", None)])
def test_exact_planner(scale, fmt, variant):
    p = rbm.random_parameters(100, 1, derive_key(0, "init"), scale)
    snap = rbm.round_parameters(p, precision.FORMATS[fmt])
    plan = rbm.plan_exact(snap)
    if variant is not None:
        assert plan.variant == variant
    assert plan.quantum > 0 and plan.bound > 0
    # all snapshot values are multiples of the quantum
    vals = np.concatenate([snap.w.real.ravel(), snap.w.imag.ravel(), snap.b.real, snap.b.imag])
    assert np.all(np.mod(vals / plan.quantum, 1.0) == 0)
    if plan.variant == 1:
        g = plan.split
        hi = np.rint(vals / g) * g
        lo = vals - hi
        # hi/lo exactly representable in the format, lo bounded by split/2
        rnd = precision.make_rounder(precision.FORMATS[fmt])
        assert np.array_equal(rnd(hi), hi) and np.array_equal(rnd(lo), lo)
        assert np.max(np.abs(lo)) <= g / 2
    _exact_sums_fit_f32(None, 200, np.random.default_rng(1), plan, snap)


def test_parameters_io_roundtrip(tmp_path):
    p = rbm.random_parameters(5, 2, derive_key(1, "io"), 0.3)
    rbm.save_parameters(p, tmp_path / "p.json")
    q = rbm.load_parameters(tmp_path / "p.json")
    assert np.array_equal(p.a, q.a) and np.array_equal(p.w, q.w)
    assert p.n_params == 5 + 10 + 50
    with pytest.raises(ValueError):
        rbm.RbmParameters(np.zeros(3), np.zeros(3), np.zeros((2, 3)))


def test_lattice_next_nearest_and_sublattice():
    assert LatticeSpec.chain(10, periodic=True).next_nearest_bonds().shape == (10, 2)
    assert LatticeSpec.square(4).next_nearest_bonds().shape == (32, 2)
    assert LatticeSpec.square(4, periodic=False).next_nearest_bonds().shape == (18, 2)
    assert LatticeSpec.square(10).next_nearest_bonds().shape == (200, 2)
    with pytest.raises(ValueError):
        LatticeSpec.square(3).sublattice()
    with pytest.raises(ValueError):
        hamiltonians.HeisenbergSpec(LatticeSpec.chain(9, periodic=True), 1.0, marshall=True)


def test_training_log_format_matches_reference(tmp_path):
    """formats.record_row/write_csv reproduce the reference's writer byte for
    byte (golden file from experiments.py's own write_csv, make_golden.py)."""
    import os

    from paper_2601_20782_b200 import formats

    recs = [{"step": 0, "energy": -1.2345678901234567, "mc_error": 0.01, "acceptance": 0.5, "sigma_hat": 0.0,
             "bound_pinsker": 0.0, "bound_theorem3": 0.0, "kappa": float("nan"), "rel_error": 1e-3},
            {"step": 1, "energy": np.float64(3.0), "mc_error": np.float32(0.25), "acceptance": 1,
             "sigma_hat": 1e-300, "bound_pinsker": 5e-301, "bound_theorem3": 2.5, "kappa": 12.0,
             "sampling_seconds": 0.5, "update_seconds": 0.25}]
    out = formats.write_csv(tmp_path / "log.csv", ["format", *formats.LOG_COLUMNS, "rel_error"],
                            [formats.record_row(("f16",), r) for r in recs])
    golden = os.path.join(os.path.dirname(__file__), "golden", "training_log_ref.csv")
    assert open(out).read() == open(golden).read()
    back = formats.read_training_log(out)
    assert back[0]["format"] == "f16" and back[1]["step"] == 1 and back[0]["energy"] == -1.23456789012346


def test_training_log_sidecar_and_samples(tmp_path):
    import json

    from paper_2601_20782_b200 import formats

    class R:
        records = [{"step": 0, "energy": 1.0, "mc_error": 0.1, "acceptance": 0.5, "sigma_hat": 0.0,
                    "bound_pinsker": 0.0, "bound_theorem3": 0.0, "kappa": 2.0}]

    path = formats.write_training_log(tmp_path / "run", {"f64": R(), "f16": R()}, {"train": {"steps": 1}}, -1.5)
    meta = json.load(open(f"{path}.meta.json"))
    assert meta["reference_energy"] == -1.5 and meta["config"] == {"train": {"steps": 1}}
    assert [r["format"] for r in formats.read_training_log(path)] == ["f64", "f16"]
    smp = np.random.default_rng(0).integers(0, 2, size=(7, 5), dtype=np.uint8)
    p = formats.save_samples(tmp_path / "s.npy", smp)
    assert np.array_equal(formats.load_samples(p), smp)


def test_shapiro_wilk_matches_reference():
    """normality.shapiro_wilk / sw_coefficients equal the reference's
    (golden from normality.py itself, tests/golden/make_golden.py gen_delta)."""
    import os

    from paper_2601_20782_b200 import normality

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "delta.npz"))
    np.testing.assert_allclose(normality.sw_coefficients(20), g["sw_a20"], rtol=1e-14, atol=1e-15)
    assert normality.shapiro_wilk(g["sw_x"]).w == pytest.approx(float(g["sw_w"]), rel=1e-13)
