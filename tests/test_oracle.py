"""The CPU oracle (oracle/) pinned to golden vectors produced by the reference
itself (tests/golden/make_golden.py).  Runs without a GPU."""
import numpy as np
import pytest

from oracle import port
from oracle import rng as orng

FMTS = ("f64", "f32", "f16", "bf16")


def test_stream_draws_match_streamset(g_rng):
    draws = port.stream_uniforms(int(g_rng["stream_key"]), 37, 50)
    assert np.array_equal(draws, g_rng["stream_draws"])
    np_draws = orng.stream_uniforms(g_rng["stream_key"], np.arange(37)[None, :], np.arange(50)[:, None])
    assert np.array_equal(np_draws, g_rng["stream_draws"])


def test_mix64_and_keys(g_rng):
    assert np.array_equal(orng.mix64(g_rng["mix_in"]), g_rng["mix_out"])
    for seed, label, key in zip(g_rng["path_seeds"], g_rng["path_labels"], g_rng["keys"]):
        path = [int(p) if p.isdigit() else p for p in str(label).split("/")]
        assert orng.derive_key(int(seed), *path) == key
    assert int(orng.derive_key(0, "chains")) == 0xA91B32726445095B


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_per_op_forward_bitwise(g_forward, fmt):
    for ci in range(int(g_forward["n_cases"])):
        p = port.Params(g_forward[f"c{ci}_{fmt}_snap_a"], g_forward[f"c{ci}_{fmt}_snap_b"], g_forward[f"c{ci}_{fmt}_snap_w"])
        bits = g_forward[f"c{ci}_bits"]
        lp, re, im = port.rounded_forward(p, bits, fmt)
        psi = g_forward[f"c{ci}_{fmt}_psi"]
        assert np.array_equal(lp, g_forward[f"c{ci}_{fmt}_lp"])
        assert np.array_equal(re, psi.real) and np.array_equal(im, psi.imag)
        assert np.array_equal(port.rounded_log_prob(p, bits, fmt), lp)


def test_f64_forward(g_forward):
    for ci in range(int(g_forward["n_cases"])):
        p = port.Params(g_forward[f"c{ci}_a"], g_forward[f"c{ci}_b"], g_forward[f"c{ci}_w"])
        lp, re, im = port.f64_forward(p, g_forward[f"c{ci}_bits"])
        ref = g_forward[f"c{ci}_f64_psi"]
        assert np.max(np.abs(re - ref.real) / np.maximum(1, np.abs(ref.real))) < 1e-13
        assert np.max(np.abs(im - ref.imag) / np.maximum(1, np.abs(ref.imag))) < 1e-13


def test_survey_kat_values(g_forward):
    # bits [1,0,1,1] per-op log p in each format
    want = {"f64": -0.37474936330837283, "f32": -0.3747496008872986, "f16": -0.37646484375, "bf16": -0.37890625}
    for fmt, v in want.items():
        assert g_forward[f"kat_{fmt}_lp"][0] == v
        if fmt != "f64":
            from paper_2601_20782_b200 import rbm
            from paper_2601_20782_b200.precision import FORMATS

            snap = rbm.round_parameters(rbm.RbmParameters(g_forward["kat_a"], g_forward["kat_b"], g_forward["kat_w"]),
                                        FORMATS[fmt])
            lp = port.rounded_log_prob(port.Params(snap.a, snap.b, snap.w), np.array([[1, 0, 1, 1]]), fmt)
            assert lp[0] == v


@pytest.mark.parametrize("kind,weight", [("flip", None), ("exchange", 6)])
@pytest.mark.parametrize("fmt", FMTS)
def test_chain_ensemble_lockstep(g_chains, g_forward, kind, weight, fmt):
    from paper_2601_20782_b200 import rbm
    from paper_2601_20782_b200.precision import FORMATS

    snap = rbm.round_parameters(rbm.RbmParameters(g_chains["a"], g_chains["b"], g_chains["w"]), FORMATS[fmt])
    ens = port.PortEnsemble(64, 12, kind, weight, port.Params(snap.a, snap.b, snap.w), fmt, int(g_chains["key"]))
    done = 0
    for cp in (0, 1, 50, 300):
        ens.run_steps(cp - done)
        done = cp
        assert np.array_equal(ens.bits, g_chains[f"{kind}_{fmt}_bits_{cp}"])
        assert ens.accepted == int(g_chains[f"{kind}_{fmt}_acc_{cp}"])
        ref = g_chains[f"{kind}_{fmt}_logp_{cp}"]
        tol = 1e-13 if fmt == "f64" else 0.0
        assert np.max(np.abs(ens.logp - ref) / np.maximum(1, np.abs(ref))) <= tol


@pytest.mark.parametrize("ri", [0, 1, 2])
@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_run_chains_layout(g_chains, ri, fmt):
    from paper_2601_20782_b200 import rbm
    from paper_2601_20782_b200.precision import FORMATS
    from paper_2601_20782_b200.rng import derive_key

    c, s, burn, thin, seed = (int(v) for v in g_chains[f"run{ri}_args"])
    snap = rbm.round_parameters(rbm.RbmParameters(g_chains["a"], g_chains["b"], g_chains["w"]), FORMATS[fmt])
    ens = port.PortEnsemble(c, 12, "flip", None, port.Params(snap.a, snap.b, snap.w), fmt, int(derive_key(seed, "chains")))
    ens.run_steps(burn)
    ens.reset_counters()
    samples = ens.collect(s, thin)
    assert np.array_equal(samples, g_chains[f"run{ri}_{fmt}_samples"])
    assert ens.accepted / ens.proposed == float(g_chains[f"run{ri}_{fmt}_rate"])


TAGS = ["tfim_chain10", "tfim_sq4", "heis_chain8", "heis_sq4", "tfim_chain20_open", "tfim_sq10"]


@pytest.mark.parametrize("tag", TAGS)
def test_local_energies(g_energy, tag):
    p = port.Params(g_energy[f"{tag}_a"], g_energy[f"{tag}_b"], g_energy[f"{tag}_w"])
    J, h = g_energy[f"{tag}_coupling"]
    ham = "tfim" if tag.startswith("tfim") else "heisenberg"
    eps = port.local_energies(p, ham, g_energy[f"{tag}_bonds"], J, h, g_energy[f"{tag}_bits"])
    ref = g_energy[f"{tag}_eps"]
    assert np.max(np.abs(eps - ref) / np.maximum(1, np.abs(ref))) < 1e-11


def test_oracle_parameters_match_reference():
    """oracle random_parameters / round_parameters (the reference arm's inputs)
    == the reference's rbm.random_parameters / round_parameters (golden)."""
    import hashlib

    from conftest import golden

    g = golden("params.npz")
    a, b, w = port.random_parameters(20, 1, orng.derive_key(0, "init"), 0.01)
    assert np.array_equal(a, g["c20_a"]) and np.array_equal(b, g["c20_b"]) and np.array_equal(w, g["c20_w"])
    for f in ("f32", "f16", "bf16"):
        assert np.array_equal(port.round_parameters(a, b, w, f)[2], g[f"c20_{f}_w"])
    for alpha in (2, 4):
        a, b, w = port.random_parameters(100, alpha, orng.derive_key(0, "init"), 0.01)
        for f in ("f64", "f32", "f16", "bf16"):
            h = hashlib.sha256()
            for arr in port.round_parameters(a, b, w, f):
                h.update(np.ascontiguousarray(arr, dtype=np.complex128).tobytes())
            assert h.hexdigest() == str(g[f"c100a{alpha}_{f}_sha256"]), (alpha, f)


def test_oracle_exact_diagonalisation_matches_reference():
    from conftest import golden

    from oracle import ed
    from paper_2601_20782_b200.lattice import LatticeSpec

    g = golden("ed.npz")
    chain10 = LatticeSpec.chain(10).bond_array()
    assert ed.ground_energy("tfim", 10, chain10, 1.0, 0.5) == pytest.approx(float(g["tfim_chain10_h0.5"]), abs=1e-10)
    assert ed.ground_energy("tfim", 10, chain10, 1.0, 1.0) == pytest.approx(float(g["tfim_chain10_h1"]), abs=1e-10)
    assert ed.ground_energy("tfim", 9, LatticeSpec.square(3).bond_array(), 1.0, 3.04) == pytest.approx(
        float(g["tfim_sq3_h3.04"]), abs=1e-10)
    assert ed.ground_energy("heisenberg", 8, LatticeSpec.chain(8).bond_array(), 1.0) == pytest.approx(
        float(g["heis_chain8"]), abs=1e-10)


def test_oracle_sparse_diagonalisation_matches_dense():
    from oracle import ed
    from paper_2601_20782_b200.lattice import LatticeSpec

    for kind, lat, j, h in (("tfim", LatticeSpec.chain(10), 1.0, 0.5), ("heisenberg", LatticeSpec.square(3), 1.0, 0.0)):
        n = lat.n_sites
        dense = ed.ground_energy(kind, n, lat.bond_array(), j, h)
        assert ed.ground_energy_sparse([(kind, lat.bond_array(), j, h)], n) == pytest.approx(dense, abs=1e-9)
