"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference lives at /root/reference, read-only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box never runs this (it has no
/root/reference); tests load the committed .npz files.  Every array here is an
output of the unmodified reference API (mpvmc), so the oracle and the CUDA path
are pinned to the reference's own numbers.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from mpvmc import rbm, sampler, vmc  # noqa: E402
from mpvmc.bounds import pinsker_tv_bound, theorem3_gaussian_bound  # noqa: E402
from mpvmc.hamiltonians import HeisenbergSpec, TfimSpec, exact_ground_state  # noqa: E402
from mpvmc.lattice import LatticeSpec  # noqa: E402
from mpvmc.precision import BF16, F16, F32, F64, RoundingMode  # noqa: E402
from mpvmc.rng import StreamSet, derive_key, mix64  # noqa: E402
from mpvmc.sampler import ChainEnsemble, Proposal, run_chains  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FMTS = {"f64": F64, "f32": F32, "f16": F16, "bf16": BF16}
PER_OP = RoundingMode.PER_OPERATION


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def gen_rng():
    paths = [(0, ("chains",)), (0, ("init",)), (7, ("train",)), (7, ("chain", 0)), (7, ("chain", 1)),
             (12345, ("params",)), (3, ("chains",)), (2**63 + 5, ("noise", 4))]
    keys = np.array([derive_key(s, *p) for s, p in paths], dtype=np.uint64)
    key = derive_key(0, "chains")
    streams = StreamSet(key, 37)
    draws = np.array([streams.next_uniform() for _ in range(50)])  # (50, 37)
    mix_in = np.array([0, 1, 2, 0xDEADBEEF, 2**64 - 1], dtype=np.uint64)
    save("rng.npz", path_seeds=np.array([s for s, _ in paths], dtype=np.uint64),
         path_labels=np.array(["/".join(map(str, p)) for _, p in paths]), keys=keys,
         stream_key=np.uint64(key), stream_draws=draws, mix_in=mix_in, mix_out=mix64(mix_in))


def random_bits(rng, n_rows, n):
    bits = rng.integers(0, 2, size=(n_rows, n), dtype=np.uint8)
    bits[0] = 0
    bits[1] = 1
    return bits


def gen_forward():
    cases = [(10, 1, 5, 0.5), (16, 2, 6, 0.3), (12, 1, 7, 0.01), (20, 1, 8, 1.0)]
    arrays = {}
    rng = np.random.default_rng(2601)
    for ci, (n, alpha, seed, scale) in enumerate(cases):
        p = rbm.random_parameters(n, alpha, derive_key(seed, "params"), scale)
        bits = random_bits(rng, 160, n)
        arrays[f"c{ci}_meta"] = np.array([n, alpha, seed, scale])
        arrays[f"c{ci}_a"], arrays[f"c{ci}_b"], arrays[f"c{ci}_w"] = p.a, p.b, p.w
        arrays[f"c{ci}_bits"] = bits
        for name, fmt in FMTS.items():
            arrays[f"c{ci}_{name}_lp"] = rbm.log_prob_batch(p, bits, fmt, PER_OP)
            arrays[f"c{ci}_{name}_psi"] = rbm.log_psi_batch(p, bits, fmt, PER_OP)
            snap = rbm.round_parameters(p, fmt)
            arrays[f"c{ci}_{name}_snap_a"] = snap.a
            arrays[f"c{ci}_{name}_snap_b"] = snap.b
            arrays[f"c{ci}_{name}_snap_w"] = snap.w
            if name != "f64":
                arrays[f"c{ci}_{name}_storage_lp"] = rbm.log_prob_batch(
                    p, bits, fmt, RoundingMode.STORAGE_ONLY)
    # SURVEY §8(c) value: p = random_parameters(4, 1, derive_key(0,"params"), 0.5), bits [1,0,1,1]
    p = rbm.random_parameters(4, 1, derive_key(0, "params"), 0.5)
    x = np.array([[1, 0, 1, 1]], dtype=np.uint8)
    for name, fmt in FMTS.items():
        arrays[f"kat_{name}_lp"] = rbm.log_prob_batch(p, x, fmt, PER_OP)
    arrays["kat_a"], arrays["kat_b"], arrays["kat_w"] = p.a, p.b, p.w
    # random_parameters for the host init (ndtri of counter uniforms)
    q = rbm.random_parameters(6, 2, derive_key(11, "init"), 0.01)
    arrays["init_a"], arrays["init_b"], arrays["init_w"] = q.a, q.b, q.w
    save("forward.npz", n_cases=np.array(len(cases)), **arrays)


def gen_chains():
    arrays = {}
    n, alpha = 12, 2
    p = rbm.random_parameters(n, alpha, derive_key(0, "params"), 0.4)
    arrays["a"], arrays["b"], arrays["w"] = p.a, p.b, p.w
    key = derive_key(3, "chains")
    arrays["key"] = np.uint64(key)
    checkpoints = [0, 1, 50, 300]
    for kind, weight in (("flip", None), ("exchange", 6)):
        for name, fmt in FMTS.items():
            ev = rbm.log_prob_evaluator(p, fmt, PER_OP)
            ens = ChainEnsemble(64, n, Proposal(kind, weight), ev, key)
            done = 0
            for cp in checkpoints:
                ens.run_steps(cp - done)
                done = cp
                arrays[f"{kind}_{name}_bits_{cp}"] = ens.bits
                arrays[f"{kind}_{name}_logp_{cp}"] = ens.log_probs
                arrays[f"{kind}_{name}_acc_{cp}"] = np.array(ens.accepted)
    # run_chains layouts
    for ri, (c, s, burn, thin) in enumerate([(64, 200, 37, 13), (50, 50, 0, 1), (40, 7, 5, 3)]):
        for name in ("f64", "f32"):
            ev = rbm.log_prob_evaluator(p, FMTS[name], PER_OP)
            samples, rate = run_chains(c, s, burn, thin, 9, ev, Proposal("flip"), n)
            arrays[f"run{ri}_{name}_samples"] = samples
            arrays[f"run{ri}_{name}_rate"] = np.array(rate)
            arrays[f"run{ri}_args"] = np.array([c, s, burn, thin, 9])
    # run_chains(4, 8, 10, 5, seed 0, f32 per-op, flip, n=4)
    p4 = rbm.random_parameters(4, 1, derive_key(0, "params"), 0.5)
    samples, rate = run_chains(4, 8, 10, 5, 0, rbm.log_prob_evaluator(p4, F32, PER_OP), Proposal("flip"), 4)
    arrays["kat4_samples"], arrays["kat4_rate"] = samples, np.array(rate)
    save("chains.npz", **arrays)


def gen_energy():
    arrays = {}
    rng = np.random.default_rng(77)
    specs = [
        ("tfim_chain10", TfimSpec(LatticeSpec.chain(10), 1.0, 0.7)),
        ("tfim_sq4", TfimSpec(LatticeSpec.square(4), 1.0, 3.04)),
        ("heis_chain8", HeisenbergSpec(LatticeSpec.chain(8, periodic=True), 1.0)),
        ("heis_sq4", HeisenbergSpec(LatticeSpec.square(4), 1.0)),
        ("tfim_chain20_open", TfimSpec(LatticeSpec.chain(20), 1.0, 1.0)),
        ("tfim_sq10", TfimSpec(LatticeSpec.square(10), 1.0, 3.04)),
    ]
    for tag, spec in specs:
        n = spec.lattice.n_sites
        p = rbm.random_parameters(n, 2, derive_key(5, tag), 0.3)
        if isinstance(spec, HeisenbergSpec):
            bits = np.zeros((48, n), dtype=np.uint8)
            for r in range(48):
                bits[r, rng.permutation(n)[: n // 2]] = 1
        else:
            bits = rng.integers(0, 2, size=(48, n), dtype=np.uint8)
        arrays[f"{tag}_bonds"] = spec.lattice.bond_array()
        arrays[f"{tag}_a"], arrays[f"{tag}_b"], arrays[f"{tag}_w"] = p.a, p.b, p.w
        arrays[f"{tag}_bits"] = bits
        arrays[f"{tag}_eps"] = vmc.local_energies(spec, rbm.log_psi_evaluator(p), bits)
        arrays[f"{tag}_coupling"] = np.array([spec.j, getattr(spec, "h", 0.0)])
    for tag, spec in [("ed_tfim8", TfimSpec(LatticeSpec.chain(8), 1.0, 1.0)),
                      ("ed_heis8", HeisenbergSpec(LatticeSpec.chain(8, periodic=True), 1.0)),
                      ("ed_tfim3x3", TfimSpec(LatticeSpec.square(3), 1.0, 3.04))]:
        e0, _ = exact_ground_state(spec)
        arrays[tag] = np.array(e0)
    # the survey's chain-4 KAT
    p = rbm.random_parameters(4, 1, derive_key(0, "params"), 0.5)
    x = np.array([[1, 0, 1, 1]], dtype=np.uint8)
    arrays["kat_tfim4"] = vmc.local_energies(TfimSpec(LatticeSpec.chain(4), 1, 1), rbm.log_psi_evaluator(p), x)
    arrays["kat_heis4"] = vmc.local_energies(HeisenbergSpec(LatticeSpec.chain(4), 1), rbm.log_psi_evaluator(p), x)
    sig = np.array([0.0, 1e-4, 1e-2, 0.3, 1.0, 2.0])
    arrays["bound_sigma"] = sig
    arrays["bound_pinsker"] = np.array([pinsker_tv_bound(s) for s in sig])
    arrays["bound_theorem3"] = np.array([theorem3_gaussian_bound(s, 0.0, 0.0) for s in sig])
    save("energy.npz", **arrays)


def gen_train():
    """Reference training runs (vmc.py:472-639) for tests/test_gpu_train.py."""
    from mpvmc.precision import F32
    from mpvmc.sampler import Proposal

    arrays = {}
    runs = {
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
    keys = ("energy", "mc_error", "acceptance", "sigma_hat", "bound_pinsker", "bound_theorem3", "kappa")
    for tag, cfg in runs.items():
        res = vmc.train(vmc.TrainConfig(**cfg))
        for k in keys:
            arrays[f"{tag}_{k}"] = np.array([r[k] for r in res.records], dtype=np.float64)
        arrays[f"{tag}_w"] = res.params.w
    save("train.npz", **arrays)


def gen_table():
    """Reference ChainEnsemble / run_chains driven by table_log_prob evaluators
    (sampler.py:254-268) -> tests/golden/table_chains.npz."""
    from mpvmc.sampler import table_log_prob, uniform_log_prob

    arrays = {}
    n = 6
    table = np.random.default_rng(11).normal(0.0, 1.5, 1 << n)
    table[5] = -np.inf  # an unreachable state
    arrays["table"] = table
    key = derive_key(8, "chains")
    arrays["key"] = np.uint64(key)
    for kind, weight in (("flip", None), ("exchange", 3)):
        ens = ChainEnsemble(40, n, Proposal(kind, weight), table_log_prob(table, n), key)
        done = 0
        for cp in (0, 1, 50, 400):
            ens.run_steps(cp - done)
            done = cp
            arrays[f"{kind}_bits_{cp}"] = ens.bits
            arrays[f"{kind}_logp_{cp}"] = ens.log_probs
            arrays[f"{kind}_acc_{cp}"] = np.array(ens.accepted)
    samples, rate = run_chains(8, 64, 5, 1, 42, uniform_log_prob(4), Proposal("flip"), 4)
    arrays["uniform_samples"], arrays["uniform_rate"] = samples, np.array(rate)
    samples, rate = run_chains(16, 64, 10, 3, 4, table_log_prob(table, n), Proposal("exchange", 3), n)
    arrays["exchange_samples"], arrays["exchange_rate"] = samples, np.array(rate)
    save("table_chains.npz", **arrays)


def gen_noisy():
    """Reference ChainEnsemble with noisy_log_prob_evaluator (rbm.py:333-352,
    408-416) -> tests/golden/noisy_chains.npz."""
    arrays = {}
    n = 10
    p = rbm.random_parameters(n, 2, derive_key(3, "noisy"), 0.3)
    arrays["a"], arrays["b"], arrays["w"] = p.a, p.b, p.w
    noise = rbm.NoiseField(0.4, 5)
    key = derive_key(6, "chains")
    arrays["key"] = np.uint64(key)
    ev = rbm.noisy_log_prob_evaluator(p, noise)
    bits = np.random.default_rng(4).integers(0, 2, size=(64, n), dtype=np.uint8)
    arrays["eval_bits"], arrays["eval_lp"] = bits, ev(bits)
    ens = ChainEnsemble(64, n, Proposal("flip"), ev, key)
    done = 0
    for cp in (0, 1, 50, 300):
        ens.run_steps(cp - done)
        done = cp
        arrays[f"bits_{cp}"], arrays[f"logp_{cp}"] = ens.bits, ens.log_probs
        arrays[f"acc_{cp}"] = np.array(ens.accepted)
    save("noisy_chains.npz", **arrays)


def gen_delta():
    """rbm.delta_distribution (rbm.py:440-469) and normality.shapiro_wilk on
    fixed inputs -> tests/golden/delta.npz."""
    from mpvmc import normality
    from mpvmc.lattice import LatticeSpec as RefLattice

    arrays = {}
    for tag, (n, alpha, seed, scale, fmt) in {
            "f16_n12": (12, 1, 16, 0.05, F16), "bf16_n8": (8, 2, 15, 0.3, BF16), "f32_n8": (8, 2, 15, 0.3, F32),
            "f16_n14": (14, 1, 3, 0.2, F16)}.items():
        p = rbm.random_parameters(n, alpha, derive_key(seed, "delta"), scale)
        summary, delta = rbm.delta_distribution(p, fmt, PER_OP, RefLattice.chain(n))
        arrays[f"{tag}_delta"] = delta
        arrays[f"{tag}_summary"] = np.array([summary.mean, summary.std, summary.skewness, summary.excess_kurtosis,
                                             summary.shapiro_wilk_w, summary.shapiro_n])
        arrays[f"{tag}_meta"] = np.array([n, alpha, seed, scale])
    x = np.random.default_rng(5).standard_t(5, size=777)
    arrays["sw_x"] = x
    arrays["sw_w"] = np.array(normality.shapiro_wilk(x).w)
    arrays["sw_a20"] = normality._sw_coefficients(20)
    save("delta.npz", **arrays)


def gen_formats():
    """The reference's training-log writer (experiments.py:222-237, 611-624) on
    fixed records -> tests/golden/training_log_ref.csv (formats.py parity)."""
    from mpvmc import experiments as ex

    recs = [{"step": 0, "energy": -1.2345678901234567, "mc_error": 0.01, "acceptance": 0.5, "sigma_hat": 0.0,
             "bound_pinsker": 0.0, "bound_theorem3": 0.0, "kappa": float("nan"), "rel_error": 1e-3},
            {"step": 1, "energy": np.float64(3.0), "mc_error": np.float32(0.25), "acceptance": 1,
             "sigma_hat": 1e-300, "bound_pinsker": 5e-301, "bound_theorem3": 2.5, "kappa": 12.0,
             "sampling_seconds": 0.5, "update_seconds": 0.25}]
    rows = [ex._record_row(("f16",), r) for r in recs]
    path = os.path.join(OUT, "training_log_ref.csv")
    ex.write_csv(path, ["format", *ex._LOG_COLUMNS, "rel_error"], rows)
    print(f"wrote {path}")


def gen_params():
    """rbm.random_parameters / round_parameters of the reference at the bench's
    shapes: full arrays at configs[0] (N=20, alpha=1), SHA-256 digests of the
    arrays' bytes at configs[1] (N=100, alpha=2) and configs[2] (alpha=4)."""
    import hashlib

    out = {}
    p = rbm.random_parameters(20, 1, derive_key(0, "init"), 0.01)
    out["c20_a"], out["c20_b"], out["c20_w"] = p.a, p.b, p.w
    for f in ("f32", "f16", "bf16"):
        r = rbm.round_parameters(p, FMTS[f])
        out[f"c20_{f}_w"] = r.w
    for alpha in (2, 4):
        p = rbm.random_parameters(100, alpha, derive_key(0, "init"), 0.01)
        for f in ("f64", "f32", "f16", "bf16"):
            r = rbm.round_parameters(p, FMTS[f])
            h = hashlib.sha256()
            for arr in (r.a, r.b, r.w):
                h.update(np.ascontiguousarray(arr, dtype=np.complex128).tobytes())
            out[f"c100a{alpha}_{f}_sha256"] = np.array(h.hexdigest())
    save("params.npz", **out)


def gen_ed():
    """Exact ground-state energies (hamiltonians.exact_ground_state) that pin
    the oracle's dense diagonalisation (the VMC precision gate's E0)."""
    cases = {"tfim_chain10_h0.5": TfimSpec(LatticeSpec.chain(10), 1.0, 0.5),
             "tfim_chain10_h1": TfimSpec(LatticeSpec.chain(10), 1.0, 1.0),
             "tfim_sq3_h3.04": TfimSpec(LatticeSpec.square(3), 1.0, 3.04),
             "heis_chain8": HeisenbergSpec(LatticeSpec.chain(8), 1.0)}
    save("ed.npz", **{k: np.float64(exact_ground_state(v)[0]) for k, v in cases.items()})


if __name__ == "__main__":
    if sys.argv[1:] == ["ed"]:
        gen_ed()
        sys.exit(0)
    if sys.argv[1:] == ["params"]:
        gen_params()
        sys.exit(0)
    if sys.argv[1:] == ["formats"]:
        gen_formats()
        sys.exit(0)
    if sys.argv[1:] == ["table"]:
        gen_table()
        sys.exit(0)
    if sys.argv[1:] == ["noisy"]:
        gen_noisy()
        sys.exit(0)
    if sys.argv[1:] == ["delta"]:
        gen_delta()
        sys.exit(0)
    gen_ed()
    gen_params()
    gen_formats()
    gen_table()
    gen_noisy()
    gen_delta()
    gen_train()
    gen_rng()
    gen_forward()
    gen_chains()
    gen_energy()
