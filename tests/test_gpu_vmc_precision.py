"""North-star VMC precision gate (row N1): the ground-state energy reached by
training with f16 / bf16 / f32 NATIVE sampling agrees with the f64-sampling
result within the paper's MH bias bound plus the across-seed spread, and every
format reaches the exact ground state.

Protocol (the reference's vmc.train, vmc.py:472-639,
and SPEC acceptance #10, read with the plateau rule because the
reference fails the per-step band itself): N=10 open TFIM chain, alpha=1, 500
SR steps, 4,096 samples, lambda 1e-3, eta 0.01, seeds 0-4, h in {0.5, 1}.
Plateau = mean energy of the last 100 steps.  Gate for each reduced format:

    |<plateau_fmt> - <plateau_f64>| <= B + 3 sqrt(s_fmt^2/5 + s_f64^2/5)

with <.> and s the mean and standard deviation over seeds and B the paper's
bias bound 2 max|eps| TV, TV <= min(Pinsker(sigma_hat), Theorem 3(sigma_hat))
averaged over the plateau records (bounds.py:78-83, 217-229), max|eps| over
the final state's samples.  E0 comes from the oracle's exact diagonalisation,
pinned to the reference's exact_ground_state (tests/golden/ed.npz).
"""
import numpy as np
import pytest

from paper_2601_20782_b200 import BF16, F16, F32, F64, RoundingMode, rbm, sampler, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec

pytestmark = pytest.mark.gpu
SEEDS = range(5)
FORMATS = (F64, F32, F16, BF16)


def _train(spec, fmt, seed, e0):
    mode = RoundingMode.PER_OPERATION if fmt is F64 else RoundingMode.NATIVE
    cfg = vmc.TrainConfig(spec, alpha=1, n_steps=500, n_samples=4096, lambda_shift=1e-3, eta=0.01,
                          sampling_format=fmt, rounding_mode=mode, seed=seed, reference_energy=e0)
    res = vmc.train(cfg)
    recs = res.records[-100:]
    plateau = float(np.mean([r["energy"] for r in recs]))
    tv = float(np.mean([min(r["bound_pinsker"], r["bound_theorem3"]) for r in recs]))
    # max |eps| over the final state's samples (the bias bound's energy scale)
    ev = rbm.log_prob_evaluator(res.params, fmt, mode)
    samples, _ = sampler.run_chains(512, 4096, 20 * spec.lattice.n_sites, spec.lattice.n_sites + 1, 99, ev,
                                    sampler.Proposal("flip"), spec.lattice.n_sites)
    eps_max = float(np.abs(vmc.local_energies(spec, rbm.log_psi_evaluator(res.params), samples)).max())
    return plateau, tv, eps_max


@pytest.mark.parametrize("h", [0.5, 1.0])
def test_vmc_ground_state_energy_reduced_vs_f64(cuda, h):
    from conftest import golden

    from oracle import ed

    spec = TfimSpec(LatticeSpec.chain(10), 1.0, h)
    e0 = ed.ground_energy("tfim", 10, spec.lattice.bond_array(), 1.0, h)
    assert e0 == pytest.approx(float(golden("ed.npz")[f"tfim_chain10_h{h:g}"]), abs=1e-10)
    out = {}
    for fmt in FORMATS:
        runs = [_train(spec, fmt, s, e0) for s in SEEDS]
        pl = np.array([r[0] for r in runs])
        out[fmt.name] = {"mean": float(pl.mean()), "std": float(pl.std(ddof=1)),
                         "tv": float(np.mean([r[1] for r in runs])), "eps_max": float(max(r[2] for r in runs)),
                         "rel_err_e0": abs(float(pl.mean()) - e0) / abs(e0)}
    print(f"\n[N1 gate] TFIM chain N=10 h={h} E0={e0:.8f}")
    for k, v in out.items():
        print(f"   {k:5s} plateau {v['mean']:.6f} +- {v['std']:.2e} (seeds)  rel err vs E0 {v['rel_err_e0']:.2e}  "
              f"TV bound {v['tv']:.2e}  max|eps| {v['eps_max']:.2f}")
    ref = out["f64"]
    for name in ("f32", "f16", "bf16"):
        v = out[name]
        bias = 2.0 * v["eps_max"] * v["tv"]
        spread = 3.0 * np.sqrt(v["std"] ** 2 / len(SEEDS) + ref["std"] ** 2 / len(SEEDS))
        assert abs(v["mean"] - ref["mean"]) <= bias + spread, (name, v, ref, bias, spread)
    for name, v in out.items():
        assert v["rel_err_e0"] < 1e-2, (name, v)
