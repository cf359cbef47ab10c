"""10x10 TFIM (h=3.04, alpha=1) minSR training with f16 NATIVE vs f64 sampling, long run:
energy per site every 100 steps and the last-200-step plateau (north-star precision leg)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2601_20782_b200 import F16, F64, RoundingMode, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
eta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for fmt in (F16, F64):
    mode = RoundingMode.NATIVE if fmt is not F64 else RoundingMode.PER_OPERATION
    c = vmc.TrainConfig(TfimSpec(LatticeSpec.square(10), 1.0, 3.04), alpha=1, n_steps=steps, n_samples=4096,
                        n_chains=1024, sampling_format=fmt, rounding_mode=mode, sr_solver="minsr",
                        compute_kappa=False, eta=eta, lambda_shift=1e-2, burn_in_sweeps=100)
    t0 = time.perf_counter()
    r = vmc.train(c, local=True).records
    e = np.array([x["energy"] for x in r]) / 100
    print(fmt.name, "wall %.1f s" % (time.perf_counter() - t0),
          " ".join("%.4f" % e[i:i + 100].mean() for i in range(0, steps, 100)),
          "| plateau(last 200) %.5f +- %.5f, mc_err %.5f, tv %.2e" % (
              e[-200:].mean(), e[-200:].std(), np.mean([x["mc_error"] for x in r[-200:]]) / 100,
              np.mean([min(x["bound_pinsker"], x["bound_theorem3"]) for x in r[-200:]])), flush=True)
