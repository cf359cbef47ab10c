"""Config-2 VMC iteration (65,536 samples, P = 20,300, device-resident CG): per-step update times."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2601_20782_b200 import F16, RoundingMode, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec

cfg = vmc.TrainConfig(TfimSpec(LatticeSpec.square(10), 1.0, 3.04), alpha=2, n_steps=6, n_samples=65536, n_chains=16384,
                      sampling_format=F16, rounding_mode=RoundingMode.NATIVE, track_timings=True, sr_solver="cg",
                      cg_tol=1e-8, burn_in_sweeps=200)
recs = vmc.train(cfg, local=True).records
for r in recs:
    print("step %d update %.1f ms sampling %.2f ms cg %d" % (r["step"], 1e3 * r["update_seconds"], 1e3 * r["sampling_seconds"],
                                                             r["cg_iterations"]))
