"""Where the config-1 VMC iteration (N=20 TFIM chain, alpha=1, 4,096 samples, dense SR) spends its time."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.precision import F16, RoundingMode

for kappa in (True, False):
    cfg = vmc.TrainConfig(TfimSpec(LatticeSpec.chain(20), 1.0, 1.0), alpha=1, n_steps=12, n_samples=4096, n_chains=1024,
                          sampling_format=F16, rounding_mode=RoundingMode.NATIVE, track_timings=True, compute_kappa=kappa)
    recs = vmc.train(cfg, local=True).records[2:]
    import numpy as np
    print("kappa", kappa, "sampling %.2f ms update %.2f ms" % (1e3 * np.median([r["sampling_seconds"] for r in recs]),
                                                           1e3 * np.median([r["update_seconds"] for r in recs])), flush=True)
cfg = vmc.TrainConfig(TfimSpec(LatticeSpec.chain(20), 1.0, 1.0), alpha=1, n_steps=4, n_samples=4096, n_chains=1024,
                      sampling_format=F16, rounding_mode=RoundingMode.NATIVE, track_timings=True)
vmc.train(cfg, local=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    vmc.train(cfg, local=True)
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
