"""Wall-clock breakdown of one end-to-end bench step through the public API
(host buffers): snapshot build, sweeps, collect (D2H), local energies (H2D + kernel + D2H)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_20782_b200 import rbm, vmc
from paper_2601_20782_b200.hamiltonians import TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.precision import F16, RoundingMode
from paper_2601_20782_b200.rng import derive_key
from paper_2601_20782_b200.sampler import ChainEnsemble, Proposal

spec = TfimSpec(LatticeSpec.square(10), 1.0, 3.04)
params = rbm.random_parameters(100, 2, derive_key(0, "init"), 0.01)
psi = rbm.log_psi_evaluator(params)
ev = rbm.log_prob_evaluator(params, F16, RoundingMode.NATIVE)
ens = ChainEnsemble(16384, 100, Proposal("flip"), ev, derive_key(0, "chains"))
ens.run_sweeps(4)
for it in range(4):
    t = [time.perf_counter()]
    ev2 = rbm.log_prob_evaluator(params, F16, RoundingMode.NATIVE); torch.cuda.synchronize(); t.append(time.perf_counter())
    ens.set_evaluator(ev2, check=False); ens.reset_counters(); ens.run_sweeps(2, check=False); torch.cuda.synchronize(); t.append(time.perf_counter())
    s = ens.collect(65536, 101); t.append(time.perf_counter())
    eps = vmc.local_energies(spec, psi, s); t.append(time.perf_counter())
    e = float(eps.real.mean()); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("snapshot %.3f  sweeps %.3f  collect %.3f  energies %.3f  mean %.3f  total %.3f ms" % (*d, sum(d)))
