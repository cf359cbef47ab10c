"""Stage timings of one ResCNN VMC iteration (the bench's config-4 leg: J1-J2
10x10, 4 residual blocks, 4,096 samples, 1,024 chains, exchange moves)."""
import sys
import time
sys.path.insert(0, "/root/repo")
import torch

from paper_2601_20782_b200 import rescnn, sampler
from paper_2601_20782_b200.hamiltonians import J1J2Spec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key
from paper_2601_20782_b200.precision import F16

spec = J1J2Spec(LatticeSpec.square(10), 1.0, 0.5, marshall=True)
L, n = 10, 100
params = rescnn.random_parameters(L, 4, derive_key(0, "init"), 0.3)
ens = None
for it in range(4):
    t = [time.perf_counter()]
    ev = rescnn.log_prob_evaluator(params, F16)
    if ens is None:
        ens = sampler.ChainEnsemble(1024, n, sampler.Proposal("exchange", n // 2), ev, derive_key(0, "chains"))
    else:
        ens.set_evaluator(ev, check=False)
        ens.run_sweeps(2, check=False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    ens.reset_counters()
    packed = ens.collect_packed(4096, n + 1)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    uniq, inverse, cnt = torch.unique(packed, dim=0, return_inverse=True, return_counts=True)
    w = cnt.to(torch.float64) / 4096
    torch.cuda.synchronize(); t.append(time.perf_counter())
    eps = rescnn.local_energies_packed(spec, params, uniq).real
    torch.cuda.synchronize(); t.append(time.perf_counter())
    o = rescnn.log_derivatives(params, uniq)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    g, _, energy = rescnn.minsr_dense(o, eps, w, 1e-2, "f32", None, False)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    lp_fmt, _ = ev.log_prob_packed(uniq)
    delta = lp_fmt - 2.0 * rescnn.log_psi_packed(params, uniq)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["snapshot+reburn", "collect", "unique", "energies", "O (autograd)", "minSR f32", "sigma_hat"]
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(" ".join(f"{k} {v:.1f}" for k, v in zip(names, d)), f"total {sum(d):.1f} ms", flush=True)
