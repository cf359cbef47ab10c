import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_20782_b200 import rescnn, sampler, F16
from paper_2601_20782_b200.hamiltonians import J1J2Spec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key
spec = J1J2Spec(LatticeSpec.square(4), 1.0, 0.5, marshall=True)
p = rescnn.random_parameters(4, 2, derive_key(0, "init"), 0.3)
ev = rescnn.log_prob_evaluator(p, F16)
ens = sampler.ChainEnsemble(512, 16, sampler.Proposal("exchange", 8), ev, derive_key(0, "chains"))
ens.run_sweeps(20)
packed = ens.collect_packed(2048, 17)
uniq, inv, cnt = torch.unique(packed, dim=0, return_inverse=True, return_counts=True)
print("uniq", uniq.shape, "acc", ens.acceptance_rate)
w = cnt.double() / 2048
eps = rescnn.local_energies_packed(spec, p, uniq).real
print("eps", eps.min().item(), eps.max().item(), torch.isfinite(eps).all().item())
o = rescnn.log_derivatives(p, uniq)
print("o", o.shape, o.abs().max().item(), torch.isfinite(o).all().item())
for prec in ("f64", "f32"):
    try:
        g, f, e = rescnn.minsr_dense(o, eps, w, 1e-3, prec)
        print(prec, "ok", g.norm().item(), e)
    except Exception as ex:
        print(prec, "fail", ex)
sw = torch.sqrt(w)
ot = sw[:, None] * (o - (w[:, None] * o).sum(0))
k = ot @ ot.T
print("K diag max", torch.diagonal(k).max().item(), "min eig", torch.linalg.eigvalsh(k)[0].item())
