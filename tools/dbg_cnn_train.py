import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, time
from paper_2601_20782_b200 import rescnn, sampler, F16
from paper_2601_20782_b200.hamiltonians import J1J2Spec, TfimSpec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key
for spec in (TfimSpec(LatticeSpec.square(4), 1.0, 3.04), J1J2Spec(LatticeSpec.square(4), 1.0, 0.5, marshall=True)):
    prop = sampler.Proposal("flip") if isinstance(spec, TfimSpec) else sampler.Proposal("exchange", 8)
    p = rescnn.random_parameters(4, 2, derive_key(0, "init"), 0.3)
    ens = None
    for step in range(60):
        ev = rescnn.log_prob_evaluator(p, F16)
        if ens is None:
            ens = sampler.ChainEnsemble(512, 16, prop, ev, derive_key(0, "chains")); ens.run_sweeps(20)
        else:
            ens.set_evaluator(ev); ens.run_sweeps(2)
        packed = ens.collect_packed(2048, 17)
        uniq, inv, cnt = torch.unique(packed, dim=0, return_inverse=True, return_counts=True)
        w = cnt.double() / 2048
        eps = rescnn.local_energies_packed(spec, p, uniq).real
        o = rescnn.log_derivatives(p, uniq)
        g, f, e = rescnn.minsr_dense(o, eps, w, 1e-2, "f64")
        if step % 5 == 0 or not torch.isfinite(g).all():
            print(type(spec).__name__, step, "E", round(e, 4), "|g|", g.norm().item(), "|F|", f.norm().item(), "|O|max", o.abs().max().item(),
                  "theta max", np.abs(p.theta).max(), "acc", round(ens.acceptance_rate, 3), flush=True)
        p = rescnn.ResCnnParameters(p.theta - 0.01 * g.cpu().numpy(), 4, 2)
