import numpy as np, sys
sys.path.insert(0, "/root/repo")
from paper_2601_20782_b200 import rbm, sampler, F64, RoundingMode
from paper_2601_20782_b200.rng import derive_key
from paper_2601_20782_b200.errors import EvaluationFailureError
p = rbm.RbmParameters(np.array([1e308, 1e308, 0], complex), np.zeros(2, complex), np.zeros((2, 3), complex))
ev = rbm.log_prob_evaluator(p, F64)
try:
    ens = sampler.ChainEnsemble(8, 3, sampler.Proposal("flip"), ev, derive_key(0, "chains"))
    print("init ok", ens.bits, ens.log_probs)
    ens.run_steps(50)
except EvaluationFailureError as e:
    print("err", e, e.context)
