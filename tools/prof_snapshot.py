"""Host-side cost of building a device snapshot (the e2e step's first call)."""
import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import rbm
from paper_2601_20782_b200.precision import F16, RoundingMode
from paper_2601_20782_b200.rng import derive_key
p = rbm.random_parameters(100, 2, derive_key(0, "init"), 0.01)
for _ in range(5):
    rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50):
    rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
torch.cuda.synchronize()
print("per snapshot %.3f ms" % ((time.perf_counter() - t) / 50 * 1e3))
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
