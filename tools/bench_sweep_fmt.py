"""Sampling rate per format at the config-2 shape (10x10 TFIM, alpha=2, 16,384 chains)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import BF16, F16, F32, F64, RoundingMode, rbm, sampler
from paper_2601_20782_b200.rng import derive_key
p = rbm.random_parameters(100, 2, derive_key(0, "init"), 0.01)
for fmt, mode in ((F16, RoundingMode.NATIVE), (BF16, RoundingMode.NATIVE), (F32, RoundingMode.NATIVE), (F64, RoundingMode.PER_OPERATION)):
    ev = rbm.log_prob_evaluator(p, fmt, mode)
    en = sampler.ChainEnsemble(16384, 100, sampler.Proposal("flip"), ev, derive_key(0, "chains"))
    en.run_steps(400)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); en.run_steps(404, check=False); b.record(); torch.cuda.synchronize()
    print(f"{fmt.name:5s} {ev.snapshot.label:28s} {16384 * 404 / (a.elapsed_time(b) / 1e3):.3e} chain-steps/s")
