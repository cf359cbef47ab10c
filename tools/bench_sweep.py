"""Time the fused sweep alone for one configuration (for ncu captures).

    python tools/bench_sweep.py N ALPHA FMT SCALE [PROPOSAL] [CHAINS]
"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import F16, BF16, F32, F64, RoundingMode, rbm, sampler
from paper_2601_20782_b200.rng import derive_key

n, alpha, fmt, scale = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], float(sys.argv[4])
prop = sys.argv[5] if len(sys.argv) > 5 else "flip"
chains = int(sys.argv[6]) if len(sys.argv) > 6 else 16384
F = {"f16": F16, "bf16": BF16, "f32": F32, "f64": F64}[fmt]
p = rbm.random_parameters(n, alpha, derive_key(0, "init"), scale)
ev = rbm.log_prob_evaluator(p, F, RoundingMode.NATIVE if fmt != "f64" else RoundingMode.PER_OPERATION)
ens = sampler.ChainEnsemble(chains, n, sampler.Proposal(prop, n // 2 if prop == "exchange" else None), ev,
                            derive_key(0, "chains"))
ens.run_steps(4 * n)
torch.cuda.synchronize()
k = 4 * (n + 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ens.run_steps(k, check=False)
e1.record()
torch.cuda.synchronize()
print(f"{ev.snapshot.label}: {chains * k / (e0.elapsed_time(e1) / 1e3):.4e} chain-steps/s, acc {ens.acceptance_rate:.3f}")
