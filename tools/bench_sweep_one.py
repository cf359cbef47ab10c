"""One format's collect-style sweep at the config-2 shape (for ncu captures):
python tools/bench_sweep_one.py FMT [N ALPHA SCALE PROPOSAL CHAINS]"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import BF16, F16, F32, F64, RoundingMode, rbm, sampler
from paper_2601_20782_b200.rng import derive_key
fmts = {"f16": F16, "bf16": BF16, "f32": F32, "f64": F64}
fmt = fmts[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
alpha = int(sys.argv[3]) if len(sys.argv) > 3 else 2
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 0.01
kind = sys.argv[5] if len(sys.argv) > 5 else "flip"
chains = int(sys.argv[6]) if len(sys.argv) > 6 else 16384
mode = RoundingMode.PER_OPERATION if fmt is F64 else RoundingMode.NATIVE
p = rbm.random_parameters(n, alpha, derive_key(0, "init"), scale)
ev = rbm.log_prob_evaluator(p, fmt, mode)
prop = sampler.Proposal(kind, n // 2 if kind == "exchange" else None)
en = sampler.ChainEnsemble(chains, n, prop, ev, derive_key(0, "chains"))
en.run_steps(4 * n)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); en.run_steps(4 * (n + 1), check=False); b.record(); torch.cuda.synchronize()
print(f"{fmt.name} {en.layout_label} {chains * 4 * (n + 1) / (a.elapsed_time(b) / 1e3):.3e} chain-steps/s")
