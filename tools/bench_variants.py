"""Sampling rate of each exact-accumulator variant the planner allows, for a
few shapes (flat and peaked states): python tools/bench_variants.py"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import BF16, F16, RoundingMode, _native, rbm, sampler
from paper_2601_20782_b200.rng import derive_key

NAMES = {_native.ACC_X1: "X1", _native.ACC_X2: "X2", _native.ACC_XI: "XI", _native.ACC_F64: "F64"}
for n, alpha, scale, fmt, kind in ((100, 1, 0.5, F16, "flip"), (100, 2, 0.5, F16, "flip"), (100, 1, 0.01, F16, "flip"),
                                   (100, 2, 0.01, BF16, "flip"), (100, 4, 0.01, BF16, "exchange"),
                                   (256, 1, 0.01, F16, "flip")):
    p = rbm.random_parameters(n, alpha, derive_key(0, "init"), scale)
    for var in (_native.ACC_X1, _native.ACC_XI, _native.ACC_X2, _native.ACC_F64):
        try:
            ev = rbm.log_prob_evaluator(p, fmt, RoundingMode.NATIVE, variant=var)
        except ValueError:
            continue
        prop = sampler.Proposal(kind, n // 2 if kind == "exchange" else None)
        en = sampler.ChainEnsemble(16384, n, prop, ev, derive_key(0, "chains"))
        en.run_steps(2 * n)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        en.run_steps(4 * (n + 1), check=False)
        b.record()
        torch.cuda.synchronize()
        print(f"N={n} a={alpha} s={scale} {fmt.name} {kind:8s} {NAMES[var]:3s} {ev.snapshot.label:26s} "
              f"{16384 * 4 * (n + 1) / (a.elapsed_time(b) / 1e3):.3e}", flush=True)
