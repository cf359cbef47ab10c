"""Flip-sweep rate of the fused kernel under forced lane layouts (experiments):
python tools/bench_layouts.py"""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2601_20782_b200 import F16, RoundingMode, _native as nat, rbm, sampler
from paper_2601_20782_b200.rng import derive_key

for alpha in (1, 2):
    p = rbm.random_parameters(100, alpha, derive_key(0, "init"), 0.01)
    for ml in (1, 8, 16, 32):
        ev = rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
        snap = ev.snapshot
        c, G, U = nat.plan_cluster(100, p.n_hidden, F16.code, RoundingMode.NATIVE.code, snap.variant, ml)
        other = object.__new__(rbm.DeviceSnapshot)
        other.__dict__.update({k: v for k, v in snap.__dict__.items() if k != "_layouts"})
        other._layouts = {}
        other._fill(snap.variant, c, G, U, c * G * U)
        ev.snapshot = other
        en = sampler.ChainEnsemble(16384, 100, sampler.Proposal("flip"), ev, derive_key(0, "chains"))
        en.run_steps(1000)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 0
        for _ in range(3):
            a.record(); en.run_steps(1010, check=False); b.record(); torch.cuda.synchronize()
            best = max(best, 16384 * 1010 / (a.elapsed_time(b) / 1e3))
        print(f"alpha={alpha} min_lanes={ml} {other.label}: {best:.4e}", flush=True)
