"""Throughput of the tcgen05 batched forward (mpv_forward_tc) beside the
CUDA-core f64 forward (mpv_snapshot_forward) on the same configurations.

Workload: the connected configurations of one configs[1] local-energy pass
(65,536 samples x 100 single flips = 6,553,600 configurations of a 10x10
lattice, RBM alpha=2), packed words resident in HBM.  Prints one JSON line."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20782_b200 import rbm  # noqa: E402
from paper_2601_20782_b200.precision import BF16, F16  # noqa: E402
from paper_2601_20782_b200.rng import derive_key  # noqa: E402


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--alpha", type=int, default=2)
    ap.add_argument("--configs", type=int, default=65536 * 100)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--fmt", default="f16")
    ap.add_argument("--no-f64", action="store_true")
    args = ap.parse_args()
    N, B = args.n, args.configs
    fmt = F16 if args.fmt == "f16" else BF16
    params = rbm.random_parameters(N, args.alpha, derive_key(0, "bench-tc"), 0.05)
    M = params.n_hidden
    words = (N + 31) // 32
    g = torch.Generator(device="cuda").manual_seed(1)
    packed = torch.randint(-2**31, 2**31 - 1, (B, words), dtype=torch.int32, device="cuda", generator=g)
    if N % 32:
        packed[:, -1] &= (1 << (N % 32)) - 1
    tc = rbm.TensorCoreForward(params, fmt)
    lp = torch.empty(B, dtype=torch.float64, device="cuda")
    ms = timed(lambda: tc.forward_packed(packed, out_lp=lp), args.reps)
    Kp = (N + 1 + 15) // 16 * 16
    out = {
        "kernel": "forward_tc_kernel", "fmt": fmt.name, "N": N, "M": M, "configs": B,
        "ms": ms, "configs_per_s": B / (ms * 1e-3),
        "tensor_tflops_algorithmic": 2.0 * B * N * 2 * M / (ms * 1e-3) / 1e12,
        "tensor_tflops_issued": 2.0 * B * Kp * 2 * ((M + 15) // 16 * 16) / (ms * 1e-3) / 1e12,
        "hidden_units_per_s": B * M / (ms * 1e-3),
    }
    re, im = torch.empty_like(lp), torch.empty_like(lp)
    ms_ph = timed(lambda: tc.forward_packed(packed, out_lp=lp, out_re=re, out_im=im), args.reps)
    out["ms_with_phase"] = ms_ph
    out["configs_per_s_with_phase"] = B / (ms_ph * 1e-3)
    if not args.no_f64:
        ev = rbm.log_psi_evaluator(params)
        sub = packed[: min(B, 65536 * 10)]
        ms64 = timed(lambda: ev.log_psi_packed(sub), max(1, args.reps // 2))
        out["f64_cuda_core_configs_per_s"] = sub.shape[0] / (ms64 * 1e-3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
