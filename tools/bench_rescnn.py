"""ResCNN (configs[3]) rates on one B200: tensor-core forward, fused MH sampling
(10x10 J1-J2, exchange moves), and one VMC iteration (f32 minSR)."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

from paper_2601_20782_b200 import BF16, F16, rescnn, sampler
from paper_2601_20782_b200.hamiltonians import J1J2Spec
from paper_2601_20782_b200.lattice import LatticeSpec
from paper_2601_20782_b200.rng import derive_key


def tm(f, reps=5):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    L, n = 10, 100
    p = rescnn.random_parameters(L, 4, derive_key(0, "init"), 0.5)
    out = {}
    B = 65536
    pk = torch.randint(-2**31, 2**31 - 1, (B, 4), dtype=torch.int32, device="cuda")
    pk[:, -1] &= (1 << (n % 32)) - 1
    for fmt in (F16, BF16):
        ev = rescnn.log_prob_evaluator(p, fmt)
        ms = tm(lambda: ev.log_prob_packed(pk))
        useful = n * (16 * 9 + 8 * 16 * 16 * 9) * 2  # flops per configuration
        issued = 144 * 9 * (16 * 16 * 9) * 2 * (2048 / (14 * 144))  # tensor flops issued per configuration
        out[f"forward_{fmt.name}"] = {"configs": B, "ms": ms, "configs_per_s": B / (ms / 1e3),
                                      "useful_tflops": useful * B / (ms / 1e3) / 1e12,
                                      "issued_tensor_tflops": issued * B / (ms / 1e3) / 1e12}
    ev64 = rescnn.log_prob_evaluator(p, rescnn.FloatFormat_f64())
    ms = tm(lambda: ev64.log_prob_packed(pk[:8192]), 2)
    out["forward_f64_dmma"] = {"configs_per_s": 8192 / (ms / 1e3)}
    ev = rescnn.log_prob_evaluator(p, F16)
    C = 16384
    ens = sampler.ChainEnsemble(C, n, sampler.Proposal("exchange", n // 2), ev, derive_key(0, "chains"))
    ens.run_steps(20)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ens.run_steps(200, check=False)
    b.record()
    torch.cuda.synchronize()
    out["mh_j1j2_10x10_exchange_f16"] = {"chains": C, "chain_steps_per_s": C * 200 / (a.elapsed_time(b) / 1e3),
                                         "acceptance": ens.acceptance_rate}
    spec = J1J2Spec(LatticeSpec.square(10), 1.0, 0.5, marshall=True)
    cfg = rescnn.CnnTrainConfig(spec, n_res=4, n_steps=4, n_samples=4096, n_chains=1024, eta=0.01, lambda_shift=1e-2,
                                proposal=sampler.Proposal("exchange", n // 2), init_scale=0.3, burn_in_sweeps=20)
    t0 = time.perf_counter()
    recs, _ = rescnn.train(cfg)
    torch.cuda.synchronize()
    out["vmc_iteration_j1j2_10x10_s4096"] = {"seconds_per_iteration_incl_burn_in": (time.perf_counter() - t0) / 4,
                                             "energy_last": recs[-1]["energy"], "sigma_hat": recs[-1]["sigma_hat"]}
    t0 = time.perf_counter()
    cfg.n_steps, cfg.burn_in_sweeps = 3, 0
    rescnn.train(cfg)
    torch.cuda.synchronize()
    out["vmc_iteration_j1j2_10x10_s4096"]["seconds_per_iteration"] = (time.perf_counter() - t0) / 3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
