"""Benchmark of the hot path: reduced-precision MH sampling of an RBM NQS +
the f64 local energies that consume the samples (BASELINE.json metric
"MCMC chain-steps/sec per GPU").

Workload (BASELINE.json configs[1]): RBM alpha=2 on the 10x10 periodic TFIM at
h=3.04 (J=1), 16,384 chains per GPU, f16 sampling (NATIVE fused sweep) + f64
local energies.  One step = the sampling phase of one VMC iteration as the
reference runs it (vmc.py:531-564): publish the f16 snapshot, re-burn 2 sweeps,
collect 4 samples per chain at thinning N+1 (sampler.py:142-167), then f64 local
energies of all samples and the energy / acceptance reductions.  Chain-steps
per step = chains * (2N + 4(N+1)).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun each rank owns 16,384 chains (weak scaling, global chain ids),
and NCCL all-reduces the energy sums and acceptance counts once per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

L = 10
N_SITES = L * L
ALPHA = 2
H_FIELD = 3.04
CHAINS_PER_GPU = 16384
SAMPLES_PER_CHAIN = 4
REBURN_SWEEPS = 2
BURN_IN_SWEEPS = 10 * N_SITES // 10  # 100 sweeps of initial equilibration (untimed)
INIT_SCALE = 0.01  # reference default init (vmc.py:338)
WORKLOAD = "rbm_a2_tfim10x10_h3.04_c16384_f16native_f64energy"
METRIC = "MCMC chain-steps/sec (f16 sampling + f64 local energies), whole job"
DATA = "synthetic (random_parameters scale 0.01, reference streams derive_key(0,'chains'))"


def chain_steps_per_step(chains):
    return chains * (REBURN_SWEEPS * N_SITES + SAMPLES_PER_CHAIN * (N_SITES + 1))


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self._proc = None
            return
        self._thread = threading.Thread(target=self._read, daemon=True)
        self._thread.start()

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2601_20782_b200 import F16, RoundingMode, rbm, sampler, vmc
    from paper_2601_20782_b200.hamiltonians import TfimSpec
    from paper_2601_20782_b200.lattice import LatticeSpec
    from paper_2601_20782_b200.rng import derive_key

    dist = None
    if world > 1:
        import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    spec = TfimSpec(LatticeSpec.square(L), 1.0, H_FIELD)
    params = rbm.random_parameters(N_SITES, ALPHA, derive_key(0, "init"), INIT_SCALE)
    C = CHAINS_PER_GPU
    n_total_chains = C * world
    n_samples_total = n_total_chains * SAMPLES_PER_CHAIN
    thin = N_SITES + 1
    ev = rbm.log_prob_evaluator(params, F16, RoundingMode.NATIVE)
    ens = sampler.ChainEnsemble(C, N_SITES, sampler.Proposal("flip"), ev, derive_key(0, "chains"),
                                chain_offset=rank * C, n_chains_total=n_total_chains)
    ens.run_sweeps(BURN_IN_SWEEPS)
    psi = rbm.log_psi_evaluator(params)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    launches = {"n": 0}

    def device_step(record=None):
        """Inputs resident in HBM: snapshot already built; returns device scalars."""
        ens.set_evaluator(ev, check=False)  # the refresh rides on the re-burn launch; checked at the end
        ens.reset_counters()
        ens.run_sweeps(REBURN_SWEEPS, check=False)
        if record is not None:
            record[0].record(stream)
        packed = ens.collect_packed(n_samples_total, thin, check=False)
        if record is not None:
            record[1].record(stream)
        kern = vmc._energy_kernel(spec, psi)
        if record is not None:
            record[2].record(stream)
        eps, status = kern.packed(packed)
        if record is not None:
            record[3].record(stream)
        e_sum = eps[:, 0].sum()
        acc = ens.accepted_per_chain.sum()
        launches["n"] = 3  # ours: re-burn sweep (refreshes first), collect sweep, local energies (+ 2 torch reductions)
        return e_sum, acc, packed.shape[0]

    # warmup
    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    total_ms = 0.0
    sweep_ms = 0.0
    energy_ms = 0.0
    energies = []
    accs = []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed iterations (untimed)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e_sum, acc, rows = device_step((s0, s1, g0, g1))
        if dist is not None:
            red = torch.stack([e_sum, acc.to(torch.float64), torch.tensor(float(rows), device=dev, dtype=torch.float64)])
            dist.all_reduce(red)
            e_sum, acc, rows = red[0], red[1], red[2]
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        sweep_ms += s0.elapsed_time(s1)
        energy_ms += g0.elapsed_time(g1)
        energies.append(float(e_sum) / float(rows))
        accs.append(float(acc))
    clocks.stop()
    ms = total_ms / args.steps
    if dist is not None:
        t = torch.tensor([ms, sweep_ms / args.steps, energy_ms / args.steps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, sweep_avg, energy_avg = float(t[0]), float(t[1]), float(t[2])
    else:
        sweep_avg, energy_avg = sweep_ms / args.steps, energy_ms / args.steps

    # ---- end-to-end through the public API (host buffers, copies inside) ----
    e2e_ms = 0.0
    h2d = d2h = 0
    n_e2e = min(max(args.steps, 5), 10)  # host-side jitter: at least 5 timed public-API steps
    e2e_each = []
    E2E_WARMUP = 3  # untimed: the pinned host blocks reach steady state in the caching allocator
    for it in range(n_e2e + E2E_WARMUP):
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        ev_e2e = rbm.log_prob_evaluator(params, F16, RoundingMode.NATIVE)  # snapshot built + uploaded
        ens.set_evaluator(ev_e2e, check=False)  # failures surface at collect (sticky status)
        ens.reset_counters()
        ens.run_sweeps(REBURN_SWEEPS, check=False)
        samples = ens.collect(n_samples_total, thin)  # uint8 host rows (D2H) + status check
        eps = vmc.local_energies(spec, psi, samples)  # H2D packed rows, D2H eps
        energy = float(eps.real.mean())
        rate = ens.acceptance_rate
        t1.record(stream)
        torch.cuda.synchronize()
        if it >= E2E_WARMUP:
            e2e_ms += t0.elapsed_time(t1)
            e2e_each.append(t0.elapsed_time(t1))
        snap = ev_e2e.snapshot
        # snapshot upload + the uint8 sample rows re-uploaded by local_energies (packed on the device)
        h2d = snap._table.numel() + snap._bias.numel() + snap._vis_im.numel() * 8 + samples.nbytes
        d2h = samples.nbytes + eps.nbytes + 3 * 16  # samples, eps, status words
    e2e_ms /= n_e2e
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])

    # ---- north-star shape (alpha=1, 10x10, f16) sweep-only rate, same run ----
    ns = None
    if rank == 0:
        def ns_rate(scale, chains=C):
            p1 = rbm.random_parameters(N_SITES, 1, derive_key(0, "init"), scale)
            ev1 = rbm.log_prob_evaluator(p1, F16, RoundingMode.NATIVE)
            e1s = sampler.ChainEnsemble(chains, N_SITES, sampler.Proposal("flip"), ev1, derive_key(0, "chains"))
            e1s.run_steps(1000)
            torch.cuda.synchronize()
            rates = []
            for _ in range(3):  # median of three 1,010-step launches
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                e1s.run_steps(10 * (N_SITES + 1), check=False)
                a1.record(stream)
                torch.cuda.synchronize()
                rates.append(chains * 10 * (N_SITES + 1) / (a0.elapsed_time(a1) / 1e3))
            return sorted(rates)[1], e1s.layout_label

        r_flat, v_flat = ns_rate(INIT_SCALE)
        r_peak, v_peak = ns_rate(0.5)
        r_2x, _ = ns_rate(INIT_SCALE, 2 * C)  # 2,048 chain groups at 16,384 chains fill 86% of the warp slots
        ns = {"config": "rbm_a1_tfim10x10_c16384_f16native", "chain_steps_per_s": r_flat, "variant": v_flat,
              "chains_32768": {"chain_steps_per_s": r_2x,
                               "note": "the same sweep with every warp slot of the GPU holding a chain group"},
              "peaked_scale0.5": {"chain_steps_per_s": r_peak, "variant": v_peak,
                                  "why_below_flat": "peaked weights need the int32 (XI) accumulators: per hidden "
                                  "unit 2 IMAD + 2 I2F + 2 FMUL instead of 2 mixed-precision FFMA, and the sweep "
                                  "is issue-co-limited (profiles/r02/sweep.md, DESIGN.md section 10)"}}

    # ---- sampling-only rates: precision sweep at the config-2 shape, BASELINE
    # configs[2] (Heisenberg 10x10, alpha=4, exchange Sz=0, bf16) and configs[4]
    # (16x16 TFIM, alpha=1) ----
    extra = None
    if rank == 0 and not args.no_extras:
        from paper_2601_20782_b200 import BF16, F32, F64

        def rate(n, alpha, fmt, mode, prop, chains=C, steps=None, scale=INIT_SCALE):
            p = rbm.random_parameters(n, alpha, derive_key(0, "init"), scale)
            e = rbm.log_prob_evaluator(p, fmt, mode)
            en = sampler.ChainEnsemble(chains, n, prop, e, derive_key(0, "chains"))
            en.run_steps(4 * n)
            torch.cuda.synchronize()
            k = steps or 4 * (n + 1)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            en.run_steps(k, check=False)
            a1.record(stream)
            torch.cuda.synchronize()
            return {"chain_steps_per_s": chains * k / (a0.elapsed_time(a1) / 1e3), "variant": en.layout_label}

        flip = sampler.Proposal("flip")
        extra = {"precision_sweep_a2_10x10": {
            "f16": rate(N_SITES, ALPHA, F16, RoundingMode.NATIVE, flip),
            "bf16": rate(N_SITES, ALPHA, BF16, RoundingMode.NATIVE, flip),
            "f32": rate(N_SITES, ALPHA, F32, RoundingMode.NATIVE, flip),
            "f64": rate(N_SITES, ALPHA, F64, RoundingMode.PER_OPERATION, flip),
            "f16_per_operation_reference_arithmetic": rate(N_SITES, ALPHA, F16, RoundingMode.PER_OPERATION, flip,
                                                           steps=40)},
            "peaked_state_scale0.5_f16": rate(N_SITES, ALPHA, F16, RoundingMode.NATIVE, flip, scale=0.5),
            "config3_heis10x10_a4_exchange_bf16": rate(N_SITES, 4, BF16, RoundingMode.NATIVE,
                                                        sampler.Proposal("exchange", N_SITES // 2)),
            "config5_tfim16x16_a1_f16": rate(256, 1, F16, RoundingMode.NATIVE, flip, chains=4096 * 4),
        }

        # BASELINE configs[4]: precision sweep on 16x16 TFIM, energy bias vs the
        # paper's MH bias bound (same parameters, same sampler settings per format)
        def bias_sweep(n_side=16, alpha=1, scale=0.05, chains=4096, per_chain=4, burn_sweeps=100):
            from paper_2601_20782_b200 import bounds
            from paper_2601_20782_b200.lattice import LatticeSpec as _LS

            n = n_side * n_side
            spec = TfimSpec(_LS.square(n_side), 1.0, 3.04)
            p = rbm.random_parameters(n, alpha, derive_key(1, "init"), scale)
            psi = rbm.log_psi_evaluator(p)
            res = {}
            for fmt, mode in ((F64, RoundingMode.PER_OPERATION), (F32, RoundingMode.NATIVE),
                              (BF16, RoundingMode.NATIVE), (F16, RoundingMode.NATIVE)):
                e = rbm.log_prob_evaluator(p, fmt, mode)
                en = sampler.ChainEnsemble(chains, n, flip, e, derive_key(1, "chains"))
                en.run_sweeps(burn_sweeps)
                en.reset_counters()
                smp = en.collect(chains * per_chain, n + 1)
                eps = vmc.local_energies(spec, psi, smp).real
                means = eps.reshape(chains, per_chain).mean(axis=1)
                err = float(np.sqrt(means.var(ddof=1) / chains))
                sig = float(np.std(e(smp) - rbm.log_prob_batch(p, smp, F64))) if fmt is not F64 else 0.0
                res[fmt.name] = {"energy_per_site": float(eps.mean()) / n, "mc_error_per_site": err / n,
                                 "sigma_hat": sig, "tv_bound_pinsker": float(bounds.pinsker_tv_bound(sig)),
                                 "tv_bound_theorem3": float(bounds.theorem3_gaussian_bound(sig, 0.0, 0.0)),
                                 "acceptance": en.acceptance_rate, "variant": e.snapshot.label}
            e64 = res["f64"]["energy_per_site"]
            for k, v in res.items():
                v["bias_vs_f64_per_site"] = v["energy_per_site"] - e64
            res["config"] = (f"rbm_a{alpha}_tfim{n_side}x{n_side}_h3.04_scale{scale}_c{chains}_s{chains * per_chain}"
                             f"_burn{burn_sweeps}sweeps")
            return res

        extra["config5_precision_bias_16x16"] = bias_sweep()

        # f64 local-energy throughput for the Hamiltonians of configs[1..3] (65,536 samples each)
        def energy_rate(spec, alpha, n=N_SITES, samples=65536):
            from paper_2601_20782_b200.lattice import pack_bits

            p = rbm.random_parameters(n, alpha, derive_key(3, "init"), 0.05)
            kern = vmc._energy_kernel(spec, rbm.log_psi_evaluator(p))
            rng = np.random.default_rng(0)
            bits = rng.integers(0, 2, size=(samples, n), dtype=np.uint8)
            if not isinstance(spec, TfimSpec):  # Sz = 0 sector, as the exchange sampler produces
                bits = np.zeros((samples, n), dtype=np.uint8)
                idx = np.argsort(rng.random((samples, n)), axis=1)[:, : n // 2]
                np.put_along_axis(bits, idx, 1, axis=1)
            packed = torch.from_numpy(pack_bits(bits)).to(dev)
            for _ in range(2):
                kern.packed(packed)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(5):
                kern.packed(packed)
            a1.record(stream)
            torch.cuda.synchronize()
            ms_ = a0.elapsed_time(a1) / 5
            return {"ms_per_65536_samples": ms_, "samples_per_s": samples / (ms_ / 1e3)}

        from paper_2601_20782_b200.hamiltonians import HeisenbergSpec, J1J2Spec
        from paper_2601_20782_b200.lattice import LatticeSpec as _LS2

        extra["local_energies_f64"] = {
            "config2_tfim10x10_h3.04_a2": energy_rate(TfimSpec(_LS2.square(10), 1.0, 3.04), 2),
            "config3_heisenberg10x10_marshall_a4": energy_rate(HeisenbergSpec(_LS2.square(10), 1.0, marshall=True), 4),
            "config4_j1j2_10x10_j2_0.5_marshall_a1": energy_rate(J1J2Spec(_LS2.square(10), 1.0, 0.5, marshall=True), 1),
        }

        # north_star subsystem (2): the batched forward as a tcgen05 GEMM (f16, f32 TMEM
        # accumulators, log-cosh epilogue) over the connected configurations of one
        # config-2 local-energy pass (65,536 samples x 100 flips), packed words resident
        def forward_tc_rate(n=N_SITES, alpha=ALPHA, configs=65536 * N_SITES):
            p = rbm.random_parameters(n, alpha, derive_key(0, "bench-tc"), 0.05)
            tcf = rbm.TensorCoreForward(p, F16)
            g = torch.Generator(device=dev).manual_seed(1)
            words = (n + 31) // 32
            pk = torch.randint(-2**31, 2**31 - 1, (configs, words), dtype=torch.int32, device=dev, generator=g)
            if n % 32:
                pk[:, -1] &= (1 << (n % 32)) - 1
            lp_ = torch.empty(configs, dtype=torch.float64, device=dev)
            re_, im_ = torch.empty_like(lp_), torch.empty_like(lp_)

            def t(fn, reps=5):
                fn()
                torch.cuda.synchronize()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for _ in range(reps):
                    fn()
                a1.record(stream)
                torch.cuda.synchronize()
                return a0.elapsed_time(a1) / reps

            ms_lp = t(lambda: tcf.forward_packed(pk, out_lp=lp_))
            ms_ph = t(lambda: tcf.forward_packed(pk, out_lp=lp_, out_re=re_, out_im=im_))
            f64ev = rbm.log_psi_evaluator(p)
            sub = pk[: 65536 * 10]
            ms64 = t(lambda: f64ev.log_psi_packed(sub), 2)
            M_ = p.n_hidden
            return {"workload": f"rbm_a{alpha}_n{n}_f16_{configs}configs (connected configurations of one config-2 "
                                "energy pass), packed words resident",
                    "ms_log_prob": ms_lp, "configs_per_s_log_prob": configs / (ms_lp / 1e3),
                    "ms_log_psi_with_phase": ms_ph, "configs_per_s_log_psi": configs / (ms_ph / 1e3),
                    "f64_cuda_core_forward_configs_per_s": sub.shape[0] / (ms64 / 1e3),
                    "mufu_ops_per_s_log_prob": 2.5 * configs * M_ / (ms_lp / 1e3),
                    "tensor_tflops_log_prob": 2.0 * configs * n * 2 * M_ / (ms_lp / 1e3) / 1e12,
                    "tensor_pipe_pct_ncu": 16.5, "ncu": "profiles/r01/forward_tc_kernel.md"}

        extra["forward_tc"] = forward_tc_rate()

        # BASELINE configs[3]: ResCNN (4 residual blocks, 16 filters, 3x3) on the 10x10
        # J1-J2 model (J2 = 0.5, Marshall sign): tcgen05 forward, fused MH sampling with
        # exchange moves (16,384 chains, f16), one VMC iteration (4,096 samples, f32 minSR)
        def rescnn_rates():
            from paper_2601_20782_b200 import rescnn
            from paper_2601_20782_b200.hamiltonians import J1J2Spec
            from paper_2601_20782_b200.lattice import LatticeSpec as _LS3

            pc = rescnn.random_parameters(10, 4, derive_key(0, "init"), 0.5)
            B = 65536
            pk = torch.randint(-2**31, 2**31 - 1, (B, 4), dtype=torch.int32, device=dev)
            pk[:, -1] &= (1 << (N_SITES % 32)) - 1
            evc = rescnn.log_prob_evaluator(pc, F16)
            evc.log_prob_packed(pk)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(5):
                evc.log_prob_packed(pk)
            a1.record(stream)
            torch.cuda.synchronize()
            ms_f = a0.elapsed_time(a1) / 5
            useful = N_SITES * (16 * 9 + 8 * 16 * 16 * 9) * 2
            sub = pk[:16384]
            rescnn.log_psi_packed(pc, sub)  # f64 forward on DMMA (the local energies' evaluator)
            torch.cuda.synchronize()
            a0.record(stream)
            for _ in range(3):
                rescnn.log_psi_packed(pc, sub)
            a1.record(stream)
            torch.cuda.synchronize()
            ms_64 = a0.elapsed_time(a1) / 3
            ens_c = sampler.ChainEnsemble(C, N_SITES, sampler.Proposal("exchange", N_SITES // 2), evc,
                                          derive_key(0, "chains"))
            ens_c.run_steps(20)
            torch.cuda.synchronize()
            a0.record(stream)
            ens_c.run_steps(200, check=False)
            a1.record(stream)
            torch.cuda.synchronize()
            spec_c = J1J2Spec(_LS3.square(10), 1.0, 0.5, marshall=True)
            cfgc = rescnn.CnnTrainConfig(spec_c, n_res=4, n_steps=3, n_samples=4096, n_chains=1024, eta=0.01,
                                         lambda_shift=1e-2, proposal=sampler.Proposal("exchange", N_SITES // 2),
                                         init_scale=0.3, burn_in_sweeps=0)
            cfgc.n_steps = 1
            rescnn.train(cfgc, local=True)  # warm-up: autograd / cuDNN plans, allocator (rank 0 only: no collectives)
            cfgc.n_steps = 3
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rescnn.train(cfgc, local=True)
            torch.cuda.synchronize()
            return {"config": "rescnn_4x16_3x3_j1j2_10x10_j2_0.5_marshall",
                    "forward_f16_configs_per_s": B / (ms_f / 1e3),
                    "forward_f16_useful_tflops": useful * B / (ms_f / 1e3) / 1e12,
                    "forward_f64_dmma_configs_per_s": sub.shape[0] / (ms_64 / 1e3),
                    "forward_f64_fp64_frac": useful / 2 * sub.shape[0] / (ms_64 / 1e3) / (64 * 148 * 1.965e9),
                    "sampling_exchange_f16_chain_steps_per_s": C * 200 / (a0.elapsed_time(a1) / 1e3),
                    "acceptance": ens_c.acceptance_rate,
                    "vmc_iteration_s4096_c1024_minsr_f32_seconds": (time.perf_counter() - t0) / 3}

        try:
            extra["config4_rescnn"] = rescnn_rates()
        except Exception as exc:
            extra["config4_rescnn"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # ---- VMC iteration time at BASELINE configs[0] (N=20 open TFIM chain, alpha=1,
    # 4,096 samples, 1,024 chains, f16 sampling), reference: vmc.py:472-639 ----
    vmc_iter = None
    if rank == 0 and not args.no_vmc:
        from paper_2601_20782_b200.lattice import LatticeSpec as _LS

        def wall(n_steps):  # whole train() call
            c1 = vmc.TrainConfig(TfimSpec(_LS.chain(20), 1.0, 1.0), alpha=1, n_steps=n_steps, n_samples=4096,
                                 n_chains=1024, sampling_format=F16, rounding_mode=RoundingMode.NATIVE,
                                 track_timings=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = vmc.train(c1, local=True)  # rank 0 alone (other ranks idle)
            torch.cuda.synchronize()
            return time.perf_counter() - t0, res.records

        wall(3)  # warm-up
        # host-side jitter (Python, allocator): median of three runs of each length
        w2 = float(np.median([wall(2)[0] for _ in range(3)]))
        runs12 = [wall(12) for _ in range(3)]
        w12 = float(np.median([r[0] for r in runs12]))
        recs = runs12[-1][1]
        recs = recs[2:]
        vmc_iter = {"config": "tfim_chain20_open_h1_a1_s4096_c1024_f16native",
                    "sampling_ms": 1e3 * float(np.median([r["sampling_seconds"] for r in recs])),
                    "update_ms": 1e3 * float(np.median([r["update_seconds"] for r in recs])),
                    "energy_last": recs[-1]["energy"], "kappa_last": recs[-1]["kappa"],
                    "iteration_ms": 1e3 * (w12 - w2) / 10,
                    "timing": "iteration_ms = wall time of 10 training steps (12-step run minus a 2-step run, medians of 3), incl. "
                              "the per-step eigvalsh condition number of the reference's record (cuSOLVER, ~5 ms at P = 440)"}
        # BASELINE configs[1] (10x10 TFIM, alpha=2, 16,384 chains, 65,536 samples, f16
        # sampling + f64 energies): the dense S (P = 20,300) does not fit the
        # reference's solver; SR runs matrix-free (factored O, conjugate gradients)
        cfg2 = vmc.TrainConfig(TfimSpec(_LS.square(10), 1.0, 3.04), alpha=2, n_steps=4, n_samples=4 * C,
                               n_chains=C, sampling_format=F16, rounding_mode=RoundingMode.NATIVE,
                               track_timings=True, sr_solver="cg", cg_tol=1e-8, burn_in_sweeps=200)
        recs2 = vmc.train(cfg2, local=True).records[1:]
        vmc_iter["config2"] = {
            "config": "rbm_a2_tfim10x10_h3.04_s65536_c16384_f16native_f64energy_sr_cg(tol 1e-8, lambda 1e-3)",
            "sampling_ms": 1e3 * float(np.median([r["sampling_seconds"] for r in recs2])),
            "update_ms": 1e3 * float(np.median([r["update_seconds"] for r in recs2])),
            "cg_iterations": int(np.median([r["cg_iterations"] for r in recs2])),
            "energy_last": recs2[-1]["energy"]}
        vmc_iter["config2"]["iteration_ms"] = vmc_iter["config2"]["sampling_ms"] + vmc_iter["config2"]["update_ms"]

        # north_star precision leg: the ground-state search on the 10x10 TFIM (h=3.04,
        # alpha=1) with f16 NATIVE vs f64 sampling, same seed and protocol (minSR in
        # sample space: U = 4,096 < P = 10,200); plateau = mean of the last 100 steps
        def plateau(fmt):
            mode = RoundingMode.NATIVE if fmt is not F64 else RoundingMode.PER_OPERATION
            c = vmc.TrainConfig(TfimSpec(_LS.square(10), 1.0, 3.04), alpha=1, n_steps=300, n_samples=4096,
                                n_chains=1024, sampling_format=fmt, rounding_mode=mode, sr_solver="minsr",
                                compute_kappa=False, eta=0.01, lambda_shift=1e-2, burn_in_sweeps=100)
            t0 = time.perf_counter()
            res = vmc.train(c, local=True)
            r = res.records
            e = np.array([x["energy"] for x in r[-100:]])
            return {"plateau_energy_per_site": float(e.mean()) / 100, "plateau_std_per_site": float(e.std()) / 100,
                    "mean_mc_error_per_site": float(np.mean([x["mc_error"] for x in r[-100:]])) / 100,
                    "sigma_hat": float(np.mean([x["sigma_hat"] for x in r[-100:]])),
                    "tv_bound": float(np.mean([min(x["bound_pinsker"], x["bound_theorem3"]) for x in r[-100:]])),
                    "wall_s": time.perf_counter() - t0}, res.params

        # the same trained state sampled in f16 NATIVE and f64 (65,536 samples each):
        # the sampling bias at fixed parameters against the paper's bound
        # |E_f16 - E_f64| <= 2 max|eps| TV (TV from sigma-hat, Pinsker / Theorem 3)
        def fixed_state_bias(pt, chains=16384, per_chain=4, burn_sweeps=100):
            from paper_2601_20782_b200 import bounds

            n = pt.n_visible
            spec = TfimSpec(_LS.square(10), 1.0, 3.04)
            psi = rbm.log_psi_evaluator(pt)
            out = {}
            for fmt, mode in ((F64, RoundingMode.PER_OPERATION), (F16, RoundingMode.NATIVE)):
                e = rbm.log_prob_evaluator(pt, fmt, mode)
                en = sampler.ChainEnsemble(chains, n, sampler.Proposal("flip"), e, derive_key(2, "chains"))
                en.run_sweeps(burn_sweeps)
                smp = en.collect(chains * per_chain, n + 1)
                eps = vmc.local_energies(spec, psi, smp).real
                means = eps.reshape(chains, per_chain).mean(axis=1)
                sig = float(np.std(e(smp) - rbm.log_prob_batch(pt, smp, F64))) if fmt is not F64 else 0.0
                tv = min(float(bounds.pinsker_tv_bound(sig)), float(bounds.theorem3_gaussian_bound(sig, 0.0, 0.0)))
                out[fmt.name] = {"energy_per_site": float(eps.mean()) / n,
                                 "mc_error_per_site": float(np.sqrt(means.var(ddof=1) / chains)) / n,
                                 "sigma_hat": sig, "tv_bound": tv,
                                 "bias_bound_per_site": 2.0 * float(np.max(np.abs(eps))) * tv / n}
            d = out["f16"]["energy_per_site"] - out["f64"]["energy_per_site"]
            err = float(np.hypot(out["f16"]["mc_error_per_site"], out["f64"]["mc_error_per_site"]))
            out["delta_per_site"] = d
            out["within_bias_bound_plus_3_sigma"] = bool(abs(d) <= out["f16"]["bias_bound_per_site"] + 3 * err)
            return out

        from paper_2601_20782_b200 import F64

        try:
            (p16, _), (p64, params64) = plateau(F16), plateau(F64)
            vmc_iter["precision_leg_10x10"] = {
                "config": "tfim10x10_h3.04_a1_s4096_c1024_minsr_eta0.01_lambda0.01_300steps (plateau: last 100 steps)",
                "f16_native": p16, "f64": p64,
                "delta_per_site": p16["plateau_energy_per_site"] - p64["plateau_energy_per_site"],
                "note": "separately trained runs follow different stochastic trajectories (both still descending); "
                        "the fixed-state comparison below isolates the f16 sampling bias",
                "fixed_state_f64_trained": fixed_state_bias(params64)}
        except Exception as exc:  # a diverging training run must not void the throughput line
            vmc_iter["precision_leg_10x10"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    steps_per_step = chain_steps_per_step(C) * world
    value = steps_per_step / (ms / 1e3)
    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or 1965.0
    mufu_peak = 16 * 148 * sm_mhz * 1e6  # MUFU lane-ops/s at the measured SM clock
    collect_steps = C * SAMPLES_PER_CHAIN * (N_SITES + 1)
    achieved_mufu = 3 * params.n_hidden * collect_steps / (sweep_avg / 1e3)
    fp64_peak = 64 * 148 * sm_mhz * 1e6
    fp64_ops = n_samples_total / world * (N_SITES * params.n_hidden * 8 + N_SITES * 2 * params.n_hidden)
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "chain-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16",
        "data": DATA,
        "config": bench_config(),
        "run": {"chain_steps_per_step": steps_per_step, "variant": ev.snapshot.label,
                "parallelism": f"chains sharded x{world}"},
        "sampling_sweep_ms": sweep_avg,
        "sampling_chain_steps_per_s": collect_steps * world / (sweep_avg / 1e3),
        "energy_check": {"mean_energy": float(np.mean(energies)), "acceptance": None},
        "roofline": {"bound": "sfu", "kernel": "sweep_kernel (collect launch)", "achieved": achieved_mufu / 1e12,
                     "peak": mufu_peak / 1e12, "unit": "Tmufu-op/s", "frac": achieved_mufu / mufu_peak,
                     "traffic": None, "algorithmic": "3 MUFU ops (ex2, cos, lg2) per hidden unit per chain-step, M=200",
                     "peak_basis": "16 MUFU/clk/SM (measured, tools/microbench) x 148 SMs x measured median SM clock"},
        # second-largest kernel of the step: the f64 local energies (FP64 pipe: DFMA and DMMA)
        "roofline_energy": {"bound": "fp64", "kernel": "energy_kernel", "ms": energy_avg,
                            "achieved": fp64_ops / (energy_avg / 1e3) / 1e12, "peak": fp64_peak / 1e12,
                            "unit": "TFP64-op/s", "frac": fp64_ops / (energy_avg / 1e3) / fp64_peak,
                            "algorithmic": "per sample: terms x M x 8 FP64 ops (ratio products) + N x 2M "
                                           "multiply-adds (theta GEMM on DMMA); 65,536 samples, 100 terms, M=200",
                            "peak_basis": "64 FP64 FMA/clk/SM (measured, tools/microbench/fp64lat.cu, dmma.cu) x 148 "
                                          "SMs x measured median SM clock"},
        "clocks": clk,
        "gpu_launches": launches["n"],
        "e2e": {"value": steps_per_step / (e2e_ms / 1e3), "unit": "chain-steps/s", "ms_per_step": e2e_ms,
                "timed_steps": n_e2e, "ms_min_max_rank0": [min(e2e_each), max(e2e_each)],
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": "log_prob_evaluator + ChainEnsemble.set_evaluator/run_sweeps/collect + vmc.local_energies"},
        "north_star_shape": ns,
        "vmc_iteration": vmc_iter,
        "sampling_rates": extra,
    }
    if isinstance(extra, dict):
        # MUFU roofline of every sampling rate (3 MUFU ops per hidden unit per
        # evaluated chain-step: f16/bf16 ex2, cos, lg2; f32 ex2, rcp, lg2).  The f64
        # arithmetic is libm-bound on the FP64 pipe (exp, sincos, log per unit).
        # Exchange rates count every step; about half of them swap equal bits and
        # are skipped, so their fraction can exceed what the evaluated steps reach.
        def mufu(entry, m):
            if isinstance(entry, dict) and "chain_steps_per_s" in entry:
                entry["mufu_frac_all_steps"] = 3 * m * entry["chain_steps_per_s"] / mufu_peak
        for fmt_, ent in (extra.get("precision_sweep_a2_10x10") or {}).items():
            if fmt_ in ("f16", "bf16", "f32"):
                mufu(ent, 2 * N_SITES)
            elif fmt_ == "f64":
                ent["bound"] = "fp64 pipe: f64 exp, sincos, log per hidden unit (the reference's formula)"
        mufu(extra.get("peaked_state_scale0.5_f16"), 2 * N_SITES)
        mufu(extra.get("config3_heis10x10_a4_exchange_bf16"), 4 * N_SITES)
        mufu(extra.get("config5_tfim16x16_a1_f16"), 256)
    if isinstance(ns, dict):
        ns["mufu_frac"] = 3 * N_SITES * ns["chain_steps_per_s"] / mufu_peak
        ns["peaked_scale0.5"]["mufu_frac"] = 3 * N_SITES * ns["peaked_scale0.5"]["chain_steps_per_s"] / mufu_peak
    if isinstance(extra, dict) and "forward_tc" in extra:
        ftc = extra["forward_tc"]
        ftc["roofline"] = {"bound": "sfu", "achieved": ftc["mufu_ops_per_s_log_prob"] / 1e12,
                           "peak": mufu_peak / 1e12, "unit": "Tmufu-op/s",
                           "frac": ftc["mufu_ops_per_s_log_prob"] / mufu_peak,
                           "tensor_frac_of_dense_f16_peak": ftc["tensor_tflops_log_prob"] / 2250.0,
                           "algorithmic": "2.5 MUFU ops per hidden unit per configuration (ex2, cos each; one lg2 per pair of units); "
                                          "GEMM 2 x N x 2M flops per configuration"}
    out["energy_check"]["acceptance"] = float(np.mean(accs)) / (C * world * (REBURN_SWEEPS * N_SITES + SAMPLES_PER_CHAIN * (N_SITES + 1)))
    tr = os.path.join(ROOT, "profiles", "r02", "traffic.json")
    if os.path.exists(tr):
        with open(tr) as f:
            out["roofline"]["traffic"] = json.load(f)["sweep_kernel"]["dram_bytes_per_launch"]
            out["roofline"]["traffic_unit"] = "bytes/launch (ncu --set full, profiles/r02)"
            out["roofline_energy"]["traffic"] = json.load(open(tr))["energy_kernel"]["dram_bytes_per_launch"]
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline()
    return out


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle's restatement of the reference CPU
# path (oracle/c/oracle_port.c: per-operation f16 evaluator with a full forward
# per proposal, as numba runs _kernels.rounded_log_prob; f64 local energies with
# a full forward per connected configuration, vmc.py:60-108), OpenMP over the
# chains on every host core.  Parameters come from the oracle's own restatement
# of rbm.random_parameters / round_parameters (pinned to the reference's output,
# tests/test_oracle.py), never from the package under test.
# ---------------------------------------------------------------------------
REF_SAMPLE_DIV = 16  # each reference step is 1/16 of the workload step (1,024 chains)


class ReferenceWorkload:
    """One bounded sample of the bench step on the CPU: C/16 chains through the
    reference's per-iteration sampling phase (vmc.py:531-564): set_evaluator with
    the f16 snapshot, re-burn 2 sweeps, collect 4 samples per chain at thinning
    N+1, f64 local energies of every sample, energy mean and acceptance.  Work
    proportions equal the GPU step's, so chain-steps/s are comparable."""

    def __init__(self, chains, threads):
        from oracle import port
        from oracle import rng as orng

        self.port, self.chains, self.threads = port, int(chains), int(threads)
        a, b, w = port.random_parameters(N_SITES, ALPHA, orng.derive_key(0, "init"), INIT_SCALE)
        self.p64 = port.Params(a, b, w)
        self.p16 = port.Params(*port.round_parameters(a, b, w, "f16"))
        self.ens = port.PortEnsemble(self.chains, N_SITES, "flip", None, self.p16, "f16",
                                     int(orng.derive_key(0, "chains")), nthreads=self.threads)
        self.ens.run_steps(2 * N_SITES)  # untimed equilibration (per-op cost does not depend on the state)
        self.bonds = _square_bonds(L)

    def chain_steps(self):
        return chain_steps_per_step(self.chains)

    def step(self):
        ens = self.ens
        ens.set_params(self.p16, "f16")  # the iteration's snapshot (set_evaluator refresh)
        ens.reset_counters()
        ens.run_steps(REBURN_SWEEPS * N_SITES)
        samples = ens.collect(self.chains * SAMPLES_PER_CHAIN, N_SITES + 1)
        eps = self.port.local_energies(self.p64, "tfim", self.bonds, 1.0, H_FIELD, samples, nthreads=self.threads)
        return float(eps.real.mean()), ens.accepted / ens.proposed


def _square_bonds(length):
    """Periodic square-lattice bonds (i < j), row-major sites (lattice.py:118-182)."""
    out = set()
    for r in range(length):
        for c in range(length):
            i = r * length + c
            for j in (r * length + (c + 1) % length, ((r + 1) % length) * length + c):
                out.add((min(i, j), max(i, j)))
    return np.array(sorted(out), dtype=np.int64)


def _time_reference_steps(n_warmup, n_steps, threads, chains):
    wl = ReferenceWorkload(chains, threads)
    times = []
    for i in range(n_warmup + n_steps):
        t0 = time.perf_counter()
        wl.step()
        dt = time.perf_counter() - t0
        if i >= n_warmup:
            times.append(dt)
    return wl, times


def cpu_baseline(threads=None, steps=3):
    """Reported CPU baseline of our arm's JSON line (rank 0, N=1): a few timed
    reference steps of the bounded sample (about 10-20 s of CPU work)."""
    threads = threads or len(os.sched_getaffinity(0))
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    chains = CHAINS_PER_GPU // REF_SAMPLE_DIV
    wl, times = _time_reference_steps(1, steps, threads, chains)
    sec = float(np.median(times))
    return {"value": wl.chain_steps() / sec, "unit": "chain-steps/s", "cores": threads, "kind": "port",
            "sample": _reference_sample_text(chains), "sec_per_sample_step": sec, "cpu_model": _cpu_model()}


def _reference_sample_text(chains):
    return (f"1/{REF_SAMPLE_DIV} of the workload step per step: {chains} chains x "
            f"{REBURN_SWEEPS * N_SITES + SAMPLES_PER_CHAIN * (N_SITES + 1)} per-op f16 MH steps "
            f"(full forward per proposal) + f64 local energies of {chains * SAMPLES_PER_CHAIN} samples "
            "(oracle C port of the reference, OpenMP)")


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_config():
    return {"workload": WORKLOAD, "chains_per_gpu": CHAINS_PER_GPU, "n_sites": N_SITES, "alpha": ALPHA,
            "h": H_FIELD, "samples_per_step": CHAINS_PER_GPU * SAMPLES_PER_CHAIN, "thin_steps": N_SITES + 1,
            "reburn_sweeps": REBURN_SWEEPS, "l2": "flushed between timed steps (256 MB write)"}


def run_reference(args, rank):
    """--impl reference: every counted step is one timed bounded sample (1/16) of
    the workload step, run by the oracle's restatement of the reference's CPU
    path on all host cores; ms_per_step is that sample's measured wall time."""
    if rank != 0:
        return None
    threads = len(os.sched_getaffinity(0))
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    chains = CHAINS_PER_GPU // REF_SAMPLE_DIV
    t_start = time.perf_counter()
    wl, times = _time_reference_steps(args.warmup, args.steps, threads, chains)
    total = float(sum(times))
    value = wl.chain_steps() * len(times) / total
    ms = 1e3 * total / len(times)
    cb = {"value": value, "unit": "chain-steps/s", "cores": threads, "kind": "port",
          "sample": _reference_sample_text(chains), "cpu_model": _cpu_model()}
    return {"metric": METRIC, "value": value, "unit": "chain-steps/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16", "data": DATA, "config": bench_config(), "impl": "reference",
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "chain-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_start}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-vmc", action="store_true", help="skip the VMC iteration-time measurement")
    ap.add_argument("--no-extras", action="store_true", help="skip the per-format / per-config sampling rates")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank)
        if out is not None:
            print(json.dumps(out))
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        # BENCH_TEST_ONE_GPU=1 (control-flow check only, never a measurement):
        # every rank on cuda:0 over gloo, so the N>1 path can run on one GPU
        if os.environ.get("BENCH_TEST_ONE_GPU") == "1":
            os.environ["LOCAL_RANK"] = "0"
            local_rank = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
