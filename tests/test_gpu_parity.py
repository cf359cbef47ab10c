"""Parity of the sm_100a path with the reference, on a B200.

Golden vectors come from the reference itself (tests/golden/make_golden.py);
larger cases use the CPU oracle (oracle/), which tests/test_oracle.py pins to
the same golden vectors.  Tolerances:
  * RNG, per-operation forward/sampling, sample layouts: bit-exact;
  * f64 forward / local energies: 1e-12 relative (reference sums through BLAS);
  * NATIVE f32 log p: 1e-5 * max(1, |log p|) vs f64 (north_star tolerance, SURVEY §0.9 floor);
  * NATIVE f16/bf16: statistical (see test_gpu_statistics.py).
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import port
from paper_2601_20782_b200 import BF16, F16, F32, F64, RoundingMode, _native, rbm, sampler
from paper_2601_20782_b200.lattice import pack_bits
from paper_2601_20782_b200.precision import FORMATS
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu
PER_OP = RoundingMode.PER_OPERATION
NATIVE = RoundingMode.NATIVE


def params_of(g, prefix=""):
    return rbm.RbmParameters(g[f"{prefix}a"], g[f"{prefix}b"], g[f"{prefix}w"])


def test_device_streams_match_streamset(cuda, g_rng):
    out = torch.empty((50, 37), dtype=torch.float64, device=cuda)
    _native.call("mpv_stream_uniforms", int(g_rng["stream_key"]), 37, 0, 0, 50, out.data_ptr(),
                 _native.stream_handle())
    assert np.array_equal(out.cpu().numpy(), g_rng["stream_draws"])
    # far chains / far draws against the oracle restatement
    out = torch.empty((16, 1000), dtype=torch.float64, device=cuda)
    _native.call("mpv_stream_uniforms", int(g_rng["stream_key"]), 1000, 123456, 10**6, 16, out.data_ptr(),
                 _native.stream_handle())
    assert np.array_equal(out.cpu().numpy(), port.stream_uniforms(int(g_rng["stream_key"]), 1000, 16, 123456, 10**6))


@pytest.mark.parametrize("fmt", ["f32", "f16", "bf16"])
def test_per_op_forward_bitwise(cuda, g_forward, fmt):
    mismatches = 0
    for ci in range(int(g_forward["n_cases"])):
        p = params_of(g_forward, f"c{ci}_")
        bits = g_forward[f"c{ci}_bits"]
        lp = rbm.log_prob_batch(p, bits, FORMATS[fmt], PER_OP)
        psi = rbm.log_psi_batch(p, bits, FORMATS[fmt], PER_OP)
        ref_lp, ref_psi = g_forward[f"c{ci}_{fmt}_lp"], g_forward[f"c{ci}_{fmt}_psi"]
        mismatches += int(np.sum(lp != ref_lp))
        assert np.array_equal(psi.real, ref_psi.real) or fmt == "f32"
        # f32 only: a CUDA-vs-glibc f64 libm ulp can land on an f32 rounding boundary
        assert np.max(np.abs(lp - ref_lp) / np.maximum(1, np.abs(ref_lp))) <= (2e-7 if fmt == "f32" else 0.0)
        assert np.max(np.abs(psi.imag - ref_psi.imag) / np.maximum(1, np.abs(ref_psi.imag))) <= (
            2e-7 if fmt == "f32" else 0.0)
    if fmt != "f32":
        assert mismatches == 0
    else:
        assert mismatches <= 2, mismatches


def test_rounded_log_prob_drop_in(cuda, g_forward):
    """mpv_rounded_log_prob has the numba kernel's argument list (_kernels.py:95-129)."""
    lib = _native.load()
    for fmt in ("f16", "bf16", "f32"):
        ci = 0
        snap = rbm.RbmParameters(g_forward[f"c{ci}_{fmt}_snap_a"], g_forward[f"c{ci}_{fmt}_snap_b"],
                                 g_forward[f"c{ci}_{fmt}_snap_w"])
        bits = torch.from_numpy(np.ascontiguousarray(g_forward[f"c{ci}_bits"])).to(cuda)
        B, N = bits.shape
        M = snap.n_hidden
        dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(cuda)  # noqa: E731
        a_re, b_re, b_im, w_re, w_im = (dev(v) for v in (snap.a.real, snap.b.real, snap.b.imag, snap.w.real,
                                                          snap.w.imag))
        out = torch.empty(B, dtype=torch.float64, device=cuda)
        scratch = torch.empty(lib.mpv_rounded_scratch_bytes(B, N, M, FORMATS[fmt].code), dtype=torch.uint8,
                              device=cuda)
        _native.call("mpv_rounded_log_prob", bits.data_ptr(), B, N, M, a_re.data_ptr(), b_re.data_ptr(),
                     b_im.data_ptr(), w_re.data_ptr(), w_im.data_ptr(), FORMATS[fmt].code, out.data_ptr(),
                     scratch.data_ptr(), _native.stream_handle())
        got = out.cpu().numpy()
        ref = g_forward[f"c{ci}_{fmt}_lp"]
        if fmt == "f32":
            assert np.max(np.abs(got - ref) / np.maximum(1, np.abs(ref))) <= 2e-7
        else:
            assert np.array_equal(got, ref)


def test_f64_and_storage_forward(cuda, g_forward):
    for ci in range(int(g_forward["n_cases"])):
        p = params_of(g_forward, f"c{ci}_")
        bits = g_forward[f"c{ci}_bits"]
        psi = rbm.log_psi_batch(p, bits, F64)
        ref = g_forward[f"c{ci}_f64_psi"]
        assert np.max(np.abs(psi - ref) / np.maximum(1, np.abs(ref))) < 1e-12
        lp = rbm.log_prob_batch(p, bits, F64)
        assert np.max(np.abs(lp - g_forward[f"c{ci}_f64_lp"]) / np.maximum(1, np.abs(lp))) < 1e-12
        for fmt in ("bf16", "f16"):
            st = rbm.log_prob_batch(p, bits, FORMATS[fmt], RoundingMode.STORAGE_ONLY)
            want = g_forward[f"c{ci}_{fmt}_storage_lp"]
            assert np.max(np.abs(st - want) / np.maximum(1, np.abs(want))) < 1e-12


def test_native_f32_within_tolerance_of_f64(cuda, g_forward):
    for ci in range(int(g_forward["n_cases"])):
        p = params_of(g_forward, f"c{ci}_")
        bits = g_forward[f"c{ci}_bits"]
        lp = rbm.log_prob_batch(p, bits, F32, NATIVE)
        ref = g_forward[f"c{ci}_f64_lp"]
        # the native f32 arithmetic vs f64 on the f32 snapshot: 1e-5 relative with a floor of 1
        assert np.max(np.abs(lp - ref) / np.maximum(1, np.abs(ref))) < 1e-5


@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_native_matches_arithmetic_model(cuda, g_forward, fmt):
    """NATIVE log p == the numpy model of its arithmetic (oracle/model.py): theta
    exact, one rounding to fmt, per-unit log cosh rounded to fmt, f32 sums; the
    tolerance covers the MUFU approximation flipping a unit's last fmt bit."""
    from oracle import model

    for ci in range(int(g_forward["n_cases"])):
        p = params_of(g_forward, f"c{ci}_")
        snap = rbm.round_parameters(p, FORMATS[fmt])
        bits = g_forward[f"c{ci}_bits"]
        lp = rbm.log_prob_batch(p, bits, FORMATS[fmt], NATIVE)
        want, tol = model.native_log_prob(snap.a, snap.b, snap.w, bits, fmt)
        assert np.all(np.abs(lp - want) <= tol), (ci, np.max(np.abs(lp - want) - tol))


@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_native_variants_identical(cuda, fmt):
    """X1, X2 and F64 accumulators hold the same exact theta: with the same
    lane layout they give bitwise identical log p; across layouts only the f32
    summation order of the hidden sum differs."""
    p = rbm.random_parameters(40, 2, derive_key(2, "variants"), 0.01)
    bits = np.random.default_rng(3).integers(0, 2, size=(300, 40), dtype=np.uint8)
    by_layout = {}
    for var in (_native.ACC_X1, _native.ACC_XI, _native.ACC_X2, _native.ACC_F64):
        try:
            ev = rbm.log_prob_evaluator(p, FORMATS[fmt], NATIVE, variant=var)
        except ValueError:
            continue
        key = (ev.snapshot.cluster, ev.snapshot.lanes_per_chain, ev.snapshot.units_per_lane)
        by_layout.setdefault(key, []).append(ev(bits))
    assert sum(len(v) for v in by_layout.values()) >= 2
    firsts = []
    for outs in by_layout.values():
        for o in outs[1:]:
            assert np.array_equal(o, outs[0])
        firsts.append(outs[0])
    for o in firsts[1:]:
        assert np.max(np.abs(o - firsts[0]) / np.maximum(1, np.abs(o))) < 2e-6


@pytest.mark.parametrize("kind", ["flip", "exchange"])
@pytest.mark.parametrize("fmt,scale", [("f16", 0.01), ("f16", 0.3), ("bf16", 0.01), ("bf16", 0.3), ("f32", 0.01)])
def test_native_variant_sweeps_identical(cuda, fmt, scale, kind):
    """MH sweeps with every exact accumulator variant (X1 / X2 / XI / F64, where
    the planner admits it) follow bitwise identical trajectories in the same
    lane layout: covers theta' formed in place and restored on rejection (flip,
    table in shared memory), the select commit (exchange), the sign-ordered
    column difference (XI exchange) and the bf16 XI scale folded into the log
    cosh.  Acceptance is mixed at these scales, so both branches run."""
    n = 40
    p = rbm.random_parameters(n, 2, derive_key(6, "variant-sweeps"), scale)
    prop = sampler.Proposal(kind)
    key = derive_key(7, "chains")
    runs = {}
    for var in (_native.ACC_X1, _native.ACC_XI, _native.ACC_X2, _native.ACC_F64):
        try:
            ev = rbm.log_prob_evaluator(p, FORMATS[fmt], NATIVE, variant=var)
        except ValueError:
            continue
        ens = sampler.ChainEnsemble(96, n, prop, ev, key)
        ens.run_steps(600)
        snap = ens._snapshot()
        layout = (snap.cluster, snap.lanes_per_chain, snap.units_per_lane)
        runs.setdefault(layout, []).append((var, ens.bits, ens.log_probs, ens.accepted, ens.collect(64, 5)))
    assert max(len(v) for v in runs.values()) >= 2, {k: [g[0] for g in v] for k, v in runs.items()}
    for group in runs.values():
        var0, bits0, lp0, acc0, smp0 = group[0]
        assert 0 < acc0 < 96 * 600  # both accepted and rejected moves
        for var, bits, lp, acc, smp in group[1:]:
            assert np.array_equal(bits, bits0), (var0, var)
            assert np.array_equal(lp, lp0), (var0, var)
            assert np.array_equal(acc, acc0) and np.array_equal(smp, smp0), (var0, var)


@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32", "f64"])
@pytest.mark.parametrize("mode", [NATIVE, PER_OP])
def test_zero_parameters_give_zero(cuda, fmt, mode):
    """ref tests/test_rbm.py:58-63; also pins that padded hidden units add exactly 0."""
    n = 13
    p = rbm.RbmParameters(np.zeros(n, complex), np.zeros(3 * n, complex), np.zeros((3 * n, n), complex))
    bits = np.random.default_rng(0).integers(0, 2, size=(64, n), dtype=np.uint8)
    assert np.array_equal(rbm.log_prob_batch(p, bits, FORMATS[fmt], mode), np.zeros(64))


@pytest.mark.parametrize("kind,weight", [("flip", None), ("exchange", 6)])
@pytest.mark.parametrize("fmt", ["f64", "f32", "f16", "bf16"])
def test_ensemble_matches_reference_trajectory(cuda, g_chains, kind, weight, fmt):
    """Device ChainEnsemble with the per-operation evaluator reproduces the
    reference ChainEnsemble step for step (f64: same decisions, log p to 1e-12)."""
    p = params_of(g_chains)
    ev = rbm.log_prob_evaluator(p, FORMATS[fmt], PER_OP)
    ens = sampler.ChainEnsemble(64, 12, sampler.Proposal(kind, weight), ev, g_chains["key"])
    done = 0
    for cp in (0, 1, 50, 300):
        ens.run_steps(cp - done)
        done = cp
        assert np.array_equal(ens.bits, g_chains[f"{kind}_{fmt}_bits_{cp}"]), cp
        assert ens.accepted == int(g_chains[f"{kind}_{fmt}_acc_{cp}"])
        ref = g_chains[f"{kind}_{fmt}_logp_{cp}"]
        tol = 1e-12 if fmt == "f64" else (2e-7 if fmt == "f32" else 0.0)
        assert np.max(np.abs(ens.log_probs - ref) / np.maximum(1, np.abs(ref))) <= tol
    assert ens.proposed == 64 * 300


@pytest.mark.parametrize("ri", [0, 1, 2])
@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_run_chains_matches_reference(cuda, g_chains, ri, fmt):
    c, s, burn, thin, seed = (int(v) for v in g_chains[f"run{ri}_args"])
    ev = rbm.log_prob_evaluator(params_of(g_chains), FORMATS[fmt], PER_OP)
    samples, rate = sampler.run_chains(c, s, burn, thin, seed, ev, sampler.Proposal("flip"), 12)
    assert np.array_equal(samples, g_chains[f"run{ri}_{fmt}_samples"])
    assert rate == float(g_chains[f"run{ri}_{fmt}_rate"])


def test_run_chains_survey_kat(cuda, g_chains):
    p = rbm.random_parameters(4, 1, derive_key(0, "params"), 0.5)
    samples, rate = sampler.run_chains(4, 8, 10, 5, 0, rbm.log_prob_evaluator(p, F32, PER_OP),
                                       sampler.Proposal("flip"), 4)
    codes = (samples * (1 << np.arange(4))).sum(axis=1)
    assert codes.tolist() == [15, 10, 11, 10, 10, 11, 15, 15]
    assert rate == 0.35
    assert np.array_equal(samples, g_chains["kat4_samples"])


@pytest.mark.parametrize("fmt,kind", [("f16", "flip"), ("bf16", "exchange"), ("f32", "flip"), ("f64", "flip")])
def test_launch_and_shard_invariance(cuda, fmt, kind):
    """A chain's trajectory depends only on (key, global chain id, step): one
    long launch == many short ones, a subset of chains == the same chains in a
    larger ensemble, and two shards == one ensemble."""
    n = 30
    p = rbm.random_parameters(n, 2, derive_key(4, "shard"), 0.3)
    mode = NATIVE if fmt != "f64" else PER_OP
    ev = rbm.log_prob_evaluator(p, FORMATS[fmt], mode)
    prop = sampler.Proposal(kind)
    key = derive_key(5, "chains")
    a = sampler.ChainEnsemble(100, n, prop, ev, key)
    a.run_steps(777)
    b = sampler.ChainEnsemble(100, n, prop, ev, key)
    for _ in range(7):
        b.run_steps(111)
    # f64 accumulators are not exact: each launch re-derives theta, so log p may
    # differ in the last ulp; the reduced formats keep theta exact (bitwise equal)
    same_lp = (lambda x, y: np.allclose(x, y, rtol=1e-13, atol=0)) if fmt == "f64" else np.array_equal
    assert np.array_equal(a.bits, b.bits) and same_lp(a.log_probs, b.log_probs)
    assert a.accepted == b.accepted
    s0 = sampler.ChainEnsemble(37, n, prop, ev, key, chain_offset=0, n_chains_total=100)
    s1 = sampler.ChainEnsemble(63, n, prop, ev, key, chain_offset=37, n_chains_total=100)
    for s in (s0, s1):
        s.run_steps(777)
    assert np.array_equal(np.concatenate([s0.bits, s1.bits]), a.bits)
    assert same_lp(np.concatenate([s0.log_probs, s1.log_probs]), a.log_probs)
    # sample rows of the shards concatenate to the single-ensemble matrix
    full = a.collect(250, 7)
    parts = [s.collect(250, 7) for s in (s0, s1)]
    assert np.array_equal(np.concatenate(parts), full)


@pytest.mark.parametrize("n,alpha,scale,kind", [
    (20, 1, 0.5, "flip"),      # configs[0] shape (N=20, alpha=1), peaked state
    (100, 2, 0.1, "flip"),     # configs[1] shape (N=100, alpha=2)
    (100, 2, 0.3, "flip"),     # configs[1] shape, more peaked (larger |log p|, more ties)
    (36, 2, 0.3, "exchange"),  # exchange moves (Sz = 0)
])
def test_native_f32_decisions_match_reference_f32(cuda, n, alpha, scale, kind):
    """NATIVE f32 (exact theta, one rounding, accurate f32 log cosh) against the
    reference per-operation f32 chain (oracle, bit-exact with the reference) in
    lockstep over 1024 chains x 2000 steps: identical decisions except
    near-threshold ties, each one checked against the stated tolerance at its
    first divergent step and then resynchronised (tests/lockstep.py; SURVEY
    §0.5, §8(c)).  The tie counts are printed (DESIGN.md §7 lists them)."""
    from lockstep import run_lockstep

    chains, steps = 1024, 2000
    p = rbm.random_parameters(n, alpha, derive_key(0, "params"), scale)
    key = derive_key(0, "chains")
    ev = rbm.log_prob_evaluator(p, F32, NATIVE)
    weight = None if kind == "flip" else n // 2
    ens = sampler.ChainEnsemble(chains, n, sampler.Proposal(kind, weight), ev, key)
    snap = rbm.round_parameters(p, F32)
    ref = port.PortEnsemble(chains, n, kind, weight, port.Params(snap.a, snap.b, snap.w), "f32", int(key))
    ties, st = run_lockstep(ens, ev, ref, snap, p, steps, kind)
    print(f"\n[f32 decisions] N={n} alpha={alpha} scale={scale} {kind}: {len(ties)} ties in "
          f"{chains * steps} chain-steps; max rel |lp - lp64| device {st['dev_vs_f64']:.2e}, "
          f"reference f32 {st['ref_vs_f64']:.2e}; device vs reference {st['dev_vs_ref']:.2e}")
    for t in ties:
        print("   tie", t)
    assert len(ties) <= 1e-4 * chains * steps


def test_exchange_conserves_sector_and_uniform_accepts(cuda):
    n = 16
    zero = rbm.RbmParameters(np.zeros(n, complex), np.zeros(n, complex), np.zeros((n, n), complex))
    for fmt, mode in ((F16, NATIVE), (F32, PER_OP), (F64, PER_OP)):
        ev = rbm.log_prob_evaluator(zero, fmt, mode)
        samples, rate = sampler.run_chains(64, 512, 20, 3, 4, ev, sampler.Proposal("exchange", 5), n)
        assert (samples.sum(axis=1) == 5).all()
        assert rate == 1.0  # flat target: every proposal accepted (ref tests/test_sampler.py:99-112)


def test_host_callable_evaluator_rejected(cuda):
    with pytest.raises(TypeError):
        sampler.ChainEnsemble(4, 3, sampler.Proposal("flip"), lambda b: np.zeros(len(b)), derive_key(0, "c"))


def test_nonfinite_log_prob_raises_with_context(cuda):
    from paper_2601_20782_b200.errors import EvaluationFailureError

    big = rbm.RbmParameters(np.full(2, 1e308, dtype=complex), np.zeros(2, complex), np.zeros((2, 2), complex))
    with pytest.raises(EvaluationFailureError) as err:
        rbm.log_prob_batch(big, np.array([[1, 1]]), F64)
    assert err.value.context["bits"].tolist() == [1, 1]
    # in a chain: the first failing proposal is reported with its configuration
    # log p = 2 * 1.2e308 overflows exactly when sites 0 and 1 are both up
    p = rbm.RbmParameters(np.array([6e307, 6e307, 0], complex), np.zeros(2, complex), np.zeros((2, 3), complex))
    for fmt, mode in ((F64, PER_OP), (F32, PER_OP), (F32, NATIVE)):
        ev = rbm.log_prob_evaluator(p, fmt, mode) if fmt is F64 else None
        if ev is None:
            continue
        with pytest.raises(EvaluationFailureError) as err:
            ens = sampler.ChainEnsemble(8, 3, sampler.Proposal("flip"), ev, derive_key(0, "chains"))
            ens.run_steps(50)
        assert err.value.context["bits"][:2].tolist() == [1, 1]


def test_deferred_failure_check_reports_the_same_failure(cuda):
    """run_sweeps/set_evaluator(check=False) skip the host synchronisation; the
    sticky status words make the next checked call (collect) raise the same
    first failure (step, chain, configuration) as immediate checking."""
    from paper_2601_20782_b200.errors import EvaluationFailureError

    p = rbm.RbmParameters(np.array([6e307, 6e307, 0], complex), np.zeros(2, complex), np.zeros((2, 3), complex))
    ev = rbm.log_prob_evaluator(p, F64)
    ctx = []
    for deferred in (False, True):
        p0 = rbm.RbmParameters(np.zeros(3, complex), np.zeros(2, complex), np.zeros((2, 3), complex))
        ens = sampler.ChainEnsemble(8, 3, sampler.Proposal("flip"), rbm.log_prob_evaluator(p0, F64),
                                    derive_key(0, "chains"))
        with pytest.raises(EvaluationFailureError) as err:
            if deferred:
                ens.set_evaluator(ev, check=False)
                ens.run_steps(50, check=False)
                ens.collect(16, 4)
            else:
                ens.set_evaluator(ev)
                ens.run_steps(50)
        ctx.append((err.value.context["step"], err.value.context["chain"], err.value.context["bits"].tolist()))
    assert ctx[0] == ctx[1]


@pytest.mark.parametrize("kind,weight", [("flip", None), ("exchange", 5)])
def test_checkpoint_resume_is_bit_identical(cuda, tmp_path, kind, weight):
    """state_dict / save_state -> a fresh ensemble continues exactly like the
    uninterrupted run (bits, log p, counters, collected samples)."""
    p = rbm.random_parameters(10, 2, derive_key(1, "ckpt"), 0.3)
    ev = rbm.log_prob_evaluator(p, F16, NATIVE)
    key = derive_key(2, "chains")
    ref = sampler.ChainEnsemble(64, 10, sampler.Proposal(kind, weight), ev, key)
    ref.run_steps(137)
    path = ref.save_state(tmp_path / "chains.npz")
    ref.run_steps(91)
    s_ref = ref.collect(256, 11)
    res = sampler.ChainEnsemble(64, 10, sampler.Proposal(kind, weight), ev, key)
    res.run_steps(3)  # diverged state, overwritten by the checkpoint
    res.load_state(path)
    res.run_steps(91)
    s_res = res.collect(256, 11)
    np.testing.assert_array_equal(s_res, s_ref)
    np.testing.assert_array_equal(res.bits, ref.bits)
    np.testing.assert_array_equal(res.log_probs, ref.log_probs)
    assert res.accepted == ref.accepted and res.proposed == ref.proposed


@pytest.mark.parametrize("n,alpha,chains,kind", [(1, 2, 5, "flip"), (2, 3, 7, "exchange"), (31, 1, 33, "flip"),
                                                 (32, "1/2", 64, "exchange"), (33, "3/11", 3, "flip"),
                                                 (65, "1/5", 40, "flip"), (97, 1, 1, "exchange")])
@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_edge_shapes_per_op_bitwise(cuda, n, alpha, chains, kind, fmt):
    """Per-operation chains bit-identical to the oracle at edge shapes: one site,
    word boundaries (31/32/33, 65, 97 sites), tiny M, odd chain counts, one chain."""
    from fractions import Fraction

    p = rbm.random_parameters(n, Fraction(alpha), derive_key(n, "edge"), 0.4)
    key = derive_key(n + 1, "chains")
    prop = sampler.Proposal(kind, None if kind == "flip" else max(1, n // 2))
    ev = rbm.log_prob_evaluator(p, FORMATS[fmt], PER_OP)
    ens = sampler.ChainEnsemble(chains, n, prop, ev, key)
    snap = rbm.round_parameters(p, FORMATS[fmt])
    ref = port.PortEnsemble(chains, n, kind, None if kind == "flip" else max(1, n // 2),
                            port.Params(snap.a, snap.b, snap.w), fmt, int(key))
    ens.run_steps(150)
    ref.run_steps(150)
    np.testing.assert_array_equal(ens.bits, ref.bits)
    np.testing.assert_array_equal(ens.log_probs, ref.logp)
    assert ens.accepted == ref.accepted


@pytest.mark.parametrize("n,alpha", [(1, 3), (2, "5/2"), (31, 1), (33, "3/11"), (65, "1/5"), (97, 2), (200, 1)])
@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32"])
def test_edge_shapes_native_model(cuda, n, alpha, fmt):
    """NATIVE fused-sweep evaluation at edge shapes (lane layouts with padded
    hidden units, word boundaries, M = 1..200) against the arithmetic model,
    and a short chain run stays consistent with its own re-evaluation."""
    from fractions import Fraction

    from oracle import model

    p = rbm.random_parameters(n, Fraction(alpha), derive_key(n, "edge-native"), 0.3)
    snap = rbm.round_parameters(p, FORMATS[fmt])
    bits = np.random.default_rng(n).integers(0, 2, size=(37, n), dtype=np.uint8)
    ev = rbm.log_prob_evaluator(p, FORMATS[fmt], NATIVE)
    want, tol = model.native_log_prob(snap.a, snap.b, snap.w, bits, fmt)
    assert np.all(np.abs(ev(bits) - want) <= tol), ev.snapshot.label
    kinds = [("flip", None)] + ([("exchange", n // 2)] if n >= 2 else [])
    for kind, weight in kinds:
        ens = sampler.ChainEnsemble(19, n, sampler.Proposal(kind, weight), ev, derive_key(3, "chains"))
        ens.run_steps(120)
        # cached log p == fresh evaluation (in the sweep's lane layout)
        np.testing.assert_array_equal(ens.log_probs, ev.for_proposal(kind)(ens.bits))
        if kind == "exchange":
            assert np.all(ens.bits.sum(axis=1) == n // 2)


@pytest.mark.parametrize("n,alpha,fmt,kind,scale", [(100, 4, "bf16", "exchange", 0.01), (256, 1, "f16", "flip", 0.01),
                                                     (100, 2, "f32", "flip", 0.3)])
def test_cluster_split_sweep(cuda, monkeypatch, n, alpha, fmt, kind, scale):
    """Opt-in cluster split (MPV_CLUSTER_SPLIT=1: the hidden units of a table
    beyond shared memory split over 2 or 4 CTAs of a thread-block cluster that
    exchange partial sums every step): log p equals the arithmetic model (and,
    for f32, the f64 value to 1e-5), chains stay consistent with fresh
    evaluations, shards reproduce the single ensemble."""
    from oracle import model

    monkeypatch.setenv("MPV_CLUSTER_SPLIT", "1")
    p = rbm.random_parameters(n, alpha, derive_key(n, "cluster"), scale)
    ev = rbm.log_prob_evaluator(p, FORMATS[fmt], NATIVE)
    assert ev.snapshot.cluster > 1, ev.snapshot.label
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, size=(500, n), dtype=np.uint8)
    got = ev(bits)
    if fmt == "f32":
        ref = rbm.log_prob_batch(p, bits, F64)
        assert np.max(np.abs(got - ref) / np.maximum(1, np.abs(ref))) < 1e-5
    else:
        r = rbm.round_parameters(p, FORMATS[fmt])
        want, tol = model.native_log_prob(r.a, r.b, r.w, bits, fmt)
        assert np.all(np.abs(got - want) <= tol)
    prop = sampler.Proposal(kind, n // 2 if kind == "exchange" else None)
    key = derive_key(2, "chains")
    a = sampler.ChainEnsemble(300, n, prop, ev, key)
    a.run_steps(700)
    np.testing.assert_array_equal(a.log_probs, ev.for_proposal(kind)(a.bits))
    s0 = sampler.ChainEnsemble(100, n, prop, ev, key, chain_offset=0, n_chains_total=300)
    s1 = sampler.ChainEnsemble(200, n, prop, ev, key, chain_offset=100, n_chains_total=300)
    for s in (s0, s1):
        s.run_steps(700)
    np.testing.assert_array_equal(np.concatenate([s0.bits, s1.bits]), a.bits)


@pytest.mark.parametrize("fmt", ["f16", "bf16", "f32", "f64"])
def test_exchange_collect_rows_equal_stepped_bits(cuda, fmt):
    """Fused exchange sweeps (one chain per warp; steps whose swap exchanges equal
    bits are skipped by the warp but still counted and recorded): the collected
    rows equal the chains' bits read after every `thin` steps of a stepped twin
    (chain-major rows, sampler.py:142-167), and the acceptance counters agree."""
    n, chains, per_chain, thin = 24, 40, 3, 5
    p = rbm.random_parameters(n, 2, derive_key(6, "xrec"), 0.3)
    mode = NATIVE if fmt != "f64" else PER_OP
    ev = rbm.log_prob_evaluator(p, FORMATS[fmt], mode)
    prop = sampler.Proposal("exchange", n // 2)
    key = derive_key(8, "chains")
    a = sampler.ChainEnsemble(chains, n, prop, ev, key)
    rows = a.collect(chains * per_chain, thin)
    b = sampler.ChainEnsemble(chains, n, prop, ev, key)
    snaps = []
    for _ in range(per_chain):
        b.run_steps(thin)
        snaps.append(b.bits.copy())
    want = np.stack(snaps, axis=1).reshape(chains * per_chain, n)  # chain-major
    assert np.array_equal(rows, want)
    assert a.accepted == b.accepted and a.proposed == b.proposed
    assert np.all(rows.sum(axis=1) == n // 2)


def test_bench_workload_full_size_properties(cuda):
    """The bench step at its full size (BASELINE configs[1]: 10x10 TFIM, alpha=2,
    16,384 chains, f16 NATIVE, 2 re-burn sweeps, 65,536 samples at thinning
    N+1), through size-independent properties: two chain shards reproduce the
    single ensemble's samples bit for bit, every chain's cached log p equals a
    fresh evaluation, and a random subsample's f64 local energies equal the
    oracle's restatement of the reference."""
    from oracle import port
    from paper_2601_20782_b200 import vmc
    from paper_2601_20782_b200.hamiltonians import TfimSpec
    from paper_2601_20782_b200.lattice import LatticeSpec

    n, chains = 100, 16384
    p = rbm.random_parameters(n, 2, derive_key(0, "init"), 0.01)
    ev = rbm.log_prob_evaluator(p, FORMATS["f16"], NATIVE)
    prop = sampler.Proposal("flip")
    key = derive_key(0, "chains")
    full = sampler.ChainEnsemble(chains, n, prop, ev, key)
    full.run_sweeps(2)
    rows = full.collect(4 * chains, n + 1)
    np.testing.assert_array_equal(full.log_probs, ev(full.bits))
    parts = []
    for off, cnt in ((0, 7000), (7000, chains - 7000)):
        s = sampler.ChainEnsemble(cnt, n, prop, ev, key, chain_offset=off, n_chains_total=chains)
        s.run_sweeps(2)
        parts.append(s.collect(4 * chains, n + 1))
    np.testing.assert_array_equal(np.concatenate(parts), rows)
    spec = TfimSpec(LatticeSpec.square(10), 1.0, 3.04)
    sub = rows[np.random.default_rng(0).choice(rows.shape[0], size=64, replace=False)]
    eps = vmc.local_energies(spec, rbm.log_psi_evaluator(p), sub)
    want = port.local_energies(port.Params(p.a, p.b, p.w), "tfim", spec.lattice.bond_array(), 1.0, 3.04, sub)
    assert np.max(np.abs(eps - want) / np.maximum(1, np.abs(want))) < 1e-11
