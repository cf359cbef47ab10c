"""Tensor-core (tcgen05) batched forward, mpv_forward_tc, against the oracle's
f64 forward of the same rounded parameters (ref: rbm.py:130-150 _fast_forward,
rbm.py:91-101 round_parameters; oracle/c/oracle_port.c f64_row).

The GEMM products are exact (x in {0,1}, f16/bf16 weights) and the kernel
accumulates theta and the log-cosh sum in f32, so the tolerance is the
north star's f32 bar: log psi within 1e-5 relative (floor 1)."""
import numpy as np
import pytest
import torch

from oracle import port
from paper_2601_20782_b200 import rbm
from paper_2601_20782_b200.precision import BF16, F16, F32
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu

CASES = [  # (N, alpha, scale, B)
    (1, 1, 0.5, 5),
    (12, 2, 0.4, 300),
    (37, 3, 0.3, 1000),      # M = 111: padded hidden columns
    (100, 2, 0.05, 5000),    # configs[1] shape
    (100, 4, 0.05, 2000),    # M = 400: two hidden chunks, B re-staged per chunk
    (256, 1, 0.05, 700),     # Kp = 256: chunk size capped by shared memory
    (333, 1, 0.03, 129),     # odd N across words, one full tile + 1
]


def _bits(B, N, seed):
    return np.random.default_rng(seed).integers(0, 2, size=(B, N), dtype=np.uint8)


def _oracle(params, fmt, bits):
    snap = rbm.round_parameters(params, fmt)
    _, re, im = port.f64_forward(port.Params(snap.a, snap.b, snap.w), bits)
    return re, im


def _conditioning(params, fmt, bits):
    """sum_i |tanh theta_i| |theta_i|: the change of log psi under a relative
    perturbation of every theta (log|cosh| is ill-conditioned near the zeros of
    cosh, where f32 theta alone moves the f64 answer)."""
    snap = rbm.round_parameters(params, fmt)
    theta = snap.b[None, :] + bits.astype(np.float64) @ snap.w.T
    return np.sum(np.abs(np.tanh(theta)) * np.abs(theta), axis=1)


@pytest.mark.parametrize("fmt", [F16, BF16], ids=["f16", "bf16"])
@pytest.mark.parametrize("N,alpha,scale,B", CASES)
def test_forward_tc_matches_f64_of_rounded(fmt, N, alpha, scale, B):
    params = rbm.random_parameters(N, alpha, derive_key(N * 7 + alpha, "tc"), scale)
    bits = _bits(B, N, N + B)
    tc = rbm.TensorCoreForward(params, fmt)
    got = tc(bits)
    re, im = _oracle(params, fmt, bits)
    # 1e-5 relative (floor 1) plus the f32-theta conditioning term (K*2^-24 ~ 1e-6 per unit)
    cond = 1e-6 * _conditioning(params, fmt, bits)
    tol_re = 1e-5 * np.maximum(1.0, np.abs(re)) + cond
    tol_im = 1e-5 * np.maximum(1.0, np.abs(im)) + cond
    assert np.all(np.abs(got.real - re) <= tol_re), np.max(np.abs(got.real - re) / tol_re)
    assert np.all(np.abs(got.imag - im) <= tol_im), np.max(np.abs(got.imag - im) / tol_im)
    # log p only (the epilogue without the phase: ex2, cos 2v, lg2 per hidden unit)
    lp = torch.empty(B, dtype=torch.float64, device=tc.device)
    tc.forward_packed(rbm.device_pack(bits, tc.device), out_lp=lp)
    lp = lp.cpu().numpy()
    tol_lp = 2.0 * tol_re
    assert np.all(np.abs(lp - 2.0 * re) <= tol_lp), np.max(np.abs(lp - 2.0 * re) / tol_lp)


def test_forward_tc_large_theta_and_log_prob():
    """|Re theta| up to ~30 (t = exp(-2u) underflow side) and out_lp = 2 Re log psi."""
    N, B = 64, 512
    params = rbm.random_parameters(N, 2, derive_key(3, "tc-big"), 1.0)
    bits = _bits(B, N, 11)
    tc = rbm.TensorCoreForward(params, F16)
    packed = rbm.device_pack(bits, tc.device)
    lp, re, im = tc.forward_packed(packed)
    want_re, want_im = _oracle(params, F16, bits)
    assert np.allclose(re.cpu().numpy(), want_re, rtol=1e-5, atol=1e-5)
    assert np.array_equal(lp.cpu().numpy(), 2.0 * re.cpu().numpy())


def test_forward_tc_deterministic_across_grids():
    """Each row's sums run in a fixed order: the grid size does not change a bit."""
    N, B = 100, 3000
    params = rbm.random_parameters(N, 2, derive_key(5, "tc-det"), 0.1)
    tc = rbm.TensorCoreForward(params, BF16)
    packed = rbm.device_pack(_bits(B, N, 7), tc.device)
    a = [t.cpu().numpy() for t in tc.forward_packed(packed)]
    b = [t.cpu().numpy() for t in tc.forward_packed(packed, max_ctas=3)]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    lp = torch.empty(B, dtype=torch.float64, device=tc.device)
    tc.forward_packed(packed, out_lp=lp)
    lp2 = torch.empty_like(lp)
    tc.forward_packed(packed, out_lp=lp2, max_ctas=5)
    assert np.array_equal(lp.cpu().numpy(), lp2.cpu().numpy())


@pytest.mark.parametrize("N,alpha,B,ctas", [
    (37, 3, 2100, 2),   # M = 111: one hidden chunk per tile, 9 tiles per CTA (the tightest mbarrier hand-off)
    (12, 20, 1900, 2),  # M = 240: three hidden chunks per tile, ragged last tile
    (100, 2, 1000, 1),  # a single CTA runs every tile of the batch
])
def test_forward_tc_many_tiles_per_cta(N, alpha, B, ctas):
    """Pipelined kernel with many tiles per CTA (A, TMEM and partial-sum buffers
    wrap many times): equal to the oracle and bit-equal to the full grid."""
    params = rbm.random_parameters(N, alpha, derive_key(N * 13 + alpha, "tc-wrap"), 0.2)
    bits = _bits(B, N, N * 3 + B)
    tc = rbm.TensorCoreForward(params, F16)
    packed = rbm.device_pack(bits, tc.device)
    few = [t.cpu().numpy() for t in tc.forward_packed(packed, max_ctas=ctas)]
    full = [t.cpu().numpy() for t in tc.forward_packed(packed)]
    for x, y in zip(few, full):
        assert np.array_equal(x, y)
    re, im = _oracle(params, F16, bits)
    cond = 1e-6 * _conditioning(params, F16, bits)
    assert np.all(np.abs(few[1] - re) <= 1e-5 * np.maximum(1.0, np.abs(re)) + cond)
    assert np.all(np.abs(few[2] - im) <= 1e-5 * np.maximum(1.0, np.abs(im)) + cond)


def test_forward_tc_rejects_other_formats_and_empty_batch():
    params = rbm.random_parameters(10, 1, derive_key(1, "tc-x"), 0.1)
    with pytest.raises(ValueError):
        rbm.TensorCoreForward(params, F32)
    tc = rbm.TensorCoreForward(params, F16)
    out = tc(np.zeros((0, 10), dtype=np.uint8))
    assert out.shape == (0,)


def test_forward_tc_full_size_subsample():
    """configs[1]-sized batch (65,536 samples x 100 flips = 6,553,600 configurations):
    a seeded subsample against the oracle, and log p == 2 Re log psi of the
    phase epilogue over the whole batch (two different epilogues, same GEMM)."""
    N, B = 100, 65536 * 100
    params = rbm.random_parameters(N, 2, derive_key(9, "tc-full"), 0.05)
    tc = rbm.TensorCoreForward(params, F16)
    g = torch.Generator(device=tc.device).manual_seed(3)
    packed = torch.randint(-2**31, 2**31 - 1, (B, 4), dtype=torch.int32, device=tc.device, generator=g)
    packed[:, -1] &= (1 << (N % 32)) - 1
    lp, re, im = tc.forward_packed(packed)
    lp_only = torch.empty_like(lp)
    tc.forward_packed(packed, out_lp=lp_only)

    def unpack(rows):
        words = packed[torch.from_numpy(rows).to(tc.device)].cpu().numpy().view(np.uint32)
        return ((words[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(len(rows), -1)[:, :N].astype(np.uint8)

    # the two epilogues agree to 4e-5 relative; rows beyond that must be the
    # ill-conditioned ones (a hidden unit near a zero of cosh), within the conditioning term
    diff = torch.abs(lp_only - lp)
    bad = torch.nonzero(diff > 4e-5 * torch.clamp(torch.abs(lp), min=1.0)).flatten().cpu().numpy()
    assert len(bad) < B // 1000, len(bad)
    if len(bad):
        cond = 4e-6 * _conditioning(params, F16, unpack(bad))
        lim = 4e-5 * np.maximum(1.0, np.abs(lp.cpu().numpy()[bad])) + cond
        assert np.all(diff.cpu().numpy()[bad] <= lim), np.max(diff.cpu().numpy()[bad] / lim)
    rows = np.random.default_rng(5).choice(B, size=3000, replace=False)
    bits = unpack(rows)
    want_re, want_im = _oracle(params, F16, bits)
    got_re = re.cpu().numpy()[rows]
    got_im = im.cpu().numpy()[rows]
    cond = 1e-6 * _conditioning(params, F16, bits)
    assert np.all(np.abs(got_re - want_re) <= 1e-5 * np.maximum(1.0, np.abs(want_re)) + cond)
    assert np.all(np.abs(got_im - want_im) <= 1e-5 * np.maximum(1.0, np.abs(want_im)) + cond)


def test_forward_tc_small_u_near_cosh_zero():
    """|Re theta| just below the 1/16 series threshold of 1 - e^{-2u} with Im theta
    near pi/2 (where the phase is most sensitive to that factor): theta = b is
    exact in f32 for the all-zero configuration, so the epilogue alone is checked
    against the f64 forward, at the 1e-5 relative bar with no conditioning term."""
    M = 128
    i = np.arange(M)
    u = np.where(i % 2 == 0, 0.06, 0.0305) * np.where(i % 4 < 2, 1.0, -1.0)
    v = np.pi / 2 + np.linspace(-0.09, 0.09, M)
    b = u + 1j * v
    params = rbm.RbmParameters(np.zeros(1, complex), b, np.zeros((M, 1), complex))
    bits = np.zeros((256, 1), dtype=np.uint8)
    for fmt in (F16, BF16):
        got = rbm.TensorCoreForward(params, fmt)(bits)
        re, im = _oracle(params, fmt, bits)
        assert np.all(np.abs(got.real - re) <= 1e-5 * np.maximum(1.0, np.abs(re)))
        assert np.all(np.abs(got.imag - im) <= 1e-5 * np.maximum(1.0, np.abs(im))), np.max(np.abs(got.imag - im))
