"""ResCNN neural quantum state on the B200 (beyond the reference: the
convolutional ansatz of /root/reference/PAPER.md:876-890, used for BASELINE
configs[3]; the reference package has none, so parity is pinned by the f64
restatement oracle/rescnn.py and by exact H psi on enumerable lattices).

    s = 1 - 2x,  h0 = Conv(s),  h_{l+1} = h_l + Conv(GELU(Conv(GELU(LN(h_l))))),
    log psi(x) = sum_{sites, channels} LN(h_n)           (real; log p = 2 log psi)

3x3 periodic convolutions with bias, 16 channels, LN over the channels of a
site (learned gain / shift, eps 1e-6), GELU in its tanh form.  Evaluation runs
in the CUDA library (csrc/rescnn.cu): a tcgen05 tensor-core forward with
f16/bf16 operands and f32 accumulation (the sampler's evaluator, fused with the
MH step), and an f64 forward on the FP64 tensor cores (DMMA; local energies,
parity).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import EvaluationFailureError
from .precision import FloatFormat, make_rounder
from .rng import gaussian_field

FILTERS = 16
TAPS = 9


def param_layout(n_res: int):
    """(name, shape) of the flat parameter vector, in order (oracle/rescnn.py)."""
    F, T = FILTERS, TAPS
    out = [("w0", (F, 1, T)), ("b0", (F,))]
    for i in range(n_res):
        out += [(f"g{i}", (F,)), (f"be{i}", (F,)), (f"w{i}a", (F, F, T)), (f"b{i}a", (F,)),
                (f"w{i}b", (F, F, T)), (f"b{i}b", (F,))]
    return out + [("gf", (F,)), ("bef", (F,))]


def n_params(n_res: int) -> int:
    return int(sum(np.prod(s) for _, s in param_layout(n_res)))


@dataclass(frozen=True)
class ResCnnParameters:
    """Flat real f64 parameters of a ResCNN on an L x L periodic lattice."""

    theta: np.ndarray
    L: int
    n_res: int = 4

    def __post_init__(self):
        th = np.ascontiguousarray(self.theta, dtype=np.float64)
        if th.shape != (n_params(self.n_res),):
            raise ValueError(f"expected {n_params(self.n_res)} parameters, got {th.shape}")
        if not np.all(np.isfinite(th)):
            raise ValueError("non-finite parameters")
        if not 3 <= self.L <= 30:
            raise ValueError("3 <= L <= 30")
        object.__setattr__(self, "theta", th)

    @property
    def n_visible(self) -> int:
        return self.L * self.L

    def unflatten(self) -> dict:
        out, k = {}, 0
        for name, shape in param_layout(self.n_res):
            size = int(np.prod(shape))
            out[name] = self.theta[k:k + size].reshape(shape)
            k += size
        return out


def random_parameters(L: int, n_res: int, key, scale: float = 1.0) -> ResCnnParameters:
    """Counter-based Gaussian init (the rbm.random_parameters field, rng.py:86-96):
    conv weights N(0, scale^2 / fan_in), biases N(0, (0.1 scale)^2), LN gains
    1 + N(0, 0.1^2), shifts N(0, 0.1^2)."""
    z = gaussian_field(key, np.arange(n_params(n_res)), 1.0)
    theta = np.empty_like(z)
    k = 0
    for name, shape in param_layout(n_res):
        size = int(np.prod(shape))
        v = z[k:k + size]
        if name.startswith("w"):
            fan_in = shape[1] * shape[2]
            v = v * scale / np.sqrt(fan_in)
        elif name.startswith("g"):
            v = 1.0 + 0.1 * v
        elif name.startswith("be"):
            v = 0.1 * v
        else:
            v = 0.1 * scale * v
        theta[k:k + size] = v
        k += size
    return ResCnnParameters(theta, L, n_res)


def _bits16(values, fmt: FloatFormat) -> np.ndarray:
    """RNE rounding to f16/bf16 (round_parameters semantics), as uint16 bit patterns."""
    v = np.asarray(values, dtype=np.float64)
    if fmt.name == "f16":
        return v.astype(np.float16).view(np.uint16)
    r = make_rounder(fmt)(v).astype(np.float32)  # exact bf16 values
    return (r.view(np.uint32) >> 16).astype(np.uint16)


def rounded_parameters(params: ResCnnParameters, fmt: FloatFormat) -> ResCnnParameters:
    """The parameters the tensor-core forward uses: convolution weights rounded
    to fmt (RNE), vectors rounded to f32 (the epilogue's precision)."""
    out = params.theta.copy()
    k = 0
    rnd = make_rounder(fmt)
    for name, shape in param_layout(params.n_res):
        size = int(np.prod(shape))
        seg = out[k:k + size]
        out[k:k + size] = rnd(seg) if name.startswith("w") else seg.astype(np.float32).astype(np.float64)
        k += size
    return ResCnnParameters(out, params.L, params.n_res)


def make_blob(params: ResCnnParameters, fmt: FloatFormat) -> np.ndarray:
    """Kernel operand blob (include/mpvmc_b200.h): per convolution and tap the
    16 x 16 B operand W[cout][cin] in the K-major core-matrix layout (element
    (n, k) at byte (n&7)*16 + (n>>3)*256 + (k>>3)*128 + (k&7)*2), then f32 vectors:
    per LN the running residual bias b0 + sum of the earlier blocks' second
    biases, the gain and the shift; then each block's first-convolution bias."""
    p = params.unflatten()
    n_res, F = params.n_res, FILTERS
    convs = [np.concatenate([p["w0"], np.zeros((F, F - 1, TAPS))], axis=1)]
    for i in range(n_res):
        convs += [p[f"w{i}a"], p[f"w{i}b"]]
    n, k = np.meshgrid(np.arange(F), np.arange(F), indexing="ij")
    off = ((n & 7) * 16 + (n >> 3) * 256 + (k >> 3) * 128 + (k & 7) * 2) // 2
    blocks = np.zeros((len(convs), TAPS, 256), dtype=np.uint16)
    for ci, w in enumerate(convs):
        bits = _bits16(w, fmt)  # [cout][cin][tap]
        for d in range(TAPS):
            blocks[ci, d, off.ravel()] = bits[:, :, d].ravel()
    vec = []
    run = p["b0"].copy()
    for i in range(n_res):
        vec += [run.copy(), p[f"g{i}"], p[f"be{i}"]]
        run = run + p[f"b{i}b"]
    vec += [run, p["gf"], p["bef"]]
    vec += [p[f"b{i}a"] for i in range(n_res)]
    vec = np.concatenate(vec).astype(np.float32)
    size = int(nat.load().mpv_rescnn_blob_bytes(params.L, n_res))
    if size == 0:
        raise ValueError(f"unsupported ResCNN shape L={params.L}, n_res={n_res}")
    out = np.zeros(size, dtype=np.uint8)
    b = blocks.view(np.uint8).ravel()
    out[:b.size] = b
    out[b.size:b.size + vec.nbytes] = vec.view(np.uint8)
    return out


class ResCnnEvaluator:
    """Device log-probability evaluator of a ResCNN (the reference evaluator
    protocol, sampler.py:49-53: uint8[B, N] -> float64[B]).  fmt f16/bf16: the
    tcgen05 forward (ChainEnsemble fuses it into the MH step); f64: the DMMA f64
    forward (2 log psi)."""

    def __init__(self, params: ResCnnParameters, fmt: FloatFormat, device=None):
        import torch

        nat.require_cuda()
        if fmt.name not in ("f16", "bf16", "f64"):
            raise ValueError("the ResCNN evaluator takes f16, bf16 (tensor cores) or f64")
        self.params, self.fmt = params, fmt
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.L, self.n_res = params.L, params.n_res
        self.n_visible = params.n_visible
        self.theta = torch.from_numpy(params.theta).to(self.device)
        self.blob = None
        if fmt.name != "f64":
            self.blob = torch.from_numpy(make_blob(params, fmt)).to(self.device)

    def log_prob_packed(self, packed):
        import torch

        packed = packed.contiguous()
        B = packed.shape[0]
        out = torch.empty(B, dtype=torch.float64, device=self.device)
        status = torch.tensor([0, 2**63 - 1], dtype=torch.int64, device=self.device)
        st = nat.stream_handle(self.device)
        if self.blob is None:
            nat.call("mpv_rescnn_forward_f64", self.theta.data_ptr(), self.L, self.n_res, packed.data_ptr(), B,
                     out.data_ptr(), st)
            out.mul_(2.0)
        else:
            nat.call("mpv_rescnn_forward", self.L, self.n_res, self.fmt.code, self.blob.data_ptr(), packed.data_ptr(),
                     B, out.data_ptr(), status.data_ptr(), st)
        return out, status

    def __call__(self, bits) -> np.ndarray:
        from .rbm import device_pack

        bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
        if bits.shape[1] != self.n_visible:
            raise ValueError(f"bit matrix has {bits.shape[1]} sites, ansatz has {self.n_visible}")
        out, status = self.log_prob_packed(device_pack(bits, self.device))
        out = out.cpu().numpy()
        if not np.all(np.isfinite(out)):
            bad = int(np.nonzero(~np.isfinite(out))[0][0])
            raise EvaluationFailureError("non-finite log probability", context={"bits": bits[bad].copy()})
        return out


def log_prob_evaluator(params: ResCnnParameters, fmt: FloatFormat, device=None) -> ResCnnEvaluator:
    return ResCnnEvaluator(params, fmt, device)


def log_psi_packed(params: ResCnnParameters, packed, device=None):
    """f64 log psi of packed configurations (device tensor)."""
    ev = ResCnnEvaluator(params, FloatFormat_f64(), device)
    lp, _ = ev.log_prob_packed(packed)
    return 0.5 * lp


def FloatFormat_f64():
    from .precision import F64

    return F64


def local_energies_packed(spec, params: ResCnnParameters, packed, device=None):
    """eps(x) = sum_x' H(x, x') psi(x') / psi(x) (the reference's local energy,
    vmc.py:60-108) for the real ResCNN amplitude: connected configurations built
    with device bit operations, every amplitude from the f64 forward.  TFIM: all
    single flips, H = h; Heisenberg / J1-J2 (optionally Marshall): anti-aligned
    bonds, H = the bond's off-diagonal coefficient.  Returns complex128 [B]."""
    import torch

    from .hamiltonians import HeisenbergSpec, J1J2Spec, TfimSpec

    dev = packed.device
    N = params.n_visible
    words = (N + 31) // 32
    B = packed.shape[0]
    packed = packed.contiguous().view(torch.int32)
    lp0 = log_psi_packed(params, packed, dev)
    sites = torch.arange(N, device=dev)
    bits = ((packed[:, sites // 32] >> (sites % 32)) & 1).to(torch.int64)  # (B, N)
    spin = 1 - 2 * bits
    if isinstance(spec, TfimSpec):
        bonds = torch.from_numpy(spec.lattice.bond_array()).to(dev)
        diag = float(spec.j) * (spin[:, bonds[:, 0]] * spin[:, bonds[:, 1]]).sum(dim=1).to(torch.float64)
        mask = torch.zeros((N, words), dtype=torch.int64, device=dev)
        mask[sites, sites // 32] = (1 << (sites % 32))
        conn = (packed.to(torch.int64)[:, None, :] ^ mask[None]).reshape(B * N, words)
        owner = torch.arange(B, device=dev).repeat_interleave(N)
        coef = torch.full((B * N,), float(spec.h), dtype=torch.float64, device=dev)
        slot = (owner, sites.repeat(B))
    elif isinstance(spec, (HeisenbergSpec, J1J2Spec)):
        b_np, jb_np, cf_np = spec.couplings()
        bonds = torch.from_numpy(b_np).to(dev)
        jb = torch.from_numpy(jb_np).to(dev)
        cf = torch.from_numpy(cf_np).to(dev)
        diag = (jb[None, :] * (spin[:, bonds[:, 0]] * spin[:, bonds[:, 1]])).sum(dim=1).to(torch.float64)
        differ = bits[:, bonds[:, 0]] != bits[:, bonds[:, 1]]  # (B, nb)
        s_idx, b_idx = torch.nonzero(differ, as_tuple=True)
        i, j = bonds[b_idx, 0], bonds[b_idx, 1]
        mask = torch.zeros((s_idx.numel(), words), dtype=torch.int64, device=dev)
        mask.scatter_(1, (i // 32)[:, None], (1 << (i % 32))[:, None])
        mask.scatter_add_(1, (j // 32)[:, None], (1 << (j % 32))[:, None])
        conn = packed.to(torch.int64)[s_idx] ^ mask
        owner = s_idx
        coef = cf[b_idx].to(torch.float64)
        slot = (s_idx, b_idx)  # each ratio's (sample, bond) cell: a fixed-order row sum below
    else:
        raise TypeError(f"unknown Hamiltonian spec {type(spec).__name__}")
    conn32 = conn.to(torch.int32).contiguous() if conn.numel() else torch.empty((0, words), dtype=torch.int32,
                                                                                     device=dev)
    lpc = log_psi_packed(params, conn32, dev)
    ratio = torch.exp(lpc - lp0[owner]) * coef
    # (sample, term) matrix summed along rows: a fixed summation order (no atomics)
    cells = torch.zeros((B, N if isinstance(spec, TfimSpec) else bonds.shape[0]), dtype=torch.float64, device=dev)
    cells[slot] = ratio
    off = cells.sum(dim=1)
    eps = diag + off
    return torch.complex(eps, torch.zeros_like(eps))


# ---------------------------------------------------------------------------
# Training (BASELINE configs[3]: "minSR in f32, chain sharding").  Sampling
# uses the fused tensor-core MH step, local energies the f64 forward; the
# per-sample log-derivatives O = d log psi / d theta come from one batched
# torch autograd backward over a torch restatement of the same network in f64
# plus per-layer site contractions (cuDNN / cuBLAS - the gradient statistics
# stay f32/f64, north_star (4)), and
# the SR step is solved in sample space (minSR) in f32 or f64, sharded.
# ---------------------------------------------------------------------------

def torch_log_psi(theta, spins, L: int, n_res: int):
    """log psi for spins (B, L, L) = 1 - 2x as a torch function of theta (autograd)."""
    import torch
    import torch.nn.functional as tf

    F, k = FILTERS, 0
    p = {}
    for name, shape in param_layout(n_res):
        size = int(np.prod(shape))
        p[name] = theta[k:k + size].reshape(shape)
        k += size

    def conv(h, w, b):
        hp = tf.pad(h, (1, 1, 1, 1), mode="circular")
        return tf.conv2d(hp, w.reshape(w.shape[0], w.shape[1], 3, 3), b)

    def ln(h, g, be):
        mu = h.mean(dim=1, keepdim=True)
        var = ((h - mu) ** 2).mean(dim=1, keepdim=True)
        return g[None, :, None, None] * (h - mu) / torch.sqrt(var + 1e-6) + be[None, :, None, None]

    h = conv(spins[:, None], p["w0"], p["b0"])
    for i in range(n_res):
        u = tf.gelu(ln(h, p[f"g{i}"], p[f"be{i}"]), approximate="tanh")
        v = tf.gelu(conv(u, p[f"w{i}a"], p[f"b{i}a"]), approximate="tanh")
        h = h + conv(v, p[f"w{i}b"], p[f"b{i}b"])
    return ln(h, p["gf"], p["bef"]).sum(dim=(1, 2, 3))


def log_derivatives(params: ResCnnParameters, packed):
    """O[s] = d log psi(x_s) / d theta (U, P) f64 on the device.

    Per-sample gradients from ONE batched backward: the samples are independent,
    so d(sum_s log psi_s)/d(output of a layer)[s] is sample s's own output
    gradient; each parametric layer's per-sample parameter gradient is then a
    contraction over the lattice sites of that output gradient with the
    layer's input (convolution: the unfolded 3x3 neighbourhoods, one batched
    f64 GEMM; bias: a site sum; LayerNorm gain/shift: sums of dy * x_hat and
    dy).  Equal to the per-sample autograd (`_log_derivatives_vmap`) to f64
    rounding (tests/test_gpu_rescnn.py)."""
    import torch
    import torch.nn.functional as tf

    dev = packed.device
    L, n, n_res = params.L, params.n_visible, params.n_res
    sites = torch.arange(n, device=dev)
    bits = ((packed.view(torch.int32)[:, sites // 32] >> (sites % 32)) & 1).to(torch.float64)
    B = bits.shape[0]
    F = FILTERS
    theta = torch.from_numpy(params.theta).to(dev)
    p, k = {}, 0
    for name, shape in param_layout(n_res):
        size = int(np.prod(shape))
        p[name] = theta[k:k + size].reshape(shape)
        k += size
    convs, lns = {}, {}  # name -> (padded input, output); name -> (x_hat, output)

    def conv(h, wn, bn):
        hp = tf.pad(h, (1, 1, 1, 1), mode="circular")
        w = p[wn]
        o = tf.conv2d(hp, w.reshape(w.shape[0], w.shape[1], 3, 3), p[bn])
        convs[wn] = (hp, o)
        return o

    def ln(h, gn, bn):
        mu = h.mean(dim=1, keepdim=True)
        var = ((h - mu) ** 2).mean(dim=1, keepdim=True)
        xh = (h - mu) / torch.sqrt(var + 1e-6)
        y = p[gn][None, :, None, None] * xh + p[bn][None, :, None, None]
        lns[gn] = (xh.detach(), y)
        return y

    with torch.enable_grad(), torch.backends.cudnn.flags(enabled=True, deterministic=True, benchmark=False):
        spins = (1.0 - 2.0 * bits).reshape(B, 1, L, L).requires_grad_(True)  # graph root
        h = conv(spins, "w0", "b0")
        for i in range(n_res):
            u = tf.gelu(ln(h, f"g{i}", f"be{i}"), approximate="tanh")
            v = tf.gelu(conv(u, f"w{i}a", f"b{i}a"), approximate="tanh")
            h = h + conv(v, f"w{i}b", f"b{i}b")
        total = ln(h, "gf", "bef").sum()
        outs = [convs[k_][1] for k_ in convs] + [lns[k_][1] for k_ in lns]
        grads = torch.autograd.grad(total, outs)
    go = dict(zip(list(convs) + list(lns), grads))
    o = torch.empty((B, n_params(n_res)), dtype=torch.float64, device=dev)
    k = 0
    for name, shape in param_layout(n_res):
        size = int(np.prod(shape))
        dst = o[:, k:k + size]
        if name.startswith("w"):
            hp, _ = convs[name]
            cin = hp.shape[1]                                  # 3x3 neighbourhoods as a strided view, one copy
            unf = hp.detach().unfold(2, 3, 1).unfold(3, 3, 1).permute(0, 1, 4, 5, 2, 3).reshape(B, cin * 9, L * L)
            g = go[name].reshape(B, F, L * L)                  # (B, Cout, L * L)
            dst.copy_(torch.bmm(g, unf.transpose(1, 2)).reshape(B, size))
        elif name.startswith("b") and not name.startswith("be"):
            dst.copy_(go["w" + name[1:]].sum(dim=(2, 3)))      # conv bias: site sum
        elif name.startswith("g"):
            xh, _ = lns[name]
            dst.copy_((go[name] * xh).sum(dim=(2, 3)))         # LN gain
        else:                                                  # LN shift be{i} / bef
            gname = "g" + name[2:] if name != "bef" else "gf"
            dst.copy_(go[gname].sum(dim=(2, 3)))
        k += size
    return o


def _log_derivatives_vmap(params: ResCnnParameters, packed, chunk: int = 1024):
    """Per-sample autograd (torch.func vmap(grad)): the test reference of log_derivatives."""
    import torch
    from torch.func import grad, vmap

    dev = packed.device
    L, n = params.L, params.n_visible
    sites = torch.arange(n, device=dev)
    bits = ((packed.view(torch.int32)[:, sites // 32] >> (sites % 32)) & 1).to(torch.float64)
    spins = (1.0 - 2.0 * bits).reshape(-1, L, L)
    theta = torch.from_numpy(params.theta).to(dev)
    one = lambda th, s: torch_log_psi(th, s[None], L, params.n_res)[0]  # noqa: E731
    g = vmap(grad(one), in_dims=(None, 0), chunk_size=chunk)
    with torch.backends.cudnn.flags(enabled=True, deterministic=True, benchmark=False):
        return g(theta, spins)  # reproducible training runs


@dataclass
class CnnTrainConfig:
    hamiltonian: object
    n_res: int = 4
    n_steps: int = 100
    n_samples: int = 4096
    n_chains: int | None = None
    eta: float = 0.01
    lambda_shift: float = 1e-3
    seed: int = 0
    sampling_format: FloatFormat = None
    proposal: object = None
    burn_in_sweeps: int = 20
    reburn_sweeps: int = 2
    init_scale: float = 0.5
    minsr_precision: str = "f32"


def minsr_dense(o, eps, w, lam: float, precision: str = "f32", group=None, sharded: bool = False):
    """Sample-space SR step for a real dense O (U, P) shard: K = O~ O~^T + lam
    with O~ = W^1/2 (O - obar), e~ = W^1/2 (eps - ebar); g = O~^T K^-1 e~
    (push-through identity; the reference's parameter-space estimators,
    vmc.py:145-229).  Across ranks the O~ rows are all-gathered and every rank
    solves the same U_total x U_total system; O~^T y sums per rank."""
    import torch

    from . import parallel
    from .vmc import _gather_rows

    red = (lambda z: parallel.all_reduce_sum(z, group)) if sharded else (lambda z: z)
    s = red(torch.cat([(w[:, None] * o).sum(0), (w * eps).sum().reshape(1)]))
    obar, ebar = s[:-1], s[-1]
    sw = torch.sqrt(w)
    ot = sw[:, None] * (o - obar[None, :])
    et = sw * (eps - ebar)
    f = red(ot.T @ et)
    dt = torch.float32 if precision == "f32" else torch.float64
    if sharded:
        ot_all, row0 = _gather_rows(ot.to(dt).contiguous(), group)
        et_all, _ = _gather_rows(et.to(dt).contiguous(), group)
    else:
        ot_all, row0, et_all = ot.to(dt), 0, et.to(dt)
    k = ot_all @ ot_all.T
    if precision == "f32":
        # the f32 Gram matrix is PSD only to its rounding floor: the shift is
        # raised to 64 ulp of the largest diagonal entry when that exceeds lam
        lam = max(lam, 64.0 * 2.0**-24 * float(torch.diagonal(k).max()))
    k = 0.5 * (k + k.T) + lam * torch.eye(k.shape[0], dtype=dt, device=k.device)
    L_, info = torch.linalg.cholesky_ex(k)
    if int(info) != 0:
        from .errors import SolverError

        raise SolverError("minSR matrix is not positive definite")
    y = torch.cholesky_solve(et_all[:, None], L_)[:, 0]
    y = y + torch.cholesky_solve((et_all - k @ y)[:, None], L_)[:, 0]
    g = red(ot.T @ y[row0:row0 + ot.shape[0]].to(torch.float64))
    return g, f, float(ebar)


def train(config: CnnTrainConfig, device=None, group=None, local: bool = False):
    """VMC of the ResCNN (the reference's _train_loop structure, vmc.py:472-639):
    per step the f16/bf16 snapshot, re-burn, collect, unique samples + weights,
    f64 local energies, O, minSR, update; records energy, split-chain error,
    acceptance, sigma_hat (fmt vs f64 log p on the unique samples)."""
    import torch
    import torch.distributed as tdist

    from . import parallel
    from .bounds import pinsker_tv_bound, theorem3_gaussian_bound
    from .precision import F16
    from .rng import derive_key
    from .sampler import ChainEnsemble, Proposal, default_chain_count
    from .vmc import device_mc_error, device_std

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    world = tdist.get_world_size(group) if (not local and tdist.is_available() and tdist.is_initialized()) else 1
    rank = tdist.get_rank(group) if world > 1 else 0
    spec = config.hamiltonian
    if len(spec.lattice.shape) != 2 or spec.lattice.shape[0] != spec.lattice.shape[1]:
        raise ValueError("the ResCNN needs a square L x L lattice")
    L = spec.lattice.shape[0]
    n = L * L
    fmt = config.sampling_format or F16
    proposal = config.proposal or Proposal("flip")
    params = random_parameters(L, config.n_res, derive_key(config.seed, "init"), config.init_scale)
    n_chains = config.n_chains or default_chain_count(config.n_samples)
    c_off, c_cnt = parallel.shard(n_chains, rank, world)
    grp = group if world > 1 else None
    ensemble = None
    records = []
    for step in range(config.n_steps):
        ev = log_prob_evaluator(params, fmt, dev)
        if ensemble is None:
            ensemble = ChainEnsemble(c_cnt, n, proposal, ev, derive_key(config.seed, "chains"), chain_offset=c_off,
                                     n_chains_total=n_chains)
            ensemble.run_sweeps(config.burn_in_sweeps)
        else:
            ensemble.set_evaluator(ev, check=False)
            ensemble.run_sweeps(config.reburn_sweeps, check=False)
        ensemble.reset_counters()
        packed = ensemble.collect_packed(config.n_samples, n + 1)
        acc = torch.tensor([float(ensemble.accepted), float(ensemble.proposed)], dtype=torch.float64, device=dev)
        if world > 1:
            parallel.all_reduce_sum(acc, grp)
        uniq, inverse, cnt = torch.unique(packed, dim=0, return_inverse=True, return_counts=True)
        w = cnt.to(torch.float64) / config.n_samples
        eps = local_energies_packed(spec, params, uniq).real
        o = log_derivatives(params, uniq)
        g, _, energy = minsr_dense(o, eps, w, config.lambda_shift, config.minsr_precision, grp, world > 1)
        if world > 1:
            counts = parallel.chain_counts(config.n_samples, n_chains, c_off, c_cnt)
            err = parallel.energy_statistics(eps[inverse], counts, 0, 1, grp)["mc_error"]
        else:
            err = device_mc_error(torch.complex(eps, torch.zeros_like(eps)), inverse, config.n_samples, n_chains)
        lp_fmt, _ = ev.log_prob_packed(uniq)
        delta = lp_fmt - 2.0 * log_psi_packed(params, uniq, dev)
        sigma_hat = device_std(delta) if delta.numel() > 1 else 0.0
        records.append({"step": step, "energy": energy, "mc_error": err, "acceptance": float(acc[0] / acc[1]),
                        "sigma_hat": sigma_hat, "bound_pinsker": pinsker_tv_bound(sigma_hat),
                        "bound_theorem3": theorem3_gaussian_bound(sigma_hat, 0.0, 0.0)})
        params = ResCnnParameters(params.theta - config.eta * g.cpu().numpy(), L, config.n_res)
    return records, params
