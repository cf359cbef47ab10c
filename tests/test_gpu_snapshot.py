"""Device-built parameter snapshots (mpv_snapshot_round / mpv_snapshot_fill)
against a numpy construction of the same kernel layout from the host rounding
(ref: rbm.py:91-101 round_parameters; layout: include/mpvmc_b200.h mpv_snapshot)."""
import numpy as np
import pytest

from paper_2601_20782_b200 import _native as nat
from paper_2601_20782_b200 import rbm
from paper_2601_20782_b200.precision import BF16, F16, F32, F64, RoundingMode
from paper_2601_20782_b200.rng import derive_key

pytestmark = pytest.mark.gpu


def _half_bits(x, fmt):
    if fmt == "f16":
        return x.astype(np.float16).view(np.uint16)
    return (x.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def _pairs(re, im, fmt):
    if fmt == "f32":
        out = np.empty(re.shape + (2,), dtype=np.float32)
        out[..., 0], out[..., 1] = re, im
        return out
    return _half_bits(re, fmt).astype(np.uint32) | (_half_bits(im, fmt).astype(np.uint32) << np.uint32(16))


def _pad16(b):
    return b + b"\0" * ((-len(b)) % 16)


def host_layout(snap, fmt, mode, variant, G, U, plan):
    """numpy restatement of the kernel layout: ([table | vis] bytes, bias bytes, vis_im)."""
    N, M = snap.n_visible, snap.n_hidden
    wt = snap.w.T
    f64 = fmt.name == "f64" or mode is RoundingMode.STORAGE_ONLY
    Mpad = M if (mode is RoundingMode.PER_OPERATION and not f64) else G * U
    wpad = np.zeros((N, Mpad), dtype=np.complex128)
    wpad[:, :M] = wt
    bpad = np.zeros(Mpad, dtype=np.complex128)
    bpad[:M] = snap.b
    if f64 or variant == nat.ACC_F64:
        table = np.stack([wpad.real, wpad.imag], -1)
        bias = np.stack([bpad.real, bpad.imag], -1)
        vis = snap.a.real.astype(np.float64)
    elif variant == nat.ACC_X1:
        table, bias = _pairs(wpad.real, wpad.imag, fmt.name), _pairs(bpad.real, bpad.imag, fmt.name)
        vis = snap.a.real.astype(np.float32)
    elif variant == nat.ACC_XI:
        q = plan.quantum
        ints = lambda x: np.rint(x / q).astype(np.int32)
        table = np.stack([ints(wpad.real), ints(wpad.imag)], -1)
        bias = np.stack([ints(bpad.real), ints(bpad.imag)], -1)
        vis = ints(snap.a.real)
    else:
        g = plan.split

        def split(x):
            hi = np.rint(x / g) * g
            return hi, x - hi

        (whr, wlr), (whi, wli) = split(wpad.real), split(wpad.imag)
        (bhr, blr), (bhi, bli) = split(bpad.real), split(bpad.imag)
        ahi, alo = split(snap.a.real)
        th, tl = _pairs(whr, whi, fmt.name), _pairs(wlr, wli, fmt.name)
        bh, bl = _pairs(bhr, bhi, fmt.name), _pairs(blr, bli, fmt.name)
        ax = -2 if fmt.name == "f32" else -1
        table, bias = np.stack([th, tl], ax), np.stack([bh, bl], ax)
        vis = np.stack([ahi, alo], -1).astype(np.float32)
    blob = _pad16(np.ascontiguousarray(table).tobytes()) + _pad16(np.ascontiguousarray(vis).tobytes())
    return blob, _pad16(np.ascontiguousarray(bias).tobytes()), snap.a.imag.astype(np.float64)


CASES = [(12, 2, 0.3), (10, 1, 0.01), (20, 2, 1.5), (16, 4, 0.05)]
MODES = [(F16, RoundingMode.NATIVE), (BF16, RoundingMode.NATIVE), (F32, RoundingMode.NATIVE),
         (F16, RoundingMode.PER_OPERATION), (BF16, RoundingMode.PER_OPERATION), (F32, RoundingMode.PER_OPERATION),
         (F16, RoundingMode.STORAGE_ONLY), (F64, RoundingMode.PER_OPERATION)]


@pytest.mark.parametrize("n,alpha,scale", CASES)
@pytest.mark.parametrize("fmt,mode", MODES, ids=lambda v: getattr(v, "name", None) or getattr(v, "value", str(v)))
def test_device_snapshot_matches_host_layout(cuda, n, alpha, scale, fmt, mode):
    p = rbm.random_parameters(n, alpha, derive_key(n, "snapshot"), scale)
    snap_host = rbm.round_parameters(p, fmt)
    variants = [None]
    if mode is RoundingMode.NATIVE:
        variants = [nat.ACC_X1, nat.ACC_XI, nat.ACC_X2, nat.ACC_F64]
    for variant in variants:
        try:
            dev = rbm.DeviceSnapshot(p, fmt, mode, variant=variant)
        except ValueError:
            continue  # variant not exact for this snapshot
        rounded = dev.params
        for x, y in ((rounded.a, snap_host.a), (rounded.b, snap_host.b), (rounded.w, snap_host.w)):
            np.testing.assert_array_equal(x.view(np.float64), y.view(np.float64))
        plan = (rbm.plan_exact(snap_host, allow_xi=fmt.name in ("f16", "bf16"))
                if mode is RoundingMode.NATIVE and fmt.name != "f64" else None)
        if plan is not None:
            assert dev.plan == plan
        blob, bias, vis_im = host_layout(snap_host, fmt, mode, dev.variant, dev.lanes_per_chain,
                                         dev.units_per_lane, plan)
        assert dev._table.cpu().numpy().tobytes() == blob, dev.label
        assert dev._bias.cpu().numpy().tobytes() == bias, dev.label
        np.testing.assert_array_equal(dev._vis_im.cpu().numpy(), vis_im)


def test_device_rounding_edge_values(cuda):
    """RNE ties, subnormals, largest finite values: device rounding == host rounding
    (overflow to inf is rejected by RbmParameters on both sides)."""
    base = [65504.0, 65519.99, 2.0**-24, 2.0**-25, 3 * 2.0**-26, 1 + 2.0**-11, 1 + 3 * 2.0**-11, 1e-40, -0.0,
            1 / 3, np.pi, -2.5e-6]
    wide = base + [1e6, -1e6, 3.3895313892515355e38, 1 + 2.0**-8, 1 + 3 * 2.0**-8, 1 + 2.0**-24]
    for fmt, vals in ((F16, base), (BF16, wide), (F32, wide)):
        vals = np.array(vals)
        p = rbm.RbmParameters(vals + 1j * vals[::-1], np.array([0.5 + 0.25j]), vals[None, :] * (1 - 1j))
        dev = rbm.DeviceSnapshot(p, fmt, RoundingMode.PER_OPERATION)
        host = rbm.round_parameters(p, fmt)
        got = dev.params
        for x, y in ((got.a, host.a), (got.b, host.b), (got.w, host.w)):
            np.testing.assert_array_equal(x.view(np.float64), y.view(np.float64))
