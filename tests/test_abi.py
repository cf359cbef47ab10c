"""The C ABI (include/mpvmc_b200.h) and the built sm_100a library, without a GPU:
the library loads, exports every declared symbol, its ctypes mirror has the
header's struct layout, and host-only entry points validate arguments."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2601_20782_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpvmc_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mpv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(nat.EXPORTED) == syms
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (mpv_\w+)", out)))
    assert exported == syms  # nothing else leaks from the library


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "mpvmc_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(mpv_snapshot), '
                   'offsetof(mpv_snapshot, table), offsetof(mpv_snapshot, vis_im), sizeof(mpv_chains), '
                   'offsetof(mpv_chains, bits), offsetof(mpv_chains, scratch_bytes));return 0;}\n')
    exe = tmp_path / "layout"
    gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(nat.Snapshot), nat.Snapshot.table.offset, nat.Snapshot.vis_im.offset,
            ctypes.sizeof(nat.Chains), nat.Chains.bits.offset, nat.Chains.scratch_bytes.offset]
    assert got == want


def test_plan_layout():
    x1 = dict(fmt=nat.FMT_F16, variant=nat.ACC_X1)
    x2 = dict(fmt=nat.FMT_F16, variant=nat.ACC_X2)
    assert nat.plan_layout(100, 100, **x1) == (4, 25)
    assert nat.plan_layout(100, 200, **x1) == (8, 25)
    assert nat.plan_layout(20, 20, **x1) == (1, 20)
    assert nat.plan_layout(100, 100, **x2) == (8, 13)
    assert nat.plan_layout(100, 200, **x2) == (16, 13)
    assert nat.plan_layout(256, 256, **x2) == (16, 16)
    assert nat.plan_layout(100, 400, nat.FMT_F64, nat.ACC_F64) == (32, 13)
    for fmt, var in [(nat.FMT_F16, nat.ACC_X1), (nat.FMT_BF16, nat.ACC_X2), (nat.FMT_F32, nat.ACC_X1),
                     (nat.FMT_F32, nat.ACC_F64), (nat.FMT_F64, nat.ACC_F64)]:
        for n, m in [(100, 8), (256, 16), (12, 24), (64, 3), (1024, 256), (100, 400)]:
            g, u = nat.plan_layout(n, m, fmt, var)
            assert g * u >= m and g >= (n + 31) // 32 and 32 % g == 0
    with pytest.raises(ValueError):
        nat.plan_layout(100, 10_000)


def test_argument_validation_without_gpu():
    lib = nat.load()
    assert lib.mpv_mh_sweep(None, None, 0, 0, 0, 0, 0, 0, None, 0, 0, 0, 0, None) == nat.MPV_ERR_ARGS
    assert b"null" in lib.mpv_last_error()
    assert lib.mpv_local_energies(0, 0, None, None, None, 0, None, 0, 0.0, 0.0, None, None, 0, None, None,
                                  None) == nat.MPV_ERR_ARGS
    assert lib.mpv_rounded_log_prob(None, 1, 4, 4, None, None, None, None, None, 0, None, None,
                                    None) == nat.MPV_ERR_ARGS
    assert b"sm_100a" in lib.mpv_version()


def test_product_has_no_cpu_fallback():
    """The product package must not import the oracle or any host evaluator."""
    pkg = os.path.join(ROOT, "paper_2601_20782_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            text = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in text.replace("oracle/", ""), fn
            assert "numba" not in text, fn


def test_forward_tc_layout_and_argument_checks():
    """Host-side contract of the tensor-core forward (no GPU needed): the
    weights blob size, the supported shapes, and the format check that fails
    before any launch."""
    lib = nat.load()
    n100 = lib.mpv_forward_tc_weights_bytes(100, 200)
    assert n100 > 0 and n100 % 256 == 0
    # B rows: (112 hidden + 16) per re/im block per chunk x Kp = 112 f16, two chunks, + a (re, im) f32
    assert n100 >= 2 * 2 * 128 * 112 * 2
    assert lib.mpv_forward_tc_weights_bytes(1, 1) > 0
    assert lib.mpv_forward_tc_weights_bytes(100, 400) > lib.mpv_forward_tc_weights_bytes(100, 200)
    assert lib.mpv_forward_tc_weights_bytes(2000, 10) == 0  # A tile beyond shared memory
    assert lib.mpv_forward_tc_weights_bytes(0, 10) == 0
    rc = lib.mpv_forward_tc_prepare(10, 10, nat.FMT_F32, ctypes.c_void_p(8), ctypes.c_void_p(8), None)
    assert rc == nat.MPV_ERR_ARGS and b"f16 or bf16" in lib.mpv_last_error()
    rc = lib.mpv_forward_tc(10, 10, nat.FMT_F16, ctypes.c_void_p(8), ctypes.c_void_p(8), 4, None, None, None, 0, None)
    assert rc == nat.MPV_ERR_ARGS  # no output requested
    assert lib.mpv_forward_tc(10, 10, nat.FMT_F16, ctypes.c_void_p(8), None, 0, None, None, None, 0, None) == nat.MPV_OK
