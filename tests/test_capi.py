"""CPU tests of the drop-in boundary: libmimw_b200.so builds, loads, exports
every entry point include/mimw_b200.h declares, and has no CPU fallback."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "mimw_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(mimw_b200_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import paper_2605_10905_b200 as P
    from paper_2605_10905_b200 import build
    build.build()
    return P.lib()


def test_header_declares_the_reference_replacements():
    names = _declared()
    for n in ("mimw_b200_oracle_gemm", "mimw_b200_oracle_multi_device_gemm",
              "mimw_b200_oracle_attention", "mimw_b200_gemm_bf16", "mimw_b200_attention_fwd",
              "mimw_b200_last_error", "mimw_b200_version"):
        assert n in names, n


def test_every_declared_symbol_is_exported(L):
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing


def test_sass_is_tcgen05_tma():
    import subprocess
    from paper_2605_10905_b200 import build
    lib = build.build()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                          text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "UTCBAR"):
        assert mnem in sass, mnem
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(L):
    import paper_2605_10905_b200 as P
    a = np.ones((4, 8), np.float32)
    b = np.ones((8, 8), np.float32)
    with pytest.raises(P.MimwError) as e:
        P.oracle_gemm(a, b)
    assert e.value.code == P.ERR_CUDA
    assert b"no sm_100" in L.mimw_b200_last_error() or b"CUDA" in L.mimw_b200_last_error().upper()


def test_shape_errors_are_reported(L):
    import paper_2605_10905_b200 as P
    with pytest.raises(P.MimwError) as e:
        P.oracle_gemm(np.ones((4, 8), np.float32), np.ones((7, 8), np.float32))
    assert e.value.code == P.ERR_SHAPE


def test_bad_enum_is_arg_error(L):
    r = L.mimw_b200_gemm_bf16(None, None, None, 4, 4, 4, 4, 4, 4, 7, 0, None)
    assert r == 4
    assert b"b_layout" in L.mimw_b200_last_error()


def test_grouped_gemm_argument_errors(L):
    """Shape / argument validation happens before any device work."""
    import ctypes
    offs = (ctypes.c_int64 * 3)(0, 5, 3)  # decreasing
    r = L.mimw_b200_grouped_gemm_bf16(None, offs, None, None, 2, 64, 64, 0, None)
    assert r == 1 and b"non-decreasing" in L.mimw_b200_last_error()
    offs = (ctypes.c_int64 * 3)(0, 5, 9)
    r = L.mimw_b200_grouped_gemm_bf16(None, offs, None, None, 2, 64, 64, 9, None)
    assert r == 4
    r = L.mimw_b200_grouped_gemm_bf16(None, None, None, None, 2, 64, 64, 0, None)
    assert r == 4


def test_oracle_grouped_gemm_is_per_group_oracle_gemm():
    import oracle
    offs = [0, 3, 3, 8]
    x = oracle.random_tile([8, 16], 1)
    w = oracle.random_tile([3, 16, 24], 2)
    ys = oracle.oracle_grouped_gemm(x, offs, w)
    assert ys[1].shape == (0, 24)
    np.testing.assert_array_equal(ys[2], oracle.oracle_gemm(x[3:8], w[2]))


def test_tile_and_variant_selectors_are_validated(L):
    """The tuning hooks reject tile / variant selectors they do not implement
    before touching any device state (no GPU needed): dense and grouped
    tile_n, grouped swap_tails, attention cta_group."""
    import paper_2605_10905_b200 as P
    nul = None
    offs = np.array([0, 4], np.int64)
    r = L.mimw_b200_gemm_bf16_ex(nul, nul, nul, 64, 64, 64, 64, 64, 64, 0, 1, 2, 0, 0, 384, nul)
    assert r == P.ERR_ARG and b"tile_n" in L.mimw_b200_last_error()
    r = L.mimw_b200_gemm_bf16_ex(nul, nul, nul, 64, 64, 64, 64, 64, 64, 0, 0, 2, 0, 0, 512, nul)  # f32 out
    assert r == P.ERR_ARG
    r = L.mimw_b200_grouped_gemm_bf16_ex(nul, offs.ctypes.data, nul, nul, 1, 512, 64, 0, 1, 0, -1, 512, nul)
    assert r == P.ERR_ARG and b"tile_n" in L.mimw_b200_last_error()  # 512-wide needs cta_group 2
    r = L.mimw_b200_grouped_gemm_bf16_ex(nul, offs.ctypes.data, nul, nul, 1, 512, 64, 0, 2, 0, 2, 0, nul)
    assert r == P.ERR_ARG and b"swap_tails" in L.mimw_b200_last_error()
