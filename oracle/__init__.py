"""TEST INFRASTRUCTURE — the CPU oracle (checker) for the B200 hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  The product package ``paper_2605_10905_b200`` never
imports it and has no CPU fallback.

Two ctypes-loaded libraries, both built by ``oracle/Makefile``:

* ``C``   — ``liboracle.so``: the plain-C restatement (``oracle.c``), each
  function citing the reference lines it restates.
* ``REF`` — ``_ref/libmimw_ref.so``: the UNMODIFIED reference sources
  (``/root/reference/proj/core/src/{oracles,case,tensor_io}.cpp``) compiled
  with a thin extern "C" shim (``ref_shim.cpp``).  ``None`` when not built.

The numpy-level helpers below mirror the reference signatures
(``core/include/mimw/oracles.hpp``): inputs are float32 row-major arrays.
"""
from __future__ import annotations

import ctypes as C_
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64 = C_.c_int64


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (+ _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _load(path):
    return C_.CDLL(path) if os.path.exists(path) else None


def _declare_c(lib):
    lib.orc_random_tile.argtypes = [_i64, C_.c_uint64, _f32p]
    lib.orc_input_seed.argtypes = [C_.c_uint64, C_.c_uint64]
    lib.orc_input_seed.restype = C_.c_uint64
    lib.orc_rel_error.argtypes = [_f32p, _f32p, _i64]
    lib.orc_rel_error.restype = C_.c_double
    lib.orc_rel_error_rows.argtypes = [_f32p, _f32p, _i64, _i64]
    lib.orc_rel_error_rows.restype = C_.c_double
    lib.orc_round_bf16_n.argtypes = [_f32p, _f32p, _i64]
    lib.orc_mx_dequant.argtypes = [_u8p, _u8p, _f32p, _i64, _i64]
    lib.orc_gemm.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, _i64]
    lib.orc_gemm_rows.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, _i64, _i64, _i64]
    lib.orc_multi_device_gemm.argtypes = [_f32p] * 5 + [_i64] * 4
    lib.orc_gemm_rowlist_mt.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, _i64, C_.c_int]
    lib.orc_attention_rowlist_mt.argtypes = [_f32p, _f32p, _f32p, _f32p, C_.c_void_p, _i64, _i64, _i64,
                                             C_.c_int, C_.c_double,
                                             np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"),
                                             _i64, C_.c_int]
    lib.orc_attention.argtypes = [_f32p, _f32p, _f32p, _f32p, C_.c_void_p,
                                  _i64, _i64, _i64, C_.c_double]
    lib.orc_attention_rows.argtypes = [_f32p, _f32p, _f32p, _f32p, C_.c_void_p,
                                       _i64, _i64, _i64, C_.c_double, _i64, _i64]
    lib.orc_simplicial_attention.argtypes = [_f32p] * 7 + [_i64] * 4 + [C_.c_double]
    lib.orc_attention_mode_rows.argtypes = [_f32p, _f32p, _f32p, _f32p, C_.c_void_p, _i64, _i64,
                                            _i64, C_.c_int, C_.c_double, _i64, _i64]
    lib.orc_attention_bwd.argtypes = [_f32p] * 7 + [_i64, _i64, _i64, C_.c_int, C_.c_double]
    lib.orc_layernorm.argtypes = [_f32p, _f32p, _f32p, C_.c_double, _f32p,
                                  _f32p, _f32p, _i64, _i64]
    lib.orc_write_tensor.argtypes = [C_.c_char_p, _f32p, C_.POINTER(_i64), C_.c_int]
    return lib


def _declare_ref(lib):
    lib.ref_random_tile.argtypes = [C_.POINTER(_i64), C_.c_int, C_.c_uint64, _f32p]
    lib.ref_rel_error.argtypes = [_f32p, _f32p, _i64]
    lib.ref_rel_error.restype = C_.c_double
    lib.ref_oracle_gemm.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, _i64]
    lib.ref_oracle_gemm_rows.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, _i64, _i64, _i64]
    lib.ref_oracle_gemm_mt.argtypes = [_f32p, _f32p, _f32p, _i64, _i64, _i64, C_.c_int]
    lib.ref_oracle_attention.argtypes = [_f32p] * 4 + [_i64, _i64, C_.c_int, C_.c_double]
    lib.ref_oracle_attention_heads_mt.argtypes = [_f32p] * 4 + [_i64, _i64, _i64, C_.c_int,
                                                              C_.c_double, C_.c_int]
    lib.ref_oracle_simplicial_attention.argtypes = [_f32p] * 7 + [_i64, _i64, C_.c_int,
                                                                C_.c_int, C_.c_double]
    lib.ref_oracle_multi_device_gemm.argtypes = [_f32p] * 5 + [_i64] * 4
    lib.ref_oracle_layernorm.argtypes = [_f32p, _f32p, _f32p, C_.c_double, _f32p, _f32p,
                                         _f32p, _i64, _i64]
    lib.ref_write_tensor.argtypes = [C_.c_char_p, _f32p, C_.POINTER(_i64), C_.c_int]
    return lib


def _libs():
    c = _load(os.path.join(HERE, "liboracle.so"))
    if c is None:
        build()
        c = _load(os.path.join(HERE, "liboracle.so"))
    r = _load(os.path.join(HERE, "_ref", "libmimw_ref.so"))
    return _declare_c(c), (_declare_ref(r) if r is not None else None)


C, REF = _libs()


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


# --------------------------------------------------------------------------
# seeded inputs / metric (tensor_io.cpp:80-88, case.cpp:82-104)
# --------------------------------------------------------------------------
def random_tile(shape, seed: int) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, np.float32)
    C.orc_random_tile(n, seed, out)
    return out.reshape(shape)


def input_seed(seed: int, k: int) -> int:
    return int(C.orc_input_seed(seed, k))


def make_inputs(shapes: dict, seed: int) -> dict:
    """``make_inputs`` (case.cpp:82-92): input k in declaration order gets
    ``random_tile(shape, seed*1000003 + k)``.  ``shapes`` is ordered."""
    return {name: random_tile(shape, input_seed(seed, k))
            for k, (name, shape) in enumerate(shapes.items())}


def rel_error(a, b) -> float:
    a, b = _f32(a), _f32(b)
    if a.shape != b.shape:
        return float("inf")
    return float(C.orc_rel_error(a.ravel(), b.ravel(), a.size))


def rel_error_rows(a, b) -> float:
    a, b = _f32(a), _f32(b)
    cols = a.shape[-1]
    return float(C.orc_rel_error_rows(a.ravel(), b.ravel(), a.size // cols, cols))


def round_bf16(x) -> np.ndarray:
    x = _f32(x)
    out = np.empty_like(x)
    C.orc_round_bf16_n(x.ravel(), out.ravel(), x.size)
    return out


def mx_dequant(q: np.ndarray, sf: np.ndarray) -> np.ndarray:
    rows, cols = q.shape
    out = np.empty((rows, cols), np.float32)
    C.orc_mx_dequant(np.ascontiguousarray(q, np.uint8), np.ascontiguousarray(sf, np.uint8),
                     out, rows, cols)
    return out


# --------------------------------------------------------------------------
# oracles (oracles.hpp:15-37)
# --------------------------------------------------------------------------
def oracle_gemm(a, b, rows=None) -> np.ndarray:
    """C = A.B (oracles.cpp:14-26); ``rows=(r0, r1)`` computes only those rows
    (exact: each c[i,j] depends only on A[i,:] and B[:,j])."""
    a, b = _f32(a), _f32(b)
    m, k = a.shape
    n = b.shape[1]
    if rows is None:
        c = np.empty((m, n), np.float32)
        C.orc_gemm(a, b, c, m, n, k)
        return c
    r0, r1 = rows
    full = np.zeros((m, n), np.float32)
    C.orc_gemm_rows(a, b, full, m, n, k, r0, r1)
    return full[r0:r1]


def oracle_gemm_rowlist(a_rows, b, threads: int | None = None) -> np.ndarray:
    """Rows of C = A.B given the gathered rows ``a_rows`` [R, K] of A and B
    [K, N]: the reference's arithmetic (oracles.cpp:17-23, float accumulator,
    ascending k) restated with a cache-friendly loop order and threads;
    bit-identical to oracle_gemm (tests/test_oracle.py)."""
    a, b = _f32(a_rows), _f32(b)
    r, k = a.shape
    n = b.shape[1]
    c = np.empty((r, n), np.float32)
    C.orc_gemm_rowlist_mt(a, b, c, r, n, k, threads or (os.cpu_count() or 1))
    return c


def oracle_attention_rowlist(q, k, v, w: int, scale: float, rows, causal: bool = True,
                             threads: int | None = None):
    """Sparse rows of one head's attention (oracles.cpp:119-145; causal=False:
    the restated every-key variant), threaded: returns (o[len(rows), D],
    lse[len(rows)])."""
    q, k, v = map(_f32, (q, k, v))
    s, d = q.shape
    rr = np.ascontiguousarray(np.asarray(rows, np.int64))
    o = np.empty((len(rr), d), np.float32)
    lse = np.empty(len(rr), np.float32)
    C.orc_attention_rowlist_mt(q, k, v, o, lse.ctypes.data, s, d, w, 1 if causal else 0, scale, rr, len(rr),
                               threads or (os.cpu_count() or 1))
    return o, lse


def oracle_grouped_gemm(x, m_offsets, w, rows=None) -> list:
    """Grouped (MoE) GEMM oracle: one ``oracle_gemm`` (oracles.cpp:14-26) per
    group, ``Y_e = X[off_e:off_e+1] . W_e`` with W as [G, K, N].  The
    reference has no grouped GEMM (parity anchored on
    oracle_gemm).  ``rows`` = optional {e: (r0, r1)} row ranges (exact)."""
    out = []
    for e in range(len(m_offsets) - 1):
        xe = x[m_offsets[e]:m_offsets[e + 1]]
        if rows is not None:
            if e not in rows:
                out.append(None)
                continue
            out.append(oracle_gemm(xe, w[e], rows=rows[e]))
        else:
            out.append(oracle_gemm(xe, w[e]) if len(xe) else np.zeros((0, w.shape[2]), np.float32))
    return out


def oracle_multi_device_gemm(a0, a1, b0, b1) -> np.ndarray:
    a0, a1, b0, b1 = map(_f32, (a0, a1, b0, b1))
    m, k0 = a0.shape
    k1, n = a1.shape[1], b0.shape[1]
    c = np.empty((m, n), np.float32)
    C.orc_multi_device_gemm(a0, a1, b0, b1, c, m, k0, k1, n)
    return c


def oracle_attention(q, k, v, w: int, scale: float, with_lse: bool = False):
    """Windowed causal attention for one head [S, D] (oracles.cpp:119-145)."""
    q, k, v = map(_f32, (q, k, v))
    s, d = q.shape
    o = np.empty((s, d), np.float32)
    lse = np.empty(s, np.float32) if with_lse else None
    C.orc_attention(q, k, v, o, lse.ctypes.data if with_lse else None, s, d, w, scale)
    return (o, lse) if with_lse else o


def oracle_attention_rows(q, k, v, w: int, scale: float, r0: int, r1: int):
    """Rows [r0, r1) of oracle_attention (exact: rows are independent in
    oracles.cpp:123-144).  Returns (o[r1-r0, D], lse[r1-r0])."""
    q, k, v = map(_f32, (q, k, v))
    s, d = q.shape
    o = np.empty((r1 - r0, d), np.float32)
    lse = np.empty(r1 - r0, np.float32)
    C.orc_attention_rows(q, k, v, o, lse.ctypes.data, s, d, w, scale, r0, r1)
    return o, lse


def oracle_attention_full(q, k, v, scale: float, rows=None):
    """NON-CAUSAL attention of one head (every key; no reference oracle —
    restated from oracles.cpp:119-145 with the key range widened, see
    oracle.c key_range).  ``rows=(r0, r1)`` computes only those rows.
    Returns (o, lse)."""
    q, k, v = map(_f32, (q, k, v))
    s, d = q.shape
    r0, r1 = rows if rows is not None else (0, s)
    o = np.empty((r1 - r0, d), np.float32)
    lse = np.empty(r1 - r0, np.float32)
    C.orc_attention_mode_rows(q, k, v, o, lse.ctypes.data, s, d, s, 0, scale, r0, r1)
    return o, lse


def oracle_attention_bwd(q, k, v, do, scale: float, causal: bool = True, w: int | None = None):
    """Gradients (dq, dk, dv) of one [S, D] head of attention (causal with
    window ``w`` as oracle_attention, or non-causal), evaluated in f64 —
    a restatement: the reference has no backward (oracle.c orc_attention_bwd)."""
    q, k, v, do = map(_f32, (q, k, v, do))
    s, d = q.shape
    dq, dk, dv = (np.empty((s, d), np.float32) for _ in range(3))
    C.orc_attention_bwd(q, k, v, do, dq, dk, dv, s, d, w if w is not None else s,
                        1 if causal else 0, scale)
    return dq, dk, dv


def oracle_simplicial_attention(q, k1, v1, k2, v2, w1: int, w2: int, scale: float):
    q, k1, v1, k2, v2 = map(_f32, (q, k1, v1, k2, v2))
    s, d = q.shape
    o = np.empty((s, d), np.float32)
    lse = np.empty(s, np.float32)
    C.orc_simplicial_attention(q, k1, v1, k2, v2, o, lse, s, d, w1, w2, scale)
    return o, lse


def oracle_simplicial_rows(q, k1, v1, k2, v2, w1: int, w2: int, scale: float, rows):
    """Selected rows of oracle_simplicial_attention (oracles.cpp:82-117), in
    float64 numpy (rows are independent, so this is exact oracle semantics for
    those rows): returns (o[len(rows), D], lse[len(rows)])."""
    q, k1, v1, k2, v2 = (np.asarray(t, np.float64) for t in (q, k1, v1, k2, v2))
    out_o, out_l = [], []
    for i in rows:
        j1 = np.arange(max(0, i - w1 + 1), i + 1)
        j2 = np.arange(max(0, i - w2 + 1), i + 1)
        s = ((q[i] * k1[j1]) @ k2[j2].T) * scale          # [|j1|, |j2|]
        m = s.max()
        e = np.exp(s - m)
        l_ = e.sum()
        p = e / l_
        o = (p[:, :, None] * v1[j1][:, None, :] * v2[j2][None, :, :]).sum(axis=(0, 1))
        out_o.append(o.astype(np.float32))
        out_l.append(np.float32(m + np.log(l_)))
    return np.stack(out_o), np.array(out_l, np.float32)


def oracle_layernorm(x, w, b, eps: float):
    x, w, b = map(_f32, (x, w, b))
    rows, n = x.shape
    y = np.empty_like(x)
    mean = np.empty(rows, np.float32)
    rstd = np.empty(rows, np.float32)
    C.orc_layernorm(x, w, b, eps, y, mean, rstd, rows, n)
    return y, mean, rstd


# --------------------------------------------------------------------------
# MIMWTNSR golden files (tensor_io.cpp:10, 30-78)
# --------------------------------------------------------------------------
def read_tensor(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:8] != b"MIMWTNSR":
        raise ValueError(f"{path}: bad magic")
    rank = int.from_bytes(raw[8:12], "little")
    shape = [int.from_bytes(raw[12 + 4 * i:16 + 4 * i], "little") for i in range(rank)]
    off = 12 + 4 * rank
    return np.frombuffer(raw[off:], dtype="<f4").reshape(shape).astype(np.float32)


def write_tensor(path: str, x) -> None:
    x = _f32(x)
    shape = (_i64 * max(1, x.ndim))(*x.shape)
    if C.orc_write_tensor(path.encode(), x.ravel(), shape, x.ndim) != 0:
        raise OSError(path)
