"""B200-native (sm_100a) hot path of arXiv 2605.10905 (TLX / MIMW).

Host-side mirror of the reference's operator API
(/root/reference/proj/core/include/mimw/oracles.hpp) over the C-ABI library
``libmimw_b200.so`` (include/mimw_b200.h):

* ``oracle_gemm(a, b)``, ``oracle_multi_device_gemm(a0, a1, b0, b1)``,
  ``oracle_attention(q, k, v, w, scale)``, ``run_oracle(name, inputs,
  scalars)`` take/return float32 numpy arrays exactly like the reference
  functions take/return ``Tile`` — same names, same argument meaning.
  ``run_oracle`` returns ``None`` for an unknown name and raises ``KeyError``
  for a missing input, as the reference does (oracles.cpp:147-201).
* ``gemm(...)``, ``attention_fwd(...)`` etc. take CUDA torch tensors (device
  pointers; torch is plumbing only) and launch on the current stream.

There is NO CPU fallback: importing works anywhere, but every compute call
raises ``MimwError`` if the library is missing or no B200 is visible.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# MIMW_B200_LIB: load another build of the library (A/B timing of two builds)
LIB_PATH = os.environ.get("MIMW_B200_LIB") or os.path.join(PKG, "libmimw_b200.so")

OK, ERR_SHAPE, ERR_UNSUPPORTED, ERR_CUDA, ERR_ARG = 0, 1, 2, 3, 4
F32, BF16 = 0, 1
B_KN, B_NK = 0, 1
PREC_BF16, PREC_F32_BF16X3, PREC_F32 = 0, 1, 2

_i64 = C.c_int64
_vp = C.c_void_p
_fp = C.POINTER(C.c_float)


class MimwError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[mimw status {code}] {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load libmimw_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MimwError(ERR_CUDA, f"{LIB_PATH} missing: run `python -m paper_2605_10905_b200.build`"
                                      " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.mimw_b200_last_error.restype = C.c_char_p
        L.mimw_b200_version.restype = C.c_int
        L.mimw_b200_oracle_gemm.argtypes = [_fp, _fp, _fp, _i64, _i64, _i64, C.c_int32]
        L.mimw_b200_oracle_multi_device_gemm.argtypes = [_fp] * 5 + [_i64] * 4 + [C.c_int32]
        L.mimw_b200_gemm_bf16.argtypes = [_vp, _vp, _vp] + [_i64] * 6 + [C.c_int32, C.c_int32, _vp]
        L.mimw_b200_gemm_bf16_ex.argtypes = ([_vp, _vp, _vp] + [_i64] * 6 +
                                             [C.c_int32] * 6 + [_vp])
        for name, types in _optional_sigs().items():
            if hasattr(L, name):
                getattr(L, name).argtypes = types
        _lib = L
    return _lib


def _optional_sigs():
    return {
        "mimw_b200_oracle_attention": [_fp, _fp, _fp, _fp, _fp, _i64, _i64, _i64, C.c_double],
        "mimw_b200_oracle_attention_ex": [_fp, _fp, _fp, _fp, _fp, _i64, _i64, _i64, C.c_double,
                                          C.c_int32],
        "mimw_b200_oracle_attention_heads": [_fp, _fp, _fp, _fp, _fp, _i64, _i64, _i64, _i64,
                                             C.c_double, C.c_int32],
        "mimw_b200_trim_pool": [],
        "mimw_b200_oracle_simplicial_attention_ex": [_fp] * 7 + [_i64] * 4 + [C.c_double, C.c_int32],
        "mimw_b200_attention_fwd": [_vp, _vp, _vp, _vp, _vp] + [_i64] * 5 + [C.c_double, _vp],
        "mimw_b200_attention_bwd": [_vp] * 5 + [_vp] + [_vp] * 3 + [_i64] * 5 + [C.c_double, _vp],
        "mimw_b200_attention_fwd_ex": [_vp, _vp, _vp, _vp, _vp] + [_i64] * 4 + [C.c_double, C.c_int32,
                                                                           C.c_int32, _vp, C.c_int32, _vp],
        "mimw_b200_gemm_mxfp8": [_vp] * 5 + [_i64] * 3 + [_vp],
        "mimw_b200_oracle_simplicial_attention": [_fp] * 7 + [_i64] * 4 + [C.c_double],
        "mimw_b200_simplicial_attention_fwd": [_vp] * 6 + [_vp] + [_i64] * 5 + [C.c_double, _vp],
        "mimw_b200_oracle_layernorm": [_fp, _fp, _fp, C.c_double, _fp, _fp, _fp, _i64, _i64],
        "mimw_b200_layernorm": [_vp] * 6 + [_i64, _i64, C.c_double, _vp],
        "mimw_b200_layernorm_ex": [_vp] * 6 + [_i64, _i64, C.c_double, C.c_int32, _vp],
        "mimw_b200_gemm_mxfp8_ex": [_vp] * 5 + [_i64] * 3 + [C.c_int32, _vp],
        "mimw_b200_grouped_gemm_bf16": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, C.c_int32, _vp],
        "mimw_b200_grouped_gemm_bf16_ex": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, C.c_int32,
                                           C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp],
    }


def _check(status: int) -> None:
    if status != OK:
        raise MimwError(status, lib().mimw_b200_last_error().decode(errors="replace"))


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32)


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(_fp)


# ---------------------------------------------------------------------------
# reference-signature mirror (host f32 "Tiles")
# ---------------------------------------------------------------------------
def oracle_gemm(a, b, precision: int = PREC_BF16) -> np.ndarray:
    """``Tile oracle_gemm(const Tile &a, const Tile &b)`` (oracles.hpp:15-16)
    on B200 tensor cores.  ``precision=PREC_F32_BF16X3`` meets the reference's
    own f32 tolerance (1e-4); the default rounds inputs to bf16 (north-star
    tolerance 1e-2)."""
    a, b = _f32(a), _f32(b)
    m, k = a.shape
    k2, n = b.shape
    if k2 != k:
        raise MimwError(ERR_SHAPE, f"dot conformance: a.shape[1]={k} != b.shape[0]={k2}")
    c = np.empty((m, n), np.float32)
    _check(lib().mimw_b200_oracle_gemm(_ptr(a), _ptr(b), _ptr(c), m, n, k, precision))
    return c


def oracle_multi_device_gemm(a0, a1, b0, b1, precision: int = PREC_BF16) -> np.ndarray:
    """``oracle_multi_device_gemm`` (oracles.hpp:24-25): [a0 | a1] . [b0 ; b1]."""
    a0, a1, b0, b1 = map(_f32, (a0, a1, b0, b1))
    m, k0 = a0.shape
    k1, n = a1.shape[1], b0.shape[1]
    if a1.shape[0] != m or b0.shape[0] != k0 or b1.shape != (k1, n):
        raise MimwError(ERR_SHAPE, "multi_device_gemm: inconsistent shapes")
    c = np.empty((m, n), np.float32)
    _check(lib().mimw_b200_oracle_multi_device_gemm(_ptr(a0), _ptr(a1), _ptr(b0), _ptr(b1),
                                                     _ptr(c), m, k0, k1, n, precision))
    return c


def oracle_attention(q, k, v, w: int, scale: float, with_lse: bool = False,
                     precision: int = PREC_BF16):
    """``void oracle_attention(q, k, v, int w, double scale, Tile *o)``
    (oracles.hpp:35-37): windowed causal softmax attention of one [S, D] head.
    ``precision=PREC_F32_BF16X3`` holds the reference's own 1e-4 on the
    tcgen05 tensor cores (split-bf16 x3 scores and P.V, f32 softmax);
    ``PREC_F32`` does with the oracle's f64 arithmetic on CUDA cores; the
    default is the fused bf16 tcgen05 kernel (1e-2)."""
    L = lib()
    if not hasattr(L, "mimw_b200_oracle_attention"):
        raise MimwError(ERR_UNSUPPORTED, "attention not built")
    q, k, v = map(_f32, (q, k, v))
    if q.ndim != 2 or k.shape != q.shape or v.shape != q.shape:
        raise MimwError(ERR_SHAPE, "q, k, v must be [S, D] of one shape")
    s, d = q.shape
    o = np.empty((s, d), np.float32)
    lse = np.empty(s, np.float32)
    _check(L.mimw_b200_oracle_attention_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), s, d, w,
                                           scale, precision))
    return (o, lse) if with_lse else o


def oracle_attention_heads(q, k, v, w: int, scale: float, with_lse: bool = False,
                           precision: int = PREC_BF16):
    """``oracle_attention`` for ``H`` independent heads in one call: q, k, v
    float32 [H, S, D]; head h equals ``oracle_attention(q[h], k[h], v[h], w,
    scale)``.  The heads are pipelined through PCIe and the B200 kernel
    (mimw_b200_oracle_attention_heads)."""
    q, k, v = map(_f32, (q, k, v))
    if q.ndim != 3 or k.shape != q.shape or v.shape != q.shape:
        raise MimwError(ERR_SHAPE, "q, k, v must be [H, S, D] of one shape")
    h, s, d = q.shape
    o = np.empty((h, s, d), np.float32)
    lse = np.empty((h, s), np.float32)
    _check(lib().mimw_b200_oracle_attention_heads(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), h, s, d,
                                                  w, scale, precision))
    return (o, lse) if with_lse else o


def trim_pool() -> None:
    """Return the library's cached device scratch to the driver."""
    _check(lib().mimw_b200_trim_pool())


def oracle_simplicial_attention(q, k1, v1, k2, v2, w1: int, w2: int, scale: float,
                                precision: int = PREC_BF16):
    """``oracle_simplicial_attention`` (oracles.hpp:31-33, oracles.cpp:82-117)
    on the B200 for one [S, D] head; returns (o, lse).  ``precision`` as for
    ``oracle_attention`` (PREC_F32 holds the reference case's 1e-3)."""
    q, k1, v1, k2, v2 = map(_f32, (q, k1, v1, k2, v2))
    s, d = q.shape
    o = np.empty((s, d), np.float32)
    lse = np.empty(s, np.float32)
    _check(lib().mimw_b200_oracle_simplicial_attention_ex(_ptr(q), _ptr(k1), _ptr(v1), _ptr(k2),
                                                          _ptr(v2), _ptr(o), _ptr(lse), s, d, w1,
                                                          w2, scale, precision))
    return o, lse


def oracle_layernorm(x, w, b, eps: float):
    """``oracle_layernorm(x, w, b, eps, &y, &mean, &rstd)`` (oracles.cpp:28-55)
    on the B200 cluster kernel; returns (y, mean, rstd)."""
    x, w, b = map(_f32, (x, w, b))
    rows, n = x.shape
    y = np.empty_like(x)
    mean = np.empty(rows, np.float32)
    rstd = np.empty(rows, np.float32)
    _check(lib().mimw_b200_oracle_layernorm(_ptr(x), _ptr(w), _ptr(b), eps, _ptr(y), _ptr(mean),
                                            _ptr(rstd), rows, n))
    return y, mean, rstd


def run_oracle(name: str, inputs: dict, scalars: dict | None = None, precision: int = PREC_BF16):
    """``run_oracle`` (oracles.cpp:147-201) dispatching to the B200 path for
    the hot-path oracles.  Unknown / off-path names return ``None``.
    ``precision``: PREC_BF16 (the tensor-core kernels, 1e-2) or any reference
    precision (PREC_F32_BF16X3 / PREC_F32: split-bf16 GEMMs and the f64-arithmetic
    attention path, which hold the reference cases' own tolerances)."""
    scalars = scalars or {}
    gp = PREC_F32_BF16X3 if precision else PREC_BF16
    if name == "gemm":
        return {"c": oracle_gemm(inputs["a"], inputs["b"], gp)}
    if name == "multi_device_gemm":
        return {"c": oracle_multi_device_gemm(inputs["a0"], inputs["a1"], inputs["b0"],
                                              inputs["b1"], gp)}
    if name == "simplicial_attention":  # scalar defaults as sc("w1", 2) ... (oracles.cpp:190-193)
        o, lse = oracle_simplicial_attention(inputs["q"], inputs["k1"], inputs["v1"], inputs["k2"],
                                             inputs["v2"], int(scalars.get("w1", 2)),
                                             int(scalars.get("w2", 16)), scalars.get("scale", 1.0),
                                             PREC_F32 if precision else PREC_BF16)
        return {"o": o, "lse": lse}
    if name == "layernorm":
        return {"y": oracle_layernorm(inputs["x"], inputs["w"], inputs["b"],
                                      scalars.get("eps", 1e-5))[0]}
    if name == "attention":
        return {"o": oracle_attention(inputs["q"], inputs["k"], inputs["v"],
                                      int(scalars.get("w", 1 << 30)), scalars.get("scale", 1.0),
                                      precision=PREC_F32 if precision else PREC_BF16)}
    return None


# ---------------------------------------------------------------------------
# device path (torch CUDA tensors as plumbing)
# ---------------------------------------------------------------------------
def _need(t, dtype, what: str, ndim: int):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise MimwError(ERR_ARG, f"{what}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise MimwError(ERR_UNSUPPORTED, f"{what}: dtype {t.dtype}, expected {dtype}")
    if t.dim() != ndim:
        raise MimwError(ERR_SHAPE, f"{what}: expected {ndim} dims, got shape {tuple(t.shape)}")


def _stream(stream):
    import torch
    return _vp(stream if stream is not None else torch.cuda.current_stream().cuda_stream)


def gemm(a, b, out=None, b_layout: int = B_KN, out_dtype=None, stream=None, cta_group: int = 2,
         raster_group: int = 0, max_clusters: int = 0, tile_n: int = 0):
    """C = A.B with bf16 A [M,K], B [K,N] (B_KN) or [N,K] (B_NK); fp32 accumulate.
    ``out`` dtype float32 or bfloat16.  ``tile_n``: C columns per CTA-pair tile
    (0 auto, 256, or 512 for bf16 out with cta_group 2)."""
    import torch
    _need(a, torch.bfloat16, "gemm a", 2)
    _need(b, torch.bfloat16, "gemm b", 2)
    if b_layout not in (B_KN, B_NK):
        raise MimwError(ERR_ARG, "bad b_layout")
    m, k = a.shape
    kb, n = (b.shape[0], b.shape[1]) if b_layout == B_KN else (b.shape[1], b.shape[0])
    if kb != k:
        raise MimwError(ERR_SHAPE, f"dot conformance: a.shape[1]={k} != K of b={kb}")
    for t, nm in ((a, "a"), (b, "b")):
        if t.stride(1) != 1:
            raise MimwError(ERR_UNSUPPORTED, f"gemm {nm}: rows must be contiguous")
    if out is not None:
        if out.dtype not in (torch.float32, torch.bfloat16) or tuple(out.shape) != (m, n) \
                or out.stride(1) != 1 or out.device != a.device:
            raise MimwError(ERR_SHAPE, f"gemm out: need an f32/bf16 [{m}, {n}] tensor with contiguous rows")
    if b.device != a.device:
        raise MimwError(ERR_ARG, "gemm: a and b on different devices")
    if out is None:
        out = torch.empty((m, n), device=a.device, dtype=out_dtype or torch.bfloat16)
    cd = F32 if out.dtype == torch.float32 else BF16
    _check(lib().mimw_b200_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, k,
                                        a.stride(0), b.stride(0), out.stride(0), b_layout, cd,
                                        cta_group, raster_group, max_clusters, tile_n, _stream(stream)))
    return out


WINDOW_NONCAUSAL = 0


def attention_fwd(q, k, v, window: int | None = None, scale: float | None = None, out=None,
                  lse=None, want_lse: bool = True, stream=None, emu: int = -1, max_ctas: int = 0,
                  trace=None, causal: bool = True, cta_group: int = 1):
    """Causal (optionally windowed) or, with ``causal=False``, non-causal
    attention forward on bf16 [B, H, S, 128] CUDA tensors.  Returns (o, lse)
    with lse fp32 [B, H, S] (natural log)."""
    import torch
    for t, nm in ((q, "q"), (k, "k"), (v, "v")):
        _need(t, torch.bfloat16, f"attention_fwd {nm}", 4)
    if k.shape != q.shape or v.shape != q.shape:
        raise MimwError(ERR_SHAPE, "attention_fwd: q, k, v must have one [B, H, S, D] shape")
    b, h, s, d = q.shape
    if out is not None and (out.shape != q.shape or out.dtype != torch.bfloat16):
        raise MimwError(ERR_SHAPE, "attention_fwd: out must be a bf16 tensor of q's shape")
    if lse is not None and (tuple(lse.shape) != (b, h, s) or lse.dtype != torch.float32
                            or not lse.is_contiguous()):
        raise MimwError(ERR_SHAPE, "attention_fwd: lse must be a contiguous f32 [B, H, S] tensor")
    if not causal:
        window = WINDOW_NONCAUSAL
    if out is None:
        out = torch.empty_like(q)
    if lse is None and want_lse:
        lse = torch.empty((b, h, s), device=q.device, dtype=torch.float32)
    if scale is None:
        scale = d ** -0.5
    if window is None:
        window = s
    for t in (q, k, v, out):
        if not t.is_contiguous():
            raise MimwError(ERR_UNSUPPORTED, "attention_fwd needs contiguous [B,H,S,D] tensors")
    if d != 128:
        raise MimwError(ERR_UNSUPPORTED, "device attention supports head_dim == 128")
    _check(lib().mimw_b200_attention_fwd_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                            lse.data_ptr() if lse is not None else None, b, h, s,
                                            window, scale, emu, max_ctas,
                                            trace.data_ptr() if trace is not None else None,
                                            cta_group, _stream(stream)))
    return out, lse


def gemm_mxfp8(a, sfa, b, sfb, out=None, stream=None, cta_group: int = 2):
    """Block-scaled FP8 GEMM: a e4m3 [M,K], sfa uint8 (UE8M0) [M,K/32],
    b e4m3 [N,K], sfb [N,K/32]  ->  bf16 [M,N] = (a*2^(sfa-127)) . (b*2^(sfb-127))^T."""
    import torch
    f8 = (torch.float8_e4m3fn, torch.uint8)
    for t, nm in ((a, "a"), (b, "b")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype not in f8 or t.dim() != 2:
            raise MimwError(ERR_ARG, f"gemm_mxfp8 {nm}: expected a 2-D e4m3 (or uint8) CUDA tensor")
    m, k = a.shape
    n = b.shape[0]
    if b.shape[1] != k:
        raise MimwError(ERR_SHAPE, f"dot conformance: a.shape[1]={k} != b.shape[1]={b.shape[1]}")
    for t, rows, nm in ((sfa, m, "sfa"), (sfb, n, "sfb")):
        _need(t, torch.uint8, f"gemm_mxfp8 {nm}", 2)
        if tuple(t.shape) != (rows, k // 32):
            raise MimwError(ERR_SHAPE, f"gemm_mxfp8 {nm}: need uint8 [{rows}, {k // 32}] (one UE8M0 per 32 K)")
    for t in (a, b, sfa, sfb):
        if not t.is_contiguous() or t.device != a.device:
            raise MimwError(ERR_UNSUPPORTED, "gemm_mxfp8 needs contiguous tensors on one device")
    if out is not None and (tuple(out.shape) != (m, n) or out.dtype != torch.bfloat16
                            or not out.is_contiguous() or out.device != a.device):
        raise MimwError(ERR_SHAPE, f"gemm_mxfp8 out: need a contiguous bf16 [{m}, {n}] tensor")
    if out is None:
        out = torch.empty((m, n), device=a.device, dtype=torch.bfloat16)
    _check(lib().mimw_b200_gemm_mxfp8_ex(a.data_ptr(), sfa.data_ptr(), b.data_ptr(), sfb.data_ptr(),
                                         out.data_ptr(), m, n, k, cta_group, _stream(stream)))
    return out


def grouped_gemm(x, m_offsets, w, out=None, w_layout: int = B_KN, stream=None, cta_group: int = 2,
                 max_clusters: int = 0, swap_tails: bool | None = None, tile_n: int = 0):
    """Grouped (MoE) GEMM: for each group e, ``out[off[e]:off[e+1]] =
    x[off[e]:off[e+1]] @ W_e`` with bf16 x [rows, K], w [G, K, N] (B_KN) or
    [G, N, K] (B_NK) CUDA tensors and ``m_offsets`` a host sequence of G+1
    non-decreasing row offsets.  Returns bf16 [rows, N].  ``tile_n``: output
    columns per CTA-pair tile (0 auto, 256, 512); ``swap_tails``: groups'
    < 256-row tails as swapped-operand tiles (None: the tile's default)."""
    import torch
    _need(x, torch.bfloat16, "grouped_gemm x", 2)
    _need(w, torch.bfloat16, "grouped_gemm w", 3)
    if w.device != x.device:
        raise MimwError(ERR_ARG, "grouped_gemm: x and w on different devices")
    offs = np.ascontiguousarray(np.asarray(m_offsets, dtype=np.int64))
    g = w.shape[0]
    if offs.shape != (g + 1,):
        raise MimwError(ERR_SHAPE, f"m_offsets must have n_groups + 1 = {g + 1} entries")
    n, k = (w.shape[2], w.shape[1]) if w_layout == B_KN else (w.shape[1], w.shape[2])
    if x.shape[1] != k:
        raise MimwError(ERR_SHAPE, f"dot conformance: x.shape[1]={x.shape[1]} != K={k}")
    if x.shape[0] < offs[-1]:
        raise MimwError(ERR_SHAPE, "x has fewer rows than m_offsets[-1]")
    for t in (x, w):
        if not t.is_contiguous():
            raise MimwError(ERR_UNSUPPORTED, "grouped_gemm needs contiguous tensors")
    if out is not None and (out.dtype != torch.bfloat16 or out.dim() != 2 or out.shape[1] != n
                            or out.shape[0] < offs[-1] or not out.is_contiguous() or out.device != x.device):
        raise MimwError(ERR_SHAPE, f"grouped_gemm out: need a contiguous bf16 [>= {int(offs[-1])}, {n}] tensor")
    if out is None:
        out = torch.empty((x.shape[0], n), device=x.device, dtype=torch.bfloat16)
    _check(lib().mimw_b200_grouped_gemm_bf16_ex(x.data_ptr(), offs.ctypes.data, w.data_ptr(),
                                                out.data_ptr(), g, n, k, w_layout, cta_group,
                                                max_clusters, -1 if swap_tails is None else int(bool(swap_tails)),
                                                tile_n, _stream(stream)))
    return out


def layernorm(x, w, b, eps: float = 1e-5, out=None, mean=None, rstd=None, stream=None,
              cluster: int = 0):
    """Cluster LayerNorm over the last dim of an f32 CUDA tensor [rows, n]."""
    import torch
    _need(x, torch.float32, "layernorm x", 2)
    if not x.is_contiguous():
        raise MimwError(ERR_UNSUPPORTED, "layernorm needs a contiguous float32 tensor")
    rows, n = x.shape
    for t, nm in ((w, "w"), (b, "b")):
        _need(t, torch.float32, f"layernorm {nm}", 1)
        if t.numel() < n or not t.is_contiguous():
            raise MimwError(ERR_SHAPE, f"layernorm {nm}: need a contiguous f32 vector of >= {n} elements")
    for t, nm in ((mean, "mean"), (rstd, "rstd")):
        if t is not None and (t.dtype != torch.float32 or t.numel() < rows or not t.is_contiguous()):
            raise MimwError(ERR_SHAPE, f"layernorm {nm}: need a contiguous f32 vector of >= {rows} elements")
    if out is not None and (out.shape != x.shape or out.dtype != torch.float32 or not out.is_contiguous()):
        raise MimwError(ERR_SHAPE, "layernorm out: need a contiguous f32 tensor of x's shape")
    if out is None:
        out = torch.empty_like(x)
    _check(lib().mimw_b200_layernorm_ex(x.data_ptr(), w.data_ptr(), b.data_ptr(), out.data_ptr(),
                                        mean.data_ptr() if mean is not None else None,
                                        rstd.data_ptr() if rstd is not None else None, rows, n,
                                        eps, cluster, _stream(stream)))
    return out


def simplicial_attention_fwd(q, k1, v1, k2, v2, w1: int, w2: int, scale: float | None = None,
                             out=None, lse=None, want_lse: bool = True, stream=None):
    """2-simplicial attention forward on bf16 CUDA tensors [BH, S, 128]."""
    import torch
    for t, nm in ((q, "q"), (k1, "k1"), (v1, "v1"), (k2, "k2"), (v2, "v2")):
        _need(t, torch.bfloat16, f"simplicial_attention_fwd {nm}", 3)
    bh, s, d = q.shape
    if d != 128:
        raise MimwError(ERR_UNSUPPORTED, "device simplicial attention supports head_dim == 128")
    for t in (q, k1, v1, k2, v2):
        if not t.is_contiguous() or t.shape != q.shape or t.device != q.device:
            raise MimwError(ERR_UNSUPPORTED, "contiguous [BH, S, 128] tensors of one shape required")
    if out is not None and (out.shape != q.shape or out.dtype != torch.bfloat16 or not out.is_contiguous()):
        raise MimwError(ERR_SHAPE, "simplicial_attention_fwd out: need a contiguous bf16 tensor of q's shape")
    if lse is not None and (tuple(lse.shape) != (bh, s) or lse.dtype != torch.float32 or not lse.is_contiguous()):
        raise MimwError(ERR_SHAPE, "simplicial_attention_fwd lse: need a contiguous f32 [BH, S] tensor")
    if out is None:
        out = torch.empty_like(q)
    if lse is None and want_lse:
        lse = torch.empty((bh, s), device=q.device, dtype=torch.float32)
    if scale is None:
        scale = d ** -0.5
    _check(lib().mimw_b200_simplicial_attention_fwd(
        q.data_ptr(), k1.data_ptr(), v1.data_ptr(), k2.data_ptr(), v2.data_ptr(), out.data_ptr(),
        lse.data_ptr() if lse is not None else None, bh, s, d, w1, w2, scale, _stream(stream)))
    return out, lse


def attention_bwd(q, k, v, o, do, lse, window: int | None = None, scale: float | None = None,
                  causal: bool = True, dq=None, dk=None, dv=None, stream=None):
    """Attention backward on bf16 [B, H, S, 128] CUDA tensors: returns (dq, dk, dv)
    given the forward's output ``o`` and ``lse`` (fp32 [B, H, S]) and the
    upstream gradient ``do``.  ``causal=False`` for non-causal attention."""
    import torch
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (o, "o"), (do, "do")):
        _need(t, torch.bfloat16, f"attention_bwd {nm}", 4)
        if t.shape != q.shape:
            raise MimwError(ERR_SHAPE, f"attention_bwd {nm}: shape {tuple(t.shape)} != q's {tuple(q.shape)}")
    b, h, s, d = q.shape
    _need(lse, torch.float32, "attention_bwd lse", 3)
    if tuple(lse.shape) != (b, h, s):
        raise MimwError(ERR_SHAPE, f"attention_bwd lse: need f32 [{b}, {h}, {s}]")
    for t, nm in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        if t is not None and (t.shape != q.shape or t.dtype != torch.bfloat16 or not t.is_contiguous()):
            raise MimwError(ERR_SHAPE, f"attention_bwd {nm}: need a contiguous bf16 tensor of q's shape")
    if d != 128:
        raise MimwError(ERR_UNSUPPORTED, "device attention supports head_dim == 128")
    for t in (q, k, v, o, do, lse):
        if not t.is_contiguous() or t.device != q.device:
            raise MimwError(ERR_UNSUPPORTED, "attention_bwd needs contiguous tensors on one device")
    if scale is None:
        scale = d ** -0.5
    if not causal:
        window = WINDOW_NONCAUSAL
    elif window is None:
        window = s
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    _check(lib().mimw_b200_attention_bwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                         do.data_ptr(), lse.data_ptr(), dq.data_ptr(),
                                         dk.data_ptr(), dv.data_ptr(), b, h, s, d, window, scale,
                                         _stream(stream)))
    return dq, dk, dv
