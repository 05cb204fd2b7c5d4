/*
 * mimw_b200.h — C-ABI of the B200-native hot path (libmimw_b200.so).
 *
 * Drop-in boundary for the reference's operator API, the pure oracle
 * functions of /root/reference/proj/core/include/mimw/oracles.hpp (which
 * the corpus driver tools/mimw.cpp:205-259 and the tests call through
 * run_oracle, oracles.cpp:147-201).  Two families of entry points:
 *
 *   mimw_b200_oracle_*   HOST f32 buffers, exactly the reference's Tile
 *                        semantics (row-major, shapes as in oracles.hpp);
 *                        copies in, runs the sm_100a kernels, copies out.
 *                        These replace the reference functions one for one.
 *   mimw_b200_*          DEVICE buffers + a cudaStream_t (as void*), the
 *                        production path (bf16 / e4m3 operands in HBM).
 *
 * Conventions: plain pointers and int64 sizes, no exceptions
 * cross the ABI, every call returns a status code; the message of the last
 * failure on the calling thread is available from mimw_b200_last_error().
 * Calls are reentrant per stream.  There is no CPU fallback: without a
 * B200 (sm_100a) device every compute entry point returns MIMW_ERR_CUDA.
 */
#ifndef MIMW_B200_H
#define MIMW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MIMW_OK 0
#define MIMW_ERR_SHAPE 1       /* dot conformance, proj/core/src/validate.cpp:314-338 */
#define MIMW_ERR_UNSUPPORTED 2 /* dtype / layout / alignment not supported */
#define MIMW_ERR_CUDA 3        /* CUDA runtime / launch failure, or no sm_100 device */
#define MIMW_ERR_ARG 4         /* null pointer or bad enum */

/* element types */
#define MIMW_F32 0
#define MIMW_BF16 1

/* B operand layout */
#define MIMW_B_KN 0 /* B[K, N] row-major — the reference's layout (oracles.cpp:21-22) */
#define MIMW_B_NK 1 /* B[N, K] row-major (K-contiguous, "NT" GEMM) */

/* precision of the host f32 entry points */
#define MIMW_PREC_BF16 0          /* inputs rounded to bf16 (RNE), fp32 accumulate */
#define MIMW_PREC_F32_BF16X3 1    /* split-bf16 x3 on tensor cores: ~1e-6 rel-err,
                                     meets the reference's own 1e-4 GEMM cases */
#define MIMW_PREC_F32 2           /* attention Tiles: the oracles' f64 score / softmax
                                     arithmetic on CUDA cores (reference tolerances
                                     1e-4 / 1e-3; for reference-scale Tiles) */

int mimw_b200_version(void);
const char *mimw_b200_last_error(void);

/* Device scratch (staging buffers, the attention-backward dQ accumulator)
 * comes from a library-private stream-ordered memory pool per device that
 * keeps freed memory for the next call; the device's default pool is never
 * modified.  This returns the private pool's cached memory of the current
 * device to the driver. */
int mimw_b200_trim_pool(void);

/* ---- GEMM:  C[M,N] = A[M,K] . B  (fp32 accumulate in TMEM) ----------------
 * Replaces: Tile oracle_gemm(const Tile &a, const Tile &b)
 *           proj/core/include/mimw/oracles.hpp:15-16 (oracles.cpp:14-26).
 * Host f32 buffers a[m*k], b[k*n] (row-major, B as [K,N]); c[m*n] written. */
int mimw_b200_oracle_gemm(const float *a, const float *b, float *c, int64_t m, int64_t n,
                          int64_t k, int32_t precision);

/* Device form: a bf16 [m, lda], b bf16 ([k, ldb] for MIMW_B_KN or [n, ldb]
 * for MIMW_B_NK), c [m, ldc] of c_dtype (MIMW_F32 or MIMW_BF16).  Leading
 * dimensions in elements; row pitches must be multiples of 16 bytes (TMA).
 * Warp-specialized kernel, 2-CTA clusters (cta_group::2); output tiles are
 * dispatched by hardware cluster launch control (gemm_clc.mimw). */
int mimw_b200_gemm_bf16(const void *a, const void *b, void *c, int64_t m, int64_t n, int64_t k,
                        int64_t lda, int64_t ldb, int64_t ldc, int32_t b_layout, int32_t c_dtype,
                        void *stream);

/* ---- Block-scaled FP8 GEMM (MXFP8) -----------------------------------------
 * C[m,n] (bf16) = sum_k e4m3(a[m,k]) 2^(sfa[m,k/32]-127) * e4m3(b[n,k]) 2^(sfb[n,k/32]-127)
 * No reference counterpart; its oracle is oracle_gemm
 * (oracles.cpp:14-26) on the dequantised Tiles.  Device buffers: a e4m3
 * [m,k], b e4m3 [n,k] (both K-contiguous), sfa ue8m0 [m,k/32], sfb ue8m0
 * [n,k/32], c bf16 [m,n]; k % 32 == 0.  tcgen05.mma.kind::mxf8f6f4.block_scale
 * with scale factors staged smem->TMEM by tcgen05.cp. */
int mimw_b200_gemm_mxfp8(const void *a, const void *sfa, const void *b, const void *sfb, void *c,
                         int64_t m, int64_t n, int64_t k, void *stream);

/* ---- Grouped (MoE) GEMM ---------------------------------------------------
 * For every group (expert) e < n_groups:
 *   y[m_offsets[e] : m_offsets[e+1], :] = x[m_offsets[e] : m_offsets[e+1], :] . W_e
 * No reference counterpart; its oracle is one
 * oracle_gemm (oracles.cpp:14-26) per group.  x bf16 [m_offsets[G], k] and
 * y bf16 [m_offsets[G], n] are DEVICE buffers with rows packed by group;
 * m_offsets is a HOST int64 array of n_groups + 1 non-decreasing row offsets
 * (empty groups allowed); w bf16 is [G, k, n] (MIMW_B_KN, the reference's
 * B layout) or [G, n, k] (MIMW_B_NK).  n and k multiples of 8.  2-CTA kernel,
 * tiles dispatched by cluster launch control; each group's < 256-row tail runs
 * as a swapped-operand tile clipped by the group's own Y tensor map. */
int mimw_b200_grouped_gemm_bf16(const void *x, const int64_t *m_offsets, const void *w, void *y,
                                int64_t n_groups, int64_t n, int64_t k, int32_t w_layout,
                                void *stream);

/* ---- K-gathered GEMM: C = [a0 | a1] . [b0 ; b1] ---------------------------
 * Replaces: Tile oracle_multi_device_gemm(a0, a1, b0, b1)
 *           oracles.hpp:24-25 (oracles.cpp:57-80).  Host f32 buffers. */
int mimw_b200_oracle_multi_device_gemm(const float *a0, const float *a1, const float *b0,
                                       const float *b1, float *c, int64_t m, int64_t k0,
                                       int64_t k1, int64_t n, int32_t precision);

/* ---- All-gather (K-gathered) multi-device GEMM -------
 * The production form of oracle_multi_device_gemm (oracles.hpp:24-25,
 * oracles.cpp:57-80) and proj/kernels/multi_device_gemm.mimw:1-79,
 * generalised from 2 to `world` devices.  Device s holds the K-split
 * a_splits[s] bf16 [m, k_splits[s]] and b_splits[s] bf16 [k_splits[s], n];
 * this call (on device `rank`) computes its row block of
 *     C = [a_0 | ... | a_{world-1}] . [b_0 ; ... ; b_{world-1}]
 * i.e. c[rows, n] (bf16, row pitch ldc) = C[row0 : row0 + rows, :].
 * a_splits[s] / b_splits[s] are pointers valid in the calling process: the
 * local split, or a peer's buffer mapped with mimw_b200_ipc_open.  One kernel
 * overlaps the gather with the GEMM: comm CTA pairs pull the peers' splits
 * over NVLink into `workspace` in 256-wide K slabs and publish each on a
 * readiness counter; the GEMM CTA pairs start on the local split and wait on a
 * slab's counter only before its first TMA load.
 * pads[p] = device p's 64-byte signal pad (inside an IPC allocation, zeroed at
 * allocation) for the device-side entry/exit barrier, with `epoch` strictly
 * increasing from 1 per call; pads == NULL skips the barrier (the caller then
 * guarantees the peers' splits are complete and stay unchanged until this call
 * has finished — e.g. all "devices" emulated on one GPU).
 * workspace: >= mimw_b200_multi_device_gemm_workspace_bytes(...), 1 KiB
 * aligned.  n and every k split multiples of 8.  comm_pairs: > 0 that many
 * dedicated comm CTA pairs (the reference's comm CTAs); < 0 a comm warp in
 * every GEMM CTA pair instead (no SM taken from the GEMM); 0 = the default.
 * max_pairs caps the GEMM CTA pairs (0 = every co-resident pair). */
#define MIMW_MAX_DEVICES 8
#define MIMW_IPC_HANDLE_BYTES 64
#define MIMW_SIGNAL_PAD_BYTES 64
int64_t mimw_b200_multi_device_gemm_workspace_bytes(int32_t rank, int32_t world,
                                                    const int64_t *k_splits, int64_t rows,
                                                    int64_t n);
int mimw_b200_multi_device_gemm(int32_t rank, int32_t world, const void *const *a_splits,
                                const void *const *b_splits, const int64_t *k_splits, int64_t m,
                                int64_t n, int64_t row0, int64_t rows, void *c, int64_t ldc,
                                void *workspace, int64_t workspace_bytes, uint32_t *const *pads,
                                uint32_t epoch, int32_t comm_pairs, int32_t max_pairs,
                                void *stream);

/* Same, with the comm pipelines' tuning knobs (0 = defaults): comm_box = box
 * rows 32 / 64 / 128 of 512 bytes (16 / 32 / 64 KiB TMA boxes), comm_agents = copy
 * pipelines per comm CTA (1..6), comm_lag = stores in flight before a slab's
 * readiness signal waits for completion (1, 2, 4, 6, 8, 12). */
int mimw_b200_multi_device_gemm_ex(int32_t rank, int32_t world, const void *const *a_splits,
                                   const void *const *b_splits, const int64_t *k_splits, int64_t m,
                                   int64_t n, int64_t row0, int64_t rows, void *c, int64_t ldc,
                                   void *workspace, int64_t workspace_bytes, uint32_t *const *pads,
                                   uint32_t epoch, int32_t comm_pairs, int32_t max_pairs,
                                   int32_t comm_box, int32_t comm_agents, int32_t comm_lag,
                                   void *stream);

/* CUDA IPC plumbing for the peer mappings: a zero-filled device allocation
 * with its 64-byte IPC handle, and the peer side's open / close. */
int mimw_b200_ipc_alloc(int64_t bytes, void **ptr, void *handle);
int mimw_b200_ipc_open(const void *handle, void **ptr);
int mimw_b200_ipc_close(void *ptr);
int mimw_b200_ipc_free(void *ptr);

/* ---- Attention forward (windowed causal softmax attention) --------------
 * Replaces: void oracle_attention(const Tile &q, const Tile &k, const Tile &v,
 *                                 int w, double scale, Tile *o)
 *           oracles.hpp:35-37 (oracles.cpp:119-145): keys j in
 *           [max(0, i-w+1), i]; w >= seq is plain causal attention.
 * Host f32 buffers q, k, v, o of [seq, d] (d <= 128; zero-padded to 128
 * internally, exact); lse[seq] (natural-log logsumexp of the scaled scores,
 * as oracle_simplicial_attention's lse, oracles.cpp:116) may be NULL. */
int mimw_b200_oracle_attention(const float *q, const float *k, const float *v, float *o,
                               float *lse, int64_t seq, int64_t d, int64_t w, double scale);

/* Batched form for `heads` independent heads stored back to back: q, k, v, o
 * host f32 [heads, seq, d], lse [heads, seq] or NULL; head h is exactly
 * oracle_attention(q[h], k[h], v[h], w, scale).  No reference counterpart
 * (the reference's callers loop over heads); one call pipelines the heads
 * through PCIe and the B200 kernel.  precision as mimw_b200_oracle_attention_ex. */
int mimw_b200_oracle_attention_heads(const float *q, const float *k, const float *v, float *o,
                                     float *lse, int64_t heads, int64_t seq, int64_t d, int64_t w,
                                     double scale, int32_t precision);

/* window value selecting non-causal attention (every key of the sequence; the
 * paper's AFN / ABC rows, PAPER.md:702-716 — no reference oracle) */
#define MIMW_WINDOW_NONCAUSAL 0

/* Same with a precision: MIMW_PREC_BF16 (the tcgen05 kernel on bf16 inputs,
 * rel-err ~3e-3, the north-star 1e-2 bar), MIMW_PREC_F32_BF16X3 (split-bf16 x3
 * scores and P.V on the tcgen05 GEMM, softmax in f32: the reference's own 1e-4,
 * acceptance.cpp:333-355) or MIMW_PREC_F32 (f64 scores on CUDA cores, one CTA
 * per query row: the reference's arithmetic, for callers that want it). */
int mimw_b200_oracle_attention_ex(const float *q, const float *k, const float *v, float *o,
                                  float *lse, int64_t seq, int64_t d, int64_t w, double scale,
                                  int32_t precision);

/* Device form: q, k, v, o bf16 [batch, heads, seq, head_dim] contiguous,
 * head_dim == 128; lse fp32 [batch, heads, seq] or NULL.  window >= 1 as in
 * the reference, or MIMW_WINDOW_NONCAUSAL.  Warp-specialized
 * kernel: TMA producer warp, single-thread tcgen05 MMA warp (S = QK^T and
 * O += PV with P in TMEM), two ping-pong softmax/correction warpgroups. */
int mimw_b200_attention_fwd(const void *q, const void *k, const void *v, void *o, float *lse,
                            int64_t batch, int64_t heads, int64_t seq, int64_t head_dim,
                            int64_t window, double scale, void *stream);

/* ---- Attention backward (PAPER.md:702-716 ABC rows) --
 * Gradients of o = softmax(scale q k^T) v (causal with `window` as the forward,
 * or MIMW_WINDOW_NONCAUSAL).  No reference counterpart (the reference has no
 * backward); oracle: the f64 restatement orc_attention_bwd in oracle/oracle.c.
 * q, k, v, o, dout, dq, dk, dv bf16 [batch, heads, seq, 128] contiguous; lse
 * fp32 [batch, heads, seq] (natural log, as written by mimw_b200_attention_fwd).
 * Any seq >= 0.  KV-stationary tcgen05 kernel (key-major S^T / dP^T so P^T and
 * dS^T feed the dV / dK MMAs from TMEM), dQ accumulated by TMA reduce-add. */
int mimw_b200_attention_bwd(const void *q, const void *k, const void *v, const void *o,
                            const void *dout, const float *lse, void *dq, void *dk, void *dv,
                            int64_t batch, int64_t heads, int64_t seq, int64_t head_dim,
                            int64_t window, double scale, void *stream);

/* ---- 2-simplicial attention forward ----------------
 * Replaces: void oracle_simplicial_attention(q, k1, v1, k2, v2, int w1, int w2,
 *                                            double scale, Tile *o, Tile *lse)
 *           proj/core/include/mimw/oracles.hpp:31-33 (oracles.cpp:82-117):
 *   s(i,j1,j2) = scale * sum_x q[i,x] k1[j1,x] k2[j2,x],
 *   o[i] = sum softmax(s) v1[j1] (.) v2[j2],  lse[i] = log sum exp s,
 *   j1 in [i-w1+1, i], j2 in [i-w2+1, i].
 * Host f32 buffers of [seq, d] (d <= 128, zero-padded to 128 internally). */
int mimw_b200_oracle_simplicial_attention(const float *q, const float *k1, const float *v1,
                                           const float *k2, const float *v2, float *o, float *lse,
                                           int64_t seq, int64_t d, int64_t w1, int64_t w2,
                                           double scale);

/* Same with a precision (MIMW_PREC_BF16 or MIMW_PREC_F32, which holds the
 * reference case's 1e-3, simplicial_attention.case). */
int mimw_b200_oracle_simplicial_attention_ex(const float *q, const float *k1, const float *v1,
                                              const float *k2, const float *v2, float *o, float *lse,
                                              int64_t seq, int64_t d, int64_t w1, int64_t w2,
                                              double scale, int32_t precision);

/* Device form: bf16 [bh, seq, 128] contiguous (bh = batch*heads), lse fp32
 * [bh, seq] or NULL.  Per K1 offset a windowed flash-attention sweep over K2/V2
 * on tcgen05 (Q (.) K1 formed elementwise into smem, V1 applied after P.V2). */
int mimw_b200_simplicial_attention_fwd(const void *q, const void *k1, const void *v1, const void *k2,
                                       const void *v2, void *o, float *lse, int64_t bh, int64_t seq,
                                       int64_t head_dim, int64_t w1, int64_t w2, double scale,
                                       void *stream);

/* ---- Cluster LayerNorm ------------------------------
 * Replaces: void oracle_layernorm(const Tile &x, const Tile &w, const Tile &b,
 *                                 double eps, Tile *y, Tile *mean, Tile *rstd)
 *           proj/core/src/oracles.cpp:28-55 (two-pass mean / variance), the
 *           computation proj/kernels/layernorm_cluster.mimw:1-62 distributes
 *           over a CTA cluster.  Host f32 buffers x[rows*n], w[n], b[n],
 *           y[rows*n]; mean / rstd [rows] may be NULL.  n <= 262144. */
int mimw_b200_oracle_layernorm(const float *x, const float *w, const float *b, double eps, float *y,
                               float *mean, float *rstd, int64_t rows, int64_t n);

/* Device form: f32 [rows, n] row-major; one thread-block cluster per row
 * (CTA slices of <= 16K columns), partial reductions exchanged through
 * distributed shared memory (st.async + remote mbarrier complete_tx). */
int mimw_b200_layernorm(const float *x, const float *w, const float *b, float *y, float *mean,
                        float *rstd, int64_t rows, int64_t n, double eps, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MIMW_B200_H */
