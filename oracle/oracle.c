/*
 * TEST INFRASTRUCTURE — the CPU oracle for the B200 hot path.
 *
 * Plain-C restatement of the reference's dense oracles and parity plumbing.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this (as the checker); the product library never links it and has no
 * CPU fallback.
 *
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   1. against tests/golden/*.tnsr, produced by the UNMODIFIED reference
 *      sources compiled here (oracle/_ref, see oracle/Makefile and
 *      tests/golden/make_golden.py), bit-for-bit;
 *   2. live against oracle/_ref on fresh seeds whenever _ref is built.
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).  Build: gcc -O2 -ffp-contract=off (no FMA
 * contraction, so float sums round exactly like the reference's
 * `s += a*b`, which g++ -O3 without -march never contracts).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* mt19937_64 — the engine behind random_tile (core/src/tensor_io.cpp:82). */
/* Standard constants from the C++ <random> specification.                 */
/* ---------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t *s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64_t *s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* random_tile: u = (rng() >> 11) * 2^-53 in [0,1); x = float(u*2-1).
 * core/src/tensor_io.cpp:80-88. */
void orc_random_tile(int64_t n, uint64_t seed, float *out) {
  mt64_t s;
  mt64_seed(&s, seed);
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
    out[i] = (float)(u * 2.0 - 1.0);
  }
}

/* make_inputs seed rule: input k of a program gets seed*1000003 + k
 * (core/src/case.cpp:82-92). */
uint64_t orc_input_seed(uint64_t seed, uint64_t k) { return seed * 1000003ULL + k; }

/* rel_error = max|a-b| / max(max|b|, 1e-30), in double (core/src/case.cpp:94-104). */
double orc_rel_error(const float *a, const float *b, int64_t n) {
  double max_abs = 1e-30, max_diff = 0;
  for (int64_t i = 0; i < n; ++i) {
    double bb = fabs((double)b[i]);
    double d = fabs((double)a[i] - (double)b[i]);
    if (bb > max_abs) max_abs = bb;
    if (d > max_diff) max_diff = d;
  }
  return max_diff / max_abs;
}

/* Per-row variant: max over rows of the row's rel_error. */
double orc_rel_error_rows(const float *a, const float *b, int64_t rows,
                          int64_t cols) {
  double worst = 0;
  for (int64_t r = 0; r < rows; ++r) {
    double e = orc_rel_error(a + r * cols, b + r * cols, cols);
    if (e > worst) worst = e;
  }
  return worst;
}

/* ---------------------------------------------------------------------- */
/* Number formats used to feed identical values to CPU and GPU.            */
/* ---------------------------------------------------------------------- */
/* f32 -> bf16 round-to-nearest-even (NaN kept quiet), returned as f32. */
float orc_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) {
    u = (u | 0x00400000u) & 0xFFFF0000u;
  } else {
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
  }
  memcpy(&x, &u, 4);
  return x;
}

void orc_round_bf16_n(const float *in, float *out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_round_bf16(in[i]);
}

/* OCP e4m3 (FN variant: no inf, S.1111.111 = NaN, max 448) decode. */
float orc_e4m3_to_f32(uint8_t v) {
  int s = v >> 7, e = (v >> 3) & 0xF, m = v & 7;
  float r;
  if (e == 0xF && m == 7) return NAN;
  if (e == 0)
    r = ldexpf((float)m, -9); /* subnormal: m/8 * 2^-6 */
  else
    r = ldexpf(1.0f + (float)m / 8.0f, e - 7);
  return s ? -r : r;
}

/* UE8M0 scale decode: 2^(e-127); 0xFF = NaN. */
float orc_ue8m0_to_f32(uint8_t e) {
  if (e == 0xFF) return NAN;
  return ldexpf(1.0f, (int)e - 127);
}

/* MX block-scaled dequantisation along K (the FP8 path's oracle input):
 * x[r, c] = e4m3(q[r, c]) * ue8m0(sf[r, c / 32]); q is [rows, cols] row-major,
 * sf is [rows, cols/32]. */
void orc_mx_dequant(const uint8_t *q, const uint8_t *sf, float *out,
                    int64_t rows, int64_t cols) {
  int64_t nb = cols / 32;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      out[r * cols + c] =
          orc_e4m3_to_f32(q[r * cols + c]) * orc_ue8m0_to_f32(sf[r * nb + c / 32]);
}

/* ---------------------------------------------------------------------- */
/* Oracles                                                                 */
/* ---------------------------------------------------------------------- */

/* C = A.B, float accumulator starting at 0.0f, ascending k
 * (core/src/oracles.cpp:14-26).  B is walked through a transposed copy for
 * cache friendliness; each c[i,j] still sums a[i,k]*b[k,j] in ascending k in
 * float, so the result is bit-identical to the reference. */
void orc_gemm_rows(const float *a, const float *b, float *c, int64_t m,
                   int64_t n, int64_t k, int64_t r0, int64_t r1) {
  (void)m;
  float *bt = (float *)malloc(sizeof(float) * (size_t)(n * k));
  for (int64_t kk = 0; kk < k; ++kk)
    for (int64_t j = 0; j < n; ++j) bt[j * k + kk] = b[kk * n + j];
  for (int64_t i = r0; i < r1; ++i) {
    const float *ar = a + i * k;
    for (int64_t j = 0; j < n; ++j) {
      const float *bc = bt + j * k;
      float s = 0.0f;
      for (int64_t kk = 0; kk < k; ++kk) s += ar[kk] * bc[kk];
      c[i * n + j] = s;
    }
  }
  free(bt);
}

void orc_gemm(const float *a, const float *b, float *c, int64_t m, int64_t n,
              int64_t k) {
  orc_gemm_rows(a, b, c, m, n, k, 0, m);
}

/* Selected rows of C = A.B for config-scale parity: c[r, :] = a[r, :] . B for
 * the R rows given as a[R, K] (gathered by the caller), B [K, N] row-major.
 * Same arithmetic as oracles.cpp:17-23 — per element a float accumulator
 * starting at 0.0f, s += a[k]*b[k][j] in ascending k, no FMA contraction —
 * so bit-identical to the reference (tests/test_oracle.py pins it), but the
 * loop runs k-outer over a block of rows and a slice of columns per thread,
 * streaming B row-contiguously (vectorised across j), so 8192^3-scale row
 * samples take seconds instead of the reference's strided walk. */
typedef struct {
  const float *a, *b;
  float *c;
  int64_t R, N, K, j0, j1;
} rowlist_job;

static void *gemm_rowlist_worker(void *arg) {
  const rowlist_job *jb = (const rowlist_job *)arg;
  const int64_t RB = 16, JB = 512;
  float acc[16 * 512];
  for (int64_t r0 = 0; r0 < jb->R; r0 += RB) {
    const int64_t rn = jb->R - r0 < RB ? jb->R - r0 : RB;
    for (int64_t j0 = jb->j0; j0 < jb->j1; j0 += JB) {
      const int64_t jn = jb->j1 - j0 < JB ? jb->j1 - j0 : JB;
      for (int64_t x = 0; x < rn * JB; ++x) acc[x] = 0.0f;
      for (int64_t kk = 0; kk < jb->K; ++kk) {
        const float *br = jb->b + kk * jb->N + j0;
        for (int64_t r = 0; r < rn; ++r) {
          const float av = jb->a[(r0 + r) * jb->K + kk];
          float *ar = acc + r * JB;
          for (int64_t j = 0; j < jn; ++j) ar[j] = ar[j] + av * br[j];
        }
      }
      for (int64_t r = 0; r < rn; ++r)
        memcpy(jb->c + (r0 + r) * jb->N + j0, acc + r * JB, sizeof(float) * (size_t)jn);
    }
  }
  return NULL;
}

void orc_gemm_rowlist_mt(const float *a, const float *b, float *c, int64_t R, int64_t N, int64_t K,
                         int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  rowlist_job jobs[256];
  const int64_t per = ((N + threads - 1) / threads + 7) / 8 * 8;
  int nt = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t j0 = t * per, j1 = j0 + per < N ? j0 + per : N;
    if (j0 >= j1) break;
    jobs[nt] = (rowlist_job){a, b, c, R, N, K, j0, j1};
    pthread_create(&th[nt], NULL, gemm_rowlist_worker, &jobs[nt]);
    ++nt;
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* Gathered GEMM: A = [a0 | a1], B = [b0 ; b1] (core/src/oracles.cpp:57-80). */
void orc_multi_device_gemm(const float *a0, const float *a1, const float *b0,
                           const float *b1, float *c, int64_t m, int64_t k0,
                           int64_t k1, int64_t n) {
  int64_t k = k0 + k1;
  float *a = (float *)malloc(sizeof(float) * (size_t)(m * k));
  float *b = (float *)malloc(sizeof(float) * (size_t)(k * n));
  for (int64_t i = 0; i < m; ++i) {
    memcpy(a + i * k, a0 + i * k0, sizeof(float) * (size_t)k0);
    memcpy(a + i * k + k0, a1 + i * k1, sizeof(float) * (size_t)k1);
  }
  memcpy(b, b0, sizeof(float) * (size_t)(k0 * n));
  memcpy(b + k0 * n, b1, sizeof(float) * (size_t)(k1 * n));
  orc_gemm(a, b, c, m, n, k);
  free(a);
  free(b);
}

/* Windowed causal softmax attention, one head (core/src/oracles.cpp:119-145):
 * keys j in [max(0, i-w+1), i]; scores in double (s += double(q)*k, then
 * *scale); m = max; l = sum exp(s-m); p = exp(s-m)/l; o[i,x] += float(p*v)
 * in ascending j with a float accumulator.  lse (not produced by the
 * reference function) is m + log(l) as in oracles.cpp:116, written only when
 * lse != NULL. */
/* Rows [r0, r1) only (each row of the reference loop is independent); o and
 * lse are indexed from row r0.  Used for row-sampled parity at S = 8192. */
void orc_attention_rows(const float *q, const float *k, const float *v, float *o,
                        float *lse, int64_t seq, int64_t d, int64_t w, double scale,
                        int64_t r0, int64_t r1) {
  double *scores = (double *)malloc(sizeof(double) * (size_t)(seq > 0 ? seq : 1));
  memset(o, 0, sizeof(float) * (size_t)((r1 - r0) * d));
  o -= r0 * d;
  if (lse) lse -= r0;
  for (int64_t i = r0; i < r1; ++i) {
    int64_t j0 = i - w + 1 > 0 ? i - w + 1 : 0;
    int64_t cnt = 0;
    for (int64_t j = j0; j <= i; ++j) {
      double s = 0;
      for (int64_t x = 0; x < d; ++x) s += (double)q[i * d + x] * k[j * d + x];
      scores[cnt++] = s * scale;
    }
    double m = -INFINITY;
    for (int64_t t = 0; t < cnt; ++t) m = scores[t] > m ? scores[t] : m;
    double l = 0;
    for (int64_t t = 0; t < cnt; ++t) l += exp(scores[t] - m);
    for (int64_t t = 0; t < cnt; ++t) {
      double p = exp(scores[t] - m) / l;
      const float *vr = v + (j0 + t) * d;
      for (int64_t x = 0; x < d; ++x) o[i * d + x] += (float)(p * vr[x]);
    }
    if (lse) lse[i] = (float)(m + log(l));
  }
  free(scores);
}

void orc_attention(const float *q, const float *k, const float *v, float *o,
                   float *lse, int64_t seq, int64_t d, int64_t w, double scale) {
  orc_attention_rows(q, k, v, o, lse, seq, d, w, scale, 0, seq);
}

/* Key range of query row i: the reference's windowed causal rule
 * (oracles.cpp:123-126), or — causal == 0 — every key of the sequence.
 * The non-causal mode has NO reference oracle (the reference's attention is
 * causal only); it is a restatement with the key range
 * widened and the reference's arithmetic otherwise unchanged (f64 scores and
 * softmax, f32 accumulation of o in ascending key order, oracles.cpp:127-144). */
static void key_range(int64_t i, int64_t seq, int64_t w, int causal, int64_t *j0, int64_t *j1) {
  if (causal) {
    *j0 = i - w + 1 > 0 ? i - w + 1 : 0;
    *j1 = i;
  } else {
    *j0 = 0;
    *j1 = seq - 1;
  }
}

void orc_attention_mode_rows(const float *q, const float *k, const float *v, float *o,
                             float *lse, int64_t seq, int64_t d, int64_t w, int causal,
                             double scale, int64_t r0, int64_t r1) {
  double *scores = (double *)malloc(sizeof(double) * (size_t)(seq > 0 ? seq : 1));
  memset(o, 0, sizeof(float) * (size_t)((r1 - r0) * d));
  o -= r0 * d;
  if (lse) lse -= r0;
  for (int64_t i = r0; i < r1; ++i) {
    int64_t j0, j1;
    key_range(i, seq, w, causal, &j0, &j1);
    int64_t cnt = 0;
    for (int64_t j = j0; j <= j1; ++j) {
      double s = 0;
      for (int64_t x = 0; x < d; ++x) s += (double)q[i * d + x] * k[j * d + x];
      scores[cnt++] = s * scale;
    }
    double m = -INFINITY;
    for (int64_t t = 0; t < cnt; ++t) m = scores[t] > m ? scores[t] : m;
    double l = 0;
    for (int64_t t = 0; t < cnt; ++t) l += exp(scores[t] - m);
    for (int64_t t = 0; t < cnt; ++t) {
      double p = exp(scores[t] - m) / l;
      const float *vr = v + (j0 + t) * d;
      for (int64_t x = 0; x < d; ++x) o[i * d + x] += (float)(p * vr[x]);
    }
    if (lse) lse[i] = (float)(m + log(l));
  }
  free(scores);
}

/* Sparse rows of one head's attention (rows[] in any order, each computed as
 * orc_attention_mode_rows(row, row + 1)), spread over pthreads; o[nrows, d],
 * lse[nrows].  For config-scale parity (one row per work item). */
typedef struct {
  const float *q, *k, *v;
  float *o, *lse;
  int64_t seq, d, w;
  int causal;
  double scale;
  const int64_t *rows;
  int64_t i0, i1;
} attn_rows_job;

static void *attn_rows_worker(void *arg) {
  const attn_rows_job *jb = (const attn_rows_job *)arg;
  for (int64_t i = jb->i0; i < jb->i1; ++i)
    orc_attention_mode_rows(jb->q, jb->k, jb->v, jb->o + i * jb->d, jb->lse ? jb->lse + i : NULL, jb->seq,
                            jb->d, jb->w, jb->causal, jb->scale, jb->rows[i], jb->rows[i] + 1);
  return NULL;
}

void orc_attention_rowlist_mt(const float *q, const float *k, const float *v, float *o, float *lse,
                              int64_t seq, int64_t d, int64_t w, int causal, double scale,
                              const int64_t *rows, int64_t nrows, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  attn_rows_job jobs[256];
  int nt = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t i0 = nrows * t / threads, i1 = nrows * (t + 1) / threads;
    if (i0 >= i1) continue;
    jobs[nt] = (attn_rows_job){q, k, v, o, lse, seq, d, w, causal, scale, rows, i0, i1};
    pthread_create(&th[nt], NULL, attn_rows_worker, &jobs[nt]);
    ++nt;
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* Attention backward for one head: the gradients of o = softmax(scale q k^T) v
 * (key ranges as key_range) with respect to q, k, v, given do.  No reference
 * counterpart (the reference has no backward): the
 * standard derivation, evaluated in f64 —
 *   P = softmax rows, dV = P^T dO, dP = dO V^T, D_i = sum_j P_ij dP_ij,
 *   dS = P (dP - D), dQ = scale dS K, dK = scale dS^T Q. */
void orc_attention_bwd(const float *q, const float *k, const float *v, const float *dout,
                       float *dq, float *dk, float *dv, int64_t seq, int64_t d, int64_t w,
                       int causal, double scale) {
  double *p = (double *)malloc(sizeof(double) * (size_t)(seq > 0 ? seq : 1));
  double *dqa = (double *)calloc((size_t)(seq * d > 0 ? seq * d : 1), sizeof(double));
  double *dka = (double *)calloc((size_t)(seq * d > 0 ? seq * d : 1), sizeof(double));
  double *dva = (double *)calloc((size_t)(seq * d > 0 ? seq * d : 1), sizeof(double));
  for (int64_t i = 0; i < seq; ++i) {
    int64_t j0, j1;
    key_range(i, seq, w, causal, &j0, &j1);
    const int64_t cnt = j1 - j0 + 1;
    double m = -INFINITY;
    for (int64_t t = 0; t < cnt; ++t) {
      double s = 0;
      for (int64_t x = 0; x < d; ++x) s += (double)q[i * d + x] * k[(j0 + t) * d + x];
      p[t] = s * scale;
      m = p[t] > m ? p[t] : m;
    }
    double l = 0;
    for (int64_t t = 0; t < cnt; ++t) {
      p[t] = exp(p[t] - m);
      l += p[t];
    }
    double di = 0;
    for (int64_t t = 0; t < cnt; ++t) {
      p[t] /= l;
      double dp = 0;
      for (int64_t x = 0; x < d; ++x) dp += (double)dout[i * d + x] * v[(j0 + t) * d + x];
      di += p[t] * dp;
    }
    for (int64_t t = 0; t < cnt; ++t) {
      const int64_t j = j0 + t;
      double dp = 0;
      for (int64_t x = 0; x < d; ++x) dp += (double)dout[i * d + x] * v[j * d + x];
      const double ds = p[t] * (dp - di);
      for (int64_t x = 0; x < d; ++x) {
        dva[j * d + x] += p[t] * dout[i * d + x];
        dqa[i * d + x] += scale * ds * k[j * d + x];
        dka[j * d + x] += scale * ds * q[i * d + x];
      }
    }
  }
  for (int64_t e = 0; e < seq * d; ++e) {
    dq[e] = (float)dqa[e];
    dk[e] = (float)dka[e];
    dv[e] = (float)dva[e];
  }
  free(p);
  free(dqa);
  free(dka);
  free(dva);
}

/* Trilinear attention with asymmetric causal windows
 * (core/src/oracles.cpp:82-117). */
void orc_simplicial_attention(const float *q, const float *k1, const float *v1,
                              const float *k2, const float *v2, float *o,
                              float *lse, int64_t seq, int64_t d, int64_t w1,
                              int64_t w2, double scale) {
  size_t cap = (size_t)((w1 < seq ? w1 : seq) * (w2 < seq ? w2 : seq) + 1);
  double *scores = (double *)malloc(sizeof(double) * cap);
  int64_t *pj1 = (int64_t *)malloc(sizeof(int64_t) * cap);
  int64_t *pj2 = (int64_t *)malloc(sizeof(int64_t) * cap);
  memset(o, 0, sizeof(float) * (size_t)(seq * d));
  for (int64_t i = 0; i < seq; ++i) {
    int64_t cnt = 0;
    for (int64_t j1 = (i - w1 + 1 > 0 ? i - w1 + 1 : 0); j1 <= i; ++j1)
      for (int64_t j2 = (i - w2 + 1 > 0 ? i - w2 + 1 : 0); j2 <= i; ++j2) {
        double s = 0;
        for (int64_t x = 0; x < d; ++x)
          s += (double)q[i * d + x] * k1[j1 * d + x] * k2[j2 * d + x];
        pj1[cnt] = j1;
        pj2[cnt] = j2;
        scores[cnt++] = s * scale;
      }
    double m = -INFINITY;
    for (int64_t t = 0; t < cnt; ++t) m = scores[t] > m ? scores[t] : m;
    double l = 0;
    for (int64_t t = 0; t < cnt; ++t) l += exp(scores[t] - m);
    for (int64_t t = 0; t < cnt; ++t) {
      double p = exp(scores[t] - m) / l;
      for (int64_t x = 0; x < d; ++x)
        o[i * d + x] += (float)(p * v1[pj1[t] * d + x] * v2[pj2[t] * d + x]);
    }
    lse[i] = (float)(m + log(l));
  }
  free(scores);
  free(pj1);
  free(pj2);
}

/* LayerNorm over rows (core/src/oracles.cpp:28-55). */
void orc_layernorm(const float *x, const float *w, const float *b, double eps,
                   float *y, float *mean, float *rstd, int64_t rows, int64_t n) {
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0;
    for (int64_t j = 0; j < n; ++j) s += x[r * n + j];
    double mu = s / (double)n;
    double v = 0;
    for (int64_t j = 0; j < n; ++j) {
      double dd = x[r * n + j] - mu;
      v += dd * dd;
    }
    v /= (double)n;
    double rs = 1.0 / sqrt(v + eps);
    if (mean) mean[r] = (float)mu;
    if (rstd) rstd[r] = (float)rs;
    for (int64_t j = 0; j < n; ++j)
      y[r * n + j] = (float)((x[r * n + j] - mu) * rs * w[j] + b[j]);
  }
}

/* ---------------------------------------------------------------------- */
/* MIMWTNSR flat tensor files (core/src/tensor_io.cpp:10, 30-78):          */
/* "MIMWTNSR", u32 rank, u32 extents, little-endian f32 payload.           */
/* ---------------------------------------------------------------------- */
int orc_write_tensor(const char *path, const float *data, const int64_t *shape,
                     int rank) {
  FILE *f = fopen(path, "wb");
  if (!f) return 1;
  fwrite("MIMWTNSR", 1, 8, f);
  uint32_t r = (uint32_t)rank;
  fwrite(&r, 4, 1, f);
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) {
    uint32_t e = (uint32_t)shape[i];
    fwrite(&e, 4, 1, f);
    n *= shape[i];
  }
  fwrite(data, 4, (size_t)n, f);
  fclose(f);
  return 0;
}
