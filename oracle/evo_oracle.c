/*
 * evo_oracle.c — plain fp64 CPU oracle for Evoformer gated multi-head attention with
 * pair bias (forward and backward).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2404_11068_b200/) never imports, links or calls it, and it shares no code,
 * header, table or constant with the CUDA path.
 *
 * What it computes (the plain definition; FlashAttention-style tiling is exact, so the
 * GPU method must reach this result up to rounding):
 *   PAPER.md L294 (§3.3.1 "Multi Head Attention"): "a pair bias term is added to the
 *     logits matrix before the softmax operation"; the kernel fuses "all operations in MHA".
 *   PAPER.md L169 (§2.1): the four MHA modules (row, column, triangle start, triangle end).
 *   SPEC.md L155-173 (attn_pair_bias_fwd/bwd): o = sigmoid(g) ⊙ (softmax(q·kᵀ·scale+bias)·v),
 *     bias [B,H,L,L] or broadcast [H,L,L]; recomputation backward; dbias reduced over the
 *     broadcast batch axis.
 *   AF2 supplementary Alg. 7 l.4-6 / Alg. 13 l.4-6 (cited by PAPER.md L178): gate
 *     g = sigmoid(Linear(x)), o = g ⊙ Σ_k a_k v_k.
 *   Mask convention (reading R5): hard mask; masked keys get weight
 *   exactly 0; a query row with no surviving key gives o = 0, lse = -inf, and contributes
 *   nothing to any gradient.
 *
 * Layouts (all contiguous, row-major, fp64):
 *   q, g, o, dout, dq, dg : [B][H][Lq][D]
 *   k, v, dk, dv          : [B][H][Lk][D]
 *   bias, dbias           : [H][Lq][Lk] (kind 1, shared over B) or [B][H][Lq][Lk] (kind 2)
 *   mask                  : [B][Lk] uint8, 1 keep / 0 drop (NULL = keep all)
 *   lse                   : [B][H][Lq]
 * No -ffast-math: IEEE exp/log.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_E_ARG 1
#define ORACLE_E_NOMEM 2

/* sigma(x) = 1 / (1 + e^-x)   (AF2 Alg. 7 line 4) */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

static const double* bias_row(int bias_kind, const double* bias, int64_t b, int64_t h,
                              int64_t H, int64_t Lq, int64_t Lk, int64_t qi) {
  if (bias_kind == 1) return bias + ((h * Lq) + qi) * Lk;
  if (bias_kind == 2) return bias + (((b * H + h) * Lq) + qi) * Lk;
  return NULL;
}

/*
 * Forward for one (b, h, qi) row, following SURVEY §8c "Forward" steps 1-4:
 *   1. s_k = scale * Σ_d Q[q,d] K[k,d] + bias(q,k), for every kept key k
 *   2. no kept key -> o = 0, lse = -inf
 *   3. m = max_k s_k; l = Σ_k exp(s_k - m); p_k = exp(s_k - m)/l (0 for masked); lse = m + ln l
 *   4. a_d = Σ_k p_k V[k,d]; o_d = sigma(G_d) a_d  (o = a without gate)
 * Writes p[Lk] (probabilities, 0 at masked keys) and a[D] (ungated attention output).
 * Returns 1 if the row has at least one kept key, 0 otherwise.
 */
static int row_forward(int64_t D, int64_t Lk, double scale, const double* qrow,
                       const double* kbase, const double* vbase, const double* brow,
                       const uint8_t* mrow, double* s, double* p, double* a, double* lse_out) {
  int any = 0;
  double m = -INFINITY;
  for (int64_t kk = 0; kk < Lk; ++kk) {
    if (mrow && !mrow[kk]) { s[kk] = 0.0; continue; }
    double dot = 0.0;
    for (int64_t d = 0; d < D; ++d) dot += qrow[d] * kbase[kk * D + d];
    s[kk] = scale * dot + (brow ? brow[kk] : 0.0);
    if (!any || s[kk] > m) m = s[kk];
    any = 1;
  }
  for (int64_t d = 0; d < D; ++d) a[d] = 0.0;
  if (!any) {
    for (int64_t kk = 0; kk < Lk; ++kk) p[kk] = 0.0;
    *lse_out = -INFINITY;
    return 0;
  }
  double l = 0.0;
  for (int64_t kk = 0; kk < Lk; ++kk) {
    if (mrow && !mrow[kk]) { p[kk] = 0.0; continue; }
    p[kk] = exp(s[kk] - m);
    l += p[kk];
  }
  for (int64_t kk = 0; kk < Lk; ++kk) p[kk] /= l;
  *lse_out = m + log(l);
  for (int64_t kk = 0; kk < Lk; ++kk) {
    if (p[kk] == 0.0) continue;
    for (int64_t d = 0; d < D; ++d) a[d] += p[kk] * vbase[kk * D + d];
  }
  return 1;
}

static int check_args(int64_t B, int64_t H, int64_t Lq, int64_t Lk, int64_t D, int bias_kind,
                      const double* bias) {
  if (B < 0 || H < 1 || Lq < 0 || Lk < 0 || D < 1) return ORACLE_E_ARG;
  if (bias_kind < 0 || bias_kind > 2) return ORACLE_E_ARG;
  if (bias_kind != 0 && bias == NULL) return ORACLE_E_ARG;
  return ORACLE_OK;
}

int oracle_attn_fwd(int64_t B, int64_t H, int64_t Lq, int64_t Lk, int64_t D, double scale,
                    const double* q, const double* k, const double* v, int bias_kind,
                    const double* bias, const uint8_t* mask, const double* g, double* o,
                    double* lse) {
  int rc = check_args(B, H, Lq, Lk, D, bias_kind, bias);
  if (rc) return rc;
  int err = 0;
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(Lk + 1));
    double* p = (double*)malloc(sizeof(double) * (size_t)(Lk + 1));
    double* a = (double*)malloc(sizeof(double) * (size_t)D);
    if (!s || !p || !a) {
#pragma omp atomic write
      err = 1;
    } else {
#pragma omp for collapse(2) schedule(static)
      for (int64_t b = 0; b < B; ++b)
        for (int64_t h = 0; h < H; ++h) {
          const double* kb = k + ((b * H + h) * Lk) * D;
          const double* vb = v + ((b * H + h) * Lk) * D;
          const uint8_t* mrow = mask ? mask + b * Lk : NULL;
          for (int64_t qi = 0; qi < Lq; ++qi) {
            int64_t row = (b * H + h) * Lq + qi;
            const double* brow = bias_row(bias_kind, bias, b, h, H, Lq, Lk, qi);
            row_forward(D, Lk, scale, q + row * D, kb, vb, brow, mrow, s, p, a, &lse[row]);
            for (int64_t d = 0; d < D; ++d)
              o[row * D + d] = g ? sigmoid(g[row * D + d]) * a[d] : a[d];
          }
        }
    }
    free(s); free(p); free(a);
  }
  return err ? ORACLE_E_NOMEM : ORACLE_OK;
}

/*
 * Backward (SURVEY §8c "Backward", derived in Appendix B and checked there in float64):
 *   1. dA = dO ⊙ sigma(G);  dG = dO ⊙ a ⊙ sigma(G)(1 - sigma(G))
 *   2. dp_k = Σ_d dA_d V[k,d];  D_q = Σ_k p_k dp_k
 *   3. ds_k = p_k (dp_k - D_q)
 *   4. dbias(h,q,k) += ds_k   (summed over b for the shared kind)
 *   5. dQ[q] += scale Σ_k ds_k K[k];  dK[k] += scale ds_k Q[q];  dV[k] += p_k dA
 * The probabilities are recomputed from the inputs (recompute backward).
 * Parallel over h; b runs serially inside so the shared dbias sum has a fixed order.
 */
int oracle_attn_bwd(int64_t B, int64_t H, int64_t Lq, int64_t Lk, int64_t D, double scale,
                    const double* q, const double* k, const double* v, int bias_kind,
                    const double* bias, const uint8_t* mask, const double* g,
                    const double* dout, double* dq, double* dk, double* dv, double* dg,
                    double* dbias) {
  int rc = check_args(B, H, Lq, Lk, D, bias_kind, bias);
  if (rc) return rc;
  memset(dq, 0, sizeof(double) * (size_t)(B * H * Lq * D));
  memset(dk, 0, sizeof(double) * (size_t)(B * H * Lk * D));
  memset(dv, 0, sizeof(double) * (size_t)(B * H * Lk * D));
  if (dg) memset(dg, 0, sizeof(double) * (size_t)(B * H * Lq * D));
  if (bias_kind == 1 && dbias) memset(dbias, 0, sizeof(double) * (size_t)(H * Lq * Lk));
  if (bias_kind == 2 && dbias) memset(dbias, 0, sizeof(double) * (size_t)(B * H * Lq * Lk));
  int err = 0;
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(Lk + 1));
    double* p = (double*)malloc(sizeof(double) * (size_t)(Lk + 1));
    double* dp = (double*)malloc(sizeof(double) * (size_t)(Lk + 1));
    double* a = (double*)malloc(sizeof(double) * (size_t)D);
    double* dA = (double*)malloc(sizeof(double) * (size_t)D);
    double lse_unused;
    if (!s || !p || !dp || !a || !dA) {
#pragma omp atomic write
      err = 1;
    } else {
#pragma omp for schedule(static)
      for (int64_t h = 0; h < H; ++h)
        for (int64_t b = 0; b < B; ++b) {
          const double* kb = k + ((b * H + h) * Lk) * D;
          const double* vb = v + ((b * H + h) * Lk) * D;
          double* dkb = dk + ((b * H + h) * Lk) * D;
          double* dvb = dv + ((b * H + h) * Lk) * D;
          const uint8_t* mrow = mask ? mask + b * Lk : NULL;
          for (int64_t qi = 0; qi < Lq; ++qi) {
            int64_t row = (b * H + h) * Lq + qi;
            const double* brow = bias_row(bias_kind, bias, b, h, H, Lq, Lk, qi);
            int live = row_forward(D, Lk, scale, q + row * D, kb, vb, brow, mrow, s, p, a,
                                   &lse_unused);
            if (!live) continue; /* fully masked row: zero contribution (reading R5) */
            /* step 1 */
            for (int64_t d = 0; d < D; ++d) {
              double go = dout[row * D + d];
              if (g) {
                double sg = sigmoid(g[row * D + d]);
                dA[d] = go * sg;
                dg[row * D + d] = go * a[d] * sg * (1.0 - sg);
              } else {
                dA[d] = go;
              }
            }
            /* step 2 */
            double Dq = 0.0;
            for (int64_t kk = 0; kk < Lk; ++kk) {
              double t = 0.0;
              for (int64_t d = 0; d < D; ++d) t += dA[d] * vb[kk * D + d];
              dp[kk] = t;
              Dq += p[kk] * t;
            }
            /* steps 3-5 */
            double* dbrow = NULL;
            if (dbias && bias_kind == 1) dbrow = dbias + ((h * Lq) + qi) * Lk;
            if (dbias && bias_kind == 2) dbrow = dbias + (((b * H + h) * Lq) + qi) * Lk;
            for (int64_t kk = 0; kk < Lk; ++kk) {
              if (mrow && !mrow[kk]) continue; /* masked key: weight exactly 0 */
              double ds = p[kk] * (dp[kk] - Dq);
              if (dbrow) dbrow[kk] += ds;
              for (int64_t d = 0; d < D; ++d) {
                dq[row * D + d] += scale * ds * kb[kk * D + d];
                dkb[kk * D + d] += scale * ds * q[row * D + d];
                dvb[kk * D + d] += p[kk] * dA[d];
              }
            }
          }
        }
    }
    free(s); free(p); free(dp); free(a); free(dA);
  }
  return err ? ORACLE_E_NOMEM : ORACLE_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
