/* fms_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of Faster Mean-shift.
 *
 * TEST INFRASTRUCTURE ONLY (see fms_oracle.h).  "P:n" = PAPER.md line n; "R#" = DESIGN.md reading.
 * Pins (tests/test_oracle_*.py, -m "not gpu"): P1 fixed points, P2 monotone ascent, P3 non-empty
 * windows, P4 closed-form centres, P5 exact recovery, P6 reduction to Alg. 1 (independent numpy
 * brute force), P7 sklearn radius/nearest-neighbour routines, P8 Eq. 14/19 closed forms and the
 * SPEC worked values, P9 selection determinism/uniformity.  No function here is "parity unpinned".
 */
#include "fms_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int fmso_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------------------------------
 * Seed selection key (R11: "Evenly random select seed vector set", Alg. 2 line 2).
 * splitmix64 (Steele/Lea/Flood) of rng_seed ^ (round+1)*0xD1B54A32D192ED03 ^ i.  The map is a
 * bijection of uint64, so keys of distinct pixels of one round never tie.
 * ------------------------------------------------------------------------------------------- */
uint64_t fmso_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t fmso_key(uint64_t rng_seed, int32_t round, int64_t i) {
  uint64_t salt = (uint64_t)(round + 1) * 0xD1B54A32D192ED03ULL;
  return fmso_splitmix64(rng_seed ^ salt ^ (uint64_t)i);
}

/* ---------------------------------------------------------------------------------------------
 * OSOP scalars.
 * Eq. 14:  P_seed/cluster = (1 - (1 - r/I)^N)^I
 * Eq. 19:  N_min = ln(1 - e^{ln(P)/I}) / ln(1 - r/I), rounded up to an integer
 *                      (R15: r/I exactly as printed in Eq. 19).
 * ------------------------------------------------------------------------------------------- */
double fmso_p_success(int64_t N, int64_t I, double r) {
  double q = r / (double)I;
  return pow(1.0 - pow(1.0 - q, (double)N), (double)I);
}

int64_t fmso_n_min(double P, int64_t I, double r) {
  if (I <= 0 || !(r > 0.0)) return INT64_MAX; /* nothing observed: keep seeding (R13) */
  double q = r / (double)I;
  if (q >= 1.0) return 1;
  double num = log(-expm1(log(P) / (double)I)); /* ln(1 - e^{ln P / I}) */
  double den = log1p(-q);                        /* ln(1 - r/I) */
  double v = ceil(num / den);
  if (v < 1.0) v = 1.0;
  if (v > 4.0e18) return INT64_MAX;
  return (int64_t)v;
}

/* R8: "If more than gamma percentage of the seed vectors are converged" -> the batch
 * stops once converged >= ceil(gamma*K); the 1e-9 guard keeps gamma*K that is an integer in exact
 * arithmetic from rounding one ulp up. */
int32_t fmso_need(double gamma, int64_t K) {
  double v = ceil(gamma * (double)K - 1e-9);
  if (v < 0.0) v = 0.0;
  return (int32_t)v;
}

/* O8 (NEXT-1): the seed count carried to the next frame of a sequence.  P:318: "The N will be
 * doubled for the next iteration [within a frame, R12] ... if N is too large compared to N_min, N
 * is reduced as N - N_min" with "too large" = N > H N_min (Eq. 21's upper bound, H = 8 P:318);
 * R18: floor at N_min.  The frame's N is the total number of seeds it used; N_min is the last
 * estimate (Eq. 19) of the frame. */
int64_t fmso_session_next(int64_t total, double nmin, double H) {
  if (!(nmin > 0.0)) return total; /* N_min infinite: nothing to reduce against */
  if ((double)total > H * nmin) {
    const int64_t m = (int64_t)nmin;
    const int64_t v = total - m;
    return v > m ? v : m;
  }
  return total;
}

/* ---------------------------------------------------------------------------------------------
 * Eq. 1 / Eq. 9: cosine distance is 1 - x.y/(|x||y|), so every embedding is
 * divided by its Euclidean norm once.  A zero or non-finite norm has no direction -> error.
 * ------------------------------------------------------------------------------------------- */
int fmso_normalize(const float* emb, int64_t n, int32_t d, double* xhat) {
  for (int64_t i = 0; i < n; ++i) {
    double ss = 0.0;
    for (int32_t k = 0; k < d; ++k) ss += (double)emb[i * d + k] * (double)emb[i * d + k];
    double nrm = sqrt(ss);
    if (!(nrm > 0.0) || !isfinite(nrm)) return FMSO_E_ZERO_NORM;
    for (int32_t k = 0; k < d; ++k) xhat[i * d + k] = (double)emb[i * d + k] / nrm;
  }
  return FMSO_OK;
}

/* ---------------------------------------------------------------------------------------------
 * Alg. 2 line 2: choose K of the candidate pixels "evenly random" (R11): the K candidates
 * with the smallest (key, index); the chosen indices are returned in ascending order.
 * ------------------------------------------------------------------------------------------- */
typedef struct { uint64_t key; int64_t i; } kv_t;

static int cmp_kv(const void* a, const void* b) {
  const kv_t* x = (const kv_t*)a;
  const kv_t* y = (const kv_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i);
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y);
}

int64_t fmso_select(const uint8_t* cand, int64_t n, int64_t K, uint64_t rng_seed, int32_t round,
                    int64_t* out) {
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) m += cand[i] ? 1 : 0;
  kv_t* all = (kv_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(kv_t));
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i)
    if (cand[i]) { all[c].key = fmso_key(rng_seed, round, i); all[c].i = i; ++c; }
  qsort(all, (size_t)m, sizeof(kv_t), cmp_kv);
  int64_t k = K < m ? K : m;
  for (int64_t j = 0; j < k; ++j) out[j] = all[j].i;
  qsort(out, (size_t)k, sizeof(int64_t), cmp_i64);
  free(all);
  return k;
}

/* ---------------------------------------------------------------------------------------------
 * Eq. 8 gated by the flat kernel Eq. 11, read as R1 (Eq. 10's printed
 * "mean of distances" is a typo for the vector mean):
 *     S_h(s) = { x_i : d(s, x_i) <= h } = { x_i : x_i.s >= tau },  tau = 1 - h   (R5, inclusive)
 *     g(s)   = sum_{x_i in S_h(s)} x_i    (ascending i)
 * The count m = |S_h(s)| is returned; m_h = g/m.  Dense evaluation over all points, as P:210
 * says ("does not search which points belong to S_h ... multiplies ... with the kernel").
 * ------------------------------------------------------------------------------------------- */
int64_t fmso_window(const double* xhat, int64_t n, int32_t d, double tau, const double* s,
                    double* g) {
  int64_t cnt = 0;
  for (int32_t k = 0; k < d; ++k) g[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double* x = xhat + i * d;
    double dot = 0.0;
    for (int32_t k = 0; k < d; ++k) dot += x[k] * s[k];
    if (dot >= tau) {
      for (int32_t k = 0; k < d; ++k) g[k] += x[k];
      ++cnt;
    }
  }
  return cnt;
}

/* ---------------------------------------------------------------------------------------------
 * NEXT-4, reading R23: Eq. 2 admits any profile k; the Gaussian profile
 * k(t) = exp(-t/2) with t = |x - s|^2 / h, and |x - s|^2 = 2 (1 - x.s) for unit vectors (Eq. 9), gives
 *     w_i = exp(-(1 - x_i.s) / h),   g(s) = sum_i w_i x_i   (ascending i; every point contributes)
 * and the mean-shift vector (Eq. 5-6 with g = -k' proportional to k) is g / sum_i w_i.
 * ------------------------------------------------------------------------------------------- */
double fmso_window_gauss(const double* xhat, int64_t n, int32_t d, double h, const double* s, double* g) {
  double wsum = 0.0;
  for (int32_t k = 0; k < d; ++k) g[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double* x = xhat + i * d;
    double dot = 0.0;
    for (int32_t k = 0; k < d; ++k) dot += x[k] * s[k];
    const double w = exp(-(1.0 - dot) / h);
    for (int32_t k = 0; k < d; ++k) g[k] += w * x[k];
    wsum += w;
  }
  return wsum;
}

/* ---------------------------------------------------------------------------------------------
 * Alg. 2 lines 4-9 with the convergence rule of P:223 and early stopping:
 * all active seeds advance once per lockstep iteration (the batched-tensor form of P:210):
 *     s' = m_h(s)/|m_h(s)| = g/|g|              (R4: renormalised onto the unit sphere)
 *     converged if |s' - s|_2 < tol             (R6: "change ... less than ... h/1,000")
 * Converged seeds freeze (R9).  The batch stops once converged >= ceil(gamma*K) (R8) or no seed is
 * active; seeds still moving are "discarded from the seed vector".  An empty window
 * (impossible for seeds started at data points, pin P3) marks the seed stalled.  Each converged
 * mode gets its intensity = |S_h(m)| (density of Eq. 2 at the mode, R10).
 * ------------------------------------------------------------------------------------------- */
int32_t fmso_lockstep(const double* xhat, int64_t n, int32_t d, double h, int32_t max_iter,
                      double tol, double gamma, int64_t K, double* seeds, uint8_t* status,
                      int64_t* intensity, int32_t* iters, int64_t* seed_iters) {
  return fmso_lockstep_p(xhat, n, d, h, max_iter, tol, gamma, K, seeds, status, intensity, iters, seed_iters,
                         FMSO_PROFILE_FLAT);
}

/* the same with the profile of the update selectable (flat: the paper; Gaussian: NEXT-4, R23) */
int32_t fmso_lockstep_p(const double* xhat, int64_t n, int32_t d, double h, int32_t max_iter,
                        double tol, double gamma, int64_t K, double* seeds, uint8_t* status,
                        int64_t* intensity, int32_t* iters, int64_t* seed_iters, int32_t profile) {
  return fmso_lockstep_m(xhat, n, d, h, max_iter, tol, gamma, K, seeds, status, intensity, iters, seed_iters,
                         profile, FMSO_METRIC_COSINE);
}

/* ---------------------------------------------------------------------------------------------
 * NEXT-4, reading R24: Eq. 3's flat kernel with the Euclidean distance of Eq. 4, which
 * Eq. 9 replaces on the paper's cosine path:
 *     S_h(s) = { x_i : |x_i - s|_2 <= h },   m_h(s) = (1/|S_h(s)|) sum_{S_h(s)} x_i   (Eq. 8 / 10)
 * on the raw embeddings (no normalisation, no renormalisation of the shifted seed).
 * ------------------------------------------------------------------------------------------- */
int64_t fmso_window_euclid(const double* x, int64_t n, int32_t d, double h, const double* s, double* g) {
  int64_t cnt = 0;
  const double h2 = h * h;
  for (int32_t k = 0; k < d; ++k) g[k] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double* xi = x + i * d;
    double d2 = 0.0;
    for (int32_t k = 0; k < d; ++k) d2 += (xi[k] - s[k]) * (xi[k] - s[k]);
    if (d2 <= h2) {
      for (int32_t k = 0; k < d; ++k) g[k] += xi[k];
      ++cnt;
    }
  }
  return cnt;
}

int32_t fmso_lockstep_m(const double* xhat, int64_t n, int32_t d, double h, int32_t max_iter,
                        double tol, double gamma, int64_t K, double* seeds, uint8_t* status,
                        int64_t* intensity, int32_t* iters, int64_t* seed_iters, int32_t profile,
                        int32_t metric) {
  const double tau = 1.0 - h;
  const int euclid = metric == FMSO_METRIC_EUCLID;
  const int32_t need = fmso_need(gamma, K);
  int32_t t_run = 0;
  *seed_iters = 0;
  for (int64_t j = 0; j < K; ++j) { status[j] = 0; intensity[j] = 0; iters[j] = 0; }
  for (int32_t t = 1; t <= max_iter; ++t) {
    int64_t active = 0;
    for (int64_t j = 0; j < K; ++j) active += status[j] == 0;
    if (active == 0) break;
    *seed_iters += active;
    t_run = t;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t j = 0; j < K; ++j) {
      if (status[j] != 0) continue;
      double g[256], sn[256];
      double* s = seeds + j * d;
      const double mass = euclid ? (double)fmso_window_euclid(xhat, n, d, h, s, g)
                          : profile == FMSO_PROFILE_GAUSS ? fmso_window_gauss(xhat, n, d, h, s, g)
                                                          : (double)fmso_window(xhat, n, d, tau, s, g);
      if (mass == 0.0) { status[j] = 2; continue; }
      double nn = 0.0;
      for (int32_t k = 0; k < d; ++k) nn += g[k] * g[k];
      nn = euclid ? mass : sqrt(nn);  /* Euclidean: the window mean; cosine: onto the sphere (R4) */
      double dd = 0.0;
      for (int32_t k = 0; k < d; ++k) {
        sn[k] = g[k] / nn;
        dd += (sn[k] - s[k]) * (sn[k] - s[k]);
      }
      for (int32_t k = 0; k < d; ++k) s[k] = sn[k];
      iters[j] = t;
      if (sqrt(dd) < tol) status[j] = 1;
    }
    int64_t conv = 0, still = 0;
    for (int64_t j = 0; j < K; ++j) { conv += status[j] == 1; still += status[j] == 0; }
    if (conv >= need || still == 0) break;
  }
  for (int64_t j = 0; j < K; ++j)
    if (status[j] == 0) status[j] = 3;
  /* intensity of a converged mode m (R10): the flat-kernel density of Eq. 2 at m up to the constant
   * 1/(n h^d), i.e. the number of points in the window centred on m. */
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t j = 0; j < K; ++j) {
    if (status[j] != 1) continue;
    double g[256];
    intensity[j] = euclid ? fmso_window_euclid(xhat, n, d, h, seeds + j * d, g)
                          : fmso_window(xhat, n, d, tau, seeds + j * d, g);
  }
  return t_run;
}

/* ---------------------------------------------------------------------------------------------
 * "Prune modes" (Alg. 1 l.12, Alg. 2 l.10; "pruned and merged if their distance is small")
 * read as R10: visit the pool in (intensity desc, origin asc) order and keep a mode unless a kept
 * centre lies within cosine distance rho (Eq. 9) of it.  Kept modes are not averaged, so every
 * centre stays an actual mean-shift fixed point.
 * ------------------------------------------------------------------------------------------- */
typedef struct { int64_t inten, origin, idx; } mrank_t;

static int cmp_mrank(const void* a, const void* b) {
  const mrank_t* x = (const mrank_t*)a;
  const mrank_t* y = (const mrank_t*)b;
  if (x->inten != y->inten) return x->inten > y->inten ? -1 : 1;
  if (x->origin != y->origin) return x->origin < y->origin ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

int64_t fmso_merge(const double* pool, const int64_t* intensity, const int64_t* origin, int64_t m,
                   int32_t d, double rho, int64_t* keep) {
  return fmso_merge_m(pool, intensity, origin, m, d, rho, keep, FMSO_METRIC_COSINE);
}

int64_t fmso_merge_m(const double* pool, const int64_t* intensity, const int64_t* origin, int64_t m,
                     int32_t d, double rho, int64_t* keep, int32_t metric) {
  mrank_t* ord = (mrank_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(mrank_t));
  for (int64_t j = 0; j < m; ++j) { ord[j].inten = intensity[j]; ord[j].origin = origin[j]; ord[j].idx = j; }
  qsort(ord, (size_t)m, sizeof(mrank_t), cmp_mrank);
  int64_t kept = 0;
  for (int64_t o = 0; o < m; ++o) {
    const double* a = pool + ord[o].idx * d;
    int ok = 1;
    for (int64_t q = 0; q < kept && ok; ++q) {
      const double* b = pool + keep[q] * d;
      if (metric == FMSO_METRIC_EUCLID) {
        double d2 = 0.0;
        for (int32_t k = 0; k < d; ++k) d2 += (a[k] - b[k]) * (a[k] - b[k]);
        if (d2 <= rho * rho) ok = 0;
      } else {
        double dot = 0.0;
        for (int32_t k = 0; k < d; ++k) dot += a[k] * b[k];
        if (1.0 - dot <= rho) ok = 0;
      }
    }
    if (ok) keep[kept++] = ord[o].idx;
  }
  free(ord);
  return kept;
}

/* ---------------------------------------------------------------------------------------------
 * Alg. 2 lines 12-14 ("all vectors are clustered according to their distance to
 * each mode"): label = argmin_k d(x, c_k) = argmax_k x.c_k, ties -> lowest k (R21).
 * covered = the nearest centre's window contains x (max_k x.c_k >= tau), used by OSOP re-seeding.
 * ------------------------------------------------------------------------------------------- */
void fmso_assign(const double* xhat, int64_t n, int32_t d, const double* centres, int64_t K,
                 double tau, int32_t* labels, uint8_t* covered, int64_t* hist) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* x = xhat + i * d;
    double best = -INFINITY;
    int32_t lab = 0;
    for (int64_t k = 0; k < K; ++k) {
      double dot = 0.0;
      for (int32_t q = 0; q < d; ++q) dot += x[q] * centres[k * d + q];
      if (dot > best) { best = dot; lab = (int32_t)k; }
    }
    labels[i] = lab;
    covered[i] = best >= tau ? 1 : 0;
  }
  for (int64_t k = 0; k < K; ++k) hist[k] = 0;
  for (int64_t i = 0; i < n; ++i) hist[labels[i]]++;
}

void fmso_assign_m(const double* x, int64_t n, int32_t d, const double* centres, int64_t K, double h,
                   int32_t* labels, uint8_t* covered, int64_t* hist, int32_t metric) {
  if (metric != FMSO_METRIC_EUCLID) {
    fmso_assign(x, n, d, centres, K, 1.0 - h, labels, covered, hist);
    return;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* xi = x + i * d;
    double best = INFINITY;
    int32_t lab = 0;
    for (int64_t k = 0; k < K; ++k) {
      double d2 = 0.0;
      for (int32_t q = 0; q < d; ++q) d2 += (xi[q] - centres[k * d + q]) * (xi[q] - centres[k * d + q]);
      if (d2 < best) { best = d2; lab = (int32_t)k; }
    }
    labels[i] = lab;
    covered[i] = best <= h * h ? 1 : 0;
  }
  for (int64_t k = 0; k < K; ++k) hist[k] = 0;
  for (int64_t i = 0; i < n; ++i) hist[labels[i]]++;
}

/* ---------------------------------------------------------------------------------------------
 * OSOP observation ("I and r are calculated from the predicted segmentation"; SPEC S:263-270
 * estimate_observation).  hist[k] = #pixels labelled k.  With has_background the largest cluster
 * (lowest k on ties) is the background (R14); I = #clusters other than the background with at least
 * min_instance_px pixels (R22; 0 = every cluster counts); r = 1 - |background| / n (the foreground
 * ratio of Eq. 13), or r = 1 without a background.  Returns the background index (-1 if none).
 * ------------------------------------------------------------------------------------------- */
int64_t fmso_observe(const int64_t* hist, int64_t K, int64_t n, int32_t has_background, int32_t min_instance_px,
                     int32_t* I_out, double* r_out) {
  int64_t bg = -1;
  if (has_background && K > 0) {
    bg = 0;
    for (int64_t k = 1; k < K; ++k)
      if (hist[k] > hist[bg]) bg = k;
  }
  int32_t I = 0;
  for (int64_t k = 0; k < K; ++k)
    if (k != bg && hist[k] >= min_instance_px) ++I;
  if (I_out) *I_out = I;
  if (r_out) *r_out = bg >= 0 ? 1.0 - (double)hist[bg] / (double)n : 1.0;
  return bg;
}

/* OSOP stop rule after round `round` (P:318 + R13, R22): stop when no uncovered unvisited pixel
 * remains (ncand == 0), every pixel has been a seed (total >= n), the round cap is reached, the seeds
 * used so far reach L * N_min (Eq. 21's lower bound; nmin = INT64_MAX is infinite), or -- with
 * saturation_stop -- the round did not raise the observed instance count (I <= I_prev, round >= 1).
 * Returns 1 to stop, 0 to run another round with "N doubled" (K_next = min(total, ncand)). */
int fmso_osop_stop(int64_t ncand, int64_t total, int64_t n, int32_t round, int32_t max_rounds, int64_t nmin,
                   double L, int32_t saturation_stop, int32_t I, int32_t I_prev) {
  if (ncand == 0 || total >= n || round + 1 >= max_rounds) return 1;
  if (nmin != INT64_MAX && (double)total >= L * (double)nmin) return 1;
  if (saturation_stop && round >= 1 && I <= I_prev) return 1;
  return 0;
}

/* ---------------------------------------------------------------------------------------------
 * The whole method: Alg. 2 wrapped in the OSOP controller of Fig. 3 / P:316-318.
 *   round 0: K_0 = N_initial (OSOP), n_seeds (FIXED) or n (ALL = Alg. 1, gamma = 1)
 *   each round: select -> lockstep mean-shift -> merge with previous centres -> assign all pixels
 *   OSOP (R12-R14, R22): observe I, r from the segmentation (background = largest cluster),
 *   N_min by Eq. 19; stop once total >= L*N_min, or no uncovered unvisited pixel remains, or all
 *   pixels were seeds, or max_rounds, or (saturation_stop) the round added no counted instance;
 *   otherwise "N will be doubled": K_next = min(total, #candidates) seeds from pixels not covered
 *   by any converged cluster (north_star reading R13).
 * ------------------------------------------------------------------------------------------- */
int fmso_cluster(const float* emb, int64_t n, int32_t d, double h, int32_t max_iter, double tol,
                 const fmso_policy* pol, int32_t* labels, double* centres, int32_t centres_cap,
                 int32_t* K_out, fmso_trace* trace) {
  if (!pol) return FMSO_E_INVALID;
  const int euclid = pol->metric == FMSO_METRIC_EUCLID;
  if (n < 1 || d < 1 || d > 256 || !(h > 0.0 && (euclid || h < 1.0)) || !(tol > 0.0) || max_iter < 1)
    return FMSO_E_INVALID;
  if (pol->metric != FMSO_METRIC_COSINE && (!euclid || pol->profile != FMSO_PROFILE_FLAT)) return FMSO_E_INVALID;
  if (pol->kind < 0 || pol->kind > 2 || pol->max_rounds < 1 || pol->max_rounds > FMSO_MAX_ROUNDS)
    return FMSO_E_INVALID;
  if (pol->kind != FMSO_SEEDS_ALL && pol->n_seeds < 1) return FMSO_E_INVALID;
  if (!(pol->gamma > 0.0 && pol->gamma <= 1.0)) return FMSO_E_INVALID;
  if (pol->kind == FMSO_SEEDS_OSOP && (!(pol->P > 0.0 && pol->P < 1.0) || !(pol->L > 0.0)))
    return FMSO_E_INVALID;
  if (pol->profile != FMSO_PROFILE_FLAT && pol->profile != FMSO_PROFILE_GAUSS) return FMSO_E_INVALID;

  const double tau = 1.0 - h;
  const double rho = h;
  int rc = FMSO_OK;
  double* xhat = (double*)malloc((size_t)n * d * sizeof(double));
  uint8_t* visited = (uint8_t*)calloc((size_t)n, 1);
  uint8_t* covered = (uint8_t*)calloc((size_t)n, 1);
  uint8_t* cand = (uint8_t*)malloc((size_t)n);
  int64_t* idx = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t cap = 64;
  double* cvec = (double*)malloc((size_t)cap * d * sizeof(double));
  int64_t* cint = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
  int64_t* corg = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
  int64_t Kc = 0;
  int64_t* hist = NULL;
  fmso_trace tr;
  memset(&tr, 0, sizeof(tr));

  if (euclid) {  /* R24: the raw embeddings (Eq. 4 needs no normalisation) */
    for (int64_t i = 0; i < n * d; ++i) xhat[i] = (double)emb[i];
  } else {
    rc = fmso_normalize(emb, n, d, xhat);
    if (rc != FMSO_OK) goto done;
  }

  int64_t total = 0, K_next = 0;
  int32_t I_prev = -1;
  for (int32_t round = 0; round < pol->max_rounds; ++round) {
    int64_t ncand = 0;
    for (int64_t i = 0; i < n; ++i) {
      cand[i] = round == 0 ? 1 : (!covered[i] && !visited[i]);
      ncand += cand[i];
    }
    int64_t Kreq = round == 0 ? (pol->kind == FMSO_SEEDS_ALL ? n : (int64_t)pol->n_seeds) : K_next;
    int64_t Kr = fmso_select(cand, n, Kreq, pol->rng_seed, round, idx);
    for (int64_t j = 0; j < Kr; ++j) visited[idx[j]] = 1;
    total += Kr;

    double* seeds = (double*)malloc((size_t)(Kr > 0 ? Kr : 1) * d * sizeof(double));
    uint8_t* st = (uint8_t*)malloc((size_t)(Kr > 0 ? Kr : 1));
    int64_t* inten = (int64_t*)malloc((size_t)(Kr > 0 ? Kr : 1) * sizeof(int64_t));
    int32_t* its = (int32_t*)malloc((size_t)(Kr > 0 ? Kr : 1) * sizeof(int32_t));
    for (int64_t j = 0; j < Kr; ++j) memcpy(seeds + j * d, xhat + idx[j] * d, (size_t)d * sizeof(double));
    double gam = pol->kind == FMSO_SEEDS_ALL ? 1.0 : pol->gamma;
    int64_t sit = 0;
    int32_t t_run = fmso_lockstep_m(xhat, n, d, h, max_iter, tol, gam, Kr, seeds, st, inten, its, &sit,
                                    pol->profile, pol->metric);

    int64_t nconv = 0, ndisc = 0;
    for (int64_t j = 0; j < Kr; ++j) { nconv += st[j] == 1; ndisc += st[j] != 1; }
    tr.round_K[round] = (int32_t)Kr;
    tr.round_iters[round] = t_run;
    tr.round_conv[round] = (int32_t)nconv;
    tr.round_disc[round] = (int32_t)ndisc;
    tr.round_seed_iters[round] = sit;
    tr.seeds_total += Kr;
    tr.seed_iters += sit;
    tr.discarded += ndisc;
    tr.rounds = round + 1;
    if (round == 0 && nconv == 0) {
      free(seeds); free(st); free(inten); free(its);
      rc = FMSO_E_STALLED;
      goto done;
    }

    /* merge: pool = previous centres U this round's converged modes */
    int64_t m = Kc + nconv;
    double* pool = (double*)malloc((size_t)m * d * sizeof(double));
    int64_t* pint = (int64_t*)malloc((size_t)m * sizeof(int64_t));
    int64_t* porg = (int64_t*)malloc((size_t)m * sizeof(int64_t));
    int64_t* keep = (int64_t*)malloc((size_t)m * sizeof(int64_t));
    memcpy(pool, cvec, (size_t)Kc * d * sizeof(double));
    memcpy(pint, cint, (size_t)Kc * sizeof(int64_t));
    memcpy(porg, corg, (size_t)Kc * sizeof(int64_t));
    int64_t p = Kc;
    for (int64_t j = 0; j < Kr; ++j)
      if (st[j] == 1) {
        memcpy(pool + p * d, seeds + j * d, (size_t)d * sizeof(double));
        pint[p] = inten[j];
        porg[p] = idx[j];
        ++p;
      }
    int64_t kept = fmso_merge_m(pool, pint, porg, m, d, rho, keep, pol->metric);
    if (kept > cap) {
      cap = kept * 2;
      cvec = (double*)realloc(cvec, (size_t)cap * d * sizeof(double));
      cint = (int64_t*)realloc(cint, (size_t)cap * sizeof(int64_t));
      corg = (int64_t*)realloc(corg, (size_t)cap * sizeof(int64_t));
    }
    for (int64_t q = 0; q < kept; ++q) {
      memcpy(cvec + q * d, pool + keep[q] * d, (size_t)d * sizeof(double));
      cint[q] = pint[keep[q]];
      corg[q] = porg[keep[q]];
    }
    Kc = kept;
    free(pool); free(pint); free(porg); free(keep);
    free(seeds); free(st); free(inten); free(its);

    /* assign every pixel to its nearest centre */
    free(hist);
    hist = (int64_t*)malloc((size_t)Kc * sizeof(int64_t));
    fmso_assign_m(xhat, n, d, cvec, Kc, h, labels, covered, hist, pol->metric);
    int64_t ncand2 = 0;
    for (int64_t i = 0; i < n; ++i) ncand2 += (!covered[i] && !visited[i]);
    tr.round_Kc[round] = (int32_t)Kc;
    tr.round_cand[round] = ncand2;

    if (pol->kind != FMSO_SEEDS_OSOP) break;

    /* OSOP (Eq. 12-19) */
    int32_t I = 0;
    double r = 1.0;
    fmso_observe(hist, Kc, n, pol->has_background, pol->min_instance_px, &I, &r);
    int64_t nmin = fmso_n_min(pol->P, I, r);
    tr.round_I[round] = I;
    tr.round_r[round] = r;
    tr.round_nmin[round] = nmin == INT64_MAX ? -1.0 : (double)nmin;
    int stop = fmso_osop_stop(ncand2, total, n, round, pol->max_rounds, nmin, pol->L, pol->saturation_stop, I,
                              I_prev);
    I_prev = I;
    if (stop) break;
    K_next = total < ncand2 ? total : ncand2;
  }

  tr.K = (int32_t)Kc;
  if (K_out) *K_out = (int32_t)Kc;
  if (Kc > centres_cap) {
    rc = FMSO_E_CAPACITY;
  } else if (centres) {
    memcpy(centres, cvec, (size_t)Kc * d * sizeof(double));
  }

done:
  if (trace) *trace = tr;
  free(xhat); free(visited); free(covered); free(cand); free(idx);
  free(cvec); free(cint); free(corg); free(hist);
  return rc;
}
