/* fms_oracle.h -- plain fp64 CPU oracle of Faster Mean-shift (arXiv 2007.14283).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2007_14283_b200/), and neither includes the other.
 *
 * Every function follows the paper step by step (PAPER.md line numbers "P:n"); where the paper is
 * silent or garbled the reading is the DESIGN.md "Readings" entry named R#.
 * All floating point is fp64; summation orders are fixed (ascending pixel index), so results are
 * bitwise identical for any OpenMP thread count.
 */
#ifndef FMS_ORACLE_H
#define FMS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FMSO_OK = 0, FMSO_E_INVALID = 2, FMSO_E_ZERO_NORM = 3, FMSO_E_STALLED = 4, FMSO_E_CAPACITY = 5 };
enum { FMSO_SEEDS_FIXED = 0, FMSO_SEEDS_OSOP = 1, FMSO_SEEDS_ALL = 2 };
#define FMSO_MAX_ROUNDS 16

typedef struct {
  int32_t kind;            /* FMSO_SEEDS_* */
  int32_t n_seeds;         /* FIXED: seed count; OSOP: N_initial (128) */
  double gamma;            /* early-stop fraction (0.9) */
  double L, H, P;          /* OSOP controller (2, 8) and coverage target (0.99) */
  int32_t has_background;  /* largest cluster is background when estimating I, r (R14) */
  int32_t min_instance_px; /* clusters smaller than this do not count toward I (R22) */
  int32_t saturation_stop; /* stop when a round adds no counted instance (R22) */
  int32_t max_rounds;      /* <= FMSO_MAX_ROUNDS */
  uint64_t rng_seed;       /* hash-priority selection salt (R11) */
  int32_t profile;         /* kernel profile of the iteration: FMSO_PROFILE_FLAT (Eq. 3/11, the paper) or
                              FMSO_PROFILE_GAUSS (NEXT-4, reading R23) */
  int32_t metric;          /* FMSO_METRIC_COSINE (Eq. 9, the paper's path) or FMSO_METRIC_EUCLID (Eq. 4,
                              NEXT-4, reading R24; flat profile only) */
} fmso_policy;
enum { FMSO_PROFILE_FLAT = 0, FMSO_PROFILE_GAUSS = 1 };
enum { FMSO_METRIC_COSINE = 0, FMSO_METRIC_EUCLID = 1 };

typedef struct {
  int32_t rounds, K;
  int64_t seeds_total, seed_iters, discarded;
  int32_t round_K[FMSO_MAX_ROUNDS];      /* seeds launched in round r (K_r) */
  int32_t round_iters[FMSO_MAX_ROUNDS];  /* lockstep iterations run */
  int32_t round_conv[FMSO_MAX_ROUNDS];   /* converged seeds */
  int32_t round_disc[FMSO_MAX_ROUNDS];   /* discarded (unconverged / stalled) seeds */
  int64_t round_seed_iters[FMSO_MAX_ROUNDS]; /* sum over t of active seeds A_t */
  int32_t round_Kc[FMSO_MAX_ROUNDS];     /* centres after merge */
  int32_t round_I[FMSO_MAX_ROUNDS];      /* observed instance count (OSOP) */
  int64_t round_cand[FMSO_MAX_ROUNDS];   /* uncovered & unvisited pixels after assignment */
  double round_r[FMSO_MAX_ROUNDS];       /* observed foreground ratio */
  double round_nmin[FMSO_MAX_ROUNDS];    /* N_min (Eq. 19); -1 = infinite */
} fmso_trace;

/* ---- scalar pieces (P8/P9 pins) ---- */
uint64_t fmso_splitmix64(uint64_t z);
uint64_t fmso_key(uint64_t rng_seed, int32_t round, int64_t i);
double fmso_p_success(int64_t N, int64_t I, double r);      /* Eq. 14 */
int64_t fmso_n_min(double P, int64_t I, double r);           /* Eq. 19; INT64_MAX if I == 0 */
int32_t fmso_need(double gamma, int64_t K);                  /* ceil(gamma*K) (R8) */
/* O8 / NEXT-1, the frame-to-frame seed count ("N is reduced as N - N_min", R12, R18):
 * N_next = total seeds of the frame; if N_next > H * N_min then N_next = max(N_next - N_min, N_min).
 * nmin < 0 means N_min = infinity (no instance observed): N_next = total. */
int64_t fmso_session_next(int64_t total, double nmin, double H);

/* OSOP observation of the segmentation (R14, R22): background = the largest
 * cluster (lowest index on ties) when has_background; I = other clusters with >= min_instance_px
 * pixels; r = 1 - |bg|/n (1 without background).  Returns the background index or -1. */
int64_t fmso_observe(const int64_t* hist, int64_t K, int64_t n, int32_t has_background, int32_t min_instance_px,
                     int32_t* I_out, double* r_out);
/* OSOP stop rule (R13, R22): 1 = stop, 0 = another round.  nmin = INT64_MAX is infinite. */
int fmso_osop_stop(int64_t ncand, int64_t total, int64_t n, int32_t round, int32_t max_rounds, int64_t nmin,
                   double L, int32_t saturation_stop, int32_t I, int32_t I_prev);

/* ---- vector pieces ---- */
int fmso_normalize(const float* emb, int64_t n, int32_t d, double* xhat);         /* Eq. 1 / 9 */
int64_t fmso_select(const uint8_t* cand, int64_t n, int64_t K, uint64_t rng_seed,
                    int32_t round, int64_t* out);                                 /* Alg. 2 l.2 */
int64_t fmso_window(const double* xhat, int64_t n, int32_t d, double tau,
                    const double* s, double* g);                                  /* Eq. 8+11 */
/* NEXT-4, reading R23: the Gaussian profile of Eq. 2, k(t) = exp(-t/2) at
 * t = |x - s|^2 / h = 2 (1 - x.s) / h for unit vectors: every point weighs w = exp(-(1 - x.s)/h).
 * g = sum_i w_i x_i (ascending i); returns sum_i w_i. */
double fmso_window_gauss(const double* xhat, int64_t n, int32_t d, double h, const double* s, double* g);
/* fmso_lockstep with the kernel profile of the update selectable (FMSO_PROFILE_*); the intensity
 * stays the flat window count |S_h(m)| (R10) for both profiles. */
int32_t fmso_lockstep_p(const double* xhat, int64_t n, int32_t d, double h, int32_t max_iter,
                        double tol, double gamma, int64_t K, double* seeds, uint8_t* status,
                        int64_t* intensity, int32_t* iters, int64_t* seed_iters, int32_t profile);
/* NEXT-4, reading R24: the Euclidean metric of Eq. 4 with the flat kernel of Eq. 3 on the
 * raw (unnormalised) embeddings: S_h(s) = { x_i : |x_i - s|_2 <= h } (inclusive), g = sum x_i
 * (ascending i); returns |S_h(s)|.  The mean-shift update is then the window mean g / |S_h(s)|. */
int64_t fmso_window_euclid(const double* x, int64_t n, int32_t d, double h, const double* s, double* g);
/* fmso_lockstep_p with the metric selectable (FMSO_METRIC_*; Euclidean needs the flat profile): the
 * Euclidean update is s' = g / |S_h(s)| without renormalisation, convergence |s' - s|_2 < tol. */
int32_t fmso_lockstep_m(const double* x, int64_t n, int32_t d, double h, int32_t max_iter, double tol,
                        double gamma, int64_t K, double* seeds, uint8_t* status, int64_t* intensity,
                        int32_t* iters, int64_t* seed_iters, int32_t profile, int32_t metric);
/* Greedy merge with the metric selectable: Euclidean keeps a mode unless |m - c|_2 <= rho. */
int64_t fmso_merge_m(const double* pool, const int64_t* intensity, const int64_t* origin, int64_t m,
                     int32_t d, double rho, int64_t* keep, int32_t metric);
/* Assignment with the metric selectable: Euclidean label = argmin_k |x - c_k|_2 (lowest k on ties),
 * covered = min_k |x - c_k|_2 <= h.  (Cosine: fmso_assign with tau = 1 - h.) */
void fmso_assign_m(const double* x, int64_t n, int32_t d, const double* centres, int64_t K, double h,
                   int32_t* labels, uint8_t* covered, int64_t* hist, int32_t metric);
/* Lockstep mean-shift over K seeds (Alg. 2 l.4-9 + early stop).  seeds[K*d] in/out, status[K]:
 * 1 converged, 2 stalled, 3 discarded.  Returns iterations run; writes, for converged seeds, the
 * intensity |S_h(m)| (flat-kernel density of Eq. 2 at the mode, R10) and per-seed iterations. */
int32_t fmso_lockstep(const double* xhat, int64_t n, int32_t d, double h, int32_t max_iter,
                      double tol, double gamma, int64_t K, double* seeds, uint8_t* status,
                      int64_t* intensity, int32_t* iters, int64_t* seed_iters);
/* Greedy merge (R10): pool rows sorted by (intensity desc, origin asc), keep unless within rho of
 * a kept centre.  Writes kept indices into keep[] in kept order; returns the kept count. */
int64_t fmso_merge(const double* pool, const int64_t* intensity, const int64_t* origin,
                   int64_t m, int32_t d, double rho, int64_t* keep);
/* Nearest-mode assignment (Alg. 2 l.12-14): label = argmax_k x.c_k (lowest k on ties). */
void fmso_assign(const double* xhat, int64_t n, int32_t d, const double* centres, int64_t K,
                 double tau, int32_t* labels, uint8_t* covered, int64_t* hist);

/* ---- full method ---- */
int fmso_cluster(const float* emb, int64_t n, int32_t d, double h, int32_t max_iter, double tol,
                 const fmso_policy* pol, int32_t* labels, double* centres, int32_t centres_cap,
                 int32_t* K_out, fmso_trace* trace);

int fmso_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
