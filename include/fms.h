/* fms.h -- C ABI of the B200 (sm_100a) Faster Mean-shift hot path (arXiv 2007.14283).
 *
 * The library clusters unit-normalised pixel embeddings with the paper's Faster Mean-shift:
 * batched lockstep mean-shift of seed vectors with a flat cosine kernel (Alg. 2, PAPER.md
 * P:179-223), online seed optimisation (OSOP, Eq. 12-21), merging of converged modes
 * ("pruned and merged if their distance is small") and nearest-mode assignment of every
 * pixel (Alg. 2 l.12-14).  Readings of the paper are listed in DESIGN.md ("R#").
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers are CUDA global-memory addresses on the
 *    context's device; host pointers are ordinary (preferably pinned) host memory.
 *  - The caller owns every input and output buffer.  Inputs are read-only and never retained
 *    after a call returns.  The context owns its workspace (grown on demand).
 *  - Every call returns an fms_status; nothing aborts.  fms_last_error(ctx) gives a message.
 *  - A context may be used by one host thread at a time; distinct contexts are independent.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *    stream-ordered and return once results are complete (K_out is a host value).
 *  - Limits of this build: 1 <= d <= 32 (rows are padded to 16 or 32 fp16 lanes), n < 2^31/B.
 */
#ifndef FMS_H
#define FMS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FMS_OK = 0,
  FMS_E_INVALID = 2,   /* usage: n<1, d<1 or d>32, h not in (0,1), tol<=0, max_iters<1, bad policy ("2") */
  FMS_E_ZERO_NORM = 3, /* a row has zero or non-finite norm: no direction (Eq. 9 needs |x|>0; "3") */
  FMS_E_STALLED = 4,   /* no seed converged in round 0 ("4") */
  FMS_E_CAPACITY = 5,  /* K > centres_cap only: the frame finished, labels are valid, *K_out = the required K */
  FMS_E_CUDA = 6,      /* CUDA runtime / launch error; message in fms_last_error */
  FMS_E_NCCL = 7,      /* reserved for the multi-GPU paths */
  FMS_E_OOM = 8,       /* workspace allocation failed */
  FMS_E_INTERNAL = 9   /* internal capacity (seed, centre or merge-pool workspace) or consistency check failed;
                          the frame's results are not valid */
} fms_status;

typedef enum {
  FMS_SEEDS_FIXED = 0, /* exactly n_seeds seeds, one round */
  FMS_SEEDS_OSOP = 1,  /* online seed optimisation (readings R12-R15, R22) */
  FMS_SEEDS_ALL = 2    /* every pixel is a seed, gamma = 1: Alg. 1 */
} fms_seed_kind;

/* Seed policy.  Defaults (fms_default_policy): OSOP, N_initial = 128, gamma = 0.9,
 * L = 2, H = 8, P = 0.99, background on, min_instance_px = 0, saturation off,
 * max_rounds = 8, rng_seed = 0. */
typedef struct {
  int32_t kind;            /* fms_seed_kind */
  int32_t n_seeds;         /* FIXED: seed count; OSOP: N_initial */
  double gamma;            /* early stop once ceil(gamma*K_r) seeds converged (R8), 0 < gamma <= 1 */
  double L, H, P;          /* OSOP: stop once seeds >= L*N_min (Eq. 21); H (session only); coverage target (Eq. 19) */
  int32_t has_background;  /* 1: the largest cluster is background when observing I, r (R14) */
  int32_t min_instance_px; /* clusters smaller than this do not count toward I (R22); 0 = paper */
  int32_t saturation_stop; /* 1: stop when a round adds no counted instance (R22) */
  int32_t max_rounds;      /* 1..16 */
  uint64_t rng_seed;       /* salt of the seed-selection hash (R11) */
} fms_seed_policy;

#define FMS_MAX_ROUNDS 16

/* Per-frame trace (identical fields to the test oracle's trace; counts are the run's own work). */
typedef struct {
  int32_t status, rounds, K, pad;
  int64_t seeds_total, seed_iters, discarded;
  int32_t round_K[FMS_MAX_ROUNDS];     /* seeds launched in round r */
  int32_t round_iters[FMS_MAX_ROUNDS]; /* lockstep iterations run in round r */
  int32_t round_conv[FMS_MAX_ROUNDS];
  int32_t round_disc[FMS_MAX_ROUNDS];
  int32_t round_Kc[FMS_MAX_ROUNDS];    /* centres after the merge of round r */
  int32_t round_I[FMS_MAX_ROUNDS];
  int64_t round_seed_iters[FMS_MAX_ROUNDS]; /* sum over t of active seeds */
  int64_t round_cand[FMS_MAX_ROUNDS];  /* uncovered & unvisited pixels after assignment */
  double round_r[FMS_MAX_ROUNDS];
  double round_nmin[FMS_MAX_ROUNDS];   /* N_min of Eq. 19, -1 = infinite */
} fms_frame_stats;

/* Per-call counters (whole batch). */
typedef struct {
  double ms_total;            /* wall time of the call on the stream (CUDA events) */
  int64_t workspace_bytes;    /* device workspace owned by the context */
  int32_t steps;              /* lockstep steps launched (including no-op tail steps) */
  int32_t iter_launches;      /* K2 launches that had work */
  double iter_ms;             /* summed K2 device time over those launches (only if profiling on) */
  int64_t iter_seed_iters;    /* sum over K2 launches of active seeds (units of work) */
  int64_t iter_items;         /* sum over K2 launches of work items */
  int64_t launches;           /* kernels this library launched during the call */
  int64_t iter_count_units;   /* sum over K2 launches of converged modes counted (intensity pass, R10) */
  int64_t host_syncs;         /* host waits on the stream during the call: 1 with the device-resident loop
                                 (option "graph", the default); one per poll with the host-polled loop */
  /* per-phase device time (ms), only with option "profile_iter" = 1 (the host-polled loop; events at the
     phase boundaries on the call's stream): K1 prep; K6 selection; the per-step control around K2
     (plan, K3 update, ctl_step, and the seed-sharding step exchange); K4 merge; K5 assignment + K7 OSOP;
     the stream idle while the host polls.  K2 itself is iter_ms. */
  double ms_prep, ms_select, ms_step_ctl, ms_merge, ms_assign, ms_host_wait;
  /* with option "guard_stats" = 1: lockstep-iteration (seed, pixel) pairs whose computed similarity lay
     within 2^-16 of tau -- the certified error bound of the 3-term fp32 similarity -- i.e. the window
     decisions (Eq. 11) the CUDA path cannot certify against the exact similarity; 0 otherwise */
  int64_t guard_pairs;
} fms_run_stats;

fms_status fms_default_policy(fms_seed_policy* out);

fms_status fms_ctx_create(void** ctx_out, int device);
void fms_ctx_destroy(void* ctx);
const char* fms_last_error(const void* ctx);
const char* fms_version(void);

/* Frame sequences (NEXT-1; the seed count N is carried from frame to
 * frame).  A session clusters one frame per fms_session_step with round 0 using the session's N
 * (initially policy->n_seeds); afterwards N = the frame's total seeds, reduced to
 * max(N - N_min, N_min) when N > H * N_min, N_min being the frame's last Eq. 19 estimate.
 * fms_session_step takes the arguments of fms_cluster (same ownership, errors and blocking) and
 * updates N only when the frame succeeded (FMS_OK or FMS_E_CAPACITY).  policy must be OSOP
 * (FMS_E_INVALID otherwise); the policy is copied.  fms_session_seeds returns the N the next
 * frame will start with (-1 for a NULL session).  The session borrows ctx (destroy it first). */
fms_status fms_session_create(void* ctx, const fms_seed_policy* policy, void** session_out);
fms_status fms_session_step(void* session, const float* emb, int64_t n, int32_t d, double bandwidth,
                            int32_t max_iters, double tol, int32_t* labels, float* centres, int32_t centres_cap,
                            int32_t* K_out, fms_frame_stats* frame_stats, fms_run_stats* run_stats, void* stream);
int64_t fms_session_seeds(const void* session);
void fms_session_destroy(void* session);

/* Seed sharding (the seeds of a round are independent mean-shift trajectories,
 * Alg. 2 l.4-9, so a round's seeds can be split over GPUs that each hold the
 * whole frame).  With world > 1, rank r iterates only the round seeds j with j % world == r; the
 * library calls `fn` at two exchange points and expects it to replace the int32 device buffer
 * `buf[0..count)` by its elementwise sum over all ranks, stream-ordered on `stream` (e.g. an
 * all-reduce through torch.distributed), returning 0 on success:
 *   - once per lockstep step: per frame (active, converged, stalled) counts, so the early-stop test
 *     converged >= ceil(gamma K_r) sees the whole round on every rank;
 *   - once per round before the merge: every owner's converged seeds (fp32 bits), statuses and
 *     intensities (non-owners contribute zeros, so the integer sum is exact).
 * Selection, merge, assignment and OSOP control then run replicated and bit-identical on every rank,
 * and every rank returns the full result.  All ranks must pass the same frames and parameters.
 * world = 1 (the default) disables sharding.  Errors: FMS_E_INVALID for rank/world out of range or
 * a NULL fn with world > 1; a nonzero return of fn makes the clustering call fail with FMS_E_NCCL. */
typedef int (*fms_exchange_fn)(void* user, int32_t* buf, int64_t count, void* stream);
fms_status fms_set_exchange(void* ctx, fms_exchange_fn fn, void* user, int32_t rank, int32_t world);

/* Seed sharding's per-round exchange as an all-gather (optional, SURVEY.md 8(e)2 "one allgather per
 * OSOP round of ... mode slots"): with fn set and seed sharding on, every rank packs only the seeds it
 * owns (j % world == rank, packed at row j / world) and `fn` must gather the ranks' int32 device
 * buffers: recv[r * count .. (r + 1) * count) = send of rank r, stream-ordered on `stream`, returning
 * 0 on success -- each rank sends 1/world of the round's rows instead of all-reducing a zero-padded
 * copy of all of them.  fn = NULL restores the all-reduce exchange.  A nonzero return fails the
 * clustering call with FMS_E_NCCL. */
typedef int (*fms_allgather_fn)(void* user, const int32_t* send, int32_t* recv, int64_t count, void* stream);
fms_status fms_set_allgather(void* ctx, fms_allgather_fn fn, void* user);

/* In-library NCCL (SURVEY.md 8(b) fms_ctx_create_dist): the sharding collectives run as NCCL calls
 * from inside the library on its stream -- no callback into the caller per lockstep step.
 * fms_nccl_unique_id writes a 128-byte ncclUniqueId (rank 0 calls it and shares the bytes, e.g.
 * through torch.distributed); every rank then calls fms_set_nccl (collective: blocks until all `world`
 * ranks joined) with mode FMS_SHARD_SEEDS (per-step counts by ncclAllReduce, per-round owned rows by
 * ncclAllGather) or FMS_SHARD_PIXELS (every exchange by ncclAllReduce; n_global / offset as in
 * fms_set_pixel_shard).  libnccl.so.2 is opened at run time (FMS_E_NCCL if it cannot be, or on an NCCL
 * error; the message names it).  One GPU per rank.  world = 1 turns sharding off.
 * fms_ctx_create_dist = fms_ctx_create + fms_set_nccl. */
enum { FMS_SHARD_SEEDS = 1, FMS_SHARD_PIXELS = 2 };
fms_status fms_nccl_unique_id(void* id_out);
fms_status fms_set_nccl(void* ctx, const void* unique_id, int32_t rank, int32_t world, int32_t mode,
                        int64_t n_global, int64_t offset);
fms_status fms_ctx_create_dist(void** ctx_out, int device, const void* unique_id, int32_t rank, int32_t world,
                               int32_t mode, int64_t n_global, int64_t offset);

/* Pixel sharding (for frames or stacks too large for one GPU).  Every window sum of
 * the lockstep iteration is a sum over pixels (Eq. 8 gated by Eq. 11, Alg. 2 l.4-9, PAPER.md
 * P:137-139), and so are the mode intensities, the label histogram that feeds I and r of
 * Eq. 19 and the coverage count of the OSOP stop rule, so a frame's pixels can be
 * split over GPUs that each hold a contiguous range.  With world > 1 this rank holds pixels
 * [offset, offset + n) of frames of n_global pixels: the clustering entry points then take n = this
 * rank's pixel count and `emb`/`labels` of this rank's rows only ([B][n][d] / [B][n]); seeds,
 * centres, K and the OSOP control are replicated, and every rank returns the same centres and K.
 * Seed origins (and so the merge order and the selection keys of R11) use the global pixel index,
 * so the result is identical to clustering the whole frame on one GPU.  The library calls `fn` (same
 * contract as fms_set_exchange: in-place elementwise int32 sum over all ranks on `stream`) after K1
 * (status), after each selection (the seed rows), after every K2 launch (the exact window sums G as
 * split int64, and counts), and after each assignment (histogram, candidate count, coverage bits).
 * Ranges of different ranks must be disjoint and cover [0, n_global); all ranks pass the same B,
 * d and parameters.  world = 1 disables it.  Seed sharding and pixel sharding are exclusive: enabling
 * one (world > 1) disables the other.  Errors: FMS_E_INVALID for rank/world out of range, a NULL fn
 * with world > 1, n_global outside [1, 2^31) or offset outside [0, n_global) (and, at the clustering
 * call, offset + n > n_global); a nonzero return of fn fails the call with FMS_E_NCCL. */
fms_status fms_set_pixel_shard(void* ctx, fms_exchange_fn fn, void* user, int32_t rank, int32_t world,
                               int64_t n_global, int64_t offset);

/* Options: "guard_stats" (0/1, default 0): count the uncertified window decisions (fms_run_stats.guard_pairs)
 *          with a K2 instantiation that tests every pair against the similarity's error bound.
 *          "pdl" (0/1, default 1): launch the lockstep-step kernels (plan, K2, K3 update, ctl_step, the
 *          step condition) with programmatic dependent launch, so each one's launch and prologue
 *          overlap its predecessor's tail (off in profiled calls).
 *          "graph" (0/1, default 1): run a single-GPU call as one CUDA graph launch whose round and
 *          lockstep-step loops are WHILE conditional nodes with device-set conditions (one host
 *          synchronisation per call); sharded and profiled calls always use the host-polled loop.
 *          "profile_iter" (0/1): time every K2 launch with CUDA events for fms_run_stats.iter_ms
 *          (forces the host-polled loop).
 *          "poll_steps" (1..64, default 4): lockstep steps launched between two host polls of the
 *          device counters (a frame that finishes early idles at most poll_steps - 1 steps).
 *          "kernel_profile" (0/1, default 0): the kernel of the mean-shift update.  0 = the paper's
 *          flat kernel (Eq. 3 / Eq. 11).  1 = Gaussian profile (SURVEY NEXT-4,
 *          DESIGN reading R23): Eq. 2's k(t) = exp(-t/2) at t = |x - s|^2 / h, i.e. every pixel
 *          weighs w = exp(-(1 - x.s)/h) in s' = normalize(sum_i w_i x_i) (fp16 weights; weights
 *          below 2^-24 flush to zero).  Intensity, merge, coverage and assignment keep the flat
 *          window in both.  Pixel sharding requires 0 (FMS_E_INVALID at the clustering call).
 *          "metric" (0/1, default 0): 0 = cosine distance on normalised embeddings (Eq. 9, the paper's
 *          path).  1 = Euclidean distance (Eq. 4, DESIGN reading R24): the
 *          raw embeddings, window |x - s|_2 <= bandwidth (any bandwidth > 0), update = window mean
 *          (no renormalisation), merge radius and coverage radius = bandwidth, label = nearest centre
 *          in L2; zero vectors are valid.  Needs d <= 30, kernel_profile 0 and no pixel sharding
 *          (FMS_E_INVALID otherwise).  centres come back in the caller's units. */
fms_status fms_set_option(void* ctx, const char* key, int64_t value);

/* Cluster one frame.  emb: device, [n][d] fp32 row-major.  labels: device int32[n] in [0, K).
 * centres: device fp32 [centres_cap][d], unit rows in merge order (intensity desc, origin asc).
 * K_out: host.  frame_stats/run_stats: host, nullable. */
fms_status fms_cluster(void* ctx, const float* emb, int64_t n, int32_t d, double bandwidth, int32_t max_iters,
                       double tol, const fms_seed_policy* policy, int32_t* labels, float* centres,
                       int32_t centres_cap, int32_t* K_out, fms_frame_stats* frame_stats,
                       fms_run_stats* run_stats, void* stream);

/* Cluster B independent frames of identical shape in one pass (the throughput entry point).
 * emb: device [B][n][d]; labels: device [B][n]; centres: device [B][centres_cap][d];
 * K_out: host int32[B]; frame_stats: host [B] or NULL.  Frames never interact. */
fms_status fms_cluster_batch(void* ctx, const float* emb, int32_t B, int64_t n, int32_t d, double bandwidth,
                             int32_t max_iters, double tol, const fms_seed_policy* policy, int32_t* labels,
                             float* centres, int32_t centres_cap, int32_t* K_out, fms_frame_stats* frame_stats,
                             fms_run_stats* run_stats, void* stream);

/* Same as fms_cluster_batch with HOST buffers: the embeddings are copied to the device, and labels /
 * centres copied back, inside the call (end-to-end entry).  The batch runs in chunks through
 * double-buffered device staging -- a first chunk of host_chunk / 4 frames (option "host_chunk",
 * default 48), then the rest split evenly into chunks of at most host_chunk: a copy stream uploads
 * chunk i+1 and downloads chunk i-1's results while chunk i is clustered (frames are independent, so
 * the results equal one fms_cluster_batch over all B frames).  Pinned host memory is needed for the
 * copies to overlap.  run_stats sums the chunks' counters. */
fms_status fms_cluster_batch_host(void* ctx, const float* emb_host, int32_t B, int64_t n, int32_t d,
                                  double bandwidth, int32_t max_iters, double tol,
                                  const fms_seed_policy* policy, int32_t* labels_host, float* centres_host,
                                  int32_t centres_cap, int32_t* K_out, fms_frame_stats* frame_stats,
                                  fms_run_stats* run_stats, void* stream);

#ifdef __cplusplus
}
#endif
#endif
