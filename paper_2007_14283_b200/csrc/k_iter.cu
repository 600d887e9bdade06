// k_iter.cu -- K2: the lockstep mean-shift iteration on 5th-generation tensor cores.
//
// One lockstep step of Alg. 2 lines 4-9 for every active seed of every frame
// in the batch, evaluated densely as P:210 prescribes ("does not search which points belong to S_h
// ... multiplies ... with the kernel function"):
//
//     C = S_hat . X_hat^T              seeds x pixels cosine similarity   (Eq. 1/9)
//     W = [C >= tau], tau = 1 - h      flat kernel, inclusive              (Eq. 11; R5)
//     G = W . X_hat                    windowed sum (count cancels, R4)    (Eq. 8 / R1)
//
// Numerics.  Pixels are stored as two fixed-point limbs held exactly in fp16, x = (hi + lo 2^-11)
// 2^-11 (|err| <= 2^-23); seeds as s = s_hi + s_lo plus s_hi 2^-11.  Then
//     2^11 C = s_hi.hi + (s_hi 2^-11).lo + s_lo.hi        (three kind::f16 MMAs, fp32 accumulate)
// decides the window with ~1e-7 error (plain fp16 would err by ~1e-4 and flip decisions), and
//     2^11 G = W.hi + 2^-11 W.lo                          (N = 2 DP MMAs over [hi | lo])
// is EXACT: the in-window weight is 2^-17 (an fp16 subnormal, see flat_kernel_pair), and 2^-17 times
// integers |v| <= 2048 summed over <= 2^13 pixels are multiples of 2^-17 below 2^7 -- within fp32's
// 24-bit significand.  Exact sums make the result independent of how pixels are split across CTAs, so work is
// balanced freely and CTAs merge with fp64 atomics (integer-valued, hence order-independent).
//
// Structure (fused-attention style; the S x N weight matrix never leaves the SM):
//   * work item = (frame, 128-seed tile, chunk of kChunkTiles 128-pixel tiles).  Persistent CTAs
//     (one per SM) take equal contiguous ranges of the item list; consecutive items of the same
//     seed tile form a segment whose G is accumulated in fp64 (shared memory) and flushed once.
//   * warp 0   : TMA producer -- seed tile (s_hi, s_hi 2^-11, s_lo) and a ring of pixel tiles
//                                (hi, lo limbs), 32B (DP=16) or 64B (DP=32) swizzled rows.
//   * warp 1   : MMA1 issuer  -- C[i % 2] = 3 MMAs (M=128, N=128, K=DP) into TMEM.
//   * warp 2   : MMA2 issuer  -- G += P[i % NP] . [hi | lo]  (A = P from TMEM, B read MN-major,
//                                M=128, N=2 DP, K=16 per instruction).  tcgen05.mma blocks its
//                                issuing thread while the tensor pipe is busy, so both MMA streams
//                                get dedicated warps.
//   * warps 3-10: epilogue    -- two groups of 4 warps (one per TMEM lane quarter) take alternate
//                                tiles: one tcgen05.ld of the whole 128-column C row, C handed back
//                                to MMA1, flat kernel -> fp16 0/1 weights P (tcgen05.st).  Group 0
//                                drains each item's G into the fp64 segment sums.
//                                Count-pass items (mode 1: the converged modes of a round) skip G
//                                and count window members (intensity, R10).
//   TMEM: 2 x 128 columns of C + NP x 64 columns of P + 2 x 2DP columns of G.
#include "fms_device.cuh"

namespace fms {

// Epilogue: two groups take alternate tiles; a group is 8 warps, two per TMEM lane quarter, each
// owning 64 of the tile's 128 columns.  Then TMA producer, MMA1 issuer, MMA2 issuer.
constexpr int kGroups = 2;
constexpr int kGroupWarps = 8;
constexpr int kEpiWarps = kGroups * kGroupWarps;
constexpr int kColsPerWarp = kBN / 2;
constexpr int kWarpTma = kEpiWarps, kWarpMma1 = kEpiWarps + 1, kWarpMma2 = kEpiWarps + 2;
constexpr int kIterThreads = (kEpiWarps + 3) * 32;

// Epilogue -> issuer hand-offs as named barriers (as in k_iter8.cu: one per C buffer, ids 1..NC, and
// one per weight buffer, ids NC + 1..NC + NP; a group's next arrival on one needs an MMA the waiting
// warp issues only after its sync); -DK2_MBAR_HANDOFF restores the mbarrier hand-offs
#ifdef K2_MBAR_HANDOFF
#define K2_RELEASE_C(b)                          \
  do {                                           \
    if (lane == 0) mbar_arrive(&c_empty[(b)]);   \
  } while (0)
#else
#define K2_RELEASE_C(b) nbar_arrive(1 + (int)(b), (kGroupWarps + 1) * 32)
#endif

template <int DP>
struct IterCfg {
  static constexpr int ROW_B = DP * 2;                    // bytes per row (fp16)
  static constexpr int TILE_B = kBN * ROW_B;              // one pixel tile (one limb)
  static constexpr int A_B = kBM * ROW_B;                 // one seed tile (one split)
  static constexpr uint32_t LAYOUT = DP == 16 ? 6u : 4u;  // SWIZZLE_32B / SWIZZLE_64B
  static constexpr uint32_t SBO = 8 * ROW_B;              // 8-row core-matrix group stride
  static constexpr int G_N = 2 * DP;                      // G columns: [hi | lo]
  // TMEM map (512 columns): C buffers (fp32 similarity) | P buffers (fp16 weights) | G buffers
  static constexpr int NC = 2;                            // C buffers (one per epilogue group)
  static constexpr int NP = DP == 16 ? 3 : 2;             // P buffers (tile mod NP)
  static constexpr int P_COL = NC * kBN;                  // 128 px of fp16 weights = 64 columns each
  static constexpr int G_COL = P_COL + NP * (kBN / 2);
  static_assert(G_COL + 2 * G_N <= 512, "TMEM budget");
  // deep TMA ring: a stage is held from its load until the weighted-sum MMA two tiles later, and
  // pixel tiles stream from HBM (~2-3 us loaded latency), so ~160 KB of tiles must be in flight
  static constexpr int STAGES = DP == 16 ? 20 : 9;
  static constexpr int GS_B = kBM * DP * 8;                // fp64 segment sums of G, [DP][kBM]
  static constexpr int SMEM = 1024 /*align slack*/ + 2 * 3 * A_B + STAGES * 2 * TILE_B + GS_B + 1024 /*barriers*/;
};

// In-window weights of two pixels -> packed fp16 pair of {0, 2^-17}, low half = first pixel.
// C and tau are 2^11-scaled fp32 numbers in [1024, 2048) near the threshold, so c - tau_m (tau_m =
// the float just below tau) is an exact multiple of 2^-13 and
//     sat(8192 c - 8192 tau_m) = [c >= tau]            (one FFMA.SAT, exact, inclusive: R5)
// The byte permute puts byte 2 of each 1.0f / 0.0f (0x80 / 0x00) over a zero byte: fp16 0x0080 =
// 2^-17 (subnormal) or 0.  A power of two keeps the weighted sums exact in fp32 (see the header);
// the drain scales by 2^17.  The FMA pipe does the compare and a single ALU op per pair packs.
__device__ __forceinline__ uint32_t flat_kernel_pair(float c0, float c1, float k_tau) {
  const float w0 = __saturatef(__fmaf_rn(c0, 8192.0f, k_tau));
  const float w1 = __saturatef(__fmaf_rn(c1, 8192.0f, k_tau));
  uint32_t m;
  asm("prmt.b32 %0, %1, %2, 0x4602;" : "=r"(m) : "r"(__float_as_uint(w0)), "r"(__float_as_uint(w1)));
  return m;
}
constexpr double kPScale = 1.0 / 131072.0;  // value of an in-window weight, 2^-17

// NEXT-4, reading R23: Gaussian profile of Eq. 2 on unit vectors, w = exp(-(1 - c)/h) =
// exp2(C ka + kb) with C = 2^11 c, ka = log2(e) / (2^11 h), kb = -log2(e) / h: one FFMA and one
// MUFU.EX2 per pixel, and one F2FP packs a pair of weights into fp16 (low half = first pixel).
// Weights below the fp16 range (< 2^-24, i.e. 1 - c > 16.6 h) flush to zero.  The weighted sums are
// no longer exact (fp16 weights, ~2^-11 relative), so results match the fp64 oracle to a tolerance.
__device__ __forceinline__ uint32_t gauss_pair(float c0, float c1, float ka, float kb) {
  float w0, w1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w0) : "f"(__fmaf_rn(c0, ka, kb)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w1) : "f"(__fmaf_rn(c1, ka, kb)));
  uint32_t m;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(m) : "f"(w1), "f"(w0));  // a -> upper half, b -> lower
  return m;
}

// Timing experiments (tools/iter_probe.cu): -DFMS_K2_VARIANT=bits switches parts of the kernel off
// (1 weighted-sum MMAs, 2 weight stores, 8/12 similarity MMAs, 16 C loads, 64 pixel loads), -DFMS_K2_TIMELINE logs a clock64 timeline of CTA 0.  The production
// build compiles both hooks away.
#ifdef FMS_K2_VARIANT
#define K2_OFF(p, bit) (FMS_K2_VARIANT & (bit))
#else
#define K2_OFF(p, bit) (0)
#endif
#ifdef FMS_K2_TIMELINE
__device__ __forceinline__ void tlog(const Params& p, int role, int tile, int ev) {
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tile < 512) p.dbg[((size_t)role * 512 + tile) * 8 + ev] = clock64();
}
#else
__device__ __forceinline__ void tlog(const Params&, int, int, int) {}
#endif

// waits of the producer / MMA warps, which share their SM sub-partitions with epilogue warps
#ifdef K2_ROLE_SLEEP
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t parity) { mbar_wait_sleep(bar, parity, K2_ROLE_SLEEP); }
#else
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
#endif
// the epilogue's wait for a similarity tile (timing experiment: -DK2_EPI_SLEEP=ns backs off)
#ifdef K2_EPI_SLEEP
__device__ __forceinline__ void epi_wait(uint64_t* bar, uint32_t parity) {
  if (!mbar_test(bar, parity)) mbar_wait_sleep(bar, parity, K2_EPI_SLEEP);
}
#else
__device__ __forceinline__ void epi_wait(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
#endif

struct ItemDesc {
  int f, tile, chunk, mode;
};
__device__ __forceinline__ ItemDesc item_desc(const Params& p, int item) {
  const int t = item / p.n_chunks;
  const TileTask tt = p.tiles[t];
  return ItemDesc{tt.f, tt.tile, item - t * p.n_chunks, tt.mode};
}

template <int DP, bool GAUSS>
__global__ void __launch_bounds__(kIterThreads, 1) iter_kernel(const __grid_constant__ TMaps tm, Params p) {
  using Cfg = IterCfg<DP>;
  pdl_wait();
  const int n_items = p.counters[0];
  // equal contiguous item ranges per CTA
  const int i_begin = (int)(((long long)n_items * blockIdx.x) / gridDim.x);
  const int i_end = (int)(((long long)n_items * (blockIdx.x + 1)) / gridDim.x);
  if (i_begin >= i_end) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // [2 buffers][s_hi, s_hs, s_lo][A_B]
  uint8_t* sX = smem + 6 * Cfg::A_B;                    // [Cfg::STAGES][hi, lo][TILE_B]
  double* gsm = reinterpret_cast<double*>(sX + Cfg::STAGES * 2 * Cfg::TILE_B);  // [DP][kBM]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(gsm) + Cfg::GS_B);
  uint64_t* x_full = bars;                    // [STAGES] pixel tile landed
  uint64_t* x_empty = x_full + Cfg::STAGES;   // [STAGES] tile's weighted sum done: stage and P free
  uint64_t* a_full = x_empty + Cfg::STAGES;   // [2] seed tile landed
  uint64_t* a_empty = a_full + 2;             // [2] seed tile consumed
  uint64_t* c_full = a_empty + 2;             // [NC] similarity ready
  uint64_t* c_empty = c_full + Cfg::NC;       // [NC] similarity loaded by the epilogue
  uint64_t* g_full = c_empty + Cfg::NC;       // [2] item's G complete (kChunkTiles commits)
  uint64_t* g_empty = g_full + 2;             // [2] G drained (and re-zeroed) by group 0
  uint64_t* p_full = g_empty + 2;             // [NP] weights written (4 quarters)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(p_full + Cfg::NP);
  static_assert(Cfg::STAGES * 2 + 8 + 2 * Cfg::NC + Cfg::NP <= 120, "barrier area");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1);
      mbar_init(&g_full[i], 1); mbar_init(&g_empty[i], 4);  // drained by 4 warps (one per quarter)
    }
    // epilogue barriers take one arrive per warp (after __syncwarp): 256 same-address arrives
    // per tile would serialise in the shared-memory atomic unit
    for (int i = 0; i < Cfg::NC; ++i) { mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], kGroupWarps); }
    for (int i = 0; i < Cfg::NP; ++i) mbar_init(&p_full[i], kGroupWarps);  // one group per tile
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == kWarpTma && lane == 0) {
    tma_prefetch(&tm.xh); tma_prefetch(&tm.xl);
    tma_prefetch(&tm.sh); tma_prefetch(&tm.ss); tma_prefetch(&tm.sl);
  }
  if (warp == kWarpMma1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (warp == kWarpTma) {
    // ================================ TMA producer ================================
    int xi = 0;
    int stage = 0;
    uint32_t sphase = 0;
    int it = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int cbeg = w.chunk * kChunkTiles;
      const int ccnt = min(kChunkTiles, p.n_ptiles - cbeg);
      role_wait(&a_empty[ab], aph ^ 1);
      if (lane == 0) {
        const int srow = w.f * p.S_pad + w.tile * kBM;
        mbar_expect_tx(&a_full[ab], 3 * Cfg::A_B);
        tma_load_2d(sA + (3 * ab + 0) * Cfg::A_B, &tm.sh, &a_full[ab], 0, srow);
        tma_load_2d(sA + (3 * ab + 1) * Cfg::A_B, &tm.ss, &a_full[ab], 0, srow);
        tma_load_2d(sA + (3 * ab + 2) * Cfg::A_B, &tm.sl, &a_full[ab], 0, srow);
      }
      __syncwarp();
      const long long row0 = (long long)w.f * p.n_pad + (long long)cbeg * kBN;
      for (int j = 0; j < ccnt; ++j) {
        role_wait(&x_empty[stage], sphase ^ 1);
        tlog(p, 0, xi, 0);
        if (lane == 0) {
          const int xrow = (int)(row0 + (long long)j * kBN);
          if (K2_OFF(p, 64)) {
            mbar_arrive(&x_full[stage]);  // timing experiment: no pixel loads
          } else {
            mbar_expect_tx(&x_full[stage], 2 * Cfg::TILE_B);
            tma_load_2d(sX + (2 * stage) * Cfg::TILE_B, &tm.xh, &x_full[stage], 0, xrow);
            tma_load_2d(sX + (2 * stage + 1) * Cfg::TILE_B, &tm.xl, &x_full[stage], 0, xrow);
          }
        }
        __syncwarp();
        ++xi;
        if (++stage == Cfg::STAGES) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp == kWarpMma1) {
    // ============================ MMA1 issuer: similarity ============================
    // C[i % NC] = 2^11 S.X^T for every tile of the CTA's stream; a C buffer is rewritten as soon as
    // the epilogue has loaded the previous tile from it (c_empty).
    constexpr uint32_t IDESC1 = idesc_f16(kBM, kBN, 0, 0);  // both operands K-major
    const uint64_t dx0 = umma_desc(smem_u32(sX), 16, Cfg::SBO, Cfg::LAYOUT);
    int stage = 0;
    uint32_t sphase = 0;
    int i = 0;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      role_wait(&a_full[ab], (it >> 1) & 1);
      tc_fence_after();
      // descriptors: computed once per item / stage and advanced by plain adds (the start-address
      // field holds the byte address >> 4 in the low bits)
      const uint64_t dah = umma_desc(smem_u32(sA + (3 * ab + 0) * Cfg::A_B), 16, Cfg::SBO, Cfg::LAYOUT);
      const uint64_t das = dah + (Cfg::A_B >> 4);
      const uint64_t dal = dah + (2 * Cfg::A_B >> 4);
      for (int j = 0; j < ccnt; ++j, ++i) {
        const uint32_t buf = i % Cfg::NC;
        tlog(p, 1, i, 0);
#ifdef K2_MBAR_HANDOFF
        if (i >= Cfg::NC) role_wait(&c_empty[buf], ((i / Cfg::NC) - 1) & 1);
#else
        if (i >= Cfg::NC) nbar_sync(1 + buf, (kGroupWarps + 1) * 32);  // C[buf] loaded by its group
#endif
        tlog(p, 1, i, 1);
        role_wait(&x_full[stage], sphase);
        tlog(p, 1, i, 2);
        tc_fence_after();
        const uint64_t dxh = dx0 + (uint64_t)(stage * (2 * Cfg::TILE_B >> 4));
        const uint64_t dxl = dxh + (Cfg::TILE_B >> 4);
        const uint32_t d = tmem + buf * kBN;
        if (!K2_OFF(p, 8)) {
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // s_hi . hi
            mma_ss_f16_el(d, dah + kk * 2, dxh + kk * 2, IDESC1, kk > 0);
        }
        if (!K2_OFF(p, 12)) {
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // + (s_hi 2^-11) . lo
            mma_ss_f16_el(d, das + kk * 2, dxl + kk * 2, IDESC1, 1u);
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // + s_lo . hi
            mma_ss_f16_el(d, dal + kk * 2, dxh + kk * 2, IDESC1, 1u);
        }
        tc_commit_el(&c_full[buf]);
        tlog(p, 1, i, 3);
        if (++stage == Cfg::STAGES) { stage = 0; sphase ^= 1; }
      }
      tc_commit_el(&a_empty[ab]);  // seed tile free once this item's MMA1s complete
    }
  } else if (warp == kWarpMma2) {
    // ========================== MMA2 issuer: weighted sum ==========================
    // G[ab] += P[i % NP] . [hi | lo] once the epilogue group has written the weights (p_full); one
    // commit frees the pixel stage and with it the weight buffer (x_empty); at the end of an item
    // hands G over (g_full).  A dedicated warp absorbs the issue stalls of a busy tensor pipe.
    constexpr uint32_t IDESC2 = idesc_f16(kBM, Cfg::G_N, 0, 1);  // B = [hi|lo] read MN-major
    const uint64_t dxg0 = umma_desc(smem_u32(sX), Cfg::TILE_B, Cfg::SBO, Cfg::LAYOUT);
    int stage = 0;
    int i = 0;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      role_wait(&g_empty[ab], ((it >> 1) & 1) ^ 1);
      const uint32_t g_tmem = tmem + Cfg::G_COL + ab * Cfg::G_N;
      for (int j = 0; j < ccnt; ++j, ++i) {
        const uint32_t pb = i % Cfg::NP;
#ifdef K2_MBAR_HANDOFF
        role_wait(&p_full[pb], (i / Cfg::NP) & 1);
#else
        nbar_sync(1 + Cfg::NC + pb, (kGroupWarps + 1) * 32);  // P[pb] stored by its group
#endif
        tc_fence_after();
        if (w.mode == 0 && !K2_OFF(p, 1)) {
          const uint64_t bd0 = dxg0 + (uint64_t)(stage * (2 * Cfg::TILE_B >> 4));
          const uint32_t pa = tmem + Cfg::P_COL + pb * (kBN / 2);
#pragma unroll
          for (int k = 0; k < kBN / 16; ++k)  // 16 pixels = 8 columns of packed fp16 weights
            mma_ts_f16_el(g_tmem, pa + k * 8, bd0 + (uint64_t)(k * (16 * Cfg::ROW_B >> 4)), IDESC2,
                          (j == 0 && k == 0) ? 0u : 1u);
        }
        tc_commit_el(&x_empty[stage]);  // pixel stage and weight buffer pb free once these complete
        if (++stage == Cfg::STAGES) stage = 0;
      }
      tc_commit_el(&g_full[ab]);
    }
  } else {
    // ================================ epilogue (warps 0..15) ================================
    // Group g handles the tiles with index % 2 == g out of C buffer g; warp (q, h) of the group
    // reads lane quarter q, columns [64 h, 64 h + 64) -- half a row, so 64 registers of C.
    const int q = warp & 3;                           // TMEM lane quarter this warp may access
    const int h = (warp >> 2) & 1;                    // column half
    const int grp = warp >> 3;
    const bool drainer = grp == 0 && h == 0;          // drains G for its quarter
    const int row = q * 32 + lane;                    // seed row within the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    // C is scaled by 2^11 (exact); k_tau = -8192 tau_m, tau_m = the float just below 2^11 tau
    const float k_tau = -8192.0f * __uint_as_float(__float_as_uint(p.tau_f * kLimb) - 1u);
    const float g_ka = GAUSS ? (float)(1.4426950408889634 / (p.h * (double)kLimb)) : 0.f;  // Gaussian (R23)
    const float g_kb = GAUSS ? (float)(-1.4426950408889634 / p.h) : 0.f;
    const uint32_t cbase = tmem + lane_base + grp * kBN + h * kColsPerWarp;
    uint32_t ctile = 0;                               // running tile index over the CTA's stream
    uint32_t mine = 0;                                // tiles handled by this group so far
    int it = 0;
    double* gs = gsm + row;                           // segment sum of 2^11 G, [k][kBM] (conflict-free)
    if (drainer) {
#pragma unroll
      for (int k = 0; k < DP; ++k) gs[k * kBM] = 0.0;
    }
    int cnt = 0;
    // Group 0 drains an item's G (and flushes a finished segment) after its first tile of the next
    // item, so the drain's waits overlap that tile instead of stalling the tile stream.
    auto drain = [&](int item_d, int it_d) {
      const ItemDesc w = item_desc(p, item_d);
      const int ab = it_d & 1;
      mbar_wait(&g_full[ab], (it_d >> 1) & 1);
      tc_fence_after();
      const uint32_t gq = tmem + lane_base + Cfg::G_COL + ab * Cfg::G_N;
      if (w.mode == 0) {
        if constexpr (DP == 16) {
          uint32_t g[2 * DP];
          tmem_ld32(gq, *reinterpret_cast<uint32_t(*)[32]>(g));
          tmem_ld_wait();
          tmem_regs_ready(*reinterpret_cast<uint32_t(*)[32]>(g));
#pragma unroll
          for (int k = 0; k < DP; ++k)
            gs[k * kBM] += (double)__uint_as_float(g[k]) + (double)__uint_as_float(g[DP + k]) * (1.0 / kLimb);
        } else {
          // DP = 32: the hi and lo halves one after the other (32 live registers instead of 64; the
          // fp64 segment sums are exact either way)
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            uint32_t g[32];
            tmem_ld32(gq + part * 32, g);
            tmem_ld_wait();
            tmem_regs_ready(g);
            const double sc = part ? 1.0 / kLimb : 1.0;
#pragma unroll
            for (int k = 0; k < 32; ++k) gs[k * kBM] += (double)__uint_as_float(g[k]) * sc;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&g_empty[ab]);
      // flush the segment when the next item belongs to another seed tile (or at the end)
      const bool last = (item_d + 1 == i_end) || ((item_d + 1) / p.n_chunks != item_d / p.n_chunks);
      if (last && w.mode == 0) {
        double* dst = p.gacc + ((size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row) * DP;
#pragma unroll
        for (int k = 0; k < DP; ++k) {
          // exact sums of multiples of 2^-28 in fp64; dividing by the power of two 2^-17 is exact
          if (gs[k * kBM] != 0.0) atomicAdd(dst + k, GAUSS ? gs[k * kBM] : gs[k * kBM] / kPScale);
          gs[k * kBM] = 0.0;
        }
      }
    };
    int pend = -1, pend_it = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      for (int j = 0; j < ccnt; ++j, ++ctile) {
        if ((int)(ctile & 1) != grp) continue;
        const int lrole = h ? 15 : 3 + grp * 4 + q;  // timeline: the h == 0 warps
        tlog(p, lrole, ctile, 0);
        epi_wait(&c_full[grp], mine & 1);
        tlog(p, lrole, ctile, 1);
        const uint32_t pb = ctile % Cfg::NP;
        tc_fence_after();
        uint32_t v[kColsPerWarp];
        if (K2_OFF(p, 128)) K2_RELEASE_C(grp);  // timing experiment: release early
        if (!K2_OFF(p, 16)) {
          tmem_ld64(cbase, v);  // one instruction: the scheduler cannot interleave math between pieces
          tmem_ld_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (!K2_OFF(p, 128)) K2_RELEASE_C(grp);  // MMA1 may overwrite C[grp]
        tlog(p, lrole, ctile, 2);
        // P[pb] is free once the weighted sum of the tile that used it last has completed: probe
        // now, use the answer after the flat kernel
        const uint32_t u = ctile - Cfg::NP;
        // (count-pass tiles too: p_full must not complete twice before MMA2 has seen the first phase)
        const bool need_free = ctile >= (uint32_t)Cfg::NP;
        bool p_free = !need_free || mbar_test(&x_empty[u % Cfg::STAGES], (u / Cfg::STAGES) & 1);
        uint32_t pk[kColsPerWarp / 2];
        if (GAUSS && w.mode == 0) {  // count passes (intensity, R10) keep the flat window
#pragma unroll
          for (int i = 0; i < kColsPerWarp / 2; ++i)
            pk[i] = gauss_pair(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]), g_ka, g_kb);
        } else {
#pragma unroll
          for (int i = 0; i < kColsPerWarp / 2; ++i)
            pk[i] = flat_kernel_pair(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]), k_tau);
        }
        tlog(p, lrole, ctile, 5);
        if (!p_free) mbar_wait(&x_empty[u % Cfg::STAGES], (u / Cfg::STAGES) & 1);
        tlog(p, lrole, ctile, 6);
        if (w.mode == 0) {
          tc_fence_after();
          if (!K2_OFF(p, 2))
            tmem_st32(tmem + lane_base + Cfg::P_COL + pb * (kBN / 2) + h * (kColsPerWarp / 2),
                      *reinterpret_cast<const uint32_t(*)[32]>(pk));
          tmem_st_wait();
        } else {
#pragma unroll
          for (int i = 0; i < kColsPerWarp / 2; ++i) cnt += __popc(pk[i] & 0x00800080u);  // bit 7 of 0x0080
        }
        tlog(p, lrole, ctile, 3);
        tc_fence_before();
        __syncwarp();
#ifdef K2_MBAR_HANDOFF
        if (lane == 0) mbar_arrive(&p_full[pb]);  // MMA2 may consume P[pb]
#else
        nbar_arrive(1 + Cfg::NC + pb, (kGroupWarps + 1) * 32);  // MMA2 may consume P[pb]
#endif
        tlog(p, lrole, ctile, 4);
        ++mine;
        if (drainer && pend >= 0) { drain(pend, pend_it); pend = -1; }
      }
      if (drainer) {
        if (pend >= 0) drain(pend, pend_it);
        pend = item;
        pend_it = it;
      }
      // count pass: each group flushes its window counts when the segment ends
      const bool last = (item + 1 == i_end) || ((item + 1) / p.n_chunks != item / p.n_chunks);
      if (last && w.mode != 0) {
        if (cnt) atomicAdd(p.cacc + (size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row, cnt);
        cnt = 0;
      }
    }
    if (drainer && pend >= 0) drain(pend, pend_it);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpMma1) tmem_dealloc(tmem, 512);
}

int iter_smem_bytes(int DP) { return DP == 16 ? IterCfg<16>::SMEM : IterCfg<32>::SMEM; }

cudaError_t launch_iter(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st) {
  const bool g = p.profile == 1;
  if (DP == 16) {
    return launch_ex(p.pdl, g ? iter_kernel<16, true> : iter_kernel<16, false>, grid, kIterThreads, IterCfg<16>::SMEM,
                     st, tm, p);
  } else {
    return launch_ex(p.pdl, g ? iter_kernel<32, true> : iter_kernel<32, false>, grid, kIterThreads, IterCfg<32>::SMEM,
                     st, tm, p);
  }
}

cudaError_t setup_iter_attrs() {
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e = cudaFuncSetAttribute(iter_kernel<16, false>, a, IterCfg<16>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(iter_kernel<16, true>, a, IterCfg<16>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(iter_kernel<32, false>, a, IterCfg<32>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(iter_kernel<32, true>, a, IterCfg<32>::SMEM);
  return e;
}

}  // namespace fms
