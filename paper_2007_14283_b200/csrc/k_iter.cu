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
//     2^11 G = W.hi + 2^-11 W.lo                          (one MMA with N = 2 DP over [hi | lo])
// is EXACT: 0/1 weights times integers |v| <= 2048 summed over <= 2^13 pixels stay below 2^24 in
// fp32.  Exact sums make the result independent of how pixels are split across CTAs, so work is
// balanced freely and merged with fp64 atomics (integer-valued, hence order-independent).
//
// Structure (fused-attention style; the S x N weight matrix never leaves the SM):
//   * work item = (frame, 128-seed tile, chunk of kChunkTiles 128-pixel tiles).  Persistent CTAs
//     (one per SM) take equal contiguous ranges of the item list; consecutive items of the same
//     seed tile form a segment whose G is accumulated in fp64 registers and flushed once.
//   * warp 0  : TMA producer  -- seed tile (s_hi, s_hi 2^-11, s_lo) and a ring of pixel tiles
//                               (hi, lo limbs), 32B (DP=16) or 64B (DP=32) swizzled rows.
//   * warp 1  : MMA issuer    -- C[buf] = 3 MMAs (M=128, N=128, K=DP) into TMEM;
//                                 G += P[buf] . [hi | lo]  (A = P from TMEM, B read MN-major,
//                                                          M=128, N=2 DP, K=16 per instruction)
//   * warps 2-9: epilogue      -- two warps per TMEM lane quarter (64 columns each, both loads in
//                                 flight before one wait): tcgen05.ld C rows, flat kernel -> fp16
//                                 0/1 weights P written back over C in TMEM (tcgen05.st); per
//                                 item G -> fp64 registers.
//                                 Count-pass items (mode 1: the converged modes of a round) skip G
//                                 and count window members (intensity, R10).
//   TMEM: 3 x 128 columns of C/P (triple buffered) + 2 x 2DP columns of G (double buffered).
#include "fms_device.cuh"

namespace fms {

constexpr int kEpiWarps = 8;                            // 2 groups x 4 warps (one per TMEM lane quarter)
constexpr int kGroupWarps = 4;                           // a group owns every other pixel tile
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kEpiWarp0 = 3;                             // warps: 0 TMA, 1 MMA1, 2 MMA2, 3..10 epilogue
constexpr int kIterThreads = kEpiWarp0 * 32 + kEpiThreads;

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
  static constexpr int NP = 2;                            // P buffers (one per epilogue group)
  static constexpr int P_COL = NC * kBN;                  // 128 px of fp16 weights = 64 columns each
  static constexpr int G_COL = P_COL + NP * (kBN / 2);
  static_assert(G_COL + 2 * G_N <= 512, "TMEM budget");
  // deep TMA ring: a stage is held from its load until the weighted-sum MMA two tiles later, and
  // pixel tiles stream from HBM (~2-3 us loaded latency), so ~160 KB of tiles must be in flight
  static constexpr int STAGES = DP == 16 ? 20 : 10;
  static constexpr int SMEM = 1024 /*align slack*/ + 2 * 3 * A_B + STAGES * 2 * TILE_B + 1024 /*barriers*/;
};

// in-window weights of two pixels -> packed fp16 {0, 1.0} pair (low half = first pixel)
__device__ __forceinline__ uint32_t flat_kernel_pair(float c0, float c1, float tau) {
  const float u0 = c0 - tau, u1 = c1 - tau;  // exact near tau (Sterbenz); sign(u) = [c < tau]
  uint32_t m;
  asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(m) : "r"(__float_as_uint(u0)), "r"(__float_as_uint(u1)));
  return ~m & 0x3C003C00u;  // sign-replicated masks select 0 (outside) or 1.0 (inside, c >= tau)
}

struct ItemDesc {
  int f, tile, chunk, mode;
};
__device__ __forceinline__ ItemDesc item_desc(const Params& p, int item) {
  const int t = item / p.n_chunks;
  const TileTask tt = p.tiles[t];
  return ItemDesc{tt.f, tt.tile, item - t * p.n_chunks, tt.mode};
}

template <int DP>
__global__ void __launch_bounds__(kIterThreads, 1) iter_kernel(const __grid_constant__ TMaps tm, Params p) {
  using Cfg = IterCfg<DP>;
  const int n_items = p.counters[0];
  // equal contiguous item ranges per CTA
  const int i_begin = (int)(((long long)n_items * blockIdx.x) / gridDim.x);
  const int i_end = (int)(((long long)n_items * (blockIdx.x + 1)) / gridDim.x);
  if (i_begin >= i_end) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // [2 buffers][s_hi, s_hs, s_lo][A_B]
  uint8_t* sX = smem + 6 * Cfg::A_B;                    // [Cfg::STAGES][hi, lo][TILE_B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + Cfg::STAGES * 2 * Cfg::TILE_B);
  uint64_t* x_full = bars;                    // [STAGES] pixel tile landed
  uint64_t* x_empty = x_full + Cfg::STAGES;   // [STAGES] pixel tile consumed (MMA1 and MMA2)
  uint64_t* a_full = x_empty + Cfg::STAGES;   // [2] seed tile landed
  uint64_t* a_empty = a_full + 2;             // [2] seed tile consumed
  uint64_t* c_full = a_empty + 2;             // [NC] similarity ready
  uint64_t* c_empty = c_full + Cfg::NC;       // [NC] similarity loaded by the epilogue
  uint64_t* p_full = c_empty + Cfg::NC;       // [NP] weights written
  uint64_t* p_free = p_full + Cfg::NP;        // [NP] weights consumed by MMA2
  uint64_t* g_full = p_free + Cfg::NP;        // [2] item's G complete
  uint64_t* g_empty = g_full + 2;             // [2] G drained by the epilogue
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(g_empty + 2);
  static_assert(Cfg::STAGES * 2 + 8 + 2 * Cfg::NC + 2 * Cfg::NP <= 120, "barrier area");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1);
      mbar_init(&g_full[i], 1); mbar_init(&g_empty[i], kGroupWarps);
    }
    // epilogue barriers take one arrive per warp (after __syncwarp): 256 same-address arrives
    // per tile would serialise in the shared-memory atomic unit
    for (int i = 0; i < Cfg::NC; ++i) { mbar_init(&c_full[i], 1); mbar_init(&c_empty[i], kGroupWarps); }
    for (int i = 0; i < Cfg::NP; ++i) { mbar_init(&p_full[i], kGroupWarps); mbar_init(&p_free[i], 1); }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm.xh); tma_prefetch(&tm.xl);
    tma_prefetch(&tm.sh); tma_prefetch(&tm.ss); tma_prefetch(&tm.sl);
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ================================ TMA producer ================================
    int stage = 0;
    uint32_t sphase = 0;
    int it = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int cbeg = w.chunk * kChunkTiles;
      const int ccnt = min(kChunkTiles, p.n_ptiles - cbeg);
      mbar_wait(&a_empty[ab], aph ^ 1);
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
        mbar_wait(&x_empty[stage], sphase ^ 1);
        if (lane == 0) {
          const int xrow = (int)(row0 + (long long)j * kBN) >> ((p.variant & 32) ? 2 : 0);
          if (p.variant & 64) {
            mbar_arrive(&x_full[stage]);  // timing experiment: no pixel loads
          } else {
            mbar_expect_tx(&x_full[stage], 2 * Cfg::TILE_B);
            tma_load_2d(sX + (2 * stage) * Cfg::TILE_B, &tm.xh, &x_full[stage], 0, xrow);
            tma_load_2d(sX + (2 * stage + 1) * Cfg::TILE_B, &tm.xl, &x_full[stage], 0, xrow);
          }
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA1 issuer: similarity ============================
    // C[i % NC] = 2^11 S.X^T for every tile of the CTA's stream; a C buffer is rewritten as soon as
    // the epilogue has loaded the previous tile from it (c_empty).
    constexpr uint32_t IDESC1 = idesc_f16(kBM, kBN, 0, 0);  // both operands K-major
    int stage = 0;
    uint32_t sphase = 0;
    int i = 0;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      mbar_wait(&a_full[ab], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t ah = smem_u32(sA + (3 * ab + 0) * Cfg::A_B);
      const uint32_t as = ah + Cfg::A_B;
      const uint32_t al = ah + 2 * Cfg::A_B;
      for (int j = 0; j < ccnt; ++j, ++i) {
        const uint32_t buf = i % Cfg::NC;
        if (i >= Cfg::NC) mbar_wait(&c_empty[buf], ((i / Cfg::NC) - 1) & 1);
        mbar_wait(&x_full[stage], sphase);
        tc_fence_after();
        const uint32_t xh = smem_u32(sX + (2 * stage) * Cfg::TILE_B);
        const uint32_t xl = xh + Cfg::TILE_B;
        const uint32_t d = tmem + buf * kBN;
        if (!(p.variant & 8)) {
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // s_hi . hi
            mma_ss_f16_el(d, umma_desc(ah + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                          umma_desc(xh + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT), IDESC1, kk > 0);
        }
        if (!(p.variant & 12)) {
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // + (s_hi 2^-11) . lo
            mma_ss_f16_el(d, umma_desc(as + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                          umma_desc(xl + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT), IDESC1, 1u);
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // + s_lo . hi
            mma_ss_f16_el(d, umma_desc(al + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                          umma_desc(xh + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT), IDESC1, 1u);
        }
        tc_commit_el(&c_full[buf]);
        if (++stage == Cfg::STAGES) { stage = 0; sphase ^= 1; }
      }
      tc_commit_el(&a_empty[ab]);  // seed tile free once this item's MMA1s complete
    }
  } else if (warp == 2) {
    // ========================== MMA2 issuer: weighted sum ==========================
    // G[ab] += P[i % NP] . [hi | lo] once the epilogue has written the weights (p_full); frees the
    // weight buffer (p_free) and the pixel stage (x_empty); at the end of an item hands G over.
    constexpr uint32_t IDESC2 = idesc_f16(kBM, Cfg::G_N, 0, 1);  // B = [hi|lo] read MN-major
    int stage = 0;
    uint32_t sphase = 0;
    int i = 0;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      mbar_wait(&g_empty[ab], ((it >> 1) & 1) ^ 1);
      const uint32_t g_tmem = tmem + Cfg::G_COL + ab * Cfg::G_N;
      for (int j = 0; j < ccnt; ++j, ++i) {
        const uint32_t pb = i % Cfg::NP;
        mbar_wait(&p_full[pb], (i / Cfg::NP) & 1);
        tc_fence_after();
        if (w.mode == 0 && !(p.variant & 1)) {
          const uint32_t xh = smem_u32(sX + (2 * stage) * Cfg::TILE_B);
#pragma unroll
          for (int k = 0; k < kBN / 16; ++k) {  // 16 pixels = 8 columns of packed fp16 weights
            const uint64_t bd = umma_desc(xh + k * 16 * Cfg::ROW_B, Cfg::TILE_B, Cfg::SBO, Cfg::LAYOUT);
            mma_ts_f16_el(g_tmem, tmem + Cfg::P_COL + pb * (kBN / 2) + k * 8, bd, IDESC2,
                          (j == 0 && k == 0) ? 0u : 1u);
          }
        }
        tc_commit_el(&p_free[pb]);
        tc_commit_el(&x_empty[stage]);
        if (++stage == Cfg::STAGES) { stage = 0; sphase ^= 1; }
      }
      tc_commit_el(&g_full[ab]);
    }
  } else {
    // ================================ epilogue (warps 3..10) ================================
    // Two groups of 4 warps (one warp per TMEM lane quarter); group g handles the tiles with
    // index % 2 == g in C buffer g and P buffer g, so each group has two tile periods to hide
    // its TMEM-load and barrier latencies.  Group 0 also drains G at the end of every item.
    const int q = warp & 3;                           // TMEM lane quarter this warp may access
    const int grp = (warp - kEpiWarp0) >> 2;          // 0 or 1
    const int row = q * 32 + lane;                    // seed row within the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const float tau = p.tau_f * kLimb;                // C is scaled by 2^11 (exact power-of-two scaling)
    const uint32_t cbase = tmem + lane_base + grp * kBN;
    const uint32_t pbase = tmem + lane_base + Cfg::P_COL + grp * (kBN / 2);
    uint32_t ctile = 0;                               // running tile index over the CTA's stream
    uint32_t mine = 0;                                // tiles handled by this group so far
    int it = 0;
    double gs[DP];                                    // segment sum of 2^11 G (exact integers / 2^11)
#pragma unroll
    for (int k = 0; k < DP; ++k) gs[k] = 0.0;
    int cnt = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      for (int j = 0; j < ccnt; ++j, ++ctile) {
        if ((int)(ctile & 1) != grp) continue;
        const uint32_t ph = mine & 1;
        mbar_wait(&c_full[grp], ph);
        if (mine >= 1) mbar_wait(&p_free[grp], (mine - 1) & 1);  // MMA2 done with our last weights
        tc_fence_after();
        __half2 acc = __float2half2_rn(0.f);
#pragma unroll
        for (int r = 0; r < 2; ++r) {  // two rounds of 64 columns
          uint32_t v[64];
          if (!(p.variant & 16)) {
            tmem_ld32(cbase + r * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
            tmem_ld32(cbase + r * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
            tmem_ld_wait();
          }
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            pk[i] = flat_kernel_pair(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]), tau);
          if (w.mode == 0) {
            if (!(p.variant & 2)) {
              tmem_st16(pbase + r * 32, *reinterpret_cast<const uint32_t(*)[16]>(pk));
              tmem_st16(pbase + r * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc = __hadd2(acc, *reinterpret_cast<const __half2*>(&pk[i]));
          }
        }
        if (w.mode == 0) {
          tmem_st_wait();
        } else {
          const float2 a2 = __half22float2(acc);  // exact: <= 64 per half per tile
          cnt += (int)(a2.x + a2.y);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&c_empty[grp]);  // MMA1 may overwrite C[grp]
          mbar_arrive(&p_full[grp]);   // MMA2 may consume P[grp]
        }
        ++mine;
      }
      if (grp == 0) {
        mbar_wait(&g_full[ab], aph);
        tc_fence_after();
        if (w.mode == 0) {
          uint32_t g[2 * DP];
          tmem_ld32(tmem + lane_base + Cfg::G_COL + ab * Cfg::G_N, *reinterpret_cast<uint32_t(*)[32]>(g));
          if constexpr (DP == 32)
            tmem_ld32(tmem + lane_base + Cfg::G_COL + ab * Cfg::G_N + 32, *reinterpret_cast<uint32_t(*)[32]>(g + 32));
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < DP; ++k)
            gs[k] += (double)__uint_as_float(g[k]) + (double)__uint_as_float(g[DP + k]) * (1.0 / kLimb);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_empty[ab]);
      }
      // flush the segment when the next item belongs to another seed tile (or at the end)
      const int t = item / p.n_chunks;
      const bool last = (item + 1 == i_end) || ((item + 1) / p.n_chunks != t);
      if (last) {
        const size_t r = (size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row;
        if (w.mode == 0) {
          if (grp == 0) {
            double* dst = p.gacc + r * DP;
#pragma unroll
            for (int k = 0; k < DP; ++k) {
              if (gs[k] != 0.0) atomicAdd(dst + k, gs[k]);
              gs[k] = 0.0;
            }
          }
        } else {
          if (cnt) atomicAdd(p.cacc + r, cnt);
          cnt = 0;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

int iter_smem_bytes(int DP) { return DP == 16 ? IterCfg<16>::SMEM : IterCfg<32>::SMEM; }

cudaError_t launch_iter(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st) {
  if (DP == 16) {
    iter_kernel<16><<<grid, kIterThreads, IterCfg<16>::SMEM, st>>>(tm, p);
  } else {
    iter_kernel<32><<<grid, kIterThreads, IterCfg<32>::SMEM, st>>>(tm, p);
  }
  return cudaGetLastError();
}

cudaError_t setup_iter_attrs() {
  cudaError_t e = cudaFuncSetAttribute(iter_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, IterCfg<16>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(iter_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, IterCfg<32>::SMEM);
}

}  // namespace fms
