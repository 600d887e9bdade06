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
//   * warps 2-5: epilogue      -- tcgen05.ld C rows, flat kernel -> fp16 0/1 weights P written back
//                                 over C in TMEM (tcgen05.st); per item G -> fp64 registers.
//                                 Count-pass items (mode 1: the converged modes of a round) skip G
//                                 and count window members (intensity, R10).
//   TMEM: 3 x 128 columns of C/P (triple buffered) + 2 x 2DP columns of G (double buffered).
#include "fms_device.cuh"

namespace fms {

template <int DP>
struct IterCfg {
  static constexpr int ROW_B = DP * 2;                    // bytes per row (fp16)
  static constexpr int TILE_B = kBN * ROW_B;              // one pixel tile (one limb)
  static constexpr int A_B = kBM * ROW_B;                 // one seed tile (one split)
  static constexpr uint32_t LAYOUT = DP == 16 ? 6u : 4u;  // SWIZZLE_32B / SWIZZLE_64B
  static constexpr uint32_t SBO = 8 * ROW_B;              // 8-row core-matrix group stride
  static constexpr int G_N = 2 * DP;                      // G columns: [hi | lo]
  static constexpr int G_COL = kCBufs * kBN;              // TMEM column of G buffer 0
  static constexpr int SMEM = 1024 /*align slack*/ + 2 * 3 * A_B + kStages * 2 * TILE_B + 1024 /*barriers*/;
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
__global__ void __launch_bounds__(192, 1) iter_kernel(const __grid_constant__ TMaps tm, Params p) {
  using Cfg = IterCfg<DP>;
  const int n_items = p.counters[0];
  // equal contiguous item ranges per CTA
  const int i_begin = (int)(((long long)n_items * blockIdx.x) / gridDim.x);
  const int i_end = (int)(((long long)n_items * (blockIdx.x + 1)) / gridDim.x);
  if (i_begin >= i_end) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // [2 buffers][s_hi, s_hs, s_lo][A_B]
  uint8_t* sX = smem + 6 * Cfg::A_B;                    // [kStages][hi, lo][TILE_B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + kStages * 2 * Cfg::TILE_B);
  uint64_t* x_full = bars;                    // [kStages]
  uint64_t* x_empty = x_full + kStages;       // [kStages]
  uint64_t* a_full = x_empty + kStages;       // [2]
  uint64_t* a_empty = a_full + 2;             // [2]
  uint64_t* c_full = a_empty + 2;             // [kCBufs]
  uint64_t* p_full = c_full + kCBufs;         // [kCBufs]
  uint64_t* g_full = p_full + kCBufs;         // [2]
  uint64_t* g_empty = g_full + 2;             // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(g_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1);
      mbar_init(&g_full[i], 1); mbar_init(&g_empty[i], 128);
    }
    for (int i = 0; i < kCBufs; ++i) { mbar_init(&c_full[i], 1); mbar_init(&p_full[i], 128); }
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
          const int xrow = (int)(row0 + (long long)j * kBN);
          mbar_expect_tx(&x_full[stage], 2 * Cfg::TILE_B);
          tma_load_2d(sX + (2 * stage) * Cfg::TILE_B, &tm.xh, &x_full[stage], 0, xrow);
          tma_load_2d(sX + (2 * stage + 1) * Cfg::TILE_B, &tm.xl, &x_full[stage], 0, xrow);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    constexpr uint32_t IDESC1 = idesc_f16(kBM, kBN, 0, 0);        // C = A . X^T, both K-major
    constexpr uint32_t IDESC2 = idesc_f16(kBM, Cfg::G_N, 0, 1);   // G += P . [hi|lo], MN-major
    int stage = 0;
    uint32_t sphase = 0;
    uint32_t ctile = 0;  // running tile counter -> C buffer index and phase
    int it = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const uint32_t g_tmem = tmem + Cfg::G_COL + ab * Cfg::G_N;
      mbar_wait(&a_full[ab], aph);
      mbar_wait(&g_empty[ab], aph ^ 1);
      tc_fence_after();
      const uint32_t ah = smem_u32(sA + (3 * ab + 0) * Cfg::A_B);
      const uint32_t as = smem_u32(sA + (3 * ab + 1) * Cfg::A_B);
      const uint32_t al = smem_u32(sA + (3 * ab + 2) * Cfg::A_B);
      int prev_stage = -1;
      uint32_t prev_buf = 0, prev_ph = 0;
      bool prev_first = true;
      for (int j = 0; j <= ccnt; ++j) {
        if (j < ccnt) {
          const uint32_t buf = ctile % kCBufs;
          mbar_wait(&x_full[stage], sphase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t xh = smem_u32(sX + (2 * stage) * Cfg::TILE_B);
            const uint32_t xl = smem_u32(sX + (2 * stage + 1) * Cfg::TILE_B);
            const uint32_t d = tmem + buf * kBN;
#pragma unroll
            for (int kk = 0; kk < DP / 16; ++kk)  // s_hi . hi
              mma_ss_f16(d, umma_desc(ah + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                         umma_desc(xh + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT), IDESC1, kk > 0);
#pragma unroll
            for (int kk = 0; kk < DP / 16; ++kk)  // + (s_hi 2^-11) . lo
              mma_ss_f16(d, umma_desc(as + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                         umma_desc(xl + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT), IDESC1, 1u);
#pragma unroll
            for (int kk = 0; kk < DP / 16; ++kk)  // + s_lo . hi
              mma_ss_f16(d, umma_desc(al + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT),
                         umma_desc(xh + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT), IDESC1, 1u);
            tc_commit(&c_full[buf]);
          }
          __syncwarp();
        }
        if (prev_stage >= 0) {
          // G += P[prev] . [hi | lo][prev]: 16 pixels per instruction; the lo limb tile is the
          // second MN atom (LBO = tile stride).  Count-pass items only release the buffer.
          mbar_wait(&p_full[prev_buf], prev_ph);
          tc_fence_after();
          if (lane == 0) {
            if (w.mode == 0) {
              const uint32_t xh = smem_u32(sX + (2 * prev_stage) * Cfg::TILE_B);
#pragma unroll
              for (int k = 0; k < kBN / 16; ++k) {
                const uint64_t bd = umma_desc(xh + k * 16 * Cfg::ROW_B, Cfg::TILE_B, Cfg::SBO, Cfg::LAYOUT);
                mma_ts_f16(g_tmem, tmem + prev_buf * kBN + k * 8, bd, IDESC2, (prev_first && k == 0) ? 0u : 1u);
              }
            }
            tc_commit(&x_empty[prev_stage]);
          }
          __syncwarp();
          prev_first = false;
        }
        if (j < ccnt) {
          prev_stage = stage;
          prev_buf = ctile % kCBufs;
          prev_ph = (ctile / kCBufs) & 1;
          ++ctile;
          if (++stage == kStages) { stage = 0; sphase ^= 1; }
        }
      }
      if (lane == 0) {
        tc_commit(&a_empty[ab]);
        tc_commit(&g_full[ab]);
      }
      __syncwarp();
    }
  } else {
    // ================================ epilogue (warps 2..5) ================================
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;          // seed row within the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const float tau = p.tau_f * kLimb;      // C is scaled by 2^11 (exact power-of-two scaling)
    uint32_t ctile = 0;
    int it = 0;
    double gs[DP];                           // segment sum of 2^11 G (exact integers / 2^11)
#pragma unroll
    for (int k = 0; k < DP; ++k) gs[k] = 0.0;
    int cnt = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const ItemDesc w = item_desc(p, item);
      const int ccnt = min(kChunkTiles, p.n_ptiles - w.chunk * kChunkTiles);
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      for (int j = 0; j < ccnt; ++j, ++ctile) {
        const uint32_t buf = ctile % kCBufs;
        mbar_wait(&c_full[buf], (ctile / kCBufs) & 1);
        tc_fence_after();
        const uint32_t tb = tmem + lane_base + buf * kBN;
        if (w.mode == 0) {
          // steady state: weights only (2 FADD + PRMT + LOP3 per pixel pair)
#pragma unroll
          for (int qq = 0; qq < kBN / 32; ++qq) {
            uint32_t v[32];
            tmem_ld32(tb + qq * 32, v);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              pk[i] = flat_kernel_pair(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]), tau);
            tmem_st16(tb + qq * 16, pk);
          }
          tmem_st_wait();
        } else {
          // count pass: window sizes of the converged modes
          __half2 acc = __float2half2_rn(0.f);
#pragma unroll
          for (int qq = 0; qq < kBN / 32; ++qq) {
            uint32_t v[32];
            tmem_ld32(tb + qq * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t pk = flat_kernel_pair(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]), tau);
              acc = __hadd2(acc, *reinterpret_cast<const __half2*>(&pk));  // exact: <= 64 per lane
            }
          }
          const float2 a2 = __half22float2(acc);
          cnt += (int)(a2.x + a2.y);
        }
        tc_fence_before();
        mbar_arrive(&p_full[buf]);
      }
      mbar_wait(&g_full[ab], aph);
      tc_fence_after();
      if (w.mode == 0) {
        uint32_t g[2 * DP];
        if constexpr (DP == 16) {
          tmem_ld32(tmem + lane_base + Cfg::G_COL + ab * Cfg::G_N, *reinterpret_cast<uint32_t(*)[32]>(g));
        } else {
          tmem_ld32(tmem + lane_base + Cfg::G_COL + ab * Cfg::G_N, *reinterpret_cast<uint32_t(*)[32]>(g));
          tmem_ld32(tmem + lane_base + Cfg::G_COL + ab * Cfg::G_N + 32, *reinterpret_cast<uint32_t(*)[32]>(g + 32));
        }
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < DP; ++k)
          gs[k] += (double)__uint_as_float(g[k]) + (double)__uint_as_float(g[DP + k]) * (1.0 / kLimb);
      }
      tc_fence_before();
      mbar_arrive(&g_empty[ab]);
      // flush the segment when the next item belongs to another seed tile (or at the end)
      const int t = item / p.n_chunks;
      const bool last = (item + 1 == i_end) || ((item + 1) / p.n_chunks != t);
      if (last) {
        const size_t r = (size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row;
        if (w.mode == 0) {
          double* dst = p.gacc + r * DP;
#pragma unroll
          for (int k = 0; k < DP; ++k) {
            if (gs[k] != 0.0) atomicAdd(dst + k, gs[k]);
            gs[k] = 0.0;
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
    iter_kernel<16><<<grid, 192, IterCfg<16>::SMEM, st>>>(tm, p);
  } else {
    iter_kernel<32><<<grid, 192, IterCfg<32>::SMEM, st>>>(tm, p);
  }
  return cudaGetLastError();
}

cudaError_t setup_iter_attrs() {
  cudaError_t e = cudaFuncSetAttribute(iter_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, IterCfg<16>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(iter_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, IterCfg<32>::SMEM);
}

}  // namespace fms
