// k_iter.cu -- K2: the lockstep mean-shift iteration on 5th-generation tensor cores.
//
// One lockstep step of Alg. 2 lines 4-9 for every active seed of every frame
// in the batch, evaluated densely as P:210 prescribes ("does not search which points belong to S_h
// ... multiplies ... with the kernel function"):
//
//     C = S_hat . X_hat^T              seeds x pixels cosine similarity   (Eq. 1/9)
//     W = [C >= tau], tau = 1 - h      flat kernel, inclusive              (Eq. 11; R5)
//     G = W . X_hat,  cnt = W . 1      windowed sums                       (Eq. 8 / R1)
//
// Structure (fused-attention style; the S x N weight matrix never leaves the SM):
//   * work item = (frame, 128-seed tile, contiguous range of 128-pixel tiles); persistent CTAs
//     (one per SM) stride over the device-built item list.
//   * warp 0  : TMA producer  -- seed tile (A) and a ring of pixel tiles (B), 32B/64B swizzled.
//   * warp 1  : MMA issuer    -- tcgen05.mma kind::f16:  C[buf] = A . X^T  (M=128, N=128, K=DP)
//                                 then G += P[buf] . X   (A = P from TMEM, B = same X tile read
//                                 MN-major, M=128, N=DP, K=16 per instruction).
//   * warps 2-5: epilogue      -- tcgen05.ld C rows, flat kernel -> fp16 0/1 weights P written back
//                                 over C in TMEM (tcgen05.st), window counts in registers; at the
//                                 end of an item, G rows -> fp32 split-pixel partials in HBM.
//   TMEM: 3 x 128 columns of C/P (triple buffered) + 2 x DP columns of G (double buffered).
// The partial sums of one (frame, seed tile) are reduced in a fixed split order by K3, so results
// do not depend on scheduling.
#include "fms_device.cuh"

namespace fms {

template <int DP>
struct IterCfg {
  static constexpr int ROW_B = DP * 2;                    // bytes per row (fp16)
  static constexpr int TILE_B = kBN * ROW_B;              // pixel tile bytes
  static constexpr int A_B = kBM * ROW_B;                 // seed tile bytes
  static constexpr uint32_t LAYOUT = DP == 16 ? 6u : 4u;  // SWIZZLE_32B / SWIZZLE_64B
  static constexpr uint32_t SBO = 8 * ROW_B;              // 8-row core-matrix group stride
  static constexpr int G_COL = kCBufs * kBN;              // TMEM column of G buffer 0
  static constexpr int SMEM = 1024 /*align slack*/ + 2 * A_B + kStages * TILE_B + 1024 /*barriers*/;
};

template <int DP>
__global__ void __launch_bounds__(192, 1)
    iter_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_s, Params p) {
  using Cfg = IterCfg<DP>;
  const int n_items = p.counters[0];
  if ((int)blockIdx.x >= n_items) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // [2][A_B]
  uint8_t* sX = smem + 2 * Cfg::A_B;                   // [kStages][TILE_B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + kStages * Cfg::TILE_B);
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
  if (warp == 0 && lane == 0) { tma_prefetch(&tm_x); tma_prefetch(&tm_s); }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ================================ TMA producer ================================
    // whole warp walks the schedule; lane 0 issues
    int stage = 0;
    uint32_t sphase = 0;
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const WorkItem w = p.items[item];
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&a_empty[ab], aph ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&a_full[ab], Cfg::A_B);
        tma_load_2d(sA + ab * Cfg::A_B, &tm_s, &a_full[ab], 0, w.f * p.S_pad + w.tile * kBM);
      }
      __syncwarp();
      const long long row0 = (long long)w.f * p.n_pad + (long long)w.begin * kBN;
      for (int j = 0; j < w.count; ++j) {
        mbar_wait(&x_empty[stage], sphase ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&x_full[stage], Cfg::TILE_B);
          tma_load_2d(sX + stage * Cfg::TILE_B, &tm_x, &x_full[stage], 0, (int)(row0 + (long long)j * kBN));
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // whole warp walks the schedule and waits; lane 0 issues tcgen05.mma / tcgen05.commit
    constexpr uint32_t IDESC1 = idesc_f16(kBM, kBN, 0, 0);  // C = A . X^T, both K-major
    constexpr uint32_t IDESC2 = idesc_f16(kBM, DP, 0, 1);   // G += P . X, X read MN-major
    int stage = 0;
    uint32_t sphase = 0;
    uint32_t ctile = 0;  // running tile counter -> C buffer index and phase
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const WorkItem w = p.items[item];
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const uint32_t g_tmem = tmem + Cfg::G_COL + ab * DP;
      mbar_wait(&a_full[ab], aph);
      mbar_wait(&g_empty[ab], aph ^ 1);
      tc_fence_after();
      const uint32_t a_addr = smem_u32(sA + ab * Cfg::A_B);
      int prev_stage = -1;
      uint32_t prev_buf = 0, prev_ph = 0;
      bool prev_first = true;
      for (int j = 0; j <= w.count; ++j) {
        if (j < w.count) {
          const uint32_t buf = ctile % kCBufs;
          mbar_wait(&x_full[stage], sphase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t x_addr = smem_u32(sX + stage * Cfg::TILE_B);
#pragma unroll
            for (int kk = 0; kk < DP / 16; ++kk) {
              const uint64_t ad = umma_desc(a_addr + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT);
              const uint64_t bd = umma_desc(x_addr + kk * 32, 16, Cfg::SBO, Cfg::LAYOUT);
              mma_ss_f16(tmem + buf * kBN, ad, bd, IDESC1, kk > 0);
            }
            tc_commit(&c_full[buf]);
          }
          __syncwarp();
        }
        if (prev_stage >= 0) {
          // G += P[prev] . X[prev]  (16 pixels per instruction, P packed 2 fp16 per column)
          mbar_wait(&p_full[prev_buf], prev_ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t x_addr = smem_u32(sX + prev_stage * Cfg::TILE_B);
#pragma unroll
            for (int k = 0; k < kBN / 16; ++k) {
              const uint64_t bd = umma_desc(x_addr + k * 16 * Cfg::ROW_B, Cfg::SBO * 2, Cfg::SBO, Cfg::LAYOUT);
              mma_ts_f16(g_tmem, tmem + prev_buf * kBN + k * 8, bd, IDESC2, (prev_first && k == 0) ? 0u : 1u);
            }
            tc_commit(&x_empty[prev_stage]);
          }
          __syncwarp();
          prev_first = false;
        }
        if (j < w.count) {
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
    const float tau = p.tau_f;
    uint32_t ctile = 0;
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const WorkItem w = p.items[item];
      const int ab = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      int cnt = 0;
      for (int j = 0; j < w.count; ++j, ++ctile) {
        const uint32_t buf = ctile % kCBufs;
        mbar_wait(&c_full[buf], (ctile / kCBufs) & 1);
        tc_fence_after();
        const uint32_t tb = tmem + lane_base + buf * kBN;
#pragma unroll
        for (int qq = 0; qq < kBN / 32; ++qq) {
          uint32_t v[32];
          tmem_ld32(tb + qq * 32, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const bool w0 = __uint_as_float(v[2 * i]) >= tau;
            const bool w1 = __uint_as_float(v[2 * i + 1]) >= tau;
            pk[i] = (w0 ? 0x3C00u : 0u) | (w1 ? 0x3C000000u : 0u);
            cnt += (int)w0 + (int)w1;
          }
          tmem_st16(tb + qq * 16, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[buf]);
      }
      mbar_wait(&g_full[ab], aph);
      tc_fence_after();
      uint32_t g[DP];
      if constexpr (DP == 16) {
        tmem_ld16(tmem + lane_base + Cfg::G_COL + ab * DP, *reinterpret_cast<uint32_t(*)[16]>(g));
      } else {
        tmem_ld32(tmem + lane_base + Cfg::G_COL + ab * DP, *reinterpret_cast<uint32_t(*)[32]>(g));
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&g_empty[ab]);
      float4* dst = reinterpret_cast<float4*>(p.part_g + ((size_t)item * kBM + row) * DP);
#pragma unroll
      for (int i = 0; i < DP / 4; ++i)
        dst[i] = make_float4(__uint_as_float(g[4 * i]), __uint_as_float(g[4 * i + 1]), __uint_as_float(g[4 * i + 2]),
                             __uint_as_float(g[4 * i + 3]));
      p.part_c[(size_t)item * kBM + row] = cnt;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template __global__ void iter_kernel<16>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                         Params);
template __global__ void iter_kernel<32>(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                         Params);

int iter_smem_bytes(int DP) { return DP == 16 ? IterCfg<16>::SMEM : IterCfg<32>::SMEM; }

cudaError_t launch_iter(int DP, const CUtensorMap& tx, const CUtensorMap& ts, const Params& p, int grid,
                        cudaStream_t st) {
  if (DP == 16) {
    iter_kernel<16><<<grid, 192, IterCfg<16>::SMEM, st>>>(tx, ts, p);
  } else {
    iter_kernel<32><<<grid, 192, IterCfg<32>::SMEM, st>>>(tx, ts, p);
  }
  return cudaGetLastError();
}

cudaError_t setup_iter_attrs() {
  cudaError_t e = cudaFuncSetAttribute(iter_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, IterCfg<16>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(iter_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, IterCfg<32>::SMEM);
}

}  // namespace fms
