// k_assign.cu -- K5 on 5th-generation tensor cores: nearest-centre labels and window coverage.
//
// Alg. 2 l.12-14: every pixel takes the label of its most similar mode,
//     label = argmax_k x_hat . c_k   (lowest k on ties, R21)
//     covered = max_k x_hat . c_k >= tau   (inside some mode's window, Eq. 11 / R5)
// plus the per-centre histogram and the count of uncovered & unvisited pixels OSOP needs (K7).
//
// The similarity block is the transpose of K2's: D[pixel][centre] = X_hat . C^T with the pixel
// tile as A (M = 128 pixels, the fp16 limb tiles K2 streams, K-major) and the frame's centres as B
// (N = Kc rounded up to 16, at most 128), with the same three-term split as K2:
//     2^11 D = hi.c_hi + lo.(c_hi 2^-11) + hi.c_lo      (fp32 accumulate, ~1e-7 error)
// so coverage takes exactly K2's window decision [2^11 x.c >= 2^11 tau] (fp32).  One TMEM lane
// per pixel turns the row argmax into a per-thread scan of Kc registers.
//
//   * warp 0   : TMA producer of pixel tiles (hi, lo); converts the frame's centres to the fp16
//                split on the fly and stores them into shared memory in the K-major swizzled layout
//                the MMA descriptor expects (double buffered by frame).
//   * warps 1-2: MMA issuers taking alternate tiles, D[i % 4] (128 TMEM columns each).
//   * warps 3-18: four groups of 4 warps (one per TMEM lane quarter) take the tiles round robin;
//                the per-pixel argmax is a dependent scan, so it needs the thread parallelism.
// Two instantiations: NMAX = 128 (frames with 1..128 centres) and 256 (129..256); frames with more
// are left to the CUDA-core kernel (assign_kernel in k_post.cu).
#include <type_traits>

#include "fms_device.cuh"

namespace fms {

constexpr int kAsgMmaWarps = 2;                 // MMA issuers, alternate tiles
constexpr int kAsgEpiWarp0 = 1 + kAsgMmaWarps;

// NMAX = the most centres a frame may have to be assigned by this instantiation (one MMA, N <= NMAX):
// 128 (frames with 1..128 centres) or 256 (129..256, e.g. C4's ~200 cells); the CUDA-core kernel
// (assign_kernel, k_post.cu) takes frames with more.  TMEM holds 512 / NMAX similarity buffers, one
// per epilogue group of 4 warps.
// Timing experiment: -DK5_TIMELINE records clock64 events of CTA 0 of the first <16, 128> launch
// ([role][tile][event]; role 0 producer, 1 MMA, 2.. epilogue warps q = 0 of each group) into a device
// array read by fms_k5_timeline (exported by that build only); the production build compiles it away.
#ifdef K5_TIMELINE
__device__ long long k5_tl[(2 + 4) * 1024 * 8];
__device__ int k5_tl_done;
#define K5_TL(role, tile, ev)                                                                        \
  do {                                                                                               \
    if (tl_on && lane == 0 && (tile) < 1024) k5_tl[((role) * 1024 + (tile)) * 8 + (ev)] = clock64(); \
  } while (0)
#else
#define K5_TL(role, tile, ev) \
  do {                        \
  } while (0)
#endif

constexpr int kAsgMaxList = 2048;  // frames listed per launch (larger batches walk all frames)

template <int DP, int NMAX>
struct AsgCfg {
  static constexpr int GROUPS = 512 / NMAX;               // epilogue groups (tile mod GROUPS)
  static constexpr int EPI_THREADS = GROUPS * 4 * 32;
  static constexpr int THREADS = kAsgEpiWarp0 * 32 + EPI_THREADS;
  static constexpr int ROW_B = DP * 2;
  static constexpr int TILE_B = kBN * ROW_B;              // one pixel tile, one limb
  static constexpr int CEN_B = NMAX * ROW_B;              // one centre split
  static constexpr uint32_t LAYOUT = DP == 16 ? 6u : 4u;  // SWIZZLE_32B / SWIZZLE_64B
  static constexpr uint32_t SBO = 8 * ROW_B;
  // K5 streams the limbs once per round (HBM-bound): as many pixel stages in flight as shared memory
  // holds next to the two centre buffers (8 stages kept the stream latency-bound at ~2.7 TB/s)
  static constexpr int FIXED = 1024 + 2 * 3 * CEN_B + 2 * NMAX * 4 + 1024;
  static constexpr int DYN_MAX = 232448 - kAsgMaxList * 4 - 1024;  // the static active-frame list and scan scratch
  static constexpr int STAGES_FIT = (DYN_MAX - FIXED) / (2 * TILE_B);
  // even: stage s is always consumed by MMA warp s % 2 (tiles alternate between the two issuers)
  static constexpr int STAGES = (STAGES_FIT < 24 ? STAGES_FIT : 24) & ~1;
  static constexpr int SMEM = FIXED + STAGES * 2 * TILE_B;
  static_assert(STAGES >= 4 && SMEM <= DYN_MAX, "shared memory");
  static_assert((2 * STAGES + 4 + 2 * GROUPS) * 8 + 4 <= 1024, "barrier area");
};

// byte offset of (row, 16-byte chunk) in a K-major tile with 32-byte (SW32) / 64-byte (SW64)
// swizzled rows -- the layout TMA writes for the pixel tiles (16-byte chunk index XOR row bits)
template <int DP>
__device__ __forceinline__ uint32_t swz_off(int row, int chunk) {
  if constexpr (DP == 16) return row * 32 + ((chunk ^ ((row >> 2) & 1)) << 4);
  else return row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4);
}


template <int NMAX>
__device__ __forceinline__ bool asg_frame_active(const Params& p, int f) {
  const FrameCtl& c = p.ctl[f];
  return c.phase == PH_POST && c.Kc > (NMAX == 128 ? 0 : 128) && c.Kc <= NMAX;
}

template <int DP, int NMAX>
__global__ void __launch_bounds__(AsgCfg<DP, NMAX>::THREADS, 1)
    assign_tc_kernel(const __grid_constant__ TMaps tm, Params p) {
  using Cfg = AsgCfg<DP, NMAX>;
#ifdef K5_TIMELINE
  const bool tl_on = blockIdx.x == 0 && NMAX == 128 && !*(volatile int*)&k5_tl_done;
#endif
  constexpr int kAsgMaxN = NMAX, kAsgGroups = Cfg::GROUPS, kAsgEpiThreads = Cfg::EPI_THREADS;
  if (NMAX > 128 && p.counters[19] <= 128) return;  // no frame of this round has 129..256 centres
  // The CTAs split the pixel tiles of the frames this instantiation assigns (a compact list of active
  // frames), not of all B frames: frames that finished OSOP earlier, or whose centre count belongs to
  // the other instantiation, would otherwise leave whole CTAs idle.  (Splitting by a per-frame cost
  // estimate, tiles x (96 + Kc), measured no faster than equal tile counts.)
  __shared__ int s_act[kAsgMaxList];
  __shared__ int s_sm[33];
  const bool listed = p.B <= kAsgMaxList;
  int n_fr = p.B;
  const int n_pt = p.n_ptiles;
  if (listed) {
    int carry = 0;
    for (int f0 = 0; f0 < p.B; f0 += blockDim.x) {
      const int f = f0 + threadIdx.x;
      const int a = (f < p.B && asg_frame_active<NMAX>(p, f)) ? 1 : 0;
      int tot;
      const int pos = carry + block_excl_scan(a, s_sm, &tot);
      if (a) s_act[pos] = f;
      carry += tot;
    }
    __syncthreads();
    n_fr = carry;
  }
  const long long n_items = (long long)n_fr * n_pt;
  const int i_begin = (int)((n_items * blockIdx.x) / gridDim.x);
  const int i_end = (int)((n_items * (blockIdx.x + 1)) / gridDim.x);
  auto frame_of = [&](int fa) { return listed ? s_act[fa] : fa; };
  if (i_begin >= i_end) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sC = smem;                                   // [2 frames][hi, hs, lo][CEN_B]
  uint8_t* sX = sC + 2 * 3 * Cfg::CEN_B;                // [STAGES][hi, lo][TILE_B]
  int* shist = reinterpret_cast<int*>(sX + Cfg::STAGES * 2 * Cfg::TILE_B);  // [2][kAsgMaxN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(shist + 2 * kAsgMaxN);
  uint64_t* x_full = bars;                   // [STAGES]
  uint64_t* x_empty = x_full + Cfg::STAGES;  // [STAGES]
  uint64_t* c_full = x_empty + Cfg::STAGES;  // [2] centres of a frame staged
  uint64_t* c_empty = c_full + 2;            // [2] last MMA of that frame done
  uint64_t* d_full = c_empty + 2;            // [kAsgGroups] similarity block ready
  uint64_t* d_empty = d_full + kAsgGroups;   // [kAsgGroups] loaded by the epilogue group
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(d_empty + kAsgGroups);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&c_full[i], 32); mbar_init(&c_empty[i], kAsgMmaWarps); }
    for (int i = 0; i < kAsgGroups; ++i) { mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], 4); }
    fence_barrier_init();
    fence_proxy_async();
  }
  for (int i = threadIdx.x; i < 2 * kAsgMaxN; i += blockDim.x) shist[i] = 0;
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ================================ producer ================================
    int stage = 0, fcount = 0;
    uint32_t sphase = 0;
    // frame by frame over the CTA's item range (every listed frame is active)
    for (int fa = i_begin / n_pt; (long long)fa * n_pt < i_end; ++fa) {
      const int f = frame_of(fa);
      if (!asg_frame_active<NMAX>(p, f)) continue;
      const int s0 = max(i_begin, fa * n_pt), s1 = min(i_end, (fa + 1) * n_pt);
      {
        // stage this frame's centre split into buffer fcount & 1 once its previous user is done
        const int cb = fcount & 1;
        mbar_wait(&c_empty[cb], ((fcount >> 1) & 1) ^ 1);
        const int Kc = p.ctl[f].Kc;
        const float* cent = p.cent + (size_t)f * p.C_cap * DP;
        uint8_t* dst = sC + cb * 3 * Cfg::CEN_B;
        const int n_rows = (Kc + 15) & ~15;
        for (int idx = lane; idx < n_rows * (DP / 8); idx += 32) {  // one 8-feature chunk per step
          const int r = idx / (DP / 8), ch = idx - r * (DP / 8);
          __align__(16) __half hi[8], hs[8], lo[8];
          float row[DP];  // the centre's operand row (augmented for the Euclidean metric, R24)
          if (r < Kc) {
            operand_row<DP>(p, f, cent + (size_t)r * DP, row);
          } else {
#pragma unroll
            for (int e = 0; e < DP; ++e) row[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) split_seed(row[ch * 8 + e], hi[e], hs[e], lo[e]);
          const uint32_t off = swz_off<DP>(r, ch);
          *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(hi);
          *reinterpret_cast<uint4*>(dst + Cfg::CEN_B + off) = *reinterpret_cast<const uint4*>(hs);
          *reinterpret_cast<uint4*>(dst + 2 * Cfg::CEN_B + off) = *reinterpret_cast<const uint4*>(lo);
        }
        fence_proxy_async();  // generic-proxy stores -> visible to the tensor core
        mbar_arrive(&c_full[cb]);
        ++fcount;
      }
      const int row0 = (int)((long long)f * p.n_pad - (long long)fa * n_pt * kBN);  // + item * kBN
      for (int item = s0; item < s1; ++item) {
        K5_TL(0, item - i_begin, 0);
        mbar_wait(&x_empty[stage], sphase ^ 1);
        K5_TL(0, item - i_begin, 1);
        if (lane == 0) {
          const int xrow = row0 + item * kBN;
          mbar_expect_tx(&x_full[stage], 2 * Cfg::TILE_B);
          tma_load_2d(sX + (2 * stage) * Cfg::TILE_B, &tm.xh, &x_full[stage], 0, xrow);
          tma_load_2d(sX + (2 * stage + 1) * Cfg::TILE_B, &tm.xl, &x_full[stage], 0, xrow);
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp <= kAsgMmaWarps) {
    // ================================ MMA issuers ================================
    // A = pixel tile (M = 128, K-major), B = centres (N = Kc rounded to 16, K-major).  Two warps take
    // alternate tiles: an issuing warp blocks while its MMAs execute, so one warp alone serialises
    // its barrier waits and commits with the tensor work.  Tile i uses D buffer i % 4 and pixel
    // stage i % STAGES, both always of the same parity, so each barrier keeps a single committer.
    const int mw = warp - 1;
    const uint64_t dx0 = umma_desc(smem_u32(sX), 16, Cfg::SBO, Cfg::LAYOUT);
    const uint64_t dc0 = umma_desc(smem_u32(sC), 16, Cfg::SBO, Cfg::LAYOUT);
    int fcount = 0, i = 0;
    uint32_t idesc = 0;
    uint64_t dch = 0, dcs = 0, dcl = 0;
    for (int fa = i_begin / n_pt; (long long)fa * n_pt < i_end; ++fa) {
      const int f = frame_of(fa);
      if (!asg_frame_active<NMAX>(p, f)) continue;
      const int s0 = max(i_begin, fa * n_pt), s1 = min(i_end, (fa + 1) * n_pt);
      {
        if (fcount > 0) tc_commit_el(&c_empty[(fcount - 1) & 1]);  // previous frame's centres free
        const int cb = fcount & 1;
        mbar_wait(&c_full[cb], (fcount >> 1) & 1);
        tc_fence_after();
        const int nN = (p.ctl[f].Kc + 15) & ~15;
        idesc = idesc_f16(kBM, nN, 0, 0);
        dch = dc0 + (uint64_t)((cb * 3 * Cfg::CEN_B) >> 4);
        dcs = dch + (Cfg::CEN_B >> 4);
        dcl = dch + (2 * Cfg::CEN_B >> 4);
        ++fcount;
      }
      for (int item = s0; item < s1; ++item, ++i) {
        if ((i & 1) != mw) continue;
        const int stage = i % Cfg::STAGES;
        const uint32_t sphase = (uint32_t)(i / Cfg::STAGES) & 1;
        const uint32_t db = i % kAsgGroups;
        K5_TL(1, i, 0);
        if (i >= kAsgGroups) mbar_wait(&d_empty[db], ((i / kAsgGroups) - 1) & 1);
        K5_TL(1, i, 1);
        mbar_wait(&x_full[stage], sphase);
        K5_TL(1, i, 2);
        tc_fence_after();
        const uint64_t dxh = dx0 + (uint64_t)(stage * (2 * Cfg::TILE_B >> 4));
        const uint64_t dxl = dxh + (Cfg::TILE_B >> 4);
        const uint32_t d = tmem + db * kAsgMaxN;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk) mma_ss_f16_el(d, dxh + kk * 2, dch + kk * 2, idesc, kk > 0);  // hi.c_hi
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk) mma_ss_f16_el(d, dxl + kk * 2, dcs + kk * 2, idesc, 1u);  // lo.c_hs
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk) mma_ss_f16_el(d, dxh + kk * 2, dcl + kk * 2, idesc, 1u);  // hi.c_lo
        tc_commit_el(&d_full[db]);
        tc_commit_el(&x_empty[stage]);
        K5_TL(1, i, 3);
      }
    }
    if (fcount > 0) tc_commit_el(&c_empty[(fcount - 1) & 1]);
  } else {
    // ================================ epilogue ================================
    const int q = warp & 3;
    const int grp = (warp - kAsgEpiWarp0) >> 2;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const float tau2 = p.tau_f * kLimb;  // D is 2^11-scaled
    int fcount = 0;
    int cand = 0;
    auto flush = [&](int f, int hb) {  // per-frame histogram and candidate count -> global
      asm volatile("bar.sync 1, %0;" ::"n"(kAsgEpiThreads) : "memory");  // the epilogue warps
      int* hs = shist + hb * kAsgMaxN;
      const int Kc = p.ctl[f].Kc;
      for (int k = threadIdx.x - kAsgEpiWarp0 * 32; k < Kc; k += kAsgEpiThreads) {
        if (hs[k]) atomicAdd(&p.hist[(size_t)f * p.C_cap + k], hs[k]);
        hs[k] = 0;
      }
      const int tot = __reduce_add_sync(0xffffffffu, cand);
      if (lane == 0 && tot) atomicAdd((unsigned long long*)&p.ctl[f].ncand, (unsigned long long)tot);
      cand = 0;
      asm volatile("bar.sync 1, %0;" ::"n"(kAsgEpiThreads) : "memory");
    };
    // Walk the CTA's item range frame by frame: a frame is active (assigned here) or not as a whole,
    // so the active items form contiguous runs and group grp takes every kAsgGroups-th of them
    // directly (the producer and the MMA warp number the same active items 0, 1, 2, ...).
    int n_act = 0;  // active items of this CTA before the current frame
    for (int fa = i_begin / p.n_ptiles; (long long)fa * p.n_ptiles < i_end; ++fa) {
      const int f = frame_of(fa);
      const int s0 = max(i_begin, fa * p.n_ptiles), s1 = min(i_end, (fa + 1) * p.n_ptiles);
      if (!asg_frame_active<NMAX>(p, f)) continue;
      ++fcount;
      const int Kc = p.ctl[f].Kc;
      for (int item = s0 + (((grp - n_act) % kAsgGroups) + kAsgGroups) % kAsgGroups; item < s1;
           item += kAsgGroups) {
        const int my = n_act + (item - s0);
        const int t = item - fa * p.n_ptiles;
        const long long px = (long long)t * kBN + q * 32 + lane;
        const uint8_t fl = px < p.n ? p.flags[flag_at(p, f, px)] : 0;  // latency overlaps the wait below
        const uint32_t db = my % kAsgGroups;
        const bool tl = q == 0;
        if (tl) K5_TL(2 + grp, my, 0);
        mbar_wait_susp(&d_full[db], (my / kAsgGroups) & 1);  // parked: the MMA warp shares its sub-partition
        if (tl) K5_TL(2 + grp, my, 1);
        tc_fence_after();
        // argmax over the row in four interleaved streams (short dependency chains); each stream
        // keeps its first maximum, the merge prefers the larger value, then the lower index
        float bv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        int bl[4] = {0, 1, 2, 3};
        const uint32_t dbase = tmem + lane_base + db * kAsgMaxN;
#ifdef K5_OFF
        const int kc_scan = (K5_OFF & 1) ? 0 : Kc;  // timing experiment: no argmax
#else
        const int kc_scan = Kc;
#endif
        for (int c0 = 0; c0 < kc_scan; c0 += 64) {
          uint32_t v[64];
          tmem_ld64(dbase + c0, v);
          tmem_ld_wait();
          // only the 16-column groups that hold centres (compile-time bodies: v stays in registers);
          // columns past Kc in the last group read as -inf
          const int nk = min(64, Kc - c0);
          auto scan = [&](auto groups) {
            constexpr int G16 = decltype(groups)::value;
#pragma unroll
            for (int k = 0; k < 16 * G16; ++k) {
              const float dv = (k < 16 * (G16 - 1) || k < nk) ? __uint_as_float(v[k]) : -INFINITY;
              if (dv > bv[k & 3]) { bv[k & 3] = dv; bl[k & 3] = c0 + k; }
            }
          };
          switch ((nk + 15) >> 4) {
            case 1: scan(std::integral_constant<int, 1>{}); break;
            case 2: scan(std::integral_constant<int, 2>{}); break;
            case 3: scan(std::integral_constant<int, 3>{}); break;
            default: scan(std::integral_constant<int, 4>{}); break;
          }
        }
        float best = bv[0];
        int lab = bl[0];
#pragma unroll
        for (int s2 = 1; s2 < 4; ++s2)
          if (bv[s2] > best || (bv[s2] == best && bl[s2] < lab)) { best = bv[s2]; lab = bl[s2]; }
        if (tl) K5_TL(2 + grp, my, 2);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[db]);
        if (px < p.n) {
          const size_t pi = (size_t)f * p.n + px;
          const bool covered = best >= tau2;
          p.flags[flag_at(p, f, px)] = (uint8_t)((fl & ~PF_COVERED) | (covered ? PF_COVERED : 0));
          labels_of(p)[pi] = lab;
          // warp-aggregated histogram: neighbouring pixels mostly share a label, and 32 same-address
          // shared atomics would serialise
          const unsigned same = __match_any_sync(__activemask(), lab);
          if ((__ffs(same) - 1) == lane) atomicAdd(&shist[((fcount - 1) & 1) * kAsgMaxN + lab], __popc(same));
          cand += (!covered && !(fl & PF_VISITED)) ? 1 : 0;
        }
        if (tl) K5_TL(2 + grp, my, 3);
      }
      n_act += s1 - s0;
      flush(f, (fcount - 1) & 1);  // every epilogue warp flushes every active frame of the range
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
#ifdef K5_TIMELINE
  if (blockIdx.x == 0 && threadIdx.x == 0 && NMAX == 128) k5_tl_done = 1;
#endif
}

#ifdef K5_TIMELINE
}  // namespace fms
extern "C" int fms_k5_timeline(long long* host, int n) {
  if (n > (int)(sizeof(fms::k5_tl) / 8)) n = (int)(sizeof(fms::k5_tl) / 8);
  return cudaMemcpyFromSymbol(host, fms::k5_tl, (size_t)n * 8) == cudaSuccess ? n : -1;
}
namespace fms {
#endif

cudaError_t setup_assign_attrs() {
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e = cudaFuncSetAttribute(assign_tc_kernel<16, 128>, a, AsgCfg<16, 128>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(assign_tc_kernel<32, 128>, a, AsgCfg<32, 128>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(assign_tc_kernel<16, 256>, a, AsgCfg<16, 256>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(assign_tc_kernel<32, 256>, a, AsgCfg<32, 256>::SMEM);
  return e;
}

// both tensor-core instantiations; a frame is assigned by the one whose centre range holds its Kc
// (CTAs of the other exit after scanning their item range)
cudaError_t launch_assign_tc(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st) {
  if (DP == 16) {
    assign_tc_kernel<16, 128><<<grid, AsgCfg<16, 128>::THREADS, AsgCfg<16, 128>::SMEM, st>>>(tm, p);
    if (p.C_cap > 128) assign_tc_kernel<16, 256><<<grid, AsgCfg<16, 256>::THREADS, AsgCfg<16, 256>::SMEM, st>>>(tm, p);
  } else {
    assign_tc_kernel<32, 128><<<grid, AsgCfg<32, 128>::THREADS, AsgCfg<32, 128>::SMEM, st>>>(tm, p);
    if (p.C_cap > 128) assign_tc_kernel<32, 256><<<grid, AsgCfg<32, 256>::THREADS, AsgCfg<32, 256>::SMEM, st>>>(tm, p);
  }
  return cudaGetLastError();
}

}  // namespace fms
