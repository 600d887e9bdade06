// k_iter8.cu -- K2 for the flat kernel (the paper's path): the lockstep mean-shift iteration with the
// weighted sum as an exact 8-bit integer contraction on the 5th-generation tensor cores.
//
// One lockstep step of Alg. 2 lines 4-9 for every active seed of every frame,
// evaluated densely as P:210 prescribes:
//
//     C = S_hat . X_hat^T              seeds x pixels cosine similarity   (Eq. 1/9)
//     W = [C >= tau], tau = 1 - h      flat kernel, inclusive              (Eq. 11; R5)
//     G = W . X_hat                    windowed sum (count cancels, R4)    (Eq. 8 / R1)
//
// Similarity: as in k_iter.cu, three kind::f16 MMAs over fixed-point fp16 limbs (s_hi.hi +
// (s_hi 2^-11).lo + s_lo.hi, error ~1e-7) into an fp32 TMEM accumulator.
//
// Weighted sum: the pixels are also stored as int8 digit planes of v = round(2^22 x_hat) =
// a 2^16 + b 2^8 + c (fms_device.cuh `digits`), 3 DP planes of 128 pixels per tile, K-major.  The
// in-window weight is the byte 255 (unsigned), so
//     Gq[:, j DP + k] = 255 sum_{in window} digit_j(x_k)        (kind::i8, s32 accumulate: EXACT)
// and G_k = (Gq[a] 2^16 + Gq[b] 2^8 + Gq[c]) / 255 = sum_{in window} v_k, an integer.  Per tile that
// is 4 MMAs of K = 32 pixels (the fp16 weighted sum needs 8 of K = 16), and the weights take 32
// TMEM columns per tile instead of 64.  Integer sums are exact for any split of the pixels, so work
// items are sized freely (plan_kernel) and CTAs merge with fp64 atomics of integers (order-free).
//
// Flat kernel in the epilogue: with C and tau_m (the float just below 2^11 tau) fp32,
//     v = C - tau_m  has its sign bit clear and a nonzero value  <=>  C > tau_m  <=>  C >= 2^11 tau
// (the rounded difference keeps the sign of the exact one and is zero only when C = tau_m).  FADD2
// forms two differences per instruction; I2IP (cvt.pack.sat.u8.s32) saturates the float bits read as
// int32 -- positive -> 255, zero or negative -> 0 -- and packs two pixels per instruction, chaining
// the previous pair into the upper half.  Four pixels' weights cost 2 FADD2 + 2 I2IP.
//
// Structure (fused-attention style; the S x N weights never leave the SM):
//   * work item = (frame, 128-seed tile, chunk of `ct` 128-pixel tiles; ct chosen per launch by
//     plan_kernel).  Persistent CTAs (one per SM) take equal contiguous ranges of the item list.
//   * warp 16  : TMA producer -- seed tile (s_hi, s_hi 2^-11, s_lo) and a ring of pixel tiles
//                                (hi, lo limbs; digit planes).
//   * warp 17  : MMA1 issuer  -- C[i % NC] = 3 MMAs (M=128, N=128, K=DP) into TMEM.
//   * warp 18  : MMA2 issuer  -- Gq += P[i % NP] . Q (kind::i8, A = P from TMEM, N = 3 DP).
//   * warps 0-15: epilogue    -- four groups of 4 warps take tiles round-robin: two tcgen05.ld of 64
//                                columns of C per warp, C handed back to MMA1 (named barrier), flat
//                                kernel -> u8 weights (tcgen05.st).  The group that handled an
//                                item's last tile drains Gq into its own int64 segment sums.
//                                Count-pass items (mode 1: the converged modes of a round) skip the
//                                weighted sum and count window members (intensity, R10).
//   TMEM: NC x 128 columns of C + NP x 32 columns of P + 3 DP columns of Gq.
#include "fms_device.cuh"

namespace fms {

namespace k8 {
#ifdef K8_EPI_WARPS
constexpr int kEpiWarps = K8_EPI_WARPS;
#else
constexpr int kEpiWarps = 16;
#endif
constexpr int kWarpTma = kEpiWarps, kWarpMma1 = kEpiWarps + 1, kWarpMma2 = kEpiWarps + 2;
constexpr int kWarpTmaQ = kEpiWarps + 3;  // producer of the digit-plane ring
constexpr int kThreads = (kEpiWarps + 4) * 32;
}  // namespace k8

template <int DP>
struct Iter8Cfg {
  // epilogue groups (tiles in flight): 4 groups of 4 warps for 16-lane rows; 32-lane rows keep 2
  // groups of 8 (their segment sums and pixel stages would not fit shared memory with 4)
#ifdef K8_GROUPS
  static constexpr int GROUPS = (DP == 16 || k8::kEpiWarps != 16) ? K8_GROUPS : 4;
#else
  static constexpr int GROUPS = 4;
#endif
  // 32-lane rows: a drain adds its sums straight to the global accumulator (fp64 atomics of exact
  // integers) instead of shared-memory segment sums, which leaves room for a deeper pixel ring
#ifdef K8_DIRECT_ALL
  static constexpr bool DIRECT = true;
#else
  static constexpr bool DIRECT = DP == 32;
#endif
  static constexpr int GROUP_WARPS = k8::kEpiWarps / GROUPS;  // a multiple of 4 (one per lane quarter)
  // 4 groups of 4 warps (the default) or 1 group of 16 warps (every warp on every tile, 32 columns
  // each: 16 TMEM loads in flight per tile; measured slower, 906 vs 805 cycles per tile).  2 groups
  // of 8 are excluded: with NC = 3 the MMA1 issuer can complete a group's c_full twice before a slow
  // warp of the group waits on it (parity aliasing), which deadlocked in a probe run.
  static constexpr int COLS_PER_WARP = kBN / (GROUP_WARPS / 4);
#ifdef K8_PART
  static constexpr int PART_MAX = K8_PART;
#else
  static constexpr int PART_MAX = 64;
#endif
  static constexpr int PART = COLS_PER_WARP < PART_MAX ? COLS_PER_WARP : PART_MAX;  // columns per tcgen05.ld
  static constexpr int PARTS = COLS_PER_WARP / PART;
  static constexpr int ROW_B = DP * 2;                    // bytes per fp16 row
  static constexpr int TILE_B = kBN * ROW_B;              // one pixel tile (one limb)
  static constexpr int A_B = kBM * ROW_B;                 // one seed tile (one split)
  static constexpr uint32_t LAYOUT = DP == 16 ? 6u : 4u;  // SWIZZLE_32B / SWIZZLE_64B (fp16 rows)
  static constexpr uint32_t SBO = 8 * ROW_B;              // 8-row core-matrix group stride
  static constexpr int NQ = 3 * DP;                       // digit planes (= Gq columns)
  static constexpr int Q_B = NQ * kBN;                    // digit planes of one tile (128 B rows, SW128)
  static constexpr int L_B = 2 * TILE_B;                  // one stage of the limb ring (hi, lo)
#ifdef K8_NC
  static constexpr int NC = DP == 16 ? K8_NC : 2;
#else
  static constexpr int NC = DP == 16 ? 3 : 2;             // C buffers
#endif
#ifdef K8_NP
  static constexpr int NP = K8_NP;
#else
  static constexpr int NP = DP == 16 ? (NC == 3 ? 2 : 3) : 3;  // P buffers (32 columns each)
#endif
  static_assert(GROUPS >= 1 && GROUPS <= 4 && k8::kEpiWarps % (4 * GROUPS) == 0,
                "epilogue layout: 4 groups of 4 warps, 1 group of 16, or 2 groups of 8 with one C buffer each");
  static constexpr int P_COL = NC * kBN;
  static constexpr int G_COL = P_COL + NP * (kBN / 4);
  static_assert(G_COL + NQ <= 512, "TMEM budget");
  // Two rings: the limbs (MMA1's B operand) free a stage when MMA1 is done with it; the digit planes
  // (MMA2's B) when MMA2 is.  A stage of the limb ring is held for a few hundred cycles, so the ring
  // prefetches far ahead of the similarity MMAs for its size.
#if defined(K8_LSTAGES) && defined(K8_QSTAGES)
  static constexpr int LSTAGES = DP == 16 ? K8_LSTAGES : 5;
  static constexpr int QSTAGES = DP == 16 ? K8_QSTAGES : 8;
#else
  static constexpr int LSTAGES = DP == 16 ? 8 : 5;
  static constexpr int QSTAGES = DP == 16 ? 10 : 8;
#endif
  static constexpr int GS_B = DIRECT ? 0 : kBM * DP * 8;  // int64 segment sums, [DP][kBM], per group
  static constexpr int SMEM = 1024 + 6 * A_B + LSTAGES * L_B + QSTAGES * Q_B + GROUPS * GS_B + 1024;
  static_assert(SMEM <= 232448, "shared memory");
  static_assert(L_B % 1024 == 0 && Q_B % 1024 == 0, "SW128 alignment of the digit planes");
};

// Work items: (frame f, chunk c of ct pixel tiles, seed tile j of f), ordered frame by frame, chunk by
// chunk, and within a chunk over the frame's seed tiles.  A frame's pixels stream from HBM once per
// step: the T_f seed tiles of a frame read the same chunk back to back (from L2), instead of each
// seed tile streaming the whole frame (pixel tiles are 14 / 28 KB, far above the tensor work's
// arithmetic intensity when every seed tile re-reads them from HBM).  Frame f's items are
// [nch tile_off(f), nch (tile_off(f) + T_f)), so the tile task at item / nch belongs to f.
struct Item8 {
  int f, tile, chunk, mode, key;  // key: frame * S_pad + tile * kBM (the segment a G drain belongs to)
  int rows;                       // active seed rows in the tile (the last tile of a frame is partial)
};
__device__ __forceinline__ Item8 item8(const Params& p, int item, int nch) {
  const int f = p.tiles[item / nch].f;
  const FrameCtl& c = p.ctl[f];
  const int T = c.n_tiles_step;
  const int L = item - nch * c.tile_off;
  const int chunk = L / T;
  const TileTask tt = p.tiles[c.tile_off + (L - chunk * T)];
  return Item8{f, tt.tile, chunk, tt.mode, f * p.S_pad + tt.tile * kBM, min(kBM, c.n_active - tt.tile * kBM)};
}

// two in-window differences per instruction: {c0 - tau_m, c1 - tau_m}
__device__ __forceinline__ void sub_tau2(uint32_t c0, uint32_t c1, float tau_m, uint32_t& d0, uint32_t& d1) {
  asm("{\n\t.reg .b64 ra, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rc, {%4, %4};\n\t"
      "add.rn.f32x2 rd, ra, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=r"(d0), "=r"(d1)
      : "r"(c0), "r"(c1), "f"(-tau_m));
}
// four pixels' weights, byte i = 255 if difference i > 0 else 0
__device__ __forceinline__ uint32_t pack_w4(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3) {
  uint32_t t, w;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(t) : "r"(d3), "r"(d2));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(d1), "r"(d0), "r"(t));
  return w;
}

// Timing experiment (tools/iter8_probe.cu): -DK8_TIMELINE logs clock64 events of CTA 0 into p.dbg,
// [role][tile][event]; the production build compiles the hook away.
// -DK8_OFF=bits switches parts off for timing: 1 MMA2, 2 MMA1, 4 C loads, 8 flat-kernel ALU,
// 16 weight stores, 32 pixel TMA loads
#ifdef K8_OFF
#define K8_SKIP(bit) (K8_OFF & (bit))
#else
#define K8_SKIP(bit) (0)
#endif
#ifdef K8_TIMELINE
#define K8_TL(role, tile, ev)                                                                  \
  do {                                                                                         \
    if (blockIdx.x == 0 && lane == 0 && (tile) < 512)                                          \
      p.dbg[((size_t)(role) * 512 + (tile)) * 8 + (ev)] = clock64();                           \
  } while (0)
#else
#define K8_TL(role, tile, ev) \
  do {                        \
  } while (0)
#endif

// Epilogue -> issuer hand-offs are named barriers (bar.arrive by the group's warps, bar.sync by the MMA
// warp; ~30 cycles against ~180 for an mbarrier arrive -> wait, tools/sync_probe.cu): one per C buffer
// (ids 1..NC) and one per weight buffer (ids NC + 1..NC + NP).  No arrival can run a phase ahead: a
// group's next arrival on a buffer's barrier needs an MMA that the waiting warp issues only after its
// sync (C: the buffer's next similarity; P: the weighted sum that frees the buffer).
// (r2: 798 -> 762 cycles per tile at 2 seed tiles per frame, 790 -> 709 at 1; tools/k9_variants.sh)
#define K8_RELEASE_C(cb) nbar_arrive(1 + (int)(cb), (kGroupWarps + 1) * 32)

// GUARD (option "guard_stats", fms_run_stats.guard_pairs): also count the iteration pairs whose
// similarity lies within the certified error bound of tau (kGuardEps), i.e. the window decisions the
// 3-term fp32 similarity cannot certify against the exact one.  A separate instantiation: the
// production kernel carries no extra instruction.
template <int DP, bool GUARD = false>
__global__ void __launch_bounds__(k8::kThreads, 1) iter8_kernel(const __grid_constant__ TMaps tm, Params p) {
  using namespace k8;
  using Cfg = Iter8Cfg<DP>;
  constexpr int kGroups = Cfg::GROUPS, kGroupWarps = Cfg::GROUP_WARPS;
  constexpr int kColsPerWarp = Cfg::COLS_PER_WARP, kParts = Cfg::PARTS, kPart = Cfg::PART;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                    // [2 buffers][s_hi, s_hs, s_lo][A_B]
  uint8_t* sX = smem + 6 * Cfg::A_B;                     // [LSTAGES][hi, lo]
  uint8_t* sQ = sX + Cfg::LSTAGES * Cfg::L_B;            // [QSTAGES][digit planes]
  long long* gsm = reinterpret_cast<long long*>(sQ + Cfg::QSTAGES * Cfg::Q_B);  // [group][DP][kBM]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(gsm) + kGroups * Cfg::GS_B);
  uint64_t* x_full = bars;                    // [LSTAGES] limbs of a pixel tile landed
  uint64_t* x_empty = x_full + Cfg::LSTAGES;  // [LSTAGES] the tile's similarity MMAs done
  uint64_t* q_full = x_empty + Cfg::LSTAGES;  // [QSTAGES] digit planes landed
  uint64_t* q_empty = q_full + Cfg::QSTAGES;  // [QSTAGES] the tile's weighted sum done: stage and P free
  uint64_t* a_full = q_empty + Cfg::QSTAGES;  // [2] seed tile landed
  uint64_t* a_empty = a_full + 2;             // [2] seed tile consumed
  // similarity ready: one barrier per epilogue GROUP (not per C buffer), so that a group never waits
  // on a barrier whose previous phase is still pending (a waiter two phases ahead would see the
  // pending phase's parity as complete)
  // c_full: per group with 4 groups (safe because MMA1 issues in order and NC < 4: the group's next
  // phase needs the group's previous tile consumed), per C buffer with 1 group (every warp consumes
  // every tile, so a buffer's next phase needs every waiter's release)
  // (2 groups: per C buffer as well -- a buffer's next phase needs its previous tile's group to have
  // released it, hence to have waited)
  constexpr int kCF = kGroups != 4 ? Cfg::NC : kGroups;
  uint64_t* c_full = a_empty + 2;             // [kCF]
  // an item's Gq complete: per group -- the group owning the item's last tile drains it, and each
  // group's drains are sequential in its own program order
  uint64_t* g_full = c_full + kCF;           // [kGroups]
  uint64_t* g_empty = g_full + kGroups;       // [1] Gq drained
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(g_empty + 1);
  static_assert(1 + Cfg::NC + Cfg::NP <= 16, "named barrier ids");
  static_assert((Cfg::LSTAGES * 2 + Cfg::QSTAGES * 2 + 5 + kCF + kGroups) * 8 + 4 <= 1024,
                "barrier area");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < Cfg::LSTAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < Cfg::QSTAGES; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < kGroups; ++i) mbar_init(&g_full[i], 1);
    mbar_init(g_empty, 4);  // drained by 4 warps (one per lane quarter)
    for (int i = 0; i < kCF; ++i) mbar_init(&c_full[i], 1);
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == kWarpTma && lane == 0) {
    tma_prefetch(&tm.xh); tma_prefetch(&tm.xl);
    tma_prefetch(&tm.sh); tma_prefetch(&tm.ss); tma_prefetch(&tm.sl);
  }
  if (warp == kWarpTmaQ && lane == 0) tma_prefetch(&tm.xq);
  if (warp == kWarpMma1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // everything above (barriers, descriptor prefetch, TMEM) overlaps the predecessor under PDL; the
  // work list below is its output
  pdl_wait();
  const int n_items = p.counters[0];
  const int ct = p.counters[12];   // pixel tiles per work item
  const int nch = p.counters[13];  // work items per seed tile
  const int i_begin = (int)(((long long)n_items * blockIdx.x) / gridDim.x);
  const int i_end = (int)(((long long)n_items * (blockIdx.x + 1)) / gridDim.x);
  if (i_begin >= i_end) {
    // no work: nothing to do but release TMEM below
  } else if (warp == kWarpTma) {
    // ================================ TMA producer ================================
    int xi = 0;
    int stage = 0;
    uint32_t sphase = 0;
    int it = 0;
    for (int item = i_begin; item < i_end; ++item, ++it) {
      const Item8 w = item8(p, item, nch);
      const int ab = it & 1;
      const int cbeg = w.chunk * ct;
      const int ccnt = min(ct, p.n_ptiles - cbeg);
      mbar_wait(&a_empty[ab], ((it >> 1) & 1) ^ 1);
      if (lane == 0) {
        const int srow = w.f * p.S_pad + w.tile * kBM;
        mbar_expect_tx(&a_full[ab], 3 * Cfg::A_B);
        tma_load_2d(sA + (3 * ab + 0) * Cfg::A_B, &tm.sh, &a_full[ab], 0, srow);
        tma_load_2d(sA + (3 * ab + 1) * Cfg::A_B, &tm.ss, &a_full[ab], 0, srow);
        tma_load_2d(sA + (3 * ab + 2) * Cfg::A_B, &tm.sl, &a_full[ab], 0, srow);
      }
      __syncwarp();
      const long long tile0 = (long long)w.f * p.n_ptiles + cbeg;
      for (int j = 0; j < ccnt; ++j) {
        mbar_wait(&x_empty[stage], sphase ^ 1);
        K8_TL(0, xi, 0);
        if (lane == 0) {
          uint8_t* st = sX + stage * Cfg::L_B;
          const int xrow = (int)((tile0 + j) * kBN);
          if (K8_SKIP(32)) {
            mbar_arrive(&x_full[stage]);
          } else {
            mbar_expect_tx(&x_full[stage], Cfg::L_B);
#ifdef K8_BULK_LIMBS  // timing experiment: contiguous 1-D copies (wrong smem layout for the MMA)
            bulk_load(st, p.Xh + (size_t)xrow * DP, Cfg::TILE_B, &x_full[stage]);
            bulk_load(st + Cfg::TILE_B, p.Xl + (size_t)xrow * DP, Cfg::TILE_B, &x_full[stage]);
#else
            tma_load_2d(st, &tm.xh, &x_full[stage], 0, xrow);
            tma_load_2d(st + Cfg::TILE_B, &tm.xl, &x_full[stage], 0, xrow);
#endif
          }
        }
        __syncwarp();
        ++xi;
        if (++stage == Cfg::LSTAGES) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp == kWarpTmaQ) {
    // ====================== TMA producer of the digit planes ======================
    int stage = 0;
    uint32_t sphase = 0;
    for (int item = i_begin; item < i_end; ++item) {
      const Item8 w = item8(p, item, nch);
      const int cbeg = w.chunk * ct;
      const int ccnt = min(ct, p.n_ptiles - cbeg);
      const long long tile0 = (long long)w.f * p.n_ptiles + cbeg;
      for (int j = 0; j < ccnt; ++j) {
        mbar_wait(&q_empty[stage], sphase ^ 1);
        if (lane == 0) {
          if (K8_SKIP(32)) {
            mbar_arrive(&q_full[stage]);
          } else {
            mbar_expect_tx(&q_full[stage], Cfg::Q_B);
#ifdef K8_BULK_DIGITS  // timing experiment: contiguous 1-D copy (wrong smem layout for the MMA)
            bulk_load(sQ + stage * Cfg::Q_B, p.Xq + (size_t)(tile0 + j) * Cfg::Q_B, Cfg::Q_B, &q_full[stage]);
#else
            tma_load_2d(sQ + stage * Cfg::Q_B, &tm.xq, &q_full[stage], 0, (int)((tile0 + j) * Cfg::NQ));
#endif
          }
        }
        __syncwarp();
        if (++stage == Cfg::QSTAGES) { stage = 0; sphase ^= 1; }
      }
    }
  } else if (warp == kWarpMma1) {
    // ============================ MMA1 issuer: similarity ============================
    constexpr uint32_t IDESC1 = idesc_f16(kBM, kBN, 0, 0);  // both operands K-major
    const uint64_t dx0 = umma_desc(smem_u32(sX), 16, Cfg::SBO, Cfg::LAYOUT);
    int stage = 0;
    uint32_t sphase = 0;
    int i = 0;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const Item8 w = item8(p, item, nch);
      const int ccnt = min(ct, p.n_ptiles - w.chunk * ct);
      const int ab = it & 1;
      mbar_wait(&a_full[ab], (it >> 1) & 1);
      tc_fence_after();
      const uint64_t dah = umma_desc(smem_u32(sA + (3 * ab + 0) * Cfg::A_B), 16, Cfg::SBO, Cfg::LAYOUT);
      const uint64_t das = dah + (Cfg::A_B >> 4);
      const uint64_t dal = dah + (2 * Cfg::A_B >> 4);
      for (int j = 0; j < ccnt; ++j, ++i) {
        const uint32_t buf = i % Cfg::NC;
        K8_TL(1, i, 0);
        if (i >= Cfg::NC) nbar_sync(1 + buf, (kGroupWarps + 1) * 32);  // C[buf] loaded by its group
        K8_TL(1, i, 1);
        mbar_wait(&x_full[stage], sphase);
        K8_TL(1, i, 2);
        tc_fence_after();
        const uint64_t dxh = dx0 + (uint64_t)(stage * (Cfg::L_B >> 4));
        const uint64_t dxl = dxh + (Cfg::TILE_B >> 4);
        const uint32_t d = tmem + buf * kBN;
        if (!K8_SKIP(2)) {
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // s_hi . hi
            mma_ss_f16_el(d, dah + kk * 2, dxh + kk * 2, IDESC1, kk > 0);
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // + (s_hi 2^-11) . lo
            mma_ss_f16_el(d, das + kk * 2, dxl + kk * 2, IDESC1, 1u);
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)  // + s_lo . hi
            mma_ss_f16_el(d, dal + kk * 2, dxh + kk * 2, IDESC1, 1u);
        }
        tc_commit_el(&c_full[kGroups != 4 ? buf : i % kGroups]);
        tc_commit_el(&x_empty[stage]);  // the limbs stage is free once these MMAs complete
        K8_TL(1, i, 3);
        if (++stage == Cfg::LSTAGES) { stage = 0; sphase ^= 1; }
      }
      tc_commit_el(&a_empty[ab]);  // seed tile free once this item's MMA1s complete
    }
  } else if (warp == kWarpMma2) {
    // ==================== MMA2 issuer: exact int8 weighted sum ====================
    // Gq (+)= P[i % NP] . Q once the epilogue group has written the weights (named barrier); one commit frees
    // the pixel stage and with it the weight buffer (x_empty); at the end of an item hands Gq over.
    constexpr uint32_t IDESC2 = idesc_i8(kBM, Cfg::NQ);
    const uint64_t dq0 = umma_desc(smem_u32(sQ), 16, 1024, 2);  // K-major SW128
    int stage = 0;
    uint32_t sphase = 0;
    int i = 0;
    const uint32_t g_tmem = tmem + Cfg::G_COL;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const Item8 w = item8(p, item, nch);
      const int ccnt = min(ct, p.n_ptiles - w.chunk * ct);
      mbar_wait(g_empty, (it & 1) ^ 1);
      tc_fence_after();
      for (int j = 0; j < ccnt; ++j, ++i) {
        const uint32_t pb = i % Cfg::NP;
        K8_TL(2, i, 0);
        nbar_sync(1 + Cfg::NC + pb, (kGroupWarps + 1) * 32);  // P[pb] stored by its group
        mbar_wait(&q_full[stage], sphase);
        K8_TL(2, i, 1);
        tc_fence_after();
        if (w.mode == 0 && !K8_SKIP(1)) {
          const uint64_t bq = dq0 + (uint64_t)(stage * (Cfg::Q_B >> 4));
          const uint32_t pa = tmem + Cfg::P_COL + pb * (kBN / 4);
#pragma unroll
          for (int k = 0; k < kBN / 32; ++k)  // 32 pixels = 8 columns of packed u8 weights
            mma_ts_i8_el(g_tmem, pa + k * 8, bq + (uint64_t)(k * 2), IDESC2, (j == 0 && k == 0) ? 0u : 1u);
        }
        tc_commit_el(&q_empty[stage]);  // digit stage and weight buffer pb free once these complete
        K8_TL(2, i, 2);
        if (++stage == Cfg::QSTAGES) { stage = 0; sphase ^= 1; }
      }
      tc_commit_el(&g_full[(i - 1) % kGroups]);  // the group that handled the item's last tile drains
    }
  } else {
    // ================================ epilogue (warps 0..15) ================================
    // kGroups groups of kGroupWarps warps take tiles round-robin; a warp reads lane quarter q and
    // kColsPerWarp columns of C in halves of 64 (one tcgen05.ld each).
    const int q = warp & 3;                           // TMEM lane quarter this warp may access
    const int h = (warp >> 2) % (kGroupWarps / 4);    // column part within the group
    const int grp = warp / kGroupWarps;
    const int row = q * 32 + lane;                    // seed row within the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    // tau_m = the float just below 2^11 tau (C is scaled by 2^11, exactly)
    const float tau_m = __uint_as_float(__float_as_uint(p.tau_f * kLimb) - 1u);
    unsigned long long gpairs = 0;  // GUARD: pairs within kGuardEps of tau (scaled by 2^11 like C)
    (void)gpairs;
    uint32_t tcur = 0;                                // running tile index over the CTA's stream
    uint32_t mine = 0;                                // tiles handled by this group so far
    long long* gs = gsm + (size_t)grp * (DP * kBM) + row;  // this group's segment sums of this row, [k][kBM]
    int seg = -1;                                     // segment (frame, seed tile) held in gs
    int seg_f = 0, seg_tile = 0;
    uint32_t drains = 0;                              // items this group has drained
    if (h == 0 && !Cfg::DIRECT) {
#pragma unroll
      for (int k = 0; k < DP; ++k) gs[k * kBM] = 0;
    }
    auto flush = [&]() {
      if (Cfg::DIRECT || seg < 0) return;
      double* dst = p.gacc + ((size_t)seg_f * p.S_pad + (size_t)seg_tile * kBM + row) * DP;
#pragma unroll
      for (int k = 0; k < DP; ++k) {
        if (gs[k * kBM] != 0) atomicAdd(dst + k, (double)gs[k * kBM]);  // exact integers (< 2^53)
        gs[k * kBM] = 0;
      }
      seg = -1;
    };
    int cnt = 0;
    for (int item = i_begin, it = 0; item < i_end; ++item, ++it) {
      const Item8 w = item8(p, item, nch);
      const int ccnt = min(ct, p.n_ptiles - w.chunk * ct);
      // the tile range of this item in the CTA's stream: [ctile, ctile + ccnt); this group's tiles
      // are those with index % kGroups == grp; the group owning the item's last tile drains its Gq
      const uint32_t base = tcur;
      const uint32_t last_tile = base + (uint32_t)ccnt - 1;
      const uint32_t first = base + (uint32_t)((grp - (int)(base % kGroups) + kGroups) % kGroups);
      for (uint32_t ctile = first; ctile <= last_tile; ctile += kGroups) {  // this group's tiles only
        const uint32_t cb = ctile % Cfg::NC;
        const uint32_t pb = ctile % Cfg::NP;
        const int role = 3 + (grp * kGroupWarps + (warp % kGroupWarps)) % 16;
        (void)role;
        K8_TL(role, ctile, 0);
        if (kGroups != 4) mbar_wait(&c_full[cb], (ctile / Cfg::NC) & 1);
        else mbar_wait(&c_full[grp], mine & 1);
        ++mine;
        K8_TL(role, ctile, 1);
        tc_fence_after();
        // P[pb] is free once the weighted sum of the tile that used it last has completed
        // (count-pass tiles too: without it a group could arrive on P[pb]'s named barrier a phase ahead)
        const uint32_t u = ctile - Cfg::NP;
        const bool need_free = ctile >= (uint32_t)Cfg::NP;
        bool p_free = !need_free;
        // a lane quarter without active seeds (the tail of a frame's last seed tile) skips its C loads,
        // flat kernel and weight stores; its rows of Gq are never drained (stale weights only reach them)
        const bool quarter_active = q * 32 < w.rows;
        if (!quarter_active) {
          tc_fence_before();
          __syncwarp();
          K8_RELEASE_C(cb);
          if (!p_free) mbar_wait(&q_empty[u % Cfg::QSTAGES], (u / Cfg::QSTAGES) & 1);
        }
#pragma unroll
        for (int part = 0; part < kParts && quarter_active; ++part) {
          const uint32_t col = (uint32_t)(h * kColsPerWarp + part * kPart);
          uint32_t v[kPart];
          if (!K8_SKIP(4)) {
            tmem_ld_n<kPart>(tmem + lane_base + cb * kBN + col, v);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < kPart; ++i) v[i] = __float_as_uint(tau_m) + (uint32_t)(i * lane);
          }
          if (part == kParts - 1) {
            K8_TL(role, ctile, 2);
            tc_fence_before();
            __syncwarp();
            K8_RELEASE_C(cb);  // MMA1 may overwrite C[cb]
          }
          if (!p_free) p_free = mbar_test(&q_empty[u % Cfg::QSTAGES], (u / Cfg::QSTAGES) & 1);
          uint32_t pk[kPart / 4];
          if (!K8_SKIP(8)) {
#pragma unroll
            for (int i = 0; i < kPart / 4; ++i) {
              uint32_t d0, d1, d2, d3;
              sub_tau2(v[4 * i], v[4 * i + 1], tau_m, d0, d1);
              sub_tau2(v[4 * i + 2], v[4 * i + 3], tau_m, d2, d3);
              pk[i] = pack_w4(d0, d1, d2, d3);
              if constexpr (GUARD) {
                if (w.mode == 0 && row < w.rows) {
                  const long long px0 = (long long)(w.chunk * ct + (ctile - base)) * kBN + col + 4 * i;
                  const float e = kGuardEps * kLimb;
                  gpairs += (px0 + 0 < p.n && fabsf(__uint_as_float(d0)) < e) + (px0 + 1 < p.n && fabsf(__uint_as_float(d1)) < e) +
                            (px0 + 2 < p.n && fabsf(__uint_as_float(d2)) < e) + (px0 + 3 < p.n && fabsf(__uint_as_float(d3)) < e);
                }
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < kPart / 4; ++i) pk[i] = v[4 * i] ^ v[4 * i + 3];
          }
          K8_TL(role, ctile, 3);
          if (!p_free) {
            mbar_wait(&q_empty[u % Cfg::QSTAGES], (u / Cfg::QSTAGES) & 1);
            p_free = true;
          }
          K8_TL(role, ctile, 4);
          if (w.mode == 0) {
            tc_fence_after();
            if (!K8_SKIP(16)) {
              tmem_st_n<kPart / 4>(tmem + lane_base + Cfg::P_COL + pb * (kBN / 4) + col / 4, pk);
            } else {
#pragma unroll
              for (int i = 0; i < kPart / 4; ++i) cnt += pk[i] & 1u;  // keeps the ALU work alive
            }
          } else {
#pragma unroll
            for (int i = 0; i < kPart / 4; ++i) cnt += __popc(pk[i]);  // 8 bits per member
          }
        }
        if (w.mode == 0 && !K8_SKIP(16)) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        nbar_arrive(1 + Cfg::NC + pb, (kGroupWarps + 1) * 32);  // MMA2 may consume P[pb]
        K8_TL(role, ctile, 5);
        if (ctile == last_tile && h == 0) {
          // ---- drain the item's Gq (this group handled its last tile) into its segment sums ----
          mbar_wait(&g_full[grp], drains & 1);
          ++drains;
          K8_TL(role, ctile, 6);
          tc_fence_after();
          if (w.mode == 0 && quarter_active) {
            if (!Cfg::DIRECT && seg != w.key) {
              flush();
              seg = w.key;
              seg_f = w.f;
              seg_tile = w.tile;
            }
            const uint32_t gq = tmem + lane_base + Cfg::G_COL;
#pragma unroll
            for (int k0 = 0; k0 < DP; k0 += 16) {
              uint32_t ga[16], gb[16], gc[16];
              tmem_ld16(gq + k0, ga);
              tmem_ld16(gq + DP + k0, gb);
              tmem_ld16(gq + 2 * DP + k0, gc);
              tmem_ld_wait();
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const long long s = (long long)(int)ga[k] * 65536ll + (long long)(int)gb[k] * 256ll + (int)gc[k];
                // s = 255 x (an integer below 2^43): the correctly rounded product is within 1e-3 of it
                const long long v = __double2ll_rn((double)s * (1.0 / 255.0));
                if constexpr (Cfg::DIRECT) {
                  if (v != 0)
                    atomicAdd(p.gacc + ((size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row) * DP + k0 + k, (double)v);
                } else {
                  gs[(k0 + k) * kBM] += v;
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(g_empty);
          K8_TL(role, ctile, 7);
        }
      }
      tcur = base + (uint32_t)ccnt;
      // count pass: each warp flushes its window counts when the segment (same seed tile) ends
      const bool last = (item + 1 == i_end) || item8(p, item + 1, nch).key != w.key;
      if (last && w.mode != 0) {
        if (cnt) atomicAdd(p.cacc + (size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row, cnt >> 3);
        cnt = 0;
      }
    }
    if (h == 0) flush();
    if constexpr (GUARD) {
      for (int o = 16; o > 0; o >>= 1) gpairs += __shfl_xor_sync(0xffffffffu, gpairs, o);
      if (lane == 0 && gpairs) atomicAdd(reinterpret_cast<unsigned long long*>(p.counters + kGuardCounter), gpairs);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpMma1) tmem_dealloc(tmem, 512);
}

int iter8_smem_bytes(int DP) { return DP == 16 ? Iter8Cfg<16>::SMEM : Iter8Cfg<32>::SMEM; }

cudaError_t launch_iter8(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st) {
  if (p.guard) {
    if (DP == 16) return launch_ex(p.pdl, iter8_kernel<16, true>, grid, k8::kThreads, Iter8Cfg<16>::SMEM, st, tm, p);
    return launch_ex(p.pdl, iter8_kernel<32, true>, grid, k8::kThreads, Iter8Cfg<32>::SMEM, st, tm, p);
  }
  if (DP == 16) return launch_ex(p.pdl, iter8_kernel<16>, grid, k8::kThreads, Iter8Cfg<16>::SMEM, st, tm, p);
  return launch_ex(p.pdl, iter8_kernel<32>, grid, k8::kThreads, Iter8Cfg<32>::SMEM, st, tm, p);
}

cudaError_t setup_iter8_attrs() {
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e = cudaFuncSetAttribute(iter8_kernel<16>, a, Iter8Cfg<16>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(iter8_kernel<32>, a, Iter8Cfg<32>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(iter8_kernel<16, true>, a, Iter8Cfg<16>::SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(iter8_kernel<32, true>, a, Iter8Cfg<32>::SMEM);
  return e;
}

}  // namespace fms
