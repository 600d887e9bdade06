// k_iter9.cu -- EXPERIMENT (not built into libfms.so; timed by tools/k9_variants.sh).  Result: exact (window
// sums identical to k_iter8.cu) but not faster: 753-830 cycles per tile against iter8's 709-762 with its
// named-barrier hand-offs.
//
// K2 for the flat kernel, 16-lane rows (the C2 path): the lockstep mean-shift iteration
// of Alg. 2 lines 4-9, evaluated densely as P:210 prescribes,
//
//     C = S_hat . X_hat^T              seeds x pixels cosine similarity   (Eq. 1/9)
//     W = [C >= tau], tau = 1 - h      flat kernel, inclusive              (Eq. 11; R5)
//     G = W . X_hat                    windowed sum (count cancels, R4)    (Eq. 8 / R1)
//
// with the same arithmetic as k_iter8.cu (3 kind::f16 MMAs over fixed-point fp16 limbs for C, the
// FADD2 + I2IP flat kernel, an exact kind::i8 weighted sum over int8 digit planes), restructured so
// that no tile waits on a cross-warp mbarrier hand-off except the tensor pipe's own commits.
//
// k_iter8.cu runs one MMA1 warp, one MMA2 warp and four epilogue groups through shared rings of C
// and weight buffers; every buffer passes through two ~200-350-cycle mbarrier hand-offs and the
// per-tile period (~750 cycles) was set by those chains, not by a unit.  Here:
//   * two GROUPS, each a self-contained pipeline: 8 epilogue warps (lane quarter q, column half h),
//     one ISSUER warp (both MMAs of the group) and one PRODUCER warp (TMA).  Group g takes every
//     other work item of the CTA's range (items i_begin + g, + 2, ...), so the groups share nothing
//     but the tensor pipe: own seed-tile buffers, pixel rings, C / P / Gq columns and segment sums.
//   * epilogue -> issuer hand-offs are named barriers (bar.arrive by the 8 epilogue warps, bar.sync
//     by the issuer; ~30 cycles): "C loaded" lets the issuer put the next tile's similarity into
//     the group's single C buffer at once, "P stored" lets it issue the weighted sum.
//   * the C buffer is released as soon as the loads land (the flat kernel and the weight stores run
//     while the next similarity is computed); the weight buffer is free when the group's previous
//     weighted sum has completed (one commit, long done by then).
// Pairs with the other group: while one group loads / converts / stores, the pipe runs the other
// group's MMAs.
//
// TMEM (512 columns): C_g = [128 g, 128 g + 128), P_g = 256 + 32 g (u8 weights, 32 columns), Gq_g =
// 320 + 48 g (3 DP = 48 int32 columns).  16-lane rows only (DP = 16); 32-lane rows stay on k_iter8.
#include "fms_device.cuh"  // built with -Ipaper_2007_14283_b200/csrc (tools/k9_variants.sh)

namespace fms {

namespace k9 {
constexpr int kGroups = 2;
constexpr int kGroupWarps = 8;                      // epilogue warps per group
constexpr int kEpiWarps = kGroups * kGroupWarps;    // warps 0..15
constexpr int kWarpIss = kEpiWarps;                 // warps 16, 17: issuer of group 0, 1
constexpr int kWarpTma = kEpiWarps + kGroups;       // warps 18, 19: producer of group 0, 1
constexpr int kThreads = (kEpiWarps + 2 * kGroups) * 32;
constexpr int kBarThreads = (kGroupWarps + 1) * 32;  // a group's epilogue warps + its issuer
constexpr int DP = 16;
constexpr int ROW_B = DP * 2;                  // bytes per fp16 row
constexpr int TILE_B = kBN * ROW_B;            // one pixel tile (one limb)
constexpr int A_B = kBM * ROW_B;               // one seed tile (one split)
constexpr uint32_t LAYOUT = 6u;                // SWIZZLE_32B (32-byte fp16 rows)
constexpr uint32_t SBO = 8 * ROW_B;            // 8-row core-matrix group stride
constexpr int NQ = 3 * DP;                     // digit planes (= Gq columns)
constexpr int Q_B = NQ * kBN;                  // digit planes of one tile (128 B rows, SW128)
constexpr int L_B = 2 * TILE_B;                // one stage of the limb ring (hi, lo)
#ifdef K9_LSTAGES
constexpr int LSTAGES = K9_LSTAGES;
#else
constexpr int LSTAGES = 4;
#endif
#ifdef K9_QSTAGES
constexpr int QSTAGES = K9_QSTAGES;
#else
constexpr int QSTAGES = 5;
#endif
constexpr int GS_B = kBM * DP * 8;             // int64 segment sums, [DP][kBM]
constexpr int P_COL = kGroups * kBN;           // 256
constexpr int G_COL = P_COL + kGroups * (kBN / 4);  // 320
static_assert(G_COL + kGroups * NQ <= 512, "TMEM budget");
// per group: 2 seed-tile buffers x 3 splits, the limb and digit rings, segment sums
constexpr int GRP_B = 6 * A_B + LSTAGES * L_B + QSTAGES * Q_B + GS_B;
constexpr int NBAR = 2 * LSTAGES + 2 * QSTAGES + 4 + 3;  // per group
constexpr int SMEM = 1024 + kGroups * GRP_B + 1024;
static_assert(SMEM <= 232448, "shared memory");
static_assert(GRP_B % 1024 == 0 && L_B % 1024 == 0 && Q_B % 1024 == 0 && (6 * A_B) % 1024 == 0, "alignment");
static_assert(kGroups * NBAR * 8 + 16 <= 1024, "barrier area");
}  // namespace k9

struct Item9 {
  int f, tile, chunk, mode, key;  // key: frame * S_pad + tile * kBM (the segment a G drain belongs to)
  int rows;                       // active seed rows in the tile
};
// same work-item order as k_iter8.cu (frame by frame, chunk by chunk, a chunk's seed tiles back to back)
__device__ __forceinline__ Item9 item9(const Params& p, int item, int nch) {
  const int f = p.tiles[item / nch].f;
  const FrameCtl& c = p.ctl[f];
  const int T = c.n_tiles_step;
  const int L = item - nch * c.tile_off;
  const int chunk = L / T;
  const TileTask tt = p.tiles[c.tile_off + (L - chunk * T)];
  return Item9{f, tt.tile, chunk, tt.mode, f * p.S_pad + tt.tile * kBM, min(kBM, c.n_active - tt.tile * kBM)};
}


// two in-window differences per instruction: {c0 - tau_m, c1 - tau_m}
__device__ __forceinline__ void sub_tau2_9(uint32_t c0, uint32_t c1, float tau_m, uint32_t& d0, uint32_t& d1) {
  asm("{\n\t.reg .b64 ra, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rc, {%4, %4};\n\t"
      "add.rn.f32x2 rd, ra, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=r"(d0), "=r"(d1)
      : "r"(c0), "r"(c1), "f"(-tau_m));
}
// four pixels' weights, byte i = 255 if difference i > 0 else 0 (see k_iter8.cu for the exactness argument)
__device__ __forceinline__ uint32_t pack_w4_9(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3) {
  uint32_t t, w;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(t) : "r"(d3), "r"(d2));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(d1), "r"(d0), "r"(t));
  return w;
}

// Timing experiment: -DK9_TIMELINE logs clock64 events of CTA 0 into p.dbg, [role][k][event], role 0/1
// = issuer of group 0/1, 2 + 8 g + w = epilogue warp w of group g; k = the group's tile ordinal.
// -DK9_OFF=bits switches parts off for timing: 1 MMA2, 2 MMA1, 4 C loads, 8 weight stores, 16 TMA loads
#ifdef K9_OFF
#define K9_SKIP(bit) (K9_OFF & (bit))
#else
#define K9_SKIP(bit) (0)
#endif
#ifdef K9_TIMELINE
#define K9_TL(role, k, ev)                                                                     \
  do {                                                                                         \
    if (blockIdx.x == 0 && lane == 0 && (k) < 512)                                             \
      p.dbg[((size_t)(role) * 512 + (k)) * 8 + (ev)] = clock64();                              \
  } while (0)
#else
#define K9_TL(role, k, ev) \
  do {                     \
  } while (0)
#endif

__global__ void __launch_bounds__(k9::kThreads, 1) iter9_kernel(const __grid_constant__ TMaps tm, Params p) {
  using namespace k9;
  const int n_items = p.counters[0];
  const int ct = p.counters[12];   // pixel tiles per work item
  const int nch = p.counters[13];  // work items per seed tile
  const int i_begin = (int)(((long long)n_items * blockIdx.x) / gridDim.x);
  const int i_end = (int)(((long long)n_items * (blockIdx.x + 1)) / gridDim.x);
  if (i_begin >= i_end) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // this warp's group
  const int g = warp < kEpiWarps ? warp / kGroupWarps : (warp < kWarpTma ? warp - kWarpIss : warp - kWarpTma);
  uint8_t* gb = smem + g * GRP_B;
  uint8_t* sA = gb;                                   // [2 buffers][s_hi, s_hs, s_lo][A_B]
  uint8_t* sX = gb + 6 * A_B;                         // [LSTAGES][hi, lo]
  uint8_t* sQ = sX + LSTAGES * L_B;                   // [QSTAGES][digit planes]
  long long* gsm = reinterpret_cast<long long*>(sQ + QSTAGES * Q_B);  // [DP][kBM]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kGroups * GRP_B) + g * NBAR;
  uint64_t* x_full = bars;                    // [LSTAGES] limbs of a pixel tile landed
  uint64_t* x_empty = x_full + LSTAGES;       // [LSTAGES] the tile's similarity MMAs done
  uint64_t* q_full = x_empty + LSTAGES;       // [QSTAGES] digit planes landed
  uint64_t* q_empty = q_full + QSTAGES;       // [QSTAGES] the tile's weighted sum done
  uint64_t* a_full = q_empty + QSTAGES;       // [2] seed tile landed
  uint64_t* a_empty = a_full + 2;             // [2] the item's similarity MMAs done
  uint64_t* c_full = a_empty + 2;             // similarity of the group's current tile in C_g
  uint64_t* p_free = c_full + 1;              // the group's previous weighted sum done (P_g free)
  uint64_t* g_full = p_free + 1;              // the item's Gq_g complete
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(smem + kGroups * GRP_B) +
                                                      kGroups * NBAR);
  const int bar_c = 1 + 2 * g;  // named barrier: C_g loaded by the group's epilogue warps
  const int bar_p = 2 + 2 * g;  // named barrier: P_g stored

  if (warp == kWarpTma + g && lane == 0) {  // each producer initialises its group's barriers
    for (int i = 0; i < LSTAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < QSTAGES; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    mbar_init(c_full, 1);
    mbar_init(p_free, 1);
    mbar_init(g_full, 1);
    fence_barrier_init();
    fence_proxy_async();
    if (g == 0) {
      tma_prefetch(&tm.xh); tma_prefetch(&tm.xl); tma_prefetch(&tm.xq);
      tma_prefetch(&tm.sh); tma_prefetch(&tm.ss); tma_prefetch(&tm.sl);
    }
  }
  if (warp == kWarpIss) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // the group's items: i_begin + g, i_begin + g + 2, ...
  const int first_item = i_begin + g;
  auto tiles_of = [&](const Item9& w) { return min(ct, p.n_ptiles - w.chunk * ct); };

  if (warp >= kWarpTma) {
    // ================================ TMA producer (group g) ================================
    int xs = 0, qs = 0;
    uint32_t xph = 0, qph = 0;
    int it = 0;
    for (int item = first_item; item < i_end; item += kGroups, ++it) {
      const Item9 w = item9(p, item, nch);
      const int ab = it & 1;
      const int cbeg = w.chunk * ct;
      const int ccnt = tiles_of(w);
      mbar_wait(&a_empty[ab], ((it >> 1) & 1) ^ 1);
      if (lane == 0) {
        const int srow = w.f * p.S_pad + w.tile * kBM;
        mbar_expect_tx(&a_full[ab], 3 * A_B);
        tma_load_2d(sA + (3 * ab + 0) * A_B, &tm.sh, &a_full[ab], 0, srow);
        tma_load_2d(sA + (3 * ab + 1) * A_B, &tm.ss, &a_full[ab], 0, srow);
        tma_load_2d(sA + (3 * ab + 2) * A_B, &tm.sl, &a_full[ab], 0, srow);
      }
      __syncwarp();
      const long long tile0 = (long long)w.f * p.n_ptiles + cbeg;
      for (int j = 0; j < ccnt; ++j) {
        mbar_wait(&x_empty[xs], xph ^ 1);
        if (lane == 0) {
          uint8_t* st = sX + xs * L_B;
          const int xrow = (int)((tile0 + j) * kBN);
          if (K9_SKIP(16)) {
            mbar_arrive(&x_full[xs]);
          } else {
            mbar_expect_tx(&x_full[xs], L_B);
            tma_load_2d(st, &tm.xh, &x_full[xs], 0, xrow);
            tma_load_2d(st + TILE_B, &tm.xl, &x_full[xs], 0, xrow);
          }
        }
        __syncwarp();
        if (++xs == LSTAGES) { xs = 0; xph ^= 1; }
        mbar_wait(&q_empty[qs], qph ^ 1);
        if (lane == 0) {
          if (K9_SKIP(16)) {
            mbar_arrive(&q_full[qs]);
          } else {
            mbar_expect_tx(&q_full[qs], Q_B);
            tma_load_2d(sQ + qs * Q_B, &tm.xq, &q_full[qs], 0, (int)((tile0 + j) * NQ));
          }
        }
        __syncwarp();
        if (++qs == QSTAGES) { qs = 0; qph ^= 1; }
      }
    }
  } else if (warp >= kWarpIss) {
    // ================================ issuer (group g) ================================
    // MMA1 of the group's tile k + 1 goes into C_g as soon as the epilogue has loaded tile k; MMA2 of
    // tile k once its weights are stored.
    constexpr uint32_t IDESC1 = idesc_f16(kBM, kBN, 0, 0);
    constexpr uint32_t IDESC2 = idesc_i8(kBM, NQ);
    const uint64_t dx0 = umma_desc(smem_u32(sX), 16, SBO, LAYOUT);
    const uint64_t dq0 = umma_desc(smem_u32(sQ), 16, 1024, 2);  // K-major SW128
    const uint64_t da0 = umma_desc(smem_u32(sA), 16, SBO, LAYOUT);
    const uint32_t c_tmem = tmem + g * kBN;
    const uint32_t p_tmem = tmem + P_COL + g * (kBN / 4);
    const uint32_t g_tmem = tmem + G_COL + g * NQ;
    // lookahead cursor of MMA1: (item, its ordinal, tile j within it, its tile count)
    int la_item = first_item, la_it = 0, la_j = 0, la_cnt = 0;
    int xs = 0;
    uint32_t xph = 0;
    uint32_t k = 0;
    auto issue_mma1 = [&]() {
      // similarity of the lookahead tile into C_g
      const int ab = la_it & 1;
      K9_TL(g, k, 4);
#ifndef K9_XPRE
      mbar_wait(&x_full[xs], xph);
#endif
      K9_TL(g, k, 5);
      tc_fence_after();
      const uint64_t dah = da0 + (uint64_t)((3 * ab) * (A_B >> 4));
      const uint64_t das = dah + (A_B >> 4);
      const uint64_t dal = dah + (2 * A_B >> 4);
      const uint64_t dxh = dx0 + (uint64_t)(xs * (L_B >> 4));
      const uint64_t dxl = dxh + (TILE_B >> 4);
      if (!K9_SKIP(2)) {
        mma_ss_f16_el(c_tmem, dah, dxh, IDESC1, 0u);  // s_hi . hi
        mma_ss_f16_el(c_tmem, das, dxl, IDESC1, 1u);  // + (s_hi 2^-11) . lo
        mma_ss_f16_el(c_tmem, dal, dxh, IDESC1, 1u);  // + s_lo . hi
      }
      tc_commit_el(c_full);
      tc_commit_el(&x_empty[xs]);
      if (++xs == LSTAGES) { xs = 0; xph ^= 1; }
    };
    // enter the first item
    bool la_ok = first_item < i_end;
    if (la_ok) {
      la_cnt = tiles_of(item9(p, la_item, nch));
      mbar_wait(&a_full[0], 0);
#ifdef K9_XPRE
      mbar_wait(&x_full[xs], xph);
#endif
      issue_mma1();
    }
    int qs = 0;
    uint32_t qph = 0;
    int it = 0;
    for (int item = first_item; item < i_end; item += kGroups, ++it) {
      const Item9 w = item9(p, item, nch);
      const int ccnt = tiles_of(w);
      for (int j = 0; j < ccnt; ++j, ++k) {
#ifdef K9_XPRE
        // the next tile's pixels (if any) while the epilogue still loads C: off the critical path
        if (la_ok && !(la_j + 1 == la_cnt && la_item + kGroups >= i_end)) mbar_wait(&x_full[xs], xph);
#endif
        nbar_sync(bar_c, kBarThreads);  // C_g of tile k loaded
        K9_TL(g, k, 0);
        tc_fence_after();
        // advance the lookahead to tile k + 1
        if (++la_j == la_cnt) {
          tc_commit_el(&a_empty[la_it & 1]);  // the item's seed tile is free once its MMA1s complete
          la_item += kGroups;
          ++la_it;
          la_j = 0;
          la_ok = la_item < i_end;
          if (la_ok) {
            la_cnt = tiles_of(item9(p, la_item, nch));
            mbar_wait(&a_full[la_it & 1], (la_it >> 1) & 1);
          }
        }
        if (la_ok) issue_mma1();
        K9_TL(g, k, 1);
        nbar_sync(bar_p, kBarThreads);  // P_g of tile k stored
        K9_TL(g, k, 2);
        tc_fence_after();
        mbar_wait(&q_full[qs], qph);
        K9_TL(g, k, 6);
        tc_fence_after();
        if (w.mode == 0 && !K9_SKIP(1)) {
          const uint64_t bq = dq0 + (uint64_t)(qs * (Q_B >> 4));
#pragma unroll
          for (int kk = 0; kk < kBN / 32; ++kk)  // 32 pixels = 8 columns of packed u8 weights
            mma_ts_i8_el(g_tmem, p_tmem + kk * 8, bq + (uint64_t)(kk * 2), IDESC2, (j == 0 && kk == 0) ? 0u : 1u);
        }
        tc_commit_el(p_free);
        tc_commit_el(&q_empty[qs]);
        if (j == ccnt - 1) tc_commit_el(g_full);
        if (++qs == QSTAGES) { qs = 0; qph ^= 1; }
        K9_TL(g, k, 3);
      }
    }
  } else {
    // ================================ epilogue (group g, 8 warps) ================================
    const int wi = warp % kGroupWarps;
    const int q = wi & 3;                 // TMEM lane quarter this warp may access
    const int h = wi >> 2;                // column half: C columns 64 h .. 64 h + 63, P columns 16 h ..
    const int row = q * 32 + lane;        // seed row within the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t c_addr = tmem + lane_base + g * kBN + h * 64;
    const uint32_t p_addr = tmem + lane_base + P_COL + g * (kBN / 4) + h * 16;
    const uint32_t gq = tmem + lane_base + G_COL + g * NQ;
    const int role = 2 + g * kGroupWarps + wi;
    (void)role;
    // tau_m = the float just below 2^11 tau (C is scaled by 2^11, exactly)
    const float tau_m = __uint_as_float(__float_as_uint(p.tau_f * kLimb) - 1u);
    long long* gs = gsm + row;            // segment sums of this row, [k][kBM]
    int seg = -1, seg_f = 0, seg_tile = 0;
    if (h == 0) {
#pragma unroll
      for (int k = 0; k < DP; ++k) gs[k * kBM] = 0;
    }
    auto flush = [&]() {
      if (seg < 0) return;
      double* dst = p.gacc + ((size_t)seg_f * p.S_pad + (size_t)seg_tile * kBM + row) * DP;
#pragma unroll
      for (int k = 0; k < DP; ++k) {
        if (gs[k * kBM] != 0) atomicAdd(dst + k, (double)gs[k * kBM]);  // exact integers (< 2^53)
        gs[k * kBM] = 0;
      }
      seg = -1;
    };
    uint32_t k = 0, drains = 0;
    int cnt = 0;
    for (int item = first_item; item < i_end; item += kGroups) {
      const Item9 w = item9(p, item, nch);
      const int ccnt = tiles_of(w);
      const bool active = q * 32 < w.rows;  // lanes without active seeds skip their loads and stores
      for (int j = 0; j < ccnt; ++j, ++k) {
        K9_TL(role, k, 0);
        mbar_wait(c_full, k & 1);
        K9_TL(role, k, 1);
        tc_fence_after();
        // C in two halves of 32 columns: the second load is in flight while the first converts (64 C
        // values, 16 packed words and the loop state would not fit the 96 registers of a 640-thread CTA)
        uint32_t pk[16];
#ifdef K9_LD64
        if (active) {
          uint32_t v[64];
          tmem_ld64(c_addr, v);
          tmem_ld_wait();
          tc_fence_before();
          nbar_arrive(bar_c, kBarThreads);  // C_g may be overwritten
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            uint32_t d0, d1, d2, d3;
            sub_tau2_9(v[4 * i], v[4 * i + 1], tau_m, d0, d1);
            sub_tau2_9(v[4 * i + 2], v[4 * i + 3], tau_m, d2, d3);
            pk[i] = pack_w4_9(d0, d1, d2, d3);
          }
        } else {
          tc_fence_before();
          nbar_arrive(bar_c, kBarThreads);
        }
#else
        if (active) {
          uint32_t va[32], vb[32];
          if (!K9_SKIP(4)) {
            tmem_ld32(c_addr, va);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) va[i] = __float_as_uint(tau_m) + (uint32_t)(i * lane);
          }
          tmem_regs_ready(va);
          if (!K9_SKIP(4)) {
            tmem_ld32(c_addr + 32, vb);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) vb[i] = __float_as_uint(tau_m) + (uint32_t)(i * lane + 7);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            uint32_t d0, d1, d2, d3;
            sub_tau2_9(va[4 * i], va[4 * i + 1], tau_m, d0, d1);
            sub_tau2_9(va[4 * i + 2], va[4 * i + 3], tau_m, d2, d3);
            pk[i] = pack_w4_9(d0, d1, d2, d3);
          }
          tmem_ld_wait();
          tmem_regs_ready(vb);
          tc_fence_before();
          nbar_arrive(bar_c, kBarThreads);  // C_g may be overwritten
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            uint32_t d0, d1, d2, d3;
            sub_tau2_9(vb[4 * i], vb[4 * i + 1], tau_m, d0, d1);
            sub_tau2_9(vb[4 * i + 2], vb[4 * i + 3], tau_m, d2, d3);
            pk[8 + i] = pack_w4_9(d0, d1, d2, d3);
          }
        } else {
          tc_fence_before();
          nbar_arrive(bar_c, kBarThreads);
        }
#endif
        K9_TL(role, k, 2);
        K9_TL(role, k, 3);
        if (k > 0) mbar_wait(p_free, (k - 1) & 1);  // the group's previous weighted sum is done with P_g
        K9_TL(role, k, 4);
        if (active) {
          if (w.mode == 0) {
            tc_fence_after();
            if (!K9_SKIP(8)) {
              tmem_st16(p_addr, pk);
              tmem_st_wait();
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) cnt += pk[i] & 1u;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) cnt += __popc(pk[i]);  // 8 bits per window member
          }
        }
        tc_fence_before();
        nbar_arrive(bar_p, kBarThreads);  // the issuer may run the weighted sum
        K9_TL(role, k, 5);
        if (j == ccnt - 1 && h == 0) {
          // ---- drain the item's Gq_g into the segment sums ----
          mbar_wait(g_full, drains & 1);
          ++drains;
          tc_fence_after();
          if (w.mode == 0 && active) {
            if (seg != w.key) {
              flush();
              seg = w.key;
              seg_f = w.f;
              seg_tile = w.tile;
            }
            uint32_t ga[16], gb2[16], gc[16];
            tmem_ld16(gq, ga);
            tmem_ld16(gq + DP, gb2);
            tmem_ld16(gq + 2 * DP, gc);
            tmem_ld_wait();
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const long long s = (long long)(int)ga[kk] * 65536ll + (long long)(int)gb2[kk] * 256ll + (int)gc[kk];
              // s = 255 x (an integer below 2^43): the correctly rounded product is within 1e-3 of it
              gs[kk * kBM] += __double2ll_rn((double)s * (1.0 / 255.0));
            }
          }
          tc_fence_before();  // ordered before the next bar_p arrive, hence before Gq_g is reset
          K9_TL(role, k, 6);
        }
      }
      // count pass: each warp flushes its window counts when its segment (same seed tile) ends
      const bool last = (item + kGroups >= i_end) || item9(p, item + kGroups, nch).key != w.key;
      if (last && w.mode != 0) {
        if (cnt) atomicAdd(p.cacc + (size_t)w.f * p.S_pad + (size_t)w.tile * kBM + row, cnt >> 3);
        cnt = 0;
      }
    }
    if (h == 0) flush();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpIss) tmem_dealloc(tmem, 512);
}

int iter9_smem_bytes() { return k9::SMEM; }

cudaError_t launch_iter9(const TMaps& tm, const Params& p, int grid, cudaStream_t st) {
  iter9_kernel<<<grid, k9::kThreads, k9::SMEM, st>>>(tm, p);
  return cudaGetLastError();
}

cudaError_t setup_iter9_attrs() {
  return cudaFuncSetAttribute(iter9_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, k9::SMEM);
}

}  // namespace fms
