// iter8_probe.cu -- time the flat-kernel K2 (k_iter8.cu) and the fp16-weighted-sum K2 (k_iter.cu) on
// the same fixed synthetic work list: B frames x T full seed tiles x n pixels, chunked like plan_kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Ipaper_2007_14283_b200/csrc \
//        -Iinclude -o tools/iter8_probe tools/iter8_probe.cu paper_2007_14283_b200/csrc/k_iter8.cu \
//        paper_2007_14283_b200/csrc/k_iter.cu -lcuda
// Run:   tools/iter8_probe [B=32] [T=2] [ct=64] [n=262144] [DP=16] [rows per frame = 128 T]
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fms_device.cuh"

namespace fms {
cudaError_t launch_iter(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st);
cudaError_t launch_iter8(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st);
cudaError_t setup_iter_attrs();
cudaError_t setup_iter8_attrs();
cudaError_t launch_iter9(const TMaps& tm, const Params& p, int grid, cudaStream_t st);
cudaError_t setup_iter9_attrs();
}  // namespace fms
using namespace fms;

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}
static void tmap(CUtensorMap* m, void* base, uint64_t rows, int DP) {
  cuuint64_t dims[2] = {(cuuint64_t)DP, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)DP * 2};
  cuuint32_t box[2] = {(cuuint32_t)DP, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     DP == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("tmap err %d\n", (int)r);
}
static void tmap_q(CUtensorMap* m, void* base, uint64_t rows, int nq) {
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, (cuuint32_t)nq};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("tmap_q err %d\n", (int)r);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__global__ void clk_kernel(unsigned long long* out) {
  const unsigned long long c0 = clock64();
  const unsigned long long t0 = globaltimer_ns();
  unsigned long long t = t0;
  while (t - t0 < 2000000) t = globaltimer_ns();
  out[0] = clock64() - c0;
  out[1] = t - t0;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int B = argc > 1 ? atoi(argv[1]) : 32, T_per_frame = argc > 2 ? atoi(argv[2]) : 2;
  const int ct = argc > 3 ? atoi(argv[3]) : 64;
  const long long n = argc > 4 ? atoll(argv[4]) : 262144;
  const int DP = argc > 5 ? atoi(argv[5]) : 16;
  // active seed rows per frame (default: every tile full); the last tile of a frame is partial otherwise
  const int rows = argc > 6 ? atoi(argv[6]) : T_per_frame * 128;
  const long long n_pad = (n + 127) / 128 * 128;
  const int S_pad = 128 * T_per_frame;
  setup_iter_attrs();
  setup_iter8_attrs();
  setup_iter9_attrs();
  Params p{};
  p.B = B; p.DP = DP; p.d = DP; p.n = n; p.n_pad = n_pad; p.n_ptiles = (int)(n_pad / 128);
  p.S_pad = S_pad; p.S_cap = S_pad; p.n_chunks = (p.n_ptiles + kChunkTiles - 1) / kChunkTiles;
  p.tau_f = 0.9f;
  p.num_sms = 148;
  __half *xh, *xl, *sh, *ss, *sl;
  int8_t* xq;
  cudaMalloc(&xh, B * n_pad * DP * 2); cudaMalloc(&xl, B * n_pad * DP * 2);
  cudaMalloc(&xq, B * n_pad * DP * 3);
  p.Xh = xh; p.Xl = xl; p.Xq = xq;  // raw pointers (the bulk-copy timing experiments read them)
  cudaMalloc(&sh, B * S_pad * DP * 2); cudaMalloc(&ss, B * S_pad * DP * 2); cudaMalloc(&sl, B * S_pad * DP * 2);
  // pixels: half of them near the seed direction (in window), half far -- the epilogue cost does not
  // depend on the data, the window sums just need to be non-trivial
  std::vector<__half> hx(B * n_pad * DP), hl(B * n_pad * DP);
  for (size_t i = 0; i < (size_t)B * n_pad; ++i)
    for (int k = 0; k < DP; ++k) {
      const bool near = (i * 2654435761u >> 7) & 1;
      const float v = k == 0 ? (near ? 0.99f : 0.3f) : ((i * 31 + k * 7) % 13 - 6) * 0.002f;
      hx[i * DP + k] = __float2half(rintf(v * 2048.f));
      hl[i * DP + k] = __float2half((float)((int)((i + k) * 2654435761u % 2048) - 1024));
    }
  cudaMemcpy(xh, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(xl, hl.data(), hl.size() * 2, cudaMemcpyHostToDevice);
  std::vector<int8_t> hq(B * n_pad * DP * 3);
  for (size_t i = 0; i < hq.size(); ++i) hq[i] = (int8_t)((i * 2654435761u >> 9) & 0xFF);
  cudaMemcpy(xq, hq.data(), hq.size(), cudaMemcpyHostToDevice);
  std::vector<__half> hs(B * S_pad * DP);
  for (size_t i = 0; i < hs.size(); ++i) hs[i] = __float2half((i % DP) == 0 ? 1.0f : 0.f);
  cudaMemcpy(sh, hs.data(), hs.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(ss, 0, hs.size() * 2);
  cudaMemset(sl, 0, hs.size() * 2);
  TMaps tm;
  tmap(&tm.xh, xh, B * n_pad, DP); tmap(&tm.xl, xl, B * n_pad, DP);
  tmap(&tm.sh, sh, B * S_pad, DP); tmap(&tm.ss, ss, B * S_pad, DP); tmap(&tm.sl, sl, B * S_pad, DP);
  tmap_q(&tm.xq, xq, (uint64_t)B * p.n_ptiles * 3 * DP, 3 * DP);
  const int T = B * T_per_frame;
  std::vector<TileTask> tt(T);
  for (int t = 0; t < T; ++t) tt[t] = TileTask{t / T_per_frame, t % T_per_frame, 0, 0, 0, 0, 0, 0};
  cudaMalloc(&p.tiles, T * sizeof(TileTask));
  cudaMemcpy(p.tiles, tt.data(), T * sizeof(TileTask), cudaMemcpyHostToDevice);
  std::vector<FrameCtl> hc(B);
  for (int f = 0; f < B; ++f) { memset(&hc[f], 0, sizeof(FrameCtl)); hc[f].tile_off = f * T_per_frame; hc[f].n_tiles_step = T_per_frame; hc[f].n_active = rows; }
  cudaMalloc(&p.ctl, B * sizeof(FrameCtl));
  cudaMemcpy(p.ctl, hc.data(), B * sizeof(FrameCtl), cudaMemcpyHostToDevice);
  cudaMalloc(&p.counters, 64 * 4);
  cudaMalloc(&p.gacc, (size_t)B * S_pad * DP * 8);
  cudaMalloc(&p.cacc, (size_t)B * S_pad * 4);
  cudaMemset(p.gacc, 0, (size_t)B * S_pad * DP * 8);
#if defined(K8_TIMELINE) || defined(K9_TIMELINE)
  cudaMalloc(&p.dbg, 19 * 512 * 8 * 8);
#endif
  unsigned long long* dclk;
  cudaMalloc(&dclk, 16);
  clk_kernel<<<1, 1>>>(dclk);
  unsigned long long hclk[2];
  cudaMemcpy(hclk, dclk, 16, cudaMemcpyDeviceToHost);
  const double ghz = (double)hclk[0] / (double)hclk[1];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double pairs = (double)T * 128 * n;
  {
    // barrier offsets (relative to the 1024-aligned dynamic smem base) for decoding stuck waits
    const int S = DP == 16 ? 9 : 6;
    const int stage_b = 2 * 128 * DP * 2 + 3 * DP * 128;
    const int bars = 6 * 128 * DP * 2 + S * stage_b + 128 * DP * 8;
    printf("barriers at smem+0x%x: x_full[%d], x_empty[%d], a_full[2], a_empty[2], c_full[NC], c_empty[NC], g_full, "
           "g_empty, p_full[NP], gs_bar[4]\n", bars, S, S);
  }
#ifdef FMS_WAIT_DEBUG
  for (int which = 0; which < 1; ++which) {
#else
  for (int which = 0; which < 3; ++which) {
#endif
    if (which == 2 && DP != 16) break;
    const int c = which != 1 ? ct : kChunkTiles;
    const int nch = (p.n_ptiles + c - 1) / c;
    int cnt[14] = {0};
    cnt[0] = T * (which != 1 ? nch : p.n_chunks);
    cnt[1] = T;
    cnt[12] = c;
    cnt[13] = nch;
    cudaMemcpy(p.counters, cnt, sizeof(cnt), cudaMemcpyHostToDevice);
    auto launch = [&]() {
      return which == 0 ? launch_iter8(DP, tm, p, 148, 0)
                        : which == 1 ? launch_iter(DP, tm, p, 148, 0) : launch_iter9(tm, p, 148, 0);
    };
    if (which == 2) cudaMemset(p.gacc, 0, (size_t)B * S_pad * DP * 8);
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
#ifdef FMS_WAIT_DEBUG
    {
      unsigned n = 0;
      cudaMemcpyFromSymbol(&n, fms_stuck_n, 4);
      unsigned long long st[64];
      cudaMemcpyFromSymbol(st, fms_stuck, sizeof(st));
      printf("stuck waits: %u\n", n);
      for (unsigned i = 0; i < n && i < 64; ++i)
        printf("  block %llu warp %llu smem 0x%05llx parity %llu\n", st[i] >> 40, (st[i] >> 32) & 0xFF,
               (st[i] >> 4) & 0xFFFFF, st[i] & 1);
    }
#endif
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double tiles_per_sm = (double)T * p.n_ptiles / 148.0;
    const double ns_tile = ms * 1e6 / tiles_per_sm;
    printf("%s DP=%d B=%d T/frame=%d ct=%d n=%lld: %.3f ms/launch, %.0f ns = %.0f cycles (%.3f GHz) per 128x128 tile per SM, "
           "%.1f TFLOP/s (4nD/pair)\n",
           which == 0 ? "iter8 (i8 weighted sum)" : which == 1 ? "iter  (f16 weighted sum)" : "iter9 (two groups)  ", DP, B, T_per_frame, c, n, ms, ns_tile,
           ns_tile * ghz, ghz, pairs * 4 * DP / (ms * 1e-3) / 1e12);
  }
  if (DP == 16) {
    // exactness cross-check: one launch of each flat-kernel K2 from zeroed sums, compared bit for bit
    const int nch = (p.n_ptiles + ct - 1) / ct;
    int cnt[14] = {0};
    cnt[0] = T * nch; cnt[1] = T; cnt[12] = ct; cnt[13] = nch;
    cudaMemcpy(p.counters, cnt, sizeof(cnt), cudaMemcpyHostToDevice);
    const size_t ng = (size_t)B * S_pad * DP;
    std::vector<double> g8(ng), g9(ng);
    cudaMemset(p.gacc, 0, ng * 8);
    launch_iter8(DP, tm, p, 148, 0);
    cudaMemcpy(g8.data(), p.gacc, ng * 8, cudaMemcpyDeviceToHost);
    cudaMemset(p.gacc, 0, ng * 8);
    launch_iter9(tm, p, 148, 0);
    cudaMemcpy(g9.data(), p.gacc, ng * 8, cudaMemcpyDeviceToHost);
    size_t bad = 0, nz = 0;
    for (size_t i = 0; i < ng; ++i) { bad += g8[i] != g9[i]; nz += g8[i] != 0; }
    printf("iter9 vs iter8 window sums: %zu of %zu differ (%zu nonzero) %s\n", bad, ng, nz, bad ? "MISMATCH" : "identical");
  }
#ifdef K9_TIMELINE
  {
    const size_t NE = 19 * 512 * 8;
    cudaMemset(p.dbg, 0, NE * 8);
    const int nch = (p.n_ptiles + ct - 1) / ct;
    int cnt[14] = {0};
    cnt[0] = T * nch; cnt[1] = T; cnt[12] = ct; cnt[13] = nch;
    cudaMemcpy(p.counters, cnt, sizeof(cnt), cudaMemcpyHostToDevice);
    launch_iter9(tm, p, 148, 0);
    cudaDeviceSynchronize();
    std::vector<long long> h(NE);
    cudaMemcpy(h.data(), p.dbg, NE * 8, cudaMemcpyDeviceToHost);
    auto ev = [&](int role, int t, int e) { return h[((size_t)role * 512 + t) * 8 + e]; };
    const long long t0 = ev(2, 0, 0);
    printf("iter9 timeline of CTA 0 (cycles from group 0 warp 0's first wait): k | group g: issuer [C synced, MMA1 issued, "
           "P synced, MMA2 issued] | warp q0h0 [cfull wait, ld+arrive, alu, pfree wait, st+arrive] | warp q1h1 [same]\n");
    for (int k = 0; k < 40; ++k) {
      printf("%3d", k);
      for (int g = 0; g < 2; ++g) {
        printf(" | g%d %6lld a%4lld x%4lld i%4lld P%4lld q%4lld i%4lld |", g, ev(g, k, 0) - t0, ev(g, k, 4) - ev(g, k, 0),
               ev(g, k, 5) - ev(g, k, 4), ev(g, k, 1) - ev(g, k, 5), ev(g, k, 2) - ev(g, k, 1), ev(g, k, 6) - ev(g, k, 2),
               ev(g, k, 3) - ev(g, k, 6));
        for (int w : {0, 5}) {
          const int r = 2 + g * 8 + w;
          printf(" %6lld[%4lld] %4lld %4lld %4lld %4lld", ev(r, k, 1) - t0, ev(r, k, 1) - ev(r, k, 0), ev(r, k, 2) - ev(r, k, 1),
                 ev(r, k, 3) - ev(r, k, 2), ev(r, k, 4) - ev(r, k, 3), ev(r, k, 5) - ev(r, k, 4));
        }
      }
      printf("\n");
    }
  }
#endif
#ifdef K8_TIMELINE
  {
    const size_t NE = 19 * 512 * 8;
    cudaMemset(p.dbg, 0, NE * 8);
    const int nch = (p.n_ptiles + ct - 1) / ct;
    int cnt[14] = {0};
    cnt[0] = T * nch; cnt[1] = T; cnt[12] = ct; cnt[13] = nch;
    cudaMemcpy(p.counters, cnt, sizeof(cnt), cudaMemcpyHostToDevice);
    launch_iter8(DP, tm, p, 148, 0);
    cudaDeviceSynchronize();
    std::vector<long long> h(NE);
    cudaMemcpy(h.data(), p.dbg, NE * 8, cudaMemcpyDeviceToHost);
    auto ev = [&](int role, int t, int e) { return h[((size_t)role * 512 + t) * 8 + e]; };
    const long long t0 = ev(1, 0, 0);
    printf("timeline of CTA 0 (cycles from MMA1's first wait): tile | TMA | MMA1: wait c_empty->ok, x_full ok, "
           "issued | MMA2: p_full ok, issued | epilogue warps (h0 q0..3, h1 q0): cfull-ok [wait], ld, alu, pfree-wait, "
           "st+arrive | drain (q0): g_full ok, done\n");
#ifndef K8_GROUPS
#define K8_GROUPS 4
#endif
    const int kG = K8_GROUPS, kGW = 16 / K8_GROUPS;
    for (int t = 0; t < 48; ++t) {
      const int g = t % kG;
      printf("%3d | %6lld | %6lld %6lld %6lld %6lld | %6lld %6lld %6lld |", t, ev(0, t, 0) - t0, ev(1, t, 0) - t0,
             ev(1, t, 1) - t0, ev(1, t, 2) - t0, ev(1, t, 3) - t0, ev(2, t, 0) - t0, ev(2, t, 1) - t0, ev(2, t, 2) - t0);
      for (int w = 0; w < (kGW < 5 ? kGW : 5); ++w) {
        const int role = 3 + g * kGW + w;
        printf(" %6lld[%4lld] %4lld %4lld %4lld %4lld |", ev(role, t, 1) - t0, ev(role, t, 1) - ev(role, t, 0),
               ev(role, t, 2) - ev(role, t, 1), ev(role, t, 3) - ev(role, t, 2), ev(role, t, 4) - ev(role, t, 3),
               ev(role, t, 5) - ev(role, t, 4));
      }
      const int r0 = 3 + g * kGW;
      if (ev(r0, t, 6)) printf(" drain %6lld %6lld", ev(r0, t, 6) - t0, ev(r0, t, 7) - t0);
      printf("\n");
    }
  }
#endif
  return 0;
}
