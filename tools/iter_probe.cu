// iter_probe.cu -- time K2 (iter_kernel) on a fixed synthetic work list, with parts switched off.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I../paper_2007_14283_b200/csrc \
//        -o iter_probe iter_probe.cu ../paper_2007_14283_b200/csrc/k_iter.cu
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fms_device.cuh"

namespace fms {
cudaError_t launch_iter(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st);
cudaError_t setup_iter_attrs();
}  // namespace fms
using namespace fms;

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}
static int g_wide = 0;  // experiment: 128-byte rows (4 pixels per TMA row), same 4 KB per box
static void tmap(CUtensorMap* m, void* base, uint64_t rows, int DP, int wide = 0) {
  const int f = wide ? 4 : 1;
  cuuint64_t dims[2] = {(cuuint64_t)DP * f, (cuuint64_t)rows / f};
  cuuint64_t strides[1] = {(cuuint64_t)DP * 2 * f};
  cuuint32_t box[2] = {(cuuint32_t)DP * f, (cuuint32_t)(128 / f)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     wide ? CU_TENSOR_MAP_SWIZZLE_128B : (DP == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B),
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("tmap err %d\n", (int)r);
}

int main(int argc, char** argv) {
  const int DP = 16;
  const int B = argc > 1 ? atoi(argv[1]) : 8, T_per_frame = argc > 2 ? atoi(argv[2]) : 2;
  g_wide = argc > 3 ? atoi(argv[3]) : 0;
  const long long n = 262144, n_pad = n;
  const int S_pad = 128 * T_per_frame;
  setup_iter_attrs();
  Params p{};
  p.B = B; p.DP = DP; p.d = 16; p.n = n; p.n_pad = n_pad; p.n_ptiles = (int)(n_pad / 128);
  p.S_pad = S_pad; p.S_cap = S_pad; p.n_chunks = (p.n_ptiles + kChunkTiles - 1) / kChunkTiles;
  p.tau_f = 0.9f;
  __half *xh, *xl, *sh, *ss, *sl;
  cudaMalloc(&xh, B * n_pad * DP * 2); cudaMalloc(&xl, B * n_pad * DP * 2);
  cudaMalloc(&sh, B * S_pad * DP * 2); cudaMalloc(&ss, B * S_pad * DP * 2); cudaMalloc(&sl, B * S_pad * DP * 2);
  std::vector<__half> hx(B * n_pad * DP);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = __float2half((float)((int)(i * 2654435761u % 4096) - 2048));
  cudaMemcpy(xh, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(xl, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  std::vector<__half> hs(B * S_pad * DP);
  for (size_t i = 0; i < hs.size(); ++i) hs[i] = __float2half(0.25f * ((i % 7) - 3) / 3.f);
  cudaMemcpy(sh, hs.data(), hs.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(ss, hs.data(), hs.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(sl, hs.data(), hs.size() * 2, cudaMemcpyHostToDevice);
  TMaps tm;
  tmap(&tm.xh, xh, B * n_pad, DP, g_wide); tmap(&tm.xl, xl, B * n_pad, DP, g_wide);
  tmap(&tm.sh, sh, B * S_pad, DP); tmap(&tm.ss, ss, B * S_pad, DP); tmap(&tm.sl, sl, B * S_pad, DP);
  const int T = B * T_per_frame;
  std::vector<TileTask> tt(T);
  for (int t = 0; t < T; ++t) tt[t] = TileTask{t / T_per_frame, t % T_per_frame, 0, 0, 0, 0, 0, 0};
  cudaMalloc(&p.tiles, T * sizeof(TileTask));
  cudaMemcpy(p.tiles, tt.data(), T * sizeof(TileTask), cudaMemcpyHostToDevice);
  cudaMalloc(&p.counters, 64 * 4);
  int cnt[2] = {T * p.n_chunks, T};
  cudaMemcpy(p.counters, cnt, 8, cudaMemcpyHostToDevice);
  cudaMalloc(&p.gacc, B * S_pad * DP * 8);
  cudaMalloc(&p.cacc, B * S_pad * 4);
  cudaMalloc(&p.dbg, 16 * 512 * 8 * 8);
  cudaMemset(p.dbg, 0, 16 * 512 * 8 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double pairs = (double)T * 128 * n;
  for (int v : {0}) {
    for (int w = 0; w < 3; ++w) launch_iter(DP, tm, p, 148, 0);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) launch_iter(DP, tm, p, 148, 0);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double tiles_per_sm = (double)T * p.n_ptiles / 148.0;
    printf("B=%d T/frame=%d variant %2d (%s%s%s%s%s%s): %.3f ms/launch, %.0f ns per 128x128 tile per SM, %.1f TFLOP/s (4nD/pair)\n", B, T_per_frame, v,
           (v & 1) ? "noMMA2 " : "", (v & 2) ? "noEpi " : "", (v & 4) ? "1termMMA1 " : "", (v & 8) ? "noMMA1 " : "",
           (v & 16) ? "noLDTM " : "", (v & 64) ? "noTMA" : "", ms,
           ms * 1e6 / tiles_per_sm, pairs * 64 / (ms * 1e-3) / 1e12);
  }
  // event timeline of CTA 0 for the full kernel
  launch_iter(DP, tm, p, 148, 0);
  cudaDeviceSynchronize();
  std::vector<long long> h(16 * 512 * 8);
  cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
  auto ev = [&](int role, int t, int e) { return h[((size_t)role * 512 + t) * 8 + e]; };
  const long long t0 = ev(1, 0, 0);
  printf("tile | prod xempty | MMA1 start cempty xfull commit | per-warp epilogue: cfull, then deltas: cfull-wait, load+release, compute, P-free wait, STTM, issue\n");
  for (int t = 0; t < 40; ++t) {
    printf("%3d | %6lld | %6lld %6lld %6lld %6lld |", t, ev(0, t, 0) - t0, ev(1, t, 0) - t0, ev(1, t, 1) - t0,
           ev(1, t, 2) - t0, ev(1, t, 3) - t0);
    const int g = t & 1;
    for (int q = 0; q < 4; ++q) {
      const int role = 3 + g * 4 + q;
      printf(" q%d %6lld %4lld %4lld %4lld %4lld %4lld %4lld |", q, ev(role, t, 1) - t0, ev(role, t, 1) - ev(role, t, 0), ev(role, t, 2) - ev(role, t, 1),
             ev(role, t, 5) - ev(role, t, 2), ev(role, t, 6) - ev(role, t, 5), ev(role, t, 3) - ev(role, t, 6),
             ev(role, t, 4) - ev(role, t, 3));
    }
    printf("\n");
  }
  return 0;
}
