// tmem_bw.cu -- TMEM read bandwidth (tcgen05.ld bytes/cycle/SM) vs loading warps and loads in flight,
// alone and next to a warp streaming kind::f16 M128 N128 K16 SS MMAs (K2's similarity MMA) into other
// columns; and the MMA rate with and without the loads.  One CTA per SM, 148 CTAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2007_14283_b200/csrc \
//        -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>

#include "fms_device.cuh"

using namespace fms;

template <int F>
__global__ void probe(int reps, int mma_reps, int ldw, unsigned long long* out, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x / 32;
  if (warp == 0) tmem_alloc(&holder, 512);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = clock64();
  uint32_t acc = 0;
  if (warp < ldw) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    for (int r = 0; r < reps; ++r) {
      const uint32_t col = (uint32_t)(((r * ldw + warp) / 4 * 32 * F) % 384);
      uint32_t v[F][32];
#pragma unroll
      for (int f = 0; f < F; ++f) tmem_ld32(tmem + lane_base + col + f * 32, v[f]);
      tmem_ld_wait();
#pragma unroll
      for (int f = 0; f < F; ++f)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= v[f][i];
    }
  } else if (warp == nw - 1 && mma_reps > 0) {
    constexpr uint32_t ID = idesc_f16(128, 128, 0, 0);
    const uint64_t da = umma_desc(smem_u32(sm), 16, 256, 6);
    const uint64_t db = umma_desc(smem_u32(sm + 8192), 16, 256, 6);
    for (int r = 0; r < mma_reps; ++r) mma_ss_f16_el(tmem + 384, da, db, ID, r > 0);
    tc_commit_el(&bar);
    mbar_wait(&bar, 0);
  }
  const unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 0x12345678) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, 8 * 148 * 32);
  cudaMalloc(&sink, 4);
  static unsigned long long h[148 * 32];
  const int reps = 512;
  auto run = [&](int F, int ldw, int mma_reps, int nthreads) {
    cudaMemset(d, 0, 8 * 148 * 32);
    for (int it = 0; it < 2; ++it) {
      if (F == 1) probe<1><<<148, nthreads, 16384>>>(ldw ? reps : 0, mma_reps, ldw, d, sink);
      else if (F == 2) probe<2><<<148, nthreads, 16384>>>(ldw ? reps / 2 : 0, mma_reps, ldw, d, sink);
      else probe<4><<<148, nthreads, 16384>>>(ldw ? reps / 4 : 0, mma_reps, ldw, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double ld = 0, mm = 0;
    for (int b = 0; b < 148; ++b) {
      unsigned long long m = 0;
      for (int w = 0; w < ldw; ++w) m = h[b * 32 + w] > m ? h[b * 32 + w] : m;
      ld += m;
      mm += h[b * 32 + nthreads / 32 - 1];
    }
    ld /= 148; mm /= 148;
    const double bytes = (double)ldw * reps * 32 * 32 * 4;
    printf("x32 x%d in flight, %2d loading warps, %s: loads %8.0f cycles = %6.1f B/cycle/SM", F, ldw,
           mma_reps ? "with MMA stream" : "alone          ", ld, ldw ? bytes / ld : 0.0);
    if (mma_reps) printf(" | %d MMAs in %8.0f cycles = %.1f cycles/MMA", mma_reps, mm, mm / mma_reps);
    printf("\n");
  };
  run(1, 0, 2000, 64);  // MMA stream alone
  for (int F : {1, 2, 4})
    for (int ldw : {4, 8, 16}) {
      run(F, ldw, 0, (ldw + 1) * 32);
      run(F, ldw, 2000, (ldw + 1) * 32);
    }
  return 0;
}
