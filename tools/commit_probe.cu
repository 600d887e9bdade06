// commit_probe.cu -- issue cost of tcgen05.commit and tcgen05.mma on sm_100a as seen by the issuing warp.
// One warp per CTA (148 CTAs) issues `reps` rounds of: (a) commits only, (b) one MMA + one commit,
// (c) one MMA + two commits, (d) MMAs only, (e) 3 MMAs + 2 commits (K2's MMA1 per tile),
// (f) 4 kind::i8 TS MMAs (N = 48) + 1 commit (K2's MMA2 per tile), then waits for the last commit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2007_14283_b200/csrc \
//        -o tools/commit_probe tools/commit_probe.cu
#include <cstdio>

#include "fms_device.cuh"
using namespace fms;

template <int MODE>
__global__ void probe(int reps, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sm[16384];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  const uint64_t ad = umma_desc(smem_u32(sm), 16, 256, 6), bd = umma_desc(smem_u32(sm + 4096), 16, 256, 6);
  const uint64_t qd = umma_desc(smem_u32(sm + 8192), 16, 1024, 2);
  constexpr uint32_t I1 = idesc_f16(128, 128, 0, 0);
  const uint32_t I2 = idesc_i8(128, 48);
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) {
      tc_commit_el(&bar[r & 7]);
    } else if (MODE == 1) {
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 0);
      tc_commit_el(&bar[r & 7]);
    } else if (MODE == 2) {
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 0);
      tc_commit_el(&bar[r & 7]);
      tc_commit_el(&bar[(r + 4) & 7]);
    } else if (MODE == 3) {
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 0);
    } else if (MODE == 4) {
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 0);
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 1);
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 1);
      tc_commit_el(&bar[r & 7]);
      tc_commit_el(&bar[(r + 4) & 7]);
    } else if (MODE == 5) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_ts_i8_el(tm + 400, tm + 256 + k * 8, qd + k * 2, I2, 1);
      tc_commit_el(&bar[r & 7]);
    } else if (MODE == 6) {
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 0);
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 1);
      mma_ss_f16_el(tm + (r & 1) * 128, ad, bd, I1, 1);
    }
  }
  unsigned long long t1 = clock64();
  // drain: one more commit and wait for it
  tc_commit_el(&bar[0]);
  __syncwarp();
  unsigned long long t2 = clock64();
  if ((threadIdx.x & 31) == 0 && warp == 0) {
    out[blockIdx.x * 2 + 0] = (t1 - t0) / reps;
    out[blockIdx.x * 2 + 1] = t2 - t1;
  }
  __syncthreads();
  // let every commit land before the TMEM is released
  for (volatile int spin = 0; spin < 200000; spin = spin + 1) {
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16 * 148);
  unsigned long long h[2 * 148];
  const char* nm[] = {"commit only", "1 MMA + 1 commit", "1 MMA + 2 commits", "1 MMA only",
                      "3 MMA + 2 commits (MMA1 tile)", "4 i8 TS MMA N=48 + 1 commit (MMA2 tile)", "3 MMA only"};
  for (int m = 0; m < 7; ++m) {
    for (int it = 0; it < 2; ++it) {
      switch (m) {
        case 0: probe<0><<<148, 32>>>(2000, d); break;
        case 1: probe<1><<<148, 32>>>(2000, d); break;
        case 2: probe<2><<<148, 32>>>(2000, d); break;
        case 3: probe<3><<<148, 32>>>(2000, d); break;
        case 4: probe<4><<<148, 32>>>(2000, d); break;
        case 5: probe<5><<<148, 32>>>(2000, d); break;
        case 6: probe<6><<<148, 32>>>(2000, d); break;
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-42s: %5llu issue cycles per round (CTA 0)\n", nm[m], h[0]);
  }
  return 0;
}
