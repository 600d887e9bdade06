// ts_probe.cu -- does a stream of tcgen05.mma slow concurrent tcgen05.ld?  Warp 0 issues `reps` MMAs
// of one kind while warps 4..11 (2 per SM sub-partition) stream 32x32b.x64 loads, as K2's epilogue
// does.  Kinds: 0 none, 1 SS kind::f16 M128 N128 K16 (K2's similarity), 2 TS kind::i8 M128 N48 K32
// (K2's weighted sum, A from TMEM), 3 SS kind::i8 M128 N48 K32 (A from shared memory), 4 TS kind::f16
// M128 N48 K16.  Reports the cycles per load and per MMA (CTA average over 148 CTAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2007_14283_b200/csrc \
//        -o tools/ts_probe tools/ts_probe.cu
#include <cstdio>

#include "fms_device.cuh"
using namespace fms;

__device__ __forceinline__ void mma_ss_i8_el(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <int KIND>
__global__ void probe(int reps, int loads, unsigned long long* out, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (KIND != 0 && reps > 0) {
      const uint64_t ad = umma_desc(smem_u32(sm), 16, 256, 6), bd = umma_desc(smem_u32(sm + 8192), 16, 256, 6);
      const uint64_t qd = umma_desc(smem_u32(sm + 16384), 16, 1024, 2);  // 48 rows x 128 B, SW128
      const uint64_t pd = umma_desc(smem_u32(sm + 24576), 16, 1024, 2);  // 128 rows x 128 B, SW128
      for (int r = 0; r < reps; ++r) {
        if (KIND == 1) {
          mma_ss_f16_el(tmem + 256 + (r & 1) * 128, ad, bd, idesc_f16(128, 128, 0, 0), r >= 2);
        } else if (KIND == 2) {
          mma_ts_i8_el(tmem + 448, tmem + 384 + (r & 7) * 8, qd + (uint64_t)((r & 3) * 2), idesc_i8(128, 48), 1);
        } else if (KIND == 3) {
          mma_ss_i8_el(tmem + 448, pd + (uint64_t)((r & 3) * 2), qd + (uint64_t)((r & 3) * 2), idesc_i8(128, 48), 1);
        } else if (KIND == 4) {
          mma_ts_f16_el(tmem + 448, tmem + 384 + (r & 7) * 8, bd, idesc_f16(128, 48, 0, 0), 1);
        }
      }
      tc_commit_el(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
    }
  } else if (warp >= 4 && warp < 12 && loads > 0) {
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    for (int r = 0; r < loads; ++r) {
      uint32_t v[64];
      tmem_ld64(tmem + lb + ((warp >> 2) & 1) * 64 + (r & 1) * 128, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 64; ++i) acc ^= v[i];
    }
    if (acc == 0x1234567u) sink[0] = acc;
  }
  unsigned long long t1 = clock64();
  if (lane == 0 && (warp == 0 || warp == 4)) out[blockIdx.x * 2 + (warp == 4)] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, 16 * 148);
  cudaMalloc(&sink, 4);
  unsigned long long h[296];
  const int smem = 48 * 1024 + 1024;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[] = {"no MMA", "SS f16 N128 K16", "TS i8 N48 K32", "SS i8 N48 K32", "TS f16 N48 K16"};
  const int reps_of[] = {0, 256, 640, 640, 640};
  for (int kind = 0; kind < 5; ++kind) {
    for (int loads : {0, 256}) {
      if (kind == 0 && loads == 0) continue;
      for (int it = 0; it < 2; ++it) {
        const int reps = reps_of[kind];
        switch (kind) {
          case 0: probe<0><<<148, 384, smem>>>(reps, loads, d, sink); break;
          case 1: probe<1><<<148, 384, smem>>>(reps, loads, d, sink); break;
          case 2: probe<2><<<148, 384, smem>>>(reps, loads, d, sink); break;
          case 3: probe<3><<<148, 384, smem>>>(reps, loads, d, sink); break;
          case 4: probe<4><<<148, 384, smem>>>(reps, loads, d, sink); break;
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double a = 0, b = 0;
      for (int i = 0; i < 148; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
      a /= 148; b /= 148;
      printf("%-18s x %3d  +  8 warps x %3d LDTM.x64:  MMA stream %7.0f cyc (%5.1f per MMA)  loads %7.0f cyc (%5.1f per load)\n",
             nm[kind], reps_of[kind], loads, a, reps_of[kind] ? a / reps_of[kind] : 0.0, b, loads ? b / loads : 0.0);
    }
  }
  return 0;
}
