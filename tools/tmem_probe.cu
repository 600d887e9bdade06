// tmem_probe.cu -- TMEM load throughput (bytes/cycle/SM) for tcgen05.ld shapes and warp counts.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2007_14283_b200/csrc -o tmem_probe tmem_probe.cu
#include <cstdio>

#include "fms_device.cuh"

using namespace fms;

__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ld_32x32b_x32_pack(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void ld_x64(uint32_t taddr, uint32_t (&v)[64]) { tmem_ld64(taddr, v); }
__device__ __forceinline__ void ld_x128(uint32_t taddr, uint32_t (&v)[128]) { tmem_ld128(taddr, v); }

template <int SHAPE>
__global__ void probe(int reps, unsigned long long* out, unsigned* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  const int nw = blockDim.x / 32;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const uint32_t col = ((r * nw + warp) / 4 * 32) & 511;
    if (SHAPE == 0) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_base + col, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= v[i];
    } else if (SHAPE == 1) {
      uint32_t v[32];
      ld_16x256b_x8(tmem + lane_base + (col & 511), v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= v[i];
    } else if (SHAPE == 2) {
      uint32_t v[16];
      ld_32x32b_x32_pack(tmem + lane_base + col, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) acc ^= v[i];
    } else if (SHAPE == 3) {
      uint32_t v[64];
      ld_x64(tmem + lane_base + ((col * 2) & 511), v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 64; ++i) acc ^= v[i];
    } else {
      uint32_t v[128];
      ld_x128(tmem + lane_base + ((col * 4) & 511), v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 128; ++i) acc ^= v[i];
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&sink, 4);
  unsigned long long h[148];
  const int reps = 256;
  for (int shape = 0; shape < 5; ++shape) {
    if (shape == 1) continue;  // 16x256b needs a different lane mapping (not used)
    for (int warps : {4, 8, 16}) {
      for (int it = 0; it < 2; ++it) {
        if (shape == 0) probe<0><<<148, warps * 32>>>(reps, d, sink);
        else if (shape == 1) probe<1><<<148, warps * 32>>>(reps, d, sink);
        else if (shape == 2) probe<2><<<148, warps * 32>>>(reps, d, sink);
        else if (shape == 3) probe<3><<<148, warps * 32>>>(reps, d, sink);
        else probe<4><<<148, warps * 32>>>(reps, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      // bytes read from TMEM per CTA: warps * reps * 32 lanes * 32 columns * 4 B (pack::16b: same cells)
      const double mult = shape == 3 ? 2.0 : shape == 4 ? 4.0 : 1.0;
      const double bytes = (double)warps * reps * 32 * 32 * 4 * mult;
      const char* nm[] = {"32x32b.x32", "16x256b.x8", "32x32b.x32.pack16", "32x32b.x64", "32x32b.x128"};
      printf("%-18s warps=%2d : %8.0f cycles, %6.1f TMEM bytes/cycle/SM\n", nm[shape], warps, avg, bytes / avg);
    }
  }
  return 0;
}
