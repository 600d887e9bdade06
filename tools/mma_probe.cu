// mma_probe.cu -- microbenchmark: cycles per tcgen05.mma for the shapes the iteration kernel uses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2007_14283_b200/csrc -o mma_probe mma_probe.cu
#include <cstdio>

#include "fms_device.cuh"

using namespace fms;

// whole warp executes; elect.sync picks the issuing lane inside the asm (operands stay uniform)
__device__ __forceinline__ void mma_ss_el(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts_el(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_el(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
               :: "r"(smem_u32(bar)) : "memory");
}

// one warp issues `reps` MMAs of one shape back to back, then commits and waits
template <int MODE>
__global__ void probe(int reps, int N, int nacc, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sm[40 * 1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 8192);
    const uint32_t idesc = idesc_f16(128, N, 0, (MODE == 1 || MODE == 3) ? 1 : 0);
    unsigned long long t0 = clock64();
    if (MODE >= 2) {
      const uint64_t ad = umma_desc(a, 16, 256, 6), bd = umma_desc(b, 16, 256, 6), bd2 = umma_desc(b, 4096, 256, 6);
      for (int r = 0; r < reps; ++r) {
        if (MODE == 2) mma_ss_el(tmem + (r & 3) * 128 * (nacc > 1), ad, bd, idesc, r >= nacc);
        else mma_ts_el(tmem + 256 + (r & 3) * 64 * (nacc > 1), tmem + (r & 7) * 8, bd2 + (uint64_t)((r & 7) * 32), idesc, r >= nacc);
      }
      commit_el(&bar);
    } else if (lane == 0) {
      for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {  // SS, K-major both (similarity GEMM)
          mma_ss_f16(tmem + (r % nacc) * 128, umma_desc(a, 16, 256, 6), umma_desc(b, 16, 256, 6), idesc, r >= nacc);
        } else {          // TS, A from TMEM, B MN-major (weighted sum)
          mma_ts_f16(tmem + 256 + (r % nacc) * 64, tmem + (r & 7) * 8, umma_desc(b, 4096, 256, 6), idesc, r >= nacc);
        }
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  struct Case { int mode, N, nacc; };
  const Case cases[] = {{0, 128, 1}, {2, 128, 1}, {2, 128, 4}, {2, 32, 1}, {2, 32, 4}, {2, 256, 1}, {2, 256, 4},
                        {3, 32, 1}, {3, 32, 4}, {3, 64, 1}, {3, 64, 4}, {3, 16, 1}, {3, 128, 1}};
  for (const Case& cs : cases) {
    const int reps = 64;
    for (int it = 0; it < 2; ++it) {
      if (cs.mode == 0) probe<0><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else if (cs.mode == 1) probe<1><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else if (cs.mode == 2) probe<2><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else probe<3><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const char* nm[] = {"SS lane0", "TS lane0", "SS elect", "TS elect"};
    printf("%s M=128 N=%3d K=16 accumulators=%d : %6.1f cycles/MMA (floor %d)\n", nm[cs.mode], cs.N,
           cs.nacc, avg / reps, 128 * cs.N / 256);
  }
  return 0;
}
