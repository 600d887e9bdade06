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
__device__ __forceinline__ void mma_ts_i8_el(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss_i8_el(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int b_mn) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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
    const uint32_t idesc = MODE >= 4 ? idesc_i8(128, N, 0) : idesc_f16(128, N, 0, (MODE == 1 || MODE == 3) ? 1 : 0);
    unsigned long long t0 = clock64();
    if (MODE >= 4) {  // kind::i8, K = 32 bytes; B K-major SW128 (rows of 128 pixels)
      const uint64_t ad = umma_desc(a, 16, 1024, 2), bd = umma_desc(b, 16, 1024, 2);
      for (int r = 0; r < reps; ++r) {
        if (MODE == 5) mma_ss_i8_el(tmem + (r & 3) * 128 * (nacc > 1), ad, bd + (uint64_t)((r & 3) * 2), idesc, r >= nacc);
        else mma_ts_i8_el(tmem + 256 + (r & 3) * 64 * (nacc > 1), tmem + (r & 7) * 8, bd + (uint64_t)((r & 3) * 2), idesc, r >= nacc);
      }
      commit_el(&bar);
    } else if (MODE >= 2) {
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

// two warps issue concurrently: warp 0 SS N=128 (similarity), warp 1 TS N=32 (weighted sum), to see
// whether the per-instruction cost of small-N MMAs is a pipe limit or a per-warp issue limit
__global__ void dual(int reps1, int reps2, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sm[40 * 1024];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t a = smem_u32(sm), b = smem_u32(sm + 8192);
  unsigned long long t0 = clock64();
  if (warp == 0 && reps1 > 0) {
    const uint64_t ad = umma_desc(a, 16, 256, 6), bd = umma_desc(b, 16, 256, 6);
    for (int r = 0; r < reps1; ++r) mma_ss_el(tmem + (r & 1) * 128, ad, bd, idesc_f16(128, 128, 0, 0), r >= 2);
    commit_el(&bar[0]);
    __syncwarp();
    mbar_wait(&bar[0], 0);
  } else if (warp == 1 && reps2 > 0) {
    const uint64_t bd2 = umma_desc(b, 4096, 256, 6);
    for (int r = 0; r < reps2; ++r)
      mma_ts_el(tmem + 384 + (r & 1) * 32, tmem + 256 + (r & 7) * 8, bd2 + (uint64_t)((r & 7) * 32), idesc_f16(128, 32, 0, 1), r >= 2);
    commit_el(&bar[1]);
    __syncwarp();
    mbar_wait(&bar[1], 0);
  }
  unsigned long long t1 = clock64();
  if (lane == 0 && warp < 2) out[blockIdx.x * 2 + warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// does MMA issue block the issuing SM sub-partition?  warp 0 issues `reps` MMAs back to back while
// warps 4 (same SMSP as warp 0) and 5 (another SMSP) run an independent ALU loop
__global__ void interfere(int reps, int mode, int iters, unsigned long long* out, float* sink) {
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
  const uint32_t a = smem_u32(sm), b = smem_u32(sm + 8192);
  if (warp == 0) {
    if (reps > 0) {
      if (mode == 0) {
        const uint64_t bd2 = umma_desc(b, 4096, 256, 6);
        for (int r = 0; r < reps; ++r)
          mma_ts_el(tmem + 384 + (r & 1) * 32, tmem + 256 + (r & 7) * 8, bd2 + (uint64_t)((r & 7) * 32), idesc_f16(128, 32, 0, 1), 1);
      } else {
        const uint64_t ad = umma_desc(a, 16, 256, 6), bd = umma_desc(b, 16, 256, 6);
        for (int r = 0; r < reps; ++r) mma_ss_el(tmem + (r & 1) * 128, ad, bd, idesc_f16(128, 128, 0, 0), 1);
      }
      commit_el(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
    }
  } else if (warp == 4 || warp == 5) {
    float x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x0 = fmaf(x0, 1.0001f, 0.5f); x1 = fmaf(x1, 1.0001f, 0.5f); x2 = fmaf(x2, 1.0001f, 0.5f); x3 = fmaf(x3, 1.0001f, 0.5f);
    }
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 2 + (warp - 4)] = t1 - t0;
    if (x0 + x1 + x2 + x3 == 1234.5f) sink[0] = x0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// does a warp spinning in mbarrier.try_wait slow the other warps of its SM sub-partition?
__global__ void spin(int mode, int iters, unsigned long long* out, float* sink) {
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
  __syncthreads();
  if (warp == 0) {
    if (mode == 1) mbar_wait(&bar, 0);                       // completes when warp 4 arrives at the end
    else if (mode == 2) mbar_wait_sleep(&bar, 0, 100);
    else if (mode == 3) { while (!stop) {} }
  } else if (warp == 4 || warp == 5) {
    float x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3, x4 = lane, x5 = lane + 1, x6 = lane + 2, x7 = lane + 3;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x0 = fmaf(x0, 1.0001f, 0.5f); x1 = fmaf(x1, 1.0001f, 0.5f); x2 = fmaf(x2, 1.0001f, 0.5f); x3 = fmaf(x3, 1.0001f, 0.5f);
      x4 = fmaf(x4, 1.0001f, 0.5f); x5 = fmaf(x5, 1.0001f, 0.5f); x6 = fmaf(x6, 1.0001f, 0.5f); x7 = fmaf(x7, 1.0001f, 0.5f);
    }
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 2 + (warp - 4)] = t1 - t0;
    if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1234.5f) sink[0] = x0;
  }
  __syncwarp();
  if (warp == 4) { if (lane == 0) { mbar_arrive(&bar); stop = 1; } }
  __syncthreads();
}

// epilogue-like ALU loop (FADD + PRMT + LOP3 per pair) next to: idle / try_wait spinner / MMA issuer
__global__ void alu_mix(int mode, int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ __align__(1024) uint8_t sm[40 * 1024];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0) {
    if (mode == 1) mbar_wait(&bar, 0);
    else if (mode == 2) {
      const uint64_t bd2 = umma_desc(smem_u32(sm + 8192), 4096, 256, 6);
      for (int r = 0; r < 1200; ++r)
        mma_ts_el(tmem + 384 + (r & 1) * 32, tmem + 256 + (r & 7) * 8, bd2 + (uint64_t)((r & 7) * 32), idesc_f16(128, 32, 0, 1), 1);
      commit_el(&bar2);
      __syncwarp();
      mbar_wait(&bar2, 0);
    }
  } else if (warp == 4 || warp == 5) {
    float c[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) c[i] = (float)(lane * 64 + i) * 0.37f;
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float u0 = c[2 * i] - 1843.2f, u1 = c[2 * i + 1] - 1843.2f;
        uint32_t m;
        asm volatile("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(m) : "r"(__float_as_uint(u0)), "r"(__float_as_uint(u1)));
        acc ^= ~m & 0x3C003C00u;
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) c[i] += 1.0f;
    }
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 2 + (warp - 4)] = t1 - t0;
    if (acc == 0x12345u) sink[0] = acc;
  }
  __syncwarp();
  if (warp == 4 && lane == 0) mbar_arrive(&bar);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// do tcgen05.ld traffic and MMA execution contend?  warp 0 issues `reps` SS N=128 MMAs (into columns
// 256..383) while warps 4..11 (2 per SM sub-partition) stream 32x32b.x64 loads from columns 0..255
__global__ void tmem_mma(int reps, int loads, unsigned long long* out, unsigned* sink) {
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
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (reps > 0) {
      const uint64_t ad = umma_desc(smem_u32(sm), 16, 256, 6), bd = umma_desc(smem_u32(sm + 8192), 16, 256, 6);
      for (int r = 0; r < reps; ++r) mma_ss_el(tmem + 256 + (r & 1) * 128, ad, bd, idesc_f16(128, 128, 0, 0), r >= 2);
      commit_el(&bar);
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
  cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  struct Case { int mode, N, nacc; };
  const Case cases[] = {{0, 128, 1}, {2, 128, 1}, {2, 128, 4}, {2, 32, 1}, {2, 32, 4}, {2, 256, 1},
                        {3, 32, 1}, {3, 32, 4}, {3, 64, 1}, {3, 64, 4}, {3, 16, 1}, {3, 128, 1},
                        {4, 32, 1}, {4, 48, 1}, {4, 48, 4}, {4, 64, 1}, {4, 64, 4}, {4, 96, 1}, {4, 128, 1}, {5, 128, 1}, {5, 128, 4}};
  for (const Case& cs : cases) {
    const int reps = 64;
    for (int it = 0; it < 2; ++it) {
      if (cs.mode == 0) probe<0><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else if (cs.mode == 1) probe<1><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else if (cs.mode == 2) probe<2><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else if (cs.mode == 3) probe<3><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else if (cs.mode == 4) probe<4><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      else probe<5><<<148, 128>>>(reps, cs.N, cs.nacc, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const char* nm[] = {"SS lane0", "TS lane0", "SS elect", "TS elect", "TS i8 K32", "SS i8 K32"};
    printf("%s M=128 N=%3d K=16 accumulators=%d : %6.1f cycles/MMA (floor %d)\n", nm[cs.mode], cs.N,
           cs.nacc, avg / reps, 128 * cs.N / 256);
  }
  {
    unsigned long long* d3;
    float* sink;
    cudaMalloc(&d3, 16 * 148);
    cudaMalloc(&sink, 4);
    unsigned long long h3[296];
    for (int mode = 0; mode < 2; ++mode)
      for (int reps : {0, 256}) {
        for (int it = 0; it < 2; ++it) interfere<<<148, 256>>>(reps, mode, 4000, d3, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h3, d3, 16 * 148, cudaMemcpyDeviceToHost);
        double w4 = 0, w5 = 0;
        for (int i = 0; i < 148; ++i) { w4 += h3[2 * i]; w5 += h3[2 * i + 1]; }
        printf("interfere: %s x%d issued by warp 0 -> ALU loop warp4 (same SMSP) %.0f cyc, warp5 (other SMSP) %.0f cyc\n",
               mode == 0 ? "TS N=32" : "SS N=128", reps, w4 / 148, w5 / 148);
      }
  }
  {
    unsigned long long* d3;
    float* sink;
    cudaMalloc(&d3, 16 * 148);
    cudaMalloc(&sink, 4);
    unsigned long long h3[296];
    const char* nm[] = {"idle", "try_wait spin", "try_wait+nanosleep(100)", "volatile smem poll"};
    for (int mode = 0; mode < 4; ++mode) {
      for (int it = 0; it < 2; ++it) spin<<<148, 256>>>(mode, 4000, d3, sink);
      cudaDeviceSynchronize();
      cudaMemcpy(h3, d3, 16 * 148, cudaMemcpyDeviceToHost);
      double w4 = 0, w5 = 0;
      for (int i = 0; i < 148; ++i) { w4 += h3[2 * i]; w5 += h3[2 * i + 1]; }
      printf("spin: warp0 %-24s -> FMA loop warp4 (same SMSP) %.0f cyc, warp5 (other SMSP) %.0f cyc\n", nm[mode], w4 / 148, w5 / 148);
    }
  }
  {
    unsigned long long* d3;
    uint32_t* sink;
    cudaMalloc(&d3, 16 * 148);
    cudaMalloc(&sink, 4);
    unsigned long long h3[296];
    const char* nm[] = {"idle", "try_wait spin", "1200 TS MMAs"};
    for (int mode = 0; mode < 3; ++mode) {
      for (int it = 0; it < 2; ++it) alu_mix<<<148, 256>>>(mode, 300, d3, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h3, d3, 16 * 148, cudaMemcpyDeviceToHost);
      double w4 = 0, w5 = 0;
      for (int i = 0; i < 148; ++i) { w4 += h3[2 * i]; w5 += h3[2 * i + 1]; }
      printf("alu_mix: warp0 %-14s -> epilogue-like loop warp4 (same SMSP) %.0f cyc, warp5 (other SMSP) %.0f cyc (%.2f cyc per pair)\n",
             nm[mode], w4 / 148, w5 / 148, w5 / 148 / (300.0 * 32));
    }
  }
  {
    unsigned long long* d4;
    unsigned* sink4;
    cudaMalloc(&d4, 16 * 148);
    cudaMalloc(&sink4, 4);
    unsigned long long h4[296];
    const int cfg[][2] = {{200, 0}, {0, 400}, {200, 400}};
    for (auto& c : cfg) {
      for (int it = 0; it < 2; ++it) tmem_mma<<<148, 384>>>(c[0], c[1], d4, sink4);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h4, d4, 16 * 148, cudaMemcpyDeviceToHost);
      double a = 0, b = 0;
      for (int i = 0; i < 148; ++i) { a += h4[2 * i]; b += h4[2 * i + 1]; }
      printf("tmem_mma: %3d SS N=128 MMAs (%.0f cyc) + 8 warps x %3d LDTM.x64 (%.0f cyc)\n", c[0], c[0] ? a / 148 : 0.0,
             c[1], c[1] ? b / 148 : 0.0);
    }
  }
  unsigned long long* d2;
  cudaMalloc(&d2, 16 * 148);
  unsigned long long h2[296];
  const int combos[][2] = {{96, 0}, {0, 256}, {96, 256}, {192, 256}};
  for (auto& c : combos) {
    for (int it = 0; it < 2; ++it) {
      dual<<<148, 128>>>(c[0], c[1], d2);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h2, d2, 16 * 148, cudaMemcpyDeviceToHost);
    double w0 = 0, w1 = 0;
    for (int i = 0; i < 148; ++i) { w0 += h2[2 * i]; w1 += h2[2 * i + 1]; }
    printf("dual: %3d x SS N=128 (warp0 %.0f cyc) + %3d x TS N=32 (warp1 %.0f cyc)\n", c[0], c[0] ? w0 / 148 : 0.0, c[1], c[1] ? w1 / 148 : 0.0);
  }
  return 0;
}
