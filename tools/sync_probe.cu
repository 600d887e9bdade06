// sync_probe.cu -- latency of the synchronisation primitives used by K2's pipeline.
#include <cstdio>

#include "fms_device.cuh"
using namespace fms;

__global__ void probe(int reps, unsigned long long* out) {
  __shared__ uint64_t bar[5];
  __shared__ __align__(1024) uint8_t sm[8192];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    // (a) tcgen05.commit with no MMA in flight, then wait on it
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      tc_commit_el(&bar[0]);
      mbar_wait(&bar[0], r & 1);
    }
    unsigned long long t1 = clock64();
    // (b) plain arrive + wait (same thread)
    for (int r = 0; r < reps; ++r) {
      if (lane == 0) mbar_arrive(&bar[1]);
      __syncwarp();
      mbar_wait(&bar[1], r & 1);
    }
    unsigned long long t2 = clock64();
    // (c) one 128x128x16 MMA + commit + wait (issue-to-completion latency)
    for (int r = 0; r < reps; ++r) {
      mma_ss_f16_el(holder, umma_desc(smem_u32(sm), 16, 256, 6), umma_desc(smem_u32(sm + 4096), 16, 256, 6), idesc_f16(128, 128, 0, 0), 0);
      tc_commit_el(&bar[2]);
      mbar_wait(&bar[2], r & 1);
    }
    unsigned long long t3 = clock64();
    if (lane == 0 && blockIdx.x == 0) {
      out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; out[2] = (t3 - t2) / reps;
    }
  }
  // (d) cross-warp handoff: warp 1 arrives, warp 0 waits, ping-pong
  __syncthreads();
  if (warp < 2) {
    unsigned long long t4 = clock64();
    for (int r = 0; r < reps; ++r) {
      // warp 0 -> warp 1 on bar[3], warp 1 -> warp 0 on bar[4]
      if (warp == 0) {
        if (lane == 0) mbar_arrive(&bar[3]);
        __syncwarp();
        mbar_wait(&bar[4], r & 1);
      } else {
        mbar_wait(&bar[3], r & 1);
        if (lane == 0) mbar_arrive(&bar[4]);
        __syncwarp();
      }
    }
    unsigned long long t5 = clock64();
    if (warp == 0 && lane == 0 && blockIdx.x == 0) out[3] = (t5 - t4) / reps;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(holder, 512);
}

// cost of waiting on / probing an already-completed phase
__global__ void done_wait(int reps, unsigned long long* out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); mbar_arrive(&bar); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) mbar_wait(&bar, 0);
  unsigned long long t1 = clock64();
  int acc = 0;
  for (int r = 0; r < reps; ++r) acc += mbar_test(&bar, 0);
  unsigned long long t2 = clock64();
  uint32_t x = 0;
  for (int r = 0; r < reps; ++r) { mbar_wait(&bar, 0); x = x * 3 + r; }
  unsigned long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = (t1 - t0) / reps;
    out[blockIdx.x * 4 + 1] = (t2 - t1) / reps;
    out[blockIdx.x * 4 + 2] = acc + (x == 7);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  unsigned long long h[4];
  probe<<<1, 64>>>(1000, d);
  probe<<<148, 64>>>(1000, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("commit(no MMA)+wait: %llu cycles\narrive+wait same warp: %llu cycles\nMMA128x128x16+commit+wait: %llu cycles\n"
         "cross-warp round trip (2 handoffs): %llu cycles\n", h[0], h[1], h[2], h[3]);
  {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 4 * 148);
    unsigned long long h[4 * 148];
    for (int it = 0; it < 2; ++it) done_wait<<<148, 32>>>(256, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("completed phase: try_wait loop %llu cyc/wait, test_wait %llu cyc/probe\n", h[0], h[1]);
  }
  return 0;
}
