// k_post.cu -- per-round post-processing: K4 merge, K5 assignment + coverage, K7 OSOP control.
//
// K4 ("modes are further pruned and merged if their distance is small"; reading R10):
//     pool = previous centres U this round's converged modes; order by (intensity desc, origin asc);
//     greedy: keep a mode unless a kept centre lies within cosine distance rho = h.  Kept modes are
//     not averaged.  One CTA per frame: bitonic sort of the pool keys in SMEM, then the greedy scan in
//     batches of 32 candidates (all kept-vs-candidate tests of a batch in parallel, the in-batch
//     chain resolved by one warp with ballots).
// K5 (Alg. 2 l.12-14): label = argmax_k x.c_k (lowest k on ties, R21); covered =
//     max_k x_hat.c_k >= tau; per-centre histogram; count of uncovered & unvisited pixels.
//     Frames with <= 128 centres run on the tensor cores (k_assign.cu); this fp32 CUDA-core scan
//     of the input covers frames with more centres.
// K7 (Eq. 12-19; readings R12-R15, R22): background = largest cluster,
//     I = #other clusters with >= min_instance_px pixels, r = 1 - |bg|/n,
//     N_min = ceil( ln(1 - e^{ln P / I}) / ln(1 - r/I) ); stop when coverage holds
//     (no candidates / total >= L N_min / total >= n / max_rounds / saturation), else double N.
#include <cub/device/device_segmented_radix_sort.cuh>

#include "fms_device.cuh"

namespace fms {

template <int DP>
__device__ __forceinline__ float dotv(const float* a, const float* b) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < DP; ++k) s = fmaf(a[k], b[k], s);
  return s;
}

constexpr int kKeptSm = 256;    // kept centres cached in SMEM during the greedy scan
constexpr int kMergeSm = 8192;  // pools up to this size are sorted in SMEM

// 1. assemble the pool (previous centres, then this round's converged seeds in seed order) and its
//    sort keys (intensity desc, origin asc); returns P (or -1 after flagging a capacity error)
template <int DP>
__device__ int merge_assemble(const Params& p, int f, unsigned long long* keys, int* vals, int P2, int* sm) {
  FrameCtl& c = p.ctl[f];
  const int Kc = c.Kc;
  const int K = c.K_r;
  const int P = Kc + c.n_conv;
  if (P > p.P_cap) {
    if (threadIdx.x == 0) { c.status = 9; c.phase = PH_ERROR; }  // FMS_E_INTERNAL: pool capacity
    return -1;
  }
  float* pool = p.pool + (size_t)f * p.P_cap * DP;
  int* pint = p.pint + (size_t)f * p.P_cap;
  int* porg = p.porg + (size_t)f * p.P_cap;
  const float* cent = p.cent + (size_t)f * p.C_cap * DP;
  for (int k = threadIdx.x; k < Kc; k += blockDim.x) {
    for (int q = 0; q < DP; ++q) pool[(size_t)k * DP + q] = cent[(size_t)k * DP + q];
    pint[k] = p.cint[(size_t)f * p.C_cap + k];
    porg[k] = p.corig[(size_t)f * p.C_cap + k];
  }
  const size_t sb = (size_t)f * p.S_cap;
  int carry = Kc;
  for (int j0 = 0; j0 < K; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    const int a = (j < K && p.sstat[sb + j] == ST_CONV) ? 1 : 0;
    int tot;
    const int pos = carry + block_excl_scan(a, sm, &tot);
    if (a) {
      for (int q = 0; q < DP; ++q) pool[(size_t)pos * DP + q] = p.seeds[(sb + j) * DP + q];
      pint[pos] = p.scnt[sb + j];
      porg[pos] = p.sorig[sb + j];
    }
    carry += tot;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P2; i += blockDim.x) {
    if (i < P) {
      keys[i] = ((unsigned long long)(0x7FFFFFFFu - (unsigned)pint[i]) << 32) | (unsigned)porg[i];
      vals[i] = i;
    } else {
      keys[i] = ~0ull;
      vals[i] = -1;
    }
  }
  __syncthreads();
  return P;
}

// 3. greedy NMS in sorted order, in batches of 32; batch candidates and the first kKeptSm kept
//    centres live in SMEM, so the serial in-batch chain never waits on global memory
template <int DP>
__device__ void merge_nms(const Params& p, int f, const int* vals, int P, float* cand, float* keptv) {
  static_assert(32 * DP <= 1024, "one prefetched candidate value per thread of a 1024-thread CTA");
  FrameCtl& c = p.ctl[f];
  __shared__ unsigned s_supp;
  __shared__ unsigned s_inb[32];  // in-batch conflicts: bit j of s_inb[i] = candidate j (< i) within rho
  __shared__ int s_kept, s_err;
  const float* pool = p.pool + (size_t)f * p.P_cap * DP;
  const int* pint = p.pint + (size_t)f * p.P_cap;
  const int* porg = p.porg + (size_t)f * p.P_cap;
  float* cent = p.cent + (size_t)f * p.C_cap * DP;
  const float thr = p.rho_f;  // keep unless x.c >= 1 - rho
  // Euclidean (R24): keep unless |m - c| <= rho = h, in the frame's scaled units
  const float rho2 = p.metric == 1 ? (float)((double)p.fscale[f] * p.h * (double)p.fscale[f] * p.h) : 0.f;
  auto close = [&](const float* a, const float* b) -> bool {
    if (p.metric != 1) return dotv<DP>(a, b) >= thr;
    float d2 = 0.f;
#pragma unroll
    for (int k = 0; k < DP; ++k) d2 = fmaf(a[k] - b[k], a[k] - b[k], d2);
    return d2 <= rho2;
  };
  if (threadIdx.x == 0) { s_kept = 0; s_err = 0; }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // a batch's candidates (32 x DP floats, one per thread: blockDim >= 32 DP) are fetched during the
  // previous batch, so no batch starts on a dependent global load
  const int t = threadIdx.x;
  auto fetch = [&](int b0) -> float {
    const int nbb = min(32, P - b0);
    if (b0 >= P || t >= nbb * DP) return 0.f;
    const int ci = t / DP, q = t - ci * DP;
    return pool[(size_t)vals[b0 + ci] * DP + q];
  };
  float cur = fetch(0);
  for (int base = 0; base < P; base += 32) {
    const int nb = min(32, P - base);
    if (threadIdx.x == 0) s_supp = 0;
    if (threadIdx.x < 32) s_inb[threadIdx.x] = 0;
    if (t < nb * DP) cand[t] = cur;
    __syncthreads();
    cur = fetch(base + 32);  // the next batch, in flight while this one is compared
    const int kept = s_kept;
    const int total = nb * kept;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int ci = idx / kept, k = idx - ci * kept;
      const float* kv = k < kKeptSm ? keptv + k * DP : cent + (size_t)k * DP;
      if (close(cand + ci * DP, kv)) atomicOr(&s_supp, 1u << ci);
    }
    // all in-batch pairs (i, j < i) at once, one per thread, instead of a serial loop per lane
    for (int idx = threadIdx.x; idx < 32 * 32; idx += blockDim.x) {
      const int i = idx >> 5, j = idx & 31;
      if (i < nb && j < i && close(cand + i * DP, cand + j * DP)) atomicOr(&s_inb[i], 1u << j);
    }
    __syncthreads();
    if (warp == 0) {
      const float* a = cand + (lane < nb ? lane : 0) * DP;
      const unsigned inb = lane < nb ? s_inb[lane] : 0u;
      const unsigned supp = s_supp;
      unsigned keep = 0;
      for (int i = 0; i < nb; ++i) {
        const int ok = (lane == i) && !((supp >> i) & 1u) && !(inb & keep);
        if (__ballot_sync(0xffffffffu, ok)) keep |= 1u << i;
      }
      if (lane < nb && ((keep >> lane) & 1u)) {
        const int pos = kept + __popc(keep & ((1u << lane) - 1u));
        if (pos < p.C_cap) {
          for (int q = 0; q < DP; ++q) {
            cent[(size_t)pos * DP + q] = a[q];
            if (pos < kKeptSm) keptv[pos * DP + q] = a[q];
          }
          p.cint[(size_t)f * p.C_cap + pos] = pint[vals[base + lane]];
          p.corig[(size_t)f * p.C_cap + pos] = porg[vals[base + lane]];
        } else {
          s_err = 1;
        }
      }
      if (lane == 0) s_kept = kept + __popc(keep);
    }
    __syncthreads();
  }
  const int Kn = s_kept;
  for (int k = threadIdx.x; k < Kn && k < p.C_cap; k += blockDim.x) p.hist[(size_t)f * p.C_cap + k] = 0;
  if (threadIdx.x == 0) {
    atomicMax(&p.counters[19], Kn);  // the largest K of the round: which assignment kernels have work
    if (s_err) { c.status = 9; c.phase = PH_ERROR; }  // FMS_E_INTERNAL: centre capacity C_cap
    c.Kc = Kn < p.C_cap ? Kn : p.C_cap;
    c.ncand = 0;
  }
}

// pools up to kMergeSm: one CTA per frame, bitonic sort of the keys in SMEM (larger pools are left
// to the global-memory path below)
template <int DP>
__global__ void __launch_bounds__(1024) merge_kernel(Params p) {
  const int f = blockIdx.x;
  if (p.ctl[f].phase != PH_POST || p.ctl[f].Kc + p.ctl[f].n_conv > kMergeSm) return;
  extern __shared__ uint8_t dsm[];
  __shared__ int sm[33];
  int P2 = 1;
  while (P2 < p.ctl[f].Kc + p.ctl[f].n_conv) P2 <<= 1;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(dsm);
  int* vals = reinterpret_cast<int*>(keys + P2);
  const int P = merge_assemble<DP>(p, f, keys, vals, P2, sm);
  if (P < 0) return;
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = keys[i], b = keys[ixj];
          if ((a > b) == up) {
            keys[i] = b; keys[ixj] = a;
            const int t = vals[i]; vals[i] = vals[ixj]; vals[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  float* cand = reinterpret_cast<float*>(vals + P2);  // [32][DP]
  merge_nms<DP>(p, f, vals, P, cand, cand + 32 * DP);
}

// larger pools (Alg. 1 merges a mode per pixel; late OSOP rounds of many-cell frames): keys in global
// memory, a CUB segmented radix sort between the two kernels.  Each frame's segment is [f P_cap,
// f P_cap + P) for a frame with P > kMergeSm and empty otherwise.
template <int DP>
__global__ void __launch_bounds__(1024) merge_pool_kernel(Params p) {
  const int f = blockIdx.x;
  const int P = p.ctl[f].Kc + p.ctl[f].n_conv;
  const bool big = p.ctl[f].phase == PH_POST && P > kMergeSm;
  if (threadIdx.x == 0) {
    p.moffs[f] = f * p.P_cap;
    p.moffs_end[f] = f * p.P_cap + (big ? P : 0);
  }
  if (!big) return;
  __shared__ int sm[33];
  const int Pa = merge_assemble<DP>(p, f, p.mkeys + (size_t)f * p.P_cap, p.mvals + (size_t)f * p.P_cap, P, sm);
  if (Pa < 0 && threadIdx.x == 0) p.moffs_end[f] = f * p.P_cap;  // capacity error flagged (phase ERROR)
}

template <int DP>
__global__ void __launch_bounds__(1024) merge_nms_kernel(Params p) {
  const int f = blockIdx.x;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_POST || c.Kc + c.n_conv <= kMergeSm) return;
  __shared__ float cand[32 * DP];
  __shared__ float keptv[kKeptSm * DP];
  merge_nms<DP>(p, f, p.mvals_sorted + (size_t)f * p.P_cap, c.Kc + c.n_conv, cand, keptv);
}

template <int DP>
__global__ void __launch_bounds__(256) assign_kernel(Params p) {
  constexpr int kAsgChunk = 8192 / DP;  // centres per SMEM chunk (32 KB)
  __shared__ float sc[kAsgChunk * DP];
  __shared__ int sh[kAsgChunk];
  __shared__ int s_cand;
  // grid (16, B): most frames go to assign_tc_kernel and their CTAs exit at once; the others are
  // covered by a block-stride loop over 256-pixel blocks
  const int f = blockIdx.y;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_POST || (c.Kc > 0 && c.Kc <= 256)) return;  // <= 256 centres: assign_tc_kernel
  const int nb = (int)((p.n + 255) / 256);
  for (int bid = blockIdx.x; bid < nb; bid += gridDim.x) {
  const int Kc = c.Kc;
  const long long i = (long long)bid * blockDim.x + threadIdx.x;
  const bool valid = i < p.n;
  float x[DP];
#pragma unroll
  for (int k = 0; k < DP; ++k) x[k] = 0.f;
  const bool euclid = p.metric == 1;
  const float sg = euclid ? p.fscale[f] : 1.f;
  if (valid) {
    const float* src = emb_of(p) + ((size_t)f * p.n + i) * p.d;
#pragma unroll
    for (int k = 0; k < DP; ++k)
      if (k < p.d) x[k] = src[k] * sg;
  }
  if (threadIdx.x == 0) s_cand = 0;
  float best = -INFINITY;
  int lab = 0;
  const float* cent = p.cent + (size_t)f * p.C_cap * DP;
  for (int k0 = 0; k0 < Kc; k0 += kAsgChunk) {
    const int nk = min(kAsgChunk, Kc - k0);
    __syncthreads();
    for (int t = threadIdx.x; t < nk * DP; t += blockDim.x) sc[t] = cent[(size_t)k0 * DP + t];
    __syncthreads();
    for (int k = 0; k < nk; ++k) {
      // Euclidean (R24): rank by x.c - |c|^2 / 2 = (|x|^2 - |x - c|^2) / 2
      const float dv = euclid ? dotv<DP>(x, sc + k * DP) - 0.5f * dotv<DP>(sc + k * DP, sc + k * DP)
                              : dotv<DP>(x, sc + k * DP);
      if (dv > best) { best = dv; lab = k0 + k; }
    }
  }
  // histogram of labels (SMEM per chunk of centres), coverage and candidate count
  int cand = 0;
  if (valid) {
    const size_t pi = (size_t)f * p.n + i;
    const double hs = (double)sg * p.h;
    const bool covered = euclid ? best >= 0.5f * (dotv<DP>(x, x) - (float)(hs * hs)) : best * p.inv[pi] >= p.tau_f;
    const uint8_t fl = p.flags[flag_at(p, f, i)];
    p.flags[flag_at(p, f, i)] = (uint8_t)((fl & ~PF_COVERED) | (covered ? PF_COVERED : 0));
    labels_of(p)[pi] = lab;
    cand = (!covered && !(fl & PF_VISITED)) ? 1 : 0;
  }
  for (int k0 = 0; k0 < Kc; k0 += kAsgChunk) {
    const int nk = min(kAsgChunk, Kc - k0);
    __syncthreads();
    for (int t = threadIdx.x; t < nk; t += blockDim.x) sh[t] = 0;
    __syncthreads();
    if (valid && lab >= k0 && lab < k0 + nk) atomicAdd(&sh[lab - k0], 1);
    __syncthreads();
    for (int t = threadIdx.x; t < nk; t += blockDim.x)
      if (sh[t]) atomicAdd(&p.hist[(size_t)f * p.C_cap + k0 + t], sh[t]);
  }
  cand = __syncthreads_count(cand);
  if (threadIdx.x == 0 && cand) atomicAdd((unsigned long long*)&c.ncand, (unsigned long long)cand);
  }
}

__global__ void osop_kernel(Params p) {
  __shared__ int sm[33];
  int not_done = 0;
  for (int f0 = 0; f0 < p.B; f0 += blockDim.x) {
    const int f = f0 + threadIdx.x;
    if (f < p.B) {
      FrameCtl& c = p.ctl[f];
      if (c.phase == PH_POST) {
        const int r = c.round;
        c.round_Kc[r] = c.Kc;
        c.round_cand[r] = c.ncand;
        if (p.kind != 1 /*OSOP*/) {
          c.phase = PH_DONE;
        } else {
          const int* hist = p.hist + (size_t)f * p.C_cap;
          int bg = -1;
          if (p.has_bg) {
            bg = 0;
            for (int k = 1; k < c.Kc; ++k)
              if (hist[k] > hist[bg]) bg = k;
          }
          int I = 0;
          for (int k = 0; k < c.Kc; ++k)
            if (k != bg && hist[k] >= p.min_px) ++I;
          const double rr = bg >= 0 ? 1.0 - (double)hist[bg] / (double)p.n_glob : 1.0;
          double nmin = -1.0;  // -1 = infinite (no instance observed)
          if (I > 0 && rr > 0.0) {
            const double q = rr / (double)I;
            if (q >= 1.0) {
              nmin = 1.0;
            } else {
              double v = ceil(log(-expm1(log(p.P) / (double)I)) / log1p(-q));
              nmin = v < 1.0 ? 1.0 : v;
            }
          }
          c.round_I[r] = I;
          c.round_r[r] = rr;
          c.round_nmin[r] = nmin;
          const bool stop = c.ncand == 0 || c.total >= p.n_glob || r + 1 >= p.max_rounds ||
                            (nmin > 0.0 && (double)c.total >= p.L * nmin) ||
                            (p.sat_stop && r >= 1 && I <= c.I_prev);
          c.I_prev = I;
          if (stop) {
            c.phase = PH_DONE;
          } else {
            c.K_next = c.total < c.ncand ? c.total : c.ncand;
            c.round = r + 1;
            c.phase = PH_SELECT;
          }
        }
      }
      if (c.phase == PH_SELECT || c.phase == PH_ITERATE || c.phase == PH_POST) not_done = 1;
    }
  }
  int tot;
  block_excl_scan(not_done, sm, &tot);
  if (threadIdx.x == 0) {
    p.counters[2] = tot;
    p.counters[18] = 0;  // largest merge pool of the next round (ctl_step)
    p.counters[19] = 0;  // largest K of the next round (merge)
  }
}

template <int DP>
__global__ void output_kernel(Params p, float* centres_out, int cap) {
  if (!centres_out) centres_out = p.io->centres;  // graph mode
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  const int Kc = c.Kc < cap ? c.Kc : cap;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < Kc * p.d; t += gridDim.x * blockDim.x) {
    const int k = t / p.d, q = t - k * p.d;
    // Euclidean: back to the caller's units (1 / sigma is a power of two: exact)
    centres_out[((size_t)f * cap + k) * p.d + q] =
        p.cent[((size_t)f * p.C_cap + k) * DP + q] * (p.metric == 1 ? 1.f / p.fscale[f] : 1.f);
  }
}

int merge_smem_bytes(int P_cap, int DP) {
  int P2 = 1;
  while (P2 < P_cap) P2 <<= 1;
  return P2 * 12 + (32 + kKeptSm) * DP * 4;
}

cudaError_t setup_post_attrs(int P_cap) {
  cudaError_t e = cudaFuncSetAttribute(merge_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       merge_smem_bytes(P_cap, 16));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(merge_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              merge_smem_bytes(P_cap, 32));
}

cudaError_t launch_assign_tc(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st);

size_t merge_sort_temp_bytes(const Params& p) {
  size_t bytes = 0;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr,
                                          (unsigned long long*)nullptr, (const int*)nullptr, (int*)nullptr,
                                          (int)((size_t)p.B * p.P_cap), p.B, (const int*)nullptr, (const int*)nullptr);
  return bytes;
}


cudaError_t launch_osop(const Params& p, cudaStream_t st) {
  osop_kernel<<<1, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

// merge, small pools (P <= kMergeSm, SMEM sort) -- every call
cudaError_t launch_merge_small(const Params& p, cudaStream_t st) {
  const int sm = merge_smem_bytes(p.P_cap < kMergeSm ? p.P_cap : kMergeSm, p.DP);
  if (p.DP == 16) merge_kernel<16><<<p.B, 1024, sm, st>>>(p);
  else merge_kernel<32><<<p.B, 1024, sm, st>>>(p);
  return cudaGetLastError();
}

// merge, large pools (global-memory sort) -- only when some frame's pool exceeds kMergeSm
// (counters[18], the largest pool of the round, set by ctl_step)
cudaError_t launch_merge_big(const Params& p, cudaStream_t st) {
  if (p.P_cap <= kMergeSm) return cudaSuccess;
  if (p.DP == 16) merge_pool_kernel<16><<<p.B, 1024, 0, st>>>(p);
  else merge_pool_kernel<32><<<p.B, 1024, 0, st>>>(p);
  size_t tb = p.msort_bytes;
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(p.msort_temp, tb, p.mkeys, p.mkeys_sorted, p.mvals,
                                                           p.mvals_sorted, (int)((size_t)p.B * p.P_cap), p.B,
                                                           p.moffs, p.moffs_end, 0, 64, st);
  if (e != cudaSuccess) return e;
  if (p.DP == 16) merge_nms_kernel<16><<<p.B, 1024, 0, st>>>(p);
  else merge_nms_kernel<32><<<p.B, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

// assignment (+ the OSOP step unless `osop` is false: pixel sharding sums the histogram over the
// ranks first)
cudaError_t launch_assign_osop(const Params& p, const TMaps& tm, int num_sms, cudaStream_t st, bool osop) {
  const dim3 ga(16, p.B);
  cudaError_t e = launch_assign_tc(p.DP, tm, p, num_sms, st);  // frames with <= 256 centres
  if (e != cudaSuccess) return e;
  if (p.DP == 16) assign_kernel<16><<<ga, 256, 0, st>>>(p);    // the rest
  else assign_kernel<32><<<ga, 256, 0, st>>>(p);
  if (osop) osop_kernel<<<1, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_output(const Params& p, float* centres_out, int cap, cudaStream_t st) {
  dim3 g(32, p.B);
  if (p.DP == 16) output_kernel<16><<<g, 256, 0, st>>>(p, centres_out, cap);
  else output_kernel<32><<<g, 256, 0, st>>>(p, centres_out, cap);
  return cudaGetLastError();
}

}  // namespace fms
