// k_shard.cu -- pixel sharding: one frame's pixels split over ranks.
//
// Rank g holds the pixels [pix_off, pix_off + n) of every frame of n_glob pixels.  Seeds, centres
// and the OSOP control block are replicated, so every data-dependent decision is taken identically
// on every rank; the only distributed quantities are sums over pixels, and those are exchanged as
// int32 sums (the caller's collective, fms_set_pixel_shard):
//
//   after K1       status (a zero-norm row on any rank fails the frame everywhere)
//   after K6       the round's seed rows: the rank holding seed pixel i writes x_i / |x_i|, the
//                  others zero, so the sum is the owner's fp32 bits
//   after K2       every lockstep step (Alg. 2 l.4-9): the window sums G = sum_{W(s)} x
//                  and counts.  K2's G is exact -- an fp64 sum of integers 2^11 hi + lo (the limbs),
//                  |G 2^11| < 2^53 -- so it travels as an int64 split into a signed high part
//                  (G >> 24) and a 24-bit low part; the ranks' sums are exact and the summed G is
//                  bit-identical to the unsharded G.  K3 (renormalise, converge) then runs
//                  replicated.
//   after K5       the label histogram (I and r of Eq. 19 need global cluster sizes), the count of
//                  uncovered unvisited pixels and the coverage bits of the owned pixels (one bit per
//                  pixel; ranges are disjoint, so the integer sum of the words is their OR) -- the
//                  next round's candidates (R13) are selected over the global pixel range.
#include <algorithm>

#include "fms_device.cuh"

namespace fms {

__device__ __forceinline__ bool pst_stepping(const FrameCtl& c) {
  return (c.phase == PH_ITERATE || c.phase == PH_COUNT) && c.n_active > 0;
}

// ---- status after K1 ----
__global__ void pstat_kernel(Params p, bool pack) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < p.B; f += gridDim.x * blockDim.x) {
    if (pack) p.pbuf[f] = p.ctl[f].status != 0 ? 1 : 0;
    else if (p.pbuf[f] != 0) p.ctl[f].status = 3;  // FMS_E_ZERO_NORM on some rank
  }
}

// ---- after K6: largest K_r of the frames about to iterate -> counters[8] ----
__global__ void psel_kmax_kernel(Params p) {
  __shared__ int m;
  if (threadIdx.x == 0) m = 0;
  __syncthreads();
  for (int f = threadIdx.x; f < p.B; f += blockDim.x)
    if (p.ctl[f].phase == PH_ITERATE) atomicMax(&m, p.ctl[f].K_r);
  __syncthreads();
  if (threadIdx.x == 0) p.counters[8] = m;
}

// seed rows [B][pkmax][DP] (fp32 bits; zero rows from ranks that do not hold the seed pixel)
template <int DP>
__global__ void psel_pack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  const int K = c.phase == PH_ITERATE ? c.K_r : 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < p.pkmax * DP; t += gridDim.x * blockDim.x) {
    const int j = t / DP;
    p.pbuf[(size_t)f * p.pkmax * DP + t] =
        j < K ? __float_as_int(p.seeds[((size_t)f * p.S_cap) * DP + t]) : 0;
  }
}
// summed rows -> master seeds and their fp16 operand rows (seed j sits at compacted row j)
template <int DP>
__global__ void psel_unpack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  if (c.phase != PH_ITERATE) return;
  const int K = c.K_r;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x) {
    const int* row = p.pbuf + ((size_t)f * p.pkmax + j) * DP;
    float* s = p.seeds + ((size_t)f * p.S_cap + j) * DP;
    __align__(16) __half sh[DP], ss[DP], sl[DP];
    float sv[DP], orow[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      sv[k] = __int_as_float(row[k]);
      s[k] = sv[k];
    }
    operand_row<DP>(p, f, sv, orow);
#pragma unroll
    for (int k = 0; k < DP; ++k) split_seed(orow[k], sh[k], ss[k], sl[k]);
    const size_t ro = (size_t)f * p.S_pad + j;
#pragma unroll
    for (int k = 0; k < DP / 8; ++k) {
      reinterpret_cast<uint4*>(p.sop + ro * DP)[k] = reinterpret_cast<const uint4*>(sh)[k];
      reinterpret_cast<uint4*>(p.sops + ro * DP)[k] = reinterpret_cast<const uint4*>(ss)[k];
      reinterpret_cast<uint4*>(p.sopl + ro * DP)[k] = reinterpret_cast<const uint4*>(sl)[k];
    }
  }
}

// ---- after K2, every step: G (an exact integer: sum of round(2^22 x), k_iter8.cu) as (hi = v >> 24,
//      lo = v & 0xFFFFFF), count ----
template <int DP>
__global__ void pstep_pack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  const int rows = pst_stepping(c) ? min(c.n_active, p.pkmax) : 0;
  constexpr int W = 2 * DP + 1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < p.pkmax * W; t += gridDim.x * blockDim.x) {
    const int j = t / W, k = t - j * W;
    int v = 0;
    if (j < rows) {
      const size_t r = (size_t)f * p.S_pad + j;
      if (k < 2 * DP) {
        const long long g = (long long)p.gacc[r * DP + (k >> 1)];  // exact integer
        v = (k & 1) ? (int)(g & 0xFFFFFF) : (int)(g >> 24);
      } else {
        v = p.cacc[r];
      }
    }
    p.pbuf[(size_t)f * p.pkmax * W + t] = v;
  }
}
template <int DP>
__global__ void pstep_unpack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  if (!pst_stepping(c)) return;
  const int rows = min(c.n_active, p.pkmax);
  constexpr int W = 2 * DP + 1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < rows * (DP + 1); t += gridDim.x * blockDim.x) {
    const int j = t / (DP + 1), k = t - j * (DP + 1);
    const int* row = p.pbuf + ((size_t)f * p.pkmax + j) * W;
    const size_t r = (size_t)f * p.S_pad + j;
    if (k < DP) {
      const long long g = (long long)row[2 * k] * 16777216ll + (long long)row[2 * k + 1];
      p.gacc[r * DP + k] = (double)g;
    } else {
      p.cacc[r] = row[2 * DP];
    }
  }
}

// ---- after K5: [B][C_cap + 2 + pcov_words]: histogram, candidate count (hi, lo), coverage bits ----
__global__ void ppost_pack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  const bool post = c.phase == PH_POST;
  const size_t W = (size_t)p.C_cap + 2 + p.pcov_words;
  int* row = p.pbuf + (size_t)f * W;
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = t0; k < p.C_cap; k += stride) row[k] = (post && k < c.Kc) ? p.hist[(size_t)f * p.C_cap + k] : 0;
  if (t0 == 0) {
    row[p.C_cap] = post ? (int)(c.ncand >> 24) : 0;
    row[p.C_cap + 1] = post ? (int)(c.ncand & 0xFFFFFF) : 0;
  }
  const long long lo = p.pix_off, hi = p.pix_off + p.n;
  for (int w = t0; w < p.pcov_words; w += stride) {
    unsigned bits = 0;
    if (post) {
      for (int b = 0; b < 32; ++b) {
        const long long i = (long long)w * 32 + b;
        if (i >= lo && i < hi && (p.flags[(size_t)f * p.n_glob + i] & PF_COVERED)) bits |= 1u << b;
      }
    }
    row[p.C_cap + 2 + w] = (int)bits;
  }
}
__global__ void ppost_unpack_kernel(Params p) {
  const int f = blockIdx.y;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_POST) return;
  const size_t W = (size_t)p.C_cap + 2 + p.pcov_words;
  const int* row = p.pbuf + (size_t)f * W;
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = t0; k < c.Kc; k += stride) p.hist[(size_t)f * p.C_cap + k] = row[k];
  for (long long i = t0; i < p.n_glob; i += stride) {
    const unsigned bits = (unsigned)row[p.C_cap + 2 + (i >> 5)];
    uint8_t* fl = p.flags + (size_t)f * p.n_glob + i;
    *fl = (uint8_t)((*fl & ~PF_COVERED) | (((bits >> (i & 31)) & 1u) ? PF_COVERED : 0));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    c.ncand = (long long)row[p.C_cap] * 16777216ll + (long long)row[p.C_cap + 1];
}

// ---- launches ----
cudaError_t launch_pstat(const Params& p, bool pack, cudaStream_t st) {
  pstat_kernel<<<1, 256, 0, st>>>(p, pack);
  return cudaGetLastError();
}
cudaError_t launch_psel_kmax(const Params& p, cudaStream_t st) {
  psel_kmax_kernel<<<1, 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_psel(const Params& p, bool pack, cudaStream_t st) {
  const dim3 g((unsigned)std::max(1, std::min(64, (p.pkmax * p.DP + 255) / 256)), p.B);
  if (p.DP == 16) {
    if (pack) psel_pack_kernel<16><<<g, 256, 0, st>>>(p);
    else psel_unpack_kernel<16><<<g, 256, 0, st>>>(p);
  } else {
    if (pack) psel_pack_kernel<32><<<g, 256, 0, st>>>(p);
    else psel_unpack_kernel<32><<<g, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}
cudaError_t launch_pstep(const Params& p, bool pack, cudaStream_t st) {
  const dim3 g((unsigned)std::max(1, std::min(64, (p.pkmax * (2 * p.DP + 1) + 255) / 256)), p.B);
  if (p.DP == 16) {
    if (pack) pstep_pack_kernel<16><<<g, 256, 0, st>>>(p);
    else pstep_unpack_kernel<16><<<g, 256, 0, st>>>(p);
  } else {
    if (pack) pstep_pack_kernel<32><<<g, 256, 0, st>>>(p);
    else pstep_unpack_kernel<32><<<g, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}
cudaError_t launch_ppost(const Params& p, bool pack, cudaStream_t st) {
  const long long work = std::max<long long>(p.C_cap, pack ? p.pcov_words : p.n_glob);
  const dim3 g((unsigned)std::max<long long>(1, std::min<long long>(256, (work + 255) / 256)), p.B);
  if (pack) ppost_pack_kernel<<<g, 256, 0, st>>>(p);
  else ppost_unpack_kernel<<<g, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace fms
