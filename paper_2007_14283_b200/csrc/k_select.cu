// k_select.cu -- K1 (normalise + quantise) and K6 (OSOP seed selection).
//
// K1: Eq. 1 / Eq. 9 -- every embedding is divided by its norm; the
//     unit vector is stored as two fixed-point limbs (integers held exactly in fp16, x ~= (hi +
//     lo 2^-11) 2^-11, |err| <= 2^-23) as the tensor-core operand (rows padded to DP, frames padded
//     to whole 128-pixel tiles with zero rows, which never enter a window since tau > 0).
// K6: Alg. 2 line 2 ("Evenly random select seed vector set"), reading R11: the K_r candidate
//     pixels with the smallest splitmix64 keys, in ascending pixel order.  Candidates are all pixels
//     in round 0 and the uncovered, unvisited pixels afterwards (north_star / R13).
//     Exact K-smallest selection without a sort of all n keys:
//       collect  -- every candidate whose key is below a threshold T sized for ~K + 4 sqrt(K) + 64
//                   survivors is appended to a per-frame sample (warp-aggregated atomics)
//       kth      -- one CTA per frame finds the K-th smallest sampled key by 8-bit MSD radix select
//                   (falls back to a radix select over all candidates if the sample was too small)
//       count / scan / write -- ordered stream compaction of {candidate, key <= kth} -> seeds
#include "fms_device.cuh"

namespace fms {

// ------------------------------------------------------------------------------------------------
__global__ void init_ctl_kernel(Params p) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.B) return;
  FrameCtl& c = p.ctl[f];
  memset(&c, 0, sizeof(FrameCtl));
  c.phase = PH_SELECT;
  c.I_prev = -1;
  for (int r = 0; r < kMaxRounds; ++r) c.round_nmin[r] = 0.0;
}

// Euclidean metric: per-frame max |x|^2 (float bits, non-negative: integer order = float order)
__global__ void maxnorm_kernel(Params p) {
  const int f = blockIdx.y;
  float m = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += (long long)gridDim.x * blockDim.x) {
    const float* x = emb_of(p) + ((size_t)f * p.n + i) * p.d;
    float ss = 0.f;
    for (int k = 0; k < p.d; ++k) ss = fmaf(x[k], x[k], ss);
    m = fmaxf(m, isfinite(ss) ? ss : INFINITY);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned*>(p.fscale) + f, __float_as_uint(m));
}
// max |x|^2 -> sigma = 2^-e with sqrt(max) < 2^e (power of two: scaling is exact)
__global__ void scale_kernel(Params p) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.B) return;
  const float m2 = p.fscale[f];
  if (!isfinite(m2)) { p.ctl[f].status = 3; p.fscale[f] = 1.f; return; }  // non-finite input
  int e = 0;
  frexpf(sqrtf(m2) * 1.0001f, &e);  // m < 2^e (the margin covers the fp32 rounding of the norm)
  p.fscale[f] = m2 > 0.f ? ldexpf(1.f, -e) : 1.f;
}

// digit planes of pixel i: byte (tile, plane, i % 128) of Xq, planes j*DP + k (k_iter8.cu's K-major
// weighted-sum operand); a warp writes 32 consecutive bytes of each plane
template <int DP>
__device__ __forceinline__ void store_digits(const Params& p, int f, long long i, const int8_t* q) {
  int8_t* base = p.Xq + ((size_t)f * p.n_ptiles + (size_t)(i >> 7)) * (3 * DP * kBN) + (i & 127);
#pragma unroll
  for (int r = 0; r < 3 * DP; ++r) base[(size_t)r * kBN] = q[r];
}

template <int DP>
__global__ void prep_euclid_kernel(Params p) {
  const int f = blockIdx.y;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_pad) return;
  __align__(16) __half h[DP];
  __align__(16) __half l[DP];
  int8_t q[3 * DP];  // digit planes a | b | c of v = round(2^22 x) (k_iter8.cu)
  if (i < p.n) {
    const float sg = p.fscale[f];
    const float* x = emb_of(p) + ((size_t)f * p.n + i) * p.d;
    float v[DP];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      v[k] = k < p.d ? x[k] * sg : 0.f;
      ss = fmaf(v[k], v[k], ss);
    }
    v[p.d] = -0.5f * ss;
    v[p.d + 1] = 1.f;
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      limbs(v[k], h[k], l[k]);
      digits(v[k], q[k], q[DP + k], q[2 * DP + k]);
    }
    p.inv[(size_t)f * p.n + i] = sg;  // seeds start at sigma x_i (select)
    p.flags[flag_at(p, f, i)] = 0;
  } else {
#pragma unroll
    for (int k = 0; k < DP; ++k) h[k] = l[k] = __float2half_rn(0.f);
#pragma unroll
    for (int k = 0; k < 3 * DP; ++k) q[k] = 0;
  }
  uint4* dst = reinterpret_cast<uint4*>(p.Xh + ((size_t)f * p.n_pad + i) * DP);
  uint4* dstl = reinterpret_cast<uint4*>(p.Xl + ((size_t)f * p.n_pad + i) * DP);
#pragma unroll
  for (int k = 0; k < DP / 8; ++k) {
    dst[k] = reinterpret_cast<const uint4*>(h)[k];
    dstl[k] = reinterpret_cast<const uint4*>(l)[k];
  }
  store_digits<DP>(p, f, i, q);
}

template <int DP>
__global__ void prep_kernel(Params p) {
  const int f = blockIdx.y;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_pad) return;
  __align__(16) __half h[DP];
  __align__(16) __half l[DP];
  int8_t q[3 * DP];  // digit planes a | b | c of v = round(2^22 x) (k_iter8.cu)
  if (i < p.n) {
    const float* x = emb_of(p) + ((size_t)f * p.n + i) * p.d;
    float v[DP];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      v[k] = k < p.d ? x[k] : 0.f;
      ss = fmaf(v[k], v[k], ss);
    }
    const float nrm = sqrtf(ss);
    float inv = 0.f;
    if (!(nrm > 0.f) || !isfinite(nrm)) {
      atomicExch(&p.ctl[f].status, 3 /*FMS_E_ZERO_NORM*/);
    } else {
      inv = 1.0f / nrm;
    }
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      limbs(v[k] * inv, h[k], l[k]);
      digits(v[k] * inv, q[k], q[DP + k], q[2 * DP + k]);
    }
    p.inv[(size_t)f * p.n + i] = inv;
    p.flags[flag_at(p, f, i)] = 0;
  } else {
#pragma unroll
    for (int k = 0; k < DP; ++k) h[k] = l[k] = __float2half_rn(0.f);
#pragma unroll
    for (int k = 0; k < 3 * DP; ++k) q[k] = 0;
  }
  uint4* dst = reinterpret_cast<uint4*>(p.Xh + ((size_t)f * p.n_pad + i) * DP);
  uint4* dstl = reinterpret_cast<uint4*>(p.Xl + ((size_t)f * p.n_pad + i) * DP);
#pragma unroll
  for (int k = 0; k < DP / 8; ++k) {
    dst[k] = reinterpret_cast<const uint4*>(h)[k];
    dstl[k] = reinterpret_cast<const uint4*>(l)[k];
  }
  store_digits<DP>(p, f, i, q);
}

// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ bool is_candidate(const Params& p, int f, int round, long long i) {
  if (round == 0) return true;
  return (p.flags[(size_t)f * p.n_glob + i] & (PF_VISITED | PF_COVERED)) == 0;  // i: global index
}

__global__ void sel_prepare_kernel(Params p) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.B) return;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT) return;
  if (c.status != 0) { c.phase = PH_ERROR; return; }
  long long ncand, Kreq;
  if (c.round == 0) {
    ncand = p.n_glob;
    Kreq = p.kind == 2 /*ALL*/ ? p.n_glob : (long long)p.n_seeds;
  } else {
    ncand = c.ncand;
    Kreq = c.K_next;
  }
  long long K = Kreq < ncand ? Kreq : ncand;
  if (K > p.S_cap) { c.status = 9 /*FMS_E_INTERNAL: seed capacity*/; c.phase = PH_ERROR; return; }
  c.K_r = (int)K;
  c.sample_count = 0;
  c.kth = ~0ull;
  if (K >= ncand) {
    c.take_all = 1;
    c.thresh = ~0ull;
  } else {
    c.take_all = 0;
    double frac = ((double)K + 4.0 * sqrt((double)K) + 64.0) / (double)ncand;
    c.thresh = frac >= 1.0 ? ~0ull : (unsigned long long)(frac * 18446744073709551616.0);
  }
}

__global__ void sel_collect_kernel(Params p) {
  const int f = blockIdx.y;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT || c.take_all) return;
  const int round = c.round;
  const unsigned long long T = c.thresh;
  const int lane = threadIdx.x & 31;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < p.n_glob; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    bool take = false;
    unsigned long long key = 0;
    if (i < p.n_glob && is_candidate(p, f, round, i)) {
      key = sel_key(p.rng_seed, round, i);
      take = key < T;
    }
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (m) {
      long long base = 0;
      if (lane == 0) base = (long long)atomicAdd((unsigned long long*)&c.sample_count, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (take) {
        long long pos = base + __popc(m & ((1u << lane) - 1));
        if (pos < p.sample_cap) p.sample[(size_t)f * p.sample_cap + pos] = key;
      }
    }
  }
}

// K-th smallest (1-based) key by MSD radix select, 8 bits per pass.  from_sample selects the key
// source: the sample buffer, or (fallback) every candidate pixel recomputed on the fly.
__device__ unsigned long long radix_kth(const Params& p, int f, int round, bool from_sample, long long count,
                                        long long k) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_k;
  if (threadIdx.x == 0) { s_prefix = 0; s_k = k; }
  unsigned long long mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    for (long long idx = threadIdx.x; idx < count; idx += blockDim.x) {
      unsigned long long key;
      if (from_sample) {
        key = p.sample[(size_t)f * p.sample_cap + idx];
      } else {
        if (!is_candidate(p, f, round, idx)) continue;
        key = sel_key(p.rng_seed, round, idx);
      }
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
    }
    __syncthreads();
    // the bin holding the k-th key: warp 0 scans the 256 bins (8 per lane) instead of one thread
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      unsigned int h8[8];
      unsigned long long part = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) { h8[u] = hist[l * 8 + u]; part += h8[u]; }
      unsigned long long incl = part;  // inclusive prefix of the lanes' 8-bin partial sums
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
      }
      const long long k0 = s_k;
      const unsigned long long excl = incl - part;
      const bool mine = (long long)excl < k0 && (long long)incl >= k0;  // exactly one lane
      if (mine) {
        long long cum = (long long)excl;
        for (int u = 0; u < 8; ++u) {
          if (cum + h8[u] >= k0) {
            s_prefix |= (unsigned long long)(l * 8 + u) << shift;
            s_k = k0 - cum;
            break;
          }
          cum += h8[u];
        }
      }
    }
    mask |= 0xFFull << shift;
    __syncthreads();
  }
  return s_prefix;
}

__global__ void sel_kth_kernel(Params p) {
  const int f = blockIdx.x;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT || c.take_all) return;
  const long long M = c.sample_count;
  const long long K = c.K_r;
  unsigned long long kth;
  if (M >= K && M <= p.sample_cap) {
    kth = radix_kth(p, f, c.round, true, M, K);
  } else {
    kth = radix_kth(p, f, c.round, false, p.n_glob, K);  // rare: sample too small / overflowed
  }
  if (threadIdx.x == 0) c.kth = kth;
}

constexpr int kSelBlock = 2048;  // pixels per block in count/write (256 threads x 8)

__device__ __forceinline__ bool is_selected(const Params& p, int f, const FrameCtl& c, long long i) {
  if (!is_candidate(p, f, c.round, i)) return false;
  if (c.take_all) return true;
  return sel_key(p.rng_seed, c.round, i) <= c.kth;
}

__global__ void sel_count_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT) return;
  const long long base = (long long)blockIdx.x * kSelBlock;
  int cnt = 0;
  for (int u = 0; u < kSelBlock / 256; ++u) {
    long long i = base + u * 256 + threadIdx.x;
    if (i < p.n_glob && is_selected(p, f, c, i)) ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 8; ++w) s += ws[w];
    p.blkcnt[(size_t)f * p.nblk_glob + blockIdx.x] = s;
  }
}

__global__ void sel_scan_kernel(Params p) {
  const int f = blockIdx.x;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT) return;
  __shared__ int sm[33];
  int carry = 0;
  for (int b0 = 0; b0 < p.nblk_glob; b0 += blockDim.x) {
    int b = b0 + threadIdx.x;
    int v = b < p.nblk_glob ? p.blkcnt[(size_t)f * p.nblk_glob + b] : 0;
    int tot;
    int ex = block_excl_scan(v, sm, &tot);
    if (b < p.nblk_glob) p.blkcnt[(size_t)f * p.nblk_glob + b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && carry != c.K_r) {
    c.status = 9;  // internal: selection count mismatch
    c.phase = PH_ERROR;
  }
}

template <int DP>
__global__ void sel_write_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT) return;
  __shared__ int sm[33];
  const long long base = (long long)blockIdx.x * kSelBlock + (long long)threadIdx.x * 8;
  unsigned sel = 0;
  for (int u = 0; u < 8; ++u) {
    long long i = base + u;
    if (i < p.n_glob && is_selected(p, f, c, i)) sel |= 1u << u;
  }
  int pos = p.blkcnt[(size_t)f * p.nblk_glob + blockIdx.x] + block_excl_scan(__popc(sel), sm, nullptr);
  for (int u = 0; u < 8; ++u) {
    if (!(sel & (1u << u))) continue;
    const long long i = base + u;
    const size_t so = (size_t)f * p.S_cap + pos;
    // pixel sharding: only the rank holding pixel i has its embedding; the others write a zero row
    // and the seed rows are summed over the ranks before the round iterates (k_shard.cu)
    const long long il = i - p.pix_off;
    const bool have = il >= 0 && il < p.n;
    const float inv = have ? p.inv[(size_t)f * p.n + il] : 0.f;
    const float* x = emb_of(p) + ((size_t)f * p.n + (have ? il : 0)) * p.d;
    float* s = p.seeds + so * DP;
    // the operand row (and accumulators) of an active seed sit at its compacted position; with seed
    // sharding only this rank's seeds (j % world == rank) are active here, at j / world
    const bool own = pos % p.world == p.rank;
    const int lp = pos / p.world;
    __align__(16) __half sh[DP], ss[DP], sl[DP];
    float sv[DP], row[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      sv[k] = (have && k < p.d) ? x[k] * inv : 0.f;
      s[k] = sv[k];
    }
    operand_row<DP>(p, f, sv, row);
#pragma unroll
    for (int k = 0; k < DP; ++k) split_seed(row[k], sh[k], ss[k], sl[k]);
    if (own) {
      const size_t ro = (size_t)f * p.S_pad + lp;
#pragma unroll
      for (int k = 0; k < DP / 8; ++k) {
        reinterpret_cast<uint4*>(p.sop + ro * DP)[k] = reinterpret_cast<const uint4*>(sh)[k];
        reinterpret_cast<uint4*>(p.sops + ro * DP)[k] = reinterpret_cast<const uint4*>(ss)[k];
        reinterpret_cast<uint4*>(p.sopl + ro * DP)[k] = reinterpret_cast<const uint4*>(sl)[k];
      }
      double* g = p.gacc + ro * DP;
#pragma unroll
      for (int k = 0; k < DP; ++k) g[k] = 0.0;
      p.cacc[ro] = 0;
      p.act[(size_t)f * p.S_cap + lp] = pos;
    }
    p.sorig[so] = (int)i;
    p.sstat[so] = ST_ACTIVE;
    p.scnt[so] = 0;
    p.flags[(size_t)f * p.n_glob + i] |= PF_VISITED;
    ++pos;
  }
}

__global__ void sel_finish_kernel(Params p) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p.B) return;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_SELECT) return;
  const int K = c.K_r;
  c.phase = PH_ITERATE;
  c.t = 0;
  const int mine = K > p.rank ? (K - 1 - p.rank) / p.world + 1 : 0;  // seeds this rank iterates
  c.n_active = mine;
  c.n_conv = 0;
  const double g = p.kind == 2 ? 1.0 : p.gamma;
  double need = ceil(g * (double)K - 1e-9);
  c.need = need < 0 ? 0 : (int)need;
  c.total += K;
  c.round_K[c.round] = K;
  c.round_seed_iters[c.round] = 0;
  if (K == 0) { c.phase = PH_POST; }
  // rows [K, roundup(K, 128)) of the last seed tile are computed too; start them at zero
  const int kpad = (mine + kBM - 1) / kBM * kBM;
  for (int r = mine; r < kpad && r < p.S_pad; ++r) {
    double* g = p.gacc + ((size_t)f * p.S_pad + r) * p.DP;
    for (int k = 0; k < p.DP; ++k) g[k] = 0.0;
    p.cacc[(size_t)f * p.S_pad + r] = 0;
  }
}

// ------------------------------------------------------------------------------------------------
cudaError_t launch_prep(const Params& p, cudaStream_t st) {
  init_ctl_kernel<<<(p.B + 127) / 128, 128, 0, st>>>(p);
  dim3 g((unsigned)((p.n_pad + 255) / 256), p.B);
  if (p.metric == 1) {
    cudaMemsetAsync(p.fscale, 0, (size_t)p.B * 4, st);
    maxnorm_kernel<<<dim3(64, p.B), 256, 0, st>>>(p);
    scale_kernel<<<(p.B + 127) / 128, 128, 0, st>>>(p);
    if (p.DP == 16) prep_euclid_kernel<16><<<g, 256, 0, st>>>(p);
    else prep_euclid_kernel<32><<<g, 256, 0, st>>>(p);
    return cudaGetLastError();
  }
  if (p.DP == 16) prep_kernel<16><<<g, 256, 0, st>>>(p);
  else prep_kernel<32><<<g, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_select(const Params& p, int num_sms, cudaStream_t st) {
  sel_prepare_kernel<<<(p.B + 127) / 128, 128, 0, st>>>(p);
  int gx = (int)((p.n_glob + 255) / 256);
  int cap = (num_sms * 8 + p.B - 1) / p.B;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  sel_collect_kernel<<<dim3(gx, p.B), 256, 0, st>>>(p);
  sel_kth_kernel<<<p.B, 1024, 0, st>>>(p);
  sel_count_kernel<<<dim3(p.nblk_glob, p.B), 256, 0, st>>>(p);
  sel_scan_kernel<<<p.B, 1024, 0, st>>>(p);
  if (p.DP == 16) sel_write_kernel<16><<<dim3(p.nblk_glob, p.B), 256, 0, st>>>(p);
  else sel_write_kernel<32><<<dim3(p.nblk_glob, p.B), 256, 0, st>>>(p);
  sel_finish_kernel<<<(p.B + 127) / 128, 128, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace fms
