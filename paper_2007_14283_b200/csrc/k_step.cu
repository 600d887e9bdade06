// k_step.cu -- per-lockstep-step control around K2: work planning, K3 (reduce + renormalise +
// converge), and the per-frame early-stop / compaction step.
//
// K3 implements, for every active seed (R4, R6):
//     G = the exact windowed sum merged by K2 (fp64 accumulator, reset after reading)
//     s' = G / |G|                      (renormalised onto the unit sphere; the count cancels)
//     delta = |s' - s|_2,  converged if delta < tol = h/1000,  converged seeds freeze (R9)
//     window count 0 -> stalled (never happens for seeds started at pixels, pin P3)
// ctl_step applies early stopping (R8): once converged >= ceil(gamma*K_r) or no seed is
// active (or max_iter), the remaining active seeds are discarded and the converged modes get one
// count pass (their intensity |S_h(m)|, R10) before the merge phase; otherwise the active seeds
// are compacted (ascending seed index) into the fp16 hi/lo operand rows.
#include <algorithm>

#include "fms_device.cuh"

namespace fms {

// one CTA: prefix over frames -> tile-task table for this step.  Work item i is chunk
// (i mod n_chunks) of tile task (i div n_chunks).
// L2 load (bypasses L1): state another CTA of the same kernel may have written (post_step_kernel)
template <bool CG, typename T>
__device__ __forceinline__ T ldx(const T* ptr) {
  if constexpr (CG) return __ldcg(ptr);
  else return *ptr;
}

template <bool CG>
__device__ void plan_body(const Params& p, int* sm, int* s_tiles_total_p) {
  int& s_tiles_total = *s_tiles_total_p;
  int carry_t = 0;
  long long units = 0, count_units = 0;  // active seeds this step (A_t) and converged modes counted
  for (int f0 = 0; f0 < p.B; f0 += blockDim.x) {
    const int f = f0 + threadIdx.x;
    int nt = 0, u_it = 0, u_ct = 0;
    if (f < p.B) {
      const FrameCtl& c = p.ctl[f];
      const int ph = ldx<CG>(&c.phase), na = ldx<CG>(&c.n_active);
      if ((ph == PH_ITERATE || ph == PH_COUNT) && na > 0) {
        nt = (na + kBM - 1) / kBM;
        (ph == PH_ITERATE ? u_it : u_ct) = na;
      }
    }
    int ti, tc;
    block_excl_scan(u_it, sm, &ti);
    block_excl_scan(u_ct, sm, &tc);
    units += ti;
    count_units += tc;
    int tt;
    const int ot = block_excl_scan(nt, sm, &tt);
    if (f < p.B) {
      FrameCtl& c = p.ctl[f];
      c.tile_off = carry_t + ot;
      c.n_tiles_step = nt;
      c.tiles_done = 0;
      c.step_conv = 0;
      c.step_stall = 0;
    }
    carry_t += tt;
  }
  if (threadIdx.x == 0) s_tiles_total = carry_t;
  __syncthreads();
  if (s_tiles_total > p.tiles_cap) {
    if (threadIdx.x == 0) { p.counters[0] = 0; p.counters[1] = 0; p.counters[5] = 1; }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int f = warp; f < p.B; f += nw) {
    const FrameCtl& c = p.ctl[f];
    const int nt = c.n_tiles_step;
    const int mode = ldx<CG>(&c.phase) == PH_COUNT ? 1 : 0;
    for (int tile = lane; tile < nt; tile += 32) p.tiles[c.tile_off + tile] = TileTask{f, tile, 0, 0, mode, 0, 0, 0};
  }
  if (threadIdx.x == 0) {
    // work items: chunks of ct pixel tiles per seed tile.  The flat-kernel K2 (k_iter8.cu) sums
    // exactly in int32 for any chunk, so ct targets ~8 items per CTA (long items drain G less often;
    // short ones keep a single frame's step spread over every SM); the Gaussian K2 (k_iter.cu) keeps
    // the fixed kChunkTiles of its fp32 accumulation.
    int ct = kChunkTiles, nch = p.n_chunks;
    if (p.profile == 0) {
      // items per CTA: 8 for large steps; down to 1 when the step has few tiles per CTA (a single
      // frame's step split into 8 x 148 items of one or two tiles paid a Gq drain and a seed-tile
      // load per tile: 27.5 us per K2 launch against ~6 us of tile work)
      const long long total = (long long)s_tiles_total * p.n_ptiles;
      long long per_cta = total / (32ll * p.num_sms);
      per_cta = per_cta < 1 ? 1 : (per_cta > 8 ? 8 : per_cta);
      const long long want = (total + per_cta * p.num_sms - 1) / (per_cta * p.num_sms);
      const long long cmax = p.DP == 16 ? p.item_tiles_max : p.item_tiles_max / 2;  // 28 KB tiles at DP = 32
      ct = (int)(want < 1 ? 1 : (want > cmax ? cmax : want));
      if (ct > p.n_ptiles) ct = p.n_ptiles;
      nch = (p.n_ptiles + ct - 1) / ct;
    }
    p.counters[12] = ct;
    p.counters[13] = nch;
    p.counters[0] = s_tiles_total * nch;
    p.counters[1] = s_tiles_total;
    p.counters[3] = 0;
    p.counters[4] = 0;  // post_step_kernel: tiles of this step done
    reinterpret_cast<long long*>(p.counters + 6)[0] = units;  // active seeds this step (A_t summed)
    reinterpret_cast<long long*>(p.counters + 10)[0] = count_units;  // converged modes counted (R10)
  }
}

__global__ void plan_kernel(Params p) {
  __shared__ int sm[33];
  __shared__ int s_tiles_total;
  pdl_wait();
  plan_body<false>(p, sm, &s_tiles_total);
}

// K3 for one tile task (128 compacted rows of one frame); returns nothing, adds the CTA's converged /
// stalled counts to the frame's step counters (one atomic each)
template <int DP, bool CG>
__device__ void update_tile(const Params& p, const TileTask& task) {
  {
    FrameCtl& c = p.ctl[task.f];
    const int j = task.tile * kBM + threadIdx.x;
    const int n_active = ldx<CG>(&c.n_active);
    int conv = 0, stall = 0;
    const size_t r = (size_t)task.f * p.S_pad + j;  // compacted row (accumulator index)
    if (task.mode == 1) {
      // count pass: intensity |S_h(m)| of a converged mode (R10)
      if (j < n_active) p.scnt[(size_t)task.f * p.S_cap + p.act[(size_t)task.f * p.S_cap + j]] = p.cacc[r];
      p.cacc[r] = 0;
    } else {
      double g[DP];
#pragma unroll
      for (int k = 0; k < DP; ++k) {
        g[k] = p.gacc[r * DP + k];
        p.gacc[r * DP + k] = 0.0;  // every row of a processed tile is reset for the next step
      }
      if (j < n_active && p.metric == 1) {
        // Euclidean (R24): s' = window mean = G[0, d) / G[d + 1] (the ones column counts the window,
        // both scaled by 2^11); no renormalisation; tolerance in the frame's scaled units
        const size_t sidx = (size_t)task.f * p.S_cap + p.act[(size_t)task.f * p.S_cap + j];
        const double cntw = g[p.d + 1];
        if (!(cntw > 0.0)) {
          p.sstat[sidx] = ST_STALLED;
          stall = 1;
        } else {
          float* s = p.seeds + sidx * DP;
          double dd = 0.0;
#pragma unroll
          for (int k = 0; k < DP; ++k) {
            const double v = k < p.d ? g[k] / cntw : 0.0;
            const double e = v - (double)ldx<CG>(&s[k]);
            dd += e * e;
            s[k] = (float)v;
          }
          if (sqrt(dd) < p.tol * (double)p.fscale[task.f]) {
            p.sstat[sidx] = ST_CONV;
            conv = 1;
          }
        }
      } else if (j < n_active) {
        const size_t sidx = (size_t)task.f * p.S_cap + p.act[(size_t)task.f * p.S_cap + j];
        double nn = 0.0;
#pragma unroll
        for (int k = 0; k < DP; ++k) nn += g[k] * g[k];
        if (!(nn > 0.0)) {
          p.sstat[sidx] = ST_STALLED;  // empty window: the 0/1-weighted sum is exactly zero
          stall = 1;
        } else {
          const double rn = 1.0 / sqrt(nn);
          float* s = p.seeds + sidx * DP;
          double dd = 0.0;
#pragma unroll
          for (int k = 0; k < DP; ++k) {
            const double v = g[k] * rn;
            const double e = v - (double)ldx<CG>(&s[k]);
            dd += e * e;
            s[k] = (float)v;
          }
          if (sqrt(dd) < p.tol) {
            p.sstat[sidx] = ST_CONV;
            conv = 1;
          }
        }
      }
    }
    // block-reduce and one atomic per CTA
    conv = __syncthreads_count(conv);
    stall = __syncthreads_count(stall);
    if (threadIdx.x == 0) {
      if (conv) atomicAdd(&c.step_conv, conv);
      if (stall) atomicAdd(&c.step_stall, stall);
    }
  }
}

template <int DP>
__global__ void __launch_bounds__(kBM) update_kernel(Params p) {
  pdl_wait();
  const int n_tiles = p.counters[1];
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) update_tile<DP, false>(p, p.tiles[t]);
}

// compact the seeds of frame f with status `want` (ascending seed index) into act / fp16 rows
template <int DP, bool CG>
__device__ int compact_seeds(const Params& p, int f, int K, uint8_t want, int* sm) {
  const size_t base = (size_t)f * p.S_cap;
  int carry = 0;
  for (int j0 = 0; j0 < K; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    // seed sharding: this rank iterates (and counts) only the seeds it owns
    const int a = (j < K && ldx<CG>(&p.sstat[base + j]) == want && j % p.world == p.rank) ? 1 : 0;
    int tot;
    const int pos = carry + block_excl_scan(a, sm, &tot);
    if (a) {
      p.act[base + pos] = j;
      const float* s = p.seeds + (base + j) * DP;
      __align__(16) __half h[DP];
      __align__(16) __half hs[DP];
      __align__(16) __half l[DP];
      float row[DP], sv[DP];
#pragma unroll
      for (int k = 0; k < DP; ++k) sv[k] = ldx<CG>(&s[k]);
      operand_row<DP>(p, f, sv, row);
#pragma unroll
      for (int k = 0; k < DP; ++k) split_seed(row[k], h[k], hs[k], l[k]);
      const size_t ro = (size_t)f * p.S_pad + pos;
      uint4* dst = reinterpret_cast<uint4*>(p.sop + ro * DP);
      uint4* dsts = reinterpret_cast<uint4*>(p.sops + ro * DP);
      uint4* dstl = reinterpret_cast<uint4*>(p.sopl + ro * DP);
#pragma unroll
      for (int k = 0; k < DP / 8; ++k) {
        dst[k] = reinterpret_cast<const uint4*>(h)[k];
        dsts[k] = reinterpret_cast<const uint4*>(hs)[k];
        dstl[k] = reinterpret_cast<const uint4*>(l)[k];
      }
    }
    carry += tot;
  }
  return carry;
}

// the early-stop / compaction step of frame f (one CTA; s_end, s_rem, sm: shared scratch)
template <int DP, bool CG>
__device__ void ctl_frame(const Params& p, int f, int* sm, int& s_end, int& s_rem) {
  FrameCtl& c = p.ctl[f];
  if (c.phase == PH_COUNT) {  // intensities written by the update kernel
    if (threadIdx.x == 0) { c.phase = PH_POST; c.n_active = 0; }
    return;
  }
  if (c.phase != PH_ITERATE) return;
  if (threadIdx.x == 0) {
    // decisions use the counts summed over the ranks (seed sharding); the compaction check uses
    // this rank's own
    int A = c.n_active, conv = ldx<CG>(&c.step_conv), stall = ldx<CG>(&c.step_stall);
    if (p.world > 1) { A = p.xchg[f * 4 + 0]; conv = p.xchg[f * 4 + 1]; stall = p.xchg[f * 4 + 2]; }
    c.t += 1;
    c.seed_iters += A;
    c.round_seed_iters[c.round] += A;
    c.n_conv += conv;
    const int rem = A - conv - stall;
    s_rem = c.n_active - ldx<CG>(&c.step_conv) - ldx<CG>(&c.step_stall);
    s_end = (c.n_conv >= c.need) || rem <= 0 || c.t >= p.max_iter;
  }
  __syncthreads();
  const int K = c.K_r;
  const size_t base = (size_t)f * p.S_cap;
  if (s_end) {
    for (int j = threadIdx.x; j < K; j += blockDim.x)
      if (ldx<CG>(&p.sstat[base + j]) == ST_ACTIVE) p.sstat[base + j] = ST_DISCARDED;
    __syncthreads();
    const int r = c.round;
    const int nconv = c.n_conv;
    // rows for the intensity pass (this rank's converged seeds; all of them without sharding)
    const int nloc = nconv > 0 ? compact_seeds<DP, CG>(p, f, K, ST_CONV, sm) : 0;
    if (threadIdx.x == 0) {
      atomicMax(&p.counters[18], c.Kc + nconv);  // merge pool size: picks the merge path (k_post.cu)
      c.round_iters[r] = c.t;
      c.round_conv[r] = nconv;
      c.round_disc[r] = K - nconv;
      c.n_active = nloc;
      if (r == 0 && nconv == 0) {
        c.status = 4;  // FMS_E_STALLED
        c.phase = PH_ERROR;
      } else if (nconv > 0) {
        c.phase = PH_COUNT;
        atomicAdd(&p.counters[3], 1);
      } else {
        c.phase = PH_POST;
      }
    }
    return;
  }
  const int carry = compact_seeds<DP, CG>(p, f, K, ST_ACTIVE, sm);
  if (threadIdx.x == 0) {
    c.n_active = carry;
    atomicAdd(&p.counters[3], 1);  // frames still iterating
    if (carry != s_rem) { c.status = 9; c.phase = PH_ERROR; }
  }
}

template <int DP>
__global__ void ctl_step_kernel(Params p) {
  __shared__ int s_end, s_rem;
  __shared__ int sm[33];
  pdl_wait();
  ctl_frame<DP, false>(p, blockIdx.x, sm, s_end, s_rem);
}

// ---------------- the fused step tail of the device-resident loop (k_graph.cu) ----------------
// One kernel per lockstep step after K2 instead of four (update, ctl_step, step_cond, plan): CTAs run
// K3 over the step's tiles; the CTA finishing a frame's last tile runs that frame's ctl_step; the CTA
// finishing the step's last tile sets the step loop's condition and plans the next step.  "Last" is
// decided by counters incremented after a __threadfence (the CUDA threadFenceReduction pattern), and
// every read of state another CTA wrote during the kernel goes to L2 (ld.global.cg: an L1 line this
// CTA cached earlier in the kernel may be stale).  Only the unsharded graph path uses it.
__device__ bool step_more(const Params& p) {  // the step loop's condition (was step_cond_kernel)
  ++p.counters[14];
  const int round_steps = ++p.counters[17];
  bool more = __ldcg(&p.counters[3]) > 0 && p.counters[5] == 0;
  if (more && round_steps > p.max_iter + 2) {
    p.counters[16] = 1;  // the step loop did not terminate
    more = false;
  }
  return more;
}

template <int DP>
__global__ void __launch_bounds__(kBM) post_step_kernel(cudaGraphConditionalHandle h, Params p) {
  __shared__ int sm[33];
  __shared__ int s_end, s_rem, s_last, s_tiles_total;
  const int n_tiles = p.counters[1];
  auto step_end = [&]() {
    // frames a plan gave no tile but whose phase still needs a ctl_step (not reached on the unsharded
    // path: an iterating or counting frame always has active rows)
    int need = 0;  // a frame without tiles whose phase still needs ctl_step (checked in parallel)
    for (int f = threadIdx.x; f < p.B; f += blockDim.x) {
      const FrameCtl& c = p.ctl[f];
      const int ph = __ldcg(&c.phase);
      need |= (ph == PH_ITERATE || ph == PH_COUNT) && c.n_tiles_step == 0;
    }
    if (__syncthreads_or(need)) {
      for (int f = 0; f < p.B; ++f) {
        const FrameCtl& c = p.ctl[f];
        const int ph = __ldcg(&c.phase);
        if ((ph == PH_ITERATE || ph == PH_COUNT) && c.n_tiles_step == 0) {
          ctl_frame<DP, true>(p, f, sm, s_end, s_rem);
          __syncthreads();
        }
      }
    }
    if (threadIdx.x == 0) {
      __threadfence();
      cudaGraphSetConditional(h, step_more(p) ? 1u : 0u);
    }
    __syncthreads();
    plan_body<true>(p, sm, &s_tiles_total);
  };
  if (n_tiles == 0) {
    if (blockIdx.x == 0) step_end();
    return;
  }
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileTask task = p.tiles[t];
    update_tile<DP, true>(p, task);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // this CTA's K3 writes before its count
      const int d = atomicAdd(&p.ctl[task.f].tiles_done, 1);
      s_last = d == p.ctl[task.f].n_tiles_step - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      ctl_frame<DP, true>(p, task.f, sm, s_end, s_rem);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      __threadfence();  // the frame's ctl_step writes before the step count
      s_last = atomicAdd(&p.counters[4], 1) == n_tiles - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      step_end();
    }
  }
}

// ---------------- seed sharding: exchange buffers around the collectives ----------------
// per step: this rank's (active, converged, stalled) counts -> xchg, summed over ranks before ctl_step
__global__ void xchg_pack_kernel(Params p) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < p.B; f += gridDim.x * blockDim.x) {
    const FrameCtl& c = p.ctl[f];
    const bool it = c.phase == PH_ITERATE;
    p.xchg[f * 4 + 0] = it ? c.n_active : 0;
    p.xchg[f * 4 + 1] = it ? c.step_conv : 0;
    p.xchg[f * 4 + 2] = it ? c.step_stall : 0;
    p.xchg[f * 4 + 3] = 0;
  }
}
// end of the round's iteration: largest K_r among frames about to merge -> counters[8]
__global__ void xkmax_kernel(Params p) {
  __shared__ int m;
  if (threadIdx.x == 0) m = 0;
  __syncthreads();
  for (int f = threadIdx.x; f < p.B; f += blockDim.x)
    if (p.ctl[f].phase == PH_POST) atomicMax(&m, p.ctl[f].K_r);
  __syncthreads();
  if (threadIdx.x == 0) p.counters[8] = m;
}
// owned seed rows (fp32 bits, status, intensity) into the round buffer, zeros elsewhere: summing
// the buffer over ranks (int32) reproduces every owner's bits exactly, since one term is nonzero
template <int DP>
__global__ void xround_pack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  const bool post = c.phase == PH_POST;
  const int K = post ? c.K_r : 0;
  const size_t base = (size_t)f * p.S_cap;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.xkmax; j += gridDim.x * blockDim.x) {
    int* row = p.xbuf + ((size_t)f * p.xkmax + j) * (DP + 2);
    const bool own = j < K && j % p.world == p.rank;
#pragma unroll
    for (int k = 0; k < DP; ++k) row[k] = own ? __float_as_int(p.seeds[(base + j) * DP + k]) : 0;
    row[DP] = own ? (int)p.sstat[base + j] : 0;
    row[DP + 1] = own ? p.scnt[base + j] : 0;
  }
}
template <int DP>
__global__ void xround_unpack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  if (c.phase != PH_POST) return;
  const int K = c.K_r;
  const size_t base = (size_t)f * p.S_cap;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x) {
    const int* row = p.xbuf + ((size_t)f * p.xkmax + j) * (DP + 2);
#pragma unroll
    for (int k = 0; k < DP; ++k) p.seeds[(base + j) * DP + k] = __int_as_float(row[k]);
    p.sstat[base + j] = (uint8_t)row[DP];
    p.scnt[base + j] = row[DP + 1];
  }
}

// all-gather layout: this rank's owned seeds j = rank + world m packed at row m; after the gather,
// seed j of frame f sits at recv[j % world][f][j / world]
template <int DP>
__global__ void xgather_pack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  const int K = c.phase == PH_POST ? c.K_r : 0;
  const size_t base = (size_t)f * p.S_cap;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < p.xkpr; m += gridDim.x * blockDim.x) {
    const int j = p.rank + p.world * m;
    int* row = p.xsend + ((size_t)f * p.xkpr + m) * (DP + 2);
    const bool own = j < K;
#pragma unroll
    for (int k = 0; k < DP; ++k) row[k] = own ? __float_as_int(p.seeds[(base + j) * DP + k]) : 0;
    row[DP] = own ? (int)p.sstat[base + j] : 0;
    row[DP + 1] = own ? p.scnt[base + j] : 0;
  }
}
template <int DP>
__global__ void xgather_unpack_kernel(Params p) {
  const int f = blockIdx.y;
  const FrameCtl& c = p.ctl[f];
  if (c.phase != PH_POST) return;
  const int K = c.K_r;
  const size_t base = (size_t)f * p.S_cap;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x) {
    const int* row = p.xrecv + (((size_t)(j % p.world) * p.B + f) * p.xkpr + j / p.world) * (DP + 2);
#pragma unroll
    for (int k = 0; k < DP; ++k) p.seeds[(base + j) * DP + k] = __int_as_float(row[k]);
    p.sstat[base + j] = (uint8_t)row[DP];
    p.scnt[base + j] = row[DP + 1];
  }
}
cudaError_t launch_xgather(const Params& p, bool pack, cudaStream_t st) {
  const int rows = pack ? p.xkpr : p.xkmax;
  const dim3 g((unsigned)std::max(1, std::min(64, (rows + 255) / 256)), p.B);
  if (p.DP == 16) {
    if (pack) xgather_pack_kernel<16><<<g, 256, 0, st>>>(p);
    else xgather_unpack_kernel<16><<<g, 256, 0, st>>>(p);
  } else {
    if (pack) xgather_pack_kernel<32><<<g, 256, 0, st>>>(p);
    else xgather_unpack_kernel<32><<<g, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_xchg_pack(const Params& p, cudaStream_t st) {
  xchg_pack_kernel<<<(p.B + 255) / 256, 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_xkmax(const Params& p, cudaStream_t st) {
  xkmax_kernel<<<1, 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_xround(const Params& p, bool pack, cudaStream_t st) {
  const dim3 g((unsigned)std::max(1, std::min(64, (p.xkmax + 255) / 256)), p.B);
  if (p.DP == 16) {
    if (pack) xround_pack_kernel<16><<<g, 256, 0, st>>>(p);
    else xround_unpack_kernel<16><<<g, 256, 0, st>>>(p);
  } else {
    if (pack) xround_pack_kernel<32><<<g, 256, 0, st>>>(p);
    else xround_unpack_kernel<32><<<g, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_plan(const Params& p, cudaStream_t st) {
  return launch_ex(p.pdl, plan_kernel, 1, 1024, 0, st, p);
}

cudaError_t launch_post_step(cudaGraphConditionalHandle h, const Params& p, int num_sms, cudaStream_t st) {
  if (p.DP == 16) post_step_kernel<16><<<num_sms, kBM, 0, st>>>(h, p);
  else post_step_kernel<32><<<num_sms, kBM, 0, st>>>(h, p);
  return cudaGetLastError();
}

cudaError_t launch_update(const Params& p, int num_sms, cudaStream_t st) {
  // grid-stride over the step's tiles; 4 CTAs per SM so a step's tiles (~160 at 96 frames) each get
  // their own CTA instead of some CTAs running two tiles' dependent-load chains back to back
  return launch_ex(p.pdl, p.DP == 16 ? update_kernel<16> : update_kernel<32>, 4 * num_sms, kBM, 0, st, p);
}
cudaError_t launch_ctl(const Params& p, cudaStream_t st) {
  return launch_ex(p.pdl, p.DP == 16 ? ctl_step_kernel<16> : ctl_step_kernel<32>, p.B, 512, 0, st, p);
}

}  // namespace fms
