// k_step.cu -- per-lockstep-step control around K2: work planning, K3 (reduce + renormalise +
// converge), and the per-frame early-stop / compaction step.
//
// K3 implements, for every active seed (R4, R6):
//     G = sum over split-pixel partials in fixed split order (fp64)
//     s' = G / |G|                      (renormalised onto the unit sphere; the count cancels)
//     delta = |s' - s|_2,  converged if delta < tol = h/1000,  converged seeds freeze (R9)
//     window count 0 -> stalled (never happens for seeds started at pixels, pin P3)
// ctl_step applies early stopping (R8): once converged >= ceil(gamma*K_r) or no seed is
// active (or max_iter), the remaining active seeds are discarded and the frame moves to the merge
// phase; otherwise the active seeds are compacted (ascending seed index) into the fp16 operand rows.
#include "fms_device.cuh"

namespace fms {

// one CTA: prefix over frames -> item table and tile-task table for this step
__global__ void plan_kernel(Params p) {
  __shared__ int sm[33];
  __shared__ int s_items_total, s_tiles_total;
  int carry_i = 0, carry_t = 0;
  for (int f0 = 0; f0 < p.B; f0 += blockDim.x) {
    const int f = f0 + threadIdx.x;
    int ni = 0, nt = 0;
    if (f < p.B) {
      FrameCtl& c = p.ctl[f];
      if (c.phase == PH_ITERATE && c.n_active > 0) {
        nt = (c.n_active + kBM - 1) / kBM;
        ni = nt * c.splits;
      }
    }
    int ti, tt;
    int oi = block_excl_scan(ni, sm, &ti);
    int ot = block_excl_scan(nt, sm, &tt);
    if (f < p.B) {
      FrameCtl& c = p.ctl[f];
      c.item_off = carry_i + oi;
      c.tile_off = carry_t + ot;
      c.n_tiles_step = nt;
      c.step_conv = 0;
      c.step_stall = 0;
    }
    carry_i += ti;
    carry_t += tt;
  }
  if (threadIdx.x == 0) {
    s_items_total = carry_i;
    s_tiles_total = carry_t;
  }
  __syncthreads();
  if (s_items_total > p.items_cap || s_tiles_total > p.tiles_cap) {
    if (threadIdx.x == 0) { p.counters[0] = 0; p.counters[1] = 0; p.counters[5] = 1; }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int f = warp; f < p.B; f += nw) {
    const FrameCtl& c = p.ctl[f];
    const int nt = c.n_tiles_step;
    if (nt == 0) continue;
    const int S = c.splits, ch = c.chunk_tiles;
    for (int idx = lane; idx < nt * S; idx += 32) {
      const int tile = idx / S, s = idx % S;
      const int begin = s * ch;
      int cnt = p.n_ptiles - begin;
      if (cnt > ch) cnt = ch;
      p.items[c.item_off + idx] = WorkItem{f, tile, begin, cnt};
    }
    for (int tile = lane; tile < nt; tile += 32) p.tiles[c.tile_off + tile] = TileTask{f, tile, c.item_off + tile * S, S};
  }
  if (threadIdx.x == 0) {
    p.counters[0] = s_items_total;
    p.counters[1] = s_tiles_total;
    p.counters[3] = 0;
    long long units = 0;
    for (int f = 0; f < p.B; ++f)
      if (p.ctl[f].n_tiles_step) units += p.ctl[f].n_active;
    reinterpret_cast<long long*>(p.counters + 6)[0] = units;  // active seeds this step (A_t summed)
  }
}

template <int DP>
__global__ void __launch_bounds__(kBM) update_kernel(Params p) {
  const int n_tiles = p.counters[1];
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const TileTask task = p.tiles[t];
    FrameCtl& c = p.ctl[task.f];
    const int j = task.tile * kBM + threadIdx.x;
    int conv = 0, stall = 0;
    if (j < c.n_active) {
      const size_t sidx = (size_t)task.f * p.S_cap + p.act[(size_t)task.f * p.S_cap + j];
      double g[DP];
#pragma unroll
      for (int k = 0; k < DP; ++k) g[k] = 0.0;
      long long cnt = 0;
      for (int s = 0; s < task.splits; ++s) {
        const size_t row = (size_t)(task.item0 + s) * kBM + threadIdx.x;
        const float4* src = reinterpret_cast<const float4*>(p.part_g + row * DP);
#pragma unroll
        for (int q = 0; q < DP / 4; ++q) {
          const float4 v = src[q];
          g[4 * q] += v.x; g[4 * q + 1] += v.y; g[4 * q + 2] += v.z; g[4 * q + 3] += v.w;
        }
        cnt += p.part_c[row];
      }
      if (cnt == 0) {
        p.sstat[sidx] = ST_STALLED;
        stall = 1;
      } else {
        double nn = 0.0;
#pragma unroll
        for (int k = 0; k < DP; ++k) nn += g[k] * g[k];
        const double rn = 1.0 / sqrt(nn);
        float* s = p.seeds + sidx * DP;
        double dd = 0.0;
#pragma unroll
        for (int k = 0; k < DP; ++k) {
          const double v = g[k] * rn;
          const double e = v - (double)s[k];
          dd += e * e;
          s[k] = (float)v;
        }
        p.scnt[sidx] = (int)cnt;
        if (sqrt(dd) < p.tol) {
          p.sstat[sidx] = ST_CONV;
          conv = 1;
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
__global__ void ctl_step_kernel(Params p) {
  const int f = blockIdx.x;
  FrameCtl& c = p.ctl[f];
  if (c.phase != PH_ITERATE) return;
  __shared__ int s_end, s_rem;
  __shared__ int sm[33];
  if (threadIdx.x == 0) {
    const int A = c.n_active;
    c.t += 1;
    c.seed_iters += A;
    c.round_seed_iters[c.round] += A;
    c.n_conv += c.step_conv;
    const int rem = A - c.step_conv - c.step_stall;
    s_rem = rem;
    s_end = (c.n_conv >= c.need) || rem <= 0 || c.t >= p.max_iter;
  }
  __syncthreads();
  const int K = c.K_r;
  const size_t base = (size_t)f * p.S_cap;
  if (s_end) {
    for (int j = threadIdx.x; j < K; j += blockDim.x)
      if (p.sstat[base + j] == ST_ACTIVE) p.sstat[base + j] = ST_DISCARDED;
    if (threadIdx.x == 0) {
      const int r = c.round;
      c.round_iters[r] = c.t;
      c.round_conv[r] = c.n_conv;
      c.round_disc[r] = K - c.n_conv;
      c.n_active = 0;
      if (r == 0 && c.n_conv == 0) {
        c.status = 4;  // FMS_E_STALLED
        c.phase = PH_ERROR;
      } else {
        c.phase = PH_POST;
      }
    }
    return;
  }
  // compact the active seeds (ascending seed index) and rebuild their fp16 operand rows
  int carry = 0;
  for (int j0 = 0; j0 < K; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    const int a = (j < K && p.sstat[base + j] == ST_ACTIVE) ? 1 : 0;
    int tot;
    const int pos = carry + block_excl_scan(a, sm, &tot);
    if (a) {
      p.act[base + pos] = j;
      const float* s = p.seeds + (base + j) * DP;
      __align__(16) __half h[DP];
#pragma unroll
      for (int k = 0; k < DP; ++k) h[k] = __float2half_rn(s[k]);
      uint4* dst = reinterpret_cast<uint4*>(p.sop + ((size_t)f * p.S_pad + pos) * DP);
#pragma unroll
      for (int k = 0; k < DP / 8; ++k) dst[k] = reinterpret_cast<const uint4*>(h)[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    c.n_active = carry;
    atomicAdd(&p.counters[3], 1);  // frames still iterating
    if (carry != s_rem) { c.status = 9; c.phase = PH_ERROR; }
  }
}

cudaError_t launch_plan(const Params& p, cudaStream_t st) {
  plan_kernel<<<1, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_update_ctl(const Params& p, int num_sms, cudaStream_t st) {
  if (p.DP == 16) {
    update_kernel<16><<<num_sms * 4, kBM, 0, st>>>(p);
    ctl_step_kernel<16><<<p.B, 256, 0, st>>>(p);
  } else {
    update_kernel<32><<<num_sms * 4, kBM, 0, st>>>(p);
    ctl_step_kernel<32><<<p.B, 256, 0, st>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace fms
