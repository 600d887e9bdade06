// k_graph.cu -- the device-resident round / step loop (CUDA graph with two nested WHILE nodes).
//
// One fms_cluster_batch call on a single GPU is one graph launch and one host synchronisation:
//
//   prologue:  counters <- 0, K1 prep
//   WHILE round_cond:                                  OSOP round
//     K6 select -> plan                                Alg. 2 l.2
//     step_cond <- 1
//     WHILE step_cond:                                 lockstep step, Alg. 2 l.4-9
//       K2 -> post_step (K3 update, ctl_step, step condition, next plan: k_step.cu)
//     K4 merge (SMEM sort; IF some pool > 8192: global sort) -> K5 assign -> K7 osop -> round_cond
//   output centres
//
// The conditions are the counters the host loop polled: counters[3] (frames still iterating after
// this step, from ctl_step) and counters[2] (frames not done, from osop).  Safety caps (max_iter + 2
// steps per round, max_rounds + 1 rounds) end a loop that would not terminate and raise
// counters[16]; counters[14] / [15] count the steps and rounds run (run statistics).
#include "fms_device.cuh"

namespace fms {

__global__ void set_cond_kernel(cudaGraphConditionalHandle h, unsigned v) { cudaGraphSetConditional(h, v); }

// the unfused step tail's condition (option fuse_step = 0; post_step_kernel folds it in otherwise)
__global__ void step_cond_kernel(cudaGraphConditionalHandle h, Params p) {
  pdl_wait();
  ++p.counters[14];
  const int round_steps = ++p.counters[17];
  bool more = p.counters[3] > 0 && p.counters[5] == 0;
  if (more && round_steps > p.max_iter + 2) {
    p.counters[16] = 1;  // the step loop did not terminate
    more = false;
  }
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

__global__ void round_cond_kernel(cudaGraphConditionalHandle h, Params p) {
  const int rounds = ++p.counters[15];
  p.counters[17] = 0;  // steps of the next round
  bool more = p.counters[2] > 0 && p.counters[5] == 0 && p.counters[16] == 0;
  if (more && rounds > p.max_rounds + 1) {
    p.counters[16] = 2;  // the round loop did not terminate
    more = false;
  }
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

// the global-memory merge path runs only when some frame's pool exceeds the SMEM sort (k_post.cu)
__global__ void big_merge_cond_kernel(cudaGraphConditionalHandle h, Params p) {
  cudaGraphSetConditional(h, p.counters[18] > 8192 ? 1u : 0u);
}
cudaError_t launch_big_merge_cond(cudaGraphConditionalHandle h, const Params& p, cudaStream_t st) {
  big_merge_cond_kernel<<<1, 1, 0, st>>>(h, p);
  return cudaGetLastError();
}

cudaError_t launch_set_cond(cudaGraphConditionalHandle h, unsigned v, cudaStream_t st) {
  set_cond_kernel<<<1, 1, 0, st>>>(h, v);
  return cudaGetLastError();
}
cudaError_t launch_step_cond(cudaGraphConditionalHandle h, const Params& p, cudaStream_t st) {
  return launch_ex(p.pdl, step_cond_kernel, 1, 1, 0, st, h, p);
}
cudaError_t launch_round_cond(cudaGraphConditionalHandle h, const Params& p, cudaStream_t st) {
  round_cond_kernel<<<1, 1, 0, st>>>(h, p);
  return cudaGetLastError();
}

}  // namespace fms
