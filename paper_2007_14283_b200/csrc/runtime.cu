// runtime.cu -- host runtime behind the C ABI (include/fms.h): context, workspace, TMA descriptors
// and the device-resident OSOP round/step loop.
//
// Control flow for a batch of B frames (every frame owns an independent FrameCtl state machine;
// the host only launches kernels and polls one small counter block):
//
//   init + K1 prep
//   repeat (rounds):                                   OSOP round
//     K6 select (7 small kernels; frames in SELECT)      Alg. 2 l.2
//     repeat (lockstep steps, polled every kPoll):       Alg. 2 l.4-9
//       plan -> K2 iter (tcgen05) -> K3 update -> ctl_step
//     K4 merge -> K5 assign -> K7 osop                   P:223, Eq. 19
//   output centres
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is opened at run time (fms_set_nccl), not linked

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fms.h"
#include "fms_device.cuh"

namespace fms {
cudaError_t launch_prep(const Params& p, cudaStream_t st);
cudaError_t launch_select(const Params& p, int num_sms, cudaStream_t st);
cudaError_t launch_plan(const Params& p, cudaStream_t st);
cudaError_t launch_iter(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st);
cudaError_t launch_iter8(int DP, const TMaps& tm, const Params& p, int grid, cudaStream_t st);
cudaError_t setup_iter8_attrs();
cudaError_t launch_set_cond(cudaGraphConditionalHandle h, unsigned v, cudaStream_t st);
cudaError_t launch_round_cond(cudaGraphConditionalHandle h, const Params& p, cudaStream_t st);
cudaError_t launch_big_merge_cond(cudaGraphConditionalHandle h, const Params& p, cudaStream_t st);
cudaError_t launch_merge_small(const Params& p, cudaStream_t st);
cudaError_t launch_merge_big(const Params& p, cudaStream_t st);
cudaError_t launch_assign_osop(const Params& p, const TMaps& tm, int num_sms, cudaStream_t st, bool osop);
cudaError_t launch_osop(const Params& p, cudaStream_t st);
cudaError_t launch_pstat(const Params& p, bool pack, cudaStream_t st);
cudaError_t launch_psel_kmax(const Params& p, cudaStream_t st);
cudaError_t launch_psel(const Params& p, bool pack, cudaStream_t st);
cudaError_t launch_pstep(const Params& p, bool pack, cudaStream_t st);
cudaError_t launch_ppost(const Params& p, bool pack, cudaStream_t st);
cudaError_t launch_update(const Params& p, int num_sms, cudaStream_t st);
cudaError_t launch_step_cond(cudaGraphConditionalHandle h, const Params& p, cudaStream_t st);
cudaError_t launch_post_step(cudaGraphConditionalHandle h, const Params& p, int num_sms, cudaStream_t st);
cudaError_t launch_ctl(const Params& p, cudaStream_t st);
cudaError_t launch_xchg_pack(const Params& p, cudaStream_t st);
cudaError_t launch_xkmax(const Params& p, cudaStream_t st);
cudaError_t launch_xround(const Params& p, bool pack, cudaStream_t st);
cudaError_t launch_xgather(const Params& p, bool pack, cudaStream_t st);
cudaError_t setup_assign_attrs();
cudaError_t launch_output(const Params& p, float* centres_out, int cap, cudaStream_t st);
cudaError_t setup_iter_attrs();
cudaError_t setup_post_attrs(int P_cap);
size_t merge_sort_temp_bytes(const Params& p);
}  // namespace fms

using namespace fms;

namespace {

constexpr int kPoll = 4;            // default lockstep steps launched between host polls
constexpr int kMaxPcap = 8192;      // merge pool capacity (SMEM bitonic sort)
constexpr int kCounters = 64;
constexpr int kProfInts = 12;       // counters snapshot per profiled K2 launch

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Ctx {
  int device = 0;
  int num_sms = 148;
  std::string err;
  bool profile = false;
  bool attrs_done = false;
  bool fresh_ws = true;
  size_t last_layout = 0;
  // device workspace (one allocation, carved per call)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // staging for the host-pointer entry point
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // pinned host scratch
  int* h_counters = nullptr;
  FrameCtl* h_ctl = nullptr;
  size_t h_ctl_cap = 0;
  // profiling
  std::vector<cudaEvent_t> ev;
  // per-phase timing (profile_iter): an event at every phase boundary of the host-polled loop; the
  // time to the next mark belongs to the mark's phase (fms_run_stats.ms_prep ... ms_host_wait)
  std::vector<cudaEvent_t> pev;
  std::vector<int> pev_phase;
  int* h_prof = nullptr;   // per launch: counters[0..kProfInts) snapshot
  size_t h_prof_cap = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  // seed sharding: the caller's in-place int32 sum over ranks (fms_set_exchange)
  fms_exchange_fn xfn = nullptr;
  void* xuser = nullptr;
  fms_allgather_fn gfn = nullptr;  // seed sharding: round exchange by all-gather of owned rows (optional)
  void* guser = nullptr;
  void* nccl_comm = nullptr;       // in-library NCCL communicator (fms_set_nccl)
  int rank = 0, world = 1;
  // pixel sharding: the caller's int32 sum; this rank holds pixels [poff, poff + n) of n_glob
  fms_exchange_fn pfn = nullptr;
  void* puser = nullptr;
  int prank = 0, pworld = 1;
  long long pn_glob = 0, poff = 0;
  void* pbuf = nullptr;  // exchange buffer, grown on demand
  size_t pbuf_bytes = 0;
  int poll = kPoll;  // lockstep steps between host polls ("poll_steps")
  int kprofile = 0;  // "kernel_profile": 0 flat (the paper), 1 Gaussian (NEXT-4)
  int metric = 0;    // "metric": 0 cosine (the paper's path), 1 Euclidean (NEXT-4)
  // host-buffer entry: chunked, double-buffered staging on a copy stream ("host_chunk")
  int host_chunk = 48;
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr}, ev_done = nullptr;
  // device-resident loop (k_graph.cu): one CUDA graph per call configuration, cached
  int use_graph = 1;             // option "graph"
  int pdl = 1;                   // option "pdl": programmatic dependent launch of the step-loop kernels
  int guard_stats = 0;           // option "guard_stats": K2 counts pairs within kGuardEps of tau
  int fuse_step = 0;             // option "fuse_step": the graph's step tail as one kernel (post_step; slower, DESIGN)
  cudaStream_t gst[3] = {nullptr, nullptr, nullptr};  // capture streams (prologue, round body, step body)
  struct GraphEntry {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    Params key{};                // Params the graph was captured with (io buffers zeroed)
    int cap = -1;
    unsigned long long used = 0;
  };
  static constexpr int kGraphCache = 4;  // the host entry alternates chunk sizes: keep a few graphs
  GraphEntry gcache[kGraphCache];
  unsigned long long gclock = 0;
  IoPtrs* h_io = nullptr;        // pinned: this call's buffers, copied to Params::io before the launch
};

// K2: the exact int8 weighted sum for the paper's flat kernel (k_iter8.cu); the fp16 one for the
// Gaussian profile (k_iter.cu, NEXT-4)
cudaError_t run_iter(const Params& p, const TMaps& tm, int grid, cudaStream_t st) {
  return p.profile == 0 ? launch_iter8(p.DP, tm, p, grid, st) : launch_iter(p.DP, tm, p, grid, st);
}

fms_status fail(Ctx* c, fms_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

#define CU(call)                                                                                  \
  do {                                                                                            \
    cudaError_t _e = (call);                                                                      \
    if (_e != cudaSuccess)                                                                        \
      return fail(c, FMS_E_CUDA, std::string(#call " failed: ") + cudaGetErrorString(_e));       \
  } while (0)

fms_status make_tmap(Ctx* c, CUtensorMap* m, void* base, uint64_t rows, int DP) {
  if (!c->encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(c, FMS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    c->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)DP, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)DP * 2};
  cuuint32_t box[2] = {(cuuint32_t)DP, (cuuint32_t)kBN};
  cuuint32_t es[2] = {1, 1};
  CUresult r = c->encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE,
                         DP == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, FMS_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return FMS_OK;
}

// int8 digit planes: rows of 128 pixels (bytes), one box = the 3 DP planes of one tile, 128B swizzle
fms_status make_tmap_q(Ctx* c, CUtensorMap* m, void* base, uint64_t rows, int nq) {
  cuuint64_t dims[2] = {(cuuint64_t)kBN, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kBN};
  cuuint32_t box[2] = {(cuuint32_t)kBN, (cuuint32_t)nq};
  cuuint32_t es[2] = {1, 1};
  CUresult r = c->encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, FMS_E_CUDA, "cuTensorMapEncodeTiled (digits) failed: " + std::to_string((int)r));
  return FMS_OK;
}

fms_status validate(Ctx* c, int32_t B, int64_t n, int32_t d, double h, int32_t max_iters, double tol,
                    const fms_seed_policy* pol) {
  if (!c) return FMS_E_INVALID;
  if (B < 1 || n < 1 || d < 1 || d > 32) return fail(c, FMS_E_INVALID, "need B>=1, n>=1, 1<=d<=32");
  if (c->metric == 1) {
    if (d > 30) return fail(c, FMS_E_INVALID, "the Euclidean metric needs d <= 30 (two augmented columns)");
    if (!(h > 0.0 && std::isfinite(h))) return fail(c, FMS_E_INVALID, "bandwidth must be > 0");
    if (c->kprofile != 0) return fail(c, FMS_E_INVALID, "the Euclidean metric uses the flat kernel");
  } else if (!(h > 0.0 && h < 1.0)) {
    return fail(c, FMS_E_INVALID, "bandwidth must be in (0,1) (cosine distance)");
  }
  if (!(tol > 0.0) || max_iters < 1) return fail(c, FMS_E_INVALID, "need tol>0 and max_iters>=1");
  if (!pol) return fail(c, FMS_E_INVALID, "policy is NULL");
  if (pol->kind < 0 || pol->kind > 2) return fail(c, FMS_E_INVALID, "bad policy kind");
  if (pol->kind != FMS_SEEDS_ALL && pol->n_seeds < 1) return fail(c, FMS_E_INVALID, "n_seeds must be >= 1");
  if (!(pol->gamma > 0.0 && pol->gamma <= 1.0)) return fail(c, FMS_E_INVALID, "gamma must be in (0,1]");
  if (pol->max_rounds < 1 || pol->max_rounds > FMS_MAX_ROUNDS) return fail(c, FMS_E_INVALID, "max_rounds in 1..16");
  if (pol->kind == FMS_SEEDS_OSOP && (!(pol->P > 0.0 && pol->P < 1.0) || !(pol->L > 0.0)))
    return fail(c, FMS_E_INVALID, "OSOP needs 0<P<1 and L>0");
  if ((double)B * (double)align_up((size_t)n, kBN) >= 2147483647.0)
    return fail(c, FMS_E_INVALID, "B*n too large for 32-bit TMA coordinates");
  return FMS_OK;
}

// carve the workspace; returns required bytes (and fills pointers if base != nullptr)
size_t carve(Params& p, uint8_t* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> void* {
    off = align_up(off, 1024);
    void* r = base ? base + off : nullptr;
    off += bytes;
    return r;
  };
  const size_t B = p.B;
  p.Xh = (__half*)take(B * p.n_pad * p.DP * 2);
  p.Xl = (__half*)take(B * p.n_pad * p.DP * 2);
  p.Xq = (int8_t*)take(B * p.n_pad * p.DP * 3);
  p.inv = (float*)take(B * p.n * 4);
  p.flags = (uint8_t*)take(B * p.n_glob);
  p.seeds = (float*)take(B * (size_t)p.S_cap * p.DP * 4);
  p.sop = (__half*)take(B * (size_t)p.S_pad * p.DP * 2);
  p.sops = (__half*)take(B * (size_t)p.S_pad * p.DP * 2);
  p.sopl = (__half*)take(B * (size_t)p.S_pad * p.DP * 2);
  p.gacc = (double*)take(B * (size_t)p.S_pad * p.DP * 8);
  p.cacc = (int*)take(B * (size_t)p.S_pad * 4);
  p.sorig = (int*)take(B * (size_t)p.S_cap * 4);
  p.sstat = (uint8_t*)take(B * (size_t)p.S_cap);
  p.scnt = (int*)take(B * (size_t)p.S_cap * 4);
  p.act = (int*)take(B * (size_t)p.S_cap * 4);
  p.cent = (float*)take(B * (size_t)p.C_cap * p.DP * 4);
  p.cint = (int*)take(B * (size_t)p.C_cap * 4);
  p.corig = (int*)take(B * (size_t)p.C_cap * 4);
  p.hist = (int*)take(B * (size_t)p.C_cap * 4);
  p.pool = (float*)take(B * (size_t)p.P_cap * p.DP * 4);
  p.pint = (int*)take(B * (size_t)p.P_cap * 4);
  p.porg = (int*)take(B * (size_t)p.P_cap * 4);
  p.tiles = (TileTask*)take((size_t)p.tiles_cap * sizeof(TileTask));
  p.counters = (int*)take(kCounters * 4);
  p.sample = (unsigned long long*)take(B * (size_t)p.sample_cap * 8);
  p.blkcnt = (int*)take(B * (size_t)p.nblk_glob * 4);
  p.ctl = (FrameCtl*)take(B * sizeof(FrameCtl));
  p.fscale = (float*)take(B * 4);
  p.io = (const IoPtrs*)take(sizeof(IoPtrs));
  if (p.P_cap > kMaxPcap) {  // merge pools above 8192 sorted in global memory
    p.mkeys = (unsigned long long*)take(B * (size_t)p.P_cap * 8);
    p.mkeys_sorted = (unsigned long long*)take(B * (size_t)p.P_cap * 8);
    p.mvals = (int*)take(B * (size_t)p.P_cap * 4);
    p.mvals_sorted = (int*)take(B * (size_t)p.P_cap * 4);
    p.moffs = (int*)take((size_t)B * 4);
    p.moffs_end = (int*)take((size_t)B * 4);
    p.msort_bytes = merge_sort_temp_bytes(p);
    p.msort_temp = take(p.msort_bytes + 16);
  }
  if (p.world > 1) {  // seed-sharding exchange buffers
    p.xchg = (int*)take((size_t)B * 4 * 4);
    p.xbuf = (int*)take((size_t)B * p.S_cap * (p.DP + 2) * 4);
    const size_t kpr = (size_t)(p.S_cap + p.world - 1) / p.world;
    p.xsend = (int*)take((size_t)B * kpr * (p.DP + 2) * 4);
    p.xrecv = (int*)take((size_t)p.world * B * kpr * (p.DP + 2) * 4);
  }
  return align_up(off, 1024);
}

// Capture the whole call (prologue, the round loop with the step loop nested in it, output) into a
// CUDA graph with two WHILE conditional nodes whose conditions the device sets (k_graph.cu).  Body
// graphs are populated by stream capture on helper streams.
fms_status build_graph(Ctx* c, const Params& p, const TMaps& tm, int32_t cap, Ctx::GraphEntry& ge) {
  for (int i = 0; i < 3; ++i)
    if (!c->gst[i]) CU(cudaStreamCreateWithFlags(&c->gst[i], cudaStreamNonBlocking));
  if (ge.exec) { cudaGraphExecDestroy(ge.exec); ge.exec = nullptr; }
  if (ge.graph) { cudaGraphDestroy(ge.graph); ge.graph = nullptr; }
  ge.cap = -1;
  cudaStream_t s0 = c->gst[0], s1 = c->gst[1], s2 = c->gst[2];
  const cudaStreamCaptureMode mode = cudaStreamCaptureModeThreadLocal;
  // at the current capture position of `s`: a kernel setting the new condition to 1, then a WHILE
  // node on it; returns the node's body graph
  auto add_cond = [&](cudaStream_t s, cudaGraphConditionalHandle* h, cudaGraph_t* body,
                      cudaGraphConditionalNodeType type) -> fms_status {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CU(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &ndeps));
    CU(cudaGraphConditionalHandleCreate(h, g, 0, 0));
    if (type == cudaGraphCondTypeWhile) CU(launch_set_cond(*h, 1u, s));
    else CU(launch_big_merge_cond(*h, p, s));
    CU(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &ndeps));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = *h;
    np.conditional.type = type;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CU(cudaGraphAddNode(&node, g, deps, ndeps, &np));
    *body = np.conditional.phGraph_out[0];
    CU(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    return FMS_OK;
  };
  cudaGraphConditionalHandle h_round, h_step;
  cudaGraph_t round_body = nullptr, step_body = nullptr;
  CU(cudaStreamBeginCapture(s0, mode));
  fms_status r = [&]() -> fms_status {
    CU(cudaMemsetAsync(p.counters, 0, kCounters * 4, s0));
    CU(launch_prep(p, s0));
    fms_status q = add_cond(s0, &h_round, &round_body, cudaGraphCondTypeWhile);
    if (q != FMS_OK) return q;
    // ---- round body: select, the step loop, merge / assign / OSOP ----
    CU(cudaStreamBeginCaptureToGraph(s1, round_body, nullptr, nullptr, 0, mode));
    q = [&]() -> fms_status {
      CU(launch_select(p, c->num_sms, s1));
      if (c->fuse_step) CU(launch_plan(p, s1));  // the round's first step; post_step plans the next ones
      fms_status q2 = add_cond(s1, &h_step, &step_body, cudaGraphCondTypeWhile);
      if (q2 != FMS_OK) return q2;
      // ---- step body ----
      CU(cudaStreamBeginCaptureToGraph(s2, step_body, nullptr, nullptr, 0, mode));
      q2 = [&]() -> fms_status {
        if (c->fuse_step) {
          CU(run_iter(p, tm, c->num_sms, s2));
          // K3 update + ctl_step + the loop condition + the next step's plan in one kernel (k_step.cu)
          CU(launch_post_step(h_step, p, c->num_sms, s2));
        } else {
          CU(launch_plan(p, s2));
          CU(run_iter(p, tm, c->num_sms, s2));
          CU(launch_update(p, c->num_sms, s2));
          CU(launch_ctl(p, s2));
          CU(launch_step_cond(h_step, p, s2));
        }
        return FMS_OK;
      }();
      cudaGraph_t gdone = nullptr;
      const cudaError_t e2 = cudaStreamEndCapture(s2, &gdone);
      if (q2 != FMS_OK) return q2;
      CU(e2);
      CU(launch_merge_small(p, s1));
      if (p.P_cap > kMaxPcap) {  // IF some pool exceeds the SMEM sort: the global-memory merge
        cudaGraphConditionalHandle h_big;
        cudaGraph_t big_body = nullptr;
        q2 = add_cond(s1, &h_big, &big_body, cudaGraphCondTypeIf);
        if (q2 != FMS_OK) return q2;
        CU(cudaStreamBeginCaptureToGraph(s2, big_body, nullptr, nullptr, 0, mode));
        const cudaError_t eb = launch_merge_big(p, s2);
        cudaGraph_t gb = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(s2, &gb);
        CU(eb);
        CU(ee);
      }
      CU(launch_assign_osop(p, tm, c->num_sms, s1, true));
      CU(launch_round_cond(h_round, p, s1));
      return FMS_OK;
    }();
    cudaGraph_t gdone = nullptr;
    const cudaError_t e1 = cudaStreamEndCapture(s1, &gdone);
    if (q != FMS_OK) return q;
    CU(e1);
    if (cap > 0) CU(launch_output(p, nullptr, cap, s0));
    return FMS_OK;
  }();
  const cudaError_t e0 = cudaStreamEndCapture(s0, &ge.graph);
  if (r != FMS_OK) {
    cudaGetLastError();
    return r;
  }
  CU(e0);
  CU(cudaGraphInstantiate(&ge.exec, ge.graph, 0));
  ge.key = p;
  ge.cap = cap;
  return FMS_OK;
}

fms_status run_batch(Ctx* c, const float* emb, int32_t B, int64_t n, int32_t d, double h, int32_t max_iters,
                     double tol, const fms_seed_policy* pol, int32_t* labels, float* centres, int32_t cap,
                     int32_t* K_out, fms_frame_stats* fs, fms_run_stats* rs, cudaStream_t st) {
  fms_status v = validate(c, B, n, d, h, max_iters, tol, pol);
  if (v != FMS_OK) return v;
  if (!emb || !labels || !K_out || (cap > 0 && !centres) || cap < 0) return fail(c, FMS_E_INVALID, "null buffer");
  CU(cudaSetDevice(c->device));
  if (!c->attrs_done) {
    CU(setup_iter_attrs());
    CU(setup_iter8_attrs());
    CU(setup_assign_attrs());
    CU(setup_post_attrs(kMaxPcap));
    CU(cudaEventCreate(&c->t0));
    CU(cudaEventCreate(&c->t1));
    c->attrs_done = true;
  }
  Params p{};
  p.B = B;
  p.d = d;
  p.DP = d + (c->metric == 1 ? 2 : 0) <= 16 ? 16 : 32;
  p.metric = c->metric;
  p.max_iter = max_iters;
  p.n = n;
  p.n_pad = (long long)align_up((size_t)n, kBN);
  p.n_ptiles = (int)(p.n_pad / kBN);
  const bool pshard = c->pworld > 1;
  if (pshard && (c->poff < 0 || c->poff + n > c->pn_glob))
    return fail(c, FMS_E_INVALID, "pixel shard [offset, offset + n) outside the frame of n_global pixels");
  if (pshard && c->kprofile != 0)
    return fail(c, FMS_E_INVALID, "pixel sharding needs the flat kernel (its window sums are exchanged exactly)");
  if (pshard && c->metric != 0)
    return fail(c, FMS_E_INVALID, "pixel sharding needs the cosine metric (the Euclidean scale is per frame)");
  p.profile = c->kprofile;
  p.n_glob = pshard ? c->pn_glob : n;
  p.pix_off = pshard ? c->poff : 0;
  p.pworld = pshard ? c->pworld : 1;
  p.prank = pshard ? c->prank : 0;
  p.nblk_glob = (int)((p.n_glob + 2047) / 2048);
  p.pcov_words = (int)((p.n_glob + 31) / 32);
  const long long ng = p.n_glob;
  long long S = pol->kind == FMS_SEEDS_FIXED ? std::min<long long>(pol->n_seeds, ng) : ng;
  p.S_cap = (int)S;
  p.S_pad = (int)align_up((size_t)S, kBM);
  p.C_cap = (int)std::min<long long>(ng, 65536);
  // the merge pool holds the previous centres plus one round's converged seeds; pools above 8192 are
  // sorted in global memory (Alg. 1 merges n modes; late OSOP rounds of many-cell frames)
  p.P_cap = (int)std::min<long long>((long long)p.C_cap + p.S_cap, INT32_MAX / 2);
  p.tiles_cap = B * (p.S_pad / kBM);
  p.n_chunks = (p.n_ptiles + kChunkTiles - 1) / kChunkTiles;
  p.items_cap = p.tiles_cap * p.n_chunks;
  p.sample_cap = (int)std::min<long long>(ng, (long long)S + 8 * (long long)std::sqrt((double)S) + 1024);
  p.nblk = (int)((n + 2047) / 2048);
  p.h = h;
  p.tau = 1.0 - h;
  p.tau_f = c->metric == 1 ? kEuclidT0 : (float)(1.0 - h);  // Euclidean: rows carry the threshold
  p.rho_f = (float)(1.0 - h);  // merge radius rho = h (R10): keep unless x.c >= 1 - rho
  p.tol = tol;
  p.kind = pol->kind;
  p.n_seeds = pol->n_seeds;
  p.has_bg = pol->has_background;
  p.min_px = pol->min_instance_px;
  p.sat_stop = pol->saturation_stop;
  p.max_rounds = pol->max_rounds;
  p.gamma = pol->gamma;
  p.L = pol->L;
  p.H = pol->H;
  p.P = pol->P;
  p.rng_seed = pol->rng_seed;
  p.rank = c->world > 1 ? c->rank : 0;
  p.world = c->world > 1 ? c->world : 1;
  p.emb = emb;
  p.labels = labels;
  p.num_sms = c->num_sms;
  p.item_tiles_max = kChunkMax;
  p.pdl = c->pdl && !c->profile;  // profiled calls time K2 with events between plain launches
  p.guard = c->guard_stats;  // r2: 16 / 32 / 48 / 64 tiles measured 1622 / 1720 / 1678 / 1625 frames/s

  const size_t need = carve(p, nullptr);
  if (need > c->ws_bytes) {
    if (c->ws) cudaFree(c->ws);
    c->ws = nullptr;
    c->ws_bytes = 0;
    if (cudaMalloc(&c->ws, need) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, FMS_E_OOM, "workspace allocation of " + std::to_string(need) + " bytes failed");
    }
    c->ws_bytes = need;
    c->fresh_ws = true;
  }
  if (c->last_layout != need + (size_t)B * 1000003u + (size_t)p.S_pad * 7u) {
    c->fresh_ws = true;  // a different carve moves the accumulators
    c->last_layout = need + (size_t)B * 1000003u + (size_t)p.S_pad * 7u;
  }
  carve(p, reinterpret_cast<uint8_t*>(c->ws));
  if ((size_t)B > c->h_ctl_cap) {
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    CU(cudaMallocHost(&c->h_ctl, sizeof(FrameCtl) * B));
    c->h_ctl_cap = B;
  }
  if (!c->h_counters) CU(cudaMallocHost(&c->h_counters, kCounters * 4));

  TMaps tm;
  fms_status ts = make_tmap(c, &tm.xh, p.Xh, (uint64_t)B * p.n_pad, p.DP);
  if (ts == FMS_OK) ts = make_tmap(c, &tm.xl, p.Xl, (uint64_t)B * p.n_pad, p.DP);
  if (ts == FMS_OK) ts = make_tmap(c, &tm.sh, p.sop, (uint64_t)B * p.S_pad, p.DP);
  if (ts == FMS_OK) ts = make_tmap(c, &tm.ss, p.sops, (uint64_t)B * p.S_pad, p.DP);
  if (ts == FMS_OK) ts = make_tmap(c, &tm.sl, p.sopl, (uint64_t)B * p.S_pad, p.DP);
  if (ts == FMS_OK) ts = make_tmap_q(c, &tm.xq, p.Xq, (uint64_t)B * p.n_ptiles * 3 * p.DP, 3 * p.DP);
  if (ts != FMS_OK) return ts;

  CU(cudaEventRecord(c->t0, st));
  CU(cudaMemsetAsync(p.counters, 0, kCounters * 4, st));
  if (c->fresh_ws) {  // accumulator rows are kept zero between steps by K3; start clean once
    CU(cudaMemsetAsync(p.gacc, 0, (size_t)B * p.S_pad * p.DP * 8, st));
    CU(cudaMemsetAsync(p.cacc, 0, (size_t)B * p.S_pad * 4, st));
    c->fresh_ws = false;
  }
  // one call on one GPU without per-launch profiling runs as one CUDA graph launch with the round
  // and step loops on the device (k_graph.cu); sharded calls (a collective between kernels) and
  // profiled calls run the host-polled loop below
  const bool gmode = c->use_graph && !pshard && p.world == 1 && !c->profile;
  enum { PHASE_PREP, PHASE_SELECT, PHASE_ITER, PHASE_STEP, PHASE_MERGE, PHASE_ASSIGN, PHASE_HOST, PHASE_END };
  int nmarks = 0;
  auto mark = [&](int phase) -> cudaError_t {  // profiled host loop only
    if (!c->profile) return cudaSuccess;
    if ((int)c->pev.size() <= nmarks) {
      cudaEvent_t e;
      cudaError_t err = cudaEventCreate(&e);
      if (err != cudaSuccess) return err;
      c->pev.push_back(e);
      c->pev_phase.push_back(0);
    }
    c->pev_phase[nmarks] = phase;
    return cudaEventRecord(c->pev[nmarks++], st);
  };
  int steps = 0, launches = 0;
  long long kernels = 2;  // init + prep
  long long syncs = 0;    // host waits on the stream during the call
  if (gmode) {
    Params key = p;
    key.emb = nullptr;
    key.labels = nullptr;
    Ctx::GraphEntry* ge = nullptr;
    for (auto& e : c->gcache)
      if (e.exec && e.cap == cap && memcmp(&key, &e.key, sizeof(Params)) == 0) ge = &e;
    if (!ge) {  // capture a new graph into the least recently used slot
      ge = &c->gcache[0];
      for (auto& e : c->gcache)
        if (e.used < ge->used) ge = &e;
      fms_status g = build_graph(c, key, tm, cap, *ge);
      if (g != FMS_OK) return g;
    }
    ge->used = ++c->gclock;
    if (!c->h_io) CU(cudaMallocHost(&c->h_io, sizeof(IoPtrs)));
    *c->h_io = IoPtrs{emb, labels, centres};
    CU(cudaMemcpyAsync((void*)p.io, c->h_io, sizeof(IoPtrs), cudaMemcpyHostToDevice, st));
    CU(cudaGraphLaunch(ge->exec, st));
  } else {
    p.io = nullptr;
    auto pgrow = [&](size_t ints) -> fms_status {  // pixel-sharding exchange buffer
      const size_t bytes = std::max<size_t>(ints, 1) * 4;
      if (bytes > c->pbuf_bytes) {
        CU(cudaStreamSynchronize(st));
        ++syncs;
        if (c->pbuf) cudaFree(c->pbuf);
        c->pbuf = nullptr;
        c->pbuf_bytes = 0;
        if (cudaMalloc(&c->pbuf, bytes) != cudaSuccess) {
          cudaGetLastError();
          return fail(c, FMS_E_OOM, "pixel-shard exchange buffer allocation failed");
        }
        c->pbuf_bytes = bytes;
      }
      p.pbuf = reinterpret_cast<int*>(c->pbuf);
      return FMS_OK;
    };
    auto pxchg = [&](size_t ints, const char* what) -> fms_status {
      if (c->pfn(c->puser, p.pbuf, (int64_t)ints, st) != 0) return fail(c, FMS_E_NCCL, std::string(what) + " exchange failed");
      return FMS_OK;
    };
    const size_t post_ints = (size_t)B * ((size_t)p.C_cap + 2 + p.pcov_words);
    if (pshard) {
      CU(cudaMemsetAsync(p.flags, 0, (size_t)B * p.n_glob, st));  // other ranks' pixels: filled by exchanges
      fms_status g = pgrow(std::max<size_t>(post_ints, B));
      if (g != FMS_OK) return g;
    }
    CU(mark(PHASE_PREP));
    CU(launch_prep(p, st));
    if (pshard) {  // a zero-norm row on any rank fails the frame on every rank
      CU(launch_pstat(p, true, st));
      fms_status g = pxchg(B, "status");
      if (g != FMS_OK) return g;
      CU(launch_pstat(p, false, st));
    }
    for (int round = 0; round < pol->max_rounds + 1; ++round) {
      CU(mark(PHASE_SELECT));
      CU(launch_select(p, c->num_sms, st));
      kernels += 7;
      if (pshard) {  // the round's seed rows come from the ranks holding the seed pixels
        CU(launch_psel_kmax(p, st));
        CU(mark(PHASE_HOST));
        CU(cudaMemcpyAsync(c->h_counters, p.counters, kCounters * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        ++syncs;
        p.pkmax = c->h_counters[8];
        fms_status g = pgrow(std::max(post_ints, (size_t)B * p.pkmax * (2 * p.DP + 1)));
        if (g != FMS_OK) return g;
        if (p.pkmax > 0) {
          CU(launch_psel(p, true, st));
          g = pxchg((size_t)B * p.pkmax * p.DP, "seed");
          if (g != FMS_OK) return g;
          CU(launch_psel(p, false, st));
          kernels += 2;
        }
        kernels += 1;
      }
      for (int s = 0; s < max_iters + c->poll; s += c->poll) {
        for (int k = 0; k < c->poll; ++k) {
          CU(mark(PHASE_STEP));
          CU(launch_plan(p, st));
          if (c->profile) {
            const size_t slot = launches;
            if (c->ev.size() < 2 * (slot + 1)) {
              cudaEvent_t e0, e1;
              CU(cudaEventCreate(&e0));
              CU(cudaEventCreate(&e1));
              c->ev.push_back(e0);
              c->ev.push_back(e1);
            }
            if (c->h_prof_cap < slot + 1) {
              size_t ncap = std::max<size_t>(256, 2 * (slot + 1));
              int* np = nullptr;
              CU(cudaMallocHost(&np, ncap * kProfInts * sizeof(int)));
              if (c->h_prof) {
                CU(cudaStreamSynchronize(st));
                ++syncs;
                memcpy(np, c->h_prof, c->h_prof_cap * kProfInts * sizeof(int));
                cudaFreeHost(c->h_prof);
              }
              c->h_prof = np;
              c->h_prof_cap = ncap;
            }
            CU(mark(PHASE_ITER));
            CU(cudaEventRecord(c->ev[2 * slot], st));
            CU(run_iter(p, tm, c->num_sms, st));
            CU(cudaEventRecord(c->ev[2 * slot + 1], st));
            CU(mark(PHASE_STEP));
            CU(cudaMemcpyAsync(c->h_prof + slot * kProfInts, p.counters, kProfInts * sizeof(int), cudaMemcpyDeviceToHost,
                               st));
            ++launches;
          } else {
            CU(run_iter(p, tm, c->num_sms, st));
          }
          if (pshard && p.pkmax > 0) {  // window sums and counts over all pixels
            CU(launch_pstep(p, true, st));
            fms_status g = pxchg((size_t)B * p.pkmax * (2 * p.DP + 1), "step");
            if (g != FMS_OK) return g;
            CU(launch_pstep(p, false, st));
            kernels += 2;
          }
          CU(launch_update(p, c->num_sms, st));
          if (p.world > 1) {  // seed sharding: per-frame step counts summed over the ranks
            CU(launch_xchg_pack(p, st));
            if (c->xfn(c->xuser, p.xchg, (int64_t)B * 4, st) != 0) return fail(c, FMS_E_NCCL, "step exchange failed");
          }
          CU(launch_ctl(p, st));
          ++steps;
          kernels += p.world > 1 ? 5 : 4;  // plan, iter, update, (exchange pack), ctl_step
        }
        CU(mark(PHASE_HOST));
        CU(cudaMemcpyAsync(c->h_counters, p.counters, kCounters * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        ++syncs;
        if (c->h_counters[5]) return fail(c, FMS_E_INTERNAL, "work-item capacity exceeded");
        if (c->h_counters[3] == 0) break;  // no frame still iterating
      }
      CU(mark(PHASE_MERGE));
      if (p.world > 1) {  // seed sharding: every rank gets every owner's converged seeds before the merge
        CU(launch_xkmax(p, st));
        CU(mark(PHASE_HOST));
        CU(cudaMemcpyAsync(c->h_counters, p.counters, kCounters * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        ++syncs;
        p.xkmax = c->h_counters[8];
        if (p.xkmax > 0 && c->gfn) {  // all-gather of every rank's owned rows (1/world of the payload each)
          p.xkpr = (p.xkmax + p.world - 1) / p.world;
          CU(launch_xgather(p, true, st));
          if (c->gfn(c->guser, p.xsend, p.xrecv, (int64_t)B * p.xkpr * (p.DP + 2), st) != 0)
            return fail(c, FMS_E_NCCL, "round all-gather failed");
          CU(launch_xgather(p, false, st));
          kernels += 2;
        } else if (p.xkmax > 0) {
          CU(launch_xround(p, true, st));
          if (c->xfn(c->xuser, p.xbuf, (int64_t)B * p.xkmax * (p.DP + 2), st) != 0)
            return fail(c, FMS_E_NCCL, "round exchange failed");
          CU(launch_xround(p, false, st));
          kernels += 2;
        }
        kernels += 1;
      }
      CU(mark(PHASE_MERGE));
      CU(launch_merge_small(p, st));
      // the global-memory merge only when a pool exceeds the SMEM sort (the last poll read counters[18])
      if (p.P_cap > kMaxPcap && c->h_counters[18] > kMaxPcap) CU(launch_merge_big(p, st));
      CU(mark(PHASE_ASSIGN));
      CU(launch_assign_osop(p, tm, c->num_sms, st, !pshard));
      kernels += 5;  // merge, assign (tensor cores, <= 128 and <= 256 centres), assign (CUDA cores), osop
      if (pshard) {  // histogram, candidate count and coverage over all pixels before the OSOP step
        CU(launch_ppost(p, true, st));
        fms_status g = pxchg(post_ints, "round");
        if (g != FMS_OK) return g;
        CU(launch_ppost(p, false, st));
        CU(launch_osop(p, st));
        kernels += 2;
      }
      CU(mark(PHASE_HOST));
      CU(cudaMemcpyAsync(c->h_counters, p.counters, kCounters * 4, cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      ++syncs;
      if (c->h_counters[2] == 0) break;  // every frame DONE (or in error)
    }
    CU(mark(PHASE_ASSIGN));
    if (cap > 0) {
      CU(launch_output(p, centres, cap, st));
      kernels += 1;
    }
  }
  CU(cudaEventRecord(c->t1, st));
  CU(cudaMemcpyAsync(c->h_ctl, p.ctl, sizeof(FrameCtl) * B, cudaMemcpyDeviceToHost, st));
  if (gmode || p.guard) CU(cudaMemcpyAsync(c->h_counters, p.counters, kCounters * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  ++syncs;
  CU(cudaGetLastError());
  if (gmode) {
    if (c->h_counters[5]) return fail(c, FMS_E_INTERNAL, "work-item capacity exceeded");
    if (c->h_counters[16]) return fail(c, FMS_E_INTERNAL, "device loop did not terminate");
    steps = c->h_counters[14];
    // prologue + per round (select 7, plan, set_cond, merge, 3 assign, osop, round_cond) + per step
    // (K2, post_step) + output
    kernels = (p.metric == 1 ? 4 : 2) + 1 + (long long)c->h_counters[15] * (c->fuse_step ? 15 : 14) +
              (long long)steps * (c->fuse_step ? 2 : 5) + (cap > 0);
  }

  fms_status result = FMS_OK;
  for (int f = 0; f < B; ++f) {
    const FrameCtl& fc = c->h_ctl[f];
    K_out[f] = fc.Kc;
    fms_status s = FMS_OK;
    if (fc.status != 0) s = (fms_status)fc.status;
    else if (fc.phase != PH_DONE) s = FMS_E_INTERNAL;
    else if (fc.Kc > cap) s = FMS_E_CAPACITY;
    if (s != FMS_OK && result == FMS_OK) {
      result = s;
      c->err = "frame " + std::to_string(f) + " status " + std::to_string((int)s);
    }
    if (fs) {
      fms_frame_stats& o = fs[f];
      memset(&o, 0, sizeof(o));
      o.status = s;
      o.rounds = std::min(fc.round + 1, FMS_MAX_ROUNDS);
      o.K = fc.Kc;
      o.seeds_total = fc.total;
      o.seed_iters = fc.seed_iters;
      long long disc = 0;
      for (int r = 0; r < o.rounds; ++r) {
        o.round_K[r] = fc.round_K[r];
        o.round_iters[r] = fc.round_iters[r];
        o.round_conv[r] = fc.round_conv[r];
        o.round_disc[r] = fc.round_disc[r];
        o.round_Kc[r] = fc.round_Kc[r];
        o.round_I[r] = fc.round_I[r];
        o.round_seed_iters[r] = fc.round_seed_iters[r];
        o.round_cand[r] = fc.round_cand[r];
        o.round_r[r] = fc.round_r[r];
        o.round_nmin[r] = fc.round_nmin[r];
        disc += fc.round_disc[r];
      }
      o.discarded = disc;
    }
  }
  if (rs) {
    memset(rs, 0, sizeof(*rs));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->t0, c->t1);
    rs->ms_total = ms;
    rs->workspace_bytes = (int64_t)c->ws_bytes;
    rs->steps = steps;
    rs->launches = kernels;
    rs->host_syncs = syncs;
    rs->guard_pairs = p.guard ? reinterpret_cast<const long long*>(c->h_counters + kGuardCounter)[0] : 0;
    if (c->profile) {
      for (int l = 0; l < launches; ++l) {
        const int* snap = c->h_prof + (size_t)l * kProfInts;
        if (snap[0] <= 0) continue;
        float t = 0.f;
        cudaEventElapsedTime(&t, c->ev[2 * l], c->ev[2 * l + 1]);
        rs->iter_ms += t;
        rs->iter_launches += 1;
        rs->iter_items += snap[0];
        rs->iter_seed_iters += reinterpret_cast<const long long*>(snap + 6)[0];
        rs->iter_count_units += reinterpret_cast<const long long*>(snap + 10)[0];
      }
      double* ph[PHASE_END] = {&rs->ms_prep, &rs->ms_select, nullptr, &rs->ms_step_ctl, &rs->ms_merge,
                               &rs->ms_assign, &rs->ms_host_wait};
      for (int i = 0; i < nmarks; ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, c->pev[i], i + 1 < nmarks ? c->pev[i + 1] : c->t1);
        if (ph[c->pev_phase[i]]) *ph[c->pev_phase[i]] += t;
      }
    }
  }
  return result;
}

// ---- in-library NCCL (fms_set_nccl): libnccl.so.2 opened at run time, so the library loads on
//      machines without it (a process that already loaded NCCL, e.g. through torch, shares that copy) ----
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};
const NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false, ok = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
      api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
      ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.all_gather && api.comm_destroy &&
           api.error_string;
    }
  }
  return ok ? &api : nullptr;
}
// the two collectives of the sharding protocols, enqueued on the library's stream
int nccl_sum_i32(void* comm, int32_t* buf, int64_t count, void* stream) {
  return nccl_api()->all_reduce(buf, buf, (size_t)count, ncclInt32, ncclSum, static_cast<ncclComm_t>(comm),
                                static_cast<cudaStream_t>(stream)) == ncclSuccess ? 0 : 1;
}
int nccl_gather_i32(void* comm, const int32_t* send, int32_t* recv, int64_t count, void* stream) {
  return nccl_api()->all_gather(send, recv, (size_t)count, ncclInt32, static_cast<ncclComm_t>(comm),
                                static_cast<cudaStream_t>(stream)) == ncclSuccess ? 0 : 1;
}

}  // namespace

extern "C" {

fms_status fms_nccl_unique_id(void* id_out) {
  const NcclApi* a = nccl_api();
  if (!id_out) return FMS_E_INVALID;
  if (!a) return FMS_E_NCCL;
  ncclUniqueId id;
  if (a->get_unique_id(&id) != ncclSuccess) return FMS_E_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return FMS_OK;
}

const char* fms_version(void) { return "fms-b200 0.1 (sm_100a, tcgen05)"; }

fms_status fms_default_policy(fms_seed_policy* o) {
  if (!o) return FMS_E_INVALID;
  memset(o, 0, sizeof(*o));
  o->kind = FMS_SEEDS_OSOP;
  o->n_seeds = 128;
  o->gamma = 0.9;
  o->L = 2.0;
  o->H = 8.0;
  o->P = 0.99;
  o->has_background = 1;
  o->max_rounds = 8;
  return FMS_OK;
}

fms_status fms_ctx_create(void** out, int device) {
  if (!out) return FMS_E_INVALID;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return FMS_E_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return FMS_E_CUDA;
  if (prop.major != 10) return FMS_E_CUDA;  // sm_100a build
  Ctx* c = new Ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  *out = c;
  return FMS_OK;
}

void fms_ctx_destroy(void* ctx) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->ws) cudaFree(c->ws);
  if (c->stage) cudaFree(c->stage);
  if (c->h_counters) cudaFreeHost(c->h_counters);
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  if (c->h_prof) cudaFreeHost(c->h_prof);
  if (c->pbuf) cudaFree(c->pbuf);
  if (c->nccl_comm && nccl_api()) nccl_api()->comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
  for (int i = 0; i < 2; ++i) {
    if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
    if (c->ev_out[i]) cudaEventDestroy(c->ev_out[i]);
  }
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (auto e : c->pev) cudaEventDestroy(e);
  for (auto& e : c->gcache) {
    if (e.exec) cudaGraphExecDestroy(e.exec);
    if (e.graph) cudaGraphDestroy(e.graph);
  }
  for (int i = 0; i < 3; ++i)
    if (c->gst[i]) cudaStreamDestroy(c->gst[i]);
  if (c->h_io) cudaFreeHost(c->h_io);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  delete c;
}

const char* fms_last_error(const void* ctx) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  return c ? c->err.c_str() : "null context";
}

fms_status fms_set_exchange(void* ctx, fms_exchange_fn fn, void* user, int32_t rank, int32_t world) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return FMS_E_INVALID;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !fn))
    return fail(c, FMS_E_INVALID, "need 0 <= rank < world and an exchange function when world > 1");
  c->xfn = fn;
  c->xuser = user;
  c->rank = rank;
  c->world = world;
  if (world > 1) {  // the two sharding modes are exclusive
    c->pfn = nullptr;
    c->pworld = 1;
    c->prank = 0;
  }
  c->fresh_ws = true;  // the carve changes (exchange buffers)
  return FMS_OK;
}

fms_status fms_set_nccl(void* ctx, const void* unique_id, int32_t rank, int32_t world, int32_t mode,
                        int64_t n_global, int64_t offset) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return FMS_E_INVALID;
  if (world < 1 || rank < 0 || rank >= world || (mode != FMS_SHARD_SEEDS && mode != FMS_SHARD_PIXELS) ||
      (world > 1 && !unique_id))
    return fail(c, FMS_E_INVALID, "need 0 <= rank < world, mode FMS_SHARD_SEEDS or FMS_SHARD_PIXELS and a unique id");
  const NcclApi* a = nccl_api();
  if (world > 1 && !a) return fail(c, FMS_E_NCCL, "libnccl.so.2 could not be opened");
  if (c->nccl_comm) {
    a->comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
    c->nccl_comm = nullptr;
  }
  if (world == 1) {  // no sharding
    fms_set_exchange(c, nullptr, nullptr, 0, 1);
    return fms_set_pixel_shard(c, nullptr, nullptr, 0, 1, n_global, offset);
  }
  CU(cudaSetDevice(c->device));
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = a->comm_init_rank(&comm, world, id, rank);
  if (r != ncclSuccess) return fail(c, FMS_E_NCCL, std::string("ncclCommInitRank: ") + a->error_string(r));
  c->nccl_comm = comm;
  if (mode == FMS_SHARD_SEEDS) {
    fms_status s = fms_set_exchange(c, nccl_sum_i32, comm, rank, world);
    if (s != FMS_OK) return s;
    return fms_set_allgather(c, nccl_gather_i32, comm);
  }
  return fms_set_pixel_shard(c, nccl_sum_i32, comm, rank, world, n_global, offset);
}

fms_status fms_ctx_create_dist(void** ctx_out, int device, const void* unique_id, int32_t rank, int32_t world,
                               int32_t mode, int64_t n_global, int64_t offset) {
  fms_status s = fms_ctx_create(ctx_out, device);
  if (s != FMS_OK) return s;
  s = fms_set_nccl(*ctx_out, unique_id, rank, world, mode, n_global, offset);
  if (s != FMS_OK) {
    fms_ctx_destroy(*ctx_out);
    *ctx_out = nullptr;
  }
  return s;
}

fms_status fms_set_allgather(void* ctx, fms_allgather_fn fn, void* user) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return FMS_E_INVALID;
  c->gfn = fn;
  c->guser = user;
  return FMS_OK;
}

fms_status fms_set_pixel_shard(void* ctx, fms_exchange_fn fn, void* user, int32_t rank, int32_t world,
                               int64_t n_global, int64_t offset) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c) return FMS_E_INVALID;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !fn))
    return fail(c, FMS_E_INVALID, "need 0 <= rank < world and an exchange function when world > 1");
  if (world > 1 && (n_global < 1 || n_global >= (1ll << 31) || offset < 0 || offset >= n_global))
    return fail(c, FMS_E_INVALID, "need 1 <= n_global < 2^31 and 0 <= offset < n_global");
  c->pfn = fn;
  c->puser = user;
  c->prank = rank;
  c->pworld = world;
  c->pn_glob = n_global;
  c->poff = offset;
  if (world > 1) {  // the two sharding modes are exclusive
    c->xfn = nullptr;
    c->world = 1;
    c->rank = 0;
  }
  c->fresh_ws = true;
  return FMS_OK;
}

fms_status fms_set_option(void* ctx, const char* key, int64_t value) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !key) return FMS_E_INVALID;
  if (!strcmp(key, "profile_iter")) {
    c->profile = value != 0;
    return FMS_OK;
  }
  if (!strcmp(key, "host_chunk")) {  // frames per chunk of fms_cluster_batch_host
    if (value < 1 || value > 1 << 20) return fail(c, FMS_E_INVALID, "host_chunk must be >= 1");
    c->host_chunk = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "metric")) {
    if (value < 0 || value > 1) return fail(c, FMS_E_INVALID, "metric must be 0 (cosine) or 1 (Euclidean)");
    c->metric = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "kernel_profile")) {
    if (value < 0 || value > 1) return fail(c, FMS_E_INVALID, "kernel_profile must be 0 (flat) or 1 (Gaussian)");
    c->kprofile = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "graph")) {  // 1: device-resident loop (one CUDA graph launch per call); 0: host-polled
    if (value < 0 || value > 1) return fail(c, FMS_E_INVALID, "graph must be 0 or 1");
    c->use_graph = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "guard_stats")) {  // 1: K2's guard-pair count (fms_run_stats.guard_pairs)
    if (value < 0 || value > 1) return fail(c, FMS_E_INVALID, "guard_stats must be 0 or 1");
    c->guard_stats = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "pdl")) {  // 1: plan / K2 / update / ctl_step / step condition launched with PDL
    if (value < 0 || value > 1) return fail(c, FMS_E_INVALID, "pdl must be 0 or 1");
    c->pdl = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "fuse_step")) {  // 1: graph step = K2 + post_step; 0: K2 + update + ctl + cond + plan
    if (value < 0 || value > 1) return fail(c, FMS_E_INVALID, "fuse_step must be 0 or 1");
    if (c->fuse_step != (int)value)
      for (auto& e : c->gcache) e.used = 0, e.cap = -1;  // captured graphs no longer match
    c->fuse_step = (int)value;
    return FMS_OK;
  }
  if (!strcmp(key, "poll_steps")) {  // a frame that finishes idles at most poll_steps - 1 steps
    if (value < 1 || value > 64) return fail(c, FMS_E_INVALID, "poll_steps must be in 1..64");
    c->poll = (int)value;
    return FMS_OK;
  }
  return fail(c, FMS_E_INVALID, std::string("unknown option ") + key);
}

fms_status fms_cluster_batch(void* ctx, const float* emb, int32_t B, int64_t n, int32_t d, double bandwidth,
                             int32_t max_iters, double tol, const fms_seed_policy* policy, int32_t* labels,
                             float* centres, int32_t centres_cap, int32_t* K_out, fms_frame_stats* frame_stats,
                             fms_run_stats* run_stats, void* stream) {
  return run_batch(static_cast<Ctx*>(ctx), emb, B, n, d, bandwidth, max_iters, tol, policy, labels, centres,
                   centres_cap, K_out, frame_stats, run_stats, static_cast<cudaStream_t>(stream));
}

fms_status fms_cluster(void* ctx, const float* emb, int64_t n, int32_t d, double bandwidth, int32_t max_iters,
                       double tol, const fms_seed_policy* policy, int32_t* labels, float* centres,
                       int32_t centres_cap, int32_t* K_out, fms_frame_stats* frame_stats,
                       fms_run_stats* run_stats, void* stream) {
  return fms_cluster_batch(ctx, emb, 1, n, d, bandwidth, max_iters, tol, policy, labels, centres, centres_cap,
                           K_out, frame_stats, run_stats, stream);
}

// ---- NEXT-1: frame sequences with the seed count carried across frames (O8) ----
struct Session {
  Ctx* c;
  fms_seed_policy pol;
  int64_t N;  // seeds for round 0 of the next frame
};

// P:318 "if N is too large compared to N_min, N is reduced as N - N_min": N_next = the frame's
// total seeds; reduced by N_min when above H * N_min, never below N_min (R18); N_min = the frame's
// last Eq. 19 estimate (-1 = infinite: no reduction)
static int64_t session_next(int64_t total, double nmin, double H) {
  if (!(nmin > 0.0) || !((double)total > H * nmin)) return total;
  const int64_t m = (int64_t)nmin;
  return std::max<int64_t>(total - m, m);
}

fms_status fms_session_create(void* ctx, const fms_seed_policy* policy, void** session_out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c || !policy || !session_out) return FMS_E_INVALID;
  if (policy->kind != FMS_SEEDS_OSOP) return fail(c, FMS_E_INVALID, "sessions carry the OSOP seed count");
  if (policy->n_seeds < 1) return fail(c, FMS_E_INVALID, "n_seeds must be >= 1");
  *session_out = new Session{c, *policy, policy->n_seeds};
  return FMS_OK;
}

int64_t fms_session_seeds(const void* session) {
  return session ? static_cast<const Session*>(session)->N : -1;
}

void fms_session_destroy(void* session) { delete static_cast<Session*>(session); }

fms_status fms_session_step(void* session, const float* emb, int64_t n, int32_t d, double bandwidth,
                            int32_t max_iters, double tol, int32_t* labels, float* centres, int32_t centres_cap,
                            int32_t* K_out, fms_frame_stats* frame_stats, fms_run_stats* run_stats, void* stream) {
  Session* s = static_cast<Session*>(session);
  if (!s) return FMS_E_INVALID;
  fms_seed_policy pol = s->pol;
  pol.n_seeds = (int32_t)std::min<int64_t>(s->N, INT32_MAX);
  fms_frame_stats fs{};
  fms_status r = fms_cluster(s->c, emb, n, d, bandwidth, max_iters, tol, &pol, labels, centres, centres_cap, K_out,
                             &fs, run_stats, stream);
  if (frame_stats) *frame_stats = fs;
  if (r == FMS_OK || r == FMS_E_CAPACITY) {
    const double nmin = fs.rounds > 0 ? fs.round_nmin[fs.rounds - 1] : -1.0;
    s->N = std::max<int64_t>(1, session_next(fs.seeds_total, nmin, s->pol.H));
  }
  return r;
}

fms_status fms_cluster_batch_host(void* ctx, const float* emb_host, int32_t B, int64_t n, int32_t d,
                                  double bandwidth, int32_t max_iters, double tol,
                                  const fms_seed_policy* policy, int32_t* labels_host, float* centres_host,
                                  int32_t centres_cap, int32_t* K_out, fms_frame_stats* frame_stats,
                                  fms_run_stats* run_stats, void* stream) {
  Ctx* c = static_cast<Ctx*>(ctx);
  fms_status v = validate(c, B, n, d, bandwidth, max_iters, tol, policy);
  if (v != FMS_OK) return v;
  if (!emb_host || !labels_host || !K_out || centres_cap < 0 || (centres_cap > 0 && !centres_host))
    return fail(c, FMS_E_INVALID, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CU(cudaSetDevice(c->device));
  // The batch runs in chunks of up to host_chunk frames with double-buffered staging: the copy
  // stream uploads chunk i+1 (and downloads chunk i-1's results) while chunk i is clustered, so the
  // PCIe transfers overlap the compute (frames are independent, so chunking changes no result).
  // chunk sizes: the first chunk is a quarter of host_chunk (its upload is the one transfer the
  // compute cannot hide), the rest split evenly in chunks of at most host_chunk frames
  const int32_t chunk = std::max(1, std::min<int32_t>(B, c->host_chunk));
  std::vector<int32_t> c_off{0};
  const int32_t first = B > chunk ? std::max<int32_t>(1, chunk / 4) : B;
  c_off.push_back(first);
  const int32_t rest = B - first, n_rest = (rest + chunk - 1) / chunk;  // the rest in even chunks
  for (int32_t r = 1; r <= n_rest; ++r) c_off.push_back(first + (int32_t)((int64_t)rest * r / n_rest));
  const int nchunks = (int)c_off.size() - 1;
  const int nbuf = nchunks > 1 ? 2 : 1;
  const size_t eb = align_up((size_t)chunk * n * d * 4, 1024);
  const size_t lb = align_up((size_t)chunk * n * 4, 1024);
  const size_t cb = align_up((size_t)chunk * std::max(centres_cap, 1) * d * 4, 1024);
  const size_t per = eb + lb + cb;
  if (per * nbuf > c->stage_bytes) {
    if (c->stage) cudaFree(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    if (cudaMalloc(&c->stage, per * nbuf) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, FMS_E_OOM, "staging allocation failed");
    }
    c->stage_bytes = per * nbuf;
  }
  if (!c->cstream) {
    CU(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  }
  cudaStream_t cs = c->cstream;
  auto buf = [&](int i) { return reinterpret_cast<uint8_t*>(c->stage) + (size_t)(i % nbuf) * per; };
  auto rows = [&](int i) { return c_off[i + 1] - c_off[i]; };
  auto h2d = [&](int i) -> cudaError_t {
    const cudaError_t e = cudaMemcpyAsync(buf(i), emb_host + (size_t)c_off[i] * n * d, (size_t)rows(i) * n * d * 4,
                                          cudaMemcpyHostToDevice, cs);
    return e != cudaSuccess ? e : cudaEventRecord(c->ev_in[i % nbuf], cs);
  };
  // the stream the caller passed must see earlier work on it before the copies start
  CU(cudaEventRecord(c->ev_done, st));
  CU(cudaStreamWaitEvent(cs, c->ev_done, 0));
  CU(h2d(0));
  fms_status result = FMS_OK;
  fms_run_stats acc{};
  for (int i = 0; i < nchunks; ++i) {
    if (i + 1 < nchunks) {
      if (i >= 1) CU(cudaStreamWaitEvent(cs, c->ev_done, 0));  // chunk i-1 no longer reads buf (i+1) % 2
      CU(h2d(i + 1));
    }
    CU(cudaStreamWaitEvent(st, c->ev_in[i % nbuf], 0));
    if (i >= nbuf) CU(cudaStreamWaitEvent(st, c->ev_out[i % nbuf], 0));  // results of chunk i-2 downloaded
    float* d_emb = reinterpret_cast<float*>(buf(i));
    int32_t* d_lab = reinterpret_cast<int32_t*>(buf(i) + eb);
    float* d_cen = reinterpret_cast<float*>(buf(i) + eb + lb);
    const int32_t Bi = rows(i);
    // rows >= K of the downloaded centres read as zeros (the device writes rows < K only)
    if (centres_cap > 0) CU(cudaMemsetAsync(d_cen, 0, (size_t)Bi * centres_cap * d * 4, st));
    fms_run_stats rs{};
    fms_status s = run_batch(c, d_emb, Bi, n, d, bandwidth, max_iters, tol, policy, d_lab, d_cen, centres_cap,
                             K_out + c_off[i], frame_stats ? frame_stats + c_off[i] : nullptr,
                             &rs, st);
    if (s != FMS_OK && s != FMS_E_CAPACITY) {
      cudaStreamSynchronize(cs);
      return s;
    }
    if (s != FMS_OK && result == FMS_OK) result = s;
    acc.ms_total += rs.ms_total;
    acc.workspace_bytes = std::max(acc.workspace_bytes, rs.workspace_bytes);
    acc.steps += rs.steps;
    acc.iter_launches += rs.iter_launches;
    acc.iter_ms += rs.iter_ms;
    acc.iter_seed_iters += rs.iter_seed_iters;
    acc.iter_items += rs.iter_items;
    acc.launches += rs.launches;
    acc.iter_count_units += rs.iter_count_units;
    acc.host_syncs += rs.host_syncs;
    CU(cudaEventRecord(c->ev_done, st));
    CU(cudaStreamWaitEvent(cs, c->ev_done, 0));
    CU(cudaMemcpyAsync(labels_host + (size_t)c_off[i] * n, d_lab, (size_t)Bi * n * 4, cudaMemcpyDeviceToHost, cs));
    if (centres_cap > 0)
      CU(cudaMemcpyAsync(centres_host + (size_t)c_off[i] * centres_cap * d, d_cen, (size_t)Bi * centres_cap * d * 4,
                         cudaMemcpyDeviceToHost, cs));
    CU(cudaEventRecord(c->ev_out[i % nbuf], cs));
  }
  CU(cudaStreamSynchronize(cs));
  if (run_stats) *run_stats = acc;
  return result;
}

}  // extern "C"
