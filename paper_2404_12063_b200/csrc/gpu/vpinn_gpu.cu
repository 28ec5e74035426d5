// C-ABI implementation of include/vpinn_gpu.h: the device context, kernel-
// variant dispatch, CUDA-graph-captured epochs and the multi-GPU attachment
// (peer memory or NCCL).  Host runtime support: host_runtime.h, nccl_loader.h.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <utility>
#include <condition_variable>
#include <thread>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <limits>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include <nccl.h>

#include "assemble.h"
#include "aux_kernels.cuh"
#include "contract_cells.cuh"
#include "contract_mf.cuh"
#include "sf_step.h"
#include "tc_selftest.cuh"
#include "tc2_step_kernel.cuh"
#include "variant.h"
#include "vpinn_gpu.h"

#include "host_runtime.h"
#include "nccl_loader.h"

namespace {

// ---------------------------------------------------------------------------
// kernel variants: (hidden width H, hidden layers D, output channels C), each
// instantiated in its own translation unit (variant_H_D_C.cu)
using vpg::Variant;
const std::vector<Variant>& variants() {
#define VPG_ITEM(H, D, C, A) vpg::variant_##H##_##D##_##C##_##A(),
  static const std::vector<Variant> v = {VPG_VARIANTS(VPG_ITEM)};
#undef VPG_ITEM
  return v;
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
inline int round4(int x) { return (x + 3) & ~3; }

}  // namespace

namespace {
int field_id(const char* name) {
  static const char* names[vpg::kFieldCount] = {"zero",     "one",     "sin2pi_u", "sin2pi_f", "sin4pi_u",
                                                "sin4pi_f", "sin8pi_u", "sin8pi_f", "gear_f",   "bump_u",
                                                "bump_f",   "sinpi_u",  "sincos_eps", "sinpi_vareps_f"};
  if (!name) return vpg::kFieldZero;
  for (int i = 0; i < vpg::kFieldCount; ++i)
    if (std::strcmp(name, names[i]) == 0) return i;
  throw Fail{VPINN_ERR_CONFIG, std::string("device assembly: unknown field '") + name + "'"};
}

// the small assembly inputs on the device (mesh, rule, basis tables)
struct AsmUpload {
  DBuf<double> nodes, xi, eta, w, bval, bdxi, bdeta;
  DBuf<int32_t> elems;
  DBuf<int> bad;
  vpg::AsmInput in{};
  void load(const vpinn_gpu_assembly* a, int64_t n_elem, int T, int Q, cudaStream_t s) {
    if (!a->nodes || !a->elements || !a->xi || !a->eta || !a->weights || !a->basis_val || !a->basis_dxi ||
        !a->basis_deta || a->n_nodes < 1)
      throw Fail{VPINN_ERR_CONFIG, "device assembly: incomplete input"};
    for (int64_t i = 0; i < 4 * n_elem; ++i)
      if (a->elements[i] < 0 || a->elements[i] >= a->n_nodes)
        throw Fail{VPINN_ERR_MESH, "device assembly: element node index out of range"};
    in.field = field_id(a->forcing);
    nodes.alloc(2 * a->n_nodes, s);
    nodes.upload(a->nodes, 2 * a->n_nodes, s);
    elems.alloc(4 * n_elem, s);
    elems.upload(a->elements, 4 * n_elem, s);
    xi.alloc(Q, s);
    xi.upload(a->xi, Q, s);
    eta.alloc(Q, s);
    eta.upload(a->eta, Q, s);
    w.alloc(Q, s);
    w.upload(a->weights, Q, s);
    bval.alloc((size_t)T * Q, s);
    bval.upload(a->basis_val, (size_t)T * Q, s);
    bdxi.alloc((size_t)T * Q, s);
    bdxi.upload(a->basis_dxi, (size_t)T * Q, s);
    bdeta.alloc((size_t)T * Q, s);
    bdeta.upload(a->basis_deta, (size_t)T * Q, s);
    bad.alloc(1, s);
    const int big = INT_MAX;
    bad.upload(&big, 1, s);
    in.nodes = nodes.p;
    in.elems = elems.p;
    in.T = T;
    in.Q = Q;
    in.xi = xi.p;
    in.eta = eta.p;
    in.w = w.p;
    in.bval = bval.p;
    in.bdxi = bdxi.p;
    in.bdeta = bdeta.p;
  }
  void check(cudaStream_t s) {
    int b = INT_MAX;
    CK(cudaMemcpyAsync(&b, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (b != INT_MAX)
      throw Fail{VPINN_ERR_MESH, "assemble: element " + std::to_string(b) +
                                     " has non-positive jacobian determinant"};
  }
};
}  // namespace

// ---------------------------------------------------------------------------
struct vpinn_gpu_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  Variant var{};
  vpg::NetDesc net{};
  int n_params = 0;
  // problem (local partition)
  int E = 0, T = 0, Q = 0, nt = 2;
  int n_int = 0, n_bnd = 0, n_sen = 0;
  long long nb_global = 0, ns_global = 0;
  float eps = 1, bx = 0, by = 0;
  int eps_source = 0, eps_idx = 0;
  double tau = 10, gamma = 10;
  DBuf<float> tens[3], forcing, bval, sval;
  DBuf<float2> pts;
  // parameters / optimiser
  DBuf<float> params, m, v;
  // per-CTA partials and the reduced vector [grad | loss words]
  DBuf<float> grad_part;
  DBuf<double> loss_part, red;
  int grad_rows = 0, loss_rows = 0, part_stride = 0;
  // trainer
  DBuf<vpg::TrainState> st;
  DBuf<unsigned> ticket;  // reduce_adam_kernel: last-CTA ticket, non-finite gradient flag
  DBuf<float> adam_bk;    // reduce_adam_kernel: (p, m, v) before the step, for an abort
  DBuf<vpg::StepRecord> rec;
  DBuf<float> lr_tab, c1_tab, c2_tab;
  int* h_flag = nullptr;  // pinned
  // set by vpinn_gpu_train: the next run_steps lifts the finished run's stop
  // (resume_kernel) or, after an abort, refuses until vpinn_gpu_adam_reset
  bool resume_pending = false;
  long long aborted_at = 0;
  // step configuration
  bool split = false;
  std::string kernel_name;  // the epoch's dominant kernel (diagnostics)
  vpg::StepArgs sargs{};  // template (fused or reverse)
  int grid_step = 0;
  size_t smem_step = 0;
  // split path
  DBuf<float> fu, fux, fuy, feps, uxb, uyb, eb, ub, e_scalar;
  vpg::ContractArgs cargs{};
  vpg::CellContractArgs ccargs{};  // fast path when Q <= 128
  bool cell_contract = false;
  int grid_cc = 0;
  int cw_warps = 8;  // warps per CTA of the warp-per-cell contraction
  bool cw_fixed = false;  // its 5x5 / 5x5 compile-time-shape variant
  size_t smem_cc = 0;
  int grid_contract = 0, grid_pen = 0, grid_fwd = 0, grid_creduce = 0;
  DBuf<float> cpart;  // row-block contraction partial adjoint columns
  DBuf<int> rr_cover;  // warp-owned-row contraction: per cell (first CTA, segment, last CTA, 0)
  cudaEvent_t contract_mid = nullptr;  // vpinn_gpu_time_contract_kernels: recorded after the streaming kernel
  size_t smem_contract = 0, smem_fwd = 0;
  // graphs
  std::map<std::tuple<int, int, double>, cudaGraphExec_t> graphs;
  // nccl
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  // peer-memory exchange (vpinn_gpu_attach_peers): this rank's mailbox, every
  // rank's mailbox mapped here (CUDA IPC)
  vpg::PeerMailbox* pbox = nullptr;
  vpg::PeerArgs peers{};
  bool peer = false;
  int grid_peer = 1;
  long long launches = 0;
  DBuf<char> flush;  // L2 flush scratch (bench)
  DBuf<long long> phase_clk;  // VPINN_PHASE_CLOCK diagnostics
  DBuf<float> tc_scratch;     // tc2 parameter-gradient scratch
  // device-assembly contexts keep the mesh, rule and basis tables: the
  // matrix-free contraction (contract_mf.cuh) works from them
  std::unique_ptr<AsmUpload> asmd;
  DBuf<float> mf_tabs, mf_rule;
  int64_t asm_e0 = 0;
  // strong form (sf_step_kernel.cuh): no tensors, f at the interior points
  bool strong = false;
  DBuf<float> sforce;
  vpg::SfKernels sfk{};
  int sf_warps = 0;
  bool sf_tc = false;               // the tcgen05 strong-form kernel (sfk.tc_*)
  int sf_block = 0, sf_pts = 0;     // its threads per CTA, points per CTA and tile
  long long n_int_global = 0;
  bool tc2 = false;           // fp16-split two-CTA tensor-core step
  bool tc2_lat = false;       // ... in its latency layout (tc2_lat: grids of <= 1 tile per SM)
  bool tc2_modes = false;     // tc2 forward / reverse modes serve the split path and evaluate
  int grid_tc2 = 0;           // 2 CTAs per SM

  ~vpinn_gpu_ctx() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);  // buffers go back to the block cache idle
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (comm && nccl().comm_destroy) nccl().comm_destroy(comm);
    if (peer)
      for (int r = 0; r < peers.world; ++r)
        if (r != rank && peers.box[r]) cudaIpcCloseMemHandle(peers.box[r]);
    if (pbox) cudaFree(pbox);
    if (h_flag) pinned_words().put(h_flag);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

void set_dev(vpinn_gpu_ctx* c) { CK(cudaSetDevice(c->device)); }

// entry points that work on the premultiplier tensors
void weak_only(const vpinn_gpu_ctx* c, const char* what) {
  if (c && c->strong) throw Fail{VPINN_ERR_CONFIG, std::string(what) + ": the context is strong-form (no tensors)"};
}

// strong form: one persistent warp-tiled kernel (1 CTA per SM, as many warps
// as the per-warp layer state fits), then the same reduce + Adam kernels
void configure_strong(vpinn_gpu_ctx* c) {
  vpg::StepArgs& a = c->sargs;
  std::memset(&a, 0, sizeof(a));
  a.E = c->E;
  a.T = c->T;
  a.Q = c->Q;
  a.pts = c->pts.p;
  a.n_int = c->n_int;
  a.n_bnd = c->n_bnd;
  a.n_sen = c->n_sen;
  a.bval = c->bval.p;
  a.sval = c->sval.p;
  a.eps = c->eps;
  a.bx = c->bx;
  a.by = c->by;
  a.eps_source = c->eps_source;
  a.eps_scalar_index = c->eps_idx;
  a.bscale = c->nb_global ? 2.0f * (float)c->tau / (float)c->nb_global : 0.0f;
  a.sscale = c->ns_global ? 2.0f * (float)c->gamma / (float)c->ns_global : 0.0f;
  // losses.hpp:445, 452: inv_n = Real(1)/Real(count), pbar = Real(2)*weight*inv_n*P
  a.inv_ni = c->n_int_global ? 1.0f / (float)c->n_int_global : 0.0f;
  a.rscale_s = (2.0f * 1.0f) * a.inv_ni;
  a.sforce = c->sforce.p;
  a.net = c->net;
  a.params = c->params.p;
  const int D = c->net.n_layers - 1;
  int maxH = 0;
  for (int l = 0; l < D; ++l) maxH = std::max(maxH, c->net.out_w[l]);
  // the tcgen05 strong-form step (sf2_step_kernel.cuh) for 2-3 hidden layers
  // of width <= 31; the warp-tiled mma.sync kernel for the other shapes
  c->sf_tc = c->sfk.tc_fused != nullptr && maxH <= 31 && !(g_test_hooks.load() & VPINN_HOOK_CUDA_CORE_STEP);
  if (c->sf_tc) {
    c->smem_step = c->sfk.tc_smem;
    for (auto fn : {c->sfk.tc_fused, c->sfk.tc_forward}) {
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_step));
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    const int P_local = c->n_int + c->n_bnd + c->n_sen;
    c->grid_step = std::max(1, std::min(c->sm_count, ceil_div(P_local, vpg::kSf2Points)));
    c->grad_rows = c->loss_rows = c->grid_step;
    c->sf_block = vpg::kSf2Threads;
    c->sf_pts = vpg::kSf2Points;
    c->tc_scratch.alloc((size_t)c->grid_step * (D - 1) * 64 * 64, c->stream);
    a.tc_scratch = c->tc_scratch.p;
    a.tc_force_spill = (g_test_hooks.load() & VPINN_HOOK_FORCE_SPILL) ? 1 : 0;
    c->kernel_name = "sf2_step_kernel<" + std::to_string(D) + "," + (c->net.sigmoid ? "sigmoid" : "tanh") +
                     "> (strong form, tcgen05 fp16 split, 256 threads, 1 CTA/SM)";
    c->part_stride = (c->grad_rows + 31) & ~31;
    c->grad_part.alloc((size_t)c->part_stride * c->n_params, c->stream);
    a.part_stride = c->part_stride;
    a.grad_part = c->grad_part.p;
    c->loss_part.alloc((size_t)c->loss_rows * vpg::kLpWords, c->stream);
    a.loss_part = c->loss_part.p;
    c->red.alloc((size_t)c->n_params + vpg::kLpWords, c->stream);
    c->e_scalar.alloc(1, c->stream);
    return;
  }
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  int w = vpg::kSfMaxWarps;
  while (w > 1 && vpg::sf_smem_bytes(D, w) > (size_t)optin) --w;
  if (vpg::sf_smem_bytes(D, w) > (size_t)optin) throw Fail{VPINN_ERR_CONFIG, "strong-form kernel does not fit shared memory"};
  c->sf_warps = w;
  c->sf_block = 32 * w;
  c->sf_pts = 16 * w;
  c->smem_step = vpg::sf_smem_bytes(D, w);
  for (auto fn : {c->sfk.fused, c->sfk.forward}) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_step));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c->sfk.fused, 32 * w, c->smem_step));
  if (occ < 1) throw Fail{VPINN_ERR_DEVICE, "strong-form kernel cannot be resident"};
  const int P_local = c->n_int + c->n_bnd + c->n_sen;
  const int tiles = ceil_div(P_local, 16);
  c->grid_step = std::max(1, std::min(occ * c->sm_count, ceil_div(tiles, w)));
  c->grad_rows = c->loss_rows = c->grid_step;
  c->kernel_name = "sf_step_kernel<" + std::to_string(D) + "," + (c->net.sigmoid ? "sigmoid" : "tanh") +
                   "> (strong form, mma.sync 3xTF32, " + std::to_string(w) + " warps/CTA)";
  c->part_stride = (c->grad_rows + 31) & ~31;
  c->grad_part.alloc((size_t)c->part_stride * c->n_params, c->stream);
  a.part_stride = c->part_stride;
  a.grad_part = c->grad_part.p;
  c->loss_part.alloc((size_t)c->loss_rows * vpg::kLpWords, c->stream);
  a.loss_part = c->loss_part.p;
  c->red.alloc((size_t)c->n_params + vpg::kLpWords, c->stream);
  c->e_scalar.alloc(1, c->stream);
}

// the warp-per-cell contraction: warps per CTA x the cell shape fixed at
// compile time for 5x5 / 5x5 cells (the benchmark gear)
const void* cw_kernel(int nw, bool fixed) {
  if (fixed)
    return nw == 16 ? (const void*)vpg::contract_warp_kernel<16, 25, 25>
                    : (nw == 12 ? (const void*)vpg::contract_warp_kernel<12, 25, 25>
                                : (const void*)vpg::contract_warp_kernel<8, 25, 25>);
  return nw == 16 ? (const void*)vpg::contract_warp_kernel<16>
                  : (nw == 12 ? (const void*)vpg::contract_warp_kernel<12> : (const void*)vpg::contract_warp_kernel<8>);
}

// the warp-owned-row contraction by points per lane (Q <= 32 MQ)
const void* rowreg_kernel(int mq) {  // mq > 0: float4 rows, M4 = mq; mq < 0: scalar, M = -mq
  switch (mq) {
    case 4: return (const void*)vpg::contract_rowreg_kernel<4, true>;
    case 8: return (const void*)vpg::contract_rowreg_kernel<8, true>;
    case 13: return (const void*)vpg::contract_rowreg_kernel<13, true>;
    case -16: return (const void*)vpg::contract_rowreg_kernel<16, false>;
    case -32: return (const void*)vpg::contract_rowreg_kernel<32, false>;
    default: return (const void*)vpg::contract_rowreg_kernel<52, false>;
  }
}
inline long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }

void configure(vpinn_gpu_ctx* c) {
  if (c->strong) {
    configure_strong(c);
    return;
  }
  // ---- fused path when a cell fits a CTA, split path otherwise ----
  const int P_local = c->n_int + c->n_bnd + c->n_sen;
  const Variant& V = c->var;
  // a cell larger than the tensor-core step's tile (the 64 class: 112
  // points) takes the split path too, on its tensor-core modes
  c->split = c->Q > vpg::kThreads ||
             (V.tc2 != nullptr && c->Q > V.tc2_mp && !(g_test_hooks.load() & VPINN_HOOK_CUDA_CORE_STEP));
  vpg::StepArgs& a = c->sargs;
  std::memset(&a, 0, sizeof(a));
  for (int t = 0; t < 3; ++t) a.tens[t] = c->tens[t].p;
  a.forcing = c->forcing.p;
  a.E = c->E;
  a.T = c->T;
  a.Q = c->Q;
  a.nt = c->nt;
  a.pts = c->pts.p;
  a.n_int = c->n_int;
  a.n_bnd = c->n_bnd;
  a.n_sen = c->n_sen;
  a.bval = c->bval.p;
  a.sval = c->sval.p;
  a.eps = c->eps;
  a.bx = c->bx;
  a.by = c->by;
  a.eps_source = c->eps_source;
  a.eps_scalar_index = c->eps_idx;
  a.inv_nt = 1.0f / (float)c->T;
  a.rscale = (2.0f * 1.0f) * a.inv_nt;
  a.bscale = c->nb_global ? 2.0f * (float)c->tau / (float)c->nb_global : 0.0f;
  a.sscale = c->ns_global ? 2.0f * (float)c->gamma / (float)c->ns_global : 0.0f;
  a.net = c->net;
  a.params = c->params.p;

  const size_t two_cta = 113 * 1024;
  int occ = 0;
  // CTAs per SM of a tensor-core step kernel: two when two of them fit the
  // SM's shared memory (width class 32: 113 KB, 256 TMEM columns each), else
  // one (width class 64: ~212 KB, all 512 TMEM columns).  The occupancy query
  // reports 1 for tcgen05 kernels; the hardware co-schedules 2 (measured).
  auto tc2_ctas_per_sm = [&](size_t smem) {
    int smsm = 0, resv = 0;
    CK(cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device));
    CK(cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, c->device));
    return 2 * (smem + resv) <= (size_t)smsm ? 2 : 1;
  };
  // the tensor-core forward / reverse modes (split path, evaluate)
  const bool tc2_modes_ok = V.tc2_fwd != nullptr && !(g_test_hooks.load() & VPINN_HOOK_CUDA_CORE_STEP);
  if (!c->split) {
    // tensor-core step: whole-cell tiles of at most tc2_mp points, the tile's
    // slab plus its contraction scratch in operand buffer A
    // whole cells per tile: as many as the points allow, at most 128 test
    // rows (the contraction's per-row scratch)
    const int tc_cells = V.tc2 ? std::max(1, std::min(V.tc2_mp / c->Q, 128 / std::max(1, c->T))) : 1;
    const int tc_rows = tc_cells * c->T;
    c->tc2 = V.tc2 != nullptr && !(g_test_hooks.load() & VPINN_HOOK_CUDA_CORE_STEP) &&
             c->Q >= 2 && c->Q <= V.tc2_mp &&
             tc_rows <= 128 &&
             (size_t)(c->nt * round4(tc_rows * c->Q + 8) +
                      (V.C == 2 ? vpg::t2::tail_floats<2>() : vpg::t2::tail_floats<1>())) * sizeof(float) <=
                 (size_t)V.tc2_buf;
    a.cells_per_tile = c->tc2 ? tc_cells : std::max(1, vpg::kThreads / c->Q);
    a.n_int_tiles = c->E ? ceil_div(c->E, a.cells_per_tile) : 0;
    a.n_tiles = a.n_int_tiles + ceil_div(c->n_bnd + c->n_sen, c->tc2 ? V.tc2_mp : vpg::kThreads);
    const int tile_rows = a.cells_per_tile * c->T;
    if (c->tc2 && (std::getenv("VPINN_PHASE_CLOCK") && std::atoi(std::getenv("VPINN_PHASE_CLOCK")) != 0)) {
      c->phase_clk.alloc((size_t)vpg::kPhaseTiles * vpg::kPhaseMarks + 3 * 1024, c->stream);
      a.phase_clk = c->phase_clk.p;
    }
    if (c->tc2) {
      a.chunk_rows = tile_rows;
      a.tstride = round4(tile_rows * c->Q + 8);
      a.stage_floats = c->nt * a.tstride;
      a.union_floats = 0;
      c->smem_step = V.tc2_smem;
      CK(cudaFuncSetAttribute(V.tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_step));
      CK(cudaFuncSetAttribute(V.tc2, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.tc2, V.tc2_nt, c->smem_step));
      if (occ < 1) throw Fail{VPINN_ERR_DEVICE, "tc2 step kernel cannot be resident"};
      occ = tc2_ctas_per_sm(c->smem_step);
      c->grid_step = std::max(1, std::min(a.n_tiles, occ * c->sm_count));
      // at most one tile per SM: the latency layout (8 units per thread, 512
      // threads) halves every thread's elementwise chain on the lone tile
      c->tc2_lat = V.tc2_lat != nullptr && a.n_tiles <= c->sm_count &&
                   !(g_test_hooks.load() & VPINN_HOOK_THROUGHPUT_LAYOUT);
      if (c->tc2_lat) {
        c->smem_step = V.tc2_lat_smem;
        CK(cudaFuncSetAttribute(V.tc2_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_step));
        occ = 1;
        c->grid_step = std::max(1, a.n_tiles);
      }
      c->tc_scratch.alloc((size_t)c->grid_step * (V.D - 1) * V.tc2_scratch, c->stream);
      a.tc_scratch = c->tc_scratch.p;
      a.tc_force_spill = (g_test_hooks.load() & VPINN_HOOK_FORCE_SPILL) ? 1 : 0;
      c->kernel_name = "tc2_step_kernel<" + std::to_string(V.H) + "," + std::to_string(V.D) + "," +
                       (V.ACT ? "sigmoid" : "tanh") + (V.C == 2 ? ",2 outputs" : "") + (c->tc2_lat ? ",8 units/thread" : "") +
                       "> (fp16 split, " + std::to_string(c->tc2_lat ? V.tc2_lat_nt : V.tc2_nt) + " threads, " +
                       std::to_string(occ) + " CTA" + (occ > 1 ? "s" : "") + "/SM)";
    } else {
      c->kernel_name = "step_kernel<" + std::to_string(V.H) + "," + std::to_string(V.D) + "," + std::to_string(V.C) +
                       "," + (V.ACT ? "sigmoid" : "tanh") + ",fused> (CUDA cores)";
      const size_t min_smem = V.smem(V.rev_need, 1);
      const size_t budget = min_smem <= two_cta ? two_cta : (size_t)227 * 1024;
      // the whole tile slab in one stage when it fits (one contraction chunk,
      // fewer barriers); otherwise a two-stage ring of half tiles or smaller
      bool single = true;
      int rows = tile_rows;
      for (;;) {
        const int tstride = round4(rows * c->Q + 8);
        const int stage = c->nt * tstride;
        const int uni = std::max(V.rev_need, single ? stage : 2 * stage);
        if (single && V.smem(uni, rows) > budget) {
          single = false;
          rows = (tile_rows + 1) / 2;
          continue;
        }
        if (V.smem(uni, rows) <= budget || rows == 1) {
          a.chunk_rows = rows;
          a.tstride = tstride;
          a.stage_floats = stage;
          a.union_floats = uni;
          break;
        }
        rows = std::max(1, rows * 3 / 4);
      }
      c->smem_step = V.smem(a.union_floats, a.chunk_rows);
      if (c->smem_step > (size_t)227 * 1024)
        throw Fail{VPINN_ERR_CONFIG, "fused step kernel does not fit shared memory"};
      CK(cudaFuncSetAttribute(V.fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_step));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.fused, vpg::kThreads, c->smem_step));
      if (occ < 1) throw Fail{VPINN_ERR_DEVICE, "fused step kernel cannot be resident"};
      c->grid_step = std::max(1, std::min(a.n_tiles, occ * c->sm_count));
    }
    c->grad_rows = c->grid_step;
    c->loss_rows = c->grid_step;
  } else if (!tc2_modes_ok) {
    // reverse kernel over all local points (the tensor-core reverse mode
    // takes this stage when the shape has one, below)
    c->kernel_name = "step_kernel<" + std::to_string(V.H) + "," + std::to_string(V.D) + "," + std::to_string(V.C) +
                     ",reverse> (split path)";
    a.n_tiles = ceil_div(P_local, vpg::kThreads);
    a.chunk_rows = 1;
    a.union_floats = V.rev_need;
    c->smem_step = V.smem(a.union_floats, 1);
    if (c->smem_step > (size_t)227 * 1024)
      throw Fail{VPINN_ERR_CONFIG, "reverse kernel does not fit shared memory"};
    CK(cudaFuncSetAttribute(V.reverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_step));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.reverse, vpg::kThreads, c->smem_step));
    if (occ < 1) throw Fail{VPINN_ERR_DEVICE, "reverse kernel cannot be resident"};
    c->grid_step = std::max(1, std::min(a.n_tiles, occ * c->sm_count));
    c->grad_rows = c->grid_step;
  }

  // ---- tc2 forward / reverse modes (split path, evaluate): any point
  // count, tanh or sigmoid, 2-3 hidden layers of width <= 63, one output ----
  {
    c->tc2_modes = tc2_modes_ok;
    if (c->tc2_modes) {
      for (vpg::StepFn fn : {V.tc2_fwd, V.tc2_rev}) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V.tc2_smem));
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      c->grid_tc2 = tc2_ctas_per_sm(V.tc2_smem) * c->sm_count;
      if (c->split) {
        // the reverse stage on the tensor cores
        a.n_tiles = ceil_div(P_local, V.tc2_mp);
        c->smem_step = V.tc2_smem;
        c->grid_step = std::max(1, std::min(a.n_tiles, c->grid_tc2));
        c->grad_rows = c->grid_step;
        c->tc_scratch.alloc((size_t)c->grid_step * (V.D - 1) * V.tc2_scratch, c->stream);
        a.tc_scratch = c->tc_scratch.p;
        c->kernel_name = "tc2_step_kernel<" + std::to_string(V.H) + "," + std::to_string(V.D) + "," +
                         (V.ACT ? "sigmoid" : "tanh") + ",reverse> (split path, fp16 split)";
      }
    }
  }

  // ---- forward kernel (evaluate; split-path first stage) ----
  // (not needed, and possibly too large, when the tensor-core forward mode serves)
  if (!c->tc2_modes) {
    c->smem_fwd = V.smem(0, 1);
    if (c->smem_fwd > (size_t)227 * 1024) throw Fail{VPINN_ERR_CONFIG, "forward kernel does not fit shared memory"};
    CK(cudaFuncSetAttribute(V.forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_fwd));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.forward, vpg::kThreads, c->smem_fwd));
    c->grid_fwd = std::max(1, occ) * c->sm_count;
  }

  // ---- standalone contraction (split path, roofline) ----
  {
    vpg::ContractArgs& ca = c->cargs;
    std::memset(&ca, 0, sizeof(ca));
    for (int t = 0; t < 3; ++t) ca.tens[t] = c->tens[t].p;
    ca.forcing = c->forcing.p;
    ca.E = c->E;
    ca.T = c->T;
    ca.Q = c->Q;
    ca.nt = c->nt;
    ca.e_fixed = c->eps;
    ca.eps_source = c->eps_source;
    ca.bx = c->bx;
    ca.by = c->by;
    ca.rscale = a.rscale;
    ca.inv_nt = a.inv_nt;
    // two ring stages of R rows (as many as fit ~200 KB, <= 16); items =
    // (cell, segment of seg_rows rows), about four per CTA, contiguous ranges
    if (c->split && c->Q > vpg::kCQMax)
      throw Fail{VPINN_ERR_CONFIG, "contraction: more than 8,192 quadrature points per cell"};
    ca.qstride = round4(c->Q);
    const size_t row_bytes = sizeof(float) * (size_t)c->nt * c->Q;
    const size_t fixed = sizeof(float) * (3 + (size_t)c->nt) * ca.qstride + 1024;
    const size_t ring_budget = (size_t)200 * 1024 > fixed ? (size_t)200 * 1024 - fixed : 0;
    // a 2-deep ring of R-row stages (measured on C3 40x40: 2 x 6 rows 41.7 us,
    // 4 x 3 rows 63.9 us -- each stage costs three CTA barriers and a serial
    // row-finish step, so fewer, larger stages win)
    ca.nstage = 2;
    ca.rows = (int)std::max<size_t>(1, std::min<size_t>({(size_t)vpg::kCRowsMax, (size_t)c->T,
                                                         ring_budget / (ca.nstage * row_bytes + 64)}));
    ca.tstride = round4(ca.rows * c->Q + 8);
    ca.stage_floats = c->nt * ca.tstride;
    c->smem_contract = vpg::contract_rows_smem_bytes(ca.stage_floats, ca.qstride, c->nt, ca.nstage);
    if (c->smem_contract > (size_t)227 * 1024)
      throw Fail{VPINN_ERR_CONFIG, "contraction kernel does not fit shared memory"};
    CK(cudaFuncSetAttribute(vpg::contract_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)c->smem_contract));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vpg::contract_rows_kernel, vpg::kCRThreads,
                                                     c->smem_contract));
    const int ctas = std::max(1, occ) * c->sm_count;
    const long long rows_total = (long long)c->E * c->T;
    const int seg = (int)std::min<long long>(c->T, std::max<long long>(1, (rows_total + 4 * ctas - 1) / (4 * ctas)));
    ca.seg_rows = std::min(c->T, ceil_div(seg, ca.rows) * ca.rows);
    ca.items_per_cell = ceil_div(c->T, ca.seg_rows);
    ca.n_items = c->E * ca.items_per_cell;
    c->grid_contract = std::max(1, std::min(ca.n_items, ctas));
    c->grid_creduce = std::max(1, std::min(ceil_div(c->E * c->Q, 256), 4 * c->sm_count));
    // two premultipliers and at most 52 points per lane: warp-owned rows
    // (contract_rowreg_kernel), one CTA per SM, row-balanced ranges
    ca.rr_mq = 0;
    if (c->nt == 2 && c->Q <= 32 * 52 && rows_total > 0) {
      const bool vec = c->Q % 4 == 0;
      const int m4 = vec ? (c->Q <= 512 ? 4 : (c->Q <= 1024 ? 8 : 13)) : (c->Q <= 512 ? 16 : (c->Q <= 1024 ? 32 : 52));
      const int vp = vpg::rr_pad_points(m4, vec);
      const int rs = round4(vp + 8);
      // row stages per warp: as many as fit (one row in flight per stage)
      int nsw = vpg::kRRMaxStages;
      while (nsw > 1 && vpg::contract_rowreg_smem_bytes(rs, ca.qstride, vp, nsw) > (size_t)227 * 1024) --nsw;
      const size_t smem = vpg::contract_rowreg_smem_bytes(rs, ca.qstride, vp, nsw);
      if (smem <= (size_t)227 * 1024) {
        ca.rr_mq = vec ? m4 : -m4;
        ca.tstride = rs;
        ca.nstage = nsw;
        const void* fn = rowreg_kernel(ca.rr_mq);
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        c->smem_contract = smem;
        c->grid_contract = (int)std::max<long long>(1, std::min<long long>(rows_total, c->sm_count));
        const long long per = ceil_div_ll(rows_total, c->grid_contract);
        ca.items_per_cell = (int)std::min<long long>(c->E, (per + c->T - 1) / c->T + 1);  // segments per CTA
        ca.n_items = c->grid_contract * ca.items_per_cell;
        // per cell: the first covering CTA, the cell's segment index in it, the last covering CTA
        const int G = c->grid_contract;
        auto row0 = [&](int b) { return (long long)(rows_total * b / G); };
        std::vector<int> cov(4 * (size_t)c->E);
        int b = 0;
        for (int k = 0; k < c->E; ++k) {
          const long long g0 = (long long)k * c->T, g1 = g0 + c->T;
          while (b + 1 < G && row0(b + 1) <= g0) ++b;
          int e = b;
          while (e + 1 < G && row0(e + 1) < g1) ++e;
          cov[4 * k] = b;
          cov[4 * k + 1] = (int)(k - row0(b) / c->T);
          cov[4 * k + 2] = e;
          cov[4 * k + 3] = 0;
        }
        c->rr_cover.alloc(cov.size(), c->stream);
        CK(cudaMemcpyAsync(c->rr_cover.p, cov.data(), cov.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
      }
    }
    c->cpart.alloc((size_t)ca.n_items * 3 * ca.qstride, c->stream);
    ca.part = c->cpart.p;
    c->grid_pen = (c->n_bnd + c->n_sen) ? std::min(64, ceil_div(c->n_bnd + c->n_sen, 256)) : 0;
  }
  // ---- whole-cell HBM-streaming contraction (warp per cell) ----
  c->cell_contract = c->E > 0;
  if (c->cell_contract) {
    vpg::CellContractArgs& cc = c->ccargs;
    std::memset(&cc, 0, sizeof(cc));
    for (int t = 0; t < 3; ++t) cc.tens[t] = c->tens[t].p;
    cc.forcing = c->forcing.p;
    cc.E = c->E;
    cc.T = c->T;
    cc.Q = c->Q;
    cc.nt = c->nt;
    cc.cc = 1;
    cc.tstride = round4(c->T * c->Q + 8);
    cc.vstride = round4(c->Q + 8);
    cc.fstride = round4(c->T + 8);
    cc.stage_floats = c->nt * cc.tstride + 3 * cc.vstride + cc.fstride;
    cc.e_fixed = c->eps;
    cc.eps_source = c->eps_source;
    cc.bx = c->bx;
    cc.by = c->by;
    cc.rscale = a.rscale;
    cc.inv_nt = a.inv_nt;
    // the most warps per CTA (8 / 12 / 16) with a >= 2-stage ring each
    const size_t budget = (size_t)227 * 1024 - 1024;
    int nw = 16, ns = 2;
    while (nw > 8 && vpg::cell_warp_smem_bytes(nw, cc.stage_floats, ns, c->T, c->Q) > budget) nw -= 4;
    cc.nstage = ns;
    c->cw_warps = nw;
    c->smem_cc = vpg::cell_warp_smem_bytes(nw, cc.stage_floats, cc.nstage, c->T, c->Q);
    if (c->smem_cc > budget) {
      c->cell_contract = false;  // cell larger than a warp's ring: row-chunked kernel
    } else {
      c->cw_fixed = c->T == 25 && c->Q == 25;
      const void* fn = cw_kernel(nw, c->cw_fixed);
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem_cc));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * nw, c->smem_cc));
      c->grid_cc = std::max(1, std::min(ceil_div(c->E, nw), std::max(1, occ) * c->sm_count));
    }
  }
  if (c->split) c->loss_rows = c->grid_contract + c->grid_pen + c->grid_step;

  // ---- buffers sized by the grids ----
  c->part_stride = (c->grad_rows + 31) & ~31;
  c->grad_part.alloc((size_t)c->part_stride * c->n_params, c->stream);
  a.part_stride = c->part_stride;
  c->loss_part.alloc((size_t)std::max(c->loss_rows, std::max(c->grid_contract, c->grid_cc)) * vpg::kLpWords, c->stream);
  c->red.alloc((size_t)c->n_params + vpg::kLpWords, c->stream);
  a.grad_part = c->grad_part.p;
  if (c->split) {
    const size_t ni = (size_t)c->n_int;
    c->fu.alloc(P_local, c->stream);
    c->fux.alloc(P_local, c->stream);
    c->fuy.alloc(P_local, c->stream);
    c->feps.alloc(P_local, c->stream);
    c->uxb.alloc(ni, c->stream);
    c->uyb.alloc(ni, c->stream);
    c->eb.alloc(ni, c->stream);
    c->ub.alloc((size_t)c->n_bnd + c->n_sen, c->stream);
    a.loss_part = c->loss_part.p + (size_t)(c->grid_contract + c->grid_pen) * vpg::kLpWords;
    a.in_ub = c->ub.p;
    a.in_uxb = c->uxb.p;
    a.in_uyb = c->uyb.p;
    a.in_eb = c->eb.p;
  } else {
    a.loss_part = c->loss_part.p;
  }
  c->e_scalar.alloc(1, c->stream);
}

// kernel launch with the programmatic-dependent-launch attribute when pdl:
// the kernel (which starts with pdl_trigger / pdl_wait) is scheduled while
// its predecessor's tail runs, hiding the launch latency between the
// epoch's kernels
template <typename... KArgs, typename... Args>
void launch_k(bool pdl, void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// programmatic dependent launch: the tensor-core step triggers its dependents
// after its tile loop (VPG_PDL_LATE), so the reduce + Adam kernel launches
// while the step CTAs write their outputs and the next epoch's step launches
// while Adam runs.  A/B (C5 gear epoch, C2 1-64 cells): 1-3% faster than no
// PDL; an early trigger (at kernel entry) was 1% slower on the gear.
constexpr bool pdl_enabled() { return true; }

void launch_fused(vpinn_gpu_ctx* c, const vpg::StepArgs& a) {
  if (c->strong)
    launch_k(pdl_enabled(), c->sf_tc ? c->sfk.tc_fused : c->sfk.fused, c->grid_step, c->sf_block, c->smem_step,
             c->stream, a);
  else if (c->tc2)
    launch_k(pdl_enabled(), c->tc2_lat ? c->var.tc2_lat : c->var.tc2, c->grid_step,
             c->tc2_lat ? c->var.tc2_lat_nt : c->var.tc2_nt, c->smem_step, c->stream, a);
  else
    c->var.fused<<<c->grid_step, vpg::kThreads, c->smem_step, c->stream>>>(a);
  CK(cudaGetLastError());
  c->launches += 1;
}

// ---- one epoch: loss + gradient (+ Adam) enqueued on the context stream ----
// row-block contraction (cells larger than a warp's ring): items, then the
// fixed-order reduction of their partial adjoint columns
void launch_contract_rows(vpinn_gpu_ctx* c, const vpg::ContractArgs& ca) {
  if (ca.n_items <= 0) return;
  if (ca.rr_mq) {
    auto fn = reinterpret_cast<void (*)(vpg::ContractArgs)>(const_cast<void*>(rowreg_kernel(ca.rr_mq)));
    fn<<<c->grid_contract, vpg::kRRThreads, c->smem_contract, c->stream>>>(ca);
    CK(cudaGetLastError());
    if (c->contract_mid) CK(cudaEventRecord(c->contract_mid, c->stream));
    vpg::contract_rowreg_reduce_kernel<<<c->grid_creduce, 256, 0, c->stream>>>(
        ca, reinterpret_cast<const int4*>(c->rr_cover.p));
    CK(cudaGetLastError());
    c->launches += 2;
    return;
  }
  vpg::contract_rows_kernel<<<c->grid_contract, vpg::kCRThreads, c->smem_contract, c->stream>>>(ca);
  CK(cudaGetLastError());
  if (c->contract_mid) CK(cudaEventRecord(c->contract_mid, c->stream));
  vpg::contract_rows_reduce_kernel<<<c->grid_creduce, 256, 0, c->stream>>>(ca);
  CK(cudaGetLastError());
  c->launches += 2;
}

vpg::AdamArgs adam_args(vpinn_gpu_ctx* c, bool tables, float lr_const, bool records, int rec_cap);

void enqueue_grad(vpinn_gpu_ctx* c, const int* stop, bool with_reduce = true) {
  const Variant& V = c->var;
  vpg::StepArgs a = c->sargs;
  a.stop_flag = stop;
  if (!c->split) {
    launch_fused(c, a);
  } else {
    const int P_local = c->n_int + c->n_bnd + c->n_sen;
    vpg::StepArgs f = a;
    f.fwd_pts = c->pts.p;
    f.n_fwd = P_local;
    f.out_u = c->fu.p;
    f.out_ux = c->fux.p;
    f.out_uy = c->fuy.p;
    f.out_eps = c->feps.p;
    f.union_floats = 0;
    if (c->tc2_modes) {
      const int grid_f = std::max(1, std::min(c->grid_tc2, ceil_div(P_local, V.tc2_mp)));
      V.tc2_fwd<<<grid_f, V.tc2_nt, V.tc2_smem, c->stream>>>(f);
    } else {
      const int grid_f = std::max(1, std::min(c->grid_fwd, ceil_div(P_local, vpg::kThreads)));
      V.forward<<<grid_f, vpg::kThreads, c->smem_fwd, c->stream>>>(f);
    }
    CK(cudaGetLastError());
    vpg::ContractArgs ca = c->cargs;
    ca.ux = c->fux.p;
    ca.uy = c->fuy.p;
    ca.eps = c->feps.p;
    ca.uxb = c->uxb.p;
    ca.uyb = c->uyb.p;
    ca.eb = c->eb.p;
    ca.e_param = c->params.p + c->net.scal_off + c->eps_idx;
    ca.loss_part = c->loss_part.p;
    ca.stop_flag = stop;
    c->launches += 1;
    launch_contract_rows(c, ca);
    if (c->grid_pen) {
      vpg::penalty_kernel<<<c->grid_pen, 256, 0, c->stream>>>(
          c->fu.p + c->n_int, c->n_bnd, c->n_sen, c->bval.p, c->sval.p, a.bscale, a.sscale,
          c->ub.p, c->loss_part.p + (size_t)c->grid_contract * vpg::kLpWords, stop);
      CK(cudaGetLastError());
      c->launches += 1;
    }
    if (c->tc2_modes)
      V.tc2_rev<<<c->grid_step, V.tc2_nt, c->smem_step, c->stream>>>(a);
    else
      V.reverse<<<c->grid_step, vpg::kThreads, c->smem_step, c->stream>>>(a);
    CK(cudaGetLastError());
    c->launches += 1;
  }
  if (!with_reduce) return;
  if (c->peer) {  // this rank's sum and the cross-rank sum in one kernel
    launch_k(pdl_enabled() && !c->split, vpg::reduce_adam_peer_kernel, c->grid_peer,
             vpg::kRAThreads, 0, c->stream, c->grad_part.p, c->grad_rows, c->part_stride, c->n_params,
             (const double*)c->loss_part.p, c->loss_rows, c->red.p, c->ticket.p, c->adam_bk.p,
             adam_args(c, false, 0.f, false, 0), c->peers, 0, stop);
    CK(cudaGetLastError());
    c->launches += 1;
    return;
  }
  vpg::reduce_kernel<<<vpg::reduce_grid(c->n_params), vpg::kRedThreads, 0, c->stream>>>(
      c->grad_part.p, c->grad_rows, c->part_stride, c->n_params, c->loss_part.p, c->loss_rows, c->red.p, stop);
  CK(cudaGetLastError());
  c->launches += 1;
  if (c->comm)
    NK(nccl().all_reduce(c->red.p, c->red.p, (size_t)c->n_params + vpg::kLpWords, ncclFloat64,
                         ncclSum, c->comm, c->stream));
}

vpg::AdamArgs adam_args(vpinn_gpu_ctx* c, bool tables, float lr_const, bool records,
                        int rec_cap) {
  vpg::AdamArgs aa{};
  aa.red = c->red.p;
  aa.n_params = c->n_params;
  aa.params = c->params.p;
  aa.m = c->m.p;
  aa.v = c->v.p;
  aa.st = c->st.p;
  aa.lr_tab = tables ? c->lr_tab.p : nullptr;
  aa.c1_tab = tables ? c->c1_tab.p : nullptr;
  aa.c2_tab = tables ? c->c2_tab.p : nullptr;
  aa.lr_const = lr_const;
  aa.rec = records ? c->rec.p : nullptr;
  aa.rec_cap = rec_cap;
  aa.n_bnd = (double)c->nb_global;
  aa.n_sen = (double)c->ns_global;
  aa.tau_f = (float)c->tau;
  aa.gamma_f = (float)c->gamma;
  aa.eps_grad_slot = c->eps_source == VPINN_EPS_SCALAR ? c->net.scal_off + c->eps_idx : -1;
  return aa;
}

void enqueue_epoch(vpinn_gpu_ctx* c, const vpg::AdamArgs& aa) {
  if (c->peer) {
    // reduce, the cross-rank sum over peer memory and Adam: one kernel
    enqueue_grad(c, &c->st.p->stopped, /*with_reduce=*/false);
    launch_k(pdl_enabled() && !c->split, vpg::reduce_adam_peer_kernel, c->grid_peer,
             vpg::kRAThreads, 0, c->stream, (const float*)c->grad_part.p, c->grad_rows, c->part_stride, c->n_params,
             (const double*)c->loss_part.p, c->loss_rows, c->red.p, c->ticket.p, c->adam_bk.p, aa, c->peers, 1,
             (const int*)&c->st.p->stopped);
    CK(cudaGetLastError());
    c->launches += 1;
    return;
  }
  if (c->comm) {
    // reduce -> ncclAllReduce -> Adam (the all-reduce sits between them)
    enqueue_grad(c, &c->st.p->stopped);
    vpg::adam_kernel<<<1, 1024, 0, c->stream>>>(aa);
    CK(cudaGetLastError());
    c->launches += 1;
    return;
  }
  enqueue_grad(c, &c->st.p->stopped, /*with_reduce=*/false);
  const float* gp = c->grad_part.p;
  const double* lp = c->loss_part.p;
  launch_k(pdl_enabled() && !c->split, vpg::reduce_adam_kernel, vpg::reduce_adam_grid(c->n_params), vpg::kRAThreads,
           0, c->stream, gp, c->grad_rows, c->part_stride, c->n_params, lp, c->loss_rows, c->red.p, c->ticket.p,
           c->adam_bk.p, aa);
  CK(cudaGetLastError());
  c->launches += 1;
}

void reset_state(vpinn_gpu_ctx* c, long long iterations, const vpinn_gpu_train_spec* spec) {
  vpg::TrainState s{};
  s.step = 0;
  s.iterations = iterations;
  s.stopped = 0;
  s.stop_reason = 0;
  s.best_loss = std::numeric_limits<double>::infinity();
  s.best_step = 0;
  s.tracks_eps = c->eps_source == VPINN_EPS_SCALAR;
  s.eps_slot = c->net.scal_off + c->eps_idx;
  if (spec) {
    s.has_eps_tol = spec->has_eps_abs_tol;
    s.has_eps_actual = spec->has_eps_actual;
    s.has_loss_tol = spec->has_loss_tol;
    s.eps_abs_tol = spec->eps_abs_tol;
    s.eps_actual = spec->eps_actual;
    s.loss_tol = spec->loss_tol;
    s.plateau_window = spec->plateau_window;
  }
  CK(cudaMemcpyAsync(c->st.p, &s, sizeof(s), cudaMemcpyHostToDevice, c->stream));
  c->resume_pending = false;
  c->aborted_at = 0;
  CK(cudaMemsetAsync(c->m.p, 0, sizeof(float) * c->n_params, c->stream));
  CK(cudaMemsetAsync(c->v.p, 0, sizeof(float) * c->n_params, c->stream));
  vpg::mark_start_kernel<<<1, 1, 0, c->stream>>>(c->st.p);
  CK(cudaGetLastError());
}

cudaGraphExec_t graph_for(vpinn_gpu_ctx* c, int kind, int steps, double lr, bool tables,
                          int rec_cap) {
  auto key = std::make_tuple(kind, steps, lr);
  auto it = c->graphs.find(key);
  if (it != c->graphs.end()) return it->second;
  const vpg::AdamArgs aa = adam_args(c, tables, (float)lr, tables, rec_cap);
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const long long before = c->launches;
  for (int s = 0; s < steps; ++s) enqueue_epoch(c, aa);
  c->launches = before;  // counted at replay
  CK(cudaStreamEndCapture(c->stream, &g));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  c->graphs[key] = ex;
  return ex;
}

// standalone contraction on device-resident derivatives: the whole-cell
// streaming kernel when a cell fits a CTA, the generic row-chunked one else.
// Returns the number of loss rows written.
int launch_contract(vpinn_gpu_ctx* c, const float* ux, const float* uy, const float* eps, float* uxb,
                    float* uyb, float* eb, float* res, const float* e_param, float rscale, double* loss_part,
                    const int* stop) {
  if (c->cell_contract) {
    vpg::CellContractArgs a = c->ccargs;
    a.ux = ux;
    a.uy = uy;
    a.eps = eps;
    a.uxb = uxb;
    a.uyb = uyb;
    a.eb = eb;
    a.res = res;
    a.e_param = e_param;
    a.rscale = rscale;
    a.loss_part = loss_part;
    a.stop_flag = stop;
    auto fn = reinterpret_cast<void (*)(vpg::CellContractArgs)>(const_cast<void*>(cw_kernel(c->cw_warps, c->cw_fixed)));
    fn<<<c->grid_cc, 32 * c->cw_warps, c->smem_cc, c->stream>>>(a);
    CK(cudaGetLastError());
    c->launches += 1;
    return c->grid_cc;
  }
  vpg::ContractArgs ca = c->cargs;
  ca.ux = ux;
  ca.uy = uy;
  ca.eps = eps;
  ca.uxb = uxb;
  ca.uyb = uyb;
  ca.eb = eb;
  ca.res = res;
  ca.e_param = e_param;
  ca.rscale = rscale;
  ca.loss_part = loss_part;
  ca.stop_flag = stop;
  launch_contract_rows(c, ca);
  return c->grid_contract;
}

// L2 flush between timed launches: write a 256 MB buffer (> 126 MB L2), then
// read it back so the write-back of the dirty lines happens here and not
// inside the next timed kernel.
void flush_l2_now(vpinn_gpu_ctx* c, char* buf) {
  const size_t bytes = (size_t)256 << 20;
  CK(cudaMemsetAsync(buf, (int)(c->launches & 0xff), bytes, c->stream));
  vpg::flush_read_kernel<<<4 * c->sm_count, 512, 0, c->stream>>>(reinterpret_cast<const int4*>(buf), bytes / 16,
                                                                 reinterpret_cast<int*>(buf));
  CK(cudaGetLastError());
}

long long launches_per_epoch(const vpinn_gpu_ctx* c) {
  // step kernel(s) + reduce + adam (fused into one kernel without a communicator)
  long long n = c->comm ? 3 : 2;
  if (c->split) n += 1 + 2 * (c->cargs.n_items > 0) + (c->grid_pen > 0);  // forward, contraction (2), penalty
  return n;
}

}  // namespace

// ===========================================================================

extern "C" {

const char* vpinn_gpu_last_error(void) { return g_err.c_str(); }

const char* vpinn_gpu_version(void) { return "vpinn-b200 0.1 (sm_100a)"; }

const char* vpinn_gpu_step_kernel(const vpinn_gpu_ctx* c) {
  if (!c) return "";
  return c->kernel_name.c_str();
}

void vpinn_gpu_partition(int64_t n_elem, int64_t n_boundary, int64_t n_sensors, int rank, int world,
                         int64_t* out6) {
  const int64_t W = world < 1 ? 1 : world, r = rank;
  out6[0] = n_elem * r / W;
  out6[1] = n_elem * (r + 1) / W;
  out6[2] = n_boundary * r / W;
  out6[3] = n_boundary * (r + 1) / W;
  out6[4] = n_sensors * r / W;
  out6[5] = n_sensors * (r + 1) / W;
}

int vpinn_gpu_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return 0;
  return p.major == 10 ? 1 : 0;
}

int vpinn_gpu_create(const vpinn_gpu_problem* pb, vpinn_gpu_ctx** out) {
  if (out) *out = nullptr;
  return guarded([&] {
    if (!pb || !out) throw Fail{VPINN_ERR_CONFIG, "vpinn_gpu_create: null argument"};
    // ---- validation (contract checks of losses.hpp:70-84, network.hpp:66-76) ----
    if (pb->n_elem < 1 || pb->n_test < 1 || pb->n_quad < 1)
      throw Fail{VPINN_ERR_CONFIG, "n_elem, n_test, n_quad must be >= 1"};
    if (pb->form != VPINN_FORM_WEAK && pb->form != VPINN_FORM_STRONG)
      throw Fail{VPINN_ERR_CONFIG, "form must be weak or strong"};
    const bool strong = pb->form == VPINN_FORM_STRONG;
    if (!strong && !pb->assembly && (!pb->grad_x || !pb->grad_y || !pb->forcing || !pb->points))
      throw Fail{VPINN_ERR_NUMERIC, "tensor kernel: tensors/forcing/points missing"};
    if (strong && !pb->assembly && (!pb->strong_forcing || !pb->points))
      throw Fail{VPINN_ERR_NUMERIC, "strong residual: forcing/points missing"};
    if (pb->n_interior != (int64_t)pb->n_elem * pb->n_quad)
      throw Fail{VPINN_ERR_NUMERIC, "evaluation does not cover the interior quadrature points"};
    if (pb->n_layer_sizes < 3 || pb->n_layer_sizes > vpg::kMaxLayers)
      throw Fail{VPINN_ERR_CONFIG, "layer_sizes: need [2, hidden..., n_out]"};
    std::vector<int> sizes(pb->layer_sizes, pb->layer_sizes + pb->n_layer_sizes);
    if (sizes.front() != 2) throw Fail{VPINN_ERR_CONFIG, "init_network: input dimension must be 2"};
    for (int s : sizes)
      if (s < 1) throw Fail{VPINN_ERR_CONFIG, "init_network: layer sizes must be >= 1"};
    const int D = (int)sizes.size() - 2, C = sizes.back();
    int maxH = 0;
    for (int l = 1; l <= D; ++l) maxH = std::max(maxH, sizes[l]);
    if (pb->eps_source == VPINN_EPS_SPATIAL && C < 2)
      throw Fail{VPINN_ERR_NUMERIC, "spatial coefficient requested but the network has no positive head"};
    if (pb->eps_source == VPINN_EPS_SCALAR &&
        (pb->eps_scalar_index < 0 || pb->eps_scalar_index >= pb->n_scalars))
      throw Fail{VPINN_ERR_NUMERIC, "coefficient scalar index out of range"};
    if (pb->activation != VPINN_ACT_TANH && pb->activation != VPINN_ACT_SIGMOID)
      throw Fail{VPINN_ERR_CONFIG, "activation must be tanh or sigmoid"};
    const Variant* var = nullptr;
    const int act = pb->activation == VPINN_ACT_SIGMOID ? 1 : 0;
    for (const auto& v : variants())
      if (v.D == D && v.C == C && v.ACT == act && v.H >= maxH && (!var || v.H < var->H)) var = &v;
    if (strong) {
      // losses.hpp:437-441 and the strong-form kernel's shape range
      if (pb->eps_source == VPINN_EPS_SPATIAL)
        throw Fail{VPINN_ERR_NUMERIC, "strong residual does not support a spatial coefficient"};
      if (C != 1) throw Fail{VPINN_ERR_CONFIG, "strong form on the GPU path: one output channel"};
      if (maxH > 32 || D > 4)
        throw Fail{VPINN_ERR_CONFIG, "strong form on the GPU path: hidden widths <= 32, at most 4 hidden layers"};
    } else if (!var)
      throw Fail{VPINN_ERR_CONFIG, "network shape not instantiated for the GPU path (hidden layers " +
                                       std::to_string(D) + ", width " + std::to_string(maxH) +
                                       ", outputs " + std::to_string(C) + ", activation " +
                                       (act ? "sigmoid" : "tanh") + ")"};
    const bool conv = pb->bx != 0.0f || pb->by != 0.0f;
    if (!strong && conv && !pb->test && !pb->assembly) throw Fail{VPINN_ERR_NUMERIC, "convection needs the test tensor"};
    const int W = std::max(1, pb->world_size), R = pb->rank;
    if (R < 0 || R >= W) throw Fail{VPINN_ERR_CONFIG, "rank out of range"};

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
      cudaGetLastError();
      throw Fail{VPINN_ERR_DEVICE, "no CUDA device: the B200 path has no CPU fallback"};
    }
    if (pb->device < 0 || pb->device >= ndev) throw Fail{VPINN_ERR_DEVICE, "device ordinal out of range"};

    // VPINN_CREATE_TIMING=1: phase wall times of this call on stderr
    const bool timing = std::getenv("VPINN_CREATE_TIMING") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto t_start = tnow();
    auto mark = [&](const char* what, cudaStream_t st) {
      if (!timing) return;
      if (st) cudaStreamSynchronize(st);
      const auto t = tnow();
      std::fprintf(stderr, "create: %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_start).count());
      t_start = t;
    };
    auto c = std::make_unique<vpinn_gpu_ctx>();
    c->device = pb->device;
    set_dev(c.get());
    // attribute queries, not cudaGetDeviceProperties (~2 ms per call)
    int cc_major = 0;
    CK(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, c->device));
    if (cc_major != 10) {
      cudaDeviceProp prop;
      CK(cudaGetDeviceProperties(&prop, c->device));
      throw Fail{VPINN_ERR_DEVICE, std::string("device ") + prop.name + " is not sm_100 (B200)"};
    }
    CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    mark("device + stream", c->stream);
    c->h_flag = pinned_words().get();
    if (!c->h_flag) throw Fail{VPINN_ERR_DEVICE, "pinned host allocation failed"};
    if (var) c->var = *var;
    c->strong = strong;
    if (strong) {
      c->sfk = vpg::sf_kernels(D, act);
      if (!c->sfk.fused) throw Fail{VPINN_ERR_CONFIG, "strong form: no kernel for this depth"};
    }
    c->n_int_global = pb->n_interior;

    // ---- network descriptor (network.hpp:98-128 offsets) ----
    vpg::NetDesc& nd = c->net;
    std::memset(&nd, 0, sizeof(nd));
    nd.n_layers = (int)sizes.size() - 1;
    int off = 0;
    for (int l = 0; l < nd.n_layers; ++l) {
      nd.in_w[l] = sizes[l];
      nd.out_w[l] = sizes[l + 1];
      nd.w_off[l] = off;
      off += sizes[l + 1] * sizes[l];
      nd.b_off[l] = off;
      off += sizes[l + 1];
    }
    nd.scal_off = off;
    nd.n_params = off + pb->n_scalars;
    nd.sigmoid = pb->activation == VPINN_ACT_SIGMOID;
    c->n_params = nd.n_params;

    // ---- partition (rank r owns contiguous cells / penalty points) ----
    const long long E = pb->n_elem, NB = pb->n_boundary, NS = pb->n_sensors;
    int64_t part[6];
    vpinn_gpu_partition(E, NB, NS, R, W, part);
    const long long e0 = part[0], e1 = part[1], b0 = part[2], b1 = part[3], s0 = part[4], s1 = part[5];
    c->E = (int)(e1 - e0);
    c->T = pb->n_test;
    c->Q = pb->n_quad;
    c->nt = conv ? 3 : 2;
    c->n_int = (int)((e1 - e0) * pb->n_quad);
    c->n_bnd = (int)(b1 - b0);
    c->n_sen = (int)(s1 - s0);
    c->nb_global = NB;
    c->ns_global = NS;
    c->eps = pb->eps;
    c->bx = pb->bx;
    c->by = pb->by;
    c->eps_source = pb->eps_source;
    c->eps_idx = pb->eps_scalar_index;
    c->tau = pb->tau;
    c->gamma = pb->gamma;
    c->rank = R;
    c->nranks = W;

    const size_t TQ = (size_t)c->T * c->Q;
    // points: cast double -> Real exactly like points_to_matrix (network.hpp:376-384)
    std::vector<float2> hp;
    hp.reserve((size_t)c->n_int + c->n_bnd + c->n_sen);
    auto push = [&](long long i) {
      hp.push_back(make_float2((float)pb->points[2 * i], (float)pb->points[2 * i + 1]));
    };
    if (!strong) {
      for (int t = 0; t < c->nt; ++t) c->tens[t].alloc(TQ * c->E, c->stream);
      c->forcing.alloc((size_t)c->T * c->E, c->stream);
    }
    if (!pb->assembly) {
      const float* src[3] = {pb->grad_x, pb->grad_y, pb->test};
      if (!strong) {
        for (int t = 0; t < c->nt; ++t) c->tens[t].upload(src[t] + TQ * e0, TQ * c->E, c->stream);
        c->forcing.upload(pb->forcing + (size_t)c->T * e0, (size_t)c->T * c->E, c->stream);
      } else {
        // commands.hpp:147-152: this rank's slice of f at the interior points
        c->sforce.alloc((size_t)c->n_int, c->stream);
        c->sforce.upload(pb->strong_forcing + e0 * pb->n_quad, (size_t)c->n_int, c->stream);
      }
      for (long long i = e0 * pb->n_quad; i < e1 * pb->n_quad; ++i) push(i);
      for (long long i = b0; i < b1; ++i) push(pb->n_interior + i);
      for (long long i = s0; i < s1; ++i) push(pb->n_interior + NB + i);
      c->pts.alloc(hp.size(), c->stream);
      c->pts.upload(hp.data(), hp.size(), c->stream);
    } else {
      // device-side assembly of this rank's cells straight into the buffers;
      // the interior points land in the head of the evaluation batch
      for (long long i = b0; i < b1; ++i) push(i);
      for (long long i = s0; i < s1; ++i) push(NB + i);
      c->pts.alloc((size_t)c->n_int + hp.size(), c->stream);
      c->pts.upload_at(c->n_int, hp.data(), hp.size(), c->stream);
      c->asmd = std::make_unique<AsmUpload>();
      AsmUpload& up = *c->asmd;
      up.load(pb->assembly, pb->n_elem, c->T, c->Q, c->stream);
      c->asm_e0 = e0;
      {
        // float copies of the basis tables and the rule for the matrix-free contraction
        const size_t TQ = (size_t)c->T * c->Q;
        std::vector<float> tabs(3 * TQ), rule(3 * (size_t)c->Q);
        for (size_t i = 0; i < TQ; ++i) {
          tabs[i] = (float)pb->assembly->basis_dxi[i];
          tabs[TQ + i] = (float)pb->assembly->basis_deta[i];
          tabs[2 * TQ + i] = (float)pb->assembly->basis_val[i];
        }
        for (int q = 0; q < c->Q; ++q) {
          rule[q] = (float)pb->assembly->xi[q];
          rule[c->Q + q] = (float)pb->assembly->eta[q];
          rule[2 * c->Q + q] = (float)pb->assembly->weights[q];
        }
        c->mf_tabs.alloc(tabs.size(), c->stream);
        c->mf_tabs.upload(tabs.data(), tabs.size(), c->stream);
        c->mf_rule.alloc(rule.size(), c->stream);
        c->mf_rule.upload(rule.data(), rule.size(), c->stream);
        CK(cudaStreamSynchronize(c->stream));  // host staging vectors go out of scope
      }
      DBuf<float> tv_tmp, fq, gx_tmp, gy_tmp;
      if (!strong) {
        float* tv = c->nt == 3 ? c->tens[2].p : nullptr;
        if (!tv) {
          tv_tmp.alloc(TQ * c->E, c->stream);
          tv = tv_tmp.p;
        }
        fq.alloc((size_t)c->n_int, c->stream);
        CK(vpg::assemble_on_device(up.in, e0, c->E, c->tens[0].p, c->tens[1].p, tv, c->forcing.p, nullptr,
                                   c->pts.p, fq.p, up.bad.p, c->stream));
      } else {
        // the points and f at them ((float)f(x_q), commands.hpp:147-152); the
        // premultipliers are built and dropped (the geometry checks still run)
        gx_tmp.alloc(TQ * c->E, c->stream);
        gy_tmp.alloc(TQ * c->E, c->stream);
        c->sforce.alloc((size_t)c->n_int, c->stream);
        CK(vpg::assemble_on_device(up.in, e0, c->E, gx_tmp.p, gy_tmp.p, nullptr, nullptr, nullptr, c->pts.p,
                                   c->sforce.p, up.bad.p, c->stream));
      }
      up.check(c->stream);
    }
    std::vector<float> bv, sv;
    for (long long i = b0; i < b1; ++i) bv.push_back((float)pb->boundary_values[i]);
    for (long long i = s0; i < s1; ++i) sv.push_back((float)pb->sensor_values[i]);
    c->bval.alloc(bv.size(), c->stream);
    c->bval.upload(bv.data(), bv.size(), c->stream);
    c->sval.alloc(sv.size(), c->stream);
    c->sval.upload(sv.data(), sv.size(), c->stream);

    c->params.alloc(c->n_params, c->stream);
    c->m.alloc(c->n_params, c->stream);
    c->v.alloc(c->n_params, c->stream);
    c->st.alloc(1, c->stream);
    c->ticket.alloc(3, c->stream);
    c->adam_bk.alloc(3 * (size_t)c->n_params, c->stream);
    mark("uploads", c->stream);
    configure(c.get());
    mark("configure", c->stream);
    reset_state(c.get(), LLONG_MAX, nullptr);
    CK(cudaStreamSynchronize(c->stream));
    *out = c.release();
  });
}

void vpinn_gpu_destroy(vpinn_gpu_ctx* ctx) { delete ctx; }

int vpinn_gpu_param_count(const vpinn_gpu_ctx* ctx) { return ctx ? ctx->n_params : -1; }

int vpinn_gpu_set_params(vpinn_gpu_ctx* c, const float* p, int n) {
  return guarded([&] {
    if (n != c->n_params) throw Fail{VPINN_ERR_NUMERIC, "from_parameters: size mismatch"};
    set_dev(c);
    CK(cudaMemcpyAsync(c->params.p, p, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vpinn_gpu_get_params(vpinn_gpu_ctx* c, float* p, int n) {
  return guarded([&] {
    if (n != c->n_params) throw Fail{VPINN_ERR_NUMERIC, "to_parameters: size mismatch"};
    set_dev(c);
    CK(cudaMemcpyAsync(p, c->params.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vpinn_gpu_loss_and_grad(vpinn_gpu_ctx* c, double* loss_parts, double* grad) {
  return guarded([&] {
    set_dev(c);
    enqueue_grad(c, nullptr);
    std::vector<double> red(c->n_params + vpg::kLpWords);
    CK(cudaMemcpyAsync(red.data(), c->red.p, sizeof(double) * red.size(), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const double* lw = red.data() + c->n_params;
    if (lw[vpg::kLpBad] != 0.0)
      throw Fail{VPINN_ERR_NUMERIC, "evaluate: non-finite network output"};
    const float Lv = (float)lw[vpg::kLpVar];
    const float Lb = c->nb_global ? (float)(lw[vpg::kLpBnd] / (double)c->nb_global) : 0.0f;
    const float Ls = c->ns_global ? (float)(lw[vpg::kLpSen] / (double)c->ns_global) : 0.0f;
    if (loss_parts) {
      loss_parts[0] = (double)(Lv + (float)c->tau * Lb + (float)c->gamma * Ls);
      loss_parts[1] = lw[vpg::kLpVar];
      loss_parts[2] = c->nb_global ? lw[vpg::kLpBnd] / (double)c->nb_global : 0.0;
      loss_parts[3] = c->ns_global ? lw[vpg::kLpSen] / (double)c->ns_global : 0.0;
    }
    if (grad) {
      for (int p = 0; p < c->n_params; ++p) grad[p] = red[p];
      if (c->eps_source == VPINN_EPS_SCALAR) grad[c->net.scal_off + c->eps_idx] += lw[vpg::kLpEpsGrad];
    }
  });
}

int vpinn_gpu_adam_reset(vpinn_gpu_ctx* c) {
  return guarded([&] {
    set_dev(c);
    reset_state(c, LLONG_MAX, nullptr);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int vpinn_gpu_run_steps(vpinn_gpu_ctx* c, int n_steps, double lr) {
  return guarded([&] {
    set_dev(c);
    if (c->aborted_at > 0)
      throw Fail{VPINN_ERR_NUMERIC, "run_steps: the last train() aborted at step " + std::to_string(c->aborted_at) +
                                        "; call vpinn_gpu_adam_reset first"};
    if (n_steps <= 0) return;
    if (c->resume_pending) {
      vpg::resume_kernel<<<1, 1, 0, c->stream>>>(c->st.p);
      CK(cudaGetLastError());
      c->resume_pending = false;
    }
    const int chunk = std::min(n_steps, 64);
    cudaGraphExec_t g = graph_for(c, 1, chunk, lr, false, 0);
    int done = 0;
    while (done + chunk <= n_steps) {
      CK(cudaGraphLaunch(g, c->stream));
      c->launches += launches_per_epoch(c) * chunk;
      done += chunk;
    }
    if (done < n_steps) {
      cudaGraphExec_t g2 = graph_for(c, 1, n_steps - done, lr, false, 0);
      CK(cudaGraphLaunch(g2, c->stream));
      c->launches += launches_per_epoch(c) * (n_steps - done);
    }
  });
}

int vpinn_gpu_synchronize(vpinn_gpu_ctx* c) {
  return guarded([&] {
    set_dev(c);
    CK(cudaStreamSynchronize(c->stream));
    vpg::TrainState s;
    CK(cudaMemcpy(&s, c->st.p, sizeof(s), cudaMemcpyDeviceToHost));
    if (s.stopped && s.stop_reason == 3)
      throw Fail{VPINN_ERR_NUMERIC, "step " + std::to_string(s.abort_step) + ": non-finite gradient"};
  });
}

int vpinn_gpu_time_steps(vpinn_gpu_ctx* c, int n_steps, double lr, double* ms_total) {
  return guarded([&] {
    set_dev(c);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c->stream));
    if (vpinn_gpu_run_steps(c, n_steps, lr) != 0) throw Fail{VPINN_ERR_DEVICE, g_err};
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_total = ms;
  });
}

namespace {
constexpr long long kGraphMinIters = 256;  // vpinn_gpu_train: shorter first runs launch directly
}

int vpinn_gpu_train(vpinn_gpu_ctx* c, const vpinn_gpu_train_spec* spec,
                    vpinn_gpu_step_record* records, vpinn_gpu_train_result* result) {
  return guarded([&] {
    if (!spec || spec->iterations < 1)
      throw Fail{VPINN_ERR_CONFIG, "train: iterations must be >= 1"};
    if (spec->lr_exponential && spec->every < 1)
      throw Fail{VPINN_ERR_CONFIG, "lr_at: every must be >= 1"};
    set_dev(c);
    const long long iters = spec->iterations;
    if (iters > INT_MAX / 2) throw Fail{VPINN_ERR_CONFIG, "train: iteration budget too large"};
    // lr_at (trainer.hpp:73-78) and the bias corrections (trainer.hpp:49-52),
    // double pow then cast, exactly as the reference computes them
    std::vector<float> lr(iters), c1(iters), c2(iters);
    for (long long t = 1; t <= iters; ++t) {
      const double l = spec->lr_exponential
                           ? spec->lr0 * std::pow(spec->decay, double((t - 1) / spec->every))
                           : spec->lr0;
      lr[t - 1] = (float)l;
      c1[t - 1] = 1.0f - (float)std::pow(0.9, double(t));
      c2[t - 1] = 1.0f - (float)std::pow(0.999, double(t));
    }
    // the tables and the record buffer keep their device addresses across
    // calls (capacity grows to a power of two): the captured epoch graphs
    // stay valid, so a repeated train() does not re-instantiate them
    if ((long long)c->lr_tab.n < iters) {
      size_t cap = 64;
      while ((long long)cap < iters) cap *= 2;
      c->lr_tab.alloc(cap, c->stream);
      c->c1_tab.alloc(cap, c->stream);
      c->c2_tab.alloc(cap, c->stream);
      c->rec.alloc(cap, c->stream);
      // tables were reallocated: drop graphs that captured the old pointers
      for (auto it = c->graphs.begin(); it != c->graphs.end();) {
        if (std::get<0>(it->first) == 2) {
          cudaGraphExecDestroy(it->second);
          it = c->graphs.erase(it);
        } else {
          ++it;
        }
      }
    }
    c->lr_tab.upload(lr.data(), iters, c->stream);
    c->c1_tab.upload(c1.data(), iters, c->stream);
    c->c2_tab.upload(c2.data(), iters, c->stream);
    reset_state(c, iters, spec);
    const int S = spec->steps_per_graph > 0 ? spec->steps_per_graph : 50;
    const int per = (int)std::min<long long>(S, iters);
    // a short run on a context without the captured epoch graph launches its
    // epochs directly (programmatic launches, the same kernels and
    // arguments): instantiating the graph costs more than the launches of a
    // few tens of epochs; longer runs capture once and replay
    // (two kernels per epoch with programmatic launch; the split path's
    // five-plus launches per epoch keep the graph: their launch gaps cost
    // ~10 us an epoch)
    const bool direct = spec->steps_per_graph <= 0 && iters < kGraphMinIters && !c->split &&
                        c->graphs.find(std::make_tuple(2, per, 0.0)) == c->graphs.end();
    if (direct) {
      const vpg::AdamArgs aa = adam_args(c, true, 0.0f, true, (int)c->rec.n);
      for (long long t = 0; t < iters; ++t) enqueue_epoch(c, aa);
    } else {
      cudaGraphExec_t g = graph_for(c, 2, per, 0.0, true, (int)c->rec.n);
      long long launched = 0;
      int since_check = 0;
      while (launched < iters) {
        CK(cudaGraphLaunch(g, c->stream));
        c->launches += launches_per_epoch(c) * per;
        launched += per;
        if (++since_check >= 20 && launched < iters) {
          since_check = 0;
          CK(cudaMemcpyAsync(c->h_flag, &c->st.p->stopped, sizeof(int), cudaMemcpyDeviceToHost,
                             c->stream));
          CK(cudaStreamSynchronize(c->stream));
          if (*c->h_flag) break;
        }
      }
    }
    vpg::TrainState s;
    CK(cudaMemcpyAsync(&s, c->st.p, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const long long ran = s.step;
    c->resume_pending = true;
    c->aborted_at = s.stop_reason == 3 ? std::max(1LL, s.abort_step) : 0;
    if (records && ran > 0) {
      std::vector<vpg::StepRecord> r(ran);
      CK(cudaMemcpy(r.data(), c->rec.p, sizeof(vpg::StepRecord) * ran, cudaMemcpyDeviceToHost));
      for (long long i = 0; i < ran; ++i) {
        records[i].total = r[i].total;
        records[i].variational = r[i].v;
        records[i].boundary = r[i].b;
        records[i].sensor = r[i].s;
        records[i].lr = r[i].lr;
        records[i].eps = r[i].eps;
        records[i].seconds = r[i].seconds;
      }
    }
    if (result) {
      result->steps_run = ran;
      result->converged = (s.stop_reason == 1 || s.stop_reason == 2) ? 1 : 0;
      result->stop_reason = s.stop_reason == 3 ? 0 : s.stop_reason;
      result->abort_step = s.stop_reason == 3 ? s.abort_step : 0;
      result->final_eps = std::numeric_limits<double>::quiet_NaN();
      if (c->eps_source == VPINN_EPS_SCALAR) {
        float e = 0;
        CK(cudaMemcpy(&e, c->params.p + c->net.scal_off + c->eps_idx, sizeof(float),
                      cudaMemcpyDeviceToHost));
        result->final_eps = e;
      }
    }
    if (s.stop_reason == 3)
      throw Fail{VPINN_ERR_NUMERIC, "step " + std::to_string(s.abort_step) +
                                        ": non-finite network output or gradient"};
  });
}

int vpinn_gpu_forward(vpinn_gpu_ctx* c, const double* points, int64_t n, int order, float* u,
                      float* du_dx, float* du_dy, float* eps) {
  return guarded([&] {
    if (order < 0 || order > 1)
      throw Fail{VPINN_ERR_CONFIG, "evaluate: order must be 0 or 1 on the GPU path"};
    if (n <= 0) return;
    set_dev(c);
    std::vector<float2> hp(n);
    for (int64_t i = 0; i < n; ++i) hp[i] = make_float2((float)points[2 * i], (float)points[2 * i + 1]);
    DBuf<float2> dp;
    DBuf<float> du, dux, duy, de;
    dp.alloc(n, c->stream);
    du.alloc(n, c->stream);
    dux.alloc(n, c->stream);
    duy.alloc(n, c->stream);
    de.alloc(n, c->stream);
    dp.upload(hp.data(), n, c->stream);
    vpg::StepArgs f = c->sargs;
    f.fwd_pts = dp.p;
    f.n_fwd = (int)n;
    f.out_u = du.p;
    f.out_ux = dux.p;
    f.out_uy = duy.p;
    f.out_eps = de.p;
    f.union_floats = 0;
    f.stop_flag = nullptr;
    if (c->strong) {
      const int grid = std::max(1, std::min(c->grid_step, ceil_div(n, c->sf_pts)));
      (c->sf_tc ? c->sfk.tc_forward : c->sfk.forward)<<<grid, c->sf_block, c->smem_step, c->stream>>>(f);
    } else if (c->tc2_modes) {
      const int grid = std::max(1, std::min(c->grid_tc2, ceil_div(n, c->var.tc2_mp)));
      c->var.tc2_fwd<<<grid, c->var.tc2_nt, c->var.tc2_smem, c->stream>>>(f);
    } else {
      const int grid = std::max(1, std::min(c->grid_fwd, ceil_div(n, vpg::kThreads)));
      c->var.forward<<<grid, vpg::kThreads, c->smem_fwd, c->stream>>>(f);
    }
    CK(cudaGetLastError());
    c->launches += 1;
    CK(cudaMemcpyAsync(u, du.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (order >= 1 && du_dx) CK(cudaMemcpyAsync(du_dx, dux.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (order >= 1 && du_dy) CK(cudaMemcpyAsync(du_dy, duy.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (eps && !c->strong && c->var.C >= 2) CK(cudaMemcpyAsync(eps, de.p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<float> chk(n);
    // network.hpp:443-447: non-finite outputs are a numeric error
    for (int64_t i = 0; i < n; ++i)
      if (!std::isfinite(u[i]) || (order >= 1 && du_dx && !std::isfinite(du_dx[i])) ||
          (order >= 1 && du_dy && !std::isfinite(du_dy[i])))
        throw Fail{VPINN_ERR_NUMERIC, "evaluate: non-finite network output"};
  });
}

int vpinn_gpu_forward2(vpinn_gpu_ctx* c, const double* points, int64_t n, float* u, float* du_dx, float* du_dy,
                       float* d2u_dx2, float* d2u_dy2) {
  return guarded([&] {
    if (!c->strong) throw Fail{VPINN_ERR_CONFIG, "evaluate order 2: strong-form contexts only"};
    if (n <= 0) return;
    set_dev(c);
    std::vector<float2> hp(n);
    for (int64_t i = 0; i < n; ++i) hp[i] = make_float2((float)points[2 * i], (float)points[2 * i + 1]);
    DBuf<float2> dp;
    DBuf<float> o[5];
    dp.alloc(n, c->stream);
    dp.upload(hp.data(), n, c->stream);
    float* host[5] = {u, du_dx, du_dy, d2u_dx2, d2u_dy2};
    for (int k = 0; k < 5; ++k)
      if (host[k]) o[k].alloc(n, c->stream);
    vpg::StepArgs f = c->sargs;
    f.fwd_pts = dp.p;
    f.n_fwd = (int)n;
    f.out_u = o[0].p;
    f.out_ux = o[1].p;
    f.out_uy = o[2].p;
    f.out_uxx = o[3].p;
    f.out_uyy = o[4].p;
    f.stop_flag = nullptr;
    const int grid = std::max(1, std::min(c->grid_step, ceil_div(n, c->sf_pts)));
    (c->sf_tc ? c->sfk.tc_forward : c->sfk.forward)<<<grid, c->sf_block, c->smem_step, c->stream>>>(f);
    CK(cudaGetLastError());
    c->launches += 1;
    for (int k = 0; k < 5; ++k)
      if (host[k]) CK(cudaMemcpyAsync(host[k], o[k].p, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 5; ++k)
      if (host[k])
        for (int64_t i = 0; i < n; ++i)
          if (!std::isfinite(host[k][i])) throw Fail{VPINN_ERR_NUMERIC, "evaluate: non-finite network output"};
  });
}

int vpinn_gpu_contract(vpinn_gpu_ctx* c, const float* du_dx, const float* du_dy, const float* eps,
                       const float* scalars, float weight, double* loss, float* residuals,
                       float* du_dx_bar, float* du_dy_bar, float* eps_bar, double* scalar_bar) {
  return guarded([&] {
    weak_only(c, "vpinn_gpu_contract");
    set_dev(c);
    if (c->eps_source == VPINN_EPS_SPATIAL && !eps)
      throw Fail{VPINN_ERR_NUMERIC, "spatial coefficient requested but no eps given"};
    if (c->eps_source == VPINN_EPS_SCALAR && !scalars)
      throw Fail{VPINN_ERR_NUMERIC, "coefficient scalar index out of range"};
    const size_t ni = (size_t)c->n_int;
    DBuf<float> ux, uy, ep, oxb, oyb, oeb, res, es;
    DBuf<double> lp;
    ux.alloc(ni, c->stream);
    uy.alloc(ni, c->stream);
    ep.alloc(ni, c->stream);
    oxb.alloc(ni, c->stream);
    oyb.alloc(ni, c->stream);
    oeb.alloc(ni, c->stream);
    res.alloc((size_t)c->E * c->T, c->stream);
    es.alloc(1, c->stream);
    lp.alloc((size_t)std::max(c->grid_contract, c->grid_cc) * vpg::kLpWords, c->stream);
    ux.upload(du_dx, ni, c->stream);
    uy.upload(du_dy, ni, c->stream);
    if (eps) ep.upload(eps, ni, c->stream);
    if (scalars) es.upload(scalars + c->eps_idx, 1, c->stream);
    const int rows = launch_contract(c, ux.p, uy.p, ep.p, oxb.p, oyb.p, oeb.p, res.p, es.p,
                                     (2.0f * weight) * c->sargs.inv_nt, lp.p, nullptr);
    std::vector<double> hl((size_t)rows * vpg::kLpWords);
    CK(cudaMemcpyAsync(hl.data(), lp.p, sizeof(double) * hl.size(), cudaMemcpyDeviceToHost, c->stream));
    if (residuals) CK(cudaMemcpyAsync(residuals, res.p, sizeof(float) * c->E * c->T, cudaMemcpyDeviceToHost, c->stream));
    if (du_dx_bar) CK(cudaMemcpyAsync(du_dx_bar, oxb.p, sizeof(float) * ni, cudaMemcpyDeviceToHost, c->stream));
    if (du_dy_bar) CK(cudaMemcpyAsync(du_dy_bar, oyb.p, sizeof(float) * ni, cudaMemcpyDeviceToHost, c->stream));
    if (eps_bar && c->eps_source == VPINN_EPS_SPATIAL)
      CK(cudaMemcpyAsync(eps_bar, oeb.p, sizeof(float) * ni, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    double l = 0.0, g = 0.0;
    for (int b = 0; b < rows; ++b) {
      l += hl[(size_t)b * vpg::kLpWords + vpg::kLpVar];
      g += hl[(size_t)b * vpg::kLpWords + vpg::kLpEpsGrad];
    }
    if (loss) *loss = l;
    if (scalar_bar && c->eps_source == VPINN_EPS_SCALAR) scalar_bar[c->eps_idx] = g;
  });
}

int vpinn_gpu_time_contract(vpinn_gpu_ctx* c, int reps, double* ms_per_launch, double* bytes) {
  return vpinn_gpu_time_contract_kernels(c, reps, ms_per_launch, nullptr, bytes);
}

int vpinn_gpu_time_contract_kernels(vpinn_gpu_ctx* c, int reps, double* ms_per_launch, double* ms_stream,
                                    double* bytes) {
  return guarded([&] {
    weak_only(c, "vpinn_gpu_time_contract");
    set_dev(c);
    const size_t ni = (size_t)c->n_int;
    DBuf<float> ux, uy, ep, oxb, oyb, oeb, es;
    DBuf<double> lp;
    ux.alloc(ni, c->stream);
    uy.alloc(ni, c->stream);
    ep.alloc(ni, c->stream);
    oxb.alloc(ni, c->stream);
    oyb.alloc(ni, c->stream);
    oeb.alloc(ni, c->stream);
    es.alloc(1, c->stream);
    lp.alloc((size_t)std::max(c->grid_contract, c->grid_cc) * vpg::kLpWords, c->stream);
    // L2 flush buffer (> 126 MB L2) between launches so each launch streams HBM
    DBuf<char> flush;
    flush.alloc((size_t)256 << 20, c->stream);
    cudaEvent_t e0, e1, em;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&em));
    // the streaming kernel alone: an event between it and the partial-column
    // reduction of the split path (the cell kernel is one launch)
    c->contract_mid = c->cell_contract ? nullptr : em;
    double total = 0.0, stream_ms = 0.0;
    for (int r = 0; r < reps + 2; ++r) {
      flush_l2_now(c, flush.p);
      CK(cudaEventRecord(e0, c->stream));
      launch_contract(c, ux.p, uy.p, ep.p, oxb.p, oyb.p, oeb.p, nullptr, es.p, c->sargs.rscale, lp.p, nullptr);
      CK(cudaEventRecord(e1, c->stream));
      CK(cudaEventSynchronize(e1));
      float ms = 0, ms1 = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (c->contract_mid) CK(cudaEventElapsedTime(&ms1, e0, em));
      else ms1 = ms;
      if (r >= 2) {
        total += ms;
        stream_ms += ms1;
      }
    }
    c->contract_mid = nullptr;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(em);
    *ms_per_launch = total / std::max(1, reps);
    if (ms_stream) *ms_stream = stream_ms / std::max(1, reps);
    const double EQ = (double)c->E * c->Q;
    double b = 4.0 * ((double)c->nt * c->E * c->T * c->Q + (double)c->E * c->T + 4.0 * EQ);
    if (c->eps_source == VPINN_EPS_SPATIAL) b += 8.0 * EQ;
    *bytes = b;
  });
}

namespace {
vpg::MfContractArgs mf_args(vpinn_gpu_ctx* c, const float* ux, const float* uy, float* oxb, float* oyb, float* res,
                            const float* es, float rscale, double* lp) {
  if (!c->asmd) throw Fail{VPINN_ERR_CONFIG, "matrix-free contraction needs a context created with an assembly input"};
  if (c->eps_source == VPINN_EPS_SPATIAL)
    throw Fail{VPINN_ERR_CONFIG, "matrix-free contraction: spatial coefficient not supported"};
  vpg::MfContractArgs m{};
  m.nodes = c->asmd->nodes.p;
  m.elems = c->asmd->elems.p;
  m.e0 = c->asm_e0;
  m.E = c->E;
  m.T = c->T;
  m.Q = c->Q;
  m.tabs = c->mf_tabs.p;
  m.rule = c->mf_rule.p;
  m.forcing = c->forcing.p;
  m.ux = ux;
  m.uy = uy;
  m.uxb = oxb;
  m.uyb = oyb;
  m.res = res;
  m.e_fixed = c->eps;
  m.e_param = es;
  m.eps_source = c->eps_source;
  m.bx = c->bx;
  m.by = c->by;
  m.rscale = rscale;
  m.inv_nt = c->sargs.inv_nt;
  m.loss_part = lp;
  return m;
}
// tile variant when a cell fits the CTA (cells_per_tile = 256 / Q), else
// the warp-per-cell kernel
int mf_cpt(vpinn_gpu_ctx* c) { return vpg::kMfTileThreads / c->Q; }
int mf_grid(vpinn_gpu_ctx* c) {
  const int cpt = mf_cpt(c);
  constexpr int per_sm = 4;
  if (cpt) return std::max(1, std::min(ceil_div(c->E, cpt), per_sm * c->sm_count));
  return std::max(1, std::min(ceil_div(c->E, vpg::kMfWarps), 8 * c->sm_count));
}
size_t mf_prepare(vpinn_gpu_ctx* c) {  // once per call site, outside any timed region
  const int cpt = mf_cpt(c);
  const size_t smem = cpt ? vpg::mf_tile_smem_bytes(c->T, c->Q, cpt) : vpg::mf_smem_bytes(c->T, c->Q);
  if (smem > (size_t)227 * 1024) throw Fail{VPINN_ERR_CONFIG, "matrix-free contraction: basis tables exceed shared memory"};
  if (cpt)
    CK(cudaFuncSetAttribute(vpg::contract_mf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  else
    CK(cudaFuncSetAttribute(vpg::contract_mf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return smem;
}
void launch_mf(vpinn_gpu_ctx* c, const vpg::MfContractArgs& m, size_t smem) {
  if (const int cpt = mf_cpt(c))
    vpg::contract_mf_tile_kernel<<<mf_grid(c), vpg::kMfTileThreads, smem, c->stream>>>(m, cpt);
  else
    vpg::contract_mf_kernel<<<mf_grid(c), 32 * vpg::kMfWarps, smem, c->stream>>>(m);
  CK(cudaGetLastError());
  c->launches += 1;
}
}  // namespace

int vpinn_gpu_contract_matrix_free(vpinn_gpu_ctx* c, const float* du_dx, const float* du_dy, const float* scalars,
                                   float weight, double* loss, float* residuals, float* du_dx_bar,
                                   float* du_dy_bar, double* scalar_bar) {
  return guarded([&] {
    weak_only(c, "vpinn_gpu_contract_matrix_free");
    set_dev(c);
    if (c->eps_source == VPINN_EPS_SCALAR && !scalars)
      throw Fail{VPINN_ERR_NUMERIC, "coefficient scalar index out of range"};
    const size_t ni = (size_t)c->n_int;
    DBuf<float> ux, uy, oxb, oyb, res, es;
    DBuf<double> lp;
    ux.alloc(ni, c->stream);
    uy.alloc(ni, c->stream);
    oxb.alloc(ni, c->stream);
    oyb.alloc(ni, c->stream);
    res.alloc((size_t)c->E * c->T, c->stream);
    es.alloc(1, c->stream);
    const int rows = mf_grid(c);
    lp.alloc((size_t)rows * vpg::kLpWords, c->stream);
    ux.upload(du_dx, ni, c->stream);
    uy.upload(du_dy, ni, c->stream);
    if (scalars) es.upload(scalars + c->eps_idx, 1, c->stream);
    launch_mf(c, mf_args(c, ux.p, uy.p, oxb.p, oyb.p, res.p, es.p, (2.0f * weight) * c->sargs.inv_nt, lp.p),
              mf_prepare(c));
    std::vector<double> hl((size_t)rows * vpg::kLpWords);
    CK(cudaMemcpyAsync(hl.data(), lp.p, sizeof(double) * hl.size(), cudaMemcpyDeviceToHost, c->stream));
    if (residuals) CK(cudaMemcpyAsync(residuals, res.p, sizeof(float) * c->E * c->T, cudaMemcpyDeviceToHost, c->stream));
    if (du_dx_bar) CK(cudaMemcpyAsync(du_dx_bar, oxb.p, sizeof(float) * ni, cudaMemcpyDeviceToHost, c->stream));
    if (du_dy_bar) CK(cudaMemcpyAsync(du_dy_bar, oyb.p, sizeof(float) * ni, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    double l = 0.0, g = 0.0;
    for (int b = 0; b < rows; ++b) {
      l += hl[(size_t)b * vpg::kLpWords + vpg::kLpVar];
      g += hl[(size_t)b * vpg::kLpWords + vpg::kLpEpsGrad];
    }
    if (loss) *loss = l;
    if (scalar_bar && c->eps_source == VPINN_EPS_SCALAR) scalar_bar[c->eps_idx] = g;
  });
}

int vpinn_gpu_time_contract_matrix_free(vpinn_gpu_ctx* c, int reps, double* ms_per_launch, double* bytes) {
  return guarded([&] {
    weak_only(c, "vpinn_gpu_time_contract_matrix_free");
    set_dev(c);
    const size_t ni = (size_t)c->n_int;
    DBuf<float> ux, uy, oxb, oyb, es;
    DBuf<double> lp;
    ux.alloc(ni, c->stream);
    uy.alloc(ni, c->stream);
    oxb.alloc(ni, c->stream);
    oyb.alloc(ni, c->stream);
    es.alloc(1, c->stream);
    lp.alloc((size_t)mf_grid(c) * vpg::kLpWords, c->stream);
    DBuf<char> flush;
    flush.alloc((size_t)256 << 20, c->stream);
    const vpg::MfContractArgs m = mf_args(c, ux.p, uy.p, oxb.p, oyb.p, nullptr, es.p, c->sargs.rscale, lp.p);
    const size_t smem = mf_prepare(c);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double total = 0.0;
    for (int r = 0; r < reps + 2; ++r) {
      flush_l2_now(c, flush.p);
      CK(cudaEventRecord(e0, c->stream));
      launch_mf(c, m, smem);
      CK(cudaEventRecord(e1, c->stream));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) total += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_launch = total / std::max(1, reps);
    // algorithmic bytes: 4 node coordinates (double) + 4 element indices per
    // cell, forcing column, u_x / u_y in, the two adjoints out
    const double EQ = (double)c->E * c->Q;
    *bytes = (double)c->E * (4 * 16 + 16) + 4.0 * ((double)c->E * c->T + 4.0 * EQ);
  });
}

int vpinn_gpu_download_tensor(vpinn_gpu_ctx* c, int which, float* out, int64_t n) {
  return guarded([&] {
    weak_only(c, "vpinn_gpu_download_tensor");
    set_dev(c);
    const DBuf<float>* b = which <= 2 ? &c->tens[which] : &c->forcing;
    if (which < 0 || which > 3) throw Fail{VPINN_ERR_CONFIG, "download: selector"};
    if (which == 2 && c->nt < 3) throw Fail{VPINN_ERR_CONFIG, "download: no test tensor uploaded"};
    if ((size_t)n != b->n) throw Fail{VPINN_ERR_CONFIG, "download: size mismatch"};
    CK(cudaMemcpy(out, b->p, sizeof(float) * n, cudaMemcpyDeviceToHost));
  });
}

int64_t vpinn_gpu_launch_count(const vpinn_gpu_ctx* c) { return c ? c->launches : -1; }

int vpinn_gpu_profile_step(vpinn_gpu_ctx* c, int reps, double* ms_mlp, double* ms_reduce,
                           double* ms_adam) {
  return guarded([&] {
    set_dev(c);
    // a diagnostic: the live parameters, Adam moments and trainer state are
    // saved here and restored at the end, so profiling leaves the run as it was
    DBuf<float> save_p, save_m, save_v;
    DBuf<vpg::TrainState> save_st;
    save_p.alloc(c->n_params, c->stream);
    save_m.alloc(c->n_params, c->stream);
    save_v.alloc(c->n_params, c->stream);
    save_st.alloc(1, c->stream);
    const size_t pb = sizeof(float) * c->n_params;
    CK(cudaMemcpyAsync(save_p.p, c->params.p, pb, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(save_m.p, c->m.p, pb, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(save_v.p, c->v.p, pb, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(save_st.p, c->st.p, sizeof(vpg::TrainState), cudaMemcpyDeviceToDevice, c->stream));
    const bool resume_pending = c->resume_pending;
    const long long aborted_at = c->aborted_at;
    reset_state(c, LLONG_MAX, nullptr);
    const vpg::AdamArgs aa = adam_args(c, false, 1e-4f, false, 0);
    cudaEvent_t ev[4];
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double t[3] = {0, 0, 0};
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaEventRecord(ev[0], c->stream));
      // the step kernels (fused, or the split chain) then reduce: time separately
      const Variant& V = c->var;
      vpg::StepArgs a = c->sargs;
      a.stop_flag = &c->st.p->stopped;
      if (!c->split) {
        launch_fused(c, a);
        CK(cudaEventRecord(ev[1], c->stream));
        vpg::reduce_kernel<<<vpg::reduce_grid(c->n_params), vpg::kRedThreads, 0, c->stream>>>(
            c->grad_part.p, c->grad_rows, c->part_stride, c->n_params, c->loss_part.p, c->loss_rows, c->red.p,
            a.stop_flag);
        CK(cudaGetLastError());
        c->launches += 1;
        if (c->comm)
          NK(nccl().all_reduce(c->red.p, c->red.p, (size_t)c->n_params + vpg::kLpWords,
                               ncclFloat64, ncclSum, c->comm, c->stream));
      } else {
        enqueue_grad(c, a.stop_flag);
        CK(cudaEventRecord(ev[1], c->stream));
      }
      CK(cudaEventRecord(ev[2], c->stream));
      vpg::adam_kernel<<<1, 1024, 0, c->stream>>>(aa);
      CK(cudaGetLastError());
      c->launches += 1;
      CK(cudaEventRecord(ev[3], c->stream));
      CK(cudaEventSynchronize(ev[3]));
      if (r >= 2) {
        float a1, a2, a3;
        CK(cudaEventElapsedTime(&a1, ev[0], ev[1]));
        CK(cudaEventElapsedTime(&a2, ev[1], ev[2]));
        CK(cudaEventElapsedTime(&a3, ev[2], ev[3]));
        t[0] += a1;
        t[1] += a2;
        t[2] += a3;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    CK(cudaMemcpyAsync(c->params.p, save_p.p, pb, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->m.p, save_m.p, pb, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->v.p, save_v.p, pb, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->st.p, save_st.p, sizeof(vpg::TrainState), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->resume_pending = resume_pending;
    c->aborted_at = aborted_at;
    *ms_mlp = t[0] / reps;
    *ms_reduce = t[1] / reps;
    *ms_adam = t[2] / reps;
  });
}

int vpinn_gpu_set_test_hooks(int flags) {
  return guarded([&] {
    if (flags & ~(VPINN_HOOK_CUDA_CORE_STEP | VPINN_HOOK_FORCE_SPILL | VPINN_HOOK_THROUGHPUT_LAYOUT))
      throw Fail{VPINN_ERR_CONFIG, "set_test_hooks: unknown flag"};
    g_test_hooks.store(flags);
  });
}

int vpinn_gpu_release_cached_memory(void) {
  return guarded([&] { block_cache().trim(); });
}

int vpinn_gpu_assemble(int device, int32_t n_elem, int32_t n_test, int32_t n_quad, const vpinn_gpu_assembly* in,
                       float* grad_x, float* grad_y, float* test, float* forcing, double* quad_points) {
  return guarded([&] {
    if (!in || !grad_x || !grad_y || n_elem < 1 || n_test < 1 || n_quad < 1)
      throw Fail{VPINN_ERR_CONFIG, "vpinn_gpu_assemble: bad arguments"};
    CK(cudaSetDevice(device));
    cudaStream_t s = nullptr;  // legacy default stream: ordered with the zero fills
    AsmUpload up;
    up.load(in, n_elem, n_test, n_quad, s);
    const size_t n = (size_t)n_elem * n_test * n_quad;
    DBuf<float> gx, gy, tv, fc, fq;
    DBuf<double> qp;
    gx.alloc(n, s);
    gy.alloc(n, s);
    tv.alloc(n, s);
    fc.alloc((size_t)n_elem * n_test, s);
    fq.alloc((size_t)n_elem * n_quad, s);
    qp.alloc((size_t)2 * n_elem * n_quad, s);
    CK(vpg::assemble_on_device(up.in, 0, n_elem, gx.p, gy.p, tv.p, forcing ? fc.p : nullptr, qp.p, nullptr, fq.p,
                               up.bad.p, s));
    up.check(s);
    CK(cudaMemcpy(grad_x, gx.p, sizeof(float) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(grad_y, gy.p, sizeof(float) * n, cudaMemcpyDeviceToHost));
    if (test) CK(cudaMemcpy(test, tv.p, sizeof(float) * n, cudaMemcpyDeviceToHost));
    if (forcing) CK(cudaMemcpy(forcing, fc.p, sizeof(float) * n_elem * n_test, cudaMemcpyDeviceToHost));
    if (quad_points)
      CK(cudaMemcpy(quad_points, qp.p, sizeof(double) * 2 * n_elem * n_quad, cudaMemcpyDeviceToHost));
  });
}

// diagnostics: the phase clocks of the last tensor-core step launch
// (VPINN_PHASE_CLOCK=1 at create), kPhaseTiles x kPhaseMarks clock64 values
int vpinn_gpu_phase_clock(vpinn_gpu_ctx* c, long long* out, int n) {
  return guarded([&] {
    set_dev(c);
    if (!c->phase_clk.p) throw Fail{VPINN_ERR_CONFIG, "phase clocks not enabled (VPINN_PHASE_CLOCK=1)"};
    const int m = std::min(n, vpg::kPhaseTiles * vpg::kPhaseMarks + 3 * 1024);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(out, c->phase_clk.p, sizeof(long long) * m, cudaMemcpyDeviceToHost));
  });
}

int vpinn_gpu_flush_l2(vpinn_gpu_ctx* c) {
  return guarded([&] {
    set_dev(c);
    if (!c->flush.p) c->flush.alloc((size_t)256 << 20, c->stream);
    flush_l2_now(c, c->flush.p);
  });
}

int vpinn_gpu_tc_probe(int device, int mode, const float* A, const float* W, const float* H, float* out) {
  return guarded([&] {
    if (mode < 0 || mode > 5) throw Fail{VPINN_ERR_CONFIG, "tc_probe: mode must be 0..5"};
    CK(cudaSetDevice(device));
    DBuf<float> dA, dW, dH, dO;
    dA.alloc(128 * 32, 0);
    dW.alloc(32 * 32, 0);
    dH.alloc(128 * 32, 0);
    dO.alloc(128 * 32 + 128 * 96, 0);
    CK(cudaMemcpy(dA.p, A, sizeof(float) * 128 * 32, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW.p, W, sizeof(float) * 32 * 32, cudaMemcpyHostToDevice));
    if (H) CK(cudaMemcpy(dH.p, H, sizeof(float) * 128 * 32, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(vpg::tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, vpg::kTcProbeSmem));
    vpg::tc_probe_kernel<<<1, 128, vpg::kTcProbeSmem>>>(mode, dA.p, dW.p, dH.p, dO.p);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dO.p, sizeof(float) * (128 * 32 + 128 * 96), cudaMemcpyDeviceToHost));
  });
}

int vpinn_gpu_measure_ffma_peak(int device, double* tflops) {
  return guarded([&] {
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    DBuf<float> out;
    out.alloc(256, 0);
    const int blocks = prop.multiProcessorCount * 8, iters = 4096;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best = 0.0;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      vpg::ffma_peak_kernel<<<blocks, 256>>>(out.p, iters, 0.999999f, 1e-7f);
      CK(cudaGetLastError());
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double flops = 2.0 * 8 * 16 * (double)iters * 256.0 * blocks;
      if (r > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tflops = best;
  });
}

int vpinn_gpu_nccl_unique_id(void* id128) {
  return guarded([&] {
    NcclUid u;
    NK(nccl().get_unique_id(&u));
    std::memcpy(id128, u.b, sizeof(u.b));
  });
}

int vpinn_gpu_peer_handle(vpinn_gpu_ctx* c, void* handle64) {
  return guarded([&] {
    set_dev(c);
    if (!c->pbox) {
      const size_t bytes = vpg::peer_mailbox_bytes(c->n_params + vpg::kLpWords);
      CK(cudaMalloc(&c->pbox, bytes));  // its own allocation: an IPC handle maps a whole allocation
      CK(cudaMemset(c->pbox, 0, bytes));
      CK(cudaDeviceSynchronize());
    }
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->pbox));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int vpinn_gpu_attach_peers(vpinn_gpu_ctx* c, const void* handles, int nranks, int rank) {
  return guarded([&] {
    if (nranks != c->nranks || rank != c->rank)
      throw Fail{VPINN_ERR_CONFIG, "attach_peers: rank/world differ from the partition"};
    if (nranks < 1 || nranks > vpg::kMaxRanks) throw Fail{VPINN_ERR_CONFIG, "attach_peers: 1..8 ranks"};
    if (!c->pbox) throw Fail{VPINN_ERR_CONFIG, "attach_peers: call vpinn_gpu_peer_handle first"};
    set_dev(c);
    vpg::PeerArgs pa{};
    pa.world = nranks;
    pa.rank = rank;
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) {
        pa.box[r] = c->pbox;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + 64 * (size_t)r, sizeof(h));
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      pa.box[r] = static_cast<vpg::PeerMailbox*>(p);
    }
    c->peers = pa;
    c->peer = true;
    // every CTA of the exchange must be resident at once (phase 2 waits for
    // all of phase 1): the grid is capped at what the device holds
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vpg::reduce_adam_peer_kernel, vpg::kRAThreads, 0));
    c->grid_peer = std::max(1, std::min(vpg::reduce_adam_grid(c->n_params), std::max(1, occ) * c->sm_count));
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  });
}

int vpinn_gpu_attach_comm(vpinn_gpu_ctx* c, const void* id128, int nranks, int rank) {
  return guarded([&] {
    if (nranks != c->nranks || rank != c->rank)
      throw Fail{VPINN_ERR_CONFIG, "attach_comm: rank/world differ from the partition"};
    set_dev(c);
    NcclUid u;
    std::memcpy(u.b, id128, sizeof(u.b));
    void* comm = nullptr;
    NK(nccl().comm_init_rank(&comm, nranks, u, rank));
    c->comm = comm;
    if (c->peer) {  // the last attachment wins: peers detached
      for (int r = 0; r < c->peers.world; ++r)
        if (r != c->rank && c->peers.box[r]) cudaIpcCloseMemHandle(c->peers.box[r]);
      c->peers = vpg::PeerArgs{};
      c->peer = false;
    }
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  });
}

}  // extern "C"
