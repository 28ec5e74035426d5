// Cross-CTA reduction, Adam + device-side trainer bookkeeping, the
// standalone HBM-streaming contraction (split path and roofline report) and
// the penalty kernel of the split path.
#pragma once

#include <type_traits>

#include "contract_cells.cuh"
#include "step_kernel.cuh"

namespace vpg {

// ---------------------------------------------------------------------------
// Cross-CTA reduction of the per-CTA partials (fp64, fixed order): one warp
// per parameter over the param-major partial rows (all loads of a lane in
// flight at once, then a fixed shuffle tree); the trailing kLpWords warps sum
// the loss words the same way.  red = [gradient | loss words].
constexpr int kRedThreads = 256;
constexpr int kRedWarps = kRedThreads / 32;

// row gw of red by one converged warp: lane c sums entries c, c + 32, ... in
// double, then a fixed xor tree; every lane returns the row's value
__device__ __forceinline__ double reduce_row(int gw, const float* __restrict__ grad_part, int n_rows, int stride,
                                             int n_params, const double* __restrict__ loss_part, int n_loss_rows,
                                             double* __restrict__ red) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (gw < n_params) {
    const float* src_f = grad_part + (size_t)gw * stride;
#pragma unroll 8
    for (int c = lane; c < n_rows; c += 32) acc += (double)src_f[c];
  } else {
    const double* src_d = loss_part + (gw - n_params);
#pragma unroll 8
    for (int c = lane; c < n_loss_rows; c += 32) acc += src_d[(size_t)c * kLpWords];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[gw] = acc;
  return acc;
}

__device__ __forceinline__ void reduce_body(const float* __restrict__ grad_part, int n_rows, int stride,
                                            int n_params, const double* __restrict__ loss_part, int n_loss_rows,
                                            double* __restrict__ red) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw < n_params + kLpWords) reduce_row(gw, grad_part, n_rows, stride, n_params, loss_part, n_loss_rows, red);
}

__host__ __device__ constexpr int reduce_grid(int n_params) { return (n_params + kLpWords + kRedWarps - 1) / kRedWarps; }
// the fused reduce + Adam: 1024-thread CTAs, so the last CTA's Adam update
// (IEEE division / square root per parameter, the epoch's serial tail) runs
// on 1024 threads
constexpr int kRAThreads = 1024;
__host__ __device__ constexpr int reduce_adam_grid(int n_params) {
  return (n_params + kLpWords + kRAThreads / 32 - 1) / (kRAThreads / 32);
}

__global__ void __launch_bounds__(kRedThreads) reduce_kernel(const float* __restrict__ grad_part, int n_rows,
                                                             int stride, int n_params,
                                                             const double* __restrict__ loss_part,
                                                             int n_loss_rows, double* __restrict__ red,
                                                             const int* stop_flag) {
  if (stop_flag != nullptr && *stop_flag != 0) return;
  reduce_body(grad_part, n_rows, stride, n_params, loss_part, n_loss_rows, red);
}

// ---------------------------------------------------------------------------
struct TrainState {
  long long step;        // completed Adam updates of the current run
  long long iterations;  // budget (stop after this many)
  int stopped;           // read by every step kernel: non-zero -> no-op
  int stop_reason;       // 0 budget, 1 coefficient within tolerance, 2 plateau, 3 abort
  long long abort_step;
  double best_loss;
  long long best_step;
  unsigned long long t_prev;
  int has_eps_tol, has_eps_actual, has_loss_tol, plateau_window;
  double eps_abs_tol, eps_actual, loss_tol;
  int tracks_eps, eps_slot;
};

struct StepRecord {
  double total, v, b, s, lr, eps, seconds, pad;
};

struct AdamArgs {
  const double* red;  // [n_params + kLpWords]
  int n_params;
  float* params;
  float* m;
  float* v;
  TrainState* st;
  const float* lr_tab;  // [iterations] per 1-based step t at index t-1, or null
  const float* c1_tab;
  const float* c2_tab;
  float lr_const;
  StepRecord* rec;  // [iterations] or null
  int rec_cap;
  double n_bnd, n_sen;  // global penalty counts
  float tau_f, gamma_f;
  int eps_grad_slot;  // parameter index receiving the scalar-eps gradient (-1 none)
};

// adam_step (trainer.hpp:34-59) for one parameter: IEEE intrinsics keep the
// update in the reference's operation order (no FMA contraction)
__device__ __forceinline__ void adam_update(float g, float m0, float v0, float p0, float lr, float c1, float c2,
                                            float& m_out, float& v_out, float& p_out) {
  const float b1 = 0.9f, b2 = 0.999f, omb1 = 1.0f - b1, omb2 = 1.0f - b2;
  const float m = __fadd_rn(__fmul_rn(b1, m0), __fmul_rn(omb1, g));
  const float v = __fadd_rn(__fmul_rn(b2, v0), __fmul_rn(omb2, __fmul_rn(g, g)));
  m_out = m;
  v_out = v;
  const float mh = __fdiv_rn(m, c1);
  const float vh = __fdiv_rn(v, c2);
  p_out = __fsub_rn(p0, __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), 1e-8f)));
}

// lr and the bias corrections of step t (trainer.hpp:49-52, 73-78): the host
// tables, or lr_const and (float)(1 - beta^t) in double
__device__ __forceinline__ void step_factors(const AdamArgs& a, long long t, float& lr, float& c1, float& c2) {
  if (a.lr_tab) {
    lr = a.lr_tab[t - 1];
    c1 = a.c1_tab[t - 1];
    c2 = a.c2_tab[t - 1];
  } else {
    lr = a.lr_const;
    c1 = 1.0f - (float)pow(0.9, (double)t);
    c2 = 1.0f - (float)pow(0.999, (double)t);
  }
}

// the loss parts in the reference's Real semantics and the train-loop
// bookkeeping after an update (trainer.hpp:316-370): history record,
// coefficient-tolerance / plateau / budget stops.  Thread 0.
__device__ __forceinline__ void train_bookkeeping(const AdamArgs& a, long long t, float lr) {
  TrainState* st = a.st;
  const int n = a.n_params;
  const double* red = a.red;
  // L2 loads: red and the parameters may come from other CTAs (reduce_adam_kernel)
  const float Lv = (float)__ldcg(&red[n + kLpVar]);
  const float Lb = a.n_bnd > 0 ? (float)(__ldcg(&red[n + kLpBnd]) / a.n_bnd) : 0.0f;
  const float Ls = a.n_sen > 0 ? (float)(__ldcg(&red[n + kLpSen]) / a.n_sen) : 0.0f;
  const float total_f = __fadd_rn(__fadd_rn(Lv, __fmul_rn(a.tau_f, Lb)), __fmul_rn(a.gamma_f, Ls));
  const double total = (double)total_f;
  const unsigned long long now = globaltimer();
  st->step = t;
  double eps_now = __longlong_as_double(0x7ff8000000000000ll);
  if (st->tracks_eps) eps_now = (double)__ldcg(&a.params[st->eps_slot]);
  if (a.rec && t - 1 < a.rec_cap) {
    StepRecord r;
    r.total = total;
    r.v = (double)Lv;
    r.b = (double)Lb;
    r.s = (double)Ls;
    r.lr = (double)lr;
    r.eps = eps_now;
    r.seconds = (double)(now - st->t_prev) * 1e-9;
    r.pad = 0.0;
    a.rec[t - 1] = r;
  }
  st->t_prev = now;
  // convergence checks, after the update (trainer.hpp:343-369)
  int stop = 0, reason = 0;
  if (st->tracks_eps && st->has_eps_tol && st->has_eps_actual) {
    if (fabs(eps_now - st->eps_actual) < st->eps_abs_tol) {
      stop = 1;
      reason = 1;
    }
  }
  if (!stop && st->has_loss_tol) {
    if (total < st->best_loss * (1.0 - st->loss_tol)) {
      st->best_loss = total;
      st->best_step = t;
    } else if (t - st->best_step >= st->plateau_window) {
      stop = 1;
      reason = 2;
    }
    if (!stop && total < st->best_loss) st->best_loss = total;
  }
  if (!stop && t >= st->iterations) {
    stop = 1;
    reason = 0;
  }
  if (stop) {
    st->stopped = 1;
    st->stop_reason = reason;
  }
}

// adam_step (trainer.hpp:34-59) + train-loop bookkeeping (trainer.hpp:316-370)
// for one epoch.  One CTA of 1024 threads.
__device__ __forceinline__ void adam_body(const AdamArgs& a) {
  TrainState* st = a.st;
  const long long t = st->step + 1;
  const int n = a.n_params;
  const double* red = a.red;
  const double eg = red[n + kLpEpsGrad];
  int bad = red[n + kLpBad] != 0.0;
  // every load of this thread's parameters issued before the abort check
  // (one round trip instead of a chain: red, then m / v / params)
  float g_loc[4], m_loc[4], v_loc[4], p_loc[4];
  int cnt = 0;
  for (int p = threadIdx.x; p < n; p += blockDim.x, ++cnt) {
    double gd = red[p];
    if (p == a.eps_grad_slot) gd += eg;
    const float g = (float)gd;
    if (!isfinite(g)) bad = 1;
    if (cnt < 4) {
      g_loc[cnt] = g;
      m_loc[cnt] = a.m[p];
      v_loc[cnt] = a.v[p];
      p_loc[cnt] = a.params[p];
    }
  }
  bad = __syncthreads_or(bad);
  float lr, c1, c2;
  if (a.lr_tab) {
    lr = a.lr_tab[t - 1];
    c1 = a.c1_tab[t - 1];
    c2 = a.c2_tab[t - 1];
  } else {
    lr = a.lr_const;
    c1 = 1.0f - (float)pow(0.9, (double)t);
    c2 = 1.0f - (float)pow(0.999, (double)t);
  }
  if (bad) {
    if (threadIdx.x == 0) {
      st->stopped = 1;
      st->stop_reason = 3;
      st->abort_step = t;
    }
    return;
  }
  cnt = 0;
  for (int p = threadIdx.x; p < n; p += blockDim.x, ++cnt) {
    float g, m0, v0, p0;
    if (cnt < 4) {
      g = g_loc[cnt];
      m0 = m_loc[cnt];
      v0 = v_loc[cnt];
      p0 = p_loc[cnt];
    } else {
      double gd = red[p];
      if (p == a.eps_grad_slot) gd += eg;
      g = (float)gd;
      m0 = a.m[p];
      v0 = a.v[p];
      p0 = a.params[p];
    }
    adam_update(g, m0, v0, p0, lr, c1, c2, a.m[p], a.v[p], a.params[p]);
  }
  __syncthreads();
  if (threadIdx.x == 0) train_bookkeeping(a, t, lr);
}

__global__ void __launch_bounds__(1024) adam_kernel(const AdamArgs a) {
  if (a.st->stopped) return;
  adam_body(a);
}

// single-GPU epoch tail: one warp per row reduces the CTA partials exactly
// as reduce_kernel does and, for a parameter row, applies Adam to that
// parameter right away (adam_update: the same expressions as adam_body),
// keeping the old (p, m, v) in bk; the last CTA to finish (atomic ticket,
// release / acquire fences) then only does the bookkeeping, or -- when a
// gradient or the step kernel's loss words were non-finite -- restores every
// parameter from bk and records the abort (adam_body's all-or-nothing
// semantics).  Two dependent global round trips fewer than reducing first
// and updating in the last CTA.  ticket[0]: CTA ticket, ticket[1]: non-finite
// gradient flag (both re-armed by the last CTA).
__global__ void __launch_bounds__(kRAThreads) reduce_adam_kernel(const float* __restrict__ grad_part, int n_rows,
                                                                   int stride, int n_params,
                                                                   const double* __restrict__ loss_part,
                                                                   int n_loss_rows, double* __restrict__ red,
                                                                   unsigned* ticket, float* bk, const AdamArgs a) {
  pdl_trigger();
  // the trainer state is this epoch's before the wait: the previous epoch's
  // tail completed before this epoch's step kernel passed its own wait, and
  // every step kernel triggers this launch only after that wait (tc2 / sf2:
  // after the tile loop; sf_step: right after the wait; step_kernel and the
  // split path: no programmatic launch)
  __shared__ int last, s_stopped;
  __shared__ long long s_t;
  __shared__ float s_f[3];  // lr, c1, c2 of this step: once per CTA, before the wait
  if (threadIdx.x == 0) {
    s_stopped = a.st->stopped;
    s_t = a.st->step + 1;
    if (!s_stopped) step_factors(a, s_t, s_f[0], s_f[1], s_f[2]);
  }
  __syncthreads();
  pdl_wait();
  if (s_stopped) return;
  const long long t = s_t;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const float lr = s_f[0], c1 = s_f[1], c2 = s_f[2];
  if (gw < n_params + kLpWords) {
    float p0 = 0.f, m0 = 0.f, v0 = 0.f;
    if (gw < n_params && lane == 0) {  // in flight with the partial loads
      p0 = a.params[gw];
      m0 = a.m[gw];
      v0 = a.v[gw];
    }
    double gd = reduce_row(gw, grad_part, n_rows, stride, n_params, loss_part, n_loss_rows, red);
    if (gw == a.eps_grad_slot)  // the scalar-eps gradient's loss word, reduced the same way
      gd += reduce_row(n_params + kLpEpsGrad, grad_part, n_rows, stride, n_params, loss_part, n_loss_rows, red);
    if (gw < n_params && lane == 0) {
      const float g = (float)gd;
      if (!isfinite(g)) atomicOr(&ticket[1], 1u);
      bk[gw] = p0;
      bk[n_params + gw] = m0;
      bk[2 * n_params + gw] = v0;
      adam_update(g, m0, v0, p0, lr, c1, c2, a.m[gw], a.v[gw], a.params[gw]);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[0], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // (other CTAs' results: L2 loads, this SM's L1 may hold lines of them)
  const int bad = __ldcg(&ticket[1]) != 0u || __ldcg(&red[n_params + kLpBad]) != 0.0;
  if (bad) {  // all or nothing: the parameters and moments of before the step
    for (int p = threadIdx.x; p < n_params; p += blockDim.x) {
      a.params[p] = __ldcg(&bk[p]);
      a.m[p] = __ldcg(&bk[n_params + p]);
      a.v[p] = __ldcg(&bk[2 * n_params + p]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ticket[0] = 0u;  // re-armed for the next epoch (graph replay)
    ticket[1] = 0u;
    if (bad) {
      a.st->stopped = 1;
      a.st->stop_reason = 3;
      a.st->abort_step = t;
    } else {
      train_bookkeeping(a, t, lr);
    }
  }
}

// ---------------------------------------------------------------------------
// Multi-GPU epoch tail over peer memory (one process per GPU,
// every rank's mailbox mapped into every other rank through CUDA IPC over
// NVLink / NVSwitch): the cross-CTA reduction, the cross-RANK sum and Adam in
// ONE kernel, instead of reduce -> ncclAllReduce -> Adam.
//   phase 1  each warp reduces one row of this rank's CTA partials (as
//            reduce_kernel) and its lanes r < W store the row into slot
//            [set][rank] of rank r's mailbox (peer stores); the last CTA to
//            finish publishes the epoch's sequence number into every rank's
//            flag[set][rank] (system-scope release after a system fence)
//   phase 2  every CTA waits for the W flags of its own mailbox, then each
//            warp sums its row over the ranks in rank order (the same bits on
//            every rank: replicas stay identical) and applies Adam to that
//            parameter (adam_update, rollback copy); the last CTA does the
//            bookkeeping (or the abort) exactly as reduce_adam_kernel.
// With adam = 0 it is the cross-rank gradient sum alone (loss_and_grad).
// Two slot sets alternate by sequence parity: a rank can run at most one
// epoch ahead of the slowest (its next tail waits for everyone's flags).
constexpr int kMaxRanks = 8;
struct PeerMailbox {
  unsigned long long flag[2][kMaxRanks];  // [set][source rank]: sequence number of the source's rows
  unsigned long long seq;                 // this rank's completed exchanges (local)
  unsigned long long pad[7];
  // double slot[2][kMaxRanks][rows] follows
};
__host__ __device__ constexpr size_t peer_mailbox_bytes(int rows) {
  return sizeof(PeerMailbox) + sizeof(double) * 2 * kMaxRanks * (size_t)rows;
}
__device__ __forceinline__ double* mbox_slot(PeerMailbox* m, int set, int src, int rows) {
  return reinterpret_cast<double*>(m + 1) + ((size_t)set * kMaxRanks + src) * rows;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
struct PeerArgs {
  PeerMailbox* box[kMaxRanks];  // every rank's mailbox in this process's address space
  int world, rank;
};

__global__ void __launch_bounds__(kRAThreads) reduce_adam_peer_kernel(const float* __restrict__ grad_part,
                                                                        int n_rows, int stride, int n_params,
                                                                        const double* __restrict__ loss_part,
                                                                        int n_loss_rows, double* __restrict__ red,
                                                                        unsigned* ticket, float* bk, const AdamArgs a,
                                                                        const PeerArgs pa, int adam,
                                                                        const int* stop_flag) {
  // the grid is at most what the device holds at once (every CTA waits in
  // phase 2 for flags the last CTA of phase 1 sets): warps stride over rows
  pdl_trigger();
  __shared__ int last, s_stopped;
  __shared__ long long s_t;
  __shared__ unsigned long long s_seq;
  __shared__ float s_f[3];
  __shared__ PeerMailbox* s_box[kMaxRanks];
  PeerMailbox* mine = pa.box[pa.rank];
  if (threadIdx.x == 0) {
    s_stopped = stop_flag != nullptr ? *stop_flag : 0;
    s_t = a.st->step + 1;
    s_seq = mine->seq + 1;
    if (adam && !s_stopped) step_factors(a, s_t, s_f[0], s_f[1], s_f[2]);
  }
  if (threadIdx.x < kMaxRanks) s_box[threadIdx.x] = pa.box[threadIdx.x];
  __syncthreads();
  pdl_wait();
  if (s_stopped) return;
  const long long t = s_t;
  const unsigned long long seq = s_seq;
  const int set = (int)(seq & 1ull);
  const int rows = n_params + kLpWords;
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5, gstride = gridDim.x * nw;
  const int w0 = blockIdx.x * nw + (int)(threadIdx.x >> 5);
  // ---- phase 1: this rank's rows into every rank's mailbox ----
  for (int gw = w0; gw < rows; gw += gstride) {
    const double v = reduce_row(gw, grad_part, n_rows, stride, n_params, loss_part, n_loss_rows, red);
    if (lane < pa.world) mbox_slot(s_box[lane], set, pa.rank, rows)[gw] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[0], 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    if (threadIdx.x == 0) ticket[0] = 0u;
    __threadfence_system();
    if (threadIdx.x < pa.world) st_release_sys_u64(&s_box[threadIdx.x]->flag[set][pa.rank], seq);
  }
  // ---- phase 2: the rank sum (fixed rank order) and the update ----
  if (threadIdx.x == 0) {
    // a peer that never arrives (a dead rank) must not hang the device: trap
    // after 30 s, the host sees a launch error instead of a hang
    const unsigned long long t0 = globaltimer();
    for (int r = 0; r < pa.world; ++r)
      while (ld_acquire_sys_u64(&mine->flag[set][r]) < seq) {
        __nanosleep(64);
        if (globaltimer() - t0 > 30000000000ull) __trap();
      }
  }
  __syncthreads();
  auto rank_sum = [&](int row) {
    double s = 0.0;
    for (int r = 0; r < pa.world; ++r) s += __ldcv(&mbox_slot(mine, set, r, rows)[row]);
    return s;
  };
  const float lr = s_f[0], c1 = s_f[1], c2 = s_f[2];
  if (lane == 0)
    for (int gw = w0; gw < rows; gw += gstride) {
      const double total = rank_sum(gw);
      red[gw] = total;
      if (adam && gw < n_params) {
        const float p0 = a.params[gw], m0 = a.m[gw], v0 = a.v[gw];
        double gd = total;
        if (gw == a.eps_grad_slot) gd += rank_sum(n_params + kLpEpsGrad);
        const float g = (float)gd;
        if (!isfinite(g)) atomicOr(&ticket[1], 1u);
        bk[gw] = p0;
        bk[n_params + gw] = m0;
        bk[2 * n_params + gw] = v0;
        adam_update(g, m0, v0, p0, lr, c1, c2, a.m[gw], a.v[gw], a.params[gw]);
      }
    }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[2], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (!adam) {
    if (threadIdx.x == 0) {
      ticket[2] = 0u;
      mine->seq = seq;
    }
    return;
  }
  const int bad = __ldcg(&ticket[1]) != 0u || __ldcg(&red[n_params + kLpBad]) != 0.0;
  if (bad) {  // all or nothing (identical decision on every rank: the same sums)
    for (int p = threadIdx.x; p < n_params; p += blockDim.x) {
      a.params[p] = __ldcg(&bk[p]);
      a.m[p] = __ldcg(&bk[n_params + p]);
      a.v[p] = __ldcg(&bk[2 * n_params + p]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ticket[1] = 0u;
    ticket[2] = 0u;
    mine->seq = seq;
    if (bad) {
      a.st->stopped = 1;
      a.st->stop_reason = 3;
      a.st->abort_step = t;
    } else {
      train_bookkeeping(a, t, s_f[0]);
    }
  }
}

__global__ void mark_start_kernel(TrainState* st) { st->t_prev = globaltimer(); }

// vpinn_gpu_run_steps after a finished vpinn_gpu_train: the run's stop
// (budget, coefficient tolerance, plateau) is lifted so further epochs run
// with no stop criteria; Adam moments and the step count are kept.  An abort
// (reason 3) stays stopped (the host refuses to resume it).
__global__ void resume_kernel(TrainState* st) {
  if (st->stopped && st->stop_reason != 3) {
    st->stopped = 0;
    st->stop_reason = 0;
    st->iterations = 0x7fffffffffffffffLL;
    st->has_eps_tol = 0;
    st->has_loss_tol = 0;
  }
  st->t_prev = globaltimer();
}

// L2 flush, second half: after the flush buffer (> L2) has been written, read
// it back so L2 holds clean lines of the flush buffer and no dirty write-back
// of it is left to compete with the next timed kernel.
__global__ void flush_read_kernel(const int4* __restrict__ buf, size_t n16, int* sink) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const int4 v = __ldcg(buf + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;  // keeps the loads; practically never taken
}

// ---------------------------------------------------------------------------
// Standalone contraction (losses.hpp:91-168) over device-resident ux/uy/eps
// for cells too large for a warp's ring (the split path, Q > 128: C3's
// 40x40 rules, forward_sine.json, inverse_eps.json).  One pass over the
// premultipliers with the work spread over (cell, row segment) ITEMS, not
// cells, so a few big cells still fill every SM:
//   contract_rows_kernel    persistent, 256 threads, two CTAs per SM; each
//                           CTA streams its items' rows through an NST-stage
//                           cp.async.bulk ring of R-row stages (~25 KB);
//                           per stage every thread takes the quadrature
//                           points q = t + 256 m of the R rows:
//                             phase A  partial dot products G_x[r,:] s_x,
//                                      G_y[r,:] s_y (, T[r,:] c) -> a fixed
//                                      warp-then-CTA reduction -> r_j and the
//                                      loss terms (losses.hpp:122-136)
//                             phase B  adjoint columns sum_j G[j][q] rbar_j,
//                                      accumulated in registers over the item
//                           and writes the item's partial columns to part
//   contract_rows_reduce    thread per (cell, q): the cell's item partials in
//                           item order -> uxb / uyb / eb (losses.hpp:145-160)
// Deterministic: fixed row / item / warp order everywhere, per-CTA loss words
// from a static item assignment.
struct ContractArgs {
  const float* tens[3];
  const float* forcing;
  int E, T, Q, nt;
  const float* ux;
  const float* uy;
  const float* eps;  // spatial source
  float* uxb;
  float* uyb;
  float* eb;
  float* res;  // optional residuals [k][j]
  float e_fixed;
  const float* e_param;  // scalar source: pointer to the trainable value
  int eps_source;
  float bx, by;
  float rscale, inv_nt;
  int rows;            // R: rows per ring stage (<= kCRowsMax)
  int seg_rows;        // rows per item (a multiple of R, or the whole cell)
  int items_per_cell;  // ceil(T / seg_rows)
  int n_items;         // E * items_per_cell
  int tstride;         // floats per tensor inside a stage (R * Q + 8, 16B multiple)
  int stage_floats;    // nt * tstride
  int nstage;          // ring depth (<= kCRMaxStages)
  int qstride;         // floats per point vector in shared memory (Q rounded to 4)
  float* part;         // [item][3][qstride] partial adjoint columns
  double* loss_part;   // [gridDim.x][kLpWords]
  const int* stop_flag;
  int rr_mq;  // contract_rowreg_kernel: M4 (> 0, float4 rows) or -M (scalar); 0: contract_rows_kernel.  items_per_cell = segments per CTA
};

constexpr int kCThreads = 256;
constexpr int kCRThreads = 512;  // contract_rows_kernel
constexpr int kCRowsMax = 16;
constexpr int kCQMax = 8192;  // points per cell this kernel serves

// ring (nstage stages) | s_x, s_y, c | adjoint column accumulators (nt) | row scalars | barriers
constexpr int kCRMaxStages = 6;
__host__ __device__ constexpr size_t contract_rows_smem_bytes(int stage_floats, int qstride, int nt, int nstage) {
  return sizeof(float) * ((size_t)nstage * stage_floats + (3 + (size_t)nt) * qstride + 3 * kCRowsMax +
                          3 * (kCRThreads / 32)) +
         sizeof(uint64_t) * kCRMaxStages + 64;
}

// rows [row0, row0 + nr) of cell k, nt tensors, into one ring stage
__device__ __forceinline__ void cr_issue(const ContractArgs& a, int k, int row0, int nr, float* stage, uint64_t* bar) {
  const size_t grow0 = (size_t)k * a.T + row0;
  uint32_t total = 0;
  for (int t = 0; t < a.nt; ++t) total += seg_of(a.tens[t] + grow0 * a.Q, (size_t)nr * a.Q).bytes;
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, total);
  for (int t = 0; t < a.nt; ++t) {
    const Seg g = seg_of(a.tens[t] + grow0 * a.Q, (size_t)nr * a.Q);
    bulk_g2s(stage + t * a.tstride, g.src, g.bytes, bar);
  }
}

// this CTA's stage sequence: its contiguous item range [i0, i1) (consecutive
// items mostly share a cell, so the cell's point vectors load rarely), each
// item split into ceil(nrows / R) stages; a cursor walks it
struct CrCursor {
  int item, sub;
};
__device__ __forceinline__ void cr_geom(const ContractArgs& a, int item, int& k, int& r_begin, int& r_end) {
  k = item / a.items_per_cell;
  const int b = item - k * a.items_per_cell;
  r_begin = b * a.seg_rows;
  r_end = min(a.T, r_begin + a.seg_rows);
}
__device__ __forceinline__ void cr_next(const ContractArgs& a, CrCursor& c) {
  int k, rb, re;
  cr_geom(a, c.item, k, rb, re);
  if (rb + (c.sub + 1) * a.rows < re) {
    ++c.sub;
  } else {
    ++c.item;
    c.sub = 0;
  }
}

__global__ void __launch_bounds__(kCRThreads, 1) contract_rows_kernel(const ContractArgs a) {
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  constexpr int NW = kCRThreads / 32;
  extern __shared__ __align__(128) float cs[];
  float* ring = cs;
  float* sx = ring + (size_t)a.nstage * a.stage_floats;
  float* sy = sx + a.qstride;
  float* cv = sy + a.qstride;
  float* acc = cv + a.qstride;                   // [nt][qstride] adjoint columns of the item
  float* rbv = acc + (size_t)a.nt * a.qstride;   // [3][kCRowsMax] rbar, r^2, rbar (gx + gy)
  float* segp = rbv + 3 * kCRowsMax;             // [row][segment][3] partial dots
  uint64_t* bars = reinterpret_cast<uint64_t*>(segp + 3 * NW);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool spatial = a.eps_source == 2;
  const bool conv = a.nt == 3;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  const int Q = a.Q;
  const int i0 = (int)((long long)a.n_items * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)a.n_items * (blockIdx.x + 1) / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < a.nstage; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  CrCursor pc{i0, 0};  // producer (thread 0)
  if (tid == 0) {
    for (int s = 0; s < a.nstage && pc.item < i1; ++s) {
      int k, rb, re;
      cr_geom(a, pc.item, k, rb, re);
      const int r0 = rb + pc.sub * a.rows;
      cr_issue(a, k, r0, min(a.rows, re - r0), ring + (size_t)s * a.stage_floats, &bars[s]);
      cr_next(a, pc);
    }
  }
  double acc_v = 0.0, acc_eg = 0.0;  // thread 0
  uint32_t parity = 0u;
  int stage_i = 0, k_prev = -1;
  for (CrCursor c{i0, 0}; c.item < i1;) {
    int k, rb, re;
    cr_geom(a, c.item, k, rb, re);
    const int r0 = rb + c.sub * a.rows, nr = min(a.rows, re - r0);
    if (c.sub == 0) {
      const size_t pb = (size_t)k * Q;
      for (int q = tid; q < Q; q += kCRThreads) {
        if (k != k_prev) {  // the cell's point vectors (s_x, s_y, bx ux + by uy)
          const float ux = a.ux[pb + q], uy = a.uy[pb + q];
          const float ep = spatial ? a.eps[pb + q] : 1.0f;
          sx[q] = spatial ? ep * ux : ux;
          sy[q] = spatial ? ep * uy : uy;
          cv[q] = a.bx * ux + a.by * uy;
        }
        acc[q] = 0.f;
        acc[a.qstride + q] = 0.f;
        if (conv) acc[2 * a.qstride + q] = 0.f;
      }
      k_prev = k;
      __syncthreads();
    }
    const int st = stage_i % a.nstage;
    mbar_wait(&bars[st], (parity >> st) & 1u);
    parity ^= 1u << st;
    const float* stage = ring + (size_t)st * a.stage_floats;
    const size_t grow0 = (size_t)k * a.T + r0;
    const float* Gx = stage + pre_of(a.tens[0] + grow0 * Q);
    const float* Gy = stage + a.tstride + pre_of(a.tens[1] + grow0 * Q);
    const float* Tv = conv ? stage + 2 * a.tstride + pre_of(a.tens[2] + grow0 * Q) : Gx;
    // phase A: warp task = (row, segment of the points); lanes over q with
    // two interleaved chains per tensor; fixed xor tree, segments summed in
    // order by one thread per row
    const int nseg = max(1, NW / nr);
    const int qseg = (Q + nseg - 1) / nseg;
    for (int task = wid; task < nr * nseg; task += NW) {
      const int r = task / nseg, sg = task - r * nseg;
      const int qa = sg * qseg, qb = min(Q, qa + qseg);
      const float* gxr = Gx + r * Q;
      const float* gyr = Gy + r * Q;
      const float* tr = Tv + r * Q;
      float gx0 = 0.f, gy0 = 0.f, t0 = 0.f, gx1 = 0.f, gy1 = 0.f, t1 = 0.f;
      int q = qa + lane;
      for (; q + 32 < qb; q += 64) {
        gx0 = fmaf(gxr[q], sx[q], gx0);
        gy0 = fmaf(gyr[q], sy[q], gy0);
        gx1 = fmaf(gxr[q + 32], sx[q + 32], gx1);
        gy1 = fmaf(gyr[q + 32], sy[q + 32], gy1);
        if (conv) {
          t0 = fmaf(tr[q], cv[q], t0);
          t1 = fmaf(tr[q + 32], cv[q + 32], t1);
        }
      }
      if (q < qb) {
        gx0 = fmaf(gxr[q], sx[q], gx0);
        gy0 = fmaf(gyr[q], sy[q], gy0);
        if (conv) t0 = fmaf(tr[q], cv[q], t0);
      }
      float gx = gx0 + gx1, gy = gy0 + gy1, t = t0 + t1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gx += __shfl_xor_sync(0xffffffffu, gx, o);
        gy += __shfl_xor_sync(0xffffffffu, gy, o);
        if (conv) t += __shfl_xor_sync(0xffffffffu, t, o);
      }
      if (lane == 0) {
        segp[3 * task + 0] = gx;
        segp[3 * task + 1] = gy;
        segp[3 * task + 2] = t;
      }
    }
    __syncthreads();
    if (tid < nr) {  // one thread per row: segments in order -> r_j
      const int r = tid;
      float gx = 0.f, gy = 0.f, t = 0.f;
      for (int sg = 0; sg < nseg; ++sg) {
        gx += segp[3 * (r * nseg + sg) + 0];
        gy += segp[3 * (r * nseg + sg) + 1];
        t += segp[3 * (r * nseg + sg) + 2];
      }
      const int j = r0 + r;
      float res = spatial ? gx + gy : e_fixed * (gx + gy);
      if (conv) res += t;
      res -= a.forcing[(size_t)k * a.T + j];
      if (a.res) a.res[(size_t)k * a.T + j] = res;
      const float rb2 = a.rscale * res;
      rbv[r] = rb2;
      rbv[kCRowsMax + r] = res * res;
      rbv[2 * kCRowsMax + r] = rb2 * (gx + gy);
    }
    __syncthreads();
    if (tid == 0)
      for (int r = 0; r < nr; ++r) {
        acc_v += (double)(rbv[kCRowsMax + r] * a.inv_nt);
        acc_eg += (double)rbv[2 * kCRowsMax + r];
      }
    // phase B: thread per point, the item's adjoint columns (even / odd rows
    // as two chains, joined in a fixed order)
    for (int q = tid; q < Q; q += kCRThreads) {
      float tx0 = acc[q], ty0 = acc[a.qstride + q], tt0 = conv ? acc[2 * a.qstride + q] : 0.f;
      float tx1 = 0.f, ty1 = 0.f, tt1 = 0.f;
      int r = 0;
      for (; r + 1 < nr; r += 2) {
        const float ra = rbv[r], rc = rbv[r + 1];
        tx0 = fmaf(Gx[r * Q + q], ra, tx0);
        ty0 = fmaf(Gy[r * Q + q], ra, ty0);
        tx1 = fmaf(Gx[(r + 1) * Q + q], rc, tx1);
        ty1 = fmaf(Gy[(r + 1) * Q + q], rc, ty1);
        if (conv) {
          tt0 = fmaf(Tv[r * Q + q], ra, tt0);
          tt1 = fmaf(Tv[(r + 1) * Q + q], rc, tt1);
        }
      }
      if (r < nr) {
        const float ra = rbv[r];
        tx0 = fmaf(Gx[r * Q + q], ra, tx0);
        ty0 = fmaf(Gy[r * Q + q], ra, ty0);
        if (conv) tt0 = fmaf(Tv[r * Q + q], ra, tt0);
      }
      acc[q] = tx0 + tx1;
      acc[a.qstride + q] = ty0 + ty1;
      if (conv) acc[2 * a.qstride + q] = tt0 + tt1;
    }
    __syncthreads();  // the stage and the row scalars are consumed
    if (tid == 0 && pc.item < i1) {
      int pk, prb, pre;
      cr_geom(a, pc.item, pk, prb, pre);
      const int pr0 = prb + pc.sub * a.rows;
      cr_issue(a, pk, pr0, min(a.rows, pre - pr0), ring + (size_t)st * a.stage_floats, &bars[st]);
      cr_next(a, pc);
    }
    ++stage_i;
    const int item = c.item;
    const bool last_sub = r0 + nr >= re;
    cr_next(a, c);
    if (last_sub) {  // the item's partial columns (each thread its own points)
      float* pp = a.part + (size_t)item * 3 * a.qstride;
      for (int q = tid; q < Q; q += kCRThreads) {
        pp[q] = acc[q];
        pp[a.qstride + q] = acc[a.qstride + q];
        if (conv) pp[2 * a.qstride + q] = acc[2 * a.qstride + q];
      }
    }
  }
  if (tid == 0) {
    double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
    for (int w = 0; w < kLpWords; ++w) lp[w] = 0.0;
    lp[kLpVar] = acc_v;
    lp[kLpEpsGrad] = acc_eg;
  }
}

// thread per (cell, q): the cell's item partials in item order -> adjoints
__global__ void contract_rows_reduce_kernel(const ContractArgs a) {
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  const size_t n = (size_t)a.E * a.Q;
  const bool spatial = a.eps_source == 2;
  const bool conv = a.nt == 3;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / a.Q), q = (int)(i - (size_t)k * a.Q);
    const float* pp = a.part + (size_t)k * a.items_per_cell * 3 * a.qstride + q;
    float tx = 0.f, ty = 0.f, tt = 0.f;
    for (int b = 0; b < a.items_per_cell; ++b, pp += 3 * a.qstride) {
      tx += pp[0];
      ty += pp[a.qstride];
      if (conv) tt += pp[2 * a.qstride];
    }
    float ox, oy;
    if (spatial) {
      const float ep = a.eps[i];
      ox = ep * tx;
      oy = ep * ty;
      if (a.eb) a.eb[i] = a.ux[i] * tx + a.uy[i] * ty;
    } else {
      ox = e_fixed * tx;
      oy = e_fixed * ty;
    }
    if (conv) {
      ox = fmaf(a.bx, tt, ox);
      oy = fmaf(a.by, tt, oy);
    }
    a.uxb[i] = ox;
    a.uyb[i] = oy;
  }
}

// ---------------------------------------------------------------------------
// Row contraction with WARP-OWNED rows (nt = 2, Q <= 1,664): the split
// path's Algorithm 3 (losses.hpp:111-166) without CTA barriers on the
// streaming path.
//   * CTA b owns the contiguous global row range [R0(b), R1(b)) of the
//     cell-major row sequence (row g = k T + j), R0(b) = floor(E T b / G):
//     row-level balance whatever E, T;
//   * inside a cell segment of that range warp w takes rows w, w + 8, ...;
//     each warp streams its rows through its OWN ring of nsw one-row
//     cp.async.bulk stages, copies a row into registers and re-issues the
//     stage for its next row at once;
//   * per row: r_j = e (G_x[j,:] s_x + G_y[j,:] s_y) - f_j (a fixed xor
//     tree), then the adjoint columns acc[q] += rbar_j G[j][q] in registers;
//   * the cell's point vectors (ux, uy, eps) arrive by cp.async.bulk into one
//     of two buffers, issued a segment ahead (float4 layout);
//   * at the end of a cell segment the eight warps' columns meet in shared
//     memory (x, then y) and are summed in warp order into the segment's
//     partial part[b * cmax + s] (s = the segment's index in the CTA's range).
// contract_rowreg_reduce_kernel then sums, per (cell, q), the partials of the
// CTAs covering the cell in CTA order.  Deterministic throughout.
constexpr int kRRThreads = 256;
constexpr int kRRWarps = kRRThreads / 32;
// points per lane: NV = 4 M4 (VEC: lane l holds q = 128 m + 4 l + i, float4
// rows, Q % 4 == 0) or M4 (scalar: q = 32 m + l); every row / vector buffer is
// padded to VP = 32 NV points; vector pads are zero and row pads finite, so
// no point needs a bounds check
__host__ __device__ constexpr int rr_pad_points(int m4, bool vec) { return vec ? 128 * m4 : 32 * m4; }
constexpr int kRRMaxStages = 8;  // row stages per warp
__host__ __device__ constexpr size_t contract_rowreg_smem_bytes(int rs, int qstride, int vpad, int nsw) {
  // per-warp ring [nsw][2][rs] | warp column slots [8][qstride] | vectors [2][3][vpad] | loss words | barriers
  return sizeof(float) * ((size_t)kRRWarps * nsw * 2 * rs + (size_t)kRRWarps * qstride + 6 * (size_t)vpad) +
         sizeof(double) * 2 * kRRWarps + sizeof(uint64_t) * (kRRWarps * kRRMaxStages + 2);
}
__device__ __forceinline__ int rr_row0(long long rows_total, int b, int G) {
  return (int)(rows_total * b / G);
}

template <int M4, bool VEC>
__global__ void __launch_bounds__(kRRThreads, 1) contract_rowreg_kernel(const ContractArgs a) {
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  constexpr int NW = kRRWarps;
  constexpr int NV = VEC ? 4 * M4 : M4;  // points per lane
  constexpr int VP = 32 * NV;            // padded points per row / vector
  extern __shared__ __align__(128) float cs[];
  const int Q = a.Q, T = a.T, rs = a.tstride, qs = a.qstride, nsw = a.nstage;
  const float* __restrict__ tx0 = a.tens[0];
  const float* __restrict__ ty0 = a.tens[1];
  float* ring = cs;                                   // [NW][nsw][2][rs], rs >= VP + 8
  float* slots = ring + (size_t)NW * nsw * 2 * rs;    // [NW][qs]
  float* vbuf = slots + (size_t)NW * qs;              // [2][3][VP]: ux, uy, eps of a segment
  double* lw = reinterpret_cast<double*>(vbuf + 6 * VP);  // [2][NW]
  uint64_t* bars = reinterpret_cast<uint64_t*>(lw + 2 * NW);  // [NW][kRRMaxStages] rows, then [2] vectors
  uint64_t* vbar = bars + NW * kRRMaxStages;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool spatial = a.eps_source == 2;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  const float rscale = a.rscale, inv_nt = a.inv_nt;
  const long long rows_total = (long long)a.E * T;
  const int R0 = rr_row0(rows_total, blockIdx.x, gridDim.x), R1 = rr_row0(rows_total, blockIdx.x + 1, gridDim.x);
  float* wring = ring + (size_t)w * nsw * 2 * rs;
  uint64_t* wbar = bars + w * kRRMaxStages;
  // pads: rows [Q, rs) of every stage and vectors [Q, VP) zero (the bulk
  // copies write [0, Q) plus at most 12 bytes of finite slop)
  for (int slot = w; slot < NW * nsw * 2; slot += NW)
    for (int i = Q + lane; i < rs; i += 32) ring[(size_t)slot * rs + i] = 0.f;
  for (int v = w; v < 6; v += NW)
    for (int i = Q + lane; i < VP; i += 32) vbuf[v * VP + i] = 0.f;
  if (tid == 0) {
    for (int i = 0; i < NW * kRRMaxStages + 2; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  __syncthreads();
  auto seg_end = [&](int g) { return min(R1, (g / T + 1) * T); };
  // the point vectors of the segment starting at row s0 into buffer vb (VEC: by
  // cp.async.bulk on vbar[vb]; scalar layout: plain loads, pads stay zero)
  auto issue_vec = [&](int s0, int vb) {
    const size_t pb = (size_t)(s0 / T) * Q;
    float* d = vbuf + vb * 3 * VP;
    const uint32_t bytes = 4u * (uint32_t)Q;
    mbar_arrive_expect_tx(&vbar[vb], (spatial ? 3u : 2u) * bytes);
    bulk_g2s(d, a.ux + pb, bytes, &vbar[vb]);
    bulk_g2s(d + VP, a.uy + pb, bytes, &vbar[vb]);
    if (spatial) bulk_g2s(d + 2 * VP, a.eps + pb, bytes, &vbar[vb]);
  };
  if constexpr (VEC) {
    if (tid == 0) {
      if (R0 < R1) issue_vec(R0, 0);
      if (seg_end(R0) < R1) issue_vec(seg_end(R0), 1);
    }
  }
  // this warp's rows: in each cell segment [s0, s1) of [R0, R1), s0 + w + NW i
  auto first_in = [&](int s0) {  // the warp's first row at or after segment start s0 (or R1)
    for (; s0 < R1; s0 = seg_end(s0))
      if (s0 + w < seg_end(s0)) return s0 + w;
    return R1;
  };
  // producer cursor (pg, end of its segment pe)
  auto next_row = [&](int& g, int& e) {
    if (g + NW < e) {
      g += NW;
    } else {
      g = first_in(e);
      e = g < R1 ? seg_end(g) : R1;
    }
  };
  auto issue = [&](int g, int st) {
    const Seg sxg = seg_of(tx0 + (size_t)g * Q, (size_t)Q), syg = seg_of(ty0 + (size_t)g * Q, (size_t)Q);
    float* stage = wring + (size_t)st * 2 * rs;
    fence_proxy_async();
    mbar_arrive_expect_tx(&wbar[st], sxg.bytes + syg.bytes);
    bulk_g2s(stage, sxg.src, sxg.bytes, &wbar[st]);
    bulk_g2s(stage + rs, syg.src, syg.bytes, &wbar[st]);
  };
  // the warp's producer cursor: nsw rows in flight, row i of the warp's
  // sequence in stage i % nsw
  int pg = first_in(R0), pe = pg < R1 ? seg_end(pg) : R1;
  for (int st = 0; st < nsw; ++st) {
    if (lane == 0 && pg < R1) issue(pg, st);
    if (pg < R1) next_row(pg, pe);
  }
  uint32_t parity = 0u;
  int cst = 0;  // consumer stage
  double lv = 0.0, leg = 0.0;  // lane 0: this warp's loss terms
  float ax[NV], ay[NV];
  // lane-local point offset of value v: VEC 128 (v / 4) + 4 lane + v % 4, scalar 32 v + lane
  auto qof = [&](int v) { return VEC ? 128 * (v >> 2) + 4 * lane + (v & 3) : 32 * v + lane; };
  int s_idx = 0;
  for (int s0 = R0; s0 < R1; s0 = seg_end(s0), ++s_idx) {
    const int s1 = seg_end(s0), k = s0 / T, vb = s_idx & 1;
    const float* vx_ = vbuf + vb * 3 * VP;
    const float* vy_ = vx_ + VP;
    const float* ve_ = vx_ + 2 * VP;
    if constexpr (VEC) {
      mbar_wait(&vbar[vb], (s_idx >> 1) & 1);
    } else {
      float* d = vbuf + vb * 3 * VP;
      const size_t pb = (size_t)k * Q;
      for (int q = tid; q < Q; q += kRRThreads) {
        d[q] = a.ux[pb + q];
        d[VP + q] = a.uy[pb + q];
        if (spatial) d[2 * VP + q] = a.eps[pb + q];
      }
      __syncthreads();
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) ax[v] = ay[v] = 0.f;
    for (int g = s0 + w; g < s1; g += NW) {
      const float frow = a.forcing[g];  // forcing (k, j) at k T + j = g
      mbar_wait(&wbar[cst], (parity >> cst) & 1u);
      parity ^= 1u << cst;
      const float* stage = wring + (size_t)cst * 2 * rs;
      float rx[NV], ry[NV];
      if constexpr (VEC) {
#pragma unroll
        for (int m = 0; m < M4; ++m) {
          const float4 x4 = lds4(stage + 128 * m + 4 * lane), y4 = lds4(stage + rs + 128 * m + 4 * lane);
          rx[4 * m] = x4.x, rx[4 * m + 1] = x4.y, rx[4 * m + 2] = x4.z, rx[4 * m + 3] = x4.w;
          ry[4 * m] = y4.x, ry[4 * m + 1] = y4.y, ry[4 * m + 2] = y4.z, ry[4 * m + 3] = y4.w;
        }
      } else {
        const float* gx = stage + pre_of(tx0 + (size_t)g * Q);
        const float* gy = stage + rs + pre_of(ty0 + (size_t)g * Q);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          rx[v] = gx[32 * v + lane];
          ry[v] = gy[32 * v + lane];
        }
      }
      __syncwarp();  // every lane has its share of the row: the stage is free
      if (lane == 0 && pg < R1) issue(pg, cst);
      if (pg < R1) next_row(pg, pe);
      cst = cst + 1 == nsw ? 0 : cst + 1;
      float d[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      auto dot = [&](auto sp) {
        constexpr bool SP = decltype(sp)::value;
#pragma unroll
        for (int v = 0; v < NV; v += (VEC ? 4 : 1)) {
          float vx[4], vy[4];
          if constexpr (VEC) {
            const float4 x4 = lds4(vx_ + qof(v)), y4 = lds4(vy_ + qof(v));
            vx[0] = x4.x, vx[1] = x4.y, vx[2] = x4.z, vx[3] = x4.w;
            vy[0] = y4.x, vy[1] = y4.y, vy[2] = y4.z, vy[3] = y4.w;
            if constexpr (SP) {
              const float4 e4 = lds4(ve_ + qof(v));
              vx[0] *= e4.x, vx[1] *= e4.y, vx[2] *= e4.z, vx[3] *= e4.w;
              vy[0] *= e4.x, vy[1] *= e4.y, vy[2] *= e4.z, vy[3] *= e4.w;
            }
          } else {
            vx[0] = vx_[qof(v)];
            vy[0] = vy_[qof(v)];
            if constexpr (SP) {
              vx[0] *= ve_[qof(v)];
              vy[0] *= ve_[qof(v)];
            }
          }
#pragma unroll
          for (int i = 0; i < (VEC ? 4 : 1); ++i) {
            d[(v + i) & 3] = fmaf(rx[v + i], vx[i], d[(v + i) & 3]);
            d[4 + ((v + i) & 3)] = fmaf(ry[v + i], vy[i], d[4 + ((v + i) & 3)]);
          }
        }
      };
      if (spatial)
        dot(std::true_type{});
      else
        dot(std::false_type{});
      float dx = (d[0] + d[1]) + (d[2] + d[3]), dy = (d[4] + d[5]) + (d[6] + d[7]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dx += __shfl_xor_sync(0xffffffffu, dx, o);
        dy += __shfl_xor_sync(0xffffffffu, dy, o);
      }
      float res = spatial ? dx + dy : e_fixed * (dx + dy);
      res -= frow;
      const float rb = rscale * res;
      if (lane == 0) {
        if (a.res) a.res[g] = res;
        lv += (double)(res * res * inv_nt);
        leg += (double)(rb * (dx + dy));
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        ax[v] = fmaf(rx[v], rb, ax[v]);
        ay[v] = fmaf(ry[v], rb, ay[v]);
      }
    }
    // the segment's columns (x, then y): warps' slots, summed in warp order
    float* pp = a.part + ((size_t)blockIdx.x * a.items_per_cell + s_idx) * 3 * qs;
    float* my = slots + (size_t)w * qs;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if constexpr (VEC) {
#pragma unroll
        for (int m = 0; m < M4; ++m) {
          const int q = 128 * m + 4 * lane;
          if (q < Q)
            sts4(my + q, t ? make_float4(ay[4 * m], ay[4 * m + 1], ay[4 * m + 2], ay[4 * m + 3])
                           : make_float4(ax[4 * m], ax[4 * m + 1], ax[4 * m + 2], ax[4 * m + 3]));
        }
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int q = qof(v);
          if (q < Q) my[q] = t ? ay[v] : ax[v];
        }
      }
      __syncthreads();
      if constexpr (VEC) {
        for (int q = 4 * tid; q < Q; q += 4 * kRRThreads) {
          float4 v = lds4(slots + q);
#pragma unroll
          for (int ww = 1; ww < NW; ++ww) {
            const float4 u = lds4(slots + (size_t)ww * qs + q);
            v.x += u.x, v.y += u.y, v.z += u.z, v.w += u.w;
          }
          *reinterpret_cast<float4*>(pp + t * qs + q) = v;
        }
      } else {
        for (int q = tid; q < Q; q += kRRThreads) {
          float v = slots[q];
#pragma unroll
          for (int ww = 1; ww < NW; ++ww) v += slots[(size_t)ww * qs + q];
          pp[t * qs + q] = v;
        }
      }
      __syncthreads();  // slots read; after t = 1 also every warp is done with vector buffer vb
    }
    if constexpr (VEC) {
      const int s2 = seg_end(s1 < R1 ? s1 : R1);  // start of segment s_idx + 2
      if (tid == 0 && s1 < R1 && s2 < R1) issue_vec(s2, vb);
    }
  }
  if (lane == 0) {
    lw[w] = lv;
    lw[NW + w] = leg;
  }
  __syncthreads();
  if (tid == 0) {
    double v = 0.0, g = 0.0;
    for (int ww = 0; ww < NW; ++ww) {
      v += lw[ww];
      g += lw[NW + ww];
    }
    double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
    for (int i = 0; i < kLpWords; ++i) lp[i] = 0.0;
    lp[kLpVar] = v;
    lp[kLpEpsGrad] = g;
  }
}

// thread per (cell, q): the partials of the CTAs covering the cell, in CTA
// order.  cover[k] = (first CTA b, its segment index for cell k, last CTA):
// the CTAs after the first start inside cell k (segment 0)
__global__ void contract_rowreg_reduce_kernel(const ContractArgs a, const int4* __restrict__ cover) {
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  const size_t n = (size_t)a.E * a.Q;
  const bool spatial = a.eps_source == 2;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  const int qs = a.qstride, cmax = a.items_per_cell;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / a.Q), q = (int)(i - (size_t)k * a.Q);
    const int4 cv = cover[k];
    const float* pp = a.part + ((size_t)cv.x * cmax + cv.y) * 3 * qs + q;
    float tx = pp[0], ty = pp[qs];
    for (int b = cv.x + 1; b <= cv.z; ++b) {
      pp = a.part + (size_t)b * cmax * 3 * qs + q;
      tx += pp[0];
      ty += pp[qs];
    }
    float ox, oy;
    if (spatial) {
      const float ep = a.eps[i];
      ox = ep * tx;
      oy = ep * ty;
      if (a.eb) a.eb[i] = a.ux[i] * tx + a.uy[i] * ty;
    } else {
      ox = e_fixed * tx;
      oy = e_fixed * ty;
    }
    a.uxb[i] = ox;
    a.uyb[i] = oy;
  }
}

// ---------------------------------------------------------------------------
// split-path penalty (losses.hpp:389-415): ub and loss words from u
__global__ void __launch_bounds__(256) penalty_kernel(const float* __restrict__ u_pen, int n_bnd,
                                                      int n_sen, const float* __restrict__ bval,
                                                      const float* __restrict__ sval,
                                                      float bscale, float sscale,
                                                      float* __restrict__ ub,
                                                      double* __restrict__ loss_part,
                                                      const int* stop_flag) {
  if (stop_flag != nullptr && *stop_flag != 0) return;
  __shared__ double red[2][8];
  double sb = 0.0, ss = 0.0;
  const int n = n_bnd + n_sen;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < n_bnd) {
      const float d = u_pen[i] - bval[i];
      sb += (double)(d * d);
      ub[i] = bscale * d;
    } else {
      const float d = u_pen[i] - sval[i - n_bnd];
      ss += (double)(d * d);
      ub[i] = sscale * d;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sb += __shfl_down_sync(0xffffffffu, sb, o);
    ss += __shfl_down_sync(0xffffffffu, ss, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = sb;
    red[1][warp] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tb = 0.0, ts = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      tb += red[0][w];
      ts += red[1][w];
    }
    double* lp = loss_part + (size_t)blockIdx.x * kLpWords;
    for (int w = 0; w < kLpWords; ++w) lp[w] = 0.0;
    lp[kLpBnd] = tb;
    lp[kLpSen] = ts;
  }
}

}  // namespace vpg

namespace vpg {

// FP32 FFMA throughput microbenchmark (roofline denominator for the
// FFMA-bound step kernel): 8 independent chains per thread, register
// operands, 2 flops per FFMA.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-7f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5f) out[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace vpg
