// Cross-CTA reduction, Adam + device-side trainer bookkeeping, the
// standalone HBM-streaming contraction (split path and roofline report) and
// the penalty kernel of the split path.
#pragma once

#include "step_kernel.cuh"

namespace vpg {

// ---------------------------------------------------------------------------
// Cross-CTA reduction of the per-CTA partials (fp64, fixed order): one warp
// per parameter over the param-major partial rows (all loads of a lane in
// flight at once, then a fixed shuffle tree); the trailing kLpWords warps sum
// the loss words the same way.  red = [gradient | loss words].
constexpr int kRedThreads = 256;
constexpr int kRedWarps = kRedThreads / 32;

__device__ __forceinline__ void reduce_body(const float* __restrict__ grad_part, int n_rows, int stride,
                                            int n_params, const double* __restrict__ loss_part, int n_loss_rows,
                                            double* __restrict__ red) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const double* src_d = nullptr;
  const float* src_f = nullptr;
  int n = 0, step = 1;
  if (gw < n_params) {
    src_f = grad_part + (size_t)gw * stride;
    n = n_rows;
  } else if (gw < n_params + kLpWords) {
    src_d = loss_part + (gw - n_params);
    n = n_loss_rows;
    step = kLpWords;
  } else {
    return;
  }
  double acc = 0.0;
  if (src_f != nullptr) {
#pragma unroll 8
    for (int c = lane; c < n; c += 32) acc += (double)src_f[c];
  } else {
#pragma unroll 8
    for (int c = lane; c < n; c += 32) acc += src_d[(size_t)c * step];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[gw] = acc;
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

// adam_step (trainer.hpp:34-59) + train-loop bookkeeping (trainer.hpp:316-370)
// for one epoch.  One CTA of 1024 threads.  IEEE intrinsics keep the update
// in the reference's operation order (no FMA contraction).
__device__ __forceinline__ void adam_body(const AdamArgs& a) {
  TrainState* st = a.st;
  const long long t = st->step + 1;
  const int n = a.n_params;
  const double* red = a.red;
  const double lw_v = red[n + kLpVar], lw_b = red[n + kLpBnd], lw_s = red[n + kLpSen];
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
  // loss parts in the reference's Real semantics
  const float Lv = (float)lw_v;
  const float Lb = a.n_bnd > 0 ? (float)(lw_b / a.n_bnd) : 0.0f;
  const float Ls = a.n_sen > 0 ? (float)(lw_s / a.n_sen) : 0.0f;
  const float total_f = __fadd_rn(__fadd_rn(Lv, __fmul_rn(a.tau_f, Lb)), __fmul_rn(a.gamma_f, Ls));
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
  const float b1 = 0.9f, b2 = 0.999f, omb1 = 1.0f - b1, omb2 = 1.0f - b2;
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
    const float m = __fadd_rn(__fmul_rn(b1, m0), __fmul_rn(omb1, g));
    const float v = __fadd_rn(__fmul_rn(b2, v0), __fmul_rn(omb2, __fmul_rn(g, g)));
    a.m[p] = m;
    a.v[p] = v;
    const float mh = __fdiv_rn(m, c1);
    const float vh = __fdiv_rn(v, c2);
    a.params[p] = __fsub_rn(p0, __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), 1e-8f)));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double total = (double)total_f;
    const unsigned long long now = globaltimer();
    st->step = t;
    double eps_now = __longlong_as_double(0x7ff8000000000000ll);
    if (st->tracks_eps) eps_now = (double)a.params[st->eps_slot];
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
}

__global__ void __launch_bounds__(1024) adam_kernel(const AdamArgs a) {
  if (a.st->stopped) return;
  adam_body(a);
}

// single-GPU epoch tail: the cross-CTA reduction of reduce_kernel, then the
// last CTA to finish (atomic ticket, release/acquire fences) applies Adam
__global__ void __launch_bounds__(kRAThreads) reduce_adam_kernel(const float* __restrict__ grad_part, int n_rows,
                                                                   int stride, int n_params,
                                                                   const double* __restrict__ loss_part,
                                                                   int n_loss_rows, double* __restrict__ red,
                                                                   unsigned* ticket, const AdamArgs a) {
  pdl_trigger();
  pdl_wait();
  if (a.st->stopped) return;
  __shared__ int last;
  reduce_body(grad_part, n_rows, stride, n_params, loss_part, n_loss_rows, red);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next epoch (graph replay)
  adam_body(a);
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
// Standalone contraction (losses.hpp:91-168) over device-resident ux/uy/eps:
// split path (Q > 128) and the HBM-roofline measurement.  256 threads; a
// tile = whole cells with at most pmax points (or one cell); premultiplier
// rows streamed through an NST-stage cp.async.bulk ring.
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
  int cells_per_tile, n_tiles;
  int chunk_rows, stage_floats, tstride, nstage;
  int pmax;
  double* loss_part;  // [gridDim.x][kLpWords]
  const int* stop_flag;
};

constexpr int kCThreads = 256;

__device__ __forceinline__ void c_issue(const ContractArgs& a, int cell0, int row0, int nrows,
                                        float* stage, uint64_t* bar) {
  const size_t grow0 = (size_t)cell0 * a.T + row0;
  uint32_t total = 0;
  const char* src[3];
  uint32_t n16[3];
  for (int t = 0; t < a.nt; ++t) {
    const char* s = reinterpret_cast<const char*>(a.tens[t] + grow0 * a.Q);
    const char* al = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(s) & ~uintptr_t(15));
    const uint32_t pre = (uint32_t)(s - al);
    n16[t] = (pre + (uint32_t)nrows * a.Q * 4u + 15u) & ~15u;
    src[t] = al;
    total += n16[t];
  }
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, total);
  for (int t = 0; t < a.nt; ++t) bulk_g2s(stage + t * a.tstride, src[t], n16[t], bar);
}

__device__ __forceinline__ const float* c_ptr(const ContractArgs& a, int cell0, int row0,
                                              const float* stage, int t) {
  const size_t grow0 = (size_t)cell0 * a.T + row0;
  const uintptr_t s = reinterpret_cast<uintptr_t>(a.tens[t] + grow0 * a.Q);
  return stage + t * a.tstride + ((s & 15u) >> 2);
}

__host__ __device__ constexpr size_t contract_smem_bytes(int pmax, int chunk_rows, int stage_floats,
                                                         int nstage) {
  return sizeof(float) * ((size_t)9 * pmax + 4 * (size_t)((chunk_rows + 3) & ~3) + 2 * 1024 +
                          (size_t)nstage * stage_floats) +
         sizeof(uint64_t) * 8 + 64;
}

__global__ void __launch_bounds__(kCThreads) contract_kernel(const ContractArgs a) {
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  extern __shared__ __align__(128) float cs[];
  float* ring = cs;
  float* sx = ring + (size_t)a.nstage * a.stage_floats;
  float* sy = sx + a.pmax;
  float* cv = sy + a.pmax;
  float* vux = cv + a.pmax;
  float* vuy = vux + a.pmax;
  float* vep = vuy + a.pmax;
  float* atx = vep + a.pmax;
  float* aty = atx + a.pmax;
  float* att = aty + a.pmax;
  const int rows4 = (a.chunk_rows + 3) & ~3;
  float* rbarv = att + a.pmax;
  float* rsqv = rbarv + rows4;
  float* rgev = rsqv + rows4;
  float* cellsq = rgev + rows4 + rows4;  // 1024
  float* cellge = cellsq + 1024;         // 1024
  uint64_t* bars = reinterpret_cast<uint64_t*>(cellge + 1024);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < a.nstage; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t parity = 0u;  // bit s = phase parity of ring stage s
  const bool spatial = a.eps_source == 2;
  const bool conv = a.nt == 3;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  double acc_v = 0.0, acc_eg = 0.0;
  for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const int cell0 = tile * a.cells_per_tile;
    const int ncell = min(a.cells_per_tile, a.E - cell0);
    const int np = ncell * a.Q;
    const int nrows = ncell * a.T;
    const int nchunks = (nrows + a.chunk_rows - 1) / a.chunk_rows;
    if (tid == 0)
      for (int c = 0; c < a.nstage && c < nchunks; ++c) {
        const int r0 = c * a.chunk_rows;
        c_issue(a, cell0, r0, min(a.chunk_rows, nrows - r0), ring + c * a.stage_floats, &bars[c]);
      }
    const size_t pb = (size_t)cell0 * a.Q;
    for (int p = tid; p < np; p += kCThreads) {
      const float ux = a.ux[pb + p], uy = a.uy[pb + p];
      const float ep = spatial ? a.eps[pb + p] : 1.0f;
      vux[p] = ux;
      vuy[p] = uy;
      vep[p] = ep;
      sx[p] = spatial ? ep * ux : ux;
      sy[p] = spatial ? ep * uy : uy;
      cv[p] = a.bx * ux + a.by * uy;
      atx[p] = 0.f;
      aty[p] = 0.f;
      att[p] = 0.f;
    }
    for (int k = tid; k < ncell; k += kCThreads) {
      cellsq[k] = 0.f;
      cellge[k] = 0.f;
    }
    __syncthreads();
    for (int c = 0; c < nchunks; ++c) {
      const int st = c % a.nstage;
      const int r0 = c * a.chunk_rows;
      const int nr = min(a.chunk_rows, nrows - r0);
      float* stage = ring + st * a.stage_floats;
      mbar_wait(&bars[st], (parity >> st) & 1u);
      parity ^= 1u << st;
      const float* Gx = c_ptr(a, cell0, r0, stage, 0);
      const float* Gy = c_ptr(a, cell0, r0, stage, 1);
      const float* Tv = conv ? c_ptr(a, cell0, r0, stage, 2) : nullptr;
      // row dot products, one WARP per row (lanes over q, fixed xor tree):
      // the large cells this kernel serves (Q > 128) make a thread-serial
      // dot of length Q the latency chain of the whole contraction
      const int lane = tid & 31, wid = tid >> 5;
      for (int r = wid; r < nr; r += kCThreads / 32) {
        const int gr = r0 + r;
        const int kk = gr / a.T;
        const int j = gr - kk * a.T;
        const float* xs = sx + kk * a.Q;
        const float* ys = sy + kk * a.Q;
        const float* gxr = Gx + (size_t)r * a.Q;
        const float* gyr = Gy + (size_t)r * a.Q;
        const float* cr = cv + kk * a.Q;
        const float* tr = conv ? Tv + (size_t)r * a.Q : gxr;
        float gx = 0.f, gy = 0.f, t = 0.f;
        for (int q = lane; q < a.Q; q += 32) {
          gx = fmaf(gxr[q], xs[q], gx);
          gy = fmaf(gyr[q], ys[q], gy);
          if (conv) t = fmaf(tr[q], cr[q], t);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          gx += __shfl_xor_sync(0xffffffffu, gx, o);
          gy += __shfl_xor_sync(0xffffffffu, gy, o);
          t += __shfl_xor_sync(0xffffffffu, t, o);
        }
        if (lane == 0) {
          float res = spatial ? gx + gy : e_fixed * (gx + gy);
          if (conv) res += t;
          res -= a.forcing[(size_t)(cell0 + kk) * a.T + j];
          if (a.res) a.res[(size_t)(cell0 + kk) * a.T + j] = res;
          rsqv[r] = res * res;
          const float rb = a.rscale * res;
          rbarv[r] = rb;
          rgev[r] = rb * (gx + gy);
        }
      }
      __syncthreads();
      // points of the cells touched by this chunk
      const int k_lo = r0 / a.T, k_hi = (r0 + nr - 1) / a.T;
      for (int p = k_lo * a.Q + tid; p < (k_hi + 1) * a.Q; p += kCThreads) {
        const int kk = p / a.Q, q = p - kk * a.Q;
        const int lo = max(r0, kk * a.T), hi = min(r0 + nr, (kk + 1) * a.T);
        float tx = atx[p], ty = aty[p], tt = att[p];
        for (int gr = lo; gr < hi; ++gr) {
          const int r = gr - r0;
          const float rb = rbarv[r];
          tx = fmaf(Gx[(size_t)r * a.Q + q], rb, tx);
          ty = fmaf(Gy[(size_t)r * a.Q + q], rb, ty);
          if (conv) tt = fmaf(Tv[(size_t)r * a.Q + q], rb, tt);
        }
        atx[p] = tx;
        aty[p] = ty;
        att[p] = tt;
      }
      for (int kk = k_lo + tid; kk <= k_hi; kk += kCThreads) {
        const int lo = max(r0, kk * a.T), hi = min(r0 + nr, (kk + 1) * a.T);
        float s = cellsq[kk], g = cellge[kk];
        for (int gr = lo; gr < hi; ++gr) {
          s += rsqv[gr - r0];
          g += rgev[gr - r0];
        }
        cellsq[kk] = s;
        cellge[kk] = g;
      }
      __syncthreads();
      if (tid == 0 && c + a.nstage < nchunks) {
        const int r2 = (c + a.nstage) * a.chunk_rows;
        c_issue(a, cell0, r2, min(a.chunk_rows, nrows - r2), stage, &bars[st]);
      }
    }
    for (int p = tid; p < np; p += kCThreads) {
      float ox, oy;
      if (spatial) {
        ox = vep[p] * atx[p];
        oy = vep[p] * aty[p];
        if (a.eb) a.eb[pb + p] = vux[p] * atx[p] + vuy[p] * aty[p];
      } else {
        ox = e_fixed * atx[p];
        oy = e_fixed * aty[p];
      }
      if (conv) {
        ox = fmaf(a.bx, att[p], ox);
        oy = fmaf(a.by, att[p], oy);
      }
      a.uxb[pb + p] = ox;
      a.uyb[pb + p] = oy;
    }
    if (tid == 0)
      for (int k = 0; k < ncell; ++k) {
        acc_v += (double)(cellsq[k] * a.inv_nt);
        acc_eg += (double)cellge[k];
      }
    __syncthreads();
  }
  if (tid == 0) {
    double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
    for (int w = 0; w < kLpWords; ++w) lp[w] = 0.0;
    lp[kLpVar] = acc_v;
    lp[kLpEpsGrad] = acc_eg;
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
