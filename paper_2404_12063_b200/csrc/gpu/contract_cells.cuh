// HBM-streaming contraction for cells of <= 128 quadrature points: the
// roofline kernel of SURVEY 8d (variational_loss_tensor, losses.hpp:91-168,
// on device-resident derivatives).  Each CTA owns a contiguous cell range
// and streams it in chunks of whole cells (cc = floor(128/Q) cells, so phase
// A has one slab row per thread and phase B one point per thread) through a
// continuous nstage-deep cp.async.bulk ring; derivatives in, adjoints
// out, both coalesced.  Every premultiplier byte is read from HBM once.
#pragma once

#include "step_kernel.cuh"

namespace vpg {

constexpr int kCCThreads = 128;
constexpr int kCCMaxStages = 4;

struct CellContractArgs {
  const float* tens[3];
  const float* forcing;
  int E, T, Q, nt;
  int cc;            // cells per chunk
  int tstride;       // floats per tensor inside a stage
  int vstride;       // floats per derivative vector inside a stage (cc*Q + 8, 16B multiple)
  int fstride;       // floats for the forcing columns inside a stage (cc*T + 8)
  int stage_floats;  // nt * tstride + 3 * vstride + fstride
  int nstage;        // ring depth (<= kCCMaxStages)
  int use_ldgsts;    // 1: all threads stage with cp.async 16 B; 0: one thread, cp.async.bulk
  const float* ux;
  const float* uy;
  const float* eps;
  float* uxb;
  float* uyb;
  float* eb;
  float* res;
  float e_fixed;
  const float* e_param;
  int eps_source;
  float bx, by;
  float rscale, inv_nt;
  double* loss_part;
  const int* stop_flag;
};

__host__ __device__ constexpr size_t cell_contract_smem_bytes(int stage_floats, int nstage) {
  return sizeof(float) * ((size_t)nstage * stage_floats + 3 * 2 * kCCThreads + 4 * kCCThreads) +
         sizeof(uint64_t) * kCCMaxStages + 64;
}

// 16-byte-aligned superset copy descriptor of [p, p + n floats)
struct Seg {
  const char* src;
  uint32_t bytes;
};
__device__ __forceinline__ Seg seg_of(const float* p, size_t n) {
  const char* s = reinterpret_cast<const char*>(p);
  const char* al = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(s) & ~uintptr_t(15));
  const uint32_t pre = (uint32_t)(s - al);
  return {al, (pre + (uint32_t)(n * 4) + 15u) & ~15u};
}

// one stage = the chunk's premultiplier slabs + its ux / uy (/ eps) and
// forcing columns, all by cp.async.bulk on one mbarrier
static __device__ __noinline__ void cc_issue(const CellContractArgs& a, int cell0, int ncell, float* stage,
                                             uint64_t* bar) {
  const size_t TQ = (size_t)a.T * a.Q;
  const size_t np = (size_t)ncell * a.Q, p0 = (size_t)cell0 * a.Q;
  Seg sg[7];
  float* dst[7];
  int n = 0;
  for (int t = 0; t < a.nt; ++t) {
    sg[n] = seg_of(a.tens[t] + (size_t)cell0 * TQ, (size_t)ncell * TQ);
    dst[n++] = stage + t * a.tstride;
  }
  float* v = stage + a.nt * a.tstride;
  sg[n] = seg_of(a.ux + p0, np);
  dst[n++] = v;
  sg[n] = seg_of(a.uy + p0, np);
  dst[n++] = v + a.vstride;
  if (a.eps_source == 2) {
    sg[n] = seg_of(a.eps + p0, np);
    dst[n++] = v + 2 * a.vstride;
  }
  sg[n] = seg_of(a.forcing + (size_t)cell0 * a.T, (size_t)ncell * a.T);
  dst[n++] = v + 3 * a.vstride;
  uint32_t total = 0;
  for (int i = 0; i < n; ++i) total += sg[i].bytes;
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, total);
  for (int i = 0; i < n; ++i) bulk_g2s(dst[i], sg[i].src, sg[i].bytes, bar);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// the same stage filled cooperatively by all threads with 16-byte cp.async
// (one commit group per stage; an empty group when there is nothing to load)
__device__ __forceinline__ void cc_issue_threads(const CellContractArgs& a, int cell0, int ncell, float* stage) {
  const size_t TQ = (size_t)a.T * a.Q;
  const size_t np = (size_t)ncell * a.Q, p0 = (size_t)cell0 * a.Q;
  auto copy = [&](const float* p, size_t n, float* dst) {
    const Seg g = seg_of(p, n);
    const uint32_t chunks = g.bytes >> 4;
    for (uint32_t i = threadIdx.x; i < chunks; i += kCCThreads)
      cp_async16(reinterpret_cast<char*>(dst) + 16 * i, g.src + 16 * i);
  };
  for (int t = 0; t < a.nt; ++t) copy(a.tens[t] + (size_t)cell0 * TQ, (size_t)ncell * TQ, stage + t * a.tstride);
  float* v = stage + a.nt * a.tstride;
  copy(a.ux + p0, np, v);
  copy(a.uy + p0, np, v + a.vstride);
  if (a.eps_source == 2) copy(a.eps + p0, np, v + 2 * a.vstride);
  copy(a.forcing + (size_t)cell0 * a.T, (size_t)ncell * a.T, v + 3 * a.vstride);
}

__device__ __forceinline__ uint32_t pre_of(const float* p) {
  return (uint32_t)((reinterpret_cast<uintptr_t>(p) & 15u) >> 2);
}

__global__ void __launch_bounds__(kCCThreads, 2) contract_cells_kernel(const CellContractArgs a) {
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  extern __shared__ __align__(128) float cs[];
  float* ring = cs;
  float* sx = ring + (size_t)a.nstage * a.stage_floats;  // [2][128]: double-buffered per chunk
  float* sy = sx + 2 * kCCThreads;
  float* cv = sy + 2 * kCCThreads;
  float* rbarv = cv + 2 * kCCThreads;
  float* rsqv = rbarv + kCCThreads;
  float* rgev = rsqv + kCCThreads;
  float* spare = rgev + kCCThreads;
  uint64_t* bars = reinterpret_cast<uint64_t*>(spare + kCCThreads);
  const int tid = threadIdx.x;
  // contiguous cell range of this CTA, in chunks of cc cells
  const int c0 = (int)((long long)a.E * blockIdx.x / gridDim.x);
  const int c1 = (int)((long long)a.E * (blockIdx.x + 1) / gridDim.x);
  const int nch = (c1 - c0 + a.cc - 1) / a.cc;
  if (tid == 0) {
    for (int s = 0; s < a.nstage; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (a.use_ldgsts) {
    // prologue: nstage-1 groups in flight, one group per stage
    for (int c = 0; c < a.nstage - 1; ++c) {
      if (c < nch) {
        const int k0 = c0 + c * a.cc;
        cc_issue_threads(a, k0, min(a.cc, c1 - k0), ring + c * a.stage_floats);
      }
      cp_async_commit();
    }
  } else if (tid == 0) {
    for (int c = 0; c < a.nstage && c < nch; ++c) {
      const int k0 = c0 + c * a.cc;
      cc_issue(a, k0, min(a.cc, c1 - k0), ring + c * a.stage_floats, &bars[c]);
    }
  }
  const bool spatial = a.eps_source == 2;
  const bool conv = a.nt == 3;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  const int T = a.T, Q = a.Q;
  const size_t TQ = (size_t)T * Q;
  double acc_v = 0.0, acc_eg = 0.0;
  uint32_t parity = 0u;
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    const int st = c % a.nstage;
    const int k0 = c0 + c * a.cc;
    const int ncell = min(a.cc, c1 - k0);
    const int np = ncell * Q, nr = ncell * T;
    float* bx_ = sx + (c & 1) * kCCThreads;
    float* by_ = sy + (c & 1) * kCCThreads;
    float* bc_ = cv + (c & 1) * kCCThreads;
    const size_t pb = (size_t)k0 * Q;
    float* stage = ring + st * a.stage_floats;
    const float* Gx = stage + pre_of(a.tens[0] + (size_t)k0 * TQ);
    const float* Gy = stage + a.tstride + pre_of(a.tens[1] + (size_t)k0 * TQ);
    const float* Tv = conv ? stage + 2 * a.tstride + pre_of(a.tens[2] + (size_t)k0 * TQ) : nullptr;
    const float* vb = stage + a.nt * a.tstride;
    const float* vux = vb + pre_of(a.ux + pb);
    const float* vuy = vb + a.vstride + pre_of(a.uy + pb);
    const float* vep = spatial ? vb + 2 * a.vstride + pre_of(a.eps + pb) : nullptr;
    const float* vf = vb + 3 * a.vstride + pre_of(a.forcing + (size_t)k0 * T);
    if (a.use_ldgsts) {
      // keep nstage-1 stages in flight: issue chunk c+nstage-1 into the stage
      // freed at the end of chunk c-1, then wait for chunk c's group
      const int cn = c + a.nstage - 1;
      if (cn < nch) {
        const int kn = c0 + cn * a.cc;
        cc_issue_threads(a, kn, min(a.cc, c1 - kn), ring + (cn % a.nstage) * a.stage_floats);
      }
      cp_async_commit();
      if (a.nstage == 2) cp_async_wait<1>();
      else if (a.nstage == 3) cp_async_wait<2>();
      else cp_async_wait<3>();
      __syncthreads();
    } else {
      mbar_wait(&bars[st], (parity >> st) & 1u);
      parity ^= 1u << st;
    }
    float ux = 0.f, uy = 0.f, ep = 1.f;
    if (tid < np) {
      ux = vux[tid];
      uy = vuy[tid];
      if (spatial) ep = vep[tid];
      bx_[tid] = spatial ? ep * ux : ux;
      by_[tid] = spatial ? ep * uy : uy;
      bc_[tid] = a.bx * ux + a.by * uy;
    }
    __syncthreads();  // derivative rows visible
    // phase A: one slab row per thread
    if (tid < nr) {
      const int kk = tid / T;
      const float* xs = bx_ + kk * Q;
      const float* ys = by_ + kk * Q;
      const float* gxr = Gx + (size_t)tid * Q;
      const float* gyr = Gy + (size_t)tid * Q;
      // four interleaved partial sums per dot product: short FMA chains
      float ax[4] = {0.f, 0.f, 0.f, 0.f}, ay[4] = {0.f, 0.f, 0.f, 0.f}, at[4] = {0.f, 0.f, 0.f, 0.f};
      const float* cr = bc_ + kk * Q;
      const float* tr = conv ? Tv + (size_t)tid * Q : gxr;
      int q = 0;
#pragma unroll 2
      for (; q + 3 < Q; q += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ax[u] = fmaf(gxr[q + u], xs[q + u], ax[u]);
          ay[u] = fmaf(gyr[q + u], ys[q + u], ay[u]);
          if (conv) at[u] = fmaf(tr[q + u], cr[q + u], at[u]);
        }
      }
      for (; q < Q; ++q) {
        ax[0] = fmaf(gxr[q], xs[q], ax[0]);
        ay[0] = fmaf(gyr[q], ys[q], ay[0]);
        if (conv) at[0] = fmaf(tr[q], cr[q], at[0]);
      }
      const float gx = (ax[0] + ax[1]) + (ax[2] + ax[3]);
      const float gy = (ay[0] + ay[1]) + (ay[2] + ay[3]);
      const float tt = (at[0] + at[1]) + (at[2] + at[3]);
      float r = spatial ? gx + gy : e_fixed * (gx + gy);
      r += tt;
      r -= vf[tid];
      if (a.res) a.res[(size_t)k0 * T + tid] = r;
      rsqv[tid] = r * r;
      const float rb = a.rscale * r;
      rbarv[tid] = rb;
      rgev[tid] = rb * (gx + gy);
    }
    __syncthreads();
    // phase B: one point per thread; all T rows of its cell are in the chunk
    if (tid < np) {
      const int kk = tid / Q, q = tid - kk * Q;
      const float* rb = rbarv + kk * T;
      const float* gxc = Gx + (size_t)kk * TQ + q;
      const float* gyc = Gy + (size_t)kk * TQ + q;
      const float* tc = conv ? Tv + (size_t)kk * TQ + q : gxc;
      float bx4[4] = {0.f, 0.f, 0.f, 0.f}, by4[4] = {0.f, 0.f, 0.f, 0.f}, bt4[4] = {0.f, 0.f, 0.f, 0.f};
      int j = 0;
#pragma unroll 2
      for (; j + 3 < T; j += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          bx4[u] = fmaf(gxc[(size_t)(j + u) * Q], rb[j + u], bx4[u]);
          by4[u] = fmaf(gyc[(size_t)(j + u) * Q], rb[j + u], by4[u]);
          if (conv) bt4[u] = fmaf(tc[(size_t)(j + u) * Q], rb[j + u], bt4[u]);
        }
      }
      for (; j < T; ++j) {
        bx4[0] = fmaf(gxc[(size_t)j * Q], rb[j], bx4[0]);
        by4[0] = fmaf(gyc[(size_t)j * Q], rb[j], by4[0]);
        if (conv) bt4[0] = fmaf(tc[(size_t)j * Q], rb[j], bt4[0]);
      }
      const float tx = (bx4[0] + bx4[1]) + (bx4[2] + bx4[3]);
      const float ty = (by4[0] + by4[1]) + (by4[2] + by4[3]);
      const float tt = (bt4[0] + bt4[1]) + (bt4[2] + bt4[3]);
      float ox, oy;
      if (spatial) {
        ox = ep * tx;
        oy = ep * ty;
        a.eb[pb + tid] = ux * tx + uy * ty;
      } else {
        ox = e_fixed * tx;
        oy = e_fixed * ty;
      }
      if (conv) {
        ox = fmaf(a.bx, tt, ox);
        oy = fmaf(a.by, tt, oy);
      }
      a.uxb[pb + tid] = ox;
      a.uyb[pb + tid] = oy;
    }
    // per-cell squared residuals and eps gradient, rows in order
    if (tid < ncell) {
      float s = 0.f, g = 0.f;
      for (int j = 0; j < T; ++j) {
        s += rsqv[tid * T + j];
        g += rgev[tid * T + j];
      }
      spare[tid] = s * a.inv_nt;
      spare[kCCThreads / 2 + tid] = g;
    }
    __syncthreads();
    if (tid == 0) {
      for (int k = 0; k < ncell; ++k) {
        acc_v += (double)spare[k];
        acc_eg += (double)spare[kCCThreads / 2 + k];
      }
      if (!a.use_ldgsts && c + a.nstage < nch) {
        const int k2 = c0 + (c + a.nstage) * a.cc;
        cc_issue(a, k2, min(a.cc, c1 - k2), stage, &bars[st]);
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

}  // namespace vpg
