// HBM-streaming whole-cell contraction: the roofline kernel of SURVEY 8d
// (variational_loss_tensor, losses.hpp:91-168, on device-resident
// derivatives).  Each warp streams whole cells (premultiplier slabs +
// ux/uy(/eps) + forcing column, one cp.async.bulk group per cell) through its
// own ring; every premultiplier byte is read from HBM once.
#pragma once

#include "step_kernel.cuh"

namespace vpg {

constexpr int kCCMaxStages = 4;

struct CellContractArgs {
  const float* tens[3];
  const float* forcing;
  int E, T, Q, nt;
  int cc;            // cells per stage (1: warp-per-cell)
  int tstride;       // floats per tensor inside a stage
  int vstride;       // floats per derivative vector inside a stage (cc*Q + 8, 16B multiple)
  int fstride;       // floats for the forcing columns inside a stage (cc*T + 8)
  int stage_floats;  // nt * tstride + 3 * vstride + fstride
  int nstage;        // ring depth (<= kCCMaxStages)
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
// forcing columns, all by cp.async.bulk on one mbarrier.  Inlined: a
// non-inlined callee would take the kernel-parameter struct through a stack
// copy (local memory), i.e. L2 round trips on every issue.
__device__ __forceinline__ void cc_issue(const CellContractArgs& a, int cell0, int ncell, float* stage,
                                         uint64_t* bar) {
  const size_t TQ = (size_t)a.T * a.Q;
  const size_t np = (size_t)ncell * a.Q, p0 = (size_t)cell0 * a.Q;
  float* v = stage + a.nt * a.tstride;
  // every segment, in a fixed order, handed to f(seg, dst); no local arrays
  auto each = [&](auto&& f) {
    f(seg_of(a.tens[0] + (size_t)cell0 * TQ, (size_t)ncell * TQ), stage);
    f(seg_of(a.tens[1] + (size_t)cell0 * TQ, (size_t)ncell * TQ), stage + a.tstride);
    if (a.nt == 3) f(seg_of(a.tens[2] + (size_t)cell0 * TQ, (size_t)ncell * TQ), stage + 2 * a.tstride);
    f(seg_of(a.ux + p0, np), v);
    f(seg_of(a.uy + p0, np), v + a.vstride);
    if (a.eps_source == 2) f(seg_of(a.eps + p0, np), v + 2 * a.vstride);
    f(seg_of(a.forcing + (size_t)cell0 * a.T, (size_t)ncell * a.T), v + 3 * a.vstride);
  };
  uint32_t total = 0;
  each([&](Seg g, float*) { total += g.bytes; });
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, total);
  each([&](Seg g, float* dst) { bulk_g2s(dst, g.src, g.bytes, bar); });
}

__device__ __forceinline__ uint32_t pre_of(const float* p) {
  return (uint32_t)((reinterpret_cast<uintptr_t>(p) & 15u) >> 2);
}

// ---------------------------------------------------------------------------
// Warp-per-cell variant: every warp owns an interleaved cell sequence
// (cell gw, gw + NW, ...) and its own nstage-deep cp.async.bulk ring, one
// cell per stage, so no CTA-wide barrier sits on the streaming path (the
// CTA-wide version above was barrier-bound at ~2.3 TB/s).  Per cell:
//   prep   lanes over q: s_x = eps*ux (spatial) or ux, s_y, c = bx*ux + by*uy
//   phase A lanes over test functions j: r_j (losses.hpp:122-136)
//   phase B lanes over quadrature points q: adjoints (losses.hpp:145-156)
// Loss words: fp32 per cell (fixed xor-shuffle tree), fp64 across cells,
// CTA partials in warp order.
constexpr int kCWMaxWarps = 16;  // warps per CTA: 8, 12 or 16, the most that fit (latency-bound lanes)

__host__ __device__ constexpr int cw_scratch_floats(int T, int Q) {
  return 3 * ((Q + 3) & ~3) + ((T + 3) & ~3);
}

__host__ __device__ constexpr size_t cell_warp_smem_bytes(int nwarps, int stage_floats, int nstage, int T, int Q) {
  return sizeof(float) * (size_t)nwarps * ((size_t)nstage * stage_floats + cw_scratch_floats(T, Q)) +
         sizeof(uint64_t) * nwarps * kCCMaxStages + sizeof(double) * 2 * nwarps + 64;
}

// FT, FQ > 0: the cell shape fixed at compile time (T = FT, Q = FQ <= 32; the
// benchmark gear's 5x5 / 5x5 cells): the point vectors of phase A and the
// residual adjoints of phase B sit in registers and every loop is unrolled
// without predication, so each premultiplier entry costs one shared-memory
// load and one FMA per phase
template <int kCWWarps, int FT = 0, int FQ = 0>
__global__ void __launch_bounds__(32 * kCWWarps, 1) contract_warp_kernel(const CellContractArgs a) {
  constexpr bool kFixed = FT > 0 && FQ > 0;
  static_assert(!kFixed || (FT <= 32 && FQ <= 32), "fixed cell shape: T, Q <= 32");
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  extern __shared__ __align__(128) float cs[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int T = kFixed ? FT : a.T, Q = kFixed ? FQ : a.Q;
  const size_t TQ = (size_t)T * Q;
  const int Q4 = (Q + 3) & ~3;
  float* ring = cs + (size_t)warp * a.nstage * a.stage_floats;
  float* scr = cs + (size_t)kCWWarps * a.nstage * a.stage_floats + (size_t)warp * cw_scratch_floats(T, Q);
  float* sxs = scr;
  float* sys = scr + Q4;
  float* cvs = scr + 2 * Q4;
  float* rbs = scr + 3 * Q4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(cs + (size_t)kCWWarps * ((size_t)a.nstage * a.stage_floats +
                                                                         cw_scratch_floats(T, Q)));
  double* red = reinterpret_cast<double*>(bars + kCWWarps * kCCMaxStages);
  uint64_t* wb = bars + warp * kCCMaxStages;
  const int gw = blockIdx.x * kCWWarps + warp;
  const int NW = gridDim.x * kCWWarps;
  const int n_my = gw < a.E ? (a.E - gw + NW - 1) / NW : 0;
  if (lane == 0) {
    for (int s = 0; s < a.nstage; ++s) mbar_init(&wb[s], 1);
    fence_mbar_init();
    for (int i = 0; i < a.nstage && i < n_my; ++i) cc_issue(a, gw + i * NW, 1, ring + i * a.stage_floats, &wb[i]);
  }
  __syncwarp();
  const bool spatial = a.eps_source == 2;
  const bool conv = a.nt == 3;
  const float e_fixed = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  double acc_v = 0.0, acc_eg = 0.0;
#pragma unroll 1
  for (int i = 0; i < n_my; ++i) {
    const int st = i % a.nstage;
    const int k = gw + i * NW;
    const size_t pb = (size_t)k * Q;
    float* stage = ring + st * a.stage_floats;
    mbar_wait(&wb[st], (uint32_t)((i / a.nstage) & 1));
    const float* Gx = stage + pre_of(a.tens[0] + (size_t)k * TQ);
    const float* Gy = stage + a.tstride + pre_of(a.tens[1] + (size_t)k * TQ);
    const float* Tv = conv ? stage + 2 * a.tstride + pre_of(a.tens[2] + (size_t)k * TQ) : nullptr;
    const float* vb = stage + a.nt * a.tstride;
    const float* vux = vb + pre_of(a.ux + pb);
    const float* vuy = vb + a.vstride + pre_of(a.uy + pb);
    const float* vep = spatial ? vb + 2 * a.vstride + pre_of(a.eps + pb) : nullptr;
    const float* vf = vb + 3 * a.vstride + pre_of(a.forcing + (size_t)k * T);
    for (int q = lane; q < Q; q += 32) {
      const float ux = vux[q], uy = vuy[q];
      const float ep = spatial ? vep[q] : 1.f;
      sxs[q] = spatial ? ep * ux : ux;
      sys[q] = spatial ? ep * uy : uy;
      cvs[q] = a.bx * ux + a.by * uy;
    }
    __syncwarp();
    // phase A: residual rows
    float lsq = 0.f, lge = 0.f;
    if constexpr (kFixed) {
      float sx[FQ], sy[FQ], cv[FQ];
#pragma unroll
      for (int q = 0; q < FQ; ++q) {
        sx[q] = sxs[q];
        sy[q] = sys[q];
        cv[q] = cvs[q];
      }
      const int j = lane;
      if (j < FT) {
        const float* gxr = Gx + j * FQ;
        const float* gyr = Gy + j * FQ;
        const float* tr = conv ? Tv + j * FQ : gxr;
        float ax[4] = {0.f, 0.f, 0.f, 0.f}, ay[4] = {0.f, 0.f, 0.f, 0.f}, at[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < FQ; ++q) {
          ax[q & 3] = fmaf(gxr[q], sx[q], ax[q & 3]);
          ay[q & 3] = fmaf(gyr[q], sy[q], ay[q & 3]);
          if (conv) at[q & 3] = fmaf(tr[q], cv[q], at[q & 3]);
        }
        const float gx = (ax[0] + ax[1]) + (ax[2] + ax[3]);
        const float gy = (ay[0] + ay[1]) + (ay[2] + ay[3]);
        const float tt = (at[0] + at[1]) + (at[2] + at[3]);
        float r = spatial ? gx + gy : e_fixed * (gx + gy);
        r += tt;
        r -= vf[j];
        if (a.res) a.res[(size_t)k * T + j] = r;
        const float rb = a.rscale * r;
        rbs[j] = rb;
        lsq = fmaf(r, r, lsq);
        lge = fmaf(rb, gx + gy, lge);
      }
    }
    for (int j = kFixed ? T : lane; j < T; j += 32) {
      const float* gxr = Gx + (size_t)j * Q;
      const float* gyr = Gy + (size_t)j * Q;
      const float* tr = conv ? Tv + (size_t)j * Q : gxr;
      float ax[4] = {0.f, 0.f, 0.f, 0.f}, ay[4] = {0.f, 0.f, 0.f, 0.f}, at[4] = {0.f, 0.f, 0.f, 0.f};
      int q = 0;
#pragma unroll 2
      for (; q + 3 < Q; q += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ax[u] = fmaf(gxr[q + u], sxs[q + u], ax[u]);
          ay[u] = fmaf(gyr[q + u], sys[q + u], ay[u]);
          if (conv) at[u] = fmaf(tr[q + u], cvs[q + u], at[u]);
        }
      }
      for (; q < Q; ++q) {
        ax[0] = fmaf(gxr[q], sxs[q], ax[0]);
        ay[0] = fmaf(gyr[q], sys[q], ay[0]);
        if (conv) at[0] = fmaf(tr[q], cvs[q], at[0]);
      }
      const float gx = (ax[0] + ax[1]) + (ax[2] + ax[3]);
      const float gy = (ay[0] + ay[1]) + (ay[2] + ay[3]);
      const float tt = (at[0] + at[1]) + (at[2] + at[3]);
      float r = spatial ? gx + gy : e_fixed * (gx + gy);
      r += tt;
      r -= vf[j];
      if (a.res) a.res[(size_t)k * T + j] = r;
      const float rb = a.rscale * r;
      rbs[j] = rb;
      lsq = fmaf(r, r, lsq);
      lge = fmaf(rb, gx + gy, lge);
    }
    __syncwarp();
    // phase B: adjoints per quadrature point
    if constexpr (kFixed) {
      float rb[FT];
#pragma unroll
      for (int j = 0; j < FT; ++j) rb[j] = rbs[j];
      const int q = lane;
      if (q < FQ) {
        const float* gxc = Gx + q;
        const float* gyc = Gy + q;
        const float* tc = conv ? Tv + q : gxc;
        float bx4[4] = {0.f, 0.f, 0.f, 0.f}, by4[4] = {0.f, 0.f, 0.f, 0.f}, bt4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < FT; ++j) {
          bx4[j & 3] = fmaf(gxc[j * FQ], rb[j], bx4[j & 3]);
          by4[j & 3] = fmaf(gyc[j * FQ], rb[j], by4[j & 3]);
          if (conv) bt4[j & 3] = fmaf(tc[j * FQ], rb[j], bt4[j & 3]);
        }
        const float tx = (bx4[0] + bx4[1]) + (bx4[2] + bx4[3]);
        const float ty = (by4[0] + by4[1]) + (by4[2] + by4[3]);
        const float tt = (bt4[0] + bt4[1]) + (bt4[2] + bt4[3]);
        float ox, oy;
        if (spatial) {
          const float ep = vep[q];
          ox = ep * tx;
          oy = ep * ty;
          a.eb[pb + q] = vux[q] * tx + vuy[q] * ty;
        } else {
          ox = e_fixed * tx;
          oy = e_fixed * ty;
        }
        if (conv) {
          ox = fmaf(a.bx, tt, ox);
          oy = fmaf(a.by, tt, oy);
        }
        a.uxb[pb + q] = ox;
        a.uyb[pb + q] = oy;
      }
    }
    for (int q = kFixed ? Q : lane; q < Q; q += 32) {
      const float* gxc = Gx + q;
      const float* gyc = Gy + q;
      const float* tc = conv ? Tv + q : gxc;
      float bx4[4] = {0.f, 0.f, 0.f, 0.f}, by4[4] = {0.f, 0.f, 0.f, 0.f}, bt4[4] = {0.f, 0.f, 0.f, 0.f};
      int j = 0;
#pragma unroll 2
      for (; j + 3 < T; j += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float rb = rbs[j + u];
          bx4[u] = fmaf(gxc[(size_t)(j + u) * Q], rb, bx4[u]);
          by4[u] = fmaf(gyc[(size_t)(j + u) * Q], rb, by4[u]);
          if (conv) bt4[u] = fmaf(tc[(size_t)(j + u) * Q], rb, bt4[u]);
        }
      }
      for (; j < T; ++j) {
        const float rb = rbs[j];
        bx4[0] = fmaf(gxc[(size_t)j * Q], rb, bx4[0]);
        by4[0] = fmaf(gyc[(size_t)j * Q], rb, by4[0]);
        if (conv) bt4[0] = fmaf(tc[(size_t)j * Q], rb, bt4[0]);
      }
      const float tx = (bx4[0] + bx4[1]) + (bx4[2] + bx4[3]);
      const float ty = (by4[0] + by4[1]) + (by4[2] + by4[3]);
      const float tt = (bt4[0] + bt4[1]) + (bt4[2] + bt4[3]);
      float ox, oy;
      if (spatial) {
        const float ep = vep[q];
        ox = ep * tx;
        oy = ep * ty;
        a.eb[pb + q] = vux[q] * tx + vuy[q] * ty;
      } else {
        ox = e_fixed * tx;
        oy = e_fixed * ty;
      }
      if (conv) {
        ox = fmaf(a.bx, tt, ox);
        oy = fmaf(a.by, tt, oy);
      }
      a.uxb[pb + q] = ox;
      a.uyb[pb + q] = oy;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lsq += __shfl_xor_sync(0xffffffffu, lsq, o);
      lge += __shfl_xor_sync(0xffffffffu, lge, o);
    }
    acc_v += (double)(lsq * a.inv_nt);
    acc_eg += (double)lge;
    __syncwarp();  // stage and scratch reads done before the refill
    if (lane == 0 && i + a.nstage < n_my) cc_issue(a, k + a.nstage * NW, 1, stage, &wb[st]);
  }
  if (lane == 0) {
    red[2 * warp] = acc_v;
    red[2 * warp + 1] = acc_eg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0, g = 0.0;
    for (int w = 0; w < kCWWarps; ++w) {
      v += red[2 * w];
      g += red[2 * w + 1];
    }
    double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
    for (int w = 0; w < kLpWords; ++w) lp[w] = 0.0;
    lp[kLpVar] = v;
    lp[kLpEpsGrad] = g;
  }
}

}  // namespace vpg
