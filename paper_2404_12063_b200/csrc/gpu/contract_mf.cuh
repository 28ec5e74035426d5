// Matrix-free variational contraction: Algorithm 3
// (variational_loss_tensor, losses.hpp:91-168) WITHOUT the precomputed
// premultiplier tensors.  The reference's premultipliers factor into the
// reference-square basis tables (basis.hpp:24-60, shared by every cell) and
// per-point geometry (geometry.hpp:75-141):
//   grad_x(k,j,q) = w_q (j22 dv_j/dxi - j12 dv_j/deta)      (the det cancels)
//   grad_y(k,j,q) = w_q (-j21 dv_j/dxi + j11 dv_j/deta)
//   test(k,j,q)   = w_q det v_j
// so, with alpha_q = w_q (j22 s_x - j21 s_y), beta_q = w_q (j11 s_y - j12 s_x)
// and gamma_q = w_q det (b_x u_x + b_y u_y),
//   g_j  = sum_q Bxi[j,q] alpha_q + Beta[j,q] beta_q     (= gx + gy)
//   t_j  = sum_q B[j,q] gamma_q,  r_j = eps g_j + t_j - F_j
// and the adjoints need only P_q = sum_j Bxi[j,q] rbar_j, M_q (Beta), V_q (B):
//   ux_bar = eps w (j22 P - j12 M) + b_x w det V,  uy_bar = eps w (j11 M - j21 P) + b_y w det V.
// HBM traffic per cell: 4 node coordinates, u_x / u_y in, the adjoints out
// and the forcing column (~4 (4 Q + T) + 40 bytes) instead of
// 4 n_t T Q bytes of premultipliers; the tables live in shared memory.
// fp32 arithmetic on the factored form: matches the tensor contraction to
// fp32 rounding (not bit-identical: the tensors are rounded from double).
#pragma once

#include "step_kernel.cuh"

namespace vpg {

struct MfContractArgs {
  const double* nodes;   // [n][2]
  const int32_t* elems;  // [E_global][4]
  int64_t e0;            // first global cell of this rank
  int E, T, Q;
  const float* tabs;     // [3][T][Q]: dv/dxi, dv/deta, v (float)
  const float* rule;     // [3][Q]: xi, eta, w (float)
  const float* forcing;  // [E][T] (local cells)
  const float* ux;       // [E*Q]
  const float* uy;
  float* uxb;
  float* uyb;
  float* res;            // [E][T] or null
  float e_fixed;
  const float* e_param;  // trainable scalar (eps_source 1)
  int eps_source;
  float bx, by;
  float rscale, inv_nt;
  double* loss_part;
};

constexpr int kMfWarps = 8;

__host__ __device__ constexpr int mf_scratch_floats(int T, int Q) {
  return 7 * ((Q + 3) & ~3) + ((T + 3) & ~3);
}
__host__ __device__ constexpr int mf_tab_floats(int T, int Q) { return (3 * T * Q + 3) & ~3; }
__host__ __device__ constexpr size_t mf_smem_bytes(int T, int Q) {
  return sizeof(float) * ((size_t)mf_tab_floats(T, Q) + 3 * ((Q + 3) & ~3) + (size_t)kMfWarps * mf_scratch_floats(T, Q)) +
         sizeof(double) * 2 * kMfWarps + 16;
}

__global__ void __launch_bounds__(32 * kMfWarps) contract_mf_kernel(const MfContractArgs a) {
  extern __shared__ __align__(16) float ms[];
  const int T = a.T, Q = a.Q, Q4 = (Q + 3) & ~3;
  float* tBx = ms;                 // [T][Q]
  float* tBy = tBx + T * Q;
  float* tB = tBy + T * Q;
  float* rxi = ms + mf_tab_floats(T, Q);  // [Q4]
  float* reta = rxi + Q4;
  float* rw = reta + Q4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* scr = rw + Q4 + (size_t)warp * mf_scratch_floats(T, Q);
  float* al = scr;                 // alpha_q
  float* be = al + Q4;             // beta_q
  float* ga = be + Q4;             // gamma_q
  float* j11 = ga + Q4;            // per-point Jacobian entries (reused by phase B)
  float* j12 = j11 + Q4;
  float* j21 = j12 + Q4;
  float* j22 = j21 + Q4;
  float* rb = j22 + Q4;            // rbar_j
  double* red = reinterpret_cast<double*>(ms + mf_tab_floats(T, Q) + 3 * Q4 + (size_t)kMfWarps * mf_scratch_floats(T, Q));
  for (int i = threadIdx.x; i < 3 * T * Q; i += blockDim.x) tBx[i] = a.tabs[i];
  for (int i = threadIdx.x; i < Q; i += blockDim.x) {
    rxi[i] = a.rule[i];
    reta[i] = a.rule[Q + i];
    rw[i] = a.rule[2 * Q + i];
  }
  __syncthreads();
  const bool conv = a.bx != 0.0f || a.by != 0.0f;
  const float e = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  double acc_v = 0.0, acc_eg = 0.0;
  const int gw = blockIdx.x * kMfWarps + warp, NW = gridDim.x * kMfWarps;
#pragma unroll 1
  for (int k = gw; k < a.E; k += NW) {
    // bilinear map of the cell (geometry.hpp:75-113), in double, per point in float
    const int4 en = reinterpret_cast<const int4*>(a.elems)[a.e0 + k];
    const double2 A = reinterpret_cast<const double2*>(a.nodes)[en.x];
    const double2 B = reinterpret_cast<const double2*>(a.nodes)[en.y];
    const double2 C = reinterpret_cast<const double2*>(a.nodes)[en.z];
    const double2 D = reinterpret_cast<const double2*>(a.nodes)[en.w];
    const float xc1 = (float)(0.25 * (-A.x + B.x + C.x - D.x)), xc2 = (float)(0.25 * (-A.x - B.x + C.x + D.x));
    const float xc3 = (float)(0.25 * (A.x - B.x + C.x - D.x));
    const float yc1 = (float)(0.25 * (-A.y + B.y + C.y - D.y)), yc2 = (float)(0.25 * (-A.y - B.y + C.y + D.y));
    const float yc3 = (float)(0.25 * (A.y - B.y + C.y - D.y));
    const size_t pb = (size_t)k * Q;
    for (int q = lane; q < Q; q += 32) {
      const float xi = rxi[q], eta = reta[q], w = rw[q];
      const float a11 = fmaf(xc3, eta, xc1), a12 = fmaf(yc3, eta, yc1);
      const float a21 = fmaf(xc3, xi, xc2), a22 = fmaf(yc3, xi, yc2);
      const float ux = a.ux[pb + q], uy = a.uy[pb + q];
      j11[q] = a11;
      j12[q] = a12;
      j21[q] = a21;
      j22[q] = a22;
      al[q] = w * (a22 * ux - a21 * uy);
      be[q] = w * (a11 * uy - a12 * ux);
      ga[q] = conv ? w * (a11 * a22 - a12 * a21) * (a.bx * ux + a.by * uy) : 0.f;
    }
    __syncwarp();
    // rows: r_j, rbar_j, per-cell sums
    float lsq = 0.f, lge = 0.f;
    for (int j = lane; j < T; j += 32) {
      const float* bx = tBx + j * Q;
      const float* by = tBy + j * Q;
      const float* bv = tB + j * Q;
      float g0 = 0.f, g1 = 0.f, t0 = 0.f;
      for (int q = 0; q < Q; ++q) {
        g0 = fmaf(bx[q], al[q], g0);
        g1 = fmaf(by[q], be[q], g1);
        if (conv) t0 = fmaf(bv[q], ga[q], t0);
      }
      const float g = g0 + g1;
      const float r = fmaf(e, g, t0) - a.forcing[(size_t)k * T + j];
      if (a.res) a.res[(size_t)k * T + j] = r;
      const float rbj = a.rscale * r;
      rb[j] = rbj;
      lsq = fmaf(r, r, lsq);
      lge = fmaf(rbj, g, lge);
    }
    __syncwarp();
    // columns: P, M, V and the adjoints
    for (int q = lane; q < Q; q += 32) {
      float P = 0.f, M = 0.f, V = 0.f;
      for (int j = 0; j < T; ++j) {
        const float r = rb[j];
        P = fmaf(tBx[j * Q + q], r, P);
        M = fmaf(tBy[j * Q + q], r, M);
        if (conv) V = fmaf(tB[j * Q + q], r, V);
      }
      const float w = rw[q];
      float ox = e * w * (j22[q] * P - j12[q] * M);
      float oy = e * w * (j11[q] * M - j21[q] * P);
      if (conv) {
        const float wv = w * (j11[q] * j22[q] - j12[q] * j21[q]) * V;
        ox = fmaf(a.bx, wv, ox);
        oy = fmaf(a.by, wv, oy);
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
    __syncwarp();
  }
  if (lane == 0) {
    red[2 * warp] = acc_v;
    red[2 * warp + 1] = acc_eg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0, g = 0.0;
    for (int w = 0; w < kMfWarps; ++w) {
      v += red[2 * w];
      g += red[2 * w + 1];
    }
    double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
    for (int w = 0; w < kLpWords; ++w) lp[w] = 0.0;
    lp[kLpVar] = v;
    lp[kLpEpsGrad] = g;
  }
}

// Tile variant: a CTA of 256 threads takes whole cells (cells_per_tile =
// 256 / Q) per tile, thread per point for the geometry and the adjoints,
// thread per (cell, row) for the residuals, so every global load of a tile
// is in flight at once (the warp-per-cell kernel above serialises them);
// the next tile's point data is prefetched into registers.
constexpr int kMfTileThreads = 256;

__host__ __device__ constexpr size_t mf_tile_smem_bytes(int T, int Q, int cpt) {
  return sizeof(float) * ((size_t)mf_tab_floats(T, Q) + 3 * ((Q + 3) & ~3) + (size_t)7 * cpt * Q +
                          (size_t)3 * cpt * T + 2 * (size_t)cpt) +
         sizeof(double) * 2 * (kMfTileThreads / 32) + 16;
}

__global__ void __launch_bounds__(kMfTileThreads) contract_mf_tile_kernel(const MfContractArgs a, int cpt) {
  extern __shared__ __align__(16) float mt[];
  const int T = a.T, Q = a.Q, Q4 = (Q + 3) & ~3;
  const int np_t = cpt * Q, nr_t = cpt * T;
  float* tBx = mt;
  float* tBy = tBx + T * Q;
  float* tB = tBy + T * Q;
  float* rxi = mt + mf_tab_floats(T, Q);
  float* reta = rxi + Q4;
  float* rw = reta + Q4;
  float* al = rw + Q4;        // [np_t]
  float* be = al + np_t;
  float* ga = be + np_t;
  float* j11 = ga + np_t;
  float* j12 = j11 + np_t;
  float* j21 = j12 + np_t;
  float* j22 = j21 + np_t;
  float* rb = j22 + np_t;     // [nr_t]
  float* rsq = rb + nr_t;
  float* rge = rsq + nr_t;
  float* cs = rge + nr_t;     // [2][cpt] per-cell sums
  double* red = reinterpret_cast<double*>(cs + 2 * cpt + ((2 * cpt) & 1) + 2);
  red = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(red) + 7) & ~uintptr_t(7));
  const int tid = threadIdx.x;
  for (int i = tid; i < 3 * T * Q; i += kMfTileThreads) tBx[i] = a.tabs[i];
  for (int i = tid; i < Q; i += kMfTileThreads) {
    rxi[i] = a.rule[i];
    reta[i] = a.rule[Q + i];
    rw[i] = a.rule[2 * Q + i];
  }
  const bool conv = a.bx != 0.0f || a.by != 0.0f;
  const float e = a.eps_source == 1 ? *a.e_param : a.e_fixed;
  const int n_tiles = (a.E + cpt - 1) / cpt;
  double acc_v = 0.0, acc_eg = 0.0;  // thread 0
  // this thread's point of a tile: (cell kk, quadrature point q)
  const int kk = tid / Q, q = tid - kk * Q;
  const bool pt = tid < np_t;
  auto load_pt = [&](int tile, float& ux, float& uy, int4& en) {
    ux = uy = 0.f;
    en = make_int4(0, 0, 0, 0);
    const int k = tile * cpt + kk;
    if (pt && tile < n_tiles && k < a.E) {
      ux = a.ux[(size_t)k * Q + q];
      uy = a.uy[(size_t)k * Q + q];
      en = reinterpret_cast<const int4*>(a.elems)[a.e0 + k];
    }
  };
  float nux, nuy;
  int4 nen;
  load_pt(blockIdx.x, nux, nuy, nen);
  __syncthreads();
#pragma unroll 1
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int k0 = tile * cpt, ncell = min(cpt, a.E - k0);
    const float ux = nux, uy = nuy;
    const int4 en = nen;
    const bool valid = pt && kk < ncell;
    if (valid) {
      const double2 A = reinterpret_cast<const double2*>(a.nodes)[en.x];
      const double2 B = reinterpret_cast<const double2*>(a.nodes)[en.y];
      const double2 C = reinterpret_cast<const double2*>(a.nodes)[en.z];
      const double2 D = reinterpret_cast<const double2*>(a.nodes)[en.w];
      const float xc1 = (float)(0.25 * (-A.x + B.x + C.x - D.x)), xc2 = (float)(0.25 * (-A.x - B.x + C.x + D.x));
      const float xc3 = (float)(0.25 * (A.x - B.x + C.x - D.x));
      const float yc1 = (float)(0.25 * (-A.y + B.y + C.y - D.y)), yc2 = (float)(0.25 * (-A.y - B.y + C.y + D.y));
      const float yc3 = (float)(0.25 * (A.y - B.y + C.y - D.y));
      const float xi = rxi[q], eta = reta[q], w = rw[q];
      const float a11 = fmaf(xc3, eta, xc1), a12 = fmaf(yc3, eta, yc1);
      const float a21 = fmaf(xc3, xi, xc2), a22 = fmaf(yc3, xi, yc2);
      j11[tid] = a11;
      j12[tid] = a12;
      j21[tid] = a21;
      j22[tid] = a22;
      al[tid] = w * (a22 * ux - a21 * uy);
      be[tid] = w * (a11 * uy - a12 * ux);
      ga[tid] = conv ? w * (a11 * a22 - a12 * a21) * (a.bx * ux + a.by * uy) : 0.f;
    }
    load_pt(tile + gridDim.x, nux, nuy, nen);  // next tile in flight
    __syncthreads();
    // rows: thread per (cell, row)
    for (int it = tid; it < ncell * T; it += kMfTileThreads) {
      const int c = it / T, j = it - c * T;
      const float* bx = tBx + j * Q;
      const float* by = tBy + j * Q;
      const float* bv = tB + j * Q;
      const float* pa = al + c * Q;
      const float* pbv = be + c * Q;
      const float* pg = ga + c * Q;
      float g0 = 0.f, g1 = 0.f, t0 = 0.f, g2 = 0.f, g3 = 0.f;
      int qq = 0;
      for (; qq + 1 < Q; qq += 2) {
        g0 = fmaf(bx[qq], pa[qq], g0);
        g1 = fmaf(by[qq], pbv[qq], g1);
        g2 = fmaf(bx[qq + 1], pa[qq + 1], g2);
        g3 = fmaf(by[qq + 1], pbv[qq + 1], g3);
        if (conv) t0 = fmaf(bv[qq + 1], pg[qq + 1], fmaf(bv[qq], pg[qq], t0));
      }
      for (; qq < Q; ++qq) {
        g0 = fmaf(bx[qq], pa[qq], g0);
        g1 = fmaf(by[qq], pbv[qq], g1);
        if (conv) t0 = fmaf(bv[qq], pg[qq], t0);
      }
      const float g = (g0 + g2) + (g1 + g3);
      const float r = fmaf(e, g, t0) - a.forcing[(size_t)(k0 + c) * T + j];
      if (a.res) a.res[(size_t)(k0 + c) * T + j] = r;
      const float rbj = a.rscale * r;
      rb[it] = rbj;
      rsq[it] = r * r;
      rge[it] = rbj * g;
    }
    __syncthreads();
    // columns: thread per point; then the per-cell sums in row order
    if (valid) {
      float P = 0.f, M = 0.f, V = 0.f;
      const float* r = rb + kk * T;
      for (int j = 0; j < T; ++j) {
        P = fmaf(tBx[j * Q + q], r[j], P);
        M = fmaf(tBy[j * Q + q], r[j], M);
        if (conv) V = fmaf(tB[j * Q + q], r[j], V);
      }
      const float w = rw[q];
      float ox = e * w * (j22[tid] * P - j12[tid] * M);
      float oy = e * w * (j11[tid] * M - j21[tid] * P);
      if (conv) {
        const float wv = w * (j11[tid] * j22[tid] - j12[tid] * j21[tid]) * V;
        ox = fmaf(a.bx, wv, ox);
        oy = fmaf(a.by, wv, oy);
      }
      const size_t pidx = (size_t)(k0 + kk) * Q + q;
      a.uxb[pidx] = ox;
      a.uyb[pidx] = oy;
    }
    if (tid < ncell) {
      const int c = tid;
      float s = 0.f, g = 0.f;
      for (int j = 0; j < T; ++j) {
        s += rsq[c * T + j];
        g += rge[c * T + j];
      }
      cs[c] = s;
      cs[cpt + c] = g;
    }
    __syncthreads();
    if (tid == 0)
      for (int c = 0; c < ncell; ++c) {
        acc_v += (double)(cs[c] * a.inv_nt);
        acc_eg += (double)cs[cpt + c];
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
