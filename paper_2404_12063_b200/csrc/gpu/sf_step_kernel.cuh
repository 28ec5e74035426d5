// Strong-form collocation step: the reference's PINN
// baseline, LossForm::strong (trainer.hpp:178-188, 246-248).
//
// Per point the network runs at ORDER 2 (network.hpp:204-282): five streams
// V (value), Tx, Ty (first derivatives) and T2x, T2y (second derivatives)
// through every layer; the loss is the pointwise residual
//   P = -eps (u_xx + u_yy) + b . grad u - f,   loss = mean P^2
// (losses.hpp:422-467) plus the boundary / sensor penalties
// (losses.hpp:389-415), and the reverse sweep is the order-2 one
// (network.hpp:287-372).  There is no contraction: the work is five GEMM
// streams per layer forward, five back, and the weight-gradient GEMM.
//
// B200 mapping.  One WARP owns a tile of 16 points and runs it end to end
// with no CTA barrier:
//   - every layer product is mma.sync m16n8k8 TF32 with a three-pass split
//     (a = a_hi + a_lo, d += a_lo b_hi + a_hi b_lo + a_hi b_hi: fp32-faithful,
//     fp32 exponent range, so unlike an fp16 split no scaling is needed);
//   - a layer's output accumulator fragment (C layout) is the next layer's A
//     fragment after a fixed permutation of the K index, so activations move
//     layer to layer in registers (the weights are stored to match);
//   - the per-layer state the reverse needs (z, TA, T2A: five [16 x 32]
//     tiles per hidden layer) lives in the warp's shared-memory slot, row
//     stride 40 floats so both the lane-private C-layout accesses and the
//     transposed reads of the weight-gradient GEMM are conflict-free;
//   - weight-gradient accumulators stay in registers for the whole kernel
//     (each (i,k) entry owned by one lane), per-unit sums are reduce-scattered
//     across the warp so each lane owns one unit; the CTA sums its warps in a
//     fixed order at the end (deterministic, no atomics).
// Hidden widths <= 32 (zero-padded exactly), one output channel, tanh or
// sigmoid, fixed or scalar eps (a spatial eps is rejected, losses.hpp:440).
#pragma once

#include "step_kernel.cuh"

// rolled GEMM k-loops keep the kernel's instruction stream small enough for
// the instruction cache (fully unrolled: 13k instructions, 44% of the stall
// samples were no_instruction)
#ifndef VPG_SF_ROLL
#define VPG_SF_ROLL 1
#endif
#define VPG_SF_STR_(x) #x
#define VPG_SF_PRAGMA_UNROLL(n) _Pragma(VPG_SF_STR_(unroll n))
#ifndef VPG_SF_LO_RN
#define VPG_SF_LO_RN 0
#endif
#ifndef VPG_SF_HI_TRUNC
#define VPG_SF_HI_TRUNC 0
#endif
#ifndef VPG_SF_CVT_RNA
#define VPG_SF_CVT_RNA 0
#endif

namespace vpg {
namespace sf {

constexpr int NU = 32;            // padded hidden width
constexpr int RS = 40;            // row stride of a [16 point][32 unit] tile
constexpr int TILE_F = 16 * RS;   // floats per tile
constexpr int WS = 40;            // weight row stride
constexpr int kMaxWarps = 8;

// per-warp slot: hidden 1..D-1 keep five tiles each (hidden 0 is recomputed;
// D == 1 keeps one tile for the final gradient reduction)
__host__ __device__ constexpr int warp_floats(int D) { return D == 1 ? TILE_F : (D - 1) * 5 * TILE_F; }
// CTA-wide: W_l and W_l^T (l = 1..D-1), W0 as float2 rows, biases, w_out
__host__ __device__ constexpr int fixed_floats(int D) {
  return (D - 1) * 2 * NU * WS + 2 * NU + D * NU + NU + 4;
}
__host__ __device__ constexpr size_t smem_bytes(int D, int warps) {
  return sizeof(float) * ((size_t)fixed_floats(D) + (size_t)warps * warp_floats(D)) + 64;
}

// round to nearest (ties away) onto the tf32 grid: two integer ops instead of
// cvt.rna.tf32.f32, which sm_100 expands to ~5 instructions with NaN / Inf
// handling (the operands here are finite; an overflowing |x| near FLT_MAX
// would round to Inf either way)
__device__ __forceinline__ uint32_t to_tf32(float x) {
#if VPG_SF_CVT_RNA
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
#else
  return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
#endif
}
// x = hi + lo, both rounded to tf32
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
#if VPG_SF_HI_TRUNC
  hi = __float_as_uint(x) & 0xffffe000u;
#else
  hi = to_tf32(x);
#endif
#if VPG_SF_LO_RN
  lo = to_tf32(x - __uint_as_float(hi));
#else
  // the MMA reads only the top 19 bits of lo (truncation): |lo| <= 2^-11 |x|,
  // so the dropped bits are below 2^-21 |x|
  lo = __float_as_uint(x - __uint_as_float(hi));
#endif
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// d += a b in three TF32 passes (a_lo b_hi, a_hi b_lo, a_hi b_hi; the lo x lo
// term is below fp32 resolution): the kernels issue the passes interleaved
// over independent accumulators (see the GEMM loops)
__device__ __forceinline__ void split4(const float (&v)[4], uint32_t (&h)[4], uint32_t (&l)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) split(v[j], h[j], l[j]);
}
__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void sts2(float* p, float a, float b) {
  *reinterpret_cast<float2*>(p) = make_float2(a, b);
}

// activation derivatives from the OUTPUT z (ActDerivs::fill, network.hpp:171-192)
template <int ACT>
__device__ __forceinline__ void derivs(float z, float& s1, float& s2, float& s3) {
  if constexpr (ACT == kActTanh) {
    s1 = 1.0f - z * z;
    s2 = -2.0f * z * s1;
    s3 = s1 * (4.0f * (z * z) - 2.0f * s1);
  } else {
    s1 = z * (1.0f - z);
    s2 = s1 * (1.0f - 2.0f * z);
    s3 = s1 * (1.0f - 6.0f * z + 6.0f * (z * z));
  }
}
template <int ACT>
__device__ __forceinline__ void derivs12(float z, float& s1, float& s2) {
  if constexpr (ACT == kActTanh) {
    s1 = 1.0f - z * z;
    s2 = -2.0f * z * s1;
  } else {
    s1 = z * (1.0f - z);
    s2 = s1 * (1.0f - 2.0f * z);
  }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// warp sums of the per-lane values v0 (unit 8 nt + 2 t) and v1 (unit
// 8 nt + 2 t + 1) over the eight lanes sharing t, added to the owner lane's
// accumulator (owner of unit 8 (g >> 1) + 2 t + (g & 1))
__device__ __forceinline__ void owner_add(float v0, float v1, int nt, int g, float& own) {
#pragma unroll
  for (int o = 4; o <= 16; o <<= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  if ((g >> 1) == nt) own += (g & 1) ? v1 : v0;
}

// slot of hidden layer l >= 1 (hidden 0 is not stored: z0 is recomputed
// from the point, TA0 = W0 columns, T2A0 = 0)
__device__ __forceinline__ float* state_slot(float* slot, int l) { return slot + (l - 1) * 5 * TILE_F; }

// state (z, TAx, TAy, T2Ax, T2Ay) of column tile nt at the lane's four C
// positions c = 2 r + e (row g + 8 r, unit 8 nt + 2 t + e); first: hidden 0,
// recomputed from the lane's points (px, py) and W0, b0
template <int ACT>
__device__ __forceinline__ void load_state_c(const float* S, const float2* sW0, const float* sB0, int nt, int g,
                                             int t, float (&st)[5][4], bool first, const float (&px)[2],
                                             const float (&py)[2]) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (first) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int u = 8 * nt + 2 * t + e;
        const float2 w = sW0[u];
        st[0][2 * r + e] = Act<ACT>::value(fmaf(w.y, py[r], w.x * px[r]) + sB0[u]);
        st[1][2 * r + e] = w.x;
        st[2][2 * r + e] = w.y;
        st[3][2 * r + e] = 0.f;
        st[4][2 * r + e] = 0.f;
      }
    } else {
      const int o = (g + 8 * r) * RS + 8 * nt + 2 * t;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const float2 v = lds2(S + s * TILE_F + o);
        st[s][2 * r] = v.x;
        st[s][2 * r + 1] = v.y;
      }
    }
  }
}

// layer outputs (network.hpp:262-276): X = z, TX = s1 TA, T2X = s2 TA^2 + s1 T2A
template <int ACT>
__device__ __forceinline__ void x_streams(float z, float tax, float tay, float t2x, float t2y, float& xv,
                                          float& xtx, float& xty, float& xt2x, float& xt2y) {
  float s1, s2;
  derivs12<ACT>(z, s1, s2);
  xv = z;
  xtx = s1 * tax;
  xty = s1 * tay;
  xt2x = s2 * (tax * tax) + s1 * t2x;
  xt2y = s2 * (tay * tay) + s1 * t2y;
}

// through the activation (network.hpp:350-370): adjoints (zb, tzx, tzy,
// t2zx, t2zy) of the layer outputs -> (Abar, TAxbar, TAybar, T2Axbar, T2Aybar)
template <int ACT>
__device__ __forceinline__ void act_reverse(float z, float tax, float tay, float t2x, float t2y, float zb, float tzx,
                                            float tzy, float t2zx, float t2zy, float (&o)[5]) {
  float s1, s2, s3;
  derivs<ACT>(z, s1, s2, s3);
  float av = s1 * zb;
  av += s2 * (tax * tzx) + s2 * (tay * tzy);
  av += s3 * ((tax * tax) * t2zx) + s2 * (t2x * t2zx) + s3 * ((tay * tay) * t2zy) + s2 * (t2y * t2zy);
  o[0] = av;
  o[1] = s1 * tzx + 2.0f * (s2 * (tax * t2zx));
  o[2] = s1 * tzy + 2.0f * (s2 * (tay * t2zy));
  o[3] = s1 * t2zx;
  o[4] = s1 * t2zy;
}

}  // namespace sf

// MODE kModeFused: loss + parameter gradient per CTA part; kModeForward:
// order-2 evaluate() at a.fwd_pts (u, u_x, u_y, u_xx, u_yy).
template <int D, int ACT, int MODE>
__global__ void __launch_bounds__(32 * sf::kMaxWarps, 1) sf_step_kernel(const StepArgs a) {
  using namespace sf;
  static_assert(D >= 1 && D <= 4, "hidden layers");
  // the trigger after the wait: the epoch tail launched early reads the
  // trainer state before its own wait (reduce_adam_kernel), which is only
  // sound once this kernel's predecessor -- the previous tail -- completed
  pdl_wait();
  pdl_trigger();
  if constexpr (MODE == kModeFused) {
    if (a.stop_flag && *a.stop_flag) return;
  }
  extern __shared__ __align__(16) float smem[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const NetDesc& net = a.net;
  const float* P = a.params;

  float* sW = smem;                                      // [D-1][NU][WS]  W_l[i][k]
  float* sWT = sW + (D - 1) * NU * WS;                   // [D-1][NU][WS]  W_l[k][i]
  float2* sW0 = reinterpret_cast<float2*>(sWT + (D - 1) * NU * WS);  // [NU] (W0[i][0], W0[i][1])
  float* sB = reinterpret_cast<float*>(sW0 + NU);        // [D][NU] hidden biases
  float* sWo = sB + D * NU;                              // [NU] output row
  float* sBo = sWo + NU;                                 // [1] output bias
  float* slot = smem + fixed_floats(D) + warp * warp_floats(D);

  // ---- weights into shared memory (zero padded to 32 units) ----
  for (int idx = threadIdx.x; idx < (D - 1) * NU * NU; idx += blockDim.x) {
    const int l = 1 + idx / (NU * NU), r = idx % (NU * NU), i = r / NU, k = r % NU;
    const int fo = net.out_w[l], fi = net.in_w[l];
    const float w = (i < fo && k < fi) ? P[net.w_off[l] + i * fi + k] : 0.0f;
    sW[(l - 1) * NU * WS + i * WS + k] = w;
    sWT[(l - 1) * NU * WS + k * WS + i] = w;
  }
  for (int i = threadIdx.x; i < NU; i += blockDim.x) {
    const bool in0 = i < net.out_w[0];
    sW0[i] = in0 ? make_float2(P[net.w_off[0] + 2 * i], P[net.w_off[0] + 2 * i + 1]) : make_float2(0.f, 0.f);
#pragma unroll
    for (int l = 0; l < D; ++l) sB[l * NU + i] = i < net.out_w[l] ? P[net.b_off[l] + i] : 0.0f;
    sWo[i] = i < net.in_w[D] ? P[net.w_off[D] + i] : 0.0f;
  }
  if (threadIdx.x == 0) sBo[0] = P[net.b_off[D]];
  const float e_val = a.eps_source == 1 ? P[net.scal_off + a.eps_scalar_index] : a.eps;
  __syncthreads();

  constexpr bool fwd = MODE == kModeForward;
  const float2* pts = fwd ? a.fwd_pts : a.pts;
  const int n_pts = fwd ? a.n_fwd : a.n_int + a.n_bnd + a.n_sen;
  const int n_tiles = (n_pts + 15) >> 4;
  const int tw = gridDim.x * nw;

  // ---- persistent gradient accumulators ----
  float gacc[D > 1 ? D - 1 : 1][2][4][4];  // W_l, l = 1..D-1: [mt][nt][c]
#pragma unroll
  for (int l = 0; l < (D > 1 ? D - 1 : 1); ++l)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int c = 0; c < 4; ++c) gacc[l][m][n][c] = 0.0f;
  // one owned unit per lane: u_own = 8 (g >> 1) + 2 t + (g & 1)
  float gb_own[D];
#pragma unroll
  for (int l = 0; l < D; ++l) gb_own[l] = 0.0f;
  // the output bias gradient sums the boundary / sensor adjoints, which
  // cancel (sum of O(tau / N) terms -> a small total): double, like the loss
  float gw0x_own = 0.f, gw0y_own = 0.f, gwo_own = 0.f;
  double gbo = 0.0;
  double acc_v = 0.0, acc_b = 0.0, acc_s = 0.0, acc_eg = 0.0;
  int bad = 0;

  const float bx = a.bx, by = a.by;
  const bool conv = bx != 0.0f || by != 0.0f;

#pragma unroll 1
  for (int tile = blockIdx.x * nw + warp; tile < n_tiles; tile += tw) {
    __syncwarp();  // the previous tile's cross-lane slot reads are complete
    const int p0 = tile << 4;
    int pr[2];
    bool valid[2];
    float px[2], py[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      pr[r] = p0 + g + 8 * r;
      valid[r] = pr[r] < n_pts;
      const float2 q = valid[r] ? pts[pr[r]] : make_float2(0.f, 0.f);
      px[r] = q.x;
      py[r] = q.y;
    }

    // ================= forward, order 2 (network.hpp:204-282) =================
    // C-layout position (nt, c): row g + 8 (c >> 1), unit 8 nt + 2 t + (c & 1).
    // Every hidden layer's state (z, TA, T2A) goes to its slot; the loops
    // over the 4 column tiles are rolled (instruction-cache footprint).
    // hidden 0 is recomputed where needed (z0 = act(W0 (x, y) + b0))
    if constexpr (D >= 2) {
#pragma unroll
      for (int l = 1; l < D; ++l) {
        float acc[5][4][4];
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[s][n][c] = 0.0f;
        const float* Wl = sW + (l - 1) * NU * WS;
        const float* Sprev = state_slot(slot, l - 1);
VPG_SF_PRAGMA_UNROLL(VPG_SF_ROLL)
        for (int kt = 0; kt < 4; ++kt) {
          // A fragments of the five input streams: positions (g, k0), (g+8, k0),
          // (g, k0+1), (g+8, k0+1) with k0 = 8 kt + 2 t (the permuted K order)
          float st[5][4];
          load_state_c<ACT>(Sprev, sW0, sB, kt, g, t, st, l == 1, px, py);
          float xs[5][4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = 2 * (q & 1) + (q >> 1);  // fragment slot q <- C position c
            x_streams<ACT>(st[0][c], st[1][c], st[2][c], st[3][c], st[4][c], xs[0][q], xs[1][q], xs[2][q],
                           xs[3][q], xs[4][q]);
          }
          uint32_t ah[5][4], al[5][4];
#pragma unroll
          for (int s = 0; s < 5; ++s) split4(xs[s], ah[s], al[s]);
          uint32_t bh[4][2], bl[4][2];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            const float2 w = lds2(Wl + (8 * nt + g) * WS + 8 * kt + 2 * t);
            split(w.x, bh[nt][0], bl[nt][0]);
            split(w.y, bh[nt][1], bl[nt][1]);
          }
          // the three split passes interleaved over the 20 independent
          // accumulators (no back-to-back dependent HMMAs)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int s = 0; s < 5; ++s) mma_tf32(acc[s][nt], al[s], bh[nt][0], bh[nt][1]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int s = 0; s < 5; ++s) mma_tf32(acc[s][nt], ah[s], bl[nt][0], bl[nt][1]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int s = 0; s < 5; ++s) mma_tf32(acc[s][nt], ah[s], bh[nt][0], bh[nt][1]);
        }
        // epilogue: z = act(A + b); state of hidden l into its slot
        float* Sl = state_slot(slot, l);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int u = 8 * nt + 2 * t + (c & 1);
            acc[0][nt][c] = Act<ACT>::value(acc[0][nt][c] + sB[l * NU + u]);
          }
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            sts2(Sl + s * TILE_F + g * RS + 8 * nt + 2 * t, acc[s][nt][0], acc[s][nt][1]);
            sts2(Sl + s * TILE_F + (g + 8) * RS + 8 * nt + 2 * t, acc[s][nt][2], acc[s][nt][3]);
          }
      }
    }

    // ---- output layer (linear): u_s = w_out . X_s (+ b_out) ----
    float* SL = state_slot(slot, D - 1);
    float part[5][2];
#pragma unroll
    for (int s = 0; s < 5; ++s) part[s][0] = part[s][1] = 0.0f;
#pragma unroll 1
    for (int nt = 0; nt < 4; ++nt) {
      float st[5][4];
      load_state_c<ACT>(SL, sW0, sB, nt, g, t, st, D == 1, px, py);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int r = c >> 1;
        const float wo = sWo[8 * nt + 2 * t + (c & 1)];
        float x[5];
        x_streams<ACT>(st[0][c], st[1][c], st[2][c], st[3][c], st[4][c], x[0], x[1], x[2], x[3], x[4]);
#pragma unroll
        for (int s = 0; s < 5; ++s) part[s][r] = fmaf(wo, x[s], part[s][r]);
      }
    }
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        part[s][r] += __shfl_xor_sync(0xffffffffu, part[s][r], 1);
        part[s][r] += __shfl_xor_sync(0xffffffffu, part[s][r], 2);
      }
    const float bo = sBo[0];
#pragma unroll
    for (int r = 0; r < 2; ++r) part[0][r] += bo;

    if constexpr (fwd) {
      if (t == 0) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
          if (valid[r]) {
            const int p = pr[r];
            if (a.out_u) a.out_u[p] = part[0][r];
            if (a.out_ux) a.out_ux[p] = part[1][r];
            if (a.out_uy) a.out_uy[p] = part[2][r];
            if (a.out_uxx) a.out_uxx[p] = part[3][r];
            if (a.out_uyy) a.out_uyy[p] = part[4][r];
          }
      }
      continue;
    }

    // ============ objective + output adjoints (trainer.hpp:246-266) ============
    float yb[5][2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int s = 0; s < 5; ++s) yb[s][r] = 0.0f;
      if (!valid[r]) continue;
      const int p = pr[r];
      const float u = part[0][r], ux = part[1][r], uy = part[2][r], uxx = part[3][r], uyy = part[4][r];
      if (!(isfinite(u) && isfinite(ux) && isfinite(uy) && isfinite(uxx) && isfinite(uyy))) bad = 1;
      if (p < a.n_int) {
        // strong_residual_loss, losses.hpp:446-466
        const float lap = uxx + uyy;
        const float Pv = __fsub_rn(__fadd_rn(__fadd_rn(__fmul_rn(-e_val, lap), __fmul_rn(bx, ux)), __fmul_rn(by, uy)),
                                   a.sforce[p]);
        if (t == 0) acc_v += (double)__fmul_rn(__fmul_rn(Pv, Pv), a.inv_ni);
        const float pbar = __fmul_rn(a.rscale_s, Pv);
        yb[3][r] = yb[4][r] = __fmul_rn(-e_val, pbar);
        if (conv) {
          yb[1][r] = __fmul_rn(bx, pbar);
          yb[2][r] = __fmul_rn(by, pbar);
        }
        if (a.eps_source == 1 && t == 0) acc_eg += (double)__fmul_rn(-lap, pbar);
      } else if (p < a.n_int + a.n_bnd) {
        const float d = u - a.bval[p - a.n_int];
        if (t == 0) acc_b += (double)(d * d);
        yb[0][r] = a.bscale * d;
      } else {
        const float d = u - a.sval[p - a.n_int - a.n_bnd];
        if (t == 0) acc_s += (double)(d * d);
        yb[0][r] = a.sscale * d;
      }
    }
    if (t == 0) gbo += (double)yb[0][0] + (double)yb[0][1];

    // ================= reverse, order 2 (network.hpp:287-372) =================
    // output layer: w_out gradient, Zbar_{D-1} = w_out (x) Ybar, and Abar of
    // the last hidden layer (in place of its state)
#pragma unroll 1
    for (int nt = 0; nt < 4; ++nt) {
      float st[5][4];
      load_state_c<ACT>(SL, sW0, sB, nt, g, t, st, D == 1, px, py);
      float gw[2] = {0.f, 0.f}, gb[2] = {0.f, 0.f}, gx[2] = {0.f, 0.f}, gy[2] = {0.f, 0.f};
      float ab[5][4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int r = c >> 1, e = c & 1;
        const float wo = sWo[8 * nt + 2 * t + e];
        float x[5];
        x_streams<ACT>(st[0][c], st[1][c], st[2][c], st[3][c], st[4][c], x[0], x[1], x[2], x[3], x[4]);
        // w_out gradient (Wbar += Abar X^T + TAxbar TXx^T + ..., 326-334)
        gw[e] += yb[0][r] * x[0] + yb[1][r] * x[1] + yb[2][r] * x[2] + yb[3][r] * x[3] + yb[4][r] * x[4];
        // Xbar = W^T Abar (340-347), then through the activation (350-370)
        float o[5];
        act_reverse<ACT>(st[0][c], st[1][c], st[2][c], st[3][c], st[4][c], wo * yb[0][r], wo * yb[1][r],
                         wo * yb[2][r], wo * yb[3][r], wo * yb[4][r], o);
#pragma unroll
        for (int s = 0; s < 5; ++s) ab[s][c] = o[s];
        gb[e] += o[0];
        if constexpr (D == 1) {
          // layer-0 gradient: X0 = (x, y), TX0 = unit vectors, T2X0 = 0
          gx[e] += o[0] * px[r] + o[1];
          gy[e] += o[0] * py[r] + o[2];
        }
      }
      owner_add(gw[0], gw[1], nt, g, gwo_own);
      owner_add(gb[0], gb[1], nt, g, gb_own[D - 1]);
      if constexpr (D == 1) {
        owner_add(gx[0], gx[1], nt, g, gw0x_own);
        owner_add(gy[0], gy[1], nt, g, gw0y_own);
      } else {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          sts2(SL + s * TILE_F + g * RS + 8 * nt + 2 * t, ab[s][0], ab[s][1]);
          sts2(SL + s * TILE_F + (g + 8) * RS + 8 * nt + 2 * t, ab[s][2], ab[s][3]);
        }
      }
    }

    if constexpr (D >= 2) {
#pragma unroll
      for (int h = D - 1; h >= 1; --h) {
        // slot h holds Abar of hidden h; hidden h-1 holds its state
        float* Ah = state_slot(slot, h);
        float* Sp = state_slot(slot, h - 1);
        __syncwarp();
        // ---- weight gradient of layer h: sum_s Abar_s^T X_s (M = i, N = k, K = points)
VPG_SF_PRAGMA_UNROLL(VPG_SF_ROLL)
        for (int kt = 0; kt < 2; ++kt) {
          const int pa = 8 * kt + t, pb = pa + 4;
          // z, s1, s2 of hidden h-1 at (points pa / pb, units 8 nt + g), shared
          // by the five streams; hidden 0 is recomputed from the points
          float zt[4][2], s1t[4][2], s2t[4][2];
          {
            float2 q[2];
            if (h == 1) {
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int pp = p0 + (i ? pb : pa);
                q[i] = pp < n_pts ? pts[pp] : make_float2(0.f, 0.f);
              }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const int k = 8 * nt + g;
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                if (h == 1) {
                  const float2 w = sW0[k];
                  zt[nt][i] = Act<ACT>::value(fmaf(w.y, q[i].y, w.x * q[i].x) + sB[k]);
                } else {
                  zt[nt][i] = Sp[(i ? pb : pa) * RS + k];
                }
                derivs12<ACT>(zt[nt][i], s1t[nt][i], s2t[nt][i]);
              }
            }
          }
VPG_SF_PRAGMA_UNROLL(VPG_SF_ROLL)
          for (int s = 0; s < 5; ++s) {
            const float* As = Ah + s * TILE_F;
            uint32_t ah[2][4], al[2][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              const float v[4] = {As[pa * RS + 16 * mt + g], As[pa * RS + 16 * mt + g + 8], As[pb * RS + 16 * mt + g],
                                  As[pb * RS + 16 * mt + g + 8]};
              split4(v, ah[mt], al[mt]);
            }
            uint32_t bh[4][2], bl[4][2];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const int k = 8 * nt + g;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int o = (q ? pb : pa) * RS + k;
                float xb;
                if (s == 0) {
                  xb = zt[nt][q];
                } else {
                  const float s1 = s1t[nt][q], s2 = s2t[nt][q];
                  float ta, t2a = 0.f;
                  if (h == 1) {
                    ta = (s == 1 || s == 3) ? sW0[k].x : sW0[k].y;
                  } else {
                    ta = Sp[((s == 1 || s == 3) ? 1 : 2) * TILE_F + o];
                    if (s >= 3) t2a = Sp[s * TILE_F + o];
                  }
                  xb = s <= 2 ? s1 * ta : s2 * (ta * ta) + s1 * t2a;
                }
                split(xb, bh[nt][q], bl[nt][q]);
              }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) mma_tf32(gacc[h - 1][mt][nt], al[mt], bh[nt][0], bh[nt][1]);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) mma_tf32(gacc[h - 1][mt][nt], ah[mt], bl[nt][0], bl[nt][1]);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) mma_tf32(gacc[h - 1][mt][nt], ah[mt], bh[nt][0], bh[nt][1]);
          }
        }
        // ---- propagation: Zbar_s = Abar_s W_h (M = points, N = k, K = i permuted)
        float zacc[5][4][4];
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
          for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int c = 0; c < 4; ++c) zacc[s][n][c] = 0.0f;
        const float* WT = sWT + (h - 1) * NU * WS;
VPG_SF_PRAGMA_UNROLL(VPG_SF_ROLL)
        for (int kt = 0; kt < 4; ++kt) {
          uint32_t bh[4][2], bl[4][2];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            const float2 w = lds2(WT + (8 * nt + g) * WS + 8 * kt + 2 * t);
            split(w.x, bh[nt][0], bl[nt][0]);
            split(w.y, bh[nt][1], bl[nt][1]);
          }
          uint32_t ah[5][4], al[5][4];
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            const float* As = Ah + s * TILE_F;
            const float2 r0 = lds2(As + g * RS + 8 * kt + 2 * t);
            const float2 r1 = lds2(As + (g + 8) * RS + 8 * kt + 2 * t);
            const float v[4] = {r0.x, r1.x, r0.y, r1.y};
            split4(v, ah[s], al[s]);
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int s = 0; s < 5; ++s) mma_tf32(zacc[s][nt], al[s], bh[nt][0], bh[nt][1]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int s = 0; s < 5; ++s) mma_tf32(zacc[s][nt], ah[s], bl[nt][0], bl[nt][1]);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int s = 0; s < 5; ++s) mma_tf32(zacc[s][nt], ah[s], bh[nt][0], bh[nt][1]);
        }
        __syncwarp();  // every lane's reads of slot h and of hidden h-1's state are done
        // Zbar of hidden h-1 parks in slot h (its Abar is consumed) so the
        // activation pass below can run as a rolled loop
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            sts2(Ah + s * TILE_F + g * RS + 8 * nt + 2 * t, zacc[s][nt][0], zacc[s][nt][1]);
            sts2(Ah + s * TILE_F + (g + 8) * RS + 8 * nt + 2 * t, zacc[s][nt][2], zacc[s][nt][3]);
          }
        // ---- through the activation of hidden h-1 ----
#pragma unroll 1
        for (int nt = 0; nt < 4; ++nt) {
          float st[5][4], zb[5][4];
          load_state_c<ACT>(Sp, sW0, sB, nt, g, t, st, h == 1, px, py);
          load_state_c<ACT>(Ah, sW0, sB, nt, g, t, zb, false, px, py);
          float gb[2] = {0.f, 0.f}, gx[2] = {0.f, 0.f}, gy[2] = {0.f, 0.f};
          float out[5][4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float o[5];
            act_reverse<ACT>(st[0][c], st[1][c], st[2][c], st[3][c], st[4][c], zb[0][c], zb[1][c], zb[2][c],
                             zb[3][c], zb[4][c], o);
#pragma unroll
            for (int s = 0; s < 5; ++s) out[s][c] = o[s];
            const int e = c & 1, r = c >> 1;
            gb[e] += o[0];
            if (h == 1) {
              gx[e] += o[0] * px[r] + o[1];
              gy[e] += o[0] * py[r] + o[2];
            }
          }
          owner_add(gb[0], gb[1], nt, g, gb_own[h - 1]);
          if (h == 1) {
            owner_add(gx[0], gx[1], nt, g, gw0x_own);
            owner_add(gy[0], gy[1], nt, g, gw0y_own);
          } else {
#pragma unroll
            for (int s = 0; s < 5; ++s) {
              sts2(Sp + s * TILE_F + g * RS + 8 * nt + 2 * t, out[s][0], out[s][1]);
              sts2(Sp + s * TILE_F + (g + 8) * RS + 8 * nt + 2 * t, out[s][2], out[s][3]);
            }
          }
        }
      }
    }
  }

  if constexpr (MODE == kModeFused) {
    // ---- per-warp gradient vector in its slot, then a fixed-order CTA sum ----
    __syncthreads();  // all warps done with their slots
    float* gv = slot;
    for (int i = lane; i < net.n_params; i += 32) gv[i] = 0.0f;
    __syncwarp();
    const int u_own = 8 * (g >> 1) + 2 * t + (g & 1);
    if (u_own < net.out_w[0]) {
      gv[net.w_off[0] + 2 * u_own] = gw0x_own;
      gv[net.w_off[0] + 2 * u_own + 1] = gw0y_own;
    }
#pragma unroll
    for (int l = 0; l < D; ++l)
      if (u_own < net.out_w[l]) gv[net.b_off[l] + u_own] = gb_own[l];
    if (u_own < net.in_w[D]) gv[net.w_off[D] + u_own] = gwo_own;
    const double gbo_w = sf::warp_sum_d(gbo);
    if (lane == 0) gv[net.b_off[D]] = (float)gbo_w;
    if constexpr (D >= 2) {
#pragma unroll
      for (int l = 1; l < D; ++l) {
        const int fo = net.out_w[l], fi = net.in_w[l];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int i = 16 * mt + g + 8 * (c >> 1), k = 8 * nt + 2 * t + (c & 1);
              if (i < fo && k < fi) gv[net.w_off[l] + i * fi + k] = gacc[l - 1][mt][nt][c];
            }
      }
    }
    const double wv = sf::warp_sum_d(acc_v), wb = sf::warp_sum_d(acc_b), ws = sf::warp_sum_d(acc_s);
    const double we = sf::warp_sum_d(acc_eg);
    const int wbad = __any_sync(0xffffffffu, bad);
    __syncthreads();
    const int wf = warp_floats(D);
    float* base = smem + fixed_floats(D);
    for (int i = threadIdx.x; i < net.n_params; i += blockDim.x) {
      float s = base[i];
      for (int w = 1; w < nw; ++w) s += base[w * wf + i];
      a.grad_part[(size_t)i * a.part_stride + blockIdx.x] = s;
    }
    __syncthreads();
    double* red = reinterpret_cast<double*>(smem);  // the weights are no longer needed
    if (lane == 0) {
      red[warp * 5 + 0] = wv;
      red[warp * 5 + 1] = wb;
      red[warp * 5 + 2] = ws;
      red[warp * 5 + 3] = we;
      red[warp * 5 + 4] = wbad ? 1.0 : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double lv = 0, lb = 0, ls = 0, le = 0, lbad = 0;
      for (int w = 0; w < nw; ++w) {
        lv += red[w * 5 + 0];
        lb += red[w * 5 + 1];
        ls += red[w * 5 + 2];
        le += red[w * 5 + 3];
        lbad += red[w * 5 + 4];
      }
      double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
      lp[kLpVar] = lv;
      lp[kLpBnd] = lb;
      lp[kLpSen] = ls;
      lp[kLpEpsGrad] = le;
      lp[kLpBad] = lbad != 0.0 ? 1.0 : 0.0;
    }
  }
}

}  // namespace vpg
