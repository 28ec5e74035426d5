// The FastVPINNs training-step kernels for sm_100a.
//
// One CTA (128 threads, one quadrature/penalty point per thread) owns a
// TILE of whole cells.  Per tile it runs, without leaving the SM:
//   1. forward with x/y tangents through the MLP (network.hpp:204-282),
//      weights in shared memory, activations in registers, per-point layer
//      state in shared memory (point-major rows, 128-bit conflict-free);
//   2. the Algorithm-3 contraction of the tile's premultiplier slabs
//      (losses.hpp:91-168), slabs streamed HBM->SMEM by cp.async.bulk (1-D
//      TMA) into a two-stage mbarrier ring issued before the forward so the
//      copy overlaps it; residuals, loss and adjoints fused per cell;
//      penalty tiles (boundary / sensors, losses.hpp:406-415) instead;
//   3. the reverse sweep (network.hpp:287-372) with parameter-gradient
//      outer products computed as per-warp 4x8 register-tiled products over
//      the warp's 32 points, combined across warps in a fixed order into
//      per-thread gradient registers (deterministic, no atomics).
// The per-CTA gradient and loss parts are reduced across CTAs by
// reduce_kernel (fp64, fixed order) and applied by adam_kernel.
//
// Every loop whose body is large is rolled and every fully unrolled region
// is short: the kernel is FFMA-bound only if its instruction stream stays in
// the instruction cache (the first profile showed no_instruction stalls).
//
// The same template also provides the split-path kernels (forward only,
// reverse from adjoints in global memory) used when a cell has more
// quadrature points than a CTA (Q > 128, e.g. 40x40 rules).
#pragma once

#include "device_utils.cuh"

namespace vpg {

constexpr int kMaxLayers = 8;

struct NetDesc {
  int n_layers;  // weight layers = hidden layers + 1
  int in_w[kMaxLayers], out_w[kMaxLayers];
  int w_off[kMaxLayers], b_off[kMaxLayers];
  int n_params;  // including trainable scalars
  int scal_off;
  int sigmoid;
};

enum : int { kModeForward = 0, kModeFused = 1, kModeReverse = 2 };

// per-CTA loss record (doubles)
enum : int { kLpVar = 0, kLpBnd = 1, kLpSen = 2, kLpEpsGrad = 3, kLpBad = 4, kLpWords = 8 };

// exchange rows (kThreads floats each, feature-major)
enum : int { kExX = 0, kExY, kExU, kExUx, kExUy, kExE, kExY1, kExSx, kExSy, kExCv, kExRows };

struct StepArgs {
  // premultipliers of this rank's cells, [k][j][q]; forcing [k][j]
  const float* tens[3];
  const float* forcing;
  int E, T, Q, nt;  // nt = tensors streamed (2: diffusion, 3: + convection)
  // points of this rank: interior (E*Q) ++ boundary ++ sensors
  const float2* pts;
  int n_int, n_bnd, n_sen;
  const float* bval;  // (float) boundary targets
  const float* sval;  // (float) sensor targets
  float eps, bx, by;
  int eps_source, eps_scalar_index;
  float inv_nt;  // Real(1)/Real(T)
  float rscale;  // Real(2)*weight*inv_nt
  float bscale;  // Real(2)*tau/Real(N_D global)
  float sscale;  // Real(2)*gamma/Real(N_S global)
  // tiling
  int cells_per_tile, n_int_tiles, n_tiles;
  int chunk_rows;    // slab rows per ring stage
  int stage_floats;  // floats per ring stage (16B multiple)
  int tstride;       // floats between tensors inside a stage
  int union_floats;
  // network
  NetDesc net;
  const float* params;
  // outputs (per CTA)
  float* grad_part;   // param-major [n_params][part_stride]: entry p*part_stride + cta
  int part_stride;    // >= gridDim.x
  double* loss_part;  // [gridDim.x][kLpWords]
  // forward mode: arbitrary points in, outputs out
  const float2* fwd_pts;
  int n_fwd;
  float* out_u;
  float* out_ux;
  float* out_uy;
  float* out_eps;
  // reverse mode: adjoints in (interior uxb/uyb/eb, penalty ub)
  const float* in_ub;
  const float* in_uxb;
  const float* in_uyb;
  const float* in_eb;
  const int* stop_flag;  // device trainer: non-zero -> no-op
  // diagnostics (VPINN_PHASE_CLOCK=1): clock64() of CTA 0's thread 0 at the
  // phase marks of its first kPhaseTiles tiles, [tile][kPhaseMarks]; else null
  long long* phase_clk;
  // tc2_step_kernel: per-CTA fp32 parameter-gradient scratch [cta][layer][64][64]
  float* tc_scratch;
  int tc_force_spill;  // test hook (VPINN_TC2_FORCE_SPILL=1): spill the accumulators every tile
  // strong form (sf_step_kernel.cuh): f at the interior points, 1/N_int
  // (global) and Real(2)*weight*inv_n; order-2 evaluate outputs
  const float* sforce;
  float inv_ni, rscale_s;
  float* out_uxx;
  float* out_uyy;
};
constexpr int kPhaseTiles = 8, kPhaseMarks = 32;

template <int H, int D, int C>
struct Layout {
  static_assert(H % 2 == 0 && H >= 4 && H <= 64, "hidden width");
  static_assert(D >= 1 && D <= 4, "hidden layers");
  static_assert(C == 1 || C == 2, "output channels");
  static constexpr int HP = (H + 3) & ~3;
  // the last hidden layer's state lives in registers when it fits
  static constexpr bool kLastRegs = (3 * H <= 96);
  // state blocks (z | TXx | TXy of one hidden layer, 3*HP floats each):
  // hidden h (1 <= h <= D-2) in block h-1; the last hidden layer in the last
  // block when it does not live in registers; block 0 always exists (forward
  // scratch for D == 2, G_0 in the reverse).
  static constexpr int kBlocksMid = (D >= 3 ? D - 2 : 0) + (kLastRegs ? 0 : 1);
  static constexpr int kBlocks = kBlocksMid > 0 ? kBlocksMid : 1;
  static constexpr int SROW0 = kBlocks * 3 * HP;
  static constexpr int SROW = ((SROW0 / 4) % 2 == 1) ? SROW0 : SROW0 + 4;
  static constexpr int SG0 = (H + 1 + 3) & ~3;
  static constexpr int SG = ((SG0 / 4) % 2 == 1) ? SG0 : SG0 + 4;
  // weights: L0 as float4 rows; hidden layers [HP][HP] + bias[HP]; the last
  // hidden layer also transposed (input-major) when it feeds registers;
  // output [C][HP] + bias[4]
  static constexpr int W0F = 4 * H;
  static constexpr int WHF = HP * HP + HP;
  static constexpr int WTF = (D >= 2 && kLastRegs) ? HP * HP : 0;
  static constexpr int WDF = C * HP + 4;
  static constexpr int WTOT = W0F + (D - 1) * WHF + WTF + WDF;
  // parameter-gradient registers per thread: thread t owns compact indices
  // t + kThreads*m (deterministic single-owner accumulation)
  static constexpr int NPMAX = 3 * H + (D - 1) * (H * H + H) + C * (H + 1) + 8;
  static constexpr int NGR = (NPMAX + kThreads - 1) / kThreads;
  static constexpr int REV_UNION = kThreads * SG;
  // per-warp parameter-gradient partials of a hidden->hidden layer; wide
  // layers (H = 50) combine them in two rounds of kWarps / 2 so the
  // reverse-phase union fits shared memory next to the 128-point state
  static constexpr int PART_GROUPS = kWarps * (HP * HP + HP) > 8192 ? 2 : 1;
  static constexpr int PART_FLOATS_H = (kWarps / PART_GROUPS) * (HP * HP + HP);
  static constexpr int REV_NEED = REV_UNION > PART_FLOATS_H ? REV_UNION : PART_FLOATS_H;
  static constexpr int OFF_W = 0;
  static constexpr int OFF_EX = OFF_W + WTOT;
  static constexpr int OFF_RED = OFF_EX + kExRows * kThreads;  // 64 doubles
  static constexpr int OFF_CELL = OFF_RED + 128;               // 2 x 128 floats
  static constexpr int OFF_STATE = OFF_CELL + 2 * kThreads;
  static constexpr int OFF_UNION = OFF_STATE + kThreads * SROW + 4;
};

template <int H, int D, int C>
__host__ __device__ constexpr size_t step_smem_bytes(int union_floats, int chunk_rows) {
  using LY = Layout<H, D, C>;
  return sizeof(float) * (size_t)(LY::OFF_UNION + union_floats + 4 * ((chunk_rows + 3) & ~3)) +
         2 * sizeof(uint64_t) + 16;
}

// ---------------------------------------------------------------------------
// small vector helpers
template <int N>
__device__ __forceinline__ void load_vec(const float* row, float (&v)[N]) {
#pragma unroll
  for (int j = 0; j < (N / 4) * 4; j += 4) {
    const float4 a = lds4(row + j);
    v[j] = a.x;
    v[j + 1] = a.y;
    v[j + 2] = a.z;
    v[j + 3] = a.w;
  }
#pragma unroll
  for (int j = (N / 4) * 4; j < N; ++j) v[j] = row[j];
}

// stores v[0..N) and zeroes the padding up to the next multiple of 4
template <int N>
__device__ __forceinline__ void store_vec(float* row, const float (&v)[N]) {
#pragma unroll
  for (int j = 0; j < (N / 4) * 4; j += 4) sts4(row + j, make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
  if constexpr (N % 4 != 0) {
    constexpr int j = (N / 4) * 4;
    float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < N % 4; ++r) t[r] = v[j + r];
    sts4(row + j, make_float4(t[0], t[1], t[2], t[3]));
  }
}

// ---------------------------------------------------------------------------
// forward helpers
// 4 output rows (i0..i0+3) x 3 streams of y = W x over H register inputs
template <int H, int HP>
__device__ __forceinline__ void mv3_rows4(const float* __restrict__ W, int i0, const float (&xz)[H],
                                          const float (&xt)[H], const float (&xu)[H],
                                          float (&a)[4], float (&tx)[4], float (&ty)[4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) a[r] = tx[r] = ty[r] = 0.0f;
#pragma unroll
  for (int j = 0; j < (H / 4) * 4; j += 4) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 w = lds4(W + (i0 + r) * HP + j);
      a[r] = fmaf(w.x, xz[j], a[r]);
      tx[r] = fmaf(w.x, xt[j], tx[r]);
      ty[r] = fmaf(w.x, xu[j], ty[r]);
      a[r] = fmaf(w.y, xz[j + 1], a[r]);
      tx[r] = fmaf(w.y, xt[j + 1], tx[r]);
      ty[r] = fmaf(w.y, xu[j + 1], ty[r]);
      a[r] = fmaf(w.z, xz[j + 2], a[r]);
      tx[r] = fmaf(w.z, xt[j + 2], tx[r]);
      ty[r] = fmaf(w.z, xu[j + 2], ty[r]);
      a[r] = fmaf(w.w, xz[j + 3], a[r]);
      tx[r] = fmaf(w.w, xt[j + 3], tx[r]);
      ty[r] = fmaf(w.w, xu[j + 3], ty[r]);
    }
  }
#pragma unroll
  for (int j = (H / 4) * 4; j < H; ++j) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float w = W[(i0 + r) * HP + j];
      a[r] = fmaf(w, xz[j], a[r]);
      tx[r] = fmaf(w, xt[j], tx[r]);
      ty[r] = fmaf(w, xu[j], ty[r]);
    }
  }
}

// hidden layer (register inputs) -> state block (z | TXx | TXy), output rows rolled
template <int H, int HP, int ACT>
__device__ __forceinline__ void hidden_to_block(const float* W, const float (&xz)[H], const float (&xt)[H],
                                                const float (&xu)[H], float* blk) {
  const float* B = W + HP * HP;
#pragma unroll 1
  for (int i0 = 0; i0 < HP; i0 += 4) {
    float a[4], tx[4], ty[4];
    mv3_rows4<H, HP>(W, i0, xz, xt, xu, a, tx, ty);
    float z[4], gx[4], gy[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      z[r] = Act<ACT>::value(a[r] + B[i0 + r]);
      const float s1 = Act<ACT>::s1(z[r]);
      gx[r] = s1 * tx[r];
      gy[r] = s1 * ty[r];
    }
    sts4(blk + i0, make_float4(z[0], z[1], z[2], z[3]));
    sts4(blk + HP + i0, make_float4(gx[0], gx[1], gx[2], gx[3]));
    sts4(blk + 2 * HP + i0, make_float4(gy[0], gy[1], gy[2], gy[3]));
  }
}

// hidden layer with inputs from a state block (own row) and outputs in
// registers: input-major, the input loop rolled, W transposed in SMEM
// ([in][out], rows of HP); accumulators oz/ot/ou sized HP.
template <int H, int HP, int ACT>
__device__ __forceinline__ void hidden_block_to_regs(const float* WT, const float* B, const float* blk,
                                                     float (&oz)[HP], float (&ot)[HP], float (&ou)[HP]) {
#pragma unroll
  for (int i = 0; i < HP; ++i) oz[i] = ot[i] = ou[i] = 0.0f;
#pragma unroll 1
  for (int j0 = 0; j0 < H; j0 += 2) {
    const float2 zz = *reinterpret_cast<const float2*>(blk + j0);
    const float2 tt = *reinterpret_cast<const float2*>(blk + HP + j0);
    const float2 uu = *reinterpret_cast<const float2*>(blk + 2 * HP + j0);
    const float zi[2] = {zz.x, zz.y}, ti[2] = {tt.x, tt.y}, ui[2] = {uu.x, uu.y};
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
#pragma unroll
      for (int i = 0; i < HP; i += 4) {
        const float4 w = lds4(WT + (j0 + jj) * HP + i);
        const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          oz[i + r] = fmaf(wv[r], zi[jj], oz[i + r]);
          ot[i + r] = fmaf(wv[r], ti[jj], ot[i + r]);
          ou[i + r] = fmaf(wv[r], ui[jj], ou[i + r]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < HP; ++i) {
    if (i < H) {
      const float z = Act<ACT>::value(oz[i] + B[i]);
      const float s1 = Act<ACT>::s1(z);
      oz[i] = z;
      ot[i] = s1 * ot[i];
      ou[i] = s1 * ou[i];
    } else {
      oz[i] = ot[i] = ou[i] = 0.0f;
    }
  }
}

// ---------------------------------------------------------------------------
// reverse helpers
// warp-level outer-product tile: acc[4x8] += sum_{p<32} G[p][o0..o0+3] (x)
// Hm[p][i0..i0+7]; G/Hm point at the warp's first row.
__device__ __forceinline__ void warp_outer_tile(const float* __restrict__ G, int sg,
                                                const float* __restrict__ Hm, int sh, int o0,
                                                int i0, float (&acc)[32]) {
#pragma unroll 4
  for (int p = 0; p < 32; ++p) {
    const float4 g = lds4(G + p * sg + o0);
    const float4 h0 = lds4(Hm + p * sh + i0);
    const float4 h1 = lds4(Hm + p * sh + i0 + 4);
    const float gv[4] = {g.x, g.y, g.z, g.w};
    const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a * 8 + b] = fmaf(gv[a], hv[b], acc[a * 8 + b]);
  }
}

// block-wide deterministic sum of one double per thread (result valid in
// thread 0); red has >= kWarps doubles
__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kWarps; ++w) s += red[w];
  return s;
}

// greg[m] (compact index tid + kThreads*m) += val(e) for e = index - lo in
// [0, cnt); only the m that can hit the range are visited (rolled loop;
// greg lives in L1-resident local memory)
template <int NGR, typename F>
__device__ __forceinline__ void own_add(float (&greg)[NGR], int tid, int lo, int cnt, F&& val) {
  const int m0 = max(0, (lo - tid + kThreads - 1) / kThreads);
  const int m1 = min(NGR, (lo + cnt - tid + kThreads - 1) / kThreads);
#pragma unroll 1
  for (int m = m0; m < m1; ++m) {
    const int e = tid + kThreads * m - lo;
    if (e >= 0 && e < cnt) greg[m] += val(e);
  }
}

// ---------------------------------------------------------------------------
// slab chunk copies (thread 0): aligned superset of each tensor's rows.
// Inlined and array-free so the kernel-parameter struct is never copied to
// the stack (local-memory round trips on every issue).
__device__ __forceinline__ void issue_chunk(const StepArgs& a, int cell0, int row0, int nrows, float* stage,
                                            uint64_t* bar) {
  const size_t grow0 = (size_t)cell0 * a.T + row0;
  auto seg = [&](int t, const char*& src) {
    const char* s = reinterpret_cast<const char*>(a.tens[t] + grow0 * a.Q);
    src = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(s) & ~uintptr_t(15));
    const uint32_t pre = (uint32_t)(s - src);
    return (pre + (uint32_t)nrows * a.Q * 4u + 15u) & ~15u;
  };
  const char* s0;
  const char* s1;
  const char* s2 = nullptr;
  const uint32_t n0 = seg(0, s0), n1 = seg(1, s1), n2 = a.nt == 3 ? seg(2, s2) : 0u;
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, n0 + n1 + n2);
  bulk_g2s(stage, s0, n0, bar);
  bulk_g2s(stage + a.tstride, s1, n1, bar);
  if (a.nt == 3) bulk_g2s(stage + 2 * a.tstride, s2, n2, bar);
}

__device__ __forceinline__ const float* chunk_ptr(const StepArgs& a, int cell0, int row0, const float* stage,
                                                  int t) {
  const size_t grow0 = (size_t)cell0 * a.T + row0;
  const uintptr_t s = reinterpret_cast<uintptr_t>(a.tens[t] + grow0 * a.Q);
  return stage + t * a.tstride + ((s & 15u) >> 2);
}

// ---------------------------------------------------------------------------
struct RevCtx {
  float* sState;
  float* srow;
  float* Gbuf;
  float* Part;
  const float* sW0;
  const float* sWh;
  const NetDesc* netp;
  float px, py;
  int tid, lane, warp;
};

// Reverse through hidden->hidden weight layer l (1 <= l <= D-1): parameter
// gradient (three streams) + propagation to hidden l-1 (network.hpp:320-358).
// On entry gA/gX/gY hold G_l for l == D-1; otherwise G_l sits in the state
// block of hidden l (written in place by the previous call).
template <int H, int D, int C, int ACT, int l, int NGR>
__device__ __forceinline__ void reverse_hidden(RevCtx& rc, float (&gA)[H], float (&gX)[H], float (&gY)[H],
                                               float (&greg)[NGR]) {
  using LY = Layout<H, D, C>;
  constexpr int HP = LY::HP;
  constexpr int SROW = LY::SROW;
  constexpr int SG = LY::SG;
  float* sState = rc.sState;
  float* srow = rc.srow;
  float* Gbuf = rc.Gbuf;
  float* Part = rc.Part;
  const float* sW0 = rc.sW0;
  const NetDesc& net = *rc.netp;
  const int tid = rc.tid, lane = rc.lane, warp = rc.warp;
  const int wrow = warp * 32;
  if constexpr (l != D - 1) {
    load_vec<H>(srow + (l - 1) * 3 * HP, gA);
    load_vec<H>(srow + (l - 1) * 3 * HP + HP, gX);
    load_vec<H>(srow + (l - 1) * 3 * HP + 2 * HP, gY);
  }
  const float* W = rc.sWh + (l - 1) * LY::WHF;
  // H operand rows: hidden l-1 = block l-2 (l >= 2) or the recomputed layer-0
  // state staged in block 0 (l == 1; block 0 is free here)
  const float* Hm;
  float z0r[l == 1 ? H : 1];
  if constexpr (l >= 2) {
    Hm = sState + wrow * SROW + (l - 2) * 3 * HP;
  } else {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float4 w = lds4(sW0 + 4 * i);
      z0r[i] = Act<ACT>::value(fmaf(w.y, rc.py, w.x * rc.px) + w.z);
    }
    Hm = sState + wrow * SROW;
  }
  constexpr int NOB = (H + 3) / 4, NIB = (H + 7) / 8, NTILE = NOB * NIB;
  constexpr int NROUND = (NTILE + 31) / 32;
  float accr[NROUND][32];
#pragma unroll
  for (int rr = 0; rr < NROUND; ++rr)
#pragma unroll
    for (int k = 0; k < 32; ++k) accr[rr][k] = 0.f;
  float bsum[(H + 31) / 32];
  // three passes: value, x-tangent, y-tangent streams
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    {
      float gsel[H];
#pragma unroll
      for (int i = 0; i < H; ++i) gsel[i] = pass == 0 ? gA[i] : (pass == 1 ? gX[i] : gY[i]);
      store_vec<H>(Gbuf + tid * SG, gsel);
    }
    if constexpr (l == 1) {
      float tv[H];
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const float4 w = lds4(sW0 + 4 * i);
        const float wsel = pass == 1 ? w.x : w.y;
        tv[i] = pass == 0 ? z0r[i] : Act<ACT>::s1(z0r[i]) * wsel;
      }
      store_vec<H>(srow, tv);
    }
    __syncthreads();
    const float* Hp = (l >= 2) ? Hm + pass * HP : Hm;
#pragma unroll
    for (int rr = 0; rr < NROUND; ++rr) {
      const int t = lane + 32 * rr;
      if (t < NTILE) {
        const int ob = t % NOB, ib = t / NOB;
        warp_outer_tile(Gbuf + wrow * SG, SG, Hp, SROW, ob * 4, ib * 8, accr[rr]);
      }
    }
    if (pass == 0) {
#pragma unroll
      for (int s = 0; s < (H + 31) / 32; ++s) {
        const int col = lane + 32 * s;
        float acc = 0.f;
        if (col < H)
#pragma unroll 4
          for (int p = 0; p < 32; ++p) acc += Gbuf[(wrow + p) * SG + col];
        bsum[s] = acc;
      }
    }
    __syncthreads();
  }
  // partials [warp][HP][HP] + bias [warp][HP], summed over warps in a fixed
  // order (in PART_GROUPS rounds for wide layers)
  constexpr int kGroups = LY::PART_GROUPS, kWpg = kWarps / kGroups;
#pragma unroll 1
  for (int grp = 0; grp < kGroups; ++grp) {
    if (warp / kWpg == grp) {
      float* pw = Part + (warp % kWpg) * (HP * HP + HP);
#pragma unroll
      for (int rr = 0; rr < NROUND; ++rr) {
        const int t = lane + 32 * rr;
        if (t < NTILE) {
          const int ob = t % NOB, ib = t / NOB;
#pragma unroll
          for (int a4 = 0; a4 < 4; ++a4) {
            const int o = ob * 4 + a4;
            if (o < HP && ib * 8 < HP)
              sts4(pw + o * HP + ib * 8, make_float4(accr[rr][a4 * 8], accr[rr][a4 * 8 + 1], accr[rr][a4 * 8 + 2],
                                                     accr[rr][a4 * 8 + 3]));
            if (o < HP && ib * 8 + 4 < HP)
              sts4(pw + o * HP + ib * 8 + 4, make_float4(accr[rr][a4 * 8 + 4], accr[rr][a4 * 8 + 5],
                                                         accr[rr][a4 * 8 + 6], accr[rr][a4 * 8 + 7]));
          }
        }
      }
#pragma unroll
      for (int s = 0; s < (H + 31) / 32; ++s) {
        const int col = lane + 32 * s;
        if (col < H) pw[HP * HP + col] = bsum[s];
      }
    }
    __syncthreads();
    {
      const int fi = net.in_w[l], fo = net.out_w[l];
      own_add(greg, tid, net.w_off[l], fo * fi, [&](int e) {
        const int o = e / fi, i = e - o * fi;
        float s = Part[o * HP + i];
#pragma unroll
        for (int w = 1; w < kWpg; ++w) s += Part[w * (HP * HP + HP) + o * HP + i];
        return s;
      });
      own_add(greg, tid, net.b_off[l], fo, [&](int o) {
        float s = Part[HP * HP + o];
#pragma unroll
        for (int w = 1; w < kWpg; ++w) s += Part[w * (HP * HP + HP) + HP * HP + o];
        return s;
      });
    }
    __syncthreads();
  }
  // propagate: Xbar = W^T Abar etc.; through hidden l-1's activation
  if constexpr (l == 1) store_vec<H>(Gbuf + tid * SG, z0r);  // own row: z0 for the chunks
#pragma unroll 1
  for (int j0 = 0; j0 < HP; j0 += 4) {
    float xb[4] = {0.f, 0.f, 0.f, 0.f}, zx[4] = {0.f, 0.f, 0.f, 0.f}, zy[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float4 w = lds4(W + i * HP + j0);
      const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        xb[r] = fmaf(wv[r], gA[i], xb[r]);
        zx[r] = fmaf(wv[r], gX[i], zx[r]);
        zy[r] = fmaf(wv[r], gY[i], zy[r]);
      }
    }
    float z[4], txv[4], tyv[4];
    float* dst;
    if constexpr (l >= 2) {
      float* blk = srow + (l - 2) * 3 * HP;
      const float4 a4 = lds4(blk + j0), b4 = lds4(blk + HP + j0), c4 = lds4(blk + 2 * HP + j0);
      z[0] = a4.x; z[1] = a4.y; z[2] = a4.z; z[3] = a4.w;
      txv[0] = b4.x; txv[1] = b4.y; txv[2] = b4.z; txv[3] = b4.w;
      tyv[0] = c4.x; tyv[1] = c4.y; tyv[2] = c4.z; tyv[3] = c4.w;
      dst = blk;
    } else {
      const float4 a4 = lds4(Gbuf + tid * SG + j0);
      z[0] = a4.x; z[1] = a4.y; z[2] = a4.z; z[3] = a4.w;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int j = min(j0 + r, H - 1);
        const float4 w = lds4(sW0 + 4 * j);
        const float s1 = Act<ACT>::s1(z[r]);
        txv[r] = s1 * w.x;
        tyv[r] = s1 * w.y;
      }
      dst = srow;  // G_0 goes to block 0
    }
    float oa[4], ox[4], oy[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float s1 = Act<ACT>::s1(z[r]), kp = Act<ACT>::kap(z[r]);
      oa[r] = fmaf(s1, xb[r], kp * fmaf(txv[r], zx[r], tyv[r] * zy[r]));
      ox[r] = s1 * zx[r];
      oy[r] = s1 * zy[r];
    }
    sts4(dst + j0, make_float4(oa[0], oa[1], oa[2], oa[3]));
    sts4(dst + HP + j0, make_float4(ox[0], ox[1], ox[2], ox[3]));
    sts4(dst + 2 * HP + j0, make_float4(oy[0], oy[1], oy[2], oy[3]));
  }
}

// ---------------------------------------------------------------------------
template <int H, int D, int C, int ACT, int MODE>
__global__ void __launch_bounds__(kThreads, 2) step_kernel(const StepArgs a) {
  using LY = Layout<H, D, C>;
  constexpr int HP = LY::HP;
  constexpr int SROW = LY::SROW;
  constexpr int SG = LY::SG;
  constexpr bool kLastRegs = LY::kLastRegs;

  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;

  extern __shared__ __align__(128) float smem[];
  float* sW0 = smem + LY::OFF_W;
  float* sWh = sW0 + LY::W0F;
  float* sWT = sWh + (D - 1) * LY::WHF;  // transposed last hidden layer
  float* sWd = sWT + LY::WTF;
  float* sEx = smem + LY::OFF_EX;
  double* sRed = reinterpret_cast<double*>(smem + LY::OFF_RED);
  float* sCell = smem + LY::OFF_CELL;  // [0,128) r^2 sums, [128,256) eps-grad sums
  float* sState = smem + LY::OFF_STATE;
  float* sUnion = smem + LY::OFF_UNION;
  float* sRows = sUnion + a.union_floats;  // rbar | rsq | rge per chunk row
  const int rows4 = (a.chunk_rows + 3) & ~3;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRows + 4 * rows4);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const NetDesc& net = a.net;
  const float* P = a.params;

  // ---- weights -> SMEM (zero-padded to the template width) ----
  for (int i = tid; i < H; i += kThreads) {
    float w0 = 0.f, w1 = 0.f, b = 0.f;
    if (i < net.out_w[0]) {
      w0 = P[net.w_off[0] + 2 * i];
      w1 = P[net.w_off[0] + 2 * i + 1];
      b = P[net.b_off[0] + i];
    }
    sts4(sW0 + 4 * i, make_float4(w0, w1, b, 0.f));
  }
  for (int l = 1; l < D; ++l) {
    float* W = sWh + (l - 1) * LY::WHF;
    const int fi = net.in_w[l], fo = net.out_w[l];
    const bool transpose = (LY::WTF > 0) && l == D - 1;
    for (int e = tid; e < LY::WHF; e += kThreads) {
      float v = 0.f;
      if (e < HP * HP) {
        const int i = e / HP, j = e - i * HP;
        if (i < fo && j < fi) v = P[net.w_off[l] + i * fi + j];
        if (transpose) sWT[j * HP + i] = v;
      } else {
        const int i = e - HP * HP;
        if (i < fo) v = P[net.b_off[l] + i];
      }
      W[e] = v;
    }
  }
  {
    const int fi = net.in_w[D];
    for (int e = tid; e < LY::WDF; e += kThreads) {
      float v = 0.f;
      if (e < C * HP) {
        const int c = e / HP, j = e - c * HP;
        if (j < fi) v = P[net.w_off[D] + c * fi + j];
      } else {
        const int c = e - C * HP;
        if (c < C) v = P[net.b_off[D] + c];
      }
      sWd[e] = v;
    }
  }
  float greg[LY::NGR];
#pragma unroll
  for (int m = 0; m < LY::NGR; ++m) greg[m] = 0.f;
  if (MODE == kModeFused && tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  for (int e = tid; e < 2 * kThreads; e += kThreads) sCell[e] = 0.f;
  __syncthreads();

  uint32_t parity = 0u;  // bit s = phase parity of ring stage s
  double acc_v = 0.0, acc_b = 0.0, acc_s = 0.0, acc_eg = 0.0;  // thread 0
  int bad = 0;

  const int n_tiles = (MODE == kModeForward) ? (a.n_fwd + kThreads - 1) / kThreads : a.n_tiles;
  const int n_pts_all = a.n_int + a.n_bnd + a.n_sen;

#pragma unroll 1
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    // ---- tile geometry ----
    bool interior = false;
    int cell0 = 0, ncell = 0, pbase = 0, np = 0;
    if (MODE == kModeFused) {
      if (tile < a.n_int_tiles) {
        interior = true;
        cell0 = tile * a.cells_per_tile;
        ncell = min(a.cells_per_tile, a.E - cell0);
        pbase = cell0 * a.Q;
        np = ncell * a.Q;
      } else {
        pbase = a.n_int + (tile - a.n_int_tiles) * kThreads;
        np = min(kThreads, n_pts_all - pbase);
      }
    } else if (MODE == kModeReverse) {
      pbase = tile * kThreads;
      np = min(kThreads, n_pts_all - pbase);
    } else {
      pbase = tile * kThreads;
      np = min(kThreads, a.n_fwd - pbase);
    }
    const int nrows_tile = ncell * a.T;
    const int nchunks = interior ? (nrows_tile + a.chunk_rows - 1) / a.chunk_rows : 0;

    // ---- prefetch the first two slab chunks (overlaps the forward) ----
    if (MODE == kModeFused && interior && tid == 0) {
      for (int c = 0; c < 2 && c < nchunks; ++c) {
        const int r0 = c * a.chunk_rows;
        issue_chunk(a, cell0, r0, min(a.chunk_rows, nrows_tile - r0), sUnion + c * a.stage_floats, &bars[c]);
      }
    }

    const bool valid = tid < np;
    float px = 0.f, py = 0.f;
    if (valid) {
      const float2 xy = (MODE == kModeForward) ? a.fwd_pts[pbase + tid] : a.pts[pbase + tid];
      px = xy.x;
      py = xy.y;
    }
    sEx[kExX * kThreads + tid] = px;
    sEx[kExY * kThreads + tid] = py;

    // =================== forward (network.hpp:239-281) ===================
    float* srow = sState + tid * SROW;
    float lz[kLastRegs ? HP : 1], lt[kLastRegs ? HP : 1], lu[kLastRegs ? HP : 1];
    {
      float z0[H], t0[H], u0[H];
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const float4 w = lds4(sW0 + 4 * i);
        const float z = Act<ACT>::value(fmaf(w.y, py, w.x * px) + w.z);
        const float s1 = Act<ACT>::s1(z);
        z0[i] = z;
        t0[i] = s1 * w.x;  // TX_1 = s1 (W0 e_x)
        u0[i] = s1 * w.y;
      }
      if constexpr (D == 1) {
        if constexpr (kLastRegs) {
#pragma unroll
          for (int i = 0; i < HP; ++i) {
            lz[i] = i < H ? z0[i] : 0.f;
            lt[i] = i < H ? t0[i] : 0.f;
            lu[i] = i < H ? u0[i] : 0.f;
          }
        } else {
          float* blk = srow + (LY::kBlocks - 1) * 3 * HP;
          store_vec<H>(blk, z0);
          store_vec<H>(blk + HP, t0);
          store_vec<H>(blk + 2 * HP, u0);
        }
      } else if constexpr (D == 2 && kLastRegs) {
        // layer 1 is the last hidden layer: stage the layer-0 state in block 0
        store_vec<H>(srow, z0);
        store_vec<H>(srow + HP, t0);
        store_vec<H>(srow + 2 * HP, u0);
      } else if constexpr (D == 2) {
        hidden_to_block<H, HP, ACT>(sWh, z0, t0, u0, srow + (LY::kBlocks - 1) * 3 * HP);
      } else {
        hidden_to_block<H, HP, ACT>(sWh, z0, t0, u0, srow);  // block 0 = hidden 1
      }
    }
    // middle hidden layers 2..D-2 (register inputs loaded from the previous block)
#pragma unroll 1
    for (int l = 2; l < D - 1; ++l) {
      float xz[H], xt[H], xu[H];
      load_vec<H>(srow + (l - 2) * 3 * HP, xz);
      load_vec<H>(srow + (l - 2) * 3 * HP + HP, xt);
      load_vec<H>(srow + (l - 2) * 3 * HP + 2 * HP, xu);
      hidden_to_block<H, HP, ACT>(sWh + (l - 1) * LY::WHF, xz, xt, xu, srow + (l - 1) * 3 * HP);
    }
    // last hidden layer D-1 >= 1
    if constexpr (D >= 2) {
      const float* Wl = sWh + (D - 2) * LY::WHF;
      if constexpr (kLastRegs) {
        const float* in_blk = (D == 2) ? srow : srow + (D - 3) * 3 * HP;
        hidden_block_to_regs<H, HP, ACT>(sWT, Wl + HP * HP, in_blk, lz, lt, lu);
      } else if constexpr (D >= 3) {
        float xz[H], xt[H], xu[H];
        load_vec<H>(srow + (D - 3) * 3 * HP, xz);
        load_vec<H>(srow + (D - 3) * 3 * HP + HP, xt);
        load_vec<H>(srow + (D - 3) * 3 * HP + 2 * HP, xu);
        hidden_to_block<H, HP, ACT>(Wl, xz, xt, xu, srow + (LY::kBlocks - 1) * 3 * HP);
      }
    }
    // output layer (linear): u, du/dx, du/dy; channel 1 -> eps head
    {
      float u = 0.f, ux = 0.f, uy = 0.f, y1 = 0.f;
      if constexpr (kLastRegs) {
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const float w = sWd[j];
          u = fmaf(w, lz[j], u);
          ux = fmaf(w, lt[j], ux);
          uy = fmaf(w, lu[j], uy);
          if constexpr (C == 2) y1 = fmaf(sWd[HP + j], lz[j], y1);
        }
      } else {
        const float* blk = srow + (LY::kBlocks - 1) * 3 * HP;
#pragma unroll 2
        for (int j = 0; j < H; ++j) {
          const float w = sWd[j];
          u = fmaf(w, blk[j], u);
          ux = fmaf(w, blk[HP + j], ux);
          uy = fmaf(w, blk[2 * HP + j], uy);
          if constexpr (C == 2) y1 = fmaf(sWd[HP + j], blk[j], y1);
        }
      }
      u += sWd[C * HP];
      if constexpr (C == 2) y1 += sWd[C * HP + 1];
      if (valid && !(finitef(u) && finitef(ux) && finitef(uy))) bad = 1;
      sEx[kExU * kThreads + tid] = u;
      sEx[kExUx * kThreads + tid] = ux;
      sEx[kExUy * kThreads + tid] = uy;
      if constexpr (C == 2) {
        sEx[kExY1 * kThreads + tid] = y1;
        sEx[kExE * kThreads + tid] = softplusf(y1);
      }
      if (MODE == kModeForward) {
        if (valid) {
          if (a.out_u) a.out_u[pbase + tid] = u;
          if (a.out_ux) a.out_ux[pbase + tid] = ux;
          if (a.out_uy) a.out_uy[pbase + tid] = uy;
          if (C == 2 && a.out_eps) a.out_eps[pbase + tid] = softplusf(y1);
        }
      }
    }
    if constexpr (MODE == kModeForward) continue;

    // =================== objective: adjoints of (u, ux, uy, eps) ===================
    float ub = 0.f, uxb = 0.f, uyb = 0.f, eb = 0.f;
    if constexpr (MODE == kModeReverse) {
      if (valid) {
        const int p = pbase + tid;
        if (p < a.n_int) {
          uxb = a.in_uxb[p];
          uyb = a.in_uyb[p];
          if (C == 2 && a.in_eb) eb = a.in_eb[p];
        } else {
          ub = a.in_ub[p - a.n_int];
        }
      }
    } else if (interior) {
      // ---------- Algorithm 3 on the tile (losses.hpp:111-166) ----------
      const bool spatial = a.eps_source == 2;
      const bool conv = a.nt == 3;
      // scalar source: the trainable coefficient is the current parameter value
      const float e_fixed = a.eps_source == 1 ? P[net.scal_off + a.eps_scalar_index] : a.eps;
      {
        const float ux = sEx[kExUx * kThreads + tid], uy = sEx[kExUy * kThreads + tid];
        const float ep = spatial ? sEx[kExE * kThreads + tid] : 1.0f;
        sEx[kExSx * kThreads + tid] = spatial ? ep * ux : ux;
        sEx[kExSy * kThreads + tid] = spatial ? ep * uy : uy;
        sEx[kExCv * kThreads + tid] = a.bx * ux + a.by * uy;
      }
      __syncthreads();
      float tx = 0.f, ty = 0.f, tt = 0.f;  // per point: Gx^T rbar, Gy^T rbar, T^T rbar
      const int myk = valid ? tid / a.Q : 0;
      const int myq = valid ? tid - myk * a.Q : 0;
      float* rbarv = sRows;
      float* rsqv = sRows + rows4;
      float* rgev = sRows + 2 * rows4;
#pragma unroll 1
      for (int c = 0; c < nchunks; ++c) {
        const int st = c & 1;
        const int r0 = c * a.chunk_rows;
        const int nr = min(a.chunk_rows, nrows_tile - r0);
        float* stage = sUnion + st * a.stage_floats;
        mbar_wait(&bars[st], (parity >> st) & 1u);
        parity ^= 1u << st;
        const float* Gx = chunk_ptr(a, cell0, r0, stage, 0);
        const float* Gy = chunk_ptr(a, cell0, r0, stage, 1);
        const float* Tv = conv ? chunk_ptr(a, cell0, r0, stage, 2) : nullptr;
        // phase A: one thread per slab row: residual r_j
        for (int r = tid; r < nr; r += kThreads) {
          const int gr = r0 + r;
          const int kk = gr / a.T;
          const int j = gr - kk * a.T;
          const float* sx = sEx + kExSx * kThreads + kk * a.Q;
          const float* sy = sEx + kExSy * kThreads + kk * a.Q;
          const float* gxr = Gx + r * a.Q;
          const float* gyr = Gy + r * a.Q;
          float gx = 0.f, gy = 0.f;
#pragma unroll 5
          for (int q = 0; q < a.Q; ++q) {
            gx = fmaf(gxr[q], sx[q], gx);
            gy = fmaf(gyr[q], sy[q], gy);
          }
          float res = spatial ? gx + gy : e_fixed * (gx + gy);
          if (conv) {
            const float* cv = sEx + kExCv * kThreads + kk * a.Q;
            const float* tr = Tv + r * a.Q;
            float t = 0.f;
#pragma unroll 5
            for (int q = 0; q < a.Q; ++q) t = fmaf(tr[q], cv[q], t);
            res += t;
          }
          res -= a.forcing[(size_t)(cell0 + kk) * a.T + j];
          rsqv[r] = res * res;
          const float rb = a.rscale * res;
          rbarv[r] = rb;
          rgev[r] = rb * (gx + gy);
        }
        __syncthreads();
        // phase B: one thread per point: adjoint contributions of the chunk rows
        if (valid) {
          const int lo = max(r0, myk * a.T), hi = min(r0 + nr, (myk + 1) * a.T);
#pragma unroll 5
          for (int gr = lo; gr < hi; ++gr) {
            const int r = gr - r0;
            const float rb = rbarv[r];
            tx = fmaf(Gx[r * a.Q + myq], rb, tx);
            ty = fmaf(Gy[r * a.Q + myq], rb, ty);
            if (conv) tt = fmaf(Tv[r * a.Q + myq], rb, tt);
          }
        }
        // per-cell squared-residual and eps-gradient sums in row order
        if (tid < ncell) {
          const int lo = max(r0, tid * a.T), hi = min(r0 + nr, (tid + 1) * a.T);
          float s = sCell[tid], g = sCell[kThreads + tid];
          for (int gr = lo; gr < hi; ++gr) {
            s += rsqv[gr - r0];
            g += rgev[gr - r0];
          }
          sCell[tid] = s;
          sCell[kThreads + tid] = g;
        }
        __syncthreads();
        if (tid == 0 && c + 2 < nchunks) {
          const int r2 = (c + 2) * a.chunk_rows;
          issue_chunk(a, cell0, r2, min(a.chunk_rows, nrows_tile - r2), stage, &bars[st]);
        }
      }
      if (valid) {
        const float ux = sEx[kExUx * kThreads + tid], uy = sEx[kExUy * kThreads + tid];
        if (spatial) {
          const float ep = sEx[kExE * kThreads + tid];
          uxb = ep * tx;
          uyb = ep * ty;
          eb = ux * tx + uy * ty;
        } else {
          uxb = e_fixed * tx;
          uyb = e_fixed * ty;
        }
        if (conv) {
          uxb = fmaf(a.bx, tt, uxb);
          uyb = fmaf(a.by, tt, uyb);
        }
      }
      if (tid == 0) {
        for (int k = 0; k < ncell; ++k) {
          acc_v += (double)(sCell[k] * a.inv_nt);
          acc_eg += (double)sCell[kThreads + k];
        }
      }
      __syncthreads();
      if (tid < ncell) {
        sCell[tid] = 0.f;
        sCell[kThreads + tid] = 0.f;
      }
    } else {
      // ---------- penalty tile (losses.hpp:389-415) ----------
      double sb = 0.0, ss = 0.0;
      if (valid) {
        const int pi = pbase + tid - a.n_int;
        const float u = sEx[kExU * kThreads + tid];
        if (pi < a.n_bnd) {
          const float d = u - a.bval[pi];
          sb = (double)(d * d);
          ub = a.bscale * d;
        } else {
          const float d = u - a.sval[pi - a.n_bnd];
          ss = (double)(d * d);
          ub = a.sscale * d;
        }
      }
      const double tb = block_sum_d(sb, sRed);
      const double ts = block_sum_d(ss, sRed + kWarps);
      if (tid == 0) {
        acc_b += tb;
        acc_s += ts;
      }
    }

    // =================== reverse (network.hpp:297-371) ===================
    float* Gbuf = sUnion;  // [kThreads][SG]
    float* Part = sUnion;  // partials (after a barrier)
    const int wrow = warp * 32;

    // ---- output layer l = D ----
    float ab1 = 0.f;
    if constexpr (C == 2) ab1 = eb * sigmoidf(sEx[kExY1 * kThreads + tid]);
    float gA[H], gX[H], gY[H];
    {
      float hz[H], ht[H], hu[H];
      if constexpr (kLastRegs) {
#pragma unroll
        for (int j = 0; j < H; ++j) {
          hz[j] = lz[j];
          ht[j] = lt[j];
          hu[j] = lu[j];
        }
      } else {
        const float* blk = srow + (LY::kBlocks - 1) * 3 * HP;
        load_vec<H>(blk, hz);
        load_vec<H>(blk + HP, ht);
        load_vec<H>(blk + 2 * HP, hu);
      }
      __syncthreads();  // union (slab) free; exchange reads done
      float csum[C][(H + 32) / 32];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float ab = (c == 0) ? ub : ab1;
        float v[H];
#pragma unroll
        for (int j = 0; j < H; ++j)
          v[j] = (c == 0) ? fmaf(uyb, hu[j], fmaf(uxb, ht[j], ab * hz[j])) : ab * hz[j];
        store_vec<H>(Gbuf + tid * SG, v);
        Gbuf[tid * SG + H] = ab;
        __syncwarp();
#pragma unroll
        for (int s = 0; s < (H + 32) / 32; ++s) {
          const int col = lane + 32 * s;
          float acc = 0.f;
          if (col <= H)
#pragma unroll 4
            for (int p = 0; p < 32; ++p) acc += Gbuf[(wrow + p) * SG + col];
          csum[c][s] = acc;
        }
        __syncwarp();
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int s = 0; s < (H + 32) / 32; ++s) {
          const int col = lane + 32 * s;
          if (col <= H) Part[(warp * C + c) * (H + 1) + col] = csum[c][s];
        }
      __syncthreads();
      {
        const int fi = net.in_w[D];
        own_add(greg, tid, net.w_off[D], C * fi, [&](int e) {
          const int c = e / fi, col = e - c * fi;
          float s = Part[c * (H + 1) + col];
#pragma unroll
          for (int w = 1; w < kWarps; ++w) s += Part[(w * C + c) * (H + 1) + col];
          return s;
        });
        own_add(greg, tid, net.b_off[D], C, [&](int c) {
          float s = Part[c * (H + 1) + H];
#pragma unroll
          for (int w = 1; w < kWarps; ++w) s += Part[(w * C + c) * (H + 1) + H];
          return s;
        });
      }
      // propagate to the last hidden layer: G_{D-1}
#pragma unroll
      for (int j = 0; j < H; ++j) {
        float xb = sWd[j] * ub;
        if constexpr (C == 2) xb = fmaf(sWd[HP + j], ab1, xb);
        const float zx = sWd[j] * uxb, zy = sWd[j] * uyb;
        const float s1 = Act<ACT>::s1(hz[j]), kp = Act<ACT>::kap(hz[j]);
        gA[j] = fmaf(s1, xb, kp * fmaf(ht[j], zx, hu[j] * zy));
        gX[j] = s1 * zx;
        gY[j] = s1 * zy;
      }
    }
    __syncthreads();

    // ---- hidden layers l = D-1 .. 1 ----
    {
      RevCtx rc{sState, srow, Gbuf, Part, sW0, sWh, &net, px, py, tid, lane, warp};
      if constexpr (D >= 4) reverse_hidden<H, D, C, ACT, 3>(rc, gA, gX, gY, greg);
      if constexpr (D >= 3) reverse_hidden<H, D, C, ACT, 2>(rc, gA, gX, gY, greg);
      if constexpr (D >= 2) reverse_hidden<H, D, C, ACT, 1>(rc, gA, gX, gY, greg);
    }
    if constexpr (D == 1) {
      // G_0 came straight from the output layer (registers)
      store_vec<H>(srow, gA);
      store_vec<H>(srow + HP, gX);
      store_vec<H>(srow + 2 * HP, gY);
    }
    __syncthreads();

    // ---- input layer l = 0: Wbar_0 += Abar x^T + TAxbar e_x^T + TAybar e_y^T ----
    {
      float s0[(H + 31) / 32], s1v[(H + 31) / 32], s2[(H + 31) / 32];
#pragma unroll
      for (int s = 0; s < (H + 31) / 32; ++s) {
        const int i = lane + 32 * s;
        float ax = 0.f, ay = 0.f, aa = 0.f, tx = 0.f, ty = 0.f;
        if (i < H) {
#pragma unroll 4
          for (int p = 0; p < 32; ++p) {
            const float* row = sState + (wrow + p) * SROW;
            const float ga = row[i];
            ax = fmaf(ga, sEx[kExX * kThreads + wrow + p], ax);
            ay = fmaf(ga, sEx[kExY * kThreads + wrow + p], ay);
            aa += ga;
            tx += row[HP + i];
            ty += row[2 * HP + i];
          }
        }
        s0[s] = ax + tx;
        s1v[s] = ay + ty;
        s2[s] = aa;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < (H + 31) / 32; ++s) {
        const int i = lane + 32 * s;
        if (i < H) {
          Part[(warp * 3 + 0) * H + i] = s0[s];
          Part[(warp * 3 + 1) * H + i] = s1v[s];
          Part[(warp * 3 + 2) * H + i] = s2[s];
        }
      }
      __syncthreads();
      const int fo = net.out_w[0];
      own_add(greg, tid, net.w_off[0], 2 * fo, [&](int e) {
        const int i = e >> 1, k = e & 1;
        float s = Part[k * H + i];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) s += Part[(w * 3 + k) * H + i];
        return s;
      });
      own_add(greg, tid, net.b_off[0], fo, [&](int i) {
        float s = Part[2 * H + i];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) s += Part[(w * 3 + 2) * H + i];
        return s;
      });
      __syncthreads();
    }
  }

  if constexpr (MODE != kModeForward) {
    // ---- per-CTA outputs ----
#pragma unroll 1
    for (int m = 0; m < LY::NGR; ++m) {
      const int e = tid + kThreads * m;
      if (e < net.n_params) a.grad_part[(size_t)e * a.part_stride + blockIdx.x] = greg[m];
    }
    const int any_bad = __syncthreads_or(bad);
    if (tid == 0) {
      double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
      lp[kLpVar] = acc_v;
      lp[kLpBnd] = acc_b;
      lp[kLpSen] = acc_s;
      lp[kLpEpsGrad] = acc_eg;
      lp[kLpBad] = any_bad ? 1.0 : 0.0;
    }
  }
}

}  // namespace vpg
