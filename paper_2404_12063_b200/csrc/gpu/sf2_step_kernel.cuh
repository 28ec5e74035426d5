// Strong-form (PINN collocation) training step on tcgen05: the network at
// order 2 (network.hpp:204-282: five streams through every layer -- value
// V, tangents Tx, Ty, second derivatives Sx = d2/dx2, Sy = d2/dy2), the
// pointwise residual P = -eps (u_xx + u_yy) + b . grad u - f at the interior
// points (strong_residual_loss, losses.hpp:422-467), the boundary / sensor
// penalties (losses.hpp:406-415) and the order-2 reverse sweep
// (network.hpp:287-372, the s1 / s2 / s3 terms).  Same machinery as
// tc2_step_kernel.cuh (its header explains the fp16 two-part split, the
// power-of-two scales from rigorous bounds and the TMEM-resident parameter
// gradient), with five streams instead of three:
//   forward      D_s[p][o] = X_s[p][:] . W[o][:]        s = V, Tx, Ty, Sx, Sy
//   propagation  D_s[p][i] = G_s[p][:] . W[:][i]
//   param grad   Wbar[o][i] = sum_{s,p} G_s[p][o] X_s[p][i]   (K = 5 streams x 128 points)
// 256 threads (point p = t % 128, units [16 g, +16), g = t / 128), 128-point
// tiles, one CTA per SM (two 80 KB operand buffers, 512 TMEM columns).
//
// Second-order bounds (on top of tc2's first-order ones; s1max = 1):
//   hidden 1      |TA| <= max |w0|, T2A = 0
//   hidden h      |TX_h| <= |TA_h|, |T2X_h| <= s2max |TA_h|^2 + |T2A_h|
//   MMA layer h   |TA_{h+1}| <= R_h |TX_h|, |T2A_{h+1}| <= R_h |T2X_h|
//   reverse       |G_A| <= |Xbar| + 2 s2max |TA| |TZbar| + 2 s3max |TA|^2 |T2Zbar|
//                          + 2 s2max |T2A| |T2Zbar|,
//                 |G_T| <= |TZbar| + 2 s2max |TA| |T2Zbar|,  |G_S| <= |T2Zbar|,
//                 through W^T with the column abs-sums C_h
// (tanh: s2max = 4 / (3 sqrt 3) < 0.77, s3max = 2; sigmoid: < 0.097, 1/8).
// The forward state of hidden layer h that the reverse needs (TA, T2A of
// its pre-activation) stays in TMEM: MMA layer l writes its accumulators to
// its own column block, so layer 1's block survives layer 2.
#pragma once

#include <type_traits>

#include "tc2_step_kernel.cuh"

namespace vpg {
namespace s2 {

constexpr int NS = 5;                // streams
constexpr int kNT = 256;
constexpr int kMP = 128;             // points per tile
constexpr int kPart = kMP * 64;      // [128][32] fp16 tile
constexpr int kStream = 2 * kPart;   // h | l parts
constexpr int kBuf = NS * kStream;   // 80 KB
constexpr int kWL = 4096;            // W of one MMA layer: h rows 0..31 | l rows 32..63
constexpr uint32_t kCols = 512;
constexpr int kDBlk = NS * 32;       // accumulator block of one MMA layer (layer l at 160 (l - 1))
constexpr int kG0 = 320;             // parameter-gradient accumulators (M = 64: layer l at lane offset 16 (l - 1))
constexpr int kZ1 = 384, kZ2 = 416, kZ0 = 448;  // z of hidden 1, hidden 2 (D = 3), the last hidden layer
constexpr float kOneBias = 20.0f;

// exchange rows ([row][128] floats)
enum : int {
  kU = 0,         // u, ux, uy, uxx, uyy (5)
  kPu = 5,        // unit group 1's output partials (5)
  kUb = 10,       // output adjoints ub, uxb, uyb, usb (uxxb = uyyb) (4)
  kRows = 14
};
// per-warp running sums of the CUDA-core gradients
enum : int { kAW0x = 0, kAW0y = 16, kAB0 = 32, kAWd = 48, kAccW = 64 };
// S_MAX words: tile maxima |ub|, max(|uxb|, |uyb|), |usb|; weight norms
enum : int { kMb = 0, kMt = 1, kMs = 2, kNW0 = 3, kNLayer = 6 };

template <int D>
struct Lay {
  static constexpr int NL = D - 1;
  static constexpr int OFF_A = 8192;  // W tiles (<= 2 x 4 KB); buffers 1024-aligned
  static constexpr int OFF_B = OFF_A + kBuf;
  static constexpr int OFF_SMALL = OFF_B + kBuf;
  // small region, in floats
  static constexpr int S_W0 = 0;               // [32][4] (w_x, w_y, b, 0)
  static constexpr int S_W0T = S_W0 + 128;     // [16][2][2] (w_x, w_y) x unit pair, * 2^kXt of X_1
  static constexpr int S_W0S = S_W0T + 64;     // [16][2][2] (w_x^2, w_y^2) x unit pair, * 2^kXs of X_1
  static constexpr int S_BIAS = S_W0S + 64;    // [2][32]
  static constexpr int S_WD = S_BIAS + 64;     // [32] + output bias at 32 (40)
  static constexpr int S_EX = S_WD + 40;       // [kRows][128]
  static constexpr int S_ACC = S_EX + kRows * 128;  // [8 warps][kAccW]
  static constexpr int S_RED = S_ACC + 8 * kAccW;   // [8 warps][5] doubles
  static constexpr int S_SC = S_RED + 80;      // floats, see kSc*
  static constexpr int S_SCI = S_SC + 48;      // ints, see kSi*
  static constexpr int S_MAX = S_SCI + 16;     // [16] uint
  static constexpr int S_BAR = S_MAX + 16;     // 4 mbarriers + TMEM slot
  static constexpr int S_END = S_BAR + 12;
  static constexpr size_t BYTES = (size_t)OFF_SMALL + sizeof(float) * S_END;
  static_assert(S_RED % 2 == 0 && S_BAR % 2 == 0 && S_W0T % 4 == 0 && S_W0S % 4 == 0, "alignment");
};
// float constants: per MMA layer l (0-based): forward unscales of the V / T /
// S streams, store scales of X_{l+1}; per hidden h (1-based, <= 3): bounds
enum : int {
  kScFv = 0,    // [2]
  kScFt = 2,    // [2]
  kScFs = 4,    // [2]
  kScXv = 6,    // [3] store scale 2^kXv of X_h (h = 1..D-1 are MMA inputs; index h - 1)
  kScXt = 9,    // [3]
  kScXs = 12,   // [3]
  kScBTA = 15,  // [4] |TA| bound of hidden h (index h)
  kScBT2A = 19, // [4] |T2A| bound of hidden h
  kScC = 23,    // [2] max column abs-sum of W_l
  kScWd = 25,   // max |wd|
  kScN = 26
};
enum : int { kSiW = 0, kSiXv = 2, kSiXt = 4, kSiXs = 6, kSiN = 8 };

template <int ACT>
struct Deriv;
// s1, s2 (and s3) of two units at once in packed fp32x2 (ActDerivs::fill,
// network.hpp:171-192, from the activation output z)
template <>
struct Deriv<kActTanh> {
  static constexpr float s2max = 0.77f, s3max = 2.0f;
  static __device__ __forceinline__ void d(float z, float& s1, float& s2, float& s3) {
    s1 = fmaf(-z, z, 1.0f);
    s2 = -2.0f * z * s1;
    s3 = s1 * (4.0f * (z * z) - 2.0f * s1);
  }
  static __device__ __forceinline__ void d12(float2 z, float2& s1, float2& s2) {
    s1 = fma2(f2(-z.x, -z.y), z, f2s(1.0f));
    s2 = mul2(mul2(f2s(-2.0f), z), s1);
  }
  static __device__ __forceinline__ void d123(float2 z, float2& s1, float2& s2, float2& s3) {
    d12(z, s1, s2);
    s3 = mul2(s1, fma2(f2s(4.0f), mul2(z, z), mul2(f2s(-2.0f), s1)));
  }
};
template <>
struct Deriv<kActSigmoid> {
  static constexpr float s2max = 0.1f, s3max = 0.15f;
  static __device__ __forceinline__ void d(float z, float& s1, float& s2, float& s3) {
    s1 = z * (1.0f - z);
    s2 = s1 * (1.0f - 2.0f * z);
    s3 = s1 * (1.0f - 6.0f * z + 6.0f * (z * z));
  }
  static __device__ __forceinline__ void d12(float2 z, float2& s1, float2& s2) {
    s1 = mul2(z, add2(f2s(1.0f), f2(-z.x, -z.y)));
    s2 = mul2(s1, fma2(f2s(-2.0f), z, f2s(1.0f)));
  }
  static __device__ __forceinline__ void d123(float2 z, float2& s1, float2& s2, float2& s3) {
    d12(z, s1, s2);
    s3 = mul2(s1, fma2(f2s(6.0f), mul2(z, z), fma2(f2s(-6.0f), z, f2s(1.0f))));
  }
};

// parameter-gradient GEMM: NS streams x 8 point blocks of K = 16
__device__ __forceinline__ void issue_param5(uint32_t acc, uint64_t da, uint64_t db, uint32_t idesc, int first,
                                             int shift, uint64_t* bar) {
  if (tc::elect_one()) {  // one elect for the group (tc2_step_kernel.cuh VPG_MMA_ELECT1)
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
#pragma unroll
      for (int kp = 0; kp < kMP / 16; ++kp) {
        const uint64_t off = (uint64_t)((s * kStream + 1024 * kp) >> 4);
        const uint64_t ad = da + off, bd = db + off;
        if (s == 0 && kp == 0 && !first && shift > 0)
          tc::mma_f16_sd(acc, ad, bd, idesc, shift);
        else
          tc::mma_bf16(acc, ad, bd, idesc, (s == 0 && kp == 0 && first) ? 0u : 1u);
      }
    }
    tc::mma_commit(bar);
  }
  __syncwarp();
}

}  // namespace s2

// MODE: kModeFused (loss + gradient parts of one epoch) or kModeForward
// (order-2 evaluate over a.fwd_pts: u, ux, uy, uxx, uyy to a.out_*)
template <int H, int D, int ACT, int MODE = kModeFused>
__global__ void __maxnreg__(255) sf2_step_kernel(const StepArgs a) {
  using namespace s2;
  static_assert(H <= 31 && (D == 2 || D == 3), "sf2 step: H <= 31, 2 or 3 hidden layers");
  using LY = Lay<D>;
  constexpr int NL = LY::NL;
  using AC = Act<ACT>;
  using DV = Deriv<ACT>;
#if !VPG_PDL_LATE
  pdl_trigger();
#endif
  pdl_wait();
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  extern __shared__ __align__(1024) char s2_raw[];
  if ((smem_u32(s2_raw) & 1023u) != 0u) __trap();
  char* sm = s2_raw;
  char* sWB = sm;
  char* bufA = sm + LY::OFF_A;
  char* bufB = sm + LY::OFF_B;
  float* sf = reinterpret_cast<float*>(sm + LY::OFF_SMALL);
  float* sW0 = sf + LY::S_W0;
  float* sW0t = sf + LY::S_W0T;
  float* sW0s = sf + LY::S_W0S;
  float* sBias = sf + LY::S_BIAS;
  float* sWd = sf + LY::S_WD;
  float* sEx = sf + LY::S_EX;
  float* sAcc = sf + LY::S_ACC;
  double* sRed = reinterpret_cast<double*>(sf + LY::S_RED);
  float* sSc = sf + LY::S_SC;
  int* sSci = reinterpret_cast<int*>(sf + LY::S_SCI);
  uint32_t* sMax = reinterpret_cast<uint32_t*>(sf + LY::S_MAX);
  uint64_t* bar_v = reinterpret_cast<uint64_t*>(sf + LY::S_BAR);
  uint64_t* bar_t = bar_v + 1;
  uint64_t* bar_w = bar_v + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar_v + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = tid & 127;
  const int ug = tid >> 7;
  const int u0 = 16 * ug;
  const NetDesc& net = a.net;
  const float* P = a.params;

  // ---------------- one-time setup (as tc2_step_kernel) ----------------
  if (warp == 0) tc::tmem_alloc(tslot, kCols);
  if (tid == 0) {
    mbar_init(bar_v, 1);
    mbar_init(bar_t, NS - 1);
    mbar_init(bar_w, 1);
    fence_mbar_init();
  }
  if (tid < 16) sMax[tid] = 0u;
  for (int i = tid; i < 8 * kAccW; i += kNT) sAcc[i] = 0.f;
  const int wl = tid >> 7, wo = (tid >> 2) & 31, wc = tid & 3;
  float wv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = 8 * wc + k;
    const int fo = wl < NL ? net.out_w[wl + 1] : 0, fi = wl < NL ? net.in_w[wl + 1] : 0;
    wv[k] = (wo < fo && i < fi) ? P[net.w_off[wl + 1] + wo * fi + i] : 0.f;
  }
  for (int i = tid; i < 32; i += kNT) {
    float w0 = 0.f, w1 = 0.f, b = (i == H) ? kOneBias : 0.f, wd = 0.f;
    if (i < net.out_w[0]) {
      w0 = P[net.w_off[0] + 2 * i];
      w1 = P[net.w_off[0] + 2 * i + 1];
      b = P[net.b_off[0] + i];
    }
    if (i < net.in_w[D]) wd = P[net.w_off[D] + i];
    sW0[4 * i] = w0;
    sW0[4 * i + 1] = w1;
    sW0[4 * i + 2] = b;
    sW0[4 * i + 3] = 0.f;
    sWd[i] = wd;
  }
  if (tid == 0) sWd[32] = P[net.b_off[D]];
  for (int l = 1; l <= NL; ++l)
    for (int o = tid; o < 32; o += kNT)
      sBias[(l - 1) * 32 + o] = o < net.out_w[l] ? P[net.b_off[l] + o] : ((o == H) ? kOneBias : 0.f);
  float* sAbs = reinterpret_cast<float*>(bufA);  // [NL][32][33]
  uint32_t* sNorm = sMax + kNW0;
  uint32_t(*s_lnorm)[3] = reinterpret_cast<uint32_t(*)[3]>(sMax + kNLayer);
  if (wl < NL) {
#pragma unroll
    for (int k = 0; k < 8; ++k) sAbs[(wl * 32 + wo) * 33 + 8 * wc + k] = fabsf(wv[k]);
  }
  __syncthreads();
  if (wl < NL) {
    float m = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) m = fmaxf(m, fabsf(wv[k]));
    t2::atomic_max_abs(&s_lnorm[wl][0], m);
  }
  if (tid < H) {
    t2::atomic_max_abs(&sNorm[0], sW0[4 * tid]);
    t2::atomic_max_abs(&sNorm[1], sW0[4 * tid + 1]);
    t2::atomic_max_abs(&sNorm[2], sWd[tid]);
  }
  if (tid < 64 * NL) {
    const int l = tid >> 6, j = tid & 31;
    const bool row = (tid & 32) == 0;
    float sum = 0.f;
    if (j < H)
      for (int k = 0; k < H; ++k) sum += row ? sAbs[(l * 32 + j) * 33 + k] : sAbs[(l * 32 + k) * 33 + j];
    t2::atomic_max_abs(&s_lnorm[l][row ? 1 : 2], sum);
  }
  __syncthreads();
  if (tid == 0) {
    // forward bounds of hidden h = 1..D: pre-activation TA / T2A
    float bta = fmaxf(__uint_as_float(sNorm[0]), __uint_as_float(sNorm[1])), bt2a = 0.f;
    for (int h = 1; h <= D; ++h) {
      sSc[kScBTA + h] = bta;
      sSc[kScBT2A + h] = bt2a;
      const float btx = bta, bt2x = DV::s2max * bta * bta + bt2a;  // |TX_h|, |T2X_h|
      if (h <= NL) {
        const int l = h - 1;  // MMA layer h, 0-based l; its input X_h
        const int kw = t2::clamp_exp(14 - tc::bound_exp(__uint_as_float(s_lnorm[l][0])));
        const int kxv = t2::clamp_exp(14 - tc::bound_exp(1.0f));
        const int kxt = t2::clamp_exp(14 - tc::bound_exp(btx));
        const int kxs = t2::clamp_exp(14 - tc::bound_exp(bt2x));
        sSci[kSiW + l] = kw;
        sSci[kSiXv + l] = kxv;
        sSci[kSiXt + l] = kxt;
        sSci[kSiXs + l] = kxs;
        sSc[kScFv + l] = tc::exp2i(-(kxv + kw));
        sSc[kScFt + l] = tc::exp2i(-(kxt + kw));
        sSc[kScFs + l] = tc::exp2i(-(kxs + kw));
        sSc[kScXv + l] = tc::exp2i(kxv);
        sSc[kScXt + l] = tc::exp2i(kxt);
        sSc[kScXs + l] = tc::exp2i(kxs);
        sSc[kScC + l] = __uint_as_float(s_lnorm[l][2]);
        const float R = __uint_as_float(s_lnorm[l][1]);
        bta = R * btx;
        bt2a = R * bt2x;
      }
    }
    sSc[kScWd] = __uint_as_float(sNorm[2]);
  }
  __syncthreads();
  for (int i = tid; i < 32; i += kNT) {  // layer-0 tangent / second-derivative weights, scaled for X_1
    const float wx = sW0[4 * i], wy = sW0[4 * i + 1];
    // unit pairs (k, k+1) adjacent per field: (wx_k, wx_k+1, wy_k, wy_k+1)
    const int pb = 4 * (i >> 1) + (i & 1);
    sW0t[pb] = wx * sSc[kScXt];
    sW0t[pb + 2] = wy * sSc[kScXt];
    sW0s[pb] = (wx * wx) * sSc[kScXs];
    sW0s[pb + 2] = (wy * wy) * sSc[kScXs];
  }
  if (wl < NL) tc::st_split8_h(sWB + wl * kWL, 32 * tc::kRowBytes, wo, wc, wv, tc::exp2i(sSci[kSiW + wl]));
  tc::fence_smem_to_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot;
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;
  const uint32_t sA = smem_u32(bufA), sB = smem_u32(bufB), sW = smem_u32(sWB);
  const uint32_t off0 = tc::sw_chunk(p, 2 * ug), off1 = tc::sw_chunk(p, 2 * ug + 1);
  const uint64_t dA_k = tc::kdesc(sA), dB_k = tc::kdesc(sB);
  const uint64_t dA_mn = tc::mndesc(sA, kPart), dB_mn = tc::mndesc(sB, kPart);
  const uint64_t dW_k = tc::kdesc(sW), dW_mn = tc::mndesc(sW, 32 * tc::kRowBytes);
  auto dblk = [&](int l) { return (uint32_t)(kDBlk * (l - 1)); };
  auto gacc = [&](int l) { return tmem + kG0 + ((uint32_t)(16 * (l - 1)) << 16); };
  // point GEMM of MMA layer l into its accumulator block: stream s by warp s
  auto issue_point_gemm = [&](bool bufb, int l, bool propagate) {
    const int s = warp;
    const uint64_t abase = (bufb ? dB_k : dA_k) + (uint64_t)((s * kStream) >> 4);
    const uint64_t wbase = (propagate ? dW_mn : dW_k) + (uint64_t)(((l - 1) * kWL) >> 4);
    const uint32_t idesc = tc::idesc_f16(128, 32, 0, propagate ? 1 : 0);
    t2::issue_point_stream<1>(tmem + dblk(l) + 32 * s, abase, wbase, idesc, propagate, kPart, kWL,
                              32 * tc::kRowBytes);
    tc::commit_warp(warp == 0 ? bar_v : bar_t);
  };
  auto issue_param_gemm = [&](int l, bool first, int shift) {
    issue_param5(gacc(l), dA_mn, dB_mn, tc::idesc_f16(64, 64, 1, 1), first ? 1 : 0, shift, bar_w);
  };
  uint32_t ph_v = 0, ph_t = 0, ph_w = 0;
  auto mma_wait = [&](uint64_t* b1, uint32_t& p1) {
    mbar_wait(b1, p1);
    p1 ^= 1u;
    tc::fence_after_sync();
  };
  auto operands_ready = [&]() {
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  };
  // this thread's 8 accumulator columns (chunk c) of stream s of MMA layer l's block
  auto dcol = [&](int l, int s, int c) { return tmem + lane_q + dblk(l) + 32 * s + u0 + 8 * c; };
  auto zcol = [&](int base, int c) { return tmem + lane_q + (uint32_t)base + u0 + 8 * c; };
  auto coff = [&](int c) { return c ? off1 : off0; };
  auto acc_units = [&](float (&v)[8], int slot, int c) {
    const float r = t2::warp_rs8(v);
    if ((lane & 3) == 0) sAcc[warp * kAccW + slot + 8 * c + t2::rs8_index(lane)] += r;
  };
  // five-stream store of 8 units (chunk c) into buffer buf with per-class scales
  // (SCALE = false: the values already carry their scales)
  auto store5 = [&](auto scale_tag, char* buf, int c, const float (&v)[8], const float (&tx)[8], const float (&ty)[8],
                    const float (&sx)[8], const float (&sy)[8], float scv, float sct, float scs) {
    constexpr bool SC = decltype(scale_tag)::value;
    const uint32_t o = coff(c);
    tc::st_split8_ho<SC>(buf, kPart, o, v, scv);
    tc::st_split8_ho<SC>(buf + kStream, kPart, o, tx, sct);
    tc::st_split8_ho<SC>(buf + 2 * kStream, kPart, o, ty, sct);
    tc::st_split8_ho<SC>(buf + 3 * kStream, kPart, o, sx, scs);
    tc::st_split8_ho<SC>(buf + 4 * kStream, kPart, o, sy, scs);
  };
  using kScaled = std::true_type;
  using kUnscaled = std::false_type;
  // X_1 of chunk c into buf: from (x, y) through layer 0 (z kept in TMEM),
  // or from that kept z (reverse)
  auto store_x1 = [&](char* buf, int c, float px, float py, bool from_tmem) {
    float z[8], tx[8], ty[8], sx[8], sy[8];
    if (from_tmem) {
      tc::tmem_ld1x8_wait(zcol(kZ1, c), z);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 w = *reinterpret_cast<const float4*>(sW0 + 4 * (u0 + 8 * c + k));
        z[k] = AC::value(fmaf(w.y, py, w.x * px) + w.z);
      }
      tc::tmem_st1x8_wait(zcol(kZ1, c), z);
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      float2 a1, a2;
      DV::d12(f2(z[k], z[k + 1]), a1, a2);
      const float4 wt = *reinterpret_cast<const float4*>(sW0t + 2 * (u0 + 8 * c + k));  // (wx, wy) of k, k+1
      const float4 ws = *reinterpret_cast<const float4*>(sW0s + 2 * (u0 + 8 * c + k));
      const float2 t1 = mul2(a1, f2(wt.x, wt.y)), t2 = mul2(a1, f2(wt.z, wt.w));
      const float2 q1 = mul2(a2, f2(ws.x, ws.y)), q2 = mul2(a2, f2(ws.z, ws.w));
      tx[k] = t1.x;
      tx[k + 1] = t1.y;
      ty[k] = t2.x;
      ty[k + 1] = t2.y;
      sx[k] = q1.x;
      sx[k + 1] = q1.y;
      sy[k] = q2.x;
      sy[k + 1] = q2.y;
    }
    tc::st_split8_ho<true>(buf, kPart, coff(c), z, sSc[kScXv]);
    tc::st_split8_ho<false>(buf + kStream, kPart, coff(c), tx, 1.f);
    tc::st_split8_ho<false>(buf + 2 * kStream, kPart, coff(c), ty, 1.f);
    tc::st_split8_ho<false>(buf + 3 * kStream, kPart, coff(c), sx, 1.f);
    tc::st_split8_ho<false>(buf + 4 * kStream, kPart, coff(c), sy, 1.f);
  };

  // per-CTA sums (thread-owned, combined in a fixed order at the end)
  double acc_v = 0.0, acc_b = 0.0, acc_s = 0.0, acc_eg = 0.0;
  int bad = 0;
  int kacc[2] = {0, 0};
  bool has[2] = {false, false}, spill[2] = {false, false};
  auto gacc_row = [&](int l) {
    const int lo = lane - 16 * (l - 1);
    return (lo >= 0 && lo < 16) ? 16 * (warp & 3) + lo : -1;
  };
  auto spill_accumulator = [&](int l, int ka, bool first) {
    float* S = a.tc_scratch + ((size_t)blockIdx.x * NL + (l - 1)) * (64 * 64);
    const float inv = tc::exp2i(-ka);
#pragma unroll 1
    for (int h2 = 0; h2 < 2; ++h2) {
      const int col0 = 32 * ug + 16 * h2;
      float v[16];
      tc::tmem_ld1x16_wait(tmem + lane_q + kG0 + col0, v);
      const int grow = gacc_row(l);
      if (grow >= 0) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          float* d = S + (col0 + k) * 64 + grow;
          *d = first ? v[k] * inv : fmaf(v[k], inv, *d);
        }
      }
    }
  };
  auto join_acc = [&](int l, int kp_nat, bool& first, int& shift) {
    const int i = l - 1;
    shift = 0;
    first = false;
    int kp = kp_nat;
    if (!has[i]) {
      first = true;
    } else if (a.tc_force_spill) {
      spill_accumulator(l, kacc[i], !spill[i]);
      spill[i] = true;
      first = true;
    } else if (kp_nat >= kacc[i]) {
      kp = kacc[i];
    } else if (kacc[i] - kp_nat <= 15) {
      shift = kacc[i] - kp_nat;
    } else {
      spill_accumulator(l, kacc[i], !spill[i]);
      spill[i] = true;
      first = true;
    }
    kacc[i] = kp;
    has[i] = true;
    return kp;
  };

  const int n_pts = MODE == kModeForward ? a.n_fwd : a.n_int + a.n_bnd + a.n_sen;
  const int n_tiles = (n_pts + kMP - 1) / kMP;
  const bool conv = a.bx != 0.f || a.by != 0.f;
  const float e_val = a.eps_source == 1 ? P[net.scal_off + a.eps_scalar_index] : a.eps;
  auto load_xy = [&](int tile, float& x, float& y) {
    x = 0.f;
    y = 0.f;
    const int gp = tile * kMP + p;
    if (tile < n_tiles && gp < n_pts) {
      const float2 xy = MODE == kModeForward ? a.fwd_pts[gp] : a.pts[gp];
      x = xy.x;
      y = xy.y;
    }
  };
  float nx, ny;
  load_xy(blockIdx.x, nx, ny);

#pragma unroll 1
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int gp = tile * kMP + p;
    const bool valid = gp < n_pts;
    const float px = nx, py = ny;
    if (tid < 3) sMax[tid] = 0u;

    // =================== forward (network.hpp:204-282, order 2) ===================
    char* x1buf = (D == 3) ? bufA : bufB;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) store_x1(x1buf, c, px, py, false);
    operands_ready();
    if (warp < NS) issue_point_gemm(D == 2, 1, false);
    float ou[5] = {0.f, 0.f, 0.f, 0.f, 0.f};  // output-layer partials (last hidden)
#pragma unroll t2::kUL
    for (int l = 1; l <= NL; ++l) {
      const bool last = l == NL;
      const float fv = sSc[kScFv + l - 1], ft = sSc[kScFt + l - 1], fs = sSc[kScFs + l - 1];
      const float* bias = sBias + 32 * (l - 1);
      mma_wait(bar_v, ph_v);
      mma_wait(bar_t, ph_t);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float d[8], ax[8], ay[8], bx2[8], by2[8];
        tc::tmem_ld1x8_wait(dcol(l, 0, c), d);
        tc::tmem_ld2x8_wait(dcol(l, 1, c), dcol(l, 2, c), ax, ay);
        tc::tmem_ld2x8_wait(dcol(l, 3, c), dcol(l, 4, c), bx2, by2);
        float z[8], tx[8], ty[8], sx[8], sy[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const int u = u0 + 8 * c + k;
          const float2 zz = AC::value2(fma2(f2(d[k], d[k + 1]), f2s(fv), f2(bias[u], bias[u + 1])));
          float2 s1, s2v;
          DV::d12(zz, s1, s2v);
          const float2 tax = mul2(f2(ax[k], ax[k + 1]), f2s(ft)), tay = mul2(f2(ay[k], ay[k + 1]), f2s(ft));
          const float2 t2ax = mul2(f2(bx2[k], bx2[k + 1]), f2s(fs)), t2ay = mul2(f2(by2[k], by2[k + 1]), f2s(fs));
          const float2 vx = mul2(s1, tax), vy = mul2(s1, tay);
          const float2 wx = fma2(s2v, mul2(tax, tax), mul2(s1, t2ax)), wy = fma2(s2v, mul2(tay, tay), mul2(s1, t2ay));
          z[k] = zz.x;
          z[k + 1] = zz.y;
          tx[k] = vx.x;
          tx[k + 1] = vx.y;
          ty[k] = vy.x;
          ty[k + 1] = vy.y;
          sx[k] = wx.x;
          sx[k + 1] = wx.y;
          sy[k] = wy.x;
          sy[k + 1] = wy.y;
          if (last) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float w = sWd[u + e];
              ou[0] = fmaf(w, z[k + e], ou[0]);
              ou[1] = fmaf(w, tx[k + e], ou[1]);
              ou[2] = fmaf(w, ty[k + e], ou[2]);
              ou[3] = fmaf(w, sx[k + e], ou[3]);
              ou[4] = fmaf(w, sy[k + e], ou[4]);
            }
          }
        }
        if (!last) {
          store5(kScaled{}, bufB, c, z, tx, ty, sx, sy, sSc[kScXv + l], sSc[kScXt + l], sSc[kScXs + l]);
          tc::tmem_st1x8_wait(zcol(kZ2, c), z);  // hidden l + 1 = 2 (D == 3)
        } else {
          tc::tmem_st1x8_wait(zcol(kZ0, c), z);
        }
      }
      if (!last) {
        operands_ready();
        if (warp < NS) issue_point_gemm(true, l + 1, false);
      }
    }
    // output layer: halves combined in order (half 0 + half 1 (+ bias))
    if (ug == 1)
#pragma unroll
      for (int s = 0; s < 5; ++s) sEx[(kPu + s) * 128 + p] = ou[s];
    __syncthreads();
    if (ug == 0) {
      float o[5];
#pragma unroll
      for (int s = 0; s < 5; ++s) o[s] = ou[s] + sEx[(kPu + s) * 128 + p];
      o[0] += sWd[32];
      if (valid && !(finitef(o[0]) && finitef(o[1]) && finitef(o[2]) && finitef(o[3]) && finitef(o[4]))) bad = 1;
      if (MODE == kModeForward && valid) {
        if (a.out_u) a.out_u[gp] = o[0];
        if (a.out_ux) a.out_ux[gp] = o[1];
        if (a.out_uy) a.out_uy[gp] = o[2];
        if (a.out_uxx) a.out_uxx[gp] = o[3];
        if (a.out_uyy) a.out_uyy[gp] = o[4];
      }
      // =================== objective (trainer.hpp:246-266) ===================
      float ub = 0.f, uxb = 0.f, uyb = 0.f, usb = 0.f;
      if (MODE == kModeFused && valid) {
        if (gp < a.n_int) {
          // strong_residual_loss, losses.hpp:446-466
          const float lap = o[3] + o[4];
          const float Pv = __fsub_rn(__fadd_rn(__fadd_rn(__fmul_rn(-e_val, lap), __fmul_rn(a.bx, o[1])),
                                               __fmul_rn(a.by, o[2])),
                                     a.sforce[gp]);
          acc_v += (double)__fmul_rn(__fmul_rn(Pv, Pv), a.inv_ni);
          const float pbar = __fmul_rn(a.rscale_s, Pv);
          usb = __fmul_rn(-e_val, pbar);
          if (conv) {
            uxb = __fmul_rn(a.bx, pbar);
            uyb = __fmul_rn(a.by, pbar);
          }
          if (a.eps_source == 1) acc_eg += (double)__fmul_rn(-lap, pbar);
        } else if (gp < a.n_int + a.n_bnd) {
          const float dd = o[0] - a.bval[gp - a.n_int];
          acc_b += (double)(dd * dd);
          ub = a.bscale * dd;
        } else {
          const float dd = o[0] - a.sval[gp - a.n_int - a.n_bnd];
          acc_s += (double)(dd * dd);
          ub = a.sscale * dd;
        }
      }
      sEx[(kUb + 0) * 128 + p] = ub;
      sEx[(kUb + 1) * 128 + p] = uxb;
      sEx[(kUb + 2) * 128 + p] = uyb;
      sEx[(kUb + 3) * 128 + p] = usb;
      t2::atomic_max_abs(&sMax[kMb], ub);
      t2::atomic_max_abs(&sMax[kMt], fmaxf(fabsf(uxb), fabsf(uyb)));
      t2::atomic_max_abs(&sMax[kMs], usb);
    }
    load_xy(tile + gridDim.x, nx, ny);
    __syncthreads();
    if constexpr (MODE == kModeForward) continue;
    const float ub = sEx[(kUb + 0) * 128 + p], uxb = sEx[(kUb + 1) * 128 + p], uyb = sEx[(kUb + 2) * 128 + p],
                usb = sEx[(kUb + 3) * 128 + p];

    // =================== reverse (network.hpp:287-372, order 2) ===================
    const float Wd = sSc[kScWd];
    // adjoint bounds entering hidden D (after the output layer)
    float bXb = Wd * __uint_as_float(sMax[kMb]), bTZ = Wd * __uint_as_float(sMax[kMt]),
          bT2Z = Wd * __uint_as_float(sMax[kMs]);
    // G bounds at hidden h from its incoming adjoint bounds
    auto g_bounds = [&](int h, float xb, float tz, float t2z, float& bga, float& bgt, float& bgs) {
      const float bta = sSc[kScBTA + h], bt2a = sSc[kScBT2A + h];
      bga = xb + 2.f * DV::s2max * bta * tz + 2.f * DV::s3max * bta * bta * t2z + 2.f * DV::s2max * bt2a * t2z;
      bgt = tz + 2.f * DV::s2max * bta * t2z;
      bgs = t2z;
    };
    // G scales for param layer l (= hidden l + 1's G, MMA layer l's inputs X_l):
    // S_G,s = 2^(kP - kX_s), one product exponent kP
    struct GS {
      float v, t, s;     // store scales of the G streams
      float pv, pt, ps;  // propagation unscales
      bool first;
      int shift;
    };
    auto g_scales = [&](int l, float bga, float bgt, float bgs) {
      GS g;
      const int kxv = sSci[kSiXv + l - 1], kxt = sSci[kSiXt + l - 1], kxs = sSci[kSiXs + l - 1],
                kw = sSci[kSiW + l - 1];
      int kp = 1 << 20;
      const int ev = tc::bound_exp(bga), et = tc::bound_exp(bgt), es = tc::bound_exp(bgs);
      if (ev > -1000) kp = min(kp, 14 - ev + kxv);
      if (et > -1000) kp = min(kp, 14 - et + kxt);
      if (es > -1000) kp = min(kp, 14 - es + kxs);
      if (kp == (1 << 20)) kp = kxv;
      kp = join_acc(l, max(-120, min(120, kp)), g.first, g.shift);
      g.v = tc::exp2i(kp - kxv);
      g.t = tc::exp2i(kp - kxt);
      g.s = tc::exp2i(kp - kxs);
      g.pv = tc::exp2i(-(kp - kxv + kw));
      g.pt = tc::exp2i(-(kp - kxt + kw));
      g.ps = tc::exp2i(-(kp - kxs + kw));
      return g;
    };
    float bga, bgt, bgs;
    g_bounds(D, bXb, bTZ, bT2Z, bga, bgt, bgs);
    GS gsc = g_scales(NL, bga, bgt, bgs);
    // ---- output layer + the last hidden layer's G ----
    {
      const float ftl = sSc[kScFt + NL - 1], fsl = sSc[kScFs + NL - 1];
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float z[8], ax[8], ay[8], bx2[8], by2[8];
        tc::tmem_ld1x8_wait(zcol(kZ0, c), z);
        tc::tmem_ld2x8_wait(dcol(NL, 1, c), dcol(NL, 2, c), ax, ay);
        tc::tmem_ld2x8_wait(dcol(NL, 3, c), dcol(NL, 4, c), bx2, by2);
        float v[8], gA[8], gTx[8], gTy[8], gSx[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const int u = u0 + 8 * c + k;
          float2 s1, s2v, s3;
          const float2 zz = f2(z[k], z[k + 1]);
          DV::d123(zz, s1, s2v, s3);
          const float2 tax = mul2(f2(ax[k], ax[k + 1]), f2s(ftl)), tay = mul2(f2(ay[k], ay[k + 1]), f2s(ftl));
          const float2 t2ax = mul2(f2(bx2[k], bx2[k + 1]), f2s(fsl)), t2ay = mul2(f2(by2[k], by2[k + 1]), f2s(fsl));
          const float2 txv = mul2(s1, tax), tyv = mul2(s1, tay);
          const float2 sxy = add2(fma2(s2v, mul2(tax, tax), mul2(s1, t2ax)), fma2(s2v, mul2(tay, tay), mul2(s1, t2ay)));
          const float2 vv = fma2(f2s(ub), zz, fma2(f2s(uxb), txv, fma2(f2s(uyb), tyv, mul2(f2s(usb), sxy))));
          const float2 w = f2(sWd[u], sWd[u + 1]);
          const float2 xb = mul2(w, f2s(ub)), tzx = mul2(w, f2s(uxb)), tzy = mul2(w, f2s(uyb)), t2z = mul2(w, f2s(usb));
          const float2 tt = fma2(tax, tax, mul2(tay, tay));  // t2z is the same for x and y (u_xxbar = u_yybar)
          float2 ga = fma2(s1, xb, mul2(s2v, fma2(tax, tzx, mul2(tay, tzy))));
          ga = fma2(s3, mul2(tt, t2z), fma2(s2v, mul2(add2(t2ax, t2ay), t2z), ga));
          const float2 s2t = mul2(mul2(f2s(2.0f), s2v), t2z);
          const float2 gtx = fma2(s1, tzx, mul2(s2t, tax)), gty = fma2(s1, tzy, mul2(s2t, tay));
          const float2 gs = mul2(s1, t2z);
          const float2 ga2 = mul2(ga, f2s(gsc.v)), gtx2 = mul2(gtx, f2s(gsc.t)), gty2 = mul2(gty, f2s(gsc.t)),
                       gs2 = mul2(gs, f2s(gsc.s));
          v[k] = vv.x;
          v[k + 1] = vv.y;
          gA[k] = ga2.x;
          gA[k + 1] = ga2.y;
          gTx[k] = gtx2.x;
          gTx[k + 1] = gtx2.y;
          gTy[k] = gty2.x;
          gTy[k + 1] = gty2.y;
          gSx[k] = gs2.x;
          gSx[k + 1] = gs2.y;
        }
        acc_units(v, kAWd, c);
        store5(kUnscaled{}, bufA, c, gA, gTx, gTy, gSx, gSx, 1.f, 1.f, 1.f);
      }
    }
    operands_ready();
    if (warp < NS) issue_point_gemm(false, NL, true);
    if (warp == NS) issue_param_gemm(NL, gsc.first, gsc.shift);
    // ---- hidden layers, last-but-one first: G of hidden h from the propagated adjoints ----
#pragma unroll t2::kUL
    for (int h = NL; h >= 1; --h) {
      // incoming adjoint bounds at hidden h: through W_h^T
      const float C = sSc[kScC + h - 1];
      bXb = C * bga;
      bTZ = C * bgt;
      bT2Z = C * bgs;
      g_bounds(h, bXb, bTZ, bT2Z, bga, bgt, bgs);
      GS g2{1.f, 1.f, 1.f, 1.f, 1.f, 1.f, false, 0};
      if (h > 1) g2 = g_scales(h - 1, bga, bgt, bgs);
      mma_wait(bar_v, ph_v);
      mma_wait(bar_t, ph_t);
      // the pre-activation TA / T2A of hidden h: MMA layer h-1's block (h >= 2), or w0 / 0
      const float fth = h >= 2 ? sSc[kScFt + h - 2] : 1.f, fsh = h >= 2 ? sSc[kScFs + h - 2] : 1.f;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float pa[8], ptx[8], pty[8], psx[8], psy[8], z[8], ax[8], ay[8], bx2[8], by2[8];
        tc::tmem_ld1x8_wait(dcol(h, 0, c), pa);
        tc::tmem_ld2x8_wait(dcol(h, 1, c), dcol(h, 2, c), ptx, pty);
        tc::tmem_ld2x8_wait(dcol(h, 3, c), dcol(h, 4, c), psx, psy);
        tc::tmem_ld1x8_wait(zcol(h == 1 ? kZ1 : kZ2, c), z);
        if (h >= 2) {
          tc::tmem_ld2x8_wait(dcol(h - 1, 1, c), dcol(h - 1, 2, c), ax, ay);
          tc::tmem_ld2x8_wait(dcol(h - 1, 3, c), dcol(h - 1, 4, c), bx2, by2);
        }
        float gA[8], gTx[8], gTy[8], gSx[8], gSy[8];
        // G of hidden h, scaled for the store (h >= 2) or not (h == 1: the input layer)
        const float2 sv2 = f2s(h >= 2 ? g2.v : 1.f), st2 = f2s(h >= 2 ? g2.t : 1.f), ss2 = f2s(h >= 2 ? g2.s : 1.f);
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const int u = u0 + 8 * c + k;
          float2 s1, s2v, s3;
          DV::d123(f2(z[k], z[k + 1]), s1, s2v, s3);
          float2 tax, tay, t2ax = f2s(0.f), t2ay = f2s(0.f);
          if (h >= 2) {
            tax = mul2(f2(ax[k], ax[k + 1]), f2s(fth));
            tay = mul2(f2(ay[k], ay[k + 1]), f2s(fth));
            t2ax = mul2(f2(bx2[k], bx2[k + 1]), f2s(fsh));
            t2ay = mul2(f2(by2[k], by2[k + 1]), f2s(fsh));
          } else {
            tax = f2(sW0[4 * u], sW0[4 * u + 4]);
            tay = f2(sW0[4 * u + 1], sW0[4 * u + 5]);
          }
          const float2 xb = mul2(f2(pa[k], pa[k + 1]), f2s(gsc.pv));
          const float2 tzx = mul2(f2(ptx[k], ptx[k + 1]), f2s(gsc.pt)), tzy = mul2(f2(pty[k], pty[k + 1]), f2s(gsc.pt));
          const float2 t2zx = mul2(f2(psx[k], psx[k + 1]), f2s(gsc.ps)), t2zy = mul2(f2(psy[k], psy[k + 1]), f2s(gsc.ps));
          float2 ga = fma2(s1, xb, mul2(s2v, fma2(tax, tzx, mul2(tay, tzy))));
          ga = fma2(s3, fma2(mul2(tax, tax), t2zx, mul2(mul2(tay, tay), t2zy)),
                    fma2(s2v, fma2(t2ax, t2zx, mul2(t2ay, t2zy)), ga));
          const float2 s22 = mul2(f2s(2.0f), s2v);
          const float2 gtx = fma2(s1, tzx, mul2(s22, mul2(tax, t2zx)));
          const float2 gty = fma2(s1, tzy, mul2(s22, mul2(tay, t2zy)));
          const float2 a2 = mul2(ga, sv2), bx3 = mul2(gtx, st2), by3 = mul2(gty, st2);
          const float2 cx3 = mul2(mul2(s1, t2zx), ss2), cy3 = mul2(mul2(s1, t2zy), ss2);
          gA[k] = a2.x;
          gA[k + 1] = a2.y;
          gTx[k] = bx3.x;
          gTx[k + 1] = bx3.y;
          gTy[k] = by3.x;
          gTy[k + 1] = by3.y;
          gSx[k] = cx3.x;
          gSx[k + 1] = cx3.y;
          gSy[k] = cy3.x;
          gSy[k + 1] = cy3.y;
        }
        if (h == 1) {
          // input layer: W0bar += Abar x^T + TAxbar e_x^T + TAybar e_y^T, b0bar += Abar
          float v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fmaf(gA[k], px, gTx[k]);
          acc_units(v, kAW0x, c);
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fmaf(gA[k], py, gTy[k]);
          acc_units(v, kAW0y, c);
          acc_units(gA, kAB0, c);
        } else {
          if (c == 0) {
            mbar_wait(bar_w, ph_w);
            ph_w ^= 1u;
            tc::fence_after_sync();
          }
          store5(kUnscaled{}, bufA, c, gA, gTx, gTy, gSx, gSy, 1.f, 1.f, 1.f);
          store_x1(bufB, c, px, py, true);  // hidden-1 output rebuilt (h - 1 == 1)
        }
      }
      if (h > 1) {
        operands_ready();
        if (warp < NS) issue_point_gemm(false, h - 1, true);
        if (warp == NS) issue_param_gemm(h - 1, g2.first, g2.shift);
        gsc = g2;
      }
    }
    mma_wait(bar_w, ph_w);  // last param GEMM done: buffers A / B free
  }

  // =================== per-CTA outputs ===================
#if VPG_PDL_LATE
  pdl_trigger();
#endif
  if constexpr (MODE == kModeForward) {
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
      tc::fence_after_sync();
      tc::tmem_dealloc(tmem, kCols);
    }
    return;
  }
  float* scr = reinterpret_cast<float*>(bufA);  // [64][65]
  for (int l = 1; l <= NL; ++l) {
    const float* S = a.tc_scratch + ((size_t)blockIdx.x * NL + (l - 1)) * (64 * 64);
    tc::fence_after_sync();
    if (has[l - 1]) {
      const float inv = tc::exp2i(-kacc[l - 1]);
#pragma unroll 1
      for (int h2 = 0; h2 < 2; ++h2) {
        const int col0 = 32 * ug + 16 * h2;
        float v[16];
        tc::tmem_ld1x16_wait(tmem + lane_q + kG0 + col0, v);
        const int grow = gacc_row(l);
        if (grow >= 0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            float x = v[k] * inv;
            if (spill[l - 1]) x += S[(col0 + k) * 64 + grow];
            scr[grow * 65 + col0 + k] = x;
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    const int fo = net.out_w[l], fi = net.in_w[l];
    for (int e = tid; e < fo * (fi + 1); e += kNT) {
      const int o = e / (fi + 1), i = e - o * (fi + 1);
      const int cc = i < fi ? i : H;
      float g = 0.f;
      if (has[l - 1])
        g = ((scr[o * 65 + cc] + scr[o * 65 + 32 + cc]) + scr[(32 + o) * 65 + cc]) + scr[(32 + o) * 65 + 32 + cc];
      const int idx = (i < fi) ? net.w_off[l] + o * fi + i : net.b_off[l] + o;
      a.grad_part[(size_t)idx * a.part_stride + blockIdx.x] = g;
    }
    __syncthreads();
  }
  for (int u = tid; u <= H; u += kNT) {
    const int h2 = u >> 4, j = u & 15;
    float w0x = 0.f, w0y = 0.f, b0 = 0.f, wd = 0.f;
    for (int w = 4 * h2; w < 4 * h2 + 4; ++w) {
      const float* A = sAcc + w * kAccW;
      w0x += A[kAW0x + j];
      w0y += A[kAW0y + j];
      b0 += A[kAB0 + j];
      wd += A[kAWd + j];
    }
    if (u < H) {
      if (u < net.out_w[0]) {
        a.grad_part[(size_t)(net.w_off[0] + 2 * u) * a.part_stride + blockIdx.x] = w0x;
        a.grad_part[(size_t)(net.w_off[0] + 2 * u + 1) * a.part_stride + blockIdx.x] = w0y;
        a.grad_part[(size_t)(net.b_off[0] + u) * a.part_stride + blockIdx.x] = b0;
      }
      if (u < net.in_w[D]) a.grad_part[(size_t)(net.w_off[D] + u) * a.part_stride + blockIdx.x] = wd;
    } else {
      a.grad_part[(size_t)net.b_off[D] * a.part_stride + blockIdx.x] = wd;
    }
  }
  if (tid == 0)
    for (int e = net.scal_off; e < net.n_params; ++e) a.grad_part[(size_t)e * a.part_stride + blockIdx.x] = 0.f;
  const int any_bad = __syncthreads_or(bad);
  {
    double v[4] = {acc_v, acc_b, acc_s, acc_eg};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 4; ++k) sRed[warp * 5 + k] = v[k];
    __syncthreads();
    if (tid == 0) {
      double lv = 0, lb = 0, ls = 0, le = 0;
      for (int w = 0; w < kNT / 32; ++w) {
        lv += sRed[w * 5 + 0];
        lb += sRed[w * 5 + 1];
        ls += sRed[w * 5 + 2];
        le += sRed[w * 5 + 3];
      }
      double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
      lp[kLpVar] = lv;
      lp[kLpBnd] = lb;
      lp[kLpSen] = ls;
      lp[kLpEpsGrad] = le;
      lp[kLpBad] = any_bad ? 1.0 : 0.0;
      for (int w = kLpBad + 1; w < kLpWords; ++w) lp[w] = 0.0;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, kCols);
  }
}

template <int D>
__host__ __device__ constexpr size_t sf2_step_smem_bytes() {
  return s2::Lay<D>::BYTES;
}

}  // namespace vpg
