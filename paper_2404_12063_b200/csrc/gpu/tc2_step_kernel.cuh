// Tensor-core FastVPINNs training step, fp16 two-part split.
//
// Per-tile semantics: forward with x/y tangents (network.hpp:204-282), the
// Algorithm-3 contraction (losses.hpp:91-168) or the penalty terms
// (losses.hpp:406-415), and the reverse sweep (network.hpp:287-372), every
// hidden->hidden GEMM on tcgen05 (s = value / x-tangent / y-tangent stream):
//   forward      D_s[p][o] = X_s[p][:] . W[o][:]        M = 128 points, N = HP, K = HP
//   propagation  D_s[p][i] = G_s[p][:] . W[:][i]        M = 128 points, N = HP, K = HP (B MN-major)
//   param grad   Wbar[o][i] = sum_{s,p} G_s[p][o] X_s[p][i]
//                                                      M = 2 HP (G h | l), N = 2 HP (X h | l),
//                                                      K = 3 streams x MP points
//
// Width classes.  Hidden units (plus the constant-one bias unit at index H)
// are padded to HP = 32 NB, NB = 1 (H <= 31) or 2 (H <= 63, the paper's
// [2,50,50,50,1] gear network); every operand tile is [MP][32] fp16 in the
// 64-byte swizzle (tc_utils.cuh), a width of 64 is two such column blocks.
//   NB = 1: 256 threads, MP = 128 points per tile, 113 KB of shared memory
//           and 256 TMEM columns -> two CTAs per SM;
//   NB = 2: 512 threads, MP = 112 points per tile (the operand buffers of
//           128 points would not fit next to the weights), ~212 KB and all
//           512 TMEM columns -> one CTA per SM.  The point GEMMs still run
//           M = 128: rows MP..127 read whatever follows the tile and their
//           accumulator lanes are never read.
//
// Precision.  Every operand is scaled by a power of two and split into two
// fp16 parts (tc_utils.cuh st_split8_ho): 22 significant bits, three products
// Ah.Bh + Ah.Bl + Al.Bh per fp32 product, accumulated in fp32 in TMEM, i.e.
// fp32-faithful.  The scales are derived from rigorous magnitude BOUNDS, not
// from the data, so no reduction sits on the critical path:
//   weights W_l              max |W_l|                                 (per CTA)
//   value stream z           |z| <= 1 (tanh / sigmoid outputs, the constant-one bias column)
//   tangent streams TX_h     |TX_1| <= max|w0|, |TX_{h+1}| <= R_h |TX_h|, R_h = max row abs-sum
//                            of W_h (one bound for the x and y tangents)
//   adjoints (reverse)       from the tile maxima of (ub, uxb, uyb) through
//                            |s1| <= 1, |kap| <= 2 and the column abs-sums of W_h
// A loose bound costs nothing measurable: fp16 keeps 2^-24 absolute spacing
// below 2^-14, i.e. ~2^-38 of the bound.  The parameter-gradient GEMM sums
// three streams with different scales, so the G scales are chosen to make
// S_G,s * S_X,s one common power of two per tile; the accumulator stays in
// TMEM across the CTA's tiles (scale-input-d when a tile needs a smaller
// product scale, a per-CTA fp32 spill for drops beyond 2^15).
//
// Shape: thread t owns point p = t % 128 (its TMEM lane) and hidden units
// [16 g, +16), g = t / 128, processed in chunks of 8.  Every unit runs the
// same branch-free code: the constant-one (bias) column H is a unit with zero
// weights and bias 20 (act(20) == 1 exactly, act' == 0), padding units have
// zero weights.  Hidden layers D in {2, 3}, one output channel.  The slab (the
// tile's premultipliers, cp.async.bulk) aliases operand buffer A.
#pragma once

#include "step_kernel.cuh"
#include "tc_utils.cuh"

#ifndef VPG_TC2_UC
#define VPG_TC2_UC 1  // unroll of the per-chunk (8-unit) loops
#endif
#ifndef VPG_TC2_UL
#define VPG_TC2_UL 2  // unroll of the per-layer loops (2: the layer-specialised code measured 7% faster)
#endif
#ifndef VPG_MMA_ELECT1
#define VPG_MMA_ELECT1 1  // one elect per MMA group (0: one per MMA; 1 measured 1.6% faster, 18% less code)
#endif
#ifndef VPG_PDL_LATE
#define VPG_PDL_LATE 1  // PDL trigger after the tile loop (the epoch tail launches during the per-CTA outputs)
#endif
#ifndef VPG_KAP_FOLD
#define VPG_KAP_FOLD 1  // tanh: kap = -2 z with the -2 folded into a scalar factor (bit-identical)
#endif
#ifndef VPG_PHASE_CLOCK
#define VPG_PHASE_CLOCK 0  // build with -DVPG_PHASE_CLOCK=1 for tools/phase_clock.py
#endif

namespace vpg {
namespace t2 {

// per width class (H = the instantiated hidden width) and hidden units per
// thread (UPT = 16: the throughput layout; UPT = 8: twice the threads on the
// same tile, the latency layout for grids of at most one tile per SM)
template <int H, int UPT = 16>
struct Cfg {
  static constexpr int NB = (H + 1 + 31) / 32;  // 32-unit column blocks (bias unit included)
  static_assert(NB == 1 || NB == 2, "tc2 step: hidden width <= 63");
  static_assert(UPT == 16 || UPT == 8, "tc2 step: 8 or 16 units per thread");
  static constexpr int HP = 32 * NB;
  static constexpr int NCH = UPT / 8;            // 8-unit chunks per thread
  static constexpr int NG = HP / UPT;            // unit groups
  static constexpr int NT = 128 * NG;            // threads
  static_assert(NT <= 512, "tc2 step: at most 512 threads");
  static constexpr int MP = NB == 1 ? 128 : 112;  // points per tile
  static constexpr int kPart = MP * 64;          // [MP][32] fp16 tile
  static constexpr int kStream = 2 * NB * kPart;  // tiles (part, block): part h blocks | part l blocks
  static constexpr int kBuf = 3 * kStream;       // 3 streams
  static constexpr int kWTile = 2 * HP * 64;     // W of one MMA layer and input block: h rows | l rows
  static constexpr int kWL = NB * kWTile;        // W of one MMA layer
  static constexpr uint32_t kCols = NB == 1 ? 256u : 512u;  // TMEM columns per CTA
  static constexpr bool kZCache = NB == 1;       // hidden-1 / hidden-2 z kept in TMEM
  static constexpr int kScratch = 4 * HP * HP;   // per-CTA fp32 spill [2HP][2HP] per MMA layer
  static constexpr int kMaxReg = 128;  // 2 x 256 or 1 x 512 threads: the whole register file
};

constexpr int kUC = VPG_TC2_UC;
constexpr int kUL = VPG_TC2_UL;
// contraction scratch after the slab in buffer A, [rows][128]: 0 bx ux + by uy,
// 4 rbar, 5 r^2, 6 rbar (gx + gy); two outputs also 1 eps, 2 y1, 3 eps ux,
// 7 eps uy, 8 y1bar, 8 + g the y1 partial of unit group g (all live between
// the forward's output layer and the reverse's first operand store)
template <int C>
constexpr int tail_floats() { return (C == 2 ? 12 : 8) * 128; }
constexpr int kTailFloats = tail_floats<1>();
enum : int { kTE = 1, kTY1 = 2, kTSx = 3, kTSy = 7, kTY1b = 8, kTY1p = 8 };
constexpr float kOneBias = 20.0f;     // bias of the constant-one unit: act(20) == 1.0f

// exchange rows ([row][128] floats).  The output-layer partials of unit
// group 1 (u, ux, uy) alias the adjoint rows, which are written only later;
// groups 2, 3 (NB = 2) have their own rows after kRows.
enum : int { kX = 0, kY, kU, kUx, kUy, kUb, kUxb, kUyb, kRows };
constexpr int kPu = kUb;

// per-warp running sums of the CUDA-core gradients: W0x | W0y | b0 | Wd (16 units each)
// (two outputs: Wd of channel 1 at kAWd2)
enum : int { kAW0x = 0, kAW0y = 16, kAB0 = 32, kAWd = 48, kAWd2 = 64 };
template <int C>
constexpr int acc_w() { return C == 2 ? 80 : 64; }

// uniform constants (floats in S_SC)
enum : int {
  kScF0 = 0,   // [2] value-stream forward unscale 2^-(kXv + kW) of MMA layer l
  kScF1 = 2,   // [2] tangent-stream forward unscale 2^-(kXt + kW)
  kScSv = 4,   // [2] value-stream scale 2^kXv of X_l (input of MMA layer l)
  kScSt = 6,   // [2] tangent-stream scale 2^kXt
  kScIt = 8,   // [2] 2^-kXt
  kScIv = 10,  // [2] 2^-kXv
  kScBt = 12,  // [4] tangent bounds of hidden 1..D outputs
  kScC = 16,   // [2] max column abs-sum of W_l
  kScWd = 18,  // max |wd|
  kScWd2 = 19,  // max |wd| of output channel 1 (two outputs)
  kScN = 20
};
// integer exponents (ints in S_SCI): kW[2], kXv[2], kXt[2]
enum : int { kSiW = 0, kSiXv = 2, kSiXt = 4, kSiN = 6 };

template <int H, int D, int C = 1, int UPT = 16>
struct Lay {
  using CF = Cfg<H, UPT>;
  static constexpr int NL = D - 1;
  static constexpr int HP = CF::HP;
  static constexpr int OFF_A = (NL * CF::kWL + 1023) & ~1023;  // W tiles first; buffers 1024-aligned
  static constexpr int OFF_B = OFF_A + CF::kBuf;
  static constexpr int OFF_SMALL = OFF_B + CF::kBuf;
  static constexpr int EX_ROWS = kRows + 3 * (CF::NG - 2);
  // small region, in floats
  static constexpr int S_W0 = 0;                       // [HP/2][4][2] unit pairs: (w_x, w_y, b, 0) x (k, k+1)
  static constexpr int S_W0S = S_W0 + 4 * HP;          // [HP/2][2][2] (w_x, w_y) x (k, k+1), * 2^kXt of X_1
  static constexpr int S_BIAS = S_W0S + 2 * HP;        // [2][HP]
  // output weights: channel 0 [HP], biases at HP, HP + 1; channel 1 at HP + 8
  static constexpr int S_WD = S_BIAS + 2 * HP;
  static constexpr int S_EX = S_WD + 2 * HP + 8;       // [EX_ROWS][128]
  static constexpr int S_ACC = S_EX + EX_ROWS * 128;   // [warps][acc_w<C>()]
  static constexpr int S_RED = S_ACC + (CF::NT / 32) * acc_w<C>();  // 2 * warps doubles
  static constexpr int S_SC = S_RED + 2 * 2 * (CF::NT / 32);   // [kScN] floats
  static constexpr int S_SCI = S_SC + kScN;            // [kSiN] ints
  static constexpr int S_MAX = S_SCI + kSiN;           // [16] uint: tile maxima, weight norms
  static constexpr int S_BAR = S_MAX + 16;             // 4 mbarriers + TMEM slot
  static constexpr int S_END = S_BAR + 12;
  static constexpr size_t BYTES = (size_t)OFF_SMALL + sizeof(float) * S_END;
  static_assert(S_RED % 2 == 0 && S_BAR % 2 == 0 && S_W0 % 4 == 0 && S_W0S % 4 == 0, "alignment");
  // TMEM columns: 0 .. 3 HP: stream accumulators; kG0: parameter-gradient
  // accumulators (NB = 1: M = 64, layer l in lanes 16 (l - 1) .. + 15 of every
  // lane quarter, both layers in the same 64 columns; NB = 2: M = 128, 128
  // columns per layer); kZ0: the last hidden layer's z; NB = 1 also keeps the
  // hidden-1 (kZ1) and hidden-2 (kZ2, D == 3) z from the forward for the reverse
  static constexpr int kG0 = 3 * HP;
  static constexpr int kZ0 = CF::NB == 1 ? 224 : kG0 + 128 * NL;
  static constexpr int kZ1 = 192;
  static constexpr int kZ2 = 160;
  static_assert(CF::NB == 2 || kG0 + 64 <= kZ2, "TMEM map");
  static_assert(kZ0 + HP <= (int)CF::kCols, "TMEM columns");
};

// S_MAX words: tile maxima of |ub|, |uxb|, |uyb|; max |w0x|, |w0y|, |wd|; per MMA
// layer (max |W|, max row abs-sum, max column abs-sum); two outputs: max |wd|
// of channel 1, tile maximum of |y1bar|
enum : int { kMb = 0, kMx = 1, kMy = 2, kNW0 = 3, kNLayer = 6, kNWd2 = 12, kMe = 13 };

// 8-value butterfly reduce-scatter over the warp's 32 lanes: afterwards lane
// l holds the sum over all lanes of value index ((l>>4)&1)*4 + ((l>>3)&1)*2 +
// ((l>>2)&1) (lanes l, l^1, l^2, l^3 agree).  Fixed order: deterministic.
__device__ __forceinline__ float warp_rs8(float (&v)[8]) {
  const int lane = threadIdx.x & 31;
  {
    const bool b = lane & 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float send = b ? v[j] : v[j + 4], keep = b ? v[j + 4] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  {
    const bool b = lane & 8;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float send = b ? v[j] : v[j + 2], keep = b ? v[j + 2] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  float r;
  {
    const bool b = lane & 4;
    const float send = b ? v[0] : v[1], keep = b ? v[1] : v[0];
    r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}
__device__ __forceinline__ int rs8_index(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }

__device__ __forceinline__ void atomic_max_abs(uint32_t* w, float v) {
  atomicMax(w, __float_as_uint(fabsf(v)));  // non-negative floats order as their bits (NaN: largest)
}
__device__ __forceinline__ int clamp_exp(int k) { return max(-60, min(60, k)); }

// point GEMM of one stream (called by a whole converged warp): the three part
// products Al.Wh, Ah.Wl, Ah.Wh into D, K = HP in steps of 16.  ablk: byte
// stride between the K blocks of A (= kPart; A part l at NB blocks); forward:
// B K-major, K block kb in W tile kb (wblk = kWTile), K step of 16 = +32 B;
// propagation: B MN-major (N across the W tiles via the descriptor's LBO),
// K step of 16 W rows = +1024 B.
template <int NB>
__device__ __forceinline__ void issue_point_stream(uint32_t d, uint64_t abase, uint64_t wbase, uint32_t idesc,
                                                   bool propagate, uint32_t kpart, uint32_t wtile, uint32_t wpart) {
#if VPG_MMA_ELECT1
  if (tc::elect_one()) {
#endif
#pragma unroll
  for (int pr = 0; pr < 3; ++pr) {
    const int pa = pr == 0 ? 1 : 0, pb = pr == 1 ? 1 : 0;
#pragma unroll
    for (int ks = 0; ks < 2 * NB; ++ks) {
      const uint32_t kb = ks >> 1, kin = ks & 1;
      const uint64_t ad = abase + (uint64_t)(((pa * NB + kb) * kpart + 32 * kin) >> 4);
      const uint32_t boff = propagate ? pb * wpart + 1024u * ks : pb * wpart + kb * wtile + 32u * kin;
#if VPG_MMA_ELECT1
      tc::mma_bf16(d, ad, wbase + (uint64_t)(boff >> 4), idesc, (pr > 0 || ks > 0) ? 1u : 0u);
#else
      tc::mma_warp(d, ad, wbase + (uint64_t)(boff >> 4), idesc, (pr > 0 || ks > 0) ? 1u : 0u);
#endif
    }
  }
#if VPG_MMA_ELECT1
  }
  __syncwarp();
#endif
}
// parameter-gradient GEMM: 3 streams x (MP / 16) point blocks of K = 16 into acc
template <int MP>
__device__ __forceinline__ void issue_param(uint32_t acc, uint64_t da, uint64_t db, uint32_t idesc, int first,
                                            int shift, uint64_t* bar, uint32_t kstream) {
#if VPG_MMA_ELECT1
  if (tc::elect_one()) {
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
#pragma unroll
      for (int kp = 0; kp < MP / 16; ++kp) {
        const uint64_t off = (uint64_t)((s * kstream + 1024 * kp) >> 4);
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
#else
#pragma unroll 1
  for (int s = 0; s < 3; ++s) {
#pragma unroll
    for (int kp = 0; kp < MP / 16; ++kp) {
      const uint64_t off = (uint64_t)((s * kstream + 1024 * kp) >> 4);
      const uint64_t ad = da + off, bd = db + off;
      if (s == 0 && kp == 0) {
        if (first)
          tc::mma_warp(acc, ad, bd, idesc, 0u);
        else if (shift > 0)
          tc::mma_warp_sd(acc, ad, bd, idesc, shift);
        else
          tc::mma_warp(acc, ad, bd, idesc, 1u);
      } else {
        tc::mma_warp(acc, ad, bd, idesc, 1u);
      }
    }
  }
  tc::commit_warp(bar);
#endif
}

}  // namespace t2

// MODE (step_kernel.cuh): kModeFused = the whole epoch on whole-cell tiles;
// kModeForward = forward over a.fwd_pts, (u, ux, uy) to a.out_*;
// kModeReverse = forward recompute + reverse from the adjoints in a.in_*
// (the split path of cells larger than a tile: forward -> contraction ->
// penalty -> reverse)
template <int H, int D, int ACT, int MODE = kModeFused, int C = 1, int UPT = 16>
__global__ void __maxnreg__((t2::Cfg<H, UPT>::kMaxReg)) tc2_step_kernel(const StepArgs a) {
  using namespace t2;
  static_assert(D == 2 || D == 3, "tc2 step: 2 or 3 hidden layers");
  static_assert(C == 1 || C == 2, "tc2 step: one output, or two (spatial-eps head)");
  using CF = Cfg<H, UPT>;
  using LY = Lay<H, D, C, UPT>;
  constexpr int NCH = CF::NCH;
  constexpr int kAccW = acc_w<C>();
  constexpr int NL = LY::NL;
  constexpr int NB = CF::NB, HP = CF::HP, NT = CF::NT, MP = CF::MP;
  constexpr int kPart = CF::kPart, kStream = CF::kStream;
  // contraction threads per row / per point: all of them when the CTA is
  // alone on its SM (NB = 2); one (unit group 0) when two CTAs share the SM,
  // whose other CTA fills the idle issue slots (splitting measured slower)
  constexpr int kCS = NT >= 512 ? NT / 128 : 1;
  using AC = Act<ACT>;

#if !VPG_PDL_LATE
  pdl_trigger();
#endif
  pdl_wait();
  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;
  if constexpr (VPG_PHASE_CLOCK != 0) {  // entry clocks (diagnostics)
    if (a.phase_clk != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
      a.phase_clk[kPhaseTiles * kPhaseMarks - 1] = clock64();
    if (a.phase_clk != nullptr && threadIdx.x == 0 && blockIdx.x < 1024) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.phase_clk[kPhaseTiles * kPhaseMarks + 3 * blockIdx.x] = (long long)globaltimer();
      a.phase_clk[kPhaseTiles * kPhaseMarks + 3 * blockIdx.x + 2] = smid;
    }
  }

  // the swizzled operand tiles need a 1024-byte aligned base; the dynamic
  // window starts aligned (no static shared memory), checked here
  extern __shared__ __align__(1024) char t2_raw[];
  if ((smem_u32(t2_raw) & 1023u) != 0u) __trap();
  char* sm = t2_raw;
  char* sWB = sm;
  char* bufA = sm + LY::OFF_A;
  char* bufB = sm + LY::OFF_B;
  float* sf = reinterpret_cast<float*>(sm + LY::OFF_SMALL);
  float* sW0 = sf + LY::S_W0;
  float* sW0s = sf + LY::S_W0S;
  // field f (0 w_x, 1 w_y, 2 b, 3 pad) of hidden-1 unit i in sW0
  auto w0_at = [](int i, int f) { return 8 * (i >> 1) + 2 * f + (i & 1); };
  float* sBias = sf + LY::S_BIAS;
  float* sWd = sf + LY::S_WD;
  float* sWd2 = sWd + HP + 8;  // output channel 1 (C == 2)
  const bool spatial = C == 2 && a.eps_source == 2;
  float* sEx = sf + LY::S_EX;
  float* sAcc = sf + LY::S_ACC;
  double* sRed = reinterpret_cast<double*>(sf + LY::S_RED);
  float* sSc = sf + LY::S_SC;
  int* sSci = reinterpret_cast<int*>(sf + LY::S_SCI);
  uint32_t* sMax = reinterpret_cast<uint32_t*>(sf + LY::S_MAX);
  uint64_t* bar_v = reinterpret_cast<uint64_t*>(sf + LY::S_BAR);
  uint64_t* bar_t = bar_v + 1;
  uint64_t* bar_w = bar_v + 2;
  uint64_t* tma_bar = bar_v + 3;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar_v + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = tid & 127;   // point of this thread == TMEM lane
  const int ug = tid >> 7;   // unit group
  const int u0 = UPT * ug;   // first hidden unit of this thread
  const uint32_t tb = (uint32_t)(u0 >> 5) * kPart;  // this thread's column block inside a part
  // MP < 128 (NB = 2): the threads of TMEM lanes MP..127 hold no point; they
  // compute on the accumulators' unused rows, never store an operand row
  // (row p of an [MP][32] tile would be row p - MP of the next one) and add
  // zeros to the per-warp gradient sums
  const bool row_ok = MP == 128 || p < MP;
  const NetDesc& net = a.net;
  const float* P = a.params;
  const float kapmax = 2.0f;  // |act''/act'|: 2 |z| (tanh) or |1 - 2z| (sigmoid)

  // ---------------- one-time setup ----------------
  auto smark = [&](int i) {
    if constexpr (VPG_PHASE_CLOCK != 0)
      if (a.phase_clk != nullptr && blockIdx.x == 0 && threadIdx.x == 0) a.phase_clk[7 * kPhaseMarks + 20 + i] = clock64();
  };
  smark(0);
  if (warp == 0) tc::tmem_alloc(tslot, CF::kCols);
  smark(1);
  if (tid == 0) {
    mbar_init(bar_v, 1);
    mbar_init(bar_t, 2);
    mbar_init(bar_w, 1);
    mbar_init(tma_bar, 1);
    fence_mbar_init();
  }
  if (tid < 16) sMax[tid] = 0u;
  for (int i = tid; i < (NT / 32) * kAccW; i += NT) sAcc[i] = 0.f;
  // every parameter load of the setup issued at once: item it = (MMA layer
  // wl, row wo, 8-column chunk wc) of the [HP][HP] padded weight matrices
  constexpr int kWItems = HP * HP / 8;
  constexpr int IPT = (NL * kWItems + NT - 1) / NT;
  float wv[IPT][8];
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int it = tid + j * NT;
    const int wl = it / kWItems, wo = (it % kWItems) / (HP / 8), wc = it % (HP / 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = 8 * wc + k;
      // narrower layers (out_w / in_w < H) are zero-padded: padded units get
      // zero weights and biases, so they never reach the outputs
      const int fo = wl < NL ? net.out_w[wl + 1] : 0, fi = wl < NL ? net.in_w[wl + 1] : 0;
      wv[j][k] = (wo < fo && i < fi) ? P[net.w_off[wl + 1] + wo * fi + i] : 0.f;
    }
  }
  for (int i = tid; i < HP; i += NT) {
    float w0 = 0.f, w1 = 0.f, b = (i == H) ? kOneBias : 0.f, wd = 0.f;
    if (i < net.out_w[0]) {
      w0 = P[net.w_off[0] + 2 * i];
      w1 = P[net.w_off[0] + 2 * i + 1];
      b = P[net.b_off[0] + i];
    }
    if (i < net.in_w[D]) wd = P[net.w_off[D] + i];
    // unit pairs (k, k+1) adjacent per field: packed fp32x2 operands load
    // as register pairs (no moves to assemble them)
    sW0[w0_at(i, 0)] = w0;
    sW0[w0_at(i, 1)] = w1;
    sW0[w0_at(i, 2)] = b;
    sW0[w0_at(i, 3)] = 0.f;
    sWd[i] = wd;
    if constexpr (C == 2) sWd2[i] = i < net.in_w[D] ? P[net.w_off[D] + net.in_w[D] + i] : 0.f;
  }
  if (tid == 0) {
    sWd[HP] = P[net.b_off[D]];
    if constexpr (C == 2) sWd[HP + 1] = P[net.b_off[D] + 1];
  }
  for (int l = 1; l <= NL; ++l)
    for (int o = tid; o < HP; o += NT)
      sBias[(l - 1) * HP + o] = o < net.out_w[l] ? P[net.b_off[l] + o] : ((o == H) ? kOneBias : 0.f);
  // |W| into buffer A (free until the first tile) for the row / column sums
  float* sAbs = reinterpret_cast<float*>(bufA);  // [NL][HP][HP + 1] (odd row stride: no bank conflicts)
  uint32_t* sNorm = sMax + kNW0;  // [0] w0x [1] w0y [2] wd
  uint32_t(*s_lnorm)[3] = reinterpret_cast<uint32_t(*)[3]>(sMax + kNLayer);  // [layer][maxabs, rowsum, colsum]
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int it = tid + j * NT;
    const int wl = it / kWItems, wo = (it % kWItems) / (HP / 8), wc = it % (HP / 8);
    if (wl < NL) {
#pragma unroll
      for (int k = 0; k < 8; ++k) sAbs[(wl * HP + wo) * (HP + 1) + 8 * wc + k] = fabsf(wv[j][k]);
    }
  }
  smark(2);
  __syncthreads();  // (also orders the sMax zero fill before any atomic below)
  smark(3);
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int wl = (tid + j * NT) / kWItems;
    if (wl < NL) {
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) m = fmaxf(m, fabsf(wv[j][k]));
      atomic_max_abs(&s_lnorm[wl][0], m);  // max: order-free
    }
  }
  // weight norms (bounds for the scales): max |w0x|, |w0y|, |wd|; per MMA
  // layer max row abs-sum R and max column abs-sum C, each sum in index order
  if (tid < H) {
    atomic_max_abs(&sNorm[0], sW0[w0_at(tid, 0)]);
    atomic_max_abs(&sNorm[1], sW0[w0_at(tid, 1)]);
    atomic_max_abs(&sNorm[2], sWd[tid]);
    if constexpr (C == 2) atomic_max_abs(&sMax[kNWd2], sWd2[tid]);
  }
  for (int t = tid; t < 2 * HP * NL; t += NT) {
    const int l = t / (2 * HP), j = t % HP;
    const bool row = ((t / HP) & 1) == 0;
    float sum = 0.f;
    if (j < H) {
      for (int k = 0; k < H; ++k) sum += row ? sAbs[(l * HP + j) * (HP + 1) + k] : sAbs[(l * HP + k) * (HP + 1) + j];
    }
    atomic_max_abs(&s_lnorm[l][row ? 1 : 2], sum);
  }
  __syncthreads();
  if (tid == 0) {
    // forward tangent bounds of hidden 1..D outputs (x and y together)
    float bt = fmaxf(__uint_as_float(sNorm[0]), __uint_as_float(sNorm[1]));
    sSc[kScBt] = bt;
    for (int h = 1; h < D; ++h) {
      bt *= __uint_as_float(s_lnorm[h - 1][1]);
      sSc[kScBt + h] = bt;
    }
    for (int l = 0; l < NL; ++l) {
      const int kw = clamp_exp(14 - tc::bound_exp(__uint_as_float(s_lnorm[l][0])));
      // X_{l+1} (input of MMA layer l+1 = hidden l+1 output): value bound 1,
      // tangent bound bt[l]
      const int kxv = clamp_exp(14 - tc::bound_exp(1.0f));
      const int kxt = clamp_exp(14 - tc::bound_exp(sSc[kScBt + l]));
      sSci[kSiW + l] = kw;
      sSci[kSiXv + l] = kxv;
      sSci[kSiXt + l] = kxt;
      sSc[kScF0 + l] = tc::exp2i(-(kxv + kw));
      sSc[kScF1 + l] = tc::exp2i(-(kxt + kw));
      sSc[kScSv + l] = tc::exp2i(kxv);
      sSc[kScSt + l] = tc::exp2i(kxt);
      sSc[kScIv + l] = tc::exp2i(-kxv);
      sSc[kScIt + l] = tc::exp2i(-kxt);
      sSc[kScC + l] = __uint_as_float(s_lnorm[l][2]);
    }
    sSc[kScWd] = __uint_as_float(sNorm[2]);
    sSc[kScWd2] = C == 2 ? __uint_as_float(sMax[kNWd2]) : 0.f;
  }
  __syncthreads();
  for (int i = tid; i < HP; i += NT) {  // layer-0 tangent weights pre-scaled for X_1
    sW0s[4 * (i >> 1) + (i & 1)] = sW0[w0_at(i, 0)] * sSc[kScSt];
    sW0s[4 * (i >> 1) + 2 + (i & 1)] = sW0[w0_at(i, 1)] * sSc[kScSt];
  }
  smark(4);
  // W tiles, scaled by 2^kW: MMA layer wl, input block ib = wc / 4: row o of
  // part h at rows 0..HP-1, part l at rows HP..2HP-1
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int it = tid + j * NT;
    const int wl = it / kWItems, wo = (it % kWItems) / (HP / 8), wc = it % (HP / 8);
    if (wl < NL)
      tc::st_split8_h(sWB + wl * CF::kWL + (wc >> 2) * CF::kWTile, HP * tc::kRowBytes, wo, wc & 3, wv[j],
                      tc::exp2i(sSci[kSiW + wl]));
  }
  tc::fence_smem_to_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot;
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;  // TMEM lane quarter of this warp
  const uint32_t sA = smem_u32(bufA), sB = smem_u32(bufB), sW = smem_u32(sWB);
  // swizzled byte offsets of this thread's two 8-unit chunks inside its block's tile
  const uint32_t off0 = tc::sw_chunk(p, (u0 & 31) >> 3) + tb;
  const uint32_t off1 = NCH == 2 ? tc::sw_chunk(p, ((u0 & 31) >> 3) + 1) + tb : off0;

  // ---------------- MMA issue ----------------
  // descriptors: start address >> 4 in the low 14 bits, so an address offset
  // is added as offset >> 4 (addresses < 256 KB: no carry out of the field)
  const uint64_t dA_k = tc::kdesc(sA), dB_k = tc::kdesc(sB);                    // K-major point operands
  const uint64_t dA_mn = tc::mndesc(sA, kPart), dB_mn = tc::mndesc(sB, kPart);  // MN-major (param GEMM)
  const uint64_t dW_k = tc::kdesc(sW), dW_mn = tc::mndesc(sW, CF::kWTile);
  // layer l's parameter-gradient accumulator (MMA address) and this warp's
  // load address of it (lane quarter base)
  auto gacc = [&](int l) {
    return NB == 1 ? tmem + LY::kG0 + ((uint32_t)(16 * (l - 1)) << 16) : tmem + LY::kG0 + 128 * (l - 1);
  };
  auto gacc_ld = [&](int l) { return tmem + lane_q + LY::kG0 + (NB == 1 ? 0 : 128 * (l - 1)); };
  // point GEMM of MMA layer l (forward, or propagation with B MN-major):
  // stream s is issued by warp s (the three streams' MMAs enter the tensor
  // pipe in parallel; each stream's accumulation order stays fixed); bar_t
  // expects the two tangent-stream arrivals
  auto issue_point_gemm = [&](bool bufb, int l, bool propagate) {
    const int s = warp;
    const uint64_t abase = (bufb ? dB_k : dA_k) + (uint64_t)((s * kStream) >> 4);
    const uint64_t wbase = (propagate ? dW_mn : dW_k) + (uint64_t)(((l - 1) * CF::kWL) >> 4);
    const uint32_t idesc = tc::idesc_f16(128, HP, 0, propagate ? 1 : 0);
    issue_point_stream<NB>(tmem + HP * s, abase, wbase, idesc, propagate, kPart, CF::kWTile, HP * tc::kRowBytes);
#if VPG_MMA_ELECT1
    if (tc::elect_one()) tc::mma_commit(warp == 0 ? bar_v : bar_t);
    __syncwarp();
#else
    tc::commit_warp(warp == 0 ? bar_v : bar_t);
#endif
  };
  // parameter gradient of MMA layer l: G parts in bufA (M = Gh | Gl), X parts
  // in bufB (N = Xh | Xl).  Accumulates in TMEM across the CTA's tiles:
  // fresh (first), or onto the accumulator scaled down by 2^-shift
  // (scale-input-d) when this tile's product scale is smaller than the
  // accumulated one
  auto issue_param_gemm = [&](int l, bool first, int shift) {
    issue_param<MP>(gacc(l), dA_mn, dB_mn, tc::idesc_f16(2 * HP, 2 * HP, 1, 1), first ? 1 : 0, shift, bar_w,
                    kStream);
  };
  uint32_t ph_v = 0, ph_t = 0, ph_w = 0, tma_phase = 0;
  // wait for MMA completion: every warp polls the mbarrier(s) itself (no CTA
  // barrier, warps run ahead)
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
  auto dcol = [&](int s, int c) { return tmem + lane_q + HP * s + u0 + 8 * c; };
  auto coff = [&](int c) { return c ? off1 : off0; };

  // layer 0 of this thread's chunk c (8 units) at (px, py): z and s1
  // (unit pairs in packed fp32x2: the same IEEE operations per lane)
  auto layer0 = [&](int c, float px, float py, float (&z)[8], float (&s1)[8]) {
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const float4 wa = *reinterpret_cast<const float4*>(sW0 + 4 * (u0 + 8 * c + k));      // w_x, w_y of k, k+1
      const float2 wb = *reinterpret_cast<const float2*>(sW0 + 4 * (u0 + 8 * c + k) + 4);  // b of k, k+1
      const float2 pre = add2(fma2(f2(wa.z, wa.w), f2s(py), mul2(f2(wa.x, wa.y), f2s(px))), wb);
      const float2 zz = AC::value2(pre), ss = AC::s1_2(zz);
      z[k] = zz.x;
      z[k + 1] = zz.y;
      s1[k] = ss.x;
      s1[k + 1] = ss.y;
    }
  };
  // X_1 (hidden-1 output) of chunk c, scaled, into buffer buf: from (x, y)
  // through layer 0 (forward; its z kept in TMEM when it fits), or from that
  // kept z (reverse: no activation evaluation)
  auto store_x1 = [&](char* buf, int c, float px, float py, bool from_tmem) {
    float z[8], s1[8], tx[8], ty[8];
    if (CF::kZCache && from_tmem) {
      tc::tmem_ld1x8_wait(tmem + lane_q + LY::kZ1 + u0 + 8 * c, z);
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const float2 ss = AC::s1_2(f2(z[k], z[k + 1]));
        s1[k] = ss.x;
        s1[k + 1] = ss.y;
      }
    } else {
      layer0(c, px, py, z, s1);
      if (CF::kZCache) tc::tmem_st1x8_wait(tmem + lane_q + LY::kZ1 + u0 + 8 * c, z);
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const float4 ws = *reinterpret_cast<const float4*>(sW0s + 2 * (u0 + 8 * c + k));  // wx, wy of k, k+1
      const float2 ss = f2(s1[k], s1[k + 1]);
      const float2 a = mul2(ss, f2(ws.x, ws.y)), b = mul2(ss, f2(ws.z, ws.w));
      tx[k] = a.x;
      tx[k + 1] = a.y;
      ty[k] = b.x;
      ty[k + 1] = b.y;
    }
    const uint32_t o = coff(c);
    if (row_ok) tc::st_split8_ho<true>(buf, NB * kPart, o, z, sSc[kScSv]);
    if (row_ok) tc::st_split8_ho<false>(buf + kStream, NB * kPart, o, tx, 1.f);
    if (row_ok) tc::st_split8_ho<false>(buf + 2 * kStream, NB * kPart, o, ty, 1.f);
  };
  // running per-warp sums of 8 unit values (units u0 + 8c + k) at slot base
  auto acc_units = [&](float (&v)[8], int slot, int c) {
    if constexpr (MP < 128) {
      if (!row_ok) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.f;
      }
    }
    const float r = warp_rs8(v);
    if ((lane & 3) == 0) sAcc[warp * kAccW + slot + 8 * c + rs8_index(lane)] += r;
  };

  // parameter-gradient accumulators: product scale exponent kacc of what
  // TMEM holds per MMA layer, and whether it holds anything yet
  int kacc0 = 0, kacc1 = 0;
  bool has0 = false, has1 = false, spill0 = false, spill1 = false;
  // G row (part * HP + o) held by this thread's TMEM lane in layer l's
  // parameter-gradient accumulator, or -1: NB = 2 (M = 128) puts row r in
  // lane r; NB = 1 (M = 64) in lane 32 (r / 16) + r % 16 + the layer's lane
  // offset 16 (l - 1)
  auto gacc_row = [&](int l) {
    if (NB == 1) {
      const int lo = lane - 16 * (l - 1);
      return (lo >= 0 && lo < 16) ? 16 * (warp & 3) + lo : -1;
    }
    return 32 * (warp & 3) + lane;
  };
  // this thread's 2HP / NG accumulator columns (X part * HP + i)
  constexpr int kColsT = 2 * HP / CF::NG;
  const int col_base = kColsT * ug;
  // rare path (an accumulator would need more than 2^-15): add the layer-l
  // accumulator, unscaled, into the per-CTA fp32 scratch ([col][row]) and
  // restart it
  auto spill_accumulator = [&](int l, int kacc, bool first) {
    float* S = a.tc_scratch + ((size_t)blockIdx.x * NL + (l - 1)) * CF::kScratch;
    const float inv = tc::exp2i(-kacc);
#pragma unroll 1
    for (int h2 = 0; h2 < kColsT / 16; ++h2) {
      const int col0 = col_base + 16 * h2;
      float v[16];
      tc::tmem_ld1x16_wait(gacc_ld(l) + col0, v);
      const int grow = gacc_row(l);
      if (grow >= 0) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          float* d = S + (col0 + k) * (2 * HP) + grow;
          *d = first ? v[k] * inv : fmaf(v[k], inv, *d);
        }
      }
    }
  };
  // this tile's product exponent for param layer l: the natural kp_nat, or
  // the accumulated one when smaller; sets how the GEMM joins the accumulator
  auto join_acc = [&](int l, int kp_nat, bool& first, int& shift) {
    const int kacc = (l == 1) ? kacc0 : kacc1;
    const bool has = (l == 1) ? has0 : has1;
    bool spill = (l == 1) ? spill0 : spill1;
    shift = 0;
    first = false;
    int kp = kp_nat;
    if (!has) {
      first = true;
    } else if (a.tc_force_spill) {
      spill_accumulator(l, kacc, !spill);
      spill = true;
      first = true;
    } else if (kp_nat >= kacc) {
      kp = kacc;
    } else if (kacc - kp_nat <= 15) {
      shift = kacc - kp_nat;
    } else {
      spill_accumulator(l, kacc, !spill);
      spill = true;
      first = true;
    }
    if (l == 1) {
      kacc0 = kp;
      has0 = true;
      spill0 = spill;
    } else {
      kacc1 = kp;
      has1 = true;
      spill1 = spill;
    }
    return kp;
  };

  // diagnostics: phase clocks of CTA 0 (StepArgs::phase_clk, -DVPG_PHASE_CLOCK=1)
  int ph_tile = 0;
  auto mark = [&](int i) {
    if constexpr (VPG_PHASE_CLOCK != 0) {
      if (a.phase_clk != nullptr && blockIdx.x == 0 && tid == 0 && ph_tile < kPhaseTiles)
        a.phase_clk[ph_tile * kPhaseMarks + i] = clock64();
    }
  };

  double acc_b = 0.0, acc_s = 0.0;  // thread 0: penalty sums
  // per-cell-slot loss sums kept by the thread that forms them (unit group
  // 1, slot = cell within the tile) and combined across the CTA in a fixed
  // order at the end
  double cell_v = 0.0, cell_eg = 0.0;
  int bad = 0;
  const int n_pts_all = a.n_int + a.n_bnd + a.n_sen;
  struct TileGeo {
    bool interior;
    int cell0, ncell, pbase, np;
  };
  const int n_tiles = MODE == kModeForward ? (a.n_fwd + MP - 1) / MP
                      : (MODE == kModeReverse ? (n_pts_all + MP - 1) / MP : a.n_tiles);
  auto geo = [&](int tile) {
    TileGeo g{false, 0, 0, 0, 0};
    if (MODE != kModeFused) {
      if (tile < n_tiles) {
        g.pbase = tile * MP;
        g.np = min(MP, (MODE == kModeForward ? a.n_fwd : n_pts_all) - g.pbase);
      }
    } else if (tile < a.n_int_tiles) {
      g.interior = true;
      g.cell0 = tile * a.cells_per_tile;
      g.ncell = min(a.cells_per_tile, a.E - g.cell0);
      g.pbase = g.cell0 * a.Q;
      g.np = g.ncell * a.Q;
    } else if (tile < a.n_tiles) {
      g.pbase = a.n_int + (tile - a.n_int_tiles) * MP;
      g.np = min(MP, n_pts_all - g.pbase);
    }
    return g;
  };
  auto load_xy = [&](const TileGeo& g, float& x, float& y) {
    x = 0.f;
    y = 0.f;
    if (p < g.np) {
      const float2 xy = MODE == kModeForward ? a.fwd_pts[g.pbase + p] : a.pts[g.pbase + p];
      x = xy.x;
      y = xy.y;
    }
  };
  smark(5);
  float nx, ny;
  load_xy(geo(blockIdx.x), nx, ny);
  // contraction scratch after the slab in buffer A
  float* tail = reinterpret_cast<float*>(bufA) + (MODE == kModeFused ? a.nt * a.tstride : 0);
  // two outputs: the spatial-eps head's rows (tail_floats)
  float* tE = tail + kTE * 128;
  float* tY1 = tail + kTY1 * 128;
  float* tSx = tail + kTSx * 128;
  float* tSy = tail + kTSy * 128;
  float* tY1b = tail + kTY1b * 128;
  float* cvr = tail;              // [128] bx ux + by uy
  float* rbarv = tail + 4 * 128;  // [128]
  float* rsqv = tail + 5 * 128;
  float* rgev = tail + 6 * 128;

#pragma unroll 1
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileGeo G = geo(tile);
    mark(0);
    const bool interior = G.interior;
    const int cell0 = G.cell0, ncell = G.ncell, np = G.np;
    const int nrows_tile = ncell * a.T;
    const bool valid = p < np;
    const float px = nx, py = ny;
    float frow = 0.f;
    // contraction row of this thread (kCS adjacent threads per row, part 0 finishes it)
    if (interior && tid % kCS == 0 && tid / kCS < nrows_tile) frow = a.forcing[(size_t)cell0 * a.T + tid / kCS];
    if (ug == 0) {
      sEx[kX * 128 + p] = px;
      sEx[kY * 128 + p] = py;
    }
    if (tid < 3) sMax[tid] = 0u;  // tile maxima of |ub|, |uxb|, |uyb| (first read after 3+ barriers)
    if (C == 2 && tid == 3) sMax[kMe] = 0u;
    // D == 2: buffer A (slab) is free from the tile start
    if (D == 2 && interior && tid == 0)
      issue_chunk(a, cell0, 0, nrows_tile, reinterpret_cast<float*>(bufA), tma_bar);

    // =================== forward ===================
    char* x1buf = (D == 3) ? bufA : bufB;  // hidden-1 output (input of MMA layer 1)
#pragma unroll kUC
    for (int c = 0; c < NCH; ++c) store_x1(x1buf + 0, c, px, py, false);
    operands_ready();
    if (warp < 3) issue_point_gemm(D == 2, 1, false);
    mark(1);
    // epilogue of MMA layer l: hidden l+1 output.  Value stream first (it
    // overlaps the tangent-stream MMAs), stored (or consumed by the output
    // layer when hidden l+1 is the last), then the tangents.
    float ou = 0.f, oux = 0.f, ouy = 0.f;  // output-layer partials (last hidden)
    float oy1 = 0.f;                      // output channel 1 (C == 2)
#pragma unroll kUL
    for (int l = 1; l <= NL; ++l) {
      const bool last = l == NL;
      const float f0 = sSc[kScF0 + l - 1];
      // tangent factor: forward unscale, times the X_{l+1} scale when stored
      const float ft = last ? sSc[kScF1 + l - 1] : sSc[kScF1 + l - 1] * sSc[kScSt + l];
      const float sv = last ? 1.f : sSc[kScSv + l];
      const float* bias = sBias + HP * (l - 1);
      float s1v[UPT];
      mma_wait(bar_v, ph_v);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        float d[8], z[8];
        tc::tmem_ld1x8_wait(dcol(0, c), d);
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const int u = u0 + 8 * c + k;
          const float2 zz = AC::value2(fma2(f2(d[k], d[k + 1]), f2s(f0), *reinterpret_cast<const float2*>(bias + u)));
          const float2 ss = mul2(AC::s1_2(zz), f2s(ft));
          z[k] = zz.x;
          z[k + 1] = zz.y;
          s1v[8 * c + k] = ss.x;
          s1v[8 * c + k + 1] = ss.y;
          if (last) {
            ou = fmaf(sWd[u], zz.x, ou);
            ou = fmaf(sWd[u + 1], zz.y, ou);
            if constexpr (C == 2) {
              oy1 = fmaf(sWd2[u], zz.x, oy1);
              oy1 = fmaf(sWd2[u + 1], zz.y, oy1);
            }
          }
        }
        if (!last) {
          if (row_ok) tc::st_split8_ho<true>(bufB, NB * kPart, coff(c), z, sv);
          if (CF::kZCache && D == 3) tc::tmem_st1x8_wait(tmem + lane_q + LY::kZ2 + u0 + 8 * c, z);
        } else
          tc::tmem_st1x8_wait(tmem + lane_q + LY::kZ0 + u0 + 8 * c, z);  // kept for the reverse
      }
      mma_wait(bar_t, ph_t);
      // D == 3: buffer A (slab) is free once MMA layer 1 is done
      if (D == 3 && l == 1 && interior && tid == 0)
        issue_chunk(a, cell0, 0, nrows_tile, reinterpret_cast<float*>(bufA), tma_bar);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        float dx[8], dy[8];
        tc::tmem_ld2x8_wait(dcol(1, c), dcol(2, c), dx, dy);
        if (last) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float w = sWd[u0 + 8 * c + k] * s1v[8 * c + k];
            oux = fmaf(w, dx[k], oux);
            ouy = fmaf(w, dy[k], ouy);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const float2 ss = f2(s1v[8 * c + k], s1v[8 * c + k + 1]);
            const float2 a = mul2(f2(dx[k], dx[k + 1]), ss), b = mul2(f2(dy[k], dy[k + 1]), ss);
            dx[k] = a.x;
            dx[k + 1] = a.y;
            dy[k] = b.x;
            dy[k + 1] = b.y;
          }
          if (row_ok) tc::st_split8_ho<false>(bufB + kStream, NB * kPart, coff(c), dx, 1.f);
          if (row_ok) tc::st_split8_ho<false>(bufB + 2 * kStream, NB * kPart, coff(c), dy, 1.f);
        }
      }
      if (!last) {
        operands_ready();
        if (warp < 3) issue_point_gemm(true, l + 1, false);
      }
      mark(1 + l);
    }
    // output layer: groups combined in order (group 0 + 1, + 2, + 3, + bias)
    if (ug >= 1) {
      const int r = ug == 1 ? kPu : kRows + 3 * (ug - 2);
      sEx[(r + 0) * 128 + p] = ou;
      sEx[(r + 1) * 128 + p] = oux;
      sEx[(r + 2) * 128 + p] = ouy;
      if constexpr (C == 2) tail[(kTY1p + ug) * 128 + p] = oy1;
    }
    __syncthreads();
    if (ug == 0) {
      float u = ou + sEx[(kPu + 0) * 128 + p], ux = oux + sEx[(kPu + 1) * 128 + p],
            uy = ouy + sEx[(kPu + 2) * 128 + p];
#pragma unroll
      for (int g = 2; g < CF::NG; ++g) {
        const int r = kRows + 3 * (g - 2);
        u += sEx[(r + 0) * 128 + p];
        ux += sEx[(r + 1) * 128 + p];
        uy += sEx[(r + 2) * 128 + p];
      }
      u += sWd[HP];
      if (valid && !(finitef(u) && finitef(ux) && finitef(uy))) bad = 1;
      sEx[kU * 128 + p] = u;
      sEx[kUx * 128 + p] = ux;
      sEx[kUy * 128 + p] = uy;
      if (interior) cvr[p] = a.bx * ux + a.by * uy;
      float ep = 0.f;
      if constexpr (C == 2) {
        // channel 1 -> eps = softplus(y1) (network.hpp:130-138, 477-483)
        float y1 = oy1;
#pragma unroll
        for (int g = 1; g < CF::NG; ++g) y1 += tail[(kTY1p + g) * 128 + p];
        y1 += sWd[HP + 1];
        if (valid && !finitef(y1)) bad = 1;
        ep = softplusf(y1);
        tY1[p] = y1;
        tE[p] = ep;
        if (spatial) {
          tSx[p] = ep * ux;
          tSy[p] = ep * uy;
        }
      }
      if (MODE == kModeForward && valid) {
        if (a.out_u) a.out_u[G.pbase + p] = u;
        if (a.out_ux) a.out_ux[G.pbase + p] = ux;
        if (a.out_uy) a.out_uy[G.pbase + p] = uy;
        if (C == 2 && a.out_eps) a.out_eps[G.pbase + p] = ep;
      }
    }
    mark(4);
    if constexpr (MODE == kModeForward) {
      load_xy(geo(tile + gridDim.x), nx, ny);
      __syncthreads();  // exchange rows read before the next tile rewrites them
      continue;
    }

    // =================== objective: adjoints of (u, ux, uy) ===================
    if (MODE == kModeReverse) {
      // the split path's contraction / penalty kernels computed them
      if (ug == 0) {
        float ubv = 0.f, ox = 0.f, oy = 0.f, y1b = 0.f;
        if (valid) {
          const int pi = G.pbase + p;
          if (pi < a.n_int) {
            ox = a.in_uxb[pi];
            oy = a.in_uyb[pi];
            if (C == 2 && spatial && a.in_eb) y1b = a.in_eb[pi] * sigmoidf(tY1[p]);
          } else {
            ubv = a.in_ub[pi - a.n_int];
          }
        }
        sEx[kUb * 128 + p] = ubv;
        sEx[kUxb * 128 + p] = ox;
        sEx[kUyb * 128 + p] = oy;
        atomic_max_abs(&sMax[kMb], ubv);
        atomic_max_abs(&sMax[kMx], ox);
        atomic_max_abs(&sMax[kMy], oy);
        if constexpr (C == 2) {
          tY1b[p] = y1b;
          atomic_max_abs(&sMax[kMe], y1b);
        }
      }
    } else if (interior) {
      const bool conv = a.nt == 3;
      const float e_fixed = a.eps_source == 1 ? P[net.scal_off + a.eps_scalar_index] : a.eps;
      if (warp == 0) mbar_wait(tma_bar, tma_phase);  // the slab has landed
      tma_phase ^= 1u;
      __syncthreads();
      mark(5);
      const float* slab = reinterpret_cast<const float*>(bufA);
      const float* T0 = chunk_ptr(a, cell0, 0, slab, 0);
      const float* T1 = chunk_ptr(a, cell0, 0, slab, 1);
      const float* T2 = conv ? chunk_ptr(a, cell0, 0, slab, 2) : T0;
      // phase A: kCS = NT / 128 adjacent threads per row, each running the
      // three dot products (G_x . ux, G_y . uy, T . (bx ux + by uy)) over its
      // share of the quadrature points as two interleaved chains; the shares
      // are combined by a fixed xor tree and part 0 finishes the residual
      // (losses.hpp:122-136)
      {
        const int r = tid / kCS, part = tid % kCS;
        float ax[4] = {0.f, 0.f, 0.f, 0.f}, ay[4] = {0.f, 0.f, 0.f, 0.f}, at[4] = {0.f, 0.f, 0.f, 0.f};
        if (r < nrows_tile) {
          const int kk = r / a.T;
          const int q1 = (a.Q * (part + 1)) / kCS;
          // spatial eps: eps ux, eps uy (the coefficient inside the integral)
          const float* sx = (spatial ? tSx : sEx + kUx * 128) + kk * a.Q;
          const float* sy = (spatial ? tSy : sEx + kUy * 128) + kk * a.Q;
          const float* sc = cvr + kk * a.Q;
          const float* gx_r = T0 + r * a.Q;
          const float* gy_r = T1 + r * a.Q;
          const float* gt_r = T2 + r * a.Q;
          int q = (a.Q * part) / kCS;
#pragma unroll 2
          for (; q + 3 < q1; q += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              ax[u] = fmaf(gx_r[q + u], sx[q + u], ax[u]);
              ay[u] = fmaf(gy_r[q + u], sy[q + u], ay[u]);
              if (conv) at[u] = fmaf(gt_r[q + u], sc[q + u], at[u]);
            }
          }
          for (; q < q1; ++q) {
            ax[0] = fmaf(gx_r[q], sx[q], ax[0]);
            ay[0] = fmaf(gy_r[q], sy[q], ay[0]);
            if (conv) at[0] = fmaf(gt_r[q], sc[q], at[0]);
          }
        }
        float gx = (ax[0] + ax[1]) + (ax[2] + ax[3]);
        float gy = (ay[0] + ay[1]) + (ay[2] + ay[3]);
        float gt = (at[0] + at[1]) + (at[2] + at[3]);
#pragma unroll
        for (int o = 1; o < kCS; o <<= 1) {
          gx += __shfl_xor_sync(0xffffffffu, gx, o);
          gy += __shfl_xor_sync(0xffffffffu, gy, o);
          gt += __shfl_xor_sync(0xffffffffu, gt, o);
        }
        if (part == 0 && r < nrows_tile) {
          float res = spatial ? gx + gy : e_fixed * (gx + gy);
          if (conv) res += gt;
          res -= frow;
          rsqv[r] = res * res;
          const float rb = a.rscale * res;
          rbarv[r] = rb;
          rgev[r] = rb * (gx + gy);
        }
      }
      __syncthreads();
      mark(6);
      // phase B: kCS adjacent threads per point, each running the three
      // adjoint columns over its share of the cell's rows; part 0 writes the
      // point's adjoints.  The last ncell threads then form the per-cell sums.
      {
        const int pt = tid / kCS, part = tid % kCS;
        float bx4[4] = {0.f, 0.f, 0.f, 0.f}, by4[4] = {0.f, 0.f, 0.f, 0.f}, bt4[4] = {0.f, 0.f, 0.f, 0.f};
        const bool pv = pt < np;
        if (pv) {
          const int myk = pt / a.Q, myq = pt - myk * a.Q;
          const float* cx = T0 + myq;
          const float* cy = T1 + myq;
          const float* ct = T2 + myq;
          int r = myk * a.T + (a.T * part) / kCS;
          const int r1 = myk * a.T + (a.T * (part + 1)) / kCS;
#pragma unroll 2
          for (; r + 3 < r1; r += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float rb = rbarv[r + u];
              bx4[u] = fmaf(cx[(r + u) * a.Q], rb, bx4[u]);
              by4[u] = fmaf(cy[(r + u) * a.Q], rb, by4[u]);
              if (conv) bt4[u] = fmaf(ct[(r + u) * a.Q], rb, bt4[u]);
            }
          }
          for (; r < r1; ++r) {
            const float rb = rbarv[r];
            bx4[0] = fmaf(cx[r * a.Q], rb, bx4[0]);
            by4[0] = fmaf(cy[r * a.Q], rb, by4[0]);
            if (conv) bt4[0] = fmaf(ct[r * a.Q], rb, bt4[0]);
          }
        }
        float sbx = (bx4[0] + bx4[1]) + (bx4[2] + bx4[3]);
        float sby = (by4[0] + by4[1]) + (by4[2] + by4[3]);
        float sbt = (bt4[0] + bt4[1]) + (bt4[2] + bt4[3]);
#pragma unroll
        for (int o = 1; o < kCS; o <<= 1) {
          sbx += __shfl_xor_sync(0xffffffffu, sbx, o);
          sby += __shfl_xor_sync(0xffffffffu, sby, o);
          sbt += __shfl_xor_sync(0xffffffffu, sbt, o);
        }
        if (part == 0 && pt < 128) {
          float ox = 0.f, oy = 0.f, y1b = 0.f;
          if (pv) {
            if (spatial) {
              // uxbar = eps Gx^T rbar, epsbar = ux Gx^T rbar + uy Gy^T rbar,
              // y1bar = epsbar softplus'(y1) (losses.hpp:145-160)
              const float ep = tE[pt];
              ox = ep * sbx;
              oy = ep * sby;
              const float eb = sEx[kUx * 128 + pt] * sbx + sEx[kUy * 128 + pt] * sby;
              y1b = eb * sigmoidf(tY1[pt]);
            } else {
              ox = e_fixed * sbx;
              oy = e_fixed * sby;
            }
            if (conv) {
              ox = fmaf(a.bx, sbt, ox);
              oy = fmaf(a.by, sbt, oy);
            }
          }
          sEx[kUb * 128 + pt] = 0.f;
          sEx[kUxb * 128 + pt] = ox;
          sEx[kUyb * 128 + pt] = oy;
          atomic_max_abs(&sMax[kMx], ox);
          atomic_max_abs(&sMax[kMy], oy);
          if constexpr (C == 2) {
            tY1b[pt] = y1b;
            atomic_max_abs(&sMax[kMe], y1b);
          }
        }
        const int cs = tid - (NT - ncell);
        if (cs >= 0) {
          float s = 0.f, g = 0.f;
          for (int r = cs * a.T; r < (cs + 1) * a.T; ++r) {
            s += rsqv[r];
            g += rgev[r];
          }
          if (MODE == kModeFused) {
            cell_v += (double)(s * a.inv_nt);
            cell_eg += (double)g;
          }
        }
      }
      mark(7);
    } else {
      // ---------- penalty tile (losses.hpp:389-415) ----------
      double sb = 0.0, ss = 0.0;
      float ubv = 0.f;
      if (ug == 0 && valid) {
        const int pi = G.pbase + p - a.n_int;
        const float u = sEx[kU * 128 + p];
        if (pi < a.n_bnd) {
          const float d = u - a.bval[pi];
          sb = (double)(d * d);
          ubv = a.bscale * d;
        } else {
          const float d = u - a.sval[pi - a.n_bnd];
          ss = (double)(d * d);
          ubv = a.sscale * d;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sb += __shfl_down_sync(0xffffffffu, sb, o);
        ss += __shfl_down_sync(0xffffffffu, ss, o);
      }
      if (ug == 0) {
        sEx[kUb * 128 + p] = ubv;
        sEx[kUxb * 128 + p] = 0.f;
        sEx[kUyb * 128 + p] = 0.f;
        if constexpr (C == 2) tY1b[p] = 0.f;
        atomic_max_abs(&sMax[kMb], ubv);
      }
      if (lane == 0 && warp < 4) {
        sRed[warp] = sb;
        sRed[8 + warp] = ss;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 0; w < 4; ++w) {
          acc_b += sRed[w];
          acc_s += sRed[8 + w];
        }
      }
    }
    load_xy(geo(tile + gridDim.x), nx, ny);  // next tile's points, in flight during the reverse
    __syncthreads();                          // adjoint rows + tile maxima visible; slab reads done
    mark(8);
    const float ub = sEx[kUb * 128 + p], uxb = sEx[kUxb * 128 + p], uyb = sEx[kUyb * 128 + p];
    const float y1b = C == 2 ? tY1b[p] : 0.f;  // adjoint of output channel 1 (read before the G stores)

    // =================== reverse ===================
    // magnitude bounds of G at the last hidden layer (value | tangents)
    const float Mb = __uint_as_float(sMax[kMb]), Mx = __uint_as_float(sMax[kMx]), My = __uint_as_float(sMax[kMy]);
    const float Wd = sSc[kScWd];
    float bGv = Wd * (Mb + kapmax * sSc[kScBt + D - 1] * (Mx + My));
    if constexpr (C == 2) bGv += sSc[kScWd2] * __uint_as_float(sMax[kMe]);
    float bGt = Wd * fmaxf(Mx, My);
    // G scales for param layer l: S_G,s = 2^(kP - kX_s) with the common
    // product exponent kP = min_s (14 - e(B_s) + kX_s); returns kP
    auto g_scales = [&](int l, float bv, float bt, float& sgv, float& sgt, float& puv, float& put, bool& first,
                        int& shift) {
      const int kxv = sSci[kSiXv + l - 1], kxt = sSci[kSiXt + l - 1], kw = sSci[kSiW + l - 1];
      const int ev = tc::bound_exp(bv), et = tc::bound_exp(bt);
      int kp = 1 << 20;
      if (ev > -1000) kp = min(kp, 14 - ev + kxv);
      if (et > -1000) kp = min(kp, 14 - et + kxt);
      if (kp == (1 << 20)) kp = kxv;
      kp = join_acc(l, max(-120, min(120, kp)), first, shift);
      sgv = tc::exp2i(kp - kxv);
      sgt = tc::exp2i(kp - kxt);
      puv = tc::exp2i(-(kp - kxv + kw));  // propagation unscale
      put = tc::exp2i(-(kp - kxt + kw));
      return kp;
    };
    float sgv, sgt, puv, put;
    bool pfirst;
    int pshift;
    g_scales(NL, bGv, bGt, sgv, sgt, puv, put, pfirst, pshift);
    // ---- output layer: Wbar_out, bbar_out (unit H: z == 1), G of the last hidden layer ----
    // the last hidden state: z kept in TMEM by the forward, the tangents
    // from MMA layer NL's accumulators
    {
      const float f1 = sSc[kScF1 + NL - 1];
      const float Ub = ub * sgv, Uxv = uxb * sgv, Uyv = uyb * sgv, Uxt = uxb * sgt, Uyt = uyb * sgt;
      const float Y1 = y1b * sgv;
#pragma unroll kUC
      for (int c = 0; c < NCH; ++c) {
        float zs[8], dx[8], dy[8];
        tc::tmem_ld1x8_wait(tmem + lane_q + LY::kZ0 + u0 + 8 * c, zs);
        tc::tmem_ld2x8_wait(dcol(1, c), dcol(2, c), dx, dy);
        float v[8], gA[8], gX[8], gY[8], v1[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const int u = u0 + 8 * c + k;
          const float2 z = f2(zs[k], zs[k + 1]);
          const float2 s1 = AC::s1_2(z);
          const float2 cc = mul2(s1, f2s(f1));
          const float2 tx = mul2(cc, f2(dx[k], dx[k + 1])), ty = mul2(cc, f2(dy[k], dy[k + 1]));
          const float2 vv = fma2(f2s(ub), z, fma2(f2s(uxb), tx, mul2(f2s(uyb), ty)));
          const float2 wd = *reinterpret_cast<const float2*>(sWd + u);
          // kap (tx Uxv + ty Uyv); for tanh z (tx (-2 Uxv) + ty (-2 Uyv)), the same bits
          const float2 kin = (VPG_KAP_FOLD && AC::kKapLinear)
                                 ? mul2(z, fma2(tx, f2s(-2.f * Uxv), mul2(ty, f2s(-2.f * Uyv))))
                                 : mul2(AC::kap2(z), fma2(tx, f2s(Uxv), mul2(ty, f2s(Uyv))));
          float2 ga = mul2(wd, fma2(s1, f2s(Ub), kin));
          if constexpr (C == 2) {  // + s1 wd1 y1bar (channel 1 sees the value stream only)
            ga = fma2(mul2(s1, f2(sWd2[u], sWd2[u + 1])), f2s(Y1), ga);
            const float2 v2 = mul2(f2s(y1b), z);
            v1[k] = v2.x;
            v1[k + 1] = v2.y;
          }
          const float2 sw = mul2(s1, wd);
          const float2 gx = mul2(sw, f2s(Uxt)), gy = mul2(sw, f2s(Uyt));
          v[k] = vv.x;
          v[k + 1] = vv.y;
          gA[k] = ga.x;
          gA[k + 1] = ga.y;
          gX[k] = gx.x;
          gX[k + 1] = gx.y;
          gY[k] = gy.x;
          gY[k + 1] = gy.y;
        }
        acc_units(v, kAWd, c);
        if constexpr (C == 2) acc_units(v1, kAWd2, c);
        const uint32_t o = coff(c);
        if (row_ok) tc::st_split8_ho<false>(bufA, NB * kPart, o, gA, 1.f);
        if (row_ok) tc::st_split8_ho<false>(bufA + kStream, NB * kPart, o, gX, 1.f);
        if (row_ok) tc::st_split8_ho<false>(bufA + 2 * kStream, NB * kPart, o, gY, 1.f);
      }
    }
    operands_ready();
    // the parameter-gradient GEMM from the warp after the point-GEMM issuers
    if (warp < 3) {
      mark(13);
      issue_point_gemm(false, NL, true);
      mark(14);
    }
    if (warp == 3) {
      issue_param_gemm(NL, pfirst, pshift);
      mark(15);
    }
    mark(9);
    // ---- hidden layers, last first: G of hidden l from the propagated adjoints ----
#pragma unroll kUL
    for (int l = NL; l >= 1; --l) {
      // hidden-l state: X_l in buffer B (MMA layer l's input)
      const float iv = sSc[kScIv + l - 1], it = sSc[kScIt + l - 1];
      // bounds of G at hidden l: propagation through W_l, then the activation
      const float C = sSc[kScC + l - 1];
      const float bxa = C * bGv, bxt = C * bGt;
      const float bv2 = bxa + kapmax * sSc[kScBt + l - 1] * 2.f * bxt, bt2 = bxt;
      float sgv2 = 1.f, sgt2 = 1.f, puv2 = 1.f, put2 = 1.f;
      bool pfirst2 = false;
      int pshift2 = 0;
      if (l > 1) g_scales(l - 1, bv2, bt2, sgv2, sgt2, puv2, put2, pfirst2, pshift2);
      // ga = s1 xa' + kap (tx xx' + ty xy'), gx = s1 xx', gy = s1 xy' with the
      // propagation unscale ('), the state unscale and the store scale folded
      const float A0 = puv * sgv2, AT = it * put * sgv2, BT = put * sgt2;
      // l > 1: G of hidden l goes to buffer A and the recomputed hidden-1
      // output to buffer B, so param GEMM l must have read both (bar_w,
      // waited for right before the first store, so the first chunk's G
      // computation overlaps it)
      mma_wait(bar_v, ph_v);
      mma_wait(bar_t, ph_t);
#pragma unroll kUC
      for (int c = 0; c < NCH; ++c) {
        float xa[8], xx[8], xy[8], z[8], tx[8], ty[8];
        tc::tmem_ld1x8_wait(dcol(0, c), xa);
        tc::tmem_ld2x8_wait(dcol(1, c), dcol(2, c), xx, xy);
        const uint32_t o = coff(c);
        if (CF::kZCache && l == 1) {
          // hidden-1 state from the kept z: tangents s1 * w0 (scaled like X_1)
          tc::tmem_ld1x8_wait(tmem + lane_q + LY::kZ1 + u0 + 8 * c, z);
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const float4 ws = *reinterpret_cast<const float4*>(sW0s + 2 * (u0 + 8 * c + k));
            const float2 ss = AC::s1_2(f2(z[k], z[k + 1]));
            const float2 a2 = mul2(ss, f2(ws.x, ws.y)), b2 = mul2(ss, f2(ws.z, ws.w));
            tx[k] = a2.x;
            tx[k + 1] = a2.y;
            ty[k] = b2.x;
            ty[k + 1] = b2.y;
          }
        } else {
          if (CF::kZCache && D == 3 && l == 2)
            tc::tmem_ld1x8_wait(tmem + lane_q + LY::kZ2 + u0 + 8 * c, z);  // kept hidden-2 z
          else
            tc::ld_join8_ho<true>(bufB, NB * kPart, o, iv, z);
          tc::ld_join8_ho<false>(bufB + kStream, NB * kPart, o, 1.f, tx);
          tc::ld_join8_ho<false>(bufB + 2 * kStream, NB * kPart, o, 1.f, ty);
        }
        float ga[8], gx[8], gy[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const float2 zz = f2(z[k], z[k + 1]);
          const float2 s1 = AC::s1_2(zz);
          // kap AT; for tanh z (-2 AT), the same bits
          const float2 kat = (VPG_KAP_FOLD && AC::kKapLinear) ? mul2(zz, f2s(-2.f * AT))
                                                              : mul2(AC::kap2(zz), f2s(AT));
          const float2 xx2 = f2(xx[k], xx[k + 1]), xy2 = f2(xy[k], xy[k + 1]);
          const float2 inner = fma2(f2(tx[k], tx[k + 1]), xx2, mul2(f2(ty[k], ty[k + 1]), xy2));
          const float2 g = fma2(mul2(s1, f2s(A0)), f2(xa[k], xa[k + 1]), mul2(kat, inner));
          const float2 sb = mul2(s1, f2s(BT));
          const float2 gxx = mul2(sb, xx2), gyy = mul2(sb, xy2);
          ga[k] = g.x;
          ga[k + 1] = g.y;
          gx[k] = gxx.x;
          gx[k + 1] = gxx.y;
          gy[k] = gyy.x;
          gy[k + 1] = gyy.y;
        }
        if (l == 1) {
          // ---- input layer: Wbar_0 += Abar x^T + TAxbar e_x^T + TAybar e_y^T; bbar_0 += Abar ----
          float v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fmaf(ga[k], px, gx[k]);
          acc_units(v, kAW0x, c);
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fmaf(ga[k], py, gy[k]);
          acc_units(v, kAW0y, c);
          acc_units(ga, kAB0, c);
        } else {
          if (c == 0) {
            mbar_wait(bar_w, ph_w);
            ph_w ^= 1u;
            tc::fence_after_sync();
          }
          if (row_ok) tc::st_split8_ho<false>(bufA, NB * kPart, o, ga, 1.f);
          if (row_ok) tc::st_split8_ho<false>(bufA + kStream, NB * kPart, o, gx, 1.f);
          if (row_ok) tc::st_split8_ho<false>(bufA + 2 * kStream, NB * kPart, o, gy, 1.f);
          store_x1(bufB, c, px, py, true);  // hidden-1 output rebuilt (l - 1 == 1)
        }
      }
      if (l > 1) {
        operands_ready();
        if (warp < 3) issue_point_gemm(false, l - 1, true);
        if (warp == 3) issue_param_gemm(l - 1, pfirst2, pshift2);
        bGv = bv2;
        bGt = bt2;
        puv = puv2;
        put = put2;
      }
      mark(9 + NL - l + 1);
    }
    mma_wait(bar_w, ph_w);  // last param GEMM done: buffers A / B free
    mark(12);
    ++ph_tile;
  }

  // =================== per-CTA outputs ===================
#if VPG_PDL_LATE
  pdl_trigger();  // the epoch tail may be scheduled while the CTAs write their outputs
#endif
  if constexpr (MODE == kModeForward) {
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
      tc::fence_after_sync();
      tc::tmem_dealloc(tmem, CF::kCols);
    }
    return;
  }
  // (1) every MMA layer's parameter-gradient accumulator (G rows h | l x X
  // columns h | l), unscaled by 2^-kacc, plus any spilled part -> shared
  // memory [2HP][2HP + 1] per layer (buffers A and B are free); the per-warp
  // loss sums -> sRed; one barrier (which also ORs the non-finite flags and
  // publishes the per-warp CUDA-core gradient sums)
  constexpr int SS = 2 * HP + 1;
  static_assert((size_t)NL * 2 * HP * SS * sizeof(float) <= 2 * (size_t)CF::kBuf, "readout scratch");
  float* scr0 = reinterpret_cast<float*>(bufA);
  tc::fence_after_sync();
  for (int l = 1; l <= NL; ++l) {
    const int kacc = (l == 1) ? kacc0 : kacc1;
    const bool has = (l == 1) ? has0 : has1, spill = (l == 1) ? spill0 : spill1;
    const float* S = a.tc_scratch + ((size_t)blockIdx.x * NL + (l - 1)) * CF::kScratch;
    float* scr = scr0 + (l - 1) * 2 * HP * SS;
    if (has) {
      const float inv = tc::exp2i(-kacc);
#pragma unroll 1
      for (int h2 = 0; h2 < kColsT / 16; ++h2) {
        const int col0 = col_base + 16 * h2;
        float v[16];
        tc::tmem_ld1x16_wait(gacc_ld(l) + col0, v);
        const int grow = gacc_row(l);
        if (grow >= 0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            float x = v[k] * inv;
            if (spill) x += S[(col0 + k) * (2 * HP) + grow];
            scr[grow * SS + col0 + k] = x;
          }
        }
      }
    }
  }
  constexpr int NW = NT / 32;
  {
    double v = cell_v, g = cell_eg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, o);
      g += __shfl_xor_sync(0xffffffffu, g, o);
    }
    if (lane == 0) {  // (sRed is free after the tile loop)
      sRed[warp] = v;
      sRed[NW + warp] = g;
    }
  }
  tc::fence_before_sync();
  const int any_bad = __syncthreads_or(bad);
  // (2) the four-block sums of both MMA layers, the CUDA-core gradients
  // (per-warp sums combined in warp order) and the loss words
  {
    const int n1 = net.out_w[1] * (net.in_w[1] + 1);
    const int n_all = n1 + (NL == 2 ? net.out_w[2] * (net.in_w[2] + 1) : 0);
    for (int e = tid; e < n_all; e += NT) {
      const int l = e < n1 ? 1 : 2;
      const int ee = l == 1 ? e : e - n1;
      const int fi = net.in_w[l];
      const int o = ee / (fi + 1), i = ee - o * (fi + 1);
      const int c = i < fi ? i : H;  // the bias gradient is the constant unit's column
      const bool has = (l == 1) ? has0 : has1;
      const float* scr = scr0 + (l - 1) * 2 * HP * SS;
      float g = 0.f;
      if (has)  // scr[row][col]: row = G part * HP + o, col = X part * HP + c
        g = ((scr[o * SS + c] + scr[o * SS + HP + c]) + scr[(HP + o) * SS + c]) + scr[(HP + o) * SS + HP + c];
      const int idx = (i < fi) ? net.w_off[l] + o * fi + i : net.b_off[l] + o;
      a.grad_part[(size_t)idx * a.part_stride + blockIdx.x] = g;
    }
  }
  for (int u = tid; u <= H; u += NT) {
    const int grp = u / UPT, j = u % UPT;  // unit group (warps 4 grp .. +3), unit within it
    float w0x = 0.f, w0y = 0.f, b0 = 0.f, wd = 0.f, wd1 = 0.f;
    for (int w = 4 * grp; w < 4 * grp + 4; ++w) {
      const float* A = sAcc + w * kAccW;
      w0x += A[kAW0x + j];
      w0y += A[kAW0y + j];
      b0 += A[kAB0 + j];
      wd += A[kAWd + j];
      if constexpr (C == 2) wd1 += A[kAWd2 + j];
    }
    if (u < H) {
      if (u < net.out_w[0]) {
        a.grad_part[(size_t)(net.w_off[0] + 2 * u) * a.part_stride + blockIdx.x] = w0x;
        a.grad_part[(size_t)(net.w_off[0] + 2 * u + 1) * a.part_stride + blockIdx.x] = w0y;
        a.grad_part[(size_t)(net.b_off[0] + u) * a.part_stride + blockIdx.x] = b0;
      }
      if (u < net.in_w[D]) {
        a.grad_part[(size_t)(net.w_off[D] + u) * a.part_stride + blockIdx.x] = wd;
        if constexpr (C == 2)
          a.grad_part[(size_t)(net.w_off[D] + net.in_w[D] + u) * a.part_stride + blockIdx.x] = wd1;
      }
    } else {
      a.grad_part[(size_t)net.b_off[D] * a.part_stride + blockIdx.x] = wd;
      if constexpr (C == 2) a.grad_part[(size_t)(net.b_off[D] + 1) * a.part_stride + blockIdx.x] = wd1;
    }
  }
  if constexpr (VPG_PHASE_CLOCK != 0)  // CTA 0 exit clock and tile count (diagnostics)
    if (a.phase_clk != nullptr && blockIdx.x == 0 && tid == 0) {
      a.phase_clk[kPhaseTiles * kPhaseMarks - 2] = clock64();
      a.phase_clk[kPhaseTiles * kPhaseMarks - 3] = ph_tile;
    }
  if constexpr (VPG_PHASE_CLOCK != 0)
    if (a.phase_clk != nullptr && tid == 0 && blockIdx.x < 1024)
      a.phase_clk[kPhaseTiles * kPhaseMarks + 3 * blockIdx.x + 1] = (long long)globaltimer();
  if (tid == 0) {
    for (int e = net.scal_off; e < net.n_params; ++e) a.grad_part[(size_t)e * a.part_stride + blockIdx.x] = 0.f;
    double acc_v = 0.0, acc_eg = 0.0;
    for (int w = 0; w < NW; ++w) {
      acc_v += sRed[w];
      acc_eg += sRed[NW + w];
    }
    double* lp = a.loss_part + (size_t)blockIdx.x * kLpWords;
    lp[kLpVar] = acc_v;
    lp[kLpBnd] = acc_b;
    lp[kLpSen] = acc_s;
    lp[kLpEpsGrad] = acc_eg;
    lp[kLpBad] = any_bad ? 1.0 : 0.0;
    for (int w = kLpBad + 1; w < kLpWords; ++w) lp[w] = 0.0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, CF::kCols);
  }
}

template <int H, int D, int C = 1, int UPT = 16>
__host__ __device__ constexpr size_t tc2_step_smem_bytes() {
  return t2::Lay<H, D, C, UPT>::BYTES;
}

}  // namespace vpg
