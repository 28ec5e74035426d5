// Tensor-core (tcgen05, split-bf16) FastVPINNs training step for sm_100a.
//
// Same per-tile semantics as step_kernel<..., kModeFused> (step_kernel.cuh):
// forward with x/y tangents (network.hpp:204-282), the Algorithm-3
// contraction (losses.hpp:91-168) or the penalty terms (losses.hpp:406-415),
// and the reverse sweep (network.hpp:287-372) — but every hidden->hidden
// GEMM runs on the 5th-generation tensor cores:
//   forward      D_s[p][o]  = X_s[p][:] . W[o][:]      M = 128 points, N = 96 (W h | m | l), K = 32
//   propagation  D_s[p][i]  = G_s[p][:] . W[:][i]      M = 128 points, N = 96, K = 32 (B MN-major)
//   param grad   Wbar[o][i] += sum_{s,p} G_s[p][o] X_s[p][i]
//                                                     M = 128 (G h | m | l | -), N = 96 (X h | m | l),
//                                                     K = 3 streams x 128 points, accumulated in
//                                                     TMEM across all tiles of the CTA
// s = value / x-tangent / y-tangent stream.  Operands are split three ways
// into bf16 and each product is the six-term sum of tc_utils.cuh with fp32
// accumulation, so the result is fp32-faithful (the parity tolerance of the
// north star holds).  The
// value stream carries a constant-one column at index H, which turns the
// parameter-gradient GEMM's column H into the bias gradient.
//
// CTA = 128*NQ threads; thread t owns point p = t % 128 (= its TMEM lane)
// and hidden units [UPT*(t/128), +UPT), UPT = 32/NQ (NQ = 4: 16 warps, the
// elementwise phases are latency-bound and need the warps).  One CTA per SM (TMEM 512 columns,
// ~170 KB shared memory).  Hidden layers D in {2, 3}, H <= 31, one output.
// Every phase is separated by a CTA barrier or an MMA-completion mbarrier;
// one elected thread issues all MMAs.
#pragma once

#include "step_kernel.cuh"
#include "tc_utils.cuh"

namespace vpg {

constexpr int kTcPart = 8192;               // one [128][32] bf16 operand tile
constexpr int kTcStream = 3 * kTcPart;      // h | m | l parts of one stream
constexpr int kTcBuf = 3 * kTcStream;       // 3 streams
constexpr int kTcW = 6144;                  // [96][32] bf16: W h | m | l rows
constexpr uint32_t kTcCols = 512;           // TMEM columns allocated
constexpr int kTcDCols = 96;                // accumulator columns per stream (h | m | l products)
constexpr int kTcAccCol = 3 * kTcDCols;     // parameter-gradient accumulators start here

// exchange rows of the tensor-core kernel ([row][128] floats)
// (kTxP0.. : output-layer partials of unit groups 1..3, 3 rows each)
enum : int { kTxX = 0, kTxY, kTxU, kTxUx, kTxUy, kTxSx, kTxSy, kTxCv, kTxUb, kTxUxb, kTxUyb, kTxP0, kTxRows = kTxP0 + 9 };

template <int D>
struct TcLayout {
  static constexpr int NL = D - 1;                      // MMA (hidden->hidden) layers
  static constexpr int OFF_W = 0;                       // NL x kTcW
  static constexpr int OFF_A = OFF_W + NL * kTcW;       // buffer A (1024-aligned)
  static constexpr int OFF_B = OFF_A + kTcBuf;          // buffer B
  static constexpr int OFF_SMALL = OFF_B + kTcBuf;      // floats from here (>= 8 KB: the
                                                        // unused 4th M block of a param-grad
                                                        // A operand in buffer B reads it)
  // small region, in floats
  static constexpr int S_W0 = 0;                        // [32][4] (w_x, w_y, b, 0)
  static constexpr int S_BIAS = S_W0 + 128;             // [NL][32]
  static constexpr int S_WD = S_BIAS + NL * 32;         // [32] output weights + [4] bias
  static constexpr int S_EX = S_WD + 36;                // [kTxRows][128]
  static constexpr int S_CSUM = S_EX + kTxRows * 128;   // [8][96] column-sum partials
  static constexpr int S_GACC = S_CSUM + 8 * 96;        // [128] small-gradient accumulators
  static constexpr int S_CELL = S_GACC + 128;           // [256] per-cell sums
  static constexpr int S_ROWS = S_CELL + 256;           // [6][128] rbar | rsq | rge | per-tensor partials
  static constexpr int S_RED = S_ROWS + 6 * 128;        // 64 doubles (128 floats)
  static constexpr int S_BAR = S_RED + 128;             // 4 mbarriers + TMEM slot (16 floats)
  static constexpr int S_END = S_BAR + 16;               // then the dedicated slab, if any
  static constexpr size_t BYTES = (size_t)OFF_SMALL + sizeof(float) * S_END + 1024;  // + alignment slack
  static_assert(S_END * 4 >= kTcPart, "small region must cover one operand tile");
  static_assert(S_END % 4 == 0, "dedicated slab must be 16-byte aligned");
  static_assert(OFF_A % 1024 == 0, "operand buffers must be 1024-byte aligned");
};

// small-gradient accumulator slots (S_GACC)
enum : int { kGaW0x = 0, kGaW0y = 32, kGaB0 = 64, kGaWd = 96 };  // kGaWd: 32 slots (H weights + bias at H)

constexpr int kTcNQ = 4;  // unit groups per point in the instantiated kernels

template <int H, int D>
__host__ __device__ constexpr size_t tc_step_smem_bytes() {
  return TcLayout<D>::BYTES;
}

// column sums over the tile's 128 points of up to 96 per-point values
// (src row p at src + p * ld), added in a fixed order to acc[0..ncols):
// lane (c, g) of a warp sums rows [16g, 16g + 16) of column c (4 columns x 8
// groups per warp), then a fixed xor tree over the 8 groups.  No barrier
// inside: the caller syncs before (src written) and orders later writes
// to src behind its next barrier; acc[c] has a single owner lane.
template <int NT>
__device__ __forceinline__ void tc_colsum(const float* src, int ld, int ncols, float* acc) {
  const int ncp = (ncols + 3) & ~3;
  for (int e = threadIdx.x; e < 8 * ncp; e += NT) {
    const int c = (e >> 5) * 4 + ((e & 31) >> 3), g = e & 7;
    float s = 0.f;
    if (c < ncols) {
#pragma unroll 4
      for (int p = 16 * g; p < 16 * g + 16; ++p) s += src[p * ld + c];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (g == 0 && c < ncols) acc[c] += s;
  }
}

template <int H, int D, int ACT, int NQ>
__global__ void __launch_bounds__(128 * NQ, 1) tc_step_kernel(const StepArgs a) {
  static_assert(H <= 31 && (D == 2 || D == 3), "tensor-core step: H <= 31, 2 or 3 hidden layers");
  static_assert(NQ == 4, "unit groups per point (the contraction maps tensors to groups 0..2)");
  constexpr int UPT = 32 / NQ;  // hidden units per thread
  constexpr int NT = 128 * NQ;  // threads
  using LY = TcLayout<D>;
  constexpr int NL = LY::NL;
  using AC = Act<ACT>;

  if (a.stop_flag != nullptr && *a.stop_flag != 0) return;

  extern __shared__ __align__(1024) char tc_raw[];
  // 1024-byte alignment by an offset on the __shared__ array itself (a cast
  // through uintptr_t would lose the address space: generic LD/ST)
  char* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
  char* sWB = sm + LY::OFF_W;
  char* bufA = sm + LY::OFF_A;
  char* bufB = sm + LY::OFF_B;
  float* sf = reinterpret_cast<float*>(sm + LY::OFF_SMALL);
  float* sW0 = sf + LY::S_W0;
  float* sBias = sf + LY::S_BIAS;
  float* sWd = sf + LY::S_WD;
  float* sEx = sf + LY::S_EX;
  float* sGacc = sf + LY::S_GACC;
  float* sCell = sf + LY::S_CELL;
  float* sRows = sf + LY::S_ROWS;
  double* sRed = reinterpret_cast<double*>(sf + LY::S_RED);
  // MMA-completion barriers: value stream (bar_v), tangent streams (bar_t),
  // parameter-gradient GEMM (bar_w); slab TMA (tma_bar)
  uint64_t* bar_v = reinterpret_cast<uint64_t*>(sf + LY::S_BAR);
  uint64_t* bar_t = bar_v + 1;
  uint64_t* bar_w = bar_v + 2;
  uint64_t* tma_bar = bar_v + 3;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar_v + 4);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int p = tid & 127;          // point of this thread == TMEM lane
  const int hh = tid >> 7;          // unit group
  const int u0 = UPT * hh;          // first hidden unit of this thread
  const NetDesc& net = a.net;
  const float* P = a.params;

  // ---- one-time setup: TMEM, barriers, weights ----
  if (warp == 0) tc::tmem_alloc(tslot, kTcCols);
  if (tid == 0) {
    mbar_init(bar_v, 1);
    mbar_init(bar_t, 1);
    mbar_init(bar_w, 1);
    mbar_init(tma_bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 32; i += NT) {
    float w0 = 0.f, w1 = 0.f, b = 0.f, wd = 0.f;
    if (i < H) {
      w0 = P[net.w_off[0] + 2 * i];
      w1 = P[net.w_off[0] + 2 * i + 1];
      b = P[net.b_off[0] + i];
      wd = P[net.w_off[D] + i];
    }
    sW0[4 * i] = w0;
    sW0[4 * i + 1] = w1;
    sW0[4 * i + 2] = b;
    sW0[4 * i + 3] = 0.f;
    sWd[i] = wd;
  }
  if (tid == 0) sWd[32] = P[net.b_off[D]];
  for (int l = 1; l <= NL; ++l) {
    char* wb = sWB + (l - 1) * kTcW;
    // row o, 8 columns per item; parts h | m | l at rows 0 | 32 | 64
    for (int e = tid; e < 32 * 4; e += NT) {
      const int o = e >> 2, c = e & 3;
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = 8 * c + k;
        v[k] = (o < H && i < H) ? P[net.w_off[l] + o * H + i] : 0.f;
      }
      tc::st_split8(wb, 32 * tc::kRowBytes, o, c, v);
    }
    for (int o = tid; o < 32; o += NT) sBias[(l - 1) * 32 + o] = o < H ? P[net.b_off[l] + o] : 0.f;
  }
  for (int e = tid; e < 128; e += NT) sGacc[e] = 0.f;
  for (int e = tid; e < 256; e += NT) sCell[e] = 0.f;
  tc::fence_smem_to_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot;
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;  // TMEM lane quarter of this warp

  // MMA helpers (thread 0 only) -------------------------------------------------
  const uint32_t sA = smem_u32(bufA), sB = smem_u32(bufB), sW = smem_u32(sWB);
  // forward (propagate == false) or propagation of layer l; A parts (K-major)
  // from buffer abuf: D_s[0:96) = h.[Wh|Wm|Wl], D_s[0:64) += m.[Wh|Wm], D_s[0:32) += l.Wh
  // commits: bar_v after the value stream, bar_t after the tangent streams
  // (a commit tracks every earlier MMA of the thread, so the propagation is
  // issued before the parameter-gradient GEMM)
  auto issue_point_gemm = [&](uint32_t abuf, int l, bool propagate) {
    const uint32_t wbase = sW + (uint32_t)(l - 1) * kTcW;
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
      const uint32_t d = tmem + kTcDCols * s;
#pragma unroll
      for (int part = 0; part < 3; ++part) {
        const uint32_t idesc = tc::idesc_bf16(128, 96 - 32 * part, 0, propagate ? 1 : 0);
        const uint32_t abase = abuf + s * kTcStream + part * kTcPart;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t bd = propagate ? tc::mndesc(wbase + 1024 * ks, 32 * tc::kRowBytes) : tc::kdesc(wbase + 32 * ks);
          tc::mma_bf16(d, tc::kdesc(abase + 32 * ks), bd, idesc, (part > 0 || ks > 0) ? 1u : 0u);
        }
      }
      if (s == 0) tc::mma_commit(bar_v);
    }
    tc::mma_commit(bar_t);
  };
  // parameter gradient of layer l: G parts in gbuf (M = h|m|l|-), X parts in xbuf (N = h|m|l)
  auto issue_param_gemm = [&](uint32_t gbuf, uint32_t xbuf, int l, bool first) {
    const uint32_t acc = tmem + kTcAccCol + kTcDCols * (l - 1);
    const uint32_t idesc = tc::idesc_bf16(128, 96, 1, 1);
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
      const uint32_t g = gbuf + s * kTcStream, x = xbuf + s * kTcStream;
#pragma unroll
      for (int kp = 0; kp < 8; ++kp)
        tc::mma_bf16(acc, tc::mndesc(g + 1024 * kp, kTcPart), tc::mndesc(x + 1024 * kp, kTcPart), idesc,
                     (first && s == 0 && kp == 0) ? 0u : 1u);
    }
    tc::mma_commit(bar_w);
  };
  uint32_t ph_v = 0, ph_t = 0, ph_w = 0, tma_phase = 0;
  auto wait_bar = [&](uint64_t* bar, uint32_t& ph) {
    mbar_wait(bar, ph);
    ph ^= 1u;
    tc::fence_after_sync();
  };
  // all threads: make smem operand writes and TMEM reads ordered before the
  // next MMA issue
  auto operands_ready = [&]() {
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  };

  // layer 0 of this thread's units for point (px, py): z, TX_x, TX_y
  auto layer0 = [&](float px, float py, float (&z)[UPT], float (&tx)[UPT], float (&ty)[UPT]) {
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
      const int u = u0 + k;
      const float4 w = *reinterpret_cast<const float4*>(sW0 + 4 * u);
      if (u < H) {
        const float zz = AC::value(fmaf(w.y, py, w.x * px) + w.z);
        const float s1 = AC::s1(zz);
        z[k] = zz;
        tx[k] = s1 * w.x;
        ty[k] = s1 * w.y;
      } else {
        z[k] = (u == H) ? 1.0f : 0.0f;  // constant-one column -> bias gradient
        tx[k] = 0.f;
        ty[k] = 0.f;
      }
    }
  };
  // the three streams of this thread's row, split into bf16 parts
  auto store3 = [&](char* buf, const float (&z)[UPT], const float (&tx)[UPT], const float (&ty)[UPT]) {
#pragma unroll
    for (int j = 0; j < UPT / 8; ++j) {
      tc::st_split8(buf, kTcPart, p, u0 / 8 + j, z + 8 * j);
      tc::st_split8(buf + kTcStream, kTcPart, p, u0 / 8 + j, tx + 8 * j);
      tc::st_split8(buf + 2 * kTcStream, kTcPart, p, u0 / 8 + j, ty + 8 * j);
    }
  };
  // read back one stream of a buffer (h + m + l)
  auto load1 = [&](const char* buf, int s, float (&v)[UPT]) {
#pragma unroll
    for (int j = 0; j < UPT / 8; ++j) tc::ld_join8(buf + s * kTcStream, kTcPart, p, u0 / 8 + j, v + 8 * j);
  };
  // accumulator of stream s: columns [0,32) + [32,64) + [64,96)
  auto acc_stream = [&](int s, float (&v)[UPT]) {
    float x0[UPT], x1[UPT], x2[UPT];
    const uint32_t col = tmem + lane_q + kTcDCols * s + u0;
    tc::tmem_ld3_wait<UPT>(col, col + 32, col + 64, x0, x1, x2);
#pragma unroll
    for (int k = 0; k < UPT; ++k) v[k] = (x0[k] + x1[k]) + x2[k];
  };

  // dedicated slab region after the small region (a.union_floats floats), or
  // none (0): the slab then aliases a free operand buffer
  const bool dedicated = a.union_floats > 0;
  char* dslab = reinterpret_cast<char*>(sf + LY::S_END);
  if (dedicated && tid == 0 && (int)blockIdx.x < a.n_int_tiles) {
    const int c0 = blockIdx.x * a.cells_per_tile;
    issue_chunk(a, c0, 0, min(a.cells_per_tile, a.E - c0) * a.T, reinterpret_cast<float*>(dslab), tma_bar);
  }

  bool first_grad = true;
  double acc_v = 0.0, acc_b = 0.0, acc_s = 0.0, acc_eg = 0.0;  // thread 0
  int bad = 0;
  const int n_pts_all = a.n_int + a.n_bnd + a.n_sen;

  // tile geometry; the point coordinates of a tile are loaded one tile ahead
  // (register prefetch) so their DRAM latency hides behind the previous tile
  struct TileGeo {
    bool interior;
    int cell0, ncell, pbase, np;
  };
  auto geo = [&](int tile) {
    TileGeo g{false, 0, 0, 0, 0};
    if (tile < a.n_int_tiles) {
      g.interior = true;
      g.cell0 = tile * a.cells_per_tile;
      g.ncell = min(a.cells_per_tile, a.E - g.cell0);
      g.pbase = g.cell0 * a.Q;
      g.np = g.ncell * a.Q;
    } else if (tile < a.n_tiles) {
      g.pbase = a.n_int + (tile - a.n_int_tiles) * 128;
      g.np = min(128, n_pts_all - g.pbase);
    }
    return g;
  };
  auto load_xy = [&](const TileGeo& g, float& x, float& y) {
    x = 0.f;
    y = 0.f;
    if (p < g.np) {
      const float2 xy = a.pts[g.pbase + p];
      x = xy.x;
      y = xy.y;
    }
  };
  // diagnostics: phase clocks of CTA 0 (StepArgs::phase_clk)
  int ph_tile = 0;
  auto mark = [&](int i) {
    if (a.phase_clk != nullptr && blockIdx.x == 0 && tid == 0 && ph_tile < kPhaseTiles)
      a.phase_clk[ph_tile * kPhaseMarks + i] = clock64();
  };
  float nx, ny;
  load_xy(geo(blockIdx.x), nx, ny);

#pragma unroll 1
  for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const TileGeo G = geo(tile);
    mark(0);
    const bool interior = G.interior;
    const int cell0 = G.cell0, ncell = G.ncell, pbase = G.pbase, np = G.np;
    const int nrows_tile = ncell * a.T;
    const bool valid = p < np;
    const float px = nx, py = ny;
    // forcing of this thread's residual row (used after the forward)
    float frow = 0.f;
    if (interior && hh == 0 && p < nrows_tile) frow = a.forcing[(size_t)cell0 * a.T + p];
    if (hh == 0) {
      sEx[kTxX * 128 + p] = px;
      sEx[kTxY * 128 + p] = py;
    }

    // =================== forward ===================
    {
      float z[UPT], tx[UPT], ty[UPT];
      layer0(px, py, z, tx, ty);
      store3(bufA, z, tx, ty);
    }
    operands_ready();
    mark(1);
    if (tid == 0) issue_point_gemm(sA, 1, false);
    // epilogue of hidden layer l (bias index bofs): the activation of the value
    // stream overlaps the tangent-stream MMAs
    auto hidden_epilogue = [&](int bofs, float (&oz)[UPT], float (&ot)[UPT], float (&ou)[UPT]) {
      float av[UPT];
      wait_bar(bar_v, ph_v);
      acc_stream(0, av);
      const float* bias = sBias + bofs;
      float s1v[UPT];
#pragma unroll
      for (int k = 0; k < UPT; ++k) {
        const int u = u0 + k;
        const float zz = (u < H) ? AC::value(av[k] + bias[u]) : ((u == H) ? 1.0f : 0.0f);
        oz[k] = zz;
        s1v[k] = (u < H) ? AC::s1(zz) : 0.f;
      }
      wait_bar(bar_t, ph_t);
      acc_stream(1, ot);
      acc_stream(2, ou);
#pragma unroll
      for (int k = 0; k < UPT; ++k) {
        ot[k] = s1v[k] * ot[k];
        ou[k] = s1v[k] * ou[k];
      }
    };
    // aliased slab: its operand buffer is free once layer 1 is done (D == 3:
    // layer-1 input consumed; D == 2: unused); a dedicated slab was prefetched
    char* slab = dedicated ? dslab : ((D == 3) ? bufA : bufB);
    float lz[UPT], lt[UPT], lu[UPT];  // last hidden layer (units u0..u0+15)
    hidden_epilogue(0, lz, lt, lu);
    mark(2);
    if (!dedicated && interior && tid == 0)
      issue_chunk(a, cell0, 0, nrows_tile, reinterpret_cast<float*>(slab), tma_bar);
    if constexpr (D == 3) {
      store3(bufB, lz, lt, lu);
      operands_ready();
      mark(3);
      if (tid == 0) issue_point_gemm(sB, 2, false);
      hidden_epilogue(32, lz, lt, lu);
      mark(4);
    }
    // output layer (linear) over this thread's units, halves combined in order
    {
      float u = 0.f, ux = 0.f, uy = 0.f;
#pragma unroll
      for (int k = 0; k < UPT; ++k) {
        if (u0 + k < H) {
          const float w = sWd[u0 + k];
          u = fmaf(w, lz[k], u);
          ux = fmaf(w, lt[k], ux);
          uy = fmaf(w, lu[k], uy);
        }
      }
      if (hh > 0) {
        sEx[(kTxP0 + 3 * (hh - 1)) * 128 + p] = u;
        sEx[(kTxP0 + 3 * (hh - 1) + 1) * 128 + p] = ux;
        sEx[(kTxP0 + 3 * (hh - 1) + 2) * 128 + p] = uy;
      }
      __syncthreads();
      if (hh == 0) {
#pragma unroll
        for (int g = 0; g < NQ - 1; ++g) {
          u += sEx[(kTxP0 + 3 * g) * 128 + p];
          ux += sEx[(kTxP0 + 3 * g + 1) * 128 + p];
          uy += sEx[(kTxP0 + 3 * g + 2) * 128 + p];
        }
        u += sWd[32];
        if (valid && !(finitef(u) && finitef(ux) && finitef(uy))) bad = 1;
        sEx[kTxU * 128 + p] = u;
        sEx[kTxUx * 128 + p] = ux;
        sEx[kTxUy * 128 + p] = uy;
      }
    }
    mark(5);

    // =================== objective: adjoints of (u, ux, uy) ===================
    float ub = 0.f, uxb = 0.f, uyb = 0.f;
    if (interior) {
      const bool conv = a.nt == 3;
      const float e_fixed = a.eps_source == 1 ? P[net.scal_off + a.eps_scalar_index] : a.eps;
      if (hh == 0) {
        const float ux = sEx[kTxUx * 128 + p], uy = sEx[kTxUy * 128 + p];
        sEx[kTxSx * 128 + p] = ux;
        sEx[kTxSy * 128 + p] = uy;
        sEx[kTxCv * 128 + p] = a.bx * ux + a.by * uy;
      }
      __syncthreads();
      mbar_wait(tma_bar, tma_phase);
      tma_phase ^= 1u;
      mark(6);
      const float* Gx = chunk_ptr(a, cell0, 0, reinterpret_cast<const float*>(slab), 0);
      const float* Gy = chunk_ptr(a, cell0, 0, reinterpret_cast<const float*>(slab), 1);
      const float* Tv = conv ? chunk_ptr(a, cell0, 0, reinterpret_cast<const float*>(slab), 2) : nullptr;
      float* rbarv = sRows;
      float* rsqv = sRows + 128;
      float* rgev = sRows + 256;
      float* part = sRows + 384;  // [3][128]: one dot product per (tensor, row) / (tensor, point)
      const int nt = a.nt;
      const float* Gt = hh == 0 ? Gx : (hh == 1 ? Gy : Tv);  // this group's tensor (hh < nt)
      // phase A: unit group g < nt computes tensor g's row dot products
      if (hh < nt && p < nrows_tile) {
        const int kk = p / a.T;
        const float* sv = sEx + (hh == 0 ? kTxSx : (hh == 1 ? kTxSy : kTxCv)) * 128 + kk * a.Q;
        const float* gr = Gt + p * a.Q;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        int q = 0;
#pragma unroll 2
        for (; q + 3 < a.Q; q += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) acc4[u] = fmaf(gr[q + u], sv[q + u], acc4[u]);
        }
        for (; q < a.Q; ++q) acc4[0] = fmaf(gr[q], sv[q], acc4[0]);
        part[hh * 128 + p] = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
      }
      __syncthreads();
      mark(7);
      // residuals r_j (losses.hpp:122-136)
      if (hh == 0 && p < nrows_tile) {
        const int kk = p / a.T;
        const float gx = part[p], gy = part[128 + p];
        float res = e_fixed * (gx + gy);
        if (conv) res += part[256 + p];
        res -= frow;  // forcing[(cell0 + kk) * T + j], prefetched
        rsqv[p] = res * res;
        const float rb = a.rscale * res;
        rbarv[p] = rb;
        rgev[p] = rb * (gx + gy);
      }
      __syncthreads();
      mark(8);
      // phase B: unit group g < nt computes tensor g's adjoint column per
      // point; group 3 the per-cell sums in row order
      if (hh < nt && valid) {
        const int myk = p / a.Q, myq = p - myk * a.Q;
        const float* gc = Gt + myq;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        int r = myk * a.T;
        const int r1 = r + a.T;
#pragma unroll 2
        for (; r + 3 < r1; r += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) acc4[u] = fmaf(gc[(r + u) * a.Q], rbarv[r + u], acc4[u]);
        }
        for (; r < r1; ++r) acc4[0] = fmaf(gc[r * a.Q], rbarv[r], acc4[0]);
        part[hh * 128 + p] = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
      }
      if (hh == 3 && p < ncell) {
        float s = 0.f, g = 0.f;
        for (int r = p * a.T; r < (p + 1) * a.T; ++r) {
          s += rsqv[r];
          g += rgev[r];
        }
        sCell[p] = s;
        sCell[128 + p] = g;
      }
      __syncthreads();
      mark(9);
      if (hh == 0) {
        float ox = 0.f, oy = 0.f;
        if (valid) {
          ox = e_fixed * part[p];
          oy = e_fixed * part[128 + p];
          if (conv) {
            const float tt = part[256 + p];
            ox = fmaf(a.bx, tt, ox);
            oy = fmaf(a.by, tt, oy);
          }
        }
        sEx[kTxUb * 128 + p] = 0.f;
        sEx[kTxUxb * 128 + p] = ox;
        sEx[kTxUyb * 128 + p] = oy;
      }
      if (tid == 0) {
        for (int k = 0; k < ncell; ++k) {
          acc_v += (double)(sCell[k] * a.inv_nt);
          acc_eg += (double)sCell[128 + k];
        }
      }
    } else {
      // ---------- penalty tile (losses.hpp:389-415) ----------
      double sb = 0.0, ss = 0.0;
      float ubv = 0.f;
      if (hh == 0 && valid) {
        const int pi = pbase + p - a.n_int;
        const float u = sEx[kTxU * 128 + p];
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
      if (hh == 0) {
        sEx[kTxUb * 128 + p] = ubv;
        sEx[kTxUxb * 128 + p] = 0.f;
        sEx[kTxUyb * 128 + p] = 0.f;
      }
      // block sums of the penalty squares (warps 0-3 hold the points)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sb += __shfl_down_sync(0xffffffffu, sb, o);
        ss += __shfl_down_sync(0xffffffffu, ss, o);
      }
      if ((tid & 31) == 0 && warp < 4) {
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
    __syncthreads();  // adjoint rows visible; slab reads done
    mark(10);
    ub = sEx[kTxUb * 128 + p];
    uxb = sEx[kTxUxb * 128 + p];
    uyb = sEx[kTxUyb * 128 + p];

    // =================== reverse ===================
    // ---- output layer: Wbar_out, bbar_out (column H: lz == 1) and G of the last hidden layer ----
    char* gbuf = (D == 3) ? bufA : bufB;  // free buffer
    {
      // [128][33] scratch: the consumed dedicated slab (refilled only after
      // the next barrier), else the G buffer before G is written
      float* vrow = reinterpret_cast<float*>(dedicated ? dslab : gbuf);
#pragma unroll
      for (int k = 0; k < UPT; ++k) vrow[p * 33 + u0 + k] = fmaf(uyb, lu[k], fmaf(uxb, lt[k], ub * lz[k]));
      __syncthreads();
      tc_colsum<NT>(vrow, 33, H + 1, sGacc + kGaWd);
      if (!dedicated) __syncthreads();  // scratch reads done before G overwrites it
      float gA[UPT], gX[UPT], gY[UPT];
#pragma unroll
      for (int k = 0; k < UPT; ++k) {
        const int u = u0 + k;
        if (u < H) {
          const float wd = sWd[u];
          const float xb = wd * ub, zx = wd * uxb, zy = wd * uyb;
          const float s1 = AC::s1(lz[k]), kp = AC::kap(lz[k]);
          gA[k] = fmaf(s1, xb, kp * fmaf(lt[k], zx, lu[k] * zy));
          gX[k] = s1 * zx;
          gY[k] = s1 * zy;
        } else {
          gA[k] = gX[k] = gY[k] = 0.f;
        }
      }
      store3(gbuf, gA, gX, gY);
    }
    operands_ready();
    mark(11);
    // ---- hidden->hidden layers, last first ----
    // propagation first (bar_v / bar_t), then the parameter-gradient GEMM
    // (bar_w); elementwise work that does not need them runs in their shadow
    char* xbuf = (gbuf == bufA) ? bufB : bufA;  // input of layer NL
    if (tid == 0) {
      issue_point_gemm(smem_u32(gbuf), NL, true);
      issue_param_gemm(smem_u32(gbuf), smem_u32(xbuf), NL, first_grad);
      if (dedicated) {
        // prefetch the next tile's slab: it lands during this reverse and the next forward
        const int nt = tile + gridDim.x;
        if (nt < a.n_int_tiles) {
          const int c0 = nt * a.cells_per_tile;
          issue_chunk(a, c0, 0, min(a.cells_per_tile, a.E - c0) * a.T, reinterpret_cast<float*>(dslab), tma_bar);
        }
      }
    }
    float z1[UPT], t1x[UPT], t1y[UPT];  // hidden-1 state, recomputed once per tile
    // G of hidden h from the propagated adjoints (TMEM) and the state (z, tx, ty)
    auto hidden_adjoint = [&](const float (&z)[UPT], const float (&tx)[UPT], const float (&ty)[UPT], float (&gA)[UPT],
                              float (&gX)[UPT], float (&gY)[UPT]) {
      float xa[UPT], xx[UPT], xy[UPT];
      wait_bar(bar_v, ph_v);
      acc_stream(0, xa);
      wait_bar(bar_t, ph_t);
      acc_stream(1, xx);
      acc_stream(2, xy);
#pragma unroll
      for (int k = 0; k < UPT; ++k) {
        if (u0 + k < H) {
          const float s1 = AC::s1(z[k]), kp = AC::kap(z[k]);
          gA[k] = fmaf(s1, xa[k], kp * fmaf(tx[k], xx[k], ty[k] * xy[k]));
          gX[k] = s1 * xx[k];
          gY[k] = s1 * xy[k];
        } else {
          gA[k] = gX[k] = gY[k] = 0.f;
        }
      }
    };
    if constexpr (D == 3) {
      float gA[UPT], gX[UPT], gY[UPT];
      {
        float z[UPT], tx[UPT], ty[UPT];
        load1(xbuf, 0, z);  // hidden-2 state (read-only for the MMAs too)
        load1(xbuf, 1, tx);
        load1(xbuf, 2, ty);
        layer0(px, py, z1, t1x, t1y);
        hidden_adjoint(z, tx, ty, gA, gX, gY);
      }
      mark(12);
      wait_bar(bar_w, ph_w);  // both operand buffers free
      __syncthreads();        // every thread has read hidden-2 state from xbuf
      store3(gbuf, gA, gX, gY);
      store3(xbuf, z1, t1x, t1y);  // layer-1 input (recomputed)
      operands_ready();
      mark(13);
      if (tid == 0) {
        issue_point_gemm(smem_u32(gbuf), 1, true);
        issue_param_gemm(smem_u32(gbuf), smem_u32(xbuf), 1, first_grad);
      }
    } else {
      layer0(px, py, z1, t1x, t1y);
    }
    first_grad = false;
    // ---- input layer: G of hidden 1 -> Wbar_0, bbar_0 ----
    {
      float ga[UPT], gx[UPT], gy[UPT];
      hidden_adjoint(z1, t1x, t1y, ga, gx, gy);
      mark(14);
      wait_bar(bar_w, ph_w);  // the parameter-gradient GEMM has read bufA / bufB
      mark(15);
      // [128][97] scratch in buffer B: its next writer comes after the next
      // tile's first barrier
      float* vrow = reinterpret_cast<float*>(bufB);
#pragma unroll
      for (int k = 0; k < UPT; ++k) {
        const int u = u0 + k;
        // Wbar_0 += Abar x^T + TAxbar e_x^T + TAybar e_y^T ; bbar_0 += Abar
        vrow[p * 97 + u] = fmaf(ga[k], px, gx[k]);
        vrow[p * 97 + 32 + u] = fmaf(ga[k], py, gy[k]);
        vrow[p * 97 + 64 + u] = ga[k];
      }
      tc::fence_before_sync();
      __syncthreads();
      tc_colsum<NT>(vrow, 97, 96, sGacc);
    }
    mark(16);
    ++ph_tile;
  }

  // =================== per-CTA outputs ===================
  // parameter-gradient accumulators (TMEM, M = 128: row m = lane m; rows
  // 0..31 / 32..63 / 64..95 = G parts h / m / l, columns [0,32) [32,64) [64,96)
  // = X parts h / m / l) -> smem [128][97] -> the six-term sum
  float* scr = reinterpret_cast<float*>(bufA);
  for (int l = 1; l <= NL; ++l) {
    tc::fence_after_sync();
    if (warp < 4 && !first_grad) {
      float v0[16], v1[16], v2[16];
      const uint32_t col = tmem + lane_q + kTcAccCol + kTcDCols * (l - 1);
#pragma unroll 1
      for (int h2 = 0; h2 < 2; ++h2) {
        tc::tmem_ld3x16_wait(col + 16 * h2, col + 32 + 16 * h2, col + 64 + 16 * h2, v0, v1, v2);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          scr[p * 97 + 16 * h2 + k] = v0[k];
          scr[p * 97 + 32 + 16 * h2 + k] = v1[k];
          scr[p * 97 + 64 + 16 * h2 + k] = v2[k];
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    const int fo = net.out_w[l], fi = net.in_w[l];
    for (int e = tid; e < fo * (fi + 1); e += NT) {
      const int o = e / (fi + 1), i = e - o * (fi + 1);
      float g = 0.f;
      if (!first_grad)
        g = ((scr[o * 97 + i] + scr[o * 97 + 32 + i]) + (scr[o * 97 + 64 + i] + scr[(32 + o) * 97 + i])) +
            (scr[(32 + o) * 97 + 32 + i] + scr[(64 + o) * 97 + i]);
      const int idx = (i < fi) ? net.w_off[l] + o * fi + i : net.b_off[l] + o;
      a.grad_part[(size_t)idx * a.part_stride + blockIdx.x] = g;
    }
    __syncthreads();
  }
  for (int i = tid; i < H; i += NT) {
    a.grad_part[(size_t)(net.w_off[0] + 2 * i) * a.part_stride + blockIdx.x] = sGacc[kGaW0x + i];
    a.grad_part[(size_t)(net.w_off[0] + 2 * i + 1) * a.part_stride + blockIdx.x] = sGacc[kGaW0y + i];
    a.grad_part[(size_t)(net.b_off[0] + i) * a.part_stride + blockIdx.x] = sGacc[kGaB0 + i];
    a.grad_part[(size_t)(net.w_off[D] + i) * a.part_stride + blockIdx.x] = sGacc[kGaWd + i];
  }
  if (tid == 0) {
    a.grad_part[(size_t)net.b_off[D] * a.part_stride + blockIdx.x] = sGacc[kGaWd + H];
    for (int e = net.scal_off; e < net.n_params; ++e) a.grad_part[(size_t)e * a.part_stride + blockIdx.x] = 0.f;
  }
  const int any_bad = __syncthreads_or(bad);
  if (tid == 0) {
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
    tc::tmem_dealloc(tmem, kTcCols);
  }
}

}  // namespace vpg
