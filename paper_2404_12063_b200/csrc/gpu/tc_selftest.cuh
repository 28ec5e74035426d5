// Known-answer probe of the three tcgen05 GEMM shapes the tensor-core MLP
// uses (one CTA, 128 threads), bf16x3 split / six products throughout:
//   mode 0  forward      out[p][o] = sum_i A[p][i] W[o][i]   (K-major A, K-major B, N = 96 h|m|l)
//   mode 1  propagation  out[p][i] = sum_o A[p][o] W[o][i]   (K-major A, MN-major B)
//   mode 2  param grad   out[o][i] = sum_p A[p][o] H[p][i]   (MN-major A, M = 128 h|m|l|-; MN-major B)
// A and H are [128][32], W is [32][32], all row-major fp32.  out needs
// 128*32 + 128*96 floats (the raw accumulator follows the result).
#pragma once

#include "tc_utils.cuh"

namespace vpg {

constexpr int kTcProbeSmem = 24576 * 2 + 6144 + 8192 + 1024 + 64;

__global__ void __launch_bounds__(128, 1) tc_probe_kernel(int mode, const float* __restrict__ A,
                                                          const float* __restrict__ W,
                                                          const float* __restrict__ H, float* __restrict__ out) {
  extern __shared__ __align__(1024) char tp_raw[];
  char* base = tp_raw + ((1024u - (smem_u32(tp_raw) & 1023u)) & 1023u);
  char* a_t = base;                   // 3 part tiles of [128][32]
  char* h_t = base + 24576;           // 3 part tiles
  char* w_t = base + 2 * 24576;       // [96][32]: W h | m | l rows
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 2 * 24576 + 6144 + 8192);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;

  if (warp == 0) tc::tmem_alloc(tslot, 128);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int c = 0; c < 4; ++c) {
    tc::st_split8(a_t, 8192, tid, c, A + tid * 32 + 8 * c);
    tc::st_split8(h_t, 8192, tid, c, H + tid * 32 + 8 * c);
    if (tid < 32) tc::st_split8(w_t, 2048, tid, c, W + tid * 32 + 8 * c);
  }
  tc::fence_smem_to_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    const uint32_t sa = smem_u32(a_t), sh = smem_u32(h_t), sw = smem_u32(w_t);
    if (mode == 0 || mode == 1) {
      const int mn = mode == 1;
      for (int part = 0; part < 3; ++part) {
        const uint32_t idesc = tc::idesc_bf16(128, 96 - 32 * part, 0, mn);
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t bd = mn ? tc::mndesc(sw + 1024 * ks, 2048) : tc::kdesc(sw + 32 * ks);
          tc::mma_bf16(tmem, tc::kdesc(sa + part * 8192 + 32 * ks), bd, idesc, (part > 0 || ks > 0) ? 1u : 0u);
        }
      }
    } else if (mode == 4) {
      // layout probe: one M = 64 chain, A MN-major (M blocks = A parts h | m),
      // B = H part h (N = 32), K = 128 points; the raw TMEM dump shows where
      // the 64 rows land
      const uint32_t idesc = tc::idesc_bf16(64, 32, 1, 1);
      for (int kp = 0; kp < 8; ++kp)
        tc::mma_bf16(tmem, tc::mndesc(sa + 1024 * kp, 8192), tc::mndesc(sh + 1024 * kp, 8192), idesc, kp > 0);
    } else if (mode == 5) {
      // the same M = 64 chain addressed at TMEM lane 16
      const uint32_t idesc = tc::idesc_bf16(64, 32, 1, 1);
      for (int kp = 0; kp < 8; ++kp)
        tc::mma_bf16(tmem + (16u << 16), tc::mndesc(sa + 1024 * kp, 8192), tc::mndesc(sh + 1024 * kp, 8192), idesc,
                     kp > 0);
    } else if (mode == 3) {
      // scale-input-d: the forward product twice, the second pass scaling the
      // accumulated first pass by 2^-2 on its first MMA: D = AW^T / 4 + AW^T
      const uint32_t idesc = tc::idesc_bf16(128, 32, 0, 0);
      for (int pass = 0; pass < 2; ++pass)
        for (int pr = 0; pr < 6; ++pr) {
          const uint32_t bb = sw + tc::kProdB[pr] * 2048;
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t ad = tc::kdesc(sa + tc::kProdA[pr] * 8192 + 32 * ks), bd = tc::kdesc(bb + 32 * ks);
            if (pass == 1 && pr == 0 && ks == 0)
              tc::mma_f16_sd(tmem, ad, bd, idesc, 2);
            else
              tc::mma_bf16(tmem, ad, bd, idesc, (pass > 0 || pr > 0 || ks > 0) ? 1u : 0u);
          }
        }
    } else {
      const uint32_t idesc = tc::idesc_bf16(128, 96, 1, 1);
      for (int kp = 0; kp < 8; ++kp)
        tc::mma_bf16(tmem, tc::mndesc(sa + 1024 * kp, 8192), tc::mndesc(sh + 1024 * kp, 8192), idesc, kp > 0);
    }
    tc::mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc::fence_after_sync();
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  float v0[16], v1[16], v2[16], v3[16], v4[16], v5[16];
  tc::tmem_ld3x16_wait(tmem + lane_base + 0, tmem + lane_base + 32, tmem + lane_base + 64, v0, v1, v2);
  tc::tmem_ld3x16_wait(tmem + lane_base + 16, tmem + lane_base + 48, tmem + lane_base + 80, v3, v4, v5);
  float* raw = out + 128 * 32;  // [128][96]
  for (int i = 0; i < 16; ++i) {
    raw[tid * 96 + i] = v0[i];
    raw[tid * 96 + 16 + i] = v3[i];
    raw[tid * 96 + 32 + i] = v1[i];
    raw[tid * 96 + 48 + i] = v4[i];
    raw[tid * 96 + 64 + i] = v2[i];
    raw[tid * 96 + 80 + i] = v5[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (mode == 3) {
    for (int i = 0; i < 32; ++i) out[tid * 32 + i] = raw[tid * 96 + i];
  } else if (mode != 2) {
    for (int i = 0; i < 32; ++i) out[tid * 32 + i] = raw[tid * 96 + i] + raw[tid * 96 + 32 + i] + raw[tid * 96 + 64 + i];
  } else {
    for (int e = tid; e < 32 * 32; e += 128) {
      const int o = e / 32, i = e % 32;
      out[e] = raw[o * 96 + i] + raw[o * 96 + 32 + i] + raw[o * 96 + 64 + i] + raw[(32 + o) * 96 + i] +
               raw[(32 + o) * 96 + 32 + i] + raw[(64 + o) * 96 + i];
    }
  }
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 128);
  }
}

}  // namespace vpg
