// Known-answer probe of the three tcgen05 GEMM shapes the tensor-core MLP
// uses (one CTA, 128 threads), 3xTF32 throughout:
//   mode 0  forward      out[p][o] = sum_i A[p][i] W[o][i]   (K-major A, K-major B, N = 64 hi|lo)
//   mode 1  propagation  out[p][i] = sum_o A[p][o] W[o][i]   (K-major A, MN-major B)
//   mode 2  param grad   out[o][i] = sum_p A[p][o] H[p][i]   (MN-major A, M = 64 hi|lo; MN-major B)
// A and H are [128][32], W is [32][32], all row-major fp32.
#pragma once

#include "tc_utils.cuh"

namespace vpg {

constexpr int kTcProbeSmem = 6 * 16384 + 8192 + 1024 + 64;

__global__ void __launch_bounds__(128, 1) tc_probe_kernel(int mode, const float* __restrict__ A,
                                                          const float* __restrict__ W,
                                                          const float* __restrict__ H, float* __restrict__ out) {
  extern __shared__ __align__(1024) char tp_raw[];
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(tp_raw) + 1023) & ~uintptr_t(1023));
  char* a_hi = base;
  char* a_lo = base + 16384;
  char* h_hi = base + 2 * 16384;
  char* h_lo = base + 3 * 16384;
  char* wbuf = base + 4 * 16384;  // rows 0..31 hi, 32..63 lo
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 4 * 16384 + 8192);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) tc::tmem_alloc(tslot, 128);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  // operand tiles (row = tid)
  for (int c = 0; c < 32; c += 4) {
    const float* ar = A + tid * 32 + c;
    tc::st_split4(a_hi, a_lo, tid, c, ar[0], ar[1], ar[2], ar[3]);
    if (mode == 2) {
      const float* hr = H + tid * 32 + c;
      tc::st_split4(h_hi, h_lo, tid, c, hr[0], hr[1], hr[2], hr[3]);
    }
    if (tid < 32) {
      const float* wr = W + tid * 32 + c;
      tc::st_split4(wbuf, wbuf + 4096, tid, c, wr[0], wr[1], wr[2], wr[3]);
    }
  }
  tc::fence_smem_to_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo), sh_hi = smem_u32(h_hi), sw = smem_u32(wbuf);
    if (mode == 0) {
      const uint32_t i64 = tc::idesc_tf32(128, 64, 0, 0), i32 = tc::idesc_tf32(128, 32, 0, 0);
      for (int ks = 0; ks < 4; ++ks)
        tc::mma_tf32(tmem, tc::sdesc(sa_hi + 32 * ks, 16, 1024), tc::sdesc(sw + 32 * ks, 16, 1024), i64, ks > 0);
      for (int ks = 0; ks < 4; ++ks)
        tc::mma_tf32(tmem, tc::sdesc(sa_lo + 32 * ks, 16, 1024), tc::sdesc(sw + 32 * ks, 16, 1024), i32, 1);
    } else if (mode == 1) {
      const uint32_t i64 = tc::idesc_tf32(128, 64, 0, 1), i32 = tc::idesc_tf32(128, 32, 0, 1);
      for (int ks = 0; ks < 4; ++ks)
        tc::mma_tf32(tmem, tc::sdesc(sa_hi + 32 * ks, 16, 1024), tc::sdesc(sw + 1024 * ks, 4096, 1024), i64,
                     ks > 0);
      for (int ks = 0; ks < 4; ++ks)
        tc::mma_tf32(tmem, tc::sdesc(sa_lo + 32 * ks, 16, 1024), tc::sdesc(sw + 1024 * ks, 4096, 1024), i32, 1);
    } else {
      const uint32_t i6464 = tc::idesc_tf32(64, 64, 1, 1);
      for (int ks = 0; ks < 16; ++ks)
        tc::mma_tf32(tmem, tc::sdesc(sa_hi + 1024 * ks, sa_lo - sa_hi, 1024),
                     tc::sdesc(sh_hi + 1024 * ks, smem_u32(h_lo) - sh_hi, 1024), i6464, ks > 0);
    }
    tc::mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc::fence_after_sync();
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  float v0[16], v1[16], v2[16], v3[16];
  tc::tmem_ld2x16_wait(tmem + lane_base + 0, tmem + lane_base + 16, v0, v1);
  tc::tmem_ld2x16_wait(tmem + lane_base + 32, tmem + lane_base + 48, v2, v3);
  if (mode != 2) {
    for (int i = 0; i < 16; ++i) {
      out[tid * 32 + i] = v0[i] + v2[i];
      out[tid * 32 + 16 + i] = v1[i] + v3[i];
    }
  } else if (lane < 16) {
    // M = 64 accumulator: row m = 16 * warp + lane (rows 32..63 = lo part of A)
    const int m = 16 * warp + lane;
    float* o = out + 128 * 32;  // raw 64 x 64 block after the first 128*32 floats
    for (int i = 0; i < 16; ++i) {
      o[m * 64 + i] = v0[i];
      o[m * 64 + 16 + i] = v1[i];
      o[m * 64 + 32 + i] = v2[i];
      o[m * 64 + 48 + i] = v3[i];
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (mode == 2) {
    const float* o = out + 128 * 32;
    __threadfence_block();
    for (int e = tid; e < 32 * 32; e += 128) {
      const int r = e / 32, c = e % 32;
      out[e] = o[r * 64 + c] + o[r * 64 + 32 + c] + o[(32 + r) * 64 + c];
    }
  }
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 128);
  }
}

}  // namespace vpg
