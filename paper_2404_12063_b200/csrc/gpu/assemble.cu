// Device-side premultiplier assembly: the reference's
// assemble_element_tensors / assemble_forcing (assembly.hpp:58-135) from the
// mesh, the reference quadrature rule and the reference-square basis tables,
// without building or uploading the E*T*Q host tensors.
//
// Bit-exactness with the host path (csrc/host/vp_problem.hpp:88-149, itself
// the same bits as the oracle): this translation unit is compiled with
// --fmad=false, so every expression below is evaluated in IEEE double in the
// host's source order (the host is built with -ffp-contract=off) and cast to
// float with round-to-nearest, exactly like static_cast<float>.  The forcing
// field is evaluated on the device in double (sin/cos/exp/... from the CUDA
// math library, <= 2 ulp in double), cast to float and summed in float in q
// order like the host; a float difference needs the double value within ~2
// ulp of a float rounding boundary (tested: identical on the parity meshes).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "assemble.h"

namespace vpg {
namespace {

struct AsmArgs {
  const double* nodes;     // [n][2]
  const int32_t* elems;    // [E][4]
  int64_t e0;              // first (global) cell of this launch
  int E, T, Q;
  const double* xi;        // [Q]
  const double* eta;
  const double* w;
  const double* bval;      // [T][Q]
  const double* bdxi;
  const double* bdeta;
  float* gx;               // [E][T][Q] (local cells)
  float* gy;
  float* tv;               // may be null (no convection) unless forcing is assembled
  double* qp;              // [E*Q][2] quadrature points (double), may be null
  float2* qpf;             // [E*Q] quadrature points cast to float (the evaluation batch), may be null
  float* fq;               // [E*Q] float(f(x_kq)) scratch
  int field;               // forcing field id, -1: none
  int* bad;                // first degenerate cell (global index), INT_MAX if none
};

// the host's named field library (vp_problem.hpp:22-62), in double
__device__ double eval_field(int id, double x, double y) {
  const double w1 = 2.0 * M_PI;
  switch (id) {
    case kFieldZero:
      return 0.0;
    case kFieldOne:
      return 1.0;
    case kFieldSin2piU:
      return -sin(w1 * x) * sin(w1 * y);
    case kFieldSin2piF:
      return -2.0 * w1 * w1 * sin(w1 * x) * sin(w1 * y);
    case kFieldSin4piU: {
      const double w = 2.0 * w1;
      return -sin(w * x) * sin(w * y);
    }
    case kFieldSin4piF: {
      const double w = 2.0 * w1;
      return -2.0 * w * w * sin(w * x) * sin(w * y);
    }
    case kFieldSin8piU: {
      const double w = 4.0 * w1;
      return -sin(w * x) * sin(w * y);
    }
    case kFieldSin8piF: {
      const double w = 4.0 * w1;
      return -2.0 * w * w * sin(w * x) * sin(w * y);
    }
    case kFieldGearF:
      return 50.0 * sin(x) + cos(x);
    case kFieldBumpU:
      return 10.0 * sin(x) * tanh(x) * exp(-0.3 * x * x);
    case kFieldBumpF: {
      const double sx = sin(x), cx = cos(x), sh = sinh(2.0 * x), ch = cosh(x), th = tanh(x);
      const double num = -9.0 * x * x * sx * sh + 60.0 * x * sx + 30.0 * x * cx * sh + 40.0 * sx * sh +
                         100.0 * sx * th - 100.0 * cx;
      return 3.0 * num * exp(-0.3 * x * x) / (50.0 * ch * ch);
    }
    case kFieldSinpiU:
      return sin(M_PI * x) * sin(M_PI * y);
    case kFieldSincosEps:
      return 0.5 * (sin(x) + cos(y));
    case kFieldSinpiVarepsF: {
      const double sx = sin(M_PI * x), cx = cos(M_PI * x);
      const double sy = sin(M_PI * y), cy = cos(M_PI * y);
      return 0.5 * M_PI *
             (2.0 * M_PI * (sin(x) + cos(y)) * sx * sy + sin(y) * sx * cy - sy * cos(x) * cx + 2.0 * sy * cx);
    }
    default:
      return 0.0;
  }
}

// one thread per (local cell k, quadrature point q): bilinear map, Jacobian,
// the T premultiplier entries of each tensor (coalesced over q for fixed j),
// the quadrature point and the forcing field value there
__global__ void assemble_tensors_kernel(const AsmArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)a.E * a.Q) return;
  const int k = (int)(i / a.Q), q = (int)(i - (int64_t)k * a.Q);
  const int64_t kg = a.e0 + k;
  const int4 e = reinterpret_cast<const int4*>(a.elems)[kg];
  const double2 A = reinterpret_cast<const double2*>(a.nodes)[e.x];
  const double2 B = reinterpret_cast<const double2*>(a.nodes)[e.y];
  const double2 Cn = reinterpret_cast<const double2*>(a.nodes)[e.z];
  const double2 Dn = reinterpret_cast<const double2*>(a.nodes)[e.w];
  // bilinear_coeffs (geometry.hpp:75-113)
  const double xc0 = 0.25 * (A.x + B.x + Cn.x + Dn.x);
  const double xc1 = 0.25 * (-A.x + B.x + Cn.x - Dn.x);
  const double xc2 = 0.25 * (-A.x - B.x + Cn.x + Dn.x);
  const double xc3 = 0.25 * (A.x - B.x + Cn.x - Dn.x);
  const double yc0 = 0.25 * (A.y + B.y + Cn.y + Dn.y);
  const double yc1 = 0.25 * (-A.y + B.y + Cn.y - Dn.y);
  const double yc2 = 0.25 * (-A.y - B.y + Cn.y + Dn.y);
  const double yc3 = 0.25 * (A.y - B.y + Cn.y - Dn.y);
  const double xi = a.xi[q], eta = a.eta[q];
  // jacobian_at
  const double j11 = xc1 + xc3 * eta;
  const double j12 = yc1 + yc3 * eta;
  const double j21 = xc2 + xc3 * xi;
  const double j22 = yc2 + yc3 * xi;
  const double det = j11 * j22 - j12 * j21;
  if (!(det > 0.0)) atomicMin(a.bad, (int)kg);
  // map_point
  const double px = xc0 + xc1 * xi + xc2 * eta + xc3 * xi * eta;
  const double py = yc0 + yc1 * xi + yc2 * eta + yc3 * xi * eta;
  if (a.qp) reinterpret_cast<double2*>(a.qp)[i] = make_double2(px, py);
  if (a.qpf) a.qpf[i] = make_float2((float)px, (float)py);
  if (a.field >= 0) a.fq[i] = (float)eval_field(a.field, px, py);
  const double wdet = a.w[q] * det;
  const double inv = 1.0 / det;
  const size_t base = (size_t)k * a.T * a.Q + q;
  for (int j = 0; j < a.T; ++j) {
    const int bj = j * a.Q + q;
    const double bdx = a.bdxi[bj], bde = a.bdeta[bj];
    const double dx = (j22 * bdx - j12 * bde) * inv;
    const double dy = (-j21 * bdx + j11 * bde) * inv;
    const size_t at = base + (size_t)j * a.Q;
    a.gx[at] = (float)(wdet * dx);
    a.gy[at] = (float)(wdet * dy);
    if (a.tv) a.tv[at] = (float)(wdet * a.bval[bj]);
  }
}

// forcing(k, j) = sum_q test(k, j, q) * fq(k, q), summed in q order in float
__global__ void assemble_forcing_kernel(const float* tv, const float* fq, float* forcing, int E, int T, int Q) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)E * T) return;
  const int64_t k = i / T;
  const float* row = tv + i * Q;
  const float* f = fq + k * Q;
  float acc = 0.0f;
  for (int q = 0; q < Q; ++q) acc += row[q] * f[q];
  forcing[i] = acc;
}

}  // namespace

cudaError_t assemble_on_device(const AsmInput& in, int64_t e0, int E, float* gx, float* gy, float* tv,
                               float* forcing, double* qp, float2* qpf, float* fq_scratch, int* bad,
                               cudaStream_t s) {
  AsmArgs a{};
  a.nodes = in.nodes;
  a.elems = in.elems;
  a.e0 = e0;
  a.E = E;
  a.T = in.T;
  a.Q = in.Q;
  a.xi = in.xi;
  a.eta = in.eta;
  a.w = in.w;
  a.bval = in.bval;
  a.bdxi = in.bdxi;
  a.bdeta = in.bdeta;
  a.gx = gx;
  a.gy = gy;
  a.tv = tv;
  a.qp = qp;
  a.qpf = qpf;
  a.fq = fq_scratch;
  a.field = fq_scratch ? in.field : -1;  // f at the points when a scratch is given
  a.bad = bad;
  const int64_t n = (int64_t)E * in.Q;
  if (n > 0) {
    assemble_tensors_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  if (forcing && E > 0) {
    const int64_t m = (int64_t)E * in.T;
    assemble_forcing_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(tv, fq_scratch, forcing, E, in.T, in.Q);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace vpg
