// Device-side premultiplier assembly (assemble.cu): the launcher shared by
// vpinn_gpu_create (assembly straight into the context's buffers) and the
// standalone vpinn_gpu_assemble probe.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace vpg {

// named fields of the host library (vp_problem.hpp:22-62)
enum : int {
  kFieldZero = 0,
  kFieldOne,
  kFieldSin2piU,
  kFieldSin2piF,
  kFieldSin4piU,
  kFieldSin4piF,
  kFieldSin8piU,
  kFieldSin8piF,
  kFieldGearF,
  kFieldBumpU,
  kFieldBumpF,
  kFieldSinpiU,
  kFieldSincosEps,
  kFieldSinpiVarepsF,
  kFieldCount
};

// device-resident inputs (small: mesh, rule, basis tables)
struct AsmInput {
  const double* nodes;   // [n_nodes][2]
  const int32_t* elems;  // [n_elem][4], CCW
  int T, Q;
  const double* xi;
  const double* eta;
  const double* w;
  const double* bval;  // [T][Q]
  const double* bdxi;
  const double* bdeta;
  int field;  // forcing field id
};

// assemble cells [e0, e0 + E) into gx/gy/tv ([E][T][Q]), forcing ([E][T]),
// quadrature points qp (double [E*Q][2]) / qpf (float2), all optional except
// gx/gy; tv is required when forcing is assembled; fq_scratch (E*Q floats)
// receives (float)f at the points when non-null (required with forcing); *bad receives the smallest degenerate global cell index (atomicMin)
cudaError_t assemble_on_device(const AsmInput& in, int64_t e0, int E, float* gx, float* gy, float* tv,
                               float* forcing, double* qp, float2* qpf, float* fq_scratch, int* bad,
                               cudaStream_t s);

}  // namespace vpg
