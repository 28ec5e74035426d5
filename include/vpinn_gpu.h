/*
 * vpinn_gpu.h — C-ABI of the B200 FastVPINNs training step.
 *
 * Drop-in boundary for the reference's C++ loss/trainer path
 * (reference proj/include/vpinn/, header-only, no FFI of its own).  Each
 * entry point names the reference code it replaces:
 *
 *   vpinn_gpu_create          ProblemAssembly upload (trainer.hpp:180-210,
 *                             layouts of assembly.hpp:34-54) + network
 *                             (network.hpp:42-62)
 *   vpinn_gpu_set/get_params  from_parameters / to_parameters
 *                             (network.hpp:98-128)
 *   vpinn_gpu_loss_and_grad   loss_and_parameter_gradient with the
 *                             CompositeObjective, tensor kernel
 *                             (network.hpp:508-531, trainer.hpp:215-268,
 *                             losses.hpp:91-168, 406-415)
 *   vpinn_gpu_train           the train() epoch loop body: lr_at + loss and
 *                             gradient + adam_step + from_parameters, with
 *                             the history/convergence rules
 *                             (trainer.hpp:275-382, 34-59, 73-78)
 *   vpinn_gpu_forward         evaluate(net, points, order) (network.hpp:414-449)
 *   vpinn_gpu_contract        variational_loss_tensor on caller-supplied
 *                             derivatives (losses.hpp:91-168)
 *
 * Conventions
 *   - plain pointers and sizes only; every host array is COPIED at create
 *     time and may be freed afterwards;
 *   - return value 0 = ok, otherwise the reference ErrorCategory code
 *     (core.hpp:17-22): 2 config, 3 mesh, 4 numeric, 5 io; 6 = device/CUDA
 *     failure (no reference equivalent: the reference has no device);
 *   - vpinn_gpu_last_error() returns the message of the last failure on the
 *     calling thread;
 *   - one context owns one device stream; calls on one context are
 *     serialised by the caller (not thread-safe), distinct contexts may be
 *     driven from distinct threads;
 *   - there is NO CPU fallback: without a usable sm_100 device every call
 *     returns 6.
 */
#ifndef VPINN_GPU_H
#define VPINN_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPINN_OK 0
#define VPINN_ERR_CONFIG 2
#define VPINN_ERR_MESH 3
#define VPINN_ERR_NUMERIC 4
#define VPINN_ERR_IO 5
#define VPINN_ERR_DEVICE 6

/* EpsSource (losses.hpp:22-26) */
#define VPINN_EPS_FIXED 0
#define VPINN_EPS_SCALAR 1
#define VPINN_EPS_SPATIAL 2

/* LossForm (trainer.hpp:178) */
#define VPINN_FORM_WEAK 0
#define VPINN_FORM_STRONG 1

/* Activation (network.hpp:31) */
#define VPINN_ACT_TANH 0
#define VPINN_ACT_SIGMOID 1

typedef struct vpinn_gpu_ctx vpinn_gpu_ctx;

/* Everything one step needs, in the reference layouts (host memory). */
/* Device-side assembly input (replaces the host's
 * assemble_element_tensors / assemble_forcing, reference
 * proj/include/vpinn/assembly.hpp:58-135): the mesh, the reference
 * tensor-product quadrature rule and the reference-square basis tables
 * (basis.hpp:24-60, row j = jy*n + jx), from which the device builds the
 * premultiplier tensors, the forcing and the interior quadrature points,
 * bit-identical to the host path (double geometry, cast at store). */
typedef struct vpinn_gpu_assembly {
  int64_t n_nodes;
  const double* nodes;     /* [n_nodes][2] */
  const int32_t* elements; /* [n_elem][4], counter-clockwise */
  const double* xi;        /* [n_quad] */
  const double* eta;       /* [n_quad] */
  const double* weights;   /* [n_quad] */
  const double* basis_val; /* [n_test][n_quad] */
  const double* basis_dxi;
  const double* basis_deta;
  const char* forcing; /* named field of the host library (zero, one, sin2pi_f, gear_f, ...) */
} vpinn_gpu_assembly;

typedef struct vpinn_gpu_problem {
  /* ElementTensors<float> (assembly.hpp:34-54): slices [k][j][q] row-major,
   * entry (k*n_test + j)*n_quad + q.  test may be NULL when there is no
   * convection term. */
  int32_t n_elem, n_test, n_quad;
  const float* grad_x;
  const float* grad_y;
  const float* test;
  /* Eigen column-major n_test x n_elem: entry k*n_test + j */
  const float* forcing;
  /* Evaluation batch [interior | boundary | sensors] as double (x,y) pairs
   * (trainer.hpp:199-209); interior = n_elem*n_quad element-major points. */
  const double* points;
  int64_t n_interior, n_boundary, n_sensors;
  const double* boundary_values; /* n_boundary, may be NULL if 0 */
  const double* sensor_values;   /* n_sensors, may be NULL if 0 */
  /* DenseNetwork shape: layer_sizes[0] == 2, all hidden widths equal or
   * smaller than the widest (narrower layers are zero-padded exactly). */
  int32_t n_layer_sizes;
  const int32_t* layer_sizes;
  int32_t activation;
  int32_t n_scalars; /* trainable scalars appended to the parameter vector */
  /* PdeCoefficients<float> (losses.hpp:28-41) and LossWeights (471-474) */
  float eps, bx, by;
  int32_t eps_source;
  int32_t eps_scalar_index;
  double tau, gamma;
  /* device ordinal; rank/world partition cells and penalty points
   * contiguously (rank r owns [floor(r*N/W), floor((r+1)*N/W))) */
  int32_t device;
  int32_t rank, world_size;
  /* non-NULL: tensors, forcing and the interior points are assembled on the
   * device from this input; grad_x/grad_y/test/forcing are then ignored and
   * points holds only [boundary | sensors] (n_interior = n_elem*n_quad) */
  const vpinn_gpu_assembly* assembly;
  /* LossForm (trainer.hpp:178, 246-248).  VPINN_FORM_STRONG replaces the
   * variational residual by the strong-form collocation residual at the
   * interior points (strong_residual_loss, losses.hpp:422-467) with order-2
   * network derivatives; grad_x/grad_y/test/forcing are then unused and
   * strong_forcing holds f at the n_interior points (commands.hpp:147-152,
   * cast to float), or is NULL with assembly set (f evaluated on the device
   * at the assembled points).  Hidden widths <= 32, one output channel,
   * fixed or scalar eps. */
  int32_t form;
  const float* strong_forcing;
} vpinn_gpu_problem;

/* TrainConfig subset (trainer.hpp:64-97) */
typedef struct vpinn_gpu_train_spec {
  int64_t iterations;
  int32_t lr_exponential; /* LrMode: 0 constant, 1 exponential */
  double lr0, decay;
  int32_t every;
  int32_t has_eps_abs_tol, has_eps_actual, has_loss_tol;
  double eps_abs_tol, eps_actual, loss_tol;
  int32_t plateau_window;
  int32_t steps_per_graph; /* steps captured per CUDA-graph launch (0 = auto) */
} vpinn_gpu_train_spec;

/* Per-step record produced by vpinn_gpu_train (all steps, caller picks the
 * history rows exactly like trainer.hpp:339-341). */
typedef struct vpinn_gpu_step_record {
  double total, variational, boundary, sensor;
  double lr;
  double eps;     /* trainable coefficient after the update, NaN if none */
  double seconds; /* device-timestamped step duration */
} vpinn_gpu_step_record;

typedef struct vpinn_gpu_train_result {
  int64_t steps_run;
  int32_t converged;
  int32_t stop_reason; /* 0 iteration budget, 1 coefficient within
                          tolerance, 2 loss plateau */
  int64_t abort_step;  /* 1-based step of a TrainingAbortError, else 0 */
  double final_eps;
} vpinn_gpu_train_result;

const char* vpinn_gpu_last_error(void);
const char* vpinn_gpu_version(void);
/* Name of the kernel that runs the epoch's fused step on this context
 * (tensor-core or CUDA-core variant; diagnostics and bench reporting). */
const char* vpinn_gpu_step_kernel(const vpinn_gpu_ctx* ctx);

/* 1 if a device the kernels were built for is present, else 0. */
int vpinn_gpu_device_ok(void);

/* The multi-GPU partition vpinn_gpu_create applies (pure host function):
 * out6 = {e0, e1, b0, b1, s0, s1}, rank owns cells [e0, e1), boundary
 * points [b0, b1), sensors [s0, s1): floor(r*N/W) .. floor((r+1)*N/W). */
void vpinn_gpu_partition(int64_t n_elem, int64_t n_boundary, int64_t n_sensors, int rank, int world,
                         int64_t* out6);

/* Uploads this rank's share of the problem's host arrays.  Arrays in
 * page-locked memory (cudaHostAlloc / cudaHostRegister) are DMA'd straight
 * from the caller's buffers at the link rate; pageable arrays of 4 MB or more
 * are staged through a process-wide pinned ring filled by a host thread pool.
 * The arrays are not referenced after the call returns. */
int vpinn_gpu_create(const vpinn_gpu_problem* problem, vpinn_gpu_ctx** out);
void vpinn_gpu_destroy(vpinn_gpu_ctx* ctx);

int vpinn_gpu_param_count(const vpinn_gpu_ctx* ctx);
int vpinn_gpu_set_params(vpinn_gpu_ctx* ctx, const float* params, int n);
int vpinn_gpu_get_params(vpinn_gpu_ctx* ctx, float* params, int n);

/* Forward + CompositeObjective + reverse, no optimiser.  loss_parts[4] =
 * {total, variational, boundary, sensor}; grad (n_params, may be NULL) in
 * to_parameters order; all after the cross-rank sum when a communicator is
 * attached. */
int vpinn_gpu_loss_and_grad(vpinn_gpu_ctx* ctx, double* loss_parts, double* grad);

/* Fresh AdamState + the epoch loop (trainer.hpp:294-370).  records has
 * room for spec->iterations entries (may be NULL). */
int vpinn_gpu_train(vpinn_gpu_ctx* ctx, const vpinn_gpu_train_spec* spec,
                    vpinn_gpu_step_record* records, vpinn_gpu_train_result* result);

/* Run n_steps further epochs of the current run with a constant learning
 * rate and NO host synchronisation (benchmark primitive; Adam state
 * persists across calls, reset by vpinn_gpu_train or vpinn_gpu_adam_reset).
 * After vpinn_gpu_train the finished run's stop (budget, tolerance, plateau)
 * is lifted and the epochs continue from its Adam state with no stop
 * criteria; after a train() that aborted (non-finite values) run_steps
 * returns VPINN_ERR_NUMERIC until vpinn_gpu_adam_reset. */
int vpinn_gpu_adam_reset(vpinn_gpu_ctx* ctx);
int vpinn_gpu_run_steps(vpinn_gpu_ctx* ctx, int n_steps, double lr);
int vpinn_gpu_synchronize(vpinn_gpu_ctx* ctx);
/* Device-side timing of n_steps run_steps epochs (CUDA events on the
 * context stream); ms_total out. */
int vpinn_gpu_time_steps(vpinn_gpu_ctx* ctx, int n_steps, double lr, double* ms_total);

/* evaluate(): order 0 or 1 at n arbitrary points (double x,y pairs).
 * u mandatory, du_dx/du_dy used when order >= 1, eps when the network has a
 * second output channel (softplus head).  NULL outputs are skipped. */
int vpinn_gpu_forward(vpinn_gpu_ctx* ctx, const double* points, int64_t n, int order,
                      float* u, float* du_dx, float* du_dy, float* eps);

/* variational_loss_tensor on caller-supplied interior derivatives
 * (n_elem*n_quad each; eps for the spatial source; scalars for the scalar
 * source).  Outputs: loss, residuals (n_test x n_elem column-major, may be
 * NULL), adjoints (may be NULL), scalar_bar (n_scalars, may be NULL). */
/* evaluate(net, points, 2) (network.hpp:414-449): u, first and second
 * derivatives at n points; NULL outputs skipped.  Strong-form contexts only
 * (the order-2 kernel is the strong-form one). */
int vpinn_gpu_forward2(vpinn_gpu_ctx* ctx, const double* points, int64_t n, float* u, float* du_dx,
                       float* du_dy, float* d2u_dx2, float* d2u_dy2);

int vpinn_gpu_contract(vpinn_gpu_ctx* ctx, const float* du_dx, const float* du_dy,
                       const float* eps, const float* scalars, float weight, double* loss,
                       float* residuals, float* du_dx_bar, float* du_dy_bar, float* eps_bar,
                       double* scalar_bar);

/* Standalone contraction kernel timing (the HBM-roofline report, SURVEY
 * §8d): reps launches on device-resident derivatives, mean ms per launch
 * and the algorithmic bytes per launch. */
int vpinn_gpu_time_contract(vpinn_gpu_ctx* ctx, int reps, double* ms_per_launch,
                            double* bytes_per_launch);
/* The same, also timing the streaming kernel alone (*ms_stream): on the split
 * path (cells larger than a warp's ring) the launch is the row kernel plus the
 * per-cell sum of its partial columns; for whole-cell contexts *ms_stream ==
 * *ms_per_launch.  Diagnostic (bench.py's roofline), replaces nothing in the
 * reference. */
int vpinn_gpu_time_contract_kernels(vpinn_gpu_ctx* ctx, int reps, double* ms_per_launch, double* ms_stream,
                                    double* bytes);

/* Read the uploaded tensors back (layout parity: must equal the host
 * arrays byte for byte).  which: 0 grad_x, 1 grad_y, 2 test, 3 forcing. */
int vpinn_gpu_download_tensor(vpinn_gpu_ctx* ctx, int which, float* out, int64_t n);

/* Kernel-launch accounting (for the bench's gpu_launches claim). */
int64_t vpinn_gpu_launch_count(const vpinn_gpu_ctx* ctx);
/* Per-step share of the step kernels measured with CUDA events on the
 * context stream over reps run_steps: fused (or forward+contract+reverse),
 * reduce, adam — milliseconds per step each.  The parameters, Adam moments
 * and trainer state are saved before and restored after: profiling does not
 * change the run. */
int vpinn_gpu_profile_step(vpinn_gpu_ctx* ctx, int reps, double* ms_mlp, double* ms_reduce,
                           double* ms_adam);

/* Write 256 MB (> the 126 MB L2) on the context stream: benchmarks call it
 * between timed epochs so every epoch streams its tensors from HBM. */
int vpinn_gpu_flush_l2(vpinn_gpu_ctx* ctx);

/* Matrix-free variational contraction: the same outputs
 * as vpinn_gpu_contract (fixed / scalar coefficient, convection) computed
 * from the reference basis tables and the per-cell geometry instead of the
 * premultiplier tensors (~4 (4 Q + T) bytes per cell of HBM traffic instead
 * of 4 n_t T Q).  Needs a context created with an assembly input; fp32, so it
 * matches the tensor contraction to rounding, not bitwise. */
int vpinn_gpu_contract_matrix_free(vpinn_gpu_ctx* ctx, const float* du_dx, const float* du_dy, const float* scalars,
                                   float weight, double* loss, float* residuals, float* du_dx_bar,
                                   float* du_dy_bar, double* scalar_bar);
int vpinn_gpu_time_contract_matrix_free(vpinn_gpu_ctx* ctx, int reps, double* ms_per_launch, double* bytes);

/* TEST HOOKS (parity tests of the alternate code paths; not for production
 * use).  Process-wide, read by every later vpinn_gpu_create:
 *   VPINN_HOOK_CUDA_CORE_STEP  the CUDA-core step kernel (step_kernel.cuh,
 *                              the one serving shapes without a tensor-core
 *                              variant) also for shapes the tensor-core step
 *                              serves, so its parity is tested on them;
 *   VPINN_HOOK_FORCE_SPILL     the tensor-core step spills its TMEM
 *                              parameter-gradient accumulators every tile
 *                              (the rare path of large scale drops);
 *   VPINN_HOOK_THROUGHPUT_LAYOUT  the tensor-core step keeps 16 units per
 *                              thread also on grids of at most one tile per
 *                              SM (where it takes the 8-unit latency layout).
 * 0 restores the defaults. */
#define VPINN_HOOK_CUDA_CORE_STEP 1
#define VPINN_HOOK_FORCE_SPILL 2
#define VPINN_HOOK_THROUGHPUT_LAYOUT 4
int vpinn_gpu_set_test_hooks(int flags);

/* Device buffers released by destroyed contexts are cached per size for
 * the next context (no cudaMalloc / device-synchronizing cudaFree on
 * re-creation); this returns every cached block to the driver. */
int vpinn_gpu_release_cached_memory(void);

/* Device-side assembly as a standalone call (host outputs, each may be NULL
 * except grad_x/grad_y): the same kernels vpinn_gpu_create runs for a
 * problem with an assembly input.  Returns 3 (mesh) for a cell with a
 * non-positive Jacobian determinant (DegenerateElementError, first cell). */
int vpinn_gpu_assemble(int device, int32_t n_elem, int32_t n_test, int32_t n_quad, const vpinn_gpu_assembly* in,
                       float* grad_x, float* grad_y, float* test, float* forcing, double* quad_points);

/* Diagnostics: clock64() phase marks of CTA 0 in the last tensor-core step
 * launch (enabled by VPINN_PHASE_CLOCK=1 in the environment at create;
 * 8 tiles x 32 marks).  Not part of the reference interface. */
int vpinn_gpu_phase_clock(vpinn_gpu_ctx* ctx, long long* out, int n);

/* FP32 FFMA throughput of `device` (TFLOP/s, best of 4 timed launches):
 * the roofline denominator of the FFMA-bound step kernel. */
int vpinn_gpu_measure_ffma_peak(int device, double* tflops);

/* Known-answer probe of the tcgen05 split-bf16 GEMM shapes used by the
 * tensor-core MLP (diagnostic).  A, H: [128][32]; W: [32][32] row-major.
 * mode 0: out[128][32] = A W^T;  mode 1: out[128][32] = A W;
 * mode 2: out[32][32] = A^T H.  out holds 128*32 + 128*96 floats (the raw
 * [128][96] accumulator follows the result). */
int vpinn_gpu_tc_probe(int device, int mode, const float* A, const float* W, const float* H, float* out);

/* Multi-GPU: rank 0 creates an NCCL unique id (128 bytes), every rank
 * attaches with the same id.  One ncclAllReduce(sum, f64) of
 * [gradient | loss parts] per epoch over NVLink. */
int vpinn_gpu_nccl_unique_id(void* id128);
int vpinn_gpu_attach_comm(vpinn_gpu_ctx* ctx, const void* id128, int nranks, int rank);

/* Multi-GPU over peer memory (one process per GPU, CUDA IPC over NVLink /
 * NVSwitch): every rank exports its mailbox (64-byte IPC handle), gathers all
 * ranks' handles in rank order (host plumbing, e.g. a gloo all-gather) and
 * attaches them.  Each epoch's tail is then ONE kernel: this rank's
 * cross-CTA reduction, the rows stored into every rank's mailbox, the
 * cross-rank sum in rank order (bitwise-identical replicas) and Adam --
 * replacing reduce -> ncclAllReduce -> Adam (the reference's train loop,
 * trainer.hpp:316-370, partitioned across ranks).  At most 8 ranks; every
 * rank must run the same epochs (the exchange is a barrier). */
/* (A later vpinn_gpu_attach_comm replaces an attached peer exchange.) */
int vpinn_gpu_peer_handle(vpinn_gpu_ctx* ctx, void* handle64);
int vpinn_gpu_attach_peers(vpinn_gpu_ctx* ctx, const void* handles, int nranks, int rank);

#ifdef __cplusplus
}
#endif

#endif /* VPINN_GPU_H */
