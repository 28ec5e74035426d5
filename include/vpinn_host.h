/*
 * vpinn_host.h — C-ABI of the host pipeline that feeds the B200 step
 * (config -> mesh -> quadrature/basis -> premultiplier assembly -> sampling
 * -> network init), so non-C++ callers (ctypes, the bench, a maintainer's
 * binding) reach the same code the C++ API in csrc/host uses.
 *
 * Reference interfaces mirrored:
 *   vpinn_host_problem_from_config  build_problem(cfg[, premade mesh])
 *                                   (reference proj/include/vpinn/commands.hpp:123-178,
 *                                   parse_config_json config.hpp:297-606)
 *   vpinn_host_problem_view         ProblemAssembly + DenseNetwork as the
 *                                   vpinn_gpu_problem arrays (trainer.hpp:180-210)
 *   vpinn_host_train                run_training_command's train_forward /
 *                                   train_inverse + evaluate_metrics
 *                                   (commands.hpp:202-258, trainer.hpp:275-446)
 *   vpinn_host_bench_case           bench_case (commands.hpp:285-341)
 *   vpinn_host_mesh_*               read_gmsh_file / generate_structured_mesh /
 *                                   skew_mesh_nodes (mesh_io.hpp:264,
 *                                   geometry.hpp:146, commands.hpp:75)
 * Return codes: 0 ok, else ErrorCategory (2 config, 3 mesh, 4 numeric,
 * 5 io, 6 device); message via vpinn_host_last_error().
 */
#ifndef VPINN_HOST_H
#define VPINN_HOST_H

#include <stddef.h>
#include <stdint.h>

#include "vpinn_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vpinn_host_problem vpinn_host_problem;
typedef struct vpinn_host_mesh vpinn_host_mesh;

/* Mesh sources overriding problem.domain (the benchmark's premade meshes). */
#define VPINN_MESH_FROM_CONFIG 0
#define VPINN_MESH_STRUCTURED 1 /* nx, ny, x0,x1,y0,y1, skew, skew_seed */
#define VPINN_MESH_GEAR 2       /* n_r, n_t: gen_fixtures.py gear recipe  */
#define VPINN_MESH_DISK 3       /* n (=nx): elliptical square->disk map    */
#define VPINN_MESH_HANDLE 4     /* an already loaded vpinn_host_mesh       */

typedef struct vpinn_mesh_source {
  int32_t kind;
  int32_t nx, ny;
  double x0, x1, y0, y1;
  double skew;
  uint64_t skew_seed;
  const vpinn_host_mesh* mesh;
} vpinn_mesh_source;

const char* vpinn_host_last_error(void);

/* ---- meshes ---- */
int vpinn_host_mesh_read_gmsh(const char* path, vpinn_host_mesh** out);
int vpinn_host_mesh_parse_gmsh(const char* text, vpinn_host_mesh** out);
int vpinn_host_mesh_make(const vpinn_mesh_source* src, vpinn_host_mesh** out);
/* counts[3] = n_nodes, n_elements, n_boundary_nodes */
void vpinn_host_mesh_counts(const vpinn_host_mesh* m, int64_t* counts);
/* nodes [n][2] (may be NULL), cells [e][4] (may be NULL), boundary ids (may be NULL) */
void vpinn_host_mesh_arrays(const vpinn_host_mesh* m, double* nodes, int32_t* cells, int32_t* boundary);
/* validate_mesh: number of degenerate / misoriented cells */
void vpinn_host_mesh_health(const vpinn_host_mesh* m, int64_t* degenerate, int64_t* misoriented);
void vpinn_host_mesh_free(vpinn_host_mesh* m);
/* MSH 4.1 text of the gear recipe (len excludes the NUL); cap 0 = size query */
int vpinn_host_gear_msh_text(int n_r, int n_t, char* buf, size_t cap, size_t* len);

/* ---- problems ---- */
int vpinn_host_problem_from_config(const char* config_json, const char* base_dir,
                                   const vpinn_mesh_source* mesh, vpinn_host_problem** out);
/* flags: VPINN_HOST_DEVICE_ASSEMBLY skips the host premultiplier assembly
 * (assembly.hpp:58-135); the view then carries a vpinn_gpu_assembly input
 * and vpinn_gpu_create builds the tensors on the device */
#define VPINN_HOST_DEVICE_ASSEMBLY 1
int vpinn_host_problem_from_config_ex(const char* config_json, const char* base_dir,
                                      const vpinn_mesh_source* mesh, int flags, vpinn_host_problem** out);
/* counts[8] = E, T, Q, n_interior, n_boundary, n_sensors, n_params, precision_downgraded */
void vpinn_host_problem_counts(const vpinn_host_problem* p, int64_t* counts);
/* plain-array view (pointers into p, valid while p lives) */
int vpinn_host_problem_view(const vpinn_host_problem* p, int device, int rank, int world,
                            vpinn_gpu_problem* view);
/* initial parameters (init_network, to_parameters order) */
void vpinn_host_problem_params(const vpinn_host_problem* p, float* out);
/* quadrature rule: xi, eta, w (n_quad each) */
void vpinn_host_problem_rule(const vpinn_host_problem* p, double* xi, double* eta, double* w);
void vpinn_host_problem_free(vpinn_host_problem* p);

/* Full training run on `device` with the config's training section; writes
 * the RunReport as JSON (history, timing median/p10/p90, metrics on the
 * output grid when problem.exact_solution is set, stop reason, final eps)
 * and returns the trained parameters in params_out (n_params, may be NULL).
 * json_len receives the report length; cap 0 = size query. */
int vpinn_host_train(vpinn_host_problem* p, int device, float* params_out, char* report_json,
                     size_t cap, size_t* json_len);

/* bench_case: median/p10/p90 seconds per step on a skewed e x e grid */
int vpinn_host_bench_case(const char* config_json, int e_per_dim, int n_test_per_dim,
                          int n_quad_per_dim, double skew, int reps, int device, double* out3);

#ifdef __cplusplus
}
#endif

#endif /* VPINN_HOST_H */
