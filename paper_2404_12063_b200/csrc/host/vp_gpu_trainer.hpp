// The reference-facing C++ API over the B200 step: build_problem from a
// FullConfig (reference commands.hpp:123-178), train() with the reference's
// loop semantics (trainer.hpp:275-382) executed on the device through
// include/vpinn_gpu.h, error metrics on the evaluation grid
// (trainer.hpp:405-446) through the device forward, and the benchmark step
// protocol of bench_case / time_epochs (commands.hpp:285-341,
// trainer.hpp:134-172).  Kernel "tensor" for the weak form and the
// strong-form collocation baseline are served; kernels loop/matrix raise
// InvalidModeError (CPU formulations; there is no CPU fallback).
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "vp_config.hpp"
#include "vpinn_gpu.h"

namespace vpinn {

struct BuiltProblem {
  Mesh mesh;
  DenseNetwork net;
  ProblemAssembly pa;
  LossWeights weights;
  bool precision_downgraded = false;  // config asked for double, device computes fp32
  // device_assembly: the premultiplier tensors, the forcing and the interior
  // points are built on the device (vpinn_gpu_assembly); pa.tensors then
  // only carries the sizes and pa.batch only [boundary | sensors]
  bool device_assembly = false;
  QuadratureRule2D rule;
  ReferenceBasis basis;
  std::string forcing;
};

inline Mesh build_domain_mesh(const DomainSpec& d) {
  if (d.kind == DomainSpec::Kind::rectangle) return generate_structured_mesh(d.nx, d.ny, d.x_range, d.y_range);
  return read_gmsh_file(d.path);
}

inline PdeCoefficients coefficients_from_config(const FullConfig& c) {
  PdeCoefficients k;
  k.eps = static_cast<float>(c.problem.eps);
  k.bx = static_cast<float>(c.problem.bx);
  k.by = static_cast<float>(c.problem.by);
  if (c.problem.pde == PdeType::cd2d_variable_eps) {
    k.source = EpsSource::spatial;
  } else if (c.network.eps_scalar_init) {
    k.source = EpsSource::scalar;
    k.eps_scalar_index = 0;
  }
  return k;
}

inline BuiltProblem build_problem(const FullConfig& cfg, std::optional<Mesh> premade = {},
                                  bool device_assembly = false) {
  const bool strong = cfg.disc.form == LossForm::strong;
  if (!strong && cfg.disc.kernel != KernelKind::tensor)
    throw InvalidModeError("the B200 path implements kernel 'tensor'; 'loop'/'matrix' are CPU formulations");
  BuiltProblem bp;
  bp.mesh = premade ? std::move(*premade) : build_domain_mesh(cfg.problem.domain);
  const Rule1D r1 = gauss_rule_1d(cfg.disc.n_quad_per_dim, cfg.disc.quadrature);
  const QuadratureRule2D rule = tensor_product_rule(r1, r1);
  const ReferenceBasis basis = reference_basis(cfg.disc.n_test_per_dim, rule);
  std::vector<std::pair<std::string, double>> scalars;
  if (cfg.network.eps_scalar_init) scalars.emplace_back("eps", *cfg.network.eps_scalar_init);
  bp.net = init_network(cfg.network.layers, cfg.seed, cfg.network.activation, scalars);
  auto& pa = bp.pa;
  bp.device_assembly = device_assembly;
  bp.rule = rule;
  bp.basis = basis;
  bp.forcing = cfg.problem.forcing;
  if (!device_assembly) {
    pa.tensors = assemble_element_tensors(bp.mesh, basis, rule);
    assemble_forcing(pa.tensors, lookup_field(cfg.problem.forcing));
  } else {
    lookup_field(cfg.problem.forcing);  // same ConfigError for an unknown name
    if (bp.mesh.n_elements() == 0) throw InvalidArgumentError("assemble: empty mesh");
    pa.tensors.n_elem = bp.mesh.n_elements();
    pa.tensors.n_test = basis.n_test();
    pa.tensors.n_quad = rule.size();
  }
  pa.coeffs = coefficients_from_config(cfg);
  pa.boundary = sample_boundary(bp.mesh, cfg.problem.n_boundary_points, lookup_field(cfg.problem.boundary_g),
                                cfg.problem.boundary_seed);
  if (cfg.problem.sensors) {
    if (cfg.problem.exact_solution.empty())
      throw ConfigError("problem.sensors: source 'exact' needs problem.exact_solution");
    pa.sensors = sample_sensors(bp.mesh, cfg.problem.sensors->count, lookup_field(cfg.problem.exact_solution),
                                cfg.problem.sensors->seed);
  }
  pa.build_batch();
  if (device_assembly) pa.n_interior = static_cast<long long>(pa.tensors.n_elem) * pa.tensors.n_quad;
  pa.strong = strong;
  if (strong && !device_assembly) {
    // commands.hpp:147-152 — strong_forcing = f at the quadrature points
    const ScalarField2D f = lookup_field(cfg.problem.forcing);
    pa.strong_forcing.resize(pa.tensors.quad_points.size());
    for (size_t i = 0; i < pa.tensors.quad_points.size(); ++i)
      pa.strong_forcing[i] = static_cast<float>(f(pa.tensors.quad_points[i].x, pa.tensors.quad_points[i].y));
  }
  bp.weights = cfg.training.weights;
  bp.precision_downgraded = cfg.precision == Precision::f64;
  return bp;
}

// ---- the plain-array view the C-ABI consumes --------------------------------
struct GpuView {
  vpinn_gpu_problem p{};
  std::vector<double> points, bvals, svals;
  std::vector<int32_t> sizes;
  // device assembly input (when bp.device_assembly)
  vpinn_gpu_assembly asm_in{};
  std::vector<double> nodes, xi, eta, w;
  std::vector<int32_t> elems;
};

inline std::unique_ptr<GpuView> make_gpu_view(const BuiltProblem& bp, int device = 0, int rank = 0, int world = 1) {
  auto v = std::make_unique<GpuView>();
  const auto& pa = bp.pa;
  const auto& t = pa.tensors;
  v->points.reserve(pa.batch.size() * 2);
  for (const auto& q : pa.batch) {
    v->points.push_back(q.x);
    v->points.push_back(q.y);
  }
  v->bvals = pa.boundary.values;
  v->svals = pa.sensors.values;
  v->sizes.assign(bp.net.layer_sizes.begin(), bp.net.layer_sizes.end());
  vpinn_gpu_problem& p = v->p;
  p.n_elem = t.n_elem;
  p.n_test = t.n_test;
  p.n_quad = t.n_quad;
  p.grad_x = t.grad_x.data();
  p.grad_y = t.grad_y.data();
  p.test = t.test.data();
  p.forcing = t.forcing.data();
  p.points = v->points.data();
  p.n_interior = pa.n_interior;
  p.n_boundary = pa.n_boundary;
  p.n_sensors = pa.n_sensors;
  p.boundary_values = v->bvals.empty() ? nullptr : v->bvals.data();
  p.sensor_values = v->svals.empty() ? nullptr : v->svals.data();
  p.n_layer_sizes = static_cast<int32_t>(v->sizes.size());
  p.layer_sizes = v->sizes.data();
  p.activation = bp.net.activation == Activation::sigmoid ? VPINN_ACT_SIGMOID : VPINN_ACT_TANH;
  p.n_scalars = static_cast<int32_t>(bp.net.scalars.size());
  p.eps = pa.coeffs.eps;
  p.bx = pa.coeffs.bx;
  p.by = pa.coeffs.by;
  p.eps_source = static_cast<int32_t>(pa.coeffs.source);
  p.eps_scalar_index = pa.coeffs.eps_scalar_index;
  p.tau = bp.weights.tau;
  p.gamma = bp.weights.gamma;
  p.device = device;
  p.rank = rank;
  p.world_size = world;
  p.form = pa.strong ? VPINN_FORM_STRONG : VPINN_FORM_WEAK;
  p.strong_forcing = pa.strong && !bp.device_assembly ? pa.strong_forcing.data() : nullptr;
  if (bp.device_assembly) {
    for (const auto& n : bp.mesh.nodes) {
      v->nodes.push_back(n.x);
      v->nodes.push_back(n.y);
    }
    for (const auto& e : bp.mesh.elements) v->elems.insert(v->elems.end(), e.begin(), e.end());
    vpinn_gpu_assembly& a = v->asm_in;
    a.n_nodes = bp.mesh.n_nodes();
    a.nodes = v->nodes.data();
    a.elements = v->elems.data();
    a.xi = bp.rule.xi.data();
    a.eta = bp.rule.eta.data();
    a.weights = bp.rule.weights.data();
    a.basis_val = bp.basis.val.data();
    a.basis_dxi = bp.basis.dxi.data();
    a.basis_deta = bp.basis.deta.data();
    a.forcing = bp.forcing.c_str();
    p.assembly = &v->asm_in;
    p.grad_x = p.grad_y = p.test = p.forcing = nullptr;
  }
  return v;
}

inline void raise_code(int rc, const std::string& where) {
  if (rc == 0) return;
  const std::string msg = where + ": " + vpinn_gpu_last_error();
  switch (rc) {
    case VPINN_ERR_CONFIG: throw ConfigError(msg);
    case VPINN_ERR_MESH: throw MeshFileError(msg);
    case VPINN_ERR_IO: throw IoError(msg);
    case VPINN_ERR_DEVICE: throw DeviceError(msg);
    default: throw ContractViolationError(msg);
  }
}

// RAII device context
class GpuContext {
 public:
  GpuContext(const BuiltProblem& bp, int device = 0, int rank = 0, int world = 1) {
    view_ = make_gpu_view(bp, device, rank, world);
    raise_code(vpinn_gpu_create(&view_->p, &ctx_), "vpinn_gpu_create");
    raise_code(vpinn_gpu_set_params(ctx_, bp.net.params.data(), static_cast<int>(bp.net.params.size())),
               "vpinn_gpu_set_params");
  }
  ~GpuContext() { vpinn_gpu_destroy(ctx_); }
  GpuContext(const GpuContext&) = delete;
  GpuContext& operator=(const GpuContext&) = delete;
  vpinn_gpu_ctx* get() const { return ctx_; }

 private:
  std::unique_ptr<GpuView> view_;
  vpinn_gpu_ctx* ctx_ = nullptr;
};

// ---- run report (trainer.hpp:99-130) ------------------------------------------
struct HistoryRow {
  std::int64_t step = 0;
  double total = 0, variational = 0, boundary = 0, sensor = 0, lr = 0;
  double eps = std::numeric_limits<double>::quiet_NaN();
};
struct TimingSummary {
  std::vector<double> samples;
  double median_s = 0, p10_s = 0, p90_s = 0;
};
struct Metrics {
  double mae = 0, rel_l2 = 0, max_err = 0;
};
struct RunReport {
  std::vector<HistoryRow> history;
  TimingSummary timing;
  Metrics metrics;
  bool converged = false;
  std::string stop_reason = "iteration budget";
  std::int64_t steps_run = 0;
  double final_eps = std::numeric_limits<double>::quiet_NaN();
  double eps_abs_error = std::numeric_limits<double>::quiet_NaN();
};

constexpr int kTimingWarmup = 10;

inline double percentile(std::vector<double> v, double p) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double pos = p * double(v.size() - 1);
  const size_t lo = static_cast<size_t>(pos), hi = std::min(lo + 1, v.size() - 1);
  const double f = pos - double(lo);
  return v[lo] * (1.0 - f) + v[hi] * f;
}

inline void summarize(TimingSummary& t) {
  t.median_s = percentile(t.samples, 0.5);
  t.p10_s = percentile(t.samples, 0.1);
  t.p90_s = percentile(t.samples, 0.9);
}

// The epoch loop on the device; history rows, timing and stop rules exactly
// as trainer.hpp:316-381 (per-step timestamps taken on the device).
inline RunReport train(DenseNetwork& net, const BuiltProblem& bp, const TrainConfig& cfg, GpuContext& gpu) {
  if (cfg.iterations < 1) throw InvalidArgumentError("train: iterations must be >= 1");
  vpinn_gpu_train_spec s{};
  s.iterations = cfg.iterations;
  s.lr_exponential = cfg.lr.mode == LrMode::exponential;
  s.lr0 = cfg.lr.lr0;
  s.decay = cfg.lr.decay;
  s.every = cfg.lr.every;
  s.has_eps_abs_tol = cfg.convergence.eps_abs_tol.has_value();
  s.has_eps_actual = cfg.convergence.eps_actual.has_value();
  s.has_loss_tol = cfg.convergence.loss_tol.has_value();
  s.eps_abs_tol = cfg.convergence.eps_abs_tol.value_or(0.0);
  s.eps_actual = cfg.convergence.eps_actual.value_or(0.0);
  s.loss_tol = cfg.convergence.loss_tol.value_or(0.0);
  s.plateau_window = cfg.convergence.plateau_window;
  std::vector<vpinn_gpu_step_record> rec(static_cast<size_t>(cfg.iterations));
  vpinn_gpu_train_result res{};
  const int rc = vpinn_gpu_train(gpu.get(), &s, rec.data(), &res);
  if (rc == VPINN_ERR_NUMERIC && res.abort_step > 0)
    throw TrainingAbortError(res.abort_step, vpinn_gpu_last_error());
  raise_code(rc, "vpinn_gpu_train");
  RunReport r;
  r.steps_run = res.steps_run;
  const bool tracks = bp.pa.coeffs.source == EpsSource::scalar;
  auto row = [&](std::int64_t step) {
    const auto& x = rec[static_cast<size_t>(step - 1)];
    HistoryRow h;
    h.step = step;
    h.total = x.total;
    h.variational = x.variational;
    h.boundary = x.boundary;
    h.sensor = x.sensor;
    h.lr = x.lr;
    if (tracks) h.eps = x.eps;
    return h;
  };
  for (std::int64_t step = 1; step <= res.steps_run; ++step) {
    if (step == 1 || step == cfg.iterations || (cfg.log_every > 0 && step % cfg.log_every == 0))
      r.history.push_back(row(step));
    if (step > kTimingWarmup &&
        (cfg.timing_window == 0 || static_cast<int>(r.timing.samples.size()) < cfg.timing_window))
      r.timing.samples.push_back(rec[static_cast<size_t>(step - 1)].seconds);
  }
  if (res.converged) {
    r.converged = true;
    r.stop_reason = res.stop_reason == 1 ? "coefficient within tolerance" : "loss plateau";
    if (r.history.empty() || r.history.back().step != res.steps_run) r.history.push_back(row(res.steps_run));
  }
  summarize(r.timing);
  // from_parameters: the device holds the trained parameters
  raise_code(vpinn_gpu_get_params(gpu.get(), net.params.data(), static_cast<int>(net.params.size())),
             "vpinn_gpu_get_params");
  for (size_t i = 0; i < net.scalars.size(); ++i)
    net.scalars[i].second = net.params[net.params.size() - net.scalars.size() + i];
  if (tracks) {
    r.final_eps = res.final_eps;
    if (cfg.convergence.eps_actual) r.eps_abs_error = std::abs(r.final_eps - *cfg.convergence.eps_actual);
  }
  return r;
}

// grid (inclusive endpoints, x fastest) and the error metrics, evaluate(order 0)
// on the device
inline Metrics evaluate_metrics(GpuContext& gpu, const ScalarField2D& exact, int nx, int ny,
                                std::pair<double, double> xr, std::pair<double, double> yr) {
  if (nx < 2 || ny < 2) throw InvalidArgumentError("grid_points: need at least 2 per axis");
  std::vector<double> pts;
  pts.reserve(static_cast<size_t>(nx) * ny * 2);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      pts.push_back(xr.first + (xr.second - xr.first) * i / (nx - 1));
      pts.push_back(yr.first + (yr.second - yr.first) * j / (ny - 1));
    }
  const int64_t n = static_cast<int64_t>(pts.size() / 2);
  std::vector<float> u(static_cast<size_t>(n));
  raise_code(vpinn_gpu_forward(gpu.get(), pts.data(), n, 0, u.data(), nullptr, nullptr, nullptr), "evaluate");
  Metrics m;
  double sa = 0, sq = 0, se = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double ue = exact(pts[2 * i], pts[2 * i + 1]);
    const double d = static_cast<double>(u[static_cast<size_t>(i)]) - ue;
    sa += std::abs(d);
    sq += d * d;
    se += ue * ue;
    m.max_err = std::max(m.max_err, std::abs(d));
  }
  m.mae = sa / double(n);
  m.rel_l2 = se > 0.0 ? std::sqrt(sq / se) : std::sqrt(sq);
  return m;
}

// bench_case step protocol: skewed e x e unit-square grid, 10 untimed
// warm-ups then `reps` device-timestamped steps (median / p10 / p90)
struct BenchmarkRow {
  int n_elem = 0, n_test = 0, n_quad = 0;
  bool supported = true;
  double median_s = 0, p10_s = 0, p90_s = 0;
};

inline BenchmarkRow bench_case(const FullConfig& cfg, int e_per_dim, int n_test, int n_quad, double skew, int reps,
                               int device = 0) {
  if (reps < 10) throw InvalidArgumentError("time_epochs: need at least 10 repetitions");
  BenchmarkRow row;
  row.n_elem = e_per_dim * e_per_dim;
  row.n_test = n_test * n_test;
  row.n_quad = n_quad * n_quad;
  Mesh mesh = generate_structured_mesh(e_per_dim, e_per_dim, {0.0, 1.0}, {0.0, 1.0});
  skew_mesh_nodes(mesh, skew, 1234);
  FullConfig c = cfg;
  c.disc.n_test_per_dim = n_test;
  c.disc.n_quad_per_dim = n_quad;
  c.disc.kernel = KernelKind::tensor;
  c.disc.form = LossForm::weak;
  BuiltProblem bp = build_problem(c, std::move(mesh));
  GpuContext gpu(bp, device);
  TrainConfig tc;
  tc.iterations = kTimingWarmup + reps;
  tc.lr.lr0 = c.training.lr.lr0;
  tc.log_every = 1;
  DenseNetwork net = bp.net;
  const RunReport r = train(net, bp, tc, gpu);
  row.median_s = r.timing.median_s;
  row.p10_s = r.timing.p10_s;
  row.p90_s = r.timing.p90_s;
  return row;
}

}  // namespace vpinn
