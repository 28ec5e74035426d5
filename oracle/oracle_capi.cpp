// CPU ORACLE C entry points — TEST INFRASTRUCTURE ONLY (see vpinn_oracle.hpp).
// Loaded through ctypes by tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline leg.  The problem builder mirrors build_problem
// (reference proj/include/vpinn/commands.hpp:123-178) for a caller-supplied
// mesh, so the oracle assembles its own tensors independently of the product.
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>

#include "vpinn_oracle.hpp"

namespace {

thread_local std::string g_err;

struct OracleSpec {
  int n_nodes;
  const double* nodes_xy;
  int n_cells;
  const int* cells;
  int n_test_1d, n_quad_1d, lobatto;
  const char* forcing;
  const char* boundary_g;
  const char* sensor_field;
  int n_boundary;
  unsigned long long boundary_seed;
  int n_sensors;
  unsigned long long sensor_seed;
  double eps, bx, by;
  int eps_source, eps_scalar_index;
  double tau, gamma;
  int n_sizes;
  const int* sizes;
  int sigmoid;
  int n_scalars;
  const double* scalar_init;
  unsigned long long seed;
  int use_double;
  int strong;  // LossForm::strong (trainer.hpp:178)
};

struct OracleTrainSpec {
  long long iterations;
  int lr_exponential;
  double lr0, decay;
  int every, log_every;
  int has_eps_tol, has_eps_actual, has_loss_tol;
  double eps_abs_tol, eps_actual, loss_tol;
  int plateau_window;
};

struct HandleBase {
  virtual ~HandleBase() = default;
  vo::Mesh mesh;
  vo::Rule2D rule;
  vo::Basis basis;
  std::string forcing_name;
  std::vector<double> init_params;
  bool dbl = false;
};

template <typename Real>
struct Handle : HandleBase {
  vo::Problem<Real> pb;
};

template <typename Real>
HandleBase* build(const OracleSpec& s) {
  auto h = std::make_unique<Handle<Real>>();
  h->dbl = std::is_same<Real, double>::value;
  for (int i = 0; i < s.n_nodes; ++i) h->mesh.nodes.push_back({s.nodes_xy[2 * i], s.nodes_xy[2 * i + 1]});
  for (int k = 0; k < s.n_cells; ++k)
    h->mesh.cells.push_back({s.cells[4 * k], s.cells[4 * k + 1], s.cells[4 * k + 2], s.cells[4 * k + 3]});
  const vo::Rule1D r1 = vo::gauss_1d(s.n_quad_1d, s.lobatto != 0);
  h->rule = vo::tensor_rule(r1, r1);
  h->basis = vo::make_basis(s.n_test_1d, h->rule);
  h->forcing_name = s.forcing;
  auto& pb = h->pb;
  pb.shape.sizes.assign(s.sizes, s.sizes + s.n_sizes);
  pb.shape.sigmoid = s.sigmoid != 0;
  pb.shape.n_scalars = s.n_scalars;
  std::vector<double> sc(s.scalar_init, s.scalar_init + s.n_scalars);
  const auto p0 = vo::init_params<Real>(pb.shape, s.seed, sc);
  h->init_params.assign(p0.begin(), p0.end());
  pb.t = vo::assemble<Real>(h->mesh, h->basis, h->rule);
  vo::assemble_forcing(pb.t, vo::named_field(s.forcing));
  pb.c.eps = static_cast<Real>(s.eps);
  pb.c.bx = static_cast<Real>(s.bx);
  pb.c.by = static_cast<Real>(s.by);
  pb.c.source = s.eps_source;
  pb.c.eps_scalar_index = s.eps_scalar_index;
  pb.tau = s.tau;
  pb.gamma = s.gamma;
  const auto bset = vo::sample_boundary(h->mesh, s.n_boundary, vo::named_field(s.boundary_g), s.boundary_seed);
  vo::PointSet sset;
  if (s.n_sensors > 0)
    sset = vo::sample_sensors(h->mesh, s.n_sensors, vo::named_field(s.sensor_field), s.sensor_seed);
  // trainer.hpp:202-209 build_batch
  pb.n_int = pb.t.qpts.size();
  pb.n_bnd = bset.pts.size();
  pb.n_sen = sset.pts.size();
  pb.batch = pb.t.qpts;
  pb.batch.insert(pb.batch.end(), bset.pts.begin(), bset.pts.end());
  pb.batch.insert(pb.batch.end(), sset.pts.begin(), sset.pts.end());
  pb.bvals = bset.vals;
  pb.svals = sset.vals;
  // commands.hpp:147-152 — strong_forcing = f at the quadrature points
  if (s.strong) {
    pb.strong = true;
    const vo::Field f = vo::named_field(s.forcing);
    pb.strong_f.resize(pb.t.qpts.size());
    for (size_t i = 0; i < pb.t.qpts.size(); ++i) pb.strong_f[i] = f(pb.t.qpts[i].x, pb.t.qpts[i].y);
  }
  return h.release();
}

template <typename Real>
vo::Problem<Real>& prob(void* h) {
  return static_cast<Handle<Real>*>(static_cast<HandleBase*>(h))->pb;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const vo::OracleError& e) {
    g_err = e.what();
    return e.cat;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

template <typename Real>
std::vector<Real> vec_of(const void* p, size_t n) {
  const Real* r = static_cast<const Real*>(p);
  return std::vector<Real>(r, r + n);
}

template <typename Real>
void copy_out(const std::vector<Real>& v, void* out) {
  if (out && !v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(Real));
}

template <typename Real>
void do_loss_and_grad(void* h, const void* params, double* parts, void* grad) {
  auto& pb = prob<Real>(h);
  std::vector<Real> par = vec_of<Real>(params, pb.shape.count()), g;
  vo::Parts<Real> pp;
  const Real tot = vo::loss_and_grad(pb, par, g, pp);
  parts[0] = tot;
  parts[1] = pp.v;
  parts[2] = pp.b;
  parts[3] = pp.s;
  copy_out(g, grad);
}

template <typename Real>
void do_evaluate(void* h, const void* params, const double* xy, long long n, int order, void* u,
                 void* ux, void* uy, void* eps, void* uxx = nullptr, void* uyy = nullptr) {
  auto& pb = prob<Real>(h);
  std::vector<vo::Pt> pts(n);
  for (long long i = 0; i < n; ++i) pts[i] = {xy[2 * i], xy[2 * i + 1]};
  const auto ev = vo::evaluate(pb.shape, static_cast<const Real*>(params), pts, order);
  copy_out(ev.u, u);
  copy_out(ev.ux, ux);
  copy_out(ev.uy, uy);
  copy_out(ev.eps, eps);
  copy_out(ev.uxx, uxx);
  copy_out(ev.uyy, uyy);
}

// strong_residual_loss on caller-supplied derivatives (losses.hpp:422-467),
// in double: the known-answer case of tests/test_losses.cpp:344-412
int strong_loss_d(const double* u, const double* ux, const double* uy, const double* uxx,
                  const double* uyy, long long n, long long begin, long long count, double eps,
                  double bx, double by, int eps_source, int eps_scalar_index, const double* scalars,
                  int n_scalars, const double* f, double weight, double* loss, double* uxb,
                  double* uyb, double* uxxb, double* uyyb, double* sb) {
  return guard([&] {
    vo::Eval<double> ev;
    ev.u.assign(u, u + n);
    ev.ux.assign(ux, ux + n);
    ev.uy.assign(uy, uy + n);
    ev.uxx.assign(uxx, uxx + n);
    ev.uyy.assign(uyy, uyy + n);
    ev.scalars.assign(scalars, scalars + n_scalars);
    vo::Coeffs<double> c;
    c.eps = eps;
    c.bx = bx;
    c.by = by;
    c.source = eps_source;
    c.eps_scalar_index = eps_scalar_index;
    vo::Adj<double> adj;
    std::vector<double> fv(f, f + count);
    *loss = vo::strong_loss(ev, begin, count, c, fv, weight, &adj);
    copy_out(adj.uxb, uxb);
    copy_out(adj.uyb, uyb);
    copy_out(adj.uxxb, uxxb);
    copy_out(adj.uyyb, uyyb);
    for (size_t i = 0; i < adj.sb.size(); ++i) sb[i] = adj.sb[i];
  });
}

template <typename Real>
vo::Eval<Real> synthetic(void* h, const void* ux, const void* uy, const void* eps,
                         const double* scalars, int n_scalars) {
  auto& pb = prob<Real>(h);
  const size_t n = static_cast<size_t>(pb.t.E) * pb.t.Q;
  vo::Eval<Real> ev;
  ev.u.assign(n, Real(0));
  ev.ux = vec_of<Real>(ux, n);
  ev.uy = vec_of<Real>(uy, n);
  if (eps) ev.eps = vec_of<Real>(eps, n);
  for (int i = 0; i < n_scalars; ++i) ev.scalars.push_back(static_cast<Real>(scalars[i]));
  return ev;
}

template <typename Real>
void do_var_loss(void* h, int loop, const void* ux, const void* uy, const void* eps,
                 const double* scalars, int n_scalars, double weight, double* loss, void* res,
                 void* uxb, void* uyb, void* epsb, double* sb) {
  auto& pb = prob<Real>(h);
  auto* hb = static_cast<HandleBase*>(h);
  const auto ev = synthetic<Real>(h, ux, uy, eps, scalars, n_scalars);
  vo::Adj<Real> adj;
  vo::VarResult<Real> r =
      loop ? vo::loop_loss(hb->mesh, hb->basis, hb->rule, vo::named_field(hb->forcing_name), ev,
                           pb.c, static_cast<Real>(weight), &adj)
           : vo::tensor_loss(pb.t, ev, pb.c, static_cast<Real>(weight), &adj);
  *loss = r.loss;
  copy_out(r.res, res);
  copy_out(adj.uxb, uxb);
  copy_out(adj.uyb, uyb);
  copy_out(adj.epsb, epsb);
  for (size_t i = 0; i < adj.sb.size(); ++i) sb[i] = adj.sb[i];
}

vo::TrainSpec to_spec(const OracleTrainSpec& t) {
  vo::TrainSpec s;
  s.iterations = t.iterations;
  s.lr.exponential = t.lr_exponential != 0;
  s.lr.lr0 = t.lr0;
  s.lr.decay = t.decay;
  s.lr.every = t.every;
  s.log_every = t.log_every;
  s.has_eps_tol = t.has_eps_tol;
  s.has_eps_actual = t.has_eps_actual;
  s.has_loss_tol = t.has_loss_tol;
  s.eps_abs_tol = t.eps_abs_tol;
  s.eps_actual = t.eps_actual;
  s.loss_tol = t.loss_tol;
  s.plateau_window = t.plateau_window;
  return s;
}

template <typename Real>
void do_train(void* h, void* params, const OracleTrainSpec& ts, double* every_step,
              long long* steps_run, int* stop_reason, double* final_eps) {
  auto& pb = prob<Real>(h);
  std::vector<Real> par = vec_of<Real>(params, pb.shape.count());
  const vo::TrainOut out = vo::train(pb, par, to_spec(ts));
  copy_out(par, params);
  for (size_t i = 0; i < out.every_step.size(); ++i)
    for (int c = 0; c < 4; ++c) every_step[4 * i + c] = out.every_step[i][c];
  *steps_run = out.steps_run;
  *stop_reason = out.stop_reason;
  *final_eps = out.final_eps;
}

// time_epochs-style timing of the full step (trainer.hpp:157-172,
// commands.hpp:330-336): warm-ups untimed, then per-step wall seconds.
template <typename Real>
void do_time_steps(void* h, void* params, double lr, int warmup, int reps, double* seconds) {
  auto& pb = prob<Real>(h);
  std::vector<Real> par = vec_of<Real>(params, pb.shape.count()), g;
  vo::AdamState<Real> st(par.size());
  vo::Parts<Real> pp;
  auto step = [&]() {
    vo::loss_and_grad(pb, par, g, pp);
    vo::adam_step(par, g, st, static_cast<Real>(lr));
  };
  for (int i = 0; i < warmup; ++i) step();
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    step();
    const auto t1 = std::chrono::steady_clock::now();
    seconds[i] = std::chrono::duration<double>(t1 - t0).count();
  }
  copy_out(par, params);
}

}  // namespace

extern "C" {

const char* vo_last_error() { return g_err.c_str(); }

void* vo_build(const OracleSpec* s) {
  HandleBase* h = nullptr;
  const int rc = guard([&] { h = s->use_double ? build<double>(*s) : build<float>(*s); });
  return rc == 0 ? h : nullptr;
}

void vo_free(void* h) { delete static_cast<HandleBase*>(h); }

int vo_is_double(void* h) { return static_cast<HandleBase*>(h)->dbl ? 1 : 0; }

// counts: E, T, Q, n_int, n_bnd, n_sen, n_params
void vo_counts(void* h, long long* out) {
  auto* hb = static_cast<HandleBase*>(h);
  auto fill = [&](auto& pb) {
    out[0] = pb.t.E;
    out[1] = pb.t.T;
    out[2] = pb.t.Q;
    out[3] = static_cast<long long>(pb.n_int);
    out[4] = static_cast<long long>(pb.n_bnd);
    out[5] = static_cast<long long>(pb.n_sen);
    out[6] = pb.shape.count();
  };
  if (hb->dbl)
    fill(prob<double>(h));
  else
    fill(prob<float>(h));
}

// which: 0 grad_x, 1 grad_y, 2 test, 3 forcing (Real), 4 batch points
// (double [P][2]), 5 boundary values, 6 sensor values (double), 7 initial
// parameters (double), 8 rule xi/eta/w (double [3][Q]), 9 strong forcing
// (double, n_int; strong problems only)
int vo_get_array(void* h, int which, void* out) {
  auto* hb = static_cast<HandleBase*>(h);
  return guard([&] {
    auto body = [&](auto& pb) {
      switch (which) {
        case 0: copy_out(pb.t.gx, out); break;
        case 1: copy_out(pb.t.gy, out); break;
        case 2: copy_out(pb.t.tv, out); break;
        case 3: copy_out(pb.t.forcing, out); break;
        case 4: {
          double* d = static_cast<double*>(out);
          for (size_t i = 0; i < pb.batch.size(); ++i) {
            d[2 * i] = pb.batch[i].x;
            d[2 * i + 1] = pb.batch[i].y;
          }
          break;
        }
        case 5: copy_out(pb.bvals, out); break;
        case 6: copy_out(pb.svals, out); break;
        case 7: copy_out(hb->init_params, out); break;
        case 9: copy_out(pb.strong_f, out); break;
        case 8: {
          double* d = static_cast<double*>(out);
          const size_t Q = hb->rule.w.size();
          for (size_t q = 0; q < Q; ++q) {
            d[q] = hb->rule.xi[q];
            d[Q + q] = hb->rule.eta[q];
            d[2 * Q + q] = hb->rule.w[q];
          }
          break;
        }
        default: throw vo::OracleError(vo::kConfig, "vo_get_array: bad selector");
      }
    };
    if (hb->dbl)
      body(prob<double>(h));
    else
      body(prob<float>(h));
  });
}

int vo_loss_and_grad(void* h, const void* params, double* parts, void* grad) {
  return guard([&] {
    if (vo_is_double(h))
      do_loss_and_grad<double>(h, params, parts, grad);
    else
      do_loss_and_grad<float>(h, params, parts, grad);
  });
}

// objective + gradient of the rank sub-problem (cells [e0,e1), boundary
// [b0,b1), sensors [s0,s1)), penalties normalised by the global counts
int vo_loss_and_grad_part(void* h, const void* params, long long e0, long long e1, long long b0,
                          long long b1, long long s0, long long s1, double* parts, void* grad) {
  return guard([&] {
    auto run = [&](auto tag) {
      using Real = decltype(tag);
      auto& pb = prob<Real>(h);
      const vo::Problem<Real> sub = vo::partition(pb, e0, e1, b0, b1, s0, s1);
      std::vector<Real> par = vec_of<Real>(params, pb.shape.count()), g;
      vo::Parts<Real> pp;
      const Real tot = vo::loss_and_grad(sub, par, g, pp);
      parts[0] = tot;
      parts[1] = pp.v;
      parts[2] = pp.b;
      parts[3] = pp.s;
      copy_out(g, grad);
    };
    if (vo_is_double(h))
      run(double{});
    else
      run(float{});
  });
}

int vo_evaluate(void* h, const void* params, const double* xy, long long n, int order, void* u,
                void* ux, void* uy, void* eps) {
  return guard([&] {
    if (vo_is_double(h))
      do_evaluate<double>(h, params, xy, n, order, u, ux, uy, eps);
    else
      do_evaluate<float>(h, params, xy, n, order, u, ux, uy, eps);
  });
}

// evaluate() at order 2: second derivatives too (network.hpp:414-449)
int vo_evaluate2(void* h, const void* params, const double* xy, long long n, void* u, void* ux,
                 void* uy, void* uxx, void* uyy) {
  return guard([&] {
    if (vo_is_double(h))
      do_evaluate<double>(h, params, xy, n, 2, u, ux, uy, nullptr, uxx, uyy);
    else
      do_evaluate<float>(h, params, xy, n, 2, u, ux, uy, nullptr, uxx, uyy);
  });
}

int vo_strong_loss(const double* u, const double* ux, const double* uy, const double* uxx,
                   const double* uyy, long long n, long long begin, long long count, double eps,
                   double bx, double by, int eps_source, int eps_scalar_index,
                   const double* scalars, int n_scalars, const double* f, double weight,
                   double* loss, double* uxb, double* uyb, double* uxxb, double* uyyb, double* sb) {
  return strong_loss_d(u, ux, uy, uxx, uyy, n, begin, count, eps, bx, by, eps_source,
                       eps_scalar_index, scalars, n_scalars, f, weight, loss, uxb, uyb, uxxb, uyyb,
                       sb);
}

int vo_var_loss(void* h, int loop, const void* ux, const void* uy, const void* eps,
                const double* scalars, int n_scalars, double weight, double* loss, void* res,
                void* uxb, void* uyb, void* epsb, double* sb) {
  return guard([&] {
    if (vo_is_double(h))
      do_var_loss<double>(h, loop, ux, uy, eps, scalars, n_scalars, weight, loss, res, uxb, uyb,
                          epsb, sb);
    else
      do_var_loss<float>(h, loop, ux, uy, eps, scalars, n_scalars, weight, loss, res, uxb, uyb,
                         epsb, sb);
  });
}

int vo_train(void* h, void* params, const OracleTrainSpec* ts, double* every_step,
             long long* steps_run, int* stop_reason, double* final_eps) {
  return guard([&] {
    if (vo_is_double(h))
      do_train<double>(h, params, *ts, every_step, steps_run, stop_reason, final_eps);
    else
      do_train<float>(h, params, *ts, every_step, steps_run, stop_reason, final_eps);
  });
}

int vo_time_steps(void* h, void* params, double lr, int warmup, int reps, double* seconds) {
  return guard([&] {
    if (vo_is_double(h))
      do_time_steps<double>(h, params, lr, warmup, reps, seconds);
    else
      do_time_steps<float>(h, params, lr, warmup, reps, seconds);
  });
}

// Adam on a plain double vector: n params, g given per step [steps][n]
int vo_adam_f64(double* p, const double* g, int n, int steps, double lr) {
  return guard([&] {
    std::vector<double> par(p, p + n);
    vo::AdamState<double> st(n);
    for (int t = 0; t < steps; ++t) {
      std::vector<double> gv(g + static_cast<size_t>(t) * n, g + static_cast<size_t>(t + 1) * n);
      vo::adam_step(par, gv, st, lr);
    }
    std::memcpy(p, par.data(), sizeof(double) * n);
  });
}

int vo_adam_f32(float* p, const float* g, int n, int steps, const double* lr) {
  return guard([&] {
    std::vector<float> par(p, p + n);
    vo::AdamState<float> st(n);
    for (int t = 0; t < steps; ++t) {
      std::vector<float> gv(g + static_cast<size_t>(t) * n, g + static_cast<size_t>(t + 1) * n);
      vo::adam_step(par, gv, st, static_cast<float>(lr[t]));
    }
    std::memcpy(p, par.data(), sizeof(float) * n);
  });
}

double vo_lr_at(int exponential, double lr0, double decay, int every, long long step) {
  vo::LrSched s;
  s.exponential = exponential != 0;
  s.lr0 = lr0;
  s.decay = decay;
  s.every = every;
  double v = 0;
  if (guard([&] { v = vo::lr_at(s, step); }) != 0) return -1.0;
  return v;
}

int vo_gauss_rule(int n, int lobatto, double* x, double* w) {
  return guard([&] {
    const auto r = vo::gauss_1d(n, lobatto != 0);
    for (int i = 0; i < n; ++i) {
      x[i] = r.x[i];
      w[i] = r.w[i];
    }
  });
}

void vo_test_fn(int k, double x, double* v, double* d) {
  const auto r = vo::test_fn_1d(k, x);
  *v = r.v;
  *d = r.d;
}

int vo_field(const char* name, const double* x, const double* y, long long n, double* out) {
  return guard([&] {
    const auto f = vo::named_field(name);
    for (long long i = 0; i < n; ++i) out[i] = f(x[i], y[i]);
  });
}

// structured + skewed mesh (geometry.hpp:146-183, commands.hpp:75-97)
int vo_structured_mesh(int nx, int ny, double x0, double x1, double y0, double y1, double skew,
                       unsigned long long skew_seed, double* nodes_xy, int* cells) {
  return guard([&] {
    vo::Mesh m = vo::structured_mesh(nx, ny, x0, x1, y0, y1);
    vo::skew_nodes(m, skew, skew_seed);
    for (size_t i = 0; i < m.nodes.size(); ++i) {
      nodes_xy[2 * i] = m.nodes[i].x;
      nodes_xy[2 * i + 1] = m.nodes[i].y;
    }
    for (size_t k = 0; k < m.cells.size(); ++k)
      for (int c = 0; c < 4; ++c) cells[4 * k + c] = m.cells[k][c];
  });
}

void vo_init_params_f64(const int* sizes, int n_sizes, unsigned long long seed, double* out) {
  vo::NetShape s;
  s.sizes.assign(sizes, sizes + n_sizes);
  const auto p = vo::init_params<double>(s, seed, {});
  std::memcpy(out, p.data(), p.size() * sizeof(double));
}

}  // extern "C"
