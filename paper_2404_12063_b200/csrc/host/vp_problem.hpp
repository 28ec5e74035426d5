// Host-side problem assembly for the B200 step: named analytic fields,
// premultiplier tensors and forcing in the reference layout, boundary and
// sensor sampling, the network parameter vector, and the evaluation batch.
// Layout and formula contracts: reference proj/include/vpinn/fields.hpp:39-125,
// assembly.hpp:34-135 and 223-304, network.hpp:42-128, trainer.hpp:180-210.
#pragma once

#include <cmath>
#include <functional>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "vp_mesh.hpp"

namespace vpinn {

using ScalarField2D = std::function<double(double, double)>;

// ---- named field library ---------------------------------------------------
inline const std::map<std::string, ScalarField2D>& field_library() {
  static const std::map<std::string, ScalarField2D> lib = [] {
    std::map<std::string, ScalarField2D> m;
    auto sin_u = [](double w) -> ScalarField2D {
      return [w](double x, double y) { return -std::sin(w * x) * std::sin(w * y); };
    };
    auto sin_f = [](double w) -> ScalarField2D {
      return [w](double x, double y) { return -2.0 * w * w * std::sin(w * x) * std::sin(w * y); };
    };
    const double w1 = 2.0 * M_PI;
    m["zero"] = [](double, double) { return 0.0; };
    m["one"] = [](double, double) { return 1.0; };
    m["sin2pi_u"] = sin_u(w1);
    m["sin2pi_f"] = sin_f(w1);
    m["sin4pi_u"] = sin_u(2.0 * w1);
    m["sin4pi_f"] = sin_f(2.0 * w1);
    m["sin8pi_u"] = sin_u(4.0 * w1);
    m["sin8pi_f"] = sin_f(4.0 * w1);
    m["gear_f"] = [](double x, double) { return 50.0 * std::sin(x) + std::cos(x); };
    m["bump_u"] = [](double x, double) {
      return 10.0 * std::sin(x) * std::tanh(x) * std::exp(-0.3 * x * x);
    };
    m["bump_f"] = [](double x, double) {
      const double sx = std::sin(x), cx = std::cos(x), sh = std::sinh(2.0 * x), ch = std::cosh(x),
                   th = std::tanh(x);
      const double num = -9.0 * x * x * sx * sh + 60.0 * x * sx + 30.0 * x * cx * sh +
                         40.0 * sx * sh + 100.0 * sx * th - 100.0 * cx;
      return 3.0 * num * std::exp(-0.3 * x * x) / (50.0 * ch * ch);
    };
    m["sinpi_u"] = [](double x, double y) { return std::sin(M_PI * x) * std::sin(M_PI * y); };
    m["sincos_eps"] = [](double x, double y) { return 0.5 * (std::sin(x) + std::cos(y)); };
    m["sinpi_vareps_f"] = [](double x, double y) {
      const double sx = std::sin(M_PI * x), cx = std::cos(M_PI * x);
      const double sy = std::sin(M_PI * y), cy = std::cos(M_PI * y);
      return 0.5 * M_PI *
             (2.0 * M_PI * (std::sin(x) + std::cos(y)) * sx * sy + std::sin(y) * sx * cy -
              sy * std::cos(x) * cx + 2.0 * sy * cx);
    };
    return m;
  }();
  return lib;
}

inline const ScalarField2D& lookup_field(const std::string& name) {
  const auto& lib = field_library();
  const auto it = lib.find(name);
  if (it == lib.end()) {
    std::string msg = "unknown field '" + name + "'; available:";
    for (const auto& kv : lib) msg += " " + kv.first;
    throw ConfigError(msg);
  }
  return it->second;
}

// ---- premultiplier tensors ----------------------------------------------------
// grad_x(k,j,q) = w_q det dv_j/dx, grad_y likewise, test(k,j,q) = w_q det v_j;
// slices row-major [k][j][q]; forcing Eigen-column-major T x E (index k*T + j).
struct ElementTensors {
  int n_elem = 0, n_test = 0, n_quad = 0;
  std::vector<float> grad_x, grad_y, test;
  std::vector<float> forcing;
  std::vector<Point2> quad_points;  // element-major k*Q + q
  bool has_forcing() const { return !forcing.empty(); }
};

// geometry in double, cast to float at store
inline ElementTensors assemble_element_tensors(const Mesh& mesh, const ReferenceBasis& basis,
                                               const QuadratureRule2D& rule) {
  ElementTensors t;
  t.n_elem = mesh.n_elements();
  t.n_test = basis.n_test();
  t.n_quad = rule.size();
  if (t.n_elem == 0) throw InvalidArgumentError("assemble: empty mesh");
  if (basis.nq != t.n_quad) throw ContractViolationError("assemble: basis was built for a different quadrature rule");
  const size_t slab = static_cast<size_t>(t.n_test) * t.n_quad;
  t.grad_x.resize(slab * t.n_elem);
  t.grad_y.resize(slab * t.n_elem);
  t.test.resize(slab * t.n_elem);
  t.quad_points.resize(static_cast<size_t>(t.n_elem) * t.n_quad);
  for (int k = 0; k < t.n_elem; ++k) {
    const BilinearCoeffs c = bilinear_coeffs(mesh, k);
    float* gx = t.grad_x.data() + slab * k;
    float* gy = t.grad_y.data() + slab * k;
    float* tv = t.test.data() + slab * k;
    for (int q = 0; q < t.n_quad; ++q) {
      const Jacobian J = jacobian_at(c, rule.xi[q], rule.eta[q]);
      if (!(J.det > 0.0))
        throw DegenerateElementError(k, "assemble: element " + std::to_string(k) +
                                            " has non-positive jacobian determinant " +
                                            std::to_string(J.det) + " at quadrature point " +
                                            std::to_string(q));
      t.quad_points[static_cast<size_t>(k) * t.n_quad + q] = map_point(c, rule.xi[q], rule.eta[q]);
      const double wdet = rule.weights[q] * J.det;
      const double inv = 1.0 / J.det;
      for (int j = 0; j < t.n_test; ++j) {
        const size_t bj = static_cast<size_t>(j) * basis.nq + q;
        const double dx = (J.j22 * basis.dxi[bj] - J.j12 * basis.deta[bj]) * inv;
        const double dy = (-J.j21 * basis.dxi[bj] + J.j11 * basis.deta[bj]) * inv;
        const size_t at = static_cast<size_t>(j) * t.n_quad + q;
        gx[at] = static_cast<float>(wdet * dx);
        gy[at] = static_cast<float>(wdet * dy);
        tv[at] = static_cast<float>(wdet * basis.val[bj]);
      }
    }
  }
  return t;
}

// forcing(j,k) = sum_q test(k,j,q) * (float) f(x_kq), summed in q order
inline void assemble_forcing(ElementTensors& t, const ScalarField2D& f) {
  t.forcing.assign(static_cast<size_t>(t.n_test) * t.n_elem, 0.0f);
  std::vector<float> fq(t.n_quad);
  for (int k = 0; k < t.n_elem; ++k) {
    for (int q = 0; q < t.n_quad; ++q) {
      const Point2 p = t.quad_points[static_cast<size_t>(k) * t.n_quad + q];
      const double v = f(p.x, p.y);
      if (!std::isfinite(v))
        throw AssemblyError("forcing is not finite at (" + std::to_string(p.x) + ", " + std::to_string(p.y) + ")");
      fq[q] = static_cast<float>(v);
    }
    for (int j = 0; j < t.n_test; ++j) {
      const float* row = t.test.data() + (static_cast<size_t>(k) * t.n_test + j) * t.n_quad;
      float acc = 0.0f;
      for (int q = 0; q < t.n_quad; ++q) acc += row[q] * fq[q];
      t.forcing[static_cast<size_t>(k) * t.n_test + j] = acc;
    }
  }
}

struct SampledPoints {
  std::vector<Point2> points;
  std::vector<double> values;
};

// arc-length uniform samples on single-incidence edges, seeded offset
inline SampledPoints sample_boundary(const Mesh& mesh, int n, const ScalarField2D& g, std::uint64_t seed) {
  if (n < 1) throw InvalidArgumentError("sample_boundary: n must be >= 1");
  const auto edges = boundary_edges(mesh);
  if (edges.empty()) throw InvalidArgumentError("sample_boundary: mesh has no boundary edges");
  std::vector<double> len(edges.size());
  double perimeter = 0.0;
  for (size_t i = 0; i < edges.size(); ++i) {
    const Point2 a = mesh.nodes[edges[i].first], b = mesh.nodes[edges[i].second];
    len[i] = std::hypot(b.x - a.x, b.y - a.y);
    perimeter += len[i];
  }
  Rng rng(seed);
  const double shift = rng.uniform();
  SampledPoints out;
  size_t e = 0;
  double walked = 0.0;
  for (int i = 0; i < n; ++i) {
    const double s = (i + shift) * perimeter / n;
    while (e + 1 < edges.size() && walked + len[e] < s) walked += len[e++];
    const double t = std::min(1.0, (s - walked) / len[e]);
    const Point2 a = mesh.nodes[edges[e].first], b = mesh.nodes[edges[e].second];
    const Point2 p{a.x + t * (b.x - a.x), a.y + t * (b.y - a.y)};
    const double v = g(p.x, p.y);
    if (!std::isfinite(v))
      throw AssemblyError("boundary data is not finite at (" + std::to_string(p.x) + ", " + std::to_string(p.y) + ")");
    out.points.push_back(p);
    out.values.push_back(v);
  }
  return out;
}

// random cell, then a random reference point mapped into it
inline SampledPoints sample_sensors(const Mesh& mesh, int n, const ScalarField2D& u, std::uint64_t seed) {
  if (n < 1) throw InvalidArgumentError("sample_sensors: n must be >= 1");
  Rng rng(seed);
  SampledPoints out;
  for (int i = 0; i < n; ++i) {
    const int k = static_cast<int>(rng.integer(static_cast<std::uint64_t>(mesh.n_elements())));
    const double xi = rng.uniform(-1.0, 1.0);
    const double eta = rng.uniform(-1.0, 1.0);
    const Point2 p = map_point(bilinear_coeffs(mesh, k), xi, eta);
    const double v = u(p.x, p.y);
    if (!std::isfinite(v))
      throw AssemblyError("sensor data is not finite at (" + std::to_string(p.x) + ", " + std::to_string(p.y) + ")");
    out.points.push_back(p);
    out.values.push_back(v);
  }
  return out;
}

// ---- network: reference parameter order (per layer W row-major, b; scalars) --
enum class Activation { tanh, sigmoid };

struct DenseNetwork {
  std::vector<int> layer_sizes;
  Activation activation = Activation::tanh;
  std::vector<std::pair<std::string, float>> scalars;
  std::vector<float> params;  // flat, to_parameters order (scalars included at the end)
  int parameter_count() const {
    int n = 0;
    for (size_t l = 0; l + 1 < layer_sizes.size(); ++l) n += layer_sizes[l + 1] * layer_sizes[l] + layer_sizes[l + 1];
    return n + static_cast<int>(scalars.size());
  }
};

// Glorot-uniform from one seeded stream, row-major per layer, zero biases
inline DenseNetwork init_network(const std::vector<int>& sizes, std::uint64_t seed,
                                 Activation act = Activation::tanh,
                                 const std::vector<std::pair<std::string, double>>& scalars = {}) {
  if (sizes.size() < 2) throw InvalidArgumentError("init_network: need at least input and output");
  for (int s : sizes)
    if (s < 1) throw InvalidArgumentError("init_network: layer sizes must be >= 1");
  if (sizes.front() != 2) throw InvalidArgumentError("init_network: input dimension must be 2");
  DenseNetwork net;
  net.layer_sizes = sizes;
  net.activation = act;
  Rng rng(seed);
  for (size_t l = 0; l + 1 < sizes.size(); ++l) {
    const int fi = sizes[l], fo = sizes[l + 1];
    const double bound = std::sqrt(6.0 / (fi + fo));
    for (int r = 0; r < fo * fi; ++r) net.params.push_back(static_cast<float>(rng.uniform(-bound, bound)));
    net.params.insert(net.params.end(), static_cast<size_t>(fo), 0.0f);
  }
  for (const auto& [name, v] : scalars) {
    net.scalars.emplace_back(name, static_cast<float>(v));
    net.params.push_back(static_cast<float>(v));
  }
  return net;
}

// ---- coefficients + the assembled problem ---------------------------------------
enum class EpsSource { fixed = 0, scalar = 1, spatial = 2 };

struct PdeCoefficients {
  float eps = 1.0f, bx = 0.0f, by = 0.0f;
  EpsSource source = EpsSource::fixed;
  int eps_scalar_index = 0;
  bool has_convection() const { return bx != 0.0f || by != 0.0f; }
};

struct LossWeights {
  double tau = 10.0, gamma = 10.0;
};

struct ProblemAssembly {
  ElementTensors tensors;
  PdeCoefficients coeffs;
  SampledPoints boundary, sensors;
  std::vector<Point2> batch;  // interior ++ boundary ++ sensors
  long long n_interior = 0, n_boundary = 0, n_sensors = 0;
  // LossForm::strong (trainer.hpp:178-188): f at the interior points, cast
  // to float as strong_residual_loss does at use (losses.hpp:450)
  bool strong = false;
  std::vector<float> strong_forcing;
  void build_batch() {
    n_interior = static_cast<long long>(tensors.quad_points.size());
    n_boundary = static_cast<long long>(boundary.points.size());
    n_sensors = static_cast<long long>(sensors.points.size());
    batch = tensors.quad_points;
    batch.insert(batch.end(), boundary.points.begin(), boundary.points.end());
    batch.insert(batch.end(), sensors.points.begin(), sensors.points.end());
  }
};

}  // namespace vpinn
