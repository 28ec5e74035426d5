// Quadrature, reference test basis and bilinear cell geometry — the host
// precompute feeding the device tensors.  Restates the reference algorithms
// (proj/include/vpinn/quadrature.hpp:20-198, basis.hpp:13-60,
// geometry.hpp:67-141) in the same floating-point operation order so the
// assembled premultipliers are the same bits as the oracle's.
#pragma once

#include <array>
#include <cmath>
#include <vector>

#include "vp_core.hpp"

namespace vpinn {

// ---- Jacobi / Legendre --------------------------------------------------
struct PolyEval {
  double value = 0.0;
  double derivative = 0.0;
};

inline double jacobi_recurrence(int n, double a, double b, double x) {
  if (n == 0) return 1.0;
  double p_prev = 1.0;
  double p = 0.5 * (a - b) + 0.5 * (a + b + 2.0) * x;
  for (int k = 2; k <= n; ++k) {
    const double s = a + b;
    const double d1 = 2.0 * k * (k + s) * (2.0 * k + s - 2.0);
    const double d2 = (2.0 * k + s - 1.0) * (a * a - b * b);
    const double d3 = (2.0 * k + s - 2.0) * (2.0 * k + s - 1.0) * (2.0 * k + s);
    const double d4 = 2.0 * (k + a - 1.0) * (k + b - 1.0) * (2.0 * k + s);
    const double p_next = ((d2 + d3 * x) * p - d4 * p_prev) / d1;
    p_prev = p;
    p = p_next;
  }
  return p;
}

inline PolyEval jacobi_polynomial(int n, double alpha, double beta, double x) {
  if (n < 0) throw InvalidArgumentError("jacobi_polynomial: order must be >= 0");
  if (!(alpha > -1.0) || !(beta > -1.0))
    throw InvalidArgumentError("jacobi_polynomial: alpha, beta must be > -1");
  PolyEval e;
  e.value = jacobi_recurrence(n, alpha, beta, x);
  if (n > 0)
    e.derivative = 0.5 * (n + alpha + beta + 1.0) * jacobi_recurrence(n - 1, alpha + 1.0, beta + 1.0, x);
  return e;
}

// 1-D test family v_k = P_{k+1} - P_{k-1} (vanishes at +-1)
inline PolyEval test_function_1d(int k, double x) {
  if (k < 1) throw InvalidArgumentError("test_function_1d: index must be >= 1");
  const PolyEval up = jacobi_polynomial(k + 1, 0.0, 0.0, x);
  const PolyEval dn = jacobi_polynomial(k - 1, 0.0, 0.0, x);
  return {up.value - dn.value, up.derivative - dn.derivative};
}

enum class QuadratureKind { gauss_legendre, gauss_lobatto };

struct Rule1D {
  std::vector<double> x, w;
  int size() const { return static_cast<int>(x.size()); }
};

inline void legendre_with_derivative(int n, double x, double& p, double& dp) {
  double q = 0.0;  // P_{m-1}
  p = 1.0;
  for (int m = 1; m <= n; ++m) {
    const double nxt = ((2.0 * m - 1.0) * x * p - (m - 1.0) * q) / m;
    q = p;
    p = nxt;
  }
  dp = (n == 0) ? 0.0 : n * (x * p - q) / (x * x - 1.0);
}

inline Rule1D gauss_rule_1d(int n, QuadratureKind kind) {
  Rule1D r;
  r.x.assign(n > 0 ? n : 0, 0.0);
  r.w.assign(n > 0 ? n : 0, 0.0);
  if (kind == QuadratureKind::gauss_legendre) {
    if (n < 1) throw InvalidArgumentError("gauss_rule_1d: legendre needs n >= 1");
    for (int i = 0; i < (n + 1) / 2; ++i) {
      double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
      double p = 0.0, dp = 0.0;
      for (int it = 0; it < 100; ++it) {
        legendre_with_derivative(n, t, p, dp);
        const double step = p / dp;
        t -= step;
        if (std::abs(step) <= 1e-15) break;
      }
      legendre_with_derivative(n, t, p, dp);
      const double wt = 2.0 / ((1.0 - t * t) * dp * dp);
      r.x[n - 1 - i] = t;
      r.x[i] = -t;
      r.w[n - 1 - i] = wt;
      r.w[i] = wt;
    }
    if (n % 2 == 1) r.x[n / 2] = 0.0;
  } else {
    if (n < 2) throw InvalidArgumentError("gauss_rule_1d: lobatto needs n >= 2");
    r.x.front() = -1.0;
    r.x.back() = 1.0;
    const double w_end = 2.0 / (static_cast<double>(n) * (n - 1.0));
    r.w.front() = w_end;
    r.w.back() = w_end;
    const int m = n - 1;
    for (int i = 1; i <= (n - 1) / 2; ++i) {
      double t = -std::cos(M_PI * i / static_cast<double>(m));
      for (int it = 0; it < 100; ++it) {
        double p = 0.0, dp = 0.0;
        legendre_with_derivative(m, t, p, dp);
        const double d2p = (2.0 * t * dp - m * (m + 1.0) * p) / (1.0 - t * t);
        const double step = dp / d2p;
        t -= step;
        if (std::abs(step) <= 1e-15) break;
      }
      double p = 0.0, dp = 0.0;
      legendre_with_derivative(m, t, p, dp);
      const double wt = 2.0 / (static_cast<double>(n) * (n - 1.0) * p * p);
      r.x[i] = t;
      r.w[i] = wt;
      r.x[n - 1 - i] = -t;
      r.w[n - 1 - i] = wt;
    }
    if (n % 2 == 1) {
      r.x[n / 2] = 0.0;
      double p = 0.0, dp = 0.0;
      legendre_with_derivative(m, 0.0, p, dp);
      r.w[n / 2] = 2.0 / (static_cast<double>(n) * (n - 1.0) * p * p);
    }
  }
  return r;
}

// Point order contract: q = iy * n_xi + ix (eta outer, xi inner).
struct QuadratureRule2D {
  std::vector<double> xi, eta, weights;
  int n_xi = 0, n_eta = 0;
  int size() const { return n_xi * n_eta; }
};

inline QuadratureRule2D tensor_product_rule(const Rule1D& rx, const Rule1D& ry) {
  QuadratureRule2D r;
  r.n_xi = rx.size();
  r.n_eta = ry.size();
  for (int iy = 0; iy < r.n_eta; ++iy)
    for (int ix = 0; ix < r.n_xi; ++ix) {
      r.xi.push_back(rx.x[ix]);
      r.eta.push_back(ry.x[iy]);
      r.weights.push_back(rx.w[ix] * ry.w[iy]);
    }
  return r;
}

// ---- reference-square basis: row j = jy*n + jx, column q, row-major ----
struct ReferenceBasis {
  int n_per_dim = 0, nq = 0;
  std::vector<double> val, dxi, deta;  // [j * nq + q]
  int n_test() const { return n_per_dim * n_per_dim; }
};

inline ReferenceBasis reference_basis(int n, const QuadratureRule2D& rule) {
  if (n < 1) throw InvalidArgumentError("reference_basis: n_test_per_dim must be >= 1");
  const int nq = rule.size();
  if (nq == 0) throw InvalidArgumentError("reference_basis: empty rule");
  ReferenceBasis b;
  b.n_per_dim = n;
  b.nq = nq;
  std::vector<PolyEval> ex(static_cast<size_t>(n) * nq), ey(ex.size());
  for (int q = 0; q < nq; ++q)
    for (int k = 0; k < n; ++k) {
      ex[static_cast<size_t>(k) * nq + q] = test_function_1d(k + 1, rule.xi[q]);
      ey[static_cast<size_t>(k) * nq + q] = test_function_1d(k + 1, rule.eta[q]);
    }
  const int nt = n * n;
  b.val.resize(static_cast<size_t>(nt) * nq);
  b.dxi.resize(b.val.size());
  b.deta.resize(b.val.size());
  for (int jy = 0; jy < n; ++jy)
    for (int jx = 0; jx < n; ++jx) {
      const size_t row = static_cast<size_t>(jy * n + jx) * nq;
      for (int q = 0; q < nq; ++q) {
        const PolyEval& a = ex[static_cast<size_t>(jx) * nq + q];
        const PolyEval& c = ey[static_cast<size_t>(jy) * nq + q];
        b.val[row + q] = a.value * c.value;
        b.dxi[row + q] = a.derivative * c.value;
        b.deta[row + q] = a.value * c.derivative;
      }
    }
  return b;
}

// ---- quadrilateral cells --------------------------------------------------
struct Point2 {
  double x = 0.0, y = 0.0;
};

struct Mesh {
  std::vector<Point2> nodes;
  std::vector<std::array<int, 4>> elements;  // CCW, vertex 0 <-> reference (-1,-1)
  std::vector<int> boundary_node_ids;        // sorted, unique
  int n_nodes() const { return static_cast<int>(nodes.size()); }
  int n_elements() const { return static_cast<int>(elements.size()); }
};

// x(xi,eta) = c0 + c1 xi + c2 eta + c3 xi eta, same for y
struct BilinearCoeffs {
  double xc0, xc1, xc2, xc3, yc0, yc1, yc2, yc3;
};

inline BilinearCoeffs bilinear_coeffs(const Mesh& m, int k) {
  const auto& e = m.elements.at(static_cast<size_t>(k));
  const Point2 a = m.nodes.at(e[0]), b = m.nodes.at(e[1]), c = m.nodes.at(e[2]), d = m.nodes.at(e[3]);
  BilinearCoeffs r;
  r.xc0 = 0.25 * (a.x + b.x + c.x + d.x);
  r.xc1 = 0.25 * (-a.x + b.x + c.x - d.x);
  r.xc2 = 0.25 * (-a.x - b.x + c.x + d.x);
  r.xc3 = 0.25 * (a.x - b.x + c.x - d.x);
  r.yc0 = 0.25 * (a.y + b.y + c.y + d.y);
  r.yc1 = 0.25 * (-a.y + b.y + c.y - d.y);
  r.yc2 = 0.25 * (-a.y - b.y + c.y + d.y);
  r.yc3 = 0.25 * (a.y - b.y + c.y - d.y);
  return r;
}

inline Point2 map_point(const BilinearCoeffs& c, double xi, double eta) {
  return {c.xc0 + c.xc1 * xi + c.xc2 * eta + c.xc3 * xi * eta,
          c.yc0 + c.yc1 * xi + c.yc2 * eta + c.yc3 * xi * eta};
}

struct Jacobian {
  double j11, j12, j21, j22, det;  // j11 = dx/dxi, j12 = dy/dxi, j21 = dx/deta, j22 = dy/deta
};

inline Jacobian jacobian_at(const BilinearCoeffs& c, double xi, double eta) {
  Jacobian j;
  j.j11 = c.xc1 + c.xc3 * eta;
  j.j12 = c.yc1 + c.yc3 * eta;
  j.j21 = c.xc2 + c.xc3 * xi;
  j.j22 = c.yc2 + c.yc3 * xi;
  j.det = j.j11 * j.j22 - j.j12 * j.j21;
  return j;
}

inline double signed_area(const Mesh& m, int k) {
  double s = 0.0;
  const auto& e = m.elements[static_cast<size_t>(k)];
  for (int i = 0; i < 4; ++i) {
    const Point2 p = m.nodes[e[i]], q = m.nodes[e[(i + 1) % 4]];
    s += p.x * q.y - q.x * p.y;
  }
  return 0.5 * s;
}

}  // namespace vpinn
