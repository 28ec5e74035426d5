// Mesh construction and loading on the host: structured grids, the
// benchmark's seeded skew, validation, boundary edges, Gmsh ASCII 2.2 / 4.1
// import, and the synthetic gear / disk generators of the benchmark configs.
// Semantics follow reference proj/include/vpinn/geometry.hpp:49-244,
// mesh_io.hpp:20-268, commands.hpp:75-97 and data/gen_fixtures.py:106-179.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <map>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "vp_discretization.hpp"

namespace vpinn {

// node (i,j) -> j*(nx+1)+i; endpoints exact; cells CCW from the lower left
inline Mesh generate_structured_mesh(int nx, int ny, std::pair<double, double> xr,
                                     std::pair<double, double> yr) {
  if (nx < 1 || ny < 1) throw InvalidArgumentError("generate_structured_mesh: nx, ny must be >= 1");
  if (!(xr.second > xr.first) || !(yr.second > yr.first))
    throw InvalidArgumentError("generate_structured_mesh: empty range");
  Mesh m;
  const double hx = (xr.second - xr.first) / nx, hy = (yr.second - yr.first) / ny;
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i)
      m.nodes.push_back({i == nx ? xr.second : xr.first + i * hx,
                         j == ny ? yr.second : yr.first + j * hy});
  const int stride = nx + 1;
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex) {
      const int v0 = ey * stride + ex;
      m.elements.push_back({v0, v0 + 1, v0 + 1 + stride, v0 + stride});
    }
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i)
      if (i == 0 || i == nx || j == 0 || j == ny) m.boundary_node_ids.push_back(j * stride + i);
  return m;
}

// edges incident to exactly one cell, ordered by (min id, max id) -- the
// order of the reference's std::map walk.  Edges are bucketed by their min
// id (counting sort), each bucket's max ids sorted; a run of length one is a
// boundary edge.  O(cells) instead of a 4-cells-node tree (gear: 5.4 ms ->
// ~0.3 ms, the largest part of a device-assembly problem build).
inline std::vector<std::pair<int, int>> boundary_edges(const Mesh& m) {
  int lo = 0, hi = -1;
  for (const auto& e : m.elements)
    for (int i = 0; i < 4; ++i) {
      lo = std::min(lo, e[i]);
      hi = std::max(hi, e[i]);
    }
  std::vector<std::pair<int, int>> out;
  if (lo >= 0) {
    std::vector<int> start(static_cast<size_t>(hi) + 2, 0);
    for (const auto& e : m.elements)
      for (int i = 0; i < 4; ++i) ++start[std::min(e[i], e[(i + 1) & 3]) + 1];
    for (size_t a = 1; a < start.size(); ++a) start[a] += start[a - 1];
    std::vector<int> fill(start.begin(), start.end() - 1), nb(static_cast<size_t>(start.back()));
    for (const auto& e : m.elements)
      for (int i = 0; i < 4; ++i) {
        const int a = e[i], b = e[(i + 1) & 3];
        nb[fill[std::min(a, b)]++] = std::max(a, b);
      }
    for (int a = 0; a <= hi; ++a) {
      const auto first = nb.begin() + start[a], last = nb.begin() + start[a + 1];
      std::sort(first, last);
      for (auto it = first; it != last;) {
        auto run = it + 1;
        while (run != last && *run == *it) ++run;
        if (run - it == 1) out.emplace_back(a, *it);
        it = run;
      }
    }
    return out;
  }
  // negative ids (a malformed mesh the validators report later): the tree walk
  std::map<std::pair<int, int>, int> count;
  for (const auto& e : m.elements)
    for (int i = 0; i < 4; ++i) {
      const int a = e[i], b = e[(i + 1) & 3];
      count[{std::min(a, b), std::max(a, b)}] += 1;
    }
  for (const auto& [edge, n] : count)
    if (n == 1) out.push_back(edge);
  return out;
}

struct MeshHealth {
  std::vector<int> degenerate, misoriented;
  bool ok() const { return degenerate.empty() && misoriented.empty(); }
};

// determinant scanned on a 5x5 reference grid incl. corners
inline MeshHealth validate_mesh(const Mesh& m) {
  MeshHealth h;
  for (int k = 0; k < m.n_elements(); ++k) {
    const BilinearCoeffs c = bilinear_coeffs(m, k);
    double lo = std::numeric_limits<double>::infinity();
    for (int iy = 0; iy <= 4; ++iy)
      for (int ix = 0; ix <= 4; ++ix) lo = std::min(lo, jacobian_at(c, -1.0 + 0.5 * ix, -1.0 + 0.5 * iy).det);
    if (!(lo > 0.0)) h.degenerate.push_back(k);
    if (!(signed_area(m, k) > 0.0)) h.misoriented.push_back(k);
  }
  return h;
}

struct BBox {
  double x0, x1, y0, y1;
};
inline BBox bounding_box(const Mesh& m) {
  if (m.nodes.empty()) throw InvalidArgumentError("bounding_box: empty mesh");
  BBox b{m.nodes[0].x, m.nodes[0].x, m.nodes[0].y, m.nodes[0].y};
  for (const auto& p : m.nodes) {
    b.x0 = std::min(b.x0, p.x);
    b.x1 = std::max(b.x1, p.x);
    b.y0 = std::min(b.y0, p.y);
    b.y1 = std::max(b.y1, p.y);
  }
  return b;
}

// seeded perturbation of interior nodes by up to amount * mean cell size
inline void skew_mesh_nodes(Mesh& m, double amount, std::uint64_t seed) {
  if (amount <= 0.0) return;
  const BBox b = bounding_box(m);
  const double h = std::sqrt((b.x1 - b.x0) * (b.y1 - b.y0) / static_cast<double>(m.n_elements()));
  const double tol = 1e-12 * std::max(b.x1 - b.x0, b.y1 - b.y0);
  Rng rng(seed);
  for (auto& p : m.nodes) {
    const bool rim = std::abs(p.x - b.x0) < tol || std::abs(p.x - b.x1) < tol ||
                     std::abs(p.y - b.y0) < tol || std::abs(p.y - b.y1) < tol;
    if (rim) continue;
    p.x += rng.uniform(-amount * h, amount * h);
    p.y += rng.uniform(-amount * h, amount * h);
  }
  if (!validate_mesh(m).ok())
    throw AssemblyError("skew_mesh_nodes: perturbation produced a degenerate element; lower the skew amount");
}

// ---- Gmsh ASCII import ----------------------------------------------------
namespace gmsh_detail {

struct Lines {
  std::vector<std::string> v;
  int after(const std::string& section) const {
    const std::string key = "$" + section;
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i] == key) return static_cast<int>(i) + 1;
    return -1;
  }
  const std::string& at(int i) const {
    if (i < 0 || static_cast<size_t>(i) >= v.size())
      throw MeshFileError("gmsh: unexpected end of file");
    return v[static_cast<size_t>(i)];
  }
};

inline std::string strip(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}

template <typename T>
T take(std::istringstream& in, int line, const char* what) {
  T v;
  if (!(in >> v))
    throw MeshFileError("gmsh: line " + std::to_string(line + 1) + ": expected " + what);
  return v;
}

struct Raw {
  std::vector<std::pair<std::int64_t, Point2>> nodes;
  std::vector<std::array<std::int64_t, 4>> quads;
  std::vector<std::int64_t> tagged;  // boundary node tags from line/point elements
  bool has_tags = false;
};

inline void element(Raw& r, int type, const std::vector<std::int64_t>& t, int line) {
  const std::string where = "gmsh: line " + std::to_string(line + 1) + ": ";
  if (type == 3) {
    if (t.size() != 4) throw MeshFileError(where + "quad needs 4 nodes");
    r.quads.push_back({t[0], t[1], t[2], t[3]});
  } else if (type == 1) {
    if (t.size() != 2) throw MeshFileError(where + "line element needs 2 nodes");
    r.tagged.push_back(t[0]);
    r.tagged.push_back(t[1]);
    r.has_tags = true;
  } else if (type == 15) {
    if (t.empty()) throw MeshFileError(where + "point element needs a node");
    r.tagged.push_back(t[0]);
    r.has_tags = true;
  } else {
    throw MeshFileError(where + "unsupported element type " + std::to_string(type) +
                        " (only quads, lines and points are accepted)");
  }
}

inline Raw v22(const Lines& f) {
  Raw r;
  int at = f.after("Nodes");
  if (at < 0) throw MeshFileError("gmsh: missing $Nodes section");
  {
    std::istringstream h(f.at(at));
    const auto n = take<std::int64_t>(h, at, "node count");
    for (std::int64_t i = 0; i < n; ++i) {
      const int ln = at + 1 + static_cast<int>(i);
      std::istringstream s(f.at(ln));
      const auto tag = take<std::int64_t>(s, ln, "node tag");
      const double x = take<double>(s, ln, "x"), y = take<double>(s, ln, "y");
      take<double>(s, ln, "z");
      r.nodes.push_back({tag, {x, y}});
    }
  }
  at = f.after("Elements");
  if (at < 0) throw MeshFileError("gmsh: missing $Elements section");
  std::istringstream h(f.at(at));
  const auto n = take<std::int64_t>(h, at, "element count");
  for (std::int64_t i = 0; i < n; ++i) {
    const int ln = at + 1 + static_cast<int>(i);
    std::istringstream s(f.at(ln));
    take<std::int64_t>(s, ln, "element tag");
    const int type = take<int>(s, ln, "element type");
    const int ntag = take<int>(s, ln, "tag count");
    for (int k = 0; k < ntag; ++k) take<std::int64_t>(s, ln, "tag");
    std::vector<std::int64_t> t;
    std::int64_t v;
    while (s >> v) t.push_back(v);
    element(r, type, t, ln);
  }
  return r;
}

inline Raw v41(const Lines& f) {
  Raw r;
  int at = f.after("Nodes");
  if (at < 0) throw MeshFileError("gmsh: missing $Nodes section");
  {
    std::istringstream h(f.at(at));
    const auto blocks = take<std::int64_t>(h, at, "block count");
    int ln = at + 1;
    for (std::int64_t b = 0; b < blocks; ++b) {
      std::istringstream bh(f.at(ln));
      take<int>(bh, ln, "entity dim");
      take<std::int64_t>(bh, ln, "entity tag");
      take<int>(bh, ln, "parametric flag");
      const auto cnt = take<std::int64_t>(bh, ln, "node count");
      ++ln;
      std::vector<std::int64_t> tags;
      for (std::int64_t i = 0; i < cnt; ++i, ++ln) {
        std::istringstream s(f.at(ln));
        tags.push_back(take<std::int64_t>(s, ln, "node tag"));
      }
      for (std::int64_t i = 0; i < cnt; ++i, ++ln) {
        std::istringstream s(f.at(ln));
        const double x = take<double>(s, ln, "x"), y = take<double>(s, ln, "y");
        take<double>(s, ln, "z");
        r.nodes.push_back({tags[static_cast<size_t>(i)], {x, y}});
      }
    }
  }
  at = f.after("Elements");
  if (at < 0) throw MeshFileError("gmsh: missing $Elements section");
  std::istringstream h(f.at(at));
  const auto blocks = take<std::int64_t>(h, at, "block count");
  int ln = at + 1;
  for (std::int64_t b = 0; b < blocks; ++b) {
    std::istringstream bh(f.at(ln));
    take<int>(bh, ln, "entity dim");
    take<std::int64_t>(bh, ln, "entity tag");
    const int type = take<int>(bh, ln, "element type");
    const auto cnt = take<std::int64_t>(bh, ln, "element count");
    ++ln;
    for (std::int64_t i = 0; i < cnt; ++i, ++ln) {
      std::istringstream s(f.at(ln));
      take<std::int64_t>(s, ln, "element tag");
      std::vector<std::int64_t> t;
      std::int64_t v;
      while (s >> v) t.push_back(v);
      element(r, type, t, ln);
    }
  }
  return r;
}

}  // namespace gmsh_detail

inline Mesh read_gmsh_ascii(std::istream& in) {
  gmsh_detail::Lines f;
  for (std::string l; std::getline(in, l);) f.v.push_back(gmsh_detail::strip(l));
  const int fm = f.after("MeshFormat");
  if (fm < 0) throw MeshFileError("gmsh: missing $MeshFormat section");
  std::istringstream fs(f.at(fm));
  std::string version;
  int file_type = 0, data_size = 0;
  if (!(fs >> version >> file_type >> data_size)) throw MeshFileError("gmsh: malformed $MeshFormat line");
  if (file_type != 0) throw MeshFileError("gmsh: binary files are not supported");
  gmsh_detail::Raw raw;
  if (version == "2.2")
    raw = gmsh_detail::v22(f);
  else if (version == "4.1")
    raw = gmsh_detail::v41(f);
  else
    throw MeshFileError("gmsh: unsupported format version '" + version + "' (supported: 2.2, 4.1)");
  if (raw.quads.empty()) throw MeshFileError("gmsh: mesh contains no quadrilateral elements");
  Mesh m;
  std::map<std::int64_t, int> index;
  for (const auto& [tag, p] : raw.nodes) {
    if (!index.emplace(tag, m.n_nodes()).second)
      throw MeshFileError("gmsh: duplicate node tag " + std::to_string(tag));
    m.nodes.push_back(p);
  }
  auto id = [&](std::int64_t tag) {
    const auto it = index.find(tag);
    if (it == index.end()) throw MeshFileError("gmsh: element references unknown node tag " + std::to_string(tag));
    return it->second;
  };
  for (const auto& q : raw.quads) {
    m.elements.push_back({id(q[0]), id(q[1]), id(q[2]), id(q[3])});
    // CCW normalisation keeping vertex 0 as the reference corner
    if (signed_area(m, m.n_elements() - 1) < 0.0) std::swap(m.elements.back()[1], m.elements.back()[3]);
  }
  std::vector<int> bnd;
  if (raw.has_tags) {
    for (const auto t : raw.tagged) bnd.push_back(id(t));
  } else {
    for (const auto& [a, b] : boundary_edges(m)) {
      bnd.push_back(a);
      bnd.push_back(b);
    }
  }
  std::sort(bnd.begin(), bnd.end());
  bnd.erase(std::unique(bnd.begin(), bnd.end()), bnd.end());
  m.boundary_node_ids = std::move(bnd);
  return m;
}

inline Mesh read_gmsh_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open mesh file: " + path);
  return read_gmsh_ascii(in);
}

// ---- synthetic benchmark meshes ----------------------------------------------
inline std::string fmt16g(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.16g", v);
  return buf;
}

// Gear-like annulus of data/gen_fixtures.py:158-179 (n_r rings x n_t
// segments, 12 teeth of amplitude 0.06, rims tagged), emitted as MSH 4.1
// text exactly as the generator writes it: n_r=6,n_t=96 is the bundled
// 576-cell fixture, n_r=16,n_t=887 the 14,192-cell gear of BASELINE C5.
inline std::string gear_msh41_text(int n_r, int n_t, int teeth = 12, double amp = 0.06,
                                   double r_in = 0.35, double r_out = 1.0) {
  if (n_r < 1 || n_t < 3) throw InvalidArgumentError("gear: n_r >= 1 and n_t >= 3");
  const double two_pi = 2.0 * M_PI;
  std::vector<std::pair<double, double>> nodes;
  for (int j = 0; j <= n_r; ++j) {
    const double s = static_cast<double>(j) / n_r;
    for (int i = 0; i < n_t; ++i) {
      const double th = two_pi * i / n_t;
      const double r = r_in + s * (r_out + amp * std::sin(teeth * th) - r_in);
      nodes.emplace_back(r * std::cos(th), r * std::sin(th));
    }
  }
  auto nid = [n_t](int i, int j) { return static_cast<long long>(j) * n_t + (i % n_t) + 1; };
  const long long nn = static_cast<long long>(nodes.size());
  std::string o;
  o.reserve(static_cast<size_t>(nn) * 48 + static_cast<size_t>(n_r) * n_t * 40);
  o += "$MeshFormat\n4.1 0 8\n$EndMeshFormat\n$Nodes\n";
  o += "1 " + std::to_string(nn) + " 1 " + std::to_string(nn) + "\n";
  o += "2 1 0 " + std::to_string(nn) + "\n";
  for (long long i = 1; i <= nn; ++i) o += std::to_string(i) + "\n";
  for (const auto& [x, y] : nodes) o += fmt16g(x) + " " + fmt16g(y) + " 0\n";
  o += "$EndNodes\n";
  const long long n_lines = 2LL * n_t, n_quads = static_cast<long long>(n_r) * n_t;
  o += "$Elements\n2 " + std::to_string(n_lines + n_quads) + " 1 " + std::to_string(n_lines + n_quads) + "\n";
  long long eid = 1;
  o += "1 1 1 " + std::to_string(n_lines) + "\n";
  for (int i = 0; i < n_t; ++i, ++eid)
    o += std::to_string(eid) + " " + std::to_string(nid(i, 0)) + " " + std::to_string(nid(i + 1, 0)) + "\n";
  for (int i = 0; i < n_t; ++i, ++eid)
    o += std::to_string(eid) + " " + std::to_string(nid(i, n_r)) + " " + std::to_string(nid(i + 1, n_r)) + "\n";
  o += "2 1 3 " + std::to_string(n_quads) + "\n";
  for (int j = 0; j < n_r; ++j)
    for (int i = 0; i < n_t; ++i, ++eid)
      o += std::to_string(eid) + " " + std::to_string(nid(i, j)) + " " + std::to_string(nid(i, j + 1)) + " " +
           std::to_string(nid(i + 1, j + 1)) + " " + std::to_string(nid(i + 1, j)) + "\n";
  o += "$EndElements\n";
  return o;
}

inline Mesh gear_mesh(int n_r, int n_t) {
  std::istringstream in(gear_msh41_text(n_r, n_t));
  return read_gmsh_ascii(in);
}

// BASELINE config C4: n x n square -> disk by the elliptical map
// (x,y) -> (x sqrt(1 - y^2/2), y sqrt(1 - x^2/2)) on [-1,1]^2, scaled by R;
// skewed, non-constant-Jacobian cells with all corner determinants > 0.
inline Mesh disk_mesh(int n, double radius = 1.0) {
  Mesh m = generate_structured_mesh(n, n, {-1.0, 1.0}, {-1.0, 1.0});
  for (auto& p : m.nodes) {
    const double x = p.x, y = p.y;
    p.x = radius * x * std::sqrt(1.0 - 0.5 * y * y);
    p.y = radius * y * std::sqrt(1.0 - 0.5 * x * x);
  }
  if (!validate_mesh(m).ok()) throw AssemblyError("disk_mesh: degenerate cell");
  return m;
}

}  // namespace vpinn
