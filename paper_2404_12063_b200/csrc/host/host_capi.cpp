// C-ABI of the host pipeline (include/vpinn_host.h) over the C++ API in
// vp_gpu_trainer.hpp.
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <tuple>

#include "vp_gpu_trainer.hpp"
#include "vpinn_host.h"

struct vpinn_host_mesh {
  vpinn::Mesh mesh;
};

struct vpinn_host_problem {
  vpinn::FullConfig cfg;
  vpinn::BuiltProblem bp;
  vpinn::QuadratureRule2D rule;
  // one view per (device, rank, world), kept for the problem's lifetime: a
  // vpinn_gpu_problem handed out earlier stays valid while the problem lives
  std::map<std::tuple<int, int, int>, std::unique_ptr<vpinn::GpuView>> views;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const vpinn::Error& e) {
    g_err = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

vpinn::Mesh mesh_from_source(const vpinn_mesh_source& s) {
  switch (s.kind) {
    case VPINN_MESH_STRUCTURED: {
      vpinn::Mesh m = vpinn::generate_structured_mesh(s.nx, s.ny, {s.x0, s.x1}, {s.y0, s.y1});
      vpinn::skew_mesh_nodes(m, s.skew, s.skew_seed);
      return m;
    }
    case VPINN_MESH_GEAR:
      return vpinn::gear_mesh(s.nx, s.ny);
    case VPINN_MESH_DISK:
      return vpinn::disk_mesh(s.nx);
    case VPINN_MESH_HANDLE:
      if (!s.mesh) throw vpinn::InvalidArgumentError("mesh source: null handle");
      return s.mesh->mesh;
    default:
      throw vpinn::InvalidArgumentError("mesh source: unknown kind " + std::to_string(s.kind));
  }
}

std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  std::ostringstream o;
  o.precision(17);
  o << v;
  return o.str();
}

}  // namespace

extern "C" {

const char* vpinn_host_last_error(void) { return g_err.c_str(); }

int vpinn_host_mesh_read_gmsh(const char* path, vpinn_host_mesh** out) {
  *out = nullptr;
  return guarded([&] {
    auto m = std::make_unique<vpinn_host_mesh>();
    m->mesh = vpinn::read_gmsh_file(path);
    *out = m.release();
  });
}

int vpinn_host_mesh_parse_gmsh(const char* text, vpinn_host_mesh** out) {
  *out = nullptr;
  return guarded([&] {
    auto m = std::make_unique<vpinn_host_mesh>();
    std::istringstream in(text ? text : "");
    m->mesh = vpinn::read_gmsh_ascii(in);
    *out = m.release();
  });
}

int vpinn_host_mesh_make(const vpinn_mesh_source* src, vpinn_host_mesh** out) {
  *out = nullptr;
  return guarded([&] {
    auto m = std::make_unique<vpinn_host_mesh>();
    m->mesh = mesh_from_source(*src);
    *out = m.release();
  });
}

void vpinn_host_mesh_counts(const vpinn_host_mesh* m, int64_t* c) {
  c[0] = m->mesh.n_nodes();
  c[1] = m->mesh.n_elements();
  c[2] = static_cast<int64_t>(m->mesh.boundary_node_ids.size());
}

void vpinn_host_mesh_arrays(const vpinn_host_mesh* m, double* nodes, int32_t* cells, int32_t* bnd) {
  const auto& M = m->mesh;
  if (nodes)
    for (int i = 0; i < M.n_nodes(); ++i) {
      nodes[2 * i] = M.nodes[i].x;
      nodes[2 * i + 1] = M.nodes[i].y;
    }
  if (cells)
    for (int k = 0; k < M.n_elements(); ++k)
      for (int c = 0; c < 4; ++c) cells[4 * k + c] = M.elements[k][c];
  if (bnd)
    for (size_t i = 0; i < M.boundary_node_ids.size(); ++i) bnd[i] = M.boundary_node_ids[i];
}

void vpinn_host_mesh_health(const vpinn_host_mesh* m, int64_t* deg, int64_t* mis) {
  const auto h = vpinn::validate_mesh(m->mesh);
  *deg = static_cast<int64_t>(h.degenerate.size());
  *mis = static_cast<int64_t>(h.misoriented.size());
}

void vpinn_host_mesh_free(vpinn_host_mesh* m) { delete m; }

int vpinn_host_gear_msh_text(int n_r, int n_t, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    const std::string t = vpinn::gear_msh41_text(n_r, n_t);
    if (len) *len = t.size();
    if (cap > 0) {
      if (cap < t.size() + 1) throw vpinn::InvalidArgumentError("gear text: buffer too small");
      std::memcpy(buf, t.c_str(), t.size() + 1);
    }
  });
}

int vpinn_host_problem_from_config(const char* json, const char* base_dir, const vpinn_mesh_source* mesh,
                                   vpinn_host_problem** out) {
  return vpinn_host_problem_from_config_ex(json, base_dir, mesh, 0, out);
}

int vpinn_host_problem_from_config_ex(const char* json, const char* base_dir, const vpinn_mesh_source* mesh,
                                      int flags, vpinn_host_problem** out) {
  *out = nullptr;
  return guarded([&] {
    auto p = std::make_unique<vpinn_host_problem>();
    p->cfg = vpinn::parse_config_text(json ? json : "", "<config>", base_dir ? base_dir : "");
    std::optional<vpinn::Mesh> premade;
    if (mesh && mesh->kind != VPINN_MESH_FROM_CONFIG) premade = mesh_from_source(*mesh);
    p->bp = vpinn::build_problem(p->cfg, std::move(premade), (flags & VPINN_HOST_DEVICE_ASSEMBLY) != 0);
    const vpinn::Rule1D r1 = vpinn::gauss_rule_1d(p->cfg.disc.n_quad_per_dim, p->cfg.disc.quadrature);
    p->rule = vpinn::tensor_product_rule(r1, r1);
    *out = p.release();
  });
}

void vpinn_host_problem_counts(const vpinn_host_problem* p, int64_t* c) {
  const auto& t = p->bp.pa.tensors;
  c[0] = t.n_elem;
  c[1] = t.n_test;
  c[2] = t.n_quad;
  c[3] = p->bp.pa.n_interior;
  c[4] = p->bp.pa.n_boundary;
  c[5] = p->bp.pa.n_sensors;
  c[6] = p->bp.net.parameter_count();
  c[7] = p->bp.precision_downgraded ? 1 : 0;
}

int vpinn_host_problem_view(const vpinn_host_problem* p, int device, int rank, int world, vpinn_gpu_problem* view) {
  return guarded([&] {
    auto* mp = const_cast<vpinn_host_problem*>(p);
    auto& slot = mp->views[std::make_tuple(device, rank, world)];
    if (!slot) slot = vpinn::make_gpu_view(p->bp, device, rank, world);
    *view = slot->p;
  });
}

void vpinn_host_problem_params(const vpinn_host_problem* p, float* out) {
  std::memcpy(out, p->bp.net.params.data(), sizeof(float) * p->bp.net.params.size());
}

void vpinn_host_problem_rule(const vpinn_host_problem* p, double* xi, double* eta, double* w) {
  for (int q = 0; q < p->rule.size(); ++q) {
    xi[q] = p->rule.xi[q];
    eta[q] = p->rule.eta[q];
    w[q] = p->rule.weights[q];
  }
}

void vpinn_host_problem_free(vpinn_host_problem* p) { delete p; }

int vpinn_host_train(vpinn_host_problem* p, int device, float* params_out, char* report, size_t cap, size_t* len) {
  return guarded([&] {
    vpinn::GpuContext gpu(p->bp, device);
    vpinn::DenseNetwork net = p->bp.net;
    vpinn::RunReport r = vpinn::train(net, p->bp, p->cfg.training, gpu);
    const auto& pr = p->cfg.problem;
    const bool has_exact = !pr.exact_solution.empty();
    if (has_exact) {
      const auto b = vpinn::bounding_box(p->bp.mesh);
      r.metrics = vpinn::evaluate_metrics(gpu, vpinn::lookup_field(pr.exact_solution), p->cfg.output.grid_nx,
                                          p->cfg.output.grid_ny, {b.x0, b.x1}, {b.y0, b.y1});
    }
    if (params_out) std::memcpy(params_out, net.params.data(), sizeof(float) * net.params.size());
    std::ostringstream o;
    o << "{\"steps_run\":" << r.steps_run << ",\"converged\":" << (r.converged ? "true" : "false")
      << ",\"stop_reason\":\"" << r.stop_reason << "\",\"final_eps\":" << jnum(r.final_eps)
      << ",\"eps_abs_error\":" << jnum(r.eps_abs_error) << ",\"precision\":\"single\""
      << ",\"precision_downgraded\":" << (p->bp.precision_downgraded ? "true" : "false") << ",\"timing\":{\"median_s\":"
      << jnum(r.timing.median_s) << ",\"p10_s\":" << jnum(r.timing.p10_s) << ",\"p90_s\":" << jnum(r.timing.p90_s)
      << ",\"samples\":" << r.timing.samples.size() << "},\"metrics\":";
    if (has_exact)
      o << "{\"mae\":" << jnum(r.metrics.mae) << ",\"rel_l2\":" << jnum(r.metrics.rel_l2)
        << ",\"max_err\":" << jnum(r.metrics.max_err) << "}";
    else
      o << "null";
    o << ",\"history\":[";
    for (size_t i = 0; i < r.history.size(); ++i) {
      const auto& h = r.history[i];
      o << (i ? "," : "") << "{\"step\":" << h.step << ",\"total\":" << jnum(h.total)
        << ",\"variational\":" << jnum(h.variational) << ",\"boundary\":" << jnum(h.boundary)
        << ",\"sensor\":" << jnum(h.sensor) << ",\"lr\":" << jnum(h.lr) << ",\"eps\":" << jnum(h.eps) << "}";
    }
    o << "]}";
    const std::string s = o.str();
    if (len) *len = s.size();
    if (cap > 0) {
      if (cap < s.size() + 1) throw vpinn::InvalidArgumentError("report buffer too small");
      std::memcpy(report, s.c_str(), s.size() + 1);
    }
  });
}

int vpinn_host_bench_case(const char* json, int e, int t, int q, double skew, int reps, int device, double* out3) {
  return guarded([&] {
    const vpinn::FullConfig cfg = vpinn::parse_config_text(json ? json : "", "<config>");
    const auto row = vpinn::bench_case(cfg, e, t, q, skew, reps, device);
    out3[0] = row.median_s;
    out3[1] = row.p10_s;
    out3[2] = row.p90_s;
  });
}

}  // extern "C"
