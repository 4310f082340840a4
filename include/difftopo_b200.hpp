// difftopo_b200.hpp -- header-only C++ facade over the C ABI (difftopo_b200.h)
// that mirrors the reference's C++ API (proj/include/difftopo/*.hpp) for the
// initial-pass path, so a reference user switches by changing the include:
//
//   #include "difftopo/diffusion.hpp"      ->   #include "difftopo_b200.hpp"
//
//   auto mesh = difftopo::load_mesh("m.off");                 // mesh_io.hpp:310
//   auto op   = difftopo::assemble_laplacian(mesh);            // operators.hpp:33
//   auto res  = difftopo::run_initial_pass(mesh, op, 0, cfg);  // diffusion.hpp:861
//   for (auto& ev : res.events) ...                            // TopologyEvent
//   auto reeb = difftopo::build_reeb(res);                     // SPEC reeb.build_reeb
//
// Errors surface as the reference's exception classes (errors.hpp).  Link
// with -ldifftopo_b200 (paper_2105_13168_b200/lib).  Define
// DIFFTOPO_B200_NO_ALIAS to keep the names in namespace difftopo_b200 only.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "difftopo_b200.h"

namespace difftopo_b200 {

using Index = std::uint32_t;
inline constexpr Index kInvalidIndex = 0xFFFFFFFFu;

struct Vec3 {
  double x = 0, y = 0, z = 0;
};

// errors.hpp
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define DTB_ERR(Name, Code)                                  \
  struct Name : Error {                                      \
    explicit Name(const std::string& m) : Error(Code, m) {} \
  };
DTB_ERR(ParseError, DTB_EPARSE)
DTB_ERR(TopologyError, DTB_ETOPOLOGY)
DTB_ERR(DegeneracyError, DTB_EDEGENERACY)
DTB_ERR(InvalidParameter, DTB_EINVALID)
DTB_ERR(DimensionMismatch, DTB_EDIMENSION)
DTB_ERR(EmptySeed, DTB_EEMPTYSEED)
DTB_ERR(ZeroColumn, DTB_EZEROCOLUMN)
DTB_ERR(InvalidSplit, DTB_EINVALIDSPLIT)
DTB_ERR(InvalidMerge, DTB_EINVALIDMERGE)
DTB_ERR(NumericalBlowup, DTB_EBLOWUP)
DTB_ERR(MaxStepsExceeded, DTB_EMAXSTEPS)
DTB_ERR(InconsistentLog, DTB_EINCONSISTENT)
DTB_ERR(DeviceError, DTB_ECUDA)
DTB_ERR(CapacityExceeded, DTB_ECAPACITY)
#undef DTB_ERR

[[noreturn]] inline void throw_code(int rc, const std::string& msg) {
  switch (rc) {
    case DTB_EPARSE: throw ParseError(msg);
    case DTB_ETOPOLOGY: throw TopologyError(msg);
    case DTB_EDEGENERACY: throw DegeneracyError(msg);
    case DTB_EINVALID: throw InvalidParameter(msg);
    case DTB_EDIMENSION: throw DimensionMismatch(msg);
    case DTB_EEMPTYSEED: throw EmptySeed(msg);
    case DTB_EZEROCOLUMN: throw ZeroColumn(msg);
    case DTB_EINVALIDSPLIT: throw InvalidSplit(msg);
    case DTB_EINVALIDMERGE: throw InvalidMerge(msg);
    case DTB_EBLOWUP: throw NumericalBlowup(msg);
    case DTB_EMAXSTEPS: throw MaxStepsExceeded(msg);
    case DTB_EINCONSISTENT: throw InconsistentLog(msg);
    case DTB_ECAPACITY: throw CapacityExceeded(msg);
    default: throw DeviceError(msg);
  }
}
inline void check(int rc) {
  if (rc != DTB_OK) throw_code(rc, dtb_last_error());
}

// mesh.hpp TriangleMesh / MeshTopologySummary
struct MeshTopologySummary {
  Index vertex_count = 0, edge_count = 0, face_count = 0;
  long euler_characteristic = 0, genus = 0;
};

class TriangleMesh {
 public:
  TriangleMesh(const std::vector<Vec3>& vertices, const std::vector<std::array<Index, 3>>& faces) {
    dtb_mesh* m = nullptr;
    check(dtb_mesh_from_arrays(reinterpret_cast<const double*>(vertices.data()), static_cast<uint32_t>(vertices.size()),
                               reinterpret_cast<const uint32_t*>(faces.data()), static_cast<uint32_t>(faces.size()),
                               &m));
    h_.reset(m, dtb_mesh_free);
  }
  static TriangleMesh generate(const std::string& spec) {
    dtb_mesh* m = nullptr;
    check(dtb_mesh_generate(spec.c_str(), &m));
    return TriangleMesh(m);
  }
  static TriangleMesh load(const std::string& path, int format = 0) {
    dtb_mesh* m = nullptr;
    check(dtb_mesh_load(path.c_str(), format, &m));
    return TriangleMesh(m);
  }
  Index vertex_count() const { return summary().vertex_count; }
  Index face_count() const { return summary().face_count; }
  Index edge_count() const { return summary().edge_count; }
  MeshTopologySummary summary() const {
    MeshTopologySummary s;
    uint32_t nv, ne, nf;
    int64_t eu, g;
    check(dtb_mesh_info(h_.get(), &nv, &ne, &nf, &eu, &g));
    s.vertex_count = nv;
    s.edge_count = ne;
    s.face_count = nf;
    s.euler_characteristic = eu;
    s.genus = g;
    return s;
  }
  std::vector<Vec3> vertices() const {
    std::vector<Vec3> v(vertex_count());
    check(dtb_mesh_vertices(h_.get(), reinterpret_cast<double*>(v.data())));
    return v;
  }
  std::vector<std::array<Index, 3>> faces() const {
    std::vector<std::array<Index, 3>> f(face_count());
    check(dtb_mesh_faces(h_.get(), reinterpret_cast<uint32_t*>(f.data())));
    return f;
  }
  void save(const std::string& path) const { check(dtb_mesh_save(h_.get(), path.c_str())); }
  dtb_mesh* handle() const { return h_.get(); }

 private:
  explicit TriangleMesh(dtb_mesh* m) : h_(m, dtb_mesh_free) {}
  std::shared_ptr<dtb_mesh> h_;
};

inline MeshTopologySummary topology_summary(const TriangleMesh& m) { return m.summary(); }
inline TriangleMesh load_mesh(const std::string& path) { return TriangleMesh::load(path); }
inline TriangleMesh generate_torus(int major, int minor, double R, double r) {
  return TriangleMesh::generate("torus:" + std::to_string(major) + ":" + std::to_string(minor) + ":" +
                                std::to_string(R) + ":" + std::to_string(r));
}
inline TriangleMesh generate_genus_g(int g, int resolution = 3) {
  return TriangleMesh::generate("genus:" + std::to_string(g) + ":" + std::to_string(resolution));
}
inline TriangleMesh generate_icosphere(int subdivisions, double radius = 1.0) {
  return TriangleMesh::generate("icosphere:" + std::to_string(subdivisions) + ":" + std::to_string(radius));
}

// operators.hpp LaplacianOperator (device resident)
class LaplacianOperator {
 public:
  explicit LaplacianOperator(dtb_laplacian* h) : h_(h, dtb_laplacian_free) {}
  double gershgorin_bound() const {
    int64_t nnz;
    double g;
    check(dtb_laplacian_info(h_.get(), &nnz, &g));
    return g;
  }
  std::vector<double> apply(const std::vector<double>& x) const {
    std::vector<double> y(x.size());
    check(dtb_laplacian_apply(h_.get(), x.data(), y.data()));
    return y;
  }
  dtb_laplacian* handle() const { return h_.get(); }

 private:
  std::shared_ptr<dtb_laplacian> h_;
};

inline LaplacianOperator assemble_laplacian(const TriangleMesh& m) {
  dtb_laplacian* op = nullptr;
  check(dtb_laplacian_assemble(m.handle(), &op));
  return LaplacianOperator(op);
}

// layer_field.hpp CoefficientScheme, diffusion.hpp DiffusionConfig
struct CoefficientScheme {
  double gradient_energy = 1.0 / 25.0, penalty = 1.0 / 125.0, contact = 1.0 / 30.0, mobility = 0.25;
};
struct DiffusionConfig {
  double dt = 0.0, band_low_threshold = 0.05, saturation = 0.999, collision_threshold = 0.1;
  int check_interval = 1;
  long max_steps = 200000;
  double covered_threshold = 0.05, seed_radius = 0.0;
  bool record_trails = true;
};

inline double stable_time_step(const LaplacianOperator& op, const CoefficientScheme& s = {}) {
  dtb_coefficients c{s.gradient_energy, s.penalty, s.contact, s.mobility};
  double dt = 0;
  check(dtb_stable_time_step(op.handle(), &c, &dt));
  return dt;
}

enum class EventKind { Seed, Split, Merge, Vanish };
inline const char* to_string(EventKind k) {
  switch (k) {
    case EventKind::Seed: return "seed";
    case EventKind::Split: return "split";
    case EventKind::Merge: return "merge";
    default: return "vanish";
  }
}

struct LoopPoint {
  Vec3 position;
  Index face = kInvalidIndex, edge = kInvalidIndex;
  double edge_t = 0.0;
  Index vertex = kInvalidIndex;
};
struct SurfaceLoop {
  std::vector<LoopPoint> points;
  bool closed = true;
  double length() const {
    double t = 0;
    for (size_t i = 0; i + 1 < points.size(); ++i) {
      const Vec3 &a = points[i].position, &b = points[i + 1].position;
      const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
      t += __builtin_sqrt(dx * dx + dy * dy + dz * dz);
    }
    return t;
  }
};
struct HandleEstimate {
  SurfaceLoop loop;
  Index layer = kInvalidIndex;
  std::vector<std::pair<Index, double>> field_snapshot;
  Index event_index = kInvalidIndex;
};
struct TopologyEvent {
  EventKind kind;
  long step = 0;
  std::vector<Index> layers, produced;
  Vec3 position{};
  std::vector<HandleEstimate> estimates;
  std::vector<Index> covered_snapshot;
};
struct LayerTrack {
  Index layer = kInvalidIndex, created_event = kInvalidIndex, consumed_event = kInvalidIndex;
  std::vector<Vec3> trail;
};

struct InitialPassResult {
  std::vector<TopologyEvent> events;
  std::vector<LayerTrack> tracks;
  double dt_used = 0;
  long steps = 0;
  Index seed_vertex = 0;
  int status = DTB_OK;  // the reference throws instead; see run_initial_pass
  std::string message;
  std::shared_ptr<dtb_result> handle;  // final field stays on the device
  long handle_estimate_count() const {
    long n = 0;
    for (const auto& e : events) n += static_cast<long>(e.estimates.size());
    return n;
  }
};

namespace detail {
inline Index id(int64_t x) { return x < 0 ? kInvalidIndex : static_cast<Index>(x); }
inline InitialPassResult read_result(dtb_result* r, Index seed) {
  InitialPassResult out;
  out.handle.reset(r, dtb_result_free);
  out.seed_vertex = seed;
  int32_t st;
  int64_t steps, nev, ntr, nest, nlay;
  check(dtb_result_summary(r, &st, &steps, &out.dt_used, &nev, &ntr, &nest, &nlay));
  out.status = st;
  out.steps = steps;
  out.message = dtb_result_message(r);
  for (int64_t i = 0; i < nev; ++i) {
    TopologyEvent ev;
    int32_t kind;
    uint32_t nl, np, ne, nc;
    double pos[3];
    check(dtb_result_event(r, i, &kind, &ev.step, pos, &nl, &np, &ne, &nc));
    ev.kind = static_cast<EventKind>(kind);
    ev.position = {pos[0], pos[1], pos[2]};
    ev.layers.resize(nl);
    ev.produced.resize(np);
    ev.covered_snapshot.resize(nc);
    check(dtb_result_event_layers(r, i, ev.layers.data(), ev.produced.data()));
    check(dtb_result_event_covered(r, i, ev.covered_snapshot.data()));
    for (uint32_t k = 0; k < ne; ++k) {
      HandleEstimate est;
      uint32_t layer, npts, nsnap;
      double length;
      check(dtb_result_estimate(r, i, k, &layer, &npts, &nsnap, &length));
      est.layer = layer;
      est.event_index = static_cast<Index>(i);
      std::vector<int64_t> e(npts), f(npts);
      std::vector<double> t(npts), xyz(3 * static_cast<size_t>(npts));
      check(dtb_result_estimate_points(r, i, k, e.data(), t.data(), f.data(), xyz.data()));
      for (uint32_t p = 0; p < npts; ++p) {
        LoopPoint lp;
        lp.edge = id(e[p]);
        lp.face = id(f[p]);
        lp.edge_t = t[p];
        lp.position = {xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]};
        est.loop.points.push_back(lp);
      }
      std::vector<uint32_t> sv(nsnap);
      std::vector<double> sx(nsnap);
      check(dtb_result_estimate_snapshot(r, i, k, sv.data(), sx.data()));
      for (uint32_t p = 0; p < nsnap; ++p) est.field_snapshot.emplace_back(sv[p], sx[p]);
      ev.estimates.push_back(std::move(est));
    }
    out.events.push_back(std::move(ev));
  }
  for (int64_t i = 0; i < ntr; ++i) {
    LayerTrack t;
    int64_t layer, cr, co;
    uint32_t n;
    check(dtb_result_track(r, i, &layer, &cr, &co, &n));
    t.layer = id(layer);
    t.created_event = id(cr);
    t.consumed_event = id(co);
    t.trail.resize(n);
    if (n) check(dtb_result_track_trail(r, i, reinterpret_cast<double*>(t.trail.data())));
    out.tracks.push_back(std::move(t));
  }
  return out;
}
}  // namespace detail

namespace detail {
inline dtb_config to_c(const DiffusionConfig& cfg) {
  dtb_config c;
  dtb_config_default(&c);
  c.dt = cfg.dt;
  c.band_low_threshold = cfg.band_low_threshold;
  c.saturation = cfg.saturation;
  c.collision_threshold = cfg.collision_threshold;
  c.check_interval = cfg.check_interval;
  c.record_trails = cfg.record_trails ? 1 : 0;
  c.max_steps = cfg.max_steps;
  c.covered_threshold = cfg.covered_threshold;
  c.seed_radius = cfg.seed_radius;
  return c;
}
}  // namespace detail

// run_initial_pass (diffusion.hpp:861).  Like the reference it throws the
// error that ended the run (e.g. MaxStepsExceeded); run_initial_pass_partial
// returns the partial log instead.
inline InitialPassResult run_initial_pass_partial(const TriangleMesh& mesh, const LaplacianOperator& op,
                                                  Index seed_vertex, const DiffusionConfig& cfg = {},
                                                  const CoefficientScheme& scheme = {}) {
  const dtb_config c = detail::to_c(cfg);
  dtb_coefficients co{scheme.gradient_energy, scheme.penalty, scheme.contact, scheme.mobility};
  dtb_result* r = nullptr;
  check(dtb_run_initial_pass(mesh.handle(), op.handle(), seed_vertex, &c, &co, &r));
  return detail::read_result(r, seed_vertex);
}

inline InitialPassResult run_initial_pass(const TriangleMesh& mesh, const LaplacianOperator& op, Index seed_vertex,
                                          const DiffusionConfig& cfg = {}, const CoefficientScheme& scheme = {}) {
  InitialPassResult r = run_initial_pass_partial(mesh, op, seed_vertex, cfg, scheme);
  if (r.status != DTB_OK) throw_code(r.status, r.message);
  return r;
}

// Library initialisation, no reference counterpart (see difftopo_b200.h).
// Opt-in hardware work queues for concurrent batch passes: call first thing,
// before any CUDA use in the process.
inline void init_work_queues(int queues = 32) { check(dtb_init_work_queues(queues)); }
// Context creation and kernel loading outside a caller's timed region.
inline void warmup() { check(dtb_warmup()); }

// Independent passes over a batch of meshes, several at once on this GPU
// (dtb_run_initial_pass_batch); item i equals
// run_initial_pass_partial(*meshes[i], *ops[i], seeds[i], cfg, scheme).
// Throws the first failing item's error.
inline std::vector<InitialPassResult> run_initial_pass_batch(const std::vector<const TriangleMesh*>& meshes,
                                                             const std::vector<const LaplacianOperator*>& ops,
                                                             const std::vector<Index>& seeds,
                                                             const DiffusionConfig& cfg = {},
                                                             const CoefficientScheme& scheme = {},
                                                             int concurrency = 0) {
  const size_t n = meshes.size();
  if (ops.size() != n || seeds.size() != n) throw std::invalid_argument("batch sizes differ");
  const dtb_config c = detail::to_c(cfg);
  dtb_coefficients co{scheme.gradient_energy, scheme.penalty, scheme.contact, scheme.mobility};
  std::vector<const dtb_mesh*> mh(n);
  std::vector<const dtb_laplacian*> oh(n);
  std::vector<uint32_t> sd(n);
  for (size_t i = 0; i < n; ++i) {
    mh[i] = meshes[i]->handle();
    oh[i] = ops[i]->handle();
    sd[i] = static_cast<uint32_t>(seeds[i]);
  }
  std::vector<dtb_result*> rs(n, nullptr);
  const int code = dtb_run_initial_pass_batch(mh.data(), oh.data(), sd.data(), static_cast<int32_t>(n), &c, &co,
                                              concurrency, rs.data(), nullptr);
  const std::string msg = code != DTB_OK ? dtb_last_error() : "";
  std::vector<InitialPassResult> out;
  for (size_t i = 0; i < n; ++i)
    if (rs[i]) out.push_back(detail::read_result(rs[i], seeds[i]));
  if (code != DTB_OK) throw_code(code, msg);
  return out;
}

// Reeb graph (SPEC reeb.build_reeb): nodes = events, arcs = layer lifetimes.
struct ReebGraph {
  struct Node {
    EventKind kind;
    Vec3 position;
    long step;
  };
  struct Edge {
    Index from, to, layer;
  };
  std::vector<Node> nodes;
  std::vector<Edge> edges;
  long cycle_rank() const { return static_cast<long>(edges.size()) - static_cast<long>(nodes.size()) + 1; }
};

inline ReebGraph build_reeb(const InitialPassResult& r) {
  ReebGraph g;
  for (const auto& e : r.events) g.nodes.push_back({e.kind, e.position, e.step});
  int64_t nn, na, rank;
  check(dtb_result_reeb(r.handle.get(), &nn, &na, &rank));
  std::vector<uint32_t> from(static_cast<size_t>(na)), to(static_cast<size_t>(na)), layer(static_cast<size_t>(na));
  if (na) check(dtb_result_reeb_arcs(r.handle.get(), from.data(), to.data(), layer.data()));
  for (int64_t i = 0; i < na; ++i) g.edges.push_back({from[i], to[i], layer[i]});
  return g;
}

}  // namespace difftopo_b200

#ifndef DIFFTOPO_B200_NO_ALIAS
namespace difftopo = difftopo_b200;
#endif
