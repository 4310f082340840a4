// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A command-line driver that compiles the UNMODIFIED reference headers
// (/root/reference/proj/include/difftopo/*.hpp, header-only C++20) and dumps
// their outputs in the formats our parity tests read.  The reference sources
// are NOT copied: `make -C oracle ref` compiles this file with
// -I/root/reference/proj/include and writes the binary to oracle/_ref/.
//
// Commands (mesh <src> is a spec string, see make_mesh() below):
//   mesh      <src> <out.dtm>             validated mesh (post orientation) + topology arrays
//   laplacian <src> <out.bin>             stiffness CSR, lumped masses, Gershgorin bound
//   run       <src> <out.json> [k=v ...]  run_initial_pass (diffusion.hpp:861) + per-step hashes
//   step      <src> <out.json> [k=v ...]  one-shot step() (diffusion.hpp:386) on seed_region init
//   isoline   <src> <values.f64> <level> <out.json>   extract_isoline (isoline.hpp:55)
//   front     <src> <out.json> [k=v ...]  run to `at` steps, then extract_front per layer
//   time      <src> [k=v ...]             wall-time `steps` advance()+check() steps (bench baseline)
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "difftopo/diffusion.hpp"
#include "difftopo/generators.hpp"
#include "difftopo/mesh_io.hpp"

using namespace difftopo;

// The reference Engine (diffusion.hpp:530) keeps its partial result private and
// drops it when run() throws MaxStepsExceeded.  The explicit-instantiation
// access rule lets this driver read those members without modifying the
// reference; it is only used to report the event prefix of runs that do not
// terminate.
template <typename Tag, typename Tag::type M>
struct Rob {
  friend typename Tag::type get(Tag) { return M; }
};
struct EngineResultTag {
  typedef InitialPassResult diffusion_detail::Engine::*type;
  friend type get(EngineResultTag);
};
struct EngineTracksTag {
  typedef std::vector<LayerTrack> diffusion_detail::Engine::*type;
  friend type get(EngineTracksTag);
};
template struct Rob<EngineResultTag, &diffusion_detail::Engine::result_>;
template struct Rob<EngineTracksTag, &diffusion_detail::Engine::tracks_>;

namespace {

std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, c)) out.push_back(tok);
  return out;
}

// Binary mesh exchange format shared with the product and the tests:
//   "DTM1" u32 nv u32 nf f64[3nv] u32[3nf]
TriangleMesh read_dtm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open " + path);
  char magic[4];
  in.read(magic, 4);
  if (std::memcmp(magic, "DTM1", 4) != 0) throw ParseError("bad dtm magic");
  uint32_t nv, nf;
  in.read(reinterpret_cast<char*>(&nv), 4);
  in.read(reinterpret_cast<char*>(&nf), 4);
  std::vector<Vec3> v(nv);
  std::vector<double> buf(3 * static_cast<size_t>(nv));
  in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * 8));
  for (uint32_t i = 0; i < nv; ++i) v[i] = {buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]};
  std::vector<uint32_t> fb(3 * static_cast<size_t>(nf));
  in.read(reinterpret_cast<char*>(fb.data()), static_cast<std::streamsize>(fb.size() * 4));
  if (!in) throw ParseError("truncated dtm");
  std::vector<std::array<Index, 3>> f(nf);
  for (uint32_t i = 0; i < nf; ++i) f[i] = {fb[3 * i], fb[3 * i + 1], fb[3 * i + 2]};
  return TriangleMesh(std::move(v), std::move(f));
}

TriangleMesh make_mesh(const std::string& spec) {
  auto p = split(spec, ':');
  const std::string& k = p[0];
  auto I = [&](size_t i) { return std::atoi(p.at(i).c_str()); };
  auto D = [&](size_t i) { return std::atof(p.at(i).c_str()); };
  if (k == "dtm") return read_dtm(spec.substr(4));
  if (k == "file") return load_mesh(spec.substr(5));
  if (k == "torus") return generate_torus(I(1), I(2), D(3), D(4));
  if (k == "torus_irr") return generate_torus_irregular(I(1), I(2), D(3), D(4), D(5), D(6), I(7));
  if (k == "genus") return generate_genus_g(I(1), I(2));
  if (k == "icosphere") return generate_icosphere(I(1), D(2));
  if (k == "limbstar") return generate_limb_star(I(1), I(2), I(3));
  if (k == "coin") return generate_coin(I(1), I(2), D(3), D(4));
  throw InvalidParameter("unknown mesh spec " + spec);
}

std::map<std::string, std::string> parse_kv(int argc, char** argv, int start) {
  std::map<std::string, std::string> kv;
  for (int i = start; i < argc; ++i) {
    std::string a = argv[i];
    auto eq = a.find('=');
    if (eq == std::string::npos) throw InvalidParameter("expected key=value, got " + a);
    kv[a.substr(0, eq)] = a.substr(eq + 1);
  }
  return kv;
}

double getd(const std::map<std::string, std::string>& kv, const char* k, double d) {
  auto it = kv.find(k);
  return it == kv.end() ? d : std::atof(it->second.c_str());
}
long getl(const std::map<std::string, std::string>& kv, const char* k, long d) {
  auto it = kv.find(k);
  return it == kv.end() ? d : std::atol(it->second.c_str());
}

DiffusionConfig make_cfg(const std::map<std::string, std::string>& kv) {
  DiffusionConfig cfg;
  cfg.dt = getd(kv, "dt", cfg.dt);
  cfg.band_low_threshold = getd(kv, "band", cfg.band_low_threshold);
  cfg.saturation = getd(kv, "sat", cfg.saturation);
  cfg.collision_threshold = getd(kv, "kappa", cfg.collision_threshold);
  cfg.check_interval = static_cast<int>(getl(kv, "check_interval", cfg.check_interval));
  cfg.max_steps = getl(kv, "max_steps", cfg.max_steps);
  cfg.covered_threshold = getd(kv, "covered", cfg.covered_threshold);
  cfg.seed_radius = getd(kv, "seed_radius", cfg.seed_radius);
  cfg.record_trails = getl(kv, "trails", 1) != 0;
  return cfg;
}

// Order-independent 64-bit digest of the whole layer field: the sum over all
// stored (layer, vertex, value-bits) triples of a splitmix64 mix.  The product
// computes the same digest on the device (csrc/field_hash), so per-step field
// equality is checked bit for bit.
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t entry_hash(uint64_t layer, uint64_t v, double val) {
  uint64_t bits;
  std::memcpy(&bits, &val, 8);
  return splitmix64(splitmix64((layer << 40) ^ v) ^ bits);
}
uint64_t field_hash(const LayerField& f) {
  uint64_t h = 0;
  for (Index id = 0; id < f.layer_count(); ++id)
    for (const auto& [v, val] : f.layer(id).values) h += entry_hash(id, v, val);
  return h;
}

struct Json {
  std::string s;
  void raw(const std::string& x) { s += x; }
  void num(double d) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", d);
    s += b;
  }
  void num(long long i) { s += std::to_string(i); }
  void vec(const Vec3& p) {
    s += "[";
    num(p.x);
    s += ",";
    num(p.y);
    s += ",";
    num(p.z);
    s += "]";
  }
  template <class T>
  void ids(const std::vector<T>& v) {
    s += "[";
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) s += ",";
      s += std::to_string(v[i]);
    }
    s += "]";
  }
  void key(const char* k) {
    if (!s.empty() && s.back() != '{' && s.back() != '[') s += ",";
    s += "\"";
    s += k;
    s += "\":";
  }
};

void write_loop(Json& j, const SurfaceLoop& loop) {
  j.raw("[");
  for (size_t i = 0; i < loop.points.size(); ++i) {
    const auto& p = loop.points[i];
    if (i) j.raw(",");
    j.raw("[");
    j.num(static_cast<long long>(p.edge == kInvalidIndex ? -1 : static_cast<long long>(p.edge)));
    j.raw(",");
    j.num(p.edge_t);
    j.raw(",");
    j.num(static_cast<long long>(p.face == kInvalidIndex ? -1 : static_cast<long long>(p.face)));
    j.raw(",");
    j.vec(p.position);
    j.raw("]");
  }
  j.raw("]");
}

void write_layer_table(Json& j, const LayerField& f) {
  j.raw("[");
  for (Index id = 0; id < f.layer_count(); ++id) {
    const auto& L = f.layer(id);
    if (id) j.raw(",");
    j.raw("{");
    j.key("id");
    j.num(static_cast<long long>(id));
    j.key("active");
    j.num(static_cast<long long>(L.active));
    j.key("cleared");
    j.num(static_cast<long long>(L.cleared));
    j.key("parent");
    j.num(static_cast<long long>(L.parent == kInvalidIndex ? -1 : static_cast<long long>(L.parent)));
    j.key("merge_parents");
    j.ids(L.merge_parents);
    j.key("created_step");
    j.num(static_cast<long long>(L.created_step));
    j.key("nnz");
    j.num(static_cast<long long>(L.values.size()));
    j.key("unsat");
    j.num(static_cast<long long>(L.unsaturated.size()));
    j.raw("}");
  }
  j.raw("]");
}

void dump_field_bin(const LayerField& f, const std::string& path) {
  // u32 layer_count, u32 V, then per layer: u32 n, n*(u32 v, f64 val) sorted by v.
  std::ofstream out(path, std::ios::binary);
  uint32_t lc = f.layer_count(), V = f.vertex_count();
  out.write(reinterpret_cast<const char*>(&lc), 4);
  out.write(reinterpret_cast<const char*>(&V), 4);
  for (Index id = 0; id < lc; ++id) {
    std::vector<std::pair<Index, double>> e(f.layer(id).values.begin(), f.layer(id).values.end());
    std::sort(e.begin(), e.end());
    uint32_t n = static_cast<uint32_t>(e.size());
    out.write(reinterpret_cast<const char*>(&n), 4);
    for (auto& [v, val] : e) {
      out.write(reinterpret_cast<const char*>(&v), 4);
      out.write(reinterpret_cast<const char*>(&val), 8);
    }
  }
}

int cmd_mesh(const std::string& src, const std::string& out_path) {
  TriangleMesh m = make_mesh(src);
  std::ofstream out(out_path, std::ios::binary);
  out.write("DTM1", 4);
  uint32_t nv = m.vertex_count(), nf = m.face_count(), ne = m.edge_count();
  out.write(reinterpret_cast<const char*>(&nv), 4);
  out.write(reinterpret_cast<const char*>(&nf), 4);
  for (const auto& p : m.vertices()) out.write(reinterpret_cast<const char*>(&p.x), 24);
  for (const auto& f : m.faces()) out.write(reinterpret_cast<const char*>(f.data()), 12);
  // Trailer with the topology indices (not part of the DTM1 body).
  out.write("TOPO", 4);
  out.write(reinterpret_cast<const char*>(&ne), 4);
  for (Index e = 0; e < ne; ++e) out.write(reinterpret_cast<const char*>(m.edge_vertices(e).data()), 8);
  for (Index e = 0; e < ne; ++e) out.write(reinterpret_cast<const char*>(m.edge_faces(e).data()), 8);
  for (Index f = 0; f < nf; ++f) out.write(reinterpret_cast<const char*>(m.face_edges(f).data()), 12);
  for (Index v = 0; v < nv; ++v) {
    auto vf = m.vertex_faces(v);
    uint32_t n = static_cast<uint32_t>(vf.size());
    out.write(reinterpret_cast<const char*>(&n), 4);
    out.write(reinterpret_cast<const char*>(vf.data()), 4 * n);
  }
  for (Index v = 0; v < nv; ++v) {
    auto vn = m.vertex_neighbors(v);
    uint32_t n = static_cast<uint32_t>(vn.size());
    out.write(reinterpret_cast<const char*>(&n), 4);
    out.write(reinterpret_cast<const char*>(vn.data()), 4 * n);
  }
  auto ts = topology_summary(m);
  std::printf("{\"V\":%u,\"E\":%u,\"F\":%u,\"genus\":%ld}\n", nv, ne, nf, ts.genus);
  return 0;
}

int cmd_laplacian(const std::string& src, const std::string& out_path) {
  TriangleMesh m = make_mesh(src);
  LaplacianOperator op = assemble_laplacian(m);
  std::ofstream out(out_path, std::ios::binary);
  uint32_t n = op.stiffness.rows;
  uint64_t nnz = op.stiffness.nnz();
  out.write(reinterpret_cast<const char*>(&n), 4);
  out.write(reinterpret_cast<const char*>(&nnz), 8);
  out.write(reinterpret_cast<const char*>(op.stiffness.row_offsets.data()), 8 * (n + 1));
  out.write(reinterpret_cast<const char*>(op.stiffness.col_indices.data()), 4 * nnz);
  out.write(reinterpret_cast<const char*>(op.stiffness.values.data()), 8 * nnz);
  out.write(reinterpret_cast<const char*>(op.vertex_mass.data()), 8 * n);
  out.write(reinterpret_cast<const char*>(&op.gershgorin_bound), 8);
  double dt = stable_time_step(op, CoefficientScheme{});
  out.write(reinterpret_cast<const char*>(&dt), 8);
  return 0;
}

int cmd_run(const std::string& src, const std::string& out_path,
            const std::map<std::string, std::string>& kv) {
  TriangleMesh m = make_mesh(src);
  LaplacianOperator op = assemble_laplacian(m);
  DiffusionConfig cfg = make_cfg(kv);
  const bool want_hash = getl(kv, "hash", 1) != 0;
  std::vector<long> dump_steps;
  if (kv.count("dump_steps"))
    for (auto& s : split(kv.at("dump_steps"), ',')) dump_steps.push_back(std::atol(s.c_str()));
  const Index seed = static_cast<Index>(getl(kv, "seed", 0));

  std::vector<uint64_t> hashes;
  std::vector<std::pair<long, std::string>> timeline;  // layer-table changes
  std::vector<Index> prev_active;
  Index prev_count = 0;
  cfg.on_check = [&](long s, const LayerField& f) {
    if (want_hash) hashes.push_back(field_hash(f));
    auto a = f.active_nonbase_layers();
    if (a != prev_active || f.layer_count() != prev_count) {
      Json j;
      write_layer_table(j, f);
      timeline.emplace_back(s, j.s);
      prev_active = a;
      prev_count = f.layer_count();
    }
    for (long d : dump_steps)
      if (d == s) dump_field_bin(f, out_path + ".step" + std::to_string(s) + ".bin");
  };

  Json j;
  j.raw("{");
  j.key("dt");
  j.num(stable_time_step(op, CoefficientScheme{}));
  auto t0 = std::chrono::steady_clock::now();
  InitialPassResult r;
  std::string status = "ok", error_type;
  {
    diffusion_detail::Engine engine(m, op, seed, cfg, CoefficientScheme{});
    try {
      r = engine.run();
    } catch (const Error& e) {
      status = "error";
      error_type = dynamic_cast<const MaxStepsExceeded*>(&e)  ? "MaxStepsExceeded"
                   : dynamic_cast<const NumericalBlowup*>(&e) ? "NumericalBlowup"
                   : dynamic_cast<const ZeroColumn*>(&e)      ? "ZeroColumn"
                                                              : "Error";
      r = std::move(engine.*get(EngineResultTag()));
      r.tracks = engine.*get(EngineTracksTag());
      r.steps = static_cast<long>(hashes.size()) * cfg.check_interval;
    }
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  j.key("status");
  j.raw("\"" + status + "\"");
  if (!error_type.empty()) {
    j.key("error_type");
    j.raw("\"" + error_type + "\"");
  }
  j.key("seconds");
  j.num(secs);
  j.key("steps");
  j.num(static_cast<long long>(r.steps));
  j.key("dt_used");
  j.num(r.dt_used);
  j.key("handle_estimates");
  j.num(static_cast<long long>(r.handle_estimate_count()));
  j.key("events");
  j.raw("[");
  for (size_t i = 0; i < r.events.size(); ++i) {
    const auto& ev = r.events[i];
    if (i) j.raw(",");
    j.raw("{");
    j.key("kind");
    j.raw(std::string("\"") + to_string(ev.kind) + "\"");
    j.key("step");
    j.num(static_cast<long long>(ev.step));
    j.key("layers");
    j.ids(ev.layers);
    j.key("produced");
    j.ids(ev.produced);
    j.key("position");
    j.vec(ev.position);
    j.key("covered");
    j.ids(ev.covered_snapshot);
    j.key("estimates");
    j.raw("[");
    for (size_t e = 0; e < ev.estimates.size(); ++e) {
      const auto& est = ev.estimates[e];
      if (e) j.raw(",");
      j.raw("{");
      j.key("layer");
      j.num(static_cast<long long>(est.layer));
      j.key("event_index");
      j.num(static_cast<long long>(est.event_index));
      j.key("length");
      j.num(est.loop.length());
      j.key("snapshot_n");
      j.num(static_cast<long long>(est.field_snapshot.size()));
      uint64_t sh = 0;
      for (const auto& [v, val] : est.field_snapshot) sh += entry_hash(est.layer, v, val);
      j.key("snapshot_hash");
      j.raw("\"" + std::to_string(sh) + "\"");
      j.key("points");
      write_loop(j, est.loop);
      j.raw("}");
    }
    j.raw("]");
    j.raw("}");
  }
  j.raw("]");
  j.key("tracks");
  j.raw("[");
  for (size_t i = 0; i < r.tracks.size(); ++i) {
    const auto& t = r.tracks[i];
    if (i) j.raw(",");
    j.raw("{");
    j.key("layer");
    j.num(static_cast<long long>(t.layer == kInvalidIndex ? -1 : static_cast<long long>(t.layer)));
    j.key("created");
    j.num(static_cast<long long>(t.created_event == kInvalidIndex ? -1 : static_cast<long long>(t.created_event)));
    j.key("consumed");
    j.num(static_cast<long long>(t.consumed_event == kInvalidIndex ? -1 : static_cast<long long>(t.consumed_event)));
    j.key("trail");
    j.raw("[");
    for (size_t k = 0; k < t.trail.size(); ++k) {
      if (k) j.raw(",");
      j.vec(t.trail[k]);
    }
    j.raw("]");
    j.raw("}");
  }
  j.raw("]");
  j.key("final_hash");
  j.raw("\"" + std::to_string(field_hash(r.field)) + "\"");
  j.key("layer_table");
  write_layer_table(j, r.field);
  j.key("hashes");
  j.raw("[");
  for (size_t i = 0; i < hashes.size(); ++i) {
    if (i) j.raw(",");
    j.raw("\"" + std::to_string(hashes[i]) + "\"");
  }
  j.raw("]");
  j.key("timeline");
  j.raw("[");
  for (size_t i = 0; i < timeline.size(); ++i) {
    if (i) j.raw(",");
    j.raw("{\"step\":" + std::to_string(timeline[i].first) + ",\"layers\":" + timeline[i].second + "}");
  }
  j.raw("]}");
  std::ofstream out(out_path);
  out << j.s << "\n";
  return 0;
}

int cmd_step(const std::string& src, const std::string& out_path,
             const std::map<std::string, std::string>& kv) {
  TriangleMesh m = make_mesh(src);
  LaplacianOperator op = assemble_laplacian(m);
  DiffusionConfig cfg = make_cfg(kv);
  CoefficientScheme scheme;
  double radius = cfg.seed_radius > 0 ? cfg.seed_radius : 1.5 * interface_length_scale(scheme);
  auto seeds = seed_region(m, static_cast<Index>(getl(kv, "seed", 0)), radius);
  LayerField field = init_field(m, seeds, scheme);
  long n = getl(kv, "n", 1);
  for (long i = 0; i < n; ++i) step(field, op, cfg);
  dump_field_bin(field, out_path + ".bin");
  Json j;
  j.raw("{");
  j.key("seeds");
  j.ids(seeds);
  j.key("hash");
  j.raw("\"" + std::to_string(field_hash(field)) + "\"");
  j.raw("}");
  std::ofstream out(out_path);
  out << j.s << "\n";
  return 0;
}

int cmd_isoline(const std::string& src, const std::string& values_path, double level,
                const std::string& out_path) {
  TriangleMesh m = make_mesh(src);
  std::vector<double> vals(m.vertex_count());
  std::ifstream in(values_path, std::ios::binary);
  in.read(reinterpret_cast<char*>(vals.data()), static_cast<std::streamsize>(8 * vals.size()));
  auto loops = extract_isoline(vals, level, m);
  Json j;
  j.raw("{");
  j.key("loops");
  j.raw("[");
  for (size_t i = 0; i < loops.size(); ++i) {
    if (i) j.raw(",");
    write_loop(j, loops[i]);
  }
  j.raw("]}");
  std::ofstream out(out_path);
  out << j.s << "\n";
  return 0;
}

// Runs `at` full steps of the initial pass, then reports extract_front and
// detect_collisions on the resulting field.
int cmd_front(const std::string& src, const std::string& out_path,
              const std::map<std::string, std::string>& kv) {
  TriangleMesh m = make_mesh(src);
  LaplacianOperator op = assemble_laplacian(m);
  DiffusionConfig cfg = make_cfg(kv);
  const long at = getl(kv, "at", 10);
  Json j;
  j.raw("{");
  bool done = false;
  cfg.on_check = [&](long s, const LayerField& f) {
    if (s != at || done) return;
    done = true;
    j.key("layers");
    j.raw("[");
    bool first = true;
    for (Index id : f.active_nonbase_layers()) {
      auto fronts = extract_front(f, id, m, cfg);
      for (auto& c : fronts) {
        if (!first) j.raw(",");
        first = false;
        j.raw("{");
        j.key("layer");
        j.num(static_cast<long long>(id));
        j.key("triangles");
        j.ids(c.triangles);
        j.key("boundary");
        j.ids(c.boundary_vertices);
        j.key("band_length");
        j.num(c.band_length);
        j.raw("}");
      }
    }
    j.raw("]");
    j.key("collisions");
    j.raw("[");
    auto groups = detect_collisions(f, cfg);
    for (size_t g = 0; g < groups.size(); ++g) {
      if (g) j.raw(",");
      j.ids(groups[g]);
    }
    j.raw("]");
    dump_field_bin(f, out_path + ".bin");
  };
  cfg.max_steps = at + 1;
  try {
    run_initial_pass(m, op, static_cast<Index>(getl(kv, "seed", 0)), cfg);
  } catch (const MaxStepsExceeded&) {
  }
  j.raw("}");
  std::ofstream out(out_path);
  out << j.s << "\n";
  return 0;
}

// Times the reference initial pass for a bounded number of steps (the CPU
// baseline of bench.py --impl reference).  Prints one JSON line.
int cmd_time(const std::string& src, const std::map<std::string, std::string>& kv) {
  auto t0 = std::chrono::steady_clock::now();
  TriangleMesh m = make_mesh(src);
  LaplacianOperator op = assemble_laplacian(m);
  double setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  DiffusionConfig cfg = make_cfg(kv);
  long steps_done = 0;
  cfg.on_check = [&](long s, const LayerField&) { steps_done = s; };
  auto t1 = std::chrono::steady_clock::now();
  std::string status = "ok";
  try {
    run_initial_pass(m, op, static_cast<Index>(getl(kv, "seed", 0)), cfg);
  } catch (const MaxStepsExceeded&) {
    status = "max_steps";
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  std::printf("{\"V\":%u,\"steps\":%ld,\"seconds\":%.6f,\"setup_seconds\":%.6f,\"status\":\"%s\"}\n",
              m.vertex_count(), steps_done, secs, setup, status.c_str());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: difftopo_ref <mesh|laplacian|run|step|isoline|front|time> ...\n");
    return 2;
  }
  std::string cmd = argv[1];
  try {
    if (cmd == "mesh") return cmd_mesh(argv[2], argv[3]);
    if (cmd == "laplacian") return cmd_laplacian(argv[2], argv[3]);
    if (cmd == "run") return cmd_run(argv[2], argv[3], parse_kv(argc, argv, 4));
    if (cmd == "step") return cmd_step(argv[2], argv[3], parse_kv(argc, argv, 4));
    if (cmd == "isoline") return cmd_isoline(argv[2], argv[3], std::atof(argv[4]), argv[5]);
    if (cmd == "front") return cmd_front(argv[2], argv[3], parse_kv(argc, argv, 4));
    if (cmd == "time") return cmd_time(argv[2], parse_kv(argc, argv, 3));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
