// extern "C" boundary (include/difftopo_b200.h).  Translates C++ exceptions
// into error codes and keeps a per-thread message.
#include "../../include/difftopo_b200.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace dtb {
double bench_barrier(int blocks, int n, int mode);
}

using namespace dtb;

// A mesh is built on the host (generators, files, unusual soups) or on the
// device (dtb_mesh_from_arrays on a GPU box); the other side is derived on
// first use.
struct dtb_mesh {
  std::shared_ptr<const Mesh> host_mesh;
  mutable std::shared_ptr<DeviceMesh> dev;
  mutable cudaStream_t stream = nullptr;
  const Mesh& host() const { return host_mesh ? *host_mesh : dev->host(); }
  Index nv() const { return host_mesh ? host_mesh->nv() : dev->nv(); }
  Index nf() const { return host_mesh ? host_mesh->nf() : dev->nf(); }
  Index ne() const { return host_mesh ? host_mesh->ne() : dev->ne(); }
  DeviceMesh& device() const {
    if (!dev) {
      if (!stream) cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
      dev = std::make_shared<DeviceMesh>(host_mesh, stream);
    }
    return *dev;
  }
  ~dtb_mesh() {
    dev.reset();
    if (stream) cudaStreamDestroy(stream);
  }
};
struct dtb_laplacian {
  std::shared_ptr<DeviceLaplacian> op;
  cudaStream_t stream = nullptr;
  ~dtb_laplacian() {
    op.reset();
    if (stream) cudaStreamDestroy(stream);
  }
};
struct dtb_field {
  std::shared_ptr<DeviceField> f;
  cudaStream_t stream = nullptr;
  ~dtb_field() {
    f.reset();
    if (stream) cudaStreamDestroy(stream);
  }
};
struct dtb_result {
  InitialPassResult r;
  std::unique_ptr<ReebGraph> reeb;
  const ReebGraph& graph() {
    if (!reeb) reeb = std::make_unique<ReebGraph>(build_reeb(r));
    return *reeb;
  }
};

namespace {

thread_local std::string g_err;
// Default number of passes a batch runs at once (each on SMs / lanes CTAs).
// Concurrent persistent passes need one hardware work queue each: the context
// has CUDA_DEVICE_MAX_CONNECTIONS of them (8 unless set), and passes whose
// streams share a queue run one after the other. With 32 queues, 16 lanes of
// 9 CTAs run the 64-mesh batch in 0.50 s against 0.68 s for 8 lanes of 18
// (tools/batch_probe.py, DESIGN "Batches").
constexpr int kBatchLanes = 8;
constexpr int kBatchLanesWide = 16;
// Hardware work queues of the CUDA context: CUDA_DEVICE_MAX_CONNECTIONS as
// the caller set it (read when a batch starts, i.e. after the caller had its
// chance to set it before creating the context), 8 when unset.  The library
// never changes the variable on its own; dtb_init_work_queues is the opt-in.
int context_work_queues() {
  const char* e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  const int q = e ? std::atoi(e) : 8;
  return std::max(1, std::min(32, q > 0 ? q : 8));
}

int default_batch_lanes() {
  const int cpus = static_cast<int>(std::thread::hardware_concurrency());
  if (context_work_queues() >= kBatchLanesWide && (cpus == 0 || cpus >= kBatchLanesWide)) return kBatchLanesWide;
  return kBatchLanes;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return DTB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return DTB_ECAPACITY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DTB_ECUDA;
  }
}

Config to_cfg(const dtb_config* c) {
  Config cfg;
  if (!c) return cfg;
  cfg.dt = c->dt;
  cfg.band_low_threshold = c->band_low_threshold;
  cfg.saturation = c->saturation;
  cfg.collision_threshold = c->collision_threshold;
  cfg.check_interval = c->check_interval;
  cfg.record_trails = c->record_trails != 0;
  cfg.max_steps = static_cast<long>(c->max_steps);
  cfg.covered_threshold = c->covered_threshold;
  cfg.seed_radius = c->seed_radius;
  cfg.record_hashes = c->record_hashes != 0;
  cfg.grid_ctas = c->grid_ctas;
  return cfg;
}
Coefficients to_coef(const dtb_coefficients* c) {
  Coefficients co;
  if (!c) return co;
  co.gradient_energy = c->gradient_energy;
  co.penalty = c->penalty;
  co.contact = c->contact;
  co.mobility = c->mobility;
  return co;
}
void need(const void* p, const char* what) {
  if (!p) fail(kInvalidParameter, std::string("null ") + what);
}
int64_t id_or_neg(Index i) { return i == kInvalid ? -1 : static_cast<int64_t>(i); }

const TopologyEvent& event_at(const dtb_result* r, int64_t i) {
  if (i < 0 || static_cast<size_t>(i) >= r->r.events.size()) fail(kInvalidParameter, "event index out of range");
  return r->r.events[static_cast<size_t>(i)];
}
const HandleEstimate& estimate_at(const dtb_result* r, int64_t ev, uint32_t k) {
  const auto& e = event_at(r, ev);
  if (k >= e.estimates.size()) fail(kInvalidParameter, "estimate index out of range");
  return e.estimates[k];
}
void copy_values(const std::vector<std::pair<Index, double>>& vals, uint32_t* v, double* x, uint32_t cap, uint32_t* n) {
  if (n) *n = static_cast<uint32_t>(vals.size());
  if (v && x && cap >= vals.size())
    for (size_t i = 0; i < vals.size(); ++i) {
      v[i] = vals[i].first;
      x[i] = vals[i].second;
    }
}

}  // namespace

extern "C" {

void dtb_config_default(dtb_config* c) {
  if (!c) return;
  Config d;
  c->dt = d.dt;
  c->band_low_threshold = d.band_low_threshold;
  c->saturation = d.saturation;
  c->collision_threshold = d.collision_threshold;
  c->check_interval = d.check_interval;
  c->record_trails = 1;
  c->max_steps = d.max_steps;
  c->covered_threshold = d.covered_threshold;
  c->seed_radius = d.seed_radius;
  c->record_hashes = 0;
  c->grid_ctas = 0;
}

void dtb_coefficients_default(dtb_coefficients* c) {
  if (!c) return;
  Coefficients d;
  c->gradient_energy = d.gradient_energy;
  c->penalty = d.penalty;
  c->contact = d.contact;
  c->mobility = d.mobility;
}

const char* dtb_last_error(void) { return g_err.c_str(); }
const char* dtb_version(void) { return "difftopo_b200 0.1 (sm_100a)"; }

int dtb_device_info(int* count, int* sms, int* major, int* minor) {
  return guard([&] {
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (count) *count = n;
    if (n == 0) fail(kCudaError, "no CUDA device");
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (sms) cuda_check(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    if (major) cuda_check(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev), "attr");
    if (minor) cuda_check(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev), "attr");
  });
}

int dtb_init_work_queues(int32_t queues) {
  return guard([&] {
    if (queues < 1 || queues > 32) fail(kInvalidParameter, "work queues must be in [1, 32]");
    // The variable is read once, when the CUDA context is created; a context
    // can only exist if libcuda is already mapped.
    if (void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD)) {
      dlclose(h);
      fail(kInvalidParameter, "a CUDA context may already exist; set CUDA_DEVICE_MAX_CONNECTIONS before it is created");
    }
    if (std::getenv("CUDA_DEVICE_MAX_CONNECTIONS")) return;  // the caller's own setting wins
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", std::to_string(queues).c_str(), 0);
  });
}

int dtb_warmup(void) {
  return guard([&] {
    // One small end-to-end call through the device paths (mesh build from a
    // soup, assembly, a pass with split/merge events): creates the context
    // and loads every kernel those paths use (CUDA loads kernels lazily, on
    // first launch), so a caller's first real call does not pay for it.
    const Mesh h = make_mesh("torus:32:16:2:0.5");
    std::vector<double> xyz(3 * static_cast<size_t>(h.nv()));
    for (Index v = 0; v < h.nv(); ++v) {
      xyz[3 * v] = h.p(v).x;
      xyz[3 * v + 1] = h.p(v).y;
      xyz[3 * v + 2] = h.p(v).z;
    }
    std::vector<std::uint32_t> f(3 * static_cast<size_t>(h.nf()));
    for (Index i = 0; i < h.nf(); ++i)
      for (int c = 0; c < 3; ++c) f[3 * i + c] = h.face(i)[c];
    struct StreamGuard {  // destroyed on every exit path, including a throw
      cudaStream_t s = nullptr;
      ~StreamGuard() {
        if (s) {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
        }
      }
    } g;
    cuda_check(cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking), "stream");
    cudaStream_t s = g.s;
    std::shared_ptr<DeviceMesh> dm = DeviceMesh::from_soup(xyz.data(), h.nv(), f.data(), h.nf(), s);
    if (!dm) dm = std::make_shared<DeviceMesh>(std::make_shared<Mesh>(h), s);
    DeviceLaplacian op(dm, s);
    Config cfg;
    cfg.max_steps = 400;
    InitialPassResult r = run_initial_pass(dm, op, 0, cfg, Coefficients{});
    (void)r;
  });
}

// ---- mesh
int dtb_mesh_from_arrays(const double* xyz, uint32_t nv, const uint32_t* faces, uint32_t nf, dtb_mesh** out) {
  return guard([&] {
    need(out, "out");
    need(xyz, "xyz");
    need(faces, "faces");
    auto m = std::make_unique<dtb_mesh>();
    // On a GPU box the soup is validated, oriented and indexed on the device;
    // the host builds it when there is no device or the input is unusual
    // (which includes every invalid input: the host raises the reference's
    // exact error).
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 && !std::getenv("DTB_HOST_MESH")) {
      cuda_check(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking), "stream");
      m->dev = DeviceMesh::from_soup(xyz, nv, faces, nf, m->stream);
    } else {
      cudaGetLastError();  // clear the no-device status
    }
    if (!m->dev) {
      std::vector<V3> v(nv);
      for (uint32_t i = 0; i < nv; ++i) v[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
      std::vector<std::array<Index, 3>> f(nf);
      std::memcpy(f.data(), faces, sizeof(uint32_t) * 3 * static_cast<size_t>(nf));
      m->host_mesh = std::make_shared<Mesh>(std::move(v), std::move(f));
    }
    *out = m.release();
  });
}

int dtb_mesh_generate(const char* spec, dtb_mesh** out) {
  return guard([&] {
    need(out, "out");
    need(spec, "spec");
    auto m = std::make_unique<dtb_mesh>();
    m->host_mesh = std::make_shared<Mesh>(make_mesh(spec));
    *out = m.release();
  });
}

int dtb_mesh_load(const char* path, int32_t format, dtb_mesh** out) {
  return guard([&] {
    need(out, "out");
    need(path, "path");
    auto m = std::make_unique<dtb_mesh>();
    m->host_mesh = std::make_shared<Mesh>(load_mesh(path, format));
    *out = m.release();
  });
}

int dtb_mesh_save(const dtb_mesh* m, const char* path) {
  return guard([&] {
    need(m, "mesh");
    need(path, "path");
    std::string p(path);
    auto ext = p.substr(p.find_last_of('.') + 1);
    if (ext == "dtm") write_dtm(m->host(), p);
    else if (ext == "ply") save_ply(m->host(), p, nullptr, true);
    else if (ext == "obj") save_obj(m->host(), p);
    else fail(kParseError, "unsupported mesh extension ." + ext);
  });
}

void dtb_mesh_free(dtb_mesh* m) { delete m; }

int dtb_mesh_info(const dtb_mesh* m, uint32_t* nv, uint32_t* ne, uint32_t* nf, int64_t* euler, int64_t* genus) {
  return guard([&] {
    need(m, "mesh");
    if (nv) *nv = m->nv();
    if (ne) *ne = m->ne();
    if (nf) *nf = m->nf();
    const long chi = static_cast<long>(m->nv()) - static_cast<long>(m->ne()) + static_cast<long>(m->nf());
    if (euler) *euler = chi;
    if (genus) {
      if ((2 - chi) % 2 != 0 || chi > 2)  // Mesh::genus
        fail(kTopologyError,
             "euler characteristic " + std::to_string(chi) + " is not that of a closed orientable surface");
      *genus = (2 - chi) / 2;
    }
  });
}

int dtb_mesh_vertices(const dtb_mesh* m, double* xyz) {
  return guard([&] {
    need(m, "mesh");
    need(xyz, "xyz");
    const Mesh& h = m->host();
    std::memcpy(xyz, h.positions().data(), sizeof(double) * 3 * h.nv());
  });
}
int dtb_mesh_faces(const dtb_mesh* m, uint32_t* f) {
  return guard([&] {
    need(m, "mesh");
    need(f, "faces");
    const Mesh& h = m->host();
    std::memcpy(f, h.faces().data(), sizeof(uint32_t) * 3 * h.nf());
  });
}
int dtb_mesh_edges(const dtb_mesh* m, uint32_t* ev, uint32_t* ef) {
  return guard([&] {
    need(m, "mesh");
    const Mesh& h = m->host();
    for (Index e = 0; e < h.ne(); ++e) {
      if (ev) {
        ev[2 * e] = h.edge_vertices(e)[0];
        ev[2 * e + 1] = h.edge_vertices(e)[1];
      }
      if (ef) {
        ef[2 * e] = h.edge_faces(e)[0];
        ef[2 * e + 1] = h.edge_faces(e)[1];
      }
    }
  });
}
int dtb_mesh_face_edges(const dtb_mesh* m, uint32_t* fe) {
  return guard([&] {
    need(m, "mesh");
    need(fe, "fe");
    const Mesh& h = m->host();
    for (Index f = 0; f < h.nf(); ++f)
      for (int k = 0; k < 3; ++k) fe[3 * f + k] = h.face_edges(f)[k];
  });
}
int dtb_mesh_adjacency(const dtb_mesh* m, uint32_t* v2v_off, uint32_t* v2v, uint32_t* v2f_off, uint32_t* v2f) {
  return guard([&] {
    need(m, "mesh");
    const Mesh& h = m->host();
    auto put = [](uint32_t* dst, const std::vector<uint32_t>& src) {
      if (dst) std::memcpy(dst, src.data(), sizeof(uint32_t) * src.size());
    };
    put(v2v_off, h.v2v_off());
    put(v2v, h.v2v());
    put(v2f_off, h.v2f_off());
    put(v2f, h.v2f());
  });
}

int dtb_seed_region(const dtb_mesh* m, uint32_t seed, double radius, uint32_t* out, uint32_t cap, uint32_t* n) {
  return guard([&] {
    need(m, "mesh");
    if (seed >= m->nv()) fail(kInvalidParameter, "seed vertex out of range");
    std::vector<Index> s;
    bool done = false;
    if (const char* e = std::getenv("DTB_SEED_DEVICE"); e && e[0] == '1') {  // parity tests of the device Dijkstra
      std::vector<unsigned> buf(8192);
      int cnt = 0;
      const DeviceMesh& d = m->device();
      cuda_check(static_cast<cudaError_t>(launch_seed_region(d.view(), seed, radius, buf.data(),
                                                             static_cast<int>(buf.size()), &cnt, m->stream)),
                 "seed region");
      if (cnt >= 0) {
        s.assign(buf.begin(), buf.begin() + cnt);
        std::sort(s.begin(), s.end());
        done = true;
      }
    }
    if (!done) s = seed_region(m->host(), seed, radius);
    if (n) *n = static_cast<uint32_t>(s.size());
    if (out && cap >= s.size()) std::memcpy(out, s.data(), sizeof(uint32_t) * s.size());
  });
}

// ---- operators
int dtb_laplacian_assemble(const dtb_mesh* m, dtb_laplacian** out) {
  return guard([&] {
    need(m, "mesh");
    need(out, "out");
    auto L = std::make_unique<dtb_laplacian>();
    cuda_check(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking), "stream");
    m->device();
    L->op = std::make_shared<DeviceLaplacian>(m->dev, L->stream);
    *out = L.release();
  });
}

int dtb_laplacian_from_csr(const dtb_mesh* m, const int32_t* off, const int32_t* col, const double* val,
                           const double* mass, int64_t nnz, double gershgorin, dtb_laplacian** out) {
  return guard([&] {
    need(m, "mesh");
    need(out, "out");
    need(off, "off");
    need(mass, "mass");
    const size_t nv = m->nv();
    auto L = std::make_unique<dtb_laplacian>();
    cuda_check(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking), "stream");
    m->device();
    std::vector<int> o(off, off + nv + 1), c(col, col + nnz);
    std::vector<double> v(val, val + nnz), ms(mass, mass + nv);
    L->op = std::make_shared<DeviceLaplacian>(m->dev, o, c, v, ms, gershgorin, L->stream);
    *out = L.release();
  });
}

void dtb_laplacian_free(dtb_laplacian* op) { delete op; }

int dtb_laplacian_info(const dtb_laplacian* op, int64_t* nnz, double* g) {
  return guard([&] {
    need(op, "op");
    if (nnz) *nnz = op->op->nnz();
    if (g) *g = op->op->gershgorin();
  });
}

int dtb_laplacian_csr(const dtb_laplacian* op, int32_t* off, int32_t* col, double* val, double* mass) {
  return guard([&] {
    need(op, "op");
    std::vector<int> o, c;
    std::vector<double> v, ms;
    op->op->download(o, c, v, ms, op->stream);
    if (off) std::memcpy(off, o.data(), sizeof(int) * o.size());
    if (col) std::memcpy(col, c.data(), sizeof(int) * c.size());
    if (val) std::memcpy(val, v.data(), sizeof(double) * v.size());
    if (mass) std::memcpy(mass, ms.data(), sizeof(double) * ms.size());
  });
}

int dtb_laplacian_apply(const dtb_laplacian* op, const double* x, double* y) {
  return guard([&] {
    need(op, "op");
    need(x, "x");
    need(y, "y");
    op->op->apply(x, y, op->stream);
  });
}

int dtb_laplacian_sweep_bench(const dtb_laplacian* op, int32_t reps, double* seconds, double* bytes) {
  return guard([&] {
    need(op, "op");
    need(seconds, "seconds");
    need(bytes, "bytes");
    if (reps < 1) fail(kInvalidParameter, "reps must be positive");
    op->op->sweep_bench(reps, op->stream, seconds, bytes);
  });
}

int dtb_stable_time_step(const dtb_laplacian* op, const dtb_coefficients* c, double* dt) {
  return guard([&] {
    need(op, "op");
    need(dt, "dt");
    *dt = stable_time_step(*op->op, to_coef(c));
  });
}

// ---- initial pass
int dtb_run_initial_pass(const dtb_mesh* m, const dtb_laplacian* op, uint32_t seed, const dtb_config* cfg,
                         const dtb_coefficients* c, dtb_result** out) {
  return guard([&] {
    need(m, "mesh");
    need(op, "op");
    need(out, "out");
    auto r = std::make_unique<dtb_result>();
    r->r = run_initial_pass(m->dev ? m->dev : (m->device(), m->dev), *op->op, seed, to_cfg(cfg), to_coef(c));
    *out = r.release();
  });
}

int dtb_run_initial_pass_batch(const dtb_mesh* const* meshes, const dtb_laplacian* const* ops,
                               const uint32_t* seeds, int32_t n, const dtb_config* cfg, const dtb_coefficients* c,
                               int32_t concurrency, dtb_result** out, int32_t* rc) {
  return guard([&] {
    need(meshes, "meshes");
    need(ops, "ops");
    need(out, "out");
    if (n < 0) fail(kInvalidParameter, "negative batch size");
    for (int32_t i = 0; i < n; ++i) {
      out[i] = nullptr;
      if (rc) rc[i] = DTB_OK;
      need(meshes[i], "mesh");
      need(ops[i], "op");
    }
    if (n == 0) return;
    int dev = 0, sms = 0;
    cuda_check(cudaGetDevice(&dev), "device");
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    const int lanes = std::max(1, std::min<int>(concurrency > 0 ? concurrency : default_batch_lanes(), n));
    Config base = to_cfg(cfg);
    // Each pass is a persistent cooperative kernel on its own stream; the
    // concurrent passes split the SMs between them.
    if (base.grid_ctas == 0) base.grid_ctas = std::max(1, sms / lanes);
    const Coefficients co = to_coef(c);
    // Device copies of host-built meshes are made here, one at a time.
    size_t max_nv = 0, max_ne = 0;
    for (int32_t i = 0; i < n; ++i) {
      meshes[i]->device();
      max_nv = std::max<size_t>(max_nv, meshes[i]->nv());
      max_ne = std::max<size_t>(max_ne, meshes[i]->ne());
    }
    // Every result keeps its workspace, so a batch that fits (about 1 KB per
    // vertex) reserves one per item; a larger one only one per lane.
    const size_t want = static_cast<size_t>(n) * max_nv * 1024 <= (size_t{16} << 30) ? static_cast<size_t>(n)
                                                                                       : static_cast<size_t>(lanes);
    DeviceMesh::reserve_fields(want, max_nv, max_ne);
    std::atomic<int32_t> next{0};
    std::vector<int32_t> codes(static_cast<size_t>(n), DTB_OK);
    std::vector<std::string> msgs(static_cast<size_t>(n));
    auto worker = [&] {
      if (cudaSetDevice(dev) != cudaSuccess) return;
      for (int32_t i; (i = next.fetch_add(1)) < n;) {
        const int code = guard([&] {
          auto r = std::make_unique<dtb_result>();
          r->r = run_initial_pass(meshes[i]->dev, *ops[i]->op, seeds ? seeds[i] : 0, base, co);
          out[i] = r.release();
        });
        codes[static_cast<size_t>(i)] = code;
        if (code != DTB_OK) msgs[static_cast<size_t>(i)] = g_err;
      }
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < lanes; ++k) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    for (int32_t i = 0; i < n; ++i) {
      if (rc) rc[i] = codes[static_cast<size_t>(i)];
      if (codes[static_cast<size_t>(i)] != DTB_OK)
        throw Error(codes[static_cast<size_t>(i)],
                    "batch item " + std::to_string(i) + ": " + msgs[static_cast<size_t>(i)]);
    }
  });
}

void dtb_result_free(dtb_result* r) { delete r; }

int dtb_result_summary(const dtb_result* r, int32_t* status, int64_t* steps, double* dt, int64_t* n_events,
                       int64_t* n_tracks, int64_t* n_est, int64_t* layer_count) {
  return guard([&] {
    need(r, "result");
    if (status) *status = r->r.status;
    if (steps) *steps = r->r.steps;
    if (dt) *dt = r->r.dt_used;
    if (n_events) *n_events = static_cast<int64_t>(r->r.events.size());
    if (n_tracks) *n_tracks = static_cast<int64_t>(r->r.tracks.size());
    if (n_est) *n_est = r->r.handle_estimate_count();
    if (layer_count) *layer_count = r->r.field ? r->r.field->layer_count() : 0;
  });
}

const char* dtb_result_message(const dtb_result* r) { return r ? r->r.message.c_str() : ""; }

int dtb_result_event(const dtb_result* r, int64_t i, int32_t* kind, int64_t* step, double* pos3, uint32_t* nl,
                     uint32_t* np, uint32_t* ne, uint32_t* nc) {
  return guard([&] {
    need(r, "result");
    const auto& e = event_at(r, i);
    if (kind) *kind = static_cast<int32_t>(e.kind);
    if (step) *step = e.step;
    if (pos3) {
      pos3[0] = e.position.x;
      pos3[1] = e.position.y;
      pos3[2] = e.position.z;
    }
    if (nl) *nl = static_cast<uint32_t>(e.layers.size());
    if (np) *np = static_cast<uint32_t>(e.produced.size());
    if (ne) *ne = static_cast<uint32_t>(e.estimates.size());
    if (nc) *nc = static_cast<uint32_t>(e.covered_snapshot.size());
  });
}

int dtb_result_event_layers(const dtb_result* r, int64_t i, uint32_t* layers, uint32_t* produced) {
  return guard([&] {
    need(r, "result");
    const auto& e = event_at(r, i);
    if (layers) std::memcpy(layers, e.layers.data(), sizeof(uint32_t) * e.layers.size());
    if (produced) std::memcpy(produced, e.produced.data(), sizeof(uint32_t) * e.produced.size());
  });
}

int dtb_result_event_covered(const dtb_result* r, int64_t i, uint32_t* covered) {
  return guard([&] {
    need(r, "result");
    const auto& e = event_at(r, i);
    if (covered) std::memcpy(covered, e.covered_snapshot.data(), sizeof(uint32_t) * e.covered_snapshot.size());
  });
}

int dtb_result_estimate(const dtb_result* r, int64_t ev, uint32_t k, uint32_t* layer, uint32_t* np, uint32_t* ns,
                        double* length) {
  return guard([&] {
    need(r, "result");
    const auto& est = estimate_at(r, ev, k);
    if (layer) *layer = est.layer;
    if (np) *np = static_cast<uint32_t>(est.loop.points.size());
    if (ns) *ns = static_cast<uint32_t>(est.field_snapshot.size());
    if (length) *length = est.loop.length();
  });
}

int dtb_result_estimate_points(const dtb_result* r, int64_t ev, uint32_t k, int64_t* edge, double* t, int64_t* face,
                               double* xyz) {
  return guard([&] {
    need(r, "result");
    const auto& est = estimate_at(r, ev, k);
    for (size_t i = 0; i < est.loop.points.size(); ++i) {
      const auto& p = est.loop.points[i];
      if (edge) edge[i] = id_or_neg(p.edge);
      if (t) t[i] = p.edge_t;
      if (face) face[i] = id_or_neg(p.face);
      if (xyz) {
        xyz[3 * i] = p.position.x;
        xyz[3 * i + 1] = p.position.y;
        xyz[3 * i + 2] = p.position.z;
      }
    }
  });
}

int dtb_result_estimate_snapshot(const dtb_result* r, int64_t ev, uint32_t k, uint32_t* v, double* x) {
  return guard([&] {
    need(r, "result");
    const auto& est = estimate_at(r, ev, k);
    for (size_t i = 0; i < est.field_snapshot.size(); ++i) {
      if (v) v[i] = est.field_snapshot[i].first;
      if (x) x[i] = est.field_snapshot[i].second;
    }
  });
}

int dtb_result_track(const dtb_result* r, int64_t i, int64_t* layer, int64_t* created, int64_t* consumed,
                     uint32_t* n_trail) {
  return guard([&] {
    need(r, "result");
    if (i < 0 || static_cast<size_t>(i) >= r->r.tracks.size()) fail(kInvalidParameter, "track index out of range");
    const auto& t = r->r.tracks[static_cast<size_t>(i)];
    if (layer) *layer = id_or_neg(t.layer);
    if (created) *created = id_or_neg(t.created_event);
    if (consumed) *consumed = id_or_neg(t.consumed_event);
    if (n_trail) *n_trail = static_cast<uint32_t>(t.trail.size());
  });
}

int dtb_result_track_trail(const dtb_result* r, int64_t i, double* xyz) {
  return guard([&] {
    need(r, "result");
    if (i < 0 || static_cast<size_t>(i) >= r->r.tracks.size()) fail(kInvalidParameter, "track index out of range");
    const auto& t = r->r.tracks[static_cast<size_t>(i)];
    if (xyz) std::memcpy(xyz, t.trail.data(), sizeof(double) * 3 * t.trail.size());
  });
}

int dtb_result_layer(const dtb_result* r, uint32_t layer, int32_t* active, int32_t* cleared, int64_t* parent,
                     int64_t* created_step, uint32_t* n_mp) {
  return guard([&] {
    need(r, "result");
    if (!r->r.field || layer >= static_cast<uint32_t>(r->r.field->layer_count()))
      fail(kInvalidParameter, "layer out of range");
    const auto& m = r->r.field->meta(layer);
    if (active) *active = m.active;
    if (cleared) *cleared = m.cleared;
    if (parent) *parent = id_or_neg(m.parent);
    if (created_step) *created_step = m.created_step;
    if (n_mp) *n_mp = static_cast<uint32_t>(m.merge_parents.size());
  });
}

int dtb_result_layer_values(const dtb_result* r, uint32_t layer, uint32_t* v, double* x, uint32_t cap, uint32_t* n) {
  return guard([&] {
    need(r, "result");
    need(r->r.field.get(), "field");
    copy_values(r->r.field->layer_values(layer), v, x, cap, n);
  });
}

int dtb_result_field_hash(const dtb_result* r, uint64_t* h) {
  return guard([&] {
    need(r, "result");
    need(r->r.field.get(), "field");
    need(h, "hash");
    *h = r->r.field->hash();
  });
}

int dtb_result_hashes(const dtb_result* r, uint64_t* out, int64_t cap, int64_t* n) {
  return guard([&] {
    need(r, "result");
    if (n) *n = static_cast<int64_t>(r->r.hashes.size());
    if (out && cap >= static_cast<int64_t>(r->r.hashes.size()))
      std::memcpy(out, r->r.hashes.data(), sizeof(uint64_t) * r->r.hashes.size());
  });
}

unsigned long long dtb_launch_count(void) { return launch_count(); }

double dtb_bench_barrier(int blocks, int n, int mode) { return bench_barrier(blocks, n, mode); }

int dtb_mesh_device_bytes(const dtb_mesh* m, uint64_t* bytes) {
  return guard([&] {
    need(m, "mesh");
    need(bytes, "bytes");
    const DeviceMesh& d = m->device();
    *bytes = 8 * (d.px.n + d.py.n + d.pz.n + d.fx.n + d.fy.n + d.fz.n) + 4 * (d.faces.n + d.edges.n) +
             4 * (d.c_off.n + d.c_col.n + d.n_off.n + d.n_col.n + d.f_off.n + d.f_col.n);
  });
}

int dtb_mesh_upload_bytes(const dtb_mesh* m, uint64_t* bytes) {
  return guard([&] {
    need(m, "mesh");
    need(bytes, "bytes");
    *bytes = m->device().h2d_bytes;
  });
}

int dtb_result_work(const dtb_result* r, uint64_t* sum_region, uint64_t* sum_interest, double* t_pass_device,
                    double* t_kernel) {
  return guard([&] {
    need(r, "result");
    if (t_kernel) *t_kernel = r->r.t_kernel;
    if (t_pass_device) *t_pass_device = r->r.t_pass_device;
    if (sum_region) *sum_region = r->r.sum_region;
    if (sum_interest) *sum_interest = r->r.sum_interest;
  });
}

int dtb_result_timing(const dtb_result* r, double* td, double* te, int64_t* launches, int64_t* checks,
                      int64_t* ksteps) {
  return guard([&] {
    need(r, "result");
    if (td) *td = r->r.t_device;
    if (te) *te = r->r.t_events;
    if (launches) *launches = r->r.launches;
    if (checks) *checks = r->r.event_checks;
    if (ksteps) *ksteps = r->r.kernel_steps;
  });
}

int dtb_result_reeb(const dtb_result* r, int64_t* nn, int64_t* na, int64_t* rank) {
  return guard([&] {
    need(r, "result");
    const auto& g = const_cast<dtb_result*>(r)->graph();
    if (nn) *nn = static_cast<int64_t>(g.nodes.size());
    if (na) *na = static_cast<int64_t>(g.arcs.size());
    if (rank) *rank = g.cycle_rank();
  });
}

int dtb_result_reeb_arcs(const dtb_result* r, uint32_t* from, uint32_t* to, uint32_t* layer) {
  return guard([&] {
    need(r, "result");
    const auto& g = const_cast<dtb_result*>(r)->graph();
    for (size_t i = 0; i < g.arcs.size(); ++i) {
      if (from) from[i] = g.arcs[i].from;
      if (to) to[i] = g.arcs[i].to;
      if (layer) layer[i] = g.arcs[i].layer;
    }
  });
}

// ---- field
int dtb_field_init(const dtb_mesh* m, const uint32_t* seeds, uint32_t n, dtb_field** out) {
  return guard([&] {
    need(m, "mesh");
    need(out, "out");
    auto F = std::make_unique<dtb_field>();
    cuda_check(cudaStreamCreateWithFlags(&F->stream, cudaStreamNonBlocking), "stream");
    m->device();
    F->f = std::make_shared<DeviceField>(m->dev, F->stream);
    std::vector<Index> s(seeds, seeds + n);
    F->f->init(s);
    *out = F.release();
  });
}

void dtb_field_free(dtb_field* f) { delete f; }

int dtb_field_step(dtb_field* f, const dtb_laplacian* op, const dtb_config* cfg, const dtb_coefficients* c) {
  return guard([&] {
    need(f, "field");
    need(op, "op");
    step(*f->f, *op->op, to_cfg(cfg), to_coef(c));
  });
}

int dtb_field_layer_count(const dtb_field* f, uint32_t* n) {
  return guard([&] {
    need(f, "field");
    if (n) *n = static_cast<uint32_t>(f->f->layer_count());
  });
}

int dtb_field_layer_values(const dtb_field* f, uint32_t layer, uint32_t* v, double* x, uint32_t cap, uint32_t* n) {
  return guard([&] {
    need(f, "field");
    copy_values(f->f->layer_values(layer), v, x, cap, n);
  });
}

int dtb_field_hash(const dtb_field* f, uint64_t* h) {
  return guard([&] {
    need(f, "field");
    need(h, "hash");
    *h = f->f->hash();
  });
}

int dtb_field_normalize(dtb_field* f) {
  return guard([&] {
    need(f, "field");
    f->f->normalize_columns();
  });
}

int dtb_field_covered_set(const dtb_field* f, double thr, uint32_t* out, uint32_t cap, uint32_t* n) {
  return guard([&] {
    need(f, "field");
    auto s = f->f->covered_set(thr);
    if (n) *n = static_cast<uint32_t>(s.size());
    if (out && cap >= s.size()) std::memcpy(out, s.data(), sizeof(uint32_t) * s.size());
  });
}

int dtb_field_extract_front(dtb_field* f, uint32_t layer, const dtb_config* cfg, uint32_t* ncomp, uint32_t* tri_counts,
                            uint32_t* bnd_counts, double* band_length, uint32_t* tris, uint32_t* bnd) {
  return guard([&] {
    need(f, "field");
    auto comps = extract_front(*f->f, layer, to_cfg(cfg));
    if (ncomp) *ncomp = static_cast<uint32_t>(comps.size());
    size_t ot = 0, ob = 0;
    for (size_t i = 0; i < comps.size(); ++i) {
      if (tri_counts) tri_counts[i] = static_cast<uint32_t>(comps[i].triangles.size());
      if (bnd_counts) bnd_counts[i] = static_cast<uint32_t>(comps[i].boundary_vertices.size());
      if (band_length) band_length[i] = comps[i].band_length;
      if (tris) std::memcpy(tris + ot, comps[i].triangles.data(), sizeof(uint32_t) * comps[i].triangles.size());
      if (bnd)
        std::memcpy(bnd + ob, comps[i].boundary_vertices.data(), sizeof(uint32_t) * comps[i].boundary_vertices.size());
      ot += comps[i].triangles.size();
      ob += comps[i].boundary_vertices.size();
    }
  });
}

int dtb_field_detect_collisions(dtb_field* f, const dtb_config* cfg, uint32_t* flat, uint32_t* sizes, uint32_t cap,
                                uint32_t* n_groups, uint32_t* n_flat) {
  return guard([&] {
    need(f, "field");
    auto groups = detect_collisions(*f->f, to_cfg(cfg));
    size_t total = 0;
    for (const auto& g : groups) total += g.size();
    if (n_groups) *n_groups = static_cast<uint32_t>(groups.size());
    if (n_flat) *n_flat = static_cast<uint32_t>(total);
    if (flat && sizes && cap >= total) {
      size_t o = 0;
      for (size_t i = 0; i < groups.size(); ++i) {
        sizes[i] = static_cast<uint32_t>(groups[i].size());
        for (Index l : groups[i]) flat[o++] = l;
      }
    }
  });
}

int dtb_field_split_layer(dtb_field* f, uint32_t layer, const uint32_t* flat, const uint32_t* sizes, uint32_t ncomp,
                          int64_t step_, uint32_t* children) {
  return guard([&] {
    need(f, "field");
    std::vector<std::vector<Index>> comps(ncomp);
    size_t o = 0;
    for (uint32_t i = 0; i < ncomp; ++i) {
      comps[i].assign(flat + o, flat + o + sizes[i]);
      o += sizes[i];
    }
    auto ch = f->f->split_layer(layer, comps, static_cast<long>(step_));
    f->f->pending_moved.clear();
    f->f->sync_active();
    if (children) std::memcpy(children, ch.data(), sizeof(uint32_t) * ch.size());
  });
}

int dtb_field_merge_layers(dtb_field* f, const uint32_t* ids, uint32_t n, int64_t step_, uint32_t* result) {
  return guard([&] {
    need(f, "field");
    std::vector<Index> v(ids, ids + n);
    const Index r = f->f->merge_layers(v, static_cast<long>(step_));
    f->f->pending_moved.clear();
    f->f->sync_active();
    if (result) *result = r;
  });
}

int dtb_extract_isoline(const dtb_mesh* m, const double* values, double level, uint32_t* n_loops, uint32_t* counts,
                        int64_t* edge, double* t, int64_t* face, double* xyz, uint32_t cap) {
  return guard([&] {
    need(m, "mesh");
    need(values, "values");
    std::vector<double> vals(values, values + m->nv());
    auto loops = extract_isoline(m->host(), vals, level);
    if (n_loops) *n_loops = static_cast<uint32_t>(loops.size());
    size_t total = 0;
    for (size_t i = 0; i < loops.size(); ++i) {
      if (counts) counts[i] = static_cast<uint32_t>(loops[i].points.size());
      total += loops[i].points.size();
    }
    if (cap < total) return;
    size_t o = 0;
    for (const auto& L : loops)
      for (const auto& p : L.points) {
        if (edge) edge[o] = id_or_neg(p.edge);
        if (t) t[o] = p.edge_t;
        if (face) face[o] = id_or_neg(p.face);
        if (xyz) {
          xyz[3 * o] = p.position.x;
          xyz[3 * o + 1] = p.position.y;
          xyz[3 * o + 2] = p.position.z;
        }
        ++o;
      }
  });
}

}  // extern "C"
