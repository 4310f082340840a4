// Host side of the initial pass: device resource management and the
// reference's event handling (diffusion.hpp Engine::check and handlers),
// executed only at steps where the device reported a topology event.
#include "engine.hpp"

#include <dlfcn.h>
#include <execinfo.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <unordered_set>

namespace dtb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCudaError, std::string(what) + ": " + cudaGetErrorString(e));
}
static void ck(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

namespace {
std::mutex g_alloc_mu;
std::multimap<size_t, void*> g_free_blocks;  // size class -> block
size_t g_cached_bytes = 0;
constexpr size_t kCacheBytes = size_t(16) << 30;  // cached large blocks (carved small ones are not counted)
constexpr size_t kSubMax = size_t(4) << 20;        // size classes carved from chunks
constexpr size_t kChunk = size_t(256) << 20;
char* g_bump = nullptr;
size_t g_bump_left = 0;

// Returns the cached large blocks to the driver (caller holds g_alloc_mu).
// Blocks carved from chunks stay cached: they cannot be freed one by one.
void release_cached_large_locked() {
  for (auto it = g_free_blocks.begin(); it != g_free_blocks.end();) {
    if (it->first <= kSubMax) {
      ++it;
      continue;
    }
    cudaFree(it->second);
    g_cached_bytes -= it->first;
    it = g_free_blocks.erase(it);
  }
  cudaGetLastError();
}

size_t size_class(size_t bytes) {
  if (bytes <= 4096) return 4096;
  size_t c = 4096;
  while (c < bytes && c < (size_t(64) << 20)) c <<= 1;  // powers of two up to 64 MiB
  if (c >= bytes) return c;
  return (bytes + (size_t(8) << 20) - 1) / (size_t(8) << 20) * (size_t(8) << 20);  // then 8 MiB granules
}
}  // namespace

// Stream-ordered allocations (cub temporaries) come from the default memory
// pool; keep its memory mapped between synchronizations instead of returning
// it to the driver every time (a re-map costs milliseconds for large blocks).
void keep_default_pool() {
  static const bool done = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      std::uint64_t keep = 8ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    return true;
  }();
  (void)done;
}

void* dev_alloc(size_t bytes) {
  keep_default_pool();
  const size_t c = size_class(bytes);
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_free_blocks.find(c);
    if (it != g_free_blocks.end()) {
      void* p = it->second;
      g_free_blocks.erase(it);
      if (c > kSubMax) g_cached_bytes -= c;
      return p;
    }
  }
  void* p = nullptr;
  if (c <= kSubMax) {
    // Small blocks are carved from 256 MiB chunks: a workspace is ~40
    // buffers, and a cudaMalloc per buffer made a cold batch of 64 passes
    // spend most of its time in the driver.  Carved blocks return to the
    // cache, never to the driver.
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    if (g_bump_left < c) {
      // The rest of the current chunk goes back to the cache as the largest
      // power-of-two classes it holds (the bump pointer stays 4 KiB aligned).
      while (g_bump_left >= 4096) {
        size_t b = 4096;
        while (b * 2 <= g_bump_left && b * 2 <= kSubMax) b *= 2;
        g_free_blocks.emplace(b, g_bump);
        g_bump += b;
        g_bump_left -= b;
      }
      void* chunk = nullptr;
      cudaError_t e = cudaMalloc(&chunk, kChunk);
      if (e != cudaSuccess) {
        cudaGetLastError();
        release_cached_large_locked();
        e = cudaMalloc(&chunk, kChunk);
      }
      cuda_check(e, "cudaMalloc");
      g_bump = static_cast<char*>(chunk);
      g_bump_left = kChunk;
    }
    p = g_bump;
    g_bump += c;
    g_bump_left -= c;
    return p;
  }
  cudaError_t e = cudaMalloc(&p, c);
  if (e != cudaSuccess) {
    // Out of memory with blocks parked in the cache: release them and retry.
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    cudaGetLastError();
    release_cached_large_locked();
    e = cudaMalloc(&p, c);
  }
  cuda_check(e, "cudaMalloc");
  return p;
}

void dev_free(void* p, size_t bytes) {
  const size_t c = size_class(bytes);
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  if (c <= kSubMax) {
    g_free_blocks.emplace(c, p);
    return;
  }
  if (g_cached_bytes + c > kCacheBytes) {
    cudaFree(p);
    return;
  }
  g_free_blocks.emplace(c, p);
  g_cached_bytes += c;
}

namespace {

template <class T>
std::vector<T> to_host(const DevBuf<T>& b, size_t n, cudaStream_t s) {
  std::vector<T> out(n);
  if (n) b.download(out.data(), n, s);
  cuda_check(cudaStreamSynchronize(s), "sync");
  return out;
}

struct UnionFind {
  std::vector<Index> parent;
  explicit UnionFind(size_t n) : parent(n) { std::iota(parent.begin(), parent.end(), Index{0}); }
  Index find(Index a) {
    while (parent[a] != a) a = parent[a] = parent[parent[a]];
    return a;
  }
  void unite(Index a, Index b) {
    a = find(a);
    b = find(b);
    if (a != b) parent[std::max(a, b)] = std::min(a, b);
  }
};

double signed_value(double value, double level) {
  double s = value - level;
  if (s == 0.0) s = 1e-12 * (1.0 + std::abs(level));
  return s;
}

double value_in(const std::vector<std::pair<Index, double>>& sorted_vals, Index v) {
  auto it = std::lower_bound(sorted_vals.begin(), sorted_vals.end(), std::make_pair(v, -1e300));
  return (it != sorted_vals.end() && it->first == v) ? it->second : 0.0;
}

template <class MV>
V3 mean_of(const MV& m, const std::vector<Index>& verts) {
  m.need_vertices(verts);
  V3 c{};
  for (Index v : verts) c = c + m.p(v);
  return verts.empty() ? c : c / static_cast<double>(verts.size());
}

}  // namespace

// ---------------------------------------------------------------------------
// DeviceMesh

DeviceMesh::DeviceMesh(std::shared_ptr<const Mesh> mesh, cudaStream_t s) : mesh_(std::move(mesh)) {
  const Mesh& m = *mesh_;
  nv_ = m.nv();
  nf_ = m.nf();
  ne_ = m.ne();
  const Index nv = nv_, nf = nf_, ne = ne_;
  static_assert(sizeof(V3) == 24 && sizeof(std::array<Index, 3>) == 12 && sizeof(std::array<Index, 2>) == 8,
                "packed host arrays are uploaded as-is");
  double maxabs = 1e-300;
  for (const V3& q : m.positions()) maxabs = std::max({maxabs, std::abs(q.x), std::abs(q.y), std::abs(q.z)});
  // Host arrays go up unchanged; SoA / fixed-point positions and the
  // front-connectivity CSR are derived on the device.
  DevBuf<double> xyz(3 * static_cast<size_t>(nv));
  xyz.upload(reinterpret_cast<const double*>(m.positions().data()), xyz.n, s);
  faces.alloc(3 * static_cast<size_t>(nf));
  faces.upload(reinterpret_cast<const unsigned*>(m.faces().data()), faces.n, s);
  edges.alloc(2 * static_cast<size_t>(ne));
  edges.upload(reinterpret_cast<const unsigned*>(&m.edge_vertices(0)[0]), edges.n, s);
  fe.alloc(3 * static_cast<size_t>(nf));
  fe.upload(reinterpret_cast<const unsigned*>(&m.face_edges(0)[0]), fe.n, s);
  ef.alloc(2 * static_cast<size_t>(ne));
  ef.upload(reinterpret_cast<const unsigned*>(&m.edge_faces(0)[0]), ef.n, s);
  n_off.alloc(nv + 1);
  n_off.upload(reinterpret_cast<const int*>(m.v2v_off().data()), n_off.n, s);
  n_col.alloc(std::max<size_t>(1, m.v2v().size()));
  n_col.upload(reinterpret_cast<const int*>(m.v2v().data()), m.v2v().size(), s);
  f_off.alloc(nv + 1);
  f_off.upload(reinterpret_cast<const int*>(m.v2f_off().data()), f_off.n, s);
  f_col.alloc(std::max<size_t>(1, m.v2f().size()));
  f_col.upload(reinterpret_cast<const int*>(m.v2f().data()), m.v2f().size(), s);
  h2d_bytes = 8 * xyz.n + 4 * (faces.n + edges.n + fe.n + ef.n + n_off.n + m.v2v().size() + f_off.n + m.v2f().size());
  derive(xyz.p, maxabs, s);
}

namespace {
// DTB_TIMING=1: stage times of mesh construction on stderr (diagnostics).
struct StageTimer {
  bool on = false;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  explicit StageTimer(cudaStream_t st) : s(st) {
    const char* e = std::getenv("DTB_TIMING");
    on = e && e[0] == '1';
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dtb] %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

std::shared_ptr<DeviceMesh> DeviceMesh::from_soup(const double* xyz, size_t nv, const std::uint32_t* soup, size_t nf,
                                                  cudaStream_t s) {
  if (nv == 0 || nf == 0 || nv >= (1u << 31) || 3 * nf >= (1u << 31)) return nullptr;
  StageTimer tm(s);
  std::shared_ptr<DeviceMesh> d(new DeviceMesh());
  // The faces go first (the build starts with them); the positions follow on
  // a side stream and land while the faces are paired (first read: the
  // geometry pass, which waits on their event).
  // One side stream and its two events per host thread and device (streams
  // belong to the device current when they were created).
  struct SideStream {
    cudaStream_t st = nullptr;
    cudaEvent_t faces_in = nullptr, xyz_in = nullptr;
    void create() {
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&faces_in, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&xyz_in, cudaEventDisableTiming);
    }
  };
  thread_local std::map<int, SideStream> sides;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "device");
  SideStream& side = sides[dev];
  if (!side.st) side.create();
  DevBuf<unsigned> in(3 * nf);
  in.upload(soup, 3 * nf, s);
  d->xyz_.alloc(3 * nv);
  const bool overlap = side.st && side.faces_in && side.xyz_in;
  if (overlap) {
    cuda_check(cudaEventRecord(side.faces_in, s), "event record");
    cuda_check(cudaStreamWaitEvent(side.st, side.faces_in, 0), "stream wait");
    d->xyz_.upload(xyz, 3 * nv, side.st);
    cuda_check(cudaEventRecord(side.xyz_in, side.st), "event record");
  } else {
    d->xyz_.upload(xyz, 3 * nv, s);
  }
  // Every exit (early returns, errors) waits for the side copy before the
  // buffers it writes can be freed; destroyed before `in` and `d`.
  struct CopyDone {
    cudaEvent_t ev;
    ~CopyDone() {
      if (ev) cudaEventSynchronize(ev);
    }
  } copy_done{overlap ? side.xyz_in : nullptr};
  const size_t ne = 3 * nf / 2;
  d->faces.alloc(3 * nf);
  d->edges.alloc(2 * ne);
  d->ef.alloc(2 * ne);
  d->fe.alloc(3 * nf);
  d->f_off.alloc(nv + 1);
  d->f_col.alloc(3 * nf);
  d->n_off.alloc(nv + 1);
  d->n_col.alloc(2 * ne);
  tm.mark("upload");
  MeshBuild b;
  b.nv = static_cast<int>(nv);
  b.nf = static_cast<int>(nf);
  b.xyz = d->xyz_.p;
  b.xyz_ready = overlap ? side.xyz_in : nullptr;
  b.soup = in.p;
  b.faces = d->faces.p;
  b.edges = d->edges.p;
  b.edge_faces = d->ef.p;
  b.face_edges = d->fe.p;
  b.v2f_off = d->f_off.p;
  b.v2f = d->f_col.p;
  b.v2v_off = d->n_off.p;
  b.v2v = d->n_col.p;
  const int rc = build_mesh(b, s);
  tm.mark("build");
  if (rc == 1) return nullptr;
  ck(rc, "device mesh construction");
  d->nv_ = static_cast<Index>(nv);
  d->nf_ = static_cast<Index>(nf);
  d->ne_ = static_cast<Index>(b.ne);
  d->h2d_bytes = 8 * 3 * nv + 4 * 3 * nf;
  d->derive(d->xyz_.p, std::max(1e-300, b.maxabs), s);
  tm.mark("derive");
  return d;
}

void DeviceMesh::derive(const double* d_xyz, double maxabs, cudaStream_t s) {
  const Index nv = nv_, nf = nf_, ne = ne_;
  // Fixed point with |coord| * 2^k <= 2^38: band sums of up to 2^25 vertices
  // stay exact in int64 (order-independent device reductions).
  const int k = 38 - static_cast<int>(std::ceil(std::log2(maxabs)));
  px.alloc(nv);
  py.alloc(nv);
  pz.alloc(nv);
  fx.alloc(nv);
  fy.alloc(nv);
  fz.alloc(nv);
  ck(launch_positions(d_xyz, static_cast<int>(nv), std::ldexp(1.0, k), px.p, py.p, pz.p, fx.p, fy.p, fz.p, s),
     "positions");
  // Front connectivity: for each vertex the higher-numbered mesh neighbours
  // and apexes of the faces across its link edges.  Two band vertices are
  // related iff their stars contain edge-adjacent faces, which makes
  // union-find over band vertices equivalent to the reference's union-find
  // over band triangles; each pair is united once, from its lower vertex.
  FrontBuild fb{};
  fb.nv = static_cast<int>(nv);
  fb.faces = faces.p;
  fb.face_edges = fe.p;
  fb.edge_faces = ef.p;
  fb.edges = edges.p;
  fb.v2v_off = n_off.p;
  fb.v2v = n_col.p;
  fb.v2f_off = f_off.p;
  fb.v2f = f_col.p;
  fb.nrel_room = 2 * static_cast<long long>(ne);
  c_off.alloc(nv + 1);
  int nnzc = 0;
  void* room = nullptr;
  const int rc = launch_front_count(fb, c_off.p, &nnzc, &room, s);
  if (rc == -1) fail(kCapacityExceeded, "vertex valence above 32");
  ck(rc, "front connectivity");
  struct RoomGuard {  // freed once the stream has finished with it (every exit syncs first)
    void* p;
    size_t bytes;
    cudaStream_t s;
    ~RoomGuard() {
      cudaStreamSynchronize(s);
      dev_free(p, bytes);
    }
  } room_guard{room, front_room_bytes(fb), s};
  c_col.alloc(static_cast<size_t>(std::max(1, nnzc)));
  ck(launch_front_fill(fb, c_off.p, c_col.p, room, s), "front connectivity");
  cuda_check(cudaStreamSynchronize(s), "mesh upload");

  view_.nv = static_cast<int>(nv);
  view_.nf = static_cast<int>(nf);
  view_.ne = static_cast<int>(ne);
  view_.px = px.p;
  view_.py = py.p;
  view_.pz = pz.p;
  view_.fx = fx.p;
  view_.fy = fy.p;
  view_.fz = fz.p;
  view_.fx_scale = std::ldexp(1.0, -k);
  view_.faces = faces.p;
  view_.edges = edges.p;
  view_.c_off = c_off.p;
  view_.c_col = c_col.p;
  view_.n_off = n_off.p;
  view_.n_col = n_col.p;
  view_.f_off = f_off.p;
  view_.f_col = f_col.p;
  view_.face_edges = fe.p;
  view_.edge_faces = ef.p;
}

std::shared_ptr<const Mesh> DeviceMesh::host_ptr() const {
  std::lock_guard<std::mutex> lk(host_mu_);
  if (mesh_) return mesh_;
  // Device-built mesh: download its arrays once (own stream, pinned staging
  // is not worth it for a one-off copy).
  if (const char* e = std::getenv("DTB_TIMING"); e && e[0] == '1') {
    std::fprintf(stderr, "[dtb] host mesh download\n");
    void* frames[16];
    const int nf = backtrace(frames, 16);
    for (int k = 0; k < nf; ++k) {
      Dl_info info{};
      if (dladdr(frames[k], &info) && info.dli_fbase)
        std::fprintf(stderr, "[dtb]   at %s+0x%lx\n", info.dli_fname,
                     static_cast<unsigned long>(static_cast<char*>(frames[k]) - static_cast<char*>(info.dli_fbase)));
    }
  }
  cudaStream_t s = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  std::vector<V3> pos(nv_);
  std::vector<std::array<Index, 3>> fcs(nf_), fed(nf_);
  std::vector<std::array<Index, 2>> ev(ne_), efs(ne_);
  std::vector<std::uint32_t> v2f_off(nv_ + 1), v2v_off(nv_ + 1);
  std::vector<Index> v2f(3 * static_cast<size_t>(nf_)), v2v(2 * static_cast<size_t>(ne_));
  auto get = [&](void* dst, const void* src, size_t bytes) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "mesh download");
  };
  get(pos.data(), xyz_.p, sizeof(V3) * nv_);
  get(fcs.data(), faces.p, 12 * static_cast<size_t>(nf_));
  get(fed.data(), fe.p, 12 * static_cast<size_t>(nf_));
  get(ev.data(), edges.p, 8 * static_cast<size_t>(ne_));
  get(efs.data(), ef.p, 8 * static_cast<size_t>(ne_));
  get(v2f_off.data(), f_off.p, 4 * (static_cast<size_t>(nv_) + 1));
  get(v2v_off.data(), n_off.p, 4 * (static_cast<size_t>(nv_) + 1));
  get(v2f.data(), f_col.p, 4 * v2f.size());
  get(v2v.data(), n_col.p, 4 * v2v.size());
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  cuda_check(e, "mesh download");
  mesh_ = std::make_shared<const Mesh>(Mesh::from_index(std::move(pos), std::move(fcs), std::move(ev), std::move(efs),
                                                        std::move(fed), std::move(v2f_off), std::move(v2f),
                                                        std::move(v2v_off), std::move(v2v)));
  return mesh_;
}

V3 DeviceMesh::position(Index v) const {
  {
    std::lock_guard<std::mutex> lk(host_mu_);
    if (mesh_) return mesh_->p(v);
  }
  V3 q;
  const size_t i = v;
  cuda_check(cudaMemcpy(&q.x, px.p + i, sizeof(double), cudaMemcpyDeviceToHost), "position");
  cuda_check(cudaMemcpy(&q.y, py.p + i, sizeof(double), cudaMemcpyDeviceToHost), "position");
  cuda_check(cudaMemcpy(&q.z, pz.p + i, sizeof(double), cudaMemcpyDeviceToHost), "position");
  return q;
}

// ---------------------------------------------------------------------------
// DeviceLaplacian

DeviceLaplacian::DeviceLaplacian(std::shared_ptr<DeviceMesh> dm, cudaStream_t s) : dm_(std::move(dm)) {
  const int nv = static_cast<int>(dm_->nv());
  off.alloc(nv + 1);
  col.alloc(static_cast<size_t>(nv) + 2 * static_cast<size_t>(dm_->ne()));
  val.alloc(col.n);
  mass.alloc(nv);
  DevBuf<double> grow(nv);
  DevBuf<int> dnnz(1);
  LapBuild b{};
  b.nv = nv;
  b.nf = static_cast<int>(dm_->nf());
  b.px = dm_->px.p;
  b.py = dm_->py.p;
  b.pz = dm_->pz.p;
  b.faces = dm_->faces.p;
  b.v2v_off = dm_->n_off.p;
  b.v2v = dm_->n_col.p;
  b.v2f_off = dm_->f_off.p;
  b.v2f = dm_->f_col.p;
  b.s_off = off.p;
  b.s_col = col.p;
  b.s_val = val.p;
  b.mass = mass.p;
  b.gersh_row = grow.p;
  DevBuf<double> gmax(1);
  b.gersh_max = gmax.p;
  b.nnz = dnnz.p;
  b.nroom = 2 * static_cast<long long>(dm_->ne());
  const int rc = launch_assemble(b, s);
  if (rc == -1) fail(kDegeneracyError, "non-finite cotangent weight");
  ck(rc, "laplacian assembly");
  nnz_ = to_host(dnnz, 1, s)[0];
  build_ell(s);
  gersh_ = std::max(0.0, to_host(gmax, 1, s)[0]);
}

DeviceLaplacian::DeviceLaplacian(std::shared_ptr<DeviceMesh> dm, const std::vector<int>& o, const std::vector<int>& c,
                                 const std::vector<double>& v, const std::vector<double>& ms, double gershgorin,
                                 cudaStream_t s)
    : dm_(std::move(dm)), nnz_(static_cast<int>(c.size())), gersh_(gershgorin) {
  const size_t nv = dm_->nv();
  if (o.size() != nv + 1 || ms.size() != nv || c.size() != v.size() || o.back() != static_cast<int>(c.size()))
    fail(kDimensionMismatch, "operator does not match the mesh");
  off.alloc(o.size());
  off.upload(o.data(), o.size(), s);
  col.alloc(std::max<size_t>(1, c.size()));
  col.upload(c.data(), c.size(), s);
  val.alloc(std::max<size_t>(1, v.size()));
  val.upload(v.data(), v.size(), s);
  mass.alloc(nv);
  mass.upload(ms.data(), nv, s);
  build_ell(s);
  cuda_check(cudaStreamSynchronize(s), "operator upload");
}

void DeviceLaplacian::download(std::vector<int>& o, std::vector<int>& c, std::vector<double>& v, std::vector<double>& ms,
                               cudaStream_t s) const {
  const size_t nv = dm_->nv();
  o = to_host(off, nv + 1, s);
  c = to_host(col, nnz_, s);
  v = to_host(val, nnz_, s);
  ms = to_host(mass, nv, s);
}

void DeviceLaplacian::apply(const double* xh, double* yh, cudaStream_t s) const {
  const int nv = static_cast<int>(dm_->nv());
  DevBuf<double> x(nv), y(nv);
  x.upload(xh, nv, s);
  ck(launch_spmv_ell(nv, e_len.p, e_col.p, e_val.p, off.p, col.p, val.p, mass.p, x.p, y.p, s), "spmv");
  y.download(yh, nv, s);
  cuda_check(cudaStreamSynchronize(s), "spmv sync");
}

// A full-mesh sweep of the operator (what a dense formulation of the step
// would read every step), timed on the device.  Every sweep follows a
// 256 MiB read that evicts L2; `reps` (flush, sweep) pairs and `reps`
// flushes alone are timed as two event-bracketed batches and the difference
// is the sweeps' time (no per-launch event overhead in it).  Algorithmic
// bytes per sweep: the padded rows (8 x 12 B + 1 B length), the mass, x once
// and y once per vertex.
void DeviceLaplacian::sweep_bench(int reps, cudaStream_t s, double* seconds, double* bytes) const {
  const int nv = static_cast<int>(dm_->nv());
  DevBuf<double> x(nv), y(nv);
  cuda_check(cudaMemsetAsync(x.p, 0, sizeof(double) * nv, s), "memset");
  DevBuf<char> flush(256u << 20);
  DevBuf<int> sink(1);
  cuda_check(cudaMemsetAsync(flush.p, 0, flush.n, s), "memset");
  struct Events {
    cudaEvent_t a = nullptr, b = nullptr;
    ~Events() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } ev;
  cuda_check(cudaEventCreate(&ev.a), "event");
  cuda_check(cudaEventCreate(&ev.b), "event");
  auto batch = [&](bool sweep) {
    cuda_check(cudaEventRecord(ev.a, s), "event");
    for (int r = 0; r < reps; ++r) {
      ck(launch_read_all(flush.p, flush.n, sink.p, s), "L2 eviction");
      if (sweep) ck(launch_spmv_ell(nv, e_len.p, e_col.p, e_val.p, off.p, col.p, val.p, mass.p, x.p, y.p, s), "spmv");
    }
    cuda_check(cudaEventRecord(ev.b, s), "event");
    cuda_check(cudaEventSynchronize(ev.b), "event");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, ev.a, ev.b), "elapsed");
    return 1e-3 * ms;
  };
  batch(true);  // warm-up
  const double with = batch(true), without = batch(false);
  *seconds = std::max(0.0, with - without) / std::max(1, reps);
  *bytes = static_cast<double>(nv) * (kEll * 12.0 + 1.0 + 8.0 + 8.0 + 8.0);
}

DevMesh DeviceLaplacian::view() const {
  DevMesh v = dm_->view();
  v.s_off = off.p;
  v.s_col = col.p;
  v.s_val = val.p;
  v.mass = mass.p;
  v.e_len = e_len.p;
  v.e_col = e_col.p;
  v.e_val = e_val.p;
  return v;
}

void DeviceLaplacian::build_ell(cudaStream_t s) {
  const size_t nv = dm_->nv();
  e_len.alloc(nv);
  e_col.alloc(nv * kEll);
  e_val.alloc(nv * kEll);
  ck(launch_ell(static_cast<int>(nv), off.p, col.p, val.p, e_len.p, e_col.p, e_val.p, s), "padded rows");
}

double stable_time_step(const DeviceLaplacian& op, const Coefficients& c) {
  const double a = c.gradient_energy;
  const double lambda = op.gershgorin() * 0.5 * a * a;
  if (lambda <= 0) fail(kInvalidParameter, "operator admits no positive time step");
  return 0.9 * 2.0 / lambda;
}

void Config::validate() const {
  if (!(band_low_threshold > 0) || !(band_low_threshold < saturation) || !(saturation <= 1.0))
    fail(kInvalidParameter, "need 0 < band threshold < saturation <= 1");
  if (!(collision_threshold > 0) || collision_threshold > 0.5)
    fail(kInvalidParameter, "collision threshold must lie in (0, 0.5]");
  if (check_interval < 1) fail(kInvalidParameter, "check interval must be >= 1");
  if (max_steps < 1) fail(kInvalidParameter, "max steps must be >= 1");
  if (grid_ctas < 0) fail(kInvalidParameter, "grid CTAs must be >= 0");
}

// Geodesic ball by Dijkstra over mesh edges (diffusion.hpp:134).
std::vector<Index> seed_region(const Mesh& mesh, Index seed, double radius) {
  std::vector<double> d(mesh.nv(), 1e300);
  std::priority_queue<std::pair<double, Index>, std::vector<std::pair<double, Index>>, std::greater<>> q;
  d[seed] = 0;
  q.push({0, seed});
  std::vector<Index> out;
  while (!q.empty()) {
    auto [dv, v] = q.top();
    q.pop();
    if (dv > d[v]) continue;
    if (dv > radius) break;
    out.push_back(v);
    for (Index o = mesh.v2v_off()[v]; o < mesh.v2v_off()[v + 1]; ++o) {
      const Index u = mesh.v2v()[o];
      const double nd = dv + dist(mesh.p(v), mesh.p(u));
      if (nd < d[u]) {
        d[u] = nd;
        q.push({nd, u});
      }
    }
  }
  std::sort(out.begin(), out.end());
  return out;
}

double SurfaceLoop::length() const {
  double total = 0;
  for (size_t i = 0; i + 1 < points.size(); ++i) total += dist(points[i].position, points[i + 1].position);
  return total;
}

V3 SurfaceLoop::centroid() const {
  V3 c{};
  double total = 0;
  for (size_t i = 0; i + 1 < points.size(); ++i) {
    const double len = dist(points[i].position, points[i + 1].position);
    c = c + (points[i].position + points[i + 1].position) * (0.5 * len);
    total += len;
  }
  if (total <= 0) return points.empty() ? V3{} : points.front().position;
  return c / total;
}

// Mesh views for host event handling.  HostView reads a host mesh; LocalMesh
// reads a device-resident mesh through gathers of just the vertices, faces
// and edges an event touches (their records are identical to the host
// mesh's), so a device-built mesh is never downloaded whole (~700 MB at 5M
// vertices).  need_*() batch the gathers; any record asked for without a
// prior need_*() is fetched on its own.
struct Row {
  const Index* b;
  const Index* e;
  const Index* begin() const { return b; }
  const Index* end() const { return e; }
};

class HostView {
 public:
  explicit HostView(const Mesh& m) : m_(m) {}
  void need_vertices(const std::vector<Index>&) const {}
  void need_faces(const std::vector<Index>&) const {}
  void need_edges(const std::vector<Index>&) const {}
  const V3& p(Index v) const { return m_.p(v); }
  Row v2v(Index v) const { return {m_.v2v().data() + m_.v2v_off()[v], m_.v2v().data() + m_.v2v_off()[v + 1]}; }
  Row v2f(Index v) const { return {m_.v2f().data() + m_.v2f_off()[v], m_.v2f().data() + m_.v2f_off()[v + 1]}; }
  const std::array<Index, 3>& face(Index f) const { return m_.face(f); }
  const std::array<Index, 3>& face_edges(Index f) const { return m_.face_edges(f); }
  const std::array<Index, 2>& edge_vertices(Index e) const { return m_.edge_vertices(e); }
  const std::array<Index, 2>& edge_faces(Index e) const { return m_.edge_faces(e); }
  Index opposite_face(Index e, Index f) const { return m_.opposite_face(e, f); }

 private:
  const Mesh& m_;
};

class LocalMesh {
 public:
  LocalMesh(const DeviceMesh& dm, cudaStream_t s) : dm_(dm), s_(s) {
    rows_.px = dm.px.p;
    rows_.py = dm.py.p;
    rows_.pz = dm.pz.p;
    rows_.v2v_off = dm.n_off.p;
    rows_.v2v = dm.n_col.p;
    rows_.v2f_off = dm.f_off.p;
    rows_.v2f = dm.f_col.p;
    rows_.faces = dm.faces.p;
    rows_.face_edges = dm.fe.p;
    rows_.edges = dm.edges.p;
    rows_.edge_faces = dm.ef.p;
  }
  void need_vertices(const std::vector<Index>& vs) const {
    std::vector<unsigned> miss = missing(vs, vert_);
    const int n = static_cast<int>(miss.size());
    if (!n) return;
    DevBuf<unsigned> list(miss.size());
    DevBuf<int> bounds(4 * miss.size()), dst(miss.size());
    DevBuf<double> pos(3 * miss.size());
    list.upload(miss.data(), miss.size(), s_);
    ck(launch_gather_vhead(rows_, list.p, n, bounds.p, pos.p, s_), "gather vertices");
    std::vector<int> hb(4 * miss.size());
    std::vector<double> hp(3 * miss.size());
    bounds.download(hb.data(), hb.size(), s_);
    pos.download(hp.data(), hp.size(), s_);
    cuda_check(cudaStreamSynchronize(s_), "gather vertices");
    std::vector<int> off(miss.size());
    size_t tot = 0;
    for (int i = 0; i < n; ++i) {
      off[i] = static_cast<int>(tot);
      tot += static_cast<size_t>(hb[4 * i + 1] - hb[4 * i]) + static_cast<size_t>(hb[4 * i + 3] - hb[4 * i + 2]);
    }
    std::vector<unsigned> hr(tot);
    if (tot) {
      DevBuf<unsigned> rows(tot);
      dst.upload(off.data(), off.size(), s_);
      ck(launch_gather_vrows(rows_, bounds.p, dst.p, n, rows.p, s_), "gather rows");
      rows.download(hr.data(), tot, s_);
      cuda_check(cudaStreamSynchronize(s_), "gather rows");
    }
    for (int i = 0; i < n; ++i) {
      VertRec r;
      r.p = V3{hp[3 * i], hp[3 * i + 1], hp[3 * i + 2]};
      const size_t a = off[i], nv2v = hb[4 * i + 1] - hb[4 * i], nv2f = hb[4 * i + 3] - hb[4 * i + 2];
      r.v2v.assign(hr.begin() + a, hr.begin() + a + nv2v);
      r.v2f.assign(hr.begin() + a + nv2v, hr.begin() + a + nv2v + nv2f);
      vert_.emplace(miss[i], std::move(r));
    }
  }
  void need_faces(const std::vector<Index>& fs) const {
    std::vector<unsigned> miss = missing(fs, face_);
    if (miss.empty()) return;
    std::vector<unsigned> h = gather(miss, 6, launch_gather_faces);
    for (size_t i = 0; i < miss.size(); ++i)
      face_.emplace(miss[i], FaceRec{{h[6 * i], h[6 * i + 1], h[6 * i + 2]}, {h[6 * i + 3], h[6 * i + 4], h[6 * i + 5]}});
  }
  void need_edges(const std::vector<Index>& es) const {
    std::vector<unsigned> miss = missing(es, edge_);
    if (miss.empty()) return;
    std::vector<unsigned> h = gather(miss, 4, launch_gather_edges);
    for (size_t i = 0; i < miss.size(); ++i)
      edge_.emplace(miss[i], EdgeRec{{h[4 * i], h[4 * i + 1]}, {h[4 * i + 2], h[4 * i + 3]}});
  }
  const V3& p(Index v) const { return vert(v).p; }
  Row v2v(Index v) const {
    const auto& r = vert(v);
    return {r.v2v.data(), r.v2v.data() + r.v2v.size()};
  }
  Row v2f(Index v) const {
    const auto& r = vert(v);
    return {r.v2f.data(), r.v2f.data() + r.v2f.size()};
  }
  const std::array<Index, 3>& face(Index f) const { return face_rec(f).v; }
  const std::array<Index, 3>& face_edges(Index f) const { return face_rec(f).e; }
  const std::array<Index, 2>& edge_vertices(Index e) const { return edge_rec(e).v; }
  const std::array<Index, 2>& edge_faces(Index e) const { return edge_rec(e).f; }
  Index opposite_face(Index e, Index f) const {
    const auto& r = edge_rec(e);
    return r.f[0] == f ? r.f[1] : r.f[0];
  }

 private:
  struct VertRec {
    V3 p;
    std::vector<Index> v2v, v2f;
  };
  struct FaceRec {
    std::array<Index, 3> v, e;
  };
  struct EdgeRec {
    std::array<Index, 2> v, f;
  };
  template <class M>
  static std::vector<unsigned> missing(const std::vector<Index>& ids, const M& have) {
    std::vector<unsigned> out;
    for (Index x : ids)
      if (!have.count(x)) out.push_back(static_cast<unsigned>(x));
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
  }
  template <class L>
  std::vector<unsigned> gather(const std::vector<unsigned>& ids, int width, L launch) const {
    DevBuf<unsigned> list(ids.size()), out(width * ids.size());
    list.upload(ids.data(), ids.size(), s_);
    ck(launch(rows_, list.p, static_cast<int>(ids.size()), out.p, s_), "gather");
    std::vector<unsigned> h(width * ids.size());
    out.download(h.data(), h.size(), s_);
    cuda_check(cudaStreamSynchronize(s_), "gather");
    return h;
  }
  const VertRec& vert(Index v) const {
    auto it = vert_.find(v);
    if (it == vert_.end()) {
      need_vertices({v});
      it = vert_.find(v);
    }
    return it->second;
  }
  const FaceRec& face_rec(Index f) const {
    auto it = face_.find(f);
    if (it == face_.end()) {
      need_faces({f});
      it = face_.find(f);
    }
    return it->second;
  }
  const EdgeRec& edge_rec(Index e) const {
    auto it = edge_.find(e);
    if (it == edge_.end()) {
      need_edges({e});
      it = edge_.find(e);
    }
    return it->second;
  }
  const DeviceMesh& dm_;
  cudaStream_t s_;
  MeshRows rows_{};
  mutable std::unordered_map<Index, VertRec> vert_;
  mutable std::unordered_map<Index, FaceRec> face_;
  mutable std::unordered_map<Index, EdgeRec> edge_;
};

// Chains edge crossings into closed loops (isoline.hpp:55-103): seeds in
// ascending edge order, each walk leaves through the face's other crossed
// edge, the closing point repeats the first.
template <class MV>
static std::vector<SurfaceLoop> chain_crossings(const MV& mesh, const std::vector<int>& e_sorted,
                                                const std::unordered_map<Index, double>& t_of) {
  {
    const std::vector<Index> es(e_sorted.begin(), e_sorted.end());
    mesh.need_edges(es);
    std::vector<Index> ends;
    for (Index e : es)
      for (Index v : mesh.edge_vertices(e)) ends.push_back(v);
    mesh.need_vertices(ends);
  }
  std::unordered_map<Index, std::array<Index, 2>> face_edges;
  for (int ei : e_sorted) {
    const Index e = static_cast<Index>(ei);
    for (Index f : mesh.edge_faces(e)) {
      auto [it, fresh] = face_edges.try_emplace(f, std::array<Index, 2>{e, kInvalid});
      if (!fresh) it->second[1] = e;
    }
  }
  std::vector<SurfaceLoop> loops;
  std::unordered_map<Index, bool> visited;
  for (int ei : e_sorted) {
    const Index seed = static_cast<Index>(ei);
    if (visited[seed]) continue;
    SurfaceLoop loop;
    Index edge = seed, face = mesh.edge_faces(seed)[0];
    while (true) {
      visited[edge] = true;
      LoopPoint p;
      p.edge = edge;
      p.edge_t = t_of.at(edge);
      const auto& ev = mesh.edge_vertices(edge);
      p.position = lerp(mesh.p(ev[0]), mesh.p(ev[1]), p.edge_t);
      p.face = face;
      loop.points.push_back(p);
      const auto& fe = face_edges.at(face);
      const Index next = fe[0] == edge ? fe[1] : fe[0];
      face = mesh.opposite_face(next, face);
      edge = next;
      if (edge == seed) break;
    }
    LoopPoint first = loop.points.front();
    first.face = loop.points.back().face;
    loop.points.push_back(first);
    loops.push_back(std::move(loop));
  }
  return loops;
}

std::vector<SurfaceLoop> extract_isoline(const Mesh& mesh, const std::vector<double>& values, double level) {
  if (values.size() != mesh.nv()) fail(kDimensionMismatch, "isoline values must cover every vertex");
  std::vector<int> es;
  std::unordered_map<Index, double> t_of;
  for (Index e = 0; e < mesh.ne(); ++e) {
    const auto& ev = mesh.edge_vertices(e);
    const double sa = signed_value(values[ev[0]], level), sb = signed_value(values[ev[1]], level);
    if (sa * sb >= 0) continue;
    es.push_back(static_cast<int>(e));
    t_of[e] = sa / (sa - sb);
  }
  return chain_crossings(HostView(mesh), es, t_of);
}

// ---------------------------------------------------------------------------
// DeviceField

DeviceField::DeviceField(std::shared_ptr<DeviceMesh> dm, cudaStream_t s) : dm_(dm.get()), keep_(std::move(dm)), s_(s) {
  setup();
}
DeviceField::DeviceField(DeviceMesh* dm, cudaStream_t s, size_t nv_cap, size_t ne_cap) : dm_(dm), s_(s) {
  setup(nv_cap, ne_cap);
}

DeviceMesh::~DeviceMesh() = default;

namespace {
// Process-wide pool of field workspaces (~600 B per vertex: columns, scratch,
// frontier and band lists, union-find parents ...).  A workspace serves any
// mesh up to its vertex capacity, so repeated passes -- on one mesh or on a
// batch of meshes -- do not re-allocate.
std::mutex g_pool_mu;
std::vector<DeviceField*> g_pool;
constexpr size_t kPoolKeep = 16;
}  // namespace

std::shared_ptr<DeviceField> DeviceMesh::acquire_field(cudaStream_t s) {
  DeviceField* f = nullptr;
  const size_t need = nv(), need_e = ne();
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    size_t best = g_pool.size();
    for (size_t i = 0; i < g_pool.size(); ++i)
      if (g_pool[i]->capacity() >= need && g_pool[i]->edge_capacity() >= need_e &&
          (best == g_pool.size() || g_pool[i]->capacity() < g_pool[best]->capacity()))
        best = i;
    if (best < g_pool.size()) {
      f = g_pool[best];
      g_pool.erase(g_pool.begin() + static_cast<std::ptrdiff_t>(best));
    }
  }
  if (f) f->retarget(this);
  else f = new DeviceField(this, s);
  f->set_stream(s);
  f->keep_ = shared_from_this();
  return std::shared_ptr<DeviceField>(f, [](DeviceField* p) {
    p->keep_.reset();
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(p);
    if (g_pool.size() > kPoolKeep) {
      delete g_pool.front();
      g_pool.erase(g_pool.begin());
    }
  });
}

void DeviceMesh::reserve_fields(size_t count, size_t nv, size_t ne) {
  size_t have = 0;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (DeviceField* f : g_pool) have += f->capacity() >= nv && f->edge_capacity() >= ne;
  }
  // Owned until they are in the pool: a failing allocation (OOM) must not
  // leak the workspaces already made.
  std::vector<std::unique_ptr<DeviceField>> made;
  for (size_t k = have; k < count; ++k)
    made.push_back(std::make_unique<DeviceField>(static_cast<DeviceMesh*>(nullptr), nullptr, nv, ne));
  cuda_check(cudaStreamSynchronize(nullptr), "reserve fields");
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool.reserve(g_pool.size() + made.size());
  // Trim the smallest workspaces first.
  for (auto& f : made) g_pool.push_back(f.release());
  std::stable_sort(g_pool.begin(), g_pool.end(),
                   [](const DeviceField* a, const DeviceField* b) { return a->capacity() < b->capacity(); });
  while (g_pool.size() > std::max(kPoolKeep, count)) {
    delete g_pool.front();
    g_pool.erase(g_pool.begin());
  }
}

namespace {
int engine_blocks(int nv, int requested = 0);
}  // namespace


void DeviceField::set_grid(int blocks) {
  const size_t total = bandpairs[0].n;
  size_t nseg = static_cast<size_t>(std::max(1, blocks));
  size_t seg = total / nseg;
  if (const char* env = std::getenv("DTB_BP_SEG")) {  // tests: short segments exercise the overflow list
    seg = std::min(total, static_cast<size_t>(std::max(1, std::atoi(env))));
    nseg = std::min(nseg, total / seg);
  }
  nseg = std::min(nseg, bpcount[0].n);
  work_.bandpair_cap = static_cast<int>(bp_ovf[0].n);
  if (const char* env = std::getenv("DTB_BP_OVF"))  // tests: a tiny overflow list must raise, not truncate
    work_.bandpair_cap = std::min(work_.bandpair_cap, std::max(0, std::atoi(env)));
  work_.bp_nseg = static_cast<int>(nseg);
  work_.bp_seg = static_cast<int>(seg);
}

void DeviceField::setup(size_t nv_cap, size_t ne_cap) {
  const size_t nv = std::max<size_t>(nv_cap, dm_ ? dm_->nv() : 0);
  const size_t ne = std::max<size_t>(ne_cap, dm_ ? dm_->ne() : 0);
  if (nv * kSlots >= 0xFFFFFFFFull) fail(kCapacityExceeded, "more than 134M vertices (32-bit union-find items)");
  cap_ = nv;
  cap_e_ = ne;
  for (int q = 0; q < 2; ++q) {
    cnt[q].alloc(nv);
    interest[q].alloc(nv);
    binfo[q].alloc(nv);
    lay[q].alloc(nv * kSlots);
    val[q].alloc(nv * kSlots);
    view_.b[q].cnt = cnt[q].p;
    view_.b[q].lay = lay[q].p;
    view_.b[q].val = val[q].p;
    view_.b[q].interest = interest[q].p;
    view_.b[q].binfo = binfo[q].p;
  }
  for (int q = 0; q < 4; ++q) {
    region[q].alloc(nv);
    ilist[q].alloc(nv);
    work_.region[q] = region[q].p;
    work_.ilist[q] = ilist[q].p;
  }
  stamp.alloc(nv);
  {
    // Trail-snap band items (two sets, by check parity): one segment per
    // engine CTA (twice the CTA's share of the vertices) plus an overflow
    // list.  The segment length follows the grid that runs the pass
    // (set_grid): a batch pass on a few CTAs gets long segments.
    const size_t nseg = static_cast<size_t>(engine_blocks(static_cast<int>(nv)));
    const size_t seg = 2 * ((nv + nseg - 1) / nseg) + 64;
    for (int q = 0; q < 2; ++q) {
      bandpairs[q].alloc(nseg * seg);
      bpcount[q].alloc(nseg);
      bp_ovf[q].alloc(2 * nv + 4096);
      bpcount[q].zero(s_);
      work_.bandpairs[q] = bandpairs[q].p;
      work_.bpcount[q] = bpcount[q].p;
      work_.bp_ovf[q] = bp_ovf[q].p;
    }
    set_grid(static_cast<int>(nseg));
  }
  parent.alloc(nv * kSlots);
  added.alloc(4 * (nv / 8 + 4096));  // four step slots
  add_stamp.alloc(nv);
  rem_stamp.alloc(nv);
  active.alloc(kMaxLayers + 1);
  aidx.alloc(kMaxLayers + 1);
  alist.alloc(kMaxActive);
  stat.alloc(4 * static_cast<size_t>(kMaxActive));
  pair_keys.alloc(kPairCap);
  pairs.alloc(4 * static_cast<size_t>(kPairCap));
  lastpos.alloc(4 * static_cast<size_t>(kMaxLayers + 1));
  // Trail ring: 8 records per vertex, between 2^16 and kTrailCap (a launch
  // stops before it can wrap, see advance_until_event).
  size_t tcap = size_t{1} << 16;
  while (tcap < 8 * nv && tcap < static_cast<size_t>(kTrailCap)) tcap <<= 1;
  trail.alloc(tcap);
  ctl.alloc(1);
  // The device seed Dijkstra's distances: all "far" between calls (the
  // kernel resets what it touched), so a pass neither allocates nor clears them.
  seed_dist.alloc(nv);
  cuda_check(cudaMemsetAsync(seed_dist.p, 0x7F, sizeof(unsigned long long) * nv, s_), "memset");
  parent.zero(s_);
  pair_keys.zero(s_);
  stat.zero(s_);
  lastpos.zero(s_);
  ctl.zero(s_);
  active.zero(s_);
  work_.stamp = stamp.p;
  // Event-time scratch (layer pulls, isoline crossings, edits): allocated once
  // so host event handling never calls cudaMalloc/cudaFree.
  const size_t ncap = std::max<size_t>(nv, ne) + 1;
  ai0.alloc(ncap);
  ai1.alloc(ncap);
  ad0.alloc(ncap);
  ad1.alloc(ncap);
  ad2.alloc(ncap);
  acnt.alloc(16);
  work_.parent = parent.p;
  work_.added = added.p;
  work_.added_cap = static_cast<int>(added.n / 4);
  work_.add_stamp = add_stamp.p;
  work_.rem_stamp = rem_stamp.p;
  work_.active = active.p;
  work_.aidx = aidx.p;
  work_.alist = alist.p;
  work_.stat = stat.p;
  work_.pair_keys = pair_keys.p;
  work_.pairs = pairs.p;
  work_.lastpos = lastpos.p;
  work_.trail = trail.p;
  work_.trail_mask = static_cast<int>(trail.n - 1);
  work_.ctl = ctl.p;
}

void DeviceField::init(const std::vector<Index>& seeds) {
  if (seeds.empty()) fail(kEmptySeed, "seed set is empty");
  const Index nv = dm_->nv();
  for (Index v : seeds)
    if (v >= nv) fail(kInvalidParameter, "seed vertex out of range");
  meta_.clear();
  meta_.resize(2);
  meta_[0].active = true;  // base layer
  meta_[1].active = true;  // seed layer
  std::vector<int> sv(seeds.begin(), seeds.end());
  std::sort(sv.begin(), sv.end());
  sv.erase(std::unique(sv.begin(), sv.end()), sv.end());
  ai0.upload(sv.data(), sv.size(), s_);
  // Union-find parents and pair keys carry the epoch of the check that wrote
  // them: a reused workspace continues the epoch count of its earlier passes,
  // so their tags are stale without clearing the arrays (a pooled workspace
  // for a 5M-vertex mesh holds 1.3 GB of parents).
  const long long epoch = read_ctl().epoch;
  ctl.zero(s_);
  stat.zero(s_);
  lastpos.zero(s_);
  // Step stamps of gained / lost band items: -1 never matches a step.
  cuda_check(cudaMemsetAsync(add_stamp.p, 0xFF, sizeof(int) * static_cast<size_t>(nv), s_), "memset");
  cuda_check(cudaMemsetAsync(rem_stamp.p, 0xFF, sizeof(int) * static_cast<size_t>(nv), s_), "memset");
  ck(launch_init_field(view_, work_, static_cast<int>(nv), ai0.p, static_cast<int>(sv.size()), s_), "init field");
  Ctl c{};
  c.base_one = static_cast<int>(nv - sv.size());
  c.epoch = epoch;
  ctl.upload(&c, 1, s_);
  sync_active();
  cuda_check(cudaStreamSynchronize(s_), "init");
}

std::vector<Index> DeviceField::active_nonbase() const {
  std::vector<Index> ids;
  for (Index id = 1; id < meta_.size(); ++id)
    if (meta_[id].active) ids.push_back(id);
  return ids;
}

void DeviceField::sync_active() {
  if (meta_.size() > static_cast<size_t>(kMaxLayers)) fail(kCapacityExceeded, "more than 65535 layers");
  // Ids at or above layer_count() never occur in columns, so only the table
  // prefix [0, layer_count) is uploaded.
  const size_t lc = meta_.size();
  std::vector<unsigned char> act(lc, 0);
  std::vector<int> ai(lc, -1), al;
  for (Index id = 1; id < lc; ++id)
    if (meta_[id].active) {
      act[id] = 1;
      ai[id] = static_cast<int>(al.size());
      al.push_back(static_cast<int>(id));
    }
  if (al.size() > static_cast<size_t>(kMaxActive)) fail(kCapacityExceeded, "too many simultaneously active layers");
  active.upload(act.data(), lc, s_);
  aidx.upload(ai.data(), lc, s_);
  if (!al.empty()) alist.upload(al.data(), al.size(), s_);
  cuda_check(cudaStreamSynchronize(s_), "sync_active");
}

Ctl DeviceField::read_ctl() const {
  Ctl c;
  ctl.download(&c, 1, s_);
  cuda_check(cudaStreamSynchronize(s_), "read ctl");
  return c;
}

std::vector<std::pair<Index, double>> DeviceField::layer_values(Index layer) const {
  const int nv = static_cast<int>(dm_->nv());
  cuda_check(cudaMemsetAsync(acnt.p, 0, sizeof(int), s_), "memset");
  ck(launch_pull_layer(view_, nv, static_cast<int>(layer), ai0.p, ad0.p, acnt.p, s_), "pull layer");
  const int n = to_host(acnt, 1, s_)[0];
  std::vector<int> hv = to_host(ai0, n, s_);
  std::vector<double> hx = to_host(ad0, n, s_);
  std::vector<std::pair<Index, double>> out(n);
  for (int i = 0; i < n; ++i) out[i] = {static_cast<Index>(hv[i]), hx[i]};
  std::sort(out.begin(), out.end());
  return out;
}

std::vector<double> DeviceField::dense_row(Index layer) const {
  const int nv = static_cast<int>(dm_->nv());
  ck(launch_dense_row(view_, nv, static_cast<int>(layer), ad0.p, s_), "dense row");
  return to_host(ad0, nv, s_);
}

std::vector<Index> DeviceField::covered_set(double threshold) const {
  const int nv = static_cast<int>(dm_->nv());
  cuda_check(cudaMemsetAsync(acnt.p, 0, sizeof(int), s_), "memset");
  ck(launch_covered(view_, nv, threshold, ai0.p, acnt.p, s_), "covered");
  const int n = to_host(acnt, 1, s_)[0];
  std::vector<int> hv = to_host(ai0, n, s_);
  std::sort(hv.begin(), hv.end());
  return std::vector<Index>(hv.begin(), hv.end());
}

unsigned long long DeviceField::hash() const {
  unsigned long long* h = reinterpret_cast<unsigned long long*>(acnt.p + 8);
  cuda_check(cudaMemsetAsync(h, 0, sizeof(unsigned long long), s_), "memset");
  ck(launch_field_hash(view_, static_cast<int>(dm_->nv()), h, s_), "hash");
  unsigned long long out = 0;
  cuda_check(cudaMemcpyAsync(&out, h, sizeof out, cudaMemcpyDeviceToHost, s_), "D2H");
  cuda_check(cudaStreamSynchronize(s_), "hash sync");
  return out;
}

int DeviceField::base_one_count() const {
  DevBuf<int> h(1);
  h.zero(s_);
  ck(launch_base_one_count(view_, static_cast<int>(dm_->nv()), h.p, s_), "base one");
  return to_host(h, 1, s_)[0];
}

void DeviceField::normalize_columns() {
  Ctl c = read_ctl();
  c.error = 0;
  ctl.upload(&c, 1, s_);
  ck(launch_normalize_all(view_, work_, static_cast<int>(dm_->nv()), prune_epsilon, s_), "normalize");
  if (read_ctl().error == kDevZeroColumn) fail(kZeroColumn, "total field extinction at a vertex");
}

void DeviceField::mark_region(const DevMesh& op_view, const std::vector<int>& verts, long stamp_value) {
  if (verts.empty()) return;
  ai1.upload(verts.data(), verts.size(), s_);
  ck(launch_mark_region(op_view, work_, ai1.p, static_cast<int>(verts.size()), stamp_value, slot4(stamp_value + 1), s_),
     "mark region");
  cuda_check(cudaStreamSynchronize(s_), "mark region sync");
}

void DeviceField::rebuild_band_list(long t) {
  const int q = slot4(t);
  cuda_check(cudaMemsetAsync(&ctl.p->ilcount[q], 0, sizeof(int), s_), "memset");
  ck(launch_rebuild_list(view_, work_, static_cast<int>(dm_->nv()), q, s_), "band list");
}

std::vector<Index> DeviceField::split_layer(Index layer, const std::vector<std::vector<Index>>& comps, long step_) {
  if (layer == 0) fail(kInvalidSplit, "cannot split the base layer");
  if (layer >= meta_.size() || meta_[layer].cleared) fail(kInvalidSplit, "no such layer");
  if (comps.size() < 2) fail(kInvalidSplit, "split needs at least two components");
  const auto vals = layer_values(layer);
  {
    std::unordered_set<Index> seen;
    for (const auto& c : comps) {
      if (c.empty()) fail(kInvalidSplit, "empty split component");
      for (Index v : c) {
        if (!seen.insert(v).second) fail(kInvalidSplit, "overlapping split components");
        auto it = std::lower_bound(vals.begin(), vals.end(), std::make_pair(v, -1e300));
        if (it == vals.end() || it->first != v) fail(kInvalidSplit, "split component vertex outside layer support");
      }
    }
  }
  std::vector<Index> children;
  std::vector<int> verts, newl;
  for (const auto& c : comps) {
    const Index child = static_cast<Index>(meta_.size());
    LayerMeta lm;
    lm.active = true;
    lm.parent = layer;
    lm.created_step = step_;
    meta_.push_back(lm);
    for (Index v : c) {
      verts.push_back(static_cast<int>(v));
      newl.push_back(static_cast<int>(child));
    }
    children.push_back(child);
  }
  if (meta_.size() > static_cast<size_t>(kMaxLayers)) fail(kCapacityExceeded, "more than 65535 layers");
  meta_[layer].active = false;
  ai0.upload(verts.data(), verts.size(), s_);
  ai1.upload(newl.data(), newl.size(), s_);
  ck(launch_relabel(view_, work_, ai0.p, ai1.p, static_cast<int>(verts.size()), static_cast<int>(layer), s_), "relabel");
  cuda_check(cudaStreamSynchronize(s_), "split");
  pending_moved.insert(pending_moved.end(), verts.begin(), verts.end());
  return children;
}

Index DeviceField::merge_layers(const std::vector<Index>& ids, long step_, std::vector<int>* touched) {
  if (ids.size() < 2) fail(kInvalidMerge, "merge needs at least two layers");
  {
    std::unordered_set<Index> seen;
    for (Index id : ids) {
      if (id == 0) fail(kInvalidMerge, "cannot merge the base layer");
      if (id >= meta_.size() || meta_[id].cleared || !meta_[id].active)
        fail(kInvalidMerge, "merge of an inactive or cleared layer");
      if (!seen.insert(id).second) fail(kInvalidMerge, "duplicate layer in merge");
    }
  }
  const Index result = static_cast<Index>(meta_.size());
  if (result >= static_cast<Index>(kMaxLayers)) fail(kCapacityExceeded, "more than 65535 layers");
  LayerMeta lm;
  lm.active = true;
  lm.parent = ids.front();
  lm.created_step = step_;
  lm.merge_parents = ids;
  meta_.push_back(lm);
  for (Index id : ids) {
    meta_[id].active = false;
    meta_[id].cleared = true;
  }
  // Values are accumulated in the order the ids are given; columns store
  // layers in ascending order, so the device sums in ascending id order.
  std::vector<int> sorted_ids(ids.begin(), ids.end());
  std::vector<int> order(sorted_ids);
  std::sort(order.begin(), order.end());
  if (order != sorted_ids) fail(kInvalidMerge, "merge ids must be ascending (reference groups are sorted)");
  const int nv = static_cast<int>(dm_->nv());
  ai1.upload(sorted_ids.data(), ids.size(), s_);
  cuda_check(cudaMemsetAsync(acnt.p, 0, sizeof(int), s_), "memset");
  ck(launch_merge(view_, work_, nv, ai1.p, static_cast<int>(ids.size()), static_cast<int>(result), ai0.p, acnt.p, s_),
     "merge");
  const int n = to_host(acnt, 1, s_)[0];
  std::vector<int> tv = to_host(ai0, n, s_);
  pending_moved.insert(pending_moved.end(), tv.begin(), tv.end());
  if (touched) *touched = tv;
  return result;
}

void DeviceField::set_inactive(Index layer) { meta_[layer].active = false; }

bool DeviceField::finished(Index layer, int nunsat) const {
  if (nunsat != 0) return false;
  const int one = 1;
  cuda_check(cudaMemcpyAsync(acnt.p + 1, &one, sizeof(int), cudaMemcpyHostToDevice, s_), "H2D");
  DevMesh m = dm_->view();
  ck(launch_finished(m, view_, static_cast<int>(layer), prune_epsilon, acnt.p + 1, s_), "finished");
  int flag = 0;
  cuda_check(cudaMemcpyAsync(&flag, acnt.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s_), "D2H");
  cuda_check(cudaStreamSynchronize(s_), "finished sync");
  return flag != 0;
}

long InitialPassResult::handle_estimate_count() const {
  long n = 0;
  for (const auto& e : events) n += static_cast<long>(e.estimates.size());
  return n;
}

// ---------------------------------------------------------------------------
// extract_front / detect_collisions / step (one-shot API)

namespace {
template <class MV>
std::vector<FrontComponent> extract_front_with(const MV& mesh, const DeviceField& field, Index layer,
                                               const Config& cfg) {
  const auto vals = field.layer_values(layer);
  std::vector<Index> band;
  for (const auto& [v, x] : vals)
    if (x < 1.0 && x > cfg.band_low_threshold && x < cfg.saturation) band.push_back(v);
  if (band.empty()) return {};
  mesh.need_vertices(band);
  std::vector<Index> tris;
  for (Index v : band)
    for (Index f : mesh.v2f(v)) tris.push_back(f);
  std::sort(tris.begin(), tris.end());
  tris.erase(std::unique(tris.begin(), tris.end()), tris.end());
  mesh.need_faces(tris);
  {
    std::vector<Index> es, corners;
    for (Index f : tris) {
      for (Index e : mesh.face_edges(f)) es.push_back(e);
      for (Index v : mesh.face(f)) corners.push_back(v);
    }
    mesh.need_edges(es);
    mesh.need_vertices(corners);
  }
  auto slot = [&](Index f) -> long {
    auto it = std::lower_bound(tris.begin(), tris.end(), f);
    return (it != tris.end() && *it == f) ? static_cast<long>(it - tris.begin()) : -1;
  };
  UnionFind uf(tris.size());
  for (Index i = 0; i < tris.size(); ++i)
    for (Index e : mesh.face_edges(tris[i])) {
      const long j = slot(mesh.opposite_face(e, tris[i]));
      if (j >= 0) uf.unite(i, static_cast<Index>(j));
    }
  std::unordered_map<Index, Index> root_comp;
  std::vector<FrontComponent> comps;
  for (Index i = 0; i < tris.size(); ++i) {
    auto [it, fresh] = root_comp.try_emplace(uf.find(i), static_cast<Index>(comps.size()));
    if (fresh) {
      comps.emplace_back();
      comps.back().layer = layer;
    }
    comps[it->second].triangles.push_back(tris[i]);
  }
  for (auto& c : comps) {
    std::vector<Index> verts;
    for (Index f : c.triangles)
      for (Index v : mesh.face(f))
        if (std::binary_search(band.begin(), band.end(), v)) verts.push_back(v);
    std::sort(verts.begin(), verts.end());
    verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
    c.boundary_vertices = std::move(verts);
    double len = 0;
    for (Index f : c.triangles) {
      V3 pts[3];
      int count = 0;
      const auto& t = mesh.face(f);
      for (int k = 0; k < 3 && count < 3; ++k) {
        const Index a = t[k], b = t[(k + 1) % 3];
        const double sa = signed_value(value_in(vals, a), 0.5), sb = signed_value(value_in(vals, b), 0.5);
        if (sa * sb >= 0) continue;
        pts[count++] = lerp(mesh.p(a), mesh.p(b), sa / (sa - sb));
      }
      if (count == 2) len += dist(pts[0], pts[1]);
    }
    c.band_length = len;
  }
  return comps;
}
}  // namespace

std::vector<FrontComponent> extract_front(const DeviceField& field, Index layer, const Config& cfg) {
  const DeviceMesh& dm = field.mesh();
  if (dm.has_host()) return extract_front_with(HostView(dm.host()), field, layer, cfg);
  return extract_front_with(LocalMesh(dm, field.stream()), field, layer, cfg);
}

namespace {

StepParams make_params(const DeviceField& field, const Config& cfg, const Coefficients& c, double dt) {
  StepParams p{};
  const auto act = field.active_nonbase();
  const double n = static_cast<double>(act.size() + 1);
  const double m = static_cast<double>(act.size());
  p.mu_n = c.mobility / n;
  p.m_mu_n = m * (c.mobility / n);
  p.w = c.penalty;
  p.e = c.contact;
  p.half_a2 = 0.5 * c.gradient_energy * c.gradient_energy;
  p.dt = dt;
  p.prune = field.prune_epsilon;
  p.band_lo = cfg.band_low_threshold;
  p.sat = cfg.saturation;
  p.kappa = cfg.collision_threshold;
  p.coll_base_limit = 1.0 - cfg.collision_threshold;
  p.extinct_limit = 1.0 - cfg.saturation;
  p.check_interval = cfg.check_interval;
  p.n_active = static_cast<int>(act.size());
  p.n_layers = field.layer_count();
  p.record_trails = cfg.record_trails ? 1 : 0;
  p.do_hash = cfg.record_hashes ? 1 : 0;
  p.do_check = 1;
  return p;
}

// Grid of the persistent kernel: at most one CTA per SM (the grid barrier's
// cost grows with the CTA count, and a step's frontier/band work rarely needs
// more than 148 x 256 threads), fewer for small meshes.
int engine_blocks(int nv, int requested) {
  // One 512-thread CTA per SM regardless of mesh size: a step's work is a
  // handful of dependent loads per frontier/band item, so more groups means
  // fewer items per group; the grid barrier costs ~1.2 us at 148 CTAs.
  // Occupancy and SM count are cached per device, filled once under a lock.
  struct Limits {
    int maxco, sms;
  };
  static std::mutex mu;
  static std::map<int, Limits> cache;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "device");
  Limits lim{};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it == cache.end()) {
      ck(dev_max_coresident_blocks(&lim.maxco), "occupancy");
      cuda_check(cudaDeviceGetAttribute(&lim.sms, cudaDevAttrMultiProcessorCount, dev), "sms");
      if (lim.maxco <= 0 || lim.sms <= 0) fail(kCudaError, "the engine kernel cannot be resident on this device");
      it = cache.emplace(dev, lim).first;
    }
    lim = it->second;
  }
  (void)nv;
  if (requested > 0) return std::min(requested, lim.maxco);
  if (const char* env = std::getenv("DTB_BLOCKS")) {
    const int b = std::atoi(env);
    if (b > 0) return std::min(b, lim.maxco);
  }
  return std::min(lim.sms, lim.maxco);
}

std::vector<std::vector<Index>> groups_from_pairs(const std::vector<unsigned>& pairs) {
  std::vector<Index> layers;
  for (unsigned p : pairs) {
    layers.push_back(p >> 16);
    layers.push_back(p & 0xFFFF);
  }
  std::sort(layers.begin(), layers.end());
  layers.erase(std::unique(layers.begin(), layers.end()), layers.end());
  auto slot = [&](Index l) { return static_cast<Index>(std::lower_bound(layers.begin(), layers.end(), l) - layers.begin()); };
  UnionFind uf(layers.size());
  for (unsigned p : pairs) uf.unite(slot(p >> 16), slot(p & 0xFFFF));
  std::map<Index, std::vector<Index>> g;
  for (Index i = 0; i < layers.size(); ++i) g[uf.find(i)].push_back(layers[i]);
  std::vector<std::vector<Index>> out;
  for (auto& [r, mem] : g)
    if (mem.size() >= 2) out.push_back(mem);
  std::sort(out.begin(), out.end());
  return out;
}

std::vector<unsigned> read_pairs(const DeviceField& field, long s) {
  const Ctl c = field.read_ctl();
  const int q = slot4(s);
  if (c.pair_overflow[q]) fail(kCapacityExceeded, "collision pair table overflow");
  std::vector<unsigned> out(static_cast<size_t>(c.npairs[q]));
  if (!out.empty()) {
    cuda_check(cudaMemcpyAsync(out.data(), field.pairs.p + static_cast<size_t>(q) * kPairCap, sizeof(unsigned) * out.size(),
                               cudaMemcpyDeviceToHost, field.stream()),
               "pairs");
    cuda_check(cudaStreamSynchronize(field.stream()), "pairs sync");
  }
  return out;
}

// Check-only kernel (stats, CCL, collisions of the current state) into the
// statistics buffer of step s's parity.
void run_check_kernel(DeviceField& field, const Config& cfg, const Coefficients& co, double dt, long s) {
  StepParams p = make_params(field, cfg, co, dt);
  p.step_begin = s;
  const int blocks = engine_blocks(static_cast<int>(field.mesh().nv()), cfg.grid_ctas);
  field.set_grid(blocks);
  field.rebuild_band_list(s);
  ck(launch_check(field.mesh().view(), field.view(), field.work(), p, blocks, field.stream()), "check kernel");
  cuda_check(cudaStreamSynchronize(field.stream()), "check sync");
  if (field.read_ctl().bandpair_overflow) fail(kCapacityExceeded, "band item list overflow (trail snap)");
}

std::vector<LayerStat> read_stats(const DeviceField& field, long s) {
  const size_t n = field.active_nonbase().size();
  std::vector<LayerStat> out(n);
  if (n) {
    cuda_check(cudaMemcpyAsync(out.data(), field.stat.p + static_cast<size_t>(slot4(s)) * kMaxActive, sizeof(LayerStat) * n,
                               cudaMemcpyDeviceToHost, field.stream()),
               "stats");
    cuda_check(cudaStreamSynchronize(field.stream()), "stats sync");
  }
  return out;
}

}  // namespace

std::vector<std::vector<Index>> detect_collisions(DeviceField& field, const Config& cfg) {
  cfg.validate();
  field.set_band(cfg.band_low_threshold, cfg.saturation);
  field.sync_active();
  if (field.active_nonbase().size() < 2) return {};
  run_check_kernel(field, cfg, Coefficients{}, 0.0, 0);
  return groups_from_pairs(read_pairs(field, 0));
}

void step(DeviceField& field, const DeviceLaplacian& op, const Config& cfg, const Coefficients& c) {
  cfg.validate();
  field.set_band(cfg.band_low_threshold, cfg.saturation);
  const double dt = cfg.dt > 0 ? cfg.dt : stable_time_step(op, c);
  field.sync_active();
  cudaStream_t s = field.stream();
  // prime_full_frontier: every support vertex of the base and active layers.
  cuda_check(cudaMemsetAsync(field.stamp.p, 0xFF, sizeof(int) * field.stamp.n, s), "stamp reset");
  DevWork w = field.work();
  w.stamp = field.stamp.p;
  Ctl ctl = field.read_ctl();
  for (int q = 0; q < 4; ++q) ctl.rcount[q] = 0;
  ctl.error = 0;
  ctl.stop_bits = 0;
  field.ctl.upload(&ctl, 1, s);
  const DevMesh m = op.view();
  ck(launch_mark_all_support(m, field.view(), w, 0, slot4(1), s), "mark support");
  field.rebuild_band_list(1);
  StepParams p = make_params(field, cfg, c, dt);
  p.step_begin = 1;
  p.step_end = 2;
  p.do_check = 0;
  ck(launch_run(m, field.view(), w, p, engine_blocks(m.nv, cfg.grid_ctas), s), "step kernel");
  cuda_check(cudaStreamSynchronize(s), "step sync");
  const Ctl after = field.read_ctl();
  if (after.error == kDevBlowup) fail(kNumericalBlowup, "non-finite rate; reduce dt");
  if (after.error == kDevZeroColumn) fail(kZeroColumn, "total field extinction at vertex " + std::to_string(after.error_vertex));
  if (after.error) fail(kCapacityExceeded, "column capacity exceeded at vertex " + std::to_string(after.error_vertex));
}

namespace {

// The initial pass (diffusion.hpp:530 Engine) with the step loop on the device.
class PassEngine {
 public:
  PassEngine(std::shared_ptr<DeviceMesh> dm, const DeviceLaplacian& op, Index seed, const Config& cfg,
             const Coefficients& co)
      : dm_(std::move(dm)), op_(op), cfg_(cfg), co_(co) {
    cfg_.validate();
    if (seed >= dm_->nv()) fail(kInvalidParameter, "seed vertex out of range");
    cuda_check(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreate(&ev0_), "event");
    cuda_check(cudaEventCreate(&ev1_), "event");
    cuda_check(cudaEventCreate(&ev0k_), "event");
    cuda_check(cudaEventCreate(&ev1k_), "event");
    cuda_check(cudaEventRecord(ev0_, s_), "event record");
    StageTimer tm(s_);
    field_ = dm_->acquire_field(s_);
    tm.mark("pass workspace");
    field_->set_band(cfg_.band_low_threshold, cfg_.saturation);
    res_.field = field_;
    res_.seed_vertex = seed;
    const double radius =
        cfg_.seed_radius > 0 ? cfg_.seed_radius : 1.5 * (co_.gradient_energy / std::sqrt(co_.penalty));
    // The Dijkstra runs on the device (a device-built mesh has no host copy
    // to download); capacity overflow falls back to the host.
    std::vector<Index> seeds;
    bool seeded = false;
    {
      std::vector<unsigned> buf(8192);
      int n = 0;
      ck(launch_seed_region(dm_->view(), seed, radius, buf.data(), static_cast<int>(buf.size()), &n, s_,
                            field_->seed_dist.p),
         "seed region");
      if (n >= 0) {
        seeds.assign(buf.begin(), buf.begin() + n);
        std::sort(seeds.begin(), seeds.end());
        seeded = true;
      }
    }
    if (!seeded) seeds = seed_region(mesh(), seed, radius);
    tm.mark("pass seed");
    field_->init(seeds);
    tm.mark("pass init");
    dt_ = cfg_.dt > 0 ? cfg_.dt : stable_time_step(op_, co_);
    res_.dt_used = dt_;
    if (cfg_.record_hashes) {
      field_->hashes.alloc(static_cast<size_t>(cfg_.max_steps) + 1);
      field_->hashes.zero(s_);
    }
    TopologyEvent ev;
    ev.kind = EventKind::Seed;
    ev.step = 0;
    ev.layers = {1};
    ev.position = dm_->position(seed);
    res_.events.push_back(ev);
    track(1).created_event = 0;
    std::vector<int> sv(seeds.begin(), seeds.end());
    field_->mark_region(op_.view(), sv, 0);
    tm.mark("pass frontier");
    blocks_ = engine_blocks(static_cast<int>(dm_->nv()), cfg_.grid_ctas);
    field_->set_grid(blocks_);
    if (const char* env = std::getenv("DTB_PHASE_PROF"); env && env[0] == '1') {
      prof_.alloc(4 * static_cast<size_t>(std::min<long>(cfg_.max_steps, 100000)) + 8 + 2 * 64 * 3 * 160 + 64);
      prof_.zero(s_);
    }
  }
  ~PassEngine() {
    // The result keeps the field: later queries on it must not use the
    // stream destroyed here.
    if (field_) {
      cudaStreamSynchronize(s_);
      field_->set_stream(nullptr);
    }
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    if (ev0k_) cudaEventDestroy(ev0k_);
    if (ev1k_) cudaEventDestroy(ev1k_);
    if (s_) cudaStreamDestroy(s_);
  }

  InitialPassResult run() {
    long step = 0;
    try {
      while (true) {
        if (step >= cfg_.max_steps) {
          res_.status = kMaxStepsExceeded;
          res_.message = "initial pass exceeded " + std::to_string(cfg_.max_steps) + " steps";
          break;
        }
        const long s = advance_until_event(step);
        if (s < 0) {  // budget exhausted without an event
          step = cfg_.max_steps;
          continue;
        }
        step = s;
        if (host_check(s)) break;
      }
    } catch (const Error& e) {
      res_.status = e.code;
      res_.message = e.what();
    }
    res_.steps = step;
    StageTimer tm(s_);
    if (prof_.p) {
      report_phases();
      instr_report();
    }
    {
      const Ctl c = field_->read_ctl();
      res_.sum_region = c.sum_region;
      res_.sum_interest = c.sum_interest;
    }
    finish_tracks();
    tm.mark("pass tracks");
    cuda_check(cudaEventRecord(ev1_, s_), "event record");
    cuda_check(cudaEventSynchronize(ev1_), "event sync");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, ev0_, ev1_), "elapsed");
    res_.t_pass_device = ms * 1e-3;
    if (cfg_.record_hashes) {
      const size_t n = static_cast<size_t>(std::min(step, cfg_.max_steps));
      std::vector<unsigned long long> h = to_host(field_->hashes, n + 1, s_);
      for (size_t i = 1; i <= n; ++i)
        if (i % static_cast<size_t>(cfg_.check_interval) == 0) res_.hashes.push_back(h[i]);
    }
    return std::move(res_);
  }

 private:
  LayerTrack& track(Index layer) {
    if (layer >= tracks_.size()) tracks_.resize(layer + 1);
    tracks_[layer].layer = layer;
    return tracks_[layer];
  }

  StepParams params() const {
    StepParams p = make_params(*field_, cfg_, co_, dt_);
    p.stop_every_check = cfg_.on_check ? 1 : 0;
    if (const char* env = std::getenv("DTB_D_FULL"); env && env[0] == '1') p.d_full = 1;
    if (const char* env = std::getenv("DTB_CERT_VERIFY"); env && env[0] == '1') p.cert_verify = 1;
    if (const char* env = std::getenv("DTB_NO_WIDE"); env && env[0] == '1') p.no_wide = 1;
    return p;
  }

  DevWork work() const {
    DevWork w = field_->work();
    if (prof_.p) {
      w.prof = prof_.p;
      w.prof_cap = static_cast<int>(prof_.n);
    }
    if (cfg_.record_hashes) {
      w.hashes = field_->hashes.p;
      w.hash_base = 0;
      w.hash_cap = static_cast<int>(field_->hashes.n);
    }
    return w;
  }

  // Runs device steps from `done`+1 until an event step (returned) or the
  // step budget (returns -1 after executing through max_steps).
  long advance_until_event(long done) {
    const auto t0 = std::chrono::steady_clock::now();
    StepParams p = params();
    const long per_launch = std::max<long>(1, (static_cast<long>(field_->trail.n) / std::max(1, p.n_active)) - 2);
    long begin = done + 1;
    while (true) {
      const long end = std::min<long>(cfg_.max_steps + 1, begin + std::min<long>(per_launch, 1L << 20));
      if (begin >= end) {
        res_.t_device += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return -1;
      }
      p.step_begin = begin;
      p.step_end = end;
      // The first check's band list, and an empty list for the frontier the
      // prologue queues (a discarded speculative update may have left one).
      field_->rebuild_band_list(begin);
      cuda_check(cudaMemsetAsync(&field_->ctl.p->rcount[slot4(begin + 1)], 0, sizeof(int), s_), "memset");
      cuda_check(cudaEventRecord(ev0k_, s_), "event record");
      ck(launch_run(op_.view(), field_->view(), work(), p, blocks_, s_), "engine launch");
      cuda_check(cudaEventRecord(ev1k_, s_), "event record");
      cuda_check(cudaStreamSynchronize(s_), "engine sync");
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, ev0k_, ev1k_), "elapsed");
      res_.t_kernel += ms * 1e-3;
      ++res_.launches;
      Ctl c = field_->read_ctl();
      drain_trails(c);
      res_.kernel_steps += c.stop_step - begin + 1;
      if (c.error) {
        res_.t_device += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (c.error == kDevBlowup) fail(kNumericalBlowup, "non-finite rate; reduce dt");
        if (c.error == kDevZeroColumn)
          fail(kZeroColumn, "total field extinction at vertex " + std::to_string(c.error_vertex));
        if (c.bandpair_overflow) fail(kCapacityExceeded, "band item list overflow (trail snap)");
        if (c.error == kDevCertificate) fail(kInconsistentLog, "split certificate held but the union-find split (DTB_CERT_VERIFY)");
        fail(kCapacityExceeded, "column capacity exceeded at vertex " + std::to_string(c.error_vertex));
      }
      if (c.stop_bits) {
        res_.t_device += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return static_cast<long>(c.stop_step);
      }
      begin = end;
    }
  }

  void drain_trails(Ctl& c) {
    if (c.ntrail == 0) return;
    if (c.ntrail > static_cast<long>(field_->trail.n)) fail(kCapacityExceeded, "trail ring overflow");
    std::vector<TrailRec> recs = to_host(field_->trail, static_cast<size_t>(c.ntrail), s_);
    std::sort(recs.begin(), recs.end(), [](const TrailRec& a, const TrailRec& b) {
      return a.step != b.step ? a.step < b.step : a.layer < b.layer;
    });
    for (const auto& r : recs) {
      if (cfg_.record_trails) track(static_cast<Index>(r.layer)).trail.push_back(V3{r.vx, r.vy, r.vz});
    }
    const int zero = 0;
    cuda_check(cudaMemcpyAsync(&field_->ctl.p->ntrail, &zero, sizeof(int), cudaMemcpyHostToDevice, s_), "ntrail");
    cuda_check(cudaStreamSynchronize(s_), "ntrail sync");
    c.ntrail = 0;
  }

  void set_lastpos(Index layer, const V3& p) {
    const double v[4] = {p.x, p.y, p.z, 1.0};
    cuda_check(cudaMemcpyAsync(field_->lastpos.p + 4 * static_cast<size_t>(layer), v, sizeof v, cudaMemcpyHostToDevice,
                               s_),
               "lastpos");
    cuda_check(cudaStreamSynchronize(s_), "lastpos sync");
  }
  bool get_lastpos(Index layer, V3& p) const {
    double v[4];
    cuda_check(cudaMemcpyAsync(v, field_->lastpos.p + 4 * static_cast<size_t>(layer), sizeof v, cudaMemcpyDeviceToHost,
                               s_),
               "lastpos");
    cuda_check(cudaStreamSynchronize(s_), "lastpos sync");
    if (v[3] == 0.0) return false;
    p = {v[0], v[1], v[2]};
    return true;
  }

  std::vector<Index> band_of(const std::vector<std::pair<Index, double>>& vals) const {
    std::vector<Index> band;
    for (const auto& [v, x] : vals)
      if (x < 1.0 && x > cfg_.band_low_threshold && x < cfg_.saturation) band.push_back(v);
    return band;
  }

  // handle_split (diffusion.hpp:642).
  bool handle_split(Index layer, const std::vector<FrontComponent>& fronts, long s) {
    const auto vals = field_->layer_values(layer);
    std::vector<Index> unsat;
    for (const auto& [v, x] : vals)
      if (x < 1.0) unsat.push_back(v);
    auto is_unsat = [&](Index v) { return std::binary_search(unsat.begin(), unsat.end(), v); };
    std::unordered_map<Index, Index> label;
    std::vector<Index> queue;
    for (Index c = 0; c < fronts.size(); ++c)
      for (Index v : fronts[c].boundary_vertices)
        if (label.emplace(v, c).second) queue.push_back(v);
    with_view([&](const auto& mv) {
      mv.need_vertices(unsat);  // the search only enters unsaturated vertices
      for (size_t head = 0; head < queue.size(); ++head) {
        const Index v = queue[head];
        const Index c = label.at(v);
        for (Index u : mv.v2v(v)) {
          if (!is_unsat(u)) continue;
          if (label.emplace(u, c).second) queue.push_back(u);
        }
      }
      return 0;
    });
    std::vector<std::vector<Index>> comps(fronts.size());
    for (Index v : unsat) {
      auto it = label.find(v);
      comps[it == label.end() ? 0 : it->second].push_back(v);
    }
    comps.erase(std::remove_if(comps.begin(), comps.end(), [](const auto& c) { return c.empty(); }), comps.end());
    if (comps.size() < 2) return false;
    std::vector<Index> parent_band;
    for (const auto& f : fronts) parent_band.insert(parent_band.end(), f.boundary_vertices.begin(), f.boundary_vertices.end());
    std::sort(parent_band.begin(), parent_band.end());
    parent_band.erase(std::unique(parent_band.begin(), parent_band.end()), parent_band.end());
    const std::vector<Index> children = field_->split_layer(layer, comps, s);
    TopologyEvent ev;
    ev.kind = EventKind::Split;
    ev.step = s;
    ev.layers = {layer};
    ev.produced = children;
    ev.position = with_view([&](const auto& mv) { return mean_of(mv, parent_band); });
    const Index idx = static_cast<Index>(res_.events.size());
    res_.events.push_back(std::move(ev));
    track(layer).consumed_event = idx;
    for (Index c : children) track(c).created_event = idx;
    return true;
  }

  // front_loop_of_layer (diffusion.hpp:606): longest mid-level isoline of the
  // layer that is not a frozen seam.
  bool front_loop(Index layer, SurfaceLoop& out) const {
    const DevMesh m = dm_->view();
    DeviceField& F = *field_;
    cuda_check(cudaMemsetAsync(F.acnt.p, 0, sizeof(int), s_), "memset");
    ck(launch_crossings(m, F.view(), static_cast<int>(layer), 0.5, F.ai0.p, F.ad0.p, F.ad1.p, F.ad2.p, F.acnt.p, s_),
       "crossings");
    const int n = to_host(F.acnt, 1, s_)[0];
    std::vector<int> e = to_host(F.ai0, n, s_);
    std::vector<double> t = to_host(F.ad0, n, s_), ba = to_host(F.ad1, n, s_), bb = to_host(F.ad2, n, s_);
    std::unordered_map<Index, double> t_of, b0, b1;
    for (int i = 0; i < n; ++i) {
      t_of[static_cast<Index>(e[i])] = t[i];
      b0[static_cast<Index>(e[i])] = ba[i];
      b1[static_cast<Index>(e[i])] = bb[i];
    }
    std::sort(e.begin(), e.end());
    std::vector<SurfaceLoop> loops = with_view([&](const auto& mv) { return chain_crossings(mv, e, t_of); });
    double best = -1;
    for (auto& loop : loops) {
      double base_mass = 0;
      size_t samples = 0;
      for (const auto& p : loop.points) {
        if (p.edge == kInvalid) continue;
        base_mass += (1.0 - p.edge_t) * b0.at(p.edge) + p.edge_t * b1.at(p.edge);
        ++samples;
      }
      if (samples == 0 || base_mass / samples < 0.01) continue;
      const double len = loop.length();
      if (len > best) {
        best = len;
        out = std::move(loop);
      }
    }
    return best > 0;
  }

  // handle_merge (diffusion.hpp:698).
  void handle_merge(const std::vector<Index>& group, long s) {
    struct FrontLoop {
      Index layer;
      SurfaceLoop loop;
      double length;
    };
    std::vector<FrontLoop> loops;
    for (Index id : group) {
      SurfaceLoop loop;
      if (front_loop(id, loop)) loops.push_back({id, std::move(loop), 0});
    }
    for (auto& fl : loops) fl.length = fl.loop.length();
    std::vector<Index> union_band;
    std::map<Index, std::vector<std::pair<Index, double>>> snaps;
    for (Index id : group) {
      auto vals = field_->layer_values(id);
      auto band = band_of(vals);
      union_band.insert(union_band.end(), band.begin(), band.end());
      snaps[id] = std::move(vals);
    }
    std::sort(union_band.begin(), union_band.end());
    union_band.erase(std::unique(union_band.begin(), union_band.end()), union_band.end());
    TopologyEvent ev;
    ev.kind = EventKind::Merge;
    ev.step = s;
    ev.layers = group;
    ev.position = with_view([&](const auto& mv) { return mean_of(mv, union_band); });
    ev.covered_snapshot = field_->covered_set(cfg_.covered_threshold);
    const Index idx = static_cast<Index>(res_.events.size());
    if (!loops.empty()) {
      size_t drop = 0;
      for (size_t i = 1; i < loops.size(); ++i)
        if (loops[i].length > loops[drop].length ||
            (loops[i].length == loops[drop].length && loops[i].layer < loops[drop].layer))
          drop = i;
      loops.erase(loops.begin() + static_cast<std::ptrdiff_t>(drop));
      std::sort(loops.begin(), loops.end(), [](const FrontLoop& a, const FrontLoop& b) {
        return a.length != b.length ? a.length < b.length : a.layer < b.layer;
      });
      for (auto& fl : loops) {
        HandleEstimate est;
        est.loop = std::move(fl.loop);
        est.layer = fl.layer;
        est.field_snapshot = snaps[fl.layer];
        est.event_index = idx;
        ev.estimates.push_back(std::move(est));
      }
    }
    const Index merged = field_->merge_layers(group, s);
    ev.produced = {merged};
    const V3 pos = ev.position;
    res_.events.push_back(std::move(ev));
    for (Index id : group) track(id).consumed_event = idx;
    track(merged).created_event = idx;
    set_lastpos(merged, pos);
  }

  void handle_vanish(Index layer, long s) {
    TopologyEvent ev;
    ev.kind = EventKind::Vanish;
    ev.step = s;
    ev.layers = {layer};
    V3 p;
    if (!get_lastpos(layer, p)) {
      std::vector<Index> support;
      for (const auto& [v, x] : field_->layer_values(layer)) support.push_back(v);
      p = with_view([&](const auto& mv) { return mean_of(mv, support); });
    }
    ev.position = p;
    const Index idx = static_cast<Index>(res_.events.size());
    res_.events.push_back(std::move(ev));
    track(layer).consumed_event = idx;
    field_->set_inactive(layer);
  }

  // check() (diffusion.hpp:807) for a step at which the device flagged an
  // event.  Returns true when the run is over.
  bool host_check(long s) {
    const auto t0 = std::chrono::steady_clock::now();
    ++res_.event_checks;
    bool changed = false;
    {
      const std::vector<LayerStat> st = read_stats(*field_, s);
      const std::vector<Index> act = field_->active_nonbase();
      for (size_t a = 0; a < act.size(); ++a) {
        if (st[a].ncomp < 2) continue;
        auto fronts = with_view([&](const auto& mv) { return extract_front_with(mv, *field_, act[a], cfg_); });
        if (fronts.size() < 2)
          fail(kInconsistentLog, "device reported a split the host front extraction does not see");
        changed |= handle_split(act[a], fronts, s);
      }
    }
    if (changed) {
      field_->sync_active();
      run_check_kernel(*field_, cfg_, co_, dt_, s);
    }
    const auto groups = groups_from_pairs(read_pairs(*field_, s));
    for (const auto& g : groups) {
      handle_merge(g, s);
      changed = true;
    }
    if (!groups.empty()) {
      field_->sync_active();
      run_check_kernel(*field_, cfg_, co_, dt_, s);
    }
    // Band anchors (device: means, snaps, trail records) and vanishing layers.
    const std::vector<Index> act = field_->active_nonbase();
    const std::vector<LayerStat> st = read_stats(*field_, s);
    StepParams p = params();
    p.step_begin = s;
    if (cfg_.record_trails) ck(launch_snap(dm_->view(), field_->view(), field_->work(), p, s_), "snap");
    ck(launch_flush(dm_->view(), field_->view(), field_->work(), p, s_), "flush");
    cuda_check(cudaStreamSynchronize(s_), "flush sync");
    Ctl c = field_->read_ctl();
    drain_trails(c);
    bool vanished = false;
    for (size_t a = 0; a < act.size(); ++a) {
      if (st[a].nband > 0) continue;
      if (field_->finished(act[a], st[a].nunsat)) {
        handle_vanish(act[a], s);
        vanished = true;
      }
    }
    if (cfg_.on_check) cfg_.on_check(s);
    bool done = false;
    const double bmax = [&] {
      double d;
      std::memcpy(&d, &c.base_max_bits[slot4(s)], 8);
      return d;
    }();
    if (c.base_one == 0 && bmax < 1.0 - cfg_.saturation) {
      for (Index l : field_->active_nonbase()) handle_vanish(l, s);
      done = true;
    } else if (field_->active_nonbase().empty()) {
      done = true;
    }
    field_->sync_active();
    // Vertices logged by split/merge join the next frontier (change log).
    if (!field_->pending_moved.empty()) {
      field_->mark_region(op_.view(), field_->pending_moved, s);
      field_->pending_moved.clear();
    }
    (void)vanished;
    if (cfg_.record_hashes && s < static_cast<long>(field_->hashes.n)) {
      const unsigned long long h = field_->hash();
      cuda_check(cudaMemcpyAsync(field_->hashes.p + s, &h, sizeof h, cudaMemcpyHostToDevice, s_), "hash");
      cuda_check(cudaStreamSynchronize(s_), "hash sync");
    }
    res_.t_events += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return done;
  }

  void finish_tracks() { res_.tracks = tracks_; }

  void report_phases() const {
    std::vector<unsigned long long> t = to_host(prof_, prof_.n, s_);
    double sum[3] = {0, 0, 0}, tot = 0;
    long n = 0, nd = 0, nx = 0;
    const size_t nstep_slots = 4 * static_cast<size_t>(std::min<long>(cfg_.max_steps, 100000));
    for (size_t i = 0; i + 4 < nstep_slots; i += 4) {
      if (!t[i] || !t[i + 3] || !t[i + 4]) continue;
      sum[0] += static_cast<double>(t[i + 1] - t[i]);
      sum[1] += static_cast<double>(t[i + 2] - t[i + 1]);
      sum[2] += static_cast<double>(t[i + 3] - t[i + 2]);
      tot += static_cast<double>(t[i + 4] - t[i]);
      nd += t[i + 1] > t[i];
      nx += t[i + 3] > t[i + 2] + 1000;  // ns: the extra union-find phases, not the timer reads
      ++n;
    }
    if (n)
      std::fprintf(stderr,
                   "[dtb] phase us/step over %ld steps: D+A %.2f  E+A %.2f  extra %.2f  step %.2f (blocks %d; "
                   "%ld steps with D+A, %ld with the extra union-find)\n",
                   n, sum[0] / n / 1e3, sum[1] / n / 1e3, sum[2] / n / 1e3, tot / n / 1e3, blocks_, nd, nx);
    {
      const size_t tb = t.size() - 64 * 3 * static_cast<size_t>(blocks_) - 16;
      std::fprintf(stderr, "[dtb]   trace (last D item of CTA0/thread0, us from phase start): list+binfo %.2f  active %.2f  probe %.2f  unite %.2f\n",
                   (t[tb + 1] - t[tb]) / 1e3, (t[tb + 2] - t[tb]) / 1e3, (t[tb + 3] - t[tb]) / 1e3, (t[tb + 4] - t[tb]) / 1e3);
    }
    // Per-CTA completion spread within each phase (steps 8..63 of the first launch).
    const size_t base = t.size() - 64 * 3 * static_cast<size_t>(blocks_);
    for (int ph = 0; ph < 3; ++ph) {
      std::vector<double> lat;
      const long off = std::min<long>(cfg_.max_steps, 100000) - 64;  // trace covers the launch's last 64 steps
      for (long st = 8; st < 64; ++st) {
        const unsigned long long t0 = off >= 0 ? t[4 * (off + st) + ph] : 0;  // phase start = previous phase's barrier exit
        if (!t0) continue;
        for (int b = 0; b < blocks_; ++b) {
          const unsigned long long tb = t[base + (st * 3 + ph) * blocks_ + b];
          if (tb > t0) lat.push_back(static_cast<double>(tb - t0) / 1e3);
        }
      }
      if (lat.empty()) continue;
      std::vector<double> work, skew;
      const size_t sbase = t.size() - 2 * 64 * 3 * static_cast<size_t>(blocks_) - 16;
      for (long st = 8; st < 64; ++st)
        for (int b = 0; b < blocks_; ++b) {
          const unsigned long long ts = t[sbase + (st * 3 + ph) * blocks_ + b];
          const unsigned long long td = t[base + (st * 3 + ph) * blocks_ + b];
          const unsigned long long t0 = off >= 0 ? t[4 * (off + st) + ph] : 0;
          if (ts && td > ts) work.push_back(static_cast<double>(td - ts) / 1e3);
          if (ts && t0 && ts > t0) skew.push_back(static_cast<double>(ts - t0) / 1e3);
        }
      std::sort(work.begin(), work.end());
      std::sort(skew.begin(), skew.end());
      if (!work.empty() && !skew.empty())
        std::fprintf(stderr, "[dtb]   phase %d CTA work (us): p50 %.2f p90 %.2f max %.2f | start skew p50 %.2f p90 %.2f max %.2f\n",
                     ph, work[work.size() / 2], work[work.size() * 9 / 10], work.back(), skew[skew.size() / 2],
                     skew[skew.size() * 9 / 10], skew.back());
      std::sort(lat.begin(), lat.end());
      std::fprintf(stderr, "[dtb]   phase %d CTA done after start (us): min %.2f p50 %.2f p90 %.2f max %.2f\n", ph,
                   lat.front(), lat[lat.size() / 2], lat[lat.size() * 9 / 10], lat.back());
      // Per step: the slowest CTA (what the barrier waits for) against the median one.
      double smax = 0, smed = 0;
      int ns = 0;
      for (long st = 8; st < 64; ++st) {
        const unsigned long long t0 = off >= 0 ? t[4 * (off + st) + ph] : 0;
        if (!t0) continue;
        std::vector<double> d;
        for (int b = 0; b < blocks_; ++b) {
          const unsigned long long tb = t[base + (st * 3 + ph) * blocks_ + b];
          if (tb > t0) d.push_back(static_cast<double>(tb - t0) / 1e3);
        }
        if (d.size() < 2) continue;
        if (ph == 1) {
          int am = 0;
          for (int b = 1; b < static_cast<int>(d.size()); ++b)
            if (d[b] > d[am]) am = b;
          std::fprintf(stderr, "%d:%.1f ", am, d[am]);
        }
        std::sort(d.begin(), d.end());
        smax += d.back();
        smed += d[d.size() / 2];
        ++ns;
      }
      if (ns)
        std::fprintf(stderr, "[dtb]   phase %d per step: slowest CTA %.2f us, median CTA %.2f us (mean over %d steps)\n",
                     ph, smax / ns, smed / ns, ns);
    }
  }

  std::shared_ptr<DeviceMesh> dm_;
  const Mesh& mesh() const { return dm_->host(); }  // downloaded on first use for device-built meshes
  // Event handlers read the mesh through a view: the host mesh when there is
  // one, else local gathers from the device (never the whole-mesh download).
  template <class F>
  auto with_view(F&& f) const -> decltype(f(std::declval<const HostView&>())) {
    if (dm_->has_host()) return f(HostView(dm_->host()));
    if (!local_) local_ = std::make_unique<LocalMesh>(*dm_, s_);
    return f(*local_);
  }
  mutable std::unique_ptr<LocalMesh> local_;
  const DeviceLaplacian& op_;
  Config cfg_;
  Coefficients co_;
  cudaStream_t s_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, ev0k_ = nullptr, ev1k_ = nullptr;
  std::shared_ptr<DeviceField> field_;
  InitialPassResult res_;
  std::vector<LayerTrack> tracks_;
  double dt_ = 0;
  int blocks_ = 1;
  DevBuf<unsigned long long> prof_;  // DTB_PHASE_PROF=1: per-step phase timestamps of the first launch
};

}  // namespace

InitialPassResult run_initial_pass(std::shared_ptr<DeviceMesh> dm, const DeviceLaplacian& op, Index seed,
                                   const Config& cfg, const Coefficients& c) {
  PassEngine e(std::move(dm), op, seed, cfg, c);
  return e.run();
}

ReebGraph build_reeb(const InitialPassResult& r) {
  ReebGraph g;
  for (const auto& ev : r.events) g.nodes.push_back({ev.kind, ev.position, ev.step});
  for (const auto& t : r.tracks) {
    if (t.layer == kInvalid || t.created_event == kInvalid || t.consumed_event == kInvalid) continue;
    if (t.consumed_event < t.created_event) fail(kInconsistentLog, "layer consumed before created");
    g.arcs.push_back({t.created_event, t.consumed_event, t.layer, t.trail});
  }
  return g;
}

}  // namespace dtb
