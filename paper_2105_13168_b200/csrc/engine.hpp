// Host orchestration of the device engine: device-resident mesh, Laplacian
// operator, layer field, and the initial pass (reference diffusion.hpp).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "kernels.h"
#include "mesh.hpp"

namespace dtb {

void cuda_check(cudaError_t e, const char* what);

// Caching device allocator: freed blocks are kept in size classes and handed
// out again, so repeated passes / meshes never pay cudaMalloc + cudaFree (the
// latter synchronises the whole device).  Bounded by kCacheBytes.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(sizeof(T) * count));
  }
  void release() {
    if (p) dev_free(p, sizeof(T) * n);
    p = nullptr;
    n = 0;
  }
  void upload(const T* src, size_t count, cudaStream_t s) {
    cuda_check(cudaMemcpyAsync(p, src, sizeof(T) * count, cudaMemcpyHostToDevice, s), "H2D");
  }
  void download(T* dst, size_t count, cudaStream_t s) const {
    cuda_check(cudaMemcpyAsync(dst, p, sizeof(T) * count, cudaMemcpyDeviceToHost, s), "D2H");
  }
  void zero(cudaStream_t s) {
    if (n) cuda_check(cudaMemsetAsync(p, 0, sizeof(T) * n, s), "memset");
  }
};

class DeviceField;

// Mesh geometry and topology resident in HBM.  Also pools the per-run field
// workspaces (columns, frontier lists, union-find parents ...) so repeated
// passes on one mesh do not re-allocate hundreds of MB.
class DeviceMesh : public std::enable_shared_from_this<DeviceMesh> {
 public:
  // Uploads a host-built mesh.
  explicit DeviceMesh(std::shared_ptr<const Mesh> mesh, cudaStream_t s);
  // Builds the mesh on the device from a triangle soup (csrc/meshbuild.cu);
  // nullptr when the host must build it (unusual or invalid input).
  static std::shared_ptr<DeviceMesh> from_soup(const double* xyz, size_t nv, const std::uint32_t* faces, size_t nf,
                                               cudaStream_t s);
  ~DeviceMesh();
  // A field workspace for this mesh from the process-wide pool.
  std::shared_ptr<DeviceField> acquire_field(cudaStream_t s);
  // Puts `count` workspaces for meshes of up to nv vertices / ne edges into
  // the process-wide pool (a batch allocates before its passes start, so no
  // pass frees device memory -- an implicit device synchronisation -- while
  // others run).
  static void reserve_fields(size_t count, size_t nv, size_t ne);
  Index nv() const { return nv_; }
  Index nf() const { return nf_; }
  Index ne() const { return ne_; }
  // The host mesh; for a device-built mesh it is downloaded on first use.
  const Mesh& host() const { return *host_ptr(); }
  std::shared_ptr<const Mesh> host_ptr() const;
  V3 position(Index v) const;  // one vertex position, without the host mesh
  bool has_host() const {
    std::lock_guard<std::mutex> lk(host_mu_);
    return static_cast<bool>(mesh_);
  }
  DevMesh view() const { return view_; }  // stiffness fields are filled by DeviceLaplacian::view()

  DevBuf<double> px, py, pz;
  DevBuf<long long> fx, fy, fz;
  DevBuf<unsigned> faces, edges, fe, ef;  // faces, edge vertices, face->edges, edge->faces
  size_t h2d_bytes = 0;  // host->device bytes of the upload
  DevBuf<int> c_off, c_col, n_off, n_col, f_off, f_col;  // front connectivity, neighbours, v2f

 private:
  DeviceMesh() = default;
  // Positions (SoA + fixed point) and the front-connectivity CSR from the
  // uploaded or device-built arrays.
  void derive(const double* d_xyz, double maxabs, cudaStream_t s);
  mutable std::mutex host_mu_;
  mutable std::shared_ptr<const Mesh> mesh_;
  DevBuf<double> xyz_;  // device-built meshes keep their positions for the host download
  Index nv_ = 0, nf_ = 0, ne_ = 0;
  DevMesh view_;
};

// Cotangent stiffness + lumped masses (operators.hpp LaplacianOperator).
class DeviceLaplacian {
 public:
  // Assembled on the device from the mesh.
  DeviceLaplacian(std::shared_ptr<DeviceMesh> dm, cudaStream_t s);
  // From a host CSR (e.g. the reference's own operator) -- for parity tests.
  DeviceLaplacian(std::shared_ptr<DeviceMesh> dm, const std::vector<int>& off, const std::vector<int>& col,
                  const std::vector<double>& val, const std::vector<double>& mass, double gershgorin, cudaStream_t s);
  int nnz() const { return nnz_; }
  double gershgorin() const { return gersh_; }
  void download(std::vector<int>& off, std::vector<int>& col, std::vector<double>& val, std::vector<double>& mass,
                cudaStream_t s) const;
  void apply(const double* x_host, double* y_host, cudaStream_t s) const;
  void sweep_bench(int reps, cudaStream_t s, double* seconds, double* bytes) const;
  std::shared_ptr<DeviceMesh> mesh() const { return dm_; }
  DevMesh view() const;
  void build_ell(cudaStream_t s);

  DevBuf<int> off, col;
  DevBuf<double> val, mass;
  DevBuf<unsigned char> e_len;  // padded rows (DevMesh::e_len)
  DevBuf<int> e_col;
  DevBuf<double> e_val;

 private:
  std::shared_ptr<DeviceMesh> dm_;
  int nnz_ = 0;
  double gersh_ = 0;
};

struct Coefficients {  // layer_field.hpp CoefficientScheme
  double gradient_energy = 1.0 / 25.0;
  double penalty = 1.0 / 125.0;
  double contact = 1.0 / 30.0;
  double mobility = 0.25;
};

struct Config {  // diffusion.hpp DiffusionConfig
  double dt = 0.0;
  double band_low_threshold = 0.05;
  double saturation = 0.999;
  double collision_threshold = 0.1;
  int check_interval = 1;
  long max_steps = 200000;
  double covered_threshold = 0.05;
  double seed_radius = 0.0;
  bool record_trails = true;
  bool record_hashes = false;  // per-check field digests (parity tooling)
  int grid_ctas = 0;           // CTAs of the persistent step kernel (0: one per SM); batches split the SMs
  std::function<void(long)> on_check;  // host hook; forces a host round trip per check
  void validate() const;
};

double stable_time_step(const DeviceLaplacian& op, const Coefficients& c);
std::vector<Index> seed_region(const Mesh& mesh, Index seed, double radius);

struct LoopPoint {
  V3 position;
  Index face = kInvalid, edge = kInvalid, vertex = kInvalid;
  double edge_t = 0.0;
};
struct SurfaceLoop {
  std::vector<LoopPoint> points;
  bool closed = true;
  double length() const;
  V3 centroid() const;
};

struct FrontComponent {
  Index layer = kInvalid;
  std::vector<Index> triangles, boundary_vertices;
  double band_length = 0;
};

enum class EventKind { Seed = 0, Split = 1, Merge = 2, Vanish = 3 };

struct HandleEstimate {
  SurfaceLoop loop;
  Index layer = kInvalid;
  std::vector<std::pair<Index, double>> field_snapshot;  // sorted by vertex
  Index event_index = kInvalid;
};

struct TopologyEvent {
  EventKind kind;
  long step = 0;
  std::vector<Index> layers, produced;
  V3 position{};
  std::vector<HandleEstimate> estimates;
  std::vector<Index> covered_snapshot;
};

struct LayerTrack {
  Index layer = kInvalid, created_event = kInvalid, consumed_event = kInvalid;
  std::vector<V3> trail;
};

struct LayerMeta {
  bool active = false, cleared = false;
  Index parent = kInvalid;
  std::vector<Index> merge_parents;
  long created_step = 0;
};

// The dynamic layer matrix Phi, resident on the device as per-vertex columns.
class DeviceField {
 public:
  DeviceField(std::shared_ptr<DeviceMesh> dm, cudaStream_t s);
  DeviceField(DeviceMesh* dm, cudaStream_t s, size_t nv_cap = 0, size_t ne_cap = 0);  // pooled (no ownership)
  // init_field (layer_field.hpp:318): base + one seed layer.
  void init(const std::vector<Index>& seeds);

  int layer_count() const { return static_cast<int>(meta_.size()); }
  const LayerMeta& meta(Index id) const { return meta_[id]; }
  std::vector<Index> active_nonbase() const;
  void sync_active();  // upload active flags / dense indices

  std::vector<std::pair<Index, double>> layer_values(Index layer) const;  // sorted by vertex
  std::vector<double> dense_row(Index layer) const;
  std::vector<Index> covered_set(double threshold) const;
  unsigned long long hash() const;
  void normalize_columns();
  std::vector<Index> split_layer(Index layer, const std::vector<std::vector<Index>>& comps, long step);
  Index merge_layers(const std::vector<Index>& ids, long step, std::vector<int>* touched = nullptr);
  void set_inactive(Index layer);
  bool finished(Index layer, int nunsat) const;  // diffusion.hpp:795
  int base_one_count() const;

  DevField view() const { return view_; }
  DevWork work() const { return work_; }
  // Band-item segments for a launch grid of `blocks` CTAs (one per CTA).
  void set_grid(int blocks);
  DeviceMesh& mesh() { return *dm_; }
  const DeviceMesh& mesh() const { return *dm_; }
  cudaStream_t stream() const { return s_; }
  void set_stream(cudaStream_t s) { s_ = s; }
  size_t capacity() const { return cap_; }
  size_t edge_capacity() const { return cap_e_; }
  void retarget(DeviceMesh* dm) { dm_ = dm; }
  void set_band(double lo, double sat) {
    work_.band_lo = lo;
    work_.sat = sat;
  }
  Ctl read_ctl() const;
  // Queues verts and their stiffness rows as the frontier of step stamp+1.
  void mark_region(const DevMesh& op_view, const std::vector<int>& verts, long stamp);
  // Before an engine or check launch whose first check is step t: the band
  // list E(t) reads, rebuilt from the interest flags (host edits and a
  // discarded speculative update leave the incremental list stale).
  void rebuild_band_list(long t);
  double prune_epsilon = 1e-9;
  // Vertices logged by split/merge edits since the last take (change log).
  std::vector<int> pending_moved;

  // storage: the two field copies (DevField::b), lists by slot4(step)
  DevBuf<unsigned char> cnt[2], interest[2], active;
  DevBuf<unsigned short> lay[2];
  DevBuf<double> val[2], lastpos;
  DevBuf<uint4> binfo[2];
  DevBuf<int> region[4], ilist[4], stamp, aidx, alist;
  DevBuf<int2> bandpairs[2], bp_ovf[2];
  DevBuf<int> bpcount[2];
  DevBuf<int> ai0, ai1, acnt;       // event-time scratch (see setup())
  DevBuf<double> ad0, ad1, ad2;
  DevBuf<unsigned long long> parent, pair_keys, hashes;
  DevBuf<int2> added;   // band items gained this step (split certificate)
  DevBuf<int> add_stamp;  // per vertex: last step it gained a band item
  DevBuf<int> rem_stamp;  // per vertex: last step it lost a band item
  DevBuf<unsigned long long> seed_dist;  // seed Dijkstra distances, kept "far" between calls
  DevBuf<unsigned> pairs;
  DevBuf<LayerStat> stat;
  DevBuf<TrailRec> trail;
  DevBuf<Ctl> ctl;

 private:
  friend class DeviceMesh;
  void setup(size_t nv_cap = 0, size_t ne_cap = 0);
  DeviceMesh* dm_;
  std::shared_ptr<DeviceMesh> keep_;  // keeps the mesh alive while the field is handed out
  size_t cap_ = 0;                    // vertex capacity of the device buffers
  size_t cap_e_ = 0;                  // edge capacity (event-time scratch)
  cudaStream_t s_;
  std::vector<LayerMeta> meta_;
  DevField view_;
  DevWork work_;
};

struct InitialPassResult {
  std::vector<TopologyEvent> events;
  std::vector<LayerTrack> tracks;
  double dt_used = 0;
  long steps = 0;
  Index seed_vertex = 0;
  int status = 0;  // ErrorCode (0 ok)
  std::string message;
  std::vector<unsigned long long> hashes;  // per check step (if recorded)
  std::shared_ptr<DeviceField> field;
  long handle_estimate_count() const;
  // Timing breakdown (seconds): device step loop vs. host event handling.
  double t_device = 0, t_events = 0;
  double t_pass_device = 0;  // CUDA-event time of the whole pass on its stream
  double t_kernel = 0;       // CUDA-event time of the persistent step-kernel launches
  long launches = 0, event_checks = 0, kernel_steps = 0;
  unsigned long long sum_region = 0, sum_interest = 0;  // device work counters
};

// extract_front (diffusion.hpp:398) on host data pulled from the device.
std::vector<FrontComponent> extract_front(const DeviceField& field, Index layer, const Config& cfg);
// detect_collisions (diffusion.hpp:475) via the device check kernel.
std::vector<std::vector<Index>> detect_collisions(DeviceField& field, const Config& cfg);
// One explicit Euler update of the whole field (diffusion.hpp:386).
void step(DeviceField& field, const DeviceLaplacian& op, const Config& cfg, const Coefficients& c);
// extract_isoline (isoline.hpp:55) of a host value array.
std::vector<SurfaceLoop> extract_isoline(const Mesh& mesh, const std::vector<double>& values, double level);

InitialPassResult run_initial_pass(std::shared_ptr<DeviceMesh> dm, const DeviceLaplacian& op, Index seed,
                                   const Config& cfg, const Coefficients& c = {});

// Reeb graph from the event log (SPEC reeb.build_reeb; nodes = events, arcs =
// layer lifetimes, embedding = the layer trails).
struct ReebGraph {
  struct Node {
    EventKind kind;
    V3 position;
    long step;
  };
  struct Arc {
    Index from, to, layer;
    std::vector<V3> embedding;
  };
  std::vector<Node> nodes;
  std::vector<Arc> arcs;
  long cycle_rank() const { return static_cast<long>(arcs.size()) - static_cast<long>(nodes.size()) + 1; }
};
ReebGraph build_reeb(const InitialPassResult& r);

}  // namespace dtb
