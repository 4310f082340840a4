// Device data layout and kernel launchers for the diffusion-front engine.
//
// HBM layout:
//   * mesh: SoA positions (3 x f64), fixed-point positions (3 x i64, for
//     order-independent band sums), faces (3 x u32), edges (2 x u32),
//     stiffness CSR (i32 offsets / i32 columns / f64 values), lumped masses,
//     the front-connectivity CSR (mesh neighbours plus the apexes opposite each
//     link edge) and the mesh neighbour CSR.
//   * field: the transposed layer matrix Phi^T as fixed-capacity columns -- per
//     vertex a count (u8) and kSlots (layer id u16, value f64) pairs sorted by
//     layer id.  Column v holds exactly the reference's owners_[v] list
//     (layer_field.hpp:310) with the values of layers_[id].values[v].
//   * work: double-buffered region lists (the reference's one-ring-dilated
//     frontier, diffusion.hpp:253-271) with per-vertex stamps, per-region-slot
//     scratch columns, the "interest" flags/list (vertices holding any value
//     strictly inside (0,1)), versioned union-find parents per (vertex, slot),
//     per-active-layer statistics and the collision pair set.
#pragma once

#include <cstddef>
#include <cstdint>

#include <vector_types.h>  // int2, uint4 (CUDA header, usable from host C++)

namespace dtb {
constexpr unsigned kBandOverflow = 0xFFFFu;
}

#ifdef __CUDACC__
namespace dtb {
// Band index of a column (see DevField::binfo).
__device__ __forceinline__ uint4 make_binfo(const unsigned short* lay, const double* val, int c, double lo,
                                            double sat) {
  unsigned L[4] = {0, 0, 0, 0}, S[4] = {0, 0, 0, 0};
  int n = 0;
  bool over = false;
  for (int j = 0; j < c; ++j) {
    const unsigned l = lay[j];
    const double x = val[j];
    if (l != 0 && x > lo && x < sat) {
      if (n < 4) {
        L[n] = l;
        S[n] = static_cast<unsigned>(j);
        ++n;
      } else {
        over = true;
      }
    }
  }
  uint4 r;
  r.x = L[0] | (L[1] << 16);
  r.y = L[2] | (L[3] << 16);
  r.z = S[0] | (S[1] << 16);
  r.w = S[2] | ((over ? kBandOverflow : S[3]) << 16);
  return r;
}
__device__ __forceinline__ unsigned binfo_layer(const uint4& b, int t) {
  const unsigned w = t < 2 ? b.x : b.y;
  return (w >> (16 * (t & 1))) & 0xFFFFu;
}
__device__ __forceinline__ unsigned binfo_slot(const uint4& b, int t) {
  const unsigned w = t < 2 ? b.z : b.w;
  return (w >> (16 * (t & 1))) & 0xFFFFu;
}
__device__ __forceinline__ bool binfo_overflow(const uint4& b) { return (b.w >> 16) == kBandOverflow; }
}  // namespace dtb
#endif

namespace dtb {

constexpr int kSlots = 32;         // max owners per vertex (column capacity)
constexpr int kMaxLayers = 65535;  // layer ids are u16
constexpr int kMaxActive = 4096;   // simultaneously active non-base layers
constexpr int kPairCap = 1 << 16;  // collision pair hash table slots
constexpr int kTrailCap = 1 << 20; // device trail ring capacity (records)
constexpr int kBlock = 512;        // threads per CTA for all engine kernels
constexpr int kEll = 8;            // padded stiffness row width (= 8-lane group)
constexpr int kRemovedItem = 1 << 30;  // layer-word flag of a lost band item in DevWork::added

// Error codes raised by device code (mirrored in mesh.hpp ErrorCode).
enum DevError : int {
  kDevOk = 0,
  kDevBlowup = 10,    // NumericalBlowup (diffusion.hpp:315)
  kDevZeroColumn = 7, // ZeroColumn (layer_field.hpp:148)
  kDevCapacity = 101, // column or candidate capacity exceeded
  kDevCertificate = 102,  // diagnostics (DTB_CERT_VERIFY=1): the split certificate held but the union-find split
};

// Stop reasons of the persistent step kernel.
enum StopBits : int {
  kStopNone = 0,
  kStopSplit = 1,      // some active layer has >= 2 band components
  kStopMerge = 2,      // a collision pair exists
  kStopVanish = 4,     // some active layer has no band and no unsaturated value
  kStopExtinct = 8,    // base layer extinct (diffusion.hpp:785)
  kStopError = 16,     // device error (see ctl.error)
  kStopEveryCheck = 32 // host requested a stop at every check (on_check hook)
};

struct DevMesh {
  int nv = 0, nf = 0, ne = 0;
  const double *px = nullptr, *py = nullptr, *pz = nullptr;
  const long long *fx = nullptr, *fy = nullptr, *fz = nullptr;  // fixed-point positions
  double fx_scale = 1.0;                                          // 2^-k
  const unsigned *faces = nullptr;                                // 3 * nf
  const unsigned *edges = nullptr;                                // 2 * ne (lo, hi)
  const int *s_off = nullptr, *s_col = nullptr;                   // stiffness CSR
  const double *s_val = nullptr, *mass = nullptr;
  // The same rows padded to kEll entries per vertex (columns -1 past the end;
  // e_len > kEll: use the CSR), so a row is one load away from the vertex id.
  const unsigned char* e_len = nullptr;
  const int* e_col = nullptr;
  const double* e_val = nullptr;
  const int *c_off = nullptr, *c_col = nullptr;                   // front connectivity
  const int *n_off = nullptr, *n_col = nullptr;                   // mesh neighbours
  const int *f_off = nullptr, *f_col = nullptr;                   // incident faces (v2f CSR)
  const unsigned *face_edges = nullptr, *edge_faces = nullptr;    // 3F (edge k joins corners k, k+1), 2E
};

// Per-step rotating slots.  The step loop runs E(s) (the check of step s)
// and A(s+1) (the update of step s+1) in one phase, so every list and
// counter that one step fills while another reads it rotates over four
// slots, slot4(t) = t & 3: a slot is cleared only two grid barriers after its
// last reader took it (the words read right after a barrier must stay put
// through the phase that follows) and before its next writer starts.
#ifdef __CUDACC__
__host__ __device__
#endif
inline int slot4(long long t) { return static_cast<int>(t & 3); }

// Control block in device memory (one per engine).  The first 112 bytes are
// the words every CTA snapshots after a grid barrier (CtlSnap).
struct Ctl {
  int rcount[4];       // frontier list sizes: frontier t is region[slot4(t)]
  int ilcount[4];      // band-list sizes: the list E(t) reads is ilist[slot4(t)]
  int error;           // DevError of a committed step
  int spec_error;      // error raised by a speculative update (next step)
  int dchange[4];      // by slot4(step): the step removed a band item (or overflowed a band index / list)
  int nadded[4];       // by slot4(step): band items added (W.added)
  int anchor_fail[4];  // by slot4(step): an added band item lacks a neighbour of the previous band
  int nbandpairs[4];   // by slot4(check): band items of that check in the overflow list
  int pad_[2];
  int error_vertex;
  int spec_error_vertex;
  int stop_bits;
  int pad0_;
  long long stop_step;       // last step executed by the kernel
  long long epoch;           // union-find / pair-set version
  int base_one;              // vertices whose base value is exactly 1.0 (between launches)
  int base_d[4];             // by slot4(step): that step's change of the count
  int base_cum[4];           // by slot4(step): the count after that step
  unsigned long long base_max_bits[4];  // by slot4(check): max base value in (0,1) (as ordered bits)
  int npairs[4];             // by slot4(check): collision pairs recorded
  int pair_overflow[4];
  int ntrail;                // trail records written (ring index)
  int bandpair_overflow;
  unsigned long long hash_acc[4];   // by slot4(check): field digest accumulator
  unsigned long long sum_region;    // work counters: frontier vertices updated
  unsigned long long sum_interest;  // band-list vertices checked
};

struct LayerStat {
  int ncomp, nband, nunsat, pad;
  long long sx, sy, sz;           // fixed-point band position sums
  unsigned long long snap;        // packed (distance bits | vertex) argmin
};

struct TrailRec {
  long long step;
  int layer, vertex;
  double mx, my, mz;  // band mean (last_band_position_)
  double vx, vy, vz;  // position of `vertex` (the trail point)
};

// One copy of the field columns.
struct FieldBuf {
  unsigned char *cnt = nullptr;   // nv
  unsigned short *lay = nullptr;  // nv * kSlots
  double *val = nullptr;          // nv * kSlots
  unsigned char *interest = nullptr;  // column holds a value strictly inside (0, 1)
  // Band index per vertex: up to 4 (layer, slot) pairs whose value lies in
  // (band_lo, sat), any activity; w's high half = 0xFFFF marks overflow.
  uint4 *binfo = nullptr;
};

// The field Phi^T, double-buffered by step parity: the update of step t
// reads b[(t-1) & 1] and writes b[t & 1] directly (no scratch, no commit
// phase).  Between launches both copies are identical; host edits write both.
struct DevField {
  FieldBuf b[2];
};

struct DevWork {
  int *region[4] = {nullptr, nullptr, nullptr, nullptr};  // frontier lists by slot4(step)
  int *stamp = nullptr;                 // per vertex: step whose update queued it
  int *ilist[4] = {nullptr, nullptr, nullptr, nullptr};   // band lists by slot4(step); dead entries skipped
  // (vertex, dense active index) band items of a check: one segment of bp_seg
  // entries per CTA (appended with a shared-memory counter, length in
  // bpcount[set][cta]), entries beyond a full segment in the overflow list
  // bp_ovf[set] (length Ctl::nbandpairs[slot4(check)]); set = check & 1.
  int2 *bandpairs[2] = {nullptr, nullptr};
  int *bpcount[2] = {nullptr, nullptr};
  int bp_nseg = 0, bp_seg = 0;
  int2 *bp_ovf[2] = {nullptr, nullptr};
  int bandpair_cap = 0;                 // capacity of each bp_ovf
  unsigned long long *parent = nullptr; // nv * kSlots versioned UF parents
  // 4 x added_cap band items (vertex, layer) gained -- or, with kRemovedItem
  // in the layer word, lost -- by slot4(step) (the split certificate's items)
  int2 *added = nullptr;
  int added_cap = 0;
  int *add_stamp = nullptr;             // per vertex: last step at which it gained a band item
  int *rem_stamp = nullptr;             // per vertex: last step at which it lost a band item
  unsigned char *active = nullptr;      // kMaxLayers + 1
  int *aidx = nullptr;                  // layer -> dense active index or -1
  int *alist = nullptr;                 // dense active index -> layer
  LayerStat *stat = nullptr;            // 4 x kMaxActive (slot4(check))
  unsigned long long *pair_keys = nullptr;  // kPairCap versioned keys
  unsigned *pairs = nullptr;            // 4 x kPairCap recorded pairs (first << 16 | second), slot4(check)
  double *lastpos = nullptr;            // 4 * (kMaxLayers + 1): x, y, z, valid
  TrailRec *trail = nullptr;            // trail_mask + 1 records (a power of two <= kTrailCap)
  int trail_mask = 0;
  unsigned long long *hashes = nullptr; // per-step field digests (optional)
  long long hash_base = 0;              // step of hashes[0]
  int hash_cap = 0;
  double band_lo = 0.05, sat = 0.999;  // band thresholds of the run (binfo maintenance)
  unsigned long long *prof = nullptr;  // optional phase timestamps (4 per step)
  int prof_cap = 0;
  Ctl *ctl = nullptr;
};

struct StepParams {
  double mu_n, m_mu_n, w, e, half_a2, dt, prune;
  double band_lo, sat, kappa, coll_base_limit, extinct_limit;
  long long step_begin, step_end;  // execute steps [step_begin, step_end)
  int check_interval;
  int n_active;
  int n_layers;  // layer ids in columns are below this (the active-flag table's length)
  int record_trails;
  int do_hash;
  int stop_every_check;
  int do_check;  // 0: advance only (one-shot step())
  int d_full;    // diagnostics: never skip the front union-find (DTB_D_FULL=1)
  int no_wide;   // diagnostics: no lane-parallel wide update (DTB_NO_WIDE=1)
  int cert_verify;  // diagnostics: run the union-find after a held certificate too, error if it splits
};

// --- launchers (kernels.cu) -------------------------------------------------
// Number of kernels this library has launched (all launchers increment it).
unsigned long long launch_count();
void note_launch(unsigned long long n = 1);
// All return a cudaError_t value as int.
int dev_max_coresident_blocks(int* out);
int launch_run(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, int blocks,
               void* stream);
int launch_check(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, int blocks,
                 void* stream);  // stats/CCL/collisions for the current state (no advance)
int launch_snap(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, void* stream);
// Writes trail / last-position records of the last check (step = p.step_begin) and resets the stats.
int launch_flush(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, void* stream);

// Laplacian assembly (laplacian.cu).
struct LapBuild {
  int nv, nf;
  const double *px, *py, *pz;
  const unsigned* faces;
  const int *v2v_off, *v2v;    // sorted mesh neighbours (CSR)
  const int *v2f_off, *v2f;    // incident faces in face order (CSR)
  int *s_off;                  // out: nv + 1
  int *s_col;                  // out: capacity nv + 2 * ne
  double *s_val;               // out
  double *mass;                // out
  double *gersh_row;           // out: per-row bound
  double *gersh_max;           // out: max over the rows (device scalar)
  int *nnz;                    // out
  long long nroom = 0;         // sum of row lengths of v2v (2E): the fill's room besides the diagonals
};
int launch_assemble(const LapBuild& b, void* stream);

// Mesh arrays built on the device (meshdev.cu).
struct FrontBuild {
  int nv;
  long long nrel_room;  // sum of valences (2E): the relation room is twice that
  const unsigned *faces, *face_edges, *edge_faces, *edges;  // 3F, 3F, 2E, 2E
  const int *v2v_off, *v2v, *v2f_off, *v2f;
};
// Records of listed vertices (positions, v2v and v2f rows), faces (corners,
// edges) and edges (ends, faces) for host event handling (meshdev.cu).
struct MeshRows {
  const double *px, *py, *pz;
  const int *v2v_off, *v2v, *v2f_off, *v2f;
  const unsigned *faces, *face_edges, *edges, *edge_faces;  // 3F, 3F, 2E, 2E
};
// bounds: 4 per vertex (v2v begin/end, v2f begin/end); pos: 3 per vertex.
int launch_gather_vhead(const MeshRows& m, const unsigned* list, int n, int* bounds, double* pos, void* stream);
// rows: vertex i's v2v row then its v2f row, from packed offset dst[i].
int launch_gather_vrows(const MeshRows& m, const int* bounds, const int* dst, int n, unsigned* rows, void* stream);
int launch_gather_faces(const MeshRows& m, const unsigned* list, int n, unsigned* out, void* stream);  // 6 per face
int launch_gather_edges(const MeshRows& m, const unsigned* list, int n, unsigned* out, void* stream);  // 4 per edge
int launch_positions(const double* xyz, int nv, double scale, double* px, double* py, double* pz, long long* fx,
                     long long* fy, long long* fz, void* stream);
void instr_report();
// seed_region on the device: *n = -1 when a capacity is exceeded (use the host).
// dist: nv words all 0x7F7F7F7F7F7F7F7F, left so (or null: a scratch copy is allocated).
int launch_seed_region(const DevMesh& m, unsigned seed, double radius, unsigned* out, int cap, int* n, void* stream,
                       unsigned long long* dist = nullptr);  // -DDTB_INSTR builds: latency histograms
// Device mesh construction (csrc/meshbuild.cu).  Returns 0 when the soup is a
// valid closed, connected, consistently oriented manifold without unused
// vertices (outputs filled, ne = 3nf/2), 1 when the host must build it (any
// other input, including every error case), else a CUDA error.
struct MeshBuild {
  int nv = 0, nf = 0, ne = 0;
  const double* xyz = nullptr;     // 3nv, device
  void* xyz_ready = nullptr;       // cudaEvent_t the stream waits on before reading xyz (or null)
  const unsigned* soup = nullptr;  // 3nf input faces, device
  unsigned *faces = nullptr, *edges = nullptr, *edge_faces = nullptr, *face_edges = nullptr;  // 3F, 2E, 2E, 3F
  int *v2f_off = nullptr, *v2f = nullptr, *v2v_off = nullptr, *v2v = nullptr;              // V+1, 3F, V+1, 2E
  double maxabs = 0;  // out: max |coordinate|
  int flipped = 0;    // out: faces were flipped to face outward
};
int build_mesh(MeshBuild& b, void* stream);
// Caching device allocator (engine.cpp), shared with the kernel-side helpers.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
// Gathers every vertex's relations into a room (returned through *room) and
// scans their counts into c_off; -1 when a vertex has too many relations.
int launch_front_count(const FrontBuild& b, int* c_off, int* nnz, void** room, void* stream);
// Moves the relations from the room to c_col; the caller frees the room
// (dev_free(room, front_room_bytes(b))) once the stream is done with it.
int launch_front_fill(const FrontBuild& b, const int* c_off, int* c_col, void* room, void* stream);
inline size_t front_room_bytes(const FrontBuild& b) {
  return sizeof(int) * (b.nrel_room > 0 ? 2 * static_cast<size_t>(b.nrel_room) : 1);
}
int launch_ell(int nv, const int* off, const int* col, const double* val, unsigned char* e_len, int* e_col,
               double* e_val, void* stream);
// Reads `bytes` of device memory (an L2 eviction without dirty lines); writes *sink only in theory.
int launch_read_all(const void* p, size_t bytes, int* sink, void* stream);
// y = M^-1 S x over the padded rows (DevMesh::e_*), CSR for longer rows; the same sums as launch_spmv.
int launch_spmv_ell(int nv, const unsigned char* e_len, const int* e_col, const double* e_val, const int* off,
                    const int* col, const double* val, const double* mass, const double* x, double* y, void* stream);
int launch_spmv(int nv, const int* off, const int* col, const double* val, const double* mass,
                const double* x, double* y, void* stream);

// Field edit / query helpers (fieldops.cu).
int launch_init_field(const DevField& f, const DevWork& w, int nv, const int* seeds, int nseeds,
                      void* stream);
// Queues verts and their stiffness rows into region[slot] with `stamp`.
int launch_mark_region(const DevMesh& m, const DevWork& w, const int* verts, int n, long long stamp,
                       int slot, void* stream);
int launch_mark_all_support(const DevMesh& m, const DevField& f, const DevWork& w, long long stamp,
                            int slot, void* stream);
// The band list ilist[slot] rebuilt from the interest flags (order free).
int launch_rebuild_list(const DevField& f, const DevWork& w, int nv, int slot, void* stream);
int launch_pull_layer(const DevField& f, int nv, int layer, int* out_v, double* out_x, int* out_n,
                      void* stream);
int launch_relabel(const DevField& f, const DevWork& w, const int* verts, const int* newlayer, int n,
                   int oldlayer, void* stream);
int launch_merge(const DevField& f, const DevWork& w, int nv, const int* group, int ngroup, int result,
                 int* touched, int* ntouched, void* stream);
int launch_covered(const DevField& f, int nv, double threshold, int* out_v, int* out_n, void* stream);
int launch_crossings(const DevMesh& m, const DevField& f, int layer, double level, int* out_e,
                     double* out_t, double* out_ba, double* out_bb, int* out_n, void* stream);
int launch_finished(const DevMesh& m, const DevField& f, int layer, double prune, int* out_flag,
                    void* stream);
int launch_field_hash(const DevField& f, int nv, unsigned long long* out, void* stream);
int launch_normalize_all(const DevField& f, const DevWork& w, int nv, double prune, void* stream);
int launch_dense_row(const DevField& f, int nv, int layer, double* out, void* stream);
int launch_base_one_count(const DevField& f, int nv, int* out, void* stream);

}  // namespace dtb
