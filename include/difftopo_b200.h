/* difftopo_b200.h -- C ABI of the B200 diffusion-front engine.
 *
 * Drop-in boundary for the reference's C++ API (proj/include/difftopo/ headers):
 * every entry point below names the reference interface it replaces.  Plain
 * pointers and sizes only; all functions return 0 on success or one of the
 * DTB_E* codes (the reference's exception classes, errors.hpp:8-33), with a
 * message available from dtb_last_error().  Variable-length outputs use the
 * two-call pattern: query the size, then pass a buffer of that size.
 *
 * Device memory, streams and kernels are internal; the library needs an
 * sm_100a GPU and fails with DTB_ECUDA when none is present (there is no CPU
 * fallback).
 */
#ifndef DIFFTOPO_B200_H
#define DIFFTOPO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (errors.hpp). */
enum {
  DTB_OK = 0,
  DTB_EPARSE = 1,          /* ParseError */
  DTB_ETOPOLOGY = 2,       /* TopologyError */
  DTB_EDEGENERACY = 3,     /* DegeneracyError */
  DTB_EINVALID = 4,        /* InvalidParameter */
  DTB_EDIMENSION = 5,      /* DimensionMismatch */
  DTB_EEMPTYSEED = 6,      /* EmptySeed */
  DTB_EZEROCOLUMN = 7,     /* ZeroColumn */
  DTB_EINVALIDSPLIT = 8,   /* InvalidSplit */
  DTB_EINVALIDMERGE = 9,   /* InvalidMerge */
  DTB_EBLOWUP = 10,        /* NumericalBlowup */
  DTB_EMAXSTEPS = 11,      /* MaxStepsExceeded */
  DTB_EINCONSISTENT = 15,  /* InconsistentLog */
  DTB_ECUDA = 100,         /* no device / CUDA runtime failure */
  DTB_ECAPACITY = 101      /* a fixed device capacity was exceeded */
};

typedef struct dtb_mesh dtb_mesh;           /* TriangleMesh (mesh.hpp:33) + its HBM copy */
typedef struct dtb_laplacian dtb_laplacian; /* LaplacianOperator (operators.hpp:16) */
typedef struct dtb_field dtb_field;         /* LayerField (layer_field.hpp:46) */
typedef struct dtb_result dtb_result;       /* InitialPassResult (diffusion.hpp:110) */

/* DiffusionConfig (diffusion.hpp:33); on_check is replaced by record_hashes. */
typedef struct {
  double dt;                  /* <= 0 selects stable_time_step */
  double band_low_threshold;  /* tau */
  double saturation;
  double collision_threshold; /* kappa */
  int32_t check_interval;
  int32_t record_trails;
  int64_t max_steps;
  double covered_threshold;
  double seed_radius;         /* <= 0: 1.5 * interface length scale */
  int32_t record_hashes;      /* per-check 64-bit field digests (parity tooling) */
  int32_t grid_ctas;          /* CTAs of the persistent step kernel; 0 = one per SM (B200: 148) */
} dtb_config;

/* CoefficientScheme (layer_field.hpp:30). */
typedef struct {
  double gradient_energy, penalty, contact, mobility;
} dtb_coefficients;

void dtb_config_default(dtb_config* cfg);
void dtb_coefficients_default(dtb_coefficients* c);
const char* dtb_last_error(void);
const char* dtb_version(void);
int dtb_device_info(int* device_count, int* sm_count, int* cc_major, int* cc_minor);
/* Library initialisation (no reference counterpart): one small end-to-end call
 * through the device paths, so the context exists and every kernel is loaded
 * before the caller's first timed call.  Optional. */
int dtb_warmup(void);
/* Opt-in (no reference counterpart): asks for `queues` hardware work queues
 * (1..32) in the CUDA context this process has not created yet, by setting
 * CUDA_DEVICE_MAX_CONNECTIONS when the caller left it unset.  Concurrent batch
 * passes each hold a queue for their whole run, so 32 lets 16 run at once.
 * Fails with DTB_EINVAL when a CUDA context may already exist (libcuda is
 * mapped); call it first thing, before any CUDA use.  The library itself never
 * changes the variable. */
int dtb_init_work_queues(int32_t queues);

/* ---- mesh (mesh.hpp, generators.hpp, mesh_io.hpp) ---------------------- */
/* TriangleMesh(vertices, faces) (mesh.hpp:150): validates, orients, indexes. */
int dtb_mesh_from_arrays(const double* xyz, uint32_t nv, const uint32_t* faces, uint32_t nf, dtb_mesh** out);
/* generate_torus / generate_genus_g / ... via a spec string, e.g.
 * "torus:64:32:2:0.5", "genus:8:45", "icosphere:3:2", "plate:8:45:6.0",
 * "gyroid:3:40:0.0:1.0" (generators.hpp). */
int dtb_mesh_generate(const char* spec, dtb_mesh** out);
/* load_mesh (mesh_io.hpp:310); format 0 = by extension, 1 OFF, 2 OBJ, 3 PLY. */
int dtb_mesh_load(const char* path, int32_t format, dtb_mesh** out);
/* save_ply / save_obj (mesh_io.hpp:327, :376) or .dtm by extension. */
int dtb_mesh_save(const dtb_mesh* m, const char* path);
void dtb_mesh_free(dtb_mesh* m);
/* topology_summary (mesh.hpp:134). */
int dtb_mesh_info(const dtb_mesh* m, uint32_t* nv, uint32_t* ne, uint32_t* nf, int64_t* euler, int64_t* genus);
int dtb_mesh_vertices(const dtb_mesh* m, double* xyz);                   /* 3 nv */
int dtb_mesh_faces(const dtb_mesh* m, uint32_t* faces);                  /* 3 nf */
int dtb_mesh_edges(const dtb_mesh* m, uint32_t* ev, uint32_t* ef);       /* 2 ne each */
int dtb_mesh_face_edges(const dtb_mesh* m, uint32_t* fe);                /* 3 nf */
/* CSR adjacency: vertex_neighbors (sorted) and vertex_faces (face order),
   mesh.hpp:57-62.  Offsets have nv+1 entries; v2v has 2 ne, v2f 3 nf. */
int dtb_mesh_adjacency(const dtb_mesh* m, uint32_t* v2v_off, uint32_t* v2v, uint32_t* v2f_off, uint32_t* v2f);
/* seed_region (diffusion.hpp:134); two-call. */
int dtb_seed_region(const dtb_mesh* m, uint32_t seed, double radius, uint32_t* out, uint32_t cap, uint32_t* n);

/* ---- operators (operators.hpp) ------------------------------------------ */
/* assemble_laplacian (operators.hpp:33), on the device. */
int dtb_laplacian_assemble(const dtb_mesh* m, dtb_laplacian** out);
/* A LaplacianOperator supplied as host CSR (e.g. the reference's own). */
int dtb_laplacian_from_csr(const dtb_mesh* m, const int32_t* off, const int32_t* col, const double* val,
                           const double* mass, int64_t nnz, double gershgorin, dtb_laplacian** out);
void dtb_laplacian_free(dtb_laplacian* op);
int dtb_laplacian_info(const dtb_laplacian* op, int64_t* nnz, double* gershgorin);
int dtb_laplacian_csr(const dtb_laplacian* op, int32_t* off, int32_t* col, double* val, double* mass);
/* LaplacianOperator::apply (operators.hpp:27): y = M^-1 S x. */
int dtb_laplacian_apply(const dtb_laplacian* op, const double* x, double* y);
/* Diagnostics (no reference counterpart): a full-mesh sweep of the operator
 * (the padded-row SpMV apply uses), timed on the device after an L2 flush;
 * mean seconds per sweep and algorithmic bytes per sweep. */
int dtb_laplacian_sweep_bench(const dtb_laplacian* op, int32_t reps, double* seconds, double* bytes);
/* stable_time_step (diffusion.hpp:58). */
int dtb_stable_time_step(const dtb_laplacian* op, const dtb_coefficients* c, double* dt);

/* ---- initial pass (diffusion.hpp:861 run_initial_pass) ------------------ */
int dtb_run_initial_pass(const dtb_mesh* m, const dtb_laplacian* op, uint32_t seed_vertex, const dtb_config* cfg,
                         const dtb_coefficients* c, dtb_result** out);
/* Batch of independent initial passes on this GPU (BASELINE configs[4]):
 * item i runs run_initial_pass(meshes[i], ops[i], seeds[i] (0 if seeds is
 * NULL)) exactly as dtb_run_initial_pass would, up to `concurrency` passes at
 * once (<= 0: 16 when CUDA_DEVICE_MAX_CONNECTIONS asks for >= 16 hardware
 * work queues -- see dtb_init_work_queues -- and the host has >= 16 threads,
 * else 8), each a persistent kernel on its own stream over
 * cfg->grid_ctas CTAs (0: SMs / concurrency).  out[i] receives the result
 * (NULL on failure) and rc[i] (optional) its code; the return value is the
 * first failing item's code.  Replaces a caller's loop over
 * Engine::run_initial_pass (diffusion.hpp:530) for independent meshes. */
int dtb_run_initial_pass_batch(const dtb_mesh* const* meshes, const dtb_laplacian* const* ops,
                               const uint32_t* seeds, int32_t n, const dtb_config* cfg, const dtb_coefficients* c,
                               int32_t concurrency, dtb_result** out, int32_t* rc);
void dtb_result_free(dtb_result* r);
/* status = DTB_OK or the error that ended the run (e.g. DTB_EMAXSTEPS); the
 * event log and tracks recorded up to that point stay available. */
int dtb_result_summary(const dtb_result* r, int32_t* status, int64_t* steps, double* dt_used, int64_t* n_events,
                       int64_t* n_tracks, int64_t* n_estimates, int64_t* layer_count);
const char* dtb_result_message(const dtb_result* r);
/* TopologyEvent (diffusion.hpp:92); kind 0 seed, 1 split, 2 merge, 3 vanish. */
int dtb_result_event(const dtb_result* r, int64_t i, int32_t* kind, int64_t* step, double* pos3, uint32_t* n_layers,
                     uint32_t* n_produced, uint32_t* n_estimates, uint32_t* n_covered);
int dtb_result_event_layers(const dtb_result* r, int64_t i, uint32_t* layers, uint32_t* produced);
int dtb_result_event_covered(const dtb_result* r, int64_t i, uint32_t* covered);
/* HandleEstimate (diffusion.hpp:85). */
int dtb_result_estimate(const dtb_result* r, int64_t ev, uint32_t k, uint32_t* layer, uint32_t* n_points,
                        uint32_t* n_snapshot, double* length);
int dtb_result_estimate_points(const dtb_result* r, int64_t ev, uint32_t k, int64_t* edge, double* t, int64_t* face,
                               double* xyz);
int dtb_result_estimate_snapshot(const dtb_result* r, int64_t ev, uint32_t k, uint32_t* v, double* x);
/* LayerTrack (diffusion.hpp:103); -1 for unset ids. */
int dtb_result_track(const dtb_result* r, int64_t i, int64_t* layer, int64_t* created, int64_t* consumed,
                     uint32_t* n_trail);
int dtb_result_track_trail(const dtb_result* r, int64_t i, double* xyz);
/* Final LayerField (InitialPassResult::field). */
int dtb_result_layer(const dtb_result* r, uint32_t layer, int32_t* active, int32_t* cleared, int64_t* parent,
                     int64_t* created_step, uint32_t* n_merge_parents);
int dtb_result_layer_values(const dtb_result* r, uint32_t layer, uint32_t* v, double* x, uint32_t cap, uint32_t* n);
int dtb_result_field_hash(const dtb_result* r, uint64_t* hash);
int dtb_result_hashes(const dtb_result* r, uint64_t* out, int64_t cap, int64_t* n);
int dtb_result_timing(const dtb_result* r, double* t_device, double* t_events, int64_t* launches,
                      int64_t* event_checks, int64_t* kernel_steps);
/* Device work counters (frontier vertices updated, band vertices checked, summed over steps) and the
 * CUDA-event duration of the whole pass on its stream and of its step-kernel launches, in seconds. */
int dtb_result_work(const dtb_result* r, uint64_t* sum_region, uint64_t* sum_interest, double* t_pass_device,
                    double* t_kernel);
/* Diagnostics: nanoseconds per grid barrier of the persistent engine (mode 0) or of
 * cooperative_groups::grid_group::sync (mode 1) with `blocks` CTAs. */
double dtb_bench_barrier(int blocks, int n, int mode);
/* Kernels launched by this library so far (process-wide counter). */
unsigned long long dtb_launch_count(void);
/* Bytes the mesh's device copy occupies (uploaded and device-derived arrays). */
int dtb_mesh_device_bytes(const dtb_mesh* m, uint64_t* bytes);
/* Bytes copied host->device to build the mesh's device copy. */
int dtb_mesh_upload_bytes(const dtb_mesh* m, uint64_t* bytes);
/* build_reeb (SPEC reeb): nodes = events, arcs = layer lifetimes. */
int dtb_result_reeb(const dtb_result* r, int64_t* n_nodes, int64_t* n_arcs, int64_t* cycle_rank);
int dtb_result_reeb_arcs(const dtb_result* r, uint32_t* from, uint32_t* to, uint32_t* layer);

/* ---- layer field (layer_field.hpp, diffusion.hpp one-shot operations) --- */
int dtb_field_init(const dtb_mesh* m, const uint32_t* seeds, uint32_t n, dtb_field** out); /* init_field */
void dtb_field_free(dtb_field* f);
int dtb_field_step(dtb_field* f, const dtb_laplacian* op, const dtb_config* cfg, const dtb_coefficients* c); /* step */
int dtb_field_layer_count(const dtb_field* f, uint32_t* n);
int dtb_field_layer_values(const dtb_field* f, uint32_t layer, uint32_t* v, double* x, uint32_t cap, uint32_t* n);
int dtb_field_hash(const dtb_field* f, uint64_t* hash);
int dtb_field_normalize(dtb_field* f);                                     /* normalize_columns */
int dtb_field_covered_set(const dtb_field* f, double threshold, uint32_t* out, uint32_t cap, uint32_t* n);
/* extract_front (diffusion.hpp:398): per component its triangle and boundary
 * vertex counts plus band length; flattened id arrays via the second call. */
int dtb_field_extract_front(dtb_field* f, uint32_t layer, const dtb_config* cfg, uint32_t* n_components,
                            uint32_t* tri_counts, uint32_t* bnd_counts, double* band_length, uint32_t* tris,
                            uint32_t* bnd);
/* detect_collisions (diffusion.hpp:475): groups flattened, sizes separately. */
int dtb_field_detect_collisions(dtb_field* f, const dtb_config* cfg, uint32_t* flat, uint32_t* sizes,
                                uint32_t cap, uint32_t* n_groups, uint32_t* n_flat);
int dtb_field_split_layer(dtb_field* f, uint32_t layer, const uint32_t* flat, const uint32_t* sizes, uint32_t ncomp,
                          int64_t step, uint32_t* children);
int dtb_field_merge_layers(dtb_field* f, const uint32_t* ids, uint32_t n, int64_t step, uint32_t* result);

/* ---- isolines (isoline.hpp:55) ------------------------------------------ */
/* Loops flattened: counts[i] points per loop (closing point repeated). */
int dtb_extract_isoline(const dtb_mesh* m, const double* values, double level, uint32_t* n_loops, uint32_t* counts,
                        int64_t* edge, double* t, int64_t* face, double* xyz, uint32_t cap);

#ifdef __cplusplus
}
#endif

#endif /* DIFFTOPO_B200_H */
