// Layer-field edits and queries used at topology events and by the one-shot
// API (reference: layer_field.hpp split_layer:155, merge_layers:197,
// covered_set:238, dense_row:256, normalize_columns:143; isoline.hpp
// edge_crossings:30; diffusion.hpp finished():795).  Dense passes over the
// column storage; they run only at events, never inside the step loop.
// Between engine launches both copies of the field (DevField::b) are
// identical: queries read b[0], edits write b[0] and mirror the column to b[1].
#include <cuda_runtime.h>

#include "kernels.h"

namespace dtb {

namespace {

constexpr int T = 256;
inline int nblk(long long n) { return static_cast<int>((n + T - 1) / T); }

__device__ __forceinline__ double value_of(const FieldBuf& F, int v, int layer) {
  const int c = F.cnt[v];
  const size_t b = static_cast<size_t>(v) * kSlots;
  for (int j = 0; j < c; ++j) {
    const int l = F.lay[b + j];
    if (l == layer) return F.val[b + j];
    if (l > layer) break;
  }
  return 0.0;
}

// Copies column v (entries, count, interest, band index) from b[0] to b[1].
__device__ __forceinline__ void mirror_col(const DevField& F, int v) {
  const FieldBuf &A = F.b[0], &B = F.b[1];
  const int c = A.cnt[v];
  const size_t b = static_cast<size_t>(v) * kSlots;
  for (int j = 0; j < c; ++j) {
    B.lay[b + j] = A.lay[b + j];
    B.val[b + j] = A.val[b + j];
  }
  B.cnt[v] = static_cast<unsigned char>(c);
  B.interest[v] = A.interest[v];
  B.binfo[v] = A.binfo[v];
}

// Recomputes the interest flag and band index of an edited column of b[0].
// (The band list is rebuilt from the flags before the next engine launch.)
__device__ __forceinline__ void refresh_interest(const FieldBuf& F, const DevWork& W, int v) {
  const int c = F.cnt[v];
  bool inter = false;
  for (int j = 0; j < c; ++j) {
    const double x = F.val[static_cast<size_t>(v) * kSlots + j];
    inter |= (x > 0.0 && x < 1.0);
  }
  F.interest[v] = inter ? 1 : 0;
  F.binfo[v] = inter ? make_binfo(F.lay + static_cast<size_t>(v) * kSlots, F.val + static_cast<size_t>(v) * kSlots, c,
                                  W.band_lo, W.sat)
                     : make_uint4(0, 0, 0, 0);
}

__global__ void k_init(DevField F, DevWork W, int nv) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  // Whole 32-byte sectors (slots 0..15 of the layer ids, 0..3 of the values):
  // a partial sector write costs the memory system a read to merge it.
  for (int q = 0; q < 2; ++q) {
    F.b[q].cnt[v] = 1;
    uint4* l = reinterpret_cast<uint4*>(F.b[q].lay + static_cast<size_t>(v) * kSlots);
    l[0] = make_uint4(0, 0, 0, 0);
    l[1] = make_uint4(0, 0, 0, 0);
    double4* x = reinterpret_cast<double4*>(F.b[q].val + static_cast<size_t>(v) * kSlots);
    x[0] = make_double4(1.0, 0.0, 0.0, 0.0);
    F.b[q].interest[v] = 0;
    F.b[q].binfo[v] = make_uint4(0, 0, 0, 0);
  }
  W.stamp[v] = -1;
}

__global__ void k_seed(DevField F, const int* seeds, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  F.b[0].lay[static_cast<size_t>(seeds[i]) * kSlots] = 1;
  F.b[1].lay[static_cast<size_t>(seeds[i]) * kSlots] = 1;
}

__device__ __forceinline__ void queue(const DevWork& W, int u, int stamp, int slot) {
  if (atomicExch(W.stamp + u, stamp) != stamp) {
    const int pos = atomicAdd(&W.ctl->rcount[slot], 1);
    W.region[slot][pos] = u;
  }
}

__global__ void k_mark(DevMesh M, DevWork W, const int* verts, int n, int stamp, int slot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int v = verts[i];
  queue(W, v, stamp, slot);
  for (int k = M.s_off[v]; k < M.s_off[v + 1]; ++k) queue(W, M.s_col[k], stamp, slot);
}

__global__ void k_mark_support(DevMesh M, DevField Fd, DevWork W, int stamp, int slot) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= M.nv) return;
  const int c = F.cnt[v];
  bool any = false;
  for (int j = 0; j < c; ++j) {
    const int l = F.lay[static_cast<size_t>(v) * kSlots + j];
    if (l == 0 || W.active[l]) any = true;
  }
  if (!any) return;
  queue(W, v, stamp, slot);
  for (int k = M.s_off[v]; k < M.s_off[v + 1]; ++k) queue(W, M.s_col[k], stamp, slot);
}

// Band list of the next engine launch: every vertex whose column holds a
// value strictly inside (0, 1), by warp-aggregated appends.
__global__ void k_rebuild_list(DevField Fd, DevWork W, int nv, int slot) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = v < nv && Fd.b[0].interest[v];
  const unsigned m = __ballot_sync(0xffffffffu, in);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&W.ctl->ilcount[slot], __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (in) W.ilist[slot][base + __popc(m & ((1u << lane) - 1u))] = v;
}

__global__ void k_pull(DevField Fd, int nv, int layer, int* out_v, double* out_x, int* out_n) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int c = F.cnt[v];
  const size_t b = static_cast<size_t>(v) * kSlots;
  for (int j = 0; j < c; ++j) {
    const int l = F.lay[b + j];
    if (l == layer) {
      const int pos = atomicAdd(out_n, 1);
      out_v[pos] = v;
      out_x[pos] = F.val[b + j];
      return;
    }
    if (l > layer) return;
  }
}

// Moves the value of `oldlayer` at each listed vertex to its new layer id
// (split_layer: row ownership changes, values do not).
__global__ void k_relabel(DevField Fd, DevWork W, const int* verts, const int* newlayer, int n, int oldlayer) {
  const FieldBuf& F = Fd.b[0];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int v = verts[i];
  const size_t b = static_cast<size_t>(v) * kSlots;
  int c = F.cnt[v];
  int j = 0;
  while (j < c && F.lay[b + j] != oldlayer) ++j;
  if (j == c) return;
  const double x = F.val[b + j];
  for (int q = j; q + 1 < c; ++q) {
    F.lay[b + q] = F.lay[b + q + 1];
    F.val[b + q] = F.val[b + q + 1];
  }
  --c;
  const int nl = newlayer[i];
  int p = c;
  while (p > 0 && F.lay[b + p - 1] > nl) {
    F.lay[b + p] = F.lay[b + p - 1];
    F.val[b + p] = F.val[b + p - 1];
    --p;
  }
  F.lay[b + p] = static_cast<unsigned short>(nl);
  F.val[b + p] = x;
  F.cnt[v] = static_cast<unsigned char>(c + 1);
  if (F.interest[v]) F.binfo[v] = make_binfo(F.lay + b, F.val + b, c + 1, W.band_lo, W.sat);
  mirror_col(Fd, v);
}

// merge_layers: per vertex, the group's values summed in ascending layer
// order from 0.0, clamped by min(., 1), stored under the new id.
__global__ void k_merge(DevField Fd, DevWork W, int nv, const int* group, int ngroup, int result, int* touched,
                        int* ntouched) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const size_t b = static_cast<size_t>(v) * kSlots;
  const int c = F.cnt[v];
  double acc = 0.0;
  bool any = false;
  int out = 0;
  for (int j = 0; j < c; ++j) {
    const int l = F.lay[b + j];
    bool in = false;
    for (int g = 0; g < ngroup; ++g) in |= (group[g] == l);
    if (in) {
      acc = acc + F.val[b + j];
      any = true;
    } else {
      F.lay[b + out] = F.lay[b + j];
      F.val[b + out] = F.val[b + j];
      ++out;
    }
  }
  if (!any) return;
  const double clamped = 1.0 < acc ? 1.0 : acc;
  int p = out;
  while (p > 0 && F.lay[b + p - 1] > result) {
    F.lay[b + p] = F.lay[b + p - 1];
    F.val[b + p] = F.val[b + p - 1];
    --p;
  }
  F.lay[b + p] = static_cast<unsigned short>(result);
  F.val[b + p] = clamped;
  F.cnt[v] = static_cast<unsigned char>(out + 1);
  refresh_interest(F, W, v);
  mirror_col(Fd, v);
  touched[atomicAdd(ntouched, 1)] = v;
}

__global__ void k_covered(DevField Fd, int nv, double threshold, int* out_v, int* out_n) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double b = (F.cnt[v] > 0 && F.lay[static_cast<size_t>(v) * kSlots] == 0) ? F.val[static_cast<size_t>(v) * kSlots]
                                                                                  : 0.0;
  if (1.0 - b >= threshold) out_v[atomicAdd(out_n, 1)] = v;
}

__device__ __forceinline__ double signed_value(double value, double level) {
  double s = value - level;
  if (s == 0.0) s = 1e-12 * (1.0 + fabs(level));
  return s;
}

__global__ void k_crossings(DevMesh M, DevField Fd, int layer, double level, int* out_e, double* out_t, double* out_ba,
                            double* out_bb, int* out_n) {
  const FieldBuf& F = Fd.b[0];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M.ne) return;
  const int a = M.edges[2 * e], b = M.edges[2 * e + 1];
  const double sa = signed_value(value_of(F, a, layer), level);
  const double sb = signed_value(value_of(F, b, layer), level);
  if (sa * sb >= 0) return;
  const int pos = atomicAdd(out_n, 1);
  out_e[pos] = e;
  out_t[pos] = sa / (sa - sb);
  out_ba[pos] = value_of(F, a, 0);
  out_bb[pos] = value_of(F, b, 0);
}

// finished() (diffusion.hpp:795) neighbour test: clears *flag if any mesh
// neighbour of the layer's support still holds base mass above the prune
// epsilon.
__global__ void k_finished(DevMesh M, DevField Fd, int layer, double prune, int* flag) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= M.nv) return;
  if (value_of(F, v, layer) == 0.0) return;
  for (int k = M.n_off[v]; k < M.n_off[v + 1]; ++k)
    if (value_of(F, M.n_col[k], 0) > prune) {
      *flag = 0;
      return;
    }
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_hash(DevField Fd, int nv, unsigned long long* out) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long h = 0;
  if (v < nv) {
    const int c = F.cnt[v];
    for (int j = 0; j < c; ++j) {
      const unsigned long long l = F.lay[static_cast<size_t>(v) * kSlots + j];
      const double x = F.val[static_cast<size_t>(v) * kSlots + j];
      h += splitmix64(splitmix64((l << 40) ^ static_cast<unsigned long long>(v)) ^
                      static_cast<unsigned long long>(__double_as_longlong(x)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(out, h);
}

__global__ void k_normalize(DevField Fd, DevWork W, int nv, double prune) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const size_t b = static_cast<size_t>(v) * kSlots;
  const int c = F.cnt[v];
  double s = 0.0;
  for (int j = 0; j < c; ++j) s = s + F.val[b + j];
  if (s <= 0.0) {
    atomicMax(&W.ctl->error, static_cast<int>(kDevZeroColumn));
    return;
  }
  if (fabs(s - 1.0) < 1e-15) return;
  int out = 0;
  for (int j = 0; j < c; ++j) {
    double q = F.val[b + j] / s;
    if (q > 1.0) q = 1.0;
    if (q < prune) continue;
    F.lay[b + out] = F.lay[b + j];
    F.val[b + out] = q;
    ++out;
  }
  F.cnt[v] = static_cast<unsigned char>(out);
  refresh_interest(F, W, v);
  mirror_col(Fd, v);
}

__global__ void k_dense_row(DevField Fd, int nv, int layer, double* out) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  out[v] = value_of(F, v, layer);
}

__global__ void k_base_one(DevField Fd, int nv, int* out) {
  const FieldBuf& F = Fd.b[0];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  bool one = false;
  if (v < nv) one = value_of(F, v, 0) == 1.0;
  const unsigned m = __ballot_sync(0xffffffffu, one);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, __popc(m));
}

}  // namespace

#define DTB_RET \
  note_launch();  \
  return static_cast<int>(cudaGetLastError())

int launch_init_field(const DevField& f, const DevWork& w, int nv, const int* seeds, int nseeds, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_init<<<nblk(nv), T, 0, s>>>(f, w, nv);
  if (nseeds) {
    k_seed<<<nblk(nseeds), T, 0, s>>>(f, seeds, nseeds);
    note_launch();
  }
  DTB_RET;
}
int launch_mark_region(const DevMesh& m, const DevWork& w, const int* verts, int n, long long stamp, int slot,
                       void* stream) {
  if (n <= 0) return 0;
  k_mark<<<nblk(n), T, 0, static_cast<cudaStream_t>(stream)>>>(m, w, verts, n, static_cast<int>(stamp), slot);
  DTB_RET;
}
int launch_mark_all_support(const DevMesh& m, const DevField& f, const DevWork& w, long long stamp, int slot,
                            void* stream) {
  k_mark_support<<<nblk(m.nv), T, 0, static_cast<cudaStream_t>(stream)>>>(m, f, w, static_cast<int>(stamp), slot);
  DTB_RET;
}
int launch_rebuild_list(const DevField& f, const DevWork& w, int nv, int slot, void* stream) {
  k_rebuild_list<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, w, nv, slot);
  DTB_RET;
}
int launch_pull_layer(const DevField& f, int nv, int layer, int* out_v, double* out_x, int* out_n, void* stream) {
  k_pull<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, nv, layer, out_v, out_x, out_n);
  DTB_RET;
}
int launch_relabel(const DevField& f, const DevWork& w, const int* verts, const int* newlayer, int n, int oldlayer,
                   void* stream) {
  if (n <= 0) return 0;
  k_relabel<<<nblk(n), T, 0, static_cast<cudaStream_t>(stream)>>>(f, w, verts, newlayer, n, oldlayer);
  DTB_RET;
}
int launch_merge(const DevField& f, const DevWork& w, int nv, const int* group, int ngroup, int result, int* touched,
                 int* ntouched, void* stream) {
  k_merge<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, w, nv, group, ngroup, result, touched, ntouched);
  DTB_RET;
}
int launch_covered(const DevField& f, int nv, double threshold, int* out_v, int* out_n, void* stream) {
  k_covered<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, nv, threshold, out_v, out_n);
  DTB_RET;
}
int launch_crossings(const DevMesh& m, const DevField& f, int layer, double level, int* out_e, double* out_t,
                     double* out_ba, double* out_bb, int* out_n, void* stream) {
  k_crossings<<<nblk(m.ne), T, 0, static_cast<cudaStream_t>(stream)>>>(m, f, layer, level, out_e, out_t, out_ba,
                                                                       out_bb, out_n);
  DTB_RET;
}
int launch_finished(const DevMesh& m, const DevField& f, int layer, double prune, int* out_flag, void* stream) {
  k_finished<<<nblk(m.nv), T, 0, static_cast<cudaStream_t>(stream)>>>(m, f, layer, prune, out_flag);
  DTB_RET;
}
int launch_field_hash(const DevField& f, int nv, unsigned long long* out, void* stream) {
  k_hash<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, nv, out);
  DTB_RET;
}
int launch_normalize_all(const DevField& f, const DevWork& w, int nv, double prune, void* stream) {
  k_normalize<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, w, nv, prune);
  DTB_RET;
}
int launch_dense_row(const DevField& f, int nv, int layer, double* out, void* stream) {
  k_dense_row<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, nv, layer, out);
  DTB_RET;
}
int launch_base_one_count(const DevField& f, int nv, int* out, void* stream) {
  k_base_one<<<nblk(nv), T, 0, static_cast<cudaStream_t>(stream)>>>(f, nv, out);
  DTB_RET;
}

}  // namespace dtb
