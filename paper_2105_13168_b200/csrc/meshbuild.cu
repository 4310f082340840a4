// Device-side mesh construction from a triangle soup: validation,
// orientation check, connectivity, outward orientation and the topology
// indices, with the reference's numbering (mesh.hpp:150-324):
//   * edges numbered by first appearance over (face, corner) slots of the
//     final orientation (mesh.hpp:272-293),
//   * vertex->face lists in face order, vertex->vertex lists sorted.
// It covers the common case -- a valid, closed, consistently oriented,
// connected manifold without unused vertices.  Anything else (including every
// error the reference raises) returns 1, and the caller rebuilds on the host
// (csrc/mesh.cpp), which follows the reference's check order and messages.
// Pairing uses a radix sort of the 3F corner slots by their unordered vertex
// pair; the indices use stable radix sorts, so their order is exactly the
// host construction's.
#include <cuda_runtime.h>

#include <cmath>
#include <cub/cub.cuh>
#include <vector>

#include "kernels.h"

namespace dtb {

namespace {

constexpr int kT = 256;
inline int nblk(long long n) { return static_cast<int>((n + kT - 1) / kT); }

enum : int { kBadSoup = 1, kBadPairing = 2, kBadOrientation = 4, kBadUnused = 8, kBadArea = 16 };

struct P3 {
  double x, y, z;
};
__device__ __forceinline__ P3 ld3(const double* xyz, unsigned v) { return {xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]}; }
__device__ __forceinline__ P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot3(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ P3 cross3(P3 a, P3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

__global__ void k_soup_check(const unsigned* soup, int nf, int nv, unsigned char* used, int* bad) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const unsigned a = soup[3 * f], b = soup[3 * f + 1], c = soup[3 * f + 2];
  const unsigned n = static_cast<unsigned>(nv);
  if (a >= n || b >= n || c >= n || a == b || b == c || a == c) {
    atomicOr(bad, kBadSoup);
    return;
  }
  used[a] = 1;
  used[b] = 1;
  used[c] = 1;
}

__global__ void k_unused(const unsigned char* used, int nv, int* bad) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv && !used[v]) atomicOr(bad, kBadUnused);
}

// Slot s = 3f + k is the directed edge corner k -> corner k+1 of input face f.
// Pairing by counting: the slots are bucketed by the lower end of their
// vertex pair (count, scan, scatter); each bucket -- a few dozen slots at
// most -- pairs its slots by the upper end.  Every unordered pair must be
// used by exactly two slots (closed manifold).  Slots of an invalid soup
// (flagged by k_soup_check) are left out.
__device__ __forceinline__ bool slot_ends(const unsigned* soup, int s, unsigned nv, unsigned& lo, unsigned& hi) {
  const int f = s / 3, k = s % 3;
  const unsigned a = soup[3 * f + k], b = soup[3 * f + (k + 1) % 3];
  lo = min(a, b);
  hi = max(a, b);
  return hi < nv;
}
__global__ void k_count_lo(const unsigned* soup, int ns, unsigned nv, int* cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned lo, hi;
  if (s < ns && slot_ends(soup, s, nv, lo, hi)) atomicAdd(cnt + lo, 1);
}
__global__ void k_scatter_lo(const unsigned* soup, int ns, unsigned nv, int* cur, unsigned* rows) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned lo, hi;
  if (s < ns && slot_ends(soup, s, nv, lo, hi)) rows[atomicAdd(cur + lo, 1)] = static_cast<unsigned>(s);
}
__global__ void k_pair_rows(const unsigned* soup, const int* off, const unsigned* rows, int nv, unsigned* partner,
                            int* bad) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int o0 = off[v], n = off[v + 1] - o0;
  constexpr int kCap = 64;
  unsigned hs[kCap];
  unsigned lo, hi;
  if (n <= kCap)
    for (int i = 0; i < n; ++i) {
      slot_ends(soup, static_cast<int>(rows[o0 + i]), static_cast<unsigned>(nv), lo, hi);
      hs[i] = hi;
    }
  for (int i = 0; i < n; ++i) {
    unsigned hi_i;
    if (n <= kCap) hi_i = hs[i];
    else slot_ends(soup, static_cast<int>(rows[o0 + i]), static_cast<unsigned>(nv), lo, hi_i);
    int m = 0, mate = -1;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      unsigned hi_j;
      if (n <= kCap) hi_j = hs[j];
      else slot_ends(soup, static_cast<int>(rows[o0 + j]), static_cast<unsigned>(nv), lo, hi_j);
      if (hi_j == hi_i) {
        ++m;
        mate = j;
      }
    }
    if (m != 1) {
      atomicOr(bad, kBadPairing);
      return;
    }
    partner[rows[o0 + i]] = rows[o0 + mate];
  }
}


// Consistent orientation: the partner slot traverses the edge the other way.
__global__ void k_orient_check(const unsigned* soup, const unsigned* partner, int ns, int* bad) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const unsigned a = soup[s];  // corner s%3 of face s/3
  if (soup[partner[s]] == a) atomicOr(bad, kBadOrientation);
}

// Connectivity of the face graph: lock-free union-find, hooking the larger
// root under the smaller.
__device__ __forceinline__ unsigned froot(unsigned* p, unsigned x) {
  while (true) {
    const unsigned q = __ldcg(p + x);
    if (q == x) return x;
    const unsigned r = __ldcg(p + q);
    if (r != q) p[x] = r;
    x = q;
  }
}
__global__ void k_face_init(unsigned* p, int nf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) p[f] = static_cast<unsigned>(f);
}
// Randomised linking (hash keys) keeps the trees shallow; linking by index
// builds long chains on meshes whose faces are numbered along strips.
__device__ __forceinline__ unsigned fkey(unsigned x) {
  x *= 0x9E3779B1u;
  x ^= x >> 15;
  x *= 0x85EBCA77u;
  return x ^ (x >> 13);
}
__device__ __forceinline__ void funite(unsigned* p, unsigned a, unsigned b) {
  while (true) {
    a = froot(p, a);
    b = froot(p, b);
    if (a == b) return;
    const unsigned ka = fkey(a), kb = fkey(b);
    if (ka < kb || (ka == kb && a < b)) {  // hook the smaller key under the larger
      const unsigned t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(p + b, b, a) == b) return;
  }
}
// Afforest-style connectivity: link every face to its partner across edge
// k (k = 0, then 1) with the trees flattened after each round; most faces
// then share one component, and the last pass unites all three edges only
// for faces outside the component of face 0.  Skipping an edge whose two
// faces are both already in that component loses nothing, so the final
// forest has exactly the components of the face graph.
__global__ void k_face_link(const unsigned* partner, int nf, unsigned* p, int k) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  funite(p, static_cast<unsigned>(f), partner[3 * f + k] / 3);
}
__global__ void k_face_flatten(unsigned* p, int nf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) p[f] = froot(p, static_cast<unsigned>(f));
}
__global__ void k_face_link_rest(const unsigned* partner, int nf, unsigned* p) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const unsigned c = froot(p, 0u);
  if (froot(p, static_cast<unsigned>(f)) == c) return;
  for (int k = 0; k < 3; ++k) funite(p, static_cast<unsigned>(f), partner[3 * f + k] / 3);
}
__global__ void k_face_roots(const unsigned* p, int nf, int* nroots) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf && p[f] == static_cast<unsigned>(f)) atomicAdd(nroots, 1);
}

// Per-block partials: bbox min/max, max |coordinate|, and the signed-volume
// terms dot(p0, cross(p1, p2)) / 6 (the host's per-face expression) with
// their absolute values.  Reduced deterministically by k_finish.
struct Red {
  double lo[3], hi[3], maxabs, vol, absvol;
};
__device__ __forceinline__ void red_merge(Red& a, const Red& b) {
  for (int c = 0; c < 3; ++c) {
    a.lo[c] = fmin(a.lo[c], b.lo[c]);
    a.hi[c] = fmax(a.hi[c], b.hi[c]);
  }
  a.maxabs = fmax(a.maxabs, b.maxabs);
  a.vol += b.vol;
  a.absvol += b.absvol;
}
__device__ __forceinline__ Red red_identity() {
  Red r;
  for (int c = 0; c < 3; ++c) {
    r.lo[c] = 1e300;  // the host bbox's initial values (mesh.cpp bbox_diagonal)
    r.hi[c] = -1e300;
  }
  r.maxabs = 0.0;
  r.vol = 0.0;
  r.absvol = 0.0;
  return r;
}
__device__ Red block_reduce(Red r) {
  __shared__ Red sh[kT];
  sh[threadIdx.x] = r;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red_merge(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  return sh[0];
}
__global__ void k_geometry(const double* xyz, int nv, const unsigned* soup, int nf, double* term, Red* part,
                           int* bad) {
  Red r = red_identity();
  const int stride = gridDim.x * blockDim.x;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const P3 p = ld3(xyz, v);
    const double c[3] = {p.x, p.y, p.z};
    if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z)) atomicOr(bad, kBadSoup);
    for (int k = 0; k < 3; ++k) {
      r.lo[k] = fmin(r.lo[k], c[k]);
      r.hi[k] = fmax(r.hi[k], c[k]);
      r.maxabs = fmax(r.maxabs, fabs(c[k]));
    }
  }
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += stride) {
    const P3 p0 = ld3(xyz, soup[3 * f]), p1 = ld3(xyz, soup[3 * f + 1]), p2 = ld3(xyz, soup[3 * f + 2]);
    const double t = dot3(p0, cross3(p1, p2)) / 6.0;
    term[f] = t;
    r.vol += t;
    r.absvol += fabs(t);
  }
  r = block_reduce(r);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}
__global__ void k_finish(const Red* part, int n, Red* out) {
  Red r = red_identity();
  for (int i = threadIdx.x; i < n; i += blockDim.x) red_merge(r, part[i]);
  r = block_reduce(r);
  if (threadIdx.x == 0) *out = r;
}

// Face area (host face_area: 0.5 * |cross(p1 - p0, p2 - p0)|) below tol.
__global__ void k_small_area(const double* xyz, const unsigned* soup, int nf, double tol, int* bad) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const P3 p0 = ld3(xyz, soup[3 * f]), p1 = ld3(xyz, soup[3 * f + 1]), p2 = ld3(xyz, soup[3 * f + 2]);
  const P3 c = cross3(sub(p1, p0), sub(p2, p0));
  if (0.5 * sqrt(dot3(c, c)) < tol) atomicOr(bad, kBadArea);
}

// Final orientation: a global flip swaps corners 1 and 2 of every face, which
// maps final corner pair k to input slot 2 - k.
__global__ void k_orient_faces(const unsigned* soup, int nf, int flipped, unsigned* faces) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const unsigned a = soup[3 * f], b = soup[3 * f + 1], c = soup[3 * f + 2];
  faces[3 * f] = a;
  faces[3 * f + 1] = flipped ? c : b;
  faces[3 * f + 2] = flipped ? b : c;
}
__global__ void k_final_partner(const unsigned* partner, int ns, int flipped, unsigned* pf, int* open) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const unsigned f = static_cast<unsigned>(s) / 3, k = static_cast<unsigned>(s) % 3;
  const unsigned po = partner[3 * f + (flipped ? 2 - k : k)];
  const unsigned g = po / 3, kg = po % 3;
  const unsigned q = 3 * g + (flipped ? 2 - kg : kg);
  pf[s] = q;
  open[s] = q > static_cast<unsigned>(s) ? 1 : 0;
}
// A slot opens its edge iff its partner comes later; edge id = rank of the
// opening slot (exclusive scan of open).
__global__ void k_edges(const unsigned* faces, const unsigned* pf, const int* eid, int ns, unsigned* edges,
                        unsigned* ef, unsigned* fe) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const unsigned q = pf[s];
  if (q <= static_cast<unsigned>(s)) return;
  const int e = eid[s];
  const int f = s / 3, k = s % 3;
  const unsigned a = faces[3 * f + k], b = faces[3 * f + (k + 1) % 3];
  edges[2 * e] = min(a, b);
  edges[2 * e + 1] = max(a, b);
  ef[2 * e] = static_cast<unsigned>(f);
  ef[2 * e + 1] = q / 3;
  fe[s] = static_cast<unsigned>(e);
  fe[q] = static_cast<unsigned>(e);
}
// Adjacency rows by counting: per-vertex counts, an exclusive scan into the
// row offsets, an atomic scatter into the rows, then each row sorted on its
// own (rows hold at most a few dozen entries).  Same rows as a stable sort of
// the (vertex, face) corners / (vertex, other end) half-edges.
__global__ void k_count_corners(const unsigned* faces, int ns, int* cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ns) atomicAdd(cnt + faces[s], 1);
}
__global__ void k_scatter_corners(const unsigned* faces, int ns, int* cur, int* v2f) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ns) v2f[atomicAdd(cur + faces[s], 1)] = s / 3;
}
__global__ void k_count_half(const unsigned* edges, int nh, int* cnt) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < nh) atomicAdd(cnt + edges[h], 1);
}
__global__ void k_scatter_half(const unsigned* edges, int nh, int* cur, int* v2v) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < nh) v2v[atomicAdd(cur + edges[h], 1)] = static_cast<int>(edges[h ^ 1]);
}
__global__ void k_sort_rows(const int* off, int nv, int* col) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int* r = col + off[v];
  const int n = off[v + 1] - off[v];
  for (int i = 1; i < n; ++i) {  // insertion sort of a short row
    const int x = r[i];
    int j = i - 1;
    while (j >= 0 && r[j] > x) {
      r[j + 1] = r[j];
      --j;
    }
    r[j + 1] = x;
  }
}


// Scratch from the engine's caching allocator (engine.cpp dev_alloc); every
// exit of build_mesh synchronizes the stream first, so blocks go back to the
// cache idle.
struct Scratch {
  cudaStream_t s;
  std::vector<std::pair<void*, size_t>> held;
  ~Scratch() {
    for (auto& h : held) dev_free(h.first, h.second);
  }
  template <class T>
  T* get(size_t n) {
    const size_t bytes = sizeof(T) * (n ? n : 1);
    void* p = dev_alloc(bytes);
    held.emplace_back(p, bytes);
    return static_cast<T*>(p);
  }
};

}  // namespace

int build_mesh(MeshBuild& b, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nv = b.nv, nf = b.nf, ns = 3 * nf;
  if (nf < 4 || nf % 2) return 1;  // tiny or odd: the host decides (and names the error)
  const int ne = ns / 2;
  Scratch sc{s, {}};
  int* bad = sc.get<int>(2);
  unsigned char* used = sc.get<unsigned char>(nv);
  unsigned long long* key1 = sc.get<unsigned long long>(ns);
  unsigned* val0 = sc.get<unsigned>(ns);
  unsigned* val1 = sc.get<unsigned>(ns);
  unsigned* partner = sc.get<unsigned>(ns);
  unsigned* fpar = sc.get<unsigned>(nf);
  double* term = sc.get<double>(nf);
  const int gblocks = 148 * 4;
  Red* part = sc.get<Red>(gblocks);
  Red* red = sc.get<Red>(1);
  if (!bad || !used || !key1 || !val0 || !val1 || !partner || !fpar || !term || !part || !red)
    return static_cast<int>(cudaErrorMemoryAllocation);
  cudaMemsetAsync(bad, 0, 2 * sizeof(int), s);
  cudaMemsetAsync(used, 0, nv, s);
  k_soup_check<<<nblk(nf), kT, 0, s>>>(b.soup, nf, nv, used, bad);
  k_unused<<<nblk(nv), kT, 0, s>>>(used, nv, bad);
  // Pair the slots by their unordered vertex pair.
  size_t tmp_bytes = 0;
  {
    int* cnt = sc.get<int>(nv + 1);
    int* off = sc.get<int>(nv + 1);
    unsigned* rows = val0;
    if (!cnt || !off) return static_cast<int>(cudaErrorMemoryAllocation);
    cudaMemsetAsync(cnt, 0, sizeof(int) * (nv + 1), s);
    k_count_lo<<<nblk(ns), kT, 0, s>>>(b.soup, ns, static_cast<unsigned>(nv), cnt);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, nv + 1, s);
    void* tmp = sc.get<char>(tmp_bytes);
    if (!tmp) return static_cast<int>(cudaErrorMemoryAllocation);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, nv + 1, s);
    cudaMemcpyAsync(cnt, off, sizeof(int) * nv, cudaMemcpyDeviceToDevice, s);  // bucket cursors
    k_scatter_lo<<<nblk(ns), kT, 0, s>>>(b.soup, ns, static_cast<unsigned>(nv), cnt, rows);
    cudaMemsetAsync(partner, 0, sizeof(unsigned) * ns, s);
    k_pair_rows<<<nblk(nv), kT, 0, s>>>(b.soup, off, rows, nv, partner, bad);
  }
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return static_cast<int>(e);
  if (hbad) return 1;
  k_orient_check<<<nblk(ns), kT, 0, s>>>(b.soup, partner, ns, bad);
  k_face_init<<<nblk(nf), kT, 0, s>>>(fpar, nf);
  for (int e = 0; e < 2; ++e) {
    k_face_link<<<nblk(nf), kT, 0, s>>>(partner, nf, fpar, e);
    k_face_flatten<<<nblk(nf), kT, 0, s>>>(fpar, nf);
  }
  k_face_link_rest<<<nblk(nf), kT, 0, s>>>(partner, nf, fpar);
  k_face_roots<<<nblk(nf), kT, 0, s>>>(fpar, nf, bad + 1);
  if (b.xyz_ready) cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(b.xyz_ready), 0);  // positions uploaded
  k_geometry<<<gblocks, kT, 0, s>>>(b.xyz, nv, b.soup, nf, term, part, bad);
  k_finish<<<1, kT, 0, s>>>(part, gblocks, red);
  int hb[2] = {0, 0};
  Red hr{};
  cudaMemcpyAsync(hb, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hr, red, sizeof(Red), cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return static_cast<int>(e);
  if (hb[0] || hb[1] != 1) return 1;
  // Outward orientation: the host sums the volume terms sequentially in face
  // order.  Any summation order is within (n-1) u sum|t| of the exact sum, so
  // a parallel sum decides the sign unless it lies within twice that bound;
  // then the terms are summed in face order on the host.
  double vol = hr.vol;
  const double bound = 2.0 * static_cast<double>(nf) * 0x1p-53 * hr.absvol;
  if (!(std::fabs(vol) > bound)) {
    std::vector<double> t(nf);
    cudaMemcpyAsync(t.data(), term, sizeof(double) * nf, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return static_cast<int>(e);
    vol = 0;
    for (double x : t) vol += x;
  }
  b.flipped = vol < 0 ? 1 : 0;
  b.maxabs = hr.maxabs;
  const double dx = hr.hi[0] - hr.lo[0], dy = hr.hi[1] - hr.lo[1], dz = hr.hi[2] - hr.lo[2];
  const double diag = std::sqrt(dx * dx + dy * dy + dz * dz);
  k_small_area<<<nblk(nf), kT, 0, s>>>(b.xyz, b.soup, nf, 1e-12 * diag * diag, bad);
  // Indices of the final orientation.
  int* open = reinterpret_cast<int*>(val0);  // val buffers are free again
  int* eid = reinterpret_cast<int*>(val1);
  unsigned* pf = reinterpret_cast<unsigned*>(key1);  // ns u32 fit in key1 (free after pairing)
  k_orient_faces<<<nblk(nf), kT, 0, s>>>(b.soup, nf, b.flipped, b.faces);
  k_final_partner<<<nblk(ns), kT, 0, s>>>(partner, ns, b.flipped, pf, open);
  tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, open, eid, ns, s);
  void* tmp2 = sc.get<char>(tmp_bytes);
  if (!tmp2) return static_cast<int>(cudaErrorMemoryAllocation);
  cub::DeviceScan::ExclusiveSum(tmp2, tmp_bytes, open, eid, ns, s);
  k_edges<<<nblk(ns), kT, 0, s>>>(b.faces, pf, eid, ns, b.edges, b.edge_faces, b.face_edges);
  // vertex -> faces (face order) and vertex -> vertices (ascending): rows by
  // counting, then each row sorted (k_sort_rows).
  {
    int* cnt = sc.get<int>(nv + 1);
    if (!cnt) return static_cast<int>(cudaErrorMemoryAllocation);
    const int nh = 2 * ne;
    for (int pass = 0; pass < 2; ++pass) {
      const int n = pass == 0 ? ns : nh;
      int* off = pass == 0 ? b.v2f_off : b.v2v_off;
      int* col = pass == 0 ? b.v2f : b.v2v;
      cudaMemsetAsync(cnt, 0, sizeof(int) * (nv + 1), s);
      if (pass == 0) k_count_corners<<<nblk(n), kT, 0, s>>>(b.faces, n, cnt);
      else k_count_half<<<nblk(n), kT, 0, s>>>(b.edges, n, cnt);
      tmp_bytes = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, nv + 1, s);
      void* tmp = sc.get<char>(tmp_bytes);
      if (!tmp) return static_cast<int>(cudaErrorMemoryAllocation);
      cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, nv + 1, s);
      cudaMemcpyAsync(cnt, off, sizeof(int) * nv, cudaMemcpyDeviceToDevice, s);  // row cursors
      if (pass == 0) k_scatter_corners<<<nblk(n), kT, 0, s>>>(b.faces, n, cnt, col);
      else k_scatter_half<<<nblk(n), kT, 0, s>>>(b.edges, n, cnt, col);
      k_sort_rows<<<nblk(nv), kT, 0, s>>>(off, nv, col);
    }
  }
  note_launch(27);
  cudaMemcpyAsync(hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return static_cast<int>(e);
  if (hb[0]) return 1;  // a near-zero-area face: the host raises it with its index
  b.ne = ne;
  return static_cast<int>(cudaGetLastError());
}

}  // namespace dtb
