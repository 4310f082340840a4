// Device-side construction of the mesh arrays the engine reads: SoA and
// fixed-point positions from the uploaded vertex array, and the
// front-connectivity CSR (for each vertex, the higher-numbered vertices it
// shares an edge with or faces across a link edge -- the relation under
// which band-vertex union-find reproduces extract_front's edge-adjacency of
// band triangles, diffusion.hpp:412-428).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <algorithm>
#include <cstring>
#include <vector>

#include "kernels.h"

namespace dtb {

namespace {

constexpr int kMaxRel = 64;  // related vertices per vertex before dedup (valence <= 32)

__global__ void k_positions(const double* xyz, int nv, double scale, double* px, double* py, double* pz, long long* fx,
                            long long* fy, long long* fz) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double x = xyz[3 * v], y = xyz[3 * v + 1], z = xyz[3 * v + 2];
  px[v] = x;
  py[v] = y;
  pz[v] = z;
  fx[v] = __double2ll_rn(x * scale);
  fy[v] = __double2ll_rn(y * scale);
  fz[v] = __double2ll_rn(z * scale);
}

// Gathers, sorts and deduplicates the related vertices u > v of v.
__device__ int related(const FrontBuild& B, int v, int* out, bool* overflow) {
  int n = 0;
  for (int q = B.v2v_off[v]; q < B.v2v_off[v + 1]; ++q) {
    const int u = B.v2v[q];
    if (u > v) {
      if (n < kMaxRel) out[n++] = u;
      else *overflow = true;
    }
  }
  for (int q = B.v2f_off[v]; q < B.v2f_off[v + 1]; ++q) {
    const int f = B.v2f[q];
    const unsigned t0 = B.faces[3 * f], t1 = B.faces[3 * f + 1];
    const int kv = t0 == static_cast<unsigned>(v) ? 0 : (t1 == static_cast<unsigned>(v) ? 1 : 2);
    const unsigned e = B.face_edges[3 * f + (kv + 1) % 3];  // the edge of f opposite v
    const unsigned g = B.edge_faces[2 * e] == static_cast<unsigned>(f) ? B.edge_faces[2 * e + 1] : B.edge_faces[2 * e];
    const unsigned a = B.edges[2 * e], b = B.edges[2 * e + 1];
    for (int k = 0; k < 3; ++k) {
      const unsigned w = B.faces[3 * g + k];
      if (w != a && w != b && static_cast<int>(w) > v) {
        if (n < kMaxRel) out[n++] = static_cast<int>(w);
        else *overflow = true;
      }
    }
  }
  for (int i = 1; i < n; ++i) {  // insertion sort of a short list
    const int x = out[i];
    int j = i - 1;
    while (j >= 0 && out[j] > x) {
      out[j + 1] = out[j];
      --j;
    }
    out[j + 1] = x;
  }
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || out[m - 1] != out[i]) out[m++] = out[i];
  return m;
}

// Relations are gathered once, into each vertex's room (2 x its valence
// entries from 2 * v2v_off[v]: a vertex has at most valence neighbours and
// valence faces), then moved to the scanned offsets.
__global__ void k_front_room(FrontBuild B, int* counts, int* overflow, int* room) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B.nv) return;
  int tmp[kMaxRel];
  bool over = false;
  const int n = related(B, v, tmp, &over);
  const int base = 2 * B.v2v_off[v], cap = 2 * (B.v2v_off[v + 1] - B.v2v_off[v]);
  if (over || n > cap) {
    *overflow = 1;
    counts[v] = 0;
    return;
  }
  for (int i = 0; i < n; ++i) room[base + i] = tmp[i];
  counts[v] = n;
}

__global__ void k_front_compact(FrontBuild B, const int* room, const int* off, int* col) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B.nv) return;
  const int base = 2 * B.v2v_off[v], dst = off[v], n = off[v + 1] - dst;
  for (int i = 0; i < n; ++i) col[dst + i] = room[base + i];
}

}  // namespace

// seed_region (diffusion.hpp:134) on the device.  The reference pops a
// Dijkstra queue until the distance exceeds the radius, so its result is
// {u : d(u) <= radius} with d the least fixed point of
//   d(u) = min over neighbours v of fl(d(v) + |p(v) - p(u)|),  d(seed) = 0
// (floating-point addition of a non-negative length is monotone, so that is
// what Dijkstra computes).  One CTA reaches the same fixed point by
// frontier-based Bellman-Ford relaxation with atomicMin on the distance bits
// (non-negative doubles order like their bit patterns); relaxations beyond the
// radius are skipped since they cannot lead back inside it.  The frontier
// lives in shared memory and each entry's row is relaxed by 8 lanes at once
// (one round of loads per level instead of one per neighbour).  Overflowing
// a capacity reports -1 and the caller uses the host.
constexpr int kSeedCap = 1 << 15;   // touched vertices
constexpr int kSeedFront = 4096;    // frontier entries per level (shared memory)
constexpr unsigned long long kFar = 0x7F7F7F7F7F7F7F7Full;  // 3.4e306, the memset pattern
struct SeedScratch {
  int touched[kSeedCap];
};

__global__ void __launch_bounds__(1024) k_seed_region(const int* off, const int* col, const double* px,
                                                      const double* py, const double* pz, unsigned seed, double radius,
                                                      unsigned long long* dist, SeedScratch* S, unsigned* out,
                                                      int cap, int* out_n) {
  __shared__ int front[2][kSeedFront];
  __shared__ int nfront[2], ntouched, overflow;
  if (threadIdx.x == 0) {
    dist[seed] = static_cast<unsigned long long>(__double_as_longlong(0.0));
    front[0][0] = static_cast<int>(seed);
    nfront[0] = 1;
    nfront[1] = 0;
    S->touched[0] = static_cast<int>(seed);
    ntouched = 1;
    overflow = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 7, g0 = threadIdx.x >> 3, ng = blockDim.x >> 3;
  int cur = 0;
  while (true) {
    const int n = nfront[cur];
    if (n == 0 || overflow) break;
    for (int i = g0; i < n; i += ng) {
      const int v = front[cur][i];
      const double dv = __longlong_as_double(static_cast<long long>(__ldcg(dist + v)));
      const double vx = px[v], vy = py[v], vz = pz[v];
      const int o1 = off[v + 1];
      for (int o = off[v] + lane; o < o1; o += 8) {
        const int u = col[o];
        const double dx = vx - px[u], dy = vy - py[u], dz = vz - pz[u];
        const double nd = dv + sqrt(dx * dx + dy * dy + dz * dz);
        if (!(nd <= radius)) continue;
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(nd));
        const unsigned long long old = atomicMin(dist + u, bits);
        if (bits < old) {
          if (old == kFar) {
            const int t = atomicAdd(&ntouched, 1);
            if (t < kSeedCap) S->touched[t] = u;
            else overflow = 1;
          }
          const int q = atomicAdd(&nfront[cur ^ 1], 1);
          if (q < kSeedFront) front[cur ^ 1][q] = u;
          else overflow = 1;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) nfront[cur] = 0;
    cur ^= 1;
    __syncthreads();
  }
  // Every touched vertex ended at d <= radius (only such values are stored).
  // out[0] = count (or -1), out[1..] = the vertices; dist back to "far".
  const int nt = min(ntouched, kSeedCap);
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int u = S->touched[i];
    if (i < cap) out[1 + i] = static_cast<unsigned>(u);
    dist[u] = kFar;
  }
  if (threadIdx.x == 0) *out_n = (overflow || nt > cap) ? -1 : nt;
}

int launch_seed_region(const DevMesh& m, unsigned seed, double radius, unsigned* out, int cap, int* n, void* stream,
                       unsigned long long* dist) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!(radius >= 0.0)) {  // NaN radius: the reference's loop breaks at once... let the host decide
    *n = -1;
    return 0;
  }
  static_assert(kFar == 0x7F7F7F7F7F7F7F7Full, "distance reset value is a memset byte pattern");
  const size_t dbytes = sizeof(unsigned long long) * static_cast<size_t>(m.nv);
  const bool own = dist == nullptr;
  if (own) {
    dist = static_cast<unsigned long long*>(dev_alloc(dbytes));
    cudaMemsetAsync(dist, 0x7F, dbytes, s);
  }
  cap = max(0, min(cap, kSeedCap));
  SeedScratch* S = static_cast<SeedScratch*>(dev_alloc(sizeof(SeedScratch)));
  const size_t obytes = sizeof(unsigned) * (static_cast<size_t>(cap) + 1);
  unsigned* dout = static_cast<unsigned*>(dev_alloc(obytes));  // count, then the vertices
  k_seed_region<<<1, 1024, 0, s>>>(m.n_off, m.n_col, m.px, m.py, m.pz, seed, radius, dist, S, dout, cap,
                                   reinterpret_cast<int*>(dout));
  note_launch();
  // One read-back of count and list (the list is at most cap words).
  std::vector<unsigned> h(static_cast<size_t>(cap) + 1);
  cudaMemcpyAsync(h.data(), dout, obytes, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  *n = static_cast<int>(h[0]);
  if (e == cudaSuccess && *n > 0) std::memcpy(out, h.data() + 1, sizeof(unsigned) * static_cast<size_t>(*n));
  if (*n < 0 && !own) cudaMemsetAsync(dist, 0x7F, dbytes, s);  // touched vertices may have gone unrecorded
  dev_free(dout, obytes);
  dev_free(S, sizeof(SeedScratch));
  if (own) dev_free(dist, dbytes);
  return static_cast<int>(e);
}

int launch_positions(const double* xyz, int nv, double scale, double* px, double* py, double* pz, long long* fx,
                     long long* fy, long long* fz, void* stream) {
  k_positions<<<(nv + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(xyz, nv, scale, px, py, pz, fx, fy, fz);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

// Count pass + exclusive scan into c_off; returns the column count through
// *nnz, or -1 when a vertex has more than kMaxRel relations.
int launch_front_count(const FrontBuild& b, int* c_off, int* nnz, void** room_out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int *counts = nullptr, *over = nullptr;
  // The room comes from the library's caching allocator (see launch_assemble);
  // the caller frees it with dev_free(room, front_room_bytes(b)) after the
  // stream has finished with it.
  int* room = static_cast<int*>(dev_alloc(front_room_bytes(b)));
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&counts), sizeof(int) * (b.nv + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&over), sizeof(int), s);
  if (e != cudaSuccess) {
    dev_free(room, front_room_bytes(b));
    return static_cast<int>(e);
  }
  cudaMemsetAsync(over, 0, sizeof(int), s);
  cudaMemsetAsync(counts + b.nv, 0, sizeof(int), s);
  const int blocks = (b.nv + 127) / 128;
  k_front_room<<<blocks, 128, 0, s>>>(b, counts, over, room);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, c_off, b.nv + 1, s);
  void* tmp = nullptr;
  cudaMallocAsync(&tmp, tmp_bytes, s);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, c_off, b.nv + 1, s);
  note_launch(3);
  int h[2] = {0, 0};
  cudaMemcpyAsync(&h[0], c_off + b.nv, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&h[1], over, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(counts, s);
  cudaFreeAsync(over, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess || h[1]) {
    dev_free(room, front_room_bytes(b));
    return e != cudaSuccess ? static_cast<int>(e) : -1;
  }
  *nnz = h[0];
  *room_out = room;
  return static_cast<int>(cudaGetLastError());
}

int launch_front_fill(const FrontBuild& b, const int* c_off, int* c_col, void* room, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_front_compact<<<(b.nv + 127) / 128, 128, 0, s>>>(b, static_cast<const int*>(room), c_off, c_col);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Local gathers for host event handling (engine.cpp LocalMesh): the records
// of listed vertices, faces and edges, so an event never downloads the whole
// mesh.  Rows are copied in two passes: bounds + positions, then the rows at
// host-computed packed offsets.
__global__ void k_gather_vhead(MeshRows m, const unsigned* list, int n, int* bounds, double* pos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned v = list[i];
  bounds[4 * i + 0] = m.v2v_off[v];
  bounds[4 * i + 1] = m.v2v_off[v + 1];
  bounds[4 * i + 2] = m.v2f_off[v];
  bounds[4 * i + 3] = m.v2f_off[v + 1];
  pos[3 * i + 0] = m.px[v];
  pos[3 * i + 1] = m.py[v];
  pos[3 * i + 2] = m.pz[v];
}

__global__ void k_gather_vrows(MeshRows m, const int* bounds, const int* dst, int n, unsigned* rows) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = dst[i];
  for (int k = bounds[4 * i]; k < bounds[4 * i + 1]; ++k) rows[o++] = static_cast<unsigned>(m.v2v[k]);
  for (int k = bounds[4 * i + 2]; k < bounds[4 * i + 3]; ++k) rows[o++] = static_cast<unsigned>(m.v2f[k]);
}

__global__ void k_gather_faces(MeshRows m, const unsigned* list, int n, unsigned* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t f = list[i];
  for (int c = 0; c < 3; ++c) {
    out[6 * i + c] = m.faces[3 * f + c];
    out[6 * i + 3 + c] = m.face_edges[3 * f + c];
  }
}

__global__ void k_gather_edges(MeshRows m, const unsigned* list, int n, unsigned* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t e = list[i];
  out[4 * i + 0] = m.edges[2 * e];
  out[4 * i + 1] = m.edges[2 * e + 1];
  out[4 * i + 2] = m.edge_faces[2 * e];
  out[4 * i + 3] = m.edge_faces[2 * e + 1];
}

int launch_gather_vhead(const MeshRows& m, const unsigned* list, int n, int* bounds, double* pos, void* stream) {
  if (n <= 0) return 0;
  k_gather_vhead<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(m, list, n, bounds, pos);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}
int launch_gather_vrows(const MeshRows& m, const int* bounds, const int* dst, int n, unsigned* rows, void* stream) {
  if (n <= 0) return 0;
  k_gather_vrows<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(m, bounds, dst, n, rows);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}
int launch_gather_faces(const MeshRows& m, const unsigned* list, int n, unsigned* out, void* stream) {
  if (n <= 0) return 0;
  k_gather_faces<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(m, list, n, out);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}
int launch_gather_edges(const MeshRows& m, const unsigned* list, int n, unsigned* out, void* stream) {
  if (n <= 0) return 0;
  k_gather_edges<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(m, list, n, out);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

}  // namespace dtb
