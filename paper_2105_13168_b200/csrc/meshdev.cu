// Device-side construction of the mesh arrays the engine reads: SoA and
// fixed-point positions from the uploaded vertex array, and the
// front-connectivity CSR (for each vertex, the higher-numbered vertices it
// shares an edge with or faces across a link edge -- the relation under
// which band-vertex union-find reproduces extract_front's edge-adjacency of
// band triangles, diffusion.hpp:412-428).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

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

__global__ void k_front_count(FrontBuild B, int* counts, int* overflow) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B.nv) return;
  int tmp[kMaxRel];
  bool over = false;
  counts[v] = related(B, v, tmp, &over);
  if (over) *overflow = 1;
}

__global__ void k_front_fill(FrontBuild B, const int* off, int* col) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B.nv) return;
  int tmp[kMaxRel];
  bool over = false;
  const int n = related(B, v, tmp, &over);
  for (int i = 0; i < n; ++i) col[off[v] + i] = tmp[i];
}

}  // namespace

int launch_positions(const double* xyz, int nv, double scale, double* px, double* py, double* pz, long long* fx,
                     long long* fy, long long* fz, void* stream) {
  k_positions<<<(nv + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(xyz, nv, scale, px, py, pz, fx, fy, fz);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

// Count pass + exclusive scan into c_off; returns the column count through
// *nnz, or -1 when a vertex has more than kMaxRel relations.
int launch_front_count(const FrontBuild& b, int* c_off, int* nnz, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int *counts = nullptr, *over = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&counts), sizeof(int) * (b.nv + 1), s);
  if (e != cudaSuccess) return static_cast<int>(e);
  cudaMallocAsync(reinterpret_cast<void**>(&over), sizeof(int), s);
  cudaMemsetAsync(over, 0, sizeof(int), s);
  cudaMemsetAsync(counts + b.nv, 0, sizeof(int), s);
  const int blocks = (b.nv + 127) / 128;
  k_front_count<<<blocks, 128, 0, s>>>(b, counts, over);
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
  if (e != cudaSuccess) return static_cast<int>(e);
  if (h[1]) return -1;
  *nnz = h[0];
  return static_cast<int>(cudaGetLastError());
}

int launch_front_fill(const FrontBuild& b, const int* c_off, int* c_col, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_front_fill<<<(b.nv + 127) / 128, 128, 0, s>>>(b, c_off, c_col);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

}  // namespace dtb
