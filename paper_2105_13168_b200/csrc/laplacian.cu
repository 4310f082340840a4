// Cotangent-Laplacian assembly on the device (reference: operators.hpp:33-70).
//
// One thread per vertex builds its stiffness row directly in CSR form: the
// sorted column set {v} U N(v), off-diagonal (v,u) = sum over the two faces of
// edge vu of 0.5 * cot(opposite angle), diagonal = -sum of the incident
// half-weights, entries that sum to exactly zero dropped (from_triplets with
// drop tolerance 0, sparse.hpp:50).  Off-diagonal sums have two terms and are
// therefore bit-identical to the reference's sort-then-sum; the diagonal sums
// 2*deg terms in face order, which can differ from the reference's
// std::sort-dependent order in the last bits (tests bound it by 8 ulp).
// Lumped masses accumulate face areas / 3 in face order exactly like the
// reference's sequential loop, so they are bit-identical.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "kernels.h"

namespace dtb {

namespace {

struct P3 {
  double x, y, z;
};
__device__ __forceinline__ P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot3(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ P3 cross3(P3 a, P3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ P3 pos(const LapBuild& b, unsigned v) { return {b.px[v], b.py[v], b.pz[v]}; }

// Half cotangent weight of edge (a, b) inside face with apex c.
__device__ __forceinline__ double half_cot(const LapBuild& B, unsigned a, unsigned b, unsigned c, bool& bad) {
  const P3 pc = pos(B, c);
  const P3 ca = sub(pos(B, a), pc), cb = sub(pos(B, b), pc);
  const double cot = dot3(ca, cb) / sqrt(dot3(cross3(ca, cb), cross3(ca, cb)));
  if (!isfinite(cot)) bad = true;
  return 0.5 * cot;
}

// Off-diagonal value of (v, u): the two incident faces' half weights.
__device__ double offdiag(const LapBuild& B, int v, int u, bool& bad) {
  double sum = 0.0;
  for (int q = B.v2f_off[v]; q < B.v2f_off[v + 1]; ++q) {
    const int f = B.v2f[q];
    const unsigned t0 = B.faces[3 * f], t1 = B.faces[3 * f + 1], t2 = B.faces[3 * f + 2];
    unsigned c;
    if ((t0 == (unsigned)v && t1 == (unsigned)u) || (t1 == (unsigned)v && t0 == (unsigned)u)) c = t2;
    else if ((t1 == (unsigned)v && t2 == (unsigned)u) || (t2 == (unsigned)v && t1 == (unsigned)u)) c = t0;
    else if ((t2 == (unsigned)v && t0 == (unsigned)u) || (t0 == (unsigned)v && t2 == (unsigned)u)) c = t1;
    else continue;
    sum = sum + half_cot(B, (unsigned)v, (unsigned)u, c, bad);
  }
  return sum;
}

// Diagonal: -w for each (face, corner-edge) incident to v, faces in order,
// corner edges k = 0, 1, 2 within a face (the reference's triplet order before
// its sort).
__device__ double diagonal(const LapBuild& B, int v, bool& bad) {
  double sum = 0.0;
  for (int q = B.v2f_off[v]; q < B.v2f_off[v + 1]; ++q) {
    const int f = B.v2f[q];
    const unsigned t[3] = {B.faces[3 * f], B.faces[3 * f + 1], B.faces[3 * f + 2]};
    for (int k = 0; k < 3; ++k) {
      const unsigned a = t[k], b = t[(k + 1) % 3], c = t[(k + 2) % 3];
      if (a != (unsigned)v && b != (unsigned)v) continue;
      sum = sum + (-half_cot(B, a, b, c, bad));
    }
  }
  return sum;
}

// Row v of the stiffness matrix in one pass over v's faces (v2f order):
// each corner edge (a, b) of a face that contains v adds -w to the diagonal
// (faces in order, corner edges k = 0, 1, 2 within a face: the reference's
// triplet order before its sort) and w to the off-diagonal of the other end,
// whose two faces therefore add in face order, 0 + w1 + w2 -- term for term
// the reference's triplet sums.  half_cot is symmetric in (a, b) bit for bit
// (the products commute and the cross product only changes sign), so one
// value serves both entries.  acc[j] belongs to the j-th neighbour of the
// sorted row; returns the row length, or -1 above kMaxValence (then
// diagonal / offdiag give the same values entry by entry).
constexpr int kMaxValence = 32;
__device__ int row_values(const LapBuild& B, int v, bool& bad, int* nbr, double* acc, double& diag) {
  const int q0 = B.v2v_off[v], deg = B.v2v_off[v + 1] - q0;
  if (deg > kMaxValence) return -1;  // the caller takes the entries one by one
  for (int j = 0; j < deg; ++j) {
    nbr[j] = B.v2v[q0 + j];
    acc[j] = 0.0;
  }
  double d = 0.0;
  for (int q = B.v2f_off[v]; q < B.v2f_off[v + 1]; ++q) {
    const int f = B.v2f[q];
    const unsigned t[3] = {B.faces[3 * f], B.faces[3 * f + 1], B.faces[3 * f + 2]};
    for (int k = 0; k < 3; ++k) {
      const unsigned a = t[k], b = t[(k + 1) % 3], c = t[(k + 2) % 3];
      if (a != (unsigned)v && b != (unsigned)v) continue;
      const double h = half_cot(B, a, b, c, bad);
      d = d + (-h);
      const int u = static_cast<int>(a == (unsigned)v ? b : a);
      for (int j = 0; j < deg; ++j)
        if (nbr[j] == u) {
          acc[j] = acc[j] + h;
          break;
        }
    }
  }
  diag = d;
  return deg;
}

// Fills row v once: its non-zero entries (the reference's triplet sums drop
// exact zeros) packed at the start of the row's room for the diagonal and
// every mesh neighbour (offset v2v_off[v] + v), the number of them in
// counts[v]; k_row_compact then moves the rows to their scanned offsets.
constexpr int kRowBad = 1;
__global__ void k_row_fill(LapBuild B, int* flags, int* counts) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= B.nv) return;
  bool bad = false;
  int nbr[kMaxValence];
  double acc[kMaxValence], d;
  const int deg = row_values(B, v, bad, nbr, acc, d);
  const bool wide = deg < 0;
  if (wide) d = diagonal(B, v, bad);
  const int o0 = B.v2v_off[v] + v;
  int o = o0;
  bool diag_done = false;
  double gersh = 0.0;
  auto emit = [&](int c, double x) {
    B.s_col[o] = c;
    B.s_val[o] = x;
    ++o;
    gersh = gersh + fabs(x);
  };
  const int q0 = B.v2v_off[v], n = B.v2v_off[v + 1] - q0;
  for (int j = 0; j < n; ++j) {
    const int u = wide ? B.v2v[q0 + j] : nbr[j];
    if (!diag_done && u > v) {
      if (d != 0.0) emit(v, d);
      diag_done = true;
    }
    const double w = wide ? offdiag(B, v, u, bad) : acc[j];
    if (w != 0.0) emit(u, w);
  }
  if (!diag_done && d != 0.0) emit(v, d);
  counts[v] = o - o0;
  if (bad) atomicOr(flags, kRowBad);
  // Lumped mass: area / 3 of every incident face, in face order.
  double m = 0.0;
  for (int q = B.v2f_off[v]; q < B.v2f_off[v + 1]; ++q) {
    const int f = B.v2f[q];
    const P3 p0 = pos(B, B.faces[3 * f]), p1 = pos(B, B.faces[3 * f + 1]), p2 = pos(B, B.faces[3 * f + 2]);
    const P3 n = cross3(sub(p1, p0), sub(p2, p0));
    const double area = 0.5 * sqrt(dot3(n, n));
    m = m + area / 3.0;
  }
  B.mass[v] = m;
  B.gersh_row[v] = gersh / m;
}

// Moves each filled row from its room (v2v_off[v] + v) to its scanned offset.
__global__ void k_row_compact(int nv, const int* v2v_off, const int* off, const int* tcol, const double* tval,
                              int* col, double* val) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int src = v2v_off[v] + v, dst = off[v], n = off[v + 1] - dst;
  for (int k = 0; k < n; ++k) {
    col[dst + k] = tcol[src + k];
    val[dst + k] = tval[src + k];
  }
}

__global__ void k_spmv(int nv, const int* off, const int* col, const double* val, const double* mass, const double* x,
                       double* y) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  double acc = 0.0;
  for (int k = off[v]; k < off[v + 1]; ++k) acc = acc + val[k] * x[col[k]];
  y[v] = acc / mass[v];
}

}  // namespace

// Returns cudaSuccess, or -1 when a cotangent weight is non-finite
// (DegeneracyError, operators.hpp:48).
int launch_assemble(const LapBuild& b, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int threads = 128, blocks = (b.nv + threads - 1) / threads;
  int* counts = nullptr;
  int* bad = nullptr;
  int* tcol = nullptr;
  double* tval = nullptr;
  const size_t room = static_cast<size_t>(b.nv) + static_cast<size_t>(b.nroom);  // diagonal + neighbours
  // The row rooms come from the library's caching allocator (a stream-ordered
  // pool allocation of this size is mapped anew after every synchronisation
  // and serialises concurrent batch lanes); freed after the closing sync.
  tcol = static_cast<int*>(dev_alloc(sizeof(int) * room));
  tval = static_cast<double*>(dev_alloc(sizeof(double) * room));
  auto release = [&]() {
    dev_free(tcol, sizeof(int) * room);
    dev_free(tval, sizeof(double) * room);
  };
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&counts), sizeof(int) * (b.nv + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), s);
  if (e != cudaSuccess) {
    cudaStreamSynchronize(s);
    release();
    return static_cast<int>(e);
  }
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  cudaMemsetAsync(counts + b.nv, 0, sizeof(int), s);
  LapBuild bt = b;  // rows filled into their rooms first
  bt.s_col = tcol;
  bt.s_val = tval;
  k_row_fill<<<blocks, threads, 0, s>>>(bt, bad, counts);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, b.s_off, b.nv + 1, s);
  void* tmp = nullptr;
  cudaMallocAsync(&tmp, tmp_bytes, s);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, b.s_off, b.nv + 1, s);
  k_row_compact<<<blocks, threads, 0, s>>>(b.nv, b.v2v_off, b.s_off, tcol, tval, b.s_col, b.s_val);
  note_launch(4);  // row fill, two scan passes, compaction
  cudaMemcpyAsync(b.nnz, b.s_off + b.nv, sizeof(int), cudaMemcpyDeviceToDevice, s);
  // Gershgorin bound: max over the rows (exact in any order).
  size_t red_bytes = 0;
  cub::DeviceReduce::Max(nullptr, red_bytes, b.gersh_row, b.gersh_max, b.nv, s);
  void* red = nullptr;
  cudaMallocAsync(&red, red_bytes, s);
  cub::DeviceReduce::Max(red, red_bytes, b.gersh_row, b.gersh_max, b.nv, s);
  note_launch(1);
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(red, s);
  cudaFreeAsync(counts, s);
  cudaFreeAsync(bad, s);
  e = cudaStreamSynchronize(s);
  release();
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaGetLastError();
  if (e != cudaSuccess) return static_cast<int>(e);
  return (hbad & kRowBad) ? -1 : 0;
}

namespace {
__global__ void k_ell(int nv, const int* off, const int* col, const double* val, unsigned char* e_len, int* e_col,
                      double* e_val) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int k0 = off[v], n = off[v + 1] - k0;
  e_len[v] = static_cast<unsigned char>(n > 255 ? 255 : n);
  for (int j = 0; j < kEll; ++j) {
    const bool ok = j < n;
    e_col[static_cast<size_t>(v) * kEll + j] = ok ? col[k0 + j] : -1;
    e_val[static_cast<size_t>(v) * kEll + j] = ok ? val[k0 + j] : 0.0;
  }
}
// The same sums over the padded rows: one thread per row reads its 8 columns
// and 8 values with six 16-byte loads, rows longer than kEll take the CSR.
// Summation order and rounding are k_spmv's.
__global__ void k_spmv_ell(int nv, const unsigned char* e_len, const int* e_col, const double* e_val, const int* off,
                           const int* col, const double* val, const double* mass, const double* x, double* y) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int n = e_len[v];
  double acc = 0.0;
  if (n <= kEll) {
    const size_t b = static_cast<size_t>(v) * kEll;
    const int4 c0 = __ldg(reinterpret_cast<const int4*>(e_col + b));
    const int4 c1 = __ldg(reinterpret_cast<const int4*>(e_col + b + 4));
    const double2 w0 = __ldg(reinterpret_cast<const double2*>(e_val + b));
    const double2 w1 = __ldg(reinterpret_cast<const double2*>(e_val + b + 2));
    const double2 w2 = __ldg(reinterpret_cast<const double2*>(e_val + b + 4));
    const double2 w3 = __ldg(reinterpret_cast<const double2*>(e_val + b + 6));
    const int cs[kEll] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const double ws[kEll] = {w0.x, w0.y, w1.x, w1.y, w2.x, w2.y, w3.x, w3.y};
    double xs[kEll];
#pragma unroll
    for (int j = 0; j < kEll; ++j) xs[j] = j < n ? __ldg(x + cs[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < kEll; ++j)
      if (j < n) acc = acc + ws[j] * xs[j];
  } else {
    for (int k = off[v]; k < off[v + 1]; ++k) acc = acc + val[k] * x[col[k]];
  }
  y[v] = acc / mass[v];
}

// Reads n 16-byte words (an L2 eviction that leaves clean lines behind, so
// the next kernel does not pay for write-backs); writes only if a word holds
// an impossible value.
__global__ void k_read_all(const int4* p, size_t n, int* sink) {
  int acc = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int4 q = __ldcs(p + i);
    acc ^= q.x ^ q.y ^ q.z ^ q.w;
  }
  if (acc == 0x7A5E1234) *sink = acc;
}

}  // namespace

int launch_ell(int nv, const int* off, const int* col, const double* val, unsigned char* e_len, int* e_col,
               double* e_val, void* stream) {
  k_ell<<<(nv + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(nv, off, col, val, e_len, e_col, e_val);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

int launch_spmv(int nv, const int* off, const int* col, const double* val, const double* mass, const double* x,
                double* y, void* stream) {
  const int threads = 256;
  k_spmv<<<(nv + threads - 1) / threads, threads, 0, static_cast<cudaStream_t>(stream)>>>(nv, off, col, val, mass, x,
                                                                                           y);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

int launch_read_all(const void* p, size_t bytes, int* sink, void* stream) {
  k_read_all<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const int4*>(p), bytes / 16, sink);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

int launch_spmv_ell(int nv, const unsigned char* e_len, const int* e_col, const double* e_val, const int* off,
                    const int* col, const double* val, const double* mass, const double* x, double* y, void* stream) {
  const int threads = 256;
  k_spmv_ell<<<(nv + threads - 1) / threads, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      nv, e_len, e_col, e_val, off, col, val, mass, x, y);
  note_launch();
  return static_cast<int>(cudaGetLastError());
}

}  // namespace dtb
