// Host mesh construction, generators and IO.  See mesh.hpp for the contract.
//
// Construction is parallel (OpenMP) wherever the reference's sequential
// semantics allow it: validation scans report the first offending face, the
// slot pairing and adjacency lists are bucketed with atomic cursors and then
// sorted per bucket (deterministic), edge numbering is a prefix sum over
// "first slot of its edge" flags.  Orientation is checked in parallel; only
// an inconsistently oriented input takes the reference's sequential BFS.
#include "mesh.hpp"

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstring>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>
#include <unordered_map>

namespace dtb {

namespace {

using U32 = std::uint32_t;

// Exclusive prefix sum in place over counts[0..n] (counts[n] becomes the total).
void exclusive_scan(std::vector<U32>& a) {
  U32 run = 0;
  for (auto& x : a) {
    const U32 c = x;
    x = run;
    run += c;
  }
}

// CSR of (key -> items) for items whose key is produced by key_of(i), with
// the items of each bucket sorted by less(a, b).  Parallel: atomic counts,
// atomic-cursor scatter, per-bucket sort.
template <class KeyOf, class Less>
void bucket_sort(std::size_t nitems, Index nkeys, KeyOf key_of, Less less, std::vector<U32>& off,
                 std::vector<U32>& items) {
  off.assign(static_cast<std::size_t>(nkeys) + 1, 0);
  std::vector<std::atomic<U32>> cnt(static_cast<std::size_t>(nkeys));
#pragma omp parallel for schedule(static)
  for (long long k = 0; k < static_cast<long long>(nkeys); ++k) cnt[k].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < static_cast<long long>(nitems); ++i)
    cnt[key_of(static_cast<std::size_t>(i))].fetch_add(1, std::memory_order_relaxed);
  for (Index k = 0; k < nkeys; ++k) off[k] = cnt[k].load(std::memory_order_relaxed);
  off[nkeys] = 0;
  exclusive_scan(off);
#pragma omp parallel for schedule(static)
  for (long long k = 0; k < static_cast<long long>(nkeys); ++k) cnt[k].store(off[k], std::memory_order_relaxed);
  items.resize(nitems);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < static_cast<long long>(nitems); ++i)
    items[cnt[key_of(static_cast<std::size_t>(i))].fetch_add(1, std::memory_order_relaxed)] = static_cast<U32>(i);
#pragma omp parallel for schedule(dynamic, 4096)
  for (long long k = 0; k < static_cast<long long>(nkeys); ++k)
    std::sort(items.begin() + off[k], items.begin() + off[k + 1], less);
}

// Groups the 3F directed face slots (slot s = 3f + k is the edge from corner k
// to corner k+1 of the ORIGINAL face) by their unordered vertex pair, bucketed
// on the smaller endpoint.  Reports non-manifold (>2 slots) and boundary (1
// slot) edges with the reference's error classes (mesh.hpp:210-221), and
// returns partner[s] = the other slot of s's edge.
std::vector<U32> pair_slots(const std::vector<std::array<Index, 3>>& faces, Index nv) {
  const std::size_t ns = faces.size() * 3;
  auto lo_of = [&](std::size_t s) {
    const auto& t = faces[s / 3];
    return std::min(t[s % 3], t[(s % 3 + 1) % 3]);
  };
  auto hi_of = [&](std::size_t s) {
    const auto& t = faces[s / 3];
    return std::max(t[s % 3], t[(s % 3 + 1) % 3]);
  };
  std::vector<U32> off, bucket;
  bucket_sort(
      ns, nv, lo_of,
      [&](U32 a, U32 b) {
        const Index ha = hi_of(a), hb = hi_of(b);
        return ha != hb ? ha < hb : a < b;
      },
      off, bucket);
  std::vector<U32> partner(ns, kInvalid);
  int nonmanifold = 0, boundary = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : nonmanifold, boundary)
  for (long long v = 0; v < static_cast<long long>(nv); ++v) {
    for (U32 i = off[v]; i < off[v + 1];) {
      U32 j = i;
      const Index h = hi_of(bucket[i]);
      while (j < off[v + 1] && hi_of(bucket[j]) == h) ++j;
      if (j - i > 2) nonmanifold = 1;
      else if (j - i == 1) boundary = 1;
      else {
        partner[bucket[i]] = bucket[i + 1];
        partner[bucket[i + 1]] = bucket[i];
      }
      i = j;
    }
  }
  if (nonmanifold) fail(kTopologyError, "non-manifold edge with more than two faces");
  if (boundary) fail(kTopologyError, "boundary edge: surface is not closed");
  return partner;
}

// Lock-free union-find over face indices (connectivity of the face graph).
Index uf_root(std::vector<std::atomic<U32>>& p, U32 x) {
  while (true) {
    const U32 q = p[x].load(std::memory_order_relaxed);
    if (q == x) return x;
    const U32 r = p[q].load(std::memory_order_relaxed);
    if (r != q) p[x].compare_exchange_weak(const_cast<U32&>(q), r, std::memory_order_relaxed);
    x = q;
  }
}

}  // namespace

Mesh::Mesh(std::vector<V3> vertices, std::vector<std::array<Index, 3>> faces)
    : pos_(std::move(vertices)), faces_(std::move(faces)) {
  if (faces_.empty()) fail(kTopologyError, "mesh has no faces");
  const Index raw = static_cast<Index>(pos_.size());
  // First face (in order) that references an out-of-range vertex or repeats
  // one; the reference checks faces in order, range before repetition.
  {
    long long first_bad = static_cast<long long>(faces_.size());
#pragma omp parallel for reduction(min : first_bad)
    for (long long i = 0; i < static_cast<long long>(faces_.size()); ++i) {
      const auto& f = faces_[i];
      const bool bad = f[0] >= raw || f[1] >= raw || f[2] >= raw || f[0] == f[1] || f[1] == f[2] || f[0] == f[2];
      if (bad && i < first_bad) first_bad = i;
    }
    if (first_bad < static_cast<long long>(faces_.size())) {
      const auto& f = faces_[first_bad];
      for (Index v : f)
        if (v >= raw) fail(kParseError, "face references vertex out of range");
      fail(kDegeneracyError, "face repeats a vertex");
    }
  }
  // Unreferenced vertices are dropped; survivors renumbered by first use.
  {
    std::vector<unsigned char> used(pos_.size(), 0);
#pragma omp parallel for
    for (long long i = 0; i < static_cast<long long>(faces_.size()); ++i)
      for (Index v : faces_[i]) used[v] = 1;
    long long unused = 0;
#pragma omp parallel for reduction(+ : unused)
    for (long long v = 0; v < static_cast<long long>(used.size()); ++v) unused += used[v] ? 0 : 1;
    if (unused) {
      std::vector<Index> remap(pos_.size(), kInvalid);
      Index next = 0;
      for (const auto& f : faces_)
        for (Index v : f)
          if (remap[v] == kInvalid) remap[v] = next++;
      std::vector<V3> compact(next);
      for (Index v = 0; v < pos_.size(); ++v)
        if (remap[v] != kInvalid) compact[remap[v]] = pos_[v];
      pos_ = std::move(compact);
      for (auto& f : faces_)
        for (Index& v : f) v = remap[v];
    }
  }
  // Duplicate faces in any vertex order are rejected: bucket the sorted
  // triples by their smallest vertex and compare within the buckets.
  {
    std::vector<std::array<Index, 3>> keys(faces_.size());
#pragma omp parallel for
    for (long long i = 0; i < static_cast<long long>(faces_.size()); ++i) {
      keys[i] = faces_[i];
      std::sort(keys[i].begin(), keys[i].end());
    }
    std::vector<U32> off, items;
    bucket_sort(
        faces_.size(), nv(), [&](std::size_t i) { return keys[i][0]; },
        [&](U32 a, U32 b) { return keys[a] != keys[b] ? keys[a] < keys[b] : a < b; }, off, items);
    int dup = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : dup)
    for (long long v = 0; v < static_cast<long long>(nv()); ++v)
      for (U32 i = off[v]; i + 1 < off[v + 1]; ++i)
        if (keys[items[i]] == keys[items[i + 1]]) dup = 1;
    if (dup) fail(kTopologyError, "duplicate face");
  }
  orient();
  const double diag = bbox_diagonal();
  const double tol = 1e-12 * diag * diag;
  long long first_small = static_cast<long long>(nf());
#pragma omp parallel for reduction(min : first_small)
  for (long long f = 0; f < static_cast<long long>(nf()); ++f)
    if (face_area(static_cast<Index>(f)) < tol && f < first_small) first_small = f;
  if (first_small < static_cast<long long>(nf()))
    fail(kDegeneracyError, "face " + std::to_string(first_small) + " has near-zero area");
  index();
}

// Breadth-first consistent orientation from face 0 (mesh.hpp:197-262): a face
// reached through an edge it traverses in the same direction as its
// predecessor is flipped (swap corners 1 and 2); a conflict on an already
// visited face means the surface is non-orientable.  The result is then
// flipped globally if the enclosed signed volume is negative.  Inputs whose
// faces are already consistent (every edge traversed in opposite directions)
// need no flips: for them only connectivity is checked, in parallel.
void Mesh::orient() {
  partner_ = pair_slots(faces_, nv());
  const std::vector<U32>& partner = partner_;
  flipped_.assign(faces_.size(), 0);
  std::vector<char>& flipped = flipped_;
  auto forward = [&](Index g, Index a, Index b) {
    const auto& t = faces_[g];
    for (int k = 0; k < 3; ++k)
      if (t[k] == a && t[(k + 1) % 3] == b) return true;
    return false;
  };
  int inconsistent = 0;
  const long long ns = static_cast<long long>(faces_.size()) * 3;
#pragma omp parallel for reduction(| : inconsistent)
  for (long long s = 0; s < ns; ++s) {
    const Index f = static_cast<Index>(s / 3);
    const int k = static_cast<int>(s % 3);
    if (forward(partner[s] / 3, faces_[f][k], faces_[f][(k + 1) % 3])) inconsistent = 1;
  }
  if (!inconsistent) {
    const Index nf = this->nf();
    std::vector<std::atomic<U32>> p(nf);
#pragma omp parallel for
    for (long long f = 0; f < static_cast<long long>(nf); ++f) p[f].store(static_cast<U32>(f), std::memory_order_relaxed);
#pragma omp parallel for
    for (long long s = 0; s < ns; ++s) {
      U32 a = static_cast<U32>(s / 3), b = partner[s] / 3;
      while (true) {
        a = uf_root(p, a);
        b = uf_root(p, b);
        if (a == b) break;
        if (a < b) std::swap(a, b);
        U32 expect = a;
        if (p[a].compare_exchange_strong(expect, b, std::memory_order_relaxed)) break;
      }
    }
    long long roots = 0;
#pragma omp parallel for reduction(+ : roots)
    for (long long f = 0; f < static_cast<long long>(nf); ++f) roots += uf_root(p, static_cast<U32>(f)) == f ? 1 : 0;
    if (roots != 1) fail(kTopologyError, "mesh has multiple connected components");
  } else {
    // Current corner-pair k of face f maps to an original slot: identity
    // when unflipped; after swap(t1,t2) the pairs (t0,t2),(t2,t1),(t1,t0) are
    // the original slots 2,1,0.
    auto orig_slot = [&](Index f, int k) { return 3 * f + (flipped[f] ? 2 - k : k); };
    std::vector<char> visited(faces_.size(), 0);
    std::vector<Index> queue;
    queue.reserve(faces_.size());
    queue.push_back(0);
    visited[0] = 1;
    std::size_t head = 0, reached = 1;
    while (head < queue.size()) {
      Index f = queue[head++];
      for (int k = 0; k < 3; ++k) {
        Index a = faces_[f][k], b = faces_[f][(k + 1) % 3];
        Index g = partner[orig_slot(f, k)] / 3;
        bool same = forward(g, a, b);
        if (!visited[g]) {
          if (same) {
            std::swap(faces_[g][1], faces_[g][2]);
            flipped[g] ^= 1;
          }
          visited[g] = 1;
          ++reached;
          queue.push_back(g);
        } else if (same) {
          fail(kTopologyError, "inconsistent orientation: surface is non-orientable");
        }
      }
    }
    if (reached != faces_.size()) fail(kTopologyError, "mesh has multiple connected components");
  }
  double vol = 0;  // sequential, in face order (the reference's rounding)
  for (const auto& t : faces_) vol += dot(pos_[t[0]], cross(pos_[t[1]], pos_[t[2]])) / 6.0;
  if (vol < 0) {
#pragma omp parallel for
    for (long long f = 0; f < static_cast<long long>(faces_.size()); ++f) {
      std::swap(faces_[f][1], faces_[f][2]);
      flipped_[f] ^= 1;
    }
  }
}

// Edges are numbered by first appearance over (face, corner) in order
// (mesh.hpp:272-293); vertex->face lists are in face order, vertex->vertex
// lists sorted.
void Mesh::index() {
  // Slot pairing of the final orientation, derived from orient()'s pairing of
  // the input corners: final corner pair k of face f is input slot
  // 3f + (flipped ? 2 - k : k).
  const std::size_t ns = faces_.size() * 3;
  std::vector<U32> partner(ns);
#pragma omp parallel for
  for (long long s = 0; s < static_cast<long long>(ns); ++s) {
    const std::size_t f = static_cast<std::size_t>(s) / 3;
    const int k = static_cast<int>(s % 3);
    const U32 orig = static_cast<U32>(3 * f + (flipped_[f] ? 2 - k : k));
    const U32 po = partner_[orig];
    const U32 g = po / 3, kg = po % 3;
    partner[s] = 3 * g + (flipped_[g] ? 2 - kg : kg);
  }
  std::vector<U32>().swap(partner_);
  std::vector<char>().swap(flipped_);
  // A slot opens its edge iff its partner comes later; edge ids are the
  // prefix count of opening slots (first appearance order).
  const int nthreads = 64;
  const std::size_t chunk = (ns + nthreads - 1) / nthreads;
  std::vector<U32> base(nthreads + 1, 0);
#pragma omp parallel for
  for (int t = 0; t < nthreads; ++t) {
    U32 c = 0;
    for (std::size_t s = t * chunk; s < std::min(ns, (t + 1) * chunk); ++s) c += partner[s] > s;
    base[t] = c;
  }
  base[nthreads] = 0;
  exclusive_scan(base);
  const Index ne = base[nthreads];
  edge_v_.resize(ne);
  edge_f_.resize(ne);
  face_e_.assign(faces_.size(), {kInvalid, kInvalid, kInvalid});
  std::vector<U32> slot_edge(ns);
#pragma omp parallel for
  for (int t = 0; t < nthreads; ++t) {
    U32 e = base[t];
    for (std::size_t s = t * chunk; s < std::min(ns, (t + 1) * chunk); ++s)
      if (partner[s] > s) {
        const Index f = static_cast<Index>(s / 3);
        const int k = static_cast<int>(s % 3);
        const Index a = faces_[f][k], b = faces_[f][(k + 1) % 3];
        edge_v_[e] = {std::min(a, b), std::max(a, b)};
        edge_f_[e] = {f, static_cast<Index>(partner[s] / 3)};
        slot_edge[s] = e++;
      }
  }
#pragma omp parallel for
  for (long long s = 0; s < static_cast<long long>(ns); ++s) {
    const U32 e = partner[s] > static_cast<U32>(s) ? slot_edge[s] : slot_edge[partner[s]];
    face_e_[s / 3][s % 3] = e;
  }
  const Index n = nv();
  bucket_sort(
      ns, n, [&](std::size_t s) { return faces_[s / 3][s % 3]; }, [](U32 a, U32 b) { return a < b; }, v2f_off_,
      v2f_);
#pragma omp parallel for
  for (long long i = 0; i < static_cast<long long>(ns); ++i) v2f_[i] /= 3;  // slot -> face (face order kept)
  bucket_sort(
      2 * static_cast<std::size_t>(ne), n,
      [&](std::size_t h) { return edge_v_[h / 2][h % 2]; },
      [&](U32 a, U32 b) { return edge_v_[a / 2][1 - a % 2] < edge_v_[b / 2][1 - b % 2]; }, v2v_off_, v2v_);
#pragma omp parallel for
  for (long long i = 0; i < static_cast<long long>(v2v_.size()); ++i) v2v_[i] = edge_v_[v2v_[i] / 2][1 - v2v_[i] % 2];
}

long Mesh::genus() const {
  long chi = euler();
  if ((2 - chi) % 2 != 0 || chi > 2)
    fail(kTopologyError, "euler characteristic " + std::to_string(chi) +
                             " is not that of a closed orientable surface");
  return (2 - chi) / 2;
}

double Mesh::bbox_diagonal() const {
  V3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
  for (const V3& q : pos_) {
    lo.x = std::min(lo.x, q.x);
    lo.y = std::min(lo.y, q.y);
    lo.z = std::min(lo.z, q.z);
    hi.x = std::max(hi.x, q.x);
    hi.y = std::max(hi.y, q.y);
    hi.z = std::max(hi.z, q.z);
  }
  return norm(hi - lo);
}

double Mesh::mean_edge_length() const {
  double total = 0;
  for (const auto& e : edge_v_) total += dist(pos_[e[0]], pos_[e[1]]);
  return edge_v_.empty() ? 0.0 : total / static_cast<double>(edge_v_.size());
}

// ---------------------------------------------------------------------------
// Generators.  Arithmetic is written in the same evaluation order as the
// reference so generated coordinates agree bit for bit (tests/test_mesh.py).

static constexpr double kPi = 3.14159265358979323846;

Mesh gen_torus(int major, int minor, double R, double r) {
  if (major < 3 || minor < 3) fail(kInvalidParameter, "torus needs at least 3 segments in each direction");
  if (!(R > r) || !(r > 0)) fail(kInvalidParameter, "torus needs R > r > 0");
  std::vector<V3> v;
  v.reserve(static_cast<std::size_t>(major) * minor);
  for (int i = 0; i < major; ++i) {
    const double theta = 2.0 * kPi * i / major;
    for (int j = 0; j < minor; ++j) {
      const double psi = 2.0 * kPi * j / minor;
      const double rad = R + r * std::cos(psi);
      v.push_back({rad * std::cos(theta), rad * std::sin(theta), r * std::sin(psi)});
    }
  }
  auto id = [&](int i, int j) { return static_cast<Index>((i % major) * minor + (j % minor)); };
  std::vector<std::array<Index, 3>> f;
  f.reserve(static_cast<std::size_t>(major) * minor * 2);
  for (int i = 0; i < major; ++i)
    for (int j = 0; j < minor; ++j) {
      f.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
      f.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
    }
  return Mesh(std::move(v), std::move(f));
}

Mesh perturb(const Mesh& m, double amplitude, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-amplitude, amplitude);
  std::vector<V3> v = m.positions();
  for (V3& q : v) {
    double dx = u(rng);
    double dy = u(rng);
    double dz = u(rng);
    q = q + V3{dx, dy, dz};
  }
  return Mesh(std::move(v), m.faces());
}

Mesh gen_torus_irregular(int major, int minor, double R, double r, double warp, double jitter,
                         unsigned seed) {
  if (major < 3 || minor < 3) fail(kInvalidParameter, "torus needs at least 3 segments in each direction");
  if (!(R > r) || !(r > 0)) fail(kInvalidParameter, "torus needs R > r > 0");
  if (warp < 0 || warp > 0.45) fail(kInvalidParameter, "warp must be in [0, 0.45]");
  std::vector<V3> v;
  for (int i = 0; i < major; ++i) {
    const double u = static_cast<double>(i) / major;
    const double theta = 2.0 * kPi * (u + warp / (2.0 * kPi) * std::sin(2.0 * kPi * u));
    for (int j = 0; j < minor; ++j) {
      const double psi = 2.0 * kPi * j / minor;
      const double rad = R + r * std::cos(psi);
      v.push_back({rad * std::cos(theta), rad * std::sin(theta), r * std::sin(psi)});
    }
  }
  auto id = [&](int i, int j) { return static_cast<Index>((i % major) * minor + (j % minor)); };
  std::vector<std::array<Index, 3>> f;
  for (int i = 0; i < major; ++i)
    for (int j = 0; j < minor; ++j) {
      f.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
      f.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
    }
  Mesh m(std::move(v), std::move(f));
  if (jitter > 0) m = perturb(m, jitter, seed);
  return m;
}

Mesh gen_icosphere(int subdivisions, double radius) {
  if (subdivisions < 0 || radius <= 0) fail(kInvalidParameter, "bad icosphere parameters");
  // Regular icosahedron: the 12 cyclic permutations of (0, +-1, +-phi).
  const double g = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<V3> v = {{-1, g, 0},  {1, g, 0},  {-1, -g, 0}, {1, -g, 0}, {0, -1, g},  {0, 1, g},
                       {0, -1, -g}, {0, 1, -g}, {g, 0, -1},  {g, 0, 1},  {-g, 0, -1}, {-g, 0, 1}};
  std::vector<std::array<Index, 3>> f = {
      {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
      {11, 10, 2}, {10, 7, 6}, {7, 1, 8},  {3, 9, 4},  {3, 4, 2},   {3, 2, 6}, {3, 6, 8},
      {3, 8, 9},  {4, 9, 5},  {2, 4, 11},  {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
  for (int s = 0; s < subdivisions; ++s) {
    std::unordered_map<std::uint64_t, Index> cache;
    auto midpoint = [&](Index a, Index b) {
      const std::uint64_t key = (static_cast<std::uint64_t>(std::min(a, b)) << 32) | std::max(a, b);
      auto it = cache.find(key);
      if (it != cache.end()) return it->second;
      const Index id = static_cast<Index>(v.size());
      v.push_back((v[a] + v[b]) * 0.5);
      cache.emplace(key, id);
      return id;
    };
    std::vector<std::array<Index, 3>> next;
    next.reserve(f.size() * 4);
    for (const auto& t : f) {
      const Index m01 = midpoint(t[0], t[1]);
      const Index m12 = midpoint(t[1], t[2]);
      const Index m20 = midpoint(t[2], t[0]);
      next.push_back({t[0], m01, m20});
      next.push_back({t[1], m12, m01});
      next.push_back({t[2], m20, m12});
      next.push_back({m01, m12, m20});
    }
    f.swap(next);
  }
  for (V3& q : v) q = unit(q) * radius;
  return Mesh(std::move(v), std::move(f));
}

namespace {

// Boundary of a union of unit lattice cells, every exposed cell face split
// into subdiv x subdiv quads of two triangles (generators.hpp:95 contract).
// Vertices are numbered by first use in the emission order below.
Mesh voxel_boundary(const int lo[3], const int hi[3], const std::function<bool(int, int, int)>& solid,
                    int subdiv, double cell) {
  std::vector<V3> v;
  std::unordered_map<std::uint64_t, Index> ids;
  const double h = cell / subdiv;
  auto vert = [&](long x, long y, long z) {
    const std::uint64_t bias = 1u << 20;
    const std::uint64_t key = (static_cast<std::uint64_t>(x + bias) << 42) |
                              (static_cast<std::uint64_t>(y + bias) << 21) |
                              static_cast<std::uint64_t>(z + bias);
    auto [it, fresh] = ids.try_emplace(key, static_cast<Index>(v.size()));
    if (fresh) v.push_back({x * h, y * h, z * h});
    return it->second;
  };
  std::vector<std::array<Index, 3>> f;
  static const int dirs[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
  const long S = subdiv;
  for (int cx = lo[0]; cx < hi[0]; ++cx)
    for (int cy = lo[1]; cy < hi[1]; ++cy)
      for (int cz = lo[2]; cz < hi[2]; ++cz) {
        if (!solid(cx, cy, cz)) continue;
        for (const auto& d : dirs) {
          if (solid(cx + d[0], cy + d[1], cz + d[2])) continue;
          // Origin of the exposed face on the sub-lattice; the face lies on
          // the far plane of the cell along a positive normal.
          const long o[3] = {(cx + (d[0] > 0)) * S, (cy + (d[1] > 0)) * S, (cz + (d[2] > 0)) * S};
          int u[3] = {0, 0, 0}, w[3] = {0, 0, 0};
          if (d[0] != 0) {
            u[1] = 1;
            w[2] = 1;
          } else if (d[1] != 0) {
            u[0] = 1;
            w[2] = 1;
          } else {
            u[0] = 1;
            w[1] = 1;
          }
          for (int a = 0; a < subdiv; ++a)
            for (int b = 0; b < subdiv; ++b) {
              auto corner = [&](int da, int db) {
                return vert(o[0] + (a + da) * u[0] + (b + db) * w[0], o[1] + (a + da) * u[1] + (b + db) * w[1],
                            o[2] + (a + da) * u[2] + (b + db) * w[2]);
              };
              const Index c00 = corner(0, 0);
              const Index c10 = corner(1, 0);
              const Index c11 = corner(1, 1);
              const Index c01 = corner(0, 1);
              f.push_back({c00, c10, c11});
              f.push_back({c00, c11, c01});
            }
        }
      }
  return Mesh(std::move(v), std::move(f));
}

}  // namespace

Mesh gen_genus_plate(int genus, int resolution, double cell) {
  if (genus < 1) fail(kInvalidParameter, "plate genus must be positive");
  if (resolution < 1) fail(kInvalidParameter, "resolution must be positive");
  if (!(cell > 0)) fail(kInvalidParameter, "cell size must be positive");
  const int hole = 2, gap = 2, depth = 1;
  const int cols = genus * hole + (genus + 1) * gap;
  const int rows = hole + 2 * gap;
  auto solid = [=](int x, int y, int z) {
    if (x < 0 || x >= cols || y < 0 || y >= rows || z < 0 || z >= depth) return false;
    if (y >= gap && y < gap + hole) {
      const int rel = x - gap, pitch = hole + gap;
      if (rel >= 0 && rel % pitch < hole && rel / pitch < genus) return false;
    }
    return true;
  };
  const int lo[3] = {0, 0, 0}, hi[3] = {cols, rows, depth};
  return voxel_boundary(lo, hi, solid, resolution, cell);
}

Mesh gen_genus(int genus, int resolution) {
  if (genus < 0) fail(kInvalidParameter, "genus must be non-negative");
  if (resolution < 1) fail(kInvalidParameter, "resolution must be positive");
  if (genus == 0) return gen_icosphere(std::min(resolution + 1, 6), 2.0);
  return gen_genus_plate(genus, resolution, 1.0);
}

Mesh gen_limb_star(int limbs, int resolution, int limb_length) {
  if (limbs < 1 || limbs > 6) fail(kInvalidParameter, "limb count must be in 1..6");
  if (limb_length < 1) fail(kInvalidParameter, "limb length must be positive");
  if (resolution < 1) fail(kInvalidParameter, "resolution must be positive");
  const int L = limb_length;
  auto arm = [L](int along, int s, int t) {
    return along >= 1 && along <= L && (s == -1 || s == 0) && (t == -1 || t == 0);
  };
  auto solid = [=](int x, int y, int z) {
    if ((x == -1 || x == 0) && (y == -1 || y == 0) && (z == -1 || z == 0)) return true;
    return (limbs > 0 && arm(x, y, z)) || (limbs > 1 && arm(-x - 1, y, z)) ||
           (limbs > 2 && arm(y, x, z)) || (limbs > 3 && arm(-y - 1, x, z)) ||
           (limbs > 4 && arm(z, x, y)) || (limbs > 5 && arm(-z - 1, x, y));
  };
  const int lo[3] = {-L - 2, -L - 2, -L - 2}, hi[3] = {L + 2, L + 2, L + 2};
  return voxel_boundary(lo, hi, solid, resolution, 1.0);
}

Mesh gen_coin(int rings, int sectors, double radius, double thickness) {
  if (rings < 1 || sectors < 3 || radius <= 0 || thickness <= 0) fail(kInvalidParameter, "bad coin parameters");
  std::vector<V3> v;
  std::vector<std::array<Index, 3>> f;
  auto disk = [&](double z) {
    const Index center = static_cast<Index>(v.size());
    v.push_back({0, 0, z});
    std::vector<std::vector<Index>> ring(rings);
    for (int i = 1; i <= rings; ++i) {
      const double rad = radius * i / rings;
      for (int j = 0; j < sectors; ++j) {
        const double ang = 2.0 * kPi * j / sectors;
        ring[i - 1].push_back(static_cast<Index>(v.size()));
        v.push_back({rad * std::cos(ang), rad * std::sin(ang), z});
      }
    }
    for (int j = 0; j < sectors; ++j) f.push_back({center, ring[0][j], ring[0][(j + 1) % sectors]});
    for (int i = 1; i < rings; ++i)
      for (int j = 0; j < sectors; ++j) {
        const Index a = ring[i - 1][j], b = ring[i - 1][(j + 1) % sectors];
        const Index c = ring[i][j], d = ring[i][(j + 1) % sectors];
        f.push_back({a, c, d});
        f.push_back({a, d, b});
      }
    return ring.back();
  };
  const std::vector<Index> top = disk(thickness / 2);
  const std::vector<Index> bottom = disk(-thickness / 2);
  for (int j = 0; j < sectors; ++j) {
    const Index a = top[j], b = top[(j + 1) % sectors];
    const Index c = bottom[j], d = bottom[(j + 1) % sectors];
    f.push_back({a, c, d});
    f.push_back({a, d, b});
  }
  return Mesh(std::move(v), std::move(f));
}

// Gyroid surface by marching tetrahedra over a periodic lattice.  The implicit
// function is sampled on an (n+1)^3 grid spanning `periods` periods (2*pi each)
// and the solid {g > level} is clipped to the sampling cube by min() with the
// cube's signed distance, so the extracted level set is closed.  Each cube is
// split into six tetrahedra sharing the main diagonal; vertices live on grid
// edges (deduplicated by edge key), so the output is a watertight 2-manifold
// whenever no sample equals the level (samples are nudged off it).
Mesh gen_gyroid(int periods, int res, double level, double scale) {
  if (periods < 1 || res < 4 || !(scale > 0)) fail(kInvalidParameter, "bad gyroid parameters");
  const int n = periods * res;  // cells per axis
  const double span = 2.0 * kPi * periods;
  const double h = span / n;
  const double margin = 0.5 * h;  // keeps the cube clip strictly inside the grid
  auto field = [&](int i, int j, int k) {
    const double x = i * h, y = j * h, z = k * h;
    double g = std::sin(x) * std::cos(y) + std::sin(y) * std::cos(z) + std::sin(z) * std::cos(x) - level;
    // Clip against the cube [margin, span - margin]^3 (negative outside).
    double c = std::min({x - margin, span - margin - x, y - margin, span - margin - y, z - margin,
                         span - margin - z});
    double s = std::min(g, c);
    if (s == 0.0) s = 1e-12;
    return s;
  };
  const int N1 = n + 1;
  std::vector<double> val(static_cast<std::size_t>(N1) * N1 * N1);
  auto gid = [&](int i, int j, int k) { return (static_cast<std::size_t>(i) * N1 + j) * N1 + k; };
  for (int i = 0; i <= n; ++i)
    for (int j = 0; j <= n; ++j)
      for (int k = 0; k <= n; ++k) val[gid(i, j, k)] = field(i, j, k);

  std::vector<V3> v;
  std::unordered_map<std::uint64_t, Index> edge_vertex;
  auto vertex_on = [&](std::size_t a, std::size_t b) {
    if (a > b) std::swap(a, b);
    const std::uint64_t key = static_cast<std::uint64_t>(a) * (static_cast<std::uint64_t>(N1) * N1 * N1) + b;
    auto [it, fresh] = edge_vertex.try_emplace(key, static_cast<Index>(v.size()));
    if (fresh) {
      const double fa = val[a], fb = val[b];
      // Crossings are kept off the grid nodes so no triangle degenerates.
      const double t = std::min(0.98, std::max(0.02, fa / (fa - fb)));
      auto coord = [&](std::size_t g) {
        const int k = static_cast<int>(g % N1), j = static_cast<int>((g / N1) % N1),
                  i = static_cast<int>(g / (static_cast<std::size_t>(N1) * N1));
        return V3{i * h, j * h, k * h};
      };
      v.push_back(lerp(coord(a), coord(b), t) * scale);
    }
    return it->second;
  };
  std::vector<std::array<Index, 3>> f;
  // Six tetrahedra around the cube diagonal 0-7 (corner bits: x=4,y=2,z=1).
  static const int tets[6][4] = {{0, 7, 4, 6}, {0, 7, 6, 2}, {0, 7, 2, 3},
                                 {0, 7, 3, 1}, {0, 7, 1, 5}, {0, 7, 5, 4}};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        std::size_t c[8];
        for (int b = 0; b < 8; ++b) c[b] = gid(i + ((b >> 2) & 1), j + ((b >> 1) & 1), k + (b & 1));
        for (const auto& t : tets) {
          std::size_t q[4] = {c[t[0]], c[t[1]], c[t[2]], c[t[3]]};
          int in[4], out[4], ni = 0, no = 0;
          for (int m = 0; m < 4; ++m) (val[q[m]] > 0 ? in[ni++] : out[no++]) = m;
          if (ni == 0 || ni == 4) continue;
          if (ni == 1 || ni == 3) {
            // One vertex separated from three: one triangle.
            const int lone = ni == 1 ? in[0] : out[0];
            int o3[3], p = 0;
            for (int m = 0; m < 4; ++m)
              if (m != lone) o3[p++] = m;
            f.push_back({vertex_on(q[lone], q[o3[0]]), vertex_on(q[lone], q[o3[1]]),
                         vertex_on(q[lone], q[o3[2]])});
          } else {
            // Two and two: a quad split into two triangles.
            const Index a = vertex_on(q[in[0]], q[out[0]]), b = vertex_on(q[in[0]], q[out[1]]);
            const Index c2 = vertex_on(q[in[1]], q[out[1]]), d = vertex_on(q[in[1]], q[out[0]]);
            f.push_back({a, b, c2});
            f.push_back({a, c2, d});
          }
        }
      }
  // Marching tetrahedra emits faces with arbitrary winding; orientation is
  // normalized by the Mesh constructor.  Only the largest connected component
  // is kept (the clipped gyroid solid is connected; tiny slivers are not).
  // Component labelling by union-find over shared edges.
  std::vector<Index> parent(f.size());
  for (Index i = 0; i < f.size(); ++i) parent[i] = i;
  std::function<Index(Index)> find = [&](Index a) {
    while (parent[a] != a) a = parent[a] = parent[parent[a]];
    return a;
  };
  std::unordered_map<std::uint64_t, Index> first_face;
  for (Index fi = 0; fi < f.size(); ++fi)
    for (int k = 0; k < 3; ++k) {
      Index a = f[fi][k], b = f[fi][(k + 1) % 3];
      const std::uint64_t key = (static_cast<std::uint64_t>(std::min(a, b)) << 32) | std::max(a, b);
      auto [it, fresh] = first_face.try_emplace(key, fi);
      if (!fresh) {
        Index ra = find(fi), rb = find(it->second);
        if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
      }
    }
  std::unordered_map<Index, std::size_t> comp_size;
  for (Index fi = 0; fi < f.size(); ++fi) ++comp_size[find(fi)];
  Index best = 0;
  std::size_t best_n = 0;
  for (auto& [root, cnt] : comp_size)
    if (cnt > best_n || (cnt == best_n && root < best)) {
      best = root;
      best_n = cnt;
    }
  std::vector<std::array<Index, 3>> kept;
  kept.reserve(best_n);
  for (Index fi = 0; fi < f.size(); ++fi)
    if (find(fi) == best) kept.push_back(f[fi]);
  return Mesh(std::move(v), std::move(kept));
}

namespace {
std::vector<std::string> split_spec(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ':')) out.push_back(tok);
  return out;
}
}  // namespace

Mesh make_mesh(const std::string& spec) {
  auto p = split_spec(spec);
  if (p.empty()) fail(kInvalidParameter, "empty mesh spec");
  auto I = [&](std::size_t i) {
    if (i >= p.size()) fail(kInvalidParameter, "mesh spec " + spec + " is missing fields");
    return std::atoi(p[i].c_str());
  };
  auto D = [&](std::size_t i) {
    if (i >= p.size()) fail(kInvalidParameter, "mesh spec " + spec + " is missing fields");
    return std::atof(p[i].c_str());
  };
  const std::string& k = p[0];
  if (k == "dtm") return read_dtm(spec.substr(4));
  if (k == "file") return load_mesh(spec.substr(5), 0);
  if (k == "torus") return gen_torus(I(1), I(2), D(3), D(4));
  if (k == "torus_irr") return gen_torus_irregular(I(1), I(2), D(3), D(4), D(5), D(6), static_cast<unsigned>(I(7)));
  if (k == "genus") return gen_genus(I(1), I(2));
  if (k == "plate") return gen_genus_plate(I(1), I(2), D(3));
  if (k == "icosphere") return gen_icosphere(I(1), D(2));
  if (k == "limbstar") return gen_limb_star(I(1), I(2), I(3));
  if (k == "coin") return gen_coin(I(1), I(2), D(3), D(4));
  if (k == "gyroid") return gen_gyroid(I(1), I(2), D(3), D(4));
  fail(kInvalidParameter, "unknown mesh spec " + spec);
}

// ---------------------------------------------------------------------------
// IO

namespace {

std::string content_line(std::istream& in) {
  std::string line;
  while (std::getline(in, line)) {
    auto i = line.find_first_not_of(" \t\r\n");
    if (i == std::string::npos || line[i] == '#') continue;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    return line;
  }
  fail(kParseError, "unexpected end of file");
}

Mesh read_off(std::istream& in) {
  {
    std::istringstream hs(content_line(in));
    std::string tag;
    hs >> tag;
    if (tag != "OFF") fail(kParseError, "missing OFF header");
  }
  std::size_t nv = 0, nf = 0, ne = 0;
  {
    std::istringstream cs(content_line(in));
    if (!(cs >> nv >> nf >> ne)) fail(kParseError, "bad OFF count line");
  }
  std::vector<V3> v(nv);
  for (auto& q : v) {
    std::istringstream ls(content_line(in));
    if (!(ls >> q.x >> q.y >> q.z)) fail(kParseError, "bad OFF vertex line");
  }
  std::vector<std::array<Index, 3>> f;
  f.reserve(nf);
  for (std::size_t i = 0; i < nf; ++i) {
    std::istringstream ls(content_line(in));
    std::size_t arity = 0;
    if (!(ls >> arity)) fail(kParseError, "bad OFF face line");
    if (arity != 3) fail(kParseError, "only triangle faces are supported");
    std::array<Index, 3> t{};
    for (auto& x : t)
      if (!(ls >> x)) fail(kParseError, "bad OFF face line");
    f.push_back(t);
  }
  return Mesh(std::move(v), std::move(f));
}

Mesh read_obj(std::istream& in) {
  std::vector<V3> v;
  std::vector<std::array<Index, 3>> f;
  std::string line;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag)) continue;
    if (tag == "v") {
      V3 q;
      if (!(ls >> q.x >> q.y >> q.z)) fail(kParseError, "bad OBJ vertex line");
      v.push_back(q);
    } else if (tag == "f") {
      std::vector<Index> poly;
      std::string tok;
      while (ls >> tok) {
        const auto slash = tok.find('/');
        long idx = std::stol(slash == std::string::npos ? tok : tok.substr(0, slash));
        if (idx < 0) idx = static_cast<long>(v.size()) + idx + 1;
        if (idx < 1 || idx > static_cast<long>(v.size())) fail(kParseError, "OBJ face index out of range");
        poly.push_back(static_cast<Index>(idx - 1));
      }
      if (poly.size() != 3) fail(kParseError, "only triangle faces are supported");
      f.push_back({poly[0], poly[1], poly[2]});
    }
  }
  if (v.empty() || f.empty()) fail(kParseError, "OBJ contains no triangle mesh");
  return Mesh(std::move(v), std::move(f));
}

std::size_t ply_size(const std::string& t) {
  if (t == "char" || t == "uchar" || t == "int8" || t == "uint8") return 1;
  if (t == "short" || t == "ushort" || t == "int16" || t == "uint16") return 2;
  if (t == "int" || t == "uint" || t == "int32" || t == "uint32" || t == "float" || t == "float32") return 4;
  if (t == "double" || t == "float64" || t == "int64" || t == "uint64") return 8;
  fail(kParseError, "unknown PLY type " + t);
}

double ply_bin(std::istream& in, const std::string& t) {
  unsigned char b[8];
  const std::size_t n = ply_size(t);
  in.read(reinterpret_cast<char*>(b), static_cast<std::streamsize>(n));
  if (!in) fail(kParseError, "truncated PLY binary payload");
  auto as = [&](auto x) {
    std::memcpy(&x, b, sizeof x);
    return static_cast<double>(x);
  };
  if (t == "float" || t == "float32") return as(float{});
  if (t == "double" || t == "float64") return as(double{});
  if (t == "char" || t == "int8") return as(std::int8_t{});
  if (t == "uchar" || t == "uint8") return as(std::uint8_t{});
  if (t == "short" || t == "int16") return as(std::int16_t{});
  if (t == "ushort" || t == "uint16") return as(std::uint16_t{});
  if (t == "int" || t == "int32") return as(std::int32_t{});
  if (t == "uint" || t == "uint32") return as(std::uint32_t{});
  if (t == "int64") return as(std::int64_t{});
  return as(std::uint64_t{});
}

Mesh read_ply(std::istream& in) {
  struct Prop {
    std::string name, type, count_type;
    bool list = false;
  };
  struct Elem {
    std::string name;
    std::size_t count = 0;
    std::vector<Prop> props;
  };
  std::string line;
  if (!std::getline(in, line)) fail(kParseError, "empty PLY file");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != "ply") fail(kParseError, "missing ply magic");
  bool binary = false;
  std::vector<Elem> elems;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ls(line);
    std::string tag;
    ls >> tag;
    if (tag == "comment" || tag == "obj_info" || tag.empty()) continue;
    if (tag == "format") {
      std::string fmt;
      ls >> fmt;
      if (fmt == "ascii") binary = false;
      else if (fmt == "binary_little_endian") binary = true;
      else fail(kParseError, "unsupported PLY format " + fmt);
    } else if (tag == "element") {
      Elem e;
      ls >> e.name >> e.count;
      elems.push_back(e);
    } else if (tag == "property") {
      if (elems.empty()) fail(kParseError, "PLY property before element");
      Prop pr;
      std::string t;
      ls >> t;
      if (t == "list") {
        pr.list = true;
        ls >> pr.count_type >> pr.type >> pr.name;
      } else {
        pr.type = t;
        ls >> pr.name;
      }
      elems.back().props.push_back(pr);
    } else if (tag == "end_header") {
      break;
    } else {
      fail(kParseError, "unexpected PLY header line: " + line);
    }
  }
  auto scalar = [&](const std::string& t) {
    if (binary) return ply_bin(in, t);
    double x;
    if (!(in >> x)) fail(kParseError, "truncated PLY ascii payload");
    return x;
  };
  std::vector<V3> v;
  std::vector<std::array<Index, 3>> f;
  for (const Elem& e : elems) {
    if (e.name == "vertex") {
      int ix = -1, iy = -1, iz = -1;
      for (std::size_t i = 0; i < e.props.size(); ++i) {
        if (e.props[i].list) fail(kParseError, "list property on PLY vertex element");
        if (e.props[i].name == "x") ix = static_cast<int>(i);
        if (e.props[i].name == "y") iy = static_cast<int>(i);
        if (e.props[i].name == "z") iz = static_cast<int>(i);
      }
      if (ix < 0 || iy < 0 || iz < 0) fail(kParseError, "PLY vertex element lacks x/y/z");
      v.resize(e.count);
      std::vector<double> row(e.props.size());
      for (std::size_t i = 0; i < e.count; ++i) {
        for (std::size_t k = 0; k < e.props.size(); ++k) row[k] = scalar(e.props[k].type);
        v[i] = {row[ix], row[iy], row[iz]};
      }
    } else {
      const bool faces = e.name == "face";
      if (faces) f.reserve(e.count);
      for (std::size_t i = 0; i < e.count; ++i)
        for (const auto& pr : e.props) {
          if (!pr.list) {
            scalar(pr.type);
            continue;
          }
          const std::size_t arity = static_cast<std::size_t>(scalar(pr.count_type));
          std::vector<long> poly(arity);
          for (auto& x : poly) x = static_cast<long>(scalar(pr.type));
          if (faces && (pr.name == "vertex_indices" || pr.name == "vertex_index")) {
            if (arity != 3) fail(kParseError, "only triangle faces are supported");
            for (long x : poly)
              if (x < 0 || x >= static_cast<long>(v.size())) fail(kParseError, "PLY face index out of range");
            f.push_back({static_cast<Index>(poly[0]), static_cast<Index>(poly[1]), static_cast<Index>(poly[2])});
          }
        }
    }
  }
  if (v.empty() || f.empty()) fail(kParseError, "PLY contains no triangle mesh");
  return Mesh(std::move(v), std::move(f));
}

}  // namespace

Mesh load_mesh(const std::string& path, int format) {
  if (format == 0) {
    const auto dot = path.find_last_of('.');
    if (dot == std::string::npos) fail(kParseError, "cannot infer mesh format from " + path);
    std::string ext = path.substr(dot + 1);
    for (char& c : ext) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    if (ext == "off") format = 1;
    else if (ext == "obj") format = 2;
    else if (ext == "ply") format = 3;
    else if (ext == "dtm") return read_dtm(path);
    else fail(kParseError, "unsupported mesh extension ." + ext);
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(kParseError, "cannot open " + path);
  switch (format) {
    case 1: return read_off(in);
    case 2: return read_obj(in);
    case 3: return read_ply(in);
    default: fail(kParseError, "unsupported format");
  }
}

Mesh read_dtm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(kParseError, "cannot open " + path);
  char magic[4];
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "DTM1", 4) != 0) fail(kParseError, "bad dtm magic");
  std::uint32_t nv = 0, nf = 0;
  in.read(reinterpret_cast<char*>(&nv), 4);
  in.read(reinterpret_cast<char*>(&nf), 4);
  std::vector<V3> v(nv);
  in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(24) * nv);
  std::vector<std::array<Index, 3>> f(nf);
  in.read(reinterpret_cast<char*>(f.data()), static_cast<std::streamsize>(12) * nf);
  if (!in) fail(kParseError, "truncated dtm");
  return Mesh(std::move(v), std::move(f));
}

void write_dtm(const Mesh& m, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(kParseError, "cannot write " + path);
  out.write("DTM1", 4);
  const std::uint32_t nv = m.nv(), nf = m.nf();
  out.write(reinterpret_cast<const char*>(&nv), 4);
  out.write(reinterpret_cast<const char*>(&nf), 4);
  out.write(reinterpret_cast<const char*>(m.positions().data()), static_cast<std::streamsize>(24) * nv);
  out.write(reinterpret_cast<const char*>(m.faces().data()), static_cast<std::streamsize>(12) * nf);
}

void save_ply(const Mesh& m, const std::string& path, const std::vector<double>* scalar, bool binary) {
  if (scalar && scalar->size() != m.nv()) fail(kDimensionMismatch, "scalar attribute size mismatch");
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(kParseError, "cannot write " + path);
  out << "ply\nformat " << (binary ? "binary_little_endian" : "ascii") << " 1.0\n";
  out << "element vertex " << m.nv() << "\nproperty double x\nproperty double y\nproperty double z\n";
  if (scalar) out << "property double quality\n";
  out << "element face " << m.nf() << "\nproperty list uchar int vertex_indices\nend_header\n";
  out.precision(17);
  for (Index v = 0; v < m.nv(); ++v) {
    const V3& q = m.p(v);
    if (binary) {
      out.write(reinterpret_cast<const char*>(&q), 24);
      if (scalar) out.write(reinterpret_cast<const char*>(&(*scalar)[v]), 8);
    } else {
      out << q.x << " " << q.y << " " << q.z;
      if (scalar) out << " " << (*scalar)[v];
      out << "\n";
    }
  }
  for (Index fi = 0; fi < m.nf(); ++fi) {
    const auto& t = m.face(fi);
    if (binary) {
      const unsigned char three = 3;
      const std::int32_t idx[3] = {static_cast<std::int32_t>(t[0]), static_cast<std::int32_t>(t[1]),
                                   static_cast<std::int32_t>(t[2])};
      out.write(reinterpret_cast<const char*>(&three), 1);
      out.write(reinterpret_cast<const char*>(idx), 12);
    } else {
      out << "3 " << t[0] << " " << t[1] << " " << t[2] << "\n";
    }
  }
}

void save_obj(const Mesh& m, const std::string& path) {
  std::ofstream out(path);
  if (!out) fail(kParseError, "cannot write " + path);
  out.precision(17);
  for (const V3& q : m.positions()) out << "v " << q.x << " " << q.y << " " << q.z << "\n";
  for (const auto& t : m.faces()) out << "f " << t[0] + 1 << " " << t[1] + 1 << " " << t[2] + 1 << "\n";
}

}  // namespace dtb
