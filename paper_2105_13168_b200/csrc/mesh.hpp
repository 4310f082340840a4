// Host-side triangle mesh: validation, orientation, topology indices,
// synthetic generators and file IO.  Semantics follow the reference
// (proj/include/difftopo/mesh.hpp:150-324, generators.hpp, mesh_io.hpp) so
// that vertex, face and edge numbering -- which appear in every output of the
// initial pass (loop anchors, isoline chaining order, event vertex sets) --
// are identical.  Construction is sort-based instead of hash-based so that
// multi-million-face meshes index in well under a second.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace dtb {

using Index = std::uint32_t;
inline constexpr Index kInvalid = 0xFFFFFFFFu;

// Error taxonomy of the reference (errors.hpp:8-33); the C-ABI maps each to a
// stable integer code (include/difftopo_b200.h).
enum ErrorCode : int {
  kOk = 0,
  kParseError = 1,
  kTopologyError = 2,
  kDegeneracyError = 3,
  kInvalidParameter = 4,
  kDimensionMismatch = 5,
  kEmptySeed = 6,
  kZeroColumn = 7,
  kInvalidSplit = 8,
  kInvalidMerge = 9,
  kNumericalBlowup = 10,
  kMaxStepsExceeded = 11,
  kUnreachable = 12,
  kStallError = 13,
  kLoopError = 14,
  kInconsistentLog = 15,
  kCudaError = 100,
  kCapacityExceeded = 101,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

struct V3 {
  double x = 0, y = 0, z = 0;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 operator/(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline double dist(V3 a, V3 b) { return norm(a - b); }
inline V3 lerp(V3 a, V3 b, double t) { return a + (b - a) * t; }
inline V3 unit(V3 a) {
  double n = norm(a);
  return n > 0 ? a / n : V3{};
}

class Mesh {
 public:
  Mesh() = default;
  // Validates a triangle soup (mesh.hpp:150 semantics): drops unreferenced
  // vertices, rejects duplicate / degenerate / open / non-manifold /
  // non-orientable / disconnected input, orients faces consistently and
  // outward, then builds edge, face-edge, vertex-face and vertex-vertex indices.
  Mesh(std::vector<V3> vertices, std::vector<std::array<Index, 3>> faces);

  // Trusted assembly from indices built elsewhere (the device builder,
  // csrc/meshbuild.cu), with the same numbering; no validation.
  static Mesh from_index(std::vector<V3> pos, std::vector<std::array<Index, 3>> faces,
                         std::vector<std::array<Index, 2>> edge_v, std::vector<std::array<Index, 2>> edge_f,
                         std::vector<std::array<Index, 3>> face_e, std::vector<std::uint32_t> v2f_off,
                         std::vector<Index> v2f, std::vector<std::uint32_t> v2v_off, std::vector<Index> v2v) {
    Mesh m;
    m.pos_ = std::move(pos);
    m.faces_ = std::move(faces);
    m.edge_v_ = std::move(edge_v);
    m.edge_f_ = std::move(edge_f);
    m.face_e_ = std::move(face_e);
    m.v2f_off_ = std::move(v2f_off);
    m.v2f_ = std::move(v2f);
    m.v2v_off_ = std::move(v2v_off);
    m.v2v_ = std::move(v2v);
    return m;
  }

  Index nv() const { return static_cast<Index>(pos_.size()); }
  Index nf() const { return static_cast<Index>(faces_.size()); }
  Index ne() const { return static_cast<Index>(edge_v_.size()); }
  long genus() const;
  long euler() const { return static_cast<long>(nv()) - static_cast<long>(ne()) + static_cast<long>(nf()); }

  const std::vector<V3>& positions() const { return pos_; }
  const std::vector<std::array<Index, 3>>& faces() const { return faces_; }
  const V3& p(Index v) const { return pos_[v]; }
  const std::array<Index, 3>& face(Index f) const { return faces_[f]; }
  const std::array<Index, 2>& edge_vertices(Index e) const { return edge_v_[e]; }
  const std::array<Index, 2>& edge_faces(Index e) const { return edge_f_[e]; }
  const std::array<Index, 3>& face_edges(Index f) const { return face_e_[f]; }
  Index opposite_face(Index e, Index f) const {
    return edge_f_[e][0] == f ? edge_f_[e][1] : edge_f_[e][0];
  }
  // CSR adjacency (offsets have nv()+1 entries).
  const std::vector<std::uint32_t>& v2f_off() const { return v2f_off_; }
  const std::vector<Index>& v2f() const { return v2f_; }
  const std::vector<std::uint32_t>& v2v_off() const { return v2v_off_; }
  const std::vector<Index>& v2v() const { return v2v_; }

  double face_area(Index f) const {
    const auto& t = faces_[f];
    return 0.5 * norm(cross(pos_[t[1]] - pos_[t[0]], pos_[t[2]] - pos_[t[0]]));
  }
  double bbox_diagonal() const;
  double mean_edge_length() const;

 private:
  void orient();
  void index();

  std::vector<V3> pos_;
  std::vector<std::array<Index, 3>> faces_;
  std::vector<std::array<Index, 2>> edge_v_, edge_f_;
  std::vector<std::array<Index, 3>> face_e_;
  std::vector<std::uint32_t> v2f_off_, v2v_off_;
  std::vector<Index> v2f_, v2v_;
  std::vector<std::uint32_t> partner_;  // construction scratch: input-corner slot pairing
  std::vector<char> flipped_;           // construction scratch: faces flipped by orient()
};

// --- synthetic generators (generators.hpp) ---------------------------------
Mesh gen_torus(int major, int minor, double R, double r);
Mesh gen_torus_irregular(int major, int minor, double R, double r, double warp, double jitter,
                         unsigned seed);
Mesh gen_icosphere(int subdivisions, double radius);
Mesh gen_genus(int genus, int resolution);
Mesh gen_limb_star(int limbs, int resolution, int limb_length);
Mesh gen_coin(int rings, int sectors, double radius, double thickness);
Mesh perturb(const Mesh& m, double amplitude, unsigned seed);
// New generators for the large benchmark configurations (not in the reference):
//   gen_genus_plate: generate_genus_g's slab with g through-holes, scaled so a
//     lattice cell spans `cell` model units (reference fixes cell = 1).
//   gen_gyroid: marching-tetrahedra surface of the gyroid level set
//     sin x cos y + sin y cos z + sin z cos x = level over `periods`^3 cells,
//     closed by intersecting with a cube, sampled at `res` points per period.
Mesh gen_genus_plate(int genus, int resolution, double cell);
Mesh gen_gyroid(int periods, int res, double level, double scale);
// Spec strings shared with oracle/ref_driver.cpp (torus:M:m:R:r, genus:g:res, ...).
Mesh make_mesh(const std::string& spec);

// --- IO (mesh_io.hpp) -------------------------------------------------------
Mesh load_mesh(const std::string& path, int format /*0 auto,1 off,2 obj,3 ply*/);
Mesh read_dtm(const std::string& path);
void write_dtm(const Mesh& m, const std::string& path);
void save_ply(const Mesh& m, const std::string& path, const std::vector<double>* scalar, bool binary);
void save_obj(const Mesh& m, const std::string& path);

}  // namespace dtb
