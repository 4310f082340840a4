// oracle/difftopo_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference initial pass (arXiv 2105.13168 artifact,
// /root/reference/proj/include/difftopo), used by tests/ and by bench.py's
// cpu_baseline as the checker -- never linked into the product.  It is written
// for clarity at small sizes: every layer is a dense row of V doubles (0 =
// absent), the frontier is a bitmap, and all loops run in the reference's
// order so every floating-point operation rounds identically:
//
//   assemble()        operators.hpp:33-70   (triplets + std::sort + sum, exact)
//   seed_ball()       diffusion.hpp:134-158
//   advance()         diffusion.hpp:242-367 (rates :313 and :343, clamp, prune,
//                                             normalize_columns layer_field.hpp:143)
//   front()           diffusion.hpp:398-470 extract_front
//   collisions()      diffusion.hpp:475-526 detect_collisions
//   split()/merge()   diffusion.hpp:642-759, layer_field.hpp:155-235
//   front_loop()      diffusion.hpp:606-629 + isoline.hpp:30-103
//   check()           diffusion.hpp:807-845
//
// Parity is pinned against the compiled reference (oracle/_ref) and the
// fixtures in tests/golden/ (tests/test_oracle.py).
//
// C ABI: orc_run(...) returns a malloc'ed JSON string in the reference
// driver's "run" format (oracle/ref_driver.cpp); orc_free releases it.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

using U = std::uint32_t;
constexpr U NONE = 0xFFFFFFFFu;

struct P {
  double x, y, z;
};
P operator+(P a, P b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
P operator-(P a, P b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
P operator*(P a, double s) { return {a.x * s, a.y * s, a.z * s}; }
P operator/(P a, double s) { return {a.x / s, a.y / s, a.z / s}; }
double dotp(P a, P b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
P crossp(P a, P b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double len(P a) { return std::sqrt(dotp(a, a)); }

struct Fail : std::runtime_error {
  std::string kind;
  Fail(const std::string& k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

// --- mesh indices of an already validated, oriented mesh --------------------
struct Topo {
  U nv = 0, nf = 0;
  std::vector<P> pos;
  std::vector<std::array<U, 3>> tri;
  std::vector<std::array<U, 2>> ev, ef;  // edge vertices (lo, hi), edge faces
  std::vector<std::array<U, 3>> fe;      // face edges
  std::vector<std::vector<U>> vf, vv;    // vertex faces (face order), sorted neighbours
  U other_face(U e, U f) const { return ef[e][0] == f ? ef[e][1] : ef[e][0]; }
};

Topo make_topo(const double* xyz, U nv, const U* faces, U nf) {
  Topo t;
  t.nv = nv;
  t.nf = nf;
  t.pos.resize(nv);
  for (U v = 0; v < nv; ++v) t.pos[v] = {xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]};
  t.tri.resize(nf);
  for (U f = 0; f < nf; ++f) t.tri[f] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
  std::map<std::pair<U, U>, U> id;
  t.fe.resize(nf);
  for (U f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      U a = t.tri[f][k], b = t.tri[f][(k + 1) % 3];
      auto key = std::make_pair(std::min(a, b), std::max(a, b));
      auto it = id.find(key);
      if (it == id.end()) {
        it = id.emplace(key, static_cast<U>(t.ev.size())).first;
        t.ev.push_back({key.first, key.second});
        t.ef.push_back({f, NONE});
      } else {
        t.ef[it->second][1] = f;
      }
      t.fe[f][k] = it->second;
    }
  t.vf.resize(nv);
  for (U f = 0; f < nf; ++f)
    for (U v : t.tri[f]) t.vf[v].push_back(f);
  t.vv.resize(nv);
  for (const auto& e : t.ev) {
    t.vv[e[0]].push_back(e[1]);
    t.vv[e[1]].push_back(e[0]);
  }
  for (auto& l : t.vv) std::sort(l.begin(), l.end());
  return t;
}

// --- operator ----------------------------------------------------------------
struct Op {
  std::vector<std::vector<std::pair<U, double>>> rows;  // sorted by column
  std::vector<double> mass;
  double gersh = 0;
};

Op assemble(const Topo& t) {
  struct Trip {
    U r, c;
    double w;
  };
  std::vector<Trip> trips;
  trips.reserve(static_cast<size_t>(t.nf) * 12);
  Op op;
  op.mass.assign(t.nv, 0.0);
  for (U f = 0; f < t.nf; ++f) {
    const auto& q = t.tri[f];
    const double area = 0.5 * len(crossp(t.pos[q[1]] - t.pos[q[0]], t.pos[q[2]] - t.pos[q[0]]));
    for (int k = 0; k < 3; ++k) op.mass[q[k]] += area / 3.0;
    for (int k = 0; k < 3; ++k) {
      const U a = q[k], b = q[(k + 1) % 3], c = q[(k + 2) % 3];
      const P ca = t.pos[a] - t.pos[c], cb = t.pos[b] - t.pos[c];
      const double cot = dotp(ca, cb) / len(crossp(ca, cb));
      if (!std::isfinite(cot)) throw Fail("DegeneracyError", "non-finite cotangent");
      const double w = 0.5 * cot;
      trips.push_back({a, b, w});
      trips.push_back({b, a, w});
      trips.push_back({a, a, -w});
      trips.push_back({b, b, -w});
    }
  }
  // The same (unstable) sort as the reference: equal keys then sum in the
  // order libstdc++'s introsort leaves them, which makes diagonals exact.
  std::sort(trips.begin(), trips.end(),
            [](const Trip& x, const Trip& y) { return x.r != y.r ? x.r < y.r : x.c < y.c; });
  op.rows.assign(t.nv, {});
  for (size_t i = 0; i < trips.size();) {
    size_t j = i;
    double s = 0;
    while (j < trips.size() && trips[j].r == trips[i].r && trips[j].c == trips[i].c) s += trips[j++].w;
    if (std::abs(s) > 0.0) op.rows[trips[i].r].push_back({trips[i].c, s});
    i = j;
  }
  for (U v = 0; v < t.nv; ++v) {
    double r = 0;
    for (const auto& e : op.rows[v]) r += std::abs(e.second);
    op.gersh = std::max(op.gersh, r / op.mass[v]);
  }
  return op;
}

// --- configuration -----------------------------------------------------------
struct Cfg {
  double dt = 0, tau = 0.05, sat = 0.999, kappa = 0.1;
  long check_interval = 1, max_steps = 200000;
  double covered = 0.05, seed_radius = 0;
  bool trails = true;
  double a = 1.0 / 25.0, w = 1.0 / 125.0, e = 1.0 / 30.0, mu = 0.25;
  double prune = 1e-9;
};

// --- hashing shared with the product and the reference driver --------------
uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t ehash(uint64_t l, uint64_t v, double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return mix(mix((l << 40) ^ v) ^ b);
}

// --- the layer matrix as dense rows ------------------------------------------
struct Layer {
  std::vector<double> row;  // 0 == absent
  bool active = false, cleared = false;
  U parent = NONE;
  std::vector<U> mparents;
  long created = 0;
};

struct Event {
  std::string kind;
  long step = 0;
  std::vector<U> layers, produced, covered;
  P pos{0, 0, 0};
  struct Est {
    U layer;
    double length;
    std::vector<std::tuple<long long, double, long long, P>> pts;
    size_t snap_n;
    uint64_t snap_hash;
  };
  std::vector<Est> est;
};

struct Track {
  U layer = NONE, created = NONE, consumed = NONE;
  std::vector<P> trail;
};

class Pass {
 public:
  Pass(const Topo& t, const Op& op, const Cfg& c) : t_(t), op_(op), c_(c), V_(t.nv) {}

  // init_field + Engine constructor (layer_field.hpp:318, diffusion.hpp:532).
  void start(U seed) {
    if (seed >= V_) throw Fail("InvalidParameter", "seed vertex out of range");
    const double radius = c_.seed_radius > 0 ? c_.seed_radius : 1.5 * (c_.a / std::sqrt(c_.w));
    std::vector<U> seeds = seed_ball(seed, radius);
    L_.assign(2, Layer{});
    L_[0].row.assign(V_, 1.0);
    L_[1].row.assign(V_, 0.0);
    L_[0].active = L_[1].active = true;
    for (U v : seeds) {
      L_[0].row[v] = 0.0;
      L_[1].row[v] = 1.0;
    }
    const double lam = op_.gersh * 0.5 * c_.a * c_.a;
    if (lam <= 0) throw Fail("InvalidParameter", "no positive time step");
    dt_ = c_.dt > 0 ? c_.dt : 0.9 * 2.0 / lam;
    Event ev;
    ev.kind = "seed";
    ev.layers = {1};
    ev.pos = t_.pos[seed];
    events_.push_back(ev);
    track(1).created = 0;
    moved_.assign(V_, 0);
    for (U v : seeds) moved_[v] = 1;
  }

  std::vector<U> seed_ball(U s, double r) const {
    std::vector<double> d(V_, 1e300);
    std::priority_queue<std::pair<double, U>, std::vector<std::pair<double, U>>, std::greater<>> pq;
    d[s] = 0;
    pq.push({0, s});
    std::vector<U> out;
    while (!pq.empty()) {
      auto [dv, v] = pq.top();
      pq.pop();
      if (dv > d[v]) continue;
      if (dv > r) break;
      out.push_back(v);
      for (U u : t_.vv[v]) {
        const double nd = dv + len(t_.pos[v] - t_.pos[u]);
        if (nd < d[u]) {
          d[u] = nd;
          pq.push({nd, u});
        }
      }
    }
    std::sort(out.begin(), out.end());
    return out;
  }

  std::vector<U> active_ids() const {
    std::vector<U> a;
    for (U i = 1; i < L_.size(); ++i)
      if (L_[i].active) a.push_back(i);
    return a;
  }
  double base(U v) const { return L_[0].row[v]; }
  double active_sum(U v) const {
    double s = 0;
    for (U i = 1; i < L_.size(); ++i)
      if (L_[i].active && L_[i].row[v] != 0.0) s += L_[i].row[v];
    return s;
  }

  // set_value with prune/clamp; reports whether the stored value changed.
  bool put(U l, U v, double x) {
    if (x > 1.0) x = 1.0;
    if (x < c_.prune) x = 0.0;
    double& cur = L_[l].row[v];
    if (cur == x) return false;
    cur = x;
    return true;
  }

  void advance() {
    const std::vector<U> act = active_ids();
    const double n = static_cast<double>(act.size() + 1), m = static_cast<double>(act.size());
    const double h2 = 0.5 * c_.a * c_.a;
    std::vector<char> region(V_, 0);
    bool any = false;
    for (U v = 0; v < V_; ++v)
      if (moved_[v]) {
        any = true;
        region[v] = 1;
        for (const auto& e : op_.rows[v]) region[e.first] = 1;
      }
    std::fill(moved_.begin(), moved_.end(), 0);
    if (!any) return;
    auto lap = [&](const std::vector<double>& x, U v) {
      double acc = 0;
      for (const auto& e : op_.rows[v]) acc += e.second * x[e.first];
      return acc / op_.mass[v];
    };
    std::vector<double> adense(V_);
    for (U v = 0; v < V_; ++v) adense[v] = active_sum(v);
    struct Up {
      U l, v;
      double x;
    };
    std::vector<Up> ups;
    for (U l : act) {
      const auto& row = L_[l].row;
      for (U v = 0; v < V_; ++v) {
        if (!region[v]) continue;
        const double phi = row[v];
        bool near = phi > 0;
        for (const auto& e : op_.rows[v])
          if (!near && row[e.first] > 0) near = true;
        if (!near) continue;
        const double pb = base(v);
        if (phi == 0.0 && pb <= c_.prune) continue;
        const double li = lap(row, v), lb = lap(L_[0].row, v);
        const double rate = -(c_.mu / n) * (c_.w * (pb - phi) + h2 * (lb - li) - c_.e * std::sqrt(std::max(phi * pb, 0.0)));
        if (!std::isfinite(rate)) throw Fail("NumericalBlowup", "non-finite rate");
        const double nx = std::clamp(phi + dt_ * rate, 0.0, 1.0);
        if (nx != phi) ups.push_back({l, v, nx});
      }
    }
    for (U v = 0; v < V_; ++v) {
      if (!region[v]) continue;
      const double pb = base(v);
      bool near = pb > 0;
      for (const auto& e : op_.rows[v])
        if (!near && base(e.first) > 0) near = true;
      if (!near) continue;
      double contact = 0;
      for (U l = 1; l < L_.size(); ++l)
        if (L_[l].active && L_[l].row[v] != 0.0) contact += std::sqrt(std::max(pb * L_[l].row[v], 0.0));
      const double rate = -(c_.mu / n) * (c_.w * adense[v] + h2 * lap(adense, v) + c_.e * contact) +
                          m * (c_.mu / n) * (c_.w * pb + h2 * lap(L_[0].row, v));
      if (!std::isfinite(rate)) throw Fail("NumericalBlowup", "non-finite rate");
      const double nx = std::clamp(pb + dt_ * rate, 0.0, 1.0);
      if (nx != pb) ups.push_back({0, v, nx});
    }
    std::vector<char> touched(V_, 0);
    for (const auto& u : ups) {
      if (put(u.l, u.v, u.x)) moved_[u.v] = 1;
      touched[u.v] = 1;
    }
    for (U v = 0; v < V_; ++v) {
      if (!touched[v]) continue;
      double s = 0;
      for (U l = 0; l < L_.size(); ++l)
        if (L_[l].row[v] != 0.0) s += L_[l].row[v];
      if (s <= 0.0) throw Fail("ZeroColumn", "total field extinction");
      if (std::abs(s - 1.0) < 1e-15) continue;
      std::vector<std::pair<U, double>> own;
      for (U l = 0; l < L_.size(); ++l)
        if (L_[l].row[v] != 0.0) own.push_back({l, L_[l].row[v]});
      for (const auto& [l, x] : own)
        if (put(l, v, x / s)) moved_[v] = 1;
    }
  }

  double sv(double x) const {  // symbolic perturbation at the 0.5 level
    double s = x - 0.5;
    if (s == 0.0) s = 1e-12 * (1.0 + 0.5);
    return s;
  }

  struct Front {
    std::vector<U> tris, bnd;
  };

  std::vector<U> band_of(U l) const {
    std::vector<U> b;
    for (U v = 0; v < V_; ++v) {
      const double x = L_[l].row[v];
      if (x > 0.0 && x < 1.0 && x > c_.tau && x < c_.sat) b.push_back(v);
    }
    return b;
  }

  std::vector<Front> front(U l) const {
    const std::vector<U> band = band_of(l);
    if (band.empty()) return {};
    std::vector<U> tris;
    for (U v : band)
      for (U f : t_.vf[v]) tris.push_back(f);
    std::sort(tris.begin(), tris.end());
    tris.erase(std::unique(tris.begin(), tris.end()), tris.end());
    std::vector<U> par(tris.size());
    std::iota(par.begin(), par.end(), 0u);
    auto find = [&](U a) {
      while (par[a] != a) a = par[a] = par[par[a]];
      return a;
    };
    auto slot = [&](U f) -> long {
      auto it = std::lower_bound(tris.begin(), tris.end(), f);
      return (it != tris.end() && *it == f) ? it - tris.begin() : -1;
    };
    for (U i = 0; i < tris.size(); ++i)
      for (U e : t_.fe[tris[i]]) {
        const long j = slot(t_.other_face(e, tris[i]));
        if (j < 0) continue;
        U a = find(i), b = find(static_cast<U>(j));
        if (a != b) par[std::max(a, b)] = std::min(a, b);
      }
    std::vector<Front> out;
    std::unordered_map<U, size_t> at;
    for (U i = 0; i < tris.size(); ++i) {
      auto [it, fresh] = at.try_emplace(find(i), out.size());
      if (fresh) out.emplace_back();
      out[it->second].tris.push_back(tris[i]);
    }
    for (auto& fr : out) {
      for (U f : fr.tris)
        for (U v : t_.tri[f])
          if (std::binary_search(band.begin(), band.end(), v)) fr.bnd.push_back(v);
      std::sort(fr.bnd.begin(), fr.bnd.end());
      fr.bnd.erase(std::unique(fr.bnd.begin(), fr.bnd.end()), fr.bnd.end());
    }
    return out;
  }

  P mean(const std::vector<U>& vs) const {
    P c{0, 0, 0};
    for (U v : vs) c = c + t_.pos[v];
    return vs.empty() ? c : c / static_cast<double>(vs.size());
  }

  Track& track(U l) {
    if (l >= tracks_.size()) tracks_.resize(l + 1);
    tracks_[l].layer = l;
    return tracks_[l];
  }

  U new_layer(U parent, long step) {
    Layer x;
    x.row.assign(V_, 0.0);
    x.active = true;
    x.parent = parent;
    x.created = step;
    L_.push_back(std::move(x));
    return static_cast<U>(L_.size() - 1);
  }

  void split(U l, const std::vector<Front>& fr, long step) {
    std::vector<U> unsat;
    for (U v = 0; v < V_; ++v)
      if (L_[l].row[v] > 0.0 && L_[l].row[v] < 1.0) unsat.push_back(v);
    std::vector<U> lab(V_, NONE);
    std::vector<U> q;
    for (U c = 0; c < fr.size(); ++c)
      for (U v : fr[c].bnd)
        if (lab[v] == NONE) {
          lab[v] = c;
          q.push_back(v);
        }
    for (size_t h = 0; h < q.size(); ++h) {
      const U v = q[h];
      for (U u : t_.vv[v]) {
        const double x = L_[l].row[u];
        if (!(x > 0.0 && x < 1.0) || lab[u] != NONE) continue;
        lab[u] = lab[v];
        q.push_back(u);
      }
    }
    std::vector<std::vector<U>> comps(fr.size());
    for (U v : unsat) comps[lab[v] == NONE ? 0 : lab[v]].push_back(v);
    comps.erase(std::remove_if(comps.begin(), comps.end(), [](const auto& c) { return c.empty(); }), comps.end());
    if (comps.size() < 2) return;
    std::vector<U> pb;
    for (const auto& f : fr) pb.insert(pb.end(), f.bnd.begin(), f.bnd.end());
    std::sort(pb.begin(), pb.end());
    pb.erase(std::unique(pb.begin(), pb.end()), pb.end());
    std::vector<U> kids;
    for (const auto& comp : comps) {
      const U k = new_layer(l, step);
      for (U v : comp) {
        L_[k].row[v] = L_[l].row[v];
        L_[l].row[v] = 0.0;
        moved_[v] = 1;
      }
      kids.push_back(k);
    }
    L_[l].active = false;
    Event ev;
    ev.kind = "split";
    ev.step = step;
    ev.layers = {l};
    ev.produced = kids;
    ev.pos = mean(pb);
    const U idx = static_cast<U>(events_.size());
    events_.push_back(ev);
    track(l).consumed = idx;
    for (U k : kids) track(k).created = idx;
  }

  std::vector<std::vector<U>> collisions() const {
    const std::vector<U> act = active_ids();
    if (act.size() < 2) return {};
    std::map<U, U> slot;
    for (U i = 0; i < act.size(); ++i) slot[act[i]] = i;
    std::vector<U> par(act.size());
    std::iota(par.begin(), par.end(), 0u);
    auto find = [&](U a) {
      while (par[a] != a) a = par[a] = par[par[a]];
      return a;
    };
    std::vector<char> in(act.size(), 0);
    for (U v = 0; v < V_; ++v) {
      bool cand = false;
      for (U l : act) {
        const double x = L_[l].row[v];
        if (x > 0.0 && x < 1.0 && x >= c_.kappa) cand = true;
      }
      if (!cand || base(v) > 1.0 - c_.kappa) continue;
      U first = NONE;
      for (U l : act) {
        const double x = L_[l].row[v];
        if (x == 0.0 || x < c_.kappa) continue;
        if (first == NONE) {
          first = slot[l];
        } else {
          U a = find(first), b = find(slot[l]);
          if (a != b) par[std::max(a, b)] = std::min(a, b);
          in[first] = in[slot[l]] = 1;
        }
      }
    }
    std::map<U, std::vector<U>> g;
    for (U i = 0; i < act.size(); ++i)
      if (in[i]) g[find(i)].push_back(act[i]);
    std::vector<std::vector<U>> out;
    for (auto& [r, mem] : g)
      if (mem.size() >= 2) out.push_back(mem);
    std::sort(out.begin(), out.end());
    return out;
  }

  struct LoopPt {
    U edge, face;
    double t;
    P pos;
  };

  // Mid-level isoline loops of a dense row (isoline.hpp:55).
  std::vector<std::vector<LoopPt>> isoline(const std::vector<double>& row) const {
    std::map<U, double> cross;  // edge -> t, ascending edge order
    for (U e = 0; e < t_.ev.size(); ++e) {
      const double a = sv(row[t_.ev[e][0]]), b = sv(row[t_.ev[e][1]]);
      if (a * b >= 0) continue;
      cross[e] = a / (a - b);
    }
    std::unordered_map<U, std::array<U, 2>> fx;
    for (const auto& [e, tt] : cross)
      for (U f : t_.ef[e]) {
        auto [it, fresh] = fx.try_emplace(f, std::array<U, 2>{e, NONE});
        if (!fresh) it->second[1] = e;
      }
    std::vector<std::vector<LoopPt>> loops;
    std::map<U, bool> seen;
    for (const auto& [seed, tt] : cross) {
      if (seen[seed]) continue;
      std::vector<LoopPt> lp;
      U e = seed, f = t_.ef[seed][0];
      do {
        seen[e] = true;
        const double te = cross.at(e);
        const P a = t_.pos[t_.ev[e][0]], b = t_.pos[t_.ev[e][1]];
        lp.push_back({e, f, te, a + (b - a) * te});
        const auto& two = fx.at(f);
        const U ne = two[0] == e ? two[1] : two[0];
        f = t_.other_face(ne, f);
        e = ne;
      } while (e != seed);
      LoopPt first = lp.front();
      first.face = lp.back().face;
      lp.push_back(first);
      loops.push_back(lp);
    }
    return loops;
  }

  static double loop_len(const std::vector<LoopPt>& lp) {
    double s = 0;
    for (size_t i = 0; i + 1 < lp.size(); ++i) s += len(lp[i].pos - lp[i + 1].pos);
    return s;
  }

  bool front_loop(U l, std::vector<LoopPt>& out) const {
    double best = -1;
    for (auto& lp : isoline(L_[l].row)) {
      double bm = 0;
      size_t ns = 0;
      for (const auto& p : lp) {
        bm += (1.0 - p.t) * base(t_.ev[p.edge][0]) + p.t * base(t_.ev[p.edge][1]);
        ++ns;
      }
      if (ns == 0 || bm / ns < 0.01) continue;
      const double L = loop_len(lp);
      if (L > best) {
        best = L;
        out = lp;
      }
    }
    return best > 0;
  }

  void merge(const std::vector<U>& g, long step) {
    struct FL {
      U l;
      std::vector<LoopPt> lp;
      double L;
    };
    std::vector<FL> fls;
    for (U l : g) {
      std::vector<LoopPt> lp;
      if (front_loop(l, lp)) fls.push_back({l, lp, loop_len(lp)});
    }
    std::vector<U> ub;
    for (U l : g) {
      auto b = band_of(l);
      ub.insert(ub.end(), b.begin(), b.end());
    }
    std::sort(ub.begin(), ub.end());
    ub.erase(std::unique(ub.begin(), ub.end()), ub.end());
    Event ev;
    ev.kind = "merge";
    ev.step = step;
    ev.layers = g;
    ev.pos = mean(ub);
    for (U v = 0; v < V_; ++v)
      if (1.0 - base(v) >= c_.covered) ev.covered.push_back(v);
    const U idx = static_cast<U>(events_.size());
    if (!fls.empty()) {
      size_t drop = 0;
      for (size_t i = 1; i < fls.size(); ++i)
        if (fls[i].L > fls[drop].L || (fls[i].L == fls[drop].L && fls[i].l < fls[drop].l)) drop = i;
      fls.erase(fls.begin() + static_cast<long>(drop));
      std::sort(fls.begin(), fls.end(), [](const FL& a, const FL& b) { return a.L != b.L ? a.L < b.L : a.l < b.l; });
      for (const auto& fl : fls) {
        Event::Est es;
        es.layer = fl.l;
        es.length = fl.L;
        for (const auto& p : fl.lp) es.pts.emplace_back(p.edge, p.t, p.face, p.pos);
        es.snap_n = 0;
        es.snap_hash = 0;
        for (U v = 0; v < V_; ++v)
          if (L_[fl.l].row[v] != 0.0) {
            ++es.snap_n;
            es.snap_hash += ehash(fl.l, v, L_[fl.l].row[v]);
          }
        ev.est.push_back(es);
      }
    }
    const U r = new_layer(g.front(), step);
    L_[r].mparents = g;
    for (U v = 0; v < V_; ++v) {
      double acc = 0;
      bool any = false;
      for (U l : g)
        if (L_[l].row[v] != 0.0) {
          acc += L_[l].row[v];
          any = true;
        }
      if (!any) continue;
      L_[r].row[v] = std::min(acc, 1.0);
      moved_[v] = 1;
      for (U l : g) L_[l].row[v] = 0.0;
    }
    for (U l : g) {
      L_[l].active = false;
      L_[l].cleared = true;
    }
    ev.produced = {r};
    events_.push_back(ev);
    for (U l : g) track(l).consumed = idx;
    track(r).created = idx;
    last_[r] = ev.pos;
  }

  void vanish(U l, long step) {
    Event ev;
    ev.kind = "vanish";
    ev.step = step;
    ev.layers = {l};
    auto it = last_.find(l);
    if (it != last_.end()) {
      ev.pos = it->second;
    } else {
      std::vector<U> sup;
      for (U v = 0; v < V_; ++v)
        if (L_[l].row[v] != 0.0) sup.push_back(v);
      ev.pos = mean(sup);
    }
    const U idx = static_cast<U>(events_.size());
    events_.push_back(ev);
    track(l).consumed = idx;
    L_[l].active = false;
  }

  bool finished(U l) const {
    for (U v = 0; v < V_; ++v) {
      const double x = L_[l].row[v];
      if (x > 0.0 && x < 1.0) return false;
    }
    for (U v = 0; v < V_; ++v)
      if (L_[l].row[v] != 0.0)
        for (U u : t_.vv[v])
          if (base(u) > c_.prune) return false;
    return true;
  }

  bool extinct() const {
    double mx = 0;
    bool any = false;
    for (U v = 0; v < V_; ++v) {
      const double b = base(v);
      if (b == 0.0) continue;
      any = true;
      if (b == 1.0) return false;
      mx = std::max(mx, b);
    }
    return !any || mx < 1.0 - c_.sat;
  }

  bool check(long step) {
    for (U l : active_ids()) {
      auto fr = front(l);
      if (fr.size() >= 2) split(l, fr, step);
    }
    for (const auto& g : collisions()) merge(g, step);
    for (U l : active_ids()) {
      auto b = band_of(l);
      if (!b.empty()) {
        const P m = mean(b);
        last_[l] = m;
        if (c_.trails) {
          double best = 1e300;
          U bv = NONE;
          for (U v : b) {
            const P d = t_.pos[v] - m;
            const double d2 = dotp(d, d);
            if (d2 < best) {
              best = d2;
              bv = v;
            }
          }
          track(l).trail.push_back(bv == NONE ? m : t_.pos[bv]);
        }
      } else if (finished(l)) {
        vanish(l, step);
      }
    }
    uint64_t h = 0;
    for (U l = 0; l < L_.size(); ++l)
      for (U v = 0; v < V_; ++v)
        if (L_[l].row[v] != 0.0) h += ehash(l, v, L_[l].row[v]);
    hashes_.push_back(h);
    if (extinct()) {
      for (U l : active_ids()) vanish(l, step);
      return true;
    }
    return active_ids().empty();
  }

  std::string run() {
    long step = 0;
    std::string status = "ok", err;
    try {
      while (true) {
        if (step >= c_.max_steps) throw Fail("MaxStepsExceeded", "max steps");
        advance();
        ++step;
        if (step % c_.check_interval == 0 && check(step)) break;
      }
    } catch (const Fail& f) {
      status = "error";
      err = f.kind;
    }
    return to_json(status, err, step);
  }

  static void num(std::string& s, double d) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", d);
    s += b;
  }
  static void pt(std::string& s, P p) {
    s += "[";
    num(s, p.x);
    s += ",";
    num(s, p.y);
    s += ",";
    num(s, p.z);
    s += "]";
  }
  template <class T>
  static void ids(std::string& s, const std::vector<T>& v) {
    s += "[";
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) s += ",";
      s += std::to_string(v[i]);
    }
    s += "]";
  }

  std::string to_json(const std::string& status, const std::string& err, long steps) const {
    std::string s = "{\"status\":\"" + status + "\"";
    if (!err.empty()) s += ",\"error_type\":\"" + err + "\"";
    s += ",\"steps\":" + std::to_string(steps) + ",\"dt_used\":";
    num(s, dt_);
    s += ",\"events\":[";
    for (size_t i = 0; i < events_.size(); ++i) {
      const auto& e = events_[i];
      if (i) s += ",";
      s += "{\"kind\":\"" + e.kind + "\",\"step\":" + std::to_string(e.step) + ",\"layers\":";
      ids(s, e.layers);
      s += ",\"produced\":";
      ids(s, e.produced);
      s += ",\"position\":";
      pt(s, e.pos);
      s += ",\"covered\":";
      ids(s, e.covered);
      s += ",\"estimates\":[";
      for (size_t k = 0; k < e.est.size(); ++k) {
        const auto& x = e.est[k];
        if (k) s += ",";
        s += "{\"layer\":" + std::to_string(x.layer) + ",\"event_index\":" + std::to_string(i) + ",\"length\":";
        num(s, x.length);
        s += ",\"snapshot_n\":" + std::to_string(x.snap_n) + ",\"snapshot_hash\":\"" + std::to_string(x.snap_hash) +
             "\",\"points\":[";
        for (size_t j = 0; j < x.pts.size(); ++j) {
          if (j) s += ",";
          s += "[" + std::to_string(std::get<0>(x.pts[j])) + ",";
          num(s, std::get<1>(x.pts[j]));
          s += "," + std::to_string(std::get<2>(x.pts[j])) + ",";
          pt(s, std::get<3>(x.pts[j]));
          s += "]";
        }
        s += "]}";
      }
      s += "]}";
    }
    s += "],\"tracks\":[";
    for (size_t i = 0; i < tracks_.size(); ++i) {
      const auto& t = tracks_[i];
      if (i) s += ",";
      auto sid = [](U x) { return x == NONE ? std::string("-1") : std::to_string(x); };
      s += "{\"layer\":" + sid(t.layer) + ",\"created\":" + sid(t.created) + ",\"consumed\":" + sid(t.consumed) +
           ",\"trail\":[";
      for (size_t k = 0; k < t.trail.size(); ++k) {
        if (k) s += ",";
        pt(s, t.trail[k]);
      }
      s += "]}";
    }
    s += "],\"hashes\":[";
    for (size_t i = 0; i < hashes_.size(); ++i) {
      if (i) s += ",";
      s += "\"" + std::to_string(hashes_[i]) + "\"";
    }
    s += "],\"layer_count\":" + std::to_string(L_.size()) + "}";
    return s;
  }

 private:
  const Topo& t_;
  const Op& op_;
  Cfg c_;
  U V_;
  double dt_ = 0;
  std::vector<Layer> L_;
  std::vector<char> moved_;
  std::vector<Event> events_;
  std::vector<Track> tracks_;
  std::map<U, P> last_;
  std::vector<uint64_t> hashes_;
};

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

// cfg: dt, tau, sat, kappa, check_interval, max_steps, covered, seed_radius, trails
// op_*: optional operator (CSR with int32 offsets); null -> assemble like the reference.
char* orc_run(const double* xyz, unsigned nv, const unsigned* faces, unsigned nf, const int* op_off,
              const int* op_col, const double* op_val, const double* op_mass, double op_gersh, unsigned seed,
              const double* cfg) {
  try {
    Topo t = make_topo(xyz, nv, faces, nf);
    Op op;
    if (op_off) {
      op.rows.assign(nv, {});
      for (unsigned v = 0; v < nv; ++v)
        for (int k = op_off[v]; k < op_off[v + 1]; ++k) op.rows[v].push_back({static_cast<U>(op_col[k]), op_val[k]});
      op.mass.assign(op_mass, op_mass + nv);
      op.gersh = op_gersh;
    } else {
      op = assemble(t);
    }
    Cfg c;
    if (cfg) {
      c.dt = cfg[0];
      c.tau = cfg[1];
      c.sat = cfg[2];
      c.kappa = cfg[3];
      c.check_interval = static_cast<long>(cfg[4]);
      c.max_steps = static_cast<long>(cfg[5]);
      c.covered = cfg[6];
      c.seed_radius = cfg[7];
      c.trails = cfg[8] != 0;
    }
    Pass p(t, op, c);
    p.start(seed);
    return dup(p.run());
  } catch (const std::exception& e) {
    return dup(std::string("{\"status\":\"fatal\",\"message\":\"") + e.what() + "\"}");
  }
}

// Assembled operator of a validated mesh: fills off (nv+1), and when col/val
// are non-null the CSR arrays and masses; returns nnz (or -1 on error).
long orc_assemble(const double* xyz, unsigned nv, const unsigned* faces, unsigned nf, int* off, int* col, double* val,
                  double* mass, double* gersh) {
  try {
    Topo t = make_topo(xyz, nv, faces, nf);
    Op op = assemble(t);
    long nnz = 0;
    for (unsigned v = 0; v < nv; ++v) {
      if (off) off[v] = static_cast<int>(nnz);
      for (const auto& e : op.rows[v]) {
        if (col) col[nnz] = static_cast<int>(e.first);
        if (val) val[nnz] = e.second;
        ++nnz;
      }
    }
    if (off) off[nv] = static_cast<int>(nnz);
    if (mass) std::memcpy(mass, op.mass.data(), sizeof(double) * nv);
    if (gersh) *gersh = op.gersh;
    return nnz;
  } catch (...) {
    return -1;
  }
}

void orc_free(char* p) { std::free(p); }

}  // extern "C"
