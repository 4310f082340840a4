// Persistent diffusion-front engine for sm_100a.
//
// One cooperative launch executes many explicit-Euler steps of the initial
// pass (reference: diffusion.hpp:242-367 advance(), diffusion.hpp:807-845
// check()) and returns to the host only when a topology event (split, merge,
// vanish, extinction), an error, or the step budget is reached.  Per step:
//
//   A  update   one thread per frontier vertex: gather the stiffness row's
//               columns, evaluate every near-support layer and the base layer
//               (Eq. 2, reference rates at diffusion.hpp:313 and :343), apply
//               set_value pruning/clamping and column normalisation, write the
//               new column to scratch.  Reads only committed state.
//   B  commit   scatter changed columns, maintain the interest flags and the
//               base==1 counter, queue the one-ring of every moved vertex as
//               the next frontier (stamped, deduplicated).
//   C  band     warp-ballot compaction of the interest flags into a list.
//   D  union    lock-free union-find over band (vertex, layer-slot) items with
//               the face-adjacency rule of extract_front (diffusion.hpp:398).
//   E  stats    roots per layer (= front components), band counts and
//               fixed-point position sums, unsaturated counts, collision pairs
//               (detect_collisions, diffusion.hpp:475), base extinction.
//
// Separated by a software grid barrier.  All arithmetic is IEEE binary64 with
// FMA contraction disabled (-fmad=false), in the reference's evaluation order,
// so every field value is bit-identical to the CPU reference.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace dtb {

void note_launch(unsigned long long n);

namespace {

constexpr int kCand = 16;  // candidate layers gathered over one stiffness row
constexpr int kWork = 24;  // working column capacity before the final size check
constexpr unsigned long long kVertMask = (1ull << 27) - 1;  // vertex bits of a snap key

__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }
__device__ __forceinline__ double max0(double x) { return x < 0.0 ? 0.0 : x; }  // std::max(x, 0.0)

__device__ __forceinline__ void raise_error(Ctl* ctl, int code, int v) {
  int prev = atomicMax(&ctl->error, code);
  if (prev < code) ctl->error_vertex = v;
}

__device__ __forceinline__ void grid_sync(Ctl* ctl) {
  const unsigned nb = gridDim.x;
  __syncthreads();
  if (nb == 1) return;
  if (threadIdx.x == 0) {
    volatile unsigned* genp = &ctl->bar_gen;
    const unsigned gen = *genp;
    __threadfence();
    const unsigned arrived = atomicAdd(&ctl->bar_count, 1u);
    if (arrived == nb - 1) {
      atomicExch(&ctl->bar_count, 0u);
      __threadfence();
      atomicAdd(&ctl->bar_gen, 1u);
    } else {
      while (*genp == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// set_value semantics (layer_field.hpp:102): clamp above 1, prune below the
// epsilon, erase zeros; `changed` records whether the stored value moved.
__device__ __forceinline__ bool col_set(unsigned short* nl, double* nx, int& nn, int l, double val, double prune,
                                        bool& changed) {
  if (val > 1.0) val = 1.0;
  if (val < prune) val = 0.0;
  int j = 0;
  while (j < nn && nl[j] < l) ++j;
  const bool found = j < nn && nl[j] == l;
  if (val == 0.0) {
    if (found) {
      for (int q = j; q + 1 < nn; ++q) {
        nl[q] = nl[q + 1];
        nx[q] = nx[q + 1];
      }
      --nn;
      changed = true;
    }
    return true;
  }
  if (found) {
    if (nx[j] != val) {
      nx[j] = val;
      changed = true;
    }
    return true;
  }
  if (nn >= kWork) return false;
  for (int q = nn; q > j; --q) {
    nl[q] = nl[q - 1];
    nx[q] = nx[q - 1];
  }
  nl[j] = static_cast<unsigned short>(l);
  nx[j] = val;
  ++nn;
  changed = true;
  return true;
}

// ---------------------------------------------------------------------------
// Phase A: one explicit Euler update of every near-support layer and the base
// layer at vertex v, reading only the committed columns.
__device__ void update_vertex(const DevMesh& M, const DevField& F, const DevWork& W, const StepParams& P,
                              int i, int v) {
  unsigned short ol[kSlots];
  double ox[kSlots];
  const int cv = F.cnt[v];
  for (int j = 0; j < cv; ++j) {
    ol[j] = F.lay[static_cast<size_t>(v) * kSlots + j];
    ox[j] = F.val[static_cast<size_t>(v) * kSlots + j];
  }
  const double phib = (cv > 0 && ol[0] == 0) ? ox[0] : 0.0;

  unsigned short cl[kCand];
  double ca[kCand];
  int nc = 0;
  double lapb = 0.0, lapt = 0.0;
  bool bnear = phib > 0.0;
  bool overflow = false;
  const int k0 = __ldg(M.s_off + v), k1 = __ldg(M.s_off + v + 1);
  for (int k = k0; k < k1; ++k) {
    const int u = __ldg(M.s_col + k);
    const double s = __ldg(M.s_val + k);
    const int cu = F.cnt[u];
    double bu = 0.0, au = 0.0;
    const size_t base = static_cast<size_t>(u) * kSlots;
    for (int j = 0; j < cu; ++j) {
      const int l = F.lay[base + j];
      const double x = F.val[base + j];
      if (l == 0) {
        bu = x;
        continue;
      }
      if (!W.active[l]) continue;
      au = au + x;
      int c = 0;
      while (c < nc && cl[c] != l) ++c;
      if (c == nc) {
        if (nc == kCand) {
          overflow = true;
          continue;
        }
        cl[nc] = static_cast<unsigned short>(l);
        ca[nc] = 0.0;
        ++nc;
      }
      ca[c] = ca[c] + s * x;
    }
    lapb = lapb + s * bu;
    lapt = lapt + s * au;
    if (bu > 0.0) bnear = true;
  }
  // Layers held at v itself are near support even if the stiffness row
  // lacks its diagonal (never on valid meshes, kept for exactness).
  for (int j = 0; j < cv; ++j) {
    const int l = ol[j];
    if (l == 0 || !W.active[l]) continue;
    int c = 0;
    while (c < nc && cl[c] != l) ++c;
    if (c == nc) {
      if (nc == kCand) {
        overflow = true;
        continue;
      }
      cl[nc] = static_cast<unsigned short>(l);
      ca[nc] = 0.0;
      ++nc;
    }
  }
  if (overflow) {
    raise_error(W.ctl, kDevCapacity, v);
    return;
  }

  const double mass = __ldg(M.mass + v);
  const double lap_b = lapb / mass;
  unsigned short nl[kWork];
  double nx[kWork];
  int nn = cv;
  for (int j = 0; j < cv; ++j) {
    nl[j] = ol[j];
    nx[j] = ox[j];
  }
  bool touched = false, changed = false, ok = true;

  for (int c = 0; c < nc; ++c) {
    const int l = cl[c];
    double phi = 0.0;
    for (int j = 0; j < cv; ++j)
      if (ol[j] == l) phi = ox[j];
    if (phi == 0.0 && phib <= P.prune) continue;
    const double lap_i = ca[c] / mass;
    const double inner = P.w * (phib - phi) + P.half_a2 * (lap_b - lap_i) - P.e * sqrt(max0(phi * phib));
    const double rate = -P.mu_n * inner;
    if (!isfinite(rate)) {
      raise_error(W.ctl, kDevBlowup, v);
      return;
    }
    const double next = clamp01(phi + P.dt * rate);
    if (next != phi) {
      touched = true;
      ok &= col_set(nl, nx, nn, l, next, P.prune, changed);
    }
  }
  if (bnear) {
    double total = 0.0, contact = 0.0;
    for (int j = 0; j < cv; ++j) {
      const int l = ol[j];
      if (l != 0 && W.active[l]) total = total + ox[j];
    }
    for (int j = 0; j < cv; ++j) {
      const int l = ol[j];
      if (l != 0 && W.active[l]) contact = contact + sqrt(max0(phib * ox[j]));
    }
    const double lap_total = lapt / mass;
    const double rate = -P.mu_n * (P.w * total + P.half_a2 * lap_total + P.e * contact) +
                        P.m_mu_n * (P.w * phib + P.half_a2 * lap_b);
    if (!isfinite(rate)) {
      raise_error(W.ctl, kDevBlowup, v);
      return;
    }
    const double next = clamp01(phib + P.dt * rate);
    if (next != phib) {
      touched = true;
      ok &= col_set(nl, nx, nn, 0, next, P.prune, changed);
    }
  }
  // Column normalisation of touched vertices (layer_field.hpp:143).
  if (touched) {
    double s = 0.0;
    for (int j = 0; j < nn; ++j) s = s + nx[j];
    if (s <= 0.0) {
      raise_error(W.ctl, kDevZeroColumn, v);
      return;
    }
    if (!(fabs(s - 1.0) < 1e-15)) {
      unsigned short sl[kWork];
      double sx[kWork];
      const int sn = nn;
      for (int j = 0; j < sn; ++j) {
        sl[j] = nl[j];
        sx[j] = nx[j];
      }
      for (int j = 0; j < sn; ++j) ok &= col_set(nl, nx, nn, sl[j], sx[j] / s, P.prune, changed);
    }
  }
  if (!ok || nn > kSlots) {
    raise_error(W.ctl, kDevCapacity, v);
    return;
  }
  const bool old_one = cv > 0 && ol[0] == 0 && ox[0] == 1.0;
  const bool new_one = nn > 0 && nl[0] == 0 && nx[0] == 1.0;
  W.scnt[i] = static_cast<unsigned char>(nn);
  const size_t o = static_cast<size_t>(i) * kSlots;
  for (int j = 0; j < nn; ++j) {
    W.slay[o + j] = nl[j];
    W.sval[o + j] = nx[j];
  }
  W.sflag[i] = static_cast<unsigned char>((changed ? 1 : 0) | (old_one ? 2 : 0) | (new_one ? 4 : 0));
}

__device__ __forceinline__ void queue_region(const DevWork& W, int u, int stamp, int nxt) {
  if (atomicExch(W.stamp + u, stamp) != stamp) {
    const int pos = atomicAdd(&W.ctl->rcount[nxt], 1);
    W.region[nxt][pos] = u;
  }
}

// Phase B for region slot i.
__device__ void commit_vertex(const DevMesh& M, const DevField& F, const DevWork& W, int i, int v, int stamp,
                              int nxt) {
  const int flag = W.sflag[i];
  if (!(flag & 1)) return;
  const int nn = W.scnt[i];
  const size_t o = static_cast<size_t>(i) * kSlots, d = static_cast<size_t>(v) * kSlots;
  bool inter = false;
  for (int j = 0; j < nn; ++j) {
    const double x = W.sval[o + j];
    F.lay[d + j] = W.slay[o + j];
    F.val[d + j] = x;
    inter |= (x > 0.0 && x < 1.0);
  }
  F.cnt[v] = static_cast<unsigned char>(nn);
  F.interest[v] = inter ? 1 : 0;
  const int delta = ((flag >> 2) & 1) - ((flag >> 1) & 1);
  if (delta) atomicAdd(&W.ctl->base_one, delta);
  queue_region(W, v, stamp, nxt);
  const int k0 = __ldg(M.s_off + v), k1 = __ldg(M.s_off + v + 1);
  for (int k = k0; k < k1; ++k) queue_region(W, __ldg(M.s_col + k), stamp, nxt);
}

__device__ __forceinline__ bool is_band(const DevWork& W, const StepParams& P, int l, double x) {
  return l != 0 && W.active[l] && x > P.band_lo && x < P.sat;
}

__device__ __forceinline__ unsigned uf_find(unsigned long long* par, unsigned x, unsigned long long ep) {
  while (true) {
    const unsigned long long p = par[x];
    if ((p >> 32) != ep) return x;
    const unsigned q = static_cast<unsigned>(p);
    if (q == x) return x;
    const unsigned long long pp = par[q];
    if ((pp >> 32) == ep && static_cast<unsigned>(pp) != q) par[x] = pp;  // path halving
    x = q;
  }
}

__device__ void uf_unite(unsigned long long* par, unsigned a, unsigned b, unsigned long long ep) {
  while (true) {
    a = uf_find(par, a, ep);
    b = uf_find(par, b, ep);
    if (a == b) return;
    if (a < b) {
      const unsigned t = a;
      a = b;
      b = t;
    }
    const unsigned long long old = par[a];
    if ((old >> 32) == ep && static_cast<unsigned>(old) != a) continue;
    const unsigned long long want = (ep << 32) | b;
    if (atomicCAS(par + a, old, want) == old) return;
  }
}

__device__ void insert_pair(const DevWork& W, unsigned key, unsigned long long ep) {
  const unsigned long long tagged = (ep << 32) | key;
  unsigned h = (key * 2654435761u) & (kPairCap - 1);
  for (int probe = 0; probe < kPairCap; ++probe) {
    unsigned long long cur = W.pair_keys[h];
    if (cur == tagged) return;
    if ((cur >> 32) != ep) {
      const unsigned long long prev = atomicCAS(W.pair_keys + h, cur, tagged);
      if (prev == cur) {
        const int pos = atomicAdd(&W.ctl->npairs, 1);
        if (pos < kPairCap) W.pairs[pos] = key;
        else W.ctl->pair_overflow = 1;
        return;
      }
      if (prev == tagged) return;
      continue;  // lost the race for this slot; re-inspect it
    }
    h = (h + 1) & (kPairCap - 1);
  }
  W.ctl->pair_overflow = 1;
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ unsigned long long entry_hash(unsigned long long layer, unsigned long long v, double x) {
  return splitmix64(splitmix64((layer << 40) ^ v) ^ static_cast<unsigned long long>(__double_as_longlong(x)));
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Phase C: interest list by warp-ballot compaction (+ optional field digest).
__device__ void phase_band_list(const DevField& F, const DevWork& W, int nv, bool hash) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  unsigned long long h = 0;
  for (int base = gwarp * 32; base < nv; base += nwarps * 32) {
    const int v = base + lane;
    const bool flag = v < nv && F.interest[v];
    const unsigned mask = __ballot_sync(0xffffffffu, flag);
    if (mask) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(&W.ctl->icount, __popc(mask));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (flag) W.ilist[pos + __popc(mask & ((1u << lane) - 1))] = v;
    }
    if (hash && v < nv) {
      const int c = F.cnt[v];
      for (int j = 0; j < c; ++j)
        h += entry_hash(F.lay[static_cast<size_t>(v) * kSlots + j], static_cast<unsigned long long>(v),
                        F.val[static_cast<size_t>(v) * kSlots + j]);
    }
  }
  if (hash) {
    h = warp_sum_u64(h);
    if (lane == 0 && h) atomicAdd(&W.ctl->hash_acc, h);
  }
}

// Phase D: union band items that share a band triangle pair.
__device__ void phase_union(const DevMesh& M, const DevField& F, const DevWork& W, const StepParams& P,
                            unsigned long long ep) {
  const int n = W.ctl->icount;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int v = W.ilist[idx];
    const int cv = F.cnt[v];
    for (int k = 0; k < cv; ++k) {
      const int l = F.lay[static_cast<size_t>(v) * kSlots + k];
      const double x = F.val[static_cast<size_t>(v) * kSlots + k];
      if (!is_band(W, P, l, x)) continue;
      const unsigned item = static_cast<unsigned>(v) * kSlots + k;
      const int c0 = __ldg(M.c_off + v), c1 = __ldg(M.c_off + v + 1);
      for (int c = c0; c < c1; ++c) {
        const int u = __ldg(M.c_col + c);
        if (u <= v) continue;
        const int cu = F.cnt[u];
        const size_t ub = static_cast<size_t>(u) * kSlots;
        for (int j = 0; j < cu; ++j) {
          const int lu = F.lay[ub + j];
          if (lu < l) continue;
          if (lu == l && is_band(W, P, l, F.val[ub + j])) uf_unite(W.parent, item, static_cast<unsigned>(u) * kSlots + j, ep);
          break;
        }
      }
    }
  }
}

// Phase E: per-layer statistics, collision pairs and base extinction data.
__device__ void phase_stats(const DevMesh& M, const DevField& F, const DevWork& W, const StepParams& P,
                            unsigned long long ep) {
  const int n = W.ctl->icount;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int v = W.ilist[idx];
    const int cv = F.cnt[v];
    const size_t b = static_cast<size_t>(v) * kSlots;
    const double base = (cv > 0 && F.lay[b] == 0) ? F.val[b] : 0.0;
    if (base > 0.0 && base < 1.0)
      atomicMax(&W.ctl->base_max_bits, static_cast<unsigned long long>(__double_as_longlong(base)));
    bool cand = false;
    for (int k = 0; k < cv; ++k) {
      const int l = F.lay[b + k];
      if (l == 0 || !W.active[l]) continue;
      const double x = F.val[b + k];
      const int a = W.aidx[l];
      LayerStat* st = W.stat + a;
      if (x > 0.0 && x < 1.0) {
        atomicAdd(&st->nunsat, 1);
        if (x >= P.kappa) cand = true;
      }
      if (x > P.band_lo && x < P.sat) {
        atomicAdd(&st->nband, 1);
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->sx), static_cast<unsigned long long>(__ldg(M.fx + v)));
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->sy), static_cast<unsigned long long>(__ldg(M.fy + v)));
        atomicAdd(reinterpret_cast<unsigned long long*>(&st->sz), static_cast<unsigned long long>(__ldg(M.fz + v)));
        const unsigned item = static_cast<unsigned>(v) * kSlots + k;
        if (uf_find(W.parent, item, ep) == item) atomicAdd(&st->ncomp, 1);
      }
    }
    if (cand && !(base > P.coll_base_limit)) {
      int first = -1;
      for (int k = 0; k < cv; ++k) {
        const int l = F.lay[b + k];
        if (l == 0 || !W.active[l]) continue;
        if (F.val[b + k] < P.kappa) continue;
        if (first < 0) first = l;
        else insert_pair(W, (static_cast<unsigned>(first) << 16) | static_cast<unsigned>(l), ep);
      }
    }
  }
}

__device__ __forceinline__ void band_mean(const DevMesh& M, const LayerStat& st, double& mx, double& my, double& mz) {
  const double n = static_cast<double>(st.nband);
  mx = (static_cast<double>(st.sx) * M.fx_scale) / n;
  my = (static_cast<double>(st.sy) * M.fx_scale) / n;
  mz = (static_cast<double>(st.sz) * M.fx_scale) / n;
}

// snap_to_band (diffusion.hpp:590): nearest band vertex to the band mean;
// packed key = distance bits (low 27 mantissa bits dropped) | vertex.
__device__ void phase_snap(const DevMesh& M, const DevField& F, const DevWork& W, const StepParams& P) {
  const int n = W.ctl->icount;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int v = W.ilist[idx];
    const int cv = F.cnt[v];
    const size_t b = static_cast<size_t>(v) * kSlots;
    for (int k = 0; k < cv; ++k) {
      const int l = F.lay[b + k];
      if (!is_band(W, P, l, F.val[b + k])) continue;
      const LayerStat* st = W.stat + W.aidx[l];
      double mx, my, mz;
      band_mean(M, *st, mx, my, mz);
      const double dx = __ldg(M.px + v) - mx, dy = __ldg(M.py + v) - my, dz = __ldg(M.pz + v) - mz;
      const double d2 = dx * dx + dy * dy + dz * dz;
      const unsigned long long key =
          (static_cast<unsigned long long>(__double_as_longlong(d2)) & ~kVertMask) | static_cast<unsigned long long>(v);
      atomicMin(&W.stat[W.aidx[l]].snap, key);
    }
  }
}

// Writes the trail record of active index a for a finished check and resets
// its statistics for the next one.
__device__ void flush_and_reset_stat(const DevMesh& M, const DevWork& W, const StepParams& P, int a, bool pend,
                                     long long pend_step) {
  LayerStat* st = W.stat + a;
  if (pend && st->nband > 0) {
    const int layer = W.alist[a];
    double mx, my, mz;
    band_mean(M, *st, mx, my, mz);
    W.lastpos[4 * layer + 0] = mx;
    W.lastpos[4 * layer + 1] = my;
    W.lastpos[4 * layer + 2] = mz;
    W.lastpos[4 * layer + 3] = 1.0;  // valid
    if (P.record_trails) {
      const int pos = atomicAdd(&W.ctl->ntrail, 1);
      TrailRec r;
      r.step = pend_step;
      r.layer = layer;
      r.vertex = static_cast<int>(st->snap & kVertMask);
      r.mx = mx;
      r.my = my;
      r.mz = mz;
      W.trail[pos & (kTrailCap - 1)] = r;
    }
  }
  st->ncomp = 0;
  st->nband = 0;
  st->nunsat = 0;
  st->sx = st->sy = st->sz = 0;
  st->snap = ~0ull;
}

__device__ int decide(const DevWork& W, const StepParams& P) {
  int bits = 0;
  for (int a = threadIdx.x; a < P.n_active; a += blockDim.x) {
    const LayerStat& st = W.stat[a];
    if (st.ncomp >= 2) bits |= kStopSplit;
    if (st.nband == 0 && st.nunsat == 0) bits |= kStopVanish;
  }
  if (threadIdx.x == 0) {
    if (W.ctl->npairs > 0 || W.ctl->pair_overflow) bits |= kStopMerge;
    const double bmax = __longlong_as_double(static_cast<long long>(W.ctl->base_max_bits));
    if (W.ctl->base_one == 0 && bmax < P.extinct_limit) bits |= kStopExtinct;
  }
  __shared__ int s_bits;
  if (threadIdx.x == 0) s_bits = 0;
  __syncthreads();
  if (bits) atomicOr(&s_bits, bits);
  __syncthreads();
  const int r = s_bits;
  __syncthreads();
  return r;
}

// mode 0: run steps; mode 1: check only (stats of the current state);
// mode 2: snap only (uses the stats and interest list of the last check).
template <int kMode>
__global__ void __launch_bounds__(kBlock) k_engine(DevMesh M, DevField F, DevWork W, StepParams P) {
  Ctl* ctl = W.ctl;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gsz = gridDim.x * blockDim.x;
  unsigned long long ep = static_cast<unsigned long long>(ctl->epoch);
  bool pend = ctl->trail_pending != 0;
  long long pend_step = ctl->trail_step;

  if (kMode == 1) {
    if (gtid < P.n_active) flush_and_reset_stat(M, W, P, gtid, false, 0);
    if (gtid == 0) {
      ctl->icount = 0;
      ctl->npairs = 0;
      ctl->pair_overflow = 0;
      ctl->base_max_bits = 0;
    }
    grid_sync(ctl);
    ++ep;
    phase_band_list(F, W, M.nv, false);
    grid_sync(ctl);
    phase_union(M, F, W, P, ep);
    grid_sync(ctl);
    phase_stats(M, F, W, P, ep);
    grid_sync(ctl);
    if (gtid == 0) ctl->epoch = static_cast<long long>(ep);
    return;
  }
  if (kMode == 2) {
    phase_snap(M, F, W, P);
    return;
  }
  if (kMode == 3) {  // write trail / last position records for a host-handled check
    if (gtid < P.n_active) flush_and_reset_stat(M, W, P, gtid, true, P.step_begin);
    return;
  }

  long long step = P.step_begin;
  int stop = 0;
  for (; step < P.step_end; ++step) {
    const int cur = static_cast<int>(step & 1), nxt = cur ^ 1;
    const bool check = P.do_check && (step % P.check_interval == 0);
    // ---- A: update (+ pending trail snap of the previous check)
    const int nR = ctl->rcount[cur];
    if (gtid == 0) {
      ctl->rcount[nxt] = 0;
      ctl->hash_acc = 0;
      ctl->sum_region += static_cast<unsigned long long>(nR);
    }
    for (int i = gtid; i < nR; i += gsz) update_vertex(M, F, W, P, i, W.region[cur][i]);
    if (pend && P.record_trails) phase_snap(M, F, W, P);
    grid_sync(ctl);
    if (ctl->error) {
      stop = kStopError;
      break;
    }
    // ---- B: commit, next frontier, trail flush, stat reset
    for (int i = gtid; i < nR; i += gsz) commit_vertex(M, F, W, i, W.region[cur][i], static_cast<int>(step), nxt);
    if (gtid < P.n_active) flush_and_reset_stat(M, W, P, gtid, pend, pend_step);
    if (gtid == 0) {
      ctl->icount = 0;
      ctl->npairs = 0;
      ctl->pair_overflow = 0;
      ctl->base_max_bits = 0;
    }
    pend = false;
    grid_sync(ctl);
    if (!check) continue;
    ++ep;
    // ---- C: interest list (+ digest)
    phase_band_list(F, W, M.nv, P.do_hash != 0);
    grid_sync(ctl);
    // ---- D: union-find over band items
    phase_union(M, F, W, P, ep);
    grid_sync(ctl);
    // ---- E: statistics and collisions
    phase_stats(M, F, W, P, ep);
    grid_sync(ctl);
    if (gtid == 0) ctl->sum_interest += static_cast<unsigned long long>(ctl->icount);
    if (P.do_hash && gtid == 0) {
      const long long slot = step - W.hash_base;
      if (slot >= 0 && slot < W.hash_cap) W.hashes[slot] = ctl->hash_acc;
    }
    int bits = decide(W, P);
    if (P.stop_every_check) bits |= kStopEveryCheck;
    if (bits) {
      stop = bits;
      break;
    }
    pend = true;
    pend_step = step;
  }
  if (stop == 0 && pend && P.record_trails) {
    // Budget exhausted right after a quiet check: finish its trail records.
    phase_snap(M, F, W, P);
    grid_sync(ctl);
  }
  if (stop == 0 && pend) {
    if (gtid < P.n_active) flush_and_reset_stat(M, W, P, gtid, true, pend_step);
    pend = false;
  }
  if (gtid == 0) {
    ctl->stop_bits = stop;
    ctl->stop_step = stop ? step : step - 1;
    ctl->epoch = static_cast<long long>(ep);
    ctl->trail_pending = 0;
  }
}

int coop_launch(const void* fn, int blocks, const DevMesh& m, const DevField& f, const DevWork& w,
                const StepParams& p, void* stream) {
  DevMesh mm = m;
  DevField ff = f;
  DevWork ww = w;
  StepParams pp = p;
  void* args[] = {&mm, &ff, &ww, &pp};
  note_launch();
  return static_cast<int>(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kBlock), args, 0,
                                                      static_cast<cudaStream_t>(stream)));
}

}  // namespace

static unsigned long long g_launches = 0;
unsigned long long launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }
void note_launch(unsigned long long n) { __atomic_fetch_add(&g_launches, n, __ATOMIC_RELAXED); }

int dev_max_coresident_blocks(int* out) {
  int dev = 0, sms = 0, per = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_engine<0>, kBlock, 0);
  if (e != cudaSuccess) return static_cast<int>(e);
  int per1 = 0, per2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_engine<1>, kBlock, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_engine<2>, kBlock, 0);
  if (per1 < per) per = per1;
  *out = sms * (per < 1 ? 1 : per);
  return 0;
}

int launch_run(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, int blocks,
               void* stream) {
  return coop_launch(reinterpret_cast<const void*>(&k_engine<0>), blocks, m, f, w, p, stream);
}

int launch_check(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, int blocks,
                 void* stream) {
  return coop_launch(reinterpret_cast<const void*>(&k_engine<1>), blocks, m, f, w, p, stream);
}

int launch_snap(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, void* stream) {
  note_launch();
  k_engine<2><<<148 * 4, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(m, f, w, p);
  return static_cast<int>(cudaGetLastError());
}

int launch_flush(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, void* stream) {
  const int blocks = (p.n_active + kBlock - 1) / kBlock;
  if (blocks == 0) return 0;
  note_launch();
  k_engine<3><<<blocks, kBlock, 0, static_cast<cudaStream_t>(stream)>>>(m, f, w, p);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace dtb
