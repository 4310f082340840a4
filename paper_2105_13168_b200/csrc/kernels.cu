#include <cstdio>
#include <cstring>
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

#include <cooperative_groups.h>

#include <cstdint>

#include "kernels.h"

namespace dtb {

void note_launch(unsigned long long n);

namespace {

constexpr int kCand = 32;  // candidate layers gathered over one stiffness row
constexpr int kWork = 48;  // working column capacity before the final size check
constexpr unsigned long long kVertMask = (1ull << 27) - 1;  // vertex bits of a snap key

__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }
__device__ __forceinline__ double max0(double x) { return x < 0.0 ? 0.0 : x; }  // std::max(x, 0.0)

// Errors of a speculative update (the next step's, computed while the
// current step's check runs) only become real if the check finds no event.
__device__ __forceinline__ void raise_error(Ctl* ctl, int code, int v, bool spec) {
  int* slot = spec ? &ctl->spec_error : &ctl->error;
  int prev = atomicMax(slot, code);
  if (prev < code) *(spec ? &ctl->spec_error_vertex : &ctl->error_vertex) = v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Build-time diagnostics (-DDTB_INSTR): per-item latency histograms of the
// step phases (B commit, D union, E stats, A fast, A slow), 128 ns * 2^b
// buckets, staged in shared memory and summed at kernel exit.
#ifdef DTB_INSTR
__device__ unsigned long long g_hist[6][16];
__shared__ unsigned s_hist[6][16];
__device__ __forceinline__ void instr_rec(int ph, unsigned long long t0) {
  const unsigned long long dt = gtimer() - t0;
  int b = 0;
  while (b < 15 && (128ull << b) < dt) ++b;
  atomicAdd(&s_hist[ph][b], 1u);
}
__device__ unsigned long long g_cp[32][2];
__shared__ unsigned s_cp[32][2];  // 32-bit: native shared atomics (64-bit ones are CAS loops)
__device__ __forceinline__ void instr_cp(int idx, unsigned long long t0) {
  if ((threadIdx.x & 7) == 0) {
    atomicAdd(&s_cp[idx][0], static_cast<unsigned>((static_cast<unsigned long long>(clock64()) - t0) >> 4));
    atomicAdd(&s_cp[idx][1], 1u);
  }
}
// Phase timeline: cycles since the CTA's phase start (set where the control
// snapshot is taken), checkpoint `idx` recorded by the first lane of each
// 8-lane group (or of each warp with instr_at_w); `dep` orders the clock read
// after the value it depends on.
__shared__ unsigned long long s_pt0;
__device__ __forceinline__ void instr_at(int idx, unsigned dep, unsigned lanes = 7) {
  // The clock read is predicated on `dep`, so it cannot issue before dep arrives.
  unsigned long long c = 0;
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0x7fffffff; @p mov.u64 %0, %%clock64; }" : "+l"(c) : "r"(dep));
  if ((threadIdx.x & lanes) == 0) {
    atomicAdd(&s_cp[idx][0], static_cast<unsigned>((c - s_pt0) >> 4));
    atomicAdd(&s_cp[idx][1], 1u);
  }
}
#define INSTR_AT(idx, dep) instr_at(idx, static_cast<unsigned>(dep))
#define INSTR_AT_W(idx, dep) instr_at(idx, static_cast<unsigned>(dep), 31)
#define INSTR_PHASE() \
  if (threadIdx.x == 0) s_pt0 = static_cast<unsigned long long>(clock64())
#define INSTR_CP(idx, t0) instr_cp(idx, t0)
#define INSTR_C0(name) const unsigned long long name = static_cast<unsigned long long>(clock64())
#define INSTR_T0(name) const unsigned long long name = gtimer()
#define INSTR_REC(ph, name, cond) \
  do {                            \
    if (cond) instr_rec(ph, name); \
  } while (0)
#else
#define INSTR_T0(name)
#define INSTR_REC(ph, name, cond)
#define INSTR_CP(idx, t0)
#define INSTR_C0(name)
#define INSTR_AT(idx, dep)
#define INSTR_AT_W(idx, dep)
#define INSTR_PHASE()
#endif

// Diagnostics (DTB_PHASE_PROF): per-CTA completion time of phase `ph` of the
// first 64 steps of a launch, recorded just before the grid barrier.
__device__ __forceinline__ unsigned long long gtimer_raw() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void block_done(const DevWork& W, long long rel_step, int ph) {
  if (!W.prof || rel_step < 0 || rel_step >= 64) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long base = W.prof_cap - 64LL * 3 * gridDim.x;
    W.prof[base + (rel_step * 3 + ph) * gridDim.x + blockIdx.x] = gtimer_raw();
  }
}
// Per-CTA phase start (barrier exit) for steps < 64: second table below the first.
__device__ __forceinline__ void block_start(const DevWork& W, long long rel_step, int ph) {
  if (!W.prof || rel_step < 0 || rel_step >= 64 || threadIdx.x != 0) return;
  const long long base = W.prof_cap - 2 * 64LL * 3 * gridDim.x - 16;
  W.prof[base + (rel_step * 3 + ph) * gridDim.x + blockIdx.x] = gtimer_raw();
}

__device__ __forceinline__ void grid_sync(Ctl*) {
  // cooperative_groups' grid barrier measured 1.2 us vs 2.6 us for a
  // counter/generation barrier with gpu-scope fences (148 CTAs, B200).
  cooperative_groups::this_grid().sync();
}

// The control words every thread needs after a barrier (list sizes, error
// flags).  One thread per CTA reads them and shares them through shared
// memory: 148 requests to the control line instead of one per warp (2,368),
// which the L2 slice holding that line would serve one by one.
struct CtlSnap {
  int rcount[4];
  int ilcount[4];
  int error;
  int spec_error;
  int dchange[4];
  int nadded[4];
  int anchor_fail[4];
  int nbandpairs[4];
  int pad_[2];
};
static_assert(sizeof(CtlSnap) == 112, "CtlSnap mirrors the first 112 bytes of Ctl");
__device__ __forceinline__ void ctl_snap(const Ctl* ctl, CtlSnap& sc) {
  if (threadIdx.x == 0) {
    const int4* src = reinterpret_cast<const int4*>(ctl);
    int4* dst = reinterpret_cast<int4*>(&sc);
#pragma unroll
    for (int q = 0; q < 7; ++q) dst[q] = __ldcg(src + q);
    INSTR_PHASE();
  }
  __syncthreads();
}
// After the barrier that completes check `step`: the control snapshot and
// the check's stop decision (decide(), same words) fetched in one round by
// warp 0; the decision lands in sc.pad_[0].
__device__ __forceinline__ void grid_sync_snap_decide(Ctl* ctl, CtlSnap& sc, const DevWork& W, const StepParams& P,
                                                      long long step);
__device__ __forceinline__ void grid_sync_snap(Ctl* ctl, CtlSnap& sc) {
  cooperative_groups::this_grid().sync();
  ctl_snap(ctl, sc);
}

// What an update tells the bookkeeping that follows it (post_update): flag
// bits 1 changed, 2 base was exactly 1, 4 base is exactly 1, 8 the new column
// is interesting, 0x80 valid (clear when the update raised an error); bi is
// the new column's band index.  Valid on the group's lane 0.
struct Hdr {
  unsigned flag;
  uint4 bi;
};
constexpr unsigned kHandled = 0x100u;  // Hdr::flag: the update path applied (on every lane of the group)

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
// layer at vertex v, reading only the committed columns.  An 8-lane group
// works on one vertex: lane j gathers stiffness neighbour j (its column's
// first kReg slots in registers), then every lane folds the neighbours in
// ascending column order through width-8 shuffles -- the reference's
// summation order -- so all lanes hold the same results.
constexpr int kG = 8;    // lanes per vertex group
constexpr int kReg = 4;  // neighbour-column slots kept in registers (packed as 2x2 u16 below)

__device__ __forceinline__ unsigned group_mask() { return 0xFFu << (threadIdx.x & 24); }

// 8-lane group operations on the lanes that execute them together: the mask
// is __activemask() (as in cooperative_groups::coalesced_threads), which
// holds whole groups -- the lanes of a group never diverge from each other in
// the update paths -- and is the same on every participating lane.  A
// per-group mask (0xFF << group) differs between the groups of a warp and
// makes each vote / reduction / shuffle ~10x slower on sm_100a
// (tools/fp64_lat.cu: redux 345 vs 31 cycles, vote.any 304 vs 44).
constexpr unsigned kFull = 0xffffffffu;
__device__ __forceinline__ bool seg_any8(bool p) {
  return ((__ballot_sync(__activemask(), p) >> (threadIdx.x & 24)) & 0xFFu) != 0;
}
__device__ __forceinline__ unsigned seg_min8(unsigned x) {
  const unsigned am = __activemask();
  x = min(x, __shfl_xor_sync(am, x, 4));
  x = min(x, __shfl_xor_sync(am, x, 2));
  return min(x, __shfl_xor_sync(am, x, 1));
}
__device__ __forceinline__ unsigned seg_max8(unsigned x) {
  const unsigned am = __activemask();
  x = max(x, __shfl_xor_sync(am, x, 4));
  x = max(x, __shfl_xor_sync(am, x, 2));
  return max(x, __shfl_xor_sync(am, x, 1));
}

// Element i of a small pointer array held in a kernel parameter, by selects:
// a dynamic index into a parameter array makes the compiler copy the whole
// parameter struct to local memory and load the pointer back from there (a
// dependent memory round trip in front of every use).
template <class T>
__device__ __forceinline__ T pick2(const T (&a)[2], int i) {
  return i ? a[1] : a[0];
}
template <class T>
__device__ __forceinline__ T pick4(const T (&a)[4], int i) {
  const T lo = (i & 1) ? a[1] : a[0];
  const T hi = (i & 1) ? a[3] : a[2];
  return (i & 2) ? hi : lo;
}
__device__ __forceinline__ FieldBuf pickf(const DevField& F, long long t) {  // F.b[t & 1]
  FieldBuf r;
  const bool odd = (t & 1) != 0;
  r.cnt = odd ? F.b[1].cnt : F.b[0].cnt;
  r.lay = odd ? F.b[1].lay : F.b[0].lay;
  r.val = odd ? F.b[1].val : F.b[0].val;
  r.interest = odd ? F.b[1].interest : F.b[0].interest;
  r.binfo = odd ? F.b[1].binfo : F.b[0].binfo;
  return r;
}

// The active flags of the layers (fixed for the whole launch) as a bitmap in
// shared memory: the update reads the activity of every layer it meets, and
// from global memory that was one more dependent round trip per vertex.
__shared__ unsigned s_act[(kMaxLayers + 1 + 31) / 32];
__device__ __forceinline__ bool is_active(unsigned l) { return (s_act[l >> 5] >> (l & 31)) & 1u; }
__device__ void load_active(const unsigned char* active, int n_layers) {
  const int nw = (min(n_layers, kMaxLayers + 1) + 31) / 32;
  for (int w = threadIdx.x; w < nw; w += blockDim.x) {
    unsigned bits = 0;
    for (int j = 0; j < 32; ++j) {
      const int l = w * 32 + j;
      if (l < n_layers && active[l]) bits |= 1u << j;
    }
    s_act[w] = bits;
  }
  for (int w = nw + threadIdx.x; w < (kMaxLayers + 1 + 31) / 32; w += blockDim.x) s_act[w] = 0;
}

// Dynamic shared memory: one slab per 8-lane group, used either for the fold
// staging of the fast update or for the work arrays of the general update
// (which would otherwise live in local memory, i.e. in L2).
constexpr int kSlabBytes = 2048;
constexpr int kDynSmem = (kBlock / kG) * kSlabBytes;
extern __shared__ double s_dyn[];
__device__ __forceinline__ char* group_slab() {
  return reinterpret_cast<char*>(s_dyn) + static_cast<size_t>(threadIdx.x / kG) * kSlabBytes;
}

// Work-to-CTA maps.  Rank r of a group (or thread) is spread round-robin over
// the CTAs so every SM gets an equal share of a short list; the "high" map
// fills each CTA from its last warp so that it does not collide with work
// mapped from the first warp in the same phase.
__device__ __forceinline__ int group_rank(int mode) {
  const int gpb = blockDim.x / kG, gl = threadIdx.x / kG;
  if (mode == 0) return (blockIdx.x * blockDim.x + threadIdx.x) / kG;
  return (mode == 2 ? gpb - 1 - gl : gl) * gridDim.x + blockIdx.x;
}

__device__ __forceinline__ void cand_add(unsigned short* cl, double* ca, int& nc, bool& overflow, int l, double t) {
  int c = 0;
  while (c < nc && cl[c] != l) ++c;
  if (c == nc) {
    if (nc == kCand) {
      overflow = true;
      return;
    }
    cl[nc] = static_cast<unsigned short>(l);
    ca[nc] = 0.0;
    ++nc;
  }
  ca[c] = ca[c] + t;
}

// The new column's band index and interest flag, computed where the column is
// produced and stored with it: make_binfo's definition over the new entries,
// interest = some value strictly inside (0, 1).  NMAX > 0: register arrays of
// that capacity (fully unrolled, constant indices); NMAX == 0: pointers into
// shared memory.
template <int NMAX, class LT, class XT>
__device__ __forceinline__ void column_header(const FieldBuf& Fo, const DevWork& W, int v, int n, const LT& lay,
                                              const XT& val, bool changed, bool old_one, bool new_one, Hdr& h) {
  unsigned L[4] = {0, 0, 0, 0}, S[4] = {0, 0, 0, 0};
  int nb = 0;
  bool over = false, inter = false;
#pragma unroll
  for (int j = 0; j < (NMAX > 0 ? NMAX : kWork); ++j) {
    if (j >= n) break;
    const unsigned l = static_cast<unsigned>(lay[j]);
    const double x = val[j];
    inter |= x > 0.0 && x < 1.0;
    if (l != 0 && x > W.band_lo && x < W.sat) {
      if (nb < 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q)  // constant indices: L and S stay in registers
          if (q == nb) {
            L[q] = l;
            S[q] = static_cast<unsigned>(j);
          }
        ++nb;
      } else {
        over = true;
      }
    }
  }
  uint4 bi = make_uint4(0, 0, 0, 0);
  if (inter) {
    bi.x = L[0] | (L[1] << 16);
    bi.y = L[2] | (L[3] << 16);
    bi.z = S[0] | (S[1] << 16);
    bi.w = S[2] | ((over ? kBandOverflow : S[3]) << 16);
  }
  Fo.binfo[v] = bi;
  Fo.cnt[v] = static_cast<unsigned char>(n);
  Fo.interest[v] = inter ? 1 : 0;
  h.bi = bi;
  h.flag = kHandled | 0x80u | (changed ? 1u : 0u) | (old_one ? 2u : 0u) | (new_one ? 4u : 0u) | (inter ? 8u : 0u);
}

__device__ Hdr update_vertex(const DevMesh& M, const FieldBuf& F, const FieldBuf& Fo, const DevWork& W,
                             const StepParams& P, int v, bool spec, int lane, unsigned gm) {
  Hdr h;
  h.flag = kHandled;
  h.bi = make_uint4(0, 0, 0, 0);
  // Work arrays in the group's shared-memory slab.  Every lane of the group
  // runs this code with the same values, so each lane reads back what it
  // (and its siblings, identically) wrote.
  double* const ox = reinterpret_cast<double*>(group_slab());
  double* const ca = ox + kSlots;
  double* const nx = ca + kCand;
  double* const sx = nx + kWork;
  unsigned short* const ol = reinterpret_cast<unsigned short*>(sx + kWork);
  unsigned short* const cl = ol + kSlots;
  unsigned short* const nl = cl + kCand;
  unsigned short* const sl = nl + kWork;
  static_assert((kSlots + kCand + 2 * kWork) * (8 + 2) <= kSlabBytes, "the general update's arrays fit the slab");
  INSTR_C0(tU);
  __syncwarp(__activemask());  // the slab may hold the fold staging of this group's previous vertex
  const int cv = F.cnt[v];
  const size_t vb = static_cast<size_t>(v) * kSlots;
  // The column is staged lane-parallel (slot j on lane j % kG), and the
  // activity of its layers is gathered into own_act (bit j: slot j holds an
  // active non-base layer) so lane 0's sequential part makes no global loads.
  unsigned own_act = 0;
  for (int jb = 0; jb < cv; jb += kG) {
    const int j = jb + lane;
    bool act = false;
    if (j < cv) {
      const int l = F.lay[vb + j];
      ol[j] = static_cast<unsigned short>(l);
      ox[j] = F.val[vb + j];
      act = l != 0 && is_active(l);
    }
    own_act |= ((__ballot_sync(__activemask(), act) >> (threadIdx.x & 24)) & 0xFFu) << jb;
  }
  __syncwarp(__activemask());
  const double phib = (cv > 0 && ol[0] == 0) ? ox[0] : 0.0;

  int nc = 0;
  double lapb = 0.0, lapt = 0.0;
  bool bnear = phib > 0.0;
  bool overflow = false;
  const int k0 = __ldg(M.s_off + v), k1 = __ldg(M.s_off + v + 1);
  for (int kb = k0; kb < k1; kb += kG) {
    const int k = kb + lane;
    const bool valid = k < k1;
    int u = 0, cu = 0;
    double s = 0.0, bu = 0.0, au = 0.0;
    unsigned short L[kReg];
    double X[kReg];
#pragma unroll
    for (int q = 0; q < kReg; ++q) {
      L[q] = 0;
      X[q] = 0.0;
    }
    unsigned amask = 0;  // bit q: neighbour slot q < min(cu, kReg) holds an active layer
    if (valid) {
      u = __ldg(M.s_col + k);
      s = __ldg(M.s_val + k);
      cu = F.cnt[u];
      const size_t b = static_cast<size_t>(u) * kSlots;
#pragma unroll
      for (int q = 0; q < kReg; ++q)
        if (q < cu) {
          L[q] = F.lay[b + q];
          X[q] = F.val[b + q];
        }
#pragma unroll
      for (int q = 0; q < kReg; ++q)
        if (q < cu) {
          if (L[q] == 0) {
            bu = X[q];
          } else if (is_active(L[q])) {
            au = au + X[q];
            amask |= 1u << q;
          }
        }
      for (int q = kReg; q < cu; ++q) {
        const int l = F.lay[b + q];
        const double x = F.val[b + q];
        if (l == 0) bu = x;
        else if (is_active(l)) au = au + x;
      }
    }
    const int nvalid = min(kG, k1 - kb);
    for (int jj = 0; jj < nvalid; ++jj) {
      const double s_ = __shfl_sync(__activemask(), s, jj, kG);
      const int cu_ = __shfl_sync(__activemask(), cu, jj, kG);
      const double bu_ = __shfl_sync(__activemask(), bu, jj, kG);
      const double au_ = __shfl_sync(__activemask(), au, jj, kG);
      const unsigned am_ = __shfl_sync(__activemask(), amask, jj, kG);
      lapb = lapb + s_ * bu_;
      lapt = lapt + s_ * au_;
      if (bu_ > 0.0) bnear = true;
#pragma unroll
      for (int q = 0; q < kReg; ++q) {
        const int l_ = __shfl_sync(__activemask(), static_cast<int>(L[q]), jj, kG);
        const double x_ = __shfl_sync(__activemask(), X[q], jj, kG);
        if (lane == 0 && ((am_ >> q) & 1)) cand_add(cl, ca, nc, overflow, l_, s_ * x_);
      }
      if (cu_ > kReg) {
        // Slots past kReg: loaded lane-parallel, added by lane 0 in slot order.
        const int u_ = __shfl_sync(__activemask(), u, jj, kG);
        const size_t b = static_cast<size_t>(u_) * kSlots;
        for (int qb = kReg; qb < cu_; qb += kG) {
          const int q = qb + lane;
          int l = 0;
          double x = 0.0;
          bool act = false;
          if (q < cu_) {
            l = F.lay[b + q];
            x = F.val[b + q];
            act = l != 0 && is_active(l);
          }
          const unsigned am = (__ballot_sync(__activemask(), act) >> (threadIdx.x & 24)) & 0xFFu;
          const int m = min(kG, cu_ - qb);
          for (int t = 0; t < m; ++t) {
            const int l_ = __shfl_sync(__activemask(), l, t, kG);
            const double x_ = __shfl_sync(__activemask(), x, t, kG);
            if (lane == 0 && ((am >> t) & 1)) cand_add(cl, ca, nc, overflow, l_, s_ * x_);
          }
        }
      }
    }
  }
  // From here on lane 0 alone: the candidate list and the working column live
  // in the group's slab, so only one lane may write them.  (Its siblings meet
  // it again at the group's next shuffle or __syncwarp.)
  if (lane != 0) return;
  // Layers held at v itself are near support even if the stiffness row
  // lacks its diagonal (never on valid meshes, kept for exactness).
  for (int j = 0; j < cv; ++j) {
    const int l = ol[j];
    if (!((own_act >> j) & 1)) continue;
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
    raise_error(W.ctl, kDevCapacity, v, spec);
    return h;
  }
#ifdef DTB_INSTR
  atomicAdd(&s_hist[5][min(nc, 15)], 1u);  // candidate layers of general-path vertices
  {
    int nown = 0;
    for (int j = 0; j < cv; ++j) nown += (own_act >> j) & 1;
    atomicAdd(&s_hist[4][min(cv, 15)], 1u);  // column length
  }
#endif

  const double mass = __ldg(M.mass + v);
  const double lap_b = lapb / mass;
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
      raise_error(W.ctl, kDevBlowup, v, spec);
      return h;
    }
    const double next = clamp01(phi + P.dt * rate);
    if (next != phi) {
      touched = true;
      ok &= col_set(nl, nx, nn, l, next, P.prune, changed);
    }
  }
  if (bnear) {
    double total = 0.0, contact = 0.0;
    for (int j = 0; j < cv; ++j)
      if ((own_act >> j) & 1) total = total + ox[j];
    for (int j = 0; j < cv; ++j)
      if ((own_act >> j) & 1) contact = contact + sqrt(max0(phib * ox[j]));
    const double lap_total = lapt / mass;
    const double rate = -P.mu_n * (P.w * total + P.half_a2 * lap_total + P.e * contact) +
                        P.m_mu_n * (P.w * phib + P.half_a2 * lap_b);
    if (!isfinite(rate)) {
      raise_error(W.ctl, kDevBlowup, v, spec);
      return h;
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
      raise_error(W.ctl, kDevZeroColumn, v, spec);
      return h;
    }
    if (!(fabs(s - 1.0) < 1e-15)) {
      const int sn = nn;
      for (int j = 0; j < sn; ++j) {
        sl[j] = nl[j];
        sx[j] = nx[j];
      }
      for (int j = 0; j < sn; ++j) ok &= col_set(nl, nx, nn, sl[j], sx[j] / s, P.prune, changed);
    }
  }
  if (!ok || nn > kSlots) {
    raise_error(W.ctl, kDevCapacity, v, spec);
    return h;
  }
  const bool old_one = cv > 0 && ol[0] == 0 && ox[0] == 1.0;
  const bool new_one = nn > 0 && nl[0] == 0 && nx[0] == 1.0;
  const size_t o = static_cast<size_t>(v) * kSlots;
  for (int j = 0; j < nn; ++j) {
    Fo.lay[o + j] = nl[j];
    Fo.val[o + j] = nx[j];
  }
  column_header<0>(Fo, W, v, nn, nl, nx, changed, old_one, new_one, h);
  return h;
}

// ---------------------------------------------------------------------------
// Lane-parallel path for wide columns (many layers around v; a high-genus
// gyroid puts 9-10 candidate layers on a third of its frontier): own column,
// neighbour columns and candidate layers of at most kWide entries, a row of
// at most kG entries.  The sequential general path's results, bit for bit:
//  * every per-candidate neighbour sum adds s_j * x_j in row order (a +0.0
//    for a neighbour without the layer is never added: the sum is the
//    sequential path's, whose candidate order does not matter -- each layer
//    is set once, and col_set of distinct layers commutes);
//  * the candidate and base rates are the same expressions, one candidate
//    per lane; the contact and total sums run in slot order on lane 0;
//  * the new column is the merge of the own column with the updated and
//    inserted layers (set_value: clamp above 1, prune below the epsilon);
//  * normalisation sums in column order on lane 0 and divides per lane.
// Not handled (flag 0, no side effects) when the case does not fit.
constexpr int kWide = 16;
struct WideSlab {  // one group's slab (kSlabBytes)
  double ox[kWide];           // own column values
  double nbx[kG][kWide];      // neighbour j's active non-base values (slot order); later the new column
  double ca[kWide];           // per-candidate neighbour sums
  double rn[kWide];           // per-candidate next values; contact terms
  unsigned short ol[kWide];   // own column layers
  unsigned short nbl[kG][kWide];
  unsigned short cl[kWide];   // candidate layers, ascending
  unsigned short nl2[2 * kWide + 8];  // new column layers
  int nbn[kG];                // neighbour j's staged entries
};
static_assert(sizeof(WideSlab) <= kSlabBytes, "the wide path's arrays fit the slab");
static_assert(sizeof(double) * (2 * kWide + 8) <= sizeof(double) * kG * kWide, "the new column fits the nbx area");

__device__ Hdr update_vertex_wide(const DevMesh& M, const FieldBuf& F, const FieldBuf& Fo, const DevWork& W,
                                  const StepParams& P, int v, bool spec, int lane) {
  Hdr h;
  h.flag = 0;
  h.bi = make_uint4(0, 0, 0, 0);
  WideSlab& S = *reinterpret_cast<WideSlab*>(group_slab());
  const int cv = F.cnt[v];
  const int k0 = __ldg(M.s_off + v), k1 = __ldg(M.s_off + v + 1);
  const int rlen = k1 - k0;
  if (cv > kWide || rlen > kG) return h;  // group-uniform
  const bool valid = lane < rlen;
  int u = 0, cu = 0;
  double s = 0.0;
  if (valid) {
    u = __ldg(M.s_col + k0 + lane);
    s = __ldg(M.s_val + k0 + lane);
    cu = F.cnt[u];
  }
  if (seg_any8(cu > kWide)) return h;
  INSTR_AT(16, cu);
  __syncwarp(__activemask());  // the slab may hold this group's previous staging
  // Own column, slot j on lane j % kG, with its activity bits.
  // Every load of the own column (slots lane, lane + kG) and of neighbour
  // lane's column (its first kWide slots: in bounds, the column holds kSlots)
  // is issued before any is used: one round trip for all of them.
  const size_t vb = static_cast<size_t>(v) * kSlots;
  const int ol0 = F.lay[vb + lane], ol1 = F.lay[vb + lane + kG];
  const double ox0 = F.val[vb + lane], ox1 = F.val[vb + lane + kG];
  const size_t b = static_cast<size_t>(u) * kSlots;
  const uint4 lw0 = *reinterpret_cast<const uint4*>(F.lay + b), lw1 = *reinterpret_cast<const uint4*>(F.lay + b + 8);
  double2 xw[kWide / 2];
#pragma unroll
  for (int k = 0; k < kWide / 2; ++k)
    xw[k] = 2 * k < cu ? *reinterpret_cast<const double2*>(F.val + b + 2 * k) : make_double2(0.0, 0.0);
  unsigned own_act = 0;
  {
    const bool a0 = lane < cv && ol0 != 0 && is_active(ol0);
    const bool a1 = lane + kG < cv && ol1 != 0 && is_active(ol1);
    if (lane < cv) {
      S.ol[lane] = static_cast<unsigned short>(ol0);
      S.ox[lane] = ox0;
    }
    if (lane + kG < cv) {
      S.ol[lane + kG] = static_cast<unsigned short>(ol1);
      S.ox[lane + kG] = ox1;
    }
    own_act = ((__ballot_sync(__activemask(), a0) >> (threadIdx.x & 24)) & 0xFFu) |
              (((__ballot_sync(__activemask(), a1) >> (threadIdx.x & 24)) & 0xFFu) << kG);
  }
  // Neighbour j's column: base value bu, active sum au (slot order), and its
  // active layers staged in slot (= ascending layer) order.
  double bu = 0.0, au = 0.0;
  int na = 0;
  {
    const unsigned lw[8] = {lw0.x, lw0.y, lw0.z, lw0.w, lw1.x, lw1.y, lw1.z, lw1.w};
#pragma unroll
    for (int q = 0; q < kWide; ++q) {
      if (q < cu) {
        const int l = static_cast<int>((lw[q / 2] >> (16 * (q & 1))) & 0xFFFFu);
        const double x = (q & 1) ? xw[q / 2].y : xw[q / 2].x;
        if (l == 0) {
          bu = x;
        } else if (is_active(l)) {
          au = au + x;
          S.nbl[lane][na] = static_cast<unsigned short>(l);
          S.nbx[lane][na] = x;
          ++na;
        }
      }
    }
  }
  S.nbn[lane] = na;
  INSTR_AT(17, na);
  const double phib = (cv > 0 && S.ol[0] == 0) ? S.ox[0] : 0.0;
  // Ordered row folds of s_j * bu_j and s_j * au_j (the general path's lapb, lapt).
  const double tb = s * bu, tt = s * au;
  double lapb = 0.0, lapt = 0.0;
  {
    const unsigned am = __activemask();
#pragma unroll
    for (int jj = 0; jj < kG; ++jj) {
      const double b_ = __shfl_sync(am, tb, jj, kG);
      const double t_ = __shfl_sync(am, tt, jj, kG);
      if (jj < rlen) {
        lapb = lapb + b_;
        lapt = lapt + t_;
      }
    }
  }
  const bool bnear = phib > 0.0 || seg_any8(valid && bu > 0.0);
  __syncwarp(__activemask());
  // Candidate layers: the ascending union of the own active layers (lane 0)
  // and the neighbours' staged layers (lane j), one per merge round.
  int nc = 0;
  {
    // Every lane walks the own column's cursor (the same on all lanes, so
    // no lane diverges before the group reduction); lane 0 offers its head.
    int pn = 0, po = 0;  // cursors: neighbour list, own column
    for (;;) {
      while (po < cv && !((own_act >> po) & 1)) ++po;
      const unsigned oh = po < cv ? static_cast<unsigned>(S.ol[po]) : 0xFFFFFFFFu;
      const unsigned nh = pn < na ? S.nbl[lane][pn] : 0xFFFFFFFFu;
      const unsigned m = seg_min8(lane == 0 ? min(nh, oh) : nh);
      if (m == 0xFFFFFFFFu) break;
      if (nc == kWide) return h;  // too many candidates: not handled (no side effects yet)
      if (lane == 0) S.cl[nc] = static_cast<unsigned short>(m);
      ++nc;
      if (pn < na && S.nbl[lane][pn] == m) ++pn;
      if (po < cv && S.ol[po] == m) ++po;
    }
  }
  __syncwarp(__activemask());
  INSTR_AT(18, nc);
  // Per-candidate neighbour sums in row order, candidates lane and lane + kG.
  {
    double acc0 = 0.0, acc1 = 0.0;
    const unsigned l0 = lane < nc ? S.cl[lane] : 0xFFFFu, l1 = lane + kG < nc ? S.cl[lane + kG] : 0xFFFFu;
    for (int jj = 0; jj < rlen; ++jj) {
      // The mask is taken per round: groups with shorter rows leave the loop
      // early, and a mask naming their lanes would wait for them forever.
      const double s_ = __shfl_sync(__activemask(), s, jj, kG);
      const int n_ = S.nbn[jj];
      for (int q = 0; q < n_; ++q) {
        const unsigned l = S.nbl[jj][q];
        if (l == l0) acc0 = acc0 + s_ * S.nbx[jj][q];
        if (l == l1) acc1 = acc1 + s_ * S.nbx[jj][q];
      }
    }
    if (lane < nc) S.ca[lane] = acc0;
    if (lane + kG < nc) S.ca[lane + kG] = acc1;
  }
  INSTR_AT(19, 1u);
  const double mass = __ldg(M.mass + v);
  const double lap_b = lapb / mass;
  // Candidate rates, one candidate per lane and round.
  bool blow = false;
  unsigned cupd = 0;  // bit c: candidate c's value moves
  for (int cb = 0; cb < nc; cb += kG) {
    const int c = cb + lane;
    bool upd = false;
    if (c < nc) {
      const unsigned l = S.cl[c];
      double phi = 0.0;
      for (int j = 0; j < cv; ++j)
        if (S.ol[j] == l) phi = S.ox[j];
      if (!(phi == 0.0 && phib <= P.prune)) {
        const double lap_i = S.ca[c] / mass;
        const double inner = P.w * (phib - phi) + P.half_a2 * (lap_b - lap_i) - P.e * sqrt(max0(phi * phib));
        const double rate = -P.mu_n * inner;
        if (!isfinite(rate)) {
          blow = true;
        } else {
          const double next = clamp01(phi + P.dt * rate);
          if (next != phi) {
            upd = true;
            S.rn[c] = next;
          }
        }
      }
    }
    cupd |= ((__ballot_sync(__activemask(), upd) >> (threadIdx.x & 24)) & 0xFFu) << cb;
  }
  if (seg_any8(blow)) {
    if (lane == 0) raise_error(W.ctl, kDevBlowup, v, spec);
    h.flag = kHandled;
    return h;
  }
  __syncwarp(__activemask());
  // Base rate: the contact terms per own slot on the lanes, the ordered sums
  // and the rate on lane 0.
  bool bupd = false;
  double bnext = 0.0;
  if (bnear) {
    for (int j = lane; j < cv; j += kG)
      if ((own_act >> j) & 1) S.nbx[0][j] = sqrt(max0(phib * S.ox[j]));
    __syncwarp(__activemask());
    if (lane == 0) {
      double total = 0.0, contact = 0.0;
      for (int j = 0; j < cv; ++j)
        if ((own_act >> j) & 1) total = total + S.ox[j];
      for (int j = 0; j < cv; ++j)
        if ((own_act >> j) & 1) contact = contact + S.nbx[0][j];
      const double lap_total = lapt / mass;
      const double rate = -P.mu_n * (P.w * total + P.half_a2 * lap_total + P.e * contact) +
                          P.m_mu_n * (P.w * phib + P.half_a2 * lap_b);
      if (!isfinite(rate)) {
        blow = true;
      } else {
        const double next = clamp01(phib + P.dt * rate);
        if (next != phib) {
          bupd = true;
          bnext = next;
        }
      }
    }
    if (__shfl_sync(__activemask(), blow, 0, kG)) {
      if (lane == 0) raise_error(W.ctl, kDevBlowup, v, spec);
      h.flag = kHandled;
      return h;
    }
    __syncwarp(__activemask());
  }
  INSTR_AT(20, static_cast<unsigned>(bupd));
  h.flag = kHandled;
  if (lane != 0) return h;  // lane 0 alone from here (the slab is its own)
  // The new column: merge of the own column and the updated / inserted
  // layers, set_value semantics (layer_field.hpp:102).
  double* const nx2 = &S.nbx[0][0];
  unsigned short* const nl2 = S.nl2;
  bool changed = false;
  const bool touched = cupd != 0 || bupd;
  int nn = 0;
  auto setv = [&](double val, double old, bool present) -> double {
    if (val > 1.0) val = 1.0;
    if (val < P.prune) val = 0.0;
    if (present ? (val != old) : (val != 0.0)) changed = true;
    return val;
  };
  int jo = 0, c = 0;
  if (bupd && phib == 0.0) {  // the base enters the column (sorted first)
    const double val = setv(bnext, 0.0, false);
    if (val != 0.0) {
      nl2[nn] = 0;
      nx2[nn] = val;
      ++nn;
    }
  }
  while (jo < cv || c < nc) {
    const unsigned lo = jo < cv ? S.ol[jo] : 0x10000u;
    const unsigned lc = c < nc ? S.cl[c] : 0x10000u;
    if (lo <= lc) {  // an own entry (possibly also a candidate)
      double val = S.ox[jo];
      if (lo == 0) {
        if (bupd) val = setv(bnext, val, true);
      } else if (lo == lc && ((cupd >> c) & 1)) {
        val = setv(S.rn[c], val, true);
      }
      if (val != 0.0) {
        nl2[nn] = static_cast<unsigned short>(lo);
        nx2[nn] = val;
        ++nn;
      }
      if (lo == lc) ++c;
      ++jo;
    } else {  // a candidate layer not in the column
      if ((cupd >> c) & 1) {
        const double val = setv(S.rn[c], 0.0, false);
        if (val != 0.0) {
          nl2[nn] = static_cast<unsigned short>(lc);
          nx2[nn] = val;
          ++nn;
        }
      }
      ++c;
    }
  }
  INSTR_AT(21, static_cast<unsigned>(nn));
  // Column normalisation of touched vertices (layer_field.hpp:143).
  if (touched) {
    double ssum = 0.0;
    for (int j = 0; j < nn; ++j) ssum = ssum + nx2[j];
    if (ssum <= 0.0) {
      raise_error(W.ctl, kDevZeroColumn, v, spec);
      return h;
    }
    if (!(fabs(ssum - 1.0) < 1e-15)) {
      int m = 0;
      for (int j = 0; j < nn; ++j) {
        double q = nx2[j] / ssum;
        if (q > 1.0) q = 1.0;
        if (q < P.prune) q = 0.0;
        if (q != nx2[j]) changed = true;
        if (q != 0.0) {
          nl2[m] = nl2[j];
          nx2[m] = q;
          ++m;
        }
      }
      nn = m;
    }
  }
  if (nn > kSlots) {
    raise_error(W.ctl, kDevCapacity, v, spec);
    return h;
  }
  INSTR_AT(22, static_cast<unsigned>(nn));
  const bool old_one = cv > 0 && S.ol[0] == 0 && S.ox[0] == 1.0;
  const bool new_one = nn > 0 && nl2[0] == 0 && nx2[0] == 1.0;
  for (int j = 0; j < nn; ++j) {
    Fo.lay[vb + j] = nl2[j];
    Fo.val[vb + j] = nx2[j];
  }
  column_header<0>(Fo, W, v, nn, nl2, nx2, changed, old_one, new_one, h);
  return h;
}

// ---------------------------------------------------------------------------
// Register-resident fast path of update_vertex for the common case -- at most
// kF owners at v, at most kF candidate layers, at most 8 owners afterwards.
// Every array index is a compile-time constant after unrolling, so nothing
// spills to local memory; the arithmetic (and its order) is exactly the slow
// path's.  Returns false, with no side effects, when the case does not fit.
constexpr int kF = 4;
constexpr int kN = 8;
constexpr int kNoLayer = 0x10000;  // sorts after every layer id

__device__ __forceinline__ void cand_add_reg(int (&Cl)[kF], double (&Ca)[kF], int& nc, bool& over, int l, double t) {
  bool found = false;
#pragma unroll
  for (int c = 0; c < kF; ++c)
    if (c < nc && Cl[c] == l) {
      Ca[c] = Ca[c] + t;
      found = true;
    }
  if (found) return;
  if (nc == kF) {
    over = true;
    return;
  }
#pragma unroll
  for (int c = 0; c < kF; ++c)
    if (c == nc) {
      Cl[c] = l;
      Ca[c] = 0.0;
      Ca[c] = Ca[c] + t;
    }
  ++nc;
}

// Inserts (l, x) into the sorted register column E[0..n).
__device__ __forceinline__ void reg_insert(int (&El)[kN], double (&Ex)[kN], int& n, int l, double x) {
  int pos = 0;
#pragma unroll
  for (int j = 0; j < kN; ++j)
    if (j < n && El[j] < l) ++pos;
#pragma unroll
  for (int j = kN - 1; j > 0; --j)
    if (j > pos && j <= n) {
      El[j] = El[j - 1];
      Ex[j] = Ex[j - 1];
    }
#pragma unroll
  for (int j = 0; j < kN; ++j)
    if (j == pos) {
      El[j] = l;
      Ex[j] = x;
    }
  ++n;
}

// Staging for the ordered neighbour folds of update_vertex_fold: lane j of a
// group parks its contributions here and lanes 0..5 each fold one column.
constexpr int kFoldCols = kF + 2;  // kF candidate layers, base laplacian, total laplacian
static_assert(kG * kFoldCols * 8 <= kSlabBytes, "the fold staging of a group fits its slab");

// Gather of the fast path for rows of at most kG stiffness entries whose
// neighbour columns fit kReg slots (the bulk of a front).  The candidate
// layers are found first (group-wide ascending union of the active layers of
// v and its neighbours), then every per-layer sum is one ordered fold: lane j
// contributes s_j * x_j, and lane c adds the group's contributions for its
// column in ascending neighbour order, exactly the reference's order.  This
// replaces the per-(neighbour, slot) candidate insertion of the generic loop
// (the longest dependent instruction chain of the step).  Returns false, with
// no side effects, when the case does not fit.
__device__ __forceinline__ bool gather_fold(const DevMesh& M, const FieldBuf& F, const DevWork& W, int v, int cv,
                                            const int (&Ol)[kF], int k0, int k1, int lane, unsigned gm, int (&Cl)[kF],
                                            double (&Ca)[kF], int& nc, double& lapb, double& lapt, bool& bnear) {
  INSTR_C0(tG);
  const int k = k0 + lane;
  const bool valid = k < k1;
  double s = 0.0, bu = 0.0, au = 0.0;
  int cu = 0;
  unsigned short L[kReg];
  double X[kReg];
  unsigned amask = 0;
#pragma unroll
  for (int q = 0; q < kReg; ++q) {
    L[q] = 0;
    X[q] = 0.0;
  }
  if (valid) {
    const int u = __ldg(M.s_col + k);
    s = __ldg(M.s_val + k);
    const size_t b = static_cast<size_t>(u) * kSlots;
    cu = F.cnt[u];
    const uint2 lw = *reinterpret_cast<const uint2*>(F.lay + b);
    const double2 x01 = *reinterpret_cast<const double2*>(F.val + b);
    const double2 x23 = *reinterpret_cast<const double2*>(F.val + b + 2);
    L[0] = static_cast<unsigned short>(lw.x & 0xFFFF);
    L[1] = static_cast<unsigned short>(lw.x >> 16);
    L[2] = static_cast<unsigned short>(lw.y & 0xFFFF);
    L[3] = static_cast<unsigned short>(lw.y >> 16);
    X[0] = x01.x;
    X[1] = x01.y;
    X[2] = x23.x;
    X[3] = x23.y;
#pragma unroll
    for (int q = 0; q < kReg; ++q)
      if (q < cu) {
        if (L[q] == 0) {
          bu = X[q];
        } else if (is_active(L[q])) {
          au = au + X[q];
          amask |= 1u << q;
        }
      }
  }
  if (seg_any8(cu > kReg)) return false;
  unsigned omask = 0;
#pragma unroll
  for (int q = 0; q < kF; ++q)
    if (q < cv && Ol[q] != 0 && is_active(Ol[q])) omask |= 1u << q;
  // Candidate layers, ascending.
  nc = 0;
  unsigned last = 0;
#pragma unroll
  for (int c = 0; c <= kF; ++c) {
    unsigned m = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < kReg; ++q)
      if (((amask >> q) & 1) && L[q] > last) m = min(m, static_cast<unsigned>(L[q]));
#pragma unroll
    for (int q = 0; q < kF; ++q)
      if (((omask >> q) & 1) && static_cast<unsigned>(Ol[q]) > last) m = min(m, static_cast<unsigned>(Ol[q]));
    m = seg_min8(m);
    if (m == 0xFFFFFFFFu) break;
    if (c == kF) return false;  // more than kF candidates
    Cl[c] = static_cast<int>(m);
    last = m;
    ++nc;
  }
  // Contributions, staged per lane.
  double* s_fold = reinterpret_cast<double*>(group_slab());  // [lane][kFoldCols]
  const int base = threadIdx.x & ~(kG - 1);
  const int gshift = threadIdx.x & 24;
  unsigned pm[kF];
#pragma unroll
  for (int c = 0; c < kF; ++c) {
    double t = 0.0;
    bool present = false;
#pragma unroll
    for (int q = 0; q < kReg; ++q)
      if (c < nc && ((amask >> q) & 1) && L[q] == Cl[c]) {
        t = s * X[q];
        present = true;
      }
    s_fold[lane * kFoldCols + c] = t;
    pm[c] = (__ballot_sync(__activemask(), present) >> gshift) & 0xFFu;
  }
  s_fold[lane * kFoldCols + kF] = s * bu;
  s_fold[lane * kFoldCols + kF + 1] = s * au;
  const unsigned vm = (__ballot_sync(__activemask(), valid) >> gshift) & 0xFFu;
  bnear = bnear || ((__ballot_sync(__activemask(), valid && bu > 0.0) >> gshift) & 0xFFu) != 0;
  __syncwarp(__activemask());
  double acc = 0.0;
  if (lane < kFoldCols) {
    unsigned use = vm;
#pragma unroll
    for (int c = 0; c < kF; ++c)
      if (lane == c) use = pm[c];
#pragma unroll
    for (int jj = 0; jj < kG; ++jj)
      if ((use >> jj) & 1) acc = acc + s_fold[jj * kFoldCols + lane];
  }
  __syncwarp(__activemask());  // s_fold is reused by the group's next vertex
#pragma unroll
  for (int c = 0; c < kF; ++c) Ca[c] = __shfl_sync(__activemask(), acc, c, kG);
  lapb = __shfl_sync(__activemask(), acc, kF, kG);
  lapt = __shfl_sync(__activemask(), acc, kF + 1, kG);
  return true;
}

// Fast path for the bulk of a single front: v and its stiffness neighbours
// carry at most the base layer and one and the same active layer L (columns
// of at most two owners, row of at most kG entries).  Then the candidate set
// is {L} and its neighbour sum equals the total-Laplacian sum: both add
// s_j * x_j(L) in row order, the latter also adding s_j * 0.0 = +-0.0 for
// neighbours without L, which leaves a sum of positive-valued terms (never
// -0.0) unchanged.  Every lane folds the two sums from shuffles and runs the
// sequential update (the general fast path's arithmetic, term for term);
// lanes 0..n-1 store the new column.
//
// The group-level votes and reductions use the mask of the lanes executing
// together (seg_any8): in the common case the whole warp, a single fast
// instruction.  Not handled (flag 0, no side effects) when the case does not
// apply; with act false the group only rides along (no side effects).
__device__ Hdr update_vertex_single(const DevMesh& M, const FieldBuf& F, const FieldBuf& Fo, const DevWork& W,
                                    const StepParams& P, int v, bool act, bool spec, int lane) {
  Hdr h;
  h.flag = 0;
  h.bi = make_uint4(0, 0, 0, 0);
  const int cv = F.cnt[v];
  const size_t vb = static_cast<size_t>(v) * kSlots;
  const unsigned own_lw = *reinterpret_cast<const unsigned*>(F.lay + vb);  // slots 0, 1
  const double2 own_x = *reinterpret_cast<const double2*>(F.val + vb);
  const double mass = __ldg(M.mass + v);
  // The padded row: lane j's entry is one load away from v.
  const int rlen = __ldg(M.e_len + v);
  const int u_e = __ldg(M.e_col + static_cast<size_t>(v) * kEll + lane);
  const double s_e = __ldg(M.e_val + static_cast<size_t>(v) * kEll + lane);
  const bool valid = lane < rlen;
  const int u = valid ? u_e : 0;
  const double s = valid ? s_e : 0.0;
  const size_t ub = static_cast<size_t>(u) * kSlots;
  const int cu = valid ? static_cast<int>(F.cnt[u]) : 0;
  const unsigned nlw = valid ? *reinterpret_cast<const unsigned*>(F.lay + ub) : 0u;
  const double2 nx = valid ? *reinterpret_cast<const double2*>(F.val + ub) : make_double2(0.0, 0.0);
  INSTR_AT(2, own_lw);
  INSTR_AT(3, nlw);
  // Own column: [base][, L] or [L].
  const unsigned o0 = own_lw & 0xFFFFu, o1 = own_lw >> 16;
  const double phib = (cv > 0 && o0 == 0) ? own_x.x : 0.0;
  unsigned ol = 0;  // own non-base layer (0: none)
  double ox = 0.0;
  bool bad = cv > 2 || rlen > kG;
  if (cv == 1 && o0 != 0) {
    ol = o0;
    ox = own_x.x;
  } else if (cv == 2) {
    if (o0 != 0) bad = true;  // two non-base owners
    ol = o1;
    ox = own_x.y;
  }
  // Neighbour column: base value and its non-base layer.
  double bu = 0.0, xl = 0.0;
  unsigned nl = 0;
  if (valid) {
    const unsigned a0 = nlw & 0xFFFFu, a1 = nlw >> 16;
    if (cu > 2) {
      bad = true;
    } else if (cu == 1) {
      if (a0 == 0) bu = nx.x;
      else {
        nl = a0;
        xl = nx.x;
      }
    } else if (cu == 2) {
      if (a0 != 0) bad = true;
      bu = nx.x;
      nl = a1;
      xl = nx.y;
    }
  }
  // Activity of the non-base layers, looked up as soon as each is known
  // (not after the group agrees on L, which would add a dependent round).
  const bool act_ok = (ol == 0 || is_active(ol)) && (nl == 0 || is_active(nl));
  // One common non-base layer L across v and its neighbours.
  const unsigned lo = seg_min8(min(nl ? nl : 0xFFFFFFFFu, ol ? ol : 0xFFFFFFFFu));
  const unsigned hi = seg_max8(max(nl, ol));
  const bool has_l = lo != 0xFFFFFFFFu;
  const bool fits = !seg_any8(bad || !act_ok) && !(has_l && lo != hi);
  if (!fits) {  // this group falls back (group-uniform); hint: the widest neighbour column
    h.bi.x = seg_max8(static_cast<unsigned>(cu));
    return h;
  }
  INSTR_AT(11, 1u);
  const unsigned L = has_l ? lo : 0u;
  // Ordered folds of s_j * bu_j and s_j * x_j(L) (au_j) over the row.
  const double tb = s * bu, tt = s * xl;
  const bool bpos = valid && bu > 0.0;
  double lapb = 0.0, lapt = 0.0;
  const int nvalid = rlen;
  const unsigned am = __activemask();  // whole groups, see seg_any8
#pragma unroll
  for (int jj = 0; jj < kG; ++jj) {
    const double b_ = __shfl_sync(am, tb, jj, kG);
    const double t_ = __shfl_sync(am, tt, jj, kG);
    if (jj < nvalid) {
      lapb = lapb + b_;
      lapt = lapt + t_;
    }
  }
  const bool bnear = phib > 0.0 || seg_any8(bpos);
  h.flag = kHandled;
  if (!act) return h;
  // ---- the sequential update (uniform across the group's lanes), written
  // without branches so the two divisions and the square root issue
  // together.  The candidate's lap_i and the base's lap_total are the same
  // quotient lapt / mass.  When v holds L (ol == L, phi == ox) the
  // candidate's contact term sqrt(phi * phib) equals the base's
  // sqrt(phib * ox) (IEEE products commute); when it does not (ol == 0,
  // ox == 0) both are +0.
  const double lap_b = lapb / mass;
  const double lap_t = lapt / mass;
  const double sq = sqrt(max0(phib * ox));
  const double phi = ol == L ? ox : 0.0;
  const bool c_on = has_l && !(phi == 0.0 && phib <= P.prune);
  const double rate_c = -P.mu_n * (P.w * (phib - phi) + P.half_a2 * (lap_b - lap_t) - P.e * sq);
  const double total = ol != 0 ? ox : 0.0, contact = ol != 0 ? sq : 0.0;  // 0.0 + x == x (x >= 0)
  const double rate_b = -P.mu_n * (P.w * total + P.half_a2 * lap_t + P.e * contact) +
                        P.m_mu_n * (P.w * phib + P.half_a2 * lap_b);
  if ((c_on && !isfinite(rate_c)) || (bnear && !isfinite(rate_b))) {
    if (lane == 0) raise_error(W.ctl, kDevBlowup, v, spec);
    return h;
  }
  const double next_c = clamp01(phi + P.dt * rate_c), next_b = clamp01(phib + P.dt * rate_b);
  const bool cupd = c_on && next_c != phi, bupd = bnear && next_b != phib;
  const bool touched = cupd || bupd;
  INSTR_AT(13, static_cast<unsigned>(__double_as_longlong(next_b)) ^ static_cast<unsigned>(__double_as_longlong(next_c)));
  // set_value (layer_field.hpp:102) on the base entry and the L entry
  // (values are already at most 1; prune below the epsilon; a stored value
  // that moves, an insertion or a removal is a change), then the column
  // [base][, L] sorted by layer.
  bool changed = false;
  const bool b_in = cv > 0 && o0 == 0, l_in = ol != 0;
  double nb = phib, nlv = l_in ? ox : 0.0;
  if (bupd) {
    const double val = next_b < P.prune ? 0.0 : next_b;
    changed |= b_in ? val != phib : val != 0.0;
    nb = val;
  }
  if (cupd) {
    const double val = next_c < P.prune ? 0.0 : next_c;
    changed |= l_in ? val != ox : val != 0.0;
    nlv = val;
  }
  unsigned El[2] = {0, 0};
  double Ex[2] = {0.0, 0.0};
  int n = 0;
  if (nb != 0.0) {
    Ex[0] = nb;
    n = 1;
  }
  if (nlv != 0.0) {
    if (n == 0) {
      El[0] = L;
      Ex[0] = nlv;
    } else {
      El[1] = L;
      Ex[1] = nlv;
    }
    ++n;
  }
  INSTR_AT(14, static_cast<unsigned>(__double_as_longlong(Ex[0])));
  // Column normalisation of touched vertices (layer_field.hpp:143), written
  // out for n <= 2 so the column stays in registers (the loop's sums and
  // divisions, term for term; both divisions issue together).
  if (touched) {
    double ssum = 0.0;
    if (n > 0) ssum = ssum + Ex[0];
    if (n > 1) ssum = ssum + Ex[1];
    if (ssum <= 0.0) {
      if (lane == 0) raise_error(W.ctl, kDevZeroColumn, v, spec);
      return h;
    }
    if (!(fabs(ssum - 1.0) < 1e-15)) {
      double q0 = Ex[0] / ssum, q1 = Ex[1] / ssum;
      if (q0 > 1.0) q0 = 1.0;
      if (q0 < P.prune) q0 = 0.0;
      if (q1 > 1.0) q1 = 1.0;
      if (q1 < P.prune) q1 = 0.0;
      if (n > 0 && q0 != Ex[0]) changed = true;
      if (n > 1 && q1 != Ex[1]) changed = true;
      const unsigned l0 = El[0], l1 = El[1];
      int m = 0;
      if (n > 0 && q0 != 0.0) {
        El[0] = l0;
        Ex[0] = q0;
        m = 1;
      }
      if (n > 1 && q1 != 0.0) {
        if (m == 0) {
          El[0] = l1;
          Ex[0] = q1;
        } else {
          El[1] = l1;
          Ex[1] = q1;
        }
        ++m;
      }
      n = m;
    }
  }
  INSTR_AT(15, static_cast<unsigned>(n));
  const bool old_one = cv > 0 && o0 == 0 && own_x.x == 1.0;
  const bool new_one = n > 0 && El[0] == 0 && Ex[0] == 1.0;
  const size_t o = static_cast<size_t>(v) * kSlots;
  if (lane < n) {
    Fo.lay[o + lane] = static_cast<unsigned short>(lane == 0 ? El[0] : El[1]);
    Fo.val[o + lane] = lane == 0 ? Ex[0] : Ex[1];
  }
  if (lane == 0) {
    // Header of a column of at most [base, L]: one band entry at most.
    const bool in0 = n > 0 && Ex[0] > 0.0 && Ex[0] < 1.0, in1 = n > 1 && Ex[1] > 0.0 && Ex[1] < 1.0;
    const bool inter = in0 || in1;
    const int bj = (n > 0 && El[0] != 0 && Ex[0] > W.band_lo && Ex[0] < W.sat)
                       ? 0
                       : ((n > 1 && El[1] != 0 && Ex[1] > W.band_lo && Ex[1] < W.sat) ? 1 : -1);
    uint4 bi = make_uint4(0, 0, 0, 0);
    if (inter && bj >= 0) {
      bi.x = bj == 0 ? El[0] : El[1];
      bi.z = static_cast<unsigned>(bj);
    }
    Fo.binfo[v] = bi;
    Fo.cnt[v] = static_cast<unsigned char>(n);
    Fo.interest[v] = inter ? 1 : 0;
    h.bi = bi;
    h.flag = kHandled | 0x80u | (changed ? 1u : 0u) | (old_one ? 2u : 0u) | (new_one ? 4u : 0u) | (inter ? 8u : 0u);
  }
  return h;
}

__device__ Hdr update_vertex_fast(const DevMesh& M, const FieldBuf& F, const FieldBuf& Fo, const DevWork& W,
                                  const StepParams& P, int v, bool spec, int lane, unsigned gm) {
  Hdr h;
  h.flag = 0;
  h.bi = make_uint4(0, 0, 0, 0);
  INSTR_AT(24, v);
  INSTR_C0(tA);
  // Every load below is independent of the counts it is masked with, so the
  // column, stiffness row and neighbour columns arrive in three dependent
  // rounds (columns hold kSlots entries; slots past the count are ignored).
  const int cv = F.cnt[v];
  const size_t vb = static_cast<size_t>(v) * kSlots;
  int Ol[kF];
  double Ox[kF];
  static_assert(kF == 4, "the column head is loaded as one 8 B and two 16 B vectors");
  {
    const uint2 lw = *reinterpret_cast<const uint2*>(F.lay + vb);
    const double2 x01 = *reinterpret_cast<const double2*>(F.val + vb);
    const double2 x23 = *reinterpret_cast<const double2*>(F.val + vb + 2);
    Ol[0] = static_cast<int>(lw.x & 0xFFFF);
    Ol[1] = static_cast<int>(lw.x >> 16);
    Ol[2] = static_cast<int>(lw.y & 0xFFFF);
    Ol[3] = static_cast<int>(lw.y >> 16);
    Ox[0] = x01.x;
    Ox[1] = x01.y;
    Ox[2] = x23.x;
    Ox[3] = x23.y;
  }
  const int k0 = __ldg(M.s_off + v), k1 = __ldg(M.s_off + v + 1);
  const double mass = __ldg(M.mass + v);
  if (cv > kF) return h;
#pragma unroll
  for (int q = 0; q < kF; ++q)
    if (q >= cv) {
      Ol[q] = kNoLayer;
      Ox[q] = 0.0;
    }
  const double phib = (cv > 0 && Ol[0] == 0) ? Ox[0] : 0.0;

  int Cl[kF];
  double Ca[kF];
#pragma unroll
  for (int c = 0; c < kF; ++c) {
    Cl[c] = kNoLayer;
    Ca[c] = 0.0;
  }
  int nc = 0;
  bool over = false;
  double lapb = 0.0, lapt = 0.0;
  bool bnear = phib > 0.0;
  const bool folded =
      k1 - k0 <= kG && gather_fold(M, F, W, v, cv, Ol, k0, k1, lane, gm, Cl, Ca, nc, lapb, lapt, bnear);
  if (!folded) {
  for (int kb = k0; kb < k1; kb += kG) {
    const int k = kb + lane;
    const bool valid = k < k1;
    int u = 0, cu = 0;
    double s = 0.0, bu = 0.0, au = 0.0;
    unsigned short L[kReg];
    double X[kReg];
#pragma unroll
    for (int q = 0; q < kReg; ++q) {
      L[q] = 0;
      X[q] = 0.0;
    }
    unsigned amask = 0;  // bit q: neighbour slot q < cu holds an active layer
    if (valid) {
      u = __ldg(M.s_col + k);
      s = __ldg(M.s_val + k);
      const size_t b = static_cast<size_t>(u) * kSlots;
      cu = F.cnt[u];
#pragma unroll
      for (int q = 0; q < kReg; ++q) {
        L[q] = F.lay[b + q];
        X[q] = F.val[b + q];
      }
#pragma unroll
      for (int q = 0; q < kReg; ++q)
        if (q < cu) {
          if (L[q] == 0) {
            bu = X[q];
          } else if (is_active(L[q])) {
            au = au + X[q];
            amask |= 1u << q;
          }
        }
      for (int q = kReg; q < cu; ++q) {
        const int l = F.lay[b + q];
        const double x = F.val[b + q];
        if (l == 0) bu = x;
        else if (is_active(l)) au = au + x;
      }
    }
    // Fold the group's neighbours in ascending column order (the reference's
    // summation order).  Unrolled with group-uniform predicates so the
    // shuffles issue ahead of the dependent additions.
    const int nvalid = min(kG, k1 - kb);
    const unsigned l01 = static_cast<unsigned>(L[0]) | (static_cast<unsigned>(L[1]) << 16);
    const unsigned l23 = static_cast<unsigned>(L[2]) | (static_cast<unsigned>(L[3]) << 16);
    const unsigned meta = static_cast<unsigned>(cu) | (amask << 8);
#pragma unroll
    for (int jj = 0; jj < kG; ++jj) {
      if (jj >= nvalid) break;
      const double s_ = __shfl_sync(__activemask(), s, jj, kG);
      const unsigned meta_ = __shfl_sync(__activemask(), meta, jj, kG);
      const double bu_ = __shfl_sync(__activemask(), bu, jj, kG);
      const double au_ = __shfl_sync(__activemask(), au, jj, kG);
      const unsigned l01_ = __shfl_sync(__activemask(), l01, jj, kG);
      const unsigned l23_ = __shfl_sync(__activemask(), l23, jj, kG);
      double x_[kReg];
#pragma unroll
      for (int q = 0; q < kReg; ++q) x_[q] = __shfl_sync(__activemask(), X[q], jj, kG);
      const int cu_ = static_cast<int>(meta_ & 0xFF);
      const unsigned am_ = meta_ >> 8;
      lapb = lapb + s_ * bu_;
      lapt = lapt + s_ * au_;
      if (bu_ > 0.0) bnear = true;
      const int lq[kReg] = {static_cast<int>(l01_ & 0xFFFF), static_cast<int>(l01_ >> 16),
                            static_cast<int>(l23_ & 0xFFFF), static_cast<int>(l23_ >> 16)};
#pragma unroll
      for (int q = 0; q < kReg; ++q)
        if ((am_ >> q) & 1) cand_add_reg(Cl, Ca, nc, over, lq[q], s_ * x_[q]);
      if (cu_ > kReg) {
        const int u_ = __shfl_sync(__activemask(), u, jj, kG);
        const size_t b = static_cast<size_t>(u_) * kSlots;
        for (int q = kReg; q < cu_; ++q) {
          const int l_ = F.lay[b + q];
          if (l_ != 0 && is_active(l_)) cand_add_reg(Cl, Ca, nc, over, l_, s_ * F.val[b + q]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kF; ++q)  // own layers (missing diagonal; never on valid meshes)
    if (q < cv && Ol[q] != 0 && is_active(Ol[q])) {
      bool found = false;
#pragma unroll
      for (int c = 0; c < kF; ++c) found |= (c < nc && Cl[c] == Ol[q]);
      if (!found) cand_add_reg(Cl, Ca, nc, over, Ol[q], 0.0);
    }
  }  // generic gather
  if (over) return h;

  const double lap_b = lapb / mass;
  // Candidate updates run one per lane (lanes 0..nc-1) and the base update on
  // lane kF, so the divisions and square roots of different layers proceed in
  // parallel instead of as one predicated chain.  Every expression is the
  // sequential code's, term for term.
  bool my_upd = false, my_blow = false;
  double my_next = 0.0;
  if (lane < nc) {
    int cl = 0;
    double ca = 0.0;
#pragma unroll
    for (int c = 0; c < kF; ++c)
      if (c == lane) {
        cl = Cl[c];
        ca = Ca[c];
      }
    double phi = 0.0;
#pragma unroll
    for (int q = 0; q < kF; ++q)
      if (Ol[q] == cl) phi = Ox[q];
    if (!(phi == 0.0 && phib <= P.prune)) {
      const double lap_i = ca / mass;
      const double inner = P.w * (phib - phi) + P.half_a2 * (lap_b - lap_i) - P.e * sqrt(max0(phi * phib));
      const double rate = -P.mu_n * inner;
      if (!isfinite(rate)) {
        my_blow = true;
      } else {
        const double next = clamp01(phi + P.dt * rate);
        if (next != phi) {
          my_upd = true;
          my_next = next;
        }
      }
    }
  }
  // Contact terms of the base update, one own slot per lane kF..kF+3.
  unsigned amask_own = 0;
#pragma unroll
  for (int q = 0; q < kF; ++q)
    if (q < cv && Ol[q] != 0 && is_active(Ol[q])) amask_own |= 1u << q;
  double cterm = 0.0;
  if (bnear && lane >= kF) {
#pragma unroll
    for (int q = 0; q < kF; ++q)
      if (lane - kF == q && ((amask_own >> q) & 1)) cterm = sqrt(max0(phib * Ox[q]));
  }
  double contact = 0.0;
#pragma unroll
  for (int q = 0; q < kF; ++q) {
    const double t = __shfl_sync(__activemask(), cterm, kF + q, kG);
    if ((amask_own >> q) & 1) contact = contact + t;
  }
  if (bnear && lane == kF) {
    double total = 0.0;
#pragma unroll
    for (int q = 0; q < kF; ++q)
      if ((amask_own >> q) & 1) total = total + Ox[q];
    const double lap_total = lapt / mass;
    const double rate = -P.mu_n * (P.w * total + P.half_a2 * lap_total + P.e * contact) +
                        P.m_mu_n * (P.w * phib + P.half_a2 * lap_b);
    if (!isfinite(rate)) {
      my_blow = true;
    } else {
      const double next = clamp01(phib + P.dt * rate);
      if (next != phib) {
        my_upd = true;
        my_next = next;
      }
    }
  }
  if (seg_any8(my_blow)) {  // every path raises the same error for v
    if (lane == 0) raise_error(W.ctl, kDevBlowup, v, spec);
    h.flag = kHandled;
    return h;
  }
  bool Cupd[kF];
  double Cn[kF];
#pragma unroll
  for (int c = 0; c < kF; ++c) {
    Cupd[c] = __shfl_sync(__activemask(), my_upd, c, kG);
    Cn[c] = __shfl_sync(__activemask(), my_next, c, kG);
  }
  const bool bupd = __shfl_sync(__activemask(), my_upd, kF, kG);
  const double bnext = __shfl_sync(__activemask(), my_next, kF, kG);
  bool touched = bupd;
#pragma unroll
  for (int c = 0; c < kF; ++c) touched |= Cupd[c];
  // Apply the updates with set_value semantics into a sorted register column.
  bool changed = false;
  int El[kN];
  double Ex[kN];
#pragma unroll
  for (int j = 0; j < kN; ++j) {
    El[j] = kNoLayer;
    Ex[j] = 0.0;
  }
  int n = 0;
#pragma unroll
  for (int q = 0; q < kF; ++q) {
    if (q >= cv) continue;
    double val = Ox[q];
    bool upd = false;
    if (Ol[q] == 0) {
      if (bupd) {
        val = bnext;
        upd = true;
      }
    } else {
#pragma unroll
      for (int c = 0; c < kF; ++c)
        if (Cupd[c] && Cl[c] == Ol[q]) {
          val = Cn[c];
          upd = true;
        }
    }
    if (upd) {
      if (val > 1.0) val = 1.0;
      if (val < P.prune) val = 0.0;
      if (val != Ox[q]) changed = true;
    }
    if (val != 0.0) {
#pragma unroll
      for (int j = 0; j < kN; ++j)
        if (j == n) {
          El[j] = Ol[q];
          Ex[j] = val;
        }
      ++n;
    }
  }
  if (bupd && phib == 0.0) {  // base enters the column
    double val = bnext;
    if (val > 1.0) val = 1.0;
    if (val < P.prune) val = 0.0;
    if (val != 0.0) {
      reg_insert(El, Ex, n, 0, val);
      changed = true;
    }
  }
#pragma unroll
  for (int c = 0; c < kF; ++c) {
    if (!Cupd[c]) continue;
    bool present = false;
#pragma unroll
    for (int q = 0; q < kF; ++q) present |= (Ol[q] == Cl[c]);
    if (present) continue;
    double val = Cn[c];
    if (val > 1.0) val = 1.0;
    if (val < P.prune) val = 0.0;
    if (val != 0.0) {
      reg_insert(El, Ex, n, Cl[c], val);
      changed = true;
    }
  }
  // Column normalisation of touched vertices (layer_field.hpp:143).
  if (touched) {
    double ssum = 0.0;
#pragma unroll
    for (int j = 0; j < kN; ++j)
      if (j < n) ssum = ssum + Ex[j];
    if (ssum <= 0.0) {
      raise_error(W.ctl, kDevZeroColumn, v, spec);
      h.flag = kHandled;
      return h;
    }
    if (!(fabs(ssum - 1.0) < 1e-15)) {
      // One entry per lane (n <= kN == kG): divide, clamp, prune, then drop
      // zeros by ballot compaction -- the sequential loop's result.
      static_assert(kN == kG, "normalisation maps one column entry to each lane");
      int el = kNoLayer;
      double ex = 0.0;
#pragma unroll
      for (int j = 0; j < kN; ++j)
        if (j == lane) {
          el = El[j];
          ex = Ex[j];
        }
      double q = 0.0;
      bool ch = false;
      if (lane < n) {
        q = ex / ssum;
        if (q > 1.0) q = 1.0;
        if (q < P.prune) q = 0.0;
        ch = q != ex;
      }
      const int gshift = threadIdx.x & 24;
      const unsigned keep = (__ballot_sync(__activemask(), lane < n && q != 0.0) >> gshift) & 0xFFu;
      changed = changed || ((__ballot_sync(__activemask(), ch) >> gshift) & 0xFFu) != 0;
      // Lane t takes the t-th surviving entry.
      const int src = __fns(keep, 0, lane + 1);
      const int srcl = src < 0 ? 0 : src & (kG - 1);
      const int nl = __shfl_sync(__activemask(), el, srcl, kG);
      const double nx = __shfl_sync(__activemask(), q, srcl, kG);
#pragma unroll
      for (int j = 0; j < kN; ++j) {
        El[j] = __shfl_sync(__activemask(), nl, j, kG);
        Ex[j] = __shfl_sync(__activemask(), nx, j, kG);
      }
      n = __popc(keep);
#pragma unroll
      for (int j = 0; j < kN; ++j)
        if (j >= n) {
          El[j] = kNoLayer;
          Ex[j] = 0.0;
        }
    }
  }
  const bool old_one = cv > 0 && Ol[0] == 0 && Ox[0] == 1.0;
  const bool new_one = n > 0 && El[0] == 0 && Ex[0] == 1.0;
  const size_t o = static_cast<size_t>(v) * kSlots;
#pragma unroll
  for (int j = 0; j < kN; ++j)
    if (j == lane && j < n) {
      Fo.lay[o + j] = static_cast<unsigned short>(El[j]);
      Fo.val[o + j] = Ex[j];
    }
  h.flag = kHandled;
  if (lane == 0) column_header<kN>(Fo, W, v, n, El, Ex, changed, old_one, new_one, h);
  INSTR_AT(25, n);
  return h;
}

// Warp-aggregated slot reservation: one atomic per warp and round instead of
// one per appended item (frontier and band lists see thousands per step).
__device__ __forceinline__ int agg_slot(int* counter, bool want) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, want);
  if (!m) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(act, base, leader);
  return want ? base + __popc(m & ((1u << lane) - 1)) : -1;
}

// Per-CTA staging of list appends: items collect in shared memory and the CTA
// reserves its global range with one atomic at the end of the phase (the
// frontier, band-list compaction and band items each see thousands of
// appends per step; one global counter would serialise them).
constexpr int kQCap = 2048;
template <class T>
struct BlockQueueT {
  int n, base;
  T buf[kQCap];
};
using BlockQueue = BlockQueueT<int>;

template <class T>
__device__ __forceinline__ void bq_push(BlockQueueT<T>& q, int* gcount, T* glist, T item, int cap = 0x7fffffff,
                                        int* overflow = nullptr) {
  const int p = atomicAdd(&q.n, 1);
  if (p < kQCap) {
    q.buf[p] = item;
  } else {  // staging full: direct append
    const int g = atomicAdd(gcount, 1);
    if (g < cap) glist[g] = item;
    else if (overflow) *overflow = 1;
  }
}

// Flushes the CTA's staged appends.  Threads [t0, t0 + nthreads) take part:
// the whole CTA (bar 0 = __syncthreads) or the warps of one role behind a
// named barrier, so the other roles of the phase never wait for it.  The next
// use of the queue is after a grid barrier, so no trailing barrier is needed.
// Non-aligned form: the threads of a warp may arrive at different times
// (bar.sync is barrier.sync.aligned, which requires converged warps).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
template <class T>
__device__ void bq_flush(BlockQueueT<T>& q, int* gcount, T* glist, int bar = 0, int t0 = 0, int nthreads = 0) {
  if (bar == 0) __syncthreads();
  else named_sync(bar, nthreads);
  const int n = min(q.n, kQCap);
  const int r = static_cast<int>(threadIdx.x) - t0;
  if (r == 0) q.base = n ? atomicAdd(gcount, n) : 0;
  if (bar == 0) __syncthreads();
  else named_sync(bar, nthreads);
  const int stride = bar == 0 ? static_cast<int>(blockDim.x) : nthreads;
  const int rr = bar == 0 ? static_cast<int>(threadIdx.x) : r;
  for (int i = rr; i < n; i += stride) glist[q.base + i] = q.buf[i];
  if (bar == 0) __syncthreads();
  else named_sync(bar, nthreads);
  if (r == 0 || (bar == 0 && threadIdx.x == 0)) q.n = 0;
}

__device__ __forceinline__ void queue_region(const DevWork& W, int u, int stamp, int slot, BlockQueue& Q) {
  if (atomicExch(W.stamp + u, stamp) != stamp) bq_push(Q, &W.ctl->rcount[slot], pick4(W.region, slot), u);
}

// What phase B (commit) did before the field was double-buffered, now run by
// the updating group right after its update of v at step t (reference:
// diffusion.hpp:253-271 change log -> next frontier): queue the one-ring of a
// changed column as frontier t+1, list a column that became interesting in
// the band list E(t) reads, record band-item changes for the split
// certificate, and carry the base==1 count.  The column itself was written to
// the step's buffer by the update.  old_bi / old_inter describe v's column
// before the step; rlen / ue are v's padded stiffness row (lane j: entry j-1).
__device__ void post_update(const DevMesh& M, const DevWork& W, int v, int t, const Hdr& h0, uint4 old_bi,
                            bool old_inter, int rlen, int ue, int lane, BlockQueue& Q) {
  const unsigned flag = __shfl_sync(__activemask(), h0.flag, 0, kG);  // whole groups, see seg_any8
  if (!(flag & 0x80u)) return;  // the update raised an error: the step is void
  const int nslot = slot4(t + 1), cp = slot4(t);
  const bool changed = (flag & 1u) != 0;
  // Lane 0's bookkeeping (band-item changes for the split certificate, see
  // anchor_test: a lost band layer -- or an overflowing band index -- marks
  // the step, gained layers are listed; a column that became interesting
  // joins the band list E(t) reads; the base==1 count) issues its atomics in
  // the same round as the one-ring claims below, so the two round trips
  // overlap.  An unchanged column has the same band index.
  unsigned gained[4] = {0, 0, 0, 0};
  int ngain = 0;
  bool lost = false;     // a lost band item the certificate does not test: the union-find runs
  unsigned rem_l = 0;    // the band layer a single-front column lost (tested by the certificate)
  const bool want_il = lane == 0 && (flag & 8u) && !old_inter;
  if (lane == 0 && changed) {
    const uint4 bi = h0.bi;
    if (old_bi.y == 0 && bi.y == 0 && (old_bi.x >> 16) == 0 && (bi.x >> 16) == 0) {
      // At most one band layer before and after (a single front): compare the two.
      const unsigned lo = old_bi.x, ln = bi.x;
      if (lo != 0 && lo != ln) rem_l = lo;
      if (ln != 0 && ln != lo) {
        gained[0] = ln;
        ngain = 1;
      }
    } else if (binfo_overflow(old_bi) || binfo_overflow(bi)) {
      lost = true;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned lo = binfo_layer(old_bi, q), ln = binfo_layer(bi, q);
        bool lo_kept = false, ln_old = false;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          lo_kept |= lo != 0 && binfo_layer(bi, r) == lo;
          ln_old |= ln != 0 && binfo_layer(old_bi, r) == ln;
        }
        lost |= lo != 0 && !lo_kept;
        if (ln != 0 && !ln_old) {
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (r == ngain) gained[r] = ln;
          ++ngain;
        }
      }
    }
  }
  const int nitems = ngain + (rem_l != 0);
  int add_pos = 0, il_pos = 0;
  if (nitems) add_pos = atomicAdd(&W.ctl->nadded[cp], nitems);
  if (want_il) il_pos = atomicAdd(&W.ctl->ilcount[cp], 1);
  bool first = false;
  if (changed) {
    // Claim the one-ring for frontier t+1 (lane 0: v itself, lane j: entry j-1).
    const int u0 = lane == 0 ? v : (lane <= rlen ? ue : -1);
    first = u0 >= 0 && atomicExch(W.stamp + u0, t) != t;
  }
  if (lane == 0) {
    if (lost) W.ctl->dchange[cp] = 1;
    if (nitems) {
      if (ngain) W.add_stamp[v] = t;
      if (rem_l) W.rem_stamp[v] = t;
      int2* items = W.added + static_cast<size_t>(cp) * W.added_cap;
#pragma unroll
      for (int r = 0; r < 5; ++r)
        if (r < nitems) {
          const int x = r < ngain ? static_cast<int>(gained[r & 3]) : static_cast<int>(rem_l) | kRemovedItem;
          if (add_pos + r < W.added_cap)
            items[add_pos + r] = make_int2(v, x);
          else
            W.ctl->dchange[cp] = 1;
        }
    }
    if (want_il) pick4(W.ilist, cp)[il_pos] = v;
    const int delta = static_cast<int>((flag >> 2) & 1u) - static_cast<int>((flag >> 1) & 1u);
    if (delta) atomicAdd(&W.ctl->base_d[cp], delta);
  }
  INSTR_AT(5, first);
  if (changed) {
    if (first) bq_push(Q, &W.ctl->rcount[nslot], pick4(W.region, nslot), lane == 0 ? v : ue);
    for (int k = lane + kG; k <= rlen; k += kG)  // entries past the group: padded row, then the CSR
      queue_region(W, k - 1 < kEll ? __ldg(M.e_col + static_cast<size_t>(v) * kEll + k - 1)
                                   : __ldg(M.s_col + __ldg(M.s_off + v) + k - 1),
                   t, nslot, Q);
  }
}

// Update of frontier entry i of step t (reading the field after t-1, writing
// the field after t) and its bookkeeping, by one 8-lane group (act false:
// no item, no side effects).
__device__ __forceinline__ void update_item(const DevMesh& M, const FieldBuf& Fi, const FieldBuf& Fo, const int* list,
                                            const DevWork& W, const StepParams& P, int t, int i, bool act, bool spec,
                                            BlockQueue& Q) {
  const int lane = threadIdx.x & (kG - 1);
  INSTR_AT(0, i);
  const int v = act ? list[i] : 0;
  INSTR_AT(1, v);
  // Loads of the bookkeeping that depend only on v, issued with the update's.
  const uint4 old_bi = Fi.binfo[v];
  const bool old_inter = Fi.interest[v] != 0;
  const int rlen = __ldg(M.e_len + v);
  const int ue = lane >= 1 ? __ldg(M.e_col + static_cast<size_t>(v) * kEll + lane - 1) : v;
  Hdr h = update_vertex_single(M, Fi, Fo, W, P, v, act, spec, lane);
#ifdef DTB_INSTR
  if (lane == 0) atomicAdd(&s_hist[3][(h.flag & kHandled) ? 0 : 1], 1u);  // single / not
#endif
  if (act && !(h.flag & kHandled)) {
    // Neighbour columns longer than kReg mostly mean more than kF candidate
    // layers, where the fast path would gather everything and then give up.
    if (h.bi.x <= static_cast<unsigned>(kReg) || P.no_wide) h = update_vertex_fast(M, Fi, Fo, W, P, v, spec, lane, group_mask());
#ifdef DTB_INSTR
    if (lane == 0) atomicAdd(&s_hist[3][(h.flag & kHandled) ? 2 : 3], 1u);  // fast / general
#endif
    if (!(h.flag & kHandled) && !P.no_wide) h = update_vertex_wide(M, Fi, Fo, W, P, v, spec, lane);
    if (!(h.flag & kHandled)) h = update_vertex(M, Fi, Fo, W, P, v, spec, lane, group_mask());
    __syncwarp(group_mask());  // the wide and general paths end on lane 0 alone: regroup
  }
  INSTR_AT(4, h.flag);
  post_update(M, W, v, t, h, old_bi, old_inter && act, rlen, ue, lane, Q);
  INSTR_AT(6, v);
}

// Updates of step t for the items rank0, rank0 + stride, ... < n of this group.
__device__ __forceinline__ void update_items(const DevMesh& M, const DevField& F, const DevWork& W, const StepParams& P,
                                             int t, int n, int rank0, int stride, bool spec, BlockQueue& Q) {
  const FieldBuf Fi = pickf(F, t - 1), Fo = pickf(F, t);  // the field after t-1 and after t
  const int* list = pick4(W.region, slot4(t));
  for (int i = rank0; i < n; i += stride) update_item(M, Fi, Fo, list, W, P, t, i, true, spec, Q);
}

__device__ __forceinline__ bool is_band(const DevWork& W, const StepParams& P, int l, double x) {
  return l != 0 && is_active(l) && x > P.band_lo && x < P.sat;
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

// Parent words are read with plain (L1-cacheable) loads: a CTA's items share
// hot roots, and measured alternatives that read through L2 (__ldcg) or
// switch to L2 reads after a lost CAS are 1.7x slower on this phase.  A
// stale L1 line can only make a non-root look like a root; the CAS against
// it then fails, the atomic evicts the line from this SM's L1, and the
// retry reads the current word.
//
// Randomised linking: the root with the smaller (hash, id) key is hooked
// under the other.  Linking by plain id turns concurrently united bands (ring
// paths with increasing ids) into pointer chains as long as the ring; random
// keys bound the expected depth by O(log n).
__device__ __forceinline__ unsigned long long uf_key(unsigned x) {
  unsigned h = x * 0x9E3779B1u;
  h ^= h >> 15;
  h *= 0x85EBCA77u;
  h ^= h >> 13;
  return (static_cast<unsigned long long>(h) << 32) | x;
}

__device__ void uf_unite(unsigned long long* par, unsigned a, unsigned b, unsigned long long ep) {
  const unsigned a0 = a, b0 = b;
  while (true) {
    a = uf_find(par, a, ep);
    b = uf_find(par, b, ep);
    if (a == b) {
      // Shortcut both starting items to the common root: later finds from
      // them (each item takes part in ~6 unions per step) are one hop.
      const unsigned long long r = (ep << 32) | a;
      if (a0 != a) par[a0] = r;
      if (b0 != a) par[b0] = r;
      return;
    }
    if (uf_key(a) > uf_key(b)) {
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

__device__ void insert_pair(const DevWork& W, unsigned key, unsigned long long ep, int cs) {
  const unsigned long long tagged = (ep << 32) | key;
  unsigned h = (key * 2654435761u) & (kPairCap - 1);
  for (int probe = 0; probe < kPairCap; ++probe) {
    unsigned long long cur = W.pair_keys[h];
    if (cur == tagged) return;
    if ((cur >> 32) != ep) {
      const unsigned long long prev = atomicCAS(W.pair_keys + h, cur, tagged);
      if (prev == cur) {
        const int pos = atomicAdd(&W.ctl->npairs[cs], 1);
        if (pos < kPairCap) W.pairs[static_cast<size_t>(cs) * kPairCap + pos] = key;
        else W.ctl->pair_overflow[cs] = 1;
        return;
      }
      if (prev == tagged) return;
      continue;  // lost the race for this slot; re-inspect it
    }
    h = (h + 1) & (kPairCap - 1);
  }
  W.ctl->pair_overflow[cs] = 1;
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

// Dense field digest (parity tooling only).
__device__ void phase_hash(const FieldBuf& F, unsigned long long* acc, int nv) {
  unsigned long long h = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv + 31; v += gridDim.x * blockDim.x) {
    if (v < nv) {
      const int c = F.cnt[v];
      for (int j = 0; j < c; ++j)
        h += entry_hash(F.lay[static_cast<size_t>(v) * kSlots + j], static_cast<unsigned long long>(v),
                        F.val[static_cast<size_t>(v) * kSlots + j]);
    }
  }
  h = warp_sum_u64(h);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(acc, h);
}

// Phase D: union band items that share a band triangle pair (extract_front's
// edge-adjacency of band triangles, expressed on band vertices).  An 8-lane
// group per list entry; lane j probes the higher-numbered related vertices
// j, j+8, ... through their band index (one 16-byte load per probe).
__device__ __forceinline__ int band_slot_of(const FieldBuf& F, const DevWork& W, const StepParams& P, int u,
                                            unsigned l) {
  const uint4 bu = F.binfo[u];
  if (!binfo_overflow(bu)) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (binfo_layer(bu, t) == l) return static_cast<int>(binfo_slot(bu, t));
    return -1;
  }
  const int cu = F.cnt[u];  // more than 4 band layers: scan the column
  const size_t ub = static_cast<size_t>(u) * kSlots;
  for (int j = 0; j < cu; ++j) {
    const unsigned lu = F.lay[ub + j];
    if (lu < l) continue;
    return (lu == l && is_band(W, P, static_cast<int>(l), F.val[ub + j])) ? j : -1;
  }
  return -1;
}

__device__ void phase_union(const DevMesh& M, const FieldBuf& F, const DevWork& W, const StepParams& P, int lslot,
                            unsigned long long ep, int g0, int ng, int n) {
  const int* list = pick4(W.ilist, lslot);
  const int lane = threadIdx.x & (kG - 1);
  const bool trace = W.prof && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long* tr = trace ? W.prof + (W.prof_cap - 64LL * 3 * gridDim.x - 16) : nullptr;
  if (trace) tr[0] = gtimer_raw();
  for (int idx = g0; idx < n; idx += ng) {
    INSTR_T0(t0);
    const int v = list[idx];
    if (!F.interest[v]) continue;
    const uint4 bv = F.binfo[v];
    if (trace) tr[1] = gtimer_raw() + (bv.x & 0);
    const int c0 = __ldg(M.c_off + v), c1 = __ldg(M.c_off + v + 1);
    const bool over = binfo_overflow(bv);
    const int nitems = over ? F.cnt[v] : 4;
    for (int t = 0; t < nitems; ++t) {
      unsigned l;
      int slot;
      if (!over) {
        l = binfo_layer(bv, t);
        if (l == 0) break;
        slot = static_cast<int>(binfo_slot(bv, t));
      } else {
        l = F.lay[static_cast<size_t>(v) * kSlots + t];
        if (!is_band(W, P, static_cast<int>(l), F.val[static_cast<size_t>(v) * kSlots + t])) continue;
        slot = t;
      }
      if (!is_active(l)) continue;
      const unsigned item = static_cast<unsigned>(v) * kSlots + slot;
      if (trace) tr[2] = gtimer_raw();
      for (int c = c0 + lane; c < c1; c += kG) {
        const int u = __ldg(M.c_col + c);  // higher-numbered related vertices only
        const int j = band_slot_of(F, W, P, u, l);
        if (trace) tr[3] = gtimer_raw() + (j & 0);
        if (j >= 0) uf_unite(W.parent, item, static_cast<unsigned>(u) * kSlots + j, ep);
        if (trace) tr[4] = gtimer_raw();
      }
    }
    INSTR_REC(1, t0, lane == 0);
  }
}

constexpr int kSmemLayers = 64;  // per-block aggregation slots for dense active indices
struct BlockStats {
  int cnt[kSmemLayers][3];  // ncomp, nband, nunsat
  long long sum[kSmemLayers][3];
  unsigned long long bmax;               // max base value in (0, 1), as ordered bits
  unsigned long long wbmax[kBlock / 32];  // per-warp maxima (each warp's leader owns its slot: no atomics)
  int nbp;                                // band items appended to this CTA's segment
};

__device__ void block_stats_init(BlockStats& S) {
  for (int i = threadIdx.x; i < kSmemLayers; i += blockDim.x) {
    S.cnt[i][0] = S.cnt[i][1] = S.cnt[i][2] = 0;
    S.sum[i][0] = S.sum[i][1] = S.sum[i][2] = 0;
  }
  if (threadIdx.x == 0) {
    S.bmax = 0;
    S.nbp = 0;
  }
  if (threadIdx.x < kBlock / 32) S.wbmax[threadIdx.x] = 0;
  __syncthreads();
}
__device__ __forceinline__ unsigned long long block_bmax(const BlockStats& S) {
  unsigned long long m = S.bmax;
  for (int w = 0; w < kBlock / 32; ++w) m = S.wbmax[w] > m ? S.wbmax[w] : m;
  return m;
}

// E's CTA-level flush for check `step` by threads [t0, t0 + nthreads) behind
// barrier `bar` (0: __syncthreads for the whole CTA; else a named barrier of
// E's own warps, so the CTA's A warps never wait for it): the base maximum,
// the CTA's band-item segment length, and the per-layer sums.
__device__ void e_flush(BlockStats& S, const DevWork& W, int n_active, long long step, int bar, int t0, int nthreads) {
  if (bar == 0) __syncthreads();
  else named_sync(bar, nthreads);
  const int cs = slot4(step), set = static_cast<int>(step & 1);
  LayerStat* g = W.stat + static_cast<size_t>(cs) * kMaxActive;
  const int r = static_cast<int>(threadIdx.x) - t0;
  // Each thread clears what it flushed, so S is ready for the next check
  // (a grid barrier later) without a CTA barrier of its own.
  if (r == 0) {
    const unsigned long long m = block_bmax(S);
    if (m) atomicMax(&W.ctl->base_max_bits[cs], m);
    if (blockIdx.x < W.bp_nseg) pick2(W.bpcount, set)[blockIdx.x] = min(S.nbp, W.bp_seg);
    if (blockIdx.x == 0)  // segments of CTAs beyond the grid
      for (int c = gridDim.x; c < W.bp_nseg; ++c) pick2(W.bpcount, set)[c] = 0;
    S.bmax = 0;
    S.nbp = 0;
    for (int w = 0; w < kBlock / 32; ++w) S.wbmax[w] = 0;
  }
  for (int a = r; a < n_active && a < kSmemLayers; a += nthreads) {
    if (S.cnt[a][0]) atomicAdd(&g[a].ncomp, S.cnt[a][0]);
    if (S.cnt[a][1]) atomicAdd(&g[a].nband, S.cnt[a][1]);
    if (S.cnt[a][2]) atomicAdd(&g[a].nunsat, S.cnt[a][2]);
    for (int c = 0; c < 3; ++c)
      if (S.sum[a][c])
        atomicAdd(reinterpret_cast<unsigned long long*>(c == 0 ? &g[a].sx : (c == 1 ? &g[a].sy : &g[a].sz)),
                  static_cast<unsigned long long>(S.sum[a][c]));
    S.cnt[a][0] = S.cnt[a][1] = S.cnt[a][2] = 0;
    S.sum[a][0] = S.sum[a][1] = S.sum[a][2] = 0;
  }
}

// Segmented warp reductions: lanes holding the same key (dense active layer
// index) combine their contributions with 32-bit __reduce_*_sync, so each
// warp issues one shared-memory atomic per layer (64-bit shared atomics are
// CAS spin loops on this architecture).
// Full-warp sum of fixed-point values (every lane converged).
__device__ __forceinline__ long long warp_sum_fx(long long x) {
  // |x| < 2^39: low 24 bits and the signed rest each sum exactly in 32 bits.
  const unsigned lo = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(x & 0xFFFFFF));
  const int hi = __reduce_add_sync(0xffffffffu, static_cast<int>(x >> 24));
  return (static_cast<long long>(hi) << 24) + static_cast<long long>(lo);
}
__device__ __forceinline__ long long seg_sum_fx(unsigned peers, long long x) {
  // |x| < 2^39: low 24 bits and the signed rest each sum exactly in 32 bits.
  const unsigned lo = __reduce_add_sync(peers, static_cast<unsigned>(x & 0xFFFFFF));
  const int hi = __reduce_add_sync(peers, static_cast<int>(x >> 24));
  return (static_cast<long long>(hi) << 24) + static_cast<long long>(lo);
}
__device__ __forceinline__ unsigned long long seg_min_u64(unsigned peers, unsigned long long x) {
  const unsigned hi = __reduce_min_sync(peers, static_cast<unsigned>(x >> 32));
  const unsigned lo = __reduce_min_sync(peers, static_cast<unsigned>(x >> 32) == hi ? static_cast<unsigned>(x) : ~0u);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}
__device__ __forceinline__ unsigned long long seg_max_u64(unsigned peers, unsigned long long x) {
  const unsigned hi = __reduce_max_sync(peers, static_cast<unsigned>(x >> 32));
  const unsigned lo = __reduce_max_sync(peers, static_cast<unsigned>(x >> 32) == hi ? static_cast<unsigned>(x) : 0u);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Split certificate (phase D is skipped when it holds).  With every check at
// consecutive steps, the previous check left each layer's band connected (or
// empty): its band triangles -- the faces with a band vertex, extract_front
// (diffusion.hpp:398) -- form one edge-connected set T.  The step turns T
// into T': faces whose band vertices were all lost leave, faces of gained
// band vertices join.  T' is still connected (or empty) when
//  * every gained item v has a mesh neighbour u that is a band item of its
//    layer before and after the step: star(v) is edge-connected and shares
//    the faces on edge uv with star(u), which lies in both T and T'; and
//  * every lost item r passes the local test below.  Let Omega be star(r)
//    plus the faces across its link edges.  If no other vertex of Omega
//    lost a band item at the step, every maximal run of left faces on a
//    path in T lies in star(r) and is entered and left through faces of
//    Omega that stay in T'; so when the faces of Omega in T' are one
//    edge-connected set (using only the edges between consecutive star
//    faces and between a star face and the face across its link edge), a
//    path in T between two faces of T' reroutes inside T'.
// Then T and T' minus the left faces is connected in T', and every joined
// face is edge-connected to it.  Items of inactive layers are not tested.
// One 8-lane group per item; a failed item sets anchor_fail (the union-find
// runs after all).  add_stamp / rem_stamp may already carry the next step's
// stamp (its update runs beside this test): a stamp past `stamp` proves
// nothing, so it never anchors and always counts as a loss (conservative).
__device__ __forceinline__ int seg_sum8(int x) {
  const unsigned am = __activemask();
  x += __shfl_xor_sync(am, x, 4);
  x += __shfl_xor_sync(am, x, 2);
  return x + __shfl_xor_sync(am, x, 1);
}
__device__ bool lost_item_ok(const DevMesh& M, const FieldBuf& F, const DevWork& W, const StepParams& P, int r,
                             unsigned l, int stamp, int lane) {
  const int f0 = __ldg(M.f_off + r), d = __ldg(M.f_off + r + 1) - f0;
  if (d > kG) return false;  // group-uniform
  const bool valid = lane < d;
  int a = -1, b = -1, w = -1;
  if (valid) {
    const int f = __ldg(M.f_col + f0 + lane);
    const unsigned t0 = __ldg(M.faces + 3 * f), t1 = __ldg(M.faces + 3 * f + 1), t2 = __ldg(M.faces + 3 * f + 2);
    const int kv = t0 == static_cast<unsigned>(r) ? 0 : (t1 == static_cast<unsigned>(r) ? 1 : 2);
    a = static_cast<int>(kv == 0 ? t1 : (kv == 1 ? t2 : t0));  // corners kv+1, kv+2: the link edge
    b = static_cast<int>(kv == 0 ? t2 : (kv == 1 ? t0 : t1));
    const unsigned e = __ldg(M.face_edges + 3 * f + (kv + 1) % 3);
    const unsigned g0 = __ldg(M.edge_faces + 2 * e), g1 = __ldg(M.edge_faces + 2 * e + 1);
    const unsigned g = g0 == static_cast<unsigned>(f) ? g1 : g0;
    if (g != static_cast<unsigned>(f) && g < static_cast<unsigned>(M.nf)) {  // not a boundary edge
      const unsigned h0 = __ldg(M.faces + 3 * g), h1 = __ldg(M.faces + 3 * g + 1), h2 = __ldg(M.faces + 3 * g + 2);
      w = static_cast<int>(h0 != static_cast<unsigned>(a) && h0 != static_cast<unsigned>(b)
                               ? h0
                               : (h1 != static_cast<unsigned>(a) && h1 != static_cast<unsigned>(b) ? h1 : h2));
    }
  }
  bool bad = false, fp = false;
  if (valid) {
    const bool in_a = band_slot_of(F, W, P, a, l) >= 0, in_b = band_slot_of(F, W, P, b, l) >= 0;
    const bool in_w = w >= 0 && band_slot_of(F, W, P, w, l) >= 0;
    fp = in_a || in_b;
    bad = (in_w && !fp) ||  // the face across the link edge would hang off a left face
          W.rem_stamp[a] >= stamp || W.rem_stamp[b] >= stamp || (w >= 0 && W.rem_stamp[w] >= stamp);
  }
  // Present star faces sharing an edge r-x: counted once from each side.
  int occ_a = 0, occ_b = 0, shared = 0;
  {
    const unsigned am = __activemask();  // whole groups
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int aj = __shfl_sync(am, a, j, kG), bj = __shfl_sync(am, b, j, kG);
      const bool pj = __shfl_sync(am, fp, j, kG);
      if (j != lane && j < d) {
        const int ha = aj == a || bj == a, hb = aj == b || bj == b;
        occ_a += ha;
        occ_b += hb;
        if (pj && fp) shared += ha + hb;
      }
    }
  }
  bad |= valid && (occ_a > 1 || occ_b > 1);  // not a manifold star: no claim
  const int np = __popc((__ballot_sync(__activemask(), fp) >> (threadIdx.x & 24)) & 0xFFu);
  const int ns = seg_sum8(shared);  // twice the shared edges
  // The present star faces form np - ns/2 runs around r (a cycle or a fan).
  return !seg_any8(bad) && 2 * np - ns <= 2;
}

__device__ void anchor_test(const DevMesh& M, const FieldBuf& F, const DevWork& W, const StepParams& P, int nadded,
                            int stamp, int g0, int ng) {
  const int cp = slot4(stamp);
  const int n = min(nadded, W.added_cap);
  const int lane = threadIdx.x & (kG - 1);
  for (int i = g0; i < n; i += ng) {  // group-uniform
    const int2 a = W.added[static_cast<size_t>(cp) * W.added_cap + i];
    const int v = a.x;
    const unsigned l = static_cast<unsigned>(a.y) & 0xFFFFu;
    if (!is_active(l)) continue;
    bool ok;
    if (a.y & kRemovedItem) {
      ok = lost_item_ok(M, F, W, P, v, l, stamp, lane);
    } else {
      // u anchors v when it is a band item of l after the step and gained
      // no band item at the step.
      const int o0 = __ldg(M.n_off + v), o1 = __ldg(M.n_off + v + 1);
      bool anchored = false;
      for (int ob = o0; ob < o1; ob += kG) {  // group-uniform rounds
        const int o = ob + lane;
        if (o < o1) {
          const int u = __ldg(M.n_col + o);
          anchored |= W.add_stamp[u] < stamp && band_slot_of(F, W, P, u, l) >= 0;
        }
        if (seg_any8(anchored)) break;
      }
      ok = seg_any8(anchored);
    }
    if (!ok && lane == 0) W.ctl->anchor_fail[cp] = 1;
  }
}

// Component roots of the band items (ncomp of phase E), for a check whose
// statistics were gathered under the split certificate that then failed.
__device__ void phase_roots(const FieldBuf& F, const DevWork& W, const StepParams& P, int lslot, int sslot,
                            unsigned long long ep, int n) {
  LayerStat* g = W.stat + static_cast<size_t>(sslot) * kMaxActive;
  const int* list = pick4(W.ilist, lslot);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int v = list[idx];
    if (!F.interest[v]) continue;
    const int cv = F.cnt[v];
    const size_t b = static_cast<size_t>(v) * kSlots;
    for (int k = 0; k < cv; ++k) {
      const int l = F.lay[b + k];
      const double x = F.val[b + k];
      if (l == 0 || !is_active(l) || !(x > P.band_lo && x < P.sat)) continue;
      const unsigned item = static_cast<unsigned>(v) * kSlots + k;
      const unsigned long long pw = W.parent[item];
      if ((pw >> 32) != ep || static_cast<unsigned>(pw) == item) atomicAdd(&g[W.aidx[l]].ncomp, 1);
    }
  }
}

// Phase E: per-layer statistics (roots = front components, band counts and
// fixed-point position sums, unsaturated counts), collision pairs, base
// extinction data, band items for the trail snap, and compaction of the band
// list into the other buffer (dead entries dropped).  Lanes walk their
// vertex's slots in lock step so contributions can be combined per warp.
// Check t = `step`: reads the field after t (F), the band list of slot4(t),
// writes stats slot4(t), band items of set t & 1, pairs slot4(t); compacts
// the list's live entries into slot4(t+1).  Threads [t0, t0 + nthreads) of
// each CTA take part (rank-major over the CTAs, so a short list spreads over
// every SM).
__device__ void phase_stats(const DevMesh& M, const FieldBuf& F, const DevWork& W, const StepParams& P, long long step,
                            unsigned long long ep, bool compact, BlockStats& S, int n, bool count_roots, int t0,
                            int nthreads) {
  const int lslot = slot4(step), nslot = slot4(step + 1), cs = slot4(step), set = static_cast<int>(step & 1);
  LayerStat* g = W.stat + static_cast<size_t>(cs) * kMaxActive;
  const int* list = pick4(W.ilist, lslot);
  const int lane = threadIdx.x & 31;
  const int rank = static_cast<int>(threadIdx.x) - t0;
  const int trip = (n + gridDim.x * nthreads - 1) / (gridDim.x * nthreads);
  for (int r = 0; r < trip; ++r) {
    const int idx = (r * nthreads + rank) * gridDim.x + blockIdx.x;
    INSTR_T0(t0);
    INSTR_C0(tE);
    const int v = idx < n ? list[idx] : -1;
    // One round of loads for everything the vertex contributes: flags, the
    // first four column slots with their union-find words, the position.
    const int vs = v >= 0 ? v : 0;
    const size_t b = static_cast<size_t>(vs) * kSlots;
    const unsigned char inter_v = F.interest[vs];
    const int cnt_v = F.cnt[vs];
    const uint2 lw = *reinterpret_cast<const uint2*>(F.lay + b);
    const double2 x01 = *reinterpret_cast<const double2*>(F.val + b);
    const double2 x23 = *reinterpret_cast<const double2*>(F.val + b + 2);
    const ulonglong2 p01 = *reinterpret_cast<const ulonglong2*>(W.parent + b);
    const ulonglong2 p23 = *reinterpret_cast<const ulonglong2*>(W.parent + b + 2);
    const long long fxv = __ldg(M.fx + vs), fyv = __ldg(M.fy + vs), fzv = __ldg(M.fz + vs);
    const int L4[4] = {static_cast<int>(lw.x & 0xFFFF), static_cast<int>(lw.x >> 16), static_cast<int>(lw.y & 0xFFFF),
                       static_cast<int>(lw.y >> 16)};
    const double X4[4] = {x01.x, x01.y, x23.x, x23.y};
    const unsigned long long P4[4] = {p01.x, p01.y, p23.x, p23.y};
    const bool live = v >= 0 && inter_v;
    if (compact) {
      // Survivors go straight to the next band list, one atomic per warp
      // (the list's order does not matter), so no flush is left for the end
      // of the phase.
      const unsigned lm = __ballot_sync(0xffffffffu, live);
      if (lm) {
        const int leader = __ffs(lm) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&W.ctl->ilcount[nslot], __popc(lm));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (live) pick4(W.ilist, nslot)[base + __popc(lm & ((1u << lane) - 1u))] = v;
      }
    }
    const int cv = live ? cnt_v : 0;
    const double base = (cv > 0 && L4[0] == 0) ? X4[0] : 0.0;
    {
      const bool has = base > 0.0 && base < 1.0;
      const unsigned m = __ballot_sync(0xffffffffu, has);
      if (m) {
        const unsigned long long bm =
            seg_max_u64(0xffffffffu, has ? static_cast<unsigned long long>(__double_as_longlong(base)) : 0ull);
        if (lane == __ffs(m) - 1) {
          unsigned long long& slot = S.wbmax[threadIdx.x >> 5];
          slot = bm > slot ? bm : slot;
        }
      }
    }
    const long long px = live ? fxv : 0, py = live ? fyv : 0, pz = live ? fzv : 0;
    bool cand = false;
    int nkappa = 0;  // active layers at or above the collision threshold
    // The base owner (layer 0, always slot 0) contributes nothing below, so
    // lanes walk their non-base slots only: one round for a single front.
    const int kb = (cv > 0 && L4[0] == 0) ? 1 : 0;
    const int kmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(cv - kb));
    for (int k2 = 0; k2 < kmax; ++k2) {
      const int k = k2 + kb;
      int a = -1;
      bool band = false, unsat = false, root = false;
      if (k < cv) {
        int l = 0;
        double x = 0.0;
        unsigned long long pw = 0;
        if (k < 4) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q == k) {
              l = L4[q];
              x = X4[q];
              pw = P4[q];
            }
        } else {
          l = F.lay[b + k];
          x = F.val[b + k];
          pw = W.parent[b + k];
        }
        if (l != 0 && is_active(l)) {
          a = W.aidx[l];
          unsat = x > 0.0 && x < 1.0;
          if (unsat && x >= P.kappa) cand = true;
          if (x >= P.kappa) ++nkappa;
          band = x > P.band_lo && x < P.sat;
          if (band) {
            // Unions are complete, so an item is a root iff its parent entry
            // is stale (never linked this epoch) or points to itself.
            const unsigned item = static_cast<unsigned>(v) * kSlots + k;
            root = count_roots && ((pw >> 32) != ep || static_cast<unsigned>(pw) == item);

          }
        }
      }
      if (P.record_trails) {
        // Band items for the trail snap: appended to this CTA's segment with
        // one shared-memory atomic per warp; the part of a batch that does
        // not fit goes to the overflow list (one global atomic).
        const unsigned bm = __ballot_sync(0xffffffffu, band);
        if (bm) {
          const int leader = __ffs(bm) - 1;
          int base = 0;
          if (lane == leader) base = atomicAdd(&S.nbp, __popc(bm));
          base = __shfl_sync(0xffffffffu, base, leader);
          const int pos = base + __popc(bm & ((1u << lane) - 1u));
          const int seg = blockIdx.x < W.bp_nseg ? W.bp_seg : 0;
          int obase = 0;
          unsigned om = 0;
          if (base + __popc(bm) > seg) {
            om = __ballot_sync(0xffffffffu, band && pos >= seg);
            const int ol = __ffs(om) - 1;
            if (lane == ol) obase = atomicAdd(&W.ctl->nbandpairs[cs], __popc(om));
            obase = __shfl_sync(0xffffffffu, obase, ol);
          }
          if (band) {
            if (pos < seg) {
              pick2(W.bandpairs, set)[static_cast<size_t>(blockIdx.x) * W.bp_seg + pos] = make_int2(v, a);
            } else {
              const int o = obase + __popc(om & ((1u << lane) - 1u));
              if (o < W.bandpair_cap) pick2(W.bp_ovf, set)[o] = make_int2(v, a);
              else {
                W.ctl->bandpair_overflow = 1;  // the trail snap would miss items: a capacity error
                raise_error(W.ctl, kDevCapacity, v, false);
              }
            }
          }
        }
      }
      // One round per distinct layer of the warp (usually one), with
      // full-warp votes and reductions: a partial-mask reduction costs ~10x
      // a full-mask one on sm_100a (tools/fp64_lat.cu).
      for (unsigned todo = __ballot_sync(0xffffffffu, a >= 0); todo;) {
        const int ldr = __ffs(todo) - 1;
        const int key = __shfl_sync(0xffffffffu, a, ldr);
        const bool mine = a == key;
        todo &= ~__ballot_sync(0xffffffffu, mine);
        const int nunsat = __popc(__ballot_sync(0xffffffffu, mine && unsat));
        const int nband = __popc(__ballot_sync(0xffffffffu, mine && band));
        const int nroot = __popc(__ballot_sync(0xffffffffu, mine && root));
        const bool mb = mine && band;
        const long long sx = warp_sum_fx(mb ? px : 0);
        const long long sy = warp_sum_fx(mb ? py : 0);
        const long long sz = warp_sum_fx(mb ? pz : 0);
        if (lane != ldr) continue;
        if (key < kSmemLayers) {
          if (nunsat) atomicAdd(&S.cnt[key][2], nunsat);
          if (nband) {
            atomicAdd(&S.cnt[key][1], nband);
            atomicAdd(reinterpret_cast<unsigned long long*>(&S.sum[key][0]), static_cast<unsigned long long>(sx));
            atomicAdd(reinterpret_cast<unsigned long long*>(&S.sum[key][1]), static_cast<unsigned long long>(sy));
            atomicAdd(reinterpret_cast<unsigned long long*>(&S.sum[key][2]), static_cast<unsigned long long>(sz));
          }
          if (nroot) atomicAdd(&S.cnt[key][0], nroot);
        } else {
          if (nunsat) atomicAdd(&g[key].nunsat, nunsat);
          if (nband) {
            atomicAdd(&g[key].nband, nband);
            atomicAdd(reinterpret_cast<unsigned long long*>(&g[key].sx), static_cast<unsigned long long>(sx));
            atomicAdd(reinterpret_cast<unsigned long long*>(&g[key].sy), static_cast<unsigned long long>(sy));
            atomicAdd(reinterpret_cast<unsigned long long*>(&g[key].sz), static_cast<unsigned long long>(sz));
          }
          if (nroot) atomicAdd(&g[key].ncomp, nroot);
        }
      }
    }
    if (cand && nkappa >= 2 && !(base > P.coll_base_limit)) {  // a pair needs two such layers
      int first = -1;
      for (int k = 0; k < cv; ++k) {
        const int l = F.lay[b + k];
        if (l == 0 || !is_active(l)) continue;
        if (F.val[b + k] < P.kappa) continue;
        if (first < 0) first = l;
        else insert_pair(W, (static_cast<unsigned>(first) << 16) | static_cast<unsigned>(l), ep, cs);
      }
    }
    INSTR_REC(2, t0, live);
  }
}

__device__ __forceinline__ void band_mean(const DevMesh& M, const LayerStat& st, double& mx, double& my, double& mz) {
  const double n = static_cast<double>(st.nband);
  mx = (static_cast<double>(st.sx) * M.fx_scale) / n;
  my = (static_cast<double>(st.sy) * M.fx_scale) / n;
  mz = (static_cast<double>(st.sz) * M.fx_scale) / n;
}

// snap_to_band (diffusion.hpp:590) over recorded band items: nearest band
// vertex to the band mean; key = distance bits (27 low bits dropped) | vertex.
// Lane `rank` of `stride` walks the list (every lane of a warp runs the same
// number of rounds so the warp-level minimum is well defined); each warp
// leader folds its minimum into the layer's statistics with one atomic.
__device__ void snap_list(const DevMesh& M, LayerStat* g, const int2* items, int n, int rank, int stride) {
  const int lane = threadIdx.x & 31;
  const int trip = (n + stride - 1) / stride;
  for (int r = 0; r < trip; ++r) {
    const int i = r * stride + rank;
    int a = -1;
    unsigned long long key = ~0ull;
    if (i < n) {
      const int2 bp = items[i];
      const int v = bp.x;
      a = bp.y;
      double mx, my, mz;
      band_mean(M, g[a], mx, my, mz);
      const double dx = __ldg(M.px + v) - mx, dy = __ldg(M.py + v) - my, dz = __ldg(M.pz + v) - mz;
      const double d2 = dx * dx + dy * dy + dz * dz;
      key = (static_cast<unsigned long long>(__double_as_longlong(d2)) & ~kVertMask) | static_cast<unsigned long long>(v);
    }
    for (unsigned todo = __ballot_sync(0xffffffffu, a >= 0); todo;) {  // full-warp rounds per layer
      const int ldr = __ffs(todo) - 1;
      const int k = __shfl_sync(0xffffffffu, a, ldr);
      const bool mine = a == k;
      todo &= ~__ballot_sync(0xffffffffu, mine);
      const unsigned long long kmin = seg_min_u64(0xffffffffu, mine ? key : ~0ull);
      if (lane == ldr) atomicMin(&g[k].snap, kmin);
    }
  }
}

// Trail snap of check `step` (its band items: set step & 1, n_ovf of them in
// the overflow list) by threads [t0, t0 + nthreads) of every CTA: each CTA
// takes the segments c = blockIdx.x (mod grid) -- in the engine its own --
// and a grid-strided share of the overflow list.
__device__ void phase_snap(const DevMesh& M, const DevWork& W, long long step, int n_ovf, int t0, int nthreads) {
  LayerStat* g = W.stat + static_cast<size_t>(slot4(step)) * kMaxActive;
  const int set = static_cast<int>(step & 1);
  const int rank = static_cast<int>(threadIdx.x) - t0;
  for (int c = blockIdx.x; c < W.bp_nseg; c += gridDim.x)
    snap_list(M, g, pick2(W.bandpairs, set) + static_cast<size_t>(c) * W.bp_seg, min(pick2(W.bpcount, set)[c], W.bp_seg), rank,
              nthreads);
  snap_list(M, g, pick2(W.bp_ovf, set), min(n_ovf, W.bandpair_cap), rank * static_cast<int>(gridDim.x) + blockIdx.x,
            static_cast<int>(gridDim.x) * nthreads);
}

__device__ void reset_stat(LayerStat* st) {
  st->ncomp = 0;
  st->nband = 0;
  st->nunsat = 0;
  st->sx = st->sy = st->sz = 0;
  st->snap = ~0ull;
}

// Writes the trail / last-position record of active index a for check `step`
// and resets its statistics slot for the check four steps later.
__device__ void flush_stat(const DevMesh& M, const DevWork& W, const StepParams& P, int a, long long step) {
  LayerStat* st = W.stat + static_cast<size_t>(slot4(step)) * kMaxActive + a;
  if (st->nband > 0) {
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
      r.step = step;
      r.layer = layer;
      r.vertex = static_cast<int>(st->snap & kVertMask);
      r.mx = mx;
      r.my = my;
      r.mz = mz;
      r.vx = M.px[r.vertex];
      r.vy = M.py[r.vertex];
      r.vz = M.pz[r.vertex];
      W.trail[pos & W.trail_mask] = r;
    }
  }
  reset_stat(st);
}
__device__ void flush_range(const DevMesh& M, const DevWork& W, const StepParams& P, long long step, int t0,
                            int nthreads) {
  for (int a = (static_cast<int>(threadIdx.x) - t0) * static_cast<int>(gridDim.x) + blockIdx.x; a < P.n_active;
       a += nthreads * static_cast<int>(gridDim.x))
    flush_stat(M, W, P, a, step);
}

// The stop decision of check `step` (diffusion.hpp:807-845): a split, a
// collision, a vanishing layer, base extinction, or a device error.  Every
// CTA reads the same words, right after the barrier that completed them.
__device__ int decide(const DevWork& W, const StepParams& P, long long step) {
  const int cs = slot4(step);
  const LayerStat* g = W.stat + static_cast<size_t>(cs) * kMaxActive;
  int bits = 0;
  for (int a = threadIdx.x; a < P.n_active; a += blockDim.x) {
    const LayerStat& st = g[a];
    if (st.ncomp >= 2) bits |= kStopSplit;
    if (st.nband == 0 && st.nunsat == 0) bits |= kStopVanish;
  }
  if (threadIdx.x == 0) {
    if (W.ctl->npairs[cs] > 0 || W.ctl->pair_overflow[cs]) bits |= kStopMerge;
    const double bmax = __longlong_as_double(static_cast<long long>(W.ctl->base_max_bits[cs]));
    if (W.ctl->base_cum[cs] == 0 && bmax < P.extinct_limit) bits |= kStopExtinct;
    if (W.ctl->bandpair_overflow) bits |= kStopError;
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

// The band list carried over a step without a check: the entries of the list
// of `step` whose column is interesting after the step join the list of
// step + 1 (what E's compaction does at a check).
__device__ void carry_list(const FieldBuf& F, const DevWork& W, long long step, int n) {
  const int* list = pick4(W.ilist, slot4(step));
  int* next = pick4(W.ilist, slot4(step + 1));
  int* count = &W.ctl->ilcount[slot4(step + 1)];
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * blockDim.x;
  // The loop condition is warp-uniform (idx - lane is the warp's first index).
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx - lane < n; idx += stride) {
    const int v = idx < n ? list[idx] : -1;
    const bool live = v >= 0 && F.interest[v];
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (!m) continue;
    const int leader = __ffs(m) - 1;
    int b = 0;
    if (lane == leader) b = atomicAdd(count, __popc(m));
    b = __shfl_sync(0xffffffffu, b, leader);
    if (live) next[b + __popc(m & ((1u << lane) - 1u))] = v;
  }
}

__device__ __forceinline__ void grid_sync_snap_decide(Ctl* ctl, CtlSnap& sc, const DevWork& W, const StepParams& P,
                                                      long long step) {
  cooperative_groups::this_grid().sync();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int cs = slot4(step);
    const LayerStat* g = W.stat + static_cast<size_t>(cs) * kMaxActive;
    int bits = 0;
    if (lane == 0) {
      const int4* src = reinterpret_cast<const int4*>(ctl);
      int4* dst = reinterpret_cast<int4*>(&sc);
#pragma unroll
      for (int q = 0; q < 7; ++q) dst[q] = __ldcg(src + q);
      if (__ldcg(&ctl->npairs[cs]) > 0 || __ldcg(&ctl->pair_overflow[cs])) bits |= kStopMerge;
      const double bmax = __longlong_as_double(static_cast<long long>(__ldcg(&ctl->base_max_bits[cs])));
      if (__ldcg(&ctl->base_cum[cs]) == 0 && bmax < P.extinct_limit) bits |= kStopExtinct;
      if (__ldcg(&ctl->bandpair_overflow)) bits |= kStopError;
    }
    for (int a = lane; a < P.n_active; a += 32) {
      const int4 c = __ldcg(reinterpret_cast<const int4*>(g + a));  // ncomp, nband, nunsat
      if (c.x >= 2) bits |= kStopSplit;
      if (c.y == 0 && c.z == 0) bits |= kStopVanish;
    }
    bits = static_cast<int>(__reduce_or_sync(kFull, static_cast<unsigned>(bits)));
    if (lane == 0) {
      sc.pad_[0] = bits;
      INSTR_PHASE();
    }
  }
  __syncthreads();
}

// ceil(n / gridDim.x) by a multiply-high with magic = ceil(2^32 / grid): exact
// while (n + grid - 1) < 2^32 / grid (the error of the product stays below
// 1 / grid); larger n divides.
__device__ __forceinline__ int ceil_div_grid(int n, unsigned magic) {
  const unsigned x = static_cast<unsigned>(n) + gridDim.x - 1;
  return x < magic ? static_cast<int>(__umulhi(x, magic)) : static_cast<int>(x / gridDim.x);
}

// Slot clears of the phase that starts step t (one thread; see slot4):
// the frontier list A(t) read, the band list / change tracking / check
// outputs of step t+2, the base delta of step t-1 (consumed), the digest of
// check t+1.
__device__ __forceinline__ void phase_resets(Ctl* ctl, long long t) {
  const int c0 = slot4(t), c2 = slot4(t + 2);
  ctl->rcount[c0] = 0;
  ctl->ilcount[c2] = 0;
  ctl->dchange[c2] = 0;
  ctl->nadded[c2] = 0;
  ctl->anchor_fail[c2] = 0;
  ctl->npairs[c2] = 0;
  ctl->pair_overflow[c2] = 0;
  ctl->base_max_bits[c2] = 0;
  ctl->nbandpairs[c2] = 0;
  ctl->base_d[slot4(t - 1)] = 0;
  ctl->hash_acc[slot4(t + 1)] = 0;
}

// mode 0: run steps; mode 1: check only (stats of the current state, step
// step_begin); mode 2: snap for that check; mode 3: flush it.
template <int kMode>
__global__ void __launch_bounds__(kBlock, 1) k_engine(DevMesh M, DevField F, DevWork W, StepParams P) {
  __shared__ BlockStats S;
  __shared__ BlockQueue Q;
  __shared__ CtlSnap SC;
  Ctl* ctl = W.ctl;
  if (threadIdx.x == 0) Q.n = 0;
  load_active(W.active, P.n_layers);
#ifdef DTB_INSTR
  for (int i = threadIdx.x; i < 6 * 16; i += blockDim.x) s_hist[i / 16][i % 16] = 0;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_cp[i / 2][i % 2] = 0;
#endif
  __syncthreads();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gsz = gridDim.x * blockDim.x;
  const int nthr = static_cast<int>(blockDim.x);
  const unsigned magicG = 0xFFFFFFFFu / gridDim.x + 1;  // ceil(2^32 / grid), see ceil_div_grid
  unsigned long long ep = static_cast<unsigned long long>(ctl->epoch);

  if (kMode == 1) {
    // The field copies are identical between launches; the band list of
    // slot4(s) was rebuilt by the host.
    const long long s = P.step_begin;
    const int cs = slot4(s);
    LayerStat* g = W.stat + static_cast<size_t>(cs) * kMaxActive;
    for (int a = gtid; a < kMaxActive; a += gsz) reset_stat(g + a);
    if (gtid == 0) {
      ctl->npairs[cs] = 0;
      ctl->pair_overflow[cs] = 0;
      ctl->base_max_bits[cs] = 0;
      ctl->nbandpairs[cs] = 0;
      ctl->bandpair_overflow = 0;
    }
    grid_sync_snap(ctl, SC);
    ++ep;
    const FieldBuf Fc = pickf(F, s);
    const int n = SC.ilcount[cs];
    phase_union(M, Fc, W, P, cs, ep, group_rank(1), gsz / kG, n);
    grid_sync(ctl);
    block_stats_init(S);
    phase_stats(M, Fc, W, P, s, ep, false, S, n, true, 0, nthr);
    e_flush(S, W, P.n_active, s, 0, 0, nthr);
    grid_sync(ctl);
    if (gtid == 0) ctl->epoch = static_cast<long long>(ep);
    return;
  }
  if (kMode == 2) {
    phase_snap(M, W, P.step_begin, ctl->nbandpairs[slot4(P.step_begin)], 0, nthr);
    return;
  }
  if (kMode == 3) {
    if (gtid < P.n_active) flush_stat(M, W, P, gtid, P.step_begin);
    return;
  }

  // ---- mode 0: the step loop.  Step s is one phase in the common case:
  //   E(s)   the check of the field after s (stats, collisions, list compaction)
  //   A(s+1) the update of step s+1 (b[s & 1] -> b[(s+1) & 1]) with its
  //          bookkeeping (next frontier, band list, certificate items)
  //   and, on other warps, the split certificate of s, the trail snap of
  //   check s-1 and the trail records of check s-2.
  // Without the certificate (4 % of the steps on configs[1]) the union-find
  // D(s) runs beside A(s+1) and E(s) takes a phase of its own.  A(s+1) is
  // speculative: when check s stops the run it is discarded (the host
  // relaunches at s+1), and its errors count only if check s does not stop.
  long long s = P.step_begin;
  int stop = 0;
  bool first_check = true;     // the first check of a launch follows host edits: always the union-find
  bool ran_spec = false;       // the stopping phase ran A(s+1)
  long long snap_step = -1;    // check whose trail snap runs in the next phase
  long long flush_step = -1;   // check whose trail records are written in the next phase
  long long last_snapped = -1; // check snapped in the phase just ended
  block_stats_init(S);  // e_flush clears it again after every check
  {  // prologue: A(step_begin), reading the field after step_begin - 1
    ctl_snap(ctl, SC);
    const long long b = P.step_begin;
    const int nR = SC.rcount[slot4(b)];
    if (gtid == 0) {
      phase_resets(ctl, b - 1);
      ctl->base_cum[slot4(b - 1)] = ctl->base_one;
      ctl->sum_region += static_cast<unsigned long long>(nR);
    }
    update_items(M, F, W, P, static_cast<int>(b), nR, group_rank(2), gsz / kG, false, Q);
    bq_flush(Q, &ctl->rcount[slot4(b + 1)], pick4(W.region, slot4(b + 1)));
    grid_sync_snap(ctl, SC);
    if (SC.error) stop = kStopError;
  }
  for (; stop == 0 && s < P.step_end; ++s) {
    const bool check = P.do_check && (P.check_interval == 1 || static_cast<int>(s) % P.check_interval == 0);
    const bool more = s + 1 < P.step_end;
    const int c0 = slot4(s);
    const FieldBuf Fs = pickf(F, s);  // the field after step s
    const int nR1 = more ? SC.rcount[slot4(s + 1)] : 0;  // frontier s+1, final since the last barrier
    const int nband = SC.ilcount[c0];
    const long long pslot = (s - P.step_begin) * 4;
    const bool prof = W.prof && gtid == 0 && pslot + 3 < W.prof_cap;
    if (prof) W.prof[pslot] = gtimer();
    if (gtid == 0) {
      phase_resets(ctl, s);
      ctl->base_cum[c0] = ctl->base_cum[slot4(s - 1)] + ctl->base_d[c0];
      ctl->sum_region += static_cast<unsigned long long>(nR1);
      if (check) ctl->sum_interest += static_cast<unsigned long long>(nband);
    }
    const long long fl = flush_step, sn = P.record_trails ? snap_step : -1;
    const int n_ovf = sn >= 0 ? SC.nbandpairs[slot4(sn)] : 0;
    // Earlier checks' trail work (no CTA barrier inside), by threads [t0, t0 + n).
    auto side = [&](int t0, int n) {
      if (fl >= 0) flush_range(M, W, P, fl, t0, n);
      if (sn >= 0) phase_snap(M, W, sn, n_ovf, t0, n);
    };
    auto run_a = [&](bool spec) {  // by whole warps
      update_items(M, F, W, P, static_cast<int>(s + 1), nR1, group_rank(2), gsz / kG, spec, Q);
    };
    const int q2 = slot4(s + 2);  // A(s+1) queues frontier s+2
    last_snapped = snap_step;
    if (!check) {
      block_start(W, s - (P.step_end - 64), 1);
      if (more) run_a(false);
      carry_list(Fs, W, s, nband);
      side(0, nthr);
      bq_flush(Q, &ctl->rcount[q2], pick4(W.region, q2));
      block_done(W, s - (P.step_end - 64), 1);
      grid_sync_snap(ctl, SC);
      if (prof) W.prof[pslot + 1] = W.prof[pslot + 2] = W.prof[pslot + 3] = gtimer();
      flush_step = snap_step;
      snap_step = -1;
      if (SC.error) {
        stop = kStopError;
        ++s;  // the failing update belongs to step s+1
        break;
      }
      continue;
    }
    ++ep;
    const bool skip = !P.d_full && P.check_interval == 1 && !first_check && !SC.dchange[c0];
    if (skip) {
      // ---- certificate holds: one phase.  E on the first warps, A on the
      // last ones, the certificate and the trail work in between; each role
      // flushes behind a barrier of its own warps.
      if (prof) W.prof[pslot + 1] = W.prof[pslot];
      block_start(W, s - (P.step_end - 64), 1);
      const int nwarps = nthr / 32;
      const int e_per_cta = ceil_div_grid(nband, magicG);
      const int a_per_cta = ceil_div_grid(nR1, magicG);
      const int e_warps = max(1, (e_per_cta + 31) / 32), a_warps = (a_per_cta + 3) / 4;
      const bool split = !P.do_hash && e_per_cta <= nthr && a_per_cta <= nthr / kG && e_warps + a_warps <= nwarps;
      if (split) {
        const int warp = threadIdx.x >> 5;
        const int m0 = e_warps, m1 = nwarps - a_warps;  // middle warps [m0, m1)
        if (warp < m0) {
          phase_stats(M, Fs, W, P, s, ep, true, S, nband, false, 0, m0 * 32);
          INSTR_AT_W(8, 0);
          if (m1 == m0) {  // no middle warps: E's warps take the rest
            anchor_test(M, Fs, W, P, SC.nadded[c0], static_cast<int>(s),
                        static_cast<int>(threadIdx.x) / kG * static_cast<int>(gridDim.x) + blockIdx.x,
                        m0 * 32 / kG * static_cast<int>(gridDim.x));
            side(0, m0 * 32);
          }
          e_flush(S, W, P.n_active, s, 1, 0, m0 * 32);
          INSTR_AT_W(9, 0);
        } else if (warp >= m1) {
          if (more) run_a(true);
          if (a_warps > 0) bq_flush(Q, &ctl->rcount[q2], pick4(W.region, q2), 2, m1 * 32, a_warps * 32);
          INSTR_AT_W(7, 0);
        } else {
          const int r = static_cast<int>(threadIdx.x) - m0 * 32, nm = (m1 - m0) * 32;
          anchor_test(M, Fs, W, P, SC.nadded[c0], static_cast<int>(s),
                      r / kG * static_cast<int>(gridDim.x) + blockIdx.x, nm / kG * static_cast<int>(gridDim.x));
          side(m0 * 32, nm);
          INSTR_AT_W(10, 0);
        }
      } else {
        if (more) run_a(true);
        phase_stats(M, Fs, W, P, s, ep, true, S, nband, false, 0, nthr);
        anchor_test(M, Fs, W, P, SC.nadded[c0], static_cast<int>(s), gtid / kG, gsz / kG);
        side(0, nthr);
        if (P.do_hash) phase_hash(Fs, &ctl->hash_acc[c0], M.nv);
        e_flush(S, W, P.n_active, s, 0, 0, nthr);
        bq_flush(Q, &ctl->rcount[q2], pick4(W.region, q2));
      }
      block_done(W, s - (P.step_end - 64), 1);
      grid_sync_snap_decide(ctl, SC, W, P, s);
      if (prof) W.prof[pslot + 2] = gtimer();
      if (SC.anchor_fail[c0] || P.cert_verify) {  // an item failed its test: the union-find after all
        block_start(W, s - (P.step_end - 64), 2);
        phase_union(M, Fs, W, P, c0, ep, group_rank(1), gsz / kG, nband);
        grid_sync(ctl);
        phase_roots(Fs, W, P, c0, c0, ep, nband);
        block_done(W, s - (P.step_end - 64), 2);
        grid_sync(ctl);
        int b2 = decide(W, P, s);  // the root counts changed
        if (P.cert_verify && !SC.anchor_fail[c0] && (b2 & kStopSplit)) {  // the certificate held wrongly
          b2 |= kStopError;
          if (gtid == 0) raise_error(ctl, kDevCertificate, -1, false);
        }
        __syncthreads();
        if (threadIdx.x == 0) SC.pad_[0] = b2;
        __syncthreads();
      }
      if (prof) W.prof[pslot + 3] = gtimer();
    } else {
      // ---- D(s) beside A(s+1) and the trail work, then E(s) with roots.
      block_start(W, s - (P.step_end - 64), 0);
      if (more) run_a(true);
      phase_union(M, Fs, W, P, c0, ep, group_rank(1), gsz / kG, nband);
      side(0, nthr);
      if (P.do_hash) phase_hash(Fs, &ctl->hash_acc[c0], M.nv);
      bq_flush(Q, &ctl->rcount[q2], pick4(W.region, q2));
      block_done(W, s - (P.step_end - 64), 0);
      grid_sync(ctl);
      if (prof) W.prof[pslot + 1] = gtimer();
      block_start(W, s - (P.step_end - 64), 1);
      phase_stats(M, Fs, W, P, s, ep, true, S, nband, true, 0, nthr);
      e_flush(S, W, P.n_active, s, 0, 0, nthr);
      block_done(W, s - (P.step_end - 64), 1);
      grid_sync_snap_decide(ctl, SC, W, P, s);
      if (prof) W.prof[pslot + 2] = W.prof[pslot + 3] = gtimer();
    }
    if (P.do_hash && gtid == 0) {
      const long long slot = s - W.hash_base;
      if (slot >= 0 && slot < W.hash_cap) W.hashes[slot] = ctl->hash_acc[c0];
    }
    first_check = false;
    int bits = SC.pad_[0];
    if (P.stop_every_check) bits |= kStopEveryCheck;
    if (bits) {
      stop = bits;
      ran_spec = more;
      break;  // A(s+1) is discarded; the host relaunches at s+1
    }
    if (SC.spec_error) {
      if (gtid == 0) {
        ctl->error = ctl->spec_error;
        ctl->error_vertex = ctl->spec_error_vertex;
      }
      stop = kStopError;
      ++s;  // the failing update belongs to step s+1
      break;
    }
    flush_step = snap_step;
    snap_step = s;
  }
  // ---- epilogue.  `last` is the last step whose results stand.
  const long long last = stop ? s : s - 1;
  if (!(stop & kStopError)) {
    if (stop) {
      // Stopped at check `last`: the host runs its snap and records; the
      // check before it was snapped in the last phase.
      if (last_snapped >= 0) flush_range(M, W, P, last_snapped, 0, nthr);
    } else {
      // Budget exhausted: finish the pending checks' trail work.
      if (flush_step >= 0) flush_range(M, W, P, flush_step, 0, nthr);
      if (snap_step >= 0) {
        if (P.record_trails) phase_snap(M, W, snap_step, SC.nbandpairs[slot4(snap_step)], 0, nthr);
        grid_sync(ctl);
        flush_range(M, W, P, snap_step, 0, nthr);
      }
    }
    // Both field copies identical again: the columns of frontier last+1 (every
    // column step `last` changed, and every column a discarded A(last+1)
    // overwrote) copied from the field after `last`.
    {
      const FieldBuf A = pickf(F, last);
      const FieldBuf B = pickf(F, last + 1);
      const int* list = pick4(W.region, slot4(last + 1));
      const int n = SC.rcount[slot4(last + 1)];
      for (int i = gtid; i < n; i += gsz) {
        const int v = list[i];
        const int c = A.cnt[v];
        const size_t vb = static_cast<size_t>(v) * kSlots;
        for (int j = 0; j < c; ++j) {
          B.lay[vb + j] = A.lay[vb + j];
          B.val[vb + j] = A.val[vb + j];
        }
        B.cnt[v] = static_cast<unsigned char>(c);
        B.interest[v] = A.interest[v];
        B.binfo[v] = A.binfo[v];
      }
    }
    if (ran_spec) {
      // Unclaim the frontier the discarded A(last+1) queued, then re-stamp
      // frontier last+1 (a vertex in both carried the newer stamp): the host
      // adds to frontier last+1 and the relaunch queues frontier last+2.
      const int* list = pick4(W.region, slot4(last + 2));
      const int n = SC.rcount[slot4(last + 2)];
      for (int i = gtid; i < n; i += gsz) W.stamp[list[i]] = -1;
      grid_sync(ctl);
      const int* cur = pick4(W.region, slot4(last + 1));
      const int nc = SC.rcount[slot4(last + 1)];
      for (int i = gtid; i < nc; i += gsz) W.stamp[cur[i]] = static_cast<int>(last);
    }
  }
  if (gtid == 0) {
    ctl->stop_bits = stop;
    ctl->stop_step = last;
    ctl->epoch = static_cast<long long>(ep);
    if (!(stop & kStopError)) ctl->base_one = ctl->base_cum[slot4(last)];
    for (int q = 0; q < 4; ++q) ctl->base_d[q] = 0;
  }
#ifdef DTB_INSTR
  __syncthreads();
  for (int i = threadIdx.x; i < 6 * 16; i += blockDim.x)
    if (s_hist[i / 16][i % 16]) atomicAdd(&g_hist[i / 16][i % 16], s_hist[i / 16][i % 16]);
  for (int i = threadIdx.x; i < 64; i += blockDim.x)
    if (s_cp[i / 2][i % 2]) atomicAdd(&g_cp[i / 2][i % 2], static_cast<unsigned long long>(s_cp[i / 2][i % 2]));
#endif
}

// Barrier microbenchmark (diagnostics): n grid barriers, no work.
__global__ void __launch_bounds__(kBlock, 1) k_barrier_bench(Ctl* ctl, int n, int mode) {
  if (mode == 0) {
    for (int i = 0; i < n; ++i) grid_sync(ctl);
  } else {
    cooperative_groups::grid_group g = cooperative_groups::this_grid();
    for (int i = 0; i < n; ++i) g.sync();
  }
}

// Shared memory above the 48 KB static limit must be opted into per kernel.
cudaError_t engine_attributes() {
  static cudaError_t done = [] {
    const void* fns[] = {reinterpret_cast<const void*>(&k_engine<0>), reinterpret_cast<const void*>(&k_engine<1>),
                         reinterpret_cast<const void*>(&k_engine<2>), reinterpret_cast<const void*>(&k_engine<3>)};
    for (const void* fn : fns) {
      const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }();
  return done;
}

int coop_launch(const void* fn, int blocks, const DevMesh& m, const DevField& f, const DevWork& w,
                const StepParams& p, void* stream) {
  DevMesh mm = m;
  DevField ff = f;
  DevWork ww = w;
  StepParams pp = p;
  void* args[] = {&mm, &ff, &ww, &pp};
  const cudaError_t ea = engine_attributes();
  if (ea != cudaSuccess) return static_cast<int>(ea);
  note_launch();
  return static_cast<int>(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kBlock), args, kDynSmem,
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
  e = engine_attributes();
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_engine<0>, kBlock, kDynSmem);
  if (e != cudaSuccess) return static_cast<int>(e);
  int per1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_engine<1>, kBlock, kDynSmem);
  if (per1 < per) per = per1;
  *out = sms * (per < 1 ? 1 : per);
  return 0;
}

void instr_report() {
#ifdef DTB_INSTR
  unsigned long long h[6][16];
  cudaMemcpyFromSymbol(h, g_hist, sizeof(h));
  static const char* names[6] = {"B commit", "D union", "E stats", "A paths(1,!1,fast,gen)", "gen cnt(v)", "gen ncand"};
  for (int p = 0; p < 6; ++p) {
    unsigned long long n = 0;
    for (int b = 0; b < 16; ++b) n += h[p][b];
    std::fprintf(stderr, "[dtb] instr %-8s n=%10llu  buckets(128ns*2^b):", names[p], n);
    for (int b = 0; b < 16; ++b) std::fprintf(stderr, " %llu", h[p][b]);
    std::fprintf(stderr, "\n");
  }
  std::memset(h, 0, sizeof(h));
  cudaMemcpyToSymbol(g_hist, h, sizeof(h));
  unsigned long long c[32][2];
  cudaMemcpyFromSymbol(c, g_cp, sizeof(c));
  std::fprintf(stderr, "[dtb] instr checkpoints (avg SM cycles since item start):");
  for (int i = 0; i < 32; ++i)
    if (c[i][1]) std::fprintf(stderr, " cp%d=%.0f", i, 16.0 * static_cast<double>(c[i][0]) / c[i][1]);
  std::fprintf(stderr, "\n");
  std::memset(c, 0, sizeof(c));
  cudaMemcpyToSymbol(g_cp, c, sizeof(c));
#endif
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
  if (const cudaError_t ea = engine_attributes(); ea != cudaSuccess) return static_cast<int>(ea);
  note_launch();
  k_engine<2><<<148 * 4, kBlock, kDynSmem, static_cast<cudaStream_t>(stream)>>>(m, f, w, p);
  return static_cast<int>(cudaGetLastError());
}

int launch_flush(const DevMesh& m, const DevField& f, const DevWork& w, const StepParams& p, void* stream) {
  const int blocks = (p.n_active + kBlock - 1) / kBlock;
  if (blocks == 0) return 0;
  if (const cudaError_t ea = engine_attributes(); ea != cudaSuccess) return static_cast<int>(ea);
  note_launch();
  k_engine<3><<<blocks, kBlock, kDynSmem, static_cast<cudaStream_t>(stream)>>>(m, f, w, p);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace dtb

namespace dtb {
// Returns nanoseconds per grid barrier (mode 0: engine barrier, 1: cooperative_groups).
double bench_barrier(int blocks, int n, int mode) {
  Ctl* ctl = nullptr;
  cudaMalloc(&ctl, sizeof(Ctl));
  cudaMemset(ctl, 0, sizeof(Ctl));
  void* args[] = {&ctl, &n, &mode};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_barrier_bench), dim3(blocks), dim3(kBlock), args, 0, 0);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_barrier_bench), dim3(blocks), dim3(kBlock), args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(ctl);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms * 1e6 / n;
}
}  // namespace dtb
