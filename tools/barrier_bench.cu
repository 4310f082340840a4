// Grid-barrier microbenchmark (diagnostics, GPU box): cooperative_groups
// grid.sync() vs a release/acquire counter barrier, n barriers per launch,
// 148 CTAs x 512 threads (the engine's grid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/barrier_bench.cu -o /tmp/bb && /tmp/bb
#include <cooperative_groups.h>
#include <cstdio>

__device__ unsigned g_count, g_gen;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense-reversal barrier: the last arriver resets the count and bumps the generation.
__device__ __forceinline__ void bar_relacq(unsigned& gen_local) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen_local;
    const unsigned old = atom_add_acq_rel(&g_count, 1);
    if (old == gridDim.x - 1) {
      g_count = 0;  // ordered before the release store below
      st_release(&g_gen, g + 1);
    } else {
      while (ld_acquire(&g_gen) == g) {
      }
    }
    gen_local = g + 1;
  }
  __syncthreads();
}

__device__ unsigned long long g_count64;
__device__ unsigned g_cnt1[16];
__device__ __forceinline__ unsigned long long atom_add64_acq_rel(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// One 64-bit arrival counter that never resets: the arrival that completes
// a multiple of the grid releases the generation.
__device__ __forceinline__ void bar_count64(unsigned& gen_local) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen_local;
    const unsigned long long old = atom_add64_acq_rel(&g_count64, 1);
    if ((old + 1) % gridDim.x == 0) {
      st_release(&g_gen, g + 1);
    } else {
      while (ld_acquire(&g_gen) == g) {
      }
    }
    gen_local = g + 1;
  }
  __syncthreads();
}
// Two levels: groups of 16 CTAs meet on their own counter; the last of each
// group arrives at the top counter.
__device__ __forceinline__ void bar_tree(unsigned& gen_local) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen_local;
    const unsigned grp = blockIdx.x / 16, ngrp = (gridDim.x + 15) / 16;
    const unsigned gsize = min(16u, gridDim.x - grp * 16);
    const unsigned o1 = atom_add_acq_rel(&g_cnt1[grp], 1);
    bool released = false;
    if ((o1 + 1) % gsize == 0) {
      const unsigned long long o2 = atom_add64_acq_rel(&g_count64, 1);
      if ((o2 + 1) % ngrp == 0) {
        st_release(&g_gen, g + 1);
        released = true;
      }
    }
    if (!released)
      while (ld_acquire(&g_gen) == g) {
      }
    gen_local = g + 1;
  }
  __syncthreads();
}

__global__ void k(int n, int mode, long long* out) {
  unsigned gen = 0;
  if (threadIdx.x == 0) gen = ld_acquire(&g_gen);
  cooperative_groups::grid_group gg = cooperative_groups::this_grid();
  gg.sync();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (mode == 0) gg.sync();
    else if (mode == 1) bar_relacq(gen);
    else if (mode == 2) bar_count64(gen);
    else bar_tree(gen);
  }
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int mode = 0; mode < 4; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      int n = 20000;
      void* args[] = {&n, &mode, &d};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k, dim3(148), dim3(512), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("mode %d (%s) rep %d: %.3f us per barrier (%.0f cycles)  err=%d\n", mode, mode == 0 ? "cg" : mode == 1 ? "rel/acq reset" : mode == 2 ? "count64" : "tree16", rep,
             ms * 1e3 / n, (double)c / n, (int)e);
    }
  return 0;
}
