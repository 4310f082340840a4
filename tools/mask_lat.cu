// Warp-operation latency with partial but uniform masks (diagnostics, GPU box):
// full warp vs 8 live lanes (the rest exited or diverged).  All three cost the
// same (~25-37 cycles); a mask that differs between the lanes' groups is what
// is slow (tools/fp64_lat.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mask_lat.cu -o tools/mask_lat && tools/mask_lat
#include <cstdio>
__global__ void k(unsigned* out, long long* cyc, int n, int mode) {
  unsigned u = threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (mode == 1 && lane >= 8) return;         // only lanes 0..7 alive (exited)
  long long t0, t1;
  if (mode == 2 && lane >= 8) {               // lanes 8..31 diverged, idle in a spin
    volatile unsigned* f = out + 64;
    while (*f == 0) {}
    return;
  }
  const unsigned am = __activemask();
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = min(u, __shfl_xor_sync(am, u, 4)) + 1;
  t1 = clock64();
  long long ts = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u += __ballot_sync(am, (u & 1) == 0) & 1u;
  t1 = clock64();
  long long tb = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_min_sync(am, u) + 1;
  t1 = clock64();
  long long tr = t1 - t0;
  out[threadIdx.x] = u;
  if (threadIdx.x == 0) { cyc[0] = ts; cyc[1] = tb; cyc[2] = tr; cyc[3] = am; }
  if (mode == 2 && threadIdx.x == 0) { __threadfence(); atomicExch(out + 64, 1u); }
}
int main() {
  unsigned* o; long long* c;
  cudaMalloc(&o, 128 * 4); cudaMalloc(&c, 8 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(o, 0, 128 * 4);
    const int n = 2000;
    k<<<1, 32>>>(o, c, n, mode);
    cudaMemset(o, 0, 128 * 4);
    k<<<1, 32>>>(o, c, n, mode);
    long long h[4];
    cudaError_t e = cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d (%s) mask %llx: shfl_xor %.1f  ballot %.1f  redux.min %.1f cycles  err %d\n", mode,
           mode == 0 ? "full warp" : mode == 1 ? "8 lanes, rest exited" : "8 lanes, rest diverged", (unsigned long long)h[3],
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, (int)e);
  }
  return 0;
}
