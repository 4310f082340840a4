// Latency microbenchmark (diagnostics, GPU box): dependent chains of fp64
// add / mul / div / sqrt and of 8-lane shuffles, one warp, cycles per op.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/fp64_lat.cu -o /tmp/fp64_lat && /tmp/fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = (x + 1.0) / b;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffu << (threadIdx.x & 24), x, (threadIdx.x + 1) & 7, 8) + 1.0;
  long long t5 = clock64();
  unsigned u = __double_as_longlong(x);
  for (int i = 0; i < n; ++i) u = __reduce_min_sync(0xffu << (threadIdx.x & 24), u + 1);
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_min_sync(0xffffffffu, u + 1);
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) u = __any_sync(0xffu << (threadIdx.x & 24), (u & 1) == 0) + u + 1;
  long long t8 = clock64();
  for (int i = 0; i < n; ++i) u = __any_sync(0xffffffffu, (u & 1) == 0) + u + 1;
  long long t9 = clock64();
  for (int i = 0; i < n; ++i) u = __shfl_sync(0xffffffffu, u, (threadIdx.x + 1) & 31) + 1;
  long long t10 = clock64();
  for (int i = 0; i < n; ++i) u = __shfl_sync(0xffu << (threadIdx.x & 24), u, (threadIdx.x + 1) & 7, 8) + 1;
  long long t11 = clock64();
  out[threadIdx.x] = x + u;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    cyc[6] = t7 - t6; cyc[7] = t8 - t7; cyc[8] = t9 - t8; cyc[9] = t10 - t9; cyc[10] = t11 - t10;
  }
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 16 * 8);
  const int n = 1000;
  for (int w = 1; w <= 16; w *= 4) {
    k<<<1, 32 * w>>>(o, c, 1.5, 1.0000003, n);
    k<<<1, 32 * w>>>(o, c, 1.5, 1.0000003, n);
    long long h[16];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("warps %2d  cycles/op: dadd %.1f  dmul %.1f  ddiv(+add) %.1f  dsqrt(+add) %.1f  shfl8.f64(+add) %.1f  redux.min(+add) %.1f\n", w,
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
    printf("          redux.min full %.1f  any8 %.1f  any32 %.1f  shfl32.u32 %.1f  shfl8.u32 %.1f\n", h[6] / (double)n,
           h[7] / (double)n, h[8] / (double)n, h[9] / (double)n, h[10] / (double)n);
  }
  return 0;
}
