// Dependent-load latency probe (diagnostics, not part of the library).
// Measures SM cycles per dependent global load of a pointer chase through an
// L2-resident array, with 1 active warp per SM vs all warps, and right after
// the array was rewritten by other SMs behind a grid barrier.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/latency_probe tools/latency_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>

__global__ void probe(unsigned* next, int n, int hops, int active_warps_per_cta, int rewrite, unsigned long long* out) {
  namespace cg = cooperative_groups;
  const int warp = threadIdx.x / 32;
  const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
  if (rewrite) {
    // every thread rewrites a slice (same values) so lines are dirty in L2 from other SMs
    for (unsigned i = gtid; i < static_cast<unsigned>(n); i += gridDim.x * blockDim.x) next[i] = next[i];
  }
  cg::this_grid().sync();
  unsigned x = (gtid * 2654435761u) % n;
  long long t0 = clock64();
  if (warp < active_warps_per_cta) {
    for (int h = 0; h < hops; ++h) x = next[x];
  }
  long long t1 = clock64();
  if (warp < active_warps_per_cta && (threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], static_cast<unsigned long long>(t1 - t0));
    atomicAdd(&out[1], 1ull);
  }
  if (x == 0xFFFFFFFFu) out[2] = x;
}

int main() {
  const int n = 1 << 22;  // 16 MB
  std::vector<unsigned> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<unsigned> next(n);
  for (int i = 0; i < n; ++i) next[perm[i]] = perm[(i + 1) % n];
  unsigned* d;
  unsigned long long* o;
  cudaMalloc(&d, sizeof(unsigned) * n);
  cudaMalloc(&o, 64);
  cudaMemcpy(d, next.data(), sizeof(unsigned) * n, cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rewrite = 0; rewrite < 2; ++rewrite)
    for (int aw : {1, 4, 16}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(o, 0, 64);
        int hops = 16, nn = n;
        void* args[] = {&d, &nn, &hops, &aw, &rewrite, &o};
        cudaLaunchCooperativeKernel((void*)probe, dim3(sms), dim3(512), args, 0, 0);
        unsigned long long h[2];
        cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        if (rep == 2)
          std::printf("rewrite=%d active_warps/SM=%2d: %.0f cycles per dependent load\n", rewrite, aw,
                      static_cast<double>(h[0]) / h[1] / hops);
      }
    }
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
