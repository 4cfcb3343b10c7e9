// Microbenchmark: cost of one "level" (bar.sync + dependent LDS chain + bar.sync)
// with 2 CTAs/SM x 9 warps, as in k_dag.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(288, 2) k(int iters, int depth, int* idx_g, unsigned long long* out, int mode) {
  extern __shared__ int sm[];
  const int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = idx_g[i];
  __syncthreads();
  if (tid >= 256) return;
  int v = tid;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode & 1) asm volatile("bar.sync 1, 256;" ::: "memory");
    for (int d = 0; d < depth; ++d) v = sm[(v + d) & 8191];
    if (mode & 2) asm volatile("bar.sync 1, 256;" ::: "memory");
  }
  unsigned long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0);
  if (v == -12345) out[0] = v;
}
int main() {
  int* idx; unsigned long long* out;
  cudaMalloc(&idx, 8192 * 4); cudaMalloc(&out, 1024 * 8);
  int h[8192]; for (int i = 0; i < 8192; ++i) h[i] = (i * 7919 + 13) & 8191;
  cudaMemcpy(idx, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int mode : {0, 2, 3}) for (int depth : {0, 1, 4, 8}) {
    k<<<296, 288, 100000>>>(1000, depth, idx, out, mode);
    cudaDeviceSynchronize();
    unsigned long long r[296]; cudaMemcpy(r, out, sizeof(r), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 296; ++i) s += r[i];
    printf("mode %d (bar before %d, after %d) depth %d: %.1f cycles/iter\n", mode, mode & 1, (mode >> 1) & 1, depth, s / 296 / 1000);
  }
  return 0;
}
