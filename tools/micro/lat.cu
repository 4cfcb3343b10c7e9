// Dependent-chain latencies on the GPU (cycles per op): DFMA, DADD, LDS.64,
// LDS.32 -> LDS.64 (indirect), shfl_xor, __syncwarp.   nvcc -arch=sm_100a lat.cu
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sd[1024];
  __shared__ int si[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sd[i] = 1.0 + i * 1e-9; si[i] = (i * 7 + 1) & 1023; }
  __syncwarp();
  double a = out[0], b = 1.0000001, c = 1e-12;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  t1 = clock64();
  cyc[0] = (t1 - t0);
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + c;
  t1 = clock64();
  cyc[1] = (t1 - t0);
  // LDS.32 pointer chase
  int p = threadIdx.x & 1023;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = si[p];
  t1 = clock64();
  cyc[2] = (t1 - t0);
  // LDS.32 -> LDS.64 -> DADD (indirect load chain)
  double acc = 0.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { p = si[p]; acc += sd[p]; }
  t1 = clock64();
  cyc[3] = (t1 - t0);
  // shfl_xor chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
  t1 = clock64();
  cyc[4] = (t1 - t0);
  // syncwarp loop
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncwarp(); a += 1e-20; }
  t1 = clock64();
  cyc[5] = (t1 - t0);
  // LDS.64 dependent through address: sd[(int)x & 1023]
  double x = sd[threadIdx.x];
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sd[((int)(x * 1e9)) & 1023];
  t1 = clock64();
  cyc[6] = (t1 - t0);
  out[1 + threadIdx.x] = a + acc + p + x;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 64 * 8);
  cudaMemset(o, 0, 4096 * 8);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n);
  k<<<1, 32>>>(o, c, n);
  long long h[8];
  cudaMemcpy(h, c, 7 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DADD", "LDS32 chase", "LDS32->LDS64+DADD", "SHFL+DADD", "syncwarp+DADD", "LDS64->cvt chase"};
  for (int i = 0; i < 7; ++i) printf("%-20s %.1f cycles/iter\n", nm[i], (double)h[i] / n);
  return 0;
}
