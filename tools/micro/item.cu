// Micro-benchmark of one packed forward item of the FRAG kernel (dag_solve.cu
// fwd_row) on synthetic shared-memory data: cycles per item for variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 item.cu -o item
#include <cstdint>
#include <cstdio>

enum { R_S = 0, R_M, R_VAL, R_SCR, R_CPOS, R_WORDS };

__device__ __forceinline__ void fwd_row(const int32_t* R, const double* vals, double* S, int i) {
  const int s = R[R_S], m = R[R_M];
  if (i >= s + m) return;
  double* f = S + R[R_SCR];
  const double* M = vals + R[R_VAL];
  const int kmax = i < s ? i : s - 1;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int idx = i, step = s + m - 1;
  int k = 0;
  for (; k + 3 <= kmax; k += 4) {
    const int i1 = idx + step, i2 = i1 + step - 1, i3 = i2 + step - 2;
    a0 = fma(M[idx], f[k], a0);
    a1 = fma(M[i1], f[k + 1], a1);
    a2 = fma(M[i2], f[k + 2], a2);
    a3 = fma(M[i3], f[k + 3], a3);
    idx = i3 + step - 3;
    step -= 4;
  }
  for (; k <= kmax; ++k) {
    a0 = fma(M[idx], f[k], a0);
    idx += step;
    --step;
  }
  const double acc = (a0 + a1) + (a2 + a3);
  if (i < s)
    S[R[R_CPOS] + i] = acc;
  else
    f[i] -= acc;
}

// variant B: only the item decode + record loads + one FMA (no loops)
__device__ __forceinline__ void fwd_row_min(const int32_t* R, const double* vals, double* S, int i) {
  const int s = R[R_S], m = R[R_M];
  if (i >= s + m) return;
  double* f = S + R[R_SCR];
  const double* M = vals + R[R_VAL];
  const double acc = M[i] * f[0];
  if (i < s)
    S[R[R_CPOS] + i] = acc;
  else
    f[i] -= acc;
}

// variant C: straight-line path for s <= 4 (predicated loads, no loops)
__device__ __forceinline__ void fwd_row_tiny(const int32_t* R, const double* vals, double* S, int i) {
  const int s = R[R_S], m = R[R_M];
  if (i >= s + m) return;
  double* f = S + R[R_SCR];
  const double* M = vals + R[R_VAL];
  const int kmax = i < s ? i : s - 1;
  const int w = s + m;
  const double m0 = M[i], f0 = f[0];
  const double m1 = kmax >= 1 ? M[w + i - 1] : 0.0, f1 = kmax >= 1 ? f[1] : 0.0;
  const double m2 = kmax >= 2 ? M[2 * w - 1 + i - 2] : 0.0, f2 = kmax >= 2 ? f[2] : 0.0;
  const double m3 = kmax >= 3 ? M[3 * w - 3 + i - 3] : 0.0, f3 = kmax >= 3 ? f[3] : 0.0;
  const double acc = fma(m1, f1, m0 * f0) + fma(m3, f3, m2 * f2);
  if (i < s)
    S[R[R_CPOS] + i] = acc;
  else
    f[i] -= acc;
}

// variant D: branch-free store (select address), int4 record
__device__ __forceinline__ void fwd_row_tiny4(const int4 R, const double* vals, double* S, int i, bool on) {
  const int s = R.x & 0xffff, m = R.x >> 16;
  const int kmax = i < s ? i : s - 1;
  const int w = s + m;
  double* f = S + R.y;
  const double* M = vals + R.z;
  const bool ok = on && i < w;
  const double m0 = ok ? M[i] : 0.0, f0 = ok ? f[0] : 0.0;
  const double m1 = ok && kmax >= 1 ? M[w + i - 1] : 0.0, f1 = ok && kmax >= 1 ? f[1] : 0.0;
  const double fi = ok && i >= s ? f[i] : 0.0;
  const double acc = fma(m1, f1, m0 * f0);
  double* dst = i < s ? S + R.w + i : f + i;
  const double val = i < s ? acc : fi - acc;
  if (ok) *dst = val;
}

template <int V>
__global__ void k(long long* out, int reps) {
  extern __shared__ __align__(16) uint8_t smem[];
  int32_t* h = reinterpret_cast<int32_t*>(smem);
  const int lane = threadIdx.x & 31;
  // 6 supernodes s=1, m=4 packed in one item (30 lanes) + records
  int32_t* recs = h;
  double* vals = reinterpret_cast<double*>(smem + 1024);
  double* S = reinterpret_cast<double*>(smem + 4096);
  int2* items = reinterpret_cast<int2*>(smem + 512);
  if (lane < 6) {
    int32_t* R = recs + R_WORDS * lane;
    R[R_S] = 1;
    R[R_M] = 4;
    R[R_VAL] = 5 * lane;
    R[R_SCR] = 5 * lane;
    R[R_CPOS] = 200 + lane;
  }
  if (lane < 6) {
    int4* r4 = reinterpret_cast<int4*>(smem + 8192);
    r4[lane] = make_int4(1 | (4 << 16), 5 * lane, 5 * lane, 200 + lane);
  }
  if (lane == 0) {
    unsigned mask = 0;
    for (int j = 0; j < 6; ++j) mask |= 1u << (5 * j);
    mask |= 1u << 30;
    items[0] = make_int2(0 | (6 << 16), (int)mask);
  }
  for (int i = lane; i < 256; i += 32) {
    vals[i] = 1.0 + i * 1e-3;
    S[i] = 0.5 + i * 1e-3;
  }
  __syncwarp();
  long long best = 1ll << 60, sum = 0;
  for (int r = 0; r < reps; ++r) {
    __syncwarp();
    const long long t0 = clock64();
    const int2 item = items[r & 0];
    const int cnt = item.x >> 16;
    const unsigned upto = (unsigned)item.y & ((2u << lane) - 1u);
    const int seg = __popc(upto) - 1;
    if (seg < cnt) {
      if (V == 0) fwd_row(recs + R_WORDS * ((item.x & 0xffff) + seg), vals, S, lane - (31 - __clz(upto)));
      if (V == 1) fwd_row_min(recs + R_WORDS * ((item.x & 0xffff) + seg), vals, S, lane - (31 - __clz(upto)));
      if (V == 2) fwd_row_tiny(recs + R_WORDS * ((item.x & 0xffff) + seg), vals, S, lane - (31 - __clz(upto)));
    }
    if (V == 3) {
      const int4* r4 = reinterpret_cast<const int4*>(smem + 8192);
      const int4 R = r4[(item.x & 0xffff) + (seg < cnt ? seg : 0)];
      fwd_row_tiny4(R, vals, S, lane - (31 - __clz(upto)), seg < cnt);
    }
    __syncwarp();
    const long long dt = clock64() - t0;
    best = dt < best ? dt : best;
    sum += dt;
  }
  if (lane == 0) {
    out[2 * V] = best;
    out[2 * V + 1] = sum / reps;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (int w = 0; w < 2; ++w) {
    k<0><<<1, 32, 16384>>>(d, 100);
    k<1><<<1, 32, 16384>>>(d, 100);
    k<2><<<1, 32, 16384>>>(d, 100);
    k<3><<<1, 32, 16384>>>(d, 100);
  }
  cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
  printf("full fwd_row item: best %lld avg %lld cycles\n", h[0], h[1]);
  printf("minimal item:      best %lld avg %lld cycles\n", h[2], h[3]);
  printf("tiny straight:     best %lld avg %lld cycles\n", h[4], h[5]);
  printf("tiny int4 brfree:  best %lld avg %lld cycles\n", h[6], h[7]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
