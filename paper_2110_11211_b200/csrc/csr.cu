// General sparse matrix on the device: y = A x for CSR input.
//
// The reference's solvers are duck-typed over `A @ v` (krylov.py:257-291,
// linalg.py:31-34) and its tests run PCG on scipy CSR matrices that are not
// grid Laplacians (test_krylov.py:154-166).  This is the device product for
// those: one thread per row, summed in stored column order with separate
// multiply and add roundings -- scipy's csr_matvec order (sparsetools
// csr.h: sum += Ax[jj] * Xx[Aj[jj]]), so results match it bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "common.h"

struct sfcdd_csr {
  int device = 0;
  int64_t rows = 0, cols = 0, nnz = 0;
  int64_t* indptr = nullptr;
  int32_t* indices = nullptr;
  double* data = nullptr;
};

namespace {

__global__ void k_csr_matvec(int64_t rows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                             const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int64_t e = ptr[r + 1];
    for (int64_t k = ptr[r]; k < e; ++k) acc = __dadd_rn(acc, __dmul_rn(val[k], x[idx[k]]));
    y[r] = acc;
  }
}

}  // namespace

using namespace sfcdd;

extern "C" int sfcdd_csr_create(int64_t rows, int64_t cols, const int64_t* indptr, const int32_t* indices,
                                const double* data, int32_t device, sfcdd_csr** out) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(rows >= 0 && cols >= 0 && out && indptr, SFCDD_EVALUE, "invalid CSR arguments");
  const int64_t nnz = indptr[rows];
  SFCDD_REQUIRE(nnz >= 0 && indptr[0] == 0, SFCDD_EVALUE, "invalid CSR row pointer");
  for (int64_t k = 0; k < nnz; ++k)
    SFCDD_REQUIRE(indices[k] >= 0 && indices[k] < cols, SFCDD_EVALUE, "column index out of range");
  CUDA_CHECK(cudaSetDevice(device));
  sfcdd_csr* m = new sfcdd_csr();
  m->device = device;
  m->rows = rows;
  m->cols = cols;
  m->nnz = nnz;
  try {
    CUDA_CHECK(cudaMalloc(&m->indptr, (rows + 1) * 8));
    CUDA_CHECK(cudaMalloc(&m->indices, std::max<int64_t>(nnz, 1) * 4));
    CUDA_CHECK(cudaMalloc(&m->data, std::max<int64_t>(nnz, 1) * 8));
    CUDA_CHECK(cudaMemcpy(m->indptr, indptr, (rows + 1) * 8, cudaMemcpyHostToDevice));
    if (nnz) {
      CUDA_CHECK(cudaMemcpy(m->indices, indices, nnz * 4, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(m->data, data, nnz * 8, cudaMemcpyHostToDevice));
    }
  } catch (...) {
    cudaFree(m->indptr);
    cudaFree(m->indices);
    cudaFree(m->data);
    delete m;
    throw;
  }
  *out = m;
  SFCDD_API_END
}

extern "C" int sfcdd_csr_matvec(sfcdd_csr* m, const double* x_dev, double* y_dev, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(m, SFCDD_EVALUE, "null handle");
  CUDA_CHECK(cudaSetDevice(m->device));
  if (m->rows == 0) return SFCDD_OK;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((m->rows + threads - 1) / threads, 148 * 32);
  k_csr_matvec<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(m->rows, m->indptr, m->indices, m->data,
                                                                       x_dev, y_dev);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" void sfcdd_csr_destroy(sfcdd_csr* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  cudaFree(m->indptr);
  cudaFree(m->indices);
  cudaFree(m->data);
  delete m;
}
