// SFC permutation entry point and the grid geometry shared by the
// permutation and stencil kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sfcdd {

constexpr int MAX_GRID_DIM = 16;

// Grid geometry for the permutation kernels (C-order lex enumeration,
// grid.py:72-75; embedding shift lmax - l_j, sfc.py:167-168).
enum Curve : int { CURVE_HILBERT = 0, CURVE_LEBESGUE = 1 };

struct GridGeom {
  int d;
  int lmax;
  int curve;  // Curve
  int64_t n;
  int64_t shape[MAX_GRID_DIM];
  int shift[MAX_GRID_DIM];
};

__device__ __forceinline__ void lex_to_lattice(const GridGeom& g, int64_t lex, uint32_t* x) {
  for (int j = g.d - 1; j >= 0; --j) {
    int64_t s = g.shape[j];
    int64_t c = lex % s;
    lex /= s;
    x[j] = (uint32_t)c << g.shift[j];
  }
}


// perm[s] = lex index of SFC rank s; rank = inverse (optional)
void sfc_perm_device(int d, const int32_t* levels, int64_t* perm, int64_t* rank, bool force_radix,
                     cudaStream_t st, int curve = CURVE_HILBERT);

}  // namespace sfcdd
