// Hilbert space-filling-curve keys and the SFC permutation of grid points
// (plus the Lebesgue / Morton curve option: the same bit interleaving of the
// raw lattice coordinates, no Hilbert transform; north star subsystem (1) --
// the reference has no Lebesgue curve, so that option is checked against the
// oracle's restatement only).
//
// Restates the Skilling transpose-form curve of the reference
// (sfc.py:56-79 _axes_to_transpose, sfc.py:81-99 _transpose_to_axes,
// sfc.py:102-117 pack/unpack) as per-point device code, and replaces the
// Python loop + sorted() of grid.sfc_permutation (grid.py:60-77) by
//   (a) dense key space  (2^(d*lmax) <= 16 N): bitmap of occupied keys +
//       popcount prefix scan -> rank(key) = #occupied keys below it;
//   (b) general case: LSD radix sort of (key, lex index), 8-bit digits.
// Keys are unique, so both give the reference's order bit-exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.h"
#include "scan.cuh"
#include "sfc.h"

namespace sfcdd {

constexpr int MAX_DIM = 64;  // encode/decode batch API (d*bits <= 128)


struct Key128 {
  uint64_t hi, lo;
};

// axes -> transpose (sfc.py:56-79); W = word type
template <typename W>
__device__ __forceinline__ void axes_to_transpose(W* x, int d, int bits) {
  const W m = W(1) << (bits - 1);
  for (W q = m; q > 1; q >>= 1) {
    const W p = q - 1;
    for (int i = 0; i < d; ++i) {
      if (x[i] & q) {
        x[0] ^= p;
      } else {
        W t = (x[0] ^ x[i]) & p;
        x[0] ^= t;
        x[i] ^= t;
      }
    }
  }
  for (int i = 1; i < d; ++i) x[i] ^= x[i - 1];
  W t = 0;
  for (W q = m; q > 1; q >>= 1)
    if (x[d - 1] & q) t ^= q - 1;
  for (int i = 0; i < d; ++i) x[i] ^= t;
}

// transpose -> axes (sfc.py:81-99)
template <typename W>
__device__ __forceinline__ void transpose_to_axes(W* x, int d, int bits) {
  W t = x[d - 1] >> 1;
  for (int i = d - 1; i > 0; --i) x[i] ^= x[i - 1];
  x[0] ^= t;
  for (int lv = 1; lv < bits; ++lv) {
    const W q = W(1) << lv;
    const W p = q - 1;
    for (int i = d - 1; i >= 0; --i) {
      if (x[i] & q) {
        x[0] ^= p;
      } else {
        W tt = (x[0] ^ x[i]) & p;
        x[0] ^= tt;
        x[i] ^= tt;
      }
    }
  }
}

// interleave MSB-first, axis 0 first (sfc.py:102-107): bit (level, i) lands
// at key position level*d + d-1-i.
template <typename W>
__device__ __forceinline__ Key128 pack_transpose(const W* x, int d, int bits) {
  Key128 k{0, 0};
  for (int level = 0; level < bits; ++level) {
    for (int i = 0; i < d; ++i) {
      uint64_t bit = (uint64_t)((x[i] >> level) & 1);
      int pos = level * d + (d - 1 - i);
      if (pos < 64)
        k.lo |= bit << pos;
      else
        k.hi |= bit << (pos - 64);
    }
  }
  return k;
}

// 64-bit key fast path for d*bits <= 64
template <typename W>
__device__ __forceinline__ uint64_t pack_transpose64(const W* x, int d, int bits) {
  uint64_t k = 0;
  for (int level = bits - 1; level >= 0; --level)
    for (int i = 0; i < d; ++i) k = (k << 1) | (uint64_t)((x[i] >> level) & 1);
  return k;
}

__global__ void k_encode(int d, int bits, int curve, const uint64_t* __restrict__ coords, int64_t n,
                         uint64_t* __restrict__ hi, uint64_t* __restrict__ lo) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t x[MAX_DIM];
  for (int j = 0; j < d; ++j) x[j] = coords[i * d + j];
  if (d == 1) {
    hi[i] = 0;
    lo[i] = x[0];
    return;
  }
  if (curve == CURVE_HILBERT) axes_to_transpose(x, d, bits);
  Key128 k = pack_transpose(x, d, bits);
  hi[i] = k.hi;
  lo[i] = k.lo;
}

__global__ void k_decode(int d, int bits, int curve, const uint64_t* __restrict__ hi,
                         const uint64_t* __restrict__ lo, int64_t n, uint64_t* __restrict__ coords) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t x[MAX_DIM];
  if (d == 1) {
    coords[i] = lo[i];
    return;
  }
  for (int j = 0; j < d; ++j) x[j] = 0;
  const uint64_t H = hi[i], L = lo[i];
  for (int level = 0; level < bits; ++level) {
    int base = level * d + d - 1;  // sfc.py:110-117
    for (int j = 0; j < d; ++j) {
      int pos = base - j;
      uint64_t bit = pos < 64 ? (L >> pos) & 1 : (H >> (pos - 64)) & 1;
      if (bit) x[j] |= uint64_t(1) << level;
    }
  }
  if (curve == CURVE_HILBERT) transpose_to_axes(x, d, bits);
  for (int j = 0; j < d; ++j) coords[i * d + j] = x[j];
}

__device__ __forceinline__ Key128 grid_key(const GridGeom& g, int64_t lex) {
  uint32_t x[MAX_GRID_DIM];
  lex_to_lattice(g, lex, x);
  if (g.d == 1) return Key128{0, x[0]};  // grid.py:69-70: identity order
  if (g.curve == CURVE_HILBERT) axes_to_transpose(x, g.d, g.lmax);
  if (g.d * g.lmax <= 64) return Key128{0, pack_transpose64(x, g.d, g.lmax)};
  return pack_transpose(x, g.d, g.lmax);
}

// ---- dense key-space path -------------------------------------------------
__global__ void k_mark(GridGeom g, uint32_t* __restrict__ bitmap) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  uint64_t key = grid_key(g, i).lo;
  atomicOr(&bitmap[key >> 5], 1u << (key & 31));
}

struct PopcIn {
  const uint32_t* bm;
  __device__ int64_t operator()(int64_t i) const { return __popc(bm[i]); }
};
struct StoreOut {
  int64_t* out;
  __device__ void operator()(int64_t i, int64_t v) const { out[i] = v; }
};

__global__ void k_rank_scatter(GridGeom g, const uint32_t* __restrict__ bitmap,
                               const int64_t* __restrict__ word_prefix, int64_t* __restrict__ perm,
                               int64_t* __restrict__ rank) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  uint64_t key = grid_key(g, i).lo;
  uint64_t w = key >> 5;
  uint32_t below = bitmap[w] & ((1u << (key & 31)) - 1u);
  int64_t r = word_prefix[w] + __popc(below);
  perm[r] = i;
  if (rank) rank[i] = r;
}

// ---- general path: LSD radix sort of (key, lex) -------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void k_keys(GridGeom g, uint64_t* __restrict__ hi, uint64_t* __restrict__ lo,
                       int64_t* __restrict__ val) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  Key128 k = grid_key(g, i);
  hi[i] = k.hi;
  lo[i] = k.lo;
  val[i] = i;
}

__device__ __forceinline__ uint32_t digit_of(uint64_t hi, uint64_t lo, int shift) {
  return shift < 64 ? (uint32_t)((lo >> shift) & 0xff) : (uint32_t)((hi >> (shift - 64)) & 0xff);
}

// counts layout: [digit][tile] so that one exclusive scan gives stable offsets
__global__ void k_rs_hist(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo, int64_t n,
                          int shift, int64_t ntiles, int64_t* __restrict__ counts) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int k = 0; k < RS_ITEMS; ++k) {
    int64_t i = base + (int64_t)k * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[digit_of(hi[i], lo[i], shift)], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// stable scatter: items of a tile are ranked in index order within each digit
__global__ void k_rs_scatter(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo,
                             const int64_t* __restrict__ val, int64_t n, int shift, int64_t ntiles,
                             const int64_t* __restrict__ offsets, uint64_t* __restrict__ ohi,
                             uint64_t* __restrict__ olo, int64_t* __restrict__ oval) {
  __shared__ int64_t run[256];
  __shared__ uint32_t wcnt[RS_THREADS / 32][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  run[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int k = 0; k < RS_ITEMS; ++k) {
    for (int w = 0; w < RS_THREADS / 32; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    int64_t i = base + (int64_t)k * RS_THREADS + threadIdx.x;
    bool valid = i < n;
    uint32_t dg = valid ? digit_of(hi[i], lo[i], shift) : 0xffffffffu;
    unsigned peers = __match_any_sync(0xffffffffu, dg);
    unsigned lt = (1u << lane) - 1u;
    uint32_t within = __popc(peers & lt);
    if (valid && within == 0) wcnt[warp][dg] = __popc(peers);
    __syncthreads();
    // per digit: prefix over warps (thread = digit)
    {
      uint32_t acc = 0;
      for (int w = 0; w < RS_THREADS / 32; ++w) {
        uint32_t c = wcnt[w][threadIdx.x];
        wcnt[w][threadIdx.x] = acc;
        acc += c;
      }
      __syncthreads();
      if (valid) {
        int64_t dst = run[dg] + wcnt[warp][dg] + within;
        ohi[dst] = hi[i];
        olo[dst] = lo[i];
        oval[dst] = val[i];
      }
      __syncthreads();
      run[threadIdx.x] += acc;
    }
    __syncthreads();
  }
}

struct Copy64 {
  const int64_t* in;
  __device__ int64_t operator()(int64_t i) const { return in[i]; }
};

__global__ void k_perm_from_sorted(const int64_t* __restrict__ val, int64_t n, int64_t* __restrict__ perm,
                                   int64_t* __restrict__ rank) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int64_t lex = val[s];
  perm[s] = lex;
  if (rank) rank[lex] = s;
}

template <typename T>
static void exclusive_scan(const T* in_dev, T* out_dev, int64_t n, T* total_dev, cudaStream_t st,
                           T* scratch /* >= ntiles */) {
  int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  Copy64 in{in_dev};
  scan_tile_sums<int64_t><<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(in, n, scratch);
  scan_tile_offsets<int64_t><<<1, SCAN_THREADS, 0, st>>>(scratch, ntiles, total_dev);
  StoreOut out{out_dev};
  scan_tiles<int64_t><<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(in, out, n, scratch);
}

static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

void sfc_perm_device(int d, const int32_t* levels, int64_t* perm, int64_t* rank, bool force_radix,
                     cudaStream_t st, int curve) {
  SFCDD_REQUIRE(d >= 1 && d <= MAX_GRID_DIM, SFCDD_EVALUE, "grid dimension must be in [1, 16]");
  SFCDD_REQUIRE(curve == CURVE_HILBERT || curve == CURVE_LEBESGUE, SFCDD_EVALUE, "unknown curve");
  GridGeom g{};
  g.d = d;
  g.curve = curve;
  g.lmax = 0;
  g.n = 1;
  for (int j = 0; j < d; ++j) {
    SFCDD_REQUIRE(levels[j] >= 1, SFCDD_EVALUE, "level vector must have positive entries");
    SFCDD_REQUIRE(levels[j] <= 32, SFCDD_EVALUE, "levels above 32 are not supported on device");
    g.lmax = std::max(g.lmax, (int)levels[j]);
  }
  for (int j = 0; j < d; ++j) {
    g.shape[j] = ((int64_t)1 << levels[j]) - 1;
    g.shift[j] = g.lmax - levels[j];
    SFCDD_REQUIRE(g.n <= ((int64_t)1 << 62) / g.shape[j], SFCDD_EOVERFLOW, "dof count exceeds 2^62");
    g.n *= g.shape[j];
  }
  SFCDD_REQUIRE(d * g.lmax <= 128, SFCDD_EVALUE, "key width exceeds 128 bits");
  const int64_t n = g.n;
  const int keybits = d * g.lmax;
  const bool dense = !force_radix && d > 1 && keybits <= 34 && ((int64_t)1 << keybits) <= 16 * n + 4096;
  if (d == 1 || dense) {
    const int kb = d == 1 ? g.lmax : keybits;
    const int64_t words = (((int64_t)1 << kb) + 31) / 32;
    const int64_t ntiles = (words + SCAN_TILE - 1) / SCAN_TILE;
    uint32_t* bitmap = nullptr;
    int64_t* prefix = nullptr;
    int64_t* scratch = nullptr;
    CUDA_CHECK(cudaMallocAsync(&bitmap, words * sizeof(uint32_t), st));
    CUDA_CHECK(cudaMallocAsync(&prefix, words * sizeof(int64_t), st));
    CUDA_CHECK(cudaMallocAsync(&scratch, (ntiles + 1) * sizeof(int64_t), st));
    CUDA_CHECK(cudaMemsetAsync(bitmap, 0, words * sizeof(uint32_t), st));
    k_mark<<<blocks_for(n, 256), 256, 0, st>>>(g, bitmap);
    PopcIn in{bitmap};
    scan_tile_sums<int64_t><<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(in, words, scratch);
    scan_tile_offsets<int64_t><<<1, SCAN_THREADS, 0, st>>>(scratch, ntiles, scratch + ntiles);
    StoreOut out{prefix};
    scan_tiles<int64_t><<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(in, out, words, scratch);
    k_rank_scatter<<<blocks_for(n, 256), 256, 0, st>>>(g, bitmap, prefix, perm, rank);
    CUDA_CHECK(cudaFreeAsync(bitmap, st));
    CUDA_CHECK(cudaFreeAsync(prefix, st));
    CUDA_CHECK(cudaFreeAsync(scratch, st));
    CUDA_CHECK(cudaGetLastError());
    return;
  }
  // general radix path
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int64_t ncount = 256 * ntiles;
  const int64_t nst = (ncount + SCAN_TILE - 1) / SCAN_TILE;
  uint64_t *hi[2], *lo[2];
  int64_t* val[2];
  int64_t *counts, *offs, *scratch;
  for (int b = 0; b < 2; ++b) {
    CUDA_CHECK(cudaMallocAsync(&hi[b], n * 8, st));
    CUDA_CHECK(cudaMallocAsync(&lo[b], n * 8, st));
    CUDA_CHECK(cudaMallocAsync(&val[b], n * 8, st));
  }
  CUDA_CHECK(cudaMallocAsync(&counts, ncount * 8, st));
  CUDA_CHECK(cudaMallocAsync(&offs, ncount * 8, st));
  CUDA_CHECK(cudaMallocAsync(&scratch, (nst + 1) * 8, st));
  k_keys<<<blocks_for(n, 256), 256, 0, st>>>(g, hi[0], lo[0], val[0]);
  int cur = 0;
  for (int shift = 0; shift < keybits; shift += 8) {
    k_rs_hist<<<(unsigned)ntiles, RS_THREADS, 0, st>>>(hi[cur], lo[cur], n, shift, ntiles, counts);
    exclusive_scan<int64_t>(counts, offs, ncount, scratch + nst, st, scratch);
    k_rs_scatter<<<(unsigned)ntiles, RS_THREADS, 0, st>>>(hi[cur], lo[cur], val[cur], n, shift, ntiles,
                                                          offs, hi[1 - cur], lo[1 - cur], val[1 - cur]);
    cur = 1 - cur;
  }
  k_perm_from_sorted<<<blocks_for(n, 256), 256, 0, st>>>(val[cur], n, perm, rank);
  for (int b = 0; b < 2; ++b) {
    CUDA_CHECK(cudaFreeAsync(hi[b], st));
    CUDA_CHECK(cudaFreeAsync(lo[b], st));
    CUDA_CHECK(cudaFreeAsync(val[b], st));
  }
  CUDA_CHECK(cudaFreeAsync(counts, st));
  CUDA_CHECK(cudaFreeAsync(offs, st));
  CUDA_CHECK(cudaFreeAsync(scratch, st));
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace sfcdd

using namespace sfcdd;

extern "C" int sfcdd_sfc_encode_curve(int curve, int dim, int bits, const uint64_t* coords_dev, int64_t n,
                                      uint64_t* keys_hi_dev, uint64_t* keys_lo_dev, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(curve == CURVE_HILBERT || curve == CURVE_LEBESGUE, SFCDD_EVALUE, "unknown curve");
  SFCDD_REQUIRE(dim >= 1 && dim <= MAX_DIM, SFCDD_EVALUE, "dimension must be in [1, 64]");
  SFCDD_REQUIRE(bits >= 1 && bits <= 64 && dim * bits <= 128, SFCDD_EVALUE, "invalid curve refinement");
  if (n <= 0) return SFCDD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  k_encode<<<blocks_for(n, 128), 128, 0, st>>>(dim, bits, curve, coords_dev, n, keys_hi_dev, keys_lo_dev);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_sfc_decode_curve(int curve, int dim, int bits, const uint64_t* keys_hi_dev,
                                      const uint64_t* keys_lo_dev, int64_t n, uint64_t* coords_dev, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(curve == CURVE_HILBERT || curve == CURVE_LEBESGUE, SFCDD_EVALUE, "unknown curve");
  SFCDD_REQUIRE(dim >= 1 && dim <= MAX_DIM, SFCDD_EVALUE, "dimension must be in [1, 64]");
  SFCDD_REQUIRE(bits >= 1 && bits <= 64 && dim * bits <= 128, SFCDD_EVALUE, "invalid curve refinement");
  if (n <= 0) return SFCDD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  k_decode<<<blocks_for(n, 128), 128, 0, st>>>(dim, bits, curve, keys_hi_dev, keys_lo_dev, n, coords_dev);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_sfc_perm_curve(int curve, int dim, const int32_t* levels_host, int64_t* perm_dev,
                                    int64_t* rank_dev, int force_radix, void* stream) {
  SFCDD_API_BEGIN
  sfc_perm_device(dim, levels_host, perm_dev, rank_dev, force_radix != 0, (cudaStream_t)stream, curve);
  SFCDD_API_END
}

extern "C" int sfcdd_sfc_encode(int dim, int bits, const uint64_t* coords_dev, int64_t n, uint64_t* keys_hi_dev,
                                uint64_t* keys_lo_dev, void* stream) {
  return sfcdd_sfc_encode_curve(CURVE_HILBERT, dim, bits, coords_dev, n, keys_hi_dev, keys_lo_dev, stream);
}

extern "C" int sfcdd_sfc_decode(int dim, int bits, const uint64_t* keys_hi_dev, const uint64_t* keys_lo_dev,
                                int64_t n, uint64_t* coords_dev, void* stream) {
  return sfcdd_sfc_decode_curve(CURVE_HILBERT, dim, bits, keys_hi_dev, keys_lo_dev, n, coords_dev, stream);
}

extern "C" int sfcdd_sfc_perm(int dim, const int32_t* levels_host, int64_t* perm_dev, int64_t* rank_dev,
                              int force_radix, void* stream) {
  return sfcdd_sfc_perm_curve(CURVE_HILBERT, dim, levels_host, perm_dev, rank_dev, force_radix, stream);
}
