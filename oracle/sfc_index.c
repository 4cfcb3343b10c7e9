/*
 * sfc_index.c -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the reference's index-set arithmetic for the sizes
 * where the Python oracle is too slow (BASELINE configs[4]: 16.6 M ... 133 M
 * points; SURVEY §8(c) "CPU restatement, needed only at C5 scale").  Used by
 * tests/ as the checker of the device permutation / partition / aggregates.
 * Citations are /root/reference/pkg/src/sfcdd/<file>:<line>.
 *
 *   hilbert_key      sfc.py:56-79 (_axes_to_transpose: Skilling's transform of
 *                    the axes to the transposed key), sfc.py:102-107
 *                    (_pack_transpose: key bits MSB first, axis 0 first),
 *                    sfc.py:120-136 (encode; d = 1 is the identity)
 *   grid point key   sfc.py:150-169 (1-based index k -> (k - 1) << (lmax - l_j))
 *   sfc_perm         grid.py:60-77 (C-order lex enumeration, last axis fastest;
 *                    perm = the lex indices sorted by key; keys are unique)
 *   partition        partition.py:64-75 (disjoint), 84-116 (enlarge with
 *                    exact rationals gamma = num / den, sums written the way
 *                    the reference writes them), 151-157 (weights)
 *   aggregates       coarse.py:21-24, 44-55 (q chunks per disjoint range)
 *
 * Only 64-bit keys (dim * lmax <= 64), which covers every BASELINE config
 * (<= 27 key bits); the generic 128-bit case is checked by the Python oracle.
 * Built by oracle/Makefile into oracle/_build/libsfcdd_oracle.so.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* sfc.py:56-79 then sfc.py:102-107 */
static uint64_t hilbert_key(int d, int bits, uint64_t* x) {
  if (d == 1) return x[0];
  const uint64_t m = (uint64_t)1 << (bits - 1);
  for (uint64_t q = m; q > 1; q >>= 1) {
    const uint64_t p = q - 1;
    for (int i = 0; i < d; ++i) {
      if (x[i] & q) {
        x[0] ^= p;
      } else {
        const uint64_t t = (x[0] ^ x[i]) & p;
        x[0] ^= t;
        x[i] ^= t;
      }
    }
  }
  for (int i = 1; i < d; ++i) x[i] ^= x[i - 1];
  uint64_t t = 0;
  for (uint64_t q = m; q > 1; q >>= 1)
    if (x[d - 1] & q) t ^= q - 1;
  for (int i = 0; i < d; ++i) x[i] ^= t;
  uint64_t key = 0;
  for (int level = bits - 1; level >= 0; --level)
    for (int i = 0; i < d; ++i) key = (key << 1) | ((x[i] >> level) & 1);
  return key;
}

int oracle_hilbert_keys(int d, int bits, const uint64_t* coords, int64_t n, uint64_t* keys) {
  if (d < 1 || d > 16 || bits < 1 || d * bits > 64) return -1;
  uint64_t x[16];
  for (int64_t i = 0; i < n; ++i) {
    memcpy(x, coords + i * d, sizeof(uint64_t) * d);
    keys[i] = hilbert_key(d, bits, x);
  }
  return 0;
}

/* grid.py:60-77 with the keys of sfc.py:150-169; LSD radix sort of
 * (key, lex index) pairs, 8-bit digits over the key bits in use */
int oracle_sfc_perm(int d, const int* levels, int64_t* perm) {
  if (d < 1 || d > 16) return -1;
  int lmax = 0;
  int64_t n = 1, shape[16];
  for (int j = 0; j < d; ++j) {
    if (levels[j] < 1 || levels[j] > 31) return -1;
    if (levels[j] > lmax) lmax = levels[j];
    shape[j] = ((int64_t)1 << levels[j]) - 1;
    n *= shape[j];
  }
  if (d * lmax > 64) return -2;
  if (d == 1) {
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    return 0;
  }
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* key2 = (uint64_t*)malloc(sizeof(uint64_t) * n);
  int64_t* idx2 = (int64_t*)malloc(sizeof(int64_t) * n);
  if (!key || !key2 || !idx2) {
    free(key);
    free(key2);
    free(idx2);
    return -3;
  }
  int64_t cnt[16] = {0}; /* odometer over the lex multi-index, last axis fastest */
  uint64_t x[16];
  for (int64_t i = 0; i < n; ++i) {
    for (int j = 0; j < d; ++j) x[j] = (uint64_t)cnt[j] << (lmax - levels[j]); /* (k-1) << (lmax-l_j) */
    key[i] = hilbert_key(d, lmax, x);
    perm[i] = i;
    for (int j = d - 1; j >= 0; --j) {
      if (++cnt[j] < shape[j]) break;
      cnt[j] = 0;
    }
  }
  const int kbits = d * lmax;
  uint64_t *ks = key, *kd = key2;
  int64_t *is = perm, *id = idx2;
  for (int sh = 0; sh < kbits; sh += 8) {
    int64_t c[257];
    memset(c, 0, sizeof c);
    for (int64_t i = 0; i < n; ++i) c[((ks[i] >> sh) & 255) + 1]++;
    for (int b = 0; b < 256; ++b) c[b + 1] += c[b];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t o = c[(ks[i] >> sh) & 255]++;
      kd[o] = ks[i];
      id[o] = is[i];
    }
    uint64_t* tk = ks;
    ks = kd;
    kd = tk;
    int64_t* ti = is;
    is = id;
    id = ti;
  }
  if (is != perm) memcpy(perm, is, sizeof(int64_t) * n);
  free(key);
  free(key2);
  free(idx2);
  return 0;
}

/* partition.py:64-75 and 84-116, exact rationals gamma = num / den */
int oracle_partition(int64_t n, int p, int64_t num, int64_t den, int64_t* dj_start, int64_t* dj_len,
                     int64_t* ov_start, int64_t* ov_len) {
  if (p < 1 || p > n || den < 1 || num < 0) return -1;
  const int64_t base = n / p, extra = n % p;
  int64_t st = 0;
  for (int i = 0; i < p; ++i) {
    dj_start[i] = st;
    dj_len[i] = i < extra ? base + 1 : base;
    st += dj_len[i];
  }
  if (num == 0) {
    memcpy(ov_start, dj_start, sizeof(int64_t) * p);
    memcpy(ov_len, dj_len, sizeof(int64_t) * p);
    return 0;
  }
  if (p < 2) return -1;
  if (2 * num + den > (int64_t)p * den) return -1;
  const int64_t whole = num / den, eta = num - whole * den; /* eta / den */
  for (int i = 0; i < p; ++i) {
    int64_t left = 0, right = 0;
    for (int64_t k = 1; k <= whole; ++k) {
      left += dj_len[((i - k) % p + p) % p];
      right += dj_len[(i + k) % p];
    }
    if (eta > 0) {
      const int64_t sl = dj_len[((i - whole - 1) % p + p) % p], sr = dj_len[(i + whole + 1) % p];
      left += (eta * sl + den - 1) / den; /* ceil(eta * size) */
      right += (eta * sr) / den;          /* floor(eta * size) */
    }
    ov_len[i] = dj_len[i] + left + right;
    ov_start[i] = ((dj_start[i] - left) % n + n) % n;
  }
  return 0;
}

/* partition.py:151-157: counts (n, nullable) and omega (p) */
int oracle_weights(int64_t n, int p, const int64_t* ov_start, const int64_t* ov_len, int32_t* counts_out,
                   double* omega) {
  int32_t* counts = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  if (!counts) return -3;
  for (int i = 0; i < p; ++i)
    for (int64_t r = 0; r < ov_len[i]; ++r) counts[(ov_start[i] + r) % n]++;
  for (int i = 0; i < p; ++i) {
    double mx = 0.0;
    for (int64_t r = 0; r < ov_len[i]; ++r) {
      const double v = 1.0 / (double)counts[(ov_start[i] + r) % n];
      if (v > mx) mx = v;
    }
    omega[i] = mx;
  }
  if (counts_out) memcpy(counts_out, counts, sizeof(int32_t) * n);
  free(counts);
  return 0;
}

/* coarse.py:21-24, 44-55: start of every aggregate (n0 + 1 entries) */
int oracle_aggregates(int p, const int64_t* dj_start, const int64_t* dj_len, int q, int64_t* bounds) {
  int64_t k = 0;
  bounds[0] = 0;
  for (int i = 0; i < p; ++i) {
    if (q < 1 || q > dj_len[i]) return -1;
    const int64_t base = dj_len[i] / q, extra = dj_len[i] % q;
    int64_t s = dj_start[i];
    for (int m = 0; m < q; ++m) {
      s += m < extra ? base + 1 : base;
      bounds[++k] = s;
    }
  }
  return 0;
}
