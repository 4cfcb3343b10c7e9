// Overlapping SFC partitions, computed by the library from (N, P, gamma).
//
// Replaces partition.disjoint_partition / enlarge / build_partition /
// compute_weights (partition.py:64-157).  Semantics pinned by the
// reference:
//   * P consecutive disjoint ranges, the first N mod P one longer;
//   * the overlapped range of subdomain i grows by floor(gamma) whole
//     neighbours on each side plus ceil(eta n_left) / floor(eta n_right)
//     points of the next ranges (eta = frac(gamma), exact rational arithmetic,
//     gamma = num/den after Fraction.limit_denominator(10**6) on the caller's
//     side), cyclically modulo N;
//   * counts[j] = number of overlapped ranges containing j, omega_i =
//     max_j 1/counts[j] over range i.
// Design: the whole-neighbour sums are differences of one cyclic prefix sum
// of the range sizes (O(P) for any gamma instead of O(P floor(gamma))); the
// cover counts are a cyclic difference array (O(N + P)); omega_i is
// 1/min(counts) over the range (IEEE division is monotone, so max(1/c) ==
// 1/min(c) exactly).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "common.h"
#include "host.h"

namespace sfcdd {

void partition_ranges(int64_t n, int32_t p, int64_t gnum, int64_t gden, std::vector<int64_t>& dj_start,
                      std::vector<int64_t>& dj_len, std::vector<int64_t>& ov_start, std::vector<int64_t>& ov_len) {
  SFCDD_REQUIRE(p >= 1 && (int64_t)p <= n, SFCDD_EVALUE,
                "need 1 <= P <= N, got P=" + std::to_string(p) + ", N=" + std::to_string(n));
  SFCDD_REQUIRE(gden >= 1, SFCDD_EVALUE, "gamma denominator must be positive");
  SFCDD_REQUIRE(gnum >= 0, SFCDD_EVALUE, "gamma must be nonnegative");
  const int64_t base = n / p, extra = n % p;
  dj_start.resize(p);
  dj_len.resize(p);
  int64_t s = 0;
  for (int32_t i = 0; i < p; ++i) {
    dj_start[i] = s;
    dj_len[i] = base + (i < extra ? 1 : 0);
    s += dj_len[i];
  }
  ov_start = dj_start;
  ov_len = dj_len;
  if (gnum == 0) return;
  SFCDD_REQUIRE(p >= 2, SFCDD_EVALUE, "overlap requires at least two subdomains");
  // 2 gamma + 1 > P  <=>  2 num + den > P den
  if ((__int128)2 * gnum + gden > (__int128)p * gden) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "2*gamma+1 = %g exceeds P = %d", (2.0 * gnum + gden) / gden, p);
    throw Error(SFCDD_EVALUE, buf);
  }
  const int64_t whole = gnum / gden, eta_num = gnum % gden;  // eta = eta_num / gden in [0, 1)
  // cyclic window sums of `whole` consecutive sizes: pre[k] = sum of sizes
  // [0, k) extended periodically over three periods (whole < P by the check above)
  std::vector<int64_t> pre(3 * (size_t)p + 1, 0);
  for (int64_t k = 0; k < 3 * (int64_t)p; ++k) pre[k + 1] = pre[k] + dj_len[k % p];
  for (int32_t i = 0; i < p; ++i) {
    // left neighbours i-whole .. i-1, right neighbours i+1 .. i+whole (mod P)
    const int64_t li = i + p;  // shift so indices stay nonnegative
    int64_t left = pre[li] - pre[li - whole];
    int64_t right = pre[li + 1 + whole] - pre[li + 1];
    if (eta_num > 0) {
      const int64_t nl = dj_len[(i - whole - 1 + 2 * (int64_t)p) % p];
      const int64_t nr = dj_len[(i + whole + 1) % p];
      const __int128 a = (__int128)eta_num * nl, b = (__int128)eta_num * nr;
      left += (int64_t)((a + gden - 1) / gden);  // ceil(eta * n_left)
      right += (int64_t)(b / gden);               // floor(eta * n_right)
    }
    const int64_t len = dj_len[i] + left + right;
    SFCDD_REQUIRE(len <= n, SFCDD_EINTERNAL, "overlapped range longer than N");
    ov_start[i] = ((dj_start[i] - left) % n + n) % n;
    ov_len[i] = len;
  }
}

void partition_weights(int64_t n, int32_t p, const int64_t* ov_start, const int64_t* ov_len, int32_t* counts,
                       double* omega) {
  std::vector<int32_t> diff((size_t)n + 1, 0);
  for (int32_t i = 0; i < p; ++i) {
    const int64_t s = ov_start[i], l = ov_len[i];
    SFCDD_REQUIRE(s >= 0 && s < n && l >= 0 && l <= n, SFCDD_EVALUE, "overlapped range out of bounds");
    if (l == 0) continue;
    const int64_t e = s + l;
    diff[s] += 1;
    if (e <= n) {
      diff[e] -= 1;
    } else {  // wraps: [s, n) and [0, e - n)
      diff[n] -= 1;
      diff[0] += 1;
      diff[e - n] -= 1;
    }
  }
  std::vector<int32_t> cnt((size_t)n);
  int32_t run = 0;
  for (int64_t j = 0; j < n; ++j) {
    run += diff[j];
    cnt[j] = run;
  }
  if (counts) std::copy(cnt.begin(), cnt.end(), counts);
  if (omega) {
    for (int32_t i = 0; i < p; ++i) {
      int32_t mn = INT32_MAX;
      for (int64_t r = 0; r < ov_len[i]; ++r) {
        int64_t g = ov_start[i] + r;
        if (g >= n) g -= n;
        mn = std::min(mn, cnt[g]);
      }
      omega[i] = ov_len[i] > 0 ? 1.0 / (double)mn : 0.0;
    }
  }
}

}  // namespace sfcdd

using namespace sfcdd;

extern "C" int sfcdd_partition(int64_t n, int32_t p, int64_t gamma_num, int64_t gamma_den, int64_t* dj_start,
                               int64_t* dj_len, int64_t* ov_start, int64_t* ov_len) {
  SFCDD_API_BEGIN
  std::vector<int64_t> ds, dl, os, ol;
  partition_ranges(n, p, gamma_num, gamma_den, ds, dl, os, ol);
  std::copy(ds.begin(), ds.end(), dj_start);
  std::copy(dl.begin(), dl.end(), dj_len);
  std::copy(os.begin(), os.end(), ov_start);
  std::copy(ol.begin(), ol.end(), ov_len);
  SFCDD_API_END
}

extern "C" int sfcdd_partition_weights(int64_t n, int32_t p, const int64_t* ov_start, const int64_t* ov_len,
                                       int32_t* counts, double* omega) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(n >= 1 && p >= 1, SFCDD_EVALUE, "need N >= 1 and P >= 1");
  partition_weights(n, p, ov_start, ov_len, counts, omega);
  SFCDD_API_END
}
