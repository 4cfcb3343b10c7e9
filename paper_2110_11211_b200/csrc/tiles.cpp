// Host construction of the SFC stencil tiles (tiles.h).
#include "tiles.h"

#include <algorithm>
#include <map>

#include "common.h"

namespace sfcdd {

HostTiles build_tiles(int d, const int64_t* shape, const int* lshift, const std::vector<int64_t>& perm) {
  SFCDD_REQUIRE(d == 2 || d == 3, SFCDD_EINTERNAL, "stencil tiles need a 2-D or 3-D grid");
  const int64_t n = (int64_t)perm.size();
  // block edge 2^b lattice cells: the largest with at most `cap` points, where
  // cap keeps >= ~4 tiles per SM of a B200 (148 SMs) and <= TILE_MAX_POINTS
  const int64_t cap = std::min<int64_t>(TILE_MAX_POINTS, std::max<int64_t>(512, n / (4 * 148)));
  auto pts = [&](int b) {
    int64_t p = 1;
    for (int j = 0; j < d; ++j) p *= b >= lshift[j] ? ((int64_t)1 << (b - lshift[j])) : 1;
    return p;
  };
  int b = 1;
  while (b < 30 && pts(b + 1) <= cap) ++b;
  {
    int lmax = 0;
    for (int j = 0; j < d; ++j) lmax = std::max<int>(lmax, (int)(64 - __builtin_clzll((uint64_t)shape[j] + 1)) - 1);
    SFCDD_REQUIRE(lmax - b <= 21, SFCDD_EINTERNAL, "grid too large for the tile block ids");
  }
  HostTiles T;
  T.d = d;
  std::vector<int64_t> stride(d);
  {
    int64_t s = 1;
    for (int j = d - 1; j >= 0; --j) {
      stride[j] = s;
      s *= shape[j];
    }
  }
  auto coords = [&](int64_t lex, int64_t* c) {
    for (int j = d - 1; j >= 0; --j) {
      c[j] = lex % shape[j];
      lex /= shape[j];
    }
  };
  // block id: per-axis block coordinates packed in 21 bits each (lmax - b <= 21)
  auto block_of = [&](const int64_t* c) {
    int64_t id = 0;
    for (int j = 0; j < d; ++j) id = (id << 21) | ((c[j] << lshift[j]) >> b);
    return id;
  };
  std::vector<int32_t> rank(n);
  for (int64_t s = 0; s < n; ++s) rank[perm[s]] = (int32_t)s;
  std::map<std::vector<int32_t>, int32_t> pool;  // dims + table -> offset
  std::vector<int64_t> seen_blocks;
  int64_t c[3], lo[3], hi[3];
  int64_t s0 = 0;
  while (s0 < n) {
    coords(perm[s0], c);
    const int64_t blk = block_of(c);
    int64_t s1 = s0;
    for (int j = 0; j < d; ++j) lo[j] = hi[j] = c[j];
    while (s1 < n) {
      int64_t cc[3];
      coords(perm[s1], cc);
      if (block_of(cc) != blk) break;
      for (int j = 0; j < d; ++j) {
        lo[j] = std::min(lo[j], cc[j]);
        hi[j] = std::max(hi[j], cc[j]);
      }
      ++s1;
    }
    seen_blocks.push_back(blk);
    const int64_t np = s1 - s0;
    int64_t box = 1;
    int32_t dm[3] = {1, 1, 1};
    for (int j = 0; j < d; ++j) {
      dm[j] = (int32_t)(hi[j] - lo[j] + 1);
      box *= dm[j];
    }
    SFCDD_REQUIRE(box == np && np <= TILE_MAX_POINTS, SFCDD_EINTERNAL,
                  "SFC block is not a full box of interior points");
    // rank -> packed box coordinates (2-D: u0 | u1 << 8; 3-D: 5 bits per axis)
    SFCDD_REQUIRE(d == 2 ? (dm[0] <= 256 && dm[1] <= 256) : (dm[0] <= 32 && dm[1] <= 32 && dm[2] <= 32),
                  SFCDD_EINTERNAL, "tile box too large for the packed table");
    std::vector<int32_t> key(dm, dm + 3);
    for (int64_t s = s0; s < s1; ++s) {
      int64_t cc[3];
      coords(perm[s], cc);
      int32_t e = 0;
      for (int j = 0; j < d; ++j) e |= (int32_t)(cc[j] - lo[j]) << (j * (d == 2 ? 8 : 5));
      key.push_back(e);
    }
    auto it = pool.find(key);
    int32_t off;
    if (it == pool.end()) {
      off = (int32_t)T.tab.size();
      for (size_t k = 3; k < key.size(); ++k) T.tab.push_back((uint16_t)key[k]);
      pool.emplace(std::move(key), off);
    } else {
      off = it->second;
    }
    T.r0.push_back((int32_t)s0);
    T.dims.insert(T.dims.end(), dm, dm + 3);
    T.tab_off.push_back(off);
    // halo: faces in box-lex order of the other axes
    T.halo_off.push_back((int32_t)T.halo.size());
    for (int j = 0; j < d; ++j)
      for (int side = 0; side < 2; ++side) {
        const int64_t cj = side == 0 ? lo[j] - 1 : hi[j] + 1;
        int64_t u[3] = {0, 0, 0};
        int64_t cnt = 1;
        for (int a = 0; a < d; ++a)
          if (a != j) cnt *= dm[a];
        for (int64_t f = 0; f < cnt; ++f) {
          // decompose f over the other axes (last fastest)
          int64_t r = f;
          for (int a = d - 1; a >= 0; --a) {
            if (a == j) continue;
            u[a] = r % dm[a];
            r /= dm[a];
          }
          if (cj < 0 || cj >= shape[j]) {
            T.halo.push_back(-1);
            continue;
          }
          int64_t lex = 0;
          for (int a = 0; a < d; ++a) lex += (a == j ? cj : lo[a] + u[a]) * stride[a];
          T.halo.push_back(rank[lex]);
        }
      }
    T.max_halo = std::max<int32_t>(T.max_halo, (int32_t)(T.halo.size() - T.halo_off.back()));
    s0 = s1;
  }
  T.ntiles = (int32_t)T.tab_off.size();
  T.r0.push_back((int32_t)n);
  T.halo_off.push_back((int32_t)T.halo.size());
  std::sort(seen_blocks.begin(), seen_blocks.end());
  SFCDD_REQUIRE(std::adjacent_find(seen_blocks.begin(), seen_blocks.end()) == seen_blocks.end(), SFCDD_EINTERNAL,
                "an SFC block is visited twice");
  return T;
}

}  // namespace sfcdd
