// Index-free stencil tiles over the SFC order (2-D and 3-D grids).
//
// Every aligned dyadic block of the Hilbert lattice is visited contiguously
// by the curve (sfc.py:56-107), so the interior points of a block are one
// contiguous SFC rank range.  A tile is such a block: its values are read
// coalesced, placed into a local lexicographic box in shared memory through a
// small rank->box table (deduplicated: blocks of equal orientation and shape
// share one table), and the (2d+1)-point stencil (grid.py:91-130) runs on the
// box; only the points across the tile faces are gathered through a halo rank
// list.  This replaces the 2d int32 neighbour indices per point that the
// stencil kernels otherwise read (16 MB per pass at C2).
#pragma once
#include <cstdint>
#include <vector>

namespace sfcdd {

constexpr int TILE_MAX_POINTS = 1024;  // points per tile (2-D 32x32, 3-D 8x8x8)

struct HostTiles {
  int d = 0;
  int32_t ntiles = 0;
  std::vector<int32_t> r0;        // ntiles + 1: rank range of each tile
  std::vector<int32_t> dims;      // ntiles * 3: box extent per axis (axis d-1 fastest; unused axes 1)
  std::vector<int32_t> tab_off;   // ntiles: offset of the tile's rank->box table in `tab`
  std::vector<uint16_t> tab;      // deduplicated tables: packed box coordinates of rank r0 + k
                                  // (2-D u0 | u1 << 8, 3-D u0 | u1 << 5 | u2 << 10)
  std::vector<int32_t> halo_off;  // ntiles + 1: offset of the tile's halo ranks
  std::vector<int32_t> halo;      // per tile, faces (axis 0 -, axis 0 +, axis 1 -, ...), each
                                  // in box-lex order of the other axes: SFC rank or -1 (outside)
  int32_t max_halo = 0;
};

// perm[s] = lex index of SFC rank s (grid.py:60-77); shape = interior points
// per axis; lshift[j] = lmax - l_j (anisotropic lattice embedding, sfc.py:150-169).
HostTiles build_tiles(int d, const int64_t* shape, const int* lshift, const std::vector<int64_t>& perm);

}  // namespace sfcdd
