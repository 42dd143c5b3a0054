// Tile schedule shared by the 1-SM and 2-SM K1 kernels (ffn_swiglu*.cu).
#pragma once

#include <cstdint>

namespace bfgpu {
namespace ffn {

enum Mode : int { kFused = 0, kGateUpOnly = 1, kDownOnly = 2 };

struct Params {
  int M, D, F, N;
  int Mt, Ft, Nt;  // m-units (128 rows 1-SM, 256 rows 2-SM), f-chunks of 128, n-chunks of 256
  int group;
  int mode;
  int num_tiles;
  int kt_d, kt_f;  // k-steps of 64 over D and over F
  float inv_d;
  float eps;
  int* flags;      // per m-tile count of finished gate/up tiles (fused mode)
  int* wave;       // 2-SM kernel: tile iterations started, summed over clusters (wave sync), or null
  int* seg;        // 2-SM fused kernel: tiles of the first two gate/up segments started (segment sync), or null
  int seg_tiles;   // ... their count: tiles [0, seg_tiles) of the fused order
  int braster;     // down-projection tiles: m-units per raster block (0: m fastest over the whole group)
};

struct Tile {
  int kind;  // 0 gate/up, 1 down
  int m;     // m-tile
  int j;     // f-chunk (kind 0) or n-chunk (kind 1)
};

__device__ __forceinline__ int group_size(const Params& p, int g) { return min(p.group, p.Mt - g * p.group); }

// Linear tile index -> tile. Segments: fused  A0 A1 B0 A2 B1 ... A(G-1) B(G-2) B(G-1)
//                                      gate/up-only A0 A1 ...; down-only B0 B1 ...
__device__ __forceinline__ Tile decode_tile(const Params& p, int t) {
  const int ngroups = (p.Mt + p.group - 1) / p.group;
  const int nseg = p.mode == kFused ? 2 * ngroups : ngroups;
  for (int s = 0; s < nseg; ++s) {
    int kind, g;
    if (p.mode == kGateUpOnly) {
      kind = 0;
      g = s;
    } else if (p.mode == kDownOnly) {
      kind = 1;
      g = s;
    } else if (s == 0) {
      kind = 0;
      g = 0;
    } else if (s == nseg - 1) {
      kind = 1;
      g = ngroups - 1;
    } else {
      kind = (s & 1) ? 0 : 1;
      g = (s & 1) ? (s + 1) / 2 : s / 2 - 1;
    }
    const int gs = group_size(p, g);
    const int cnt = gs * (kind == 0 ? p.Ft : p.Nt);
    if (t < cnt) {
      if (kind == 1 && p.braster > 0 && gs > p.braster) {
        // blocks of braster m-units, n-chunks in order, m fastest inside a block: a wave of
        // down tiles then reads H for braster m-units and Ut for a few n-chunks, instead of
        // H for the whole group
        for (int mb = 0;; mb += p.braster) {
          const int bsz = min(p.braster, gs - mb);
          if (t < bsz * p.Nt) return Tile{1, g * p.group + mb + t % bsz, t / bsz};
          t -= bsz * p.Nt;
        }
      }
      return Tile{kind, g * p.group + t % gs, t / gs};
    }
    t -= cnt;
  }
  return Tile{-1, 0, 0};
}

}  // namespace ffn
}  // namespace bfgpu
