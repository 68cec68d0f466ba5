// phj_common.cuh -- shared device helpers for the sm_100a patchy SL engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/phj.h"

namespace phj {

#ifndef PHJ_CTA_WARPS
#define PHJ_CTA_WARPS 8
#endif
#ifndef PHJ_NB2D
#define PHJ_NB2D 2
#endif
constexpr int kThreads = 32 * PHJ_CTA_WARPS;
constexpr int kWarps = kThreads / 32;
constexpr int kCtasPerSm = 16 / PHJ_CTA_WARPS;  // 16 resident warps per SM
constexpr int kMaxPatches = 1024;
constexpr int kSmemPatchReduce = 64;  // per-CTA patch max reduction when R <= 64

// Work/activity unit = one warp "block" of nodes: LY rows x (LX lanes * NB
// consecutive nodes) along the fastest internal axis, one plane of internal
// axis 0 in 3D (so the stencil class -- internal axis 0 -- is warp-uniform).
// Each lane keeps its NB nodes' 3^D neighbourhood in registers.
template <int D> struct Blk;
#ifndef PHJ_LX2D
#define PHJ_LX2D 8
#endif
#ifndef PHJ_NB3D
#define PHJ_NB3D 2
#endif
#ifndef PHJ_LX3D
#define PHJ_LX3D 4
#endif
template <> struct Blk<2> {
  static constexpr int NB = PHJ_NB2D, LX = PHJ_LX2D, LY = 32 / LX, BX = LX * NB, BY = LY;
};
template <> struct Blk<3> {
  static constexpr int NB = PHJ_NB3D, LX = PHJ_LX3D, LY = 32 / LX, BX = LX * NB, BY = LY;
};

struct TileGrid {
  int n[3];  // blocks per internal axis (axis 0 slowest)
  int total;
};

template <int D>
__host__ __device__ inline TileGrid make_tile_grid(const phj_grid& g) {
  TileGrid t;
  using B = Blk<D>;
  if (D == 2) {
    t.n[0] = (int)((g.shape[0] + B::BY - 1) / B::BY);
    t.n[1] = (int)((g.shape[1] + B::BX - 1) / B::BX);
    t.n[2] = 1;
    t.total = t.n[0] * t.n[1];
  } else {
    t.n[0] = (int)g.shape[0];
    t.n[1] = (int)((g.shape[1] + B::BY - 1) / B::BY);
    t.n[2] = (int)((g.shape[2] + B::BX - 1) / B::BX);
    t.total = t.n[0] * t.n[1] * t.n[2];
  }
  return t;
}

// Interior index of this lane's first node in block `t`; returns false when
// the lane's row lies outside the grid (lanes stay in warp votes regardless).
template <int D>
__device__ inline bool lane_nodes(const phj_grid& g, const TileGrid& tg, int t, int lane, int c[3]) {
  using B = Blk<D>;
  const int ly = lane / B::LX, lx = lane % B::LX;
  if (D == 2) {
    const int bx = t % tg.n[1], by = t / tg.n[1];
    c[0] = by * B::BY + ly;
    c[1] = bx * B::BX + lx * B::NB;
    c[2] = 0;
    return c[0] < g.shape[0];
  } else {
    const int bx = t % tg.n[2];
    const int r = t / tg.n[2];
    const int by = r % tg.n[1], bz = r / tg.n[1];
    c[0] = bz;
    c[1] = by * B::BY + ly;
    c[2] = bx * B::BX + lx * B::NB;
    return c[1] < g.shape[1];
  }
}

// Mark the 3^D neighbour blocks of block `t` active for the next sweep
// (lane nid of a warp whose block changed).
template <int D>
__device__ inline void mark_neighbour(const TileGrid& tg, const phj_grid& g, int t, int nid,
                                      int* next_flags, int* next_list, int* next_count) {
  int c[3], n[3] = {tg.n[0], tg.n[1], tg.n[2]};
  if (D == 2) {
    c[1] = t % n[1];
    c[0] = t / n[1];
    int d0 = nid / 3 - 1, d1 = nid % 3 - 1;
    int a = c[0] + d0, b = c[1] + d1;
    if (g.periodic[0]) a = (a + n[0]) % n[0];
    if (a < 0 || a >= n[0] || b < 0 || b >= n[1]) return;
    int nt = a * n[1] + b;
    if (atomicExch(&next_flags[nt], 1) == 0) next_list[atomicAdd(next_count, 1)] = nt;
  } else {
    c[2] = t % n[2];
    int r = t / n[2];
    c[1] = r % n[1];
    c[0] = r / n[1];
    int d0 = nid / 9 - 1, d1 = (nid / 3) % 3 - 1, d2 = nid % 3 - 1;
    int a = c[0] + d0, b = c[1] + d1, e = c[2] + d2;
    if (g.periodic[0]) a = (a + n[0]) % n[0];
    if (a < 0 || a >= n[0] || b < 0 || b >= n[1] || e < 0 || e >= n[2]) return;
    int nt = (a * n[1] + b) * n[2] + e;
    if (atomicExch(&next_flags[nt], 1) == 0) next_list[atomicAdd(next_count, 1)] = nt;
  }
}

// Colour-mask variant (transport): OR the changed colours into the
// neighbour's next-sweep mask; the first setter appends the block.
template <int D>
__device__ inline void mark_neighbour_mask(const TileGrid& tg, const phj_grid& g, int t, int nid,
                                           unsigned long long bits, unsigned long long* next_mask,
                                           int* next_list, int* next_count) {
  int n[3] = {tg.n[0], tg.n[1], tg.n[2]};
  int nt;
  if (D == 2) {
    int a = t / n[1] + nid / 3 - 1, b = t % n[1] + nid % 3 - 1;
    if (g.periodic[0]) a = (a + n[0]) % n[0];
    if (a < 0 || a >= n[0] || b < 0 || b >= n[1]) return;
    nt = a * n[1] + b;
  } else {
    const int r = t / n[2];
    int a = r / n[1] + nid / 9 - 1, b = r % n[1] + (nid / 3) % 3 - 1, e = t % n[2] + nid % 3 - 1;
    if (g.periodic[0]) a = (a + n[0]) % n[0];
    if (a < 0 || a >= n[0] || b < 0 || b >= n[1] || e < 0 || e >= n[2]) return;
    nt = (a * n[1] + b) * n[2] + e;
  }
  if (atomicOr(&next_mask[nt], bits) == 0ull) next_list[atomicAdd(next_count, 1)] = nt;
}

// Workspace carve-up shared by solve/transport.
struct Workspace {
  int* list[2];
  int* flags[2];
  int* counts;  // [max_sweeps + 2] active blocks per sweep
  int* take;    // [max_sweeps + 2] dynamic work counters
  unsigned long long* cmask[2];  // transport: per-block active-colour masks
};

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

template <int D>
inline int64_t workspace_bytes(const phj_grid& g, int max_sweeps) {
  TileGrid tg = make_tile_grid<D>(g);
  int64_t b = 0;
  b += 4 * align_up((int64_t)tg.total * 4, 256);
  b += 2 * align_up((int64_t)(max_sweeps + 2) * 4, 256);
  b += 2 * align_up((int64_t)tg.total * 8, 256);
  return b;
}

template <int D>
inline Workspace carve(const phj_grid& g, void* base, int max_sweeps) {
  TileGrid tg = make_tile_grid<D>(g);
  char* p = (char*)base;
  Workspace w;
  int64_t tb = align_up((int64_t)tg.total * 4, 256);
  w.list[0] = (int*)p; p += tb;
  w.list[1] = (int*)p; p += tb;
  w.flags[0] = (int*)p; p += tb;
  w.flags[1] = (int*)p; p += tb;
  w.counts = (int*)p; p += align_up((int64_t)(max_sweeps + 2) * 4, 256);
  w.take = (int*)p; p += align_up((int64_t)(max_sweeps + 2) * 4, 256);
  w.cmask[0] = (unsigned long long*)p; p += align_up((int64_t)tg.total * 8, 256);
  w.cmask[1] = (unsigned long long*)p;
  return w;
}

__device__ inline unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

template <typename T> __device__ __host__ constexpr T big_value();
template <> __device__ __host__ constexpr double big_value<double>() { return 1.0e300; }
template <> __device__ __host__ constexpr float big_value<float>() { return 1.0e30f; }

__device__ inline double ld_cg(const double* p) { return __ldcg(p); }
__device__ inline unsigned long long ld_cg(const unsigned long long* p) { return __ldcg(p); }
__device__ inline int ld_cg(const int* p) { return __ldcg(p); }

}  // namespace phj

// error plumbing shared by the .cu translation units
void phj_set_error(const char* fmt, ...);
void phj_count_launch(int n);  // every kernel launch of the library bumps this
int phj_check_cuda(cudaError_t e, const char* what);
#define PHJ_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return phj_check_cuda(_e, #call); \
  } while (0)
