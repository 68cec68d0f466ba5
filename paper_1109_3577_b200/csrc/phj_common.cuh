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
#ifndef PHJ_MIN_CTAS
#define PHJ_MIN_CTAS (16 / PHJ_CTA_WARPS)  // 16 resident warps per SM
#endif
constexpr int kCtasPerSm = PHJ_MIN_CTAS;
constexpr int kMaxPatches = 1024;
constexpr int kMaxColors = 4096;  // transport colours (>= kMaxPatches)
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

// n / d for 0 <= n < 2^31 by multiply-high ("round-up" magic number, the
// usual replacement for a runtime integer division); set up on the host.
struct FastDiv {
  uint32_t d, m, l;
  __host__ void init(uint32_t dd) {
    d = dd < 1 ? 1 : dd;
    l = 0;
    while ((1ull << l) < d) ++l;
    m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
  }
  __device__ __forceinline__ int div(int n) const {
    return (int)((__umulhi((uint32_t)n, m) + (uint32_t)n) >> l);
  }
};

struct TileGrid {
  int n[3];  // blocks per internal axis (axis 0 slowest)
  int total;
  FastDiv f1, f2;  // division by n[1], n[2]
};

template <int D>
__host__ inline TileGrid make_tile_grid(const phj_grid& g) {
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
  t.f1.init((uint32_t)t.n[1]);
  t.f2.init((uint32_t)t.n[2]);
  return t;
}

// block id -> block coordinates along internal axes (axis 0 slowest)
template <int D>
__device__ __forceinline__ void decode_block(const TileGrid& tg, int t, int b[3]) {
  if (D == 2) {
    b[0] = tg.f1.div(t);
    b[1] = t - b[0] * tg.n[1];
    b[2] = 0;
  } else {
    const int r = tg.f2.div(t);
    b[2] = t - r * tg.n[2];
    b[0] = tg.f1.div(r);
    b[1] = r - b[0] * tg.n[1];
  }
}

// Interior index of this lane's first node in block `t`; returns false when
// the lane's row lies outside the grid (lanes stay in warp votes regardless).
template <int D>
__device__ inline bool lane_nodes(const phj_grid& g, const TileGrid& tg, int t, int lane, int c[3]) {
  using B = Blk<D>;
  const int ly = lane / B::LX, lx = lane % B::LX;
  int b[3];
  decode_block<D>(tg, t, b);
  if (D == 2) {
    c[0] = b[0] * B::BY + ly;
    c[1] = b[1] * B::BX + lx * B::NB;
    c[2] = 0;
    return c[0] < g.shape[0];
  } else {
    c[0] = b[0];
    c[1] = b[1] * B::BY + ly;
    c[2] = b[2] * B::BX + lx * B::NB;
    return c[1] < g.shape[1];
  }
}

// Id of neighbour nid (0 .. 3^D - 1) of block t, -1 outside the grid.
template <int D>
__device__ inline int neighbour_block(const TileGrid& tg, const phj_grid& g, int t, int nid) {
  const int* n = tg.n;
  int b[3];
  decode_block<D>(tg, t, b);
  if (D == 2) {
    int a = b[0] + nid / 3 - 1, c = b[1] + nid % 3 - 1;
    if (g.periodic[0]) a = a < 0 ? a + n[0] : (a >= n[0] ? a - n[0] : a);
    if (a < 0 || a >= n[0] || c < 0 || c >= n[1]) return -1;
    return a * n[1] + c;
  } else {
    int a = b[0] + nid / 9 - 1, c = b[1] + (nid / 3) % 3 - 1, e = b[2] + nid % 3 - 1;
    if (g.periodic[0]) a = a < 0 ? a + n[0] : (a >= n[0] ? a - n[0] : a);
    if (a < 0 || a >= n[0] || c < 0 || c >= n[1] || e < 0 || e >= n[2]) return -1;
    return (a * n[1] + c) * n[2] + e;
  }
}

// Colour-mask marking (transport): OR the changed colours into neighbour
// nid's next-sweep mask; the first setter appends the block.
template <int D>
__device__ inline void mark_neighbour_mask(const TileGrid& tg, const phj_grid& g, int t, int nid,
                                           unsigned long long bits, unsigned long long* next_mask,
                                           int* next_list, int* next_count) {
  const int nt = neighbour_block<D>(tg, g, t, nid);
  if (nt < 0) return;
  if (atomicOr(&next_mask[nt], bits) == 0ull) next_list[atomicAdd(next_count, 1)] = nt;
}

// Workspace carve-up shared by solve/transport.
struct Workspace {
  int* list[2];
  int* flags[2];
  int* counts;  // [max_sweeps + 2] active blocks per sweep
  int* take;    // [max_sweeps + 2] dynamic work counters
  unsigned long long* cmask[2];  // transport: per-block active-colour masks
  // per-sweep max change per patch / colour, one 128-byte line per entry
  // (all CTAs reduce into these with atomics right before the grid barrier
  // and read them right after it: packed into one line, those requests
  // serialise on one L2 slice), six buffers by sweep: the two-sweep
  // transport zeroes sweeps 2m+2, 2m+3 during pass m while it accumulates
  // 2m, 2m+1 and slow CTAs may still read 2m-2, 2m-1 after the previous
  // barrier (with three buffers the zeroing hit entries still being read and
  // CTAs could take different stop decisions -- a rare grid-barrier hang)
  unsigned long long* pmax;  // [kMaxBufs][kMaxColors * kMaxPad]
  // asynchronous solve: FIFO ring of block ids, capacity blocks + warps
  // (at most one queued entry per block and one waiting ticket per warp)
  unsigned long long* ring;  // [total + kRingExtra] sequence-numbered cells
};

constexpr int kRingExtra = 1 << 16;  // >= resident warps of any async launch

constexpr int kMaxPad = 16;  // u64 per entry = 128 B
constexpr int kMaxBufs = 6;  // per-sweep max-change buffers (see Workspace::pmax)

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

template <int D>
inline int64_t workspace_bytes(const phj_grid& g, int max_sweeps) {
  TileGrid tg = make_tile_grid<D>(g);
  int64_t b = 0;
  b += 4 * align_up((int64_t)tg.total * 4, 256);
  b += 2 * align_up((int64_t)(max_sweeps + 2) * 4, 256);
  b += 2 * align_up((int64_t)tg.total * 8, 256);
  b += kMaxBufs * (int64_t)kMaxColors * kMaxPad * 8;
  b += align_up(((int64_t)tg.total + kRingExtra) * 8, 256);
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
  w.cmask[1] = (unsigned long long*)p; p += align_up((int64_t)tg.total * 8, 256);
  w.pmax = (unsigned long long*)p;
  p += kMaxBufs * (int64_t)kMaxColors * kMaxPad * 8;
  w.ring = (unsigned long long*)p;
  return w;
}

// the padded max-change entries of sweep sw
__device__ __forceinline__ unsigned long long* sweep_max_slots(const Workspace& w, int sw) {
  return w.pmax + (int64_t)(sw % kMaxBufs) * kMaxColors * kMaxPad;
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
