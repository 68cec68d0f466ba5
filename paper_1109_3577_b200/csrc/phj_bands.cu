// phj_bands.cu -- the schedule of the value-ordered ("banded") passes
// (patchy.band_schedule): per warp block the time range of
// its scheduled nodes from the lifted field, then one CSR row of block visits
// per sweep.  Three small launches and two 16-byte device->host reads per
// schedule instead of a dozen eager tensor ops and a sort.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "phj_common.cuh"

namespace phj {

struct BandScratch {
  unsigned long long* tmin;  // [total] bits of the smallest node time (~0 = no node)
  unsigned long long* tmax;  // [total]
  int* lo;                   // [total] first sweep visiting the block
  int* hi;                   // [total] last relaxing sweep (copy visit at hi + 1)
  unsigned long long* glob;  // [4]: max time bits, entries, n_band, blocks
  int* diff;                 // [rows] row-count differences, then counts
  int* cursor;               // [rows]
};

inline int64_t band_rows(int max_bands, int lo_w, int hi_w) {
  return (int64_t)max_bands + lo_w + hi_w + 8;
}

template <int D>
inline BandScratch carve_bands(const phj_grid& g, void* base, int64_t rows) {
  const TileGrid tg = make_tile_grid<D>(g);
  char* p = (char*)base;
  BandScratch s;
  const int64_t t8 = align_up((int64_t)tg.total * 8, 256), t4 = align_up((int64_t)tg.total * 4, 256);
  s.tmin = (unsigned long long*)p; p += t8;
  s.tmax = (unsigned long long*)p; p += t8;
  s.lo = (int*)p; p += t4;
  s.hi = (int*)p; p += t4;
  s.glob = (unsigned long long*)p; p += 256;
  s.diff = (int*)p; p += align_up(rows * 4, 256);
  s.cursor = (int*)p;
  return s;
}

template <int D>
inline int64_t band_scratch_bytes(const phj_grid& g, int64_t rows) {
  const TileGrid tg = make_tile_grid<D>(g);
  return 2 * align_up((int64_t)tg.total * 8, 256) + 2 * align_up((int64_t)tg.total * 4, 256) +
         256 + 2 * align_up(rows * 4, 256);
}

// One warp per warp block (the Blk<D> lane -> node map of the sweeps): the
// smallest / largest key of its scheduled nodes by a warp reduction, the
// time transform (monotone) applied to the two extremes only.
template <int D, typename T>
__global__ void band_times_kernel(phj_grid g, TileGrid tg, const T* __restrict__ key, int kruzkov,
                                  const uint8_t* __restrict__ nodes, BandScratch s) {
  using B = Blk<D>;
  constexpr int last = D - 1;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  unsigned long long lmax = 0ull;
  for (int b = gw; b < tg.total; b += nw) {
    int c[3];
    const bool ok = lane_nodes<D>(g, tg, b, lane, c);
    int64_t ser = 0, f = 0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      ser = ser * g.shape[ax] + c[ax];
      f += (int64_t)(c[ax] + 1) * g.strides[ax];
    }
    double vmin = 1.0e300, vmax = -1.0;
#pragma unroll
    for (int r = 0; r < B::NB; ++r) {
      if (!(ok && c[last] + r < g.shape[last]) || !nodes[ser + r]) continue;
      const double v = (double)key[f + r];
      vmin = fmin(vmin, v);
      vmax = fmax(vmax, v);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      vmin = fmin(vmin, __shfl_xor_sync(FULL, vmin, off));
      vmax = fmax(vmax, __shfl_xor_sync(FULL, vmax, off));
    }
    if (lane == 0) {
      unsigned long long b0 = ~0ull, b1 = 0ull;
      if (vmin < 1.0e300) {  // the block holds a scheduled node
        double t0 = vmin, t1 = vmax;
        if (kruzkov) {
          t0 = -log1p(-fmin(t0, 1.0 - 1e-16));
          t1 = -log1p(-fmin(t1, 1.0 - 1e-16));
        }
        b0 = (unsigned long long)__double_as_longlong(fmax(t0, 0.0));
        b1 = (unsigned long long)__double_as_longlong(fmax(t1, 0.0));
        lmax = max(lmax, b1);
      }
      s.tmin[b] = b0;
      s.tmax[b] = b1;
    }
  }
  if (lane == 0 && lmax) atomicMax(&s.glob[0], lmax);
}

__global__ void band_ranges_kernel(int total, double delta, int lo_w, int hi_w, int max_row,
                                   BandScratch s) {
  unsigned long long entries = 0ull, blocks = 0ull, top = 0ull;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < total; b += gridDim.x * blockDim.x) {
    s.lo[b] = -1;
    if (s.tmin[b] == ~0ull) continue;
    const double t0 = __longlong_as_double((long long)s.tmin[b]);
    const double t1 = __longlong_as_double((long long)s.tmax[b]);
    const int k0 = (int)fmin(floor(t0 / delta), (double)max_row);
    const int k1 = (int)fmin(floor(t1 / delta), (double)max_row);
    const int lo = max(0, k0 - hi_w), hi = k1 + lo_w;
    s.lo[b] = lo;
    s.hi[b] = hi;
    entries += (unsigned long long)(hi - lo + 2);
    top = max(top, (unsigned long long)(hi + 2));
    blocks += 1ull;
    atomicAdd(&s.diff[lo], 1);
    atomicSub(&s.diff[hi + 2], 1);
  }
  // totals: one atomic per warp instead of three per block on one address
  for (int off = 16; off > 0; off >>= 1) {
    entries += __shfl_xor_sync(0xffffffffu, entries, off);
    blocks += __shfl_xor_sync(0xffffffffu, blocks, off);
    top = max(top, __shfl_xor_sync(0xffffffffu, top, off));
  }
  if ((threadIdx.x & 31) == 0 && blocks) {
    atomicAdd(&s.glob[1], entries);
    atomicMax(&s.glob[2], top);
    atomicAdd(&s.glob[3], blocks);
  }
}

// row offsets: counts = prefix sums of the differences (one CTA, rows small)
__global__ void band_offsets_kernel(int n_band, int final_row, int n_blocks, BandScratch s,
                                    int32_t* off) {
  if (threadIdx.x == 0) {
    int run = 0, pos = 0;
    off[0] = 0;
    for (int r = 0; r < n_band; ++r) {
      run += s.diff[r];
      pos += run;
      off[r + 1] = pos;
    }
    if (final_row) off[n_band + 1] = pos + n_blocks;
  }
  for (int r = threadIdx.x; r <= n_band; r += blockDim.x) s.cursor[r] = 0;
}

// Append block id `val` to row r; the lanes of the warp appending to the same
// row in this step share one cursor atomic (neighbouring blocks have nearly
// the same rows, so a step touches a handful of rows).  All lanes call;
// inactive ones pass r < 0.
__device__ __forceinline__ void band_append(int r, int val, const BandScratch& s,
                                            const int32_t* __restrict__ off,
                                            int32_t* __restrict__ list) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned peers = __match_any_sync(FULL, r);
  if (r < 0) return;
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&s.cursor[r], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  list[off[r] + base + __popc(peers & ((1u << lane) - 1u))] = val;
}

// every third bit of x (Morton decode of one coordinate)
__device__ __forceinline__ unsigned compact3(unsigned long long x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
  x = (x ^ (x >> 32)) & 0x1fffffull;
  return (unsigned)x;
}
__device__ __forceinline__ unsigned compact2(unsigned long long x) {
  x &= 0x5555555555555555ull;
  x = (x ^ (x >> 1)) & 0x3333333333333333ull;
  x = (x ^ (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
  x = (x ^ (x >> 4)) & 0x00ff00ff00ff00ffull;
  x = (x ^ (x >> 8)) & 0x0000ffff0000ffffull;
  x = (x ^ (x >> 16)) & 0xffffffffull;
  return (unsigned)x;
}

// Block id of position i of the fill order, or -1: blocks are appended in
// Morton order of their coordinates (3D: cubes of kZ planes x 1 x 1 blocks
// along a Morton curve over (plane / kZ, row block, column block)), so the
// blocks a sweep's warps hold at the same time are neighbours in all
// directions and share their halo rows through L1/L2 instead of DRAM.
constexpr int kZ = 8;
template <int D>
__device__ __forceinline__ int fill_order_block(const TileGrid& tg, long long i) {
  if (D == 3) {
    const unsigned long long code = (unsigned long long)(i / kZ);
    const int z = (int)compact3(code >> 2) * kZ + (int)(i % kZ);
    const int y = (int)compact3(code >> 1), x = (int)compact3(code);
    if (z >= tg.n[0] || y >= tg.n[1] || x >= tg.n[2]) return -1;
    return (z * tg.n[1] + y) * tg.n[2] + x;
  } else {
    const int y = (int)compact2((unsigned long long)i >> 1), x = (int)compact2((unsigned long long)i);
    if (y >= tg.n[0] || x >= tg.n[1]) return -1;
    return y * tg.n[1] + x;
  }
}

template <int D>
__global__ void band_fill_kernel(TileGrid tg, long long n_pos, int n_band, int final_row,
                                 BandScratch s, const int32_t* __restrict__ off,
                                 int32_t* __restrict__ list) {
  const unsigned FULL = 0xffffffffu;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long rounds = (n_pos + stride - 1) / stride;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long k = 0; k < rounds; ++k, i += stride) {
    const int b = i < n_pos ? fill_order_block<D>(tg, i) : -1;
    const int lo = b >= 0 ? s.lo[b] : -1;
    const int hi = lo < 0 ? -2 : s.hi[b];
    // the warp walks rows from its smallest lo to its largest hi + 1
    int wlo = lo < 0 ? 0x7fffffff : lo, whi = hi + 1;
    for (int o = 16; o > 0; o >>= 1) {
      wlo = min(wlo, __shfl_xor_sync(FULL, wlo, o));
      whi = max(whi, __shfl_xor_sync(FULL, whi, o));
    }
    for (int r = wlo; r <= whi; ++r) {
      const bool in = lo >= 0 && r >= lo && r <= hi + 1;
      band_append(in ? r : -1, r <= hi ? b : -b - 1, s, off, list);  // hi + 1: the copy visit
    }
    if (final_row && __any_sync(FULL, lo >= 0))
      band_append(lo >= 0 ? n_band : -1, b, s, off, list);
  }
}

}  // namespace phj

using namespace phj;

extern "C" int phj_num_sms(void);

extern "C" int64_t phj_band_scratch_bytes(const phj_grid* g, int32_t max_bands, int32_t lo_w,
                                          int32_t hi_w) {
  if (!g || max_bands < 1) return -1;
  const int64_t rows = band_rows(max_bands, lo_w, hi_w);
  return g->dim == 2 ? band_scratch_bytes<2>(*g, rows) : band_scratch_bytes<3>(*g, rows);
}

template <int D>
static int band_count_impl(const phj_grid* g, int32_t dtype, int32_t rule, const void* key,
                           const uint8_t* nodes, double delta_min, int32_t max_bands,
                           int32_t lo_w, int32_t hi_w, void* scratch, int64_t* out,
                           cudaStream_t st) {
  const TileGrid tg = make_tile_grid<D>(*g);
  const int64_t rows = band_rows(max_bands, lo_w, hi_w);
  BandScratch s = carve_bands<D>(*g, scratch, rows);
  PHJ_CUDA(cudaMemsetAsync(s.glob, 0, 32, st));
  PHJ_CUDA(cudaMemsetAsync(s.diff, 0, 4 * (size_t)rows, st));
  const int nb = (int)std::min<int64_t>(((int64_t)tg.total + 7) / 8, 8 * phj_num_sms());
  const int kr = rule == PHJ_RULE_KRUZKOV;
  if (dtype == PHJ_F32)
    band_times_kernel<D, float><<<std::max(nb, 1), 256, 0, st>>>(*g, tg, (const float*)key, kr,
                                                                  nodes, s);
  else
    band_times_kernel<D, double><<<std::max(nb, 1), 256, 0, st>>>(*g, tg, (const double*)key, kr,
                                                                   nodes, s);
  phj_count_launch(1);
  unsigned long long tmax_bits = 0ull;
  PHJ_CUDA(cudaMemcpyAsync(&tmax_bits, s.glob, 8, cudaMemcpyDeviceToHost, st));
  PHJ_CUDA(cudaStreamSynchronize(st));
  double tmax = 0.0;
  memcpy(&tmax, &tmax_bits, 8);
  // bands of width delta_min, widened so that at most max_bands exist
  const double delta = std::max(delta_min, tmax / (double)max_bands);
  const int nbb = (int)std::min<int64_t>((tg.total + 255) / 256, 8 * phj_num_sms());
  band_ranges_kernel<<<std::max(nbb, 1), 256, 0, st>>>(tg.total, delta, lo_w, hi_w, max_bands,
                                                        s);
  phj_count_launch(1);
  unsigned long long gl[4];
  PHJ_CUDA(cudaMemcpyAsync(gl, s.glob, 32, cudaMemcpyDeviceToHost, st));
  PHJ_CUDA(cudaStreamSynchronize(st));
  out[0] = (int64_t)gl[1];  // entries (without the final row)
  out[1] = (int64_t)gl[2];  // n_band
  out[2] = (int64_t)gl[3];  // blocks with scheduled nodes
  memcpy(&out[3], &delta, 8);
  return PHJ_OK;
}

extern "C" int phj_band_count(const phj_grid* g, int32_t dtype, int32_t rule, const void* key,
                              const uint8_t* nodes, double delta_min, int32_t max_bands,
                              int32_t lo_w, int32_t hi_w, void* scratch, int64_t* out,
                              void* stream) {
  if (!g || !key || !nodes || !scratch || !out || max_bands < 1 || lo_w < 0 || hi_w < 0 ||
      !(delta_min > 0.0) || (g->dim != 2 && g->dim != 3)) {
    phj_set_error("phj_band_count: bad arguments");
    return PHJ_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return g->dim == 2 ? band_count_impl<2>(g, dtype, rule, key, nodes, delta_min, max_bands, lo_w,
                                          hi_w, scratch, out, st)
                     : band_count_impl<3>(g, dtype, rule, key, nodes, delta_min, max_bands, lo_w,
                                          hi_w, scratch, out, st);
}

extern "C" int phj_band_fill(const phj_grid* g, int32_t max_bands, int32_t lo_w, int32_t hi_w,
                             int32_t n_band, int32_t n_blocks, int32_t final_row, void* scratch,
                             int32_t* band_list, int32_t* band_off, void* stream) {
  if (!g || !scratch || !band_list || !band_off || n_band < 1 ||
      n_band > band_rows(max_bands, lo_w, hi_w) - 2) {
    phj_set_error("phj_band_fill: bad arguments");
    return PHJ_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = band_rows(max_bands, lo_w, hi_w);
  const bool d3 = g->dim == 3;
  BandScratch s = d3 ? carve_bands<3>(*g, scratch, rows) : carve_bands<2>(*g, scratch, rows);
  const TileGrid tg = d3 ? make_tile_grid<3>(*g) : make_tile_grid<2>(*g);
  band_offsets_kernel<<<1, 256, 0, st>>>(n_band, final_row, n_blocks, s, band_off);
  phj_count_launch(1);
  // positions of the Morton fill order (power-of-two cube around the block grid)
  int bits = 0;
  const int ext0 = d3 ? (tg.n[0] + kZ - 1) / kZ : tg.n[0];
  const int ext_max = std::max(ext0, std::max(tg.n[1], d3 ? tg.n[2] : 1));
  while ((1 << bits) < ext_max) ++bits;
  const long long n_pos = d3 ? ((long long)kZ << (3 * bits)) : (1ll << (2 * bits));
  // few threads per round: a round appends a compact piece of the curve (the
  // order inside a round is the arrival order of its warps)
  const int nbb = (int)std::min<long long>((n_pos + 255) / 256, 2 * phj_num_sms());
  if (d3)
    band_fill_kernel<3><<<std::max(nbb, 1), 256, 0, st>>>(tg, n_pos, n_band, final_row, s,
                                                           band_off, band_list);
  else
    band_fill_kernel<2><<<std::max(nbb, 1), 256, 0, st>>>(tg, n_pos, n_band, final_row, s,
                                                           band_off, band_list);
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}
