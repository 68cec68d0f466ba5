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

// warp block of internal serial s (Blk<D> geometry, axis 0 slowest)
template <int D>
__device__ __forceinline__ int block_of(const phj_grid& g, const TileGrid& tg, int64_t s) {
  using B = Blk<D>;
  if (D == 3) {
    const int64_t i2 = s % g.shape[2], r = s / g.shape[2];
    const int64_t i1 = r % g.shape[1], i0 = r / g.shape[1];
    return (int)((i0 * tg.n[1] + i1 / B::BY) * tg.n[2] + i2 / B::BX);
  } else {
    const int64_t i1 = s % g.shape[1], i0 = s / g.shape[1];
    return (int)((i0 / B::BY) * tg.n[1] + i1 / B::BX);
  }
}

template <int D, typename T>
__global__ void band_times_kernel(phj_grid g, TileGrid tg, const T* __restrict__ key, int kruzkov,
                                  const uint8_t* __restrict__ nodes, BandScratch s) {
  const int64_t n = g.shape[0] * g.shape[1] * (D == 3 ? g.shape[2] : 1);
  unsigned long long lmax = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!nodes[i]) continue;
    int c[3];
    int64_t r = i;
    for (int ax = D - 1; ax >= 0; --ax) {
      c[ax] = (int)(r % g.shape[ax]);
      r /= g.shape[ax];
    }
    int64_t f = 0;
    for (int ax = 0; ax < D; ++ax) f += (int64_t)(c[ax] + 1) * g.strides[ax];
    double t = (double)key[f];
    if (kruzkov) t = -log1p(-fmin(t, 1.0 - 1e-16));
    t = fmax(t, 0.0);
    const unsigned long long bits = (unsigned long long)__double_as_longlong(t);
    const int b = block_of<D>(g, tg, i);
    atomicMin(&s.tmin[b], bits);
    atomicMax(&s.tmax[b], bits);
    lmax = max(lmax, bits);
  }
  for (int off = 16; off > 0; off >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
  if ((threadIdx.x & 31) == 0 && lmax) atomicMax(&s.glob[0], lmax);
}

__global__ void band_ranges_kernel(int total, double delta, int lo_w, int hi_w, int max_row,
                                   BandScratch s) {
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
    atomicAdd(&s.glob[1], (unsigned long long)(hi - lo + 2));
    atomicMax(&s.glob[2], (unsigned long long)(hi + 2));
    atomicAdd(&s.glob[3], 1ull);
    atomicAdd(&s.diff[lo], 1);
    atomicSub(&s.diff[hi + 2], 1);
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

__global__ void band_fill_kernel(int total, int n_band, int final_row, BandScratch s,
                                 const int32_t* __restrict__ off, int32_t* __restrict__ list) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < total; b += gridDim.x * blockDim.x) {
    const int lo = s.lo[b];
    if (lo < 0) continue;
    const int hi = s.hi[b];
    for (int r = lo; r <= hi; ++r) list[off[r] + atomicAdd(&s.cursor[r], 1)] = b;
    list[off[hi + 1] + atomicAdd(&s.cursor[hi + 1], 1)] = -b - 1;  // copy visit
    if (final_row) list[off[n_band] + atomicAdd(&s.cursor[n_band], 1)] = b;
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
  PHJ_CUDA(cudaMemsetAsync(s.tmin, 0xff, 8 * (size_t)tg.total, st));
  PHJ_CUDA(cudaMemsetAsync(s.tmax, 0, 8 * (size_t)tg.total, st));
  PHJ_CUDA(cudaMemsetAsync(s.glob, 0, 32, st));
  PHJ_CUDA(cudaMemsetAsync(s.diff, 0, 4 * (size_t)rows, st));
  const int64_t n = g->shape[0] * g->shape[1] * (D == 3 ? g->shape[2] : 1);
  const int nb = (int)std::min<int64_t>((n + 255) / 256, 8 * phj_num_sms());
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
  const int total = d3 ? make_tile_grid<3>(*g).total : make_tile_grid<2>(*g).total;
  band_offsets_kernel<<<1, 256, 0, st>>>(n_band, final_row, n_blocks, s, band_off);
  phj_count_launch(1);
  const int nbb = (int)std::min<int64_t>((total + 255) / 256, 8 * phj_num_sms());
  band_fill_kernel<<<std::max(nbb, 1), 256, 0, st>>>(total, n_band, final_row, s, band_off,
                                                      band_list);
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}
