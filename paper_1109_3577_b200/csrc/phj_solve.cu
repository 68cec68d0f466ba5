// phj_solve.cu -- the semi-Lagrangian value sweep, colour transport and
// feedback extraction for sm_100a.
//
// Design:
//  * Jacobi iteration with two ext buffers; the whole fixed-point loop runs
//    inside ONE cooperative persistent launch (grid.sync between sweeps), so
//    there is no host round trip per sweep (reference loop: solver.py:256-273).
//  * Work and activity unit = a warp block (Blk<D>: 4 rows x 32 / 16 nodes).
//    A block is re-swept only if a block in its 3^D neighbourhood changed in
//    the previous sweep -- exact: a node whose stencil inputs did not change
//    reproduces its previous value (monotone min).  Warps fetch active blocks
//    from the sweep's list with an atomic counter; no CTA barrier inside a
//    sweep.
//  * Each lane keeps its NB nodes' 3^D neighbourhood in registers; per-control
//    corner weights come from shared memory as warp broadcasts.  Controls are
//    grouped by foot octant on the host, which makes every register index a
//    compile-time constant; two controls are evaluated per iteration for ILP.
//  * State constraints (patch solves) are per-node 3^D "foreign" bitmasks; a
//    warp with no foreign neighbour takes the rejection-free path.
//  * Per-patch convergence: patch p stops at the first sweep whose max change
//    over p is <= tol, exactly like one reference solve() per patch
//    (patchy.py:362-377); later sweeps copy its nodes through unchanged.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "phj_common.cuh"

namespace cg = cooperative_groups;

namespace phj {

struct SolveParams {
  phj_grid g;
  TileGrid tg;
  int n_classes, nc, n_real;
  const int32_t* oct_start;
  const uint32_t* nzmask;
  const double* weights;
  const double* cost;
  void* v[2];
  const int16_t* lab;
  const uint32_t* fmask;
  const void* coef;
  double coef0;
  int R;
  int max_sweeps;
  const uint8_t* mine;
  double tol;
  Workspace ws;
  unsigned long long* maxch;  // [max_sweeps * R], double bits
  int32_t* patch_sweeps;
  unsigned long long* evals;
  int32_t* info;
};

template <int D, typename T>
struct StencilSmem {
  T* w;          // [nent][2^D]
  T* a;          // [nent] beta (KRUZKOV) or cost (REF), COST_CTRL only
  T* b;          // [nent] 1 - beta
  uint32_t* nz;  // [nent]
  int* oct;      // [ncls][2^D + 1]
  static __host__ __device__ int64_t bytes(int ncls, int nc) {
    int64_t nent = (int64_t)ncls * nc;
    int64_t b = nent * (1 << D) * sizeof(T) + 2 * nent * sizeof(T);
    b = (b + 15) / 16 * 16;
    b += nent * 4 + (int64_t)ncls * ((1 << D) + 1) * 4;
    return (b + 15) / 16 * 16;
  }
};

template <int D, typename T>
__device__ inline StencilSmem<D, T> carve_stencil(unsigned char* base, int ncls, int nc) {
  StencilSmem<D, T> s;
  int64_t nent = (int64_t)ncls * nc;
  s.w = (T*)base;
  s.a = s.w + nent * (1 << D);
  s.b = s.a + nent;
  unsigned char* p = (unsigned char*)(s.b + nent);
  p = base + ((p - base + 15) / 16 * 16);
  s.nz = (uint32_t*)p;
  s.oct = (int*)(s.nz + nent);
  return s;
}

template <int D, typename T, int RULE>
__device__ inline void stage_stencil(const StencilSmem<D, T>& s, int ncls, int nc,
                                     const int32_t* oct_start, const uint32_t* nzmask,
                                     const double* weights, const double* cost) {
  const int nent = ncls * nc;
  constexpr int NC = 1 << D;
  for (int i = threadIdx.x; i < nent; i += blockDim.x) {
    // weights in T with the last nonzero one set so that their sequential
    // sum in T is exactly 1 (I[1] == 1, see dynamics._weights_for)
    T w[NC];
    int last = 0;
    for (int k = 0; k < NC; ++k) {
      w[k] = (T)weights[(int64_t)i * NC + k];
      if (w[k] != T(0)) last = k;
    }
    T sum = T(0);
    for (int k = 0; k < last; ++k) sum = sum + w[k];
    w[last] = T(1) - sum;
    for (int k = 0; k < NC; ++k) s.w[(int64_t)i * NC + k] = w[k];
  }
  for (int i = threadIdx.x; i < nent; i += blockDim.x) {
    s.nz[i] = nzmask[i];
    double c = cost ? cost[i] : 0.0;
    if (RULE == PHJ_RULE_KRUZKOV) {
      // 1 - beta is exact in T (Sterbenz), so beta * 1 + (1 - beta) == 1
      const T beta = (T)exp(-c);
      s.a[i] = beta;
      s.b[i] = T(1) - beta;
    } else {
      s.a[i] = (T)c;
      s.b[i] = (T)0;
    }
  }
  for (int i = threadIdx.x; i < ncls * ((1 << D) + 1); i += blockDim.x) s.oct[i] = oct_start[i];
}

// Neighbourhood register block: NR rows (3^(D-1)) x (NB + 2) columns.
template <int D, typename T, int NB>
struct Nbhd {
  static constexpr int NR = (D == 2) ? 3 : 9;
  T v[NR][NB + 2];
};

// value of corner K of octant O for node r (compile-time after unrolling)
template <int D, int NB, int O, int K, typename T>
__device__ __forceinline__ T corner_val(const Nbhd<D, T, NB>& nb, int r) {
  // internal axis ax: offset = (octant bit ? 0 : -1) + corner bit
  constexpr int off0 = (((O >> 0) & 1) ? 0 : -1) + ((K >> 0) & 1);
  constexpr int off1 = (((O >> 1) & 1) ? 0 : -1) + ((K >> 1) & 1);
  if constexpr (D == 2) {
    return nb.v[off0 + 1][r + off1 + 1];
  } else {
    constexpr int off2 = (((O >> 2) & 1) ? 0 : -1) + ((K >> 2) & 1);
    return nb.v[(off0 + 1) * 3 + (off1 + 1)][r + off2 + 1];
  }
}

template <int D, typename T, int NB, int O, int K>
struct CornerSum {
  __device__ __forceinline__ static T run(const Nbhd<D, T, NB>& nb, const T* w, int r, T acc) {
    acc = fma(w[K], corner_val<D, NB, O, K>(nb, r), acc);
    return CornerSum<D, T, NB, O, K + 1>::run(nb, w, r, acc);
  }
};
template <int D, typename T, int NB, int O>
struct CornerSum<D, T, NB, O, (1 << D)> {
  __device__ __forceinline__ static T run(const Nbhd<D, T, NB>&, const T*, int, T acc) {
    return acc;
  }
};

// One corner step K of U*NB interleaved interpolation chains.
template <int D, typename T, int NB, int O, int U, int K>
struct ChainStep {
  __device__ __forceinline__ static void run(const Nbhd<D, T, NB>& nb, const T (&w)[U][1 << D],
                                             T (&acc)[U][NB]) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NB; ++r) acc[u][r] = fma(w[u][K], corner_val<D, NB, O, K>(nb, r), acc[u][r]);
    ChainStep<D, T, NB, O, U, K + 1>::run(nb, w, acc);
  }
};
template <int D, typename T, int NB, int O, int U>
struct ChainStep<D, T, NB, O, U, (1 << D)> {
  __device__ __forceinline__ static void run(const Nbhd<D, T, NB>&, const T (&)[U][1 << D],
                                             T (&)[U][NB]) {}
};

template <int D, typename T, int NB, int O>
__device__ __forceinline__ T interp(const Nbhd<D, T, NB>& nb, const T* w, int r) {
  T acc = w[0] * corner_val<D, NB, O, 0>(nb, r);
  return CornerSum<D, T, NB, O, 1>::run(nb, w, r, acc);
}

template <typename T, int N>
__device__ __forceinline__ void load_weights(const T* src, T* w) {
  if constexpr (sizeof(T) == 8 && N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      double2 q = reinterpret_cast<const double2*>(src)[i];
      w[2 * i] = q.x;
      w[2 * i + 1] = q.y;
    }
  } else if constexpr (sizeof(T) == 4 && N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      float4 q = reinterpret_cast<const float4*>(src)[i];
      w[4 * i] = q.x;
      w[4 * i + 1] = q.y;
      w[4 * i + 2] = q.z;
      w[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = src[i];
  }
}

// Candidate post-processing: per-entry cost (COST_CTRL), the per-candidate
// rule in feedback mode, and state-constraint rejection.
template <typename T, int RULE, int COST, bool SLOW, int MODE>
__device__ __forceinline__ T finish_cand(T acc, T ca, T cb, T ncoef, uint32_t fm, uint32_t nz) {
  if constexpr (COST == PHJ_COST_CTRL) {
    acc = (RULE == PHJ_RULE_KRUZKOV) ? fma(ca, acc, cb) : acc + ca;
  } else if constexpr (MODE == 1) {
    // feedback applies the rule per candidate (SURVEY App. A hoisting caveat)
    acc = (RULE == PHJ_RULE_KRUZKOV) ? fma(ncoef, acc, T(1) - ncoef) : acc + ncoef;
  }
  if constexpr (SLOW) {
    if (fm & nz) acc = big_value<T>();
  }
  return acc;
}

// Running minimum of non-negative candidates.  For fp64 the compare runs on
// the bit patterns as int64 (same order for values >= 0; candidates are
// convex combinations of non-negative values plus non-negative costs), which
// keeps the FP64 pipe for the interpolation FMAs; fp32 uses FMNMX.
#ifndef PHJ_MIN_INT
#define PHJ_MIN_INT 1
#endif
#ifndef PHJ_KUNROLL2
#define PHJ_KUNROLL2 4
#endif
template <typename T>
struct MinAcc;
template <>
struct MinAcc<double> {
#if PHJ_MIN_INT
  long long b;
  __device__ __forceinline__ void init() { b = __double_as_longlong(big_value<double>()); }
  __device__ __forceinline__ void take(double x) { b = min(b, __double_as_longlong(x)); }
  __device__ __forceinline__ double get() const { return __longlong_as_double(b); }
#else
  double b;
  __device__ __forceinline__ void init() { b = big_value<double>(); }
  __device__ __forceinline__ void take(double x) { b = x < b ? x : b; }
  __device__ __forceinline__ double get() const { return b; }
#endif
};
template <>
struct MinAcc<float> {
  float b;
  __device__ __forceinline__ void init() { b = big_value<float>(); }
  __device__ __forceinline__ void take(float x) { b = fminf(b, x); }
  __device__ __forceinline__ float get() const { return b; }
};

// Argmin with the lowest original control index on ties (feedback mode).
template <typename T>
__device__ __forceinline__ void take_arg(T acc, int cidx, T& best, int& bidx) {
  if (acc < best || (acc == best && cidx < bidx && acc < big_value<T>())) {
    best = acc;
    bidx = cidx;
  }
}

// Evaluate all controls of octant O for the NB nodes of this lane, U entries
// per iteration (the host pads every octant group to a multiple of U).
// MODE 0: min (sweep, into mn); MODE 1: argmin with the lowest original
// index on ties (feedback, into best/bidx).
template <int D, typename T, int NB, int RULE, int COST, bool SLOW, int MODE, int O>
__device__ __forceinline__ void eval_octant(const Nbhd<D, T, NB>& nb, const StencilSmem<D, T>& s,
                                            const int* os, const uint32_t (&fm)[NB],
                                            const T (&ncoef)[NB], const int32_t* ctrl_map,
                                            MinAcc<T> (&mn)[NB], T (&best)[NB], int (&bidx)[NB]) {
  constexpr int NC = 1 << D;
  constexpr int U = (D == 2) ? PHJ_KUNROLL2 : PHJ_UNROLL(D);  // divides the host padding
  const int e0 = os[O], e1 = os[O + 1];
  for (int e = e0; e < e1; e += U) {
    T w[U][NC];
#pragma unroll
    for (int u = 0; u < U; ++u) load_weights<T, NC>(s.w + (int64_t)(e + u) * NC, w[u]);
    T ca[U], cb[U];
    uint32_t nz[U];
    int ci[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ca[u] = T(0);
      cb[u] = T(0);
      nz[u] = 0;
      ci[u] = 0;
      if constexpr (COST == PHJ_COST_CTRL) {
        ca[u] = s.a[e + u];
        cb[u] = s.b[e + u];
      }
      if constexpr (SLOW) nz[u] = s.nz[e + u];
      if constexpr (MODE == 1) ci[u] = ctrl_map[e + u];
    }
    // corner-major order: U*NB independent FMA chains advance one corner per
    // step, so consecutive FP64 instructions never depend on each other
    // (DFMA latency ~8 cycles, 2-cycle issue per warp on sm_100).
    T acc[U][NB];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NB; ++r) acc[u][r] = w[u][0] * corner_val<D, NB, O, 0>(nb, r);
    ChainStep<D, T, NB, O, U, 1>::run(nb, w, acc);
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      T x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        x[u] = finish_cand<T, RULE, COST, SLOW, MODE>(acc[u][r], ca[u], cb[u], ncoef[r], fm[r],
                                                      nz[u]);
      if constexpr (MODE == 0) {
        // pairwise tree over the U candidates, one link into the running min
#pragma unroll
        for (int st = 1; st < U; st <<= 1)
#pragma unroll
          for (int u = 0; u + st < U; u += 2 * st) x[u] = x[u + st] < x[u] ? x[u + st] : x[u];
        mn[r].take(x[0]);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) take_arg<T>(x[u], ci[u], best[r], bidx[r]);
      }
    }
  }
}

template <int D, typename T, int NB, int RULE, int COST, bool SLOW, int MODE, int O = 0>
struct EvalAll {
  __device__ __forceinline__ static void run(const Nbhd<D, T, NB>& nb, const StencilSmem<D, T>& s,
                                             const int* os, const uint32_t (&fm)[NB],
                                             const T (&ncoef)[NB], const int32_t* ctrl_map,
                                             MinAcc<T> (&mn)[NB], T (&best)[NB], int (&bidx)[NB]) {
    eval_octant<D, T, NB, RULE, COST, SLOW, MODE, O>(nb, s, os, fm, ncoef, ctrl_map, mn, best,
                                                     bidx);
    EvalAll<D, T, NB, RULE, COST, SLOW, MODE, O + 1>::run(nb, s, os, fm, ncoef, ctrl_map, mn, best,
                                                         bidx);
  }
};
template <int D, typename T, int NB, int RULE, int COST, bool SLOW, int MODE>
struct EvalAll<D, T, NB, RULE, COST, SLOW, MODE, (1 << D)> {
  __device__ __forceinline__ static void run(const Nbhd<D, T, NB>&, const StencilSmem<D, T>&,
                                             const int*, const uint32_t (&)[NB], const T (&)[NB],
                                             const int32_t*, MinAcc<T> (&)[NB], T (&)[NB],
                                             int (&)[NB]) {}
};

template <int D>
__device__ inline int64_t ext_flat(const phj_grid& g, const int c[3]) {
  if constexpr (D == 2) return (int64_t)(c[0] + 1) * g.strides[0] + (c[1] + 1);
  else return (int64_t)(c[0] + 1) * g.strides[0] + (int64_t)(c[1] + 1) * g.strides[1] + (c[2] + 1);
}

template <int D>
__device__ inline int64_t serial_of(const phj_grid& g, const int c[3]) {
  if constexpr (D == 2) return (int64_t)c[0] * g.shape[1] + c[1];
  else return ((int64_t)c[0] * g.shape[1] + c[1]) * g.shape[2] + c[2];
}

// Load the 3^D neighbourhood (clamped to the ext array) of NB nodes.
template <int D, typename T, int NB>
__device__ __forceinline__ void load_nbhd(const phj_grid& g, const T* __restrict__ v, const int c[3],
                                          Nbhd<D, T, NB>& nb) {
  constexpr int last = D - 1;
  const int64_t xmax = g.ext[last] - 1;
  const int64_t x0 = c[last];  // ext index of the column left of node 0
  if constexpr (D == 2) {
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      int64_t row = (int64_t)min((int64_t)(c[0] + dy), (int64_t)(g.ext[0] - 1)) * g.strides[0];
#pragma unroll
      for (int dx = 0; dx < NB + 2; ++dx) nb.v[dy][dx] = v[row + min(x0 + dx, xmax)];
    }
  } else {
#pragma unroll
    for (int dz = 0; dz < 3; ++dz) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
        int64_t row = (int64_t)min((int64_t)(c[0] + dz), (int64_t)(g.ext[0] - 1)) * g.strides[0] +
                      (int64_t)min((int64_t)(c[1] + dy), (int64_t)(g.ext[1] - 1)) * g.strides[1];
#pragma unroll
        for (int dx = 0; dx < NB + 2; ++dx) nb.v[dz * 3 + dy][dx] = v[row + min(x0 + dx, xmax)];
      }
    }
  }
}

template <typename T>
__device__ inline void atomic_max_change(unsigned long long* addr, T ch) {
  atomicMax(addr, dbits((double)ch));
}

// One block of the value sweep, processed by one warp.  Returns (warp-
// uniform) whether any node changed.
template <int D, typename T, int RULE, int COST>
__device__ bool sweep_block(const SolveParams& p, const StencilSmem<D, T>& s, int blk,
                            const T* __restrict__ vin, T* __restrict__ vout, const int* s_done,
                            unsigned long long* s_max, unsigned long long* gmax_row,
                            unsigned long long& evals) {
  constexpr int NB = Blk<D>::NB;
  constexpr int last = D - 1;
  const unsigned FULL = 0xffffffffu;
  const phj_grid& g = p.g;
  const int lane = threadIdx.x & 31;
  int c[3];
  const bool row_ok = lane_nodes<D>(g, p.tg, blk, lane, c);
  const int64_t f0 = ext_flat<D>(g, c);
  const int cls = p.n_classes > 1 ? c[0] : 0;
  const int* os = s.oct + cls * ((1 << D) + 1);
  const int nadm = p.n_real;

  // Issue every per-node load of the block up front (labels, coefficients,
  // foreign masks, the 3^D value neighbourhood) so their latencies overlap;
  // out-of-range lanes read a clamped in-bounds address and are masked.
  const int64_t nlast = (int64_t)g.ext[0] * g.strides[0] - 1;
  int labv[NB];
  uint32_t fm[NB];
  T ncoef[NB];
  bool in[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    in[r] = row_ok && c[last] + r < g.shape[last];
    const int64_t fr = min(f0 + r, nlast);
    labv[r] = p.lab[fr];
    fm[r] = p.fmask[fr];
    ncoef[r] = (COST == PHJ_COST_NODE && p.coef) ? ((const T*)p.coef)[fr] : (T)p.coef0;
  }
  Nbhd<D, T, NB> nb;
  load_nbhd<D, T, NB>(g, vin, c, nb);
  bool comp[NB], copy[NB];
  bool any_comp = false, any_copy = false;
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    if (!in[r]) labv[r] = -1;
    comp[r] = false;
    copy[r] = false;
    if (labv[r] >= 0) {
      if (s_done[labv[r]] != 0x7fffffff || (COST == PHJ_COST_NODE && ncoef[r] < T(0))) {
        copy[r] = true;
      } else {
        comp[r] = true;
        any_comp = true;
      }
    }
    if (!comp[r]) fm[r] = 0;
    any_copy |= copy[r];
  }
  bool changed = false;
  T mych[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) mych[r] = T(0);
  const int64_t M0 = g.shape[0];
  const bool per0 = g.periodic[0] != 0;
  const int64_t ghost_shift = M0 * g.strides[0];

  if (__any_sync(FULL, any_comp)) {
    MinAcc<T> mn[NB];
    T best[NB];
    int bidx[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      mn[r].init();
      best[r] = big_value<T>();
      bidx[r] = 0;
    }
    uint32_t fmo = 0;
#pragma unroll
    for (int r = 0; r < NB; ++r) fmo |= fm[r];
    if (__any_sync(FULL, fmo != 0))
      EvalAll<D, T, NB, RULE, COST, true, 0>::run(nb, s, os, fm, ncoef, nullptr, mn, best, bidx);
    else
      EvalAll<D, T, NB, RULE, COST, false, 0>::run(nb, s, os, fm, ncoef, nullptr, mn, best, bidx);
#pragma unroll
    for (int r = 0; r < NB; ++r) best[r] = mn[r].get();
    constexpr int CR = (D == 2) ? 1 : 4;  // centre row of the register block
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (!(comp[r] || copy[r])) continue;
      const T old = nb.v[CR][r + 1];
      T nv = old;
      if (comp[r]) {
        evals += (unsigned long long)nadm;
        T cand = best[r];
        if constexpr (COST == PHJ_COST_NODE) {
          cand = (RULE == PHJ_RULE_KRUZKOV) ? fma(ncoef[r], best[r], T(1) - ncoef[r])
                                            : best[r] + ncoef[r];
        }
        if (cand < old) {
          nv = cand;
          mych[r] = old - cand;
          changed = true;
        }
      }
      vout[f0 + r] = nv;
      if (per0) {
        if (c[0] == 0) vout[f0 + r + ghost_shift] = nv;
        else if (c[0] == M0 - 1) vout[f0 + r - ghost_shift] = nv;
      }
    }
  } else if (any_copy) {
    constexpr int CR = (D == 2) ? 1 : 4;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (!copy[r]) continue;
      const T old = nb.v[CR][r + 1];
      vout[f0 + r] = old;
      if (per0) {
        if (c[0] == 0) vout[f0 + r + ghost_shift] = old;
        else if (c[0] == M0 - 1) vout[f0 + r - ghost_shift] = old;
      }
    }
  }

  // per-patch max change
  const bool wchanged = __any_sync(FULL, changed);
  if (wchanged) {
    int l0 = -1;
#pragma unroll
    for (int r = 0; r < NB; ++r)
      if (mych[r] > T(0)) l0 = labv[r];
    const int lref = __reduce_max_sync(FULL, l0);
    bool uni = true;
#pragma unroll
    for (int r = 0; r < NB; ++r) uni &= (mych[r] == T(0)) || (labv[r] == lref);
    if (__all_sync(FULL, uni)) {
      T m = T(0);
#pragma unroll
      for (int r = 0; r < NB; ++r) m = max(m, mych[r]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(FULL, m, off));
      if (lane == 0 && m > T(0)) {
        if (p.R <= kSmemPatchReduce) atomic_max_change(&s_max[lref], m);
        else atomic_max_change(&gmax_row[lref], m);
      }
    } else {
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        if (mych[r] > T(0)) {
          if (p.R <= kSmemPatchReduce) atomic_max_change(&s_max[labv[r]], mych[r]);
          else atomic_max_change(&gmax_row[labv[r]], mych[r]);
        }
      }
    }
  }
  return wchanged;
}

template <int D, typename T, int RULE, int COST>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) solve_kernel(const __grid_constant__ SolveParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::grid_group grid = cg::this_grid();
  StencilSmem<D, T> s = carve_stencil<D, T>(smem, p.n_classes, p.nc);
  int* s_done = (int*)(smem + StencilSmem<D, T>::bytes(p.n_classes, p.nc));
  unsigned long long* s_max = (unsigned long long*)(s_done + ((p.R + 1) / 2 * 2));
  stage_stencil<D, T, RULE>(s, p.n_classes, p.nc, p.oct_start, p.nzmask, p.weights, p.cost);
  for (int i = threadIdx.x; i < p.R; i += blockDim.x)
    s_done[i] = (p.mine == nullptr || p.mine[i]) ? 0x7fffffff : 0;
  __syncthreads();

  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  unsigned long long evals = 0;
  int blocks_done = 0;
  int sw = 0, buf = 0;
  const int nshared = min(p.R, kSmemPatchReduce);
  for (;;) {
    const T* vin = (const T*)p.v[buf];
    T* vout = (T*)p.v[buf ^ 1];
    const int cnt = ld_cg(&p.ws.counts[sw]);
    const int* list = p.ws.list[sw & 1];
    int* cur_flags = p.ws.flags[sw & 1];
    int* nxt_flags = p.ws.flags[(sw + 1) & 1];
    int* nxt_list = p.ws.list[(sw + 1) & 1];
    int* nxt_cnt = &p.ws.counts[sw + 1];
    int* take = &p.ws.take[sw];
    unsigned long long* gmax_row = p.maxch + (int64_t)sw * p.R;
    for (int i = threadIdx.x; i < nshared; i += blockDim.x) s_max[i] = 0ull;
    __syncthreads();
    // Work items are claimed two ahead and their block ids read one ahead, so
    // the claim (atomic) and list-read round trips overlap a block's compute;
    // the first claim of a warp is its static index.
    const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * kWarps;
    int item = gwarp;
    int blk = item < cnt ? __ldcg(&list[item]) : 0;
    int nxt_l0 = 0;
    if (lane == 0) nxt_l0 = nwarps + atomicAdd(take, 1);
    while (item < cnt) {
      const int nxt = __shfl_sync(FULL, nxt_l0, 0);
      const int nblk = nxt < cnt ? __ldcg(&list[nxt]) : 0;
      if (lane == 0 && nxt < cnt) nxt_l0 = nwarps + atomicAdd(take, 1);
      if (lane == 0) cur_flags[blk] = 0;
      const bool ch = sweep_block<D, T, RULE, COST>(p, s, blk, vin, vout, s_done, s_max, gmax_row,
                                                    evals);
      ++blocks_done;
      if (ch && lane < (D == 2 ? 9 : 27))
        mark_neighbour<D>(p.tg, p.g, blk, lane, nxt_flags, nxt_list, nxt_cnt);
      item = nxt;
      blk = nblk;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nshared; i += blockDim.x)
      if (s_max[i]) atomicMax(&gmax_row[i], s_max[i]);
    grid.sync();
    ++sw;
    buf ^= 1;
    int pending = 0;
    for (int i = threadIdx.x; i < p.R; i += blockDim.x) {
      if (s_done[i] == 0x7fffffff) {
        const double mc = __longlong_as_double((long long)ld_cg(&gmax_row[i]));
        if (mc <= p.tol) s_done[i] = sw;
        else pending = 1;
      }
    }
    const int any_pending = __syncthreads_or(pending);
    if (!any_pending || sw >= p.max_sweeps) break;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < p.R; i += blockDim.x) {
      const int d = s_done[i];
      p.patch_sweeps[i] = (d == 0x7fffffff) ? -sw : d;
    }
    if (threadIdx.x == 0) {
      p.info[0] = sw;
      p.info[1] = buf;
    }
  }
  __shared__ unsigned long long s_ev;
  __shared__ int s_blk;
  if (threadIdx.x == 0) {
    s_ev = 0;
    s_blk = 0;
  }
  __syncthreads();
  atomicAdd(&s_ev, evals);
  if (lane == 0) atomicAdd(&s_blk, blocks_done);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(p.evals, s_ev);
    atomicAdd(&p.info[2], s_blk);
  }
}

// Initial active block list: every block holding a node to sweep (solve:
// label >= 0 of a mine patch; transport: a mover).  One warp per block.
template <int D>
__global__ void build_list_kernel(phj_grid g, TileGrid tg, const int16_t* __restrict__ lab,
                                  const uint8_t* __restrict__ mine, int* flags, int* list,
                                  int* count, int want_movers, const int32_t* __restrict__ fb,
                                  const int8_t* __restrict__ kind, unsigned long long* mask0,
                                  unsigned long long mask_all) {
  constexpr int NB = Blk<D>::NB;
  const int lane = threadIdx.x & 31;
  const int blk = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (blk >= tg.total) return;  // whole warp
  int c[3];
  const bool row_ok = lane_nodes<D>(g, tg, blk, lane, c);
  bool any = false;
  if (row_ok) {
    const int64_t f0 = ext_flat<D>(g, c);
    const int64_t s0 = serial_of<D>(g, c);
    for (int r = 0; r < NB; ++r) {
      if (c[D - 1] + r >= g.shape[D - 1]) break;
      if (want_movers) {
        any |= fb[s0 + r] >= 0 && kind[s0 + r] == 0;
      } else {
        const int l = lab[f0 + r];
        any |= l >= 0 && (mine == nullptr || mine[l]);
      }
    }
  }
  if (__any_sync(0xffffffffu, any) && lane == 0) {
    flags[blk] = 1;
    if (mask0) mask0[blk] = mask_all;
    list[atomicAdd(count, 1)] = blk;
  }
}

// ---------------------------------------------------------------------------
// colour transport (patchy.py:183-219): phi_i <- I[phi](x_i + h f(x_i, a*_i))
//
// All R colours in one launch, phi stored colour-major ([R][ext] planes) so
// a warp's reads of one corner of one colour are contiguous.  Each lane owns
// NB nodes of the warp block; a mover's foot cell (entry -> octant, weights)
// is resolved once per block and all 2^D x R corner loads are independent.
// Colour j stops at the first sweep whose max |change| over colour j is
// <= tol (one reference transport_color loop per colour); afterwards it is
// copied through.

struct TransportParams {
  phj_grid g;
  TileGrid tg;
  int n_classes, nc;
  const int32_t* oct_start;
  const int32_t* ctrl;
  const double* weights;
  double* phi[2];
  const int32_t* fb;
  const int8_t* kind;
  const int32_t* ent;  // per internal serial: stencil entry of the mover's feedback, or -1
  int R;
  int64_t plane;       // ext nodes per colour plane
  double tol;
  double act_eps;      // block-colour changes above this re-activate neighbours
  int max_sweeps;
  Workspace ws;
  unsigned long long* maxch;  // [max_sweeps * R], double bits
  int32_t* color_sweeps;      // [R]
  int32_t* info;
  unsigned long long* updates;
};

template <int D>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) transport_kernel(const __grid_constant__ TransportParams p) {
  using B = Blk<D>;
  constexpr int NC = 1 << D;
  constexpr int NB = B::NB;
  constexpr int last = D - 1;
  extern __shared__ __align__(16) unsigned char smem[];
  cg::grid_group grid = cg::this_grid();
  const int nent = p.n_classes * p.nc;
  const int R = p.R;
  // weights corner-major with an odd pitch: lanes of a warp hold different
  // entries, so [k][e] keeps their reads on distinct banks
  const int wpitch = nent | 1;
  double* s_w = (double*)smem;                                                     // [NC][wpitch]
  unsigned long long* s_max = (unsigned long long*)(s_w + (int64_t)wpitch * NC);   // [R]
  int* s_done = (int*)(s_max + R);                                                 // [R]
  signed char* s_oct = (signed char*)(s_done + R);                                 // [nent]
  for (int i = threadIdx.x; i < nent * NC; i += blockDim.x)
    s_w[(i % NC) * wpitch + i / NC] = p.weights[i];
  for (int i = threadIdx.x; i < R; i += blockDim.x) s_done[i] = 0x7fffffff;
  for (int cls = 0; cls < p.n_classes; ++cls) {
    const int32_t* os = p.oct_start + cls * (NC + 1);
    for (int e = os[0] + threadIdx.x; e < os[NC]; e += blockDim.x) {
      int oc = 0;
      while (oc < NC - 1 && e >= os[oc + 1]) ++oc;
      s_oct[e] = (signed char)oc;
    }
  }
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const phj_grid& g = p.g;
  const int lane = threadIdx.x & 31;
  const int64_t M0 = g.shape[0];
  const bool per0 = g.periodic[0] != 0;
  const int64_t ghost_shift = M0 * g.strides[0];
  int64_t coff[NC];  // corner offsets from the lower corner (bit ax = +stride_ax)
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    int64_t o = 0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax)
      if ((k >> ax) & 1) o += g.strides[ax];
    coff[k] = o;
  }
  unsigned long long upd = 0;
  int sw = 0, buf = 0;
  for (;;) {
    const double* pin = p.phi[buf];
    double* pout = p.phi[buf ^ 1];
    const int cnt = ld_cg(&p.ws.counts[sw]);
    const int* list = p.ws.list[sw & 1];
    int* cur_flags = p.ws.flags[sw & 1];
    unsigned long long* cur_mask = p.ws.cmask[sw & 1];
    int* take = &p.ws.take[sw];
    for (int i = threadIdx.x; i < R; i += blockDim.x) s_max[i] = 0ull;
    __syncthreads();
    const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * kWarps;
    int item = gwarp;
    while (item < cnt) {
      int nxt_l0 = 0;
      if (lane == 0) nxt_l0 = nwarps + atomicAdd(take, 1);
      const int blk = __ldcg(&list[item]);
      // colours active in this block: those a neighbour block changed in the
      // previous sweep (exact per colour, like the block skipping)
      unsigned long long cm = 0;
      if (lane == 0) {
        cm = __ldcg(&cur_mask[blk]);
        cur_mask[blk] = 0ull;
        cur_flags[blk] = 0;
      }
      cm = __shfl_sync(FULL, cm, 0);
      int c[3];
      const bool row_ok = lane_nodes<D>(g, p.tg, blk, lane, c);
      const int64_t f0 = ext_flat<D>(g, c);
      const int64_t s0 = serial_of<D>(g, c);
      int e[NB];
      int64_t base[NB];
      double w[NB][NC];
      bool any = false;
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        const bool in = row_ok && c[last] + r < g.shape[last];
        e[r] = in ? __ldg(&p.ent[s0 + r]) : -1;
        base[r] = f0 + r;
        if (e[r] >= 0) {
          const int oc = s_oct[e[r]];
#pragma unroll
          for (int ax = 0; ax < D; ++ax)
            if (!((oc >> ax) & 1)) base[r] -= g.strides[ax];
#pragma unroll
          for (int k = 0; k < NC; ++k) w[r][k] = s_w[k * wpitch + e[r]];
          any = true;
          ++upd;
        }
      }
      unsigned long long changed = 0;
      if (__any_sync(FULL, any)) {
        const bool masked = R <= 64;
        unsigned long long todo = cm;
        for (int jj = 0; masked ? (todo != 0ull) : (jj < R); ++jj) {
          int j = jj;
          if (masked) {
            j = __ffsll((long long)todo) - 1;
            todo &= todo - 1;
          }
          const bool live = s_done[j] == 0x7fffffff;
          const double* pj = pin + (int64_t)j * p.plane;
          double* qj = pout + (int64_t)j * p.plane;
          double lmax = 0.0;
          double acc[NB], old[NB];
#pragma unroll
          for (int r = 0; r < NB; ++r) {
            acc[r] = 0.0;
            old[r] = 0.0;
            if (e[r] >= 0) {
              old[r] = pj[f0 + r];
#pragma unroll
              for (int k = 0; k < NC; ++k) acc[r] = fma(w[r][k], pj[base[r] + coff[k]], acc[r]);
            }
          }
#pragma unroll
          for (int r = 0; r < NB; ++r) {
            if (e[r] < 0) continue;
            const double nv = live ? acc[r] : old[r];
            lmax = fmax(lmax, fabs(old[r] - nv));
            qj[f0 + r] = nv;
            if (per0) {
              if (c[0] == 0) qj[f0 + r + ghost_shift] = nv;
              else if (c[0] == M0 - 1) qj[f0 + r - ghost_shift] = nv;
            }
          }
          if (__any_sync(FULL, lmax > 0.0)) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) lmax = fmax(lmax, __shfl_xor_sync(FULL, lmax, off));
            if (lane == 0) atomicMax(&s_max[j], dbits(lmax));
            // activity threshold: changes <= act_eps (a small fraction of the
            // stopping tolerance) do not re-activate the neighbourhood
            if (lmax > p.act_eps) changed |= (j < 64) ? (1ull << j) : ~0ull;
          }
        }
      }
      if (changed && lane < (D == 2 ? 9 : 27))
        mark_neighbour_mask<D>(p.tg, g, blk, lane, changed, p.ws.cmask[(sw + 1) & 1],
                               p.ws.list[(sw + 1) & 1], &p.ws.counts[sw + 1]);
      item = __shfl_sync(FULL, nxt_l0, 0);
    }
    __syncthreads();
    unsigned long long* grow = p.maxch + (int64_t)sw * R;
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      if (s_max[i]) atomicMax(&grow[i], s_max[i]);
    grid.sync();
    ++sw;
    buf ^= 1;
    int pending = 0;
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      if (s_done[i] == 0x7fffffff) {
        const double mc = __longlong_as_double((long long)ld_cg(&grow[i]));
        if (mc <= p.tol) s_done[i] = sw;
        else pending = 1;
      }
    }
    const int any_pending = __syncthreads_or(pending);
    if (!any_pending || sw >= p.max_sweeps) break;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      p.color_sweeps[i] = (s_done[i] == 0x7fffffff) ? -sw : s_done[i];
    if (threadIdx.x == 0) {
      p.info[0] = sw;
      p.info[1] = buf;
    }
  }
  __shared__ unsigned long long s_up;
  if (threadIdx.x == 0) s_up = 0;
  __syncthreads();
  atomicAdd(&s_up, upd);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(p.updates, s_up);
}

// Mover -> stencil entry of its feedback control (patchy.py:165-180: movers
// are free nodes with a defined feedback and an admissible foot).
template <int D>
__global__ void transport_entries_kernel(phj_grid g, int ncls, int nc,
                                         const int32_t* __restrict__ oct_start,
                                         const int32_t* __restrict__ ctrl,
                                         const int32_t* __restrict__ fb,
                                         const int8_t* __restrict__ kind, int32_t* __restrict__ ent) {
  extern __shared__ int s_inv[];  // [ncls][nc]
  constexpr int NC = 1 << D;
  for (int i = threadIdx.x; i < ncls * nc; i += blockDim.x) s_inv[i] = -1;
  __syncthreads();
  for (int cls = 0; cls < ncls; ++cls) {
    const int32_t* os = oct_start + cls * (NC + 1);
    for (int e = os[0] + threadIdx.x; e < os[NC]; e += blockDim.x) s_inv[cls * nc + ctrl[e]] = e;
    __syncthreads();
  }
  const int64_t N = g.shape[0] * g.shape[1] * (D == 3 ? g.shape[2] : 1);
  const int64_t plane = N / g.shape[0];
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < N;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int a = fb[s];
    int e = -1;
    if (a >= 0 && a < nc && kind[s] == 0) e = s_inv[(ncls > 1 ? (int)(s / plane) : 0) * nc + a];
    ent[s] = e;
  }
}

// ---------------------------------------------------------------------------
// feedback (extract_feedback, solver.py:413-443; feedback_batch _kernels.py:109-167)

struct FeedbackParams {
  phj_grid g;
  TileGrid tg;
  int n_classes, nc, n_real;
  const int32_t* oct_start;
  const int32_t* ctrl;
  const uint32_t* nzmask;
  const double* weights;
  const double* cost;
  const void* v;
  const int8_t* kind;
  const uint32_t* fmask;
  const void* coef;
  double coef0;
  double unreach;
  int32_t* out;
  unsigned long long* evals;
};

template <int D, typename T, int RULE, int COST>
__global__ void __launch_bounds__(kThreads) feedback_kernel(const __grid_constant__ FeedbackParams p) {
  constexpr int NB = Blk<D>::NB;
  constexpr int last = D - 1;
  extern __shared__ __align__(16) unsigned char smem[];
  StencilSmem<D, T> s = carve_stencil<D, T>(smem, p.n_classes, p.nc);
  int* s_ctrl = (int*)(smem + StencilSmem<D, T>::bytes(p.n_classes, p.nc));
  stage_stencil<D, T, RULE>(s, p.n_classes, p.nc, p.oct_start, p.nzmask, p.weights, p.cost);
  for (int i = threadIdx.x; i < p.n_classes * p.nc; i += blockDim.x) s_ctrl[i] = p.ctrl[i];
  __syncthreads();
  const phj_grid& g = p.g;
  const int lane = threadIdx.x & 31;
  unsigned long long ev = 0;
  const T* v = (const T*)p.v;
  for (int blk = blockIdx.x * kWarps + (threadIdx.x >> 5); blk < p.tg.total;
       blk += gridDim.x * kWarps) {
    int c[3];
    const bool row_ok = lane_nodes<D>(g, p.tg, blk, lane, c);
    const int64_t f0 = ext_flat<D>(g, c);
    const int64_t s0 = serial_of<D>(g, c);
    const int cls = p.n_classes > 1 ? c[0] : 0;
    const int* os = s.oct + cls * ((1 << D) + 1);
    const int nadm = p.n_real;
    bool comp[NB];
    uint32_t fm[NB];
    T ncoef[NB];
    bool any = false;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const bool in = row_ok && c[last] + r < g.shape[last];
      comp[r] = false;
      fm[r] = 0;
      ncoef[r] = (T)p.coef0;
      if (in) {
        p.out[s0 + r] = -1;
        if (COST == PHJ_COST_NODE && p.coef) ncoef[r] = ((const T*)p.coef)[f0 + r];
        const bool adm = !(COST == PHJ_COST_NODE && ncoef[r] < T(0));
        if (p.kind[s0 + r] == 0 && (double)v[f0 + r] < p.unreach && adm) {
          comp[r] = true;
          fm[r] = p.fmask[f0 + r];
          any = true;
        }
      }
    }
    if (!__any_sync(0xffffffffu, any)) continue;
    Nbhd<D, T, NB> nb;
    load_nbhd<D, T, NB>(g, v, c, nb);
    MinAcc<T> mn[NB];
    T best[NB];
    int bidx[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      best[r] = big_value<T>();
      bidx[r] = 0x7fffffff;
    }
    EvalAll<D, T, NB, RULE, COST, true, 1>::run(nb, s, os, fm, ncoef, s_ctrl, mn, best, bidx);
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (!comp[r]) continue;
      ev += nadm;
      p.out[s0 + r] = (best[r] < big_value<T>()) ? bidx[r] : -1;
    }
  }
  __shared__ unsigned long long s_ev;
  if (threadIdx.x == 0) s_ev = 0;
  __syncthreads();
  atomicAdd(&s_ev, ev);
  __syncthreads();
  if (threadIdx.x == 0 && p.evals) atomicAdd(p.evals, s_ev);
}

// ---------------------------------------------------------------------------
// foreign masks

template <int D>
__global__ void fmask_kernel(phj_grid g, const int16_t* __restrict__ lab,
                             const uint8_t* __restrict__ hard, uint32_t* __restrict__ fmask) {
  const int64_t N = g.shape[0] * g.shape[1] * (D == 3 ? g.shape[2] : 1);
  for (int64_t sidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sidx < N;
       sidx += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = sidx;
    int c[3] = {0, 0, 0};
    for (int ax = D - 1; ax >= 0; --ax) {
      c[ax] = (int)(rem % g.shape[ax]);
      rem /= g.shape[ax];
    }
    const int64_t f = ext_flat<D>(g, c);
    uint32_t m = 0;
    const int own = lab ? lab[f] : 0;
    if (!lab || own >= 0) {
      constexpr int NP = (D == 2) ? 9 : 27;
      for (int q = 0; q < NP; ++q) {
        int64_t off = 0;
        if (D == 2) {
          off = (int64_t)(q / 3 - 1) * g.strides[0] + (q % 3 - 1);
        } else {
          off = (int64_t)(q / 9 - 1) * g.strides[0] + (int64_t)((q / 3) % 3 - 1) * g.strides[1] +
                (q % 3 - 1);
        }
        bool foreign;
        if (lab) {
          const int l = lab[f + off];
          foreign = !(l == own || l == PHJ_LAB_TARGET || l == PHJ_LAB_FIXED);
        } else {
          foreign = hard[f + off] != 0;
        }
        if (foreign) m |= (1u << q);
      }
    }
    fmask[f] = m;
  }
}

}  // namespace phj

using namespace phj;

// ---------------------------------------------------------------------------
// host side

static int g_num_sms = 0;

extern "C" int phj_num_sms(void) {
  if (g_num_sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

extern "C" int64_t phj_blocks_total(const phj_grid* g) {
  if (!g) return -1;
  return g->dim == 2 ? make_tile_grid<2>(*g).total : make_tile_grid<3>(*g).total;
}

extern "C" int64_t phj_solve_workspace_bytes(const phj_grid* g, int32_t n_patches,
                                             int32_t max_sweeps) {
  (void)n_patches;
  if (!g) return -1;
  return g->dim == 2 ? workspace_bytes<2>(*g, max_sweeps) : workspace_bytes<3>(*g, max_sweeps);
}

// Cooperative persistent launch: as many CTAs as are co-resident, capped by
// the work (8 warps per CTA, one block per warp per step).
template <typename K>
static int coop_launch(K kernel, int want_blocks, size_t smem, void** args, cudaStream_t stream,
                       int* launched) {
  PHJ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  PHJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem));
  if (occ < 1) {
    phj_set_error("kernel cannot be resident (smem %zu B)", smem);
    return PHJ_ERR_UNSUPPORTED;
  }
  int blocks = std::min(want_blocks, occ * phj_num_sms());
  if (const char* cap = getenv("PHJ_MAX_BLOCKS")) blocks = std::min(blocks, atoi(cap));
  if (blocks < 1) blocks = 1;
  if (launched) *launched = blocks;
  PHJ_CUDA(cudaLaunchCooperativeKernel((void*)kernel, dim3(blocks), dim3(kThreads), args, smem,
                                       stream));
  phj_count_launch(1);
  return PHJ_OK;
}

template <int D, typename T, int RULE, int COST>
static int solve_impl(const phj_solve_args* a) {
  cudaStream_t stream = (cudaStream_t)a->stream;
  SolveParams p;
  p.g = a->grid;
  p.tg = make_tile_grid<D>(a->grid);
  p.n_classes = a->st.n_classes;
  p.nc = a->st.n_controls;
  p.n_real = a->st.n_real;
  p.oct_start = a->st.oct_start;
  p.nzmask = a->st.nzmask;
  p.weights = a->st.weights;
  p.cost = a->st.cost;
  p.v[0] = a->v0;
  p.v[1] = a->v1;
  p.lab = a->lab;
  p.fmask = a->fmask;
  p.coef = a->coef;
  p.coef0 = a->coef0;
  p.R = a->n_patches;
  p.max_sweeps = a->max_sweeps;
  p.mine = a->mine;
  p.tol = a->tol;
  p.ws = carve<D>(a->grid, a->workspace, a->max_sweeps);
  p.maxch = (unsigned long long*)a->maxch_hist;
  p.patch_sweeps = a->patch_sweeps;
  p.evals = a->evals;
  p.info = a->info;
  const int64_t ws_bytes = workspace_bytes<D>(a->grid, a->max_sweeps);
  PHJ_CUDA(cudaMemsetAsync(a->workspace, 0, ws_bytes, stream));
  PHJ_CUDA(cudaMemsetAsync(a->maxch_hist, 0, sizeof(double) * (size_t)a->max_sweeps * a->n_patches,
                           stream));
  PHJ_CUDA(cudaMemsetAsync(a->evals, 0, sizeof(unsigned long long), stream));
  PHJ_CUDA(cudaMemsetAsync(a->info, 0, 4 * sizeof(int32_t), stream));
  build_list_kernel<D><<<(p.tg.total + kWarps - 1) / kWarps, kThreads, 0, stream>>>(
      p.g, p.tg, p.lab, p.mine, p.ws.flags[0], p.ws.list[0], p.ws.counts, 0, nullptr, nullptr,
      nullptr, 0ull);
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  size_t smem = (size_t)StencilSmem<D, T>::bytes(p.n_classes, p.nc) +
                (size_t)((p.R + 1) / 2 * 2) * 4 + (size_t)std::min(p.R, kSmemPatchReduce) * 8 + 16;
  void* args[] = {(void*)&p};
  int launched = 0;
  int rc = coop_launch(solve_kernel<D, T, RULE, COST>, (p.tg.total + kWarps - 1) / kWarps, smem,
                       args, stream, &launched);
  if (rc) return rc;
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}

extern "C" int phj_solve(const phj_solve_args* a) {
  if (!a || (a->grid.dim != 2 && a->grid.dim != 3) || !a->v0 || !a->v1 || !a->lab || !a->fmask ||
      !a->workspace || !a->maxch_hist || !a->patch_sweeps || !a->evals || !a->info) {
    phj_set_error("phj_solve: missing argument");
    return PHJ_ERR_ARG;
  }
  if (a->n_patches < 1 || a->n_patches > kMaxPatches || a->max_sweeps < 1) {
    phj_set_error("phj_solve: n_patches must be in [1, %d], max_sweeps >= 1", kMaxPatches);
    return PHJ_ERR_ARG;
  }
  if (a->grid.periodic[1] || a->grid.periodic[2]) {
    phj_set_error("phj_solve: only internal axis 0 may be periodic");
    return PHJ_ERR_UNSUPPORTED;
  }
  if (a->grid.dim == 2 && a->st.n_classes != 1) {
    phj_set_error("phj_solve: stencil classes need a 3D grid (class axis = internal axis 0)");
    return PHJ_ERR_UNSUPPORTED;
  }
  if (a->rule == PHJ_RULE_REF && a->dtype == PHJ_F32) {
    phj_set_error("phj_solve: the reference (sentinel) rule is fp64 only");
    return PHJ_ERR_UNSUPPORTED;
  }
  const int D = a->grid.dim, f32 = a->dtype == PHJ_F32, krz = a->rule == PHJ_RULE_KRUZKOV,
            cc = a->st.cost_mode == PHJ_COST_CTRL;
#define PHJ_DISPATCH(DD, TT, RR, CC)                                                        \
  if (D == DD && f32 == (sizeof(TT) == 4) && krz == (RR == PHJ_RULE_KRUZKOV) &&           \
      cc == (CC == PHJ_COST_CTRL))                                                         \
    return solve_impl<DD, TT, RR, CC>(a);
  PHJ_DISPATCH(2, double, PHJ_RULE_REF, PHJ_COST_NODE)
  PHJ_DISPATCH(2, double, PHJ_RULE_REF, PHJ_COST_CTRL)
  PHJ_DISPATCH(2, double, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_DISPATCH(2, double, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
  PHJ_DISPATCH(2, float, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_DISPATCH(2, float, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
  PHJ_DISPATCH(3, double, PHJ_RULE_REF, PHJ_COST_NODE)
  PHJ_DISPATCH(3, double, PHJ_RULE_REF, PHJ_COST_CTRL)
  PHJ_DISPATCH(3, double, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_DISPATCH(3, double, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
  PHJ_DISPATCH(3, float, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_DISPATCH(3, float, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
#undef PHJ_DISPATCH
  phj_set_error("phj_solve: unsupported combination");
  return PHJ_ERR_UNSUPPORTED;
}

template <int D>
static int transport_impl(const phj_transport_args* a) {
  cudaStream_t stream = (cudaStream_t)a->stream;
  TransportParams p;
  p.g = a->grid;
  p.tg = make_tile_grid<D>(a->grid);
  p.n_classes = a->st.n_classes;
  p.nc = a->st.n_controls;
  p.oct_start = a->st.oct_start;
  p.ctrl = a->st.ctrl;
  p.weights = a->st.weights;
  p.phi[0] = a->phi0;
  p.phi[1] = a->phi1;
  p.fb = a->fb;
  p.kind = a->kind;
  p.ent = a->ent_scratch;
  p.R = a->n_colors;
  p.plane = a->grid.ext[0] * a->grid.ext[1] * (D == 3 ? a->grid.ext[2] : 1);
  p.tol = a->tol;
  p.act_eps = a->act_eps;
  p.max_sweeps = a->max_sweeps;
  p.ws = carve<D>(a->grid, a->workspace, a->max_sweeps);
  p.maxch = (unsigned long long*)a->maxch_hist;
  p.color_sweeps = a->color_sweeps;
  p.info = a->info;
  p.updates = a->updates;
  const int64_t ws_bytes = workspace_bytes<D>(a->grid, a->max_sweeps);
  PHJ_CUDA(cudaMemsetAsync(a->workspace, 0, ws_bytes, stream));
  PHJ_CUDA(cudaMemsetAsync(a->maxch_hist, 0, 8 * (size_t)a->max_sweeps * p.R, stream));
  PHJ_CUDA(cudaMemsetAsync(a->info, 0, 4 * sizeof(int32_t), stream));
  PHJ_CUDA(cudaMemsetAsync(a->updates, 0, sizeof(unsigned long long), stream));
  {
    const int64_t N = p.g.shape[0] * p.g.shape[1] * (D == 3 ? p.g.shape[2] : 1);
    const int nb = (int)std::min<int64_t>((N + 255) / 256, 16 * phj_num_sms());
    const size_t sm = (size_t)p.n_classes * p.nc * 4;
    auto k = transport_entries_kernel<D>;
    PHJ_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k<<<std::max(nb, 1), 256, sm, stream>>>(p.g, p.n_classes, p.nc, p.oct_start, p.ctrl, p.fb,
                                            p.kind, a->ent_scratch);
    phj_count_launch(1);
  }
  build_list_kernel<D><<<(p.tg.total + kWarps - 1) / kWarps, kThreads, 0, stream>>>(
      p.g, p.tg, nullptr, nullptr, p.ws.flags[0], p.ws.list[0], p.ws.counts, 1, p.fb, p.kind,
      p.ws.cmask[0], p.R >= 64 ? ~0ull : ((1ull << p.R) - 1ull));
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  const int nent = p.n_classes * p.nc;
  size_t smem = (size_t)(nent | 1) * (1 << D) * 8 + (size_t)p.R * 12 + (size_t)nent + 16;
  void* args[] = {(void*)&p};
  return coop_launch(transport_kernel<D>, (p.tg.total + kWarps - 1) / kWarps, smem, args, stream,
                     nullptr);
}

extern "C" int phj_transport(const phj_transport_args* a) {
  if (!a || !a->phi0 || !a->phi1 || !a->fb || !a->kind || !a->ent_scratch || !a->workspace ||
      !a->info || !a->updates || a->max_sweeps < 1) {
    phj_set_error("phj_transport: missing argument");
    return PHJ_ERR_ARG;
  }
  if (a->grid.periodic[1] || a->grid.periodic[2]) {
    phj_set_error("phj_transport: only internal axis 0 may be periodic");
    return PHJ_ERR_UNSUPPORTED;
  }
  if (a->n_colors < 1 || a->n_colors > 4096 || !a->maxch_hist || !a->color_sweeps) {
    phj_set_error("phj_transport: n_colors must be in [1, 4096]");
    return PHJ_ERR_ARG;
  }
  return a->grid.dim == 2 ? transport_impl<2>(a) : transport_impl<3>(a);
}

template <int D, typename T, int RULE, int COST>
static int feedback_impl(const phj_grid* g, const phj_stencil* st, const void* v,
                         const int8_t* kind, const uint32_t* fmask, const void* coef,
                         double coef0, double unreach, int32_t* out, unsigned long long* evals,
                         cudaStream_t stream) {
  FeedbackParams p;
  p.g = *g;
  p.tg = make_tile_grid<D>(*g);
  p.n_classes = st->n_classes;
  p.nc = st->n_controls;
  p.n_real = st->n_real;
  p.oct_start = st->oct_start;
  p.ctrl = st->ctrl;
  p.nzmask = st->nzmask;
  p.weights = st->weights;
  p.cost = st->cost;
  p.v = v;
  p.kind = kind;
  p.fmask = fmask;
  p.coef = coef;
  p.coef0 = coef0;
  p.unreach = unreach;
  p.out = out;
  p.evals = evals;
  size_t smem = (size_t)StencilSmem<D, T>::bytes(p.n_classes, p.nc) +
                (size_t)p.n_classes * p.nc * 4 + 16;
  auto k = feedback_kernel<D, T, RULE, COST>;
  PHJ_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = std::min((p.tg.total + kWarps - 1) / kWarps, 8 * phj_num_sms());
  k<<<blocks, kThreads, smem, stream>>>(p);
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}

extern "C" int phj_feedback(const phj_grid* g, const phj_stencil* st, int32_t dtype, int32_t rule,
                            const void* v, const int8_t* kind, const uint32_t* fmask,
                            const void* coef, double coef0, double unreach, int32_t* out,
                            unsigned long long* evals, void* stream) {
  if (!g || !st || !v || !kind || !fmask || !out) {
    phj_set_error("phj_feedback: missing argument");
    return PHJ_ERR_ARG;
  }
  if (rule == PHJ_RULE_REF && dtype == PHJ_F32) {
    phj_set_error("phj_feedback: the reference (sentinel) rule is fp64 only");
    return PHJ_ERR_UNSUPPORTED;
  }
  if (g->dim == 2 && st->n_classes != 1) {
    phj_set_error("phj_feedback: stencil classes need a 3D grid");
    return PHJ_ERR_UNSUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int D = g->dim, f32 = dtype == PHJ_F32, krz = rule == PHJ_RULE_KRUZKOV,
            cc = st->cost_mode == PHJ_COST_CTRL;
#define PHJ_FB(DD, TT, RR, CC)                                                             \
  if (D == DD && f32 == (sizeof(TT) == 4) && krz == (RR == PHJ_RULE_KRUZKOV) &&           \
      cc == (CC == PHJ_COST_CTRL))                                                         \
    return feedback_impl<DD, TT, RR, CC>(g, st, v, kind, fmask, coef, coef0, unreach, out, \
                                         evals, s);
  PHJ_FB(2, double, PHJ_RULE_REF, PHJ_COST_NODE)
  PHJ_FB(2, double, PHJ_RULE_REF, PHJ_COST_CTRL)
  PHJ_FB(2, double, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_FB(2, double, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
  PHJ_FB(2, float, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_FB(2, float, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
  PHJ_FB(3, double, PHJ_RULE_REF, PHJ_COST_NODE)
  PHJ_FB(3, double, PHJ_RULE_REF, PHJ_COST_CTRL)
  PHJ_FB(3, double, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_FB(3, double, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
  PHJ_FB(3, float, PHJ_RULE_KRUZKOV, PHJ_COST_NODE)
  PHJ_FB(3, float, PHJ_RULE_KRUZKOV, PHJ_COST_CTRL)
#undef PHJ_FB
  phj_set_error("phj_feedback: unsupported combination");
  return PHJ_ERR_UNSUPPORTED;
}

static int fmask_launch(const phj_grid* g, const int16_t* lab, const uint8_t* hard,
                        uint32_t* fmask, cudaStream_t s) {
  const int64_t N = g->shape[0] * g->shape[1] * (g->dim == 3 ? g->shape[2] : 1);
  int blocks = (int)std::min<int64_t>((N + 255) / 256, 32 * phj_num_sms());
  if (blocks < 1) blocks = 1;
  if (g->dim == 2) fmask_kernel<2><<<blocks, 256, 0, s>>>(*g, lab, hard, fmask);
  else fmask_kernel<3><<<blocks, 256, 0, s>>>(*g, lab, hard, fmask);
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}

extern "C" int phj_fmask_from_labels(const phj_grid* g, const int16_t* lab, uint32_t* fmask,
                                     void* stream) {
  if (!g || !lab || !fmask) {
    phj_set_error("phj_fmask_from_labels: missing argument");
    return PHJ_ERR_ARG;
  }
  return fmask_launch(g, lab, nullptr, fmask, (cudaStream_t)stream);
}

extern "C" int phj_fmask_from_hard(const phj_grid* g, const uint8_t* hard, uint32_t* fmask,
                                   void* stream) {
  if (!g || !hard || !fmask) {
    phj_set_error("phj_fmask_from_hard: missing argument");
    return PHJ_ERR_ARG;
  }
  return fmask_launch(g, nullptr, hard, fmask, (cudaStream_t)stream);
}
