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
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "phj_common.cuh"

namespace cg = cooperative_groups;

namespace phj {

// Optional per-phase cycle accounting (diagnostic builds only, -DPHJ_TIMING).
#ifdef PHJ_TIMING
// visit timeline of the asynchronous kernels: visits per 20 us bin since the
// first visit of the launch (diagnostic builds only)
__device__ unsigned int g_visit_bins[4096];
__device__ unsigned long long g_visit_kind[4];  // solve visits by outcome: 0 / small / big change
__device__ unsigned long long g_t0;
__device__ __forceinline__ void timeline_visit() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  unsigned long long t0 = *(volatile unsigned long long*)&g_t0;
  if (t0 == 0ull) {
    atomicCAS(&g_t0, 0ull, t);
    t0 = *(volatile unsigned long long*)&g_t0;
  }
  const unsigned long long b = (t - t0) / 20000ull;
  atomicAdd(&g_visit_bins[b < 4095 ? b : 4095], 1u);
}
__device__ unsigned long long g_phase_cycles[12];
struct PhaseTimer {
  unsigned long long acc[12];
  long long prev;
  __device__ void start() {
    for (int i = 0; i < 12; ++i) acc[i] = 0;
    prev = clock64();
  }
  __device__ void mark(int i) {
    long long t = clock64();
    acc[i] += (unsigned long long)(t - prev);
    prev = t;
  }
};
#else
struct PhaseTimer {
  __device__ void start() {}
  __device__ void mark(int) {}
};
#endif

struct SolveParams {
  phj_grid g;
  TileGrid tg;
  int n_classes, nc, n_real;
  const int32_t* oct_start;
  const int32_t* ctrl;  // original control per stencil entry (padding detection)
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
  unsigned long long* pcount;  // [R][3] node relaxations, logical, executed evals (or NULL)
  int32_t* info;
  int prune;  // exact octant pruning on (PHJ_SOLVE_NO_PRUNE clears it)
  double act;  // a node change marks the neighbour blocks only if > act (0 = exact)
  int inner;   // block-local relaxations per sweep (>= 1)
  // AO3 conical reduction (NULL ao3_fb = off)
  const int32_t* ao3_fb;
  const unsigned long long* ao3_mask;
  const int32_t* ao3_count;
  int ao3_words;
  // value-ordered pass (solve_kernel): sweeps < n_band visit band_list rows
  // (b: relax block b, -b-1: copy its nodes to the other buffer); sweep
  // n_band visits row n_band (every block of the pass) as a normal sweep;
  // band_only ends the launch there (the asynchronous schedule continues)
  const int32_t* band_list;
  const int32_t* band_off;
  int n_band;
  int band_only;
};

__device__ __forceinline__ int entry_block(int e) { return e < 0 ? -e - 1 : e; }

template <int D, typename T>
struct StencilSmem {
  T* w;          // [nent][2^D]
  T* a;          // [nent] beta (KRUZKOV) or cost (REF), COST_CTRL only
  T* b;          // [nent] 1 - beta
  uint32_t* nz;  // [nent]
  int* oct;      // [ncls][2^D + 1]
  int* oreal;    // [ncls][2^D] real (non-padding) entries per octant (solve kernels)
  static __host__ __device__ int64_t bytes(int ncls, int nc) {
    int64_t nent = (int64_t)ncls * nc;
    int64_t b = nent * (1 << D) * sizeof(T) + 2 * nent * sizeof(T);
    b = (b + 15) / 16 * 16;
    b += nent * 4 + (int64_t)ncls * ((1 << D) + 1) * 4 + (int64_t)ncls * (1 << D) * 4;
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
  s.oreal = s.oct + (int64_t)ncls * ((1 << D) + 1);
  return s;
}

// Entries [src0, src0 + n) of the global stencil into entries [dst0, ...) of
// a staged copy, threads t0, t0 + tstride, ...
template <int D, typename T, int RULE>
__device__ inline void stage_entries(const StencilSmem<D, T>& s, int dst0, int src0, int n,
                                     int t0, int tstride, const uint32_t* nzmask,
                                     const double* weights, const double* cost) {
  constexpr int NC = 1 << D;
  for (int i = t0; i < n; i += tstride) {
    const int src = src0 + i, dst = dst0 + i;
    // weights in T with the last nonzero one set so that their sequential
    // sum in T is exactly 1 (I[1] == 1, see dynamics._weights_for)
    T w[NC];
    int last = 0;
    for (int k = 0; k < NC; ++k) {
      w[k] = (T)weights[(int64_t)src * NC + k];
      if (w[k] != T(0)) last = k;
    }
    T sum = T(0);
    for (int k = 0; k < last; ++k) sum = sum + w[k];
    w[last] = T(1) - sum;
    for (int k = 0; k < NC; ++k) s.w[(int64_t)dst * NC + k] = w[k];
    s.nz[dst] = nzmask[src];
    const double c = cost ? cost[src] : 0.0;
    if (RULE == PHJ_RULE_KRUZKOV) {
      // 1 - beta is exact in T (Sterbenz), so beta * 1 + (1 - beta) == 1
      const T beta = (T)exp(-c);
      s.a[dst] = beta;
      s.b[dst] = T(1) - beta;
    } else {
      s.a[dst] = (T)c;
      s.b[dst] = (T)0;
    }
  }
}

// Shared-memory stencil area of the solve kernel: the whole stencil for a
// single class, else one private single-class slot per warp (multi-class
// stencils -- one class per heading -- are too big to stage per CTA and a
// warp block lies in one class).
template <int D, typename T>
__host__ __device__ inline int64_t solve_stencil_slot(int nc) {
  return align_up(StencilSmem<D, T>::bytes(1, nc), 16);
}
template <int D, typename T>
__host__ __device__ inline int64_t solve_stencil_bytes(int ncls, int nc) {
  return ncls > 1 ? kWarps * solve_stencil_slot<D, T>(nc) : StencilSmem<D, T>::bytes(ncls, nc);
}

// Real (non-padding) entries of octant group [e0, e1): the host pads a group
// by repeating its last entry (dynamics.build_stencil), every control lies in
// one octant, so an entry is padding iff it repeats its predecessor's control.
__device__ inline int real_entries(const int32_t* ctrl, int e0, int e1) {
  if (!ctrl) return e1 - e0;
  int n = 0;
  for (int e = e0; e < e1; ++e) n += (e == e0 || __ldg(&ctrl[e]) != __ldg(&ctrl[e - 1]));
  return n;
}

template <int D, typename T, int RULE>
__device__ inline void stage_stencil(const StencilSmem<D, T>& s, int ncls, int nc,
                                     const int32_t* oct_start, const uint32_t* nzmask,
                                     const double* weights, const double* cost,
                                     const int32_t* ctrl = nullptr) {
  constexpr int NC = 1 << D;
  stage_entries<D, T, RULE>(s, 0, 0, ncls * nc, threadIdx.x, blockDim.x, nzmask, weights, cost);
  for (int i = threadIdx.x; i < ncls * (NC + 1); i += blockDim.x) s.oct[i] = oct_start[i];
  for (int i = threadIdx.x; i < ncls * NC; i += blockDim.x) {
    const int cls = i / NC, O = i % NC;
    s.oreal[i] = real_entries(ctrl, oct_start[cls * (NC + 1) + O], oct_start[cls * (NC + 1) + O + 1]);
  }
}

// One class of a multi-class stencil (Dubins: one per heading) into a
// warp's private staged copy (class index 0 there), by the warp's lanes.
template <int D, typename T, int RULE>
__device__ inline void stage_class(const StencilSmem<D, T>& s, int cls, int nc, int lane,
                                   const int32_t* oct_start, const uint32_t* nzmask,
                                   const double* weights, const double* cost,
                                   const int32_t* ctrl = nullptr) {
  constexpr int NC = 1 << D;
  stage_entries<D, T, RULE>(s, 0, cls * nc, nc, lane, 32, nzmask, weights, cost);
  if (lane <= NC) s.oct[lane] = oct_start[cls * (NC + 1) + lane] - cls * nc;
  if (lane < NC)
    s.oreal[lane] = real_entries(ctrl, oct_start[cls * (NC + 1) + lane],
                                 oct_start[cls * (NC + 1) + lane + 1]);
}

// Neighbourhood sources.  Evaluation code asks a source for corner K of
// octant O of the lane's node r (all compile-time after unrolling):
//  * Nbhd  -- the full 3^D neighbourhood of the NB nodes in registers
//             (feedback extraction);
//  * OctNb -- only the 2^D-corner cells of ONE octant, loaded from the
//             warp's staged tile right before that octant is evaluated
//             (value sweep; keeps the 3D register footprint small).
// Corner K, internal axis i: offset (O_i ? 0 : -1) + K_i from the node.
template <int D, typename T, int NB>
struct Nbhd {
  static constexpr int NR = (D == 2) ? 3 : 9;
  T v[NR][NB + 2];
  template <int O, int K>
  __device__ __forceinline__ T corner(int r) const {
    constexpr int off0 = (((O >> 0) & 1) ? 0 : -1) + ((K >> 0) & 1);
    constexpr int off1 = (((O >> 1) & 1) ? 0 : -1) + ((K >> 1) & 1);
    if constexpr (D == 2) {
      return v[off0 + 1][r + off1 + 1];
    } else {
      constexpr int off2 = (((O >> 2) & 1) ? 0 : -1) + ((K >> 2) & 1);
      return v[(off0 + 1) * 3 + (off1 + 1)][r + off2 + 1];
    }
  }
};

// Octant view of a full register neighbourhood (compile-time octant).
template <int D, typename T, int NB, int O>
struct NbhdOct {
  const Nbhd<D, T, NB>& nb;
  template <int K>
  __device__ __forceinline__ T corner(int r) const {
    return nb.template corner<O, K>(r);
  }
};

// One corner step K of U*NB interleaved interpolation chains over a cell
// source (corner<K>(r) of one octant).
template <int D, typename T, int NB, int U, int K, typename Src>
struct ChainStep {
  __device__ __forceinline__ static void run(const Src& cell, const T (&w)[U][1 << D],
                                             T (&acc)[U][NB]) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NB; ++r)
        acc[u][r] = fma(w[u][K], cell.template corner<K>(r), acc[u][r]);
    ChainStep<D, T, NB, U, K + 1, Src>::run(cell, w, acc);
  }
};
template <int D, typename T, int NB, int U, typename Src>
struct ChainStep<D, T, NB, U, (1 << D), Src> {
  __device__ __forceinline__ static void run(const Src&, const T (&)[U][1 << D], T (&)[U][NB]) {}
};

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
__device__ __forceinline__ T finish_cand(T acc, T ca, T cb, T ncoef, uint32_t fm, uint32_t nz,
                                         bool ok = true) {
  if constexpr (COST == PHJ_COST_CTRL) {
    acc = (RULE == PHJ_RULE_KRUZKOV) ? fma(ca, acc, cb) : acc + ca;
  } else if constexpr (MODE == 1) {
    // feedback applies the rule per candidate (SURVEY App. A hoisting caveat)
    acc = (RULE == PHJ_RULE_KRUZKOV) ? fma(ncoef, acc, T(1) - ncoef) : acc + ncoef;
  }
  if constexpr (SLOW) {
    if ((fm & nz) || !ok) acc = big_value<T>();
  }
  return acc;
}

// Running minimum of non-negative candidates.  For fp64 the compare runs on
// the bit patterns as int64 (same order for values >= 0; candidates are
// convex combinations of non-negative values plus non-negative costs), which
// keeps the FP64 pipe for the interpolation FMAs; fp32 uses FMNMX.
#ifndef PHJ_MIN_INT
#define PHJ_MIN_INT 0
#endif
#ifndef PHJ_KUNROLL2
#define PHJ_KUNROLL2 4
#endif
#ifndef PHJ_PRUNE
#define PHJ_PRUNE 1
#endif
#ifndef PHJ_WPIPE
#define PHJ_WPIPE 0
#endif
#ifndef PHJ_MINU
#define PHJ_MINU 0
#endif
#ifndef PHJ_CTRL_REGNB
#define PHJ_CTRL_REGNB 0
#endif
#ifndef PHJ_SKIP_EMPTY_OCT
#define PHJ_SKIP_EMPTY_OCT 1
#endif
#ifndef PHJ_EARLY_STAGE
#define PHJ_EARLY_STAGE 0
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
// AO3 conical control reduction (solver.py:446-476): per node, the stencil
// entries allowed by its feedback control, as a bitmask over entry index
// (up to 128 entries).
template <int NB>
struct Allowed {
  unsigned long long w[NB][2];
};

template <int D, typename T, int NB, int RULE, int COST, bool SLOW, int MODE, typename Src,
          bool AO3 = false>
__device__ __forceinline__ void eval_octant(const Src& cell, int O, const StencilSmem<D, T>& s,
                                            const int* os, const uint32_t (&fm)[NB],
                                            const T (&ncoef)[NB], const int32_t* ctrl_map,
                                            MinAcc<T> (&mn)[NB], T (&best)[NB], int (&bidx)[NB],
                                            const Allowed<NB>* al = nullptr) {
  static_assert(!AO3 || SLOW, "AO3 rejects candidates on the SLOW path");
  constexpr int NC = 1 << D;
  constexpr int U = (D == 2) ? PHJ_KUNROLL2 : PHJ_UNROLL(D);  // divides the host padding
  const int e0 = os[O], e1 = os[O + 1];
  if (e0 >= e1) return;
#if PHJ_MINU
  // one running min per unrolled entry slot: no cross-slot compare chain
  // inside the loop, merged into mn after the octant
  MinAcc<T> mu[U][NB];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int r = 0; r < NB; ++r) mu[u][r].init();
#endif
  // U entries from e: corner-major order -- U*NB independent FMA chains
  // advance one corner per step, so consecutive FP64 instructions never
  // depend on each other (DFMA latency ~8 cycles, 2-cycle issue per warp).
  auto step = [&](const T (&w)[U][NC], int e) {
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
    T acc[U][NB];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NB; ++r) acc[u][r] = w[u][0] * cell.template corner<0>(r);
    ChainStep<D, T, NB, U, 1, Src>::run(cell, w, acc);
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      T x[U];
      unsigned long long aw = 0ull;
      if constexpr (AO3) aw = (e >> 6) ? al->w[r][1] : al->w[r][0];  // U | 64: one word
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bool ok = true;
        if constexpr (AO3) ok = (aw >> ((e + u) & 63)) & 1ull;
        x[u] = finish_cand<T, RULE, COST, SLOW, MODE>(acc[u][r], ca[u], cb[u], ncoef[r], fm[r],
                                                      nz[u], ok);
      }
      if constexpr (MODE == 0) {
#if PHJ_MINU
#pragma unroll
        for (int u = 0; u < U; ++u) mu[u][r].take(x[u]);
#else
        // pairwise tree over the U candidates, one link into the running min
#pragma unroll
        for (int st = 1; st < U; st <<= 1)
#pragma unroll
          for (int u = 0; u + st < U; u += 2 * st) x[u] = x[u + st] < x[u] ? x[u + st] : x[u];
        mn[r].take(x[0]);
#endif
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) take_arg<T>(x[u], ci[u], best[r], bidx[r]);
      }
    }
  };
  auto load = [&](T (&w)[U][NC], int e) {
#pragma unroll
    for (int u = 0; u < U; ++u) load_weights<T, NC>(s.w + (int64_t)(e + u) * NC, w[u]);
  };
#if PHJ_WPIPE
  // weights double-buffered one step ahead (the shared-memory latency of a
  // step's weights overlaps the previous step's FMA chains)
  const int elast = e1 - U;
  T wa[U][NC], wb[U][NC];
  load(wa, e0);
  for (int e = e0; e < e1; e += 2 * U) {
    load(wb, min(e + U, elast));
    step(wa, e);
    if (e + U >= e1) break;
    load(wa, min(e + 2 * U, elast));
    step(wb, e + U);
  }
#else
  for (int e = e0; e < e1; e += U) {
    T w[U][NC];
    load(w, e);
    step(w, e);
  }
#endif
#if PHJ_MINU
  if constexpr (MODE == 0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < NB; ++r) mn[r].take(mu[u][r].get());
  }
#endif
}

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// All octants in order; `hook` runs once, right after octant 0 (the solve
// sweep issues the next block's loads there so they overlap the rest).
template <int D, typename T, int NB, int RULE, int COST, bool SLOW, int MODE, bool AO3 = false,
          int O = 0>
struct EvalAll {
  template <typename Hook>
  __device__ __forceinline__ static void run(const Nbhd<D, T, NB>& nb, const StencilSmem<D, T>& s,
                                             const int* os, const uint32_t (&fm)[NB],
                                             const T (&ncoef)[NB], const int32_t* ctrl_map,
                                             MinAcc<T> (&mn)[NB], T (&best)[NB], int (&bidx)[NB],
                                             const Hook& hook, const Allowed<NB>* al = nullptr) {
    eval_octant<D, T, NB, RULE, COST, SLOW, MODE, NbhdOct<D, T, NB, O>, AO3>(
        NbhdOct<D, T, NB, O>{nb}, O, s, os, fm, ncoef, ctrl_map, mn, best, bidx, al);
    if constexpr (O == 0) hook();
    EvalAll<D, T, NB, RULE, COST, SLOW, MODE, AO3, O + 1>::run(nb, s, os, fm, ncoef, ctrl_map, mn,
                                                              best, bidx, hook, al);
  }
};
template <int D, typename T, int NB, int RULE, int COST, bool SLOW, int MODE, bool AO3>
struct EvalAll<D, T, NB, RULE, COST, SLOW, MODE, AO3, (1 << D)> {
  template <typename Hook>
  __device__ __forceinline__ static void run(const Nbhd<D, T, NB>&, const StencilSmem<D, T>&,
                                             const int*, const uint32_t (&)[NB], const T (&)[NB],
                                             const int32_t*, MinAcc<T> (&)[NB], T (&)[NB],
                                             int (&)[NB], const Hook&, const Allowed<NB>* = nullptr) {}
};

// ---- octant pruning (MODE 0, per-node cost) --------------------------------
// Every candidate of octant O is a convex combination of the octant's 2^D
// corner values (non-negative weights summing exactly to 1 in T, fma chain
// with non-negative terms), so in floating point it is >= min corner *
// (1 - 2^D u).  An octant whose corner minimum (lowered by a margin of many
// ulps) is not below the node's running minimum cannot lower it: skipping
// it leaves the minimum bit-identical.  Values are >= 0, so the order of
// their bit patterns as integers is the order of the values.
template <typename T>
struct OrdKey;
template <>
struct OrdKey<double> {
  // coarse key: the high word (monotone in the value for x >= 0); the
  // bound test below only compares coarse keys, which is conservative
  using I = int;
  static __device__ __forceinline__ I coarse(double x) { return __double2hiint(x); }
};
template <>
struct OrdKey<float> {
  using I = int;
  static __device__ __forceinline__ I coarse(float x) { return __float_as_int(x); }
};

template <int D, typename T, int NB, int K, typename Src>
struct CornerMin {
  __device__ __forceinline__ static int run(const Src& cell, int r, int m) {
    m = min(m, OrdKey<T>::coarse(cell.template corner<K>(r)));
    return CornerMin<D, T, NB, K + 1, Src>::run(cell, r, m);
  }
};
template <int D, typename T, int NB, typename Src>
struct CornerMin<D, T, NB, (1 << D), Src> {
  __device__ __forceinline__ static int run(const Src&, int, int m) { return m; }
};

// Does any computing node of the lane still need the octant of `cell`?
// Skip only if  coarse(min corner) - margin >= coarse(best): for fp64
// (coarse = high word, margin 2) the min corner is then >= 2^32 ulps above
// best, for fp32 (full key, margin 64) >= 64 ulps -- both far above the
// rounding of a 2^D-term convex combination (<= 2^D/2 ulps below its min).
template <int D, typename T, int NB, typename Src>
__device__ __forceinline__ bool octant_needed(const Src& cell, const bool (&comp)[NB],
                                              const MinAcc<T> (&mn)[NB]) {
  using K = OrdKey<T>;
  constexpr int margin = sizeof(T) == 8 ? 2 : 64;
  bool need = false;
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    const int cmin = CornerMin<D, T, NB, 1, Src>::run(cell, r, K::coarse(cell.template corner<0>(r)));
    need |= comp[r] && cmin - margin < K::coarse(mn[r].get());
  }
  return need;
}

// ---- the warp's staged halo tile ---------------------------------------------
// Warp-block halo tile: the union of the 3^D neighbourhoods of a block's
// nodes (ext values, clamped like load_nbhd), staged into shared memory by
// the whole warp with cp.async -- every ext value is fetched once per block,
// and the copy of the next block overlaps the current block's control loop.
template <int D>
struct TileShape {
  using B = Blk<D>;
  static constexpr int RB = B::BY + 2;                    // rows per plane
  static constexpr int R = (D == 2) ? RB : 3 * RB;        // rows (x 3 planes in 3D)
  static constexpr int C = B::BX + 2 + ((B::BX + 2) % 2 == 0);  // columns (odd pitch: banks)
  // 3D solve tiles (8-wide blocks, 2 nodes per lane): rows alternate between
  // pitch 11 and 13 (row r starts at 12 r - (r & 1)).  A half-warp's 16 lanes
  // (4 consecutive rows x 4 lanes 2 elements apart) then read 16 distinct
  // 8-byte banks for every row / column / plane shift of the octant loads;
  // with the constant odd pitch 11 two of them collided and every LDS.64 of
  // the cell loads took 4 wavefronts instead of 2 (ncu: 13.7 G excess
  // wavefronts per config-5 pass, the shared-memory pipe at 76 % of peak).
  static constexpr bool SWZ = D == 3 && B::BX == 8 && B::NB == 2 && RB % 2 == 0;
  static constexpr int P = 12;  // mean pitch of the swizzled layout
  __host__ __device__ static constexpr int row(int r) { return SWZ ? P * r - (r & 1) : r * C; }
  static constexpr int N = SWZ ? R * P : R * C;
};

// +1 / -1 for lanes on odd / even block rows: the offset between a lane's
// row and the next one is P + sg in the swizzled layout (two rows: 2 P).
template <int D>
__device__ __forceinline__ int lane_sg(int lane) {
  return ((lane / Blk<D>::LX) & 1) ? 1 : -1;
}

// The lane's origin in the tile (its first node's 3^D neighbourhood starts
// here) and the element of that node displaced by (d0, d1[, d2]).
template <int D, typename T>
__device__ __forceinline__ const T* lane_tile(const T* tile, int lane) {
  using B = Blk<D>;
  using S = TileShape<D>;
  return tile + S::row(lane / B::LX) + (lane % B::LX) * B::NB;
}
// offset from the lane origin to (plane dp, row dy) of its neighbourhood
template <int D>
__device__ __forceinline__ int tile_rel(int sg, int dp, int dy) {
  using S = TileShape<D>;
  if constexpr (S::SWZ) return S::P * (dp * S::RB + dy) + ((dy & 1) ? sg : 0);
  else return (dp * S::RB + dy) * S::C;
}
template <int D, typename T>
__device__ __forceinline__ T tile_at(const T* lt, int sg, int d0, int d1, int d2 = 0) {
  using S = TileShape<D>;
  if constexpr (D == 2) return lt[(1 + d0) * S::C + 1 + d1];
  else return lt[tile_rel<D>(sg, 1 + d0, 1 + d1) + 1 + d2];
}

// The 2^D-corner cells of one octant (runtime O) for the lane's NB nodes;
// the accessors are octant-independent, so one copy of the control loop
// serves every octant.
template <int D, typename T, int NB>
struct OctNb {
  static constexpr int NR = 1 << (D - 1);
  T v[NR][NB + 1];
  template <int K>
  __device__ __forceinline__ T corner(int r) const {
    if constexpr (D == 2) return v[K & 1][r + ((K >> 1) & 1)];
    else return v[(K & 1) * 2 + ((K >> 1) & 1)][r + ((K >> 2) & 1)];
  }
  __device__ __forceinline__ void load(const T* lt, int O, int sg) {
    using S = TileShape<D>;
    const int b0 = O & 1, b1 = (O >> 1) & 1, b2 = (O >> 2) & 1;
    if constexpr (D == 2) {
      const T* t0 = lt + b0 * S::C + b1;
#pragma unroll
      for (int k0 = 0; k0 < 2; ++k0)
#pragma unroll
        for (int j = 0; j <= NB; ++j) v[k0][j] = t0[k0 * S::C + j];
    } else {
      // rows b1 and b1 + 1 of planes b0 and b0 + 1 (two row bases: the row
      // pitch depends on the row parity in the swizzled layout)
      const T* ta = lt + tile_rel<D>(sg, b0, b1) + b2;
      const T* tb = lt + tile_rel<D>(sg, b0, b1 + 1) + b2;
      constexpr int PS = S::SWZ ? S::P * S::RB : S::RB * S::C;  // plane stride
#pragma unroll
      for (int k0 = 0; k0 < 2; ++k0)
#pragma unroll
        for (int j = 0; j <= NB; ++j) {
          v[k0 * 2][j] = ta[k0 * PS + j];
          v[k0 * 2 + 1][j] = tb[k0 * PS + j];
        }
    }
  }
};

// the octant of steepest descent at the lane's first node, majority over
// the warp (warp-uniform)
template <int D, typename T>
__device__ __forceinline__ int preferred_octant(const T* lt, int sg) {
  const unsigned FULL = 0xffffffffu;
  bool down[D];
  if constexpr (D == 2) {
    down[0] = tile_at<D>(lt, sg, 1, 0) < tile_at<D>(lt, sg, -1, 0);
    down[1] = tile_at<D>(lt, sg, 0, 1) < tile_at<D>(lt, sg, 0, -1);
  } else {
    down[0] = tile_at<D>(lt, sg, 1, 0, 0) < tile_at<D>(lt, sg, -1, 0, 0);
    down[1] = tile_at<D>(lt, sg, 0, 1, 0) < tile_at<D>(lt, sg, 0, -1, 0);
    down[2] = tile_at<D>(lt, sg, 0, 0, 1) < tile_at<D>(lt, sg, 0, 0, -1);
  }
  int o = 0;
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (__popc(__ballot_sync(FULL, down[i])) >= 16) o |= 1 << i;
  return o;
}

// Sweep evaluation of one block from its staged tile: with per-node costs
// the warp's preferred octant first, then the others unless pruned; with
// per-control costs every octant in order.  `hook` runs once, after the
// first octant.  Returns the stencil entries evaluated per node; `n_real`
// gets the real (non-padding) ones among them.
template <int D, typename T, int NB, int RULE, int COST, bool SLOW, typename Hook,
          bool AO3 = false>
__device__ __forceinline__ int eval_sweep(const T* lt, bool prune_on, const StencilSmem<D, T>& s,
                                          const int* os, const uint32_t (&fm)[NB],
                                          const T (&ncoef)[NB], const bool (&comp)[NB],
                                          MinAcc<T> (&mn)[NB], T (&best)[NB], int (&bidx)[NB],
                                          const Hook& hook, int& n_real,
                                          const Allowed<NB>* al = nullptr, bool warm = false) {
#if PHJ_CTRL_REGNB
  if constexpr (COST == PHJ_COST_CTRL) {
    // per-control costs (no pruning), few controls: the whole neighbourhood
    // in registers, compile-time octants
    Nbhd<D, T, NB> nb;
    using S = TileShape<D>;
    static_assert(!S::SWZ, "register-neighbourhood path assumes the constant tile pitch");
    if constexpr (D == 2) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < NB + 2; ++dx) nb.v[dy][dx] = lt[dy * S::C + dx];
    } else {
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < NB + 2; ++dx) nb.v[dz * 3 + dy][dx] = lt[(dz * S::RB + dy) * S::C + dx];
    }
    EvalAll<D, T, NB, RULE, COST, SLOW, 0>::run(nb, s, os, fm, ncoef, nullptr, mn, best, bidx, hook);
    n_real = 0;
#pragma unroll
    for (int O = 0; O < (1 << D); ++O) n_real += s.oreal[O];
    return os[1 << D] - os[0];
  }
#endif
  constexpr bool CAN_PRUNE = COST == PHJ_COST_NODE && PHJ_PRUNE;
  const bool prune = CAN_PRUNE && prune_on;
  const int sg = lane_sg<D>(threadIdx.x & 31);
  const int first = prune ? preferred_octant<D, T>(lt, sg) : 0;
  OctNb<D, T, NB> cell;
  cell.load(lt, first, sg);
  int n_ent = 0;
  n_real = 0;
  // warm: the running minima start at the previous block-local relaxation's
  // minima (an upper bound of the new ones: values only decreased), so the
  // preferred octant is prunable too
  if (!(prune && warm) || __any_sync(0xffffffffu, octant_needed<D, T, NB>(cell, comp, mn))) {
    eval_octant<D, T, NB, RULE, COST, SLOW, 0, OctNb<D, T, NB>, AO3>(cell, first, s, os, fm,
                                                                     ncoef, nullptr, mn, best,
                                                                     bidx, al);
    n_ent = os[first + 1] - os[first];
    n_real = s.oreal[first];
  }
  hook();
#pragma unroll 1
  for (int O = 0; O < (1 << D); ++O) {
#if PHJ_SKIP_EMPTY_OCT
    if (O == first || os[O] == os[O + 1]) continue;
#else
    if (O == first) continue;
#endif
    cell.load(lt, O, sg);
    if (prune && !__any_sync(0xffffffffu, octant_needed<D, T, NB>(cell, comp, mn))) continue;
    eval_octant<D, T, NB, RULE, COST, SLOW, 0, OctNb<D, T, NB>, AO3>(cell, O, s, os, fm, ncoef,
                                                                     nullptr, mn, best, bidx, al);
    n_ent += os[O + 1] - os[O];
    n_real += s.oreal[O];
  }
  return n_ent;
}

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

template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(src), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Per-node inputs of a staged block: node coefficients, foreign masks and
// labels (int16, copied as the 32-bit words covering each row).
template <int D, typename T>
struct NodeStage {
  using B = Blk<D>;
  static constexpr int NN = B::BY * B::BX;
  static constexpr int LW = B::BX / 2 + 1;  // label words per row
  T coef[NN];
  uint32_t fm[NN];
  int32_t fb[NN];  // AO3: feedback control per node
  uint32_t labw[B::BY * LW];
};

// Stage block blk (halo tile of v + node inputs) into the warp's buffers as
// one cp.async group.  Lanes own tile row segments (one base address each,
// immediate column offsets); only blocks at the far grid edge (partial
// blocks) clamp addresses into the arrays -- lanes whose nodes lie outside
// the grid are masked by the consumer.
template <int D>
struct StagePlan {
  using B = Blk<D>;
  using S = TileShape<D>;
  static constexpr int W = B::BX + 2;  // tile columns
  static constexpr int seg() {
    int s = 32 / S::R;
    while (s > 1 && W % s != 0) --s;
    return s < 1 ? 1 : s;
  }
  static constexpr int SEG = seg();      // lanes per tile row
  static constexpr int SW = W / SEG;     // columns per lane
  static constexpr int LPR = 32 / B::BY; // lanes per node row
  static constexpr int NPL = B::BX / LPR;  // nodes per lane
  static_assert(S::R * SEG <= 32, "tile rows exceed the warp");
  static_assert(B::BX % LPR == 0, "node row split");
};

template <int D, typename T, int COST>
__device__ __forceinline__ void stage_block(const SolveParams& p, const T* __restrict__ v, int blk,
                                            T* tile, NodeStage<D, T>* ns, int lane) {
  using B = Blk<D>;
  using S = TileShape<D>;
  using NS = NodeStage<D, T>;
  using P = StagePlan<D>;
  const phj_grid& g = p.g;
  int b[3];
  decode_block<D>(p.tg, blk, b);
  // ext flat index of the tile origin, row stride, extent checks
  int64_t o, rs, s0x;
  int row0, col0, rmax, cmax;
  bool full;
  if constexpr (D == 2) {
    row0 = b[0] * B::BY;
    col0 = b[1] * B::BX;
    rs = g.strides[0];
    s0x = 0;
    o = (int64_t)row0 * rs + col0;
    rmax = (int)g.ext[0] - 1;
    cmax = (int)g.ext[1] - 1;
    full = (b[0] + 1) * B::BY <= g.shape[0] && (b[1] + 1) * B::BX <= g.shape[1];
  } else {
    row0 = b[1] * B::BY;
    col0 = b[2] * B::BX;
    rs = g.strides[1];
    s0x = g.strides[0];
    o = (int64_t)b[0] * s0x + (int64_t)row0 * rs + col0;
    rmax = (int)g.ext[1] - 1;
    cmax = (int)g.ext[2] - 1;
    full = (b[1] + 1) * B::BY <= g.shape[1] && (b[2] + 1) * B::BX <= g.shape[2];
  }
  // halo tile: lane -> (row, segment)
  if (lane < S::R * P::SEG) {
    const int r = lane / P::SEG, sg = lane - r * P::SEG;
    int pl = 0, rr = r;
    if constexpr (D == 3) {
      pl = r / S::RB;
      rr = r - pl * S::RB;
    }
    const int c0 = sg * P::SW;
    T* dst = tile + S::row(r) + c0;
    if (full) {
      const T* src = v + o + pl * s0x + (int64_t)rr * rs + c0;
#pragma unroll
      for (int j = 0; j < P::SW; ++j) cp_async<sizeof(T)>(dst + j, src + j);
    } else {
      const int rc = min(row0 + rr, rmax) - row0;
      const T* src = v + o + pl * s0x + (int64_t)rc * rs;
#pragma unroll
      for (int j = 0; j < P::SW; ++j)
        cp_async<sizeof(T)>(dst + j, src + (min(col0 + c0 + j, cmax) - col0));
    }
  }
  // node inputs: lane -> (node row, NPL consecutive nodes, label words)
  {
    const int ly = lane / P::LPR, q = lane - ly * P::LPR;
    const int64_t nlast = (int64_t)g.ext[0] * g.strides[0] - 1;
    const int64_t fr = o + s0x + rs + 1 + (int64_t)ly * rs;  // ext index of the row's node 0
    const bool stage_coef = COST == PHJ_COST_NODE && p.coef != nullptr;
    const int j0 = q * P::NPL;
#pragma unroll
    for (int k = 0; k < P::NPL; ++k) {
      const int j = j0 + k;
      const int64_t f = full ? fr + j : min(fr + j, nlast);
      cp_async<4>(&ns->fm[ly * B::BX + j], p.fmask + f);
      if (stage_coef) cp_async<sizeof(T)>(&ns->coef[ly * B::BX + j], (const T*)p.coef + f);
      if (p.ao3_fb) cp_async<4>(&ns->fb[ly * B::BX + j], p.ao3_fb + f);
    }
    const int64_t wmax = (nlast - 1) >> 1;  // last whole 32-bit word of the label array
    const uint32_t* labw = (const uint32_t*)p.lab;
    const int64_t w0 = fr >> 1;
#pragma unroll
    for (int w = q; w < NS::LW; w += P::LPR) {
      const int64_t wi = full ? w0 + w : min(w0 + w, wmax);
      cp_async<4>(&ns->labw[ly * NS::LW + w], labw + wi);
    }
  }
  cp_async_commit();
}

// Warp-local running max change of the patch the warp's recent blocks
// belonged to; flushed into the CTA (or global) per-patch max when the
// patch changes and at the end of the sweep.
struct PatchMax {
  int lab;
  double m;
};

__device__ __forceinline__ void flush_patch_max(const SolveParams& p, PatchMax& pm,
                                                unsigned long long* s_max,
                                                unsigned long long* gmax_row) {
  if (pm.lab >= 0 && (threadIdx.x & 31) == 0) {
    if (p.R <= kSmemPatchReduce) atomicMax(&s_max[pm.lab], dbits(pm.m));
    else atomicMax(&gmax_row[pm.lab * kMaxPad], dbits(pm.m));
  }
  pm.lab = -1;
  pm.m = 0.0;
}

// Per-patch work counters of one block visit (SweepStats per patch, also
// under the asynchronous schedule): node relaxations, logical candidate
// evaluations (admissible controls of each relaxation), executed candidate
// evaluations (real stencil entries after pruning).  Warp-aggregated when
// every computing node of the warp is in one patch; per-CTA shared counters
// for R <= kSmemPatchReduce.
template <int NB>
__device__ __forceinline__ void add_patch_counts(const SolveParams& p, unsigned long long* s_pc,
                                                 const bool (&comp)[NB], const int (&labv)[NB],
                                                 const int (&fc)[NB], int iters,
                                                 unsigned real_it) {
  const unsigned FULL = 0xffffffffu;
  unsigned long long* cnt = p.R <= kSmemPatchReduce ? s_pc : p.pcount;
  int l0 = -1, ncomp = 0;
  unsigned n = 0, e = 0;
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    if (!comp[r]) continue;
    l0 = labv[r];
    ++ncomp;
    n += (unsigned)iters;
    e += (unsigned)(fc[r] * iters);
  }
  const int lref = __reduce_max_sync(FULL, l0);
  bool uni = true;
#pragma unroll
  for (int r = 0; r < NB; ++r) uni &= !comp[r] || labv[r] == lref;
  if (__all_sync(FULL, uni)) {
    const unsigned wn = __reduce_add_sync(FULL, n);
    const unsigned we = __reduce_add_sync(FULL, e);
    const unsigned wx = __reduce_add_sync(FULL, real_it * (unsigned)ncomp);
    if ((threadIdx.x & 31) == 0 && lref >= 0) {
      atomicAdd(&cnt[lref * 3 + 0], (unsigned long long)wn);
      atomicAdd(&cnt[lref * 3 + 1], (unsigned long long)we);
      atomicAdd(&cnt[lref * 3 + 2], (unsigned long long)wx);
    }
  } else {
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (!comp[r]) continue;
      atomicAdd(&cnt[labv[r] * 3 + 0], (unsigned long long)iters);
      atomicAdd(&cnt[labv[r] * 3 + 1], (unsigned long long)(fc[r] * iters));
      atomicAdd(&cnt[labv[r] * 3 + 2], (unsigned long long)real_it);
    }
  }
}

// One block of the value sweep, processed by one warp from its staged halo
// tile and node inputs.  `hook` (the next block's loads, deferred marks)
// runs exactly once.  Returns (warp-uniform) whether any node changed.
template <int D, typename T, int RULE, int COST, typename Hook>
__device__ __forceinline__ int sweep_block(const SolveParams& p, const StencilSmem<D, T>& s,
                                            int blk, const T* tile, const NodeStage<D, T>* ns,
                                            T* __restrict__ vout, const int* s_done,
                                            unsigned long long* s_max, unsigned long long* gmax_row,
                                            unsigned long long& evals, unsigned long long& exec,
                                            unsigned long long& xreal, unsigned long long* s_pc,
                                            PatchMax& pm, PhaseTimer& tm, const Hook& hook,
                                            bool force_copy = false) {
  using B = Blk<D>;
  using S = TileShape<D>;
  using NS = NodeStage<D, T>;
  constexpr int NB = B::NB;
  constexpr int last = D - 1;
  const unsigned FULL = 0xffffffffu;
  const phj_grid& g = p.g;
  const int lane = threadIdx.x & 31;
  int c[3];
  const bool row_ok = lane_nodes<D>(g, p.tg, blk, lane, c);
  const int64_t f0 = ext_flat<D>(g, c);
  // the solve kernel's staged stencil holds this block's class at index 0
  // (single-class stencils, or the warp's private class slot)
  const int* os = s.oct;
  const int nadm = p.n_real;
  const int ly = lane / B::LX, lx = lane % B::LX;
  const int lshift = (int)((f0 - lx * NB) & 1);  // label half-word offset of the row
  const bool stage_coef = COST == PHJ_COST_NODE && p.coef != nullptr;
  const T* lt = lane_tile<D>(tile, lane);
  const int sg = lane_sg<D>(lane);

  int labv[NB];
  uint32_t fm[NB];
  T ncoef[NB];
  bool comp[NB], copy[NB];
  bool any_comp = false, any_copy = false;
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    const bool in = row_ok && c[last] + r < g.shape[last];
    const int j = lx * NB + r;
    const int hw = lshift + j;
    const uint32_t word = ns->labw[ly * NS::LW + (hw >> 1)];
    const int lab = (int)(int16_t)(uint16_t)(word >> ((hw & 1) * 16));
    labv[r] = in ? lab : -1;
    fm[r] = ns->fm[ly * B::BX + j];
    ncoef[r] = stage_coef ? ns->coef[ly * B::BX + j] : (T)p.coef0;
    comp[r] = false;
    copy[r] = false;
    if (labv[r] >= 0) {
      if (force_copy || s_done[labv[r]] != 0x7fffffff ||
          (COST == PHJ_COST_NODE && ncoef[r] < T(0))) {
        copy[r] = true;
      } else {
        comp[r] = true;
        any_comp = true;
      }
    }
    if (!comp[r]) fm[r] = 0;
    any_copy |= copy[r];
  }
  bool changed = false, big = false;
  T mych[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) mych[r] = T(0);
  const int64_t M0 = g.shape[0];
  const bool per0 = g.periodic[0] != 0;
  const int64_t ghost_shift = M0 * g.strides[0];

  const bool warp_comp = __any_sync(FULL, any_comp);
  tm.mark(2);
  if (warp_comp) {
    uint32_t fmo = 0;
#pragma unroll
    for (int r = 0; r < NB; ++r) fmo |= fm[r];
    const bool slow = __any_sync(FULL, fmo != 0);
    // per-node AO3 masks (loaded once per block)
    Allowed<NB> al;
    if (p.ao3_fb) {
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        const int f = comp[r] ? ns->fb[ly * B::BX + lx * NB + r] : -1;
#pragma unroll
        for (int w = 0; w < 2; ++w)
          al.w[r][w] = (f >= 0 && w < p.ao3_words) ? __ldg(&p.ao3_mask[f * p.ao3_words + w])
                                                   : ~0ull;
      }
    }
    unsigned long long fcnt_sum = 0;
    int fc[NB];
    int ncomp = 0;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      fc[r] = 0;
      if (!comp[r]) continue;
      int fcnt = nadm;
      if (p.ao3_fb) {
        const int f = ns->fb[ly * B::BX + lx * NB + r];
        if (f >= 0) fcnt = __ldg(&p.ao3_count[f]);
      }
      fc[r] = fcnt;
      ++ncomp;
      fcnt_sum += (unsigned long long)fcnt;
    }
    unsigned real_it = 0;
    int iters = 0;
    // old values, then up to p.inner block-local relaxations: the halo ring
    // stays at the sweep's input, the block's own nodes are relaxed in the
    // staged tile (deterministic: independent of the schedule)
    T old[NB], cur[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      old[r] = (D == 2) ? tile_at<D>(lt, sg, 0, r) : tile_at<D>(lt, sg, 0, 0, r);
      cur[r] = old[r];
    }
    bool hooked = false;
    auto once = [&]() {
      if (!hooked) {
        hooked = true;
        hook();
      }
    };
    // minima of the previous block-local relaxation: upper bounds of the next
    // ones (tile values only decrease; candidates are monotone in them)
    T warmv[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) warmv[r] = big_value<T>();
    for (int it = 0;;) {
      MinAcc<T> mn[NB];
      T best[NB];
      int bidx[NB];
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        mn[r].init();
        mn[r].take(warmv[r]);
        best[r] = big_value<T>();
        bidx[r] = 0;
      }
      const bool warm = it > 0;
      int n_ent, n_real;
      if (p.ao3_fb) {
        n_ent = eval_sweep<D, T, NB, RULE, COST, true, decltype(once), true>(
            lt, p.prune != 0, s, os, fm, ncoef, comp, mn, best, bidx, once, n_real, &al, warm);
      } else if (slow) {
        n_ent = eval_sweep<D, T, NB, RULE, COST, true>(lt, p.prune != 0, s, os, fm, ncoef, comp,
                                                       mn, best, bidx, once, n_real, nullptr, warm);
      } else {
        n_ent = eval_sweep<D, T, NB, RULE, COST, false>(lt, p.prune != 0, s, os, fm, ncoef, comp,
                                                        mn, best, bidx, once, n_real, nullptr,
                                                        warm);
      }
      exec += (unsigned long long)n_ent * NB;
      evals += fcnt_sum;
      real_it += (unsigned)n_real;
      ++iters;
      bool moved = false;
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        if (!comp[r]) continue;
        const T b = mn[r].get();
        warmv[r] = b;
        T cand = b;
        if constexpr (COST == PHJ_COST_NODE) {
          cand = (RULE == PHJ_RULE_KRUZKOV) ? fma(ncoef[r], b, T(1) - ncoef[r]) : b + ncoef[r];
        }
        if (cand < cur[r]) {
          // another block-local relaxation only for changes above the
          // activity threshold (the same test as the neighbour marking)
          if constexpr (RULE == PHJ_RULE_KRUZKOV) moved |= cur[r] - cand > T(p.act) * (T(1) - cand);
          else moved |= cur[r] - cand > T(p.act) * max(T(1), cand);
          cur[r] = cand;
        }
      }
      if (++it >= p.inner || !__any_sync(FULL, moved)) break;
      // publish the relaxed values to the lanes whose neighbourhoods hold them
      T* ltw = const_cast<T*>(lt);
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        if (D == 2) ltw[S::C + 1 + r] = cur[r];
        else ltw[tile_rel<D>(sg, 1, 1) + 1 + r] = cur[r];
      }
      __syncwarp();
    }
    tm.mark(3);
    xreal += (unsigned long long)real_it * (unsigned long long)ncomp;
    if (p.pcount) add_patch_counts<NB>(p, s_pc, comp, labv, fc, iters, real_it);
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (!(comp[r] || copy[r])) continue;
      T nv = old[r];
      if (comp[r] && cur[r] < old[r]) {
        nv = cur[r];
        mych[r] = old[r] - cur[r];
        changed = true;
        if constexpr (RULE == PHJ_RULE_KRUZKOV) big |= mych[r] > T(p.act) * (T(1) - nv);
        else big |= mych[r] > T(p.act) * max(T(1), nv);
      }
      vout[f0 + r] = nv;
      if (per0) {
        if (c[0] == 0) vout[f0 + r + ghost_shift] = nv;
        else if (c[0] == M0 - 1) vout[f0 + r - ghost_shift] = nv;
      }
    }
  } else {
    hook();
    if (any_copy) {
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        if (!copy[r]) continue;
        const T old = (D == 2) ? tile_at<D>(lt, sg, 0, r) : tile_at<D>(lt, sg, 0, 0, r);
        vout[f0 + r] = old;
        if (per0) {
          if (c[0] == 0) vout[f0 + r + ghost_shift] = old;
          else if (c[0] == M0 - 1) vout[f0 + r - ghost_shift] = old;
        }
      }
    }
  }

  // per-patch max change
  const bool wchanged = __any_sync(FULL, changed);
  tm.mark(4);
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
      if (lref != pm.lab) flush_patch_max(p, pm, s_max, gmax_row);
      pm.lab = lref;
      pm.m = max(pm.m, (double)m);
    } else {
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        if (mych[r] > T(0)) {
          if (p.R <= kSmemPatchReduce) atomic_max_change(&s_max[labv[r]], mych[r]);
          else atomic_max_change(&gmax_row[labv[r] * kMaxPad], mych[r]);
        }
      }
    }
  }
  tm.mark(5);
  // 2: a change above the activity threshold (mark the 3^D neighbourhood),
  // 1: only smaller changes (re-sweep this block once: both ping-pong
  // buffers must hold its new values), 0: unchanged
  return wchanged ? (__any_sync(FULL, big) ? 2 : 1) : 0;
}

// Deferred neighbour marking: a changed block's flag exchanges are issued
// at its end (stage A), the list slots are reserved with one warp-aggregated
// atomic at the next block's hook (stage B) and written one block later --
// no atomic round trip is waited for inside a block.
template <int D>
struct MarkQueue {
  int a_nt, a_old;           // A: neighbour id (-1 none), exchanged flag
  int b_nt, b_rank, b_base;  // B: reserved slot (b_base on lane 0)
  bool has_b;
  __device__ __forceinline__ void init() {
    a_nt = -1;
    a_old = 1;
    b_nt = -1;
    b_rank = 0;
    b_base = 0;
    has_b = false;
  }
  __device__ __forceinline__ void issue(const TileGrid& tg, const phj_grid& g, int blk, int ch,
                                        int lane, int* flags) {
    a_nt = -1;
    constexpr int self = D == 2 ? 4 : 13;
    if ((ch == 2 && lane < (D == 2 ? 9 : 27)) || (ch == 1 && lane == self)) {
      const int nt = neighbour_block<D>(tg, g, blk, lane);
      if (nt >= 0) {
        a_nt = nt;
        a_old = atomicExch(&flags[nt], 1);
      }
    }
  }
  // transport: OR the changed colours into the neighbours' next masks; the
  // first setter (old mask 0) appends the block
  // (append = false: OR only, e.g. into the sticky masks of the banded pass)
  __device__ __forceinline__ void issue_mask(const TileGrid& tg, const phj_grid& g, int blk,
                                             unsigned long long bits, int lane,
                                             unsigned long long* masks, bool append = true) {
    a_nt = -1;
    if (bits != 0ull && lane < (D == 2 ? 9 : 27)) {
      const int nt = neighbour_block<D>(tg, g, blk, lane);
      if (nt >= 0) {
        if (append) {
          const bool first = atomicOr(&masks[nt], bits) == 0ull;
          a_nt = nt;
          a_old = !first;
        } else {
          // sticky masks: a reduction (no value returned, nothing to wait for)
          atomicOr(&masks[nt], bits);
        }
      }
    }
  }
  __device__ __forceinline__ void reserve(int lane, int* cnt) {
    const bool want = a_nt >= 0 && a_old == 0;
    const unsigned bal = __ballot_sync(0xffffffffu, want);
    b_nt = want ? a_nt : -1;
    b_rank = __popc(bal & ((1u << lane) - 1u));
    if (bal != 0u && lane == 0) b_base = atomicAdd(cnt, __popc(bal));
    has_b = bal != 0u;
    a_nt = -1;
  }
  __device__ __forceinline__ void store(int* list) {
    if (has_b) {
      const int base = __shfl_sync(0xffffffffu, b_base, 0);
      if (b_nt >= 0) list[base + b_rank] = b_nt;
      has_b = false;
      b_nt = -1;
    }
  }
};

template <int D, typename T>
__host__ __device__ constexpr int64_t solve_tile_bytes() {
  return (int64_t)kWarps * 2 * TileShape<D>::N * sizeof(T) +
         (int64_t)kWarps * 2 * sizeof(NodeStage<D, T>);
}

// WCLS: multi-class stencil staged per warp (compile-time, so single-class
// launches keep fixed shared-memory addressing)
template <int D, typename T, int RULE, int COST, bool WCLS>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) solve_kernel(const __grid_constant__ SolveParams p) {
  constexpr int NB = Blk<D>::NB;
  using S = TileShape<D>;
  extern __shared__ __align__(16) unsigned char smem[];
  cg::grid_group grid = cg::this_grid();
  constexpr bool warp_cls = WCLS;
  const int64_t sbytes = solve_stencil_bytes<D, T>(WCLS ? 2 : 1, p.nc);
  StencilSmem<D, T> s =
      WCLS ? carve_stencil<D, T>(smem + (threadIdx.x >> 5) * solve_stencil_slot<D, T>(p.nc), 1,
                                 p.nc)
           : carve_stencil<D, T>(smem, 1, p.nc);
  int* s_done = (int*)(smem + sbytes);
  unsigned long long* s_max = (unsigned long long*)(s_done + ((p.R + 1) / 2 * 2));
  unsigned long long* s_pc = s_max + min(p.R, kSmemPatchReduce);  // [min(R,64)][3]
  T* tiles = (T*)(smem + align_up(sbytes + (int64_t)((p.R + 1) / 2 * 2) * 4 +
                                      (int64_t)min(p.R, kSmemPatchReduce) * 8 * 4,
                                  16));
  T* wtile = tiles + (threadIdx.x >> 5) * 2 * S::N;
  NodeStage<D, T>* wnodes =
      (NodeStage<D, T>*)(tiles + kWarps * 2 * S::N) + (threadIdx.x >> 5) * 2;
  if (!warp_cls)
    stage_stencil<D, T, RULE>(s, p.n_classes, p.nc, p.oct_start, p.nzmask, p.weights, p.cost,
                              p.ctrl);
  int wcls = -1;  // class held by this warp's slot
  for (int i = threadIdx.x; i < p.R; i += blockDim.x)
    s_done[i] = (p.mine == nullptr || p.mine[i]) ? 0x7fffffff : 0;
  for (int i = threadIdx.x; i < min(p.R, kSmemPatchReduce) * 3; i += blockDim.x) s_pc[i] = 0ull;
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  unsigned long long evals = 0, exec = 0, xreal = 0;
  int blocks_done = 0;
  int sw = 0, buf = 0, stage = 0;
  const int nshared = min(p.R, kSmemPatchReduce);
  const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * kWarps;
  // Work items of a sweep: the first is the warp's static index, later ones
  // are claimed one ahead with an atomic (lane 0 keeps the raw ticket so the
  // round trip is only waited for at the next item; the first dynamic claim
  // of a sweep is issued before the previous sweep's barrier).  Block ids
  // are read one ahead and the next block's tile / node inputs are loaded
  // during the current block.
  int ticket = 0;
  if (lane == 0) ticket = atomicAdd(&p.ws.take[0], 1);
  MarkQueue<D> mq;
  mq.init();
  PhaseTimer tm;
  tm.start();
  for (;;) {
    const T* vin = (const T*)p.v[buf];
    T* vout = (T*)p.v[buf ^ 1];
    const bool banded = sw < p.n_band;               // value-ordered pass
    const bool csr = p.n_band > 0 && sw <= p.n_band;  // list from the band schedule
    const int cnt = csr ? (p.band_off[sw + 1] - p.band_off[sw]) : ld_cg(&p.ws.counts[sw]);
    const int* list = csr ? p.band_list + p.band_off[sw] : p.ws.list[sw & 1];
    int* cur_flags = p.ws.flags[sw & 1];
    int* nxt_flags = p.ws.flags[(sw + 1) & 1];
    int* nxt_list = p.ws.list[(sw + 1) & 1];
    int* nxt_cnt = &p.ws.counts[sw + 1];
    int* take = &p.ws.take[sw];
    unsigned long long* gmax_row = sweep_max_slots(p.ws, sw);  // padded: entry i at i * kMaxPad
    if (blockIdx.x == 0) {
      unsigned long long* z = sweep_max_slots(p.ws, sw + 1);
      for (int i = threadIdx.x; i < p.R; i += blockDim.x) z[i * kMaxPad] = 0ull;
    }
    for (int i = threadIdx.x; i < nshared; i += blockDim.x) s_max[i] = 0ull;
    __syncthreads();
    int item = gwarp;
    int blk = item < cnt ? __ldcg(&list[item]) : 0;  // raw entry (banded: -b-1 = copy)
    if (item < cnt)
      stage_block<D, T, COST>(p, vin, entry_block(blk), wtile + stage * S::N, wnodes + stage, lane);
    PatchMax pm{-1, 0.0};
#if PHJ_EARLY_STAGE
    // block ids are read two ahead so the next block's staging can start as
    // soon as the current block's tile has landed
    int nxt = nwarps + __shfl_sync(FULL, ticket, 0);
    int nblk = (item < cnt && nxt < cnt) ? __ldcg(&list[nxt]) : 0;
    if (lane == 0 && item < cnt && nxt < cnt) ticket = atomicAdd(take, 1);
#endif
    tm.mark(0);
    while (item < cnt) {
#if PHJ_EARLY_STAGE
      const int nn = nwarps + __shfl_sync(FULL, ticket, 0);
      const int nnblk = (nxt < cnt && nn < cnt) ? __ldcg(&list[nn]) : 0;
      if (lane == 0 && nxt < cnt && nn < cnt) ticket = atomicAdd(take, 1);
#else
      const int nxt = nwarps + __shfl_sync(FULL, ticket, 0);
      const int nblk = nxt < cnt ? __ldcg(&list[nxt]) : 0;
      if (lane == 0 && nxt < cnt) ticket = atomicAdd(take, 1);
#endif
      const bool copy_visit = blk < 0;
      const int bid = entry_block(blk);
      if (lane == 0) cur_flags[bid] = 0;
      if (warp_cls) {
        int bc[3];
        decode_block<D>(p.tg, bid, bc);
        if (bc[0] != wcls) {
          __syncwarp();
          stage_class<D, T, RULE>(s, bc[0], p.nc, lane, p.oct_start, p.nzmask, p.weights, p.cost, p.ctrl);
          wcls = bc[0];
        }
      }
      cp_async_wait_all();
      __syncwarp();
#if PHJ_EARLY_STAGE
      mq.store(nxt_list);
      mq.reserve(lane, nxt_cnt);
      if (nxt < cnt)
        stage_block<D, T, COST>(p, vin, entry_block(nblk), wtile + (stage ^ 1) * S::N,
                                wnodes + (stage ^ 1), lane);
      auto hook = []() {};
#else
      auto hook = [&]() {
        mq.store(nxt_list);
        mq.reserve(lane, nxt_cnt);
        if (nxt < cnt)
          stage_block<D, T, COST>(p, vin, entry_block(nblk), wtile + (stage ^ 1) * S::N,
                                  wnodes + (stage ^ 1), lane);
      };
#endif
      tm.mark(1);
      const int ch = sweep_block<D, T, RULE, COST>(p, s, bid, wtile + stage * S::N, wnodes + stage,
                                                    vout, s_done, s_max, gmax_row, evals, exec,
                                                    xreal, s_pc, pm, tm, hook, copy_visit);
      ++blocks_done;
#ifdef PHJ_TIMING
      if (lane == 0 && banded) atomicAdd(&g_visit_kind[copy_visit ? 3 : ch], 1ull);
#endif
      // the band schedule, not the activity, drives the pass
      mq.issue(p.tg, p.g, bid, banded ? 0 : ch, lane, nxt_flags);
      tm.mark(6);
      __syncwarp();  // the buffers of this block are refilled two blocks later
      item = nxt;
      blk = nblk;
#if PHJ_EARLY_STAGE
      nxt = nn;
      nblk = nnblk;
#endif
      stage ^= 1;
    }
    if (lane == 0 && sw + 1 <= p.max_sweeps) ticket = atomicAdd(&p.ws.take[sw + 1], 1);
    mq.store(nxt_list);
    mq.reserve(lane, nxt_cnt);
    mq.store(nxt_list);
    flush_patch_max(p, pm, s_max, gmax_row);
    tm.mark(8);
    __syncthreads();
    tm.mark(9);
    for (int i = threadIdx.x; i < nshared; i += blockDim.x)
      if (s_max[i]) atomicMax(&gmax_row[i * kMaxPad], s_max[i]);
    grid.sync();
    tm.mark(10);
    ++sw;
    buf ^= 1;
    int pending = 0;
    for (int i = threadIdx.x; i < p.R; i += blockDim.x) {
      if (s_done[i] == 0x7fffffff) {
        const unsigned long long mb = ld_cg(&gmax_row[i * kMaxPad]);
        if (blockIdx.x == 0) p.maxch[(int64_t)(sw - 1) * p.R + i] = mb;
        const double mc = __longlong_as_double((long long)mb);
        // no per-patch stop inside the value-ordered pass (its sweeps see a
        // window of the patch only)
        if (sw > p.n_band && mc <= p.tol) s_done[i] = sw;
        else pending = 1;
      }
    }
    const int any_pending = __syncthreads_or(pending);
    tm.mark(7);
    if (p.band_only && sw >= p.n_band) break;
    if (!any_pending || sw >= p.max_sweeps) break;
  }
#ifdef PHJ_TIMING
  if (lane == 0)
    for (int i = 0; i < 12; ++i) atomicAdd(&g_phase_cycles[i], tm.acc[i]);
#endif
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
  __shared__ unsigned long long s_ev, s_ex, s_xr;
  __shared__ int s_blk;
  if (threadIdx.x == 0) {
    s_ev = 0;
    s_ex = 0;
    s_xr = 0;
    s_blk = 0;
  }
  __syncthreads();
  atomicAdd(&s_ev, evals);
  atomicAdd(&s_ex, exec);
  atomicAdd(&s_xr, xreal);
  if (lane == 0) atomicAdd(&s_blk, blocks_done);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&p.evals[0], s_ev);
    atomicAdd(&p.evals[1], s_ex);
    atomicAdd(&p.evals[2], s_xr);
    atomicAdd(&p.info[2], s_blk);
  }
  if (p.pcount && p.R <= kSmemPatchReduce)
    for (int i = threadIdx.x; i < p.R * 3; i += blockDim.x)
      if (s_pc[i]) atomicAdd(&p.pcount[i], s_pc[i]);
}

// ---------------------------------------------------------------------------
// Asynchronous (chaotic) relaxation of the same fixed point -- no grid
// barrier.  One value buffer updated in place; work = a FIFO ring of block
// ids with one state word per block:
//   0 idle, 1 queued, 2 being swept, 3 being swept + dirty (a neighbour
//   changed after the sweep started; the sweeper re-queues the block).
// A block is therefore never swept by two warps at once, each node is
// written only by its block's sweeper, and every value stays an upper bound
// of the fixed point that never rises (the SL map is monotone; any mixture
// of newer and older neighbour values >= v* maps to a value >= v*).  A node
// change above the activity threshold re-queues the 3^D block neighbourhood
// (the block itself included); the solve ends when nothing is queued or
// being swept (`pending` = 0), i.e. when no node of a swept block can change
// by more than the threshold -- the fixed point to within the threshold.
// The FIFO is a bounded ring of 64-bit cells with per-cell sequence numbers
// (high word) so a slow ticket holder can never miss or lose an entry when
// the ring laps: a push at position p waits for seq == p and stores p + 1, a
// pop with ticket t waits for seq == t + 1 and stores t + cap.  Capacity =
// blocks + launched warps (at most one queued entry per block, one waiting
// ticket per warp).  Tickets are claimed only by idle warps (claiming one
// ahead while busy lets a push wait on a ticket whose busy holder is itself
// waiting in a push -- a cycle, observed); a push at position P can then only
// wait on the reader of P - cap, who waits on the push of P - cap: a strictly
// descending chain, so pushes always complete.
struct AsyncQ {
  unsigned long long* ring;  // [cap] (seq << 32) | block id
  int* state;                // [blocks]
  unsigned int* head;        // tickets taken
  // low word: push positions reserved beyond the initial n0; high word:
  // queued + in-flight blocks minus n0 (one atomic updates both)
  unsigned long long* tp;
  int* abort;                // processing budget exhausted
  unsigned int* swept;       // blocks swept (budget; flushed per warp in batches)
};

template <int D>
__device__ __forceinline__ AsyncQ async_queue(const Workspace& ws) {
  AsyncQ q;
  q.ring = ws.ring;
  q.state = ws.flags[0];
  q.head = (unsigned int*)&ws.take[0];
  q.abort = &ws.take[3];
  q.swept = (unsigned int*)&ws.take[4];
  q.tp = (unsigned long long*)&ws.take[6];
  return q;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *(const volatile unsigned long long*)p;
}

__device__ __forceinline__ int async_pending(const AsyncQ& q) {
  return (int)(unsigned)(ld_volatile_u64(q.tp) >> 32);
}

// lane-0 pop with ticket t: the next block id, or -1 once nothing is queued
// or in flight (or the budget ran out)
__device__ __forceinline__ int async_pop(const AsyncQ& q, unsigned cap, int n0, unsigned budget) {
  const unsigned t = atomicAdd(q.head, 1u);
  unsigned long long* cell = &q.ring[t % cap];
  unsigned ns = 32;
  for (;;) {
    const unsigned long long c = ld_volatile_u64(cell);
    if ((unsigned)(c >> 32) == t + 1u) {
      *(volatile unsigned long long*)cell = ((unsigned long long)(t + cap) << 32) | 0xffffffffull;
      return (int)(unsigned)(c & 0xffffffffull);
    }
    if (n0 + async_pending(q) == 0 || *(const volatile int*)q.abort) return -1;
    if (*(const volatile unsigned*)q.swept >= budget) {  // idle warps watch the budget
      atomicExch(q.abort, 1);
      return -1;
    }
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : ns;
  }
}

// push of block `blk` at absolute position `pos` (the cell is free unless a
// previous-lap ticket holder left on an abort)
__device__ __forceinline__ void async_push(const AsyncQ& q, unsigned cap, unsigned pos, int blk) {
  unsigned long long* cell = &q.ring[pos % cap];
  while ((unsigned)(ld_volatile_u64(cell) >> 32) != pos) {
    if (*(const volatile int*)q.abort) return;
    __nanosleep(64);
  }
  atomicExch(cell, ((unsigned long long)(pos + 1u) << 32) | (unsigned)blk);
}

// Release the visited block (back to idle, or re-queued when a neighbour
// dirtied it during the visit) and queue the neighbours whose state went
// 0 -> 1 (`want` lanes), with ONE atomic on the packed (pending, positions)
// word: pending += pushes - (released ? 1 : 0), so it cannot reach 0 while
// work remains.  The caller has fenced its value writes before marking.
__device__ __forceinline__ void async_requeue_release(const AsyncQ& q, unsigned cap, int n0,
                                                      int blk, bool want, int nt, int lane,
                                                      unsigned budget, unsigned& swept_local) {
  const unsigned FULL = 0xffffffffu;
  int dirty = 0;
  if (lane == 0) {
    const int old = atomicCAS(&q.state[blk], 2, 0);
    if (old == 3) {
      atomicExch(&q.state[blk], 1);
      dirty = 1;
    }
  }
  const unsigned bal = __ballot_sync(FULL, want);
  unsigned base = 0;
  if (lane == 0) {
    const int npush = __popc(bal);
    const int dpend = npush - (dirty ? 0 : 1);
    const unsigned npos = (unsigned)(npush + dirty);
    const unsigned long long add =
        ((unsigned long long)(unsigned)dpend << 32) + (unsigned long long)npos;
    base = (unsigned)atomicAdd(q.tp, add);
    if (dirty) async_push(q, cap, (unsigned)n0 + base + (unsigned)npush, blk);
    atomicAdd(q.swept, 1u);  // result unused: a fire-and-forget reduction
    if (++swept_local == 32u) {
      if (*(const volatile unsigned*)q.swept >= budget) atomicExch(q.abort, 1);
      swept_local = 0u;
    }
  }
  base = __shfl_sync(FULL, base, 0);
  if (want) async_push(q, cap, (unsigned)n0 + base + __popc(bal & ((1u << lane) - 1u)), nt);
}



// initial ring: positions < n0 hold the build_list blocks, the rest are free
__global__ void async_ring_init(unsigned long long* ring, unsigned cap, const int* list,
                                const int* count) {
  const unsigned n0 = (unsigned)*count;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x)
    ring[i] = i < n0 ? (((unsigned long long)(i + 1u) << 32) | (unsigned)list[i])
                     : (((unsigned long long)i << 32) | 0xffffffffull);
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}
__device__ __forceinline__ int ld_volatile(const int* p) {
  return *(const volatile int*)p;
}

template <int D, typename T, int RULE, int COST, bool WCLS>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    solve_async_kernel(const __grid_constant__ SolveParams p, unsigned int budget) {
  using S = TileShape<D>;
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool warp_cls = WCLS;
  const int64_t sbytes = solve_stencil_bytes<D, T>(WCLS ? 2 : 1, p.nc);
  StencilSmem<D, T> s =
      WCLS ? carve_stencil<D, T>(smem + (threadIdx.x >> 5) * solve_stencil_slot<D, T>(p.nc), 1,
                                 p.nc)
           : carve_stencil<D, T>(smem, 1, p.nc);
  int* s_done = (int*)(smem + sbytes);
  unsigned long long* s_max = (unsigned long long*)(s_done + ((p.R + 1) / 2 * 2));
  unsigned long long* s_pc = s_max + min(p.R, kSmemPatchReduce);  // [min(R,64)][3]
  T* tiles = (T*)(smem + align_up(sbytes + (int64_t)((p.R + 1) / 2 * 2) * 4 +
                                      (int64_t)min(p.R, kSmemPatchReduce) * 8 * 4,
                                  16));
  T* wtile = tiles + (threadIdx.x >> 5) * 2 * S::N;
  NodeStage<D, T>* wnodes =
      (NodeStage<D, T>*)(tiles + kWarps * 2 * S::N) + (threadIdx.x >> 5) * 2;
  if (!warp_cls)
    stage_stencil<D, T, RULE>(s, p.n_classes, p.nc, p.oct_start, p.nzmask, p.weights, p.cost,
                              p.ctrl);
  int wcls = -1;
  for (int i = threadIdx.x; i < p.R; i += blockDim.x)
    s_done[i] = (p.mine == nullptr || p.mine[i]) ? 0x7fffffff : 0;
  for (int i = threadIdx.x; i < min(p.R, kSmemPatchReduce); i += blockDim.x) s_max[i] = 0ull;
  for (int i = threadIdx.x; i < min(p.R, kSmemPatchReduce) * 3; i += blockDim.x) s_pc[i] = 0ull;
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const AsyncQ q = async_queue<D>(p.ws);
  const int n0 = ld_cg(&p.ws.counts[0]);
  const unsigned cap = (unsigned)p.tg.total + (unsigned)(gridDim.x * kWarps);
  unsigned swept_local = 0;
  unsigned long long* gmax_row = sweep_max_slots(p.ws, 0);
  unsigned long long evals = 0, exec = 0, xreal = 0;
  int blocks_done = 0;
  PatchMax pm{-1, 0.0};
  PhaseTimer tm;
  tm.start();
  constexpr int NNB = D == 2 ? 9 : 27;
  constexpr int self = D == 2 ? 4 : 13;
  for (;;) {
    // -- pop: one ticket per warp, wait for its slot (or for the end) --------
    int blk = -1;
    // warp-uniform: lanes still finishing their pushes read the flag later
    if (__shfl_sync(FULL, lane == 0 ? ld_volatile(q.abort) : 0, 0)) break;
    if (lane == 0) {
      blk = async_pop(q, cap, n0, budget);
      if (blk >= 0) {
        atomicExch(&q.state[blk], 2);
      }
    }
    blk = __shfl_sync(FULL, blk, 0);
    if (blk < 0) break;
    fence_acq_rel_gpu();  // neighbour values are read after the slot / state
    tm.mark(0);
    if (warp_cls) {
      int bc[3];
      decode_block<D>(p.tg, blk, bc);
      if (bc[0] != wcls) {
        __syncwarp();
        stage_class<D, T, RULE>(s, bc[0], p.nc, lane, p.oct_start, p.nzmask, p.weights, p.cost, p.ctrl);
        wcls = bc[0];
      }
    }
    stage_block<D, T, COST>(p, (const T*)p.v[0], blk, wtile, wnodes, lane);
    cp_async_wait_all();
    __syncwarp();
    tm.mark(1);
    auto hook = []() {};
    const int ch = sweep_block<D, T, RULE, COST>(p, s, blk, wtile, wnodes, (T*)p.v[0], s_done,
                                                 s_max, gmax_row, evals, exec, xreal, s_pc, pm,
                                                 tm, hook);
    ++blocks_done;
#ifdef PHJ_TIMING
    if (lane == 0) atomicAdd(&g_visit_kind[ch], 1ull);
#endif
    // -- re-queue the neighbourhood of a changed block ------------------------
    bool want = false;
    int nt = -1;
    if (ch != 0) __threadfence();  // node values before the state words (release too)
    __syncwarp();
    if (ch == 2) {
      if (lane < NNB) {
        nt = neighbour_block<D>(p.tg, p.g, blk, lane);
        if (nt >= 0) want = atomicOr(&q.state[nt], 1) == 0;
      }
    }
#ifdef PHJ_TIMING
    if (lane == 0) timeline_visit();
#endif
    async_requeue_release(q, cap, n0, blk, want, nt, lane, budget, swept_local);
    tm.mark(6);
  }
  flush_patch_max(p, pm, s_max, gmax_row);
#ifdef PHJ_TIMING
  if (lane == 0)
    for (int i = 0; i < 12; ++i) atomicAdd(&g_phase_cycles[i], tm.acc[i]);
#endif
  __shared__ unsigned long long s_ev, s_ex, s_xr;
  __shared__ int s_blk;
  if (threadIdx.x == 0) {
    s_ev = 0;
    s_ex = 0;
    s_xr = 0;
    s_blk = 0;
  }
  __syncthreads();
  atomicAdd(&s_ev, evals);
  atomicAdd(&s_ex, exec);
  atomicAdd(&s_xr, xreal);
  if (lane == 0) atomicAdd(&s_blk, blocks_done);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&p.evals[0], s_ev);
    atomicAdd(&p.evals[1], s_ex);
    atomicAdd(&p.evals[2], s_xr);
    atomicAdd(&p.info[2], s_blk);
  }
  if (p.pcount && p.R <= kSmemPatchReduce)
    for (int i = threadIdx.x; i < p.R * 3; i += blockDim.x)
      if (s_pc[i]) atomicAdd(&p.pcount[i], s_pc[i]);
}

// Per-patch results of an asynchronous solve: "sweeps" = blocks swept /
// initial blocks (rounded up; an equivalent sweep count), negated when the
// budget ran out.
__global__ void async_finish_kernel(Workspace ws, int R, const uint8_t* mine,
                                    int32_t* patch_sweeps, int32_t* info) {
  // equivalent sweeps: block visits / blocks holding work (take[5], counted
  // by the async solve's build_list; the transport queues all of them)
  const int n0 = max(1, ws.take[5] > 0 ? ws.take[5] : ws.counts[0]);
  const unsigned swept = (unsigned)ws.take[4];
  const int eq = (int)((swept + (unsigned)n0 - 1u) / (unsigned)n0);
  const bool aborted = ws.take[3] != 0;
  for (int i = threadIdx.x; i < R; i += blockDim.x)
    patch_sweeps[i] = (mine == nullptr || mine[i]) ? (aborted ? -eq : max(eq, 1)) : 0;
  if (threadIdx.x == 0) {
    info[0] = max(eq, 1);
    info[1] = 0;
  }
}

// Colour transport seeding: OR colour j into the masks of the 3^D block
// neighbourhood of every node of part j.  A mover whose 3^D neighbourhood
// holds no part-j node starts at phi_j = 0 with every foot corner at 0, so
// only seeded (block, colour) pairs can change in the first sweep / visit.
template <int D>
__global__ void transport_seed_kernel(phj_grid g, TileGrid tg, const int64_t* __restrict__ flat,
                                      const int32_t* __restrict__ col, int64_t n,
                                      unsigned long long* __restrict__ mask) {
  using B = Blk<D>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t f = flat[i];
    int c[3];
    for (int ax = 0; ax < D; ++ax) {
      c[ax] = (int)(f / g.strides[ax]) - 1;
      f -= (int64_t)(c[ax] + 1) * g.strides[ax];
    }
    int t;
    if (D == 2) t = (c[0] / B::BY) * tg.n[1] + c[1] / B::BX;
    else t = (c[0] * tg.n[1] + c[1] / B::BY) * tg.n[2] + c[2] / B::BX;
    const unsigned long long bit = 1ull << col[i];
    for (int q = 0; q < (D == 2 ? 9 : 27); ++q) {
      const int nb = neighbour_block<D>(tg, g, t, q);
      if (nb >= 0) atomicOr(&mask[nb], bit);
    }
  }
}

// Initial active block list: every block holding a node to sweep (solve:
// label >= 0 of a mine patch; transport: a mover).  One warp per block.
template <int D>
__global__ void build_list_kernel(phj_grid g, TileGrid tg, const int16_t* __restrict__ lab,
                                  const uint8_t* __restrict__ mine, int* flags, int* list,
                                  int* count, int want_movers, const int32_t* __restrict__ fb,
                                  const int8_t* __restrict__ kind, unsigned long long* mask0,
                                  unsigned long long mask_all, const void* __restrict__ vfin = nullptr,
                                  int vfin_f32 = 0, double finite_below = 0.0,
                                  int* n_work = nullptr, int seeded = 0) {
  constexpr int NB = Blk<D>::NB;
  const int lane = threadIdx.x & 31;
  const int blk = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (blk >= tg.total) return;  // whole warp
  int c[3];
  const bool row_ok = lane_nodes<D>(g, tg, blk, lane, c);
  bool any = false, work = false;
  if (row_ok) {
    const int64_t f0 = ext_flat<D>(g, c);
    const int64_t s0 = serial_of<D>(g, c);
    for (int r = 0; r < NB; ++r) {
      if (c[D - 1] + r >= g.shape[D - 1]) break;
      if (want_movers) {
        const bool mv = fb[s0 + r] >= 0 && kind[s0 + r] == 0;
        any |= mv;
        work |= mv;
      } else {
        const int l = lab[f0 + r];
        bool take = l >= 0 && (mine == nullptr || mine[l]);
        work |= take;
        if (take && vfin) {
          // value solves: a node can only move if some value in its 3^D
          // neighbourhood is below the unreached level or its own value is
          // above it (with every corner unreached, every candidate equals
          // the unreached level exactly) -- cold solves start at the blocks
          // next to the target instead of every block
          bool fin = (vfin_f32 ? (double)((const float*)vfin)[f0 + r]
                               : ((const double*)vfin)[f0 + r]) > finite_below;
          for (int q = 0; q < (D == 2 ? 9 : 27); ++q) {
            int64_t off;
            if (D == 2) off = (int64_t)(q / 3 - 1) * g.strides[0] + (q % 3 - 1);
            else
              off = (int64_t)(q / 9 - 1) * g.strides[0] + (int64_t)((q / 3) % 3 - 1) * g.strides[1] +
                    (q % 3 - 1);
            const double x = vfin_f32 ? (double)((const float*)vfin)[f0 + r + off]
                                      : ((const double*)vfin)[f0 + r + off];
            fin |= x < finite_below;
          }
          take = fin;
        }
        any |= take;
      }
    }
  }
  if (n_work && __any_sync(0xffffffffu, work) && lane == 0) atomicAdd(n_work, 1);
  // seeded transport: only blocks whose colour mask was seeded next to a part
  if (seeded) any = any && mask0[blk] != 0ull;
  if (__any_sync(0xffffffffu, any) && lane == 0) {
    flags[blk] = 1;
    if (mask0 && !seeded) mask0[blk] = mask_all;
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
  void* phi[2];        // colour-major [R][ext] planes of PT (double or float)
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
  // value-ordered pass (transport_kernel only): sweeps < n_band visit
  // band_list[band_off[s] ..] (b: update, -b-1: copy to the other buffer)
  const int32_t* band_list;
  const int32_t* band_off;
  int n_band;
  int chunk;  // list entries per work ticket (1 or 2; transport_kernel)
};

#ifndef PHJ_TRANSPORT_CTAS
#define PHJ_TRANSPORT_CTAS 2
#endif
template <int D, typename PT>
__global__ void __launch_bounds__(kThreads, PHJ_TRANSPORT_CTAS) transport_kernel(const __grid_constant__ TransportParams p) {
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
  const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * kWarps;
  // Items are claimed two ahead (raw tickets on lane 0, first dynamic claims
  // of a sweep issued before the previous barrier), block ids read one
  // ahead, and a block's colour mask and mover entries are loaded while the
  // previous block is processed: an item's own work is a few FMAs per colour,
  // so without the lookahead each item would wait on 3 dependent round trips.
  int ticket = 0, ticket2 = 0;
  if (lane == 0) {
    ticket = atomicAdd(&p.ws.take[0], 1);
    ticket2 = atomicAdd(&p.ws.take[0], 1);
  }
  MarkQueue<D> mq;
  mq.init();
  // value-ordered pass: the colours that reached a block accumulate in a
  // sticky mask (never cleared), the array the first Jacobi sweep consumes
  unsigned long long* sticky = p.ws.cmask[p.n_band & 1];
  for (;;) {
    const PT* pin = (const PT*)p.phi[buf];
    PT* pout = (PT*)p.phi[buf ^ 1];
    const bool banded = sw < p.n_band;
    if (p.n_band > 0 && sw == p.n_band) {
      // end of the pass: every block some colour has reached enters the
      // first Jacobi sweep with all of its colours
      int* l0 = p.ws.list[sw & 1];
      for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < p.tg.total;
           b += gridDim.x * blockDim.x)
        if (__ldcg(&sticky[b]) != 0ull) l0[atomicAdd(&p.ws.counts[sw], 1)] = b;
      grid.sync();
    }
    const int cnt = banded ? (p.band_off[sw + 1] - p.band_off[sw]) : ld_cg(&p.ws.counts[sw]);
    const int* list = banded ? p.band_list + p.band_off[sw] : p.ws.list[sw & 1];
    int* cur_flags = p.ws.flags[sw & 1];
    unsigned long long* cur_mask = banded ? sticky : p.ws.cmask[sw & 1];
    unsigned long long* nxt_mask = banded ? sticky : p.ws.cmask[(sw + 1) & 1];
    int* nxt_list = p.ws.list[(sw + 1) & 1];
    int* nxt_cnt = &p.ws.counts[sw + 1];
    int* take = &p.ws.take[sw];
    for (int i = threadIdx.x; i < R; i += blockDim.x) s_max[i] = 0ull;
    if (blockIdx.x == 0) {
      unsigned long long* z = sweep_max_slots(p.ws, sw + 1);
      for (int i = threadIdx.x; i < R; i += blockDim.x) z[i * kMaxPad] = 0ull;
    }
    __syncthreads();
    // Lane -> node map of this kernel.  3D (8 x 8 plane blocks): node r of a
    // lane is row (lane / 8) + 4 r, column lane % 8, so a warp-wide gather of
    // one corner covers 4 rows of 8 consecutive elements (the shared Blk<3>
    // map -- 2 consecutive nodes per lane -- makes it 8 rows of 4 elements
    // 16 bytes apart: twice the L1 wavefronts, and the two nodes' requests
    // hit the same sectors).  2D: the Blk<2> map.
    constexpr bool kRowSplit = D == 3 && B::BY == 8 && B::BX == 8 && NB == 2;
    auto locate = [&](int b, bool (&in)[NB], int64_t (&ff)[NB], int64_t (&ss)[NB], int& c0) {
      if constexpr (kRowSplit) {
        int bb[3];
        decode_block<D>(p.tg, b, bb);
        c0 = bb[0];
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          int cc[3] = {bb[0], bb[1] * 8 + (lane >> 3) + 4 * r, bb[2] * 8 + (lane & 7)};
          in[r] = cc[1] < g.shape[1] && cc[2] < g.shape[2];
          ff[r] = ext_flat<D>(g, cc);
          ss[r] = serial_of<D>(g, cc);
        }
      } else {
        int cc[3];
        const bool rok = lane_nodes<D>(g, p.tg, b, lane, cc);
        c0 = cc[0];
        const int64_t f0 = ext_flat<D>(g, cc), s0 = serial_of<D>(g, cc);
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          in[r] = rok && cc[last] + r < g.shape[last];
          ff[r] = f0 + r;
          ss[r] = s0 + r;
        }
      }
    };
    // prefetch of one item: its colour mask (lane 0) and mover entries
    auto prefetch = [&](int b, unsigned long long& pcm, int (&pe)[NB]) {
      b = b < 0 ? -b - 1 : b;  // banded copy entries
      bool in[NB];
      int64_t ff[NB], ss[NB];
      int c0;
      locate(b, in, ff, ss, c0);
      pcm = 0ull;
      if (lane == 0) {
        pcm = __ldcg(&cur_mask[b]);
        if (!banded) cur_mask[b] = 0ull;
        cur_flags[b] = 0;
      }
#pragma unroll
      for (int r = 0; r < NB; ++r) pe[r] = in[r] ? __ldg(&p.ent[ss[r]]) : -1;
    };
    // A ticket buys kChunk consecutive list entries: the claims of a sweep all
    // hit one counter, and same-address atomics serialise in L2 (54 k tickets
    // of a config-5 sweep: 38 us, scripts/atomic_ticket_probe.cu), a floor
    // every rank of a multi-GPU run pays in full.  Dynamic item q >= 1 of the
    // warp is entry nwarps + kChunk * T[(q - 1) / kChunk + 1] + (q - 1) % kChunk.
    // One entry per ticket keeps a single GPU best balanced (C5 transport
    // 127 vs 130 ms with pairs); a rank that owns few colours finds most
    // entries empty and is bound by the claims: pairs (PHJ_TRANSPORT_PAIRS)
    // take rank 0 of 8 from 47.8 to 36.5 ms.
    const int kChunk = p.chunk;
    int item = gwarp;
    int blk = item < cnt ? __ldcg(&list[item]) : 0;
    int nxt = nwarps + kChunk * __shfl_sync(FULL, ticket, 0);  // q = 1: first entry of ticket 1
    int qn = 1;                                                // stream position of nxt
    int nblk = (item < cnt && nxt < cnt) ? __ldcg(&list[nxt]) : 0;
    unsigned long long cm_l0 = 0ull;
    int e[NB];
    if (item < cnt) prefetch(blk, cm_l0, e);
    while (item < cnt) {
      // lookahead: the item after next (a new ticket every kChunk items: the
      // one claimed kChunk iterations ago), next block's inputs
      int nn;
      if ((qn & (kChunk - 1)) == 0) {
        nn = nwarps + kChunk * __shfl_sync(FULL, ticket2, 0);
        if (lane == 0) {
          ticket = ticket2;
          if (nxt < cnt && nn < cnt) ticket2 = atomicAdd(take, 1);
        }
      } else {
        nn = nxt + 1;
      }
      ++qn;
      const int nnblk = (nxt < cnt && nn < cnt) ? __ldcg(&list[nn]) : 0;
      unsigned long long ncm_l0 = 0ull;
      int ne[NB];
#pragma unroll
      for (int r = 0; r < NB; ++r) ne[r] = -1;
      if (nxt < cnt) prefetch(nblk, ncm_l0, ne);
      mq.store(nxt_list);
      mq.reserve(lane, nxt_cnt);

      // colours active in this block: those a neighbour block changed in the
      // previous sweep (exact per colour, like the block skipping)
      const unsigned long long cm = __shfl_sync(FULL, cm_l0, 0);
      const bool copy_only = blk < 0;  // banded: last visit, copy to the other buffer
      const int bid = copy_only ? -blk - 1 : blk;
      bool in_grid[NB];
      int64_t fr[NB], sr_unused[NB];  // ext flat index of the lane's nodes
      int c0;                         // their index along internal axis 0
      locate(bid, in_grid, fr, sr_unused, c0);
      int64_t base[NB];
      bool any = false;
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        base[r] = fr[r];
        if (e[r] >= 0) {
          const int oc = s_oct[e[r]];
#pragma unroll
          for (int ax = 0; ax < D; ++ax)
            if (!((oc >> ax) & 1)) base[r] -= g.strides[ax];
          any = true;
          upd += copy_only ? 0 : 1;
        }
      }
      unsigned long long changed = 0;
      if (copy_only && __any_sync(FULL, any)) {
        // banded pass, last visit of the block: its movers' values into the
        // other buffer (no gathers; the values did not change in this sweep)
        unsigned long long todo = cm;
        while (todo) {
          const int j = __ffsll((long long)todo) - 1;
          todo &= todo - 1;
          const PT* pj = pin + (int64_t)j * p.plane;
          PT* qj = pout + (int64_t)j * p.plane;
#pragma unroll
          for (int r = 0; r < NB; ++r) {
            if (e[r] < 0) continue;
            const PT v = pj[fr[r]];
            qj[fr[r]] = v;
            if (per0) {
              if (c0 == 0) qj[fr[r] + ghost_shift] = v;
              else if (c0 == M0 - 1) qj[fr[r] - ghost_shift] = v;
            }
          }
        }
      } else if (__any_sync(FULL, any)) {
        // corner pairs along the last axis are adjacent elements: one offset
        // per pair (NC / 2 per node), the partner is the next element.  Nodes
        // without an entry read their own cell (values unused).
        constexpr int NP = NC / 2;
        constexpr int KL = 1 << last;  // corner bit of the last axis
        // (lanes of a partial block at the far grid edge lie outside the
        // array: they read a clamped in-plane location)
        int64_t fsafe[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r) fsafe[r] = min(fr[r], p.plane - 2);
        int64_t poff[NB][NP];
#pragma unroll
        for (int r = 0; r < NB; ++r)
#pragma unroll
          for (int m = 0; m < NP; ++m) poff[r][m] = e[r] >= 0 ? base[r] + coff[m] : fsafe[r];
        // colours in batches of CB: all corner loads of a batch are in flight
        // together.  3D: one colour per batch -- a block holds 3.6 colours on
        // average at config 5, so pairs waste a slot on odd counts (C5 151 ->
        // 141 ms, profiles/r2y_transport_variants.jsonl)
#ifndef PHJ_TCB2
#define PHJ_TCB2 1
#endif
#ifndef PHJ_TCB3
#define PHJ_TCB3 1
#endif
        constexpr int CB = (D == 2) ? PHJ_TCB2 : PHJ_TCB3;
        const bool masked = R <= 64;
        unsigned long long todo = masked ? cm : 0ull;
        int jnext = 0;  // unmasked (R > 64): every colour in order
        for (;;) {
          int js[CB];
          bool anyj = false;
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            if (masked) {
              js[q] = todo ? __ffsll((long long)todo) - 1 : -1;
              todo &= todo ? todo - 1 : 0ull;
            } else {
              js[q] = jnext < R ? jnext : -1;
              ++jnext;
            }
            anyj |= js[q] >= 0;
          }
          if (!anyj) break;
          // an empty slot of the last batch re-reads slot 0's colour (unused)
          PT cv[CB][NB][NC], ov[CB][NB];
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            const PT* pj = pin + (int64_t)(js[q] >= 0 ? js[q] : js[0]) * p.plane;
#pragma unroll
            for (int r = 0; r < NB; ++r) {
#pragma unroll
              for (int m = 0; m < NP; ++m) {
                const PT* pr = pj + poff[r][m];
                cv[q][r][m] = pr[0];
                cv[q][r][m + KL] = pr[1];
              }
              // the node's old value (it is also a corner of its foot cell:
              // an L1 hit)
              ov[q][r] = pj[fsafe[r]];
            }
          }
          double lmax[CB];
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            lmax[q] = 0.0;
            if (js[q] < 0) continue;
            const int j = js[q];
            const bool live = !copy_only && s_done[j] == 0x7fffffff;
            PT* qj = pout + (int64_t)j * p.plane;
#pragma unroll
            for (int r = 0; r < NB; ++r) {
              if (e[r] < 0) continue;
              double acc = 0.0;
              const double old = (double)ov[q][r];
#pragma unroll
              for (int k = 0; k < NC; ++k)
                acc = fma(s_w[k * wpitch + e[r]], (double)cv[q][r][k], acc);
              const PT nv = live ? (PT)acc : ov[q][r];  // changes measured on the stored value
              lmax[q] = fmax(lmax[q], fabs(old - (double)nv));
              qj[fr[r]] = nv;
              if (per0) {
                if (c0 == 0) qj[fr[r] + ghost_shift] = nv;
                else if (c0 == M0 - 1) qj[fr[r] - ghost_shift] = nv;
              }
            }
          }
          // warp maximum on the bit patterns (values >= 0: the integer order
          // of (high, low) words is the value order) -- two REDUX per colour
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            const int hi = __double2hiint(lmax[q]);
            const int mh = __reduce_max_sync(FULL, hi);
            const unsigned lo = hi == mh ? (unsigned)__double2loint(lmax[q]) : 0u;
            const unsigned ml = __reduce_max_sync(FULL, lo);
            lmax[q] = __hiloint2double(mh, (int)ml);
          }
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            if (js[q] < 0 || !(lmax[q] > 0.0)) continue;
            const int j = js[q];
            if (lane == 0) atomicMax(&s_max[j], dbits(lmax[q]));
            // activity threshold: changes <= act_eps (a small fraction of the
            // stopping tolerance) do not re-activate the neighbourhood
            if (lmax[q] > p.act_eps) changed |= (j < 64) ? (1ull << j) : ~0ull;
          }
        }
      }
      mq.issue_mask(p.tg, g, bid, changed, lane, nxt_mask, !banded);
      item = nxt;
      blk = nblk;
      nxt = nn;
      nblk = nnblk;
      cm_l0 = ncm_l0;
#pragma unroll
      for (int r = 0; r < NB; ++r) e[r] = ne[r];
    }
    if (lane == 0 && sw + 1 <= p.max_sweeps) {
      // the two leading claims of the next sweep
      ticket = atomicAdd(&p.ws.take[sw + 1], 1);
      ticket2 = atomicAdd(&p.ws.take[sw + 1], 1);
    }
    mq.store(nxt_list);
    mq.reserve(lane, nxt_cnt);
    mq.store(nxt_list);
    __syncthreads();
    unsigned long long* grow = sweep_max_slots(p.ws, sw);  // padded: entry i at i * kMaxPad
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      if (s_max[i]) atomicMax(&grow[i * kMaxPad], s_max[i]);
    grid.sync();
    ++sw;
    buf ^= 1;
    int pending = 0;
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      if (s_done[i] == 0x7fffffff) {
        const unsigned long long mb = ld_cg(&grow[i * kMaxPad]);
        if (blockIdx.x == 0) p.maxch[(int64_t)(sw - 1) * R + i] = mb;
        const double mc = __longlong_as_double((long long)mb);
        // no stop inside the value-ordered pass (its sweeps see a window only)
        if (sw > p.n_band && mc <= p.tol) s_done[i] = sw;
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

// ---------------------------------------------------------------------------
// Asynchronous colour transport (PHJ_TRANSPORT_ASYNC): the same block FIFO
// and state machine as solve_async_kernel, one phi buffer updated in place,
// per-block pending-colour masks (OR-ed by the neighbours that changed those
// colours).  phi only grows (from the 0/1 start, every read mixture is <= the
// fixed point and >= the values the previous update of the node read; the
// FMA chain of non-negative weights is monotone), so the iteration converges
// to the fixed point; a colour change above act_eps re-queues the 3^D block
// neighbourhood for that colour.
// A visit stages the halo tiles of up to kTC pending colours at once (all
// their L2 loads in flight together), relaxes the block's movers up to
// `inner` times in shared memory (halo fixed, own values updated in place),
// and writes back the changed own values.
template <int D>
struct TTile {
  static constexpr int TC = D == 2 ? 8 : 4;  // colours staged per chunk
  static constexpr int N = TileShape<D>::N;
};

template <int D, typename PT>
__global__ void __launch_bounds__(kThreads, PHJ_TRANSPORT_CTAS)
    transport_async_kernel(const __grid_constant__ TransportParams p, int inner,
                           unsigned int budget) {
  using B = Blk<D>;
  using S = TileShape<D>;
  constexpr int NC = 1 << D;
  constexpr int NB = B::NB;
  constexpr int last = D - 1;
  constexpr int TC = TTile<D>::TC;
  constexpr int W = B::BX + 2;  // tile columns used
  constexpr int NT = S::R * W;  // tile elements used
  extern __shared__ __align__(16) unsigned char smem[];
  const int nent = p.n_classes * p.nc;
  const int R = p.R;
  const int wpitch = nent | 1;
  double* s_w = (double*)smem;                                           // [NC][wpitch]
  double* s_tiles = s_w + (int64_t)wpitch * NC;                          // [warps][TC][N]
  signed char* s_oct = (signed char*)(s_tiles + (int64_t)kWarps * TC * S::N);  // [nent]
  for (int i = threadIdx.x; i < nent * NC; i += blockDim.x)
    s_w[(i % NC) * wpitch + i / NC] = p.weights[i];
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
  double* wt = s_tiles + (int64_t)(threadIdx.x >> 5) * TC * S::N;
  const int64_t M0 = g.shape[0];
  const bool per0 = g.periodic[0] != 0;
  const int64_t ghost_shift = M0 * g.strides[0];
  // tile strides per internal axis and corner offsets (bit ax = +1 on axis ax)
  int tstr[3];
  if constexpr (D == 2) {
    tstr[0] = S::C;
    tstr[1] = 1;
    tstr[2] = 0;
  } else {
    tstr[0] = S::RB * S::C;
    tstr[1] = S::C;
    tstr[2] = 1;
  }
  int tcoff[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    int o = 0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax)
      if ((k >> ax) & 1) o += tstr[ax];
    tcoff[k] = o;
  }
  const int nlast = (int)0;
  (void)nlast;
  const AsyncQ q = async_queue<D>(p.ws);
  unsigned long long* cmask = p.ws.cmask[0];
  const int n0 = ld_cg(&p.ws.counts[0]);
  const unsigned cap = (unsigned)p.tg.total + (unsigned)(gridDim.x * kWarps);
  unsigned swept_local = 0;
  PT* phi = (PT*)p.phi[0];
  unsigned long long upd = 0;
  constexpr int NNB = D == 2 ? 9 : 27;
  const int ly = lane / B::LX, lx = lane % B::LX;
  // this lane's node r sits at tile index tnode + r
  const int tnode = D == 2 ? (ly + 1) * S::C + lx * NB + 1
                           : (S::RB + ly + 1) * S::C + lx * NB + 1;
  PhaseTimer tm;
  tm.start();
  for (;;) {
    int blk = -1;
    unsigned long long cm = 0ull;
    if (__shfl_sync(FULL, lane == 0 ? ld_volatile(q.abort) : 0, 0)) break;
    if (lane == 0) {
      blk = async_pop(q, cap, n0, budget);
      if (blk >= 0) {
        atomicExch(&q.state[blk], 2);
        cm = atomicExch(&cmask[blk], 0ull);
      }
    }
    blk = __shfl_sync(FULL, blk, 0);
    if (blk < 0) break;
    cm = __shfl_sync(FULL, cm, 0);
    fence_acq_rel_gpu();
    tm.mark(0);
    int c[3];
    const bool row_ok = lane_nodes<D>(g, p.tg, blk, lane, c);
    const int64_t f0 = ext_flat<D>(g, c);
    const int64_t s0 = serial_of<D>(g, c);
    int e[NB], tb[NB];
    bool anym = false;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const bool in = row_ok && c[last] + r < g.shape[last];
      e[r] = in ? __ldg(&p.ent[s0 + r]) : -1;
      tb[r] = tnode + r;
      if (e[r] >= 0) {
        anym = true;
        const int oc = s_oct[e[r]];
#pragma unroll
        for (int ax = 0; ax < D; ++ax)
          if (!((oc >> ax) & 1)) tb[r] -= tstr[ax];
      }
    }
    // tile origin (ext coordinates of the block's lower halo corner) and the
    // clamps for partial blocks at the far grid edge
    int b[3];
    decode_block<D>(p.tg, blk, b);
    int64_t o, rs, s0x;
    int row0, col0, rmax, cmax;
    if constexpr (D == 2) {
      row0 = b[0] * B::BY;
      col0 = b[1] * B::BX;
      rs = g.strides[0];
      s0x = 0;
      o = (int64_t)row0 * rs + col0;
      rmax = (int)g.ext[0] - 1;
      cmax = (int)g.ext[1] - 1;
    } else {
      row0 = b[1] * B::BY;
      col0 = b[2] * B::BX;
      rs = g.strides[1];
      s0x = g.strides[0];
      o = (int64_t)b[0] * s0x + (int64_t)row0 * rs + col0;
      rmax = (int)g.ext[1] - 1;
      cmax = (int)g.ext[2] - 1;
    }
    unsigned long long changed = 0ull;
    bool anywrote = false;
    const bool work = __any_sync(FULL, anym) && cm != 0ull;
    const bool masked = R <= 64;
    unsigned long long todo = work ? (masked ? cm : ~0ull) : 0ull;
    int jnext = 0;
    while (todo) {
      // next chunk of pending colours
      int js[TC];
      int nj = 0;
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        int j = -1;
        if (masked) {
          if (todo) {
            j = __ffsll((long long)todo) - 1;
            todo &= todo - 1;
          }
        } else if (jnext < R) {
          j = jnext++;
          if (jnext >= R) todo = 0ull;
        }
        js[t] = j;
        nj += j >= 0;
      }
      if (!masked && jnext >= R) todo = 0ull;
      // stage: every halo value of every chunk colour, loads issued together
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        if (js[t] < 0) continue;
        const PT* pj = phi + (int64_t)js[t] * p.plane;
        double* tt = wt + t * S::N;
#pragma unroll
        for (int i0 = 0; i0 < NT; i0 += 32) {
          const int i = i0 + lane;
          if (i < NT) {
            const int rr = i / W, cc = i - rr * W;
            int pl = 0, ry = rr;
            if constexpr (D == 3) {
              pl = rr / S::RB;
              ry = rr - pl * S::RB;
            }
            const int yy = min(row0 + ry, rmax) - row0, xx = min(col0 + cc, cmax) - col0;
            tt[rr * S::C + cc] = (double)__ldcg(pj + o + pl * s0x + (int64_t)yy * rs + xx);
          }
        }
      }
      __syncwarp();
      tm.mark(1);
      unsigned long long wrote = 0ull;
      for (int it = 0; it < inner; ++it) {
        unsigned long long bigm = 0ull;
#pragma unroll
        for (int t = 0; t < TC; ++t) {
          if (js[t] < 0) continue;
          double* tt = wt + t * S::N;
          bool big = false, any = false;
#pragma unroll
          for (int r = 0; r < NB; ++r) {
            if (e[r] < 0) continue;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < NC; ++k) acc = fma(s_w[k * wpitch + e[r]], tt[tb[r] + tcoff[k]], acc);
            const double old = tt[tnode + r];
            ++upd;
            const double nv = (double)(PT)acc;  // the value the field will hold
            if (nv > old) {
              big |= nv - old > p.act_eps;
              any = true;
              tt[tnode + r] = nv;
            }
          }
          if (__any_sync(FULL, any)) wrote |= 1ull << t;
          if (__any_sync(FULL, big)) bigm |= 1ull << t;
        }
        if (bigm == 0ull) break;
#pragma unroll
        for (int t = 0; t < TC; ++t)
          if ((bigm >> t) & 1ull) changed |= (js[t] < 64) ? (1ull << js[t]) : ~0ull;
        __syncwarp();
      }
      tm.mark(3);
      // write back the block's changed colours
      anywrote |= wrote != 0ull;
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        if (!((wrote >> t) & 1ull)) continue;
        PT* pj = phi + (int64_t)js[t] * p.plane;
        const double* tt = wt + t * S::N;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          if (e[r] < 0) continue;
          const PT v = (PT)tt[tnode + r];
          pj[f0 + r] = v;
          if (per0) {
            if (c[0] == 0) pj[f0 + r + ghost_shift] = v;
            else if (c[0] == M0 - 1) pj[f0 + r - ghost_shift] = v;
          }
        }
      }
      __syncwarp();  // the tiles are restaged by the next chunk
      (void)nj;
      tm.mark(4);
    }
    // re-queue the neighbourhood for the changed colours
    bool want = false;
    int nt = -1;
    if (anywrote) __threadfence();  // phi values before the state words (release too)
    __syncwarp();
    if (changed) {
      if (lane < NNB) {
        nt = neighbour_block<D>(p.tg, g, blk, lane);
        if (nt >= 0) {
          atomicOr(&cmask[nt], changed);
          want = atomicOr(&q.state[nt], 1) == 0;
        }
      }
    }
#ifdef PHJ_TIMING
    if (lane == 0) timeline_visit();
#endif
    async_requeue_release(q, cap, n0, blk, want, nt, lane, budget, swept_local);
    tm.mark(6);
  }
#ifdef PHJ_TIMING
  if (lane == 0)
    for (int i = 0; i < 12; ++i) atomicAdd(&g_phase_cycles[i], tm.acc[i]);
#endif
  __shared__ unsigned long long s_up;
  if (threadIdx.x == 0) s_up = 0;
  __syncthreads();
  atomicAdd(&s_up, upd);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(p.updates, s_up);
}

// ---------------------------------------------------------------------------
// Two Jacobi sweeps per grid barrier (default transport; PHJ_TRANSPORT_T1=1
// selects the one-sweep kernel above).
//
// The transport is a linear map with fixed feet, so an active block can run
// sweeps k and k+1 back to back: it stages its 2-ring halo of colour j,
// computes sweep k on the block plus a 1-node ring (the ring values are the
// same Jacobi images the neighbour blocks compute; recomputing them costs a
// few FMAs per node), then sweep k+1 on its own nodes from shared memory.
// Only the sweep-(k+1) values are written, into the other buffer, so no
// block ever reads a value another block overwrites in the same pass.
// Activity: a block is swept for colour j in pass m if colour j changed (by
// more than act_eps) in pass m-1 within its neighbourhood -- 3x3 blocks in
// 2D, and +-2 planes along internal axis 0 in 3D (blocks are one plane
// thick there, and a change reaches two planes in one pass).  Per-colour
// stopping is decided per sweep exactly as in the one-sweep kernel (max
// change over the swept nodes of each of the two sweeps); a colour that
// stops after the first sweep of a pass gets that sweep recomputed densely
// from the pass's input buffer at the end.
template <int D>
struct T2Shape {
  using B = Blk<D>;
  static constexpr int PL = (D == 2) ? 1 : 5;         // axis-0 planes in the tile (3D)
  static constexpr int RB = B::BY + 4;                // rows per plane
  static constexpr int W = B::BX + 4;                 // columns
  static constexpr int C = W + (W % 2 == 0);          // row pitch (odd: banks)
  static constexpr int N = PL * RB * C;
  static constexpr int RPL = (D == 2) ? 1 : 3;        // ring planes
  static constexpr int RRB = B::BY + 2;               // ring rows per plane
  static constexpr int RW = B::BX + 2;                // ring columns
  static constexpr int RN = RPL * RRB * RW;
  static constexpr int NNB = (D == 2) ? 9 : 45;       // neighbour blocks marked
};

template <int D>
struct T2Warp {  // per-warp shared memory
  double tile[T2Shape<D>::N];
  double ring[T2Shape<D>::RN];
  int rent[T2Shape<D>::RN];  // stencil entry of each ring node (-1: holds its value)
};

// neighbour nid of block t for the two-sweep transport (-1 outside)
template <int D>
__device__ inline int t2_neighbour(const TileGrid& tg, const phj_grid& g, int t, int nid) {
  if (D == 2) return neighbour_block<D>(tg, g, t, nid);
  const int* n = tg.n;
  int b[3];
  decode_block<D>(tg, t, b);
  int a = b[0] + nid / 9 - 2, c = b[1] + (nid / 3) % 3 - 1, e = b[2] + nid % 3 - 1;
  if (g.periodic[0]) a = ((a % n[0]) + n[0]) % n[0];
  if (a < 0 || a >= n[0] || c < 0 || c >= n[1] || e < 0 || e >= n[2]) return -1;
  return (a * n[1] + c) * n[2] + e;
}

// interior index along internal axis 0 -> ext index, wrapped on a periodic
// axis and clamped otherwise (clamped values only feed non-movers)
__device__ __forceinline__ int t2_axis0_ext(const phj_grid& g, int q) {
  const int n0 = (int)g.shape[0];
  if (g.periodic[0]) q = ((q % n0) + n0) % n0;
  else q = max(-1, min(q, n0));
  return q + 1;
}

template <int D>
__global__ void __launch_bounds__(kThreads, PHJ_TRANSPORT_CTAS)
    transport_kernel2(const __grid_constant__ TransportParams p) {
  using B = Blk<D>;
  using S = T2Shape<D>;
  constexpr int NC = 1 << D;
  constexpr int NB = B::NB;
  extern __shared__ __align__(16) unsigned char smem[];
  cg::grid_group grid = cg::this_grid();
  const int nent = p.n_classes * p.nc;
  const int R = p.R;
  // weights corner-major with an odd pitch (as in transport_kernel)
  const int wpitch = nent | 1;
  double* s_w = (double*)smem;                                                   // [NC][wpitch]
  unsigned long long* s_max = (unsigned long long*)(s_w + (int64_t)wpitch * NC);  // [2][R]
  int* s_done = (int*)(s_max + 2 * R);                      // [R] sweeps done (0x7fffffff running)
  signed char* s_oct = (signed char*)(s_done + R);          // [nent]
  T2Warp<D>* wsm =
      (T2Warp<D>*)(smem + align_up((int64_t)wpitch * NC * 8 + 16 * R + 4 * R + nent, 16)) +
      (threadIdx.x >> 5);
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
  const int ly = lane / B::LX, lx = lane % B::LX;
  const int64_t M0 = g.shape[0];
  const bool per0 = g.periodic[0] != 0;
  const int64_t ghost_shift = M0 * g.strides[0];
  // corner offsets (bit ax = +1 along axis ax) in tile and ring coordinates
  int toff[NC], roff[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    int t = 0, r = 0;
    if (D == 2) {
      t = ((k & 1) ? S::C : 0) + ((k >> 1) & 1);
      r = ((k & 1) ? S::RW : 0) + ((k >> 1) & 1);
    } else {
      t = ((k & 1) ? S::RB * S::C : 0) + (((k >> 1) & 1) ? S::C : 0) + ((k >> 2) & 1);
      r = ((k & 1) ? S::RRB * S::RW : 0) + (((k >> 1) & 1) ? S::RW : 0) + ((k >> 2) & 1);
    }
    toff[k] = t;
    roff[k] = r;
  }
  unsigned long long upd = 0;
  int m = 0, buf = 0;
  const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * kWarps;
  int ticket = 0;
  if (lane == 0) ticket = atomicAdd(&p.ws.take[0], 1);
  for (;;) {
    const double* pin = (const double*)p.phi[buf];
    double* pout = (double*)p.phi[buf ^ 1];
    const int cnt = ld_cg(&p.ws.counts[m]);
    const int* list = p.ws.list[m & 1];
    int* cur_flags = p.ws.flags[m & 1];
    unsigned long long* cur_mask = p.ws.cmask[m & 1];
    unsigned long long* nxt_mask = p.ws.cmask[(m + 1) & 1];
    int* nxt_list = p.ws.list[(m + 1) & 1];
    int* nxt_cnt = &p.ws.counts[m + 1];
    int* take = &p.ws.take[m];
    for (int i = threadIdx.x; i < 2 * R; i += blockDim.x) s_max[i] = 0ull;
    if (blockIdx.x == 0) {
      unsigned long long* z0 = sweep_max_slots(p.ws, 2 * m + 2);
      unsigned long long* z1 = sweep_max_slots(p.ws, 2 * m + 3);
      for (int i = threadIdx.x; i < R; i += blockDim.x) {
        z0[i * kMaxPad] = 0ull;
        z1[i * kMaxPad] = 0ull;
      }
    }
    __syncthreads();
    int item = gwarp;
    while (item < cnt) {
      const int blk = __ldcg(&list[item]);
      const int nxt = nwarps + __shfl_sync(FULL, ticket, 0);
      if (lane == 0 && nxt < cnt) ticket = atomicAdd(take, 1);
      unsigned long long cm = 0ull;
      if (lane == 0) {
        cm = __ldcg(&cur_mask[blk]);
        cur_mask[blk] = 0ull;
        cur_flags[blk] = 0;
      }
      cm = __shfl_sync(FULL, cm, 0);
      int bc[3];
      decode_block<D>(p.tg, blk, bc);
      // block origin: interior coordinates of its first node
      const int o0 = (D == 2) ? bc[0] * B::BY : bc[0];
      const int o1 = (D == 2) ? bc[1] * B::BX : bc[1] * B::BY;
      const int o2 = (D == 2) ? 0 : bc[2] * B::BX;
      // ring entries (stencil entry of each ring node's feedback, -1 = holds)
      for (int q = lane; q < S::RN; q += 32) {
        int i0, i1, i2 = 0;
        if (D == 2) {
          i0 = o0 - 1 + q / S::RW;
          i1 = o1 - 1 + q % S::RW;
        } else {
          const int pl = q / (S::RRB * S::RW), rem = q - pl * S::RRB * S::RW;
          i0 = o0 - 1 + pl;
          i1 = o1 - 1 + rem / S::RW;
          i2 = o2 - 1 + rem % S::RW;
        }
        if (per0) i0 = ((i0 % (int)M0) + (int)M0) % (int)M0;
        int e = -1;
        const bool inside = i0 >= 0 && i0 < M0 && i1 >= 0 && i1 < g.shape[1] &&
                            (D == 2 || (i2 >= 0 && i2 < g.shape[2]));
        if (inside) {
          const int64_t sidx = (D == 2) ? (int64_t)i0 * g.shape[1] + i1
                                        : ((int64_t)i0 * g.shape[1] + i1) * g.shape[2] + i2;
          e = __ldg(&p.ent[sidx]);
        }
        wsm->rent[q] = e;
      }
      __syncwarp();
      // own nodes: ring position and interior validity
      int rpos[NB];
      bool own_in[NB];
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        const int rr = ly + 1, rc = lx * NB + r + 1;
        rpos[r] = (D == 2) ? rr * S::RW + rc : (1 * S::RRB + rr) * S::RW + rc;
        const int i1 = (D == 2) ? o0 + ly : o1 + ly;
        const int ilast = (D == 2) ? o1 + lx * NB + r : o2 + lx * NB + r;
        own_in[r] = (D == 2) ? (i1 < M0 && ilast < g.shape[1])
                             : (i1 < g.shape[1] && ilast < g.shape[2]);
        if (own_in[r] && wsm->rent[rpos[r]] >= 0) upd += 2;  // two sweeps
      }
      unsigned long long changed = 0ull;
      const bool masked = R <= 64;
      unsigned long long todo = masked ? cm : 0ull;
      int jnext = 0;
      for (;;) {
        int j;
        if (masked) {
          if (!todo) break;
          j = __ffsll((long long)todo) - 1;
          todo &= todo - 1;
        } else {
          if (jnext >= R) break;
          j = jnext++;
        }
        if (s_done[j] != 0x7fffffff) continue;  // stopped colours are never touched again
        const double* pj = pin + (int64_t)j * p.plane;
        double* qj = pout + (int64_t)j * p.plane;
        // stage the 2-ring tile of colour j (rows wrapped / clamped on axis 0)
        for (int rrow = lane; rrow < S::PL * S::RB; rrow += 32) {
          int64_t rbase;
          if (D == 2) {
            const int e0 = t2_axis0_ext(g, o0 - 2 + rrow);
            rbase = (int64_t)e0 * g.strides[0];
          } else {
            const int pl = rrow / S::RB, rr = rrow - pl * S::RB;
            const int e0 = t2_axis0_ext(g, o0 - 2 + pl);
            const int e1 = max(0, min(o1 - 1 + rr, (int)g.ext[1] - 1));
            rbase = (int64_t)e0 * g.strides[0] + (int64_t)e1 * g.strides[1];
          }
          const int cmax = (int)g.ext[D - 1] - 1;
          const int c0 = (D == 2) ? o1 - 1 : o2 - 1;
#pragma unroll
          for (int c = 0; c < S::W; ++c)
            cp_async<8>(&wsm->tile[rrow * S::C + c], pj + rbase + max(0, min(c0 + c, cmax)));
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        // sweep k on the block + 1-node ring
        for (int q = lane; q < S::RN; q += 32) {
          int tp;
          if (D == 2) tp = (q / S::RW + 1) * S::C + q % S::RW + 1;
          else {
            const int pl = q / (S::RRB * S::RW), rem = q - pl * S::RRB * S::RW;
            tp = ((pl + 1) * S::RB + rem / S::RW + 1) * S::C + rem % S::RW + 1;
          }
          const int e = wsm->rent[q];
          double v = wsm->tile[tp];
          if (e >= 0) {
            const int oc = s_oct[e];
            int lo = tp;  // lower corner of the foot cell
            if (D == 2) {
              if (!(oc & 1)) lo -= S::C;
              if (!((oc >> 1) & 1)) lo -= 1;
            } else {
              if (!(oc & 1)) lo -= S::RB * S::C;
              if (!((oc >> 1) & 1)) lo -= S::C;
              if (!((oc >> 2) & 1)) lo -= 1;
            }
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < NC; ++k) acc = fma(s_w[k * wpitch + e], wsm->tile[lo + toff[k]], acc);
            v = acc;
          }
          wsm->ring[q] = v;
        }
        __syncwarp();
        // sweep k + 1 on the own nodes
        double l0 = 0.0, l1 = 0.0;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          if (!own_in[r]) continue;
          const int q = rpos[r];
          const int e = wsm->rent[q];
          if (e < 0) continue;
          int tp;
          if (D == 2) tp = (q / S::RW + 1) * S::C + q % S::RW + 1;
          else {
            const int pl = q / (S::RRB * S::RW), rem = q - pl * S::RRB * S::RW;
            tp = ((pl + 1) * S::RB + rem / S::RW + 1) * S::C + rem % S::RW + 1;
          }
          const double vk = wsm->ring[q];
          l0 = fmax(l0, fabs(wsm->tile[tp] - vk));
          const int oc = s_oct[e];
          int lo = q;
          if (D == 2) {
            if (!(oc & 1)) lo -= S::RW;
            if (!((oc >> 1) & 1)) lo -= 1;
          } else {
            if (!(oc & 1)) lo -= S::RRB * S::RW;
            if (!((oc >> 1) & 1)) lo -= S::RW;
            if (!((oc >> 2) & 1)) lo -= 1;
          }
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < NC; ++k) acc = fma(s_w[k * wpitch + e], wsm->ring[lo + roff[k]], acc);
          l1 = fmax(l1, fabs(vk - acc));
          int c[3];
          if (D == 2) {
            c[0] = o0 + ly;
            c[1] = o1 + lx * NB + r;
          } else {
            c[0] = o0;
            c[1] = o1 + ly;
            c[2] = o2 + lx * NB + r;
          }
          const int64_t f = ext_flat<D>(g, c);
          qj[f] = acc;
          if (per0) {
            if (c[0] == 0) qj[f + ghost_shift] = acc;
            else if (c[0] == M0 - 1) qj[f - ghost_shift] = acc;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          l0 = fmax(l0, __shfl_xor_sync(FULL, l0, off));
          l1 = fmax(l1, __shfl_xor_sync(FULL, l1, off));
        }
        if (lane == 0) {
          if (l0 > 0.0) atomicMax(&s_max[j], dbits(l0));
          if (l1 > 0.0) atomicMax(&s_max[R + j], dbits(l1));
        }
        if (fmax(l0, l1) > p.act_eps) changed |= (j < 64) ? (1ull << j) : ~0ull;
        __syncwarp();
      }
      // mark the neighbourhood for the next pass
      for (int base = 0; base < S::NNB; base += 32) {
        const int nid = base + lane;
        int want = 0, nt = -1;
        if (changed && nid < S::NNB) {
          nt = t2_neighbour<D>(p.tg, g, blk, nid);
          if (nt >= 0 && atomicOr(&nxt_mask[nt], changed) == 0ull) want = 1;
        }
        const unsigned bal = __ballot_sync(FULL, want);
        if (bal) {
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(nxt_cnt, __popc(bal));
          b0 = __shfl_sync(FULL, b0, 0);
          if (want) nxt_list[b0 + __popc(bal & ((1u << lane) - 1u))] = nt;
        }
      }
      item = nxt;
    }
    if (lane == 0 && 2 * m + 2 < p.max_sweeps) ticket = atomicAdd(&p.ws.take[m + 1], 1);
    __syncthreads();
    unsigned long long* g0 = sweep_max_slots(p.ws, 2 * m);
    unsigned long long* g1 = sweep_max_slots(p.ws, 2 * m + 1);
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      if (s_max[i]) atomicMax(&g0[i * kMaxPad], s_max[i]);
      if (s_max[R + i]) atomicMax(&g1[i * kMaxPad], s_max[R + i]);
    }
    grid.sync();
    ++m;
    buf ^= 1;
    int pending = 0;
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      if (s_done[i] == 0x7fffffff) {
        const unsigned long long b0 = ld_cg(&g0[i * kMaxPad]), b1 = ld_cg(&g1[i * kMaxPad]);
        if (blockIdx.x == 0) {
          p.maxch[(int64_t)(2 * m - 2) * R + i] = b0;
          if (2 * m - 1 < p.max_sweeps) p.maxch[(int64_t)(2 * m - 1) * R + i] = b1;
        }
        if (__longlong_as_double((long long)b0) <= p.tol) s_done[i] = 2 * m - 1;
        else if (__longlong_as_double((long long)b1) <= p.tol) s_done[i] = 2 * m;
        else pending = 1;
      }
    }
    const int any_pending = __syncthreads_or(pending);
    if (!any_pending || 2 * m >= p.max_sweeps) break;
  }
  // colours that stopped after the first sweep of their last pass: that sweep
  // again, densely over the movers, from the pass's input buffer into its
  // output buffer (which then holds every colour's result)
  grid.sync();
  const int64_t N = g.shape[0] * g.shape[1] * (D == 3 ? g.shape[2] : 1);
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < R; ++j) {
    const int d = s_done[j];
    if (d == 0x7fffffff || !(d & 1)) continue;
    const int mj = (d - 1) / 2;  // pass that held the stop
    const double* rj = (const double*)p.phi[mj & 1] + (int64_t)j * p.plane;
    double* wj = (double*)p.phi[(mj + 1) & 1] + (int64_t)j * p.plane;
    for (int64_t sidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; sidx < N; sidx += gstride) {
      const int e = __ldg(&p.ent[sidx]);
      if (e < 0) continue;
      int c[3];
      if (D == 2) {
        c[0] = (int)(sidx / g.shape[1]);
        c[1] = (int)(sidx % g.shape[1]);
        c[2] = 0;
      } else {
        c[2] = (int)(sidx % g.shape[2]);
        const int64_t r2 = sidx / g.shape[2];
        c[1] = (int)(r2 % g.shape[1]);
        c[0] = (int)(r2 / g.shape[1]);
      }
      const int64_t f = ext_flat<D>(g, c);
      const int oc = s_oct[e];
      int64_t lo = f;
#pragma unroll
      for (int ax = 0; ax < D; ++ax)
        if (!((oc >> ax) & 1)) lo -= g.strides[ax];
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        int64_t o = 0;
#pragma unroll
        for (int ax = 0; ax < D; ++ax)
          if ((k >> ax) & 1) o += g.strides[ax];
        acc = fma(__ldg(&p.weights[(int64_t)e * NC + k]), rj[lo + o], acc);
      }
      wj[f] = acc;
      if (per0) {
        if (c[0] == 0) wj[f + ghost_shift] = acc;
        else if (c[0] == M0 - 1) wj[f - ghost_shift] = acc;
      }
    }
  }
  grid.sync();
  // every colour's result into buffer 0 (the output buffer of its last pass)
  const int mfin = m;  // passes run
  for (int j = 0; j < R; ++j) {
    const int d = s_done[j];
    const int mj = (d == 0x7fffffff) ? mfin - 1 : (d - 1) / 2;
    if (((mj + 1) & 1) == 0) continue;
    const double* src = (const double*)p.phi[1] + (int64_t)j * p.plane;
    double* dst = (double*)p.phi[0] + (int64_t)j * p.plane;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < p.plane; f += gstride)
      dst[f] = src[f];
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < R; i += blockDim.x)
      p.color_sweeps[i] = (s_done[i] == 0x7fffffff) ? -(2 * mfin) : s_done[i];
    if (threadIdx.x == 0) {
      p.info[0] = 2 * mfin;
      p.info[1] = 0;
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
  // allowed controls (solver.extract_feedback(allowed=...)): per ext node a
  // row of allow_mask ([rows][allow_words] bitmask over stencil entries) and
  // allow_count (admissible allowed controls); NULL allow_row = all allowed
  const int32_t* allow_row;
  const unsigned long long* allow_mask;
  const int32_t* allow_count;
  int allow_words;
  // blocks [blk_begin, blk_end): a slab of block rows along internal axis 0
  // (ranks of a multi-GPU run split the stage by slabs)
  int blk_begin, blk_end;
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
  for (int blk = p.blk_begin + blockIdx.x * kWarps + (threadIdx.x >> 5); blk < p.blk_end;
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
    int cnt[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) cnt[r] = nadm;
    if (p.allow_row) {
      Allowed<NB> al;
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        const int row = comp[r] ? __ldg(&p.allow_row[f0 + r]) : -1;
#pragma unroll
        for (int w = 0; w < 2; ++w)
          al.w[r][w] = (row >= 0 && w < p.allow_words)
                           ? __ldg(&p.allow_mask[(int64_t)row * p.allow_words + w])
                           : ~0ull;
        if (row >= 0) cnt[r] = __ldg(&p.allow_count[row]);
      }
      EvalAll<D, T, NB, RULE, COST, true, 1, true>::run(nb, s, os, fm, ncoef, s_ctrl, mn, best,
                                                        bidx, NoHook(), &al);
    } else {
      EvalAll<D, T, NB, RULE, COST, true, 1>::run(nb, s, os, fm, ncoef, s_ctrl, mn, best, bidx,
                                                   NoHook());
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (!comp[r]) continue;
      ev += cnt[r];
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

extern "C" int32_t phj_unroll(int32_t dim) { return PHJ_UNROLL(dim); }

extern "C" int phj_block_dims(int32_t dim, int32_t* out) {
  if (!out || (dim != 2 && dim != 3)) {
    phj_set_error("phj_block_dims: dim must be 2 or 3");
    return PHJ_ERR_ARG;
  }
  if (dim == 2) {
    out[0] = Blk<2>::BY;
    out[1] = Blk<2>::BX;
    out[2] = 1;
  } else {
    out[0] = 1;
    out[1] = Blk<3>::BY;
    out[2] = Blk<3>::BX;
  }
  return PHJ_OK;
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

// Persistent non-cooperative launch (no grid barrier): all co-resident CTAs
// (at most kRingExtra warps: the async ring holds one waiting ticket per warp).
template <typename K>
static int persistent_blocks(K kernel, size_t smem, int* blocks) {
  PHJ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  PHJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem));
  if (occ < 1) {
    phj_set_error("kernel cannot be resident (smem %zu B)", smem);
    return PHJ_ERR_UNSUPPORTED;
  }
  int b = std::min(occ * phj_num_sms(), kRingExtra / kWarps);
  if (const char* cap = getenv("PHJ_MAX_BLOCKS")) b = std::min(b, atoi(cap));
  *blocks = b < 1 ? 1 : b;
  return PHJ_OK;
}

// ring cells for an asynchronous launch of `blocks` CTAs, then the launch
template <typename K>
static int async_launch(K kernel, size_t smem, void** args, const Workspace& ws, int total,
                        cudaStream_t stream) {
  int blocks = 0;
  if (int rc = persistent_blocks(kernel, smem, &blocks)) return rc;
  const unsigned cap = (unsigned)total + (unsigned)(blocks * kWarps);
  async_ring_init<<<std::min(1024, (int)((cap + 255) / 256)), 256, 0, stream>>>(
      ws.ring, cap, ws.list[0], ws.counts);
  phj_count_launch(1);
  PHJ_CUDA(cudaLaunchKernel((void*)kernel, dim3(blocks), dim3(kThreads), args, smem, stream));
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
  p.ctrl = a->st.ctrl;
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
  p.pcount = a->patch_counts;
  p.info = a->info;
  p.prune = (a->options & PHJ_SOLVE_NO_PRUNE) ? 0 : 1;
  p.act = a->act_tol;
  p.inner = a->inner_sweeps < 1 ? 1 : a->inner_sweeps;
  p.ao3_fb = a->ao3_fb;
  p.ao3_mask = a->ao3_mask;
  p.ao3_count = a->ao3_count;
  p.ao3_words = a->ao3_words;
  const bool async = (a->options & PHJ_SOLVE_ASYNC) != 0;
  const bool banded = a->band_off && a->band_list && a->n_band > 0;
  p.band_list = banded ? a->band_list : nullptr;
  p.band_off = banded ? a->band_off : nullptr;
  p.n_band = banded ? a->n_band : 0;
  p.band_only = 0;
  if (banded && a->n_band >= a->max_sweeps) {
    phj_set_error("phj_solve: the band schedule needs n_band < max_sweeps");
    return PHJ_ERR_ARG;
  }
  const int64_t ws_bytes = workspace_bytes<D>(a->grid, a->max_sweeps);
  PHJ_CUDA(cudaMemsetAsync(a->workspace, 0, ws_bytes, stream));
  PHJ_CUDA(cudaMemsetAsync(a->maxch_hist, 0, sizeof(double) * (size_t)a->max_sweeps * a->n_patches,
                           stream));
  PHJ_CUDA(cudaMemsetAsync(a->evals, 0, 3 * sizeof(unsigned long long), stream));
  if (a->patch_counts)
    PHJ_CUDA(cudaMemsetAsync(a->patch_counts, 0, 3 * sizeof(unsigned long long) * a->n_patches,
                             stream));
  PHJ_CUDA(cudaMemsetAsync(a->info, 0, 4 * sizeof(int32_t), stream));
  size_t smem = (size_t)align_up(solve_stencil_bytes<D, T>(p.n_classes, p.nc) +
                                     (int64_t)((p.R + 1) / 2 * 2) * 4 +
                                     (int64_t)std::min(p.R, kSmemPatchReduce) * 8 * 4,
                                 16) +
                (size_t)solve_tile_bytes<D, T>();
  if (banded && async) {
    // the value-ordered pass alone (cooperative Jacobi sweeps over the band
    // schedule), then the asynchronous relaxation from its result: both
    // buffers hold the pass's values (every block ends with a copy visit)
    SolveParams pb = p;
    pb.band_only = 1;
    // block-local relaxations per visit in the pass (0: the schedule's)
    if (a->band_inner > 0) pb.inner = a->band_inner;
    void* bargs[] = {(void*)&pb};
    int rc = (D == 3 && p.n_classes > 1)
                 ? coop_launch(solve_kernel<D, T, RULE, COST, D == 3>,
                               (p.tg.total + kWarps - 1) / kWarps, smem, bargs, stream, nullptr)
                 : coop_launch(solve_kernel<D, T, RULE, COST, false>,
                               (p.tg.total + kWarps - 1) / kWarps, smem, bargs, stream, nullptr);
    if (rc) return rc;
    PHJ_CUDA(cudaMemsetAsync(a->workspace, 0, ws_bytes, stream));
    p.n_band = 0;
    p.band_list = nullptr;
    p.band_off = nullptr;
  }
  // initial blocks: those that can move from the start field (exact: from
  // the unreached start a block with no reached value within its 3^D
  // neighbourhood reproduces itself)
  if (!(banded && !async)) {
    build_list_kernel<D><<<(p.tg.total + kWarps - 1) / kWarps, kThreads, 0, stream>>>(
      p.g, p.tg, p.lab, p.mine, p.ws.flags[0], p.ws.list[0], p.ws.counts, 0,
      nullptr, nullptr,
      nullptr, 0ull, a->v0, sizeof(T) == 4, RULE == PHJ_RULE_KRUZKOV ? 1.0 : 1.0e9,
      async ? &p.ws.take[5] : nullptr);
    phj_count_launch(1);
  }
  PHJ_CUDA(cudaGetLastError());
  if (async) {
    const long long want = (long long)a->max_sweeps * (long long)p.tg.total;
    unsigned int budget = (unsigned int)std::min(want, (long long)0x7fffffff);
    void* aargs[] = {(void*)&p, (void*)&budget};
    int rc = (D == 3 && p.n_classes > 1)
                 ? async_launch(solve_async_kernel<D, T, RULE, COST, D == 3>, smem, aargs, p.ws,
                                p.tg.total, stream)
                 : async_launch(solve_async_kernel<D, T, RULE, COST, false>, smem, aargs, p.ws,
                                p.tg.total, stream);
    if (rc) return rc;
    async_finish_kernel<<<1, 256, 0, stream>>>(p.ws, p.R, p.mine, p.patch_sweeps, p.info);
    phj_count_launch(1);
    PHJ_CUDA(cudaGetLastError());
    return PHJ_OK;
  }
  void* args[] = {(void*)&p};
  int launched = 0;
  int rc = (D == 3 && p.n_classes > 1)
               ? coop_launch(solve_kernel<D, T, RULE, COST, D == 3>,
                             (p.tg.total + kWarps - 1) / kWarps, smem, args, stream, &launched)
               : coop_launch(solve_kernel<D, T, RULE, COST, false>,
                             (p.tg.total + kWarps - 1) / kWarps, smem, args, stream, &launched);
  if (rc) return rc;
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}

#ifdef PHJ_TIMING
// diagnostic: summed per-warp cycles of the solve kernel phases since the last call
extern "C" int phj_dbg_visit_kinds(unsigned long long* out) {
  PHJ_CUDA(cudaMemcpyFromSymbol(out, g_visit_kind, 4 * sizeof(unsigned long long)));
  unsigned long long z[4] = {0, 0, 0, 0};
  PHJ_CUDA(cudaMemcpyToSymbol(g_visit_kind, z, sizeof(z)));
  return PHJ_OK;
}
extern "C" int phj_dbg_timeline(unsigned int* bins) {
  PHJ_CUDA(cudaMemcpyFromSymbol(bins, g_visit_bins, 4096 * sizeof(unsigned int)));
  static unsigned int zb[4096];
  unsigned long long z = 0ull;
  PHJ_CUDA(cudaMemcpyToSymbol(g_visit_bins, zb, sizeof(zb)));
  PHJ_CUDA(cudaMemcpyToSymbol(g_t0, &z, sizeof(z)));
  return PHJ_OK;
}
extern "C" int phj_dbg_phase_cycles(unsigned long long* out) {
  PHJ_CUDA(cudaMemcpyFromSymbol(out, g_phase_cycles, 12 * sizeof(unsigned long long)));
  unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  PHJ_CUDA(cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)));
  return PHJ_OK;
}
#endif

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
  if (!(a->act_tol >= 0.0)) {
    phj_set_error("phj_solve: act_tol must be >= 0");
    return PHJ_ERR_ARG;
  }
  if (a->ao3_fb && (!a->ao3_mask || !a->ao3_count || a->ao3_words < 1 || a->ao3_words > 2 ||
                    a->st.n_classes != 1)) {
    phj_set_error("phj_solve: AO3 needs masks/counts, 1..2 mask words (<= 128 stencil entries) "
                  "and a single-class stencil");
    return PHJ_ERR_ARG;
  }
  if (((uintptr_t)a->lab & 3) != 0) {
    phj_set_error("phj_solve: lab must be 4-byte aligned (staged as 32-bit words)");
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
  const bool async = (a->options & PHJ_TRANSPORT_ASYNC) != 0;
  const bool banded = a->band_off && a->band_list && a->n_band > 0 && !async;
  p.band_list = banded ? a->band_list : nullptr;
  p.band_off = banded ? a->band_off : nullptr;
  p.n_band = banded ? a->n_band : 0;
  p.chunk = (a->options & PHJ_TRANSPORT_PAIRS) ? 2 : 1;
  if (banded && (a->n_band >= a->max_sweeps || p.R > 64)) {
    phj_set_error("phj_transport: the banded pass needs n_band < max_sweeps and <= 64 colours");
    return PHJ_ERR_ARG;
  }
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
  const bool seeded = a->seed_flat && a->n_seed > 0 && p.R <= 64;
  if (seeded) {
    const int nb = (int)std::min<int64_t>((a->n_seed + 255) / 256, 4 * phj_num_sms());
    // banded: the seeds start the sticky masks (see transport_kernel)
    transport_seed_kernel<D><<<std::max(nb, 1), 256, 0, stream>>>(
        p.g, p.tg, a->seed_flat, a->seed_col, a->n_seed, p.ws.cmask[banded ? (p.n_band & 1) : 0]);
    phj_count_launch(1);
  }
  if (banded && !seeded) {
    // every mover block starts with every colour
    const unsigned long long all = p.R >= 64 ? ~0ull : ((1ull << p.R) - 1ull);
    PHJ_CUDA(cudaMemsetAsync(p.ws.cmask[p.n_band & 1], 0, 8 * (size_t)p.tg.total, stream));
    std::vector<unsigned long long> h((size_t)p.tg.total, all);
    PHJ_CUDA(cudaMemcpyAsync(p.ws.cmask[p.n_band & 1], h.data(), 8 * (size_t)p.tg.total,
                             cudaMemcpyHostToDevice, stream));
    PHJ_CUDA(cudaStreamSynchronize(stream));
  }
  if (!banded) {
    build_list_kernel<D><<<(p.tg.total + kWarps - 1) / kWarps, kThreads, 0, stream>>>(
      p.g, p.tg, nullptr, nullptr, p.ws.flags[0], p.ws.list[0], p.ws.counts,
      1, p.fb, p.kind,
      p.ws.cmask[0], p.R >= 64 ? ~0ull : ((1ull << p.R) - 1ull), nullptr, 0, 0.0,
      async ? &p.ws.take[5] : nullptr, seeded ? 1 : 0);
    phj_count_launch(1);
  }
  PHJ_CUDA(cudaGetLastError());
  const int nent = p.n_classes * p.nc;
  if (async) {
    int inner = a->inner_sweeps < 1 ? 1 : a->inner_sweeps;
    const long long want = (long long)a->max_sweeps * (long long)p.tg.total;
    unsigned int budget = (unsigned int)std::min(want, (long long)0x7fffffff);
    void* aargs[] = {(void*)&p, (void*)&inner, (void*)&budget};
    const size_t smem = (size_t)(nent | 1) * (1 << D) * 8 +
                        (size_t)kWarps * TTile<D>::TC * TileShape<D>::N * 8 + (size_t)nent + 16;
    int rc = a->phi_dtype == PHJ_F32
                 ? async_launch(transport_async_kernel<D, float>, smem, aargs, p.ws, p.tg.total,
                                stream)
                 : async_launch(transport_async_kernel<D, double>, smem, aargs, p.ws, p.tg.total,
                                stream);
    if (rc) return rc;
    async_finish_kernel<<<1, 256, 0, stream>>>(p.ws, p.R, nullptr, p.color_sweeps, p.info);
    phj_count_launch(1);
    PHJ_CUDA(cudaGetLastError());
    return PHJ_OK;
  }
  void* args[] = {(void*)&p};
  // two sweeps per barrier pay in 2D only (3D: the 2-ring halo is 5 planes
  // deep and the activity must reach +-2 planes -- measured 2x slower)
  static const bool one_sweep = getenv("PHJ_TRANSPORT_T1") && atoi(getenv("PHJ_TRANSPORT_T1"));
  if (one_sweep || D == 3 || a->phi_dtype == PHJ_F32 || banded) {  // fp32 phi / banded: one-sweep kernel
    size_t smem = (size_t)(nent | 1) * (1 << D) * 8 + (size_t)p.R * 12 + (size_t)nent + 16;
    if (a->phi_dtype == PHJ_F32)
      return coop_launch(transport_kernel<D, float>, (p.tg.total + kWarps - 1) / kWarps, smem,
                         args, stream, nullptr);
    return coop_launch(transport_kernel<D, double>, (p.tg.total + kWarps - 1) / kWarps, smem, args,
                       stream, nullptr);
  }
  size_t smem = (size_t)align_up((int64_t)(nent | 1) * (1 << D) * 8 + 16 * (int64_t)p.R +
                                     4 * (int64_t)p.R + nent,
                                 16) +
                (size_t)kWarps * sizeof(T2Warp<D>);
  return coop_launch(transport_kernel2<D>, (p.tg.total + kWarps - 1) / kWarps, smem, args, stream,
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
  if (a->phi_dtype != PHJ_F64 && a->phi_dtype != PHJ_F32) {
    phj_set_error("phj_transport: phi_dtype must be PHJ_F64 or PHJ_F32");
    return PHJ_ERR_ARG;
  }
  if (a->n_colors < 1 || a->n_colors > kMaxColors || !a->maxch_hist || !a->color_sweeps) {
    phj_set_error("phj_transport: n_colors must be in [1, %d]", kMaxColors);
    return PHJ_ERR_ARG;
  }
  return a->grid.dim == 2 ? transport_impl<2>(a) : transport_impl<3>(a);
}

template <int D, typename T, int RULE, int COST>
static int feedback_impl(const phj_grid* g, const phj_stencil* st, const void* v,
                         const int8_t* kind, const uint32_t* fmask, const void* coef,
                         double coef0, double unreach, const int32_t* allow_row,
                         const unsigned long long* allow_mask, const int32_t* allow_count,
                         int32_t allow_words, int32_t* out, unsigned long long* evals,
                         int32_t slab_begin, int32_t slab_end, cudaStream_t stream) {
  FeedbackParams p;
  p.g = *g;
  p.tg = make_tile_grid<D>(*g);
  {
    // slabs count block rows along internal axis 0 (slab_end < 0: all)
    const int per_row = p.tg.total / p.tg.n[0];
    const int r0 = slab_end < 0 ? 0 : std::max(0, std::min(slab_begin, p.tg.n[0]));
    const int r1 = slab_end < 0 ? p.tg.n[0] : std::max(r0, std::min(slab_end, p.tg.n[0]));
    p.blk_begin = r0 * per_row;
    p.blk_end = r1 * per_row;
  }
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
  p.allow_row = allow_row;
  p.allow_mask = allow_mask;
  p.allow_count = allow_count;
  p.allow_words = allow_words;
  size_t smem = (size_t)StencilSmem<D, T>::bytes(p.n_classes, p.nc) +
                (size_t)p.n_classes * p.nc * 4 + 16;
  auto k = feedback_kernel<D, T, RULE, COST>;
  PHJ_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (p.blk_end <= p.blk_begin) return PHJ_OK;
  int blocks = std::min((p.blk_end - p.blk_begin + kWarps - 1) / kWarps, 8 * phj_num_sms());
  k<<<blocks, kThreads, smem, stream>>>(p);
  phj_count_launch(1);
  PHJ_CUDA(cudaGetLastError());
  return PHJ_OK;
}

extern "C" int phj_feedback_slab(const phj_grid* g, const phj_stencil* st, int32_t dtype,
                                    int32_t rule, const void* v, const int8_t* kind,
                                    const uint32_t* fmask, const void* coef, double coef0,
                                    double unreach, const int32_t* allow_row,
                                    const unsigned long long* allow_mask,
                                    const int32_t* allow_count, int32_t allow_words,
                                    int32_t* out, unsigned long long* evals, int32_t slab_begin,
                                    int32_t slab_end, void* stream) {
  if (!g || !st || !v || !kind || !fmask || !out) {
    phj_set_error("phj_feedback: missing argument");
    return PHJ_ERR_ARG;
  }
  if (allow_row && (!allow_mask || !allow_count || allow_words < 1 || allow_words > 2 ||
                    st->n_classes != 1)) {
    phj_set_error("phj_feedback: allowed masks need counts, 1..2 words (<= 128 stencil "
                  "entries) and a single-class stencil");
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
    return feedback_impl<DD, TT, RR, CC>(g, st, v, kind, fmask, coef, coef0, unreach,      \
                                         allow_row, allow_mask, allow_count, allow_words, out, \
                                         evals, slab_begin, slab_end, s);
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

extern "C" int phj_feedback_allowed(const phj_grid* g, const phj_stencil* st, int32_t dtype,
                                    int32_t rule, const void* v, const int8_t* kind,
                                    const uint32_t* fmask, const void* coef, double coef0,
                                    double unreach, const int32_t* allow_row,
                                    const unsigned long long* allow_mask,
                                    const int32_t* allow_count, int32_t allow_words,
                                    int32_t* out, unsigned long long* evals, void* stream) {
  return phj_feedback_slab(g, st, dtype, rule, v, kind, fmask, coef, coef0, unreach, allow_row,
                           allow_mask, allow_count, allow_words, out, evals, 0, -1, stream);
}

extern "C" int phj_feedback(const phj_grid* g, const phj_stencil* st, int32_t dtype, int32_t rule,
                            const void* v, const int8_t* kind, const uint32_t* fmask,
                            const void* coef, double coef0, double unreach, int32_t* out,
                            unsigned long long* evals, void* stream) {
  return phj_feedback_allowed(g, st, dtype, rule, v, kind, fmask, coef, coef0, unreach, nullptr,
                              nullptr, nullptr, 0, out, evals, stream);
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
