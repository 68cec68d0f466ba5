/*
 * phj_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the reference patchyhjb hot loops, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 * The product path (paper_1109_3577_b200/) never links or calls this file.
 *
 * Followed line by line (all paths under /root/reference/pkg/src/patchyhjb/):
 *   og_point/og_foot  : solver.py:170-188 (F, |F|, h=k/|F|, foot=X+h F, cost)
 *                       grid.py:123-152 (locate_many: t, floor, clip, snap)
 *   og_sweep          : _kernels.py:18-106 (sweep_batch), GS in place or Jacobi
 *   og_feedback       : _kernels.py:109-167 (feedback_batch)
 *   og_transport      : _kernels.py:170-204 (transport_batch)
 *   og_lift           : grid.py:242-261 (interpolate_many, saturating)
 *
 * Extensions beyond the reference (documented in DESIGN.md):
 *   - rule OG_RULE_KRUZKOV: candidate value beta*I + (1-beta), beta=exp(-cost)
 *     (BASELINE.json north_star); OG_RULE_REF is the reference update I+cost.
 *   - Jacobi mode (read u_in, write u_out) next to the reference GS mode.
 *   - periodic axes (corner indices wrap), Dubins dynamics f=(cos th, sin th, a).
 *
 * Arithmetic mirrors numba's IEEE code: compile with -ffp-contract=off and
 * without -ffast-math so a*b+c is never fused (see oracle/Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OG_BIG 1.0e300
#define OG_SNAP 1.0e-12

enum { OG_DYN_TABLE = 0, OG_DYN_SCALED = 1, OG_DYN_DUBINS = 2 };
enum { OG_RULE_REF = 0, OG_RULE_KRUZKOV = 1 };

typedef struct {
  int32_t dim;
  int32_t periodic[3];
  int64_t shape[3];
  int64_t ext[3];
  int64_t strides[3];
  double lo[3];
  double spacing[3];
  double ext_lo[3];
  double k;
} og_grid;

typedef struct {
  int32_t kind;
  int32_t nc;
  int32_t m;
  int32_t pad;
  const double* controls; /* [nc*m] */
  const double* speed;    /* SCALED: per interior serial */
  const double* F;        /* TABLE: [N*nc*dim] velocities */
  const double* cost_l;   /* optional running cost [N*nc] (ref rule only) */
  double eps_speed;
} og_dyn;

static void og_unravel(const og_grid* g, int64_t s, int64_t idx[3]) {
  for (int ax = g->dim - 1; ax >= 0; --ax) {
    idx[ax] = s % g->shape[ax];
    s /= g->shape[ax];
  }
}

/* flat extended index of interior serial s (grid.py:99-106) */
static int64_t og_iflat(const og_grid* g, int64_t s) {
  int64_t idx[3];
  og_unravel(g, s, idx);
  int64_t f = 0;
  for (int ax = 0; ax < g->dim; ++ax) f += (idx[ax] + 1) * g->strides[ax];
  return f;
}

/* node coordinates: lo + i*spacing (grid.py:89-97) */
static void og_point(const og_grid* g, int64_t s, double X[3]) {
  int64_t idx[3];
  og_unravel(g, s, idx);
  for (int ax = 0; ax < g->dim; ++ax) X[ax] = g->lo[ax] + (double)idx[ax] * g->spacing[ax];
}

/* locate_many for one point (grid.py:138-152): ext-cell + snapped locals */
static void og_locate(const og_grid* g, const double P[3], int64_t cell[3], double loc[3]) {
  for (int ax = 0; ax < g->dim; ++ax) {
    double t = (P[ax] - g->ext_lo[ax]) / g->spacing[ax];
    double fl = floor(t);
    int64_t c = (int64_t)fl;
    int64_t nmax = g->ext[ax] - 1;
    if (c < 0) c = 0;
    if (c > nmax - 1) c = nmax - 1;
    double l = t - (double)c;
    if (l < OG_SNAP) l = 0.0;
    if (l > 1.0 - OG_SNAP) l = 1.0;
    cell[ax] = c;
    loc[ax] = l;
  }
}

/* Candidate foot of (serial s at point X, control c); returns 0 when
 * inadmissible (|f| < eps_speed, solver.py:176-179).  solver.py:175-188.
 * X = og_point(s), hoisted out of the control loops by the callers. */
static int og_foot_at(const og_grid* g, const og_dyn* dy, int64_t s, const double X[3], int c,
                      int64_t cell[3], double loc[3], double* cost) {
  const int d = g->dim;
  double F[3] = {0.0, 0.0, 0.0};
  if (dy->kind == OG_DYN_SCALED) {
    double sp = dy->speed[s];
    for (int ax = 0; ax < d; ++ax) F[ax] = sp * dy->controls[c * dy->m + ax];
  } else if (dy->kind == OG_DYN_TABLE) {
    const double* f = dy->F + ((int64_t)s * dy->nc + c) * d;
    for (int ax = 0; ax < d; ++ax) F[ax] = f[ax];
  } else { /* DUBINS: (cos th, sin th, a), th = last coordinate */
    F[0] = cos(X[2]);
    F[1] = sin(X[2]);
    F[2] = dy->controls[c * dy->m];
  }
  double ss = F[0] * F[0];
  for (int ax = 1; ax < d; ++ax) ss = ss + F[ax] * F[ax];
  double speed = sqrt(ss);
  if (!(speed >= dy->eps_speed)) return 0;
  double h = g->k / speed;
  double P[3];
  for (int ax = 0; ax < d; ++ax) P[ax] = X[ax] + h * F[ax];
  og_locate(g, P, cell, loc);
  *cost = dy->cost_l ? h * dy->cost_l[(int64_t)s * dy->nc + c] : h;
  return 1;
}

static int og_foot(const og_grid* g, const og_dyn* dy, int64_t s, int c,
                   int64_t cell[3], double loc[3], double* cost) {
  double X[3];
  og_point(g, s, X);
  return og_foot_at(g, dy, s, X, c, cell, loc, cost);
}

/* flat index of corner `corner` (bit ax = upper face on axis ax) of an ext
 * cell; periodic axes wrap ghost indices onto the opposite interior layer. */
static int64_t og_corner(const og_grid* g, const int64_t cell[3], int corner) {
  int64_t f = 0;
  for (int ax = 0; ax < g->dim; ++ax) {
    int64_t e = cell[ax] + ((corner >> ax) & 1);
    if (g->periodic[ax]) {
      int64_t M = g->shape[ax];
      if (e == 0) e = M;
      else if (e == M + 1) e = 1;
    }
    f += e * g->strides[ax];
  }
  return f;
}

static double og_weight(int dim, const double loc[3], int corner) {
  double w = 1.0;
  for (int ax = 0; ax < dim; ++ax) {
    double t = loc[ax];
    if ((corner >> ax) & 1) w *= t;
    else w *= 1.0 - t;
  }
  return w;
}

/* Weights (og_weight's products, same order: 1.0 * axis 0 * axis 1 ...)
 * and flat indices (og_corner) of all corners of one candidate cell. */
static inline void og_cell_corners(const og_grid* g, const int64_t cell[3], const double loc[3],
                                   double w[8], int64_t f[8]) {
  const int d = g->dim;
  const int ncorner = 1 << d;
  double lo_w[3], hi_w[3];
  int64_t lo_f[3], hi_f[3];
  for (int ax = 0; ax < d; ++ax) {
    hi_w[ax] = loc[ax];
    lo_w[ax] = 1.0 - loc[ax];
    int64_t e0 = cell[ax], e1 = cell[ax] + 1;
    if (g->periodic[ax]) {
      int64_t M = g->shape[ax];
      if (e0 == 0) e0 = M; else if (e0 == M + 1) e0 = 1;
      if (e1 == 0) e1 = M; else if (e1 == M + 1) e1 = 1;
    }
    lo_f[ax] = e0 * g->strides[ax];
    hi_f[ax] = e1 * g->strides[ax];
  }
  for (int corner = 0; corner < ncorner; ++corner) {
    double ww = 1.0;
    int64_t ff = 0;
    for (int ax = 0; ax < d; ++ax) {
      if ((corner >> ax) & 1) { ww *= hi_w[ax]; ff += hi_f[ax]; }
      else { ww *= lo_w[ax]; ff += lo_f[ax]; }
    }
    w[corner] = ww;
    f[corner] = ff;
  }
}

static inline double og_apply_rule(int rule, double v, double cost) {
  if (rule == OG_RULE_REF) return v + cost;
  double beta = exp(-cost);
  return beta * v + (1.0 - beta);
}

/* Relax one node (the body of _kernels.py:57-105). */
static void og_relax(const og_grid* g, const og_dyn* dy, int64_t s,
                     const double* rd_live, const uint8_t* active, const double* frozen,
                     const uint8_t* hard, const uint8_t* allowed, int rule,
                     double* best_out, int64_t* nevals) {
  const int ncorner = 1 << g->dim;
  double best = OG_BIG, X[3];
  og_point(g, s, X);
  for (int c = 0; c < dy->nc; ++c) {
    int64_t cell[3];
    double loc[3], cost;
    if (!og_foot_at(g, dy, s, X, c, cell, loc, &cost)) continue;
    if (allowed && allowed[(int64_t)s * dy->nc + c] == 0) continue;
    *nevals += 1;
    double v = 0.0, wc[8];
    int64_t fc[8];
    int rejected = 0;
    og_cell_corners(g, cell, loc, wc, fc);
    for (int corner = 0; corner < ncorner; ++corner) {
      double w = wc[corner];
      if (w == 0.0) continue;
      int64_t f2 = fc[corner];
      if (hard[f2] != 0) {
        rejected = 1;
        break;
      }
      double cv = (active == 0 || active[f2] != 0) ? rd_live[f2] : frozen[f2];
      v += w * cv;
    }
    if (rejected) continue;
    v = og_apply_rule(rule, v, cost);
    if (v < best) best = v;
  }
  *best_out = best;
}

/*
 * One sweep over order[0:n] (sweep_batch, _kernels.py:18-106).
 *   u_in == NULL : Gauss-Seidel in place on u (reference semantics, serial).
 *   u_in != NULL : Jacobi, reads u_in (live) / frozen, writes u (caller copies
 *                  u_in into u first so untouched nodes carry over).
 * active == NULL means all-active; frozen == NULL means frozen = live array.
 * sentinel is the obstacle value (1e9 reference rule, 1.0 Kruzkov).
 */
void og_sweep(const og_grid* g, const og_dyn* dy, double* u, const double* u_in,
              const int64_t* order, int64_t n, const uint8_t* kind,
              const uint8_t* active, const double* frozen, const uint8_t* hard,
              const uint8_t* allowed, double sentinel, int rule, int nthreads,
              double* out_maxch, int64_t* out_nrelax, int64_t* out_nevals) {
  double maxch = 0.0;
  int64_t nevals = 0;
  if (u_in == 0) {
    const double* fr = frozen ? frozen : u;
    for (int64_t oi = 0; oi < n; ++oi) {
      int64_t s = order[oi];
      int64_t fi = og_iflat(g, s);
      uint8_t k = kind[s];
      if (k == 1) { u[fi] = 0.0; continue; }
      if (k == 2) { u[fi] = sentinel; continue; }
      double old = u[fi], best;
      og_relax(g, dy, s, u, active, fr, hard, allowed, rule, &best, &nevals);
      if (best < old) {
        u[fi] = best;
        double ch = old - best;
        if (ch > maxch) maxch = ch;
      }
    }
  } else {
    const double* fr = frozen ? frozen : u_in;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads) reduction(max : maxch) reduction(+ : nevals)
#endif
    for (int64_t oi = 0; oi < n; ++oi) {
      int64_t s = order[oi];
      int64_t fi = og_iflat(g, s);
      uint8_t k = kind[s];
      if (k == 1) { u[fi] = 0.0; continue; }
      if (k == 2) { u[fi] = sentinel; continue; }
      double old = u_in[fi], best;
      int64_t ev = 0;
      og_relax(g, dy, s, u_in, active, fr, hard, allowed, rule, &best, &ev);
      nevals += ev;
      if (best < old) {
        u[fi] = best;
        double ch = old - best;
        if (ch > maxch) maxch = ch;
      } else {
        u[fi] = old;
      }
    }
  }
  *out_maxch = maxch;
  *out_nrelax = n;
  *out_nevals = nevals;
}

/*
 * Argmin control per interior serial (feedback_batch, _kernels.py:109-167).
 * Dirichlet-style reads of u, reject on hard, strict < (lowest index wins).
 * `unreach` is the "own value too large" threshold (0.5*sentinel reference,
 * 1.0 Kruzkov).  Candidate values use the same rule as the sweep.
 */
int64_t og_feedback(const og_grid* g, const og_dyn* dy, const double* u,
                    const uint8_t* kind, const uint8_t* hard, const uint8_t* allowed,
                    double unreach, int rule, int nthreads, int32_t* out,
                    double* gap_out) {
  const int64_t N = g->shape[0] * g->shape[1] * (g->dim == 3 ? g->shape[2] : 1);
  const int ncorner = 1 << g->dim;
  int64_t nevals = 0;
#ifdef _OPENMP
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads) reduction(+ : nevals)
#endif
  for (int64_t s = 0; s < N; ++s) {
    int64_t fi = og_iflat(g, s);
    out[s] = -1;
    if (gap_out) gap_out[s] = OG_BIG;
    if (kind[s] != 0) continue;
    if (u[fi] >= unreach) continue;
    double best = OG_BIG, second = OG_BIG, X[3];
    int32_t bc = -1;
    og_point(g, s, X);
    for (int c = 0; c < dy->nc; ++c) {
      int64_t cell[3];
      double loc[3], cost;
      if (!og_foot_at(g, dy, s, X, c, cell, loc, &cost)) continue;
      if (allowed && allowed[s * dy->nc + c] == 0) continue;
      nevals += 1;
      double v = 0.0, wc[8];
      int64_t fc[8];
      int rejected = 0;
      og_cell_corners(g, cell, loc, wc, fc);
      for (int corner = 0; corner < ncorner; ++corner) {
        double w = wc[corner];
        if (w == 0.0) continue;
        int64_t f2 = fc[corner];
        if (hard[f2] != 0) { rejected = 1; break; }
        v += w * u[f2];
      }
      if (rejected) continue;
      v = og_apply_rule(rule, v, cost);
      if (v < best) {
        second = best;
        best = v;
        bc = c;
      } else if (v < second) {
        second = v;
      }
    }
    out[s] = bc;
    /* best-vs-second gap: the tie diagnostic of the parity protocol */
    if (gap_out) gap_out[s] = (bc >= 0 && second < OG_BIG) ? second - best : OG_BIG;
  }
  return nevals;
}

/*
 * Feet of an explicit (serial, control) list: ext cells + snapped locals +
 * cost (-1 when inadmissible).  Used for transport feet (patchy.py:165-180).
 */
void og_feet(const og_grid* g, const og_dyn* dy, const int64_t* serials,
             const int32_t* ctrl, int64_t n, int64_t* cell_out, double* loc_out,
             double* cost_out) {
  const int d = g->dim;
  for (int64_t i = 0; i < n; ++i) {
    int64_t cell[3] = {0, 0, 0};
    double loc[3] = {0, 0, 0}, cost = -1.0;
    if (ctrl[i] >= 0 && !og_foot(g, dy, serials[i], ctrl[i], cell, loc, &cost)) cost = -1.0;
    for (int ax = 0; ax < d; ++ax) {
      cell_out[i * d + ax] = cell[ax];
      loc_out[i * d + ax] = loc[ax];
    }
    cost_out[i] = cost;
  }
}

/*
 * One transport pass over movers (transport_batch, _kernels.py:170-204):
 * phi_i <- sum_{w != 0} w * phi(corner).  phi_in == NULL: GS in place;
 * otherwise Jacobi (phi_in -> phi).  Returns max |change|.
 */
double og_transport(const og_grid* g, double* phi, const double* phi_in,
                    const int64_t* movers, int64_t n, const int64_t* cells,
                    const double* locs, int nthreads) {
  const int d = g->dim;
  const int ncorner = 1 << d;
  double maxch = 0.0;
  if (phi_in == 0) {
    for (int64_t oi = 0; oi < n; ++oi) {
      int64_t s = movers[oi];
      int64_t fi = og_iflat(g, s);
      double v = 0.0;
      for (int corner = 0; corner < ncorner; ++corner) {
        double w = og_weight(d, locs + oi * d, corner);
        if (w != 0.0) v += w * phi[og_corner(g, cells + oi * d, corner)];
      }
      double ch = phi[fi] - v;
      if (ch < 0.0) ch = -ch;
      phi[fi] = v;
      if (ch > maxch) maxch = ch;
    }
  } else {
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(max : maxch)
#endif
    for (int64_t oi = 0; oi < n; ++oi) {
      int64_t s = movers[oi];
      int64_t fi = og_iflat(g, s);
      double v = 0.0;
      for (int corner = 0; corner < ncorner; ++corner) {
        double w = og_weight(d, locs + oi * d, corner);
        if (w != 0.0) v += w * phi_in[og_corner(g, cells + oi * d, corner)];
      }
      double ch = phi_in[fi] - v;
      if (ch < 0.0) ch = -ch;
      phi[fi] = v;
      if (ch > maxch) maxch = ch;
    }
  }
  return maxch;
}

/*
 * Saturating multilinear lift of a coarse field onto fine interior nodes
 * (interpolate_many, grid.py:242-261, used at patchy.py:146-148).  Corner
 * sums follow numpy's reduction order: sequential for 4 terms, the pairwise
 * tree for 8 (np.add.reduce over a length-8 contiguous row).
 */
void og_lift(const og_grid* gc, const double* uc, const og_grid* gf, double* out,
             double sat_threshold, double sat_value, int saturate, int nthreads) {
  const int d = gf->dim;
  const int ncorner = 1 << d;
  const int64_t N = gf->shape[0] * gf->shape[1] * (d == 3 ? gf->shape[2] : 1);
#ifdef _OPENMP
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
  for (int64_t s = 0; s < N; ++s) {
    double X[3], loc[3], terms[8];
    int64_t cell[3];
    og_point(gf, s, X);
    og_locate(gc, X, cell, loc);
    int bad = 0;
    for (int corner = 0; corner < ncorner; ++corner) {
      double w = og_weight(d, loc, corner);
      double cv = uc[og_corner(gc, cell, corner)];
      terms[corner] = w * cv;
      if (w > 0.0 && cv >= sat_threshold) bad = 1;
    }
    double v;
    if (ncorner == 4) {
      v = terms[0] + terms[1];
      v = v + terms[2];
      v = v + terms[3];
    } else {
      v = ((terms[0] + terms[1]) + (terms[2] + terms[3])) +
          ((terms[4] + terms[5]) + (terms[6] + terms[7]));
    }
    out[s] = (saturate && bad) ? sat_value : v;
  }
}

/*
 * Fixed-point residual certificate of a converged patch solve (full-size
 * parity, tests/test_gpu_fullsize.py).  One Jacobi application of the
 * reference relaxation (_kernels.py:57-100) to a given field u WITHOUT the
 * monotone write of :101-105, under the state constraint of a given patch
 * map: a nonzero-weight corner is readable iff it is an interior node whose
 * label is the node's own patch or TARGET (patchy.py:369-371 active = patch
 * u target; solver.py:247 hard = hard_base | ~active).
 *   lab_ext : int32 per ext node (patchy.py:40-45 codes): >= 0 patch, -2
 *             TARGET, other < 0 blocked (UNREACHABLE / OBSTACLE / ghost);
 *             periodic ghosts are never read (corners wrap).
 *   unreach : 1.0 (Kruzkov) or 0.5*sentinel (reference rule).
 * out[0] = max |T(u)_i - u_i| over free patch nodes with u_i < unreach
 * out[1] = serial where out[0] is attained
 * cnt[0] = free patch nodes with u >= unreach but T(u) < unreach (1 - 1e-9) (missed)
 * cnt[1] = free patch nodes with u < unreach but T(u) >= unreach (spurious)
 * cnt[2] = target nodes with u != 0
 * cnt[3] = blocked nodes with u < unreach
 * cnt[4] = free patch nodes with u < unreach (the certified set)
 * cnt[5] = candidate evaluations
 * missed_list (optional, 2 x missed_cap entries): serials of the missed nodes,
 *   then (from missed_cap on) of the spurious ones
 */
void og_residual(const og_grid* g, const og_dyn* dy, const double* u, const uint8_t* kind,
                 const int32_t* lab_ext, double unreach, int rule, int nthreads,
                 double* out, int64_t* cnt, int64_t* missed_list, int64_t missed_cap) {
  const int64_t N = g->shape[0] * g->shape[1] * (g->dim == 3 ? g->shape[2] : 1);
  const int ncorner = 1 << g->dim;
  double rmax = 0.0;
  int64_t at = -1, missed = 0, spurious = 0, badt = 0, badb = 0, ncert = 0, nevals = 0;
  if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads) reduction(+ : missed, spurious, badt, badb, ncert, nevals)
#endif
  {
    double lmax = 0.0;
    int64_t lat = -1;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1024)
#endif
    for (int64_t s = 0; s < N; ++s) {
      const int64_t fi = og_iflat(g, s);
      const int32_t L = lab_ext[fi];
      if (kind[s] == 1 || L == -2) {
        if (u[fi] != 0.0) badt += 1;
        continue;
      }
      if (L < 0 || kind[s] != 0) {
        if (u[fi] < unreach) badb += 1;
        continue;
      }
      double best = OG_BIG, X[3];
      og_point(g, s, X);
      for (int c = 0; c < dy->nc; ++c) {
        int64_t cell[3];
        double loc[3], cost;
        if (!og_foot_at(g, dy, s, X, c, cell, loc, &cost)) continue;
        nevals += 1;
        double v = 0.0, wc[8];
        int64_t fc[8];
        int rejected = 0;
        og_cell_corners(g, cell, loc, wc, fc);
        for (int corner = 0; corner < ncorner; ++corner) {
          if (wc[corner] == 0.0) continue;
          const int32_t L2 = lab_ext[fc[corner]];
          if (!(L2 == L || L2 == -2)) { rejected = 1; break; }
          v += wc[corner] * u[fc[corner]];
        }
        if (rejected) continue;
        v = og_apply_rule(rule, v, cost);
        if (v < best) best = v;
      }
      /* margin: values within 1e-9 (relative) of the unreached level are at
       * the floating-point floor of the Kruzkov transform (v = 1 - 1 ulp is
       * T ~ 37), and a candidate over unreached corners only is 1 up to the
       * rounding of the reference's per-node weights (their sum is 1 only
       * to ~1 ulp, grid.py:227-239): neither side counts them as reached */
      const double thr = unreach * (1.0 - 1.0e-9);
      if (u[fi] >= unreach) {
        if (best < thr) {
          int64_t k;
#ifdef _OPENMP
#pragma omp atomic capture
#endif
          k = missed++;
          if (missed_list && k < missed_cap) missed_list[k] = s;
        }
        continue;
      }
      if (best >= unreach && u[fi] < thr) {
        int64_t k;
#ifdef _OPENMP
#pragma omp atomic capture
#endif
        k = spurious++;
        if (missed_list && k < missed_cap) missed_list[missed_cap + k] = s;
        continue;
      }
      if (best > unreach) best = unreach;
      ncert += 1;
      double r = best - u[fi];
      if (r < 0.0) r = -r;
      if (r > lmax) { lmax = r; lat = s; }
    }
#ifdef _OPENMP
#pragma omp critical
#endif
    {
      if (lmax > rmax) { rmax = lmax; at = lat; }
    }
  }
  out[0] = rmax;
  out[1] = (double)at;
  cnt[0] = missed; cnt[1] = spurious; cnt[2] = badt; cnt[3] = badb; cnt[4] = ncert;
  cnt[5] = nevals;
}

/*
 * Transport residual of one colour field (transport_batch, _kernels.py:
 * 179-204, one Jacobi application without the update): max over movers
 * (patchy.py:165-180: feedback >= 0, free, admissible foot) of
 * |phi_i - sum_{w != 0} w phi(corner)|.  Feet on the fly from the feedback
 * control (solver.py:175-188).  Returns the residual; *n_movers counts.
 */
double og_transport_residual(const og_grid* g, const og_dyn* dy, const int32_t* fb,
                             const uint8_t* kind, const double* phi, int nthreads,
                             int64_t* n_movers) {
  const int64_t N = g->shape[0] * g->shape[1] * (g->dim == 3 ? g->shape[2] : 1);
  const int ncorner = 1 << g->dim;
  double rmax = 0.0;
  int64_t nm = 0;
  if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(max : rmax) reduction(+ : nm)
#endif
  for (int64_t s = 0; s < N; ++s) {
    if (kind[s] != 0 || fb[s] < 0) continue;
    int64_t cell[3];
    double loc[3], cost;
    if (!og_foot(g, dy, s, fb[s], cell, loc, &cost)) continue;
    nm += 1;
    double v = 0.0;
    for (int corner = 0; corner < ncorner; ++corner) {
      double w = og_weight(g->dim, loc, corner);
      if (w != 0.0) v += w * phi[og_corner(g, cell, corner)];
    }
    double r = phi[og_iflat(g, s)] - v;
    if (r < 0.0) r = -r;
    if (r > rmax) rmax = r;
  }
  *n_movers = nm;
  return rmax;
}

/* max over serials of |f(...)| for eps_speed (solver.py:162-168). */
double og_max_speed(const og_grid* g, const og_dyn* dy) {
  const int d = g->dim;
  const int64_t N = g->shape[0] * g->shape[1] * (d == 3 ? g->shape[2] : 1);
  double mx = 0.0;
  for (int64_t s = 0; s < N; ++s) {
    double X[3];
    og_point(g, s, X);
    for (int c = 0; c < dy->nc; ++c) {
      double F[3] = {0, 0, 0};
      if (dy->kind == OG_DYN_SCALED) {
        for (int ax = 0; ax < d; ++ax) F[ax] = dy->speed[s] * dy->controls[c * dy->m + ax];
      } else if (dy->kind == OG_DYN_TABLE) {
        for (int ax = 0; ax < d; ++ax) F[ax] = dy->F[(s * dy->nc + c) * d + ax];
      } else {
        F[0] = cos(X[2]);
        F[1] = sin(X[2]);
        F[2] = dy->controls[c * dy->m];
      }
      double ss = F[0] * F[0];
      for (int ax = 1; ax < d; ++ax) ss = ss + F[ax] * F[ax];
      double sp = sqrt(ss);
      if (sp > mx) mx = sp;
    }
  }
  return mx;
}

int og_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
