/*
 * phj.h -- C ABI of libphj.so, the B200 (sm_100a) patchy semi-Lagrangian
 * HJB engine.  Plain C types only: every array is a raw DEVICE pointer owned
 * by the caller (the Python host package keeps them in torch tensors), every
 * call takes the CUDA stream to run on and returns PHJ_OK or an error code
 * (phj_last_error() gives the message; no C++ exception crosses the ABI).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/patchyhjb/):
 *   phj_solve            _kernels.sweep_batch       _kernels.py:18-106, driven by
 *                        solver.solve               solver.py:201-279 (whole loop
 *                        on device: sweeps, convergence, per-patch stop) and by
 *                        patchy.solve_patches       patchy.py:304-389 (all patches
 *                        in one launch)
 *   phj_feedback         _kernels.feedback_batch    _kernels.py:109-167,
 *                        solver.extract_feedback    solver.py:413-443
 *   phj_transport        _kernels.transport_batch   _kernels.py:170-204,
 *                        patchy.transport_color     patchy.py:183-219
 *   phj_lift             grid.interpolate_many      grid.py:242-261 (patchy.py:146-148)
 *   phj_argmax_update,   patchy.assemble_patches    patchy.py:236-301
 *   phj_assemble_*
 *   phj_classify         solver.classify_nodes      solver.py:101-108
 *   phj_error_partials   analysis.error_report      analysis.py:50-63
 *
 * Layout: fields are ghost-padded C-order arrays (grid.py:69-85), one ghost
 * layer, last internal axis fastest.  The host may permute user axes so that
 * a stencil "class" axis (Dubins heading) is internal axis 0; periodic axes
 * keep ghost layers as copies of the opposite interior layer.
 */
#ifndef PHJ_H
#define PHJ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHJ_OK 0
#define PHJ_ERR_ARG 1
#define PHJ_ERR_CUDA 2
#define PHJ_ERR_UNSUPPORTED 3

#define PHJ_F64 0
#define PHJ_F32 1

#define PHJ_RULE_REF 0     /* u <- min_a I[u](x + h f) + h      (reference)   */
#define PHJ_RULE_KRUZKOV 1 /* v <- min_a beta I[v](x + h f) + 1 - beta        */

#define PHJ_COST_NODE 0 /* step cost per node (f = c(x) a, |a| = 1): hoisted  */
#define PHJ_COST_CTRL 1 /* step cost per stencil entry (translation/Dubins)   */

/* patch labels in the ext label array (int16) */
#define PHJ_LAB_FIXED (-1)  /* not swept, readable (frozen / inactive data)    */
#define PHJ_LAB_TARGET (-2) /* target: value 0, readable by every patch       */
#define PHJ_LAB_HARD (-3)   /* ghost / obstacle / unreachable: never readable */

/* patch-map codes (patchy.py:40-43) */
#define PHJ_UNREACHABLE (-1)
#define PHJ_TARGET (-2)
#define PHJ_OBSTACLE (-3)
#define PHJ_UNCOVERED (-4)

typedef struct phj_grid {
  int32_t dim;         /* 2 or 3 */
  int32_t periodic[3]; /* per internal axis */
  int64_t shape[3];    /* interior nodes per internal axis */
  int64_t ext[3];      /* shape + 2 */
  int64_t strides[3];  /* ext strides in nodes */
  double lo[3];
  double spacing[3];
  double ext_lo[3];
  double k; /* step length |h f| = k (grid.py:67) */
} phj_grid;

/* entries evaluated per inner-loop iteration; each octant group of a class
 * holds a multiple of this many entries (query a build with phj_unroll) */
#ifndef PHJ_UNROLL3
#define PHJ_UNROLL3 2
#endif
#define PHJ_UNROLL(dim) ((dim) == 2 ? 4 : PHJ_UNROLL3)

/* Node-independent interpolation stencils, one set per class (class index =
 * interior index along internal axis 0 when n_classes > 1).  Entries of a
 * class are sorted by foot octant; octant bit ax = foot on the + side of
 * internal axis ax, corner bit ax = upper face of that octant cell.  All
 * pointers are device pointers. */
typedef struct phj_stencil {
  int32_t dim;
  int32_t n_classes;
  int32_t n_controls; /* entry slots per class (octant groups padded to a
                         multiple of PHJ_UNROLL(dim) by repeating an entry) */
  int32_t cost_mode;  /* PHJ_COST_NODE or PHJ_COST_CTRL */
  int32_t n_real;     /* admissible controls per class (work accounting) */
  int32_t pad_;
  const int32_t* oct_start; /* [n_classes][2^dim + 1] */
  const int32_t* ctrl;      /* [n_classes][nc] original control index */
  const uint32_t* nzmask;   /* [n_classes][nc] nonzero-weight 3^dim positions */
  const double* weights;    /* [n_classes][nc][2^dim] */
  const double* cost;       /* [n_classes][nc] step cost (COST_CTRL); < 0 skips */
} phj_stencil;

typedef struct phj_solve_args {
  phj_grid grid;
  phj_stencil st;
  int32_t dtype; /* PHJ_F64 / PHJ_F32 */
  int32_t rule;  /* PHJ_RULE_* */
  void* v0;      /* ext field, ping */
  void* v1;      /* ext field, pong; both hold the start field on entry */
  const int16_t* lab;     /* ext labels: >= 0 patch id (swept), PHJ_LAB_* */
  const uint32_t* fmask;  /* ext foreign-position masks (phj_fmask_*) */
  const void* coef;       /* per ext node: h (REF) or beta (KRUZKOV) in dtype,
                             < 0 = no admissible control; NULL => coef0 */
  double coef0;
  int32_t n_patches;
  int32_t max_sweeps;
  const uint8_t* mine; /* [n_patches] patches this device sweeps; NULL = all */
  double tol;
  void* workspace;            /* phj_solve_workspace_bytes() bytes */
  int32_t* patch_sweeps;      /* out [n_patches]: sweeps to converge, -(cap) if not */
  double* maxch_hist;         /* out [max_sweeps * n_patches], may be NULL */
  unsigned long long* evals;  /* out [3]: [0] candidate evaluations of the swept nodes
                                 (nodes x admissible controls, per block-local
                                 relaxation), [1] stencil-entry evaluations executed
                                 (incl. padding and masked lanes, after pruning),
                                 [2] real candidate evaluations executed (computing
                                 nodes x non-padding entries, after pruning) */
  int32_t* info;              /* out [4]: total sweeps, index of result buffer,
                                 tiles processed, launches */
  /* AO3 conical control reduction (solver.py:446-476; NULL ao3_fb = off):
   * a node with feedback control f >= 0 only evaluates the stencil entries
   * whose bits are set in ao3_mask[f * ao3_words ...] (entry index order of
   * the class-0 stencil, 64 entries per word) and counts ao3_count[f]
   * candidate evaluations; f < 0 keeps every entry. */
  const int32_t* ao3_fb;                /* ext layout, feedback control per node or -1 */
  const unsigned long long* ao3_mask;   /* [n_controls][ao3_words] */
  const int32_t* ao3_count;             /* [n_controls] */
  int32_t ao3_words;                    /* 1 or 2 */
  int32_t options;            /* PHJ_SOLVE_* bits, 0 = defaults */
  /* activity threshold: a node change re-activates the neighbour blocks only
   * if it exceeds act_tol in time units (KRUZKOV: dv > act_tol * (1 - v),
   * REF: du > act_tol * max(1, u)); smaller changes re-sweep their own block
   * once.  0 = exact Jacobi activity. */
  double act_tol;
  /* block-local relaxations per sweep (<= 1: one, plain Jacobi): the block's
   * nodes are relaxed up to this many times from the staged tile with the
   * halo ring held at the sweep's input -- block-Jacobi with inner
   * iterations, same fixed point, schedule-independent */
  int32_t inner_sweeps;
  /* out [n_patches][3] or NULL: per patch, node relaxations, logical candidate
   * evaluations (evals[0] split by patch) and real executed ones (evals[2]);
   * the reference's per-patch SweepStats counters (solver.py:79-88) under both
   * schedules */
  unsigned long long* patch_counts;
  /* optional value-ordered pass (NULL band_off = off):
   * sweep s < n_band visits exactly the blocks band_list[band_off[s] ..
   * band_off[s+1]) (entry b = relax block b, -b-1 = copy its nodes into the
   * other buffer: its last visit), sweep n_band visits row n_band (every
   * block of the pass) as an ordinary Jacobi sweep; per-patch stopping starts
   * after it.  With PHJ_SOLVE_ASYNC the pass runs alone and the asynchronous
   * relaxation continues from its result.  Rows come from the lifted field's
   * time-to-target (patchy.band_schedule); n_band < max_sweeps. */
  const int32_t* band_list;
  const int32_t* band_off;   /* [n_band + 2] */
  int32_t n_band;
  int32_t band_inner;        /* block-local relaxations per visit in the pass
                                (0 = inner_sweeps) */
  void* stream;               /* cudaStream_t */
} phj_solve_args;

/* phj_solve_args.options: evaluate every octant (disable the exact octant
 * pruning; for verification -- results are bit-identical either way) */
#define PHJ_SOLVE_NO_PRUNE 1
/* asynchronous (chaotic) relaxation in one buffer instead of barrier-separated
 * Jacobi sweeps: same fixed point, to within act_tol (> 0 required); result
 * in v0, patch_sweeps = equivalent sweeps (blocks swept / initial blocks),
 * maxch_hist untouched */
#define PHJ_SOLVE_ASYNC 2

int64_t phj_solve_workspace_bytes(const phj_grid* g, int32_t n_patches, int32_t max_sweeps);
/* PHJ_UNROLL(dim) this library was built with (octant-group padding) */
int32_t phj_unroll(int32_t dim);
/* number of warp blocks (work/activity units) of a grid (diagnostics) */
int64_t phj_blocks_total(const phj_grid* g);
/* warp-block extent along the internal axes (block = planes x rows x nodes,
 * axis 0 slowest): out[0..2]; 2D grids use out[0..1] */
int phj_block_dims(int32_t dim, int32_t* out);

/* Schedule of a value-ordered pass (the band_list / band_off rows of
 * phj_solve_args and phj_transport_args).  `key` is the
 * lifted working field (ext layout, dtype; Kruzkov v is turned into
 * T = -log(1 - v)), `nodes` one byte per internal serial (1 = scheduled).
 * Bands are floor(T / delta) with delta = max(delta_min, T_max / max_bands);
 * a block is relaxed at sweeps [min band - hi_w, max band + lo_w] of its nodes
 * and copied one sweep later.  phj_band_count synchronises the stream and
 * returns out[0] = entries (without the final row), out[1] = n_band,
 * out[2] = scheduled blocks, out[3] = delta (double bits); phj_band_fill then
 * writes band_list [out[0] (+ out[2] with final_row)] and band_off
 * [n_band + 1 (+ 1)] (final_row: row n_band = every scheduled block).
 * Rows are in no particular block order. */
int64_t phj_band_scratch_bytes(const phj_grid* g, int32_t max_bands, int32_t lo_w, int32_t hi_w);
int phj_band_count(const phj_grid* g, int32_t dtype, int32_t rule, const void* key,
                   const uint8_t* nodes, double delta_min, int32_t max_bands, int32_t lo_w,
                   int32_t hi_w, void* scratch, int64_t* out, void* stream);
int phj_band_fill(const phj_grid* g, int32_t max_bands, int32_t lo_w, int32_t hi_w,
                  int32_t n_band, int32_t n_blocks, int32_t final_row, void* scratch,
                  int32_t* band_list, int32_t* band_off, void* stream);
int phj_solve(const phj_solve_args* a);

/* foreign-position masks: bit p set when 3^dim neighbour p of the node is not
 * readable by it.  From patch labels (corner label not in {own, TARGET,
 * FIXED}) or from a caller hard mask (uint8 per ext node, non-zero = hard). */
int phj_fmask_from_labels(const phj_grid* g, const int16_t* lab, uint32_t* fmask, void* stream);
int phj_fmask_from_hard(const phj_grid* g, const uint8_t* hard, uint32_t* fmask, void* stream);

/* Argmin control per interior serial (out is indexed by internal serial).
 * unreach: own-value threshold (0.5*sentinel REF, 1.0 KRUZKOV); reads reject
 * only where `fmask` (built from the ghost/obstacle hard mask) says so.
 * The rule is applied per candidate and ties go to the lowest ORIGINAL
 * control index (strict <, _kernels.py:162-165). */
int phj_feedback(const phj_grid* g, const phj_stencil* st, int32_t dtype, int32_t rule,
                 const void* v, const int8_t* kind, const uint32_t* fmask, const void* coef,
                 double coef0, double unreach, int32_t* out, unsigned long long* evals,
                 void* stream);
/* phj_feedback restricted per node (solver.extract_feedback(allowed=...),
 * _kernels.py:71-75): allow_row per ext node (-1 = all controls) indexes
 * allow_mask [rows][allow_words] (bit e = stencil entry e allowed) and
 * allow_count [rows] (allowed admissible controls, the evaluation count).
 * Single-class stencils, <= 128 entries (allow_words 1..2). */
int phj_feedback_allowed(const phj_grid* g, const phj_stencil* st, int32_t dtype, int32_t rule,
                         const void* v, const int8_t* kind, const uint32_t* fmask,
                         const void* coef, double coef0, double unreach,
                         const int32_t* allow_row, const unsigned long long* allow_mask,
                         const int32_t* allow_count, int32_t allow_words, int32_t* out,
                         unsigned long long* evals, void* stream);

/* phj_feedback_allowed on a slab of the grid: block rows [slab_begin,
 * slab_end) along internal axis 0 (phj_block_dims[0] node layers each;
 * slab_end < 0 = the whole grid).  Only the nodes of the slab are written
 * to `out` and counted in `evals` (accumulated, not reset).  The ranks of a
 * multi-GPU run split the feedback stage by slabs and all-gather `out`
 * (paper_1109_3577_b200/dist.py; the reference's feedback loop over all
 * serials, solver.py:413-443, has no such split). */
int phj_feedback_slab(const phj_grid* g, const phj_stencil* st, int32_t dtype, int32_t rule,
                      const void* v, const int8_t* kind, const uint32_t* fmask, const void* coef,
                      double coef0, double unreach, const int32_t* allow_row,
                      const unsigned long long* allow_mask, const int32_t* allow_count,
                      int32_t allow_words, int32_t* out, unsigned long long* evals,
                      int32_t slab_begin, int32_t slab_end, void* stream);

/* Colour transport of all target parts at once, each to its own
 * max|change| <= tol (Jacobi, whole loop on device, one launch).  phi0/phi1
 * are colour-major [n_colors][ext nodes] doubles holding the start fields
 * (1 on the part, 0 elsewhere); movers have fb >= 0 and kind == 0. */
typedef struct phj_transport_args {
  phj_grid grid;
  phj_stencil st;
  void* phi0;           /* [n_colors][ext] in phi_dtype */
  void* phi1;
  const int32_t* fb;    /* per internal serial, original control index or -1 */
  const int8_t* kind;   /* per internal serial */
  int32_t* ent_scratch; /* [interior nodes] int32 scratch (mover -> stencil entry) */
  int32_t n_colors;
  double tol;
  double act_eps;       /* a block re-activates its neighbours for colour j only
                           when some node of it changed colour j by more than
                           this (0 = exact Jacobi activity) */
  int32_t max_sweeps;
  void* workspace;      /* phj_solve_workspace_bytes(g, 1, max_sweeps) */
  double* maxch_hist;   /* out [max_sweeps][n_colors] */
  int32_t* color_sweeps; /* out [n_colors]: sweeps to converge, -(cap) if not */
  int32_t* info;        /* out [4]: total sweeps, result buffer, -, - */
  unsigned long long* updates; /* out [1]: mover updates performed */
  int32_t options;      /* PHJ_TRANSPORT_* bits */
  int32_t inner_sweeps; /* async: relaxations of a colour per block visit (>= 1) */
  int32_t phi_dtype;    /* PHJ_F64 (0) or PHJ_F32: storage of the colour fields
                           (accumulation is fp64 either way) */
  /* optional seeding (n_colors <= 64): the part nodes (internal ext flat
   * index, colour) -- only blocks next to a part of colour j start active for
   * colour j (exact: elsewhere phi_j = 0 on every foot corner); NULL = every
   * mover block starts active for every colour */
  const int64_t* seed_flat;
  const int32_t* seed_col;
  int64_t n_seed;
  /* optional value-ordered pass before the Jacobi sweeps (Jacobi transport
   * only; NULL band_off = off): sweep s < n_band processes exactly the blocks
   * band_list[band_off[s] .. band_off[s+1]) (entry b = Jacobi update of block
   * b's movers for the colours that have reached it; -b-1 = copy its movers'
   * values into the other buffer, its last visit).  Built by the host from
   * the lifted field's time-to-target (patchy.transport_bands): a node is
   * updated while its time band is within a window sliding outward from the
   * target, so the colour masses are carried across the domain in one pass;
   * the Jacobi sweeps that follow stop at max change <= tol as usual. */
  const int32_t* band_list;
  const int32_t* band_off;   /* [n_band + 1] */
  int32_t n_band;
  void* stream;
} phj_transport_args;

/* phj_transport_args.options: asynchronous in-place transport (block FIFO, no
 * grid barrier; phi1 unused, result in phi0): every colour converges until
 * no node changes by more than act_eps; color_sweeps = equivalent sweeps
 * */
#define PHJ_TRANSPORT_ASYNC 1
/* Jacobi transport: a work ticket buys two consecutive list entries instead
 * of one (half the same-address claims per sweep; for launches that own few
 * of the colours -- a rank of a multi-GPU run -- and find most entries empty) */
#define PHJ_TRANSPORT_PAIRS 2

/* argmax over the colours of a [n_colors][ext] colour field (strict >,
 * lowest colour on ties, patchy.py:251-256) */
int phj_argmax_colors(const phj_grid* g, const double* phi, int32_t n_colors, double* best_val,
                      int32_t* best_idx, void* stream);
/* the same over colour fields stored in phi_dtype (PHJ_F64 / PHJ_F32);
 * quantum > 0 compares floor(phi / quantum) * quantum instead (colours within
 * rounding noise tie exactly; lowest colour wins), 0 = strict argmax */
int phj_argmax_colors_t(const phj_grid* g, const void* phi, int32_t phi_dtype, int32_t n_colors,
                        double quantum, double* best_val, int32_t* best_idx, void* stream);
int phj_transport(const phj_transport_args* a);

/* Saturating multilinear lift of a coarse ext field to fine ext interior. */
/* multilinear interpolation of an ext field (dtype) at n arbitrary points
 * (row-major [n][dim] doubles in the grid's coordinates): grid.interpolate_many
 * (grid.py:242-261) semantics -- 1e-9 bounds tolerance on the ghost-extended
 * box (ood[i] = 1 outside), snapped locals, saturation to sat_value when a
 * nonzero-weight corner is >= sat_threshold (saturate != 0); out in double.
 * Used by analysis.trace_trajectory (analysis.py:82-139). */
int phj_interpolate_points(const phj_grid* g, int32_t dtype, const void* field,
                           const double* points, int64_t n, double sat_threshold,
                           double sat_value, int32_t saturate, double* out, int8_t* ood,
                           void* stream);
int phj_lift(const phj_grid* gc, const phj_grid* gf, int32_t dtype, const void* vc, void* vf,
             double sat_threshold, double sat_value, int32_t saturate, void* stream);

/* running argmax over colour fields (strict >, patchy.py:251-256) */
int phj_argmax_update(const phj_grid* g, const double* phi, int32_t j, double* best_val,
                      int32_t* best_idx, void* stream);
/* codes (patchy.py:258-262) */
int phj_assemble_codes(const phj_grid* g, const double* best_val, const int32_t* best_idx,
                       const uint8_t* mask, const int8_t* kind, int32_t* color, void* stream);
/* one order-free majority-repair pass (patchy.py:264-282); n_filled/n_open out */
int phj_assemble_repair(const phj_grid* g, const int32_t* color_in, int32_t* color_out,
                        int32_t n_colors, int32_t* counters, void* stream);
/* leftovers -> 0, boundary flags, patch labels for the solve (patchy.py:284-300) */
/* patch sizes: counts[c] = #{s < n : color[s] == c}, 0 <= c < n_colors <= 16384
 * (the per-patch node counts of patchy.py:293-300 / the LPT weights) */
int phj_count_labels(const int32_t* color, int64_t n, int32_t n_colors,
                     unsigned long long* counts, void* stream);
int phj_assemble_finish(const phj_grid* g, int32_t* color, uint8_t* boundary, int16_t* lab,
                        int32_t* counters, void* stream);

/* node classification for analytic targets/obstacles: kind per serial */
typedef struct phj_shapes {
  int32_t n_balls;
  const double* balls; /* host: [n][5] centre[3], radius, ncomp (leading coords) */
  int32_t n_planes;
  const double* planes; /* host: [n][3] axis, offset, tol */
  int32_t n_obst_circles;
  const double* obst_circles; /* host: [n][5] cx, cy, cz, r, ncomp */
  int32_t n_obst_boxes;
  const double* obst_boxes; /* host: [n][7] ncomp, lo[3], hi[3] */
} phj_shapes;
int phj_classify(const phj_grid* g, const phj_shapes* shapes, const int32_t* user_axis,
                 int8_t* kind, void* stream);

/* per-node coefficient: h = k / speed (REF) or beta = exp(-h) (KRUZKOV);
 * speed from an analytic model or a per-serial array; < eps => -1. */
typedef struct phj_speed_model {
  int32_t kind;     /* 0 constant, 1 array, 2 sin-product: c0 + amp * prod sin(w x_ax) */
  double c0;
  double amp;
  double omega[3];  /* per user axis, 0 => factor omitted */
  double ctrl_norm; /* |a| of the (unit) control set */
  double eps;       /* degeneracy threshold on |f| */
  const double* speed; /* kind 1: per internal serial, device */
} phj_speed_model;
int phj_node_coef(const phj_grid* g, const phj_speed_model* m, const int32_t* user_axis,
                  int32_t dtype, int32_t rule, void* coef, void* stream);

/* field init/merge: v = target ? 0 : unreached everywhere (ghosts included) */
int phj_init_field(const phj_grid* g, int32_t dtype, const int8_t* kind, double unreached,
                   void* v, void* stream);
/* T <-> Kruzkov v conversions over a whole ext array (n entries) */
int phj_to_kruzkov(int64_t n, int32_t dtype, const double* T, void* v, double half_sentinel,
                   void* stream);
int phj_from_kruzkov(int64_t n, int32_t dtype, const void* v, double* T, double sentinel,
                     void* stream);
/* copy interior ghost layers for periodic axes; elem_bytes = bytes per node
 * (1, 2, 4, 8, or a multiple of 8 for node-major multi-value fields) */
int phj_sync_periodic(const phj_grid* g, int32_t elem_bytes, void* v, void* stream);

/* E1/Einf partial sums: out[0]=sum|a-b|, out[1]=max, out[2]=compared count */
int phj_error_partials(int64_t n, const double* a, const double* b, double half_a,
                       double half_b, double* out, void* stream);

/* FP64/FP32 pipe peak microbenchmark: flops executed into out[0] */
int phj_peak_flops(int32_t dtype, int32_t iters, double* sink, void* stream);

const char* phj_last_error(void);
int phj_num_sms(void);
/* number of kernels this library has launched in the process (bench evidence) */
unsigned long long phj_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PHJ_H */
