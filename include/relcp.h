/*
 * relcp.h -- C ABI of the B200-native ReLCP hot path (arXiv 2506.14097,
 * "Smooth-Rigid-Body Contact as a ReLCP", Palmer, Aktulga, Gao).
 *
 * Library: paper_2506_14097_b200/lib/librelcp.so (CUDA, sm_100a, fp64).
 *
 * Citations: P:Lnnn = line of the paper text with the section /
 * equation in parentheses; R<k> = reading k in DESIGN.md §2.
 *
 * Conventions (all calls):
 *   - every call returns an int status: RELCP_OK (0), an error (< 0) or a
 *     warning (> 0).  relcp_last_error(ctx) holds a one-line message.
 *   - every array in relcp_bodies / relcp_constraints is a CALLER-OWNED
 *     DEVICE pointer (cudaMalloc / torch CUDA tensor), fp64 unless noted,
 *     contiguous, in the layout stated beside it.  The library never
 *     allocates or frees caller-visible memory; it owns only its internal
 *     workspace (cell list, candidate pairs, body-major CSR of D, per-body
 *     mobility blocks, reduction partials), freed by relcp_destroy.
 *   - all device work is enqueued on the stream given to relcp_create.
 *     Calls whose OUTPUT SIZE is data dependent (generate, check/augment,
 *     step) or that report a host-visible result (solve) synchronise that
 *     stream before returning; relcp_delassus_apply / relcp_wrench do not.
 *   - there is no CPU fallback: without a CUDA device every call that does
 *     work returns RELCP_E_CUDA.
 *   - results are bitwise deterministic run to run (no floating-point
 *     atomics; every reduction has a fixed order).
 *
 * Notation (§2.1.1, P:L151-157 Eq. collision_ft):
 *   body b: centre x_b, unit quaternion (s, w), velocity U = (u, w).
 *   constraint alpha between bodies a = ia < b = ib: outward unit normal n of
 *   a, lever arms r_a = y_a - x_a, r_b = y_b - x_b at the shared-normal points
 *   y_a, y_b, torque arms t_a = r_a x n, t_b = r_b x n.
 *   Row of D^T: [-n, -t_a, n, t_b]   (App. A23; Phi_dot)
 *   Column of D: wrench -[n; t_a] on a, +[n; t_b] on b (F_a = -n gamma,
 *   T_a = -(y_a - x_a) x n gamma).
 *   W_b: M_b^{-1} (inertial) or the local-drag mobility
 *   (overdamped, Eq. ellipsoid_mobility), frozen at C^k.
 *   A = s D^T W D, s = dt^2 (inertial) or dt (overdamped).
 *   LCP: 0 <= g = A lambda + q  _|_  lambda >= 0 (Lemma 3; the
 *   paper writes b = -q).
 */
#ifndef RELCP_H
#define RELCP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define RELCP_OK 0
#define RELCP_E_ARG (-1)        /* bad argument (NULL pointer, size, param)  */
#define RELCP_E_CUDA (-2)       /* CUDA error or no device                   */
#define RELCP_E_CAPACITY (-3)   /* constraint store too small; see required  */
#define RELCP_E_DEGENERATE (-4) /* coincident body centres in a pair (R4)    */
#define RELCP_E_NAN (-5)        /* NaN/Inf in the LCP iterate                */
#define RELCP_E_STATE (-6)      /* call order violated (e.g. no operator)    */
#define RELCP_W_MAX_ITER 1      /* LCP stopped at lcp_max_iter, converged=0  */
#define RELCP_W_RECURSION_CAP 2 /* ReLCP stopped at max_recursions (R15)     */
#define RELCP_W_SNSD_NONCONV 3  /* some SNSD Newton solves not certified     */

#define RELCP_INERTIAL 0   /* U+ = U + dt M^-1 F  (Eq. law_inertia)   */
#define RELCP_OVERDAMPED 1 /* U = M F, local drag (Eq. law_overdamped) */

#define RELCP_MAX_REC 64 /* size of the per-recursion arrays in the step report */

typedef struct relcp_ctx relcp_ctx;

/* Parameters.  relcp_default_params fills the values in brackets. */
typedef struct relcp_params {
    int32_t dynamics;     /* RELCP_INERTIAL | RELCP_OVERDAMPED [INERTIAL]          */
    int32_t max_recursions; /* ReLCP recursion cap [50] (R15)                      */
    double dt;            /* time step [1e-3]                                      */
    double eps_ncp;       /* overlap tolerance, absolute [1e-5] (R3)       */
    double cutoff;        /* SNSD cutoff for A_0 [0.1] (R5)         */
    double lcp_tol;       /* residual tol, r = ||min(lambda, g)||_inf [1e-8] (R2)  */
    int64_t lcp_max_iter; /* [100000]                                              */
    int32_t check_every;  /* LCP iterations between host convergence reads [32]    */
    int32_t power_iters;  /* power iterations for L, alpha_0 = 1/L [20] (R1)       */
    double box[3];        /* periodic box lengths; 0 = that axis not periodic [0]  */
    double xi;            /* drag coefficient (overdamped) [1.0]          */
    int32_t n_dirs;       /* SNSD multistart sample size for overlaps [256] (R4)   */
    int32_t solver;       /* RELCP_SOLVER_BB [default] | RELCP_SOLVER_APGD         */
    int32_t reorder;      /* relcp_step's internal body order: RELCP_REORDER_OFF,
                             _AUTO [default: from RELCP_REORDER_MIN_BODIES bodies,
                             when fewer than RELCP_REORDER_COHERENT of the
                             consecutive caller bodies (b, b+1) lie in the same
                             or adjacent cells], _ON (see relcp_step)              */
    int32_t layout;       /* operator layout of the LCP solve: RELCP_LAYOUT_CSR |
                             RELCP_LAYOUT_JDS | RELCP_LAYOUT_AUTO [default: JDS
                             for RELCP_LAYOUT_JDS_MIN_BODIES <= N and
                             N_C <= RELCP_LAYOUT_JDS_MAX_ROWS, else CSR].  JDS
                             needs a store sorted by ia and rows with
                             t . n ~ 0 (else CSR).  Results agree to rounding
                             (DESIGN.md §5). */
    int32_t cluster;      /* BB solves of small stores (N <= 8192 bodies,
                             N_C <= 16384 rows, CSR layout) run the whole
                             iteration loop in one 16-CTA thread-block cluster
                             (DESIGN.md §5 "small stores") [1]; 0 = per-pass
                             kernels.  Same iterates up to rounding.          */
    int32_t snsd_cert;    /* ellipsoid SNSD: accept a certified Newton maximum
                             of an overlapping pair without the multistart
                             when its depth is below half the smallest radius
                             of curvature of A + B (curvature certificate,
                             DESIGN.md R29) [1]; 0 = always multistart.      */
    int32_t k6_pipe;      /* 1: K6 of sorted CSR stores from 65,536 bodies runs
                             the TMA-staged pipeline over per-group records
                             (k6pipe.cuh; bitwise equal to the per-warp kernel,
                             measured 3.1x slower) [0]          */
    int32_t k6_bpw;       /* bodies per warp of the CSR K6 on sorted stores:
                             0 = auto [default: RELCP_K6_BPW_SMALL for N <=
                             RELCP_K6_SMALL_N bodies, else 32], or 8 / 16 / 32.
                             Each body's summation order does not depend on it
                             (bitwise identical results).      */
} relcp_params;

#define RELCP_K6_SMALL_N 65536
#define RELCP_K6_BPW_SMALL 8

#define RELCP_REORDER_OFF 0
#define RELCP_REORDER_AUTO 1
#define RELCP_REORDER_ON 2
#define RELCP_REORDER_MIN_BODIES 65536
#define RELCP_REORDER_COHERENT 0.5

/* Operator layout (params.layout; DESIGN.md §5 "K6 layouts").  CSR: K6 reads
 * the a-side rows in the store's order through shared-memory tiles and the
 * b-side entries from a CSR copy.  JDS: op_prepare permutes the rows of every
 * 32-body group into a per-warp jagged-diagonal order (lanes sorted by
 * degree, column j = every lane's j-th row); the solve runs on a private copy
 * in that order (ids, compact rows, q, lambda, g) and writes lambda and g
 * back in the caller's row order; K6 streams whole columns and sums them
 * from shared memory without bank conflicts.  Measured equal in time to CSR
 * at cfg5 and cfg4 (HBM-streaming stores: +-1 %), 12 % faster per iteration
 * at cfg3 (431k rows, an L2-sized store), 45 % slower at cfg2 (20k bodies,
 * skewed degrees), with ~20 % less DRAM traffic (profiles/README.md): AUTO
 * picks JDS in the mid regime only.  The fused APGD solver always uses CSR. */
#define RELCP_LAYOUT_CSR 0
#define RELCP_LAYOUT_JDS 1
#define RELCP_LAYOUT_AUTO 2
#define RELCP_LAYOUT_JDS_MIN_BODIES 65536
#define RELCP_LAYOUT_JDS_MAX_ROWS 2097152

/* LCP solvers (the paper names only the family; reading R1):
 *   BB   Barzilai-Borwein projected gradient (alternating BB1 / BB2 steps);
 *   APGD Nesterov-accelerated projected gradient, step 1/(1.1 L), gradient
 *        adaptive restart.  Same kernels and bytes per iteration (+2 vectors).
 *   APGD_FUSED  the same APGD iterates with one fewer pass over the a-side
 *        rows: the row pass also takes the projected step and forms the
 *        a-side wrench sums of the next iterate, the scatter adds the b-side
 *        (fewer bytes per iteration).  Needs the library's sorted store order
 *        (plain APGD otherwise). */
#define RELCP_SOLVER_BB 0
#define RELCP_SOLVER_APGD 1
#define RELCP_SOLVER_APGD_FUSED 2

/* Body view (SoA by field, each field row-major per body).
 *   pos         (n,3)  centre x_b                                  in/out (step)
 *   quat        (n,4)  unit quaternion (s, wx, wy, wz), P:L66      in/out (step)
 *   axes        (n,3)  semi-axes (e1, e2, e3) in the body frame    in
 *   vel         (n,6)  (u, omega), world frame; may be NULL for
 *                      overdamped bodies                           in/out (step)
 *   inv_mass    (n)    1/m   (inertial; may be NULL if overdamped) in
 *   inv_inertia (n,3)  1/I_k, principal body-frame (inertial)      in
 *   kinematic   (n) int32, 1 = prescribed velocity (W_b = 0); NULL = none
 *   shape       (n) int32, RELCP_SHAPE_ELLIPSOID (axes = semi-axes) or
 *               RELCP_SHAPE_SPHEROCYLINDER (axes[0] = half the centreline
 *               length l/2 along body x, axes[1] = cap radius r; SNSD =
 *               segment distance minus radii; drag length l + 2r);
 *               or RELCP_SHAPE_TORUS (axes[0] = major radius R of the
 *               centreline circle in the body x-y plane, axes[1] = minor radius
 *               r; SNSD = centreline-circle distance minus radii, P:L1080;
 *               drag length 2 (R + r));
 *               NULL = all ellipsoids.  Mixed-shape pairs are not defined by
 *               the paper: E_DEGENERATE. */
#define RELCP_SHAPE_ELLIPSOID 0
#define RELCP_SHAPE_SPHEROCYLINDER 1
#define RELCP_SHAPE_TORUS 2
typedef struct relcp_bodies {
    int64_t n;
    double *pos;
    double *quat;
    const double *axes;
    double *vel;
    const double *inv_mass;
    const double *inv_inertia;
    const int32_t *kinematic;
    const int32_t *shape;
} relcp_bodies;

/* Constraint store: SoA, append-only within a step (App. D1).
 *   count        host-side element count (in/out; library updates it).
 *   ia, ib, gen  (capacity) int32: body ids (ia < ib) and the recursion index
 *                that appended the row (0 = A_0).  Rows the library writes
 *                (generate, check/augment, step) keep the whole store sorted
 *                by (ia, ib, gen) (R18) provided the rows already present are
 *                (ia, ib)-sorted; a store in another order is appended to
 *                unchanged (every call accepts any row order).
 *   n, ta, tb    (3, capacity) planes: component k of row alpha at
 *                [k*capacity + alpha]; unit normal n, torque arms t_a, t_b
 *                frozen at the discovery configuration (R9).
 *   phi          (capacity) signed distance at the discovery configuration.
 *   q            (capacity) LCP right-hand side (q = -b).
 *   lambda       (capacity) multipliers gamma (in: warm start; out: solution).
 *   g            (capacity) gap g = A lambda + q written by the solver; may be
 *                NULL for calls that do not solve. */
typedef struct relcp_constraints {
    int64_t capacity;
    int64_t count;
    int32_t *ia, *ib, *gen;
    double *n, *ta, *tb;
    double *phi, *q, *lambda, *g;
} relcp_constraints;

typedef struct relcp_solve_report {
    int64_t iterations; /* BB projected-gradient iterations (R1)             */
    double residual;    /* ||min(lambda, g)||_inf at exit (R2)                */
    int32_t converged;  /* residual <= lcp_tol                                */
    int32_t pad;
    double objective;   /* f = -1/2 lambda^T A lambda          */
    double L;           /* power-iteration estimate of ||A||_2                 */
} relcp_solve_report;

typedef struct relcp_step_report {
    int32_t recursions;                 /* augmentations performed (n of Alg. 1) */
    int32_t status;                     /* 0 | RELCP_W_RECURSION_CAP             */
    int64_t n_pairs;                    /* candidate pairs at the final margin   */
    double margin;                      /* final broadphase margin (R7)          */
    double max_overlap;                 /* max(0, -min Phi) at the accepted C    */
    int64_t n_c[RELCP_MAX_REC];         /* N_C of LCP n                          */
    int64_t lcp_iters[RELCP_MAX_REC];   /* iterations of LCP n                   */
    double residual[RELCP_MAX_REC];     /* residual of LCP n                     */
    double f_n[RELCP_MAX_REC];          /* f_n = -1/2 x^T A_n x        */
    double ms_generate, ms_solve, ms_check; /* wall time per phase (events)      */
    int64_t snsd_nonconv;               /* SNSD solves not certified (all calls) */
    int64_t n_guard;                    /* pairs of this step's SNSD scans with   */
                                        /* |Phi - threshold| < 1e-10 (cutoff at   */
                                        /* generation, -eps_ncp at checks): the   */
                                        /* R14 guard band, where another correct  */
                                        /* fp64 code may decide the other way     */
} relcp_step_report;

/* ---------------------------------------------------------------- context */

/* Fill *p with the defaults listed in relcp_params. */
void relcp_default_params(relcp_params *p);

/* Create a context bound to `cuda_stream` (a cudaStream_t; NULL = legacy
 * default stream).  Errors: E_ARG (p NULL or invalid), E_CUDA. */
int relcp_create(relcp_ctx **out, const relcp_params *p, void *cuda_stream);
int relcp_destroy(relcp_ctx *ctx);
const char *relcp_last_error(const relcp_ctx *ctx);
/* Replace the parameters (e.g. dt or box between steps). */
int relcp_set_params(relcp_ctx *ctx, const relcp_params *p);

/* ------------------------------------------------------------- hot path */

/* a1-a3: broadphase (cell list, candidate pairs with
 *   |x_b - x_a|_min-image < R_a + R_b + cutoff, R = largest semi-axis;
 *   "near-contacting pairs"), SNSD of every pair at the
 *   bodies' configuration (definition R4), and the A_0 rows
 *   of pairs with Phi < cutoff (R5), appended in (ia, ib) order with gen = 0,
 *   lambda = 0 and q = Phi + dt row.U_free, U_free = vel (inertial,
 *   P:L557-561; F_ext = 0 here) or 0 (overdamped).
 *   The store is RESET (count = 0) first.  *n_out = rows written.
 *   Keeps the candidate pairs, W and U_free in the context for
 *   relcp_check_and_augment.  Synchronises once.
 * Errors: E_CAPACITY (cs->count = required rows, nothing written),
 *   E_DEGENERATE; warning W_SNSD_NONCONV. */
int relcp_generate_contacts(relcp_ctx *ctx, const relcp_bodies *bodies, relcp_constraints *cs,
                            int64_t *n_out);

/* Load a GIVEN constraint network (e.g. BASELINE cfg4's chainmail links)
 * into the store, replacing its content: m rows with body ids ia < ib,
 * normals n and lever arms ra = y_a - x_a, rb = y_b - x_b as (3, m) planes,
 * gaps phi (m); all caller-owned device arrays.  Forms t_a = ra x n,
 * t_b = rb x n, q = phi + dt row.U_free with U_free = vel
 * (inertial, F_ext = 0) or 0 (overdamped), lambda = 0,
 * gen = 0, in the given row order (rows sorted by (ia, ib) take the fast
 * operator path).  Errors: E_ARG, E_CAPACITY (cs->count = m). */
int relcp_load_constraints(relcp_ctx *ctx, const relcp_bodies *bodies, relcp_constraints *cs, int64_t m,
                           const int32_t *ia, const int32_t *ib, const double *n, const double *ra,
                           const double *rb, const double *phi);

/* Build the operator for the current store: per-body W blocks at the bodies'
 * configuration (frozen C^k) and the body-major CSR of D.  Must be called
 * again after the caller edits ia/ib/n/ta/tb/count.  Generate, solve,
 * check/augment and step (re)build it themselves. */
int relcp_prepare_operator(relcp_ctx *ctx, const relcp_bodies *bodies, const relcp_constraints *cs);

/* a5: y = scale * D^T W D x for the prepared operator (P:L154-157, P:L207-211,
 * P:L627).  x, y: device, length cs->count (may not alias).  Asynchronous.
 * Errors: E_ARG, E_STATE (operator not prepared for this count). */
int relcp_delassus_apply(relcp_ctx *ctx, const relcp_bodies *bodies, const relcp_constraints *cs,
                         const double *x, double *y, double scale);

/* Body wrench F = D x and velocity U = W D x, (n,6) each, either may be NULL.
 * Asynchronous.  Errors as relcp_delassus_apply. */
int relcp_wrench(relcp_ctx *ctx, const relcp_bodies *bodies, const relcp_constraints *cs,
                 const double *x, double *F, double *U);

/* a6: solve 0 <= A lambda + q _|_ lambda >= 0 in place (Lemma 3, P:L280-299;
 * Barzilai-Borwein projected gradient, R1).  lambda in = warm start
 * (projected onto lambda >= 0), out = solution; cs->g = A lambda + q.
 * Prepares the operator if needed.  Synchronises once per check_every
 * iterations.  Warning W_MAX_ITER (last iterate returned); error E_NAN. */
int relcp_solve_lcp(relcp_ctx *ctx, const relcp_bodies *bodies, relcp_constraints *cs,
                    relcp_solve_report *rep);

/* a7-a8: trial configuration C_{n+1} = C^k + dt G^k U_tot, U_tot = U_free +
 * sigma W D lambda (sigma = dt inertial, 1 overdamped, R6),
 * SNSD of the context's candidate pairs at C_{n+1} (margin widened per R7),
 * and append of every pair with Phi < -eps_ncp (R10) with gen =
 * `recursion`, geometry frozen at C_{n+1} (R9), lambda = 0 and
 * q = Phi - s row.(W D lambda) (Thm 1 RHS b_n = A_n iota(x_{n-1}) - g~,
 * P:L587; retained q unchanged).  *n_appended = 0 <=> stopping rule
 * (P:L646-648).  *min_phi = min Phi over the pairs at C_{n+1}.
 * `Ck` = the bodies at the start of the step (unchanged).  Requires a prior
 * relcp_generate_contacts on the same bodies.  Synchronises.
 * Errors: E_STATE, E_CAPACITY (cs->count = required rows), E_DEGENERATE. */
int relcp_check_and_augment(relcp_ctx *ctx, const relcp_bodies *Ck, relcp_constraints *cs,
                            int32_t recursion, int64_t *n_appended, double *min_phi);

/* One ReLCP time step: Algorithm 1, inertial form Eq.
 * relcp_inertial.  f_ext: (n,6) device or NULL (= 0).  Updates
 * pos (wrapped into the periodic box), quat (normalised) and vel in place:
 * C^{k+1} = accepted trial configuration, U^{k+1} = U_free + sigma W D lambda.
 * `scratch` is the constraint store used for the step (its final content is
 * the step's A_c, rows (ia < ib) sorted by (ia, ib, gen), R18).  Warning
 * W_RECURSION_CAP (the last trial configuration is accepted and flagged).
 * Internal body order (params.reorder): the step may run on a
 * relabelled copy of the bodies in spatial cell order (cells ~ the mean
 * spacing, row-major, ties by caller id) and of the store, so that the
 * operator's gathers stay local whatever order the caller keeps its bodies in;
 * labels are arbitrary, and the results are translated back (ids,
 * rows re-oriented to ia < ib with n' = -n, t_a' = -t_b, t_b' = -t_a, sorted)
 * before return.  Extra device memory: one more store of scratch->capacity
 * rows and a copy of the body arrays.  After a reordered step, relcp_get_pairs
 * returns the step's pairs in caller ids (i < j) in internal order and
 * relcp_check_and_augment needs a new relcp_generate_contacts. */
int relcp_step(relcp_ctx *ctx, relcp_bodies *inout, const double *f_ext, relcp_constraints *scratch,
               relcp_step_report *rep);

/* Candidate pairs currently held by the context (after generate / augment):
 * *n_pairs = count; if pi/pj non-NULL (device, capacity cap) they receive the
 * pairs in (i, j) lexicographic order (after a reordered relcp_step: caller
 * ids with i < j, in the internal order).  Synchronises. */
int relcp_get_pairs(relcp_ctx *ctx, int32_t *pi, int32_t *pj, int64_t cap, int64_t *n_pairs);

/* Counters kept by the context since creation / the last reset:
 *   launches          kernels this context launched (all entry points)
 *   lcp_iterations    BB iterations executed (K6 scatter + K7 gather pairs)
 * and, when timing is on (relcp_set_timing(ctx, 1)), CUDA-event durations on
 * the context stream:
 *   iter_ms / iter_timed    summed duration / count of the timed LCP
 *                           iterations: the first batch of each solve (direct
 *                           launches, events around each kernel) and every
 *                           CUDA-graph batch that ran all its iterations
 *                           (events around the graph launch);
 *   scatter_ms / gather_ms  summed K6 / K7 (or fused row pass / b-side scatter)
 *                           durations over the split_timed iterations of the
 *                           direct batches;
 *   n_guard                 SNSD-scanned pairs inside the R14 guard band
 *                           |Phi - threshold| < 1e-10 (generation: cutoff;
 *                           checks: -eps_ncp), over every generate / check
 *                           since the reset (timing off or on);
 *   jds_solves              LCP solves run on the JDS operator layout since
 *                           the reset (params.layout);
 *   op_layout               layout of the operator prepared last
 *                           (RELCP_LAYOUT_CSR or RELCP_LAYOUT_JDS);
 *   cluster_solves          BB solves run by the single-cluster loop
 *                           (params.cluster) since the reset;
 *   snsd_multistart         ellipsoid pairs that went to the SNSD multistart
 *                           (overlapping, not certified by R29) since the
 *                           reset. */
typedef struct relcp_stats {
    int64_t launches;
    int64_t lcp_iterations;
    int64_t iter_timed;
    double scatter_ms;
    double gather_ms;
    int64_t split_timed;
    double iter_ms;
    int64_t n_guard;
    int64_t jds_solves;
    int32_t op_layout;
    int32_t pad;
    int64_t cluster_solves;
    int64_t snsd_multistart;
} relcp_stats;
int relcp_get_stats(relcp_ctx *ctx, relcp_stats *out);
int relcp_reset_stats(relcp_ctx *ctx);
int relcp_set_timing(relcp_ctx *ctx, int32_t on);

/* SNSD of explicit pairs (device arrays, length n_pairs) at the given bodies:
 * phi (P), nrm (3,P) planes, ra (3,P), rb (3,P) planes (r = y - x), status
 * (P) int32 0 ok / 1 coincident centres / 2 not certified.  Asynchronous. */
int relcp_snsd_pairs(relcp_ctx *ctx, const relcp_bodies *bodies, int64_t n_pairs, const int32_t *pi,
                     const int32_t *pj, double *phi, double *nrm, double *ra, double *rb, int32_t *status);

/* ------------------------------------------------ domain decomposition
 * SURVEY §8(e) / §8(f) rank 4 (the paper's solver is distributed over spatial
 * domains with MPI).  Bodies are split into K contiguous index ranges
 * [part_off[k], part_off[k+1]) (part_off[0] = 0, part_off[K] = n); constraint
 * alpha belongs to the part owning ia (rows must be sorted by ia, R18, so a
 * part's rows are one contiguous range [row_lo, row_hi)); a part's ghosts are
 * the ib of its rows owned elsewhere.  Per apply / BB iteration the ghost
 * partial wrenches go to their owners, which add them in ascending part order
 * (deterministic, no atomics) before applying W, and the owners' U go back to
 * the ghost slots (48 B per boundary body and direction); the BB dot products
 * and residual are combined over the parts (fixed part order, or one grouped
 * NCCL all-reduce of <= 6 doubles).  DESIGN.md §8. */
typedef struct relcp_dd relcp_dd;
typedef struct relcp_dd_info {
    int64_t n_own;      /* owned bodies                                   */
    int64_t n_ghost;    /* ghost bodies (ib of owned rows owned elsewhere) */
    int64_t row_lo, row_hi; /* owned rows of the ia-sorted store          */
    int64_t n_recv;     /* halo slots received (ghost partials of others) */
    int64_t n_boundary; /* owned bodies that receive halo partials        */
} relcp_dd_info;

/* Host-only partition plan of part `part` (no device needed): info, and when
 * non-NULL ghost[n_ghost] (global ids, ascending), gseg[K+1] (ghost segment of
 * each owner part), rseg[K+1] (receive-slot segment of each source part),
 * recv_list[n_recv] (owned local id of each receive slot; the slots of source
 * p hold p's ghosts owned here, in p's ghost order).  ia/ib: host arrays.
 * Errors: E_ARG (bad offsets, rows not sorted by ia, ia == ib, ids out of range). */
int relcp_dd_plan_host(int32_t nparts, const int64_t *part_off, int64_t nc, const int32_t *ia, const int32_t *ib,
                       int32_t part, relcp_dd_info *info, int64_t *ghost, int64_t *gseg, int64_t *rseg,
                       int32_t *recv_list);
/* 128-byte NCCL unique id for relcp_dd_create in NCCL mode (rank 0 makes it,
 * the caller broadcasts it).  E_CUDA if libnccl.so.2 cannot be loaded. */
int relcp_dd_nccl_unique_id(void *out128);
/* rank < 0: VIRTUAL mode, all K parts in this process on this device (halo
 * exchange by device copies).  rank >= 0: NCCL mode, this process holds part
 * `rank` of K ranks (one GPU each; nccl_uid from relcp_dd_nccl_unique_id). */
int relcp_dd_create(relcp_dd **out, const relcp_params *p, void *cuda_stream, int32_t nparts,
                    const int64_t *part_off, int32_t rank, const void *nccl_uid);
int relcp_dd_destroy(relcp_dd *dd);
const char *relcp_dd_last_error(const relcp_dd *dd);
/* Partition (bodies, constraints) -- global device arrays as in relcp_prepare_
 * operator; the store must stay in place (q / lambda / g are used through
 * views) until the next load.  Synchronises. */
int relcp_dd_load(relcp_dd *dd, const relcp_bodies *bodies, const relcp_constraints *cs);
int relcp_dd_info_get(relcp_dd *dd, int32_t part, relcp_dd_info *info);
/* y = scale D^T W D x over the parts (x, y: device, global row order; NCCL
 * mode writes this rank's rows only).  Asynchronous. */
int relcp_dd_delassus_apply(relcp_dd *dd, const double *x, double *y, double scale);
/* U (n, 6) of the owned bodies of the local parts after the last apply /
 * solve, into a global (n, 6) device array.  Asynchronous. */
int relcp_dd_get_u(relcp_dd *dd, double *U);
/* relcp_solve_lcp over the parts (BB, same parameters); cs = the loaded store.
 * Returns OK, W_MAX_ITER or E_NAN like relcp_solve_lcp.  Synchronises. */
int relcp_dd_solve_lcp(relcp_dd *dd, relcp_constraints *cs, relcp_solve_report *rep);
/* One ReLCP step (Algorithm 1; same contract, report and codes as
 * relcp_step, in the caller's body order) whose LCP solves are the
 * domain-decomposed BB solve above on each recursion's store, and whose SNSD
 * phases (generation at C^k, every check at the trial configuration) are
 * split by the owner of i: each part scans the candidate pairs of its bodies.
 * The broadphase, trial configuration, q and the store merge are replicated
 * (every rank passes all bodies and the whole store and, after the exchanges,
 * holds the same store, in the single-domain row order).  NCCL: after each
 * SNSD phase the ranks all-reduce the counts and statistics and exchange their
 * appended rows; after each solve their rows' lambda and g (grouped send /
 * recv).  DESIGN.md §8. */
int relcp_dd_step(relcp_dd *dd, relcp_bodies *bodies, const double *f_ext, relcp_constraints *cs,
                  relcp_step_report *rep);

#ifdef __cplusplus
}
#endif
#endif /* RELCP_H */
