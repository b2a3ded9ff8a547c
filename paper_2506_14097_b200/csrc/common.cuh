// Internal header of librelcp.so (B200 / sm_100a, fp64).  Not part of the ABI.
// Citations: P:Lnnn = paper line; R<k> = DESIGN.md reading k.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>
#include <utility>

#include "../../include/relcp.h"

// Debug build only (-DRELCP_PHASE_TIMING, tools/phases.py): synchronise and
// print the host time since the previous mark.  Compiled out of librelcp.so.
#ifdef RELCP_PHASE_TIMING
#include <chrono>
inline std::chrono::steady_clock::time_point relcp_phase_last = std::chrono::steady_clock::now();  // one per .so
inline void relcp_phase_mark(cudaStream_t st, const char *name) {
    auto &last = relcp_phase_last;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[phase] %-24s %9.3f ms\n", name, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}
#define PHASE(ctx, name) relcp_phase_mark((ctx)->stream, name)
#else
#define PHASE(ctx, name) ((void)0)
#endif

#define RELCP_NT 256          // threads per block for streaming kernels
#define RELCP_SM_COUNT 148    // B200
#define RELCP_MAX_DIRS 1024   // cap on the SNSD start sample
// R14 guard band: pairs with |Phi - threshold| below this are counted (n_guard):
// two correct fp64 codes may decide them differently (R14)
#define RELCP_GUARD_BAND 1e-10

// ------------------------------------------------------------ device buffer
template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t cap = 0;  // elements
    cudaError_t grow(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = n + n / 4 + 64;
        cudaError_t e = cudaMalloc((void **)&p, want * sizeof(T));
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    void swap(DevBuf &o) {
        T *tp = p;
        p = o.p;
        o.p = tp;
        const size_t tc = cap;
        cap = o.cap;
        o.cap = tc;
    }
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }  // relcp_destroy's `delete ctx` frees every buffer
};

// Device-side state of one LCP solve (BB projected gradient, R1).
struct LcpState {
    double alpha;   // current step length
    double L;       // ||A|| estimate (power iteration)
    double resid;   // ||min(x, g)||_inf of the current iterate
    double ss, sy, yy;
    double obj;     // x^T (g - q) = x^T A x
    double pnorm;   // power iteration: scale applied to the input vector
    double tol;
    long long iter;     // completed iterations
    long long max_iter;
    int done;
    int conv;
    int nan;
    int par;        // APGD: 0 -> (x, g) current, 1 -> (xb, gb) current
    double theta;   // APGD momentum parameter
    double beta;    // APGD extrapolation weight for the next step
    double alpha_next;  // fused BB: step of the pass after the next (one-step delay)
    // BB nonmonotone safeguard (GLL / SPG line search, lcp.cu): the last
    // RELCP_GLL_M objective values f(x) = 1/2 x^T (g + q), the step t along
    // d = x+ - x of the last update and whether the current iterate is the
    // blend x + t d of the two slots (fix = 1) rather than the full step.
    double f_cur;
    double fhist[10];
    double t_ls;
    int fix;
    int n_ls;        // iterations whose full BB step the line search shortened
};
#define RELCP_GLL_M 10

// power iteration step (finalize of k_gather's ||A v||^2): L = ||A v||, the next
// input is scaled by 1/L
__device__ __forceinline__ void power_finalize(LcpState *st, const double *acc) {
    double nrm = sqrt(acc[0]);
    st->L = nrm;
    st->pnorm = nrm > 0.0 ? 1.0 / nrm : 0.0;
}

// Per-body mobility block W_b in a single 7-double form, stored as 7 SoA
// planes W[k * nb + b]:
//   U_lin = w[0] * F_lin ;  U_ang = S F_ang, S symmetric = {w1..w6} =
//   (xx, xy, xz, yy, yz, zz).  Inertial: w0 = 1/m, S = R I^-1 R^T;
//   overdamped local drag: w0 = 1/(xi L), S = 12/(xi L^3) I.
#define RELCP_WSTRIDE 7

struct relcp_ctx {
    relcp_params p;
    cudaStream_t stream;
    int own_stream = 0;  // created by relcp_create (caller passed the legacy stream)
    char err[512];

    // operator (prepared for `op_nc` rows and `op_nb` bodies)
    int64_t op_nc = -1, op_nb = -1;
    const void *op_key_ia = nullptr;
    int op_sorted = 0;               // store sorted by ia: a-side read from the store (K6)
    int64_t op_cap = 0;              // store plane stride
    const double *op_n = nullptr, *op_ta = nullptr;
    int64_t op_rs = 0;               // compact row plane stride (= op_nc)
    DevBuf<double> rc;               // (6, op_nc) compact rows (rows.cuh), for the row passes
    int op_compact = 0;              // every row has t . n ~ 0: row passes read rc
    DevBuf<int> pa;                  // (nb + 1) a-side row pointer of a sorted store
    DevBuf<int> mi;                  // merge scratch (3, rows)
    DevBuf<double> md;               // merge scratch (13, rows)
    DevBuf<double> W;        // (nb, 8)
    DevBuf<int> row_ptr;     // (nb + 1)
    DevBuf<int> deg;         // (nb)  scratch
    DevBuf<int> fill;        // (nb)  scratch
    DevBuf<int> ecid;        // (2 nc) constraint index of each half entry (body-major)
    DevBuf<double> ew;       // (6, 2 nc) signed wrench payload, body-major
    DevBuf<double> U;        // (nb, 6) U = W D x of the last scatter
    DevBuf<double> F;        // (nb, 6) scratch for relcp_wrench
    DevBuf<double> partials; // (blocks, 4)
    DevBuf<unsigned> counter;
    DevBuf<LcpState> st;
    DevBuf<double> vtmp;     // (nc) power iteration / apply scratch
    DevBuf<double> apgd_buf; // (2, nc) APGD second iterate (x', g'); fused BB: x'
    DevBuf<double> Fa;       // (6, nb) fused BB: a-side wrench sums of the next iterate
    // JDS operator layout (params.layout, operator.cu "JDS"): rows in slot order
    int op_jds = 0;          // the operator was prepared in the JDS layout
    int jds_enable = 1;      // 0: never (domain-decomposition part contexts)
    int64_t jds_solves = 0;  // solves on the JDS layout since the stats reset
    int64_t cluster_solves = 0;  // BB solves by the single-cluster loop since the reset
    int cl_ok = -1;          // cluster launch possible (-1: not probed yet)
    int pdl = 0;             // K6 / K7 launches with programmatic dependent launch (lcp.cu batches)
    int k6p_attr = 0;        // k_scatter_pipe's dynamic shared-memory limit set
    int op_k6r = 0;          // per-group K6 records built (k6pipe.cuh)
    DevBuf<long long> k6r_sz, k6r_off;  // (groups + 1) record sizes / offsets (bytes)
    DevBuf<unsigned char> k6r_rec;      // the records
    double L_reuse = 0.0;    // relcp_step: ||A|| of this step's previous LCP (0: none; R1)
    int64_t L_reuse_nc = 0;  // its row count
    DevBuf<long long> dstat; // (4) device-side counters: [0] SNSD multistart pairs
    DevBuf<int> jperm;       // (nc) slot -> store row
    DevBuf<int> jiperm;      // (nc) store row -> slot
    DevBuf<int> jameta;      // (32 nwarp) a-side lane -> degree << 5 | local body
    DevBuf<int> jbmeta;      // (32 nwarp) b-side lane -> degree << 5 | local body
    DevBuf<int> jbcid;       // (nc) b-side entry (JDS order) -> slot of its row
    DevBuf<double> jbpay;    // (4, nc) b-side entry compact payload (u, v, t_b,j1, t_b,j2)
    DevBuf<int> jia, jib;    // (nc) ids in slot order
    DevBuf<double> jq, jx, jg;  // (nc) q, lambda, g in slot order (the solve's private view)
    DevBuf<double> jtmp;     // (nc) slot-order copy of a caller's x (apply / wrench / check)
    DevBuf<double> rc2;      // (6, nc) permutation scratch for rc
    LcpState *st_host = nullptr;  // pinned mirror

    // step state (from generate_contacts at C^k)
    int64_t step_nb = -1;
    const double *step_pos_key = nullptr;
    DevBuf<int> pi, pj;      // candidate pairs
    int64_t npairs = 0;
    double margin = 0.0;
    DevBuf<double> Sig;      // (nb, 6) shape matrices at the config being tested
    DevBuf<double> ufree;    // (nb, 6)
    DevBuf<double> utot;     // (nb, 6)
    DevBuf<double> ptrial;   // (nb, 3)
    DevBuf<double> qtrial;   // (nb, 4)
    DevBuf<double> rad;      // (nb)
    // pair temporaries
    DevBuf<double> tphi, tn, tra, trb;  // (P), (3,P) planes
    DevBuf<int> tflag, tstat;
    DevBuf<int> multi;          // pairs needing the SNSD multistart (stage 2)
    DevBuf<int> nlist;          // ellipsoid pairs under the SNSD bound (Newton stage 1)
    DevBuf<double> dirs;        // (3, dirs_n) multistart directions (k_dirs)
    DevBuf<float> dirs32;       // the same, fp32 (stage-2 screening)
    int dirs_n = 0;
    DevBuf<long long> scan_ll;  // scan scratch
    DevBuf<long long> scan_tmp;
    DevBuf<int> cell_count, cell_start, cell_fill, cell_items, body_cell;
    DevBuf<long long> pair_cnt;  // per body pair counts (then offsets)
    int64_t pair_lo = 0, pair_n = -1;  // SNSD / append over pairs [pair_lo, pair_lo + pair_n) (-1: all)
    int bp_cap = 0;              // slot-row capacity of the single-pass broadphase (0: two-pass)
    DevBuf<int> bp_tmp;          // (nb, bp_cap) slot rows
    DevBuf<double> red;          // small reduction buffer
    double *red_host = nullptr;  // pinned (64 doubles)
    int64_t snsd_nonconv_total = 0;
    int64_t n_guard_total = 0;   // R14 guard-band pairs since the last reset

    // internal body order of relcp_step (order.cu)
    DevBuf<int> ord_perm, ord_inv, ord_cell, ord_cnt, ord_start, ord_key;
    DevBuf<double> ob_pos, ob_quat, ob_axes, ob_vel, ob_im, ob_ii, ob_fext;
    DevBuf<int> ob_kin, ob_shape;
    DevBuf<int> os_i;      // internal store ids (3, cap)
    DevBuf<double> os_d;   // internal store values (13, cap)
    int pairs_internal = 0;  // ctx->pi / pj hold internal ids (ord_perm maps them)

    // counters / timing (relcp_get_stats)
    int64_t launches = 0;
    int64_t lcp_iterations = 0;
    int timing = 0;
    int64_t iter_timed = 0, split_timed = 0;
    double scatter_ms = 0.0, gather_ms = 0.0, iter_ms = 0.0;
    cudaEvent_t ev[3 * 64 + 2] = {};  // per-kernel events of a direct batch + 2 around a graph launch
    int ev_ready = 0;
};

// ------------------------------------------------------------ error helpers
int set_err(relcp_ctx *c, int code, const char *fmt, ...);

#define CK(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess)                                                     \
            return set_err(ctx, RELCP_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, \
                           cudaGetErrorString(e_));                                \
    } while (0)

#define CKL()                                                                      \
    do {                                                                           \
        ++ctx->launches;                                                           \
        cudaError_t e_ = cudaGetLastError();                                       \
        if (e_ != cudaSuccess)                                                     \
            return set_err(ctx, RELCP_E_CUDA, "%s:%d launch: %s", __FILE__, __LINE__, \
                           cudaGetErrorString(e_));                                \
    } while (0)

#define CKS(expr)                  \
    do {                           \
        int s_ = (expr);           \
        if (s_ < 0) return s_;     \
    } while (0)

static inline int grid_for(int64_t n, int nt = RELCP_NT, int per_sm = 8) {
    int64_t g = (n + nt - 1) / nt;
    int64_t cap = (int64_t)RELCP_SM_COUNT * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ------------------------------------------------------------ programmatic dependent launch
// The LCP iteration kernels (K6, K7) are launched with programmatic stream
// serialisation when ctx->pdl is set (inside the solve's batches): the next
// kernel's CTAs are scheduled while the previous one drains, and wait in
// pdl_wait() (griddepcontrol.wait: the previous grid completed and its memory
// is visible) before touching its outputs; pdl_open() lets the next kernel be
// scheduled early.  Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_open() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_k(bool pdl, void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st,
                                   Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ internal API
// operator.cu
int op_prepare(relcp_ctx *ctx, const relcp_bodies *b, const relcp_constraints *cs);
int op_build_W(relcp_ctx *ctx, const relcp_bodies *b, double *W);
// scatter followed by W: U = W D x_eff; mode 0 x_eff = x, 1 BB projected step,
// 2 APGD projected step from (x, g) / (xb, gb) (device parity picks current)
// slots: x / g / xb / gb are in the JDS slot order (the solve's private view);
// otherwise (store order) a JDS operator first permutes x into slot order
int op_scatter(relcp_ctx *ctx, int64_t nb, const double *x, const double *g, int mode,
               const double *xscale_dev, double *U, double *F, const double *xb = nullptr,
               const double *gb = nullptr, int slots = 0);
// JDS operator: cs is either the solve's slot-order view (cs->ia == ctx->jia.p)
// or the caller's store (y is then written through the slot -> row permutation)
int op_gather_apply(relcp_ctx *ctx, const relcp_constraints *cs, const double *U, double *y, double scale,
                    int norm2, double *acc_out = nullptr);
// fused BB row pass (g_{k+1}, x_{k+2}, a-side sums Fa, BB reductions)
int op_fused_rows(relcp_ctx *ctx, const relcp_constraints *cs, int64_t nb, double s, double *xA, double *xB);int op_row_dot_U(relcp_ctx *ctx, const relcp_constraints *cs, int64_t begin, int64_t end, const double *U,
                 double coef, double *out_add);
// store.cu
int store_merge_appended(relcp_ctx *ctx, relcp_constraints *cs, int64_t n_old, int64_t m);
int store_is_sorted_by_ia(relcp_ctx *ctx, const relcp_constraints *cs, int *sorted_host);
// lcp.cu
int lcp_solve(relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs, relcp_solve_report *rep);
// abi.cu: Algorithm 1 (relcp_step without the internal body order) with the LCP
// solves delegated to `solve` (dd.cu relcp_dd_step)
typedef int (*relcp_solve_cb)(void *user, relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs,
                              relcp_solve_report *rep);
// Domain-decomposed SNSD of generation and checks (dd.cu relcp_dd_step): the
// candidate pairs (sorted by i) are split by the owner of i (body ranges
// off[0..K]); rank < 0: every part here, in part order (VIRTUAL); rank >= 0:
// this rank's part, then `reduce` sums / mins the statistics over the ranks
// (vals: [0..K) flagged rows per part (this rank's entry set, others 0), K: sum
// of degenerate pairs, K+1: non-certified, K+2: guard band, K+3: -min Phi) and
// `exchange` places every rank's appended rows at their offsets.
struct DistSpec {
    int K = 1;
    const int64_t *off = nullptr;
    int rank = -1;
    int (*reduce)(void *user, double *vals, int n) = nullptr;
    int (*exchange)(void *user, relcp_constraints *cs, int64_t base, const int64_t *cnt) = nullptr;
    void *user = nullptr;
};
int step_entry(relcp_ctx *ctx, relcp_bodies *b, const double *f_ext, relcp_constraints *cs, relcp_step_report *rep,
               relcp_solve_cb solve, void *user, const DistSpec *dist = nullptr);
// split-reduction pieces of the BB solve for the domain-decomposed solve (dd.cu):
// each writes its part's block-reduced partials to acc_out (device) instead of
// finalizing; lcp_dd_finalize applies the finalize step of `kind` to ctx->st
// from partials already combined over every part.
enum { DD_POWER = 0, DD_INIT = 1, DD_ITER = 2, DD_FINISH = 3, DD_OBJECTIVE = 4 };
int lcp_dd_nvals(int kind);                       // partials per kind
const int *lcp_dd_ops(int kind);                  // 0 sum, 1 max per partial
int lcp_dd_state_init(relcp_ctx *ctx, int64_t nc_global);
int lcp_dd_project_fill(relcp_ctx *ctx, int64_t nc, double *lambda, double *v, double val);
int lcp_dd_init(relcp_ctx *ctx, const relcp_constraints *cs, double s, double *acc_out);
int lcp_dd_iter(relcp_ctx *ctx, const relcp_constraints *cs, double s, double *xB, double *gB, double *acc_out);
int lcp_dd_finish(relcp_ctx *ctx, int64_t nc, double *x, double *g, const double *xo, const double *go,
                  double *acc_out);
int lcp_dd_objective(relcp_ctx *ctx, int64_t nc, const double *x, const double *g, const double *q,
                     double *acc_out);
int lcp_dd_finalize(relcp_ctx *ctx, int kind, const double *acc_dev);
double lcp_scale(const relcp_ctx *ctx);
// order.cu (relcp_step's internal body order)
int ord_body_perm(relcp_ctx *ctx, int64_t nb, const double *pos, double *coherent);
int ord_bodies_in(relcp_ctx *ctx, const relcp_bodies *b, const double *f_ext, relcp_bodies *bi,
                  const double **f_ext_i);
int ord_bodies_out(relcp_ctx *ctx, const relcp_bodies *bi, relcp_bodies *b);
int ord_store(relcp_ctx *ctx, const relcp_constraints *cs, relcp_constraints *ci);
int ord_store_out(relcp_ctx *ctx, int64_t nb, const relcp_constraints *ci, relcp_constraints *cs);
int ord_pairs_out(relcp_ctx *ctx, int64_t np, int32_t *oi, int32_t *oj);
// scan.cu
int scan_exclusive_ll(relcp_ctx *ctx, const long long *in, long long *out, int64_t n, long long *total_host);
int scan_exclusive_int(relcp_ctx *ctx, const int *in, int *out, int64_t n, int *total_host);
// geometry.cu
int geo_shape_matrices(relcp_ctx *ctx, int64_t nb, const double *quat, const double *axes, const int32_t *shape,
                       double *Sig);
int geo_broadphase(relcp_ctx *ctx, int64_t nb, const double *pos, const double *rad, double margin);
// reject_above: pairs whose rigorous lower bound Phi >= F(d/|d|) reaches it are
// not solved (status 3, phi = the bound); +INFINITY = solve every pair.
int geo_snsd(relcp_ctx *ctx, int64_t np, const int *pi, const int *pj, const double *pos, const double *Sig,
             double *phi, double *nrm, double *ra, double *rb, int *status, int64_t planes, double reject_above,
             const int32_t *shape, const double *axes);
