// C ABI entry points (include/relcp.h) and the ReLCP step orchestration
// (Algorithm 1; inertial form Eq. relcp_inertial).
#include <chrono>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: phase ranges for Nsight timelines

#include <vector>

#include "common.cuh"
#include "reduce.cuh"

int set_err(relcp_ctx *c, int code, const char *fmt, ...) {
    if (c) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(c->err, sizeof(c->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

static double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

static int check_params(const relcp_params *p) {
    if (!p) return 0;
    if (p->dynamics != RELCP_INERTIAL && p->dynamics != RELCP_OVERDAMPED) return 0;
    if (!(p->dt > 0.0) || !(p->eps_ncp >= 0.0) || !(p->cutoff >= 0.0) || !(p->lcp_tol > 0.0)) return 0;
    if (p->max_recursions < 0 || p->max_recursions > RELCP_MAX_REC - 1) return 0;
    for (int k = 0; k < 3; ++k)
        if (!(p->box[k] >= 0.0)) return 0;
    if (p->dynamics == RELCP_OVERDAMPED && !(p->xi > 0.0)) return 0;
    if (p->solver != RELCP_SOLVER_BB && p->solver != RELCP_SOLVER_APGD && p->solver != RELCP_SOLVER_APGD_FUSED)
        return 0;
    if (p->reorder < RELCP_REORDER_OFF || p->reorder > RELCP_REORDER_ON) return 0;
    if (p->layout < RELCP_LAYOUT_CSR || p->layout > RELCP_LAYOUT_AUTO) return 0;
    if (p->k6_bpw != 0 && p->k6_bpw != 8 && p->k6_bpw != 16 && p->k6_bpw != 32) return 0;
    return 1;
}

// ------------------------------------------------------------ body kernels
// bounding radius: largest semi-axis (ellipsoid) or half-length + radius (rod)
__global__ void k_radius(int64_t nb, const double *__restrict__ axes, const int32_t *__restrict__ shape,
                         double *__restrict__ rad) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        rad[b] = (shape && (shape[b] == RELCP_SHAPE_SPHEROCYLINDER || shape[b] == RELCP_SHAPE_TORUS))
                     ? axes[3 * b] + axes[3 * b + 1]
                     : fmax(axes[3 * b], fmax(axes[3 * b + 1], axes[3 * b + 2]));
}

// U_free = U^k + dt M^-1 F_ext (inertial, kinematic: U^k) or
// M F_ext (overdamped).  W is the (nb, 8) block array.
__global__ void k_ufree(int64_t nb, int dyn, double dt, const double *__restrict__ vel,
                        const double *__restrict__ fext, const double *__restrict__ W,
                        const int32_t *__restrict__ kin, double *__restrict__ uf) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        double w[7];
        for (int k = 0; k < 7; ++k) w[k] = W[k * nb + b];  // SoA planes
        double f[6] = {0, 0, 0, 0, 0, 0};
        if (fext)
            for (int k = 0; k < 6; ++k) f[k] = fext[6 * b + k];
        double wf[6] = {w[0] * f[0], w[0] * f[1], w[0] * f[2], w[1] * f[3] + w[2] * f[4] + w[3] * f[5],
                        w[2] * f[3] + w[4] * f[4] + w[5] * f[5], w[3] * f[3] + w[5] * f[4] + w[6] * f[5]};
        const bool k = kin && kin[b] != 0;
        for (int c = 0; c < 6; ++c) {
            double v = vel ? vel[6 * b + c] : 0.0;
            uf[6 * b + c] = dyn == RELCP_INERTIAL ? (k ? v : v + dt * wf[c]) : wf[c];
        }
    }
}

// Trial configuration C_{n+1} = C^k + dt G^k U_tot, U_tot = U_free + sigma Uc
// (R6): x += dt u, q += dt/2 (0, omega) (x) q^k.  Also the
// largest centre displacement (for the margin rule R7) in part/out.
__global__ void __launch_bounds__(RELCP_NT) k_trial(int64_t nb, double dt, double sigma,
                                                    const double *__restrict__ pos, const double *__restrict__ quat,
                                                    const double *__restrict__ uf, const double *__restrict__ Uc,
                                                    double *__restrict__ utot, double *__restrict__ pt,
                                                    double *__restrict__ qt, double *part, unsigned *counter,
                                                    double *out) {
    __shared__ double sh[32];
    double acc[1] = {0.0};
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        double u[6];
        for (int c = 0; c < 6; ++c) {
            u[c] = uf[6 * b + c] + sigma * Uc[6 * b + c];
            utot[6 * b + c] = u[c];
        }
        double d2 = 0.0;
        for (int c = 0; c < 3; ++c) {
            double dx = dt * u[c];
            pt[3 * b + c] = pos[3 * b + c] + dx;
            d2 += dx * dx;
        }
        const double s = quat[4 * b], x = quat[4 * b + 1], y = quat[4 * b + 2], z = quat[4 * b + 3];
        const double wx = u[3], wy = u[4], wz = u[5];
        // (0, w) (x) (s, v) = (-w.v, s w + w x v)
        qt[4 * b] = s + 0.5 * dt * (-(wx * x + wy * y + wz * z));
        qt[4 * b + 1] = x + 0.5 * dt * (s * wx + (wy * z - wz * y));
        qt[4 * b + 2] = y + 0.5 * dt * (s * wy + (wz * x - wx * z));
        qt[4 * b + 3] = z + 0.5 * dt * (s * wz + (wx * y - wy * x));
        acc[0] = fmax(acc[0], d2);
    }
    const int ops[1] = {1};
    if (grid_reduce_last<1>(acc, ops, part, counter, sh) && threadIdx.x == 0) out[0] = sqrt(acc[0]);
}

// Accept C^{k+1} = C_{n+1}: wrap positions into the periodic box
// (every axis with box[c] > 0),
// normalise quaternions, U^{k+1} = U_tot.
__global__ void k_accept(int64_t nb, double bx, double by, double bz, const double *__restrict__ pt,
                         const double *__restrict__ qt, const double *__restrict__ utot, double *pos, double *quat,
                         double *vel) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const double bxs[3] = {bx, by, bz};
        for (int c = 0; c < 3; ++c) {  // each periodic axis separately (box[c] > 0)
            double v = pt[3 * b + c];
            if (bxs[c] > 0.0) v -= bxs[c] * floor(v / bxs[c]);
            pos[3 * b + c] = v;
        }
        double s = qt[4 * b], x = qt[4 * b + 1], y = qt[4 * b + 2], z = qt[4 * b + 3];
        double inv = 1.0 / sqrt(s * s + x * x + y * y + z * z);
        quat[4 * b] = s * inv;
        quat[4 * b + 1] = x * inv;
        quat[4 * b + 2] = y * inv;
        quat[4 * b + 3] = z * inv;
        if (vel)
            for (int c = 0; c < 6; ++c) vel[6 * b + c] = utot[6 * b + c];
    }
}

// ------------------------------------------------------------ pair kernels
// flag[k] = keep pair k; counts of degenerate / non-certified pairs, min phi, and
// the pairs inside the R14 guard band |Phi - thresh| < RELCP_GUARD_BAND.
__global__ void __launch_bounds__(RELCP_NT) k_flag(int64_t np, const double *__restrict__ phi,
                                                   const int *__restrict__ stat, double thresh, int *__restrict__ flag,
                                                   double *part, unsigned *counter, double *out) {
    __shared__ double sh[4 * 32];
    double acc[4] = {0.0, 0.0, INFINITY, 0.0};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < np; k += (int64_t)gridDim.x * blockDim.x) {
        const int s = stat[k];
        const double f = phi[k];
        flag[k] = (s != 1 && f < thresh) ? 1 : 0;
        acc[0] += s == 1 ? 1.0 : 0.0;
        acc[1] += s == 2 ? 1.0 : 0.0;
        if (s != 1) acc[2] = fmin(acc[2], f);
        // R14 guard band: a decision another correct fp64 code may take the other way
        if (s != 1 && fabs(f - thresh) < RELCP_GUARD_BAND) acc[3] += 1.0;
    }
    const int ops[4] = {0, 0, 2, 0};
    if (grid_reduce_last<4>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        out[0] = acc[0];
        out[1] = acc[1];
        out[2] = acc[2];
        out[3] = acc[3];
    }
}

// Order-preserving append of flagged pairs at rows base + offset[k]:
// t_a = r_a x n, t_b = r_b x n, lambda = 0, q = phi.
__global__ void k_append(int64_t np, const int *__restrict__ flag, const int *__restrict__ off,
                         const int *__restrict__ pi, const int *__restrict__ pj, const double *__restrict__ phi,
                         const double *__restrict__ nrm, const double *__restrict__ ra, const double *__restrict__ rb,
                         int64_t planes, int64_t base, int gen, int64_t cap, int32_t *ia, int32_t *ib, int32_t *gv,
                         double *n, double *ta, double *tb, double *phio, double *q, double *lam) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < np; k += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[k]) continue;
        const int64_t a = base + off[k];
        const double nx = nrm[k], ny = nrm[planes + k], nz = nrm[2 * planes + k];
        const double ax = ra[k], ay = ra[planes + k], az = ra[2 * planes + k];
        const double bx = rb[k], by = rb[planes + k], bz = rb[2 * planes + k];
        ia[a] = pi[k];
        ib[a] = pj[k];
        gv[a] = gen;
        n[a] = nx; n[cap + a] = ny; n[2 * cap + a] = nz;
        ta[a] = ay * nz - az * ny; ta[cap + a] = az * nx - ax * nz; ta[2 * cap + a] = ax * ny - ay * nx;
        tb[a] = by * nz - bz * ny; tb[cap + a] = bz * nx - bx * nz; tb[2 * cap + a] = bx * ny - by * nx;
        phio[a] = phi[k];
        q[a] = phi[k];
        lam[a] = 0.0;
    }
}

// Given rows (relcp_load_constraints): t = r x n, q = phi, lambda = 0, gen = 0.
__global__ void k_load_rows(int64_t m, const int32_t *__restrict__ ia_in, const int32_t *__restrict__ ib_in,
                            const double *__restrict__ nrm, const double *__restrict__ ra,
                            const double *__restrict__ rb, const double *__restrict__ phi, int64_t cap, int32_t *ia,
                            int32_t *ib, int32_t *gv, double *n, double *ta, double *tb, double *phio, double *q,
                            double *lam) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        const double nx = nrm[k], ny = nrm[m + k], nz = nrm[2 * m + k];
        const double ax = ra[k], ay = ra[m + k], az = ra[2 * m + k];
        const double bx = rb[k], by = rb[m + k], bz = rb[2 * m + k];
        ia[k] = ia_in[k];
        ib[k] = ib_in[k];
        gv[k] = 0;
        n[k] = nx; n[cap + k] = ny; n[2 * cap + k] = nz;
        ta[k] = ay * nz - az * ny; ta[cap + k] = az * nx - ax * nz; ta[2 * cap + k] = ax * ny - ay * nx;
        tb[k] = by * nz - bz * ny; tb[cap + k] = bz * nx - bx * nz; tb[2 * cap + k] = bx * ny - by * nx;
        phio[k] = phi[k];
        q[k] = phi[k];
        lam[k] = 0.0;
    }
}

// ------------------------------------------------------------ helpers
static int ensure_common(relcp_ctx *ctx, int64_t nb) {
    CK(ctx->Sig.grow(6 * nb));
    CK(ctx->ufree.grow(6 * nb));
    CK(ctx->utot.grow(6 * nb));
    CK(ctx->ptrial.grow(3 * nb));
    CK(ctx->qtrial.grow(4 * nb));
    CK(ctx->rad.grow(nb));
    CK(ctx->W.grow(RELCP_WSTRIDE * nb));
    CK(ctx->U.grow(6 * nb));
    return RELCP_OK;
}

static int check_views(relcp_ctx *ctx, const relcp_bodies *b, const relcp_constraints *cs) {
    if (!ctx) return RELCP_E_ARG;
    if (!b || b->n <= 0 || !b->pos || !b->quat || !b->axes)
        return set_err(ctx, RELCP_E_ARG, "bodies: n > 0, pos, quat and axes are required");
    if (b->n >= (1ll << 31)) return set_err(ctx, RELCP_E_ARG, "bodies: n must fit int32");
    if (!cs || !cs->ia || !cs->ib || !cs->gen || !cs->n || !cs->ta || !cs->tb || !cs->phi || !cs->q || !cs->lambda ||
        cs->capacity < 0 || cs->count < 0 || cs->count > cs->capacity)
        return set_err(ctx, RELCP_E_ARG, "constraints: every array and 0 <= count <= capacity are required");
    return RELCP_OK;
}

static int grow_pair_tmp(relcp_ctx *ctx, int64_t np) {
    int64_t m = np > 0 ? np : 1;
    CK(ctx->tphi.grow(m));
    CK(ctx->tn.grow(3 * m));
    CK(ctx->tra.grow(3 * m));
    CK(ctx->trb.grow(3 * m));
    CK(ctx->tflag.grow(m + 1));
    CK(ctx->tstat.grow(m));
    CK(ctx->scan_ll.grow(m + 1));
    return RELCP_OK;
}

// SNSD over the context's pairs at (pos, Sig); flag Phi < thresh; scan.
// Returns the number of flagged pairs in *nflag, min phi, counts.
static int snsd_flag_scan(relcp_ctx *ctx, const double *pos, const int32_t *shape, const double *axes,
                          double thresh, int *nflag, double *minphi, int64_t *ndegen, int64_t *nnonconv) {
    const int64_t p0 = ctx->pair_lo, np = ctx->pair_n >= 0 ? ctx->pair_n : ctx->npairs;
    CKS(grow_pair_tmp(ctx, np));
    *nflag = 0;
    *minphi = INFINITY;
    *ndegen = 0;
    *nnonconv = 0;
    if (np == 0) return RELCP_OK;
    if (np >= (1ll << 31) - 1) return set_err(ctx, RELCP_E_ARG, "too many candidate pairs");
    // pairs whose lower bound Phi >= F(d/|d|) is >= max(thresh, 0) can neither be
    // flagged nor lower min(Phi) below 0: they are not solved (status 3)
    CKS(geo_snsd(ctx, np, ctx->pi.p + p0, ctx->pj.p + p0, pos, ctx->Sig.p, ctx->tphi.p, ctx->tn.p, ctx->tra.p,
                 ctx->trb.p, ctx->tstat.p, np, thresh > 0.0 ? thresh : 0.0, shape, axes));
    PHASE(ctx, "snsd.kernels");
    k_flag<<<grid_for(np), RELCP_NT, 0, ctx->stream>>>(np, ctx->tphi.p, ctx->tstat.p, thresh, ctx->tflag.p,
                                                       ctx->partials.p, ctx->counter.p, ctx->red.p);
    CKL();
    int *off = (int *)ctx->scan_ll.p;
    CK(cudaMemsetAsync(ctx->tflag.p + np, 0, sizeof(int), ctx->stream));
    int total = 0;
    CKS(scan_exclusive_int(ctx, ctx->tflag.p, off, np + 1, &total));  // syncs
    CK(cudaMemcpyAsync(ctx->red_host, ctx->red.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *nflag = total;
    *ndegen = (int64_t)ctx->red_host[0];
    *nnonconv = (int64_t)ctx->red_host[1];
    *minphi = ctx->red_host[2];
    ctx->n_guard_total += (int64_t)ctx->red_host[3];
    PHASE(ctx, "snsd.flag_scan");
    return RELCP_OK;
}

static int append_flagged(relcp_ctx *ctx, relcp_constraints *cs, int gen, int64_t nflag) {
    const int64_t p0 = ctx->pair_lo, np = ctx->pair_n >= 0 ? ctx->pair_n : ctx->npairs;
    if (nflag == 0) return RELCP_OK;
    int *off = (int *)ctx->scan_ll.p;
    k_append<<<grid_for(np), RELCP_NT, 0, ctx->stream>>>(np, ctx->tflag.p, off, ctx->pi.p + p0, ctx->pj.p + p0, ctx->tphi.p,
                                                         ctx->tn.p, ctx->tra.p, ctx->trb.p, np, cs->count, gen,
                                                         cs->capacity, cs->ia, cs->ib, cs->gen, cs->n, cs->ta, cs->tb,
                                                         cs->phi, cs->q, cs->lambda);
    CKL();
    return RELCP_OK;
}

static double op_s(const relcp_ctx *ctx) {
    return ctx->p.dynamics == RELCP_INERTIAL ? ctx->p.dt * ctx->p.dt : ctx->p.dt;
}
static double op_sigma(const relcp_ctx *ctx) { return ctx->p.dynamics == RELCP_INERTIAL ? ctx->p.dt : 1.0; }

// first pair of every part: pairs are sorted by i, part k owns i in [off[k], off[k+1])
__global__ void k_pair_bounds(int64_t np, const int *__restrict__ pi, int K, const int64_t *__restrict__ off,
                              long long *__restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > K) return;
    const int64_t key = off[k];
    int64_t lo = 0, hi = np;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)pi[mid] < key) lo = mid + 1; else hi = mid;
    }
    out[k] = lo;
}

// SNSD + flag (+ append when `append`) over the candidate pairs, whole or split
// over the parts of `ds` (DistSpec); the appended rows of all parts land at
// cs->count in part order (the single-domain order: pairs sorted by i), and
// cs->count advances by the total.  Returns the statistics of all parts.
static int flag_append(relcp_ctx *ctx, const double *pos, const int32_t *shape, const double *axes, double thresh,
                       relcp_constraints *cs, int gen, bool append, const DistSpec *ds, int64_t *nflag_out,
                       double *minphi_out, int64_t *ndeg_out, int64_t *nnc_out) {
    if (!ds || ds->K <= 1) {
        ctx->pair_lo = 0;
        ctx->pair_n = -1;
        int nflag;
        CKS(snsd_flag_scan(ctx, pos, shape, axes, thresh, &nflag, minphi_out, ndeg_out, nnc_out));
        *nflag_out = nflag;
        if (append && nflag > 0 && *ndeg_out == 0 && cs->count + nflag <= cs->capacity) {
            CKS(append_flagged(ctx, cs, gen, nflag));
            cs->count += nflag;
        }
        return RELCP_OK;
    }
    const int K = ds->K;
    std::vector<long long> pb(K + 1);
    {
        DevBuf<int64_t> doff;
        DevBuf<long long> dpb;
        CK(doff.grow(K + 1));
        CK(dpb.grow(K + 1));
        CK(cudaMemcpyAsync(doff.p, ds->off, sizeof(int64_t) * (K + 1), cudaMemcpyHostToDevice, ctx->stream));
        k_pair_bounds<<<1, 64 * ((K + 64) / 64), 0, ctx->stream>>>(ctx->npairs, ctx->pi.p, K, doff.p, dpb.p);
        CKL();
        CK(cudaMemcpyAsync(pb.data(), dpb.p, sizeof(long long) * (K + 1), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    std::vector<double> vals(K + 4, 0.0);
    vals[K + 3] = -INFINITY;  // -min Phi
    const int64_t guard0 = ctx->n_guard_total;
    std::vector<int64_t> cnt(K, 0);
    const int64_t base = cs->count;
    int64_t placed = 0;
    for (int k = 0; k < K; ++k) {
        if (ds->rank >= 0 && k != ds->rank) continue;
        ctx->pair_lo = pb[k];
        ctx->pair_n = pb[k + 1] - pb[k];
        int nflag;
        double mp;
        int64_t nd, nn;
        CKS(snsd_flag_scan(ctx, pos, shape, axes, thresh, &nflag, &mp, &nd, &nn));
        cnt[k] = nflag;
        vals[k] = nflag;
        vals[K] += nd;
        vals[K + 1] += nn;
        vals[K + 3] = fmax(vals[K + 3], -mp);
        // VIRTUAL: append each part at once, in part order (the next part's scan reuses the temporaries)
        if (ds->rank < 0 && append && nflag > 0 && nd == 0 && base + placed + nflag <= cs->capacity) {
            cs->count = base + placed;
            CKS(append_flagged(ctx, cs, gen, nflag));
        }
        placed += nflag;
    }
    vals[K + 2] = (double)(ctx->n_guard_total - guard0);
    ctx->n_guard_total = guard0;
    if (ds->rank >= 0 && ds->reduce) CKS(ds->reduce(ds->user, vals.data(), K + 4));
    int64_t total = 0;
    for (int k = 0; k < K; ++k) total += (int64_t)vals[k];
    *nflag_out = total;
    *ndeg_out = (int64_t)vals[K];
    *nnc_out = (int64_t)vals[K + 1];
    ctx->n_guard_total += (int64_t)vals[K + 2];
    *minphi_out = -vals[K + 3];
    cs->count = base;
    if (append && total > 0 && *ndeg_out == 0 && base + total <= cs->capacity) {
        if (ds->rank >= 0) {  // this rank's rows at their offset, then every rank's rows everywhere
            int64_t pre = 0;
            for (int k = 0; k < ds->rank; ++k) pre += (int64_t)vals[k];
            cs->count = base + pre;
            CKS(append_flagged(ctx, cs, gen, (int64_t)vals[ds->rank]));
            for (int k = 0; k < K; ++k) cnt[k] = (int64_t)vals[k];
            cs->count = base;
            if (ds->exchange) CKS(ds->exchange(ds->user, cs, base, cnt.data()));
        }
        cs->count = base + total;
    }
    ctx->pair_lo = 0;
    ctx->pair_n = -1;
    return RELCP_OK;
}

// a1-a3 with a given U_free (device, nb x 6) already in ctx->ufree.
static int generate_impl(relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs, int64_t *n_out,
                         const DistSpec *ds = nullptr) {
    const int64_t nb = b->n;
    CKS(ensure_common(ctx, nb));
    k_radius<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, b->axes, b->shape, ctx->rad.p);
    CKL();
    CKS(geo_shape_matrices(ctx, nb, b->quat, b->axes, b->shape, ctx->Sig.p));
    PHASE(ctx, "gen.shape");
    ctx->margin = ctx->p.cutoff > 0.0 ? ctx->p.cutoff : 1e-3;
    CKS(geo_broadphase(ctx, nb, b->pos, ctx->rad.p, ctx->margin));
    PHASE(ctx, "gen.broadphase");
    int64_t nflag;
    double minphi;
    int64_t ndeg, nnc;
    cs->count = 0;
    CKS(flag_append(ctx, b->pos, b->shape, b->axes, ctx->p.cutoff, cs, 0, true, ds, &nflag, &minphi, &ndeg, &nnc));
    ctx->step_nb = nb;
    ctx->step_pos_key = b->pos;
    ctx->op_nc = -1;
    ctx->snsd_nonconv_total += nnc;
    if (ndeg > 0) return set_err(ctx, RELCP_E_DEGENERATE, "generate: %lld pairs with coincident centres", (long long)ndeg);
    if (nflag > cs->capacity) {
        cs->count = nflag;
        return set_err(ctx, RELCP_E_CAPACITY, "generate: %lld rows needed, capacity %lld", (long long)nflag,
                       (long long)cs->capacity);
    }
    cs->count = nflag;
    // q_0 = Phi_0 + dt row . U_free   (Phi~_0)
    CKS(op_row_dot_U(ctx, cs, 0, nflag, ctx->ufree.p, ctx->p.dt, cs->q));
    if (n_out) *n_out = nflag;
    CK(cudaStreamSynchronize(ctx->stream));
    PHASE(ctx, "gen.append");
    return nnc > 0 ? RELCP_W_SNSD_NONCONV : RELCP_OK;
}

// a7-a8 for the current store; Uc = W D lambda computed here.
static int check_impl(relcp_ctx *ctx, const relcp_bodies *Ck, relcp_constraints *cs, int gen, int allow_append,
                      int64_t *n_app, double *min_phi, const DistSpec *ds = nullptr) {
    const int64_t nb = Ck->n;
    if (ctx->step_nb != nb || ctx->step_pos_key != Ck->pos)
        return set_err(ctx, RELCP_E_STATE, "check_and_augment: call relcp_generate_contacts on these bodies first");
    PHASE(ctx, "chk.enter");
    if (ctx->op_nc != cs->count || ctx->op_nb != nb || ctx->op_key_ia != cs->ia) CKS(op_prepare(ctx, Ck, cs));
    PHASE(ctx, "chk.prepare");
    // Uc = W D lambda
    if (cs->count > 0)
        CKS(op_scatter(ctx, nb, cs->lambda, nullptr, 0, nullptr, ctx->U.p, nullptr));
    else
        CK(cudaMemsetAsync(ctx->U.p, 0, sizeof(double) * 6 * nb, ctx->stream));
    k_trial<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, ctx->p.dt, op_sigma(ctx), Ck->pos, Ck->quat, ctx->ufree.p,
                                                        ctx->U.p, ctx->utot.p, ctx->ptrial.p, ctx->qtrial.p,
                                                        ctx->partials.p, ctx->counter.p, ctx->red.p);
    CKL();
    CK(cudaMemcpyAsync(ctx->red_host, ctx->red.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const double delta = ctx->red_host[0];
    PHASE(ctx, "chk.scatter_trial");
    if (!isfinite(delta))
        return set_err(ctx, RELCP_E_NAN, "check: non-finite trial displacement (velocities or multipliers)");
    // R7: widen the candidate margin until it exceeds the largest approach 2 delta
    double m = ctx->margin;
    while (m <= 2.0 * delta) m *= 2.0;
    if (m != ctx->margin) {
        ctx->margin = m;
        CKS(geo_broadphase(ctx, nb, Ck->pos, ctx->rad.p, m));
    }
    PHASE(ctx, "chk.broadphase");
    CKS(geo_shape_matrices(ctx, nb, ctx->qtrial.p, Ck->axes, Ck->shape, ctx->Sig.p));
    PHASE(ctx, "chk.shape");
    int64_t nflag;
    double minphi;
    int64_t ndeg, nnc;
    const int64_t base = cs->count;
    CKS(flag_append(ctx, ctx->ptrial.p, Ck->shape, Ck->axes, -ctx->p.eps_ncp, cs, gen, allow_append != 0, ds, &nflag,
                    &minphi, &ndeg, &nnc));
    ctx->snsd_nonconv_total += nnc;
    if (min_phi) *min_phi = minphi;
    if (n_app) *n_app = nflag;
    if (ndeg > 0) return set_err(ctx, RELCP_E_DEGENERATE, "check: %lld pairs with coincident centres", (long long)ndeg);
    if (!allow_append || nflag == 0) return nnc > 0 ? RELCP_W_SNSD_NONCONV : RELCP_OK;
    if (base + nflag > cs->capacity) {
        cs->count = base + nflag;
        return set_err(ctx, RELCP_E_CAPACITY, "augment: %lld rows needed, capacity %lld", (long long)cs->count,
                       (long long)cs->capacity);
    }
    PHASE(ctx, "chk.append");
    // q_new = Phi(C_n) - s row . (W D lambda)   (b_n = A_n iota(x) - Phi~)
    CKS(op_row_dot_U(ctx, cs, base, base + nflag, ctx->U.p, -op_s(ctx), cs->q));
    // keep the store sorted by (ia, ib, gen) (R18): stable merge of the new block
    PHASE(ctx, "chk.rowdot");
    CKS(store_merge_appended(ctx, cs, base, nflag));
    ctx->op_nc = -1;
    CK(cudaStreamSynchronize(ctx->stream));
    PHASE(ctx, "chk.merge");
    return nnc > 0 ? RELCP_W_SNSD_NONCONV : RELCP_OK;
}

// ------------------------------------------------------------ ABI
extern "C" {

void relcp_default_params(relcp_params *p) {
    if (!p) return;
    memset(p, 0, sizeof(*p));
    p->dynamics = RELCP_INERTIAL;
    p->max_recursions = 50;
    p->dt = 1e-3;
    p->eps_ncp = 1e-5;
    p->cutoff = 0.1;
    p->lcp_tol = 1e-8;
    p->lcp_max_iter = 100000;
    p->check_every = 32;
    p->power_iters = 20;
    p->xi = 1.0;
    p->n_dirs = 256;
    p->reorder = RELCP_REORDER_AUTO;
    p->layout = RELCP_LAYOUT_AUTO;
    p->cluster = 1;
    p->snsd_cert = 1;
    p->k6_pipe = 0;
    p->k6_bpw = 0;
}

int relcp_create(relcp_ctx **out, const relcp_params *p, void *cuda_stream) {
    if (!out) return RELCP_E_ARG;
    *out = nullptr;
    if (!check_params(p)) return RELCP_E_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return RELCP_E_CUDA;
    }
    relcp_ctx *ctx = new relcp_ctx();
    ctx->p = *p;
    ctx->stream = (cudaStream_t)cuda_stream;
    if (!ctx->stream) {
        // the legacy default stream cannot be captured into CUDA graphs: use an
        // own BLOCKING stream (implicitly ordered with the legacy stream)
        if (cudaStreamCreate(&ctx->stream) != cudaSuccess) {
            delete ctx;
            return RELCP_E_CUDA;
        }
        ctx->own_stream = 1;
    }
    ctx->err[0] = 0;
    auto fail = [&](int code) {
        relcp_destroy(ctx);
        return code;
    };
    if (ctx->partials.grow(8 * 4096) != cudaSuccess || ctx->counter.grow(4) != cudaSuccess ||
        ctx->st.grow(1) != cudaSuccess || ctx->red.grow(64) != cudaSuccess)
        return fail(RELCP_E_CUDA);
    if (cudaMallocHost((void **)&ctx->st_host, sizeof(LcpState)) != cudaSuccess) return fail(RELCP_E_CUDA);
    if (cudaMallocHost((void **)&ctx->red_host, 64 * sizeof(double)) != cudaSuccess) return fail(RELCP_E_CUDA);
    if (cudaMemset(ctx->counter.p, 0, ctx->counter.cap * sizeof(unsigned)) != cudaSuccess) return fail(RELCP_E_CUDA);
    if (cudaMemset(ctx->st.p, 0, sizeof(LcpState)) != cudaSuccess) return fail(RELCP_E_CUDA);
    *out = ctx;
    return RELCP_OK;
}

int relcp_destroy(relcp_ctx *ctx) {
    if (!ctx) return RELCP_OK;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ctx->W.release(); ctx->row_ptr.release(); ctx->deg.release(); ctx->fill.release();
    ctx->ecid.release(); ctx->ew.release(); ctx->U.release(); ctx->F.release();
    ctx->partials.release(); ctx->counter.release(); ctx->st.release(); ctx->vtmp.release();
    ctx->pi.release(); ctx->pj.release(); ctx->Sig.release(); ctx->ufree.release(); ctx->utot.release();
    ctx->ptrial.release(); ctx->qtrial.release(); ctx->rad.release();
    ctx->tphi.release(); ctx->tn.release(); ctx->tra.release(); ctx->trb.release();
    ctx->tflag.release(); ctx->tstat.release(); ctx->scan_ll.release(); ctx->scan_tmp.release();
    ctx->cell_count.release(); ctx->cell_start.release(); ctx->cell_fill.release(); ctx->cell_items.release();
    ctx->body_cell.release(); ctx->pair_cnt.release(); ctx->red.release();
    ctx->ord_perm.release(); ctx->ord_inv.release(); ctx->ord_cell.release(); ctx->ord_cnt.release();
    ctx->ord_start.release(); ctx->ord_key.release(); ctx->ob_pos.release(); ctx->ob_quat.release();
    ctx->ob_axes.release(); ctx->ob_vel.release(); ctx->ob_im.release(); ctx->ob_ii.release(); ctx->ob_fext.release();
    ctx->ob_kin.release(); ctx->ob_shape.release(); ctx->os_i.release(); ctx->os_d.release();
    if (ctx->ev_ready)
        for (int k = 0; k < 3 * 64 + 2; ++k) cudaEventDestroy(ctx->ev[k]);
    if (ctx->st_host) cudaFreeHost(ctx->st_host);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->red_host) cudaFreeHost(ctx->red_host);
    delete ctx;
    return RELCP_OK;
}

const char *relcp_last_error(const relcp_ctx *ctx) { return ctx ? ctx->err : "null context"; }

int relcp_set_params(relcp_ctx *ctx, const relcp_params *p) {
    if (!ctx) return RELCP_E_ARG;
    if (!check_params(p)) return set_err(ctx, RELCP_E_ARG, "set_params: invalid parameters");
    ctx->p = *p;
    ctx->op_nc = -1;
    return RELCP_OK;
}

int relcp_generate_contacts(relcp_ctx *ctx, const relcp_bodies *bodies, relcp_constraints *cs, int64_t *n_out) {
    CKS(check_views(ctx, bodies, cs));
    ctx->pairs_internal = 0;
    const int64_t nb = bodies->n;
    CKS(ensure_common(ctx, nb));
    if (ctx->p.dynamics == RELCP_INERTIAL && !bodies->vel)
        return set_err(ctx, RELCP_E_ARG, "generate: inertial dynamics needs vel");
    CKS(op_build_W(ctx, bodies, ctx->W.p));
    k_ufree<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, ctx->p.dynamics, ctx->p.dt, bodies->vel, nullptr,
                                                        ctx->W.p, bodies->kinematic, ctx->ufree.p);
    CKL();
    return generate_impl(ctx, bodies, cs, n_out);
}

int relcp_load_constraints(relcp_ctx *ctx, const relcp_bodies *bodies, relcp_constraints *cs, int64_t m,
                           const int32_t *ia, const int32_t *ib, const double *n, const double *ra,
                           const double *rb, const double *phi) {
    CKS(check_views(ctx, bodies, cs));
    if (m < 0 || (m > 0 && (!ia || !ib || !n || !ra || !rb || !phi)))
        return set_err(ctx, RELCP_E_ARG, "load_constraints: m >= 0 and all row arrays required");
    if (m > cs->capacity) {
        cs->count = m;
        return set_err(ctx, RELCP_E_CAPACITY, "load_constraints: %lld rows, capacity %lld", (long long)m,
                       (long long)cs->capacity);
    }
    if (ctx->p.dynamics == RELCP_INERTIAL && !bodies->vel)
        return set_err(ctx, RELCP_E_ARG, "load_constraints: inertial dynamics needs vel");
    const int64_t nb = bodies->n;
    CKS(ensure_common(ctx, nb));
    CKS(op_build_W(ctx, bodies, ctx->W.p));
    k_ufree<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, ctx->p.dynamics, ctx->p.dt, bodies->vel, nullptr,
                                                        ctx->W.p, bodies->kinematic, ctx->ufree.p);
    CKL();
    if (m > 0) {
        k_load_rows<<<grid_for(m), RELCP_NT, 0, ctx->stream>>>(m, ia, ib, n, ra, rb, phi, cs->capacity, cs->ia, cs->ib,
                                                               cs->gen, cs->n, cs->ta, cs->tb, cs->phi, cs->q,
                                                               cs->lambda);
        CKL();
    }
    cs->count = m;
    CKS(op_row_dot_U(ctx, cs, 0, m, ctx->ufree.p, ctx->p.dt, cs->q));  // q = Phi_0 + dt row.U_free
    ctx->op_nc = -1;
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

int relcp_prepare_operator(relcp_ctx *ctx, const relcp_bodies *bodies, const relcp_constraints *cs) {
    if (!ctx) return RELCP_E_ARG;
    if (!bodies || bodies->n <= 0 || !cs || cs->count < 0 || cs->count > cs->capacity || !cs->ia || !cs->ib ||
        !cs->n || !cs->ta || !cs->tb)
        return set_err(ctx, RELCP_E_ARG, "prepare: bad views");
    CKS(op_prepare(ctx, bodies, cs));
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

static int op_ready(relcp_ctx *ctx, const relcp_bodies *b, const relcp_constraints *cs) {
    if (!b || !cs) return set_err(ctx, RELCP_E_ARG, "null view");
    if (ctx->op_nc != cs->count || ctx->op_nb != b->n || ctx->op_key_ia != cs->ia)
        return set_err(ctx, RELCP_E_STATE, "operator not prepared for this store (call relcp_prepare_operator)");
    return RELCP_OK;
}

int relcp_delassus_apply(relcp_ctx *ctx, const relcp_bodies *bodies, const relcp_constraints *cs, const double *x,
                         double *y, double scale) {
    if (!ctx) return RELCP_E_ARG;
    CKS(op_ready(ctx, bodies, cs));
    if (cs->count > 0 && (!x || !y || x == y)) return set_err(ctx, RELCP_E_ARG, "apply: x, y required and distinct");
    if (cs->count == 0) return RELCP_OK;
    CKS(op_scatter(ctx, bodies->n, x, nullptr, 0, nullptr, ctx->U.p, nullptr));
    CKS(op_gather_apply(ctx, cs, ctx->U.p, y, scale, 0));
    return RELCP_OK;
}

int relcp_wrench(relcp_ctx *ctx, const relcp_bodies *bodies, const relcp_constraints *cs, const double *x, double *F,
                 double *U) {
    if (!ctx) return RELCP_E_ARG;
    CKS(op_ready(ctx, bodies, cs));
    const int64_t nb = bodies->n;
    CK(ctx->F.grow(6 * nb));
    if (cs->count == 0) {
        if (F) CK(cudaMemsetAsync(F, 0, sizeof(double) * 6 * nb, ctx->stream));
        if (U) CK(cudaMemsetAsync(U, 0, sizeof(double) * 6 * nb, ctx->stream));
        return RELCP_OK;
    }
    if (!x) return set_err(ctx, RELCP_E_ARG, "wrench: x required");
    CKS(op_scatter(ctx, nb, x, nullptr, 0, nullptr, U ? U : ctx->U.p, F));
    return RELCP_OK;
}

int relcp_solve_lcp(relcp_ctx *ctx, const relcp_bodies *bodies, relcp_constraints *cs, relcp_solve_report *rep) {
    if (!ctx) return RELCP_E_ARG;
    if (!bodies || bodies->n <= 0 || !cs || cs->count < 0 || cs->count > cs->capacity)
        return set_err(ctx, RELCP_E_ARG, "solve: bad views");
    return lcp_solve(ctx, bodies, cs, rep);
}

int relcp_check_and_augment(relcp_ctx *ctx, const relcp_bodies *Ck, relcp_constraints *cs, int32_t recursion,
                            int64_t *n_appended, double *min_phi) {
    CKS(check_views(ctx, Ck, cs));
    if (ctx->pairs_internal) return set_err(ctx, RELCP_E_STATE, "check_and_augment: call relcp_generate_contacts first");
    return check_impl(ctx, Ck, cs, recursion, 1, n_appended, min_phi);
}

}  // extern "C"

// Algorithm 1 on one body labelling; relcp_step wraps it with the
// internal body order (order.cu)
static int step_core(relcp_ctx *ctx, relcp_bodies *b, const double *f_ext, relcp_constraints *cs,
                     relcp_step_report *rep, relcp_solve_cb solve = nullptr, void *user = nullptr,
                     const DistSpec *ds = nullptr) {
    relcp_step_report R;
    memset(&R, 0, sizeof(R));
    const int64_t nb = b->n;
    CKS(ensure_common(ctx, nb));
    PHASE(ctx, "step.enter");
    const int64_t guard0 = ctx->n_guard_total;
    double t0 = now_ms();
    // W frozen at C^k; U_free (P:L557-561 / P:L522)
    CKS(op_build_W(ctx, b, ctx->W.p));
    k_ufree<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, ctx->p.dynamics, ctx->p.dt, b->vel, f_ext, ctx->W.p,
                                                        b->kinematic, ctx->ufree.p);
    CKL();
    PHASE(ctx, "step.W_ufree");
    int64_t n0 = 0;
    nvtxRangePushA("relcp_generate");
    int rc = generate_impl(ctx, b, cs, &n0, ds);  // Alg. 1 lines 1-2
    nvtxRangePop();
    if (rc < 0) return rc;
    int warn = rc;
    double t1 = now_ms();
    R.ms_generate = t1 - t0;
    int recursion = 0;
    ctx->L_reuse = 0.0;
    for (;;) {
        relcp_solve_report sr;
        double ts = now_ms();
        nvtxRangePushA("relcp_solve_lcp");
        PHASE(ctx, "solve.enter");
        rc = solve ? solve(user, ctx, b, cs, &sr) : lcp_solve(ctx, b, cs, &sr);  // lines 3 / 10
        PHASE(ctx, "solve.done");
        nvtxRangePop();
        R.ms_solve += now_ms() - ts;
        ctx->L_reuse = rc < 0 ? 0.0 : sr.L;  // later recursions of this step may reuse it (R1)
        ctx->L_reuse_nc = cs->count;
        if (rc < 0) return rc;
        if (rc == RELCP_W_MAX_ITER) warn = rc;
        R.n_c[recursion] = cs->count;
        R.lcp_iters[recursion] = sr.iterations;
        R.residual[recursion] = sr.residual;
        R.f_n[recursion] = sr.objective;
        // line 5: overlap check at C_{n+1}; lines 6-9 append
        double tc = now_ms();
        int64_t napp = 0;
        double minphi = INFINITY;
        const int allow = recursion < ctx->p.max_recursions;
        nvtxRangePushA("relcp_check_and_augment");
        rc = check_impl(ctx, b, cs, recursion + 1, allow, &napp, &minphi, ds);
        nvtxRangePop();
        R.ms_check += now_ms() - tc;
        if (rc < 0) return rc;
        if (rc == RELCP_W_SNSD_NONCONV) warn = rc;
        R.max_overlap = minphi < 0.0 ? -minphi : 0.0;
        if (napp == 0) break;
        if (!allow) {
            R.status = RELCP_W_RECURSION_CAP;
            break;
        }
        ++recursion;
    }
    ctx->L_reuse = 0.0;
    R.recursions = recursion;
    R.n_pairs = ctx->npairs;
    R.margin = ctx->margin;
    R.snsd_nonconv = ctx->snsd_nonconv_total;
    R.n_guard = ctx->n_guard_total - guard0;
    // line 14: accept C^{k+1} = C_{n+1}, U^{k+1} = U_tot
    k_accept<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, ctx->p.box[0], ctx->p.box[1], ctx->p.box[2],
                                                         ctx->ptrial.p, ctx->qtrial.p, ctx->utot.p, b->pos, b->quat,
                                                         b->vel);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));
    PHASE(ctx, "step.accept");
    ctx->step_nb = -1;  // bodies moved: the pair list is stale
    if (rep) *rep = R;
    if (R.status) return R.status;
    return warn > 0 ? warn : RELCP_OK;
}

// Algorithm 1 in the caller's body order with another LCP solver (the
// domain-decomposed solve, dd.cu relcp_dd_step)
int step_entry(relcp_ctx *ctx, relcp_bodies *b, const double *f_ext, relcp_constraints *cs, relcp_step_report *rep,
               relcp_solve_cb solve, void *user, const DistSpec *ds) {
    CKS(check_views(ctx, b, cs));
    if (!cs->g) return set_err(ctx, RELCP_E_ARG, "step: constraints.g is required");
    if (ctx->p.dynamics == RELCP_INERTIAL && !b->vel) return set_err(ctx, RELCP_E_ARG, "step: inertial needs vel");
    ctx->pairs_internal = 0;
    return step_core(ctx, b, f_ext, cs, rep, solve, user, ds);
}

extern "C" {

int relcp_step(relcp_ctx *ctx, relcp_bodies *b, const double *f_ext, relcp_constraints *cs, relcp_step_report *rep) {
    CKS(check_views(ctx, b, cs));
    if (!cs->g) return set_err(ctx, RELCP_E_ARG, "step: constraints.g is required");
    if (ctx->p.dynamics == RELCP_INERTIAL && !b->vel) return set_err(ctx, RELCP_E_ARG, "step: inertial needs vel");
    const bool on = ctx->p.reorder == RELCP_REORDER_ON;
    const bool maybe = ctx->p.reorder == RELCP_REORDER_AUTO && b->n >= RELCP_REORDER_MIN_BODIES;
    ctx->pairs_internal = 0;
    if (!on && !maybe) return step_core(ctx, b, f_ext, cs, rep);
    // internal cell order: relabel, run Algorithm 1, translate back (order.cu);
    // AUTO keeps the caller's order when it already follows space
    PHASE(ctx, "step.enter");
    double coh = 0.0;
    CKS(ord_body_perm(ctx, b->n, b->pos, on ? nullptr : &coh));
    if (!on && coh >= RELCP_REORDER_COHERENT) return step_core(ctx, b, f_ext, cs, rep);
    relcp_bodies bi;
    const double *fi = nullptr;
    CKS(ord_bodies_in(ctx, b, f_ext, &bi, &fi));
    relcp_constraints ci;
    CKS(ord_store(ctx, cs, &ci));
    PHASE(ctx, "step.reorder_in");
    const int rc = step_core(ctx, &bi, fi, &ci, rep);
    ctx->pairs_internal = 1;
    if (rc == RELCP_E_CAPACITY) cs->count = ci.count;
    if (rc < 0) return rc;
    CKS(ord_bodies_out(ctx, &bi, b));
    CKS(ord_store_out(ctx, b->n, &ci, cs));
    ctx->op_nc = -1;  // the operator was prepared on the internal store
    CK(cudaStreamSynchronize(ctx->stream));
    PHASE(ctx, "step.reorder_out");
    return rc;
}

int relcp_get_stats(relcp_ctx *ctx, relcp_stats *out) {
    if (!ctx || !out) return RELCP_E_ARG;
    out->launches = ctx->launches;
    out->lcp_iterations = ctx->lcp_iterations;
    out->iter_timed = ctx->iter_timed;
    out->scatter_ms = ctx->scatter_ms;
    out->gather_ms = ctx->gather_ms;
    out->split_timed = ctx->split_timed;
    out->iter_ms = ctx->iter_ms;
    out->n_guard = ctx->n_guard_total;
    out->jds_solves = ctx->jds_solves;
    out->op_layout = ctx->op_jds ? RELCP_LAYOUT_JDS : RELCP_LAYOUT_CSR;
    out->pad = 0;
    out->cluster_solves = ctx->cluster_solves;
    long long nm = 0;
    if (ctx->dstat.p && (cudaMemcpyAsync(&nm, ctx->dstat.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream) !=
                             cudaSuccess || cudaStreamSynchronize(ctx->stream) != cudaSuccess))
        return set_err(ctx, RELCP_E_CUDA, "stats: device counters");
    out->snsd_multistart = nm;
    return RELCP_OK;
}

int relcp_reset_stats(relcp_ctx *ctx) {
    if (!ctx) return RELCP_E_ARG;
    ctx->launches = 0;
    ctx->lcp_iterations = 0;
    ctx->iter_timed = ctx->split_timed = 0;
    ctx->scatter_ms = ctx->gather_ms = ctx->iter_ms = 0.0;
    ctx->n_guard_total = 0;
    ctx->jds_solves = 0;
    ctx->cluster_solves = 0;
    if (ctx->dstat.p && cudaMemsetAsync(ctx->dstat.p, 0, 4 * sizeof(long long), ctx->stream) != cudaSuccess)
        return set_err(ctx, RELCP_E_CUDA, "reset_stats: device counters");
    return RELCP_OK;
}

int relcp_set_timing(relcp_ctx *ctx, int32_t on) {
    if (!ctx) return RELCP_E_ARG;
    ctx->timing = on != 0;
    return RELCP_OK;
}

int relcp_get_pairs(relcp_ctx *ctx, int32_t *pi, int32_t *pj, int64_t cap, int64_t *n_pairs) {
    if (!ctx) return RELCP_E_ARG;
    if (n_pairs) *n_pairs = ctx->npairs;
    if (pi && pj) {
        int64_t m = ctx->npairs < cap ? ctx->npairs : cap;
        if (m > 0 && ctx->pairs_internal) {
            CKS(ord_pairs_out(ctx, m, pi, pj));
        } else if (m > 0) {
            CK(cudaMemcpyAsync(pi, ctx->pi.p, sizeof(int) * m, cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemcpyAsync(pj, ctx->pj.p, sizeof(int) * m, cudaMemcpyDeviceToDevice, ctx->stream));
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

int relcp_snsd_pairs(relcp_ctx *ctx, const relcp_bodies *b, int64_t n_pairs, const int32_t *pi, const int32_t *pj,
                     double *phi, double *nrm, double *ra, double *rb, int32_t *status) {
    if (!ctx) return RELCP_E_ARG;
    if (!b || b->n <= 0 || !b->pos || !b->quat || !b->axes || n_pairs < 0)
        return set_err(ctx, RELCP_E_ARG, "snsd: bad bodies");
    if (n_pairs == 0) return RELCP_OK;
    if (!pi || !pj || !phi || !nrm || !ra || !rb || !status) return set_err(ctx, RELCP_E_ARG, "snsd: null output");
    CK(ctx->Sig.grow(6 * b->n));
    CKS(geo_shape_matrices(ctx, b->n, b->quat, b->axes, b->shape, ctx->Sig.p));
    CKS(geo_snsd(ctx, n_pairs, pi, pj, b->pos, ctx->Sig.p, phi, nrm, ra, rb, status, n_pairs, INFINITY, b->shape,
                 b->axes));
    ctx->step_nb = -1;  // Sig overwritten
    return RELCP_OK;
}

}  // extern "C"
