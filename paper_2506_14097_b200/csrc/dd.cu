// Domain decomposition of the Delassus operator and of the BB solve
// (the paper's own solver is distributed with
// MPI over spatial domains, "FDPS ... Zoltan2 ... Trilinos").
//
// Partition (relcp_dd_plan_host):
//   * bodies: K contiguous index ranges [off[k], off[k+1]) -- with the
//     library's spatially coherent body order these are slabs of the box;
//   * constraint alpha is owned by the part that owns ia; the store is sorted
//     by ia (R18), so part k's rows are one contiguous store range [r_lo, r_hi)
//     and the local store is a view of the global planes (n, t, q, lambda, g);
//   * local bodies = owned (local ids 0 .. n_own-1, in global order) then the
//     ghosts: the ib of owned rows owned elsewhere, sorted by global id, hence
//     grouped by owner part (segment gseg[q] .. gseg[q+1] for owner q).
// One apply y = s D^T W D x (and one BB iteration) per part:
//   1. K6 over the local rows -> partial wrenches F of owned AND ghost bodies;
//   2. ghost partials -> owners (part q receives from every p, in ascending p,
//      into recvF segment rseg[p]); the owner adds them to its own sum in that
//      fixed order and applies W (k_dd_add_W): deterministic, no atomics;
//   3. U of boundary bodies -> the parts that hold them as ghosts (written
//      straight into their ghost slots: same segment order as step 2);
//   4. K7 over the local rows (gather + projected step + partial reductions);
//      the BB dot products / residual are combined over the parts (fixed part
//      order; NCCL all-reduce across ranks) before the step-size update.
// Transports: VIRTUAL = all K parts in this process on one device, exchange
// by device copies (the correctness / determinism vehicle on one GPU); NCCL =
// this process holds part `rank` of K ranks, exchange by grouped NCCL
// send/recv of exactly the halo bytes (48 B per boundary body and direction)
// and one grouped all-reduce of <= 6 doubles per iteration.  NCCL is loaded
// at run time (dlopen of libnccl.so.2, the one torch already loaded).
#include <dlfcn.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

// ------------------------------------------------------------ NCCL (run-time loaded)
typedef struct {
    char internal[128];
} dd_nccl_uid;
typedef void *dd_nccl_comm;
enum { ncclDouble_ = 8, ncclSum_ = 0, ncclMax_ = 2 };
struct NcclApi {
    void *h = nullptr;
    int (*GetUniqueId)(dd_nccl_uid *) = nullptr;
    int (*CommInitRank)(dd_nccl_comm *, int, dd_nccl_uid, int) = nullptr;
    int (*CommDestroy)(dd_nccl_comm) = nullptr;
    int (*Send)(const void *, size_t, int, int, dd_nccl_comm, cudaStream_t) = nullptr;
    int (*Recv)(void *, size_t, int, int, dd_nccl_comm, cudaStream_t) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, dd_nccl_comm, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
    bool load() {
        if (h) return true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
            if (!h) h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
#define NSYM(f) f = (decltype(f))dlsym(h, "nccl" #f)
        NSYM(GetUniqueId); NSYM(CommInitRank); NSYM(CommDestroy); NSYM(Send); NSYM(Recv); NSYM(AllReduce);
        NSYM(GroupStart); NSYM(GroupEnd); NSYM(GetErrorString);
#undef NSYM
        return GetUniqueId && CommInitRank && CommDestroy && Send && Recv && AllReduce && GroupStart && GroupEnd;
    }
};
static NcclApi g_nccl;

// ------------------------------------------------------------ host plan
struct DDPlan {
    int64_t lo = 0, hi = 0, r_lo = 0, r_hi = 0;
    std::vector<int64_t> ghost;      // ghost global ids, ascending
    std::vector<int64_t> gseg;       // K+1: ghost segment of each owner part
    std::vector<int64_t> rseg;       // K+1: recv-slot segment of each source part
    std::vector<int32_t> recv_list;  // owned local id of each recv slot
    std::vector<int32_t> bnd, bnd_ptr, bnd_slot;  // boundary CSR: owned id -> recv slots (ascending part)
};

static void ghosts_of(int K, const int64_t *off, const int32_t *ia, const int32_t *ib, int64_t nc, int k,
                      int64_t &r_lo, int64_t &r_hi, std::vector<int64_t> &ghost) {
    r_lo = std::lower_bound(ia, ia + nc, (int32_t)off[k]) - ia;
    r_hi = std::lower_bound(ia, ia + nc, (int32_t)off[k + 1]) - ia;
    ghost.clear();
    for (int64_t r = r_lo; r < r_hi; ++r)
        if (ib[r] < off[k] || ib[r] >= off[k + 1]) ghost.push_back(ib[r]);
    std::sort(ghost.begin(), ghost.end());
    ghost.erase(std::unique(ghost.begin(), ghost.end()), ghost.end());
}

// Returns 0, or -1 when the rows are not sorted by ia / reference bad bodies.
static int build_plan(int K, const int64_t *off, const int32_t *ia, const int32_t *ib, int64_t nc, int k,
                      DDPlan &P) {
    for (int64_t r = 0; r < nc; ++r) {
        if (r > 0 && ia[r] < ia[r - 1]) return -1;
        if (ia[r] < off[0] || ia[r] >= off[K] || ib[r] < off[0] || ib[r] >= off[K] || ia[r] == ib[r]) return -1;
    }
    P.lo = off[k];
    P.hi = off[k + 1];
    ghosts_of(K, off, ia, ib, nc, k, P.r_lo, P.r_hi, P.ghost);
    P.gseg.assign(K + 1, 0);
    for (int q = 0; q <= K; ++q)
        P.gseg[q] = std::lower_bound(P.ghost.begin(), P.ghost.end(), off[q]) - P.ghost.begin();
    // receive side: every other part's ghosts owned by k, in ascending part order
    P.rseg.assign(K + 1, 0);
    P.recv_list.clear();
    std::vector<int64_t> gp;
    for (int p = 0; p < K; ++p) {
        P.rseg[p] = (int64_t)P.recv_list.size();
        if (p == k) continue;
        int64_t a, b;
        ghosts_of(K, off, ia, ib, nc, p, a, b, gp);
        auto s = std::lower_bound(gp.begin(), gp.end(), off[k]);
        auto e = std::lower_bound(gp.begin(), gp.end(), off[k + 1]);
        for (auto it = s; it != e; ++it) P.recv_list.push_back((int32_t)(*it - off[k]));
    }
    P.rseg[K] = (int64_t)P.recv_list.size();
    // boundary CSR: owned body -> its recv slots in ascending slot (= part) order
    std::vector<std::pair<int32_t, int32_t>> js;
    js.reserve(P.recv_list.size());
    for (size_t s = 0; s < P.recv_list.size(); ++s) js.push_back({P.recv_list[s], (int32_t)s});
    std::sort(js.begin(), js.end());
    P.bnd.clear();
    P.bnd_ptr.assign(1, 0);
    P.bnd_slot.clear();
    for (size_t i = 0; i < js.size(); ++i) {
        if (i == 0 || js[i].first != js[i - 1].first) {
            if (i > 0) P.bnd_ptr.push_back((int32_t)P.bnd_slot.size());
            P.bnd.push_back(js[i].first);
        }
        P.bnd_slot.push_back(js[i].second);
    }
    if (!js.empty()) P.bnd_ptr.push_back((int32_t)P.bnd_slot.size());
    return 0;
}

extern "C" int relcp_dd_plan_host(int32_t nparts, const int64_t *part_off, int64_t nc, const int32_t *ia,
                                  const int32_t *ib, int32_t part, relcp_dd_info *info, int64_t *ghost,
                                  int64_t *gseg, int64_t *rseg, int32_t *recv_list) {
    if (nparts < 1 || !part_off || part < 0 || part >= nparts || nc < 0 || (nc > 0 && (!ia || !ib)) || !info)
        return RELCP_E_ARG;
    for (int k = 0; k < nparts; ++k)
        if (part_off[k + 1] < part_off[k]) return RELCP_E_ARG;
    DDPlan P;
    if (build_plan(nparts, part_off, ia, ib, nc, part, P) != 0) return RELCP_E_ARG;
    info->n_own = P.hi - P.lo;
    info->n_ghost = (int64_t)P.ghost.size();
    info->row_lo = P.r_lo;
    info->row_hi = P.r_hi;
    info->n_recv = (int64_t)P.recv_list.size();
    info->n_boundary = (int64_t)P.bnd.size();
    if (ghost) std::copy(P.ghost.begin(), P.ghost.end(), ghost);
    if (gseg) std::copy(P.gseg.begin(), P.gseg.end(), gseg);
    if (rseg) std::copy(P.rseg.begin(), P.rseg.end(), rseg);
    if (recv_list) std::copy(P.recv_list.begin(), P.recv_list.end(), recv_list);
    return RELCP_OK;
}

// ------------------------------------------------------------ device parts
struct DDPart {
    int k = 0;
    DDPlan plan;
    int64_t n_loc = 0;
    bool empty = false;        // owns no body (hence no row, no ghost, no halo)
    relcp_ctx *ctx = nullptr;  // this part's operator (CSR, W, U, LCP state)
    DevBuf<int32_t> ia, ib;    // local ids of the owned rows
    DevBuf<double> quat, axes, inv_mass, inv_inertia;
    DevBuf<int32_t> kin, shape;
    DevBuf<int64_t> gids;      // global id of each local body
    DevBuf<double> F;          // (n_loc, 6) partial wrenches of the last scatter
    DevBuf<double> recvF, sendU;  // (n_recv, 6)
    DevBuf<int32_t> recv_list, bnd, bnd_ptr, bnd_slot;
    relcp_bodies bodies{};
    relcp_constraints cs{};
};

struct relcp_dd {
    relcp_ctx *ctx = nullptr;  // error messages, launch counter, stream
    int K = 1, rank = -1;      // rank < 0: all parts here (VIRTUAL)
    std::vector<int64_t> off;
    std::vector<DDPart *> parts;
    int64_t nb = 0, nc = 0;
    const void *key_ia = nullptr;
    DevBuf<double> acc;        // (K, 8) per-part partials
    DevBuf<double> acc_comb;   // (8) combined
    DevBuf<double> xB, gB, vtmp;
    dd_nccl_comm comm = nullptr;
    int64_t iterations = 0;
    std::vector<int64_t> roff;  // (K + 1) row range of every part in the loaded store
};

__global__ void k_dd_gather_bodies(int64_t n, const int64_t *__restrict__ gid, const double *quat,
                                   const double *axes, const double *inv_mass, const double *inv_inertia,
                                   const int32_t *kin, const int32_t *shape, double *oq, double *oa, double *om,
                                   double *oi, int32_t *ok, int32_t *os) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = gid[b];
        for (int c = 0; c < 4; ++c) oq[4 * b + c] = quat[4 * g + c];
        for (int c = 0; c < 3; ++c) oa[3 * b + c] = axes[3 * g + c];
        if (inv_mass) om[b] = inv_mass[g];
        if (inv_inertia)
            for (int c = 0; c < 3; ++c) oi[3 * b + c] = inv_inertia[3 * g + c];
        if (kin) ok[b] = kin[g];
        if (shape) os[b] = shape[g];
    }
}

// local ids: ia - lo; ib - lo if owned, else n_own + rank in the ghost list
__global__ void k_dd_local_rows(int64_t m, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib,
                                int64_t lo, int64_t hi, const int64_t *__restrict__ ghost, int64_t ng, int64_t n_own,
                                int32_t *la, int32_t *lb) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        la[r] = (int32_t)(ia[r] - lo);
        const int64_t j = ib[r];
        if (j >= lo && j < hi) {
            lb[r] = (int32_t)(j - lo);
        } else {
            int64_t a = 0, b = ng;  // lower_bound in the sorted ghost list
            while (a < b) {
                const int64_t c = (a + b) >> 1;
                if (ghost[c] < j) a = c + 1; else b = c;
            }
            lb[r] = (int32_t)(n_own + a);
        }
    }
}

// owner side of the halo sum: F_j += recvF[slots of j] (ascending source part),
// then U_j = W_j F_j (W SoA planes of this part, stride n_loc)
__global__ void k_dd_add_W(int64_t nbnd, const int32_t *__restrict__ bnd, const int32_t *__restrict__ ptr,
                           const int32_t *__restrict__ slot, const double *__restrict__ recvF,
                           const double *__restrict__ W, int64_t n_loc, double *F, double *U) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbnd; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = bnd[i];
        double f[6];
        for (int c = 0; c < 6; ++c) f[c] = F[6 * j + c];
        for (int s = ptr[i]; s < ptr[i + 1]; ++s)
            for (int c = 0; c < 6; ++c) f[c] += recvF[6 * (int64_t)slot[s] + c];
        const double w0 = W[j], s00 = W[n_loc + j], s01 = W[2 * n_loc + j], s02 = W[3 * n_loc + j],
                     s11 = W[4 * n_loc + j], s12 = W[5 * n_loc + j], s22 = W[6 * n_loc + j];
        for (int c = 0; c < 6; ++c) F[6 * j + c] = f[c];
        U[6 * j + 0] = w0 * f[0];
        U[6 * j + 1] = w0 * f[1];
        U[6 * j + 2] = w0 * f[2];
        U[6 * j + 3] = s00 * f[3] + s01 * f[4] + s02 * f[5];
        U[6 * j + 4] = s01 * f[3] + s11 * f[4] + s12 * f[5];
        U[6 * j + 5] = s02 * f[3] + s12 * f[4] + s22 * f[5];
    }
}

__global__ void k_dd_pack_U(int64_t n, const int32_t *__restrict__ list, const double *__restrict__ U, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 6 * n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = U[6 * (int64_t)list[i / 6] + i % 6];
}

// combine the parts' partials in part order (sum or max per value)
__global__ void k_dd_combine(const double *__restrict__ acc, int K, int nv, int ops_bits, double *out) {
    for (int v = 0; v < nv; ++v) {
        const bool mx = (ops_bits >> v) & 1;
        double a = mx ? -INFINITY : 0.0;
        for (int k = 0; k < K; ++k) a = mx ? fmax(a, acc[8 * k + v]) : a + acc[8 * k + v];
        out[v] = a;
    }
}

static int ops_bits(int kind) {
    int bits = 0;
    const int *o = lcp_dd_ops(kind);
    for (int v = 0; v < lcp_dd_nvals(kind); ++v) bits |= (o[v] ? 1 : 0) << v;
    return bits;
}

#define DDCTX relcp_ctx *ctx = dd->ctx

static int nccl_check(relcp_dd *dd, int r, const char *what) {
    DDCTX;
    if (r != 0)
        return set_err(ctx, RELCP_E_CUDA, "dd: %s failed: %s", what,
                       g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
    return RELCP_OK;
}

// halo step 2: ghost partial wrenches -> owners' recvF
static int exchange_F(relcp_dd *dd) {
    DDCTX;
    const int K = dd->K;
    if (dd->rank < 0) {
        for (DDPart *q : dd->parts)
            for (DDPart *p : dd->parts) {
                if (p == q) continue;
                const int64_t cnt = p->plan.gseg[q->k + 1] - p->plan.gseg[q->k];
                if (cnt == 0) continue;
                const double *src = p->F.p + 6 * (p->plan.hi - p->plan.lo + p->plan.gseg[q->k]);
                double *dst = q->recvF.p + 6 * q->plan.rseg[p->k];
                CK(cudaMemcpyAsync(dst, src, sizeof(double) * 6 * cnt, cudaMemcpyDeviceToDevice, ctx->stream));
            }
        return RELCP_OK;
    }
    DDPart *me = dd->parts[0];
    const int64_t n_own = me->plan.hi - me->plan.lo;
    CKS(nccl_check(dd, g_nccl.GroupStart(), "ncclGroupStart"));
    for (int q = 0; q < K; ++q) {
        if (q == dd->rank) continue;
        const int64_t cs_ = me->plan.gseg[q + 1] - me->plan.gseg[q];
        if (cs_) CKS(nccl_check(dd, g_nccl.Send(me->F.p + 6 * (n_own + me->plan.gseg[q]), 6 * cs_, ncclDouble_, q,
                                                dd->comm, ctx->stream), "ncclSend"));
        const int64_t cr = me->plan.rseg[q + 1] - me->plan.rseg[q];
        if (cr) CKS(nccl_check(dd, g_nccl.Recv(me->recvF.p + 6 * me->plan.rseg[q], 6 * cr, ncclDouble_, q, dd->comm,
                                                ctx->stream), "ncclRecv"));
    }
    CKS(nccl_check(dd, g_nccl.GroupEnd(), "ncclGroupEnd"));
    return RELCP_OK;
}

// halo step 3: U of boundary bodies -> the ghost slots of the parts holding them
static int exchange_U(relcp_dd *dd) {
    DDCTX;
    const int K = dd->K;
    if (dd->rank < 0) {
        for (DDPart *q : dd->parts)
            for (DDPart *p : dd->parts) {
                if (p == q) continue;
                const int64_t cnt = q->plan.rseg[p->k + 1] - q->plan.rseg[p->k];
                if (cnt == 0) continue;
                const double *src = q->sendU.p + 6 * q->plan.rseg[p->k];
                double *dst = p->ctx->U.p + 6 * (p->plan.hi - p->plan.lo + p->plan.gseg[q->k]);
                CK(cudaMemcpyAsync(dst, src, sizeof(double) * 6 * cnt, cudaMemcpyDeviceToDevice, ctx->stream));
            }
        return RELCP_OK;
    }
    DDPart *me = dd->parts[0];
    const int64_t n_own = me->plan.hi - me->plan.lo;
    CKS(nccl_check(dd, g_nccl.GroupStart(), "ncclGroupStart"));
    for (int p = 0; p < K; ++p) {
        if (p == dd->rank) continue;
        const int64_t cs_ = me->plan.rseg[p + 1] - me->plan.rseg[p];
        if (cs_) CKS(nccl_check(dd, g_nccl.Send(me->sendU.p + 6 * me->plan.rseg[p], 6 * cs_, ncclDouble_, p, dd->comm,
                                                ctx->stream), "ncclSend"));
        const int64_t cr = me->plan.gseg[p + 1] - me->plan.gseg[p];
        if (cr) CKS(nccl_check(dd, g_nccl.Recv(me->ctx->U.p + 6 * (n_own + me->plan.gseg[p]), 6 * cr, ncclDouble_, p,
                                                dd->comm, ctx->stream), "ncclRecv"));
    }
    CKS(nccl_check(dd, g_nccl.GroupEnd(), "ncclGroupEnd"));
    return RELCP_OK;
}

// U = W D x over every part (K6 -> halo sum -> W -> halo U); mode / slots as op_scatter
static int dd_scatter(relcp_dd *dd, const double *x, const double *g, int mode, bool power, const double *xb,
                      const double *gb) {
    DDCTX;
    for (DDPart *p : dd->parts) {
        if (p->empty) continue;
        const int64_t r0 = p->plan.r_lo;
        CKS(op_scatter(p->ctx, p->n_loc, x + r0, g ? g + r0 : nullptr, mode, power ? &p->ctx->st.p->pnorm : nullptr,
                       p->ctx->U.p, p->F.p, xb ? xb + r0 : nullptr, gb ? gb + r0 : nullptr));
    }
    CKS(exchange_F(dd));
    for (DDPart *p : dd->parts) {
        const int64_t nbnd = (int64_t)p->plan.bnd.size();
        if (nbnd) {
            k_dd_add_W<<<grid_for(nbnd), RELCP_NT, 0, ctx->stream>>>(nbnd, p->bnd.p, p->bnd_ptr.p, p->bnd_slot.p,
                                                                     p->recvF.p, p->ctx->W.p, p->n_loc, p->F.p,
                                                                     p->ctx->U.p);
            CKL();
        }
        const int64_t nr = (int64_t)p->plan.recv_list.size();
        if (nr) {
            k_dd_pack_U<<<grid_for(6 * nr), RELCP_NT, 0, ctx->stream>>>(nr, p->recv_list.p, p->ctx->U.p, p->sendU.p);
            CKL();
        }
    }
    CKS(exchange_U(dd));
    return RELCP_OK;
}

// combine the per-part partials of `kind` and finalize every part's LCP state
static int dd_reduce(relcp_dd *dd, int kind) {
    DDCTX;
    const int nv = lcp_dd_nvals(kind);
    if (dd->rank < 0) {
        k_dd_combine<<<1, 1, 0, ctx->stream>>>(dd->acc.p, dd->K, nv, ops_bits(kind), dd->acc_comb.p);
        CKL();
        for (DDPart *p : dd->parts) CKS(lcp_dd_finalize(p->ctx, kind, dd->acc_comb.p));
        return RELCP_OK;
    }
    const int *o = lcp_dd_ops(kind);
    CKS(nccl_check(dd, g_nccl.GroupStart(), "ncclGroupStart"));
    for (int v = 0; v < nv; ++v)
        CKS(nccl_check(dd, g_nccl.AllReduce(dd->acc.p + v, dd->acc_comb.p + v, 1, ncclDouble_,
                                            o[v] ? ncclMax_ : ncclSum_, dd->comm, ctx->stream), "ncclAllReduce"));
    CKS(nccl_check(dd, g_nccl.GroupEnd(), "ncclGroupEnd"));
    CKS(lcp_dd_finalize(dd->parts[0]->ctx, kind, dd->acc_comb.p));
    return RELCP_OK;
}

static double *acc_slot(relcp_dd *dd, DDPart *p) { return dd->acc.p + 8 * (dd->rank < 0 ? p->k : 0); }

static void dd_free(relcp_dd *dd) {
    for (DDPart *p : dd->parts) {
        if (p->ctx) relcp_destroy(p->ctx);
        delete p;
    }
    dd->parts.clear();
}

extern "C" int relcp_dd_nccl_unique_id(void *out128) {
    if (!out128) return RELCP_E_ARG;
    if (!g_nccl.load()) return RELCP_E_CUDA;
    dd_nccl_uid u;
    if (g_nccl.GetUniqueId(&u) != 0) return RELCP_E_CUDA;
    memcpy(out128, &u, sizeof(u));
    return RELCP_OK;
}

extern "C" int relcp_dd_create(relcp_dd **out, const relcp_params *p, void *stream, int32_t nparts,
                               const int64_t *part_off, int32_t rank, const void *nccl_uid) {
    if (!out || !p || nparts < 1 || !part_off || rank >= nparts) return RELCP_E_ARG;
    *out = nullptr;
    for (int k = 0; k < nparts; ++k)
        if (part_off[k + 1] < part_off[k] || part_off[0] != 0) return RELCP_E_ARG;
    relcp_dd *dd = new relcp_dd();
    int rc = relcp_create(&dd->ctx, p, stream);
    if (rc != RELCP_OK) {
        delete dd;
        return rc;
    }
    dd->ctx->jds_enable = 0;  // parts run the CSR layout (halo partials in body order)
    dd->K = nparts;
    dd->rank = rank;
    dd->off.assign(part_off, part_off + nparts + 1);
    relcp_ctx *ctx = dd->ctx;
    auto fail = [&](int code) {
        relcp_dd_destroy(dd);
        return code;
    };
    if (dd->acc.grow(8 * (size_t)nparts) != cudaSuccess || dd->acc_comb.grow(8) != cudaSuccess)
        return fail(RELCP_E_CUDA);
    if (rank >= 0) {
        if (!nccl_uid) return fail(set_err(ctx, RELCP_E_ARG, "dd: NCCL mode needs the unique id"));
        if (!g_nccl.load()) return fail(RELCP_E_CUDA);
        dd_nccl_uid u;
        memcpy(&u, nccl_uid, sizeof(u));
        if (g_nccl.CommInitRank(&dd->comm, nparts, u, rank) != 0) return fail(RELCP_E_CUDA);
    }
    *out = dd;
    return RELCP_OK;
}

extern "C" int relcp_dd_destroy(relcp_dd *dd) {
    if (!dd) return RELCP_OK;
    if (dd->ctx && dd->ctx->stream) cudaStreamSynchronize(dd->ctx->stream);
    dd_free(dd);
    if (dd->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(dd->comm);
    dd->acc.release(); dd->acc_comb.release(); dd->xB.release(); dd->gB.release(); dd->vtmp.release();
    if (dd->ctx) relcp_destroy(dd->ctx);
    delete dd;
    return RELCP_OK;
}

extern "C" const char *relcp_dd_last_error(const relcp_dd *dd) { return dd && dd->ctx ? dd->ctx->err : "null dd"; }

// Partition the operator of (bodies, rows): every part's local store view,
// ghost bodies, halo maps and operator (body-major CSR, W).
extern "C" int relcp_dd_load(relcp_dd *dd, const relcp_bodies *b, const relcp_constraints *cs) {
    if (!dd) return RELCP_E_ARG;
    DDCTX;
    if (!b || b->n <= 0 || !b->quat || !b->axes || !cs || !cs->ia || !cs->ib || !cs->n || !cs->ta || !cs->tb ||
        cs->count < 0 || cs->count > cs->capacity)
        return set_err(ctx, RELCP_E_ARG, "dd_load: bodies (quat, axes) and rows required");
    if (dd->off[dd->K] != b->n) return set_err(ctx, RELCP_E_ARG, "dd_load: part offsets must end at n bodies");
    const int64_t nc = cs->count;
    std::vector<int32_t> ia(nc), ib(nc);
    if (nc) {
        CK(cudaMemcpyAsync(ia.data(), cs->ia, 4 * nc, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(ib.data(), cs->ib, 4 * nc, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    dd_free(dd);
    dd->roff.assign(dd->K + 1, nc);
    for (int k = 0; k <= dd->K; ++k)  // rows sorted by ia: part k owns [roff[k], roff[k+1])
        dd->roff[k] = std::lower_bound(ia.begin(), ia.end(), (int32_t)std::min<int64_t>(dd->off[k], INT32_MAX)) -
                      ia.begin();
    for (int k = 0; k < dd->K; ++k) {
        if (dd->rank >= 0 && k != dd->rank) continue;
        DDPart *P = new DDPart();
        dd->parts.push_back(P);
        P->k = k;
        if (build_plan(dd->K, dd->off.data(), ia.data(), ib.data(), nc, k, P->plan) != 0)
            return set_err(ctx, RELCP_E_ARG, "dd_load: rows must be sorted by ia, with ia != ib in range");
        const DDPlan &pl = P->plan;
        const int64_t n_own = pl.hi - pl.lo, ng = (int64_t)pl.ghost.size(), m = pl.r_hi - pl.r_lo;
        P->n_loc = n_own + ng;
        int rc = relcp_create(&P->ctx, &ctx->p, ctx->stream);
        if (rc != RELCP_OK) return set_err(ctx, rc, "dd_load: part context");
        P->ctx->jds_enable = 0;
        P->empty = P->n_loc == 0;  // keeps its LCP state (reductions), no operator
        if (P->empty) continue;
        const int64_t nl = P->n_loc;
        CK(P->gids.grow(nl)); CK(P->quat.grow(4 * nl)); CK(P->axes.grow(3 * nl)); CK(P->inv_mass.grow(nl));
        CK(P->inv_inertia.grow(3 * nl)); CK(P->kin.grow(nl)); CK(P->shape.grow(nl)); CK(P->F.grow(6 * nl));
        CK(P->ia.grow(m > 0 ? m : 1)); CK(P->ib.grow(m > 0 ? m : 1));
        std::vector<int64_t> gid(nl);
        for (int64_t j = 0; j < n_own; ++j) gid[j] = pl.lo + j;
        for (int64_t j = 0; j < ng; ++j) gid[n_own + j] = pl.ghost[j];
        CK(cudaMemcpyAsync(P->gids.p, gid.data(), 8 * nl, cudaMemcpyHostToDevice, ctx->stream));
        k_dd_gather_bodies<<<grid_for(nl), RELCP_NT, 0, ctx->stream>>>(
            nl, P->gids.p, b->quat, b->axes, b->inv_mass, b->inv_inertia, b->kinematic, b->shape, P->quat.p, P->axes.p,
            P->inv_mass.p, P->inv_inertia.p, P->kin.p, P->shape.p);
        CKL();
        DevBuf<int64_t> dghost;
        CK(dghost.grow(ng > 0 ? ng : 1));
        if (ng) CK(cudaMemcpyAsync(dghost.p, pl.ghost.data(), 8 * ng, cudaMemcpyHostToDevice, ctx->stream));
        if (m) {
            k_dd_local_rows<<<grid_for(m), RELCP_NT, 0, ctx->stream>>>(m, cs->ia + pl.r_lo, cs->ib + pl.r_lo, pl.lo,
                                                                       pl.hi, dghost.p, ng, n_own, P->ia.p, P->ib.p);
            CKL();
        }
        const int64_t nr = (int64_t)pl.recv_list.size(), nbd = (int64_t)pl.bnd.size();
        CK(P->recvF.grow(6 * (nr > 0 ? nr : 1))); CK(P->sendU.grow(6 * (nr > 0 ? nr : 1)));
        CK(P->recv_list.grow(nr > 0 ? nr : 1)); CK(P->bnd.grow(nbd > 0 ? nbd : 1));
        CK(P->bnd_ptr.grow(nbd + 1)); CK(P->bnd_slot.grow(nr > 0 ? nr : 1));
        if (nr) {
            CK(cudaMemcpyAsync(P->recv_list.p, pl.recv_list.data(), 4 * nr, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync(P->bnd_slot.p, pl.bnd_slot.data(), 4 * nr, cudaMemcpyHostToDevice, ctx->stream));
        }
        if (nbd) {
            CK(cudaMemcpyAsync(P->bnd.p, pl.bnd.data(), 4 * nbd, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync(P->bnd_ptr.p, pl.bnd_ptr.data(), 4 * (nbd + 1), cudaMemcpyHostToDevice, ctx->stream));
        }
        P->bodies = relcp_bodies{};
        P->bodies.n = nl;
        P->bodies.pos = P->axes.p;  // not read by the operator (non-null for the view checks)
        P->bodies.quat = P->quat.p;
        P->bodies.axes = P->axes.p;
        P->bodies.inv_mass = b->inv_mass ? P->inv_mass.p : nullptr;
        P->bodies.inv_inertia = b->inv_inertia ? P->inv_inertia.p : nullptr;
        P->bodies.kinematic = b->kinematic ? P->kin.p : nullptr;
        P->bodies.shape = b->shape ? P->shape.p : nullptr;
        // local store: a view of the global planes at row offset r_lo (plane stride = capacity)
        relcp_constraints &c = P->cs;
        c = *cs;
        const int64_t r0 = pl.r_lo;
        c.count = m;  // capacity stays the global plane stride
        c.ia = P->ia.p;
        c.ib = P->ib.p;
        c.gen = cs->gen ? cs->gen + r0 : nullptr;
        c.n = cs->n + r0;
        c.ta = cs->ta + r0;
        c.tb = cs->tb + r0;
        c.phi = cs->phi ? cs->phi + r0 : nullptr;
        c.q = cs->q ? cs->q + r0 : nullptr;
        c.lambda = cs->lambda ? cs->lambda + r0 : nullptr;
        c.g = cs->g ? cs->g + r0 : nullptr;
        CKS(op_prepare(P->ctx, &P->bodies, &c));
        CK(cudaStreamSynchronize(ctx->stream));  // dghost is released at scope end
    }
    dd->nb = b->n;
    dd->nc = nc;
    dd->key_ia = cs->ia;
    CK(dd->vtmp.grow(nc > 0 ? nc : 1));
    CK(dd->xB.grow(nc > 0 ? nc : 1));
    CK(dd->gB.grow(nc > 0 ? nc : 1));
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

extern "C" int relcp_dd_info_get(relcp_dd *dd, int32_t part, relcp_dd_info *info) {
    if (!dd || !info) return RELCP_E_ARG;
    for (DDPart *p : dd->parts)
        if (p->k == part) {
            info->n_own = p->plan.hi - p->plan.lo;
            info->n_ghost = (int64_t)p->plan.ghost.size();
            info->row_lo = p->plan.r_lo;
            info->row_hi = p->plan.r_hi;
            info->n_recv = (int64_t)p->plan.recv_list.size();
            info->n_boundary = (int64_t)p->plan.bnd.size();
            return RELCP_OK;
        }
    return RELCP_E_ARG;
}

static int check_loaded(relcp_dd *dd, const relcp_constraints *cs) {
    DDCTX;
    if (dd->parts.empty()) return set_err(ctx, RELCP_E_STATE, "dd: no operator loaded (relcp_dd_load)");
    if (cs && (cs->ia != dd->key_ia || cs->count != dd->nc))
        return set_err(ctx, RELCP_E_STATE, "dd: store differs from the loaded one");
    return RELCP_OK;
}

// y = scale D^T W D x over the parts; x, y: global row order (device).  In NCCL
// mode only this rank's rows [row_lo, row_hi) of y are written.
extern "C" int relcp_dd_delassus_apply(relcp_dd *dd, const double *x, double *y, double scale) {
    if (!dd) return RELCP_E_ARG;
    DDCTX;
    CKS(check_loaded(dd, nullptr));
    if (dd->nc > 0 && (!x || !y || x == y)) return set_err(ctx, RELCP_E_ARG, "dd apply: x, y required and distinct");
    CKS(dd_scatter(dd, x, nullptr, 0, false, nullptr, nullptr));
    for (DDPart *p : dd->parts)
        if (!p->empty) CKS(op_gather_apply(p->ctx, &p->cs, p->ctx->U.p, y + p->plan.r_lo, scale, 0));
    return RELCP_OK;
}

// U (n, 6) of the owned bodies of every local part (after the last scatter / solve)
extern "C" int relcp_dd_get_u(relcp_dd *dd, double *U_global) {
    if (!dd || !U_global) return RELCP_E_ARG;
    DDCTX;
    CKS(check_loaded(dd, nullptr));
    for (DDPart *p : dd->parts) {
        const int64_t n_own = p->plan.hi - p->plan.lo;
        if (n_own)
            CK(cudaMemcpyAsync(U_global + 6 * p->plan.lo, p->ctx->U.p, sizeof(double) * 6 * n_own,
                               cudaMemcpyDeviceToDevice, ctx->stream));
    }
    return RELCP_OK;
}

// BB projected gradient (lcp.cu) over the parts: the same iterates as the
// single-domain solve up to the association of the halo sums and reductions.
extern "C" int relcp_dd_solve_lcp(relcp_dd *dd, relcp_constraints *cs, relcp_solve_report *rep) {
    if (!dd || !cs) return RELCP_E_ARG;
    DDCTX;
    CKS(check_loaded(dd, cs));
    if (!cs->q || !cs->lambda || !cs->g) return set_err(ctx, RELCP_E_ARG, "dd solve: q, lambda and g required");
    for (DDPart *p : dd->parts) {  // the views follow the caller's q / lambda / g
        const int64_t r0 = p->plan.r_lo;
        p->cs.q = cs->q + r0;
        p->cs.lambda = cs->lambda + r0;
        p->cs.g = cs->g + r0;
    }
    const double s = lcp_scale(ctx);
    cudaStream_t st = ctx->stream;
    const int64_t nc = dd->nc;
    for (DDPart *p : dd->parts) {
        p->ctx->p = ctx->p;
        CKS(lcp_dd_state_init(p->ctx, nc));
    }
    if (nc == 0) {
        if (rep) memset(rep, 0, sizeof(*rep));
        if (rep) rep->converged = 1;
        CK(cudaStreamSynchronize(st));
        return RELCP_OK;
    }
    auto zero_acc = [&]() -> int {
        CK(cudaMemsetAsync(dd->acc.p, 0, sizeof(double) * 8 * (dd->rank < 0 ? dd->K : 1), st));
        return RELCP_OK;
    };
    for (DDPart *p : dd->parts)
        CKS(lcp_dd_project_fill(p->ctx, p->cs.count, p->cs.lambda, dd->vtmp.p + p->plan.r_lo, 1.0));
    for (int it = 0; it < ctx->p.power_iters; ++it) {  // L = ||A|| (alpha_0 = 1/L, R1)
        CKS(dd_scatter(dd, dd->vtmp.p, nullptr, 0, true, nullptr, nullptr));
        CKS(zero_acc());
        for (DDPart *p : dd->parts)
            if (!p->empty)
                CKS(op_gather_apply(p->ctx, &p->cs, p->ctx->U.p, dd->vtmp.p + p->plan.r_lo, s, 1, acc_slot(dd, p)));
        CKS(dd_reduce(dd, DD_POWER));
    }
    CKS(dd_scatter(dd, cs->lambda, nullptr, 0, false, nullptr, nullptr));
    CKS(zero_acc());
    for (DDPart *p : dd->parts)
        if (!p->empty) CKS(lcp_dd_init(p->ctx, &p->cs, s, acc_slot(dd, p)));
    CKS(dd_reduce(dd, DD_INIT));
    const int batch = ctx->p.check_every > 0 ? ctx->p.check_every : 32;
    LcpState *h = dd->parts[0]->ctx->st_host;
    long long it_before = 0;
    for (;;) {
        CK(cudaMemcpyAsync(h, dd->parts[0]->ctx->st.p, sizeof(LcpState), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        ctx->lcp_iterations += h->iter - it_before;
        it_before = h->iter;
        if (h->done) break;
        for (int j = 0; j < batch; ++j) {
            CKS(dd_scatter(dd, cs->lambda, cs->g, 1, false, dd->xB.p, dd->gB.p));
            CKS(zero_acc());
            for (DDPart *p : dd->parts)
                if (!p->empty)
                    CKS(lcp_dd_iter(p->ctx, &p->cs, s, dd->xB.p + p->plan.r_lo, dd->gB.p + p->plan.r_lo,
                                    acc_slot(dd, p)));
            CKS(dd_reduce(dd, DD_ITER));
        }
    }
    const bool pb = h->par != 0;
    if (h->fix) {  // ended on a shortened step: blend of the two slots
        CKS(zero_acc());
        for (DDPart *p : dd->parts) {
            const int64_t r0 = p->plan.r_lo, m = p->cs.count;
            double *xa = cs->lambda + r0, *ga = cs->g + r0, *xb = dd->xB.p + r0, *gb = dd->gB.p + r0;
            if (m) CKS(lcp_dd_finish(p->ctx, m, pb ? xb : xa, pb ? gb : ga, pb ? xa : xb, pb ? ga : gb, acc_slot(dd, p)));
        }
        CKS(dd_reduce(dd, DD_FINISH));
    }
    if (pb)
        for (DDPart *p : dd->parts) {
            const int64_t r0 = p->plan.r_lo, m = p->cs.count;
            if (!m) continue;
            CK(cudaMemcpyAsync(cs->lambda + r0, dd->xB.p + r0, 8 * m, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(cs->g + r0, dd->gB.p + r0, 8 * m, cudaMemcpyDeviceToDevice, st));
        }
    CKS(zero_acc());
    for (DDPart *p : dd->parts)
        if (p->cs.count) CKS(lcp_dd_objective(p->ctx, p->cs.count, p->cs.lambda, p->cs.g, p->cs.q, acc_slot(dd, p)));
    CKS(dd_reduce(dd, DD_OBJECTIVE));
    CK(cudaMemcpyAsync(h, dd->parts[0]->ctx->st.p, sizeof(LcpState), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (rep) {
        rep->iterations = h->iter;
        rep->residual = h->resid;
        rep->converged = h->conv;
        rep->objective = -0.5 * h->obj;
        rep->L = h->L;
    }
    if (h->nan) return set_err(ctx, RELCP_E_NAN, "dd solve: non-finite iterate after %lld iterations", h->iter);
    return h->conv ? RELCP_OK : RELCP_W_MAX_ITER;
}

// ------------------------------------------------------------ domain-decomposed ReLCP step
// Algorithm 1 with every LCP solve distributed (relcp_dd_solve_lcp
// on the store of the current recursion) and the SNSD of generation and checks
// split by the owner of i (each rank scans the candidate pairs of its bodies;
// the broadphase, trial configuration, q and the store merge stay replicated:
// every rank holds all body states and, after the exchanges, the same store).
// NCCL: after each SNSD phase the ranks all-reduce the counts / statistics and
// exchange their appended rows; after each solve their rows' lambda and g
// (grouped send / recv), so the replicated check sees the whole solution
// (DESIGN.md §8).
static int dd_allgather_rows(relcp_dd *dd, relcp_constraints *cs) {
    DDCTX;
    if (dd->rank < 0 || dd->K == 1) return RELCP_OK;
    const int me = dd->rank;
    const int64_t m0 = dd->roff[me], mm = dd->roff[me + 1] - m0;
    for (double *v : {cs->lambda, cs->g}) {
        CKS(nccl_check(dd, g_nccl.GroupStart(), "ncclGroupStart"));
        for (int q = 0; q < dd->K; ++q) {
            if (q == me) continue;
            if (mm) CKS(nccl_check(dd, g_nccl.Send(v + m0, mm, ncclDouble_, q, dd->comm, ctx->stream), "ncclSend"));
            const int64_t r0 = dd->roff[q], rm = dd->roff[q + 1] - r0;
            if (rm) CKS(nccl_check(dd, g_nccl.Recv(v + r0, rm, ncclDouble_, q, dd->comm, ctx->stream), "ncclRecv"));
        }
        CKS(nccl_check(dd, g_nccl.GroupEnd(), "ncclGroupEnd"));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

static int dd_step_solve(void *user, relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs,
                         relcp_solve_report *rep) {
    relcp_dd *dd = (relcp_dd *)user;
    (void)ctx;
    int rc = relcp_dd_load(dd, b, cs);
    if (rc < 0) return rc;
    rc = relcp_dd_solve_lcp(dd, cs, rep);
    if (rc < 0) return rc;
    const int rg = dd_allgather_rows(dd, cs);
    return rg < 0 ? rg : rc;
}

// the SNSD phases split by the owner of i (DistSpec, abi.cu flag_append): the
// statistics of every rank summed (counts, degenerate, non-certified, guard
// band) and max-reduced (-min Phi) in two all-reduces
static int dd_reduce_stats(void *user, double *vals, int n) {
    relcp_dd *dd = (relcp_dd *)user;
    DDCTX;
    DevBuf<double> d;
    CK(d.grow(n));
    CK(cudaMemcpyAsync(d.p, vals, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CKS(nccl_check(dd, g_nccl.AllReduce(d.p, d.p, n - 1, ncclDouble_, ncclSum_, dd->comm, ctx->stream),
                   "ncclAllReduce"));
    CKS(nccl_check(dd, g_nccl.AllReduce(d.p + n - 1, d.p + n - 1, 1, ncclDouble_, ncclMax_, dd->comm, ctx->stream),
                   "ncclAllReduce"));
    CK(cudaMemcpyAsync(vals, d.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

// every rank's appended rows [base + pre_q, base + pre_q + cnt[q]) of every
// store plane to every other rank (grouped send / recv)
static int dd_exchange_rows(void *user, relcp_constraints *cs, int64_t base, const int64_t *cnt) {
    relcp_dd *dd = (relcp_dd *)user;
    DDCTX;
    const int K = dd->K, me = dd->rank;
    std::vector<int64_t> pre(K + 1, 0);
    for (int q = 0; q < K; ++q) pre[q + 1] = pre[q] + cnt[q];
    const int64_t cap = cs->capacity;
    struct Plane {
        void *p;
        int esz;
    };
    std::vector<Plane> planes = {{cs->ia, 4}, {cs->ib, 4}, {cs->gen, 4}, {cs->phi, 8}, {cs->q, 8}, {cs->lambda, 8}};
    for (int k = 0; k < 3; ++k) {
        planes.push_back({cs->n + k * cap, 8});
        planes.push_back({cs->ta + k * cap, 8});
        planes.push_back({cs->tb + k * cap, 8});
    }
    CKS(nccl_check(dd, g_nccl.GroupStart(), "ncclGroupStart"));
    for (const Plane &pl : planes) {
        char *p = (char *)pl.p;
        if (!p) continue;
        const int esz = pl.esz;
        for (int q = 0; q < K; ++q) {
            if (q == me) continue;
            // ncclInt32 = 2 for 4-byte planes, ncclDouble = 8
            const int dt = esz == 4 ? 2 : ncclDouble_;
            if (cnt[me]) CKS(nccl_check(dd, g_nccl.Send(p + esz * (base + pre[me]), cnt[me], dt, q, dd->comm,
                                                        ctx->stream), "ncclSend"));
            if (cnt[q]) CKS(nccl_check(dd, g_nccl.Recv(p + esz * (base + pre[q]), cnt[q], dt, q, dd->comm,
                                                       ctx->stream), "ncclRecv"));
        }
    }
    CKS(nccl_check(dd, g_nccl.GroupEnd(), "ncclGroupEnd"));
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}

extern "C" int relcp_dd_step(relcp_dd *dd, relcp_bodies *b, const double *f_ext, relcp_constraints *cs,
                             relcp_step_report *rep) {
    if (!dd) return RELCP_E_ARG;
    DDCTX;
    if (!b || dd->off[dd->K] != b->n) return set_err(ctx, RELCP_E_ARG, "dd_step: part offsets must end at n bodies");
    DistSpec ds;
    ds.K = dd->K;
    ds.off = dd->off.data();
    ds.rank = dd->rank;
    ds.reduce = dd_reduce_stats;
    ds.exchange = dd_exchange_rows;
    ds.user = dd;
    return step_entry(ctx, b, f_ext, cs, rep, dd_step_solve, dd, &ds);
}
