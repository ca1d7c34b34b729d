// dist.cu -- row-slab distributed V-cycle.
//
// The fine levels 0..K-1 are partitioned into contiguous row slabs (one per
// rank) whose starts are multiples of 2^K, so a coarse row J is owned by the
// owner of fine row 2J on every distributed level.  Each rank stores its owned
// rows plus BMG_HALO ghost rows on each side -- the row warm-up of the fused
// streaming kernels -- and refreshes the ghost rows with ONE grouped exchange
// per leg and field (deep halo: the 2*nu colour passes of a leg need no
// exchange in between).  Level K and below are replicated: the level-K right-
// hand side is all-gathered, every rank runs the same inner single-GPU
// V-cycle (bmg_solver on the level-K operator, gathered once at setup), and
// each reads the rows of the correction it needs.  The kernels are the single-
// GPU kernels on row-offset views (Op::roff/ylo/yhi), so the iterate is
// bitwise identical to the single-GPU iterate.
//
// Transports: NCCL (one rank per process; libnccl is dlopen'ed, grouped
// ncclSend/ncclRecv over NVLink for ghost rows and all-gathers, ncclAllReduce
// for norms) or loopback (all ranks in this process on the current GPU, ghost
// rows copied device-to-device) -- the latter exercises the partition, the
// exchange schedule and the slab kernels on one GPU (tests/test_gpu_dist.py).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <string>
#include <vector>

#include "bmg.h"
#include "bmg_internal.cuh"
#include "dist.cuh"
#include "fused.cuh"

namespace bmg {

namespace {

long long rpitch(int nx) { return ((long long)nx + 2 + 31) / 32 * 32; }

struct Nccl {
    void *h = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*errstr)(ncclResult_t) = nullptr;
    bool load(const char *path, std::string &err)
    {
        h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("dlopen NCCL: ") + dlerror();
            return false;
        }
        groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
        groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
        send = (decltype(send))dlsym(h, "ncclSend");
        recv = (decltype(recv))dlsym(h, "ncclRecv");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        errstr = (decltype(errstr))dlsym(h, "ncclGetErrorString");
        if (!groupStart || !groupEnd || !send || !recv || !allReduce || !errstr) {
            err = "NCCL symbols missing";
            return false;
        }
        return true;
    }
};

// One slab level of one rank.  Pointers are global-row indexed (allocation
// shifted by -roff*pitch); the level-0 u/f of an NCCL rank are the caller's.
struct SLevel {
    int nx = 0, ny = 0, kind = 9;
    long long pitch = 0;
    int ylo = 1, yhi = 1, roff = 0, nrows = 0;
    double *pl[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    double *u = nullptr, *f = nullptr, *T = nullptr;
    double *ci[8] = {nullptr};  // weights from level l+1 (rows of level l+1's slab)
    Op op() const
    {
        Op A;
        A.nx = nx;
        A.ny = ny;
        A.kind = kind;
        A.pitch = pitch;
        A.O = pl[0];
        A.W = pl[1];
        A.S = pl[2];
        A.SW = pl[3];
        A.NW = pl[4];
        A.ylo = ylo;
        A.yhi = yhi;
        A.roff = roff;
        A.nrows = nrows;
        return A;
    }
};

struct SRank {
    int rank = 0;
    std::vector<SLevel> lv;  // 0..K (level K: slab rows of the gathered level)
    FusedPlan fp;
    int *d_err = nullptr;
    double *partials = nullptr, *d_norm = nullptr;
};

}  // namespace

struct DistSolver {
    int P = 1, K = 1, nx = 0, ny = 0, kind0 = 5;
    bool loopback = false;
    bmg_params_t prm;
    std::vector<int> yb;  // fine-row slab boundaries b_0..b_P
    std::vector<SRank> ranks;
    bmg_solver_t inner = nullptr;  // levels K.. on every rank
    double *fK = nullptr, *xK = nullptr;  // inner rhs / iterate (full level K, global rows)
    double *plK = nullptr;                // full level-K planes (inner setup input)
    long long pitchK = 0;
    int nxK = 0, nyK = 0;
    Nccl nccl;
    ncclComm_t comm = nullptr;
    int my_rank = 0;  // NCCL mode
    double *h_norm = nullptr;
    std::vector<void *> allocs;
    // peer mode (bmg_comm_t.peer): per rank index, per distributed level, the neighbours'
    // T / u / f ([0] lower, [1] upper neighbour; global-row indexed), the flag arrays
    // (mine: [0] signals of the lower neighbour, [1] of the upper one, [2] the next
    // expected count) and the IPC mappings to close
    bool peer = false;
    struct PeerPtrs {
        double *T[2] = {nullptr, nullptr}, *u[2] = {nullptr, nullptr}, *f[2] = {nullptr, nullptr};
    };
    std::vector<std::vector<PeerPtrs>> pp;
    unsigned long long *flags = nullptr, *nflags[2] = {nullptr, nullptr};
    int *d_perr = nullptr;
    std::vector<void *> ipc;
};

// ------------------------------------------------------------------ partition
// Owned rows at level l of rank p: J with 2^l J in [b_p, b_{p+1}).
static void owned(const std::vector<int> &yb, int p, int l, int nyl, int *lo, int *hi)
{
    const long long s = 1LL << l;
    int a = (int)((yb[p] + s - 1) / s), b = (int)((yb[p + 1] + s - 1) / s);
    *lo = std::max(a, 1);
    *hi = std::min(b, nyl + 1);
}

// Boundaries for K distributed levels and the largest admissible K.
static int partition(int nx, int ny, int P, const bmg_params_t &prm, std::vector<int> &yb)
{
    int L = 1;
    {
        int a = nx, b = ny;
        while (std::min(a, b) > prm.coarsest && (prm.max_levels <= 0 || L < prm.max_levels)) {
            a /= 2;
            b /= 2;
            L++;
        }
    }
    const int minrows = std::max(prm.agglom_rows, 2 * BMG_HALO);
    int bestK = 0;
    std::vector<int> best;
    for (int K = 1; K <= L - 1 && K < 30; K++) {
        const long long s = 1LL << K;
        std::vector<int> b(P + 1);
        b[0] = 1;
        b[P] = ny + 1;
        for (int p = 1; p < P; p++)
            b[p] = (int)(((long long)p * (ny + 1) / P + s / 2) / s * s);
        bool ok = true;
        for (int p = 0; p < P && ok; p++)
            if (b[p + 1] <= b[p])
                ok = false;
        int nyl = ny;
        for (int l = 0; l < K && ok; l++) {
            for (int p = 0; p < P && ok; p++) {
                int lo, hi;
                owned(b, p, l, nyl, &lo, &hi);
                if (hi - lo < minrows)
                    ok = false;
            }
            nyl /= 2;
        }
        if (!ok)
            break;
        bestK = K;
        best = b;
    }
    yb = best;
    return bestK;
}

// ------------------------------------------------------------------ exchange
// Which buffer of a slab level a ghost-row exchange refreshes.
enum Field { F_U, F_F, F_T, F_PL, F_CI };

static int nplanes(const SLevel &v, Field fd) { return fd == F_PL ? (v.kind == 9 ? 5 : 3) : fd == F_CI ? 8 : 1; }

static double *field_ptr(SLevel &v, SLevel *vc, Field fd, int q)
{
    switch (fd) {
    case F_U: return v.u;
    case F_F: return v.f;
    case F_T: return v.T;
    case F_PL: return v.pl[q];
    case F_CI: return v.ci[q];
    }
    (void)vc;
    return nullptr;
}

// Ghost rows of rank p at level l: lower [roff, ylo), upper [yhi, roff+nrows) --
// owned rows of p-1 / p+1 (slabs are contiguous and at least 2*HALO rows high).
// CI planes live on the rows of level l+1, so they are exchanged as level l+1.
static bmg_status_t exchange(DistSolver *d, int l, Field fd, cudaStream_t s, std::string &err)
{
    const int P = d->P;
    if (P == 1)
        return BMG_OK;
    const int la = fd == F_CI ? l + 1 : l;  // level whose rows the field lives on
    if (d->loopback) {
        for (int p = 0; p < P; p++) {
            SLevel &v = d->ranks[p].lv[la];
            SLevel &vs = d->ranks[p].lv[l];
            for (int q = 0; q < nplanes(vs, fd); q++) {
                double *dst = field_ptr(fd == F_CI ? vs : v, nullptr, fd, q);
                if (p > 0 && v.ylo > v.roff) {
                    SLevel &vs2 = d->ranks[p - 1].lv[l];
                    const double *src = field_ptr(fd == F_CI ? vs2 : d->ranks[p - 1].lv[la], nullptr, fd, q);
                    cudaMemcpyAsync(dst + (long long)v.roff * v.pitch, src + (long long)v.roff * v.pitch,
                                    sizeof(double) * (size_t)(v.ylo - v.roff) * v.pitch, cudaMemcpyDeviceToDevice, s);
                }
                if (p + 1 < P && v.roff + v.nrows > v.yhi) {
                    SLevel &vs2 = d->ranks[p + 1].lv[l];
                    const double *src = field_ptr(fd == F_CI ? vs2 : d->ranks[p + 1].lv[la], nullptr, fd, q);
                    cudaMemcpyAsync(dst + (long long)v.yhi * v.pitch, src + (long long)v.yhi * v.pitch,
                                    sizeof(double) * (size_t)(v.roff + v.nrows - v.yhi) * v.pitch,
                                    cudaMemcpyDeviceToDevice, s);
                }
            }
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            err = std::string("loopback exchange: ") + cudaGetErrorString(e);
            return BMG_ECUDA;
        }
        return BMG_OK;
    }
    // NCCL: this process holds rank my_rank.
    SRank &R = d->ranks[0];
    const int p = R.rank;
    SLevel &v = R.lv[la];
    SLevel &vs = R.lv[l];
    const int nyl = v.ny;
    const int G = BMG_HALO;
    ncclResult_t r = d->nccl.groupStart();
    for (int q = 0; q < nplanes(vs, fd) && r == ncclSuccess; q++) {
        double *a = field_ptr(fd == F_CI ? vs : v, nullptr, fd, q);
        const long long P_ = v.pitch;
        if (p > 0) {
            // my lower ghost rows [max(ylo-G,0), ylo) from p-1; p-1's upper ghost rows = my rows [ylo, ylo+G)
            const int g0 = std::max(v.ylo - G, 0);
            const int s1 = std::min(v.ylo + G, nyl + 2);
            r = d->nccl.recv(a + g0 * P_, (size_t)(v.ylo - g0) * P_, ncclDouble, p - 1, d->comm, s);
            if (r == ncclSuccess)
                r = d->nccl.send(a + (long long)v.ylo * P_, (size_t)(s1 - v.ylo) * P_, ncclDouble, p - 1, d->comm, s);
        }
        if (p + 1 < P && r == ncclSuccess) {
            const int g1 = std::min(v.yhi + G, nyl + 2);
            const int s0 = std::max(v.yhi - G, 0);
            r = d->nccl.recv(a + (long long)v.yhi * P_, (size_t)(g1 - v.yhi) * P_, ncclDouble, p + 1, d->comm, s);
            if (r == ncclSuccess)
                r = d->nccl.send(a + (long long)s0 * P_, (size_t)(v.yhi - s0) * P_, ncclDouble, p + 1, d->comm, s);
        }
    }
    ncclResult_t r2 = d->nccl.groupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
        err = std::string("NCCL exchange: ") + d->nccl.errstr(r != ncclSuccess ? r : r2);
        return BMG_ENCCL;
    }
    return BMG_OK;
}

// All-gather the owned level-K rows [ylo, yhi) into the full array `full` (global
// rows, pitch pitchK, `nplanes` planes of stride npk) on every rank.  which = 0:
// the rows come from the slab's planes; which = 1: they are already in `full`.
// Two exchanges as ONE NCCL group (nested groups launch at the outermost end):
// one communication kernel per leg instead of one per field.
static bmg_status_t exchange2(DistSolver *d, int l1, Field f1, int l2, Field f2, cudaStream_t s, std::string &err)
{
    if (d->P == 1)
        return BMG_OK;
    if (d->loopback) {
        bmg_status_t rc = exchange(d, l1, f1, s, err);
        return rc == BMG_OK ? exchange(d, l2, f2, s, err) : rc;
    }
    ncclResult_t r = d->nccl.groupStart();
    bmg_status_t rc = r == ncclSuccess ? exchange(d, l1, f1, s, err) : BMG_ENCCL;
    if (rc == BMG_OK)
        rc = exchange(d, l2, f2, s, err);
    ncclResult_t r2 = d->nccl.groupEnd();
    if (rc == BMG_OK && (r != ncclSuccess || r2 != ncclSuccess)) {
        err = std::string("NCCL exchange group: ") + d->nccl.errstr(r != ncclSuccess ? r : r2);
        return BMG_ENCCL;
    }
    return rc;
}

static bmg_status_t allgather_rows(DistSolver *d, double *full, long long npk, int nplanes, int which,
                                   cudaStream_t s, std::string &err)
{
    const int K = d->K;
    if (d->loopback) {
        for (auto &R : d->ranks) {
            SLevel &v = R.lv[K];
            for (int q = 0; q < nplanes && which == 0; q++) {
                const double *src = v.pl[q];
                cudaMemcpyAsync(full + q * npk + (long long)v.ylo * v.pitch, src + (long long)v.ylo * v.pitch,
                                sizeof(double) * (size_t)(v.yhi - v.ylo) * v.pitch, cudaMemcpyDeviceToDevice, s);
            }
        }
        return BMG_OK;
    }
    SRank &R = d->ranks[0];
    SLevel &v = R.lv[K];
    ncclResult_t r = d->nccl.groupStart();
    for (int q = 0; q < nplanes && r == ncclSuccess; q++) {
        double *dst = full + q * npk;
        const double *src = v.pl[q];
        if (which == 0)
            cudaMemcpyAsync(dst + (long long)v.ylo * v.pitch, src + (long long)v.ylo * v.pitch,
                            sizeof(double) * (size_t)(v.yhi - v.ylo) * v.pitch, cudaMemcpyDeviceToDevice, s);
        for (int o = 0; o < d->P && r == ncclSuccess; o++) {
            if (o == R.rank)
                continue;
            int lo, hi;
            owned(d->yb, o, K, d->nyK, &lo, &hi);
            r = d->nccl.recv(dst + (long long)lo * d->pitchK, (size_t)(hi - lo) * d->pitchK, ncclDouble, o, d->comm, s);
            if (r == ncclSuccess)
                r = d->nccl.send(dst + (long long)v.ylo * d->pitchK, (size_t)(v.yhi - v.ylo) * d->pitchK, ncclDouble,
                                 o, d->comm, s);
        }
    }
    ncclResult_t r2 = d->nccl.groupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
        err = std::string("NCCL all-gather: ") + d->nccl.errstr(r != ncclSuccess ? r : r2);
        return BMG_ENCCL;
    }
    return BMG_OK;
}

// ------------------------------------------------------------------ setup
#define DTRY(x)                   \
    do {                          \
        bmg_status_t s_ = (x);    \
        if (s_ != BMG_OK)         \
            return s_;            \
    } while (0)
#define DCK(call)                                                                                     \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) {                                                                      \
            err = std::string(#call) + ": " + cudaGetErrorString(e_);                                 \
            return e_ == cudaErrorMemoryAllocation ? BMG_ENOMEM : BMG_ECUDA;                          \
        }                                                                                             \
    } while (0)

static bmg_status_t dmalloc(DistSolver *d, double **p, size_t n, std::string &err)
{
    void *q = nullptr;
    DCK(cudaMalloc(&q, n * sizeof(double)));
    d->allocs.push_back(q);
    *p = (double *)q;
    return BMG_OK;
}

// Geometry and zeroed storage of slab level l of rank p.
static bmg_status_t alloc_level(DistSolver *d, SRank &R, int l, int nx, int ny, int kind, long long pitch, bool user0,
                                cudaStream_t s, std::string &err)
{
    SLevel &v = R.lv[l];
    v.nx = nx;
    v.ny = ny;
    v.kind = kind;
    v.pitch = pitch;
    owned(d->yb, R.rank, l, ny, &v.ylo, &v.yhi);
    v.roff = std::max(v.ylo - BMG_HALO, 0);
    v.nrows = std::min(v.yhi + BMG_HALO, ny + 2) - v.roff;
    const size_t np = (size_t)v.nrows * pitch;
    const long long sh = (long long)v.roff * pitch;
    const int npl = kind == 9 ? 5 : 3;
    double *blk = nullptr;
    DTRY(dmalloc(d, &blk, np * npl, err));
    DCK(cudaMemsetAsync(blk, 0, np * npl * sizeof(double), s));
    for (int k = 0; k < npl; k++)
        v.pl[k] = blk + k * np - sh;
    double *t = nullptr;
    DTRY(dmalloc(d, &t, np, err));
    DCK(cudaMemsetAsync(t, 0, np * sizeof(double), s));
    v.T = t - sh;
    if (!user0) {
        double *u = nullptr, *f = nullptr;
        DTRY(dmalloc(d, &u, np, err));
        DTRY(dmalloc(d, &f, np, err));
        DCK(cudaMemsetAsync(u, 0, np * sizeof(double), s));
        DCK(cudaMemsetAsync(f, 0, np * sizeof(double), s));
        v.u = u - sh;
        v.f = f - sh;
    }
    return BMG_OK;
}

static CIv civ_of(const SRank &R, int l)
{
    CIv c;
    const SLevel &vc = R.lv[l + 1];
    c.pitch = vc.pitch;
    c.roff = vc.roff;
    c.nrows = vc.nrows;
    for (int k = 0; k < 8; k++)
        c.w[k] = R.lv[l].ci[k];
    return c;
}

bmg_status_t dist_partition(int nx, int ny, int nranks, const bmg_params_t *prm, int *ybounds, int *kdist)
{
    if (nx < 1 || ny < 1 || nranks < 1 || !ybounds || !kdist)
        return BMG_EINVAL;
    bmg_params_t p;
    if (prm)
        p = *prm;
    else
        bmg_params_default(&p);
    std::vector<int> yb;
    int K = partition(nx, ny, nranks, p, yb);
    if (K < 1)
        return BMG_EINVAL;
    for (int i = 0; i <= nranks; i++)
        ybounds[i] = yb[i];
    *kdist = K;
    return BMG_OK;
}

// ------------------------------------------------------------------ peer mode (in-kernel ghost rows)
// One thread signals: after a leg, increment my count in each neighbour's flag array
// (system scope: the pushes of the leg, ordered before by the leg kernel's own system
// fences, are visible to the neighbour before it sees the count).
__global__ void k_peer_signal(unsigned long long *lo, unsigned long long *hi)
{
    __threadfence_system();
    if (lo)
        atomicAdd_system(&lo[1], 1ULL);  // I am my lower neighbour's upper neighbour
    if (hi)
        atomicAdd_system(&hi[0], 1ULL);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Before a leg: wait until each neighbour has signalled as many legs as I have waited
// for before (SPMD: every rank runs the same leg sequence), then count this wait.
// Bounded: a neighbour that never signals sets ERR_PEER instead of hanging the GPU.
__global__ void k_peer_wait(unsigned long long *mine, int has_lo, int has_hi, int *err)
{
    const unsigned long long e = mine[2];
    long long spins = 0;
    while ((has_lo && ld_acquire_sys(&mine[0]) < e) || (has_hi && ld_acquire_sys(&mine[1]) < e)) {
        __nanosleep(200);
        if (++spins > 50000000LL) {  // ~10 s
            atomicOr(err, ERR_PEER);
            break;
        }
    }
    __threadfence_system();
    mine[2] = e + 1;
}

static void peer_wait(DistSolver *d, cudaStream_t s)
{
    if (d->loopback)
        return;  // the ranks' legs run in stream order
    const int p = d->my_rank;
    k_peer_wait<<<1, 1, 0, s>>>(d->flags, p > 0, p + 1 < d->P, d->d_perr);
}

static void peer_signal(DistSolver *d, cudaStream_t s)
{
    if (d->loopback)
        return;
    k_peer_signal<<<1, 1, 0, s>>>(d->nflags[0], d->nflags[1]);
}

// Map the neighbours' T (every distributed level) and u, f (levels >= 1) arrays and flag
// arrays: loopback -- the other slabs of this process; NCCL -- CUDA IPC handles of the
// allocations, swapped with the neighbours by one grouped send/recv.
static bmg_status_t peer_setup(DistSolver *d, cudaStream_t s, std::string &err)
{
    const int K = d->K;
    if (K > 32) {
        err = "peer mode: more than 32 distributed levels";
        return BMG_EINVAL;
    }
    d->pp.assign(d->ranks.size(), std::vector<DistSolver::PeerPtrs>(K));
    if (d->loopback) {
        const int P = (int)d->ranks.size();
        for (int p = 0; p < P; p++)
            for (int l = 0; l < K; l++)
                for (int side = 0; side < 2; side++) {
                    const int q = side == 0 ? p - 1 : p + 1;
                    if (q < 0 || q >= P)
                        continue;
                    SLevel &v = d->ranks[q].lv[l];
                    d->pp[p][l].T[side] = v.T;
                    if (l > 0) {
                        d->pp[p][l].u[side] = v.u;
                        d->pp[p][l].f[side] = v.f;
                    }
                }
        return BMG_OK;
    }
    DCK(cudaMalloc(&d->flags, 4 * sizeof(unsigned long long)));
    d->allocs.push_back(d->flags);
    DCK(cudaMemsetAsync(d->flags, 0, 4 * sizeof(unsigned long long), s));
    DCK(cudaMalloc(&d->d_perr, sizeof(int)));
    d->allocs.push_back(d->d_perr);
    DCK(cudaMemsetAsync(d->d_perr, 0, sizeof(int), s));
    struct Msg {
        cudaIpcMemHandle_t T[32], u[32], f[32], flags;
        int roff[32];
    };
    Msg mine;
    memset(&mine, 0, sizeof mine);
    SRank &R = d->ranks[0];
    for (int l = 0; l < K; l++) {
        SLevel &v = R.lv[l];
        const long long sh = (long long)v.roff * v.pitch;
        mine.roff[l] = v.roff;
        DCK(cudaIpcGetMemHandle(&mine.T[l], v.T + sh));
        if (l > 0) {
            DCK(cudaIpcGetMemHandle(&mine.u[l], v.u + sh));
            DCK(cudaIpcGetMemHandle(&mine.f[l], v.f + sh));
        }
    }
    DCK(cudaIpcGetMemHandle(&mine.flags, d->flags));
    const size_t nd = (sizeof(Msg) + 7) / 8;  // as doubles
    double *buf = nullptr;
    DTRY(dmalloc(d, &buf, 3 * nd, err));
    DCK(cudaMemcpyAsync(buf, &mine, sizeof(Msg), cudaMemcpyHostToDevice, s));
    const int p = d->my_rank, P = d->P;
    ncclResult_t r = d->nccl.groupStart();
    for (int side = 0; side < 2 && r == ncclSuccess; side++) {
        const int q = side == 0 ? p - 1 : p + 1;
        if (q < 0 || q >= P)
            continue;
        r = d->nccl.recv(buf + (1 + side) * nd, nd, ncclDouble, q, d->comm, s);
        if (r == ncclSuccess)
            r = d->nccl.send(buf, nd, ncclDouble, q, d->comm, s);
    }
    ncclResult_t r2 = d->nccl.groupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
        err = std::string("peer handle exchange: ") + d->nccl.errstr(r != ncclSuccess ? r : r2);
        return BMG_ENCCL;
    }
    Msg nb[2];
    DCK(cudaMemcpyAsync(&nb[0], buf + nd, sizeof(Msg), cudaMemcpyDeviceToHost, s));
    DCK(cudaMemcpyAsync(&nb[1], buf + 2 * nd, sizeof(Msg), cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    auto open = [&](const cudaIpcMemHandle_t &h, void **out) -> bmg_status_t {
        DCK(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
        d->ipc.push_back(*out);
        return BMG_OK;
    };
    for (int side = 0; side < 2; side++) {
        const int q = side == 0 ? p - 1 : p + 1;
        if (q < 0 || q >= P)
            continue;
        void *m = nullptr;
        DTRY(open(nb[side].flags, &m));
        d->nflags[side] = (unsigned long long *)m;
        for (int l = 0; l < K; l++) {
            const long long sh = (long long)nb[side].roff[l] * R.lv[l].pitch;
            DTRY(open(nb[side].T[l], &m));
            d->pp[0][l].T[side] = (double *)m - sh;
            if (l > 0) {
                DTRY(open(nb[side].u[l], &m));
                d->pp[0][l].u[side] = (double *)m - sh;
                DTRY(open(nb[side].f[l], &m));
                d->pp[0][l].f[side] = (double *)m - sh;
            }
        }
    }
    return BMG_OK;
}

// the push of rank index ri's leg at level l: `fine` its output array's neighbour copies,
// `coarse` those of f_{l+1} (down legs, l+1 < K) -- nullptr: no push of that kind
static Push make_push(DistSolver *d, int ri, int l, double *const fine[2], double *const coarse[2])
{
    Push q;
    const SLevel &v = d->ranks[ri].lv[l];
    q.halo = BMG_HALO;
    q.ylo = v.ylo;
    q.yhi = v.yhi;
    if (fine) {
        q.lo = fine[0];
        q.hi = fine[1];
    }
    if (coarse && l + 1 < d->K) {
        const SLevel &c = d->ranks[ri].lv[l + 1];
        q.clo = coarse[0];
        q.chi = coarse[1];
        q.cylo = c.ylo;
        q.cyhi = c.yhi;
    }
    return q;
}

bmg_status_t dist_setup(const bmg_stencil_t *st, const bmg_comm_t *cm, const bmg_params_t *prm, cudaStream_t s,
                        DistSolver **out, std::string &err)
{
    *out = nullptr;
    DistSolver *d = new DistSolver();
    auto fail = [&](bmg_status_t rc) {
        dist_destroy(d);
        return rc;
    };
    if (prm)
        d->prm = *prm;
    else
        bmg_params_default(&d->prm);
    d->P = cm->nranks;
    d->loopback = cm->loopback != 0;
    d->peer = cm->peer != 0;
    d->nx = st->nx;
    d->ny = st->ny;
    d->kind0 = st->kind;
    if (!d->prm.fused || d->prm.relax != BMG_RELAX_POINT || d->prm.cycle_sym != 0 || d->prm.affine != 0 || (d->prm.nu1 != 1 && d->prm.nu1 != 2) ||
        (d->prm.nu2 != 1 && d->prm.nu2 != 2)) {
        err = "distributed solver needs the fused point-GS kernels (params.fused = 1, relax = BMG_RELAX_POINT, cycle_sym = 0, affine = 0, "
              "nu1, nu2 in {1, 2})";
        return fail(BMG_EINVAL);
    }
    d->K = partition(st->nx, st->ny, d->P, d->prm, d->yb);
    if (d->K < 1) {
        err = "grid too small for this many ranks (slabs below agglom_rows)";
        return fail(BMG_EINVAL);
    }
    if (!d->loopback) {
        if (!d->nccl.load(cm->nccl_lib, err))
            return fail(BMG_ENCCL);
        d->comm = (ncclComm_t)cm->nccl_comm;
        d->my_rank = cm->rank;
        if (!d->comm || cm->rank < 0 || cm->rank >= d->P) {
            err = "bad NCCL communicator or rank";
            return fail(BMG_EINVAL);
        }
    }
    const int nloc = d->loopback ? d->P : 1;
    d->ranks.resize(nloc);
    const int K = d->K;
    for (int i = 0; i < nloc; i++) {
        SRank &R = d->ranks[i];
        R.rank = d->loopback ? i : cm->rank;
        R.lv.resize(K + 1);
        int nx = st->nx, ny = st->ny;
        for (int l = 0; l <= K; l++) {
            const int kind = l == 0 ? st->kind : 9;
            const long long pitch = l == 0 ? st->pitch : rpitch(nx);
            // level 0 u/f: the caller's arrays (NCCL) or internal copies (loopback)
            DTRY(alloc_level(d, R, l, nx, ny, kind, pitch, l == 0 && !d->loopback, s, err) == BMG_OK
                     ? BMG_OK
                     : fail(BMG_ENOMEM));
            nx /= 2;
            ny /= 2;
        }
        for (int l = 0; l < K; l++) {  // weights from level l+1 live on level l+1's slab rows
            SLevel &vc = R.lv[l + 1];
            const size_t np = (size_t)vc.nrows * vc.pitch;
            double *blk = nullptr;
            if (dmalloc(d, &blk, np * 8, err) != BMG_OK)
                return fail(BMG_ENOMEM);
            cudaMemsetAsync(blk, 0, np * 8 * sizeof(double), s);
            for (int k = 0; k < 8; k++)
                R.lv[l].ci[k] = blk + k * np - (long long)vc.roff * vc.pitch;
        }
        void *q = nullptr;
        if (cudaMalloc(&q, 64 * sizeof(int)) != cudaSuccess)
            return fail(BMG_ENOMEM);
        d->allocs.push_back(q);
        R.d_err = (int *)q;
        cudaMemsetAsync(R.d_err, 0, 64 * sizeof(int), s);
        if (dmalloc(d, &R.partials, NORM_BLOCKS + 8, err) != BMG_OK || dmalloc(d, &R.d_norm, 8, err) != BMG_OK)
            return fail(BMG_ENOMEM);
        // fused plans of the slab levels (chunking over the owned rows)
        for (int l = 0; l < K; l++) {
            SLevel &v = R.lv[l];
            fused_plan_level(R.fp, l, v.nx, v.yhi - v.ylo, v.pitch, v.kind, d->prm.nu1, d->prm.nu2,
                             (v.pitch & 1) == 0);
            if (!(R.fp.lv[l].down && R.fp.lv[l].up)) {
                err = "slab level not supported by the fused kernels";
                return fail(BMG_EINVAL);
            }
        }
    }
    cudaMallocHost(&d->h_norm, 8 * sizeof(double));

    // S0: ingest the owned rows (and ring rows) of each rank's slab
    for (auto &R : d->ranks) {
        SLevel &v = R.lv[0];
        const long long srcsh = d->loopback ? 0 : (long long)v.roff * v.pitch;  // caller planes: local or global
        const double *src[5];
        for (int k = 0; k < 5; k++)
            src[k] = st->plane[k] ? st->plane[k] - srcsh : nullptr;
        int j0 = v.ylo == 1 ? 0 : v.ylo, j1 = v.yhi == v.ny + 1 ? v.ny + 2 : v.yhi;
        launch_ingest(v.nx, v.ny, v.kind, v.pitch, src, v.pl, R.d_err, s, j0, j1);
    }
    DTRY(exchange(d, 0, F_PL, s, err) == BMG_OK ? BMG_OK : fail(BMG_ENCCL));
    // S1 + S2 on the slab levels
    for (int l = 0; l < K; l++) {
        for (auto &R : d->ranks) {
            SLevel &v = R.lv[l], &vc = R.lv[l + 1];
            const int J0 = std::max(1, vc.ylo - 1);
            const int J1 = vc.yhi == vc.ny + 1 ? vc.ny + 1 : vc.yhi - 1;
            launch_setup_interp(v.op(), v.ci, vc.pitch, R.d_err, s, J0, J1);
        }
        DTRY(exchange(d, l, F_CI, s, err) == BMG_OK ? BMG_OK : fail(BMG_ENCCL));
        for (auto &R : d->ranks) {
            SLevel &v = R.lv[l], &vc = R.lv[l + 1];
            launch_setup_rap(v.op(), civ_of(R, l), vc.nx, vc.ny, vc.pitch, vc.pl, s, vc.ylo, vc.yhi - 1);
        }
        if (l + 1 < K)
            DTRY(exchange(d, l + 1, F_PL, s, err) == BMG_OK ? BMG_OK : fail(BMG_ENCCL));
    }
    // S3: gather the level-K operator, build the replicated inner solver
    {
        const SLevel &vK = d->ranks[0].lv[K];
        d->nxK = vK.nx;
        d->nyK = vK.ny;
        d->pitchK = vK.pitch;
        const long long npk = (long long)(d->nyK + 2) * d->pitchK;
        if (dmalloc(d, &d->plK, (size_t)npk * 5, err) != BMG_OK || dmalloc(d, &d->fK, (size_t)npk, err) != BMG_OK ||
            dmalloc(d, &d->xK, (size_t)npk, err) != BMG_OK)
            return fail(BMG_ENOMEM);
        cudaMemsetAsync(d->plK, 0, npk * 5 * sizeof(double), s);
        cudaMemsetAsync(d->fK, 0, npk * sizeof(double), s);
        cudaMemsetAsync(d->xK, 0, npk * sizeof(double), s);
        DTRY(allgather_rows(d, d->plK, npk, 5, 0, s, err) == BMG_OK ? BMG_OK : fail(BMG_ENCCL));
        int herr = 0;
        for (auto &R : d->ranks) {
            int e = 0;
            cudaMemcpyAsync(&e, R.d_err, sizeof(int), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            herr |= e;
        }
        if (cudaGetLastError() != cudaSuccess) {
            err = "CUDA error in distributed setup";
            return fail(BMG_ECUDA);
        }
        if (herr & ERR_DIAG) {
            err = "stencil diagonal a_O <= 0 at an interior point";
            return fail(BMG_EINVAL);
        }
        if (herr & ERR_DEN) {
            err = "interpolation denominator <= 0";
            return fail(BMG_EINVAL);
        }
        bmg_stencil_t sk;
        sk.kind = 9;
        sk.nx = d->nxK;
        sk.ny = d->nyK;
        sk.pitch = d->pitchK;
        for (int k = 0; k < 5; k++)
            sk.plane[k] = d->plK + k * npk;
        // the inner solver continues the SAME ladder from level K: partition() already
        // counted max_levels from level 0, so the inner hierarchy gets what is left
        bmg_params_t pin = d->prm;
        if (pin.max_levels > 0)
            pin.max_levels -= K;
        bmg_status_t rc = bmg_setup(&sk, &pin, s, &d->inner);
        if (rc != BMG_OK) {
            err = std::string("inner solver setup: ") + bmg_last_error_detail();
            return fail(rc);
        }
    }
    if (d->peer) {
        bmg_status_t rc = peer_setup(d, s, err);
        if (rc != BMG_OK)
            return fail(rc);
    }
    *out = d;
    return BMG_OK;
}

void dist_destroy(DistSolver *d)
{
    if (!d)
        return;
    cudaDeviceSynchronize();
    if (d->inner)
        bmg_destroy(d->inner);
    for (void *p : d->ipc)
        cudaIpcCloseMemHandle(p);
    for (void *p : d->allocs)
        cudaFree(p);
    if (d->h_norm)
        cudaFreeHost(d->h_norm);
    delete d;
}

bmg_solver_t dist_inner_solver(DistSolver *d) { return d->inner; }

void dist_local_rows(DistSolver *d, int *row0, int *nrows, int *ylo, int *yhi, int *kdist)
{
    const SLevel &v = d->ranks[0].lv[0];
    if (row0)
        *row0 = v.roff;
    if (nrows)
        *nrows = v.nrows;
    if (ylo)
        *ylo = v.ylo;
    if (yhi)
        *yhi = v.yhi;
    if (kdist)
        *kdist = d->K;
}

// ------------------------------------------------------------------ cycle
// Loopback: scatter the global rhs/x rows into every rank's level-0 arrays.
static void lb_scatter(DistSolver *d, const double *rhs, const double *x, cudaStream_t s)
{
    for (auto &R : d->ranks) {
        SLevel &v = R.lv[0];
        const long long o = (long long)v.roff * v.pitch;
        const size_t n = sizeof(double) * (size_t)v.nrows * v.pitch;
        cudaMemcpyAsync(v.f + o, rhs + o, n, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(v.u + o, x + o, n, cudaMemcpyDeviceToDevice, s);
    }
}

static void lb_gather(DistSolver *d, double *x, cudaStream_t s)
{
    for (auto &R : d->ranks) {
        SLevel &v = R.lv[0];
        const long long o = (long long)v.ylo * v.pitch;
        cudaMemcpyAsync(x + o, v.u + o, sizeof(double) * (size_t)(v.yhi - v.ylo) * v.pitch, cudaMemcpyDeviceToDevice,
                        s);
    }
}

static bmg_status_t one_cycle(DistSolver *d, cudaStream_t s, std::string &err)
{
    const int K = d->K;
    int n = 0;
    for (int l = 0; l < K; l++) {
        // level 0: u and f in one group; a coarse level starts from zero (c9), which
        // its fused down leg does not read -- only f's ghost rows move (peer mode: pushed
        // by the level above's restriction; wait for the neighbours' previous leg)
        if (l == 0)
            DTRY(exchange2(d, 0, F_U, 0, F_F, s, err));
        else if (!d->peer)
            DTRY(exchange(d, l, F_F, s, err));
        if (d->peer)
            peer_wait(d, s);
        for (size_t ri = 0; ri < d->ranks.size(); ri++) {
            SRank &R = d->ranks[ri];
            SLevel &v = R.lv[l];
            const bool last = l + 1 == K;
            double *fc = last ? d->fK : R.lv[l + 1].f;
            Push q;
            if (d->peer)
                q = make_push(d, (int)ri, l, d->pp[ri][l].T, last ? nullptr : d->pp[ri][l + 1].f);
            if (!fused_down(R.fp, l, v.op(), civ_of(R, l), v.f, l == 0 ? v.u : nullptr, v.T, fc, nullptr, s, &n,
                            d->peer ? &q : nullptr)) {
                err = "fused down leg rejected a slab level";
                return BMG_EINVAL;
            }
        }
        if (d->peer)
            peer_signal(d, s);
    }
    // level K: all-gather f_K, one inner V-cycle from a zero guess
    if (!d->loopback) {
        const long long npk = (long long)(d->nyK + 2) * d->pitchK;
        DTRY(allgather_rows(d, d->fK, npk, 1, 1, s, err));
    }
    cudaMemsetAsync(d->xK, 0, sizeof(double) * (size_t)(d->nyK + 2) * d->pitchK, s);
    DTRY(bmg_vcycle(d->inner, d->fK, d->xK, 1, s));
    for (int l = K - 1; l >= 0; l--) {
        if (d->peer)
            peer_wait(d, s);  // T_l and u_{l+1} were pushed by the neighbours' earlier legs
        else if (l + 1 < K)
            DTRY(exchange2(d, l, F_T, l + 1, F_U, s, err));
        else
            DTRY(exchange(d, l, F_T, s, err));
        for (size_t ri = 0; ri < d->ranks.size(); ri++) {
            SRank &R = d->ranks[ri];
            SLevel &v = R.lv[l];
            const bool last = l + 1 == K;
            const double *ec = last ? d->xK : R.lv[l + 1].u;
            const int eroff = last ? 0 : R.lv[l + 1].roff;
            const int enrows = last ? d->nyK + 2 : R.lv[l + 1].nrows;
            // level 0's u is the caller's array: its ghost rows move with the cycle-start exchange
            Push q;
            if (d->peer && l > 0)
                q = make_push(d, (int)ri, l, d->pp[ri][l].u, nullptr);
            if (!fused_up(R.fp, l, v.op(), civ_of(R, l), v.f, v.T, ec, eroff, enrows, v.u, s, &n,
                          d->peer && l > 0 ? &q : nullptr)) {
                err = "fused up leg rejected a slab level";
                return BMG_EINVAL;
            }
        }
        if (d->peer)
            peer_signal(d, s);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        err = std::string("distributed cycle: ") + cudaGetErrorString(e);
        return BMG_ECUDA;
    }
    return BMG_OK;
}

// In loopback mode the K=... level-K rhs rows are written by every rank's down leg
// straight into the shared fK (disjoint owned rows), so no all-gather is needed.
bmg_status_t dist_vcycle(DistSolver *d, const double *rhs, double *x, int ncycles, cudaStream_t s, std::string &err)
{
    if (d->loopback)
        lb_scatter(d, rhs, x, s);
    else {
        SLevel &v = d->ranks[0].lv[0];
        const long long sh = (long long)v.roff * v.pitch;
        v.f = const_cast<double *>(rhs) - sh;  // caller's local arrays (rows [roff, roff+nrows))
        v.u = x - sh;
    }
    for (int c = 0; c < ncycles; c++)
        DTRY(one_cycle(d, s, err));
    if (d->loopback)
        lb_gather(d, x, s);
    return BMG_OK;
}

bmg_status_t dist_resid_norm(DistSolver *d, const double *rhs, const double *x, double *norm, cudaStream_t s,
                             std::string &err)
{
    if (d->loopback)
        lb_scatter(d, rhs, x, s);
    else {
        SLevel &v = d->ranks[0].lv[0];
        const long long sh = (long long)v.roff * v.pitch;
        v.f = const_cast<double *>(rhs) - sh;
        v.u = const_cast<double *>(x) - sh;
    }
    DTRY(exchange(d, 0, F_U, s, err));
    double acc = 0.0;
    for (auto &R : d->ranks) {
        SLevel &v = R.lv[0];
        launch_resid_norm(v.op(), v.f, v.u, nullptr, R.partials, R.d_norm, s);
        cudaMemcpyAsync(d->h_norm, R.d_norm, sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        acc += d->h_norm[0] * d->h_norm[0];
    }
    if (!d->loopback && d->P > 1) {
        // all-reduce the local sum of squares (one double) over NCCL
        SRank &R = d->ranks[0];
        d->h_norm[1] = acc;
        cudaMemcpyAsync(R.d_norm + 1, &d->h_norm[1], sizeof(double), cudaMemcpyHostToDevice, s);
        ncclResult_t r = d->nccl.allReduce(R.d_norm + 1, R.d_norm + 2, 1, ncclDouble, ncclSum, d->comm, s);
        if (r != ncclSuccess) {
            err = std::string("NCCL all-reduce: ") + d->nccl.errstr(r);
            return BMG_ENCCL;
        }
        cudaMemcpyAsync(&d->h_norm[2], R.d_norm + 2, sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        acc = d->h_norm[2];
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        err = std::string("distributed norm: ") + cudaGetErrorString(e);
        return BMG_ECUDA;
    }
    if (d->peer && d->d_perr) {  // a peer wait that gave up (a neighbour never signalled)
        int pe = 0;
        cudaMemcpy(&pe, d->d_perr, sizeof(int), cudaMemcpyDeviceToHost);
        if (pe & ERR_PEER) {
            err = "peer mode: a neighbour's leg signal never arrived (wait timed out)";
            return BMG_ENCCL;
        }
    }
    *norm = sqrt(acc);
    return BMG_OK;
}

}  // namespace bmg
