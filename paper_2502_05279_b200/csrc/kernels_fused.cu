// kernels_fused.cu -- fused streaming kernels for the large levels
// (interface in fused.cuh).
//
// Down leg of a level in ONE pass over HBM (row step t):
//   split of the freshly landed row t; colour stage k = 1..NS (NS = 2 nu1) of
//   multicolour GS (c6) on row t-2k; residual on row t-2NS-2; restriction
//   (fig:restrict_kernel) of coarse row J = (t-2NS-4)/2; store of
//   the final iterate row t-2NS-3.
// Up leg in ONE pass:
//   split of row t; interpolation + correction (c7) on row t-1; stage k on
//   row t-1-2k; store of row t-2NS-2.
// Each task runs in its own warp group; groups are decoupled: a group waits only
// on the step-completion mbarriers of the groups it reads from (or whose ring
// slots it overwrites), so a slow task delays its consumers, not the whole CTA.
// A 9-point row stage is two colour phases (even columns, then odd columns)
// ordered by a barrier over its group only.
//
// Memory path: rows of u_in, f and the operator planes arrive by tensor TMA
// (one 2-D box for u and f each, one 3-D box for the plane block; mbarrier
// complete_tx) into a staging ring D rows ahead, in natural order.  A split task de-interleaves
// each row into [even columns | odd columns] halves of the main ring, so every
// compute access -- a colour pass touches every other column -- is a run of
// consecutive doubles across a warp (no shared-memory bank conflicts).  Coarse
// rows (interpolation weights, coarse correction) use their own 4-slot ring.
// A CTA owns TX output columns x a chunk of rows and recomputes an x halo H
// and a row warm-up that its neighbours own (same per-point arithmetic, so the
// owners' values are reproduced exactly); u is ping-ponged (u_in -> u_out).
//
// Thread mapping: NG warp-aligned task groups; a thread owns PPT column pairs
// h (smem columns 2h, 2h+1), h lane-consecutive.  Each group does one kind of
// task per step (a colour stage, a residual parity, store, restriction, split),
// loading all operands of its points before the arithmetic.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

#include "fused.cuh"

namespace bmg {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

// try_wait suspend-time hint (ns): a waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-polling and taking issue slots.
#ifndef BMG_WAIT_HINT
#define BMG_WAIT_HINT 0x989680
#endif
// BMG_WAIT_NS > 0: poll with mbarrier.test_wait and back off BMG_WAIT_NS ns between
// probes (fewer issue slots spent by waiting warps) instead of the try_wait loop.
#ifndef BMG_WAIT_NS
#define BMG_WAIT_NS 0
#endif
__device__ __forceinline__ bool mbar_test(uint32_t addr, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity)
{
    if (BMG_WAIT_NS > 0) {
        while (!mbar_test(smem_u32(b), parity))
            __nanosleep(BMG_WAIT_NS);
        return;
    }
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_LOOP:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_LOOP;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity), "r"(BMG_WAIT_HINT)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// barrier among the `n` threads (whole warps) of one task group
__device__ __forceinline__ void group_sync(int id, int n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Tiled tensor TMA: one box (out-of-bounds elements zero-filled) into smem.
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *m, int x, int y, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(smem_u32(b))
        : "memory");
}

__device__ __forceinline__ void tma_3d(void *dst, const CUtensorMap *m, int x, int y, int z, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b))
        : "memory");
}

// L2 prefetch of one tensor box (no shared memory, no completion): the rows far
// ahead of the shared-memory ring are pulled into L2 so that the ring's TMA loads
// hit L2 -- the ring's depth (bytes in flight per SM) is bounded by shared memory.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *m, int x, int y)
{
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(x), "r"(y)
                 : "memory");
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *m, int x, int y, int z)
{
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(x), "r"(y), "r"(z)
                 : "memory");
}

// rows beyond the ring's prefetch depth D that are prefetched into L2 (0: none; measured no
// gain at 4..32 rows, DESIGN §10 -- kept as a tuning knob)
#ifndef BMG_L2PF
#define BMG_L2PF 0
#endif

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// ------------------------------------------------------------------ configuration
constexpr int DC = 4;  // coarse-row prefetch distance (row steps), up leg (4-slot ring)
constexpr int DC_DN = 3;  // down leg (3-slot weight ring: 2 slots in use + 1 in flight)
constexpr int CH = 4;  // coarse halo columns on each side of a strip
constexpr int NSLOT = 32;  // slots of each task group's step-completion ring

// streamed arrays: index into the shared-memory array blocks
enum { A_U = 0, A_F = 1, A_O = 2, A_W = 3, A_S = 4, A_SW = 5, A_NW = 6 };

template <int KIND, int NS, int WD, int D, bool UP, int PPT, int E>
struct Cfg {
    static constexpr int NA = KIND == 5 ? 5 : 7;                // streamed arrays
    static constexpr int NM = NA + 1;                           // main-ring arrays: + 1/O
    static constexpr int A_DI = NA;                             // main-ring index of 1/O
    static constexpr int CSL = UP ? 4 : 3;                      // coarse-row ring slots
    // weight planes per coarse row: the up leg interpolates with all 8; the down
    // leg restricts a residual that vanishes on the colour relaxed last (DESIGN
    // §5.2), so it needs only the other half: the 4 Z-point weights (5-point
    // levels) or the 4 X/Y weights (9-point levels), one contiguous block
    // The up leg's first colour pass recomputes its points from the other colours
    // only, so their correction is never read: a 5-point up leg corrects only X/Y
    // points (4 X/Y weight planes); a 9-point one skips the C injection (all 8).
    static constexpr int NWP = UP ? (KIND == 5 ? 4 : 8) : 4;
    static constexpr int WP0 = UP ? (KIND == 5 ? CI_LR : 0) : (KIND == 5 ? CI_LNE : CI_LR);  // first plane
    static constexpr int PASSES = KIND == 5 ? NS : 2 * NS;      // colour passes (x halo shrink)
    static constexpr int H0 = UP ? PASSES : PASSES + 2;         // + residual + restriction
    static constexpr int H = ((H0 < 2 ? 2 : H0) + 1) & ~1;      // even (16-byte TMA alignment)
    static constexpr int TX = WD - 2 * H;                      // output columns (multiple of 4)
    static constexpr int HW = WD / 2;                          // half row (one parity)
    static constexpr int RM = (UP ? 2 * NS + 3 : 2 * NS + 4) + E;  // main (split) ring rows; E = extra slack
    static constexpr int SD = D + 1;                           // staging (natural) ring rows
    static constexpr int AM = RM * WD, AS = SD * WD;           // doubles per array block
    static constexpr int WC = (TX / 2 + 2 * CH + 15) / 16 * 16;  // coarse box width (128-B rows)
    static constexpr int NPG = HW / PPT;                       // threads per task group
    static constexpr int NSPLIT = 2;                           // split task groups
    // one warp group per colour stage (a 9-point stage is active every other row step,
    // so its group may take two steps per row), + residual/correction, store, restriction, split
    static constexpr int NG = UP ? NS + 3 + NSPLIT : NS + 4 + NSPLIT;
    static constexpr int NTW = NG * NPG;                       // worker threads
    static constexpr int NT = NTW + 32;                        // + one TMA producer warp
    static constexpr size_t SMEM_DBL =
        (size_t)NM * AM + (size_t)NA * AS + (UP ? 4 * (size_t)WC : 4 * (size_t)WD) + (size_t)NWP * CSL * (size_t)WC;
    static constexpr size_t SMEM = SMEM_DBL * 8 + (SD + 4 + (size_t)NG * NSLOT) * 8;
    static_assert(TX % 4 == 0 && TX > 0, "strip width");
    static_assert(NPG % 32 == 0, "task groups must be whole warps");
};

// Step-completion rings, one per waiting task: ring r slot (t mod NSLOT)
// completes when every warp of the groups that task depends on has finished
// row step t (each warp arrives once, after __syncwarp).  A task therefore waits
// on exactly one mbarrier per step.  Every dependency cycle of the pipeline
// spans fewer than NSLOT steps, so no warp is ever NSLOT steps ahead of a waiter
// or of another warp arriving on the same ring.
struct Rings {
    uint32_t base;  // shared-memory address of ring 0, slot 0
    int lo;         // first row step
    __device__ __forceinline__ uint32_t at(int r, int t) const
    {
        return base + 8u * (uint32_t)(r * NSLOT + ((t - lo) & (NSLOT - 1)));
    }
    __device__ __forceinline__ void arrive(int r, int t) const
    {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(at(r, t)) : "memory");
    }
    __device__ __forceinline__ void wait(int r, int t) const
    {
        if (t < lo)
            return;
        const uint32_t par = ((t - lo) / NSLOT) & 1;
        if (BMG_WAIT_NS > 0) {
            while (!mbar_test(at(r, t), par))
                __nanosleep(BMG_WAIT_NS);
            return;
        }
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "RWAIT:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
            "@!P1 bra RWAIT;\n"
            "}\n" ::"r"(at(r, t)),
            "r"(par), "r"(BMG_WAIT_HINT)
            : "memory");
    }
    // end of step t for one warp: arrive on rings a, b, c (-1: none)
    __device__ __forceinline__ void done(int t, int a, int b, int c) const
    {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
            if (a >= 0)
                arrive(a, t);
            if (b >= 0)
                arrive(b, t);
            if (c >= 0)
                arrive(c, t);
        }
    }
};

struct FArgs {
    Op A;
    CIv ci;
    const double *f, *uin, *ec;
    double *uout, *fc, *uc;
    int nstrips, chunk, ncx, ncy;
    int eroff;  // stored-row offset of the coarse correction e (up leg)
    int uzero;  // down leg: u_in == 0 (a coarse level's zero start, c9) -- not read
    Push push;  // ghost rows also stored into the neighbours' arrays (peer mode)
};

// Peer mode (Push): the owned row w (columns c, c+1) also into the neighbours' ghost
// rows when it lies within `halo` rows of the slab's edge; system fence so that the
// leg's completion signal (dist.cu) orders these remote stores.  Out of line: the
// single-GPU legs pay one uniform branch.
__device__ __noinline__ void push_row(const Push &q, int w, long long off, int c, int nx, double ve, double vo)
{
    double *t[2] = {q.lo && w < q.ylo + q.halo ? q.lo : nullptr, q.hi && w >= q.yhi - q.halo ? q.hi : nullptr};
    for (int k = 0; k < 2; k++) {
        if (!t[k])
            continue;
        double *dst = t[k] + off;
        if (c >= 1 && c + 1 <= nx)
            *reinterpret_cast<double2 *>(dst) = make_double2(ve, vo);
        else {
            if (c >= 1 && c <= nx)
                dst[0] = ve;
            if (c + 1 >= 1 && c + 1 <= nx)
                dst[1] = vo;
        }
        __threadfence_system();
    }
}

__device__ __noinline__ void push_coarse(const Push &q, int J, long long off, double v)
{
    if (q.clo && J < q.cylo + q.halo) {
        q.clo[off] = v;
        __threadfence_system();
    }
    if (q.chi && J >= q.cyhi - q.halo) {
        q.chi[off] = v;
        __threadfence_system();
    }
}

// TMA descriptors of one launch (kernel parameter, __grid_constant__):
// u (rows of u_in), f, a (the operator's plane block, 3-D), c (the 8 weight
// planes, 3-D), e (coarse correction, up leg).
struct TMaps {
    CUtensorMap u, f, a, c, e;
};

// ring slot of the row `d` rows behind the newest (ts = slot of row t)
template <int R>
__device__ __forceinline__ int back(int ts, int d)
{
    int s = ts - d;
    return s < 0 ? s + R : s;
}

// Offsets (within a split row) of smem column sc = 2h+par and of its x neighbours.
struct Col {
    int same, left, right;
};
template <int HW>
__device__ __forceinline__ Col col_of(int h, int par)
{
    Col c;
    c.same = par * HW + h;
    c.left = (1 - par) * HW + h + par - 1;
    c.right = c.left + 1;
    return c;
}

// Loads of the operands of one point (row bases b0/bm/bp = slot*WD of rows r, r-1, r+1),
// off-diagonal terms in fig:stencil_operator order SW,S,SE,W,E,NW,N,NE; `o` is
// main-ring array OI (A_O: the diagonal; the colour passes load 1/a_pp instead).
template <int KIND, int AM, int OI>
struct PointOps {
    double a[8], u[8], f, o, uc;
    __device__ __forceinline__ void load(const double *sm, int b0, int bm, int bp, const Col &c, bool with_uc)
    {
        if (KIND == 5) {
            a[0] = sm[A_S * AM + b0 + c.same];
            u[0] = sm[A_U * AM + bm + c.same];
            a[1] = sm[A_W * AM + b0 + c.same];
            u[1] = sm[A_U * AM + b0 + c.left];
            a[2] = sm[A_W * AM + b0 + c.right];
            u[2] = sm[A_U * AM + b0 + c.right];
            a[3] = sm[A_S * AM + bp + c.same];
            u[3] = sm[A_U * AM + bp + c.same];
        } else {
            a[0] = sm[A_SW * AM + b0 + c.same];
            u[0] = sm[A_U * AM + bm + c.left];
            a[1] = sm[A_S * AM + b0 + c.same];
            u[1] = sm[A_U * AM + bm + c.same];
            a[2] = sm[A_NW * AM + bm + c.right];
            u[2] = sm[A_U * AM + bm + c.right];
            a[3] = sm[A_W * AM + b0 + c.same];
            u[3] = sm[A_U * AM + b0 + c.left];
            a[4] = sm[A_W * AM + b0 + c.right];
            u[4] = sm[A_U * AM + b0 + c.right];
            a[5] = sm[A_NW * AM + b0 + c.same];
            u[5] = sm[A_U * AM + bp + c.left];
            a[6] = sm[A_S * AM + bp + c.same];
            u[6] = sm[A_U * AM + bp + c.same];
            a[7] = sm[A_SW * AM + bp + c.right];
            u[7] = sm[A_U * AM + bp + c.right];
        }
        f = sm[A_F * AM + b0 + c.same];
        o = sm[OI * AM + b0 + c.same];
        if (with_uc)
            uc = sm[A_U * AM + b0 + c.same];
    }
    __device__ __forceinline__ double offdiag() const
    {
        constexpr int NT = KIND == 5 ? 4 : 8;
        double acc = a[0] * u[0];
#pragma unroll
        for (int q = 1; q < NT; q++)
            acc += a[q] * u[q];
        return acc;
    }
};

// Per-thread column data for its PPT pairs, both parities (loop invariant).
// Neighbour offsets of a split row never leave the row (par 0: left/right in
// the odd half; par 1: in the even half), so no clamping is needed; `on` marks
// the points inside [1,nx] that may be stored.
template <int PPT>
struct Cols {
    Col c[2][PPT];
    bool on[2][PPT];
};

template <int WD, int PPT, int NPG>
__device__ __forceinline__ Cols<PPT> make_cols(int m, int xl, int nx)
{
    constexpr int HW = WD / 2;
    Cols<PPT> k;
#pragma unroll
    for (int par = 0; par < 2; par++)
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            const int h = m + p * NPG, sc = 2 * h + par, c = xl + sc;
            k.c[par][p] = col_of<HW>(h, par);
            k.on[par][p] = c >= 1 && c <= nx && sc >= 1 && sc <= WD - 2;
        }
    return k;
}

// One colour pass (c6: u <- (f - sum_{q!=p} a_pq u_q) / a_pp) on row r for this
// thread's PPT pairs, column parity PAR.  Points outside [1,nx] are computed but not stored.
// The division is a multiplication by 1/a_pp (rcp_pos, bmg_internal.cuh), formed
// once per point and row pass by the split task: it keeps the
// reciprocal's dependent FP64 chain off the colour stages, whose latency bounds
// the pipeline's row step.
template <int KIND, int AM, int WD, int PPT, int PAR>
__device__ __forceinline__ void colour_pass(double *sm, int s0, int sm1, int sp1, const Cols<PPT> &k)
{
    PointOps<KIND, AM, KIND == 5 ? 5 : 7> pt[PPT];
#pragma unroll
    for (int p = 0; p < PPT; p++)
        pt[p].load(sm, s0 * WD, sm1 * WD, sp1 * WD, k.c[PAR][p], false);
#pragma unroll
    for (int p = 0; p < PPT; p++) {
        const double v = (pt[p].f - pt[p].offdiag()) * pt[p].o;
        if (k.on[PAR][p])
            sm[A_U * AM + s0 * WD + k.c[PAR][p].same] = v;
    }
}

template <int KIND, int AM, int WD, int PPT>
__device__ __forceinline__ void colour_pass(double *sm, int s0, int sm1, int sp1, int par, const Cols<PPT> &k)
{
    if (par)
        colour_pass<KIND, AM, WD, PPT, 1>(sm, s0, sm1, sp1, k);
    else
        colour_pass<KIND, AM, WD, PPT, 0>(sm, s0, sm1, sp1, k);
}

// The two colour phases of a 9-point row stage (forward order: even columns, then odd),
// phase B reusing what phase A of the same thread already holds.  A thread owns the
// column pair (2h, 2h+1): phase A updates 2h, phase B 2h+1, and B's operands include
// A's u at rows r-1 and r+1 (columns 2h, 2h+1), A's own new value u(2h) and the coupling
// W(2h+1) (= E of 2h): 6 of B's 18 shared-memory loads.  Same terms in the same order
// as colour_pass, so the same bits.  `bar`: the group's named barrier (B reads A's
// results of the neighbouring lanes).
template <int AM, int WD, int PPT>
__device__ __forceinline__ void colour_pair9(double *sm, int s0, int sm1, int sp1, const Cols<PPT> &k, int bar,
                                             int nthreads)
{
    constexpr int OI = 7;
    const int b0 = s0 * WD, bm = sm1 * WD, bp = sp1 * WD;
    double keep[PPT][6];  // u(r-1,2h), u(r-1,2h+1), u(r+1,2h), u(r+1,2h+1), W(2h+1), new u(2h)
#pragma unroll
    for (int p = 0; p < PPT; p++) {
        const Col c = k.c[0][p];  // same = h, left = HW+h-1 (2h-1), right = HW+h (2h+1)
        double a[8], u[8];
        a[0] = sm[A_SW * AM + b0 + c.same];
        u[0] = sm[A_U * AM + bm + c.left];
        a[1] = sm[A_S * AM + b0 + c.same];
        u[1] = sm[A_U * AM + bm + c.same];
        a[2] = sm[A_NW * AM + bm + c.right];
        u[2] = sm[A_U * AM + bm + c.right];
        a[3] = sm[A_W * AM + b0 + c.same];
        u[3] = sm[A_U * AM + b0 + c.left];
        a[4] = sm[A_W * AM + b0 + c.right];
        u[4] = sm[A_U * AM + b0 + c.right];
        a[5] = sm[A_NW * AM + b0 + c.same];
        u[5] = sm[A_U * AM + bp + c.left];
        a[6] = sm[A_S * AM + bp + c.same];
        u[6] = sm[A_U * AM + bp + c.same];
        a[7] = sm[A_SW * AM + bp + c.right];
        u[7] = sm[A_U * AM + bp + c.right];
        const double f = sm[A_F * AM + b0 + c.same], o = sm[OI * AM + b0 + c.same];
        double acc = a[0] * u[0];
#pragma unroll
        for (int q = 1; q < 8; q++)
            acc += a[q] * u[q];
        const double v = (f - acc) * o;
        if (k.on[0][p])
            sm[A_U * AM + b0 + c.same] = v;
        keep[p][0] = u[1];
        keep[p][1] = u[2];
        keep[p][2] = u[6];
        keep[p][3] = u[7];
        keep[p][4] = a[4];
        keep[p][5] = k.on[0][p] ? v : sm[A_U * AM + b0 + c.same];
    }
    group_sync(bar, nthreads);
#pragma unroll
    for (int p = 0; p < PPT; p++) {
        const Col c = k.c[1][p];  // same = HW+h (2h+1), left = h (2h), right = h+1 (2h+2)
        double a[8], u[8];
        a[0] = sm[A_SW * AM + b0 + c.same];
        u[0] = keep[p][0];
        a[1] = sm[A_S * AM + b0 + c.same];
        u[1] = keep[p][1];
        a[2] = sm[A_NW * AM + bm + c.right];
        u[2] = sm[A_U * AM + bm + c.right];
        a[3] = keep[p][4];
        u[3] = keep[p][5];
        a[4] = sm[A_W * AM + b0 + c.right];
        u[4] = sm[A_U * AM + b0 + c.right];
        a[5] = sm[A_NW * AM + b0 + c.same];
        u[5] = keep[p][2];
        a[6] = sm[A_S * AM + bp + c.same];
        u[6] = keep[p][3];
        a[7] = sm[A_SW * AM + bp + c.right];
        u[7] = sm[A_U * AM + bp + c.right];
        const double f = sm[A_F * AM + b0 + c.same], o = sm[OI * AM + b0 + c.same];
        double acc = a[0] * u[0];
#pragma unroll
        for (int q = 1; q < 8; q++)
            acc += a[q] * u[q];
        if (k.on[1][p])
            sm[A_U * AM + b0 + c.same] = (f - acc) * o;
    }
}

// De-interleave staging row (natural order, slot ss) into main ring row (slot s0)
// for arrays [q0, q1): even columns to the first half, odd to the second.
// DI: also form 1/a_pp (rcp_pos) into main-ring array NA.
template <int NA, int AM, int WD, int PPT, int NPG, bool DI>
__device__ __forceinline__ void split_row(double *smM, const double *smS, int ss, int s0, int q0, int q1, int m)
{
    constexpr int HW = WD / 2;
    if (DI) {
        double2 v[PPT];
#pragma unroll
        for (int p = 0; p < PPT; p++)
            v[p] = *reinterpret_cast<const double2 *>(smS + (ss * NA + A_O) * WD + 2 * (m + p * NPG));
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            double *row = smM + NA * AM + s0 * WD;
            row[m + p * NPG] = rcp_pos(v[p].x);  // ring / out-of-range columns: never stored
            row[HW + m + p * NPG] = rcp_pos(v[p].y);
        }
    }
#pragma unroll
    for (int q = 0; q < 7; q++) {
        if (q < q0 || q >= q1)
            continue;
        double2 v[PPT];
#pragma unroll
        for (int p = 0; p < PPT; p++)
            v[p] = *reinterpret_cast<const double2 *>(smS + (ss * NA + q) * WD + 2 * (m + p * NPG));
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            double *row = smM + q * AM + s0 * WD;
            row[m + p * NPG] = v[p].x;
            row[HW + m + p * NPG] = v[p].y;
        }
    }
}

// ------------------------------------------------------------------ down kernel
// PUSH: the peer mode's ghost-row stores (a separate instance: the single-GPU legs'
// code is unchanged by them)
template <int KIND, int NS, int WD, int D, int PPT, int E, bool PUSH = false>
__global__ void __launch_bounds__(Cfg<KIND, NS, WD, D, false, PPT, E>::NT, 1)
    k_fused_down(FArgs a, const __grid_constant__ TMaps tmaps)
{
    using C = Cfg<KIND, NS, WD, D, false, PPT, E>;
    constexpr int NA = C::NA, H = C::H, TX = C::TX, WC = C::WC, HW = C::HW, NPG = C::NPG;
    constexpr int RM = C::RM, SD = C::SD, AM = C::AM, AS = C::AS;
    extern __shared__ __align__(128) double sm[];
    double *smS = sm + C::NM * AM;              // staging ring (natural rows)
    double *sR = smS + NA * AS;                 // residual ring [4][WD], split
    double *sC = sR + 4 * WD;                   // weights ring [4][8][WC]
    uint64_t *bar = (uint64_t *)(sC + C::NWP * C::CSL * WC); // SD staging + 4 coarse

    const int nx = a.A.nx, ny = a.A.ny, ncx = a.ncx;
    const long long P = a.A.pitch, CP = a.ci.pitch;
    const int strip = blockIdx.x % a.nstrips, chunk = blockIdx.x / a.nstrips;
    const int x0 = strip * TX, xl = x0 - H;
    const int ya = a.A.ylo + chunk * a.chunk, yb = min(a.A.yhi, ya + a.chunk);
    if (ya >= yb)
        return;
    const int lo = max(ya - NS - 2, a.A.roff), hi = min(yb + NS + 1, a.A.roff + a.A.nrows - 1);
    const int cxl = x0 / 2 - CH;
    const int Jlo = (ya + 1) / 2, Jhi = min((yb - 1) / 2, a.ncy);  // restricted rows: 2J in [ya, yb)
    const int Kend = Jhi >= Jlo ? Jhi + 1 : Jlo - 1;

    const int tid = threadIdx.x, grp = tid / NPG, m = tid % NPG;
    const bool producer = tid == C::NTW;  // lane 0 of the producer warp issues every TMA copy
    // Task groups (warp-aligned, one task per row step):
    //  5-point: 0..NS-1 colour stage k = grp+1; NS, NS+1 residual of even/odd columns;
    //           NS+2 store; NS+3 restriction; NS+4, NS+5 split.
    //  9-point: 0..NS-1 colour stage k = grp+1, active on every other row step (its row
    //           parity), phase A even columns, phase B odd; then as 5-point.
    constexpr int NSG = NS;  // colour-stage groups
    constexpr int G_RES = NSG, G_STORE = NSG + 2, G_SPLIT = NSG + 4;  // restriction: NSG + 3
    // Rings (waiter <- groups it depends on, at step t-1 unless noted):
    //  g < NSG  stage group g <- split (g = 0) or stage group g-1: row r+1 = t-2k+1
    //  R_RES    residual <- last stage group(s) (row rr+1), restriction (residual-ring slot)
    //  R_STORE  store <- last stage group(s), at step t-3
    //  R_RESTR  restriction <- residual groups
    //  R_SPLIT  split <- residual groups, store (the main slot's old row t-RM)
    //  R_PROD   producer <- split groups (staging slot of row t-1), restriction (weight slot)
    constexpr int W = NPG / 32;
    constexpr int R_RES = NSG, R_STORE = NSG + 1, R_RESTR = NSG + 2, R_SPLIT = NSG + 3, R_PROD = NSG + 4;
    constexpr int NR = NSG + 5;
    static_assert(NR <= C::NG, "ring space");
    const Rings rg{smem_u32(bar + SD + 4), lo};

    if (a.uzero)  // the zero start is never read from HBM: its staging rows stay 0
        for (int i = tid; i < SD * WD; i += C::NT)
            smS[(i / WD) * (NA * WD) + A_U * WD + i % WD] = 0.0;
    if (tid == 0) {
        for (int i = 0; i < SD + 4; i++)
            mbar_init(&bar[i], 1);
        for (int r = 0; r < NR; r++) {
            const int cnt = r < NSG ? (r == 0 ? 2 * W : W)
                            : r == R_RES ? (KIND == 5 ? 2 : 3) * W
                            : r == R_STORE ? (KIND == 5 ? 1 : 2) * W
                            : r == R_RESTR ? 2 * W : 3 * W;
            for (int q = 0; q < NSLOT; q++)
                mbar_init(bar + SD + 4 + r * NSLOT + q, cnt);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // Staging slot s holds NA natural rows [U | F | O W S (SW NW)], one TMA box
    // each for u and f and ONE 3-D box for the operator's plane block.
    int Knext = Jlo;
    auto issue_row = [&](int row) {
        const int slot = (row - lo) % SD;
        uint64_t *b = &bar[slot];
        mbar_arrive_tx(b, (uint32_t)((a.uzero ? NA - 1 : NA) * WD * 8));
        double *d = smS + slot * (NA * WD);
        if (!a.uzero)
            tma_2d(d + A_U * WD, &tmaps.u, xl, row - a.A.roff, b);
        tma_2d(d + A_F * WD, &tmaps.f, xl, row - a.A.roff, b);
        tma_3d(d + A_O * WD, &tmaps.a, xl, row - a.A.roff, 0, b);
    };
    auto issue_coarse = [&](int t) {
        while (Knext <= Kend) {
            const int use = (Knext == Jlo) ? 2 * Jlo + 2 * NS + 4 : 2 * Knext + 2 * NS + 2;
            if (use - DC_DN > t)
                break;
            const int slot = (Knext - Jlo) % C::CSL;
            uint64_t *b = &bar[SD + slot];
            mbar_arrive_tx(b, (uint32_t)(C::NWP * WC * 8));
            tma_3d(sC + slot * C::NWP * WC, &tmaps.c, cxl, Knext - a.ci.roff, C::WP0, b);
            Knext++;
        }
    };
    if (producer)
        for (int row = lo; row <= min(lo + D - 1, hi); row++)
            issue_row(row);

    const Cols<PPT> kc = make_cols<WD, PPT, NPG>(m, xl, nx);

    // residual of row rr at the columns of parity e of this thread's pairs;
    // 0 off the interior (the restriction reads the ring as zeros)
    auto resid_par = [&](int rr, int s0, int sm1, int sp1, auto PARC) {
        constexpr int e = decltype(PARC)::value;
        const bool rin = rr >= 1 && rr <= ny;
        PointOps<KIND, AM, A_O> pt[PPT];
#pragma unroll
        for (int p = 0; p < PPT; p++)
            pt[p].load(sm, s0 * WD, sm1 * WD, sp1 * WD, kc.c[e][p], true);
        double *rrow = sR + (rr & 3) * WD;
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            const double v = pt[p].f - (pt[p].o * pt[p].uc + pt[p].offdiag());
            rrow[kc.c[e][p].same] = (rin && kc.on[e][p]) ? v : 0.0;
        }
    };
    auto resid_task = [&](int rr, int s0, int sm1, int sp1, int e) {
        if (rr < ya - 1 || rr > yb || rr < 0 || rr > ny + 1)
            return;
        // the colour relaxed last has zero residual (each of its points was just
        // solved against final neighbours of the other colours); the restriction
        // never reads it: 5-point black (i + rr odd), 9-point colour 3 (i, rr odd)
        if (KIND == 5 ? ((e + rr) & 1) : (e & rr & 1))
            return;
        if (e)
            resid_par(rr, s0, sm1, sp1, std::integral_constant<int, 1>());
        else
            resid_par(rr, s0, sm1, sp1, std::integral_constant<int, 0>());
    };
    // store of the final iterate row w (main slot sw), columns (2h, 2h+1) of the owned strip
    auto store_task = [&](int w, int sw) {
        if (w < ya || w >= yb)
            return;
        const double *urow = sm + A_U * AM + sw * WD;
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            const int h = m + p * NPG, sc = 2 * h, c = xl + sc;
            if (sc < H || sc >= H + TX)
                continue;
            double *dst = a.uout + (long long)w * P + c;
            const double ve = urow[h], vo = urow[HW + h];
            if (c >= 1 && c + 1 <= nx)
                *reinterpret_cast<double2 *>(dst) = make_double2(ve, vo);
            else {
                if (c >= 1 && c <= nx)
                    dst[0] = ve;
                if (c + 1 >= 1 && c + 1 <= nx)
                    dst[1] = vo;
            }
            if constexpr (PUSH)
                push_row(a.push, w, (long long)w * P + c, c, nx, ve, vo);
        }
    };
    // restriction (fig:restrict_kernel) of coarse row J at the coarse points centred on columns 2h
    auto restrict_task = [&](int J) {
        constexpr int CS = C::CSL;
        mbar_wait(&bar[SD + (J - Jlo) % CS], ((J - Jlo) / CS) & 1);
        mbar_wait(&bar[SD + (J + 1 - Jlo) % CS], ((J + 1 - Jlo) / CS) & 1);
        const double *rm = sR + ((2 * J - 1) & 3) * WD, *r0 = sR + ((2 * J) & 3) * WD,
                     *rp = sR + ((2 * J + 1) & 3) * WD;
        constexpr int NW = C::NWP, P0 = C::WP0;  // weight planes in the ring slots: [P0, P0 + NW)
        const double *c0 = sC + ((J - Jlo) % CS) * NW * WC, *c1 = sC + ((J + 1 - Jlo) % CS) * NW * WC;
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            const int h = m + p * NPG;
            const int I = xl / 2 + h;
            if (I < x0 / 2 || I >= x0 / 2 + TX / 2 || I < 1 || I > ncx)
                continue;
            const int ic = I - cxl;
            // split residual rows: column 2h -> [h], 2h-1 -> [HW+h-1], 2h+1 -> [HW+h].
            // fig:restrict_kernel's terms in listing order, without those whose
            // residual vanishes: 5-point levels keep the centre and the four Z
            // (corner) terms, 9-point levels the centre and the four X/Y terms.
            double v;
            if (KIND == 5) {
                v = c0[(CI_LNE - P0) * WC + ic] * rm[HW + h - 1];
                v += c0[(CI_LNW - P0) * WC + ic + 1] * rm[HW + h];
                v += r0[h];
                v += c1[(CI_LSE - P0) * WC + ic] * rp[HW + h - 1];
                v += c1[(CI_LSW - P0) * WC + ic + 1] * rp[HW + h];
            } else {
                v = c0[(CI_LA - P0) * WC + ic] * rm[h];
                v += c0[(CI_LR - P0) * WC + ic] * r0[HW + h - 1];
                v += r0[h];
                v += c0[(CI_LL - P0) * WC + ic + 1] * r0[HW + h];
                v += c1[(CI_LB - P0) * WC + ic] * rp[h];
            }
            a.fc[(long long)J * CP + I] = v;
            if constexpr (PUSH)
                push_coarse(a.push, J, (long long)J * CP + I, v);
            if (a.uc)
                a.uc[(long long)J * CP + I] = 0.0;
        }
    };

    // Decoupled pipeline: each group waits only on its own ring, i.e. on the
    // groups whose results (RAW) or ring slots (WAR) it touches, so stages
    // overlap instead of meeting at a CTA-wide barrier every step.
    constexpr int QSPLIT = KIND == 5 ? 3 : 4;  // arrays [0,QSPLIT) by the first split group
    const int tend = yb + 2 * NS + 3;
    if (grp >= C::NG) {
        if (!producer)
            return;
        for (int t = lo; t <= tend; t++) {
            rg.wait(R_PROD, t - 1);
            // No proxy fence: staging slots are only READ by generic-proxy code before
            // the TMA (async proxy) overwrites them, ordered by the mbarrier wait above.
            if (t + D <= hi)
                issue_row(t + D);
            if (BMG_L2PF > 0 && t + D + BMG_L2PF <= hi) {
                const int row = t + D + BMG_L2PF - a.A.roff;
                if (!a.uzero)
                    tma_prefetch_2d(&tmaps.u, xl, row);
                tma_prefetch_2d(&tmaps.f, xl, row);
                tma_prefetch_3d(&tmaps.a, xl, row, 0);
            }
            issue_coarse(t);
        }
        return;
    }
    // rings this group arrives on after each step
    int a0 = -1, a1 = -1, a2 = -1;
    if (grp >= G_SPLIT) {
        a0 = 0, a1 = R_PROD;
    } else if (grp < NSG) {
        if (grp + 1 < NSG)
            a0 = grp + 1;
        // the stages that finalise rows: the last one (5-point) / the last sweep's two (9-point)
        if (grp >= NSG - (KIND == 9 ? 2 : 1))
            a1 = R_RES, a2 = R_STORE;
    } else if (grp < G_STORE) {
        a0 = R_SPLIT, a1 = R_RESTR;
    } else if (grp == G_STORE) {
        a0 = R_SPLIT;
    } else {
        a0 = R_RES, a1 = R_PROD;
    }
    int tm = 0, tsd = 0;  // main / staging ring slots of row t
    for (int t = lo; t <= tend; t++, tm = (tm + 1 == RM) ? 0 : tm + 1, tsd = (tsd + 1 == SD) ? 0 : tsd + 1) {
        if (grp >= G_SPLIT) {
            rg.wait(R_SPLIT, t - 1 - E);
            if (t <= hi) {
                mbar_wait(&bar[tsd], ((t - lo) / SD) & 1);
                if (grp == G_SPLIT)
                    split_row<NA, AM, WD, PPT, NPG, false>(sm, smS, tsd, tm, 0, QSPLIT, m);
                else
                    split_row<NA, AM, WD, PPT, NPG, true>(sm, smS, tsd, tm, QSPLIT, NA, m);
            }
        } else if (grp < NSG) {
            // a 9-point stage's idle step (every other one) reads and writes nothing, so it
            // arrives without waiting (the idle steps of its consumers follow it)
            if (KIND == 5 || ((t + grp + 1) & 1))
                rg.wait(grp, t - 1);
            if (KIND == 5) {
                const int k = grp + 1, d = 2 * k, r = t - d;
                if (r > lo && r < hi && r >= 1 && r <= ny)
                    colour_pass<KIND, AM, WD, PPT>(sm, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1),
                                                   (((k - 1) & 1) - r) & 1, kc);
            } else {
                // 9-point stage k is active at step t iff (t - 2k) & 1 == (k - 1) & 1, i.e. (t + k) odd
                const int k = grp + 1, d = 2 * k, r = t - d;
                const bool act = ((t + k) & 1) && r > lo && r < hi && r >= 1 && r <= ny;
                if (act)  // uniform over the group; phase B waits on the group's barrier inside.
                    // No trailing barrier: the group's next active step (two steps on) works two
                    // rows higher; consumers wait on the per-warp ring arrivals
                    colour_pair9<AM, WD, PPT>(sm, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1), kc,
                                              1 + grp, NPG);
            }
        } else if (grp < G_STORE) {
            rg.wait(R_RES, t - 1);
            const int d = 2 * NS + 2;
            resid_task(t - d, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1), grp - G_RES);
        } else if (grp == G_STORE) {
            rg.wait(R_STORE, t - 3);
            store_task(t - 2 * NS - 3, back<RM>(tm, 2 * NS + 3));
        } else {
            rg.wait(R_RESTR, t - 1);
            const int jr = t - 2 * NS - 4;
            const int J = jr >> 1;
            if (jr >= 0 && !(jr & 1) && J >= Jlo && J <= Jhi)
                restrict_task(J);
        }
        rg.done(t, a0, a1, a2);
    }
}

// ------------------------------------------------------------------ up kernel
// REV (the symmetric cycle's adjoint post-smoother, c12): colours in reverse
// order -- 5-point black before red, 9-point 3, 2, 1, 0 (odd rows first, odd
// columns first) -- and the correction skips the points of that first pass.
template <int KIND, int NS, int WD, int D, int PPT, int E, bool REV = false, bool PUSH = false>
__global__ void __launch_bounds__(Cfg<KIND, NS, WD, D, true, PPT, E>::NT, 1)
    k_fused_up(FArgs a, const __grid_constant__ TMaps tmaps)
{
    using C = Cfg<KIND, NS, WD, D, true, PPT, E>;
    // weight planes fetched: 5-point forward -> X/Y half, reversed -> Z half; 9-point all
    constexpr int P0 = (KIND == 5 && REV) ? CI_LNE : C::WP0;
    constexpr int NA = C::NA, H = C::H, TX = C::TX, WC = C::WC, HW = C::HW, NPG = C::NPG;
    constexpr int RM = C::RM, SD = C::SD, AM = C::AM, AS = C::AS;
    extern __shared__ __align__(128) double sm[];
    double *smS = sm + C::NM * AM;              // staging ring
    double *sE = smS + NA * AS;                 // coarse correction ring [4][WC]
    double *sC = sE + 4 * WC;                   // weights ring [4][8][WC]
    uint64_t *bar = (uint64_t *)(sC + C::NWP * C::CSL * WC);

    const int nx = a.A.nx, ny = a.A.ny;
    const long long P = a.A.pitch;
    const int strip = blockIdx.x % a.nstrips, chunk = blockIdx.x / a.nstrips;
    const int x0 = strip * TX, xl = x0 - H;
    const int ya = a.A.ylo + chunk * a.chunk, yb = min(a.A.yhi, ya + a.chunk);
    if (ya >= yb)
        return;
    const int lo = max(ya - NS, a.A.roff), hi = min(yb + NS - 1, a.A.roff + a.A.nrows - 1);
    const int lo1 = max(lo, 1), hi1 = min(hi, ny);  // corrected rows
    const int cxl = x0 / 2 - CH;
    const int Klo = lo1 / 2, Khi = (hi1 + 1) / 2;

    const int tid = threadIdx.x, grp = tid / NPG, m = tid % NPG;
    const bool producer = tid == C::NTW;  // lane 0 of the producer warp issues every TMA copy
    // Task groups:
    //  5-point: 0,1 correction of even/odd columns; 2..NS+1 stage k = grp-1;
    //           NS+2 store; NS+3, NS+4 split.
    //  9-point: 0..NS-1 stage k = grp+1 (active every other row step; phase A, B);
    //           NS, NS+1 correction; NS+2 store; NS+3, NS+4 split.
    constexpr int NSG = NS;
    constexpr int G_ST0 = KIND == 5 ? 2 : 0, G_CORR = KIND == 5 ? 0 : NSG;
    constexpr int G_SPLIT = NSG + 3;  // store: NSG + 2
    // Rings (waiter <- groups it depends on, at step t-1):
    //  g < NSG  stage group g <- correction groups (g = 0: row r+1 = t-2) or stage group g-1
    //  R_CORR   correction <- split groups (row t-1)
    //  R_STORE  store <- last stage group(s)
    //  R_SPLIT  split <- last stage group(s) (reads the slot's old row t-RM), store
    //  R_PROD   producer <- split groups (staging slot), correction groups (coarse slots)
    constexpr int W = NPG / 32;
    constexpr int R_CORR = NSG, R_STORE = NSG + 1, R_SPLIT = NSG + 2, R_PROD = NSG + 3, NR = NSG + 4;
    static_assert(NR <= C::NG, "ring space");
    const Rings rg{smem_u32(bar + SD + 4), lo};

    if (tid == 0) {
        for (int i = 0; i < SD + 4; i++)
            mbar_init(&bar[i], 1);
        for (int r = 0; r < NR; r++) {
            const int cnt = r < NSG ? (r == 0 ? 2 * W : W)
                            : r == R_CORR ? 2 * W
                            : r == R_STORE ? (KIND == 5 ? 1 : 2) * W
                            : r == R_SPLIT ? (KIND == 5 ? 2 : 3) * W : 4 * W;
            for (int q = 0; q < NSLOT; q++)
                mbar_init(bar + SD + 4 + r * NSLOT + q, cnt);
        }
        fence_mbar_init();
    }
    __syncthreads();

    int Knext = Klo;
    auto issue_row = [&](int row) {
        const int slot = (row - lo) % SD;
        uint64_t *b = &bar[slot];
        mbar_arrive_tx(b, (uint32_t)(NA * WD * 8));
        double *d = smS + slot * (NA * WD);
        tma_2d(d + A_U * WD, &tmaps.u, xl, row - a.A.roff, b);
        tma_2d(d + A_F * WD, &tmaps.f, xl, row - a.A.roff, b);
        tma_3d(d + A_O * WD, &tmaps.a, xl, row - a.A.roff, 0, b);
    };
    auto issue_coarse = [&](int t) {
        while (Knext <= Khi) {
            const int use = max(2 * Knext - 1, lo1) + 1;
            if (use - DC > t)
                break;
            const int slot = (Knext - Klo) & 3;
            uint64_t *b = &bar[SD + slot];
            mbar_arrive_tx(b, (uint32_t)((1 + C::NWP) * WC * 8));
            tma_2d(sE + slot * WC, &tmaps.e, cxl, Knext - a.eroff, b);
            tma_3d(sC + slot * C::NWP * WC, &tmaps.c, cxl, Knext - a.ci.roff, P0, b);
            Knext++;
        }
    };
    if (producer)
        for (int row = lo; row <= min(lo + D - 1, hi); row++)
            issue_row(row);

    // u += P e (c7) on row x (main slot sx) at the columns of parity e of this thread's
    // pairs; same operand order as k_interp_add.  Point type is uniform over the group.
    // Points of the first colour pass (5-point: C and Z; 9-point: C) are skipped:
    // that pass overwrites them from their neighbours alone, so the result is
    // bitwise the same as correcting them.
    constexpr int NW = C::NWP;
    auto correct_task = [&](int x, int sx, int e) {
        if (x < lo1 || x > hi1)
            return;
        const bool first_pass = KIND == 5 ? (REV ? ((e + x) & 1) : !((e + x) & 1))
                                          : (REV ? (e && (x & 1)) : (!e && !(x & 1)));
        if (first_pass)
            return;
        const int Ka = x >> 1, Kb = (x + 1) >> 1;
        mbar_wait(&bar[SD + ((Ka - Klo) & 3)], ((Ka - Klo) >> 2) & 1);
        mbar_wait(&bar[SD + ((Kb - Klo) & 3)], ((Kb - Klo) >> 2) & 1);
        double *u0 = sm + A_U * AM + sx * WD + e * HW;
        const bool rodd = x & 1;
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            const int h = m + p * NPG, c = xl + 2 * h + e;
            if (c < 1 || c > nx)
                continue;
            double s;
            if (!e && !rodd) {  // C point
                s = sE[((x / 2 - Klo) & 3) * WC + (c / 2 - cxl)];
            } else if (e && !rodd) {  // X point (2I-1, 2J)
                const int I = (c + 1) / 2, Jx = x / 2, ic = I - cxl;
                const double *ev = sE + ((Jx - Klo) & 3) * WC;
                const double *w = sC + ((Jx - Klo) & 3) * NW * WC;
                s = w[(CI_LL - P0) * WC + ic] * ev[ic - 1];
                s += w[(CI_LR - P0) * WC + ic] * ev[ic];
            } else if (!e && rodd) {  // Y point (2I, 2J-1)
                const int I = c / 2, Jy = (x + 1) / 2, ic = I - cxl;
                const double *e0 = sE + ((Jy - 1 - Klo) & 3) * WC, *e1 = sE + ((Jy - Klo) & 3) * WC;
                const double *w = sC + ((Jy - Klo) & 3) * NW * WC;
                s = w[(CI_LB - P0) * WC + ic] * e0[ic];
                s += w[(CI_LA - P0) * WC + ic] * e1[ic];
            } else {  // Z point (2I-1, 2J-1)
                const int I = (c + 1) / 2, Jz = (x + 1) / 2, ic = I - cxl;
                const double *e0 = sE + ((Jz - 1 - Klo) & 3) * WC, *e1 = sE + ((Jz - Klo) & 3) * WC;
                const double *w = sC + ((Jz - Klo) & 3) * NW * WC;
                s = w[(CI_LSW - P0) * WC + ic] * e0[ic - 1];
                s += w[(CI_LSE - P0) * WC + ic] * e0[ic];
                s += w[(CI_LNW - P0) * WC + ic] * e1[ic - 1];
                s += w[(CI_LNE - P0) * WC + ic] * e1[ic];
            }
            u0[h] += s;
        }
    };
    auto store_task = [&](int w, int sw) {
        if (w < ya || w >= yb)
            return;
        const double *urow = sm + A_U * AM + sw * WD;
#pragma unroll
        for (int p = 0; p < PPT; p++) {
            const int h = m + p * NPG, sc = 2 * h, c = xl + sc;
            if (sc < H || sc >= H + TX)
                continue;
            double *dst = a.uout + (long long)w * P + c;
            const double ve = urow[h], vo = urow[HW + h];
            if (c >= 1 && c + 1 <= nx)
                *reinterpret_cast<double2 *>(dst) = make_double2(ve, vo);
            else {
                if (c >= 1 && c <= nx)
                    dst[0] = ve;
                if (c + 1 >= 1 && c + 1 <= nx)
                    dst[1] = vo;
            }
            if constexpr (PUSH)
                push_row(a.push, w, (long long)w * P + c, c, nx, ve, vo);
        }
    };

    const Cols<PPT> kc = make_cols<WD, PPT, NPG>(m, xl, nx);

    constexpr int QSPLIT = KIND == 5 ? 3 : 4;
    const int tend = yb + 2 * NS + 1;
    if (grp >= C::NG) {
        if (!producer)
            return;
        for (int t = lo; t <= tend; t++) {
            rg.wait(R_PROD, t - 1);
            if (t + D <= hi)
                issue_row(t + D);
            if (BMG_L2PF > 0 && t + D + BMG_L2PF <= hi) {
                const int row = t + D + BMG_L2PF - a.A.roff;
                tma_prefetch_2d(&tmaps.u, xl, row);
                tma_prefetch_2d(&tmaps.f, xl, row);
                tma_prefetch_3d(&tmaps.a, xl, row, 0);
            }
            issue_coarse(t);
        }
        return;
    }
    int a0 = -1, a1 = -1, a2 = -1;
    if (grp >= G_SPLIT) {
        a0 = R_CORR, a1 = R_PROD;
    } else if (grp == G_CORR || grp == G_CORR + 1) {
        a0 = 0, a1 = R_PROD;
    } else if (grp < G_ST0 + NSG) {
        const int g = grp - G_ST0;
        if (g + 1 < NSG)
            a0 = g + 1;
        if (g >= NSG - (KIND == 9 ? 2 : 1))
            a1 = R_SPLIT, a2 = R_STORE;
    } else {
        a0 = R_SPLIT;
    }
    int tm = 0, tsd = 0;
    for (int t = lo; t <= tend; t++, tm = (tm + 1 == RM) ? 0 : tm + 1, tsd = (tsd + 1 == SD) ? 0 : tsd + 1) {
        if (grp >= G_SPLIT) {
            rg.wait(R_SPLIT, t - 1 - E);
            if (t <= hi) {
                mbar_wait(&bar[tsd], ((t - lo) / SD) & 1);
                if (grp == G_SPLIT)
                    split_row<NA, AM, WD, PPT, NPG, false>(sm, smS, tsd, tm, 0, QSPLIT, m);
                else
                    split_row<NA, AM, WD, PPT, NPG, true>(sm, smS, tsd, tm, QSPLIT, NA, m);
            }
        } else if (grp == G_CORR || grp == G_CORR + 1) {
            rg.wait(R_CORR, t - 1);
            correct_task(t - 1, back<RM>(tm, 1), grp - G_CORR);
        } else if (grp < G_ST0 + NSG) {
            if (KIND == 5 || (((t + grp - G_ST0 + 1) & 1) == (REV ? 1 : 0)))  // idle 9-point steps: no wait
                rg.wait(grp - G_ST0, t - 1);
            if (KIND == 5) {
                const int k = grp - G_ST0 + 1, d = 2 * k + 1, r = t - d;
                const int col = REV ? (k & 1) : ((k - 1) & 1);  // stage k's colour
                if (r > lo && r < hi && r >= 1 && r <= ny)
                    colour_pass<KIND, AM, WD, PPT>(sm, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1),
                                                   (col - r) & 1, kc);
            } else {
                // active 9-point row stage(s): k with (t-1-2k) & 1 == (k-1) & 1, i.e. (t + k) even
                // (REV: (t + k) odd -- odd rows first -- and odd columns before even)
                const int k = grp - G_ST0 + 1, d = 2 * k + 1, r = t - d;
                const bool act = (((t + k) & 1) == (REV ? 1 : 0)) && r > lo && r < hi && r >= 1 && r <= ny;
                if (act) {  // uniform over the group
                    if (REV) {
                        colour_pass<KIND, AM, WD, PPT>(sm, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1),
                                                       1, kc);
                        group_sync(1 + grp, NPG);
                        colour_pass<KIND, AM, WD, PPT>(sm, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1),
                                                       0, kc);
                    } else {
                        colour_pair9<AM, WD, PPT>(sm, back<RM>(tm, d), back<RM>(tm, d + 1), back<RM>(tm, d - 1), kc,
                                                  1 + grp, NPG);
                    }
                }
            }
        } else {
            rg.wait(R_STORE, t - 1);
            store_task(t - 2 * NS - 2, back<RM>(tm, 2 * NS + 2));
        }
        rg.done(t, a0, a1, a2);
    }
}

// ------------------------------------------------------------------ host side
// Per-device limits and kernel attributes: cudaFuncSetAttribute applies to the
// device current at the call, so a handle set up on another GPU of the same
// process gets its own; guarded for concurrent setups.
constexpr int MAX_DEV = 64;
struct DevInfo {
    int sms = 148;
    size_t smem_optin = 227 * 1024, smem_sm = 228 * 1024;
};
static DevInfo g_dev[MAX_DEV];
static std::once_flag g_dev_once[MAX_DEV];

static int cur_device()
{
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < MAX_DEV ? dev : 0;
}

static void set_all_attrs();

// Limits of the current device (queried, and the fused kernels' attributes set, once per device).
static const DevInfo &device_limits()
{
    const int dev = cur_device();
    std::call_once(g_dev_once[dev], [dev]() {
        int v = 0;
        DevInfo &d = g_dev[dev];
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            d.sms = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess && v > 0)
            d.smem_optin = (size_t)v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) == cudaSuccess && v > 0)
            d.smem_sm = (size_t)v;
        set_all_attrs();
    });
    return g_dev[dev];
}

// Deepest TMA prefetch (rows, <= 4) whose shared-memory footprint fits a CTA.
constexpr size_t SMEM_CTA_MAX = 232448;  // 227 KB opt-in
#ifndef BMG_DMAX
#define BMG_DMAX 4
#endif
template <int KIND, int NS, int WD, bool UP, int PPT, int E, int DM = BMG_DMAX>
constexpr int pick_D()
{
    if constexpr (DM <= 2)
        return 2;
    else
        return Cfg<KIND, NS, WD, DM, UP, PPT, E>::SMEM <= SMEM_CTA_MAX ? DM : pick_D<KIND, NS, WD, UP, PPT, E, DM - 1>();
}

// Kernel instances: (kind, NS) -> (WD, D, pairs per thread).  WD = smem row width.
template <int KIND, int NS>
struct Inst {
#ifndef BMG_WD5
#define BMG_WD5 256
#endif
#ifndef BMG_WD9DN
#define BMG_WD9DN 192
#endif
#ifndef BMG_WD9UP
#define BMG_WD9UP 256
#endif
    static constexpr int WD_DN = KIND == 5 ? BMG_WD5 : BMG_WD9DN;

#ifndef BMG_PPT5
#define BMG_PPT5 2
#endif
#ifndef BMG_PPT9DN
#define BMG_PPT9DN 3  // one warp per task group (352 threads): 4095^2 9-point down leg 0.434 -> 0.415 ms against 1
#endif
    static constexpr int PPT_DN = KIND == 5 ? BMG_PPT5 : BMG_PPT9DN;
#ifndef BMG_WD5UP
#define BMG_WD5UP 128  // 5-point up leg: 128-column strips (2 CTAs/SM); swept 64..256 x 1..4 pairs,
                       // 8191^2 up leg 0.826 -> 0.815 ms against 256
#endif
#ifndef BMG_PPT5UP
#define BMG_PPT5UP BMG_PPT5
#endif
    static constexpr int WD_UP = KIND == 5 ? BMG_WD5UP : (NS == 4 ? 192 : BMG_WD9UP);

#ifndef BMG_PPT9UP
#define BMG_PPT9UP 2
#endif
    static constexpr int PPT_UP = KIND == 5 ? BMG_PPT5UP : (NS == 4 ? 1 : BMG_PPT9UP);
#ifndef BMG_E5DN
#define BMG_E5DN 0
#endif
#ifndef BMG_E9DN
#define BMG_E9DN 1  // one main-ring slack row: 4095^2 9-point down leg 0.415 -> 0.381 ms (with 3 pairs per thread)
#endif
#ifndef BMG_E5UP
#define BMG_E5UP 0
#endif
#ifndef BMG_E9UP
#define BMG_E9UP 1  // one main-ring slack row: 4095^2 9-point up leg 0.277 -> 0.274 ms
#endif
    static constexpr int E_DN = KIND == 5 ? BMG_E5DN : BMG_E9DN;  // main-ring slack rows
    static constexpr int E_UP = KIND == 5 ? BMG_E5UP : BMG_E9UP;
    static constexpr int D_DN = pick_D<KIND, NS, WD_DN, false, PPT_DN, E_DN>();
    static constexpr int D_UP = pick_D<KIND, NS, WD_UP, true, PPT_UP, E_UP>();
    using CD = Cfg<KIND, NS, WD_DN, D_DN, false, PPT_DN, E_DN>;
    using CU = Cfg<KIND, NS, WD_UP, D_UP, true, PPT_UP, E_UP>;
};

template <int KIND, int NS>
static void fill_geom(FusedGeom &g, bool up)
{
    using I = Inst<KIND, NS>;
    if (!up) {
        using C = typename I::CD;
        g.TX = C::TX, g.H = C::H, g.WD = I::WD_DN, g.WC = C::WC, g.R = C::RM, g.D = I::D_DN, g.threads = C::NT;
        g.smem = C::SMEM;
    } else {
        using C = typename I::CU;
        g.TX = C::TX, g.H = C::H, g.WD = I::WD_UP, g.WC = C::WC, g.R = C::RM, g.D = I::D_UP, g.threads = C::NT;
        g.smem = C::SMEM;
    }
    g.NS = NS;
}

template <int KIND, int NS>
static void set_attrs(size_t optin)
{
    using I = Inst<KIND, NS>;
    constexpr size_t sd = I::CD::SMEM, su = I::CU::SMEM;
    if (sd <= optin) {
        cudaFuncSetAttribute(k_fused_down<KIND, NS, I::WD_DN, I::D_DN, I::PPT_DN, I::E_DN>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd);
        cudaFuncSetAttribute(k_fused_down<KIND, NS, I::WD_DN, I::D_DN, I::PPT_DN, I::E_DN, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd);
    }
    if (su <= optin) {
        cudaFuncSetAttribute(k_fused_up<KIND, NS, I::WD_UP, I::D_UP, I::PPT_UP, I::E_UP>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)su);
        cudaFuncSetAttribute(k_fused_up<KIND, NS, I::WD_UP, I::D_UP, I::PPT_UP, I::E_UP, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)su);
        cudaFuncSetAttribute(k_fused_up<KIND, NS, I::WD_UP, I::D_UP, I::PPT_UP, I::E_UP, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)su);
    }
    cudaGetLastError();  // an unsupported instance is simply not planned (plan_grid checks the size)
}

// called once per device, inside device_limits()
static void set_all_attrs()
{
    const size_t optin = g_dev[cur_device()].smem_optin;
    set_attrs<5, 2>(optin);
    set_attrs<5, 4>(optin);
    set_attrs<9, 2>(optin);
    set_attrs<9, 4>(optin);
}

// Grid for one kernel: strips of TX columns x chunks of rows, chosen to balance
// the per-SM work over waves (warm-up rows counted as overhead).
static void plan_grid(FusedGeom &g, int nx, int ny, int warm)
{
    const DevInfo &dv = device_limits();
    g.ok = false;
    if (g.smem > dv.smem_optin)
        return;
    int occ = (int)(dv.smem_sm / (g.smem + 1024));
    occ = std::min(occ, 2048 / g.threads);
    if (occ < 1)
        return;
    const int slots = dv.sms * occ;
    g.nstrips = nx / g.TX + 1;
    double best = 1e300;
    // every chunk count (at most (ny+1)/8): the cost model is cheap, and rounding a per-wave
    // count can overshoot the slots by a few CTAs and cost a whole extra wave (1023^2: 5
    // strips x 30 chunks = 150 CTAs on 148 slots)
    for (int nc = 1; nc <= std::max(1, (ny + 1) / 8); nc++) {
        const int chunk = (ny + 1 + nc - 1) / nc;
        const int nch = (ny + 1 + chunk - 1) / chunk;
        const long long units = (long long)g.nstrips * nch;
        const long long waves = (units + slots - 1) / slots;
#ifndef BMG_PLAN_K
#define BMG_PLAN_K 0  // per-CTA fixed cost in row steps beyond the warm-up (swept 0/8/16/32: 0 best at 8191^2, others within 0.1 %)
#endif
        const double cost = (double)waves * (chunk + warm + BMG_PLAN_K);
        if (cost < best) {
            best = cost;
            g.nchunks = nch;
            g.chunk = chunk;
            g.ok = true;
        }
    }
}

bmg_status_t fused_plan_level(FusedPlan &fp, int l, int nx, int ny, long long pitch, int kind, int nu1, int nu2,
                              bool aligned, bool rev)
{
    LevelPlan &lp = fp.lv[l];
    lp.down = lp.up = false;
    if (!aligned || (pitch & 1) || nx < 8 || ny < 8 || nx > (1 << 24) || pitch > (1LL << 30))
        return BMG_OK;
    if ((nu1 != 1 && nu1 != 2) || (nu2 != 1 && nu2 != 2))
        return BMG_OK;
    device_limits();  // per device: limits + kernel attributes
    const int nsd = 2 * nu1, nsu = 2 * nu2;
    if (kind == 5) {
        nsd == 2 ? fill_geom<5, 2>(lp.gd, false) : fill_geom<5, 4>(lp.gd, false);
        nsu == 2 ? fill_geom<5, 2>(lp.gu, true) : fill_geom<5, 4>(lp.gu, true);
    } else {
        nsd == 2 ? fill_geom<9, 2>(lp.gd, false) : fill_geom<9, 4>(lp.gd, false);
        nsu == 2 ? fill_geom<9, 2>(lp.gu, true) : fill_geom<9, 4>(lp.gu, true);
    }
    plan_grid(lp.gd, nx, ny, 2 * nsd + 4);
    plan_grid(lp.gu, nx, ny, 2 * nsu + 2);
    lp.gu.rev = rev;
    lp.down = lp.gd.ok;
    lp.up = lp.gu.ok;
    if (getenv("BMG_SETUP_TRACE"))  // tuning aid: the plan of this level's legs
        for (const FusedGeom *g : {&lp.gd, &lp.gu})
            fprintf(stderr,
                    "fused plan l=%d %dx%d kind %d %s: ok %d TX %d WD %d D %d threads %d smem %d B, %d strips x %d "
                    "chunks of %d rows (%d CTAs, %d/SM)\n",
                    l, nx, ny, kind, g == &lp.gd ? "down" : "up", (int)g->ok, g->TX, g->WD, g->D, g->threads,
                    (int)g->smem, g->nstrips, g->nchunks, g->chunk, g->nstrips * g->nchunks,
                    (int)std::min<long long>(device_limits().smem_sm / (g->smem + 1024), 2048 / g->threads));
    return BMG_OK;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

static bool ptrs_ok(const Op &A, const CIv &ci, std::initializer_list<const void *> extra)
{
    if (!aligned16(A.O) || !aligned16(A.W) || !aligned16(A.S))
        return false;
    if (A.kind == 9 && (!aligned16(A.SW) || !aligned16(A.NW)))
        return false;
    if (ci.pitch & 1)
        return false;
    for (int k = 0; k < 8; k++)
        if (!aligned16(ci.w[k]))
            return false;
    for (const void *p : extra)
        if (p && !aligned16(p))
            return false;
    return true;
}

// ---- TMA tensor maps (driver entry point fetched through the runtime; no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
        cudaGetLastError();
    }
    return fn;
}

// rank-3 fp64 map over `planes` planes of rows x width elements (row pitch, plane
// stride in elements); box = bw columns x 1 row x bz planes (bz = 0: all planes).
// Rank 2 when planes == 0.
static bool make_map(CUtensorMap *m, const double *base, long long width, long long rows, long long pitch,
                     long long pstride, int planes, int bw, int bz = 0)
{
    auto fn = encode_fn();
    if (!fn)
        return false;
    cuuint64_t dims[3] = {(cuuint64_t)width, (cuuint64_t)rows, (cuuint64_t)(planes > 0 ? planes : 1)};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pstride * 8};
    cuuint32_t box[3] = {(cuuint32_t)bw, 1, (cuuint32_t)(planes > 0 ? (bz > 0 ? bz : planes) : 1)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, planes > 0 ? 3 : 2, (void *)base, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Maps of one fused launch: the planes and the weights must be contiguous blocks.
static bool make_maps(TMaps &tm, const FusedGeom &g, const Op &A, const CIv &ci, const double *uin, const double *f,
                      const double *ec, int eroff, int enrows)
{
    const long long np = (long long)A.nrows * A.pitch;  // plane stride of the (slab) block
    const int npl = A.kind == 9 ? 5 : 3;
    const double *pl[5] = {A.O, A.W, A.S, A.SW, A.NW};
    for (int k = 1; k < npl; k++)
        if (pl[k] != A.O + k * np)
            return false;
    const int ncx = A.nx / 2;
    const long long npc = (long long)ci.nrows * ci.pitch;
    for (int k = 1; k < 8; k++)
        if (ci.w[k] != ci.w[0] + k * npc)
            return false;
    bool ok = make_map(&tm.u, uin + A.roff * A.pitch, A.nx + 2, A.nrows, A.pitch, 0, 0, g.WD) &&
              make_map(&tm.f, f + A.roff * A.pitch, A.nx + 2, A.nrows, A.pitch, 0, 0, g.WD) &&
              make_map(&tm.a, A.O + A.roff * A.pitch, A.nx + 2, A.nrows, A.pitch, np, npl, g.WD) &&
              // the down leg (ec == nullptr) and the 5-point up leg fetch 4 of the 8 weight planes
              make_map(&tm.c, ci.w[0] + ci.roff * ci.pitch, ncx + 2, ci.nrows, ci.pitch, npc, 8, g.WC,
                       ec && A.kind == 9 ? 8 : 4);
    if (ok && ec)
        ok = make_map(&tm.e, ec + (long long)eroff * ci.pitch, ncx + 2, enrows, ci.pitch, 0, 0, g.WC);
    else
        tm.e = tm.c;
    return ok;
}

template <int KIND, int NS>
static void launch_down(const FusedGeom &g, const FArgs &a, const TMaps &tm, cudaStream_t s)
{
    using I = Inst<KIND, NS>;
    if (a.push.halo)
        k_fused_down<KIND, NS, I::WD_DN, I::D_DN, I::PPT_DN, I::E_DN, true>
            <<<g.nstrips * g.nchunks, g.threads, g.smem, s>>>(a, tm);
    else
        k_fused_down<KIND, NS, I::WD_DN, I::D_DN, I::PPT_DN, I::E_DN><<<g.nstrips * g.nchunks, g.threads, g.smem, s>>>(a,
                                                                                                                   tm);
}

template <int KIND, int NS>
static void launch_up(const FusedGeom &g, const FArgs &a, const TMaps &tm, cudaStream_t s)
{
    using I = Inst<KIND, NS>;
    if (g.rev)
        k_fused_up<KIND, NS, I::WD_UP, I::D_UP, I::PPT_UP, I::E_UP, true><<<g.nstrips * g.nchunks, g.threads, g.smem,
                                                                            s>>>(a, tm);
    else if (a.push.halo)
        k_fused_up<KIND, NS, I::WD_UP, I::D_UP, I::PPT_UP, I::E_UP, false, true>
            <<<g.nstrips * g.nchunks, g.threads, g.smem, s>>>(a, tm);
    else
        k_fused_up<KIND, NS, I::WD_UP, I::D_UP, I::PPT_UP, I::E_UP><<<g.nstrips * g.nchunks, g.threads, g.smem, s>>>(a,
                                                                                                                   tm);
}

static FArgs make_args(const FusedGeom &g, const Op &A, const CIv &ci)
{
    FArgs a;
    a.A = A;
    a.ci = ci;
    a.f = a.uin = a.ec = nullptr;
    a.uout = a.fc = a.uc = nullptr;
    a.nstrips = g.nstrips;
    a.chunk = g.chunk;
    a.ncx = A.nx / 2;
    a.ncy = A.ny / 2;
    a.eroff = 0;
    a.uzero = 0;
    return a;
}

bool fused_down(const FusedPlan &fp, int l, const Op &A, const CIv &ci, const double *f, const double *uin,
                double *uout, double *fc, double *uc, cudaStream_t s, int *nlaunch, const Push *push)
{
    if (l >= 32 || !fp.lv[l].down || !ptrs_ok(A, ci, {f, uin, uout, fc, uc}))
        return false;
    const FusedGeom &g = fp.lv[l].gd;
    FArgs a = make_args(g, A, ci);
    a.f = f;
    a.uin = uin;
    a.uout = uout;
    a.fc = fc;
    a.uc = uc;
    a.uzero = uin == nullptr;
    if (push)
        a.push = *push;
    TMaps tm;
    if (!make_maps(tm, g, A, ci, uin ? uin : f, f, nullptr, 0, 0))  // uzero: u map unused
        return false;
    if (A.kind == 5)
        g.NS == 2 ? launch_down<5, 2>(g, a, tm, s) : launch_down<5, 4>(g, a, tm, s);
    else
        g.NS == 2 ? launch_down<9, 2>(g, a, tm, s) : launch_down<9, 4>(g, a, tm, s);
    if (nlaunch)
        *nlaunch += 1;
    return true;
}

bool fused_up(const FusedPlan &fp, int l, const Op &A, const CIv &ci, const double *f, const double *uin,
              const double *ec, int eroff, int enrows, double *uout, cudaStream_t s, int *nlaunch, const Push *push)
{
    if (l >= 32 || !fp.lv[l].up || !ptrs_ok(A, ci, {f, uin, uout, ec}))
        return false;
    const FusedGeom &g = fp.lv[l].gu;
    FArgs a = make_args(g, A, ci);
    a.f = f;
    a.uin = uin;
    a.ec = ec;
    a.uout = uout;
    if (push)
        a.push = *push;
    TMaps tm;
    a.eroff = eroff;
    if (!make_maps(tm, g, A, ci, uin, f, ec, eroff, enrows))
        return false;
    if (A.kind == 5)
        g.NS == 2 ? launch_up<5, 2>(g, a, tm, s) : launch_up<5, 4>(g, a, tm, s);
    else
        g.NS == 2 ? launch_up<9, 2>(g, a, tm, s) : launch_up<9, 4>(g, a, tm, s);
    if (nlaunch)
        *nlaunch += 1;
    return true;
}

}  // namespace bmg
