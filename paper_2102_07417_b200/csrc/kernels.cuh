// Device kernels of the amgb200 solve path (sm_100a, fp64, HBM-bound).
//
// * spmv_tiles: persistent CSR SpMV.  Rows are cut at upload into tiles of
//   <= TILE_NNZ stored entries / <= TILE_ROWS rows; each CTA walks its tiles
//   round-robin and stages a tile's contiguous value / column / offset
//   ranges in shared memory with cp.async.bulk (TMA bulk engine, mbarrier
//   completion, STAGES-deep ring), so every HBM byte is moved by fully
//   coalesced 16-byte-aligned bulk transfers and the next tiles are in
//   flight while the current one is reduced.
//   Row sums follow the reference order exactly (amgkit/sparse.py:212-217 ->
//   np.add.reduceat, restated in oracle/rowsum.c):
//       y_i = p_0 + pairwise(p_1 .. p_{L-1}),  p_k = a_k * x[c_k] (rounded)
//   with numpy's eight strided accumulators mapped onto LANES lanes per row
//   and its ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) combine done as a shuffle
//   butterfly -- so a row sum is bit-identical to the reference's.
//   Fused epilogues: y = s | y = b - s | y = b + w*s | y = w*s | y = b + s,
//   plus an optional deterministic dot partial sum_i y_i * d_i.
// * vector kernels for the PCG recurrences (krylov.py:40-92) with fused
//   dot partials; every reduction is fixed-order (per-CTA partials, the last
//   CTA to finish folds them in index order) -- no fp atomics, so repeated
//   solves are bitwise identical.
// * coarse_chol: dense forward/back substitution with the lower Cholesky
//   factor staged in shared memory (hierarchy.py:149-152, dpotrs).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

// AMG_CHECKS builds (paper_2102_07417_b200.build.build_checked_library; the
// stand-in for compute-sanitizer, which this GPU pool does not allow): index
// and protocol invariants of the kernels checked on the device, a violation
// prints its site and traps (the launch fails with an error).
#ifdef AMG_CHECKS
#define AMG_CHECK(cond)                                                                                   \
    do {                                                                                                  \
        if (!(cond)) {                                                                                    \
            printf("amgb200 check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,    \
                   (int)blockIdx.x, (int)threadIdx.x);                                                   \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define AMG_CHECK(cond) \
    do {                \
    } while (0)
#endif

namespace amg {

constexpr int TILE_THREADS = 256;

enum Epi { EPI_PLAIN = 0, EPI_RESID = 1, EPI_AXPYW = 2, EPI_SETW = 3, EPI_ADD = 4 };

enum Fin {
    FIN_NONE = 0,
    FIN_BNORM,
    FIN_INIT_RES,
    FIN_INIT_RZ,
    FIN_CURV,
    FIN_UPDATE,
    FIN_RECOMPUTE,
    FIN_TRUE,
    FIN_RZ,
    FIN_STORE,  // store raw sum into ctl->scratch (tests / diagnostics)
    FIN_LOCAL   // multi-GPU: this rank's partial -> ctl->part_local (all-gathered, then finalized)
};

constexpr int MAX_RANKS = 64;

// Device-resident PCG state: the control flow of krylov.py:40-92 evaluated
// on the GPU so an iteration never waits for the host.
struct PcgCtl {
    int active;        // 1 while the loop runs (0 after convergence / failure / max_iters)
    int do_recompute;  // this iteration replaces r by b - A x (recompute_every)
    int need_true;     // recurrence relres <= rtol: evaluate the true residual
    int converged;
    int status;        // 0 ok, 3 = not SPD
    int it;            // current iteration number
    int max_iters;
    int recompute_every;
    int record;
    int pad_;
    double rtol, bnorm, rz, curv, alpha, beta, relres, curv_fail, scratch;
    double *hist;
    double part_local;
    double part_all[MAX_RANKS];
};

struct SpmvArgs {
    const int32_t *off;
    const int32_t *col;
    const double *val;
    const double *x;  // gathered vector
    double *y;        // output
    const double *b;  // epilogue operand (may alias y)
    double omega;
    const double *dotw;  // dot partner (nullptr: no dot)
    double *partials;
    unsigned *ticket;
    int fin;
    PcgCtl *ctl;
    const int *gate1;
    const int *gate2;
    // row-range launches (multi-GPU interior / boundary split): a kernel's
    // virtual row v is row rlo + v + (v >= rsplit ? rgap : 0); identity
    // (0, INT_MAX, 0) by default.  rlo, rsplit, rgap are multiples of 128, so
    // 32-row slices and 128-row SELL-sigma windows map whole.
    int rlo, rsplit, rgap;
    // reductions over two launches: pmode 0 = this launch finalizes alone;
    // 1 = store partials[pbase + cta] only; 2 = store, then the last CTA folds
    // partials[0, pbase + grid) (the first launch wrote [0, pbase))
    int pmode, pbase;
    int pcap;  // partial slots available (2 x max grid): AMG_CHECKS bound for pbase + grid
};

__device__ __forceinline__ int vrow(const SpmvArgs &a, int v) { return a.rlo + v + (v >= a.rsplit ? a.rgap : 0); }
// (AMG_CHECKS: spmv_finalize checks the two-launch partial slots against the scratch size)

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ bool gate_open(const int *g1, const int *g2)
{
    return (g1 == nullptr || *(volatile const int *)g1) && (g2 == nullptr || *(volatile const int *)g2);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Programmatic dependent launch: a kernel may start (and stage its static
// matrix tiles) while its predecessor drains; it must call pdl_wait() before
// touching anything the predecessor writes.  No-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Bulk copy with an L2 eviction policy (matrix streams are read once:
// evict_first keeps the gathered vectors resident in L2).
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, unsigned bytes, uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ double prod(double a, double x) { return __dmul_rn(a, x); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// Fixed-shape block reduction (deterministic).  Result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (l < NT / 32) ? red[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

__device__ void apply_fin(int fin, double v, PcgCtl *c)
{
    switch (fin) {
    case FIN_BNORM: c->bnorm = sqrt(v); break;
    case FIN_INIT_RES: {
        double rr = sqrt(v) / c->bnorm;
        c->relres = rr;
        if (c->record) c->hist[0] = rr;
        if (rr <= c->rtol) { c->converged = 1; c->active = 0; }
        break;
    }
    case FIN_INIT_RZ: c->rz = v; break;
    case FIN_CURV:
        c->it += 1;
        c->curv = v;
        if (v <= 0.0) {  // krylov.py:67-72 (NaN passes, as in the reference)
            c->status = 3;
            c->curv_fail = v;
            c->active = 0;
        } else {
            c->alpha = c->rz / v;
        }
        break;
    case FIN_UPDATE:
        if (c->it % c->recompute_every == 0) {
            c->do_recompute = 1;
        } else {
            double rr = sqrt(v) / c->bnorm;
            c->relres = rr;
            if (c->record) c->hist[c->it] = rr;
            c->need_true = rr <= c->rtol;
        }
        break;
    case FIN_RECOMPUTE: {
        c->do_recompute = 0;
        double rr = sqrt(v) / c->bnorm;
        c->relres = rr;
        if (c->record) c->hist[c->it] = rr;
        c->need_true = rr <= c->rtol;
        break;
    }
    case FIN_TRUE: {
        c->need_true = 0;
        double rr = sqrt(v) / c->bnorm;
        c->relres = rr;
        if (rr <= c->rtol) { c->converged = 1; c->active = 0; }
        break;
    }
    case FIN_RZ:
        c->beta = v / c->rz;
        c->rz = v;
        break;
    case FIN_STORE: c->scratch = v; break;
    case FIN_LOCAL: c->part_local = v; break;
    default: break;
    }
}

// Per-CTA partial -> last CTA folds all partials in index order and applies
// the finalize op.  `v` must be the block sum held by thread 0.
template <int NT>
__device__ __forceinline__ void grid_finalize(double v, double *partials, unsigned *ticket, int fin, PcgCtl *ctl)
{
    __shared__ int s_last;
    __shared__ double s_red[NT / 32];
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = v;
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        AMG_CHECK(t < gridDim.x);  // the ticket was left at 0 by the previous reduction
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {  // the whole last CTA folds the partials: fixed assignment + fixed tree
        __threadfence();
        double a = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) a += __ldcg(partials + i);
        a = block_sum<NT>(a, s_red);
        if (threadIdx.x == 0) {
            apply_fin(fin, a, ctl);
            *ticket = 0u;
            __threadfence();
        }
    }
}

// As grid_finalize, for the second kernel of a pair: this grid's partials go
// to partials[base + blockIdx.x] and the last CTA folds partials[0, base + gridDim.x)
// (the first kernel, complete before this one passed griddepcontrol.wait,
// wrote partials[0, base)).
template <int NT>
__device__ __forceinline__ void grid_finalize_pair(double v, double *partials, int base, unsigned *ticket, int fin,
                                                   PcgCtl *ctl)
{
    __shared__ int s_last;
    __shared__ double s_red[NT / 32];
    if (threadIdx.x == 0) {
        partials[base + blockIdx.x] = v;
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        AMG_CHECK(t < gridDim.x);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        double a = 0.0;
        for (int i = threadIdx.x; i < base + (int)gridDim.x; i += NT) a += __ldcg(partials + i);
        a = block_sum<NT>(a, s_red);
        if (threadIdx.x == 0) {
            apply_fin(fin, a, ctl);
            *ticket = 0u;
            __threadfence();
        }
    }
}

// SpMV reductions (pmode, see SpmvArgs)
template <int NT>
__device__ __forceinline__ void spmv_finalize(double v, const SpmvArgs &a)
{
    AMG_CHECK(a.pmode == 0 || a.pbase + (int)gridDim.x <= a.pcap);
    if (a.pmode == 0) grid_finalize<NT>(v, a.partials, a.ticket, a.fin, a.ctl);
    else if (a.pmode == 1) { if (threadIdx.x == 0) a.partials[a.pbase + blockIdx.x] = v; }
    else grid_finalize_pair<NT>(v, a.partials, a.pbase, a.ticket, a.fin, a.ctl);
}

// ---------------------------------------------------------------- SpMV

// numpy's pairwise sum over products read through `P` (leaf: n <= 128).
template <class PF>
__device__ __forceinline__ double pairwise_leaf(const PF &P, int base, int n)
{
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = add(r, P(base + i));
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = P(base + j);
    int i = 8;
    const int main = n - (n % 8);
    for (; i < main; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = add(r[j], P(base + i + j));
    }
    double res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
    for (; i < n; ++i) res = add(res, P(base + i));
    return res;
}

__device__ __forceinline__ int pairwise_split(int n)
{
    int n2 = n / 2;
    return n2 - n2 % 8;
}

// Full pairwise sum with numpy's recursive split (n > 128 -> halves at
// n/2 - (n/2) % 8), evaluated with an explicit stack (no device recursion).
template <class PF>
__device__ __noinline__ double pairwise_sum(const PF &P, int base, int n)
{
    if (n <= 128) return pairwise_leaf(P, base, n);
    int fb[32], fn[32];
    double fl[32];
    int fs[32];
    int sp = 0;
    int b = base, m = n;
    double ret;
    for (;;) {
        while (m > 128) {  // descend to the left child
            fb[sp] = b;
            fn[sp] = m;
            fs[sp] = 0;
            ++sp;
            m = pairwise_split(m);
        }
        ret = pairwise_leaf(P, b, m);
        bool descend = false;
        while (sp > 0) {
            const int t = sp - 1;
            if (fs[t] == 0) {  // left done: evaluate the right child
                fl[t] = ret;
                fs[t] = 1;
                const int n2 = pairwise_split(fn[t]);
                b = fb[t] + n2;
                m = fn[t] - n2;
                descend = true;
                break;
            }
            ret = add(fl[t], ret);
            --sp;
        }
        if (!descend) return ret;
    }
}

// Row sum in numpy order for one row whose PRODUCTS p_k sit at smem
// positions [lo - vdelta, hi - vdelta).  Executed by the LANES lanes of a
// group; the result is valid in the group's lane 0.
template <int LANES>
__device__ __forceinline__ double row_sum_staged(const double *__restrict__ ps, int vdelta, int lo, int hi, int lane,
                                                 unsigned gmask)
{
    auto P = [&](int k) -> double { return ps[k - vdelta]; };
    const int len = hi - lo;
    if (len <= 0) return 0.0;
    const int n = len - 1;
    const int base = lo + 1;
    if (n < 8 || n > 128) {
        double s = 0.0;
        if (lane == 0) {
            double res;
            if (n < 8) {
                res = 0.0;
                for (int i = 0; i < n; ++i) res = add(res, P(base + i));
            } else {
                res = pairwise_sum(P, base, n);
            }
            s = add(P(lo), res);
        }
        return s;
    }
    constexpr int M = 8 / LANES;  // accumulators per lane: r_{lane + m*LANES}
    const int main = n - (n % 8);
    double acc[M];
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = P(base + lane + m * LANES);
    for (int i = 8; i < main; i += 8) {
#pragma unroll
        for (int m = 0; m < M; ++m) acc[m] = add(acc[m], P(base + i + lane + m * LANES));
    }
    double res;
    if constexpr (LANES == 1) {
        res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
    } else if constexpr (LANES == 2) {
        // lane j holds r_j, r_{j+2}, r_{j+4}, r_{j+6}
        double u[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) u[m] = add(acc[m], __shfl_xor_sync(gmask, acc[m], 1));
        res = add(add(u[0], u[1]), add(u[2], u[3]));
    } else if constexpr (LANES == 4) {
        // lane j holds r_j, r_{j+4}
        double s0 = add(acc[0], __shfl_xor_sync(gmask, acc[0], 1));
        double s1 = add(acc[1], __shfl_xor_sync(gmask, acc[1], 1));
        s0 = add(s0, __shfl_xor_sync(gmask, s0, 2));
        s1 = add(s1, __shfl_xor_sync(gmask, s1, 2));
        res = add(s0, s1);
    } else {
        double t = acc[0];
        t = add(t, __shfl_xor_sync(gmask, t, 1));
        t = add(t, __shfl_xor_sync(gmask, t, 2));
        t = add(t, __shfl_xor_sync(gmask, t, 4));
        res = t;
    }
    double out = 0.0;
    if (lane == 0) {
        for (int i = main; i < n; ++i) res = add(res, P(base + i));
        out = add(P(lo), res);
    }
    return out;
}

template <int EPI>
__device__ __forceinline__ double epilogue(double s, const double *b, int64_t row, double omega)
{
    if constexpr (EPI == EPI_PLAIN) return s;
    if constexpr (EPI == EPI_RESID) return __dsub_rn(b[row], s);
    if constexpr (EPI == EPI_AXPYW) return add(b[row], __dmul_rn(omega, s));
    if constexpr (EPI == EPI_SETW) return __dmul_rn(omega, s);
    if constexpr (EPI == EPI_ADD) return add(b[row], s);
    return s;
}

// ---------------------------------------------------------------- SpMV, direct

// Register-only CSR SpMV: a group of LANES lanes owns a row; every load of
// the row (values, columns, then x gathers) is issued before the first add,
// and the sum is formed in the reference order (numpy's 8 strided
// accumulators over the lanes, shuffle-butterfly combine, sequential tail,
// p0 first).  No shared memory and no barriers, so occupancy is limited only
// by registers -- latency is hidden by many independent row groups.
// Rows with n = len - 1 > DIRECT_MAXN follow numpy's recursive split, every
// leaf summed by the whole lane group (direct_tree).
constexpr int DIRECT_THREADS = 256;

// matrix loads go through L1: with one lane per row a warp's 32 rows are
// contiguous, and L1 merges the per-lane strided loads (evict-first measured
// slower on B200: 255 vs 204 us for the 27-pt A0)
__device__ __forceinline__ double ldm(const double *p) { return __ldg(p); }
__device__ __forceinline__ int ldm(const int32_t *p) { return __ldg(p); }
constexpr int DIRECT_MAXN = 128;

// One pairwise leaf (8 <= n <= 128 products starting at `base`) in numpy's
// order -- 8 strided accumulators spread over the LANES lanes of a group,
// butterfly combine, sequential tail -- with every load of the leaf issued
// before the first add.  The result is valid (and identical) in all lanes.
template <int LANES>
__device__ __forceinline__ double direct_leaf(const double *__restrict__ val, const int32_t *__restrict__ col,
                                              const double *__restrict__ x, int base, int n, int lane, unsigned gmask)
{
    constexpr int M = 8 / LANES;  // accumulators per lane: r_{lane + m*LANES}
    const int main = n - (n % 8);
    const int its = main / 8;
    // tail (n % 8 entries): spread over the lanes, issued with the main loads
    const int ntail = n - main;
    constexpr int TT = (7 + LANES - 1) / LANES;  // tail entries per lane (tail <= 7)
    double tpa[TT];
#pragma unroll
    for (int j = 0; j < TT; ++j) {
        const int t = lane + j * LANES;
        tpa[j] = (t < ntail) ? prod(ldm(val + base + main + t), __ldg(x + ldm(col + base + main + t))) : 0.0;
    }
    // main rounds in chunks of R = LANES rounds: 8 loads in flight per lane per chunk
    constexpr int R = LANES;
    double acc[M];
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = 0.0;
    for (int c0 = 0; c0 < its; c0 += R) {
        double pv[R][M];
        int pc[R][M];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int m = 0; m < M; ++m)
                if (c0 + r < its) {
                    const int k = base + (c0 + r) * 8 + lane + m * LANES;
                    pv[r][m] = ldm(val + k);
                    pc[r][m] = ldm(col + k);
                }
        double xg[R][M];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int m = 0; m < M; ++m)
                if (c0 + r < its) xg[r][m] = __ldg(x + pc[r][m]);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int m = 0; m < M; ++m)
                if (c0 + r < its) {
                    const double pr = prod(pv[r][m], xg[r][m]);
                    acc[m] = (c0 + r == 0) ? pr : add(acc[m], pr);
                }
    }
    double res;
    if constexpr (LANES == 1) {
        res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
    } else if constexpr (LANES == 2) {
        double u[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) u[m] = add(acc[m], __shfl_xor_sync(gmask, acc[m], 1));
        res = add(add(u[0], u[1]), add(u[2], u[3]));
    } else if constexpr (LANES == 4) {
        double s0 = add(acc[0], __shfl_xor_sync(gmask, acc[0], 1));
        double s1 = add(acc[1], __shfl_xor_sync(gmask, acc[1], 1));
        s0 = add(s0, __shfl_xor_sync(gmask, s0, 2));
        s1 = add(s1, __shfl_xor_sync(gmask, s1, 2));
        res = add(s0, s1);
    } else {
        double t = acc[0];
        t = add(t, __shfl_xor_sync(gmask, t, 1));
        t = add(t, __shfl_xor_sync(gmask, t, 2));
        t = add(t, __shfl_xor_sync(gmask, t, 4));
        res = t;
    }
    // sequential tail (entries main..n-1 held by lanes t % LANES), broadcast to every lane
#pragma unroll
    for (int t = 0; t < 7; ++t) {
        const double v = (LANES == 1) ? tpa[t] : __shfl_sync(gmask, tpa[t / LANES], t % LANES, LANES);
        if (t < ntail) res = add(res, v);
    }
    return res;
}

// numpy's pairwise sum for n > 128 (split at n/2 - (n/2) % 8, leaves of
// 64..128 products) with the explicit-stack walk of pairwise_sum; the walk is
// uniform over the lane group and every leaf is a direct_leaf of all lanes.
template <int LANES>
__device__ __noinline__ double direct_tree(const double *__restrict__ val, const int32_t *__restrict__ col,
                                           const double *__restrict__ x, int base, int n, int lane, unsigned gmask)
{
    int fb[26], fn[26], fs[26];
    double fl[26];
    int sp = 0;
    int b = base, m = n;
    double ret;
    for (;;) {
        while (m > 128) {  // descend to the left child
            fb[sp] = b;
            fn[sp] = m;
            fs[sp] = 0;
            ++sp;
            m = pairwise_split(m);
        }
        ret = direct_leaf<LANES>(val, col, x, b, m, lane, gmask);
        bool descend = false;
        while (sp > 0) {
            const int t = sp - 1;
            if (fs[t] == 0) {  // left done: evaluate the right child
                fl[t] = ret;
                fs[t] = 1;
                const int n2 = pairwise_split(fn[t]);
                b = fb[t] + n2;
                m = fn[t] - n2;
                descend = true;
                break;
            }
            ret = add(fl[t], ret);
            --sp;
        }
        if (!descend) return ret;
    }
}

template <int EPI, int LANES>
__global__ void __launch_bounds__(DIRECT_THREADS, 4) spmv_direct(const SpmvArgs a, int nrows)
{
    __shared__ double red[DIRECT_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int lane = threadIdx.x % LANES;
    const int grp_in_warp = (threadIdx.x & 31) / LANES;
    const unsigned gmask = (LANES == 32) ? 0xffffffffu : (((1u << LANES) - 1u) << (grp_in_warp * LANES));
    const int ngroups = gridDim.x * (DIRECT_THREADS / LANES);
    const int g0 = blockIdx.x * (DIRECT_THREADS / LANES) + threadIdx.x / LANES;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const int32_t *__restrict__ off = a.off;
    const int32_t *__restrict__ col = a.col;
    const double *__restrict__ val = a.val;
    const double *__restrict__ x = a.x;
    double dacc = 0.0;
    // row offsets of the next row are fetched one iteration ahead
    int nlo = 0, nhi = 0;
    if (g0 < nrows) {
        const int r = vrow(a, g0);
        nlo = __ldg(off + r);
        nhi = __ldg(off + r + 1);
    }
    for (int v = g0; v < nrows; v += ngroups) {
        const int row = vrow(a, v);
        const int lo = nlo, hi = nhi;
        if (v + ngroups < nrows) {
            const int r = vrow(a, v + ngroups);
            nlo = __ldg(off + r);
            nhi = __ldg(off + r + 1);
        }
        const int n = hi - lo - 1;
        double bv = 0.0, wv = 0.0;
        if (lane == 0) {
            if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
            if (want_dot && !self_dot) wv = a.dotw[row];
        }
        double sum;
        if (n < 0) {
            sum = 0.0;
        } else if (n < 8) {
            // sequential: p0 + (((0 + p1) + p2) + ...); one lane per entry, gathered by shuffles
            double pk = 0.0;
            if (lane <= n) pk = prod(ldm(val + lo + lane), __ldg(x + ldm(col + lo + lane)));
            if constexpr (LANES >= 8) {
                double res = 0.0;
#pragma unroll
                for (int t = 1; t < 8; ++t) {
                    const double pt = __shfl_sync(gmask, pk, t, LANES);
                    if (t <= n) res = add(res, pt);
                }
                sum = add(__shfl_sync(gmask, pk, 0, LANES), res);
            } else {
                // fewer lanes than entries: each lane holds entries lane, lane+LANES, ...
                double pe[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) pe[t] = 0.0;
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if ((t % LANES) == lane && t <= n) pe[t] = prod(ldm(val + lo + t), __ldg(x + ldm(col + lo + t)));
                double res = 0.0;
#pragma unroll
                for (int t = 1; t < 8; ++t) {
                    const double pt = (LANES == 1) ? pe[t] : __shfl_sync(gmask, pe[t], t % LANES, LANES);
                    if (t <= n) res = add(res, pt);
                }
                const double p0 = (LANES == 1) ? pe[0] : __shfl_sync(gmask, pe[0], 0, LANES);
                sum = add(p0, res);
            }
        } else {
            // p0 issued with the first leaf's loads; n > DIRECT_MAXN walks numpy's
            // recursive split with every leaf summed by the whole lane group
            const double p0 = (lane == 0) ? prod(ldm(val + lo), __ldg(x + ldm(col + lo))) : 0.0;
            const double res = (n <= DIRECT_MAXN) ? direct_leaf<LANES>(val, col, x, lo + 1, n, lane, gmask)
                                                  : direct_tree<LANES>(val, col, x, lo + 1, n, lane, gmask);
            sum = add(p0, res);
        }
        if (lane == 0) {
            double yv;
            if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
            else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
            else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
            else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
            else yv = sum;
            a.y[row] = yv;
            if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
        }
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<DIRECT_THREADS>(dacc, red);
        spmv_finalize<DIRECT_THREADS>(v, a);
    }
}

// ---------------------------------------------------------------- SpMV, long rows

// Rows of several pairwise leaves (n > 128: coarse Galerkin operators of
// elasticity / aggressive coarsening).  The leaves only depend on the row
// lengths, so they are listed once at upload (numpy's split at
// n/2 - (n/2) % 8, leaves of 64..128 products) and every SpMV runs in two
// launches: spmv_leaves sums every leaf of the matrix side by side (8 lanes
// per leaf, direct_leaf), spmv_leafsum forms each row as p0 + the leaf sums
// folded in the tree's order, with the epilogue and the fused dot.  Rows with
// 8 <= n <= 128 are a single leaf; rows with n < 8 are summed in spmv_leafsum.
struct LeafArgs {
    const int2 *leaf;         // (first product index, products) per leaf, rows in order
    int nleaves;
    double *lsum;             // leaf sums
    const int32_t *row_leaf;  // first leaf of each row (nrows + 1)
};

// numpy's pairwise tree over a row's leaf sums (n = products after p0).
__device__ __forceinline__ double leaf_tree_combine(const double *sl, int n)
{
    int fn[26], fs[26];
    double fl[26];
    int sp = 0, m = n, j = 0;
    double ret;
    for (;;) {
        while (m > 128) {
            fn[sp] = m;
            fs[sp] = 0;
            ++sp;
            m = pairwise_split(m);
        }
        ret = sl[j++];
        bool descend = false;
        while (sp > 0) {
            const int t = sp - 1;
            if (fs[t] == 0) {
                fl[t] = ret;
                fs[t] = 1;
                m = fn[t] - pairwise_split(fn[t]);
                descend = true;
                break;
            }
            ret = add(fl[t], ret);
            --sp;
        }
        if (!descend) return ret;
    }
}

__global__ void __launch_bounds__(DIRECT_THREADS, 4) spmv_leaves(const SpmvArgs a, const LeafArgs la)
{
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int lane = threadIdx.x % 8;
    const unsigned tmask = 0xffu << ((threadIdx.x & 31) & ~7);
    const int teams = gridDim.x * (DIRECT_THREADS / 8);
    for (int v = blockIdx.x * (DIRECT_THREADS / 8) + threadIdx.x / 8; v < la.nleaves; v += teams) {
        const int2 d = __ldg(la.leaf + v);
        const double s = direct_leaf<8>(a.val, a.col, a.x, d.x, d.y, lane, tmask);
        if (lane == 0) la.lsum[v] = s;
    }
}

template <int EPI>
__global__ void __launch_bounds__(DIRECT_THREADS) spmv_leafsum(const SpmvArgs a, const LeafArgs la, int nrows)
{
    __shared__ double red[DIRECT_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    double dacc = 0.0;
    for (int row = blockIdx.x * DIRECT_THREADS + threadIdx.x; row < nrows; row += gridDim.x * DIRECT_THREADS) {
        const int lo = __ldg(a.off + row), hi = __ldg(a.off + row + 1);
        const int n = hi - lo - 1;
        double bv = 0.0, wv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
        if (want_dot && !self_dot) wv = a.dotw[row];
        double sum = 0.0;
        if (n >= 0) {
            const double p0 = prod(ldm(a.val + lo), __ldg(a.x + ldm(a.col + lo)));
            double res = 0.0;
            if (n < 8) {
                for (int t = 1; t <= n; ++t) res = add(res, prod(ldm(a.val + lo + t), __ldg(a.x + ldm(a.col + lo + t))));
            } else {
                const double *ls = la.lsum + __ldg(la.row_leaf + row);
                res = (n <= 128) ? ls[0] : leaf_tree_combine(ls, n);
            }
            sum = add(p0, res);
        }
        double yv;
        if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
        else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
        else yv = sum;
        a.y[row] = yv;
        if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<DIRECT_THREADS>(dacc, red);
        grid_finalize<DIRECT_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// ---------------------------------------------------------------- SpMV, padded-aligned rows

// Padded-aligned CSR (device-only layout for rows averaging >= ~12 entries):
// row i's entries start at pstart[i] with pstart[i] % 4 == 3, so entry 1 --
// the start of numpy's 8-wide rounds -- is 16-byte aligned for both the
// values (double2) and the columns (int4).  One lane per row; a round of 8
// entries is 4 double2 + 2 int4 loads (L1 sector lookups per entry drop ~3x
// versus scalar loads), gathers and sums exactly as the reference orders them.
constexpr int VEC_SPMV_THREADS = 256;

struct PadArgs {
    const int32_t *pstart;  // nrows + 1 padded row starts (== 3 mod 4)
    const double *pval;     // padded values (16-byte aligned base)
    const int32_t *pcol;    // padded columns
};

template <int EPI, int MINB = 4>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, MINB) spmv_vec(const SpmvArgs a, const PadArgs pa, int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    double dacc = 0.0;
    const int v0 = blockIdx.x * VEC_SPMV_THREADS + threadIdx.x;
    int nlo = 0, nhi = 0, nps = 0;
    int prow = 0;  // row of the next virtual position (row-range launches)
    if (v0 < nrows) {
        prow = vrow(a, v0);
        nlo = __ldg(a.off + prow);
        nhi = __ldg(a.off + prow + 1);
        nps = __ldg(pa.pstart + prow);
    }
    for (int pos = v0; pos < nrows; pos += nthreads) {
        const int row = prow;
        const int len = nhi - nlo;
        const int ps = nps;
        if (pos + nthreads < nrows) {  // next row's offsets one step ahead
            prow = vrow(a, pos + nthreads);
            nlo = __ldg(a.off + prow);
            nhi = __ldg(a.off + prow + 1);
            nps = __ldg(pa.pstart + prow);
        }
        double bv = 0.0, wv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
        if (want_dot && !self_dot) wv = a.dotw[row];
        const int n = len - 1;
        double sum = 0.0;
        if (n >= 0 && n <= 128) {
            const double p0 = prod(__ldg(pa.pval + ps), __ldg(x + __ldg(pa.pcol + ps)));
            const int b1 = ps + 1;  // 16-byte aligned
            const double2 *v2 = reinterpret_cast<const double2 *>(pa.pval + b1);
            const int4 *c4 = reinterpret_cast<const int4 *>(pa.pcol + b1);
            auto round8 = [&](int r, double p[8]) {
                const int4 ca = __ldg(c4 + 2 * r), cb = __ldg(c4 + 2 * r + 1);
                const double2 va = __ldg(v2 + 4 * r), vb = __ldg(v2 + 4 * r + 1), vc = __ldg(v2 + 4 * r + 2),
                              vd = __ldg(v2 + 4 * r + 3);
                p[0] = prod(va.x, __ldg(x + ca.x));
                p[1] = prod(va.y, __ldg(x + ca.y));
                p[2] = prod(vb.x, __ldg(x + ca.z));
                p[3] = prod(vb.y, __ldg(x + ca.w));
                p[4] = prod(vc.x, __ldg(x + cb.x));
                p[5] = prod(vc.y, __ldg(x + cb.y));
                p[6] = prod(vd.x, __ldg(x + cb.z));
                p[7] = prod(vd.y, __ldg(x + cb.w));
            };
            // masked round (entries beyond `cnt` belong to padding / the next row: not used)
            auto round8m = [&](int r, int cnt, double p[8]) {
                const int4 ca = __ldg(c4 + 2 * r);
                const int4 cb = cnt > 4 ? __ldg(c4 + 2 * r + 1) : make_int4(0, 0, 0, 0);
                const double2 va = __ldg(v2 + 4 * r);
                const double2 vb = cnt > 2 ? __ldg(v2 + 4 * r + 1) : make_double2(0.0, 0.0);
                const double2 vc = cnt > 4 ? __ldg(v2 + 4 * r + 2) : make_double2(0.0, 0.0);
                const double2 vd = cnt > 6 ? __ldg(v2 + 4 * r + 3) : make_double2(0.0, 0.0);
                const int cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
                const double vv[8] = {va.x, va.y, vb.x, vb.y, vc.x, vc.y, vd.x, vd.y};
#pragma unroll
                for (int t = 0; t < 8; ++t) p[t] = (t < cnt) ? prod(vv[t], __ldg(x + cc[t])) : 0.0;
            };
            double res;
            // the first round is shared by short (n < 8) and long rows, so a warp
            // with mixed row lengths diverges only in the (cheap) arithmetic
            double acc[8];
            round8m(0, n < 8 ? n : 8, acc);
            if (n < 8) {
                res = 0.0;
#pragma unroll
                for (int t = 0; t < 7; ++t)
                    if (t < n) res = add(res, acc[t]);
            } else {
                const int main = n - (n % 8);
                const int its = main / 8;
                for (int r = 1; r < its; ++r) {
                    double p[8];
                    round8(r, p);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = add(acc[j], p[j]);
                }
                res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
                const int ntail = n - main;
                if (ntail > 0) {
                    double p[8];
                    round8m(its, ntail, p);
#pragma unroll
                    for (int t = 0; t < 7; ++t)
                        if (t < ntail) res = add(res, p[t]);
                }
            }
            sum = add(p0, res);
        } else if (n > 128) {
            auto P = [&](int k) -> double { return prod(__ldg(pa.pval + ps + k), __ldg(x + __ldg(pa.pcol + ps + k))); };
            sum = add(P(0), pairwise_sum(P, 1, n));
        }
        double yv;
        if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
        else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
        else yv = sum;
        a.y[row] = yv;
        if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        spmv_finalize<VEC_SPMV_THREADS>(v, a);
    }
}

// ---------------------------------------------------------------- SpMV, stencil patterns

// Stencil-pattern CSR (device-only layout for square operators whose rows
// use at most 255 distinct relative column patterns, e.g. the 27-point
// fine-grid operators of the BASELINE configs): row i stores a 1-byte
// pattern id and its values in the padded-aligned layout; its columns are
// i + rel[pattern][k] with the pattern table in shared memory (staged before
// griddepcontrol.wait).  The 4-byte column stream disappears and the x
// gathers no longer wait on a global column load.  Same products, same
// reference summation order as spmv_vec.
constexpr int PAT_MAX = 255;
constexpr int PAT_MAX_REL = 8192;  // total relative offsets over all patterns

struct PatArgs {
    const int32_t *pstart;  // padded row starts (== 3 mod 4)
    const double *pval;
    const uint8_t *pid;     // pattern id per row
    const int32_t *rel;     // concatenated relative offsets (col - row)
    const int32_t *pbeg;    // npat + 1 starts into rel
    int npat;
    int nrel;
};

template <int EPI>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, 4) spmv_pat(const SpmvArgs a, const PatArgs pa, int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    __shared__ int32_t s_rel[PAT_MAX_REL];
    __shared__ int32_t s_beg[PAT_MAX + 1];
    for (int i = threadIdx.x; i < pa.nrel; i += blockDim.x) s_rel[i] = pa.rel[i];
    for (int i = threadIdx.x; i <= pa.npat; i += blockDim.x) s_beg[i] = pa.pbeg[i];
    __syncthreads();
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    double dacc = 0.0;
    int row = blockIdx.x * VEC_SPMV_THREADS + threadIdx.x;
    int nps = 0, npid = 0;
    if (row < nrows) {
        nps = __ldg(pa.pstart + row);
        npid = __ldg(pa.pid + row);
    }
    for (; row < nrows; row += nthreads) {
        const int ps = nps, pid = npid;
        if (row + nthreads < nrows) {
            nps = __ldg(pa.pstart + row + nthreads);
            npid = __ldg(pa.pid + row + nthreads);
        }
        double bv = 0.0, wv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
        if (want_dot && !self_dot) wv = a.dotw[row];
        const int rb = s_beg[pid];
        const int len = s_beg[pid + 1] - rb;
        const int32_t *rl = s_rel + rb;
        const int n = len - 1;
        double sum = 0.0;
        if (n >= 0 && n <= 128) {
            const double p0 = prod(__ldg(pa.pval + ps), __ldg(x + row + rl[0]));
            const double2 *v2 = reinterpret_cast<const double2 *>(pa.pval + ps + 1);
            const int32_t *r1 = rl + 1;
            auto round8 = [&](int r, double p[8]) {
                const double2 va = __ldg(v2 + 4 * r), vb = __ldg(v2 + 4 * r + 1), vc = __ldg(v2 + 4 * r + 2),
                              vd = __ldg(v2 + 4 * r + 3);
                const int k = 8 * r;
                p[0] = prod(va.x, __ldg(x + row + r1[k]));
                p[1] = prod(va.y, __ldg(x + row + r1[k + 1]));
                p[2] = prod(vb.x, __ldg(x + row + r1[k + 2]));
                p[3] = prod(vb.y, __ldg(x + row + r1[k + 3]));
                p[4] = prod(vc.x, __ldg(x + row + r1[k + 4]));
                p[5] = prod(vc.y, __ldg(x + row + r1[k + 5]));
                p[6] = prod(vd.x, __ldg(x + row + r1[k + 6]));
                p[7] = prod(vd.y, __ldg(x + row + r1[k + 7]));
            };
            auto round8m = [&](int r, int cnt, double p[8]) {
                const double2 va = __ldg(v2 + 4 * r);
                const double2 vb = cnt > 2 ? __ldg(v2 + 4 * r + 1) : make_double2(0.0, 0.0);
                const double2 vc = cnt > 4 ? __ldg(v2 + 4 * r + 2) : make_double2(0.0, 0.0);
                const double2 vd = cnt > 6 ? __ldg(v2 + 4 * r + 3) : make_double2(0.0, 0.0);
                const double vv[8] = {va.x, va.y, vb.x, vb.y, vc.x, vc.y, vd.x, vd.y};
                const int k = 8 * r;
#pragma unroll
                for (int t = 0; t < 8; ++t) p[t] = (t < cnt) ? prod(vv[t], __ldg(x + row + r1[k + t])) : 0.0;
            };
            double res;
            double acc[8];
            round8m(0, n < 8 ? n : 8, acc);
            if (n < 8) {
                res = 0.0;
#pragma unroll
                for (int t = 0; t < 7; ++t)
                    if (t < n) res = add(res, acc[t]);
            } else {
                const int main = n - (n % 8);
                const int its = main / 8;
                for (int r = 1; r < its; ++r) {
                    double p[8];
                    round8(r, p);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = add(acc[j], p[j]);
                }
                res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
                const int ntail = n - main;
                if (ntail > 0) {
                    double p[8];
                    round8m(its, ntail, p);
#pragma unroll
                    for (int t = 0; t < 7; ++t)
                        if (t < ntail) res = add(res, p[t]);
                }
            }
            sum = add(p0, res);
        } else if (n > 128) {
            auto P = [&](int k) -> double { return prod(__ldg(pa.pval + ps + k), __ldg(x + row + rl[k])); };
            sum = add(P(0), pairwise_sum(P, 1, n));
        }
        double yv;
        if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
        else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
        else yv = sum;
        a.y[row] = yv;
        if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        grid_finalize<VEC_SPMV_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// ---------------------------------------------------------------- SpMV, SELL-32 slices

// SELL-32 (sliced ELLPACK, slice = 32 consecutive rows = one warp): entry k
// of the slice's rows is stored contiguously (sval[sbeg + 32 k + lane]), so
// every value / column load of a warp is one fully coalesced 256 / 128-byte
// access.  Lane = row, each lane sums its own row in the reference order
// (p0 + numpy pairwise over 8 strided accumulators), so results are
// bit-identical.  Columns come from the stencil-pattern table (PAT) or from
// the SELL column array.  Used where slices are uniform (padding <= ~10%).
struct SellArgs {
    const int32_t *sbeg;    // per slice: start (entries) of the slice block
    const double *sval;
    const int32_t *scol;    // nullptr with PAT
    const uint8_t *len;     // row lengths (<= 129)
    const uint8_t *pid;     // PAT: pattern id per row
    const int32_t *rel;
    const int32_t *pbeg;
    int npat, nrel;
    const int32_t *perm;    // SELL-sigma: original row of each slice position (nullptr: identity)
};

template <int EPI, bool PAT>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, PAT ? 5 : 4) spmv_sell(const SpmvArgs a, const SellArgs sa, int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    __shared__ int32_t s_rel[PAT ? PAT_MAX_REL : 1];
    __shared__ int32_t s_beg[PAT ? PAT_MAX + 1 : 1];
    if constexpr (PAT) {
        for (int i = threadIdx.x; i < sa.nrel; i += blockDim.x) s_rel[i] = sa.rel[i];
        for (int i = threadIdx.x; i <= sa.npat; i += blockDim.x) s_beg[i] = sa.pbeg[i];
        __syncthreads();
    }
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int lane = threadIdx.x & 31;
    const int nslices = (nrows + 31) >> 5;
    const int wstride = gridDim.x * (VEC_SPMV_THREADS / 32);
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    double dacc = 0.0;
    for (int sl = blockIdx.x * (VEC_SPMV_THREADS / 32) + (threadIdx.x >> 5); sl < nslices; sl += wstride) {
        const int pos = sl * 32 + lane;  // slice position (== row unless rows are sigma-sorted)
        const bool live = pos < nrows;
        const int sb = __ldg(sa.sbeg + sl);
        int len = 0, rb = 0, row = pos;
        if (live) {
            len = __ldg(sa.len + pos);
            if (sa.perm) row = __ldg(sa.perm + pos);
            if constexpr (PAT) rb = s_beg[__ldg(sa.pid + row)];
        }
        double bv = 0.0, wv = 0.0;
        if (live) {
            if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
            if (want_dot && !self_dot) wv = a.dotw[row];
        }
        const double *vb = sa.sval + sb + lane;
        const int32_t *cb = PAT ? nullptr : sa.scol + sb + lane;
        auto P = [&](int k) -> double {
            const int c = PAT ? row + s_rel[rb + k] : __ldg(cb + 32 * k);
            return prod(__ldg(vb + 32 * k), __ldg(x + c));
        };
        const int n = len - 1;
        double sum = 0.0;
        if (n >= 0 && n <= 128) {
            double acc[8];
            // first round shared by short and long rows (masked)
            const int c0 = n < 8 ? n : 8;
            const double p0 = P(0);
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[t] = (t < c0) ? P(1 + t) : 0.0;
            double res;
            if (n < 8) {
                res = 0.0;
#pragma unroll
                for (int t = 0; t < 7; ++t)
                    if (t < n) res = add(res, acc[t]);
            } else {
                const int main = n - (n % 8);
                for (int i = 8; i < main; i += 8) {
                    double p[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) p[t] = P(1 + i + t);
#pragma unroll
                    for (int t = 0; t < 8; ++t) acc[t] = add(acc[t], p[t]);
                }
                res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
                const int ntail = n - main;
                double p[7];
#pragma unroll
                for (int t = 0; t < 7; ++t) p[t] = (t < ntail) ? P(1 + main + t) : 0.0;
#pragma unroll
                for (int t = 0; t < 7; ++t)
                    if (t < ntail) res = add(res, p[t]);
            }
            sum = add(p0, res);
        } else if (n > 128) {
            sum = add(P(0), pairwise_sum(P, 1, n));
        }
        if (live) {
            double yv;
            if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
            else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
            else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
            else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
            else yv = sum;
            a.y[row] = yv;
            if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
        }
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        grid_finalize<VEC_SPMV_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// ---------------------------------------------------------------- SpMV, symmetric stencil diagonals

// Symmetric stencil layout (device-only, chosen at upload for square operators
// that are BITWISE symmetric, a_ij == a_ji, and whose rows use few relative
// column patterns -- the fine-grid operators of configs 1, 2 and 4): only the
// diagonals d >= 0 are stored, as nu arrays of npad doubles,
//     uval[j * npad + i] = a(i, i + d_j),
// and an entry of row i below the diagonal (d < 0) is read from its mirror,
//     a(i, i + d) = a(i + d, i) = uval[j(-d) * npad + i + d].
// Lane = row, consecutive rows per warp, so both reads are coalesced; the
// mirror read touches a line read by the sweep |d| rows earlier (an L2 hit),
// so HBM sees ~half of the value stream of a full copy.  Per pattern entry k
// the smem table holds {rel, voff}: column = row + rel, value = uval[row +
// voff].  Entries are visited in the row's stored (ascending column) order and
// summed in the reference order (p0 + numpy pairwise), so every row sum is
// bit-identical to amgkit/sparse.py:212-217.
// Pattern tables live in __constant__ memory: warp-uniform reads are
// constant-cache broadcasts (LDC) and stay off the LSU pipe, which the value
// and x streams saturate.  SYMD_SLOTS tables per device, handed out per matrix
// at upload (capi.cu symd_slot_*).
constexpr int SYMD_SLOTS = 8;
constexpr int SYMD_TAB = 4096;           // pattern entries over all tables of a device (32 KB)
constexpr int SYMD_BEG_MAX = PAT_MAX + 1;
// entry {rel, y}: column = row + rel; value = stored diagonal j of row r2 = row + (below ? rel : 0)
// (its mirror when below the diagonal): y = j * npad + (r2 - row) diagonal-major, or
// y = ((r2 - row) << 6) | j slice-blocked
__constant__ int2 c_symd_tab[SYMD_TAB];
__constant__ int32_t c_symd_beg[SYMD_SLOTS * SYMD_BEG_MAX];   // absolute starts into c_symd_tab

struct SymArgs {
    const double *uval;
    const uint8_t *pid;  // pattern id per row
    int slot;
    int chunk;  // > 0: CTA b sweeps rows [b*chunk, (b+1)*chunk) in 256-row steps (x and mirror lines
                // reused from L1 by the next step); 0: grid-stride over 256-row blocks
    int w32;    // slice-blocked storage (BLK): the nu diagonals of each 32-row slice contiguous,
                // uval[(i/32)*w32 + 32 j + i%32], w32 = 32 nu
    int npad;   // diagonal-major storage (!BLK): uval[j * npad + i]
    int tbase, nent, npat;  // this matrix's entries in c_symd_tab (staged to smem by the TSM variant)
};

// value index of pattern entry {rel, y} for `row`
template <bool BLK>
__device__ __forceinline__ int symd_vidx(int row, int y, int w32)
{
    if constexpr (!BLK) return row + y;
    const int r2 = row + (y >> 6);
    return (r2 >> 5) * w32 + ((y & 63) << 5) + (r2 & 31);
}

// reference row sum of P(0..len-1): p0 + numpy pairwise(p1..), as spmv_sell
template <bool LONG, class PF>
__device__ __forceinline__ double ref_row_sum(const PF &P, int len)
{
    const int n = len - 1;
    double sum = 0.0;
    if (n >= 0 && n <= 128) {
        double acc[8];
        const int c0 = n < 8 ? n : 8;
        const double p0 = P(0);
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = (t < c0) ? P(1 + t) : 0.0;
        double res;
        if (n < 8) {
            res = 0.0;
#pragma unroll
            for (int t = 0; t < 7; ++t)
                if (t < n) res = add(res, acc[t]);
        } else {
            const int main = n - (n % 8);
            for (int i = 8; i < main; i += 8) {
                double p[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) p[t] = P(1 + i + t);
#pragma unroll
                for (int t = 0; t < 8; ++t) acc[t] = add(acc[t], p[t]);
            }
            res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
            const int ntail = n - main;
            double p[7];
#pragma unroll
            for (int t = 0; t < 7; ++t) p[t] = (t < ntail) ? P(1 + main + t) : 0.0;
#pragma unroll
            for (int t = 0; t < 7; ++t)
                if (t < ntail) res = add(res, p[t]);
        }
        sum = add(p0, res);
    } else if (LONG && n > 128) {
        sum = add(P(0), pairwise_sum(P, 1, n));
    }
    return sum;
}

template <int EPI, int MINB, bool BLK, bool TSM = false>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, MINB) spmv_symd(const SpmvArgs a, const SymArgs sa, int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    extern __shared__ int2 symd_stab[];  // TSM: the pattern table staged in smem (entries, then starts)
    int32_t *symd_sbeg = reinterpret_cast<int32_t *>(symd_stab + (TSM ? sa.nent : 0));
    if constexpr (TSM) {
        for (int i = threadIdx.x; i < sa.nent; i += blockDim.x) symd_stab[i] = c_symd_tab[sa.tbase + i];
        for (int i = threadIdx.x; i <= sa.npat; i += blockDim.x)
            symd_sbeg[i] = c_symd_beg[sa.slot * SYMD_BEG_MAX + i] - sa.tbase;
        __syncthreads();
    }
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    const double *__restrict__ uv = sa.uval;
    const int bbase = sa.slot * SYMD_BEG_MAX;
    double dacc = 0.0;
    const int r0 = sa.chunk ? blockIdx.x * sa.chunk : blockIdx.x * VEC_SPMV_THREADS;
    const int rend = sa.chunk ? min(nrows, r0 + sa.chunk) : nrows;
    const int step = sa.chunk ? VEC_SPMV_THREADS : nthreads;
    for (int row = r0 + threadIdx.x; row < rend; row += step) {
        const int pid = __ldg(sa.pid + row);
        double bv = 0.0, wv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
        if (want_dot && !self_dot) wv = a.dotw[row];
        const int rb = TSM ? symd_sbeg[pid] : c_symd_beg[bbase + pid];
        const int len = (TSM ? symd_sbeg[pid + 1] : c_symd_beg[bbase + pid + 1]) - rb;
        auto P = [&](int k) -> double {
            const int2 q = TSM ? symd_stab[rb + k] : c_symd_tab[rb + k];
            return prod(__ldg(uv + symd_vidx<BLK>(row, q.y, sa.w32)), __ldg(x + (row + q.x)));
        };
        const double sum = ref_row_sum<false>(P, len);  // pattern rows have <= 129 entries
        double yv;
        if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
        else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
        else yv = sum;
        a.y[row] = yv;
        if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        grid_finalize<VEC_SPMV_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// Interior fast path for 27-entry rows (the 27-point operator of configs 2 / 5): when all 32
// rows of a warp have the most frequent pattern, the pattern is not decoded from the
// constant-memory table -- every column offset and every value offset (own diagonal, or the
// mirror's slice-blocked position) is a kernel parameter, i.e. a constant-bank operand of the
// address arithmetic, and the 27 products are folded by straight-line code in the reference
// order (p0 + pairwise over p1..p26: 8 accumulators x 3 rounds, tree, 2-entry tail).  The
// table-driven loop spends ~24 instructions per entry (ncu: 45% of the issue slots at 660
// instructions per 32 rows); this path ~9.  A mirror entry a(i, i - d) sits in row i - d's
// slice: with i = 32 s + l the offset from the row's own slot takes two values, split at
// lane l = d mod 32 (voffA for lanes >= thr, voffB below).
struct SymFast {
    int pat;                 // pattern id of the interior rows (-1: no fast path)
    int thr[27];
    long long xoff[27];      // column offset in bytes
    long long voffA[27], voffB[27];
};

#ifndef SYMD27_MINB
#define SYMD27_MINB 4
#endif
template <int EPI>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, SYMD27_MINB) spmv_symd27(const SpmvArgs a, const SymArgs sa, const SymFast fa,
                                                                    int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const int lane = threadIdx.x & 31;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    const double *__restrict__ uv = sa.uval;
    const int bbase = sa.slot * SYMD_BEG_MAX;
    double dacc = 0.0;
    const int r0 = sa.chunk ? blockIdx.x * sa.chunk : blockIdx.x * VEC_SPMV_THREADS;
    const int rend = sa.chunk ? min(nrows, r0 + sa.chunk) : nrows;
    const int step = sa.chunk ? VEC_SPMV_THREADS : nthreads;
    // warp-uniform trip count (the vote needs every lane); lanes beyond the last row idle
    for (int row = r0 + threadIdx.x; row - lane < rend; row += step) {
        const bool inr = row < rend;
        const int pid = inr ? __ldg(sa.pid + row) : -1;
        double bv = 0.0, wv = 0.0, sum = 0.0;
        if (inr) {
            if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
            if (want_dot && !self_dot) wv = a.dotw[row];
        }
        if (__all_sync(0xffffffffu, pid == fa.pat)) {
            const char *xr = reinterpret_cast<const char *>(x + row);
            const char *vr = reinterpret_cast<const char *>(uv + ((row >> 5) * sa.w32 + (row & 31)));
            auto PV = [&](int k) -> double {
                const long long vo = (lane >= fa.thr[k]) ? fa.voffA[k] : fa.voffB[k];
                return prod(__ldg(reinterpret_cast<const double *>(vr + vo)),
                            __ldg(reinterpret_cast<const double *>(xr + fa.xoff[k])));
            };
            const double p0 = PV(0);
            double acc[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[t] = PV(1 + t);
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[t] = add(acc[t], PV(9 + t));
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[t] = add(acc[t], PV(17 + t));
            double res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
            res = add(res, PV(25));
            res = add(res, PV(26));
            sum = add(p0, res);
        } else if (inr) {
            const int rb = c_symd_beg[bbase + pid];
            const int len = c_symd_beg[bbase + pid + 1] - rb;
            auto P = [&](int k) -> double {
                const int2 q = c_symd_tab[rb + k];
                return prod(__ldg(uv + symd_vidx<true>(row, q.y, sa.w32)), __ldg(x + (row + q.x)));
            };
            sum = ref_row_sum<false>(P, len);
        }
        if (inr) {
            double yv;
            if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
            else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
            else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
            else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
            else yv = sum;
            a.y[row] = yv;
            if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
        }
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        grid_finalize<VEC_SPMV_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// Fixed-slot variant for matrices whose rows have at most FL entries (the
// stencil operators: FL = 8 covers 7-point, FL = 32 the 27-point rows).  Every
// lane walks the same FL statically unrolled slots, slot k live iff k < len:
// all loads of a row are independent and issued together (no round-by-round
// dependency), and rows of different lengths in one warp (boundary rows) do
// not diverge -- the reference summation order for the lane's own len is
// realised with predicated adds:
//   n = len - 1 < 8 : res = p1 + p2 + ... (sequential), y = p0 + res
//   n >= 8          : acc_t = p_{1+t} + p_{9+t} + ... over the main part
//                     (main = n - n % 8), ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)),
//                     then the n % 8 tail sequentially, y = p0 + res
// exactly as ref_row_sum / numpy's pairwise_sum (n <= 128 here).
// Reference row sum (p0 + numpy pairwise) of the first len of FL products
// held in registers, realised with predicated adds (no divergence between
// rows of different lengths):
//   n = len - 1 < 8 : res = p1 + p2 + ... (sequential), y = p0 + res
//   n >= 8          : acc_t = p_{1+t} + p_{9+t} + ... over the main part
//                     (main = n - n % 8), ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)),
//                     then the n % 8 tail sequentially, y = p0 + res
// exactly as ref_row_sum / numpy's pairwise_sum (len <= FL <= 129).
template <int FL>
__device__ __forceinline__ double ref_sum_fixed(const double (&p)[FL], int len)
{
    const int n = len - 1;
    double res = 0.0;
    if (FL <= 8 || n < 8) {  // len <= FL: arrays of <= 8 products never reach the 8-accumulator part
#pragma unroll
        for (int k = 1; k < (FL < 8 ? FL : 8); ++k)
            if (k <= n) res = add(res, p[k]);
    } else {
        const int main = n - (n % 8);
        double acc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = (1 + t < FL) ? p[1 + t] : 0.0;
#pragma unroll
        for (int k = 9; k < FL; ++k)
            if (k <= main) acc[(k - 1) % 8] = add(acc[(k - 1) % 8], p[k]);
        res = add(add(add(acc[0], acc[1]), add(acc[2], acc[3])), add(add(acc[4], acc[5]), add(acc[6], acc[7])));
#pragma unroll
        for (int k = 9; k < FL; ++k)
            if (k > main && k <= n) res = add(res, p[k]);
    }
    return len > 0 ? add(p[0], res) : 0.0;
}

template <int EPI, int FL, int MINB, bool BLK>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, MINB) spmv_symd_fixed(const SpmvArgs a, const SymArgs sa,
                                                                                     int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    const double *__restrict__ uv = sa.uval;
    const int bbase = sa.slot * SYMD_BEG_MAX;
    double dacc = 0.0;
    const int r0 = sa.chunk ? blockIdx.x * sa.chunk : blockIdx.x * VEC_SPMV_THREADS;
    const int rend = sa.chunk ? min(nrows, r0 + sa.chunk) : nrows;
    const int step = sa.chunk ? VEC_SPMV_THREADS : nthreads;
    int row = r0 + threadIdx.x;
    int npid = row < rend ? __ldg(sa.pid + row) : 0;
    for (; row < rend; row += step) {
        const int pid = npid;
        if (row + step < rend) npid = __ldg(sa.pid + row + step);
        double bv = 0.0, wv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
        if (want_dot && !self_dot) wv = a.dotw[row];
        const int rb = c_symd_beg[bbase + pid];
        const int len = c_symd_beg[bbase + pid + 1] - rb;
        double p[FL];
#pragma unroll
        for (int k = 0; k < FL; ++k) {
            p[k] = 0.0;
            if (k < len) {
                const int2 q = c_symd_tab[rb + k];
                p[k] = prod(__ldg(uv + symd_vidx<BLK>(row, q.y, sa.w32)), __ldg(x + (row + q.x)));
            }
        }
        const double sum = ref_sum_fixed<FL>(p, len);
        double yv;
        if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
        else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
        else yv = sum;
        a.y[row] = yv;
        if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        grid_finalize<VEC_SPMV_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// ---------------------------------------------------------------- SpMV, warp-cooperative CSR

// Plain CSR (no extra copy), one warp per group of 32 consecutive rows: the
// group's entries [off[r0], off[r0 + 32]) are contiguous, so the warp streams
// values and columns with fully coalesced loads (lane-strided entries, all of
// a lane's loads issued before the first gather), gathers x, and parks the
// products in a per-warp shared-memory buffer; then lane l sums row r0 + l
// from the buffer in the reference order (row_sum_staged: p0 + numpy
// pairwise).  Versus one lane per row walking its own row, every warp-level
// load touches 1-2 lines instead of ~32, and no padding is moved.  Groups
// with more than WCSR_BUF entries go through the buffer in row chunks.
constexpr int WCSR_THREADS = 256;
constexpr int WCSR_BUF = 640;   // products per warp (5.3 KB with the skew; 8 warps = 42 KB per CTA)
// buffer slot of product k: one pad slot every 16 (rows starting 16 products
// apart -- the same bank -- land on different banks when lanes sum their rows)
__device__ __forceinline__ int wslot(int k) { return k + (k >> 4); }
constexpr int WCSR_UNROLL = 10; // entries per lane issued together (one pass of a <= 320-entry group)

// reference row sum (p0 + numpy pairwise) of the products in skewed slots [lo, hi)
__device__ __forceinline__ double wcsr_row_sum(const double *ps, int lo, int hi)
{
    auto P = [&](int k) -> double { return ps[wslot(k)]; };
    const int n = hi - lo - 1;
    if (n < 0) return 0.0;
    return add(P(lo), n <= 128 ? pairwise_leaf(P, lo + 1, n) : pairwise_sum(P, lo + 1, n));
}

template <int EPI>
__global__ void __launch_bounds__(WCSR_THREADS, 3) spmv_wcsr(const SpmvArgs a, int nrows)
{
    __shared__ double red[WCSR_THREADS / 32];
    __shared__ double buf[WCSR_THREADS / 32][WCSR_BUF + WCSR_BUF / 16];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *ps = buf[warp];
    const int ngroups = (nrows + 31) >> 5;
    const int gstride = gridDim.x * (WCSR_THREADS / 32);
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const int32_t *__restrict__ off = a.off;
    const int32_t *__restrict__ col = a.col;
    const double *__restrict__ val = a.val;
    const double *__restrict__ x = a.x;
    double dacc = 0.0;
    int g = blockIdx.x * (WCSR_THREADS / 32) + warp;
    // offsets of this lane's row, one group ahead
    int nlo = 0, nhi = 0, nrow = -1;
    auto fetch = [&](int gg) {
        const int v = gg * 32 + lane;
        nrow = v < nrows ? vrow(a, v) : -1;
        if (nrow >= 0) {
            nlo = __ldg(off + nrow);
            nhi = __ldg(off + nrow + 1);
        } else {
            nlo = nhi = -1;
        }
    };
    if (g < ngroups) fetch(g);
    for (; g < ngroups; g += gstride) {
        const int row = nrow;
        const int lo = nlo, hi = nhi;
        if (g + gstride < ngroups) fetch(g + gstride);
        double bv = 0.0, wv = 0.0;
        if (row >= 0) {
            if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
            if (want_dot && !self_dot) wv = a.dotw[row];
        }
        // group entry range: rows of a group are consecutive (range starts are 128-aligned)
        const int k0 = __shfl_sync(0xffffffffu, lo, 0);
        int last = 31;
        {
            const unsigned live = __ballot_sync(0xffffffffu, row >= 0);
            last = 31 - __clz(live);
        }
        const int k1 = __shfl_sync(0xffffffffu, hi, last);
        double sum = 0.0;
        if (k1 - k0 <= WCSR_BUF) {
            const int nk = k1 - k0;
            for (int kb = 0; kb < nk; kb += 32 * WCSR_UNROLL) {
                double pv[WCSR_UNROLL];
                int pc[WCSR_UNROLL];
                // clamped (not predicated) loads keep pv / pc in registers
#pragma unroll
                for (int u = 0; u < WCSR_UNROLL; ++u) {
                    const int k = min(kb + u * 32 + lane, nk - 1);
                    pv[u] = __ldg(val + k0 + k);
                    pc[u] = __ldg(col + k0 + k);
                }
#pragma unroll
                for (int u = 0; u < WCSR_UNROLL; ++u) {
                    const double xv = __ldg(x + pc[u]);
                    const int k = kb + u * 32 + lane;
                    AMG_CHECK(k >= nk || wslot(k) < WCSR_BUF + WCSR_BUF / 16);
                    if (k < nk) ps[wslot(k)] = prod(pv[u], xv);
                }
            }
            __syncwarp();
            if (row >= 0) sum = wcsr_row_sum(ps, lo - k0, hi - k0);
            __syncwarp();
        } else {
            // a heavy group: its rows through the buffer in chunks of whole rows
            // (a single row longer than the buffer sums straight from global memory)
            int rs = 0;  // first lane of the chunk
            while (rs <= last) {
                const int ks = __shfl_sync(0xffffffffu, lo, rs);
                int re = rs;  // chunk = lanes [rs, re]
                while (re < last && __shfl_sync(0xffffffffu, hi, re + 1) - ks <= WCSR_BUF) ++re;
                const int ke = __shfl_sync(0xffffffffu, hi, re);
                if (ke - ks <= WCSR_BUF) {
                    for (int k = lane; k < ke - ks; k += 32) ps[wslot(k)] = prod(__ldg(val + ks + k), __ldg(x + __ldg(col + ks + k)));
                    __syncwarp();
                    if (lane >= rs && lane <= re && row >= 0) sum = wcsr_row_sum(ps, lo - ks, hi - ks);
                    __syncwarp();
                } else if (lane == rs && row >= 0) {
                    auto P = [&](int k) -> double { return prod(__ldg(val + k), __ldg(x + __ldg(col + k))); };
                    const int n = hi - lo - 1;
                    sum = n < 0 ? 0.0 : add(P(lo), pairwise_sum(P, lo + 1, n));
                }
                rs = re + 1;
            }
        }
        if (row >= 0) {
            double yv;
            if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
            else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
            else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
            else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
            else yv = sum;
            a.y[row] = yv;
            if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
        }
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<WCSR_THREADS>(dacc, red);
        spmv_finalize<WCSR_THREADS>(v, a);
    }
}

// ---------------------------------------------------------------- SpMV, row-class dictionary

// Operators whose rows fall into few distinct (column-offset tuple, value
// tuple) classes -- constant-coefficient stencils and the FSAI factors built
// from them (config 1 / config 4 level 0: A 27 classes, G 7, G^T 14 of
// 262 k rows) -- are stored as ONE class id per row (1 or 2 bytes) plus a
// class table {start, offsets, values} held in shared memory.  A row then
// costs its class id, its x gathers and its y store: the value and column
// streams disappear from HBM.  Entry k of a row is val[k] * x[row + rel[k]]
// with exactly the stored value, summed in the reference order (p0 + numpy
// pairwise, ref_sum_fixed), so every row is bit-identical to the CSR SpMV.
struct DictArgs {
    const void *cls;      // uint8_t or uint16_t per row (WIDE)
    const int32_t *beg;   // class starts [ncls + 1]
    const int32_t *rel;   // column offset col - row per entry
    const double *val;    // value per entry
    int ncls, nent;
    // the most frequent class (rows of <= 8 entries; -1: none): its offsets and values travel as
    // kernel parameters, i.e. constant-bank operands -- a warp whose 32 rows all have it (the
    // interior of a stencil operator) reads no table at all
    int mcls, mlen;
    int32_t mrel[8];
    long long moff[8];  // mrel in bytes (64-bit: the interior path adds it to the row's x pointer)
    double mval[8];
};

// ROWS rows per thread and step (rows row, row + nthreads, ...), all gathers issued before the
// first sum.  Only ROWS = 1 is instantiated: two rows helped the table-driven path (G0 27.6 ->
// 20.2 us) but lose to one row once the interior path is lean (16.5 us); a contiguous row chunk
// per CTA (x lines reused from L1: hit rate 27 -> 50%, 37% fewer L2 sectors, ncu) was never faster.
// ML > 0: the most frequent class has ML entries (compile time): the interior path is ML
// independent gathers at constant-bank offsets, ML products with constant-bank values and
// the reference-order sum of exactly ML terms -- no predicates, no table (ncu on the general
// path: 61% of the issue slots busy with 145 instructions per 32 rows).
template <int EPI, int FL, bool WIDE, int ROWS, int ML = 0>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, (ROWS > 1 || FL > 8) ? 4 : 5) spmv_dict(const SpmvArgs a, const DictArgs d,
                                                                                          int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    extern __shared__ double dict_sm[];  // val[nent] | rel[nent] | beg[ncls + 1]
    double *sval = dict_sm;
    int32_t *srel = reinterpret_cast<int32_t *>(dict_sm + d.nent);
    int32_t *sbeg = srel + d.nent;
    for (int i = threadIdx.x; i < d.nent; i += blockDim.x) {  // static data: staged before the PDL wait
        sval[i] = d.val[i];
        srel[i] = d.rel[i];
    }
    for (int i = threadIdx.x; i <= d.ncls; i += blockDim.x) sbeg[i] = d.beg[i];
    __syncthreads();
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    auto cls_at = [&](int r) -> int {
        if constexpr (WIDE) return __ldg(reinterpret_cast<const uint16_t *>(d.cls) + r);
        else return __ldg(reinterpret_cast<const uint8_t *>(d.cls) + r);
    };
    double dacc = 0.0;
    const int rstep = nthreads;  // distance of a thread's consecutive rows
    const int rend = nrows;
    int row0 = blockIdx.x * VEC_SPMV_THREADS + threadIdx.x;
    auto cls_of = [&](int r) -> int { return r < rend ? cls_at(r) : 0; };
    int ncl[ROWS];
#pragma unroll
    for (int q = 0; q < ROWS; ++q) ncl[q] = cls_of(row0 + q * rstep);
    // warp-uniform trip count (the vote below needs every lane): lanes beyond the last row idle
    for (; row0 - (int)(threadIdx.x & 31) < rend; row0 += ROWS * rstep) {
        int len[ROWS];
        bool fast[ROWS];
        double p[ROWS][FL], bv[ROWS], wv[ROWS];
#pragma unroll
        for (int q = 0; q < ROWS; ++q) {
            const int row = row0 + q * rstep;
            const int c = ncl[q];
            ncl[q] = cls_of(row + ROWS * rstep);  // the class one step ahead
            AMG_CHECK(c >= 0 && c < d.ncls);
            bv[q] = wv[q] = 0.0;
            if (row < rend) {
                if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv[q] = a.b[row];
                if (want_dot && !self_dot) wv[q] = a.dotw[row];
            }
            fast[q] = false;
            len[q] = 0;
            if constexpr (ML > 0) fast[q] = __all_sync(0xffffffffu, c == d.mcls && row < rend);
            if (fast[q]) {
                if constexpr (ML > 0) {
                    const char *xr = reinterpret_cast<const char *>(x + row);
#pragma unroll
                    for (int k = 0; k < ML; ++k)
                        p[q][k] = prod(d.mval[k], __ldg(reinterpret_cast<const double *>(xr + d.moff[k])));
                }
            } else {
                const int rb = sbeg[c];
                len[q] = row < rend ? sbeg[c + 1] - rb : 0;
                AMG_CHECK(len[q] >= 0 && len[q] <= FL && rb + len[q] <= d.nent);
#pragma unroll
                for (int k = 0; k < FL; ++k) {
                    p[q][k] = 0.0;
                    if (k < len[q]) p[q][k] = prod(sval[rb + k], __ldg(x + (row + srel[rb + k])));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < ROWS; ++q) {
            const int row = row0 + q * rstep;
            if (row < rend) {
                double sum;
                if (ML > 0 && fast[q]) {
                    double t[ML > 0 ? ML : 1];
#pragma unroll
                    for (int k = 0; k < ML; ++k) t[k] = p[q][k];
                    sum = ref_sum_fixed<(ML > 0 ? ML : 1)>(t, ML);
                } else {
                    sum = ref_sum_fixed<FL>(p[q], len[q]);
                }
                double yv;
                if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv[q], sum);
                else if constexpr (EPI == EPI_AXPYW) yv = add(bv[q], __dmul_rn(a.omega, sum));
                else if constexpr (EPI == EPI_ADD) yv = add(bv[q], sum);
                else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
                else yv = sum;
                a.y[row] = yv;
                if (want_dot) dacc = fma(yv, self_dot ? yv : wv[q], dacc);
            }
        }
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        grid_finalize<VEC_SPMV_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

// ---------------------------------------------------------------- SpMV, uniform-width SELL-32

// Every 32-row slice padded to the same width W (taken where that costs
// <= 10%: the FSAI factors G, 9 entries on every row): entry k of row i sits
// at (i/32)*32W + 32k + i%32, so a lane's addresses follow from its row alone.
// All W value / column loads are issued at once (padding slots hold value 0
// and column = row, and are never summed), the x gathers in the next step --
// two dependent memory steps per row instead of slice offset -> length ->
// values -> gathers.  Sum over the lane's own len in the reference order.
struct SellUArgs {
    const double *val;
    const int32_t *col;
    const uint8_t *len;
    int W;
    // PLEN layouts: the rows of each 32-row slice sit in its lanes sorted by length (descending,
    // stable), perm[slot] = the row's position inside the slice.  The live lanes of a slot are then
    // a prefix, so skipping the padding skips whole sectors (unsorted, slot 2 of an interpolation
    // operator has ~40% of its lanes live but touches ~87% of its sectors); the warp still works
    // on the same 32 neighbouring rows and the y store stays one 256-byte segment.  nullptr: slot = row.
    const uint8_t *perm;
    // VD kernels: rows whose VALUE tuples fall into <= 255 classes (the interpolation of a
    // constant-coefficient problem: config 4's P_0 holds 8 distinct weights in 30 M entries) store one
    // class id per slot; the table {length, values} sits in shared memory, so a row streams its
    // columns (4 B per entry) and one byte -- no values, no length.
    const uint8_t *cls;
    const double *vtab;   // [ncls][FL]
    const int32_t *vlen;  // [ncls]
    int ncls;
    // VD == 2: too many value TUPLES but <= 256 distinct VALUES (config 4's P^T_0: 5-entry rows of
    // the same 8 weights): one value id per stored entry (1 B instead of 8, same slot layout as col),
    // the value table (vtab[0 .. ncls)) in shared memory; lengths come from `len` as usual.
    const uint8_t *vid;
};

// Software-pipelined: the next row's columns and length are loaded one
// iteration ahead, so a row's W value loads and its x gathers leave together
// (one dependent memory step per row instead of length -> values/columns ->
// gathers).
// PLEN: slots at or beyond the row's length are not loaded (no bytes for padding): short ragged
// rows (interpolation P, 1..8 entries) pad their slices freely.
template <int EPI, int FL, bool PLEN, int VD = 0>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, FL <= 4 ? 6 : FL <= 9 ? 4 : 3) spmv_sellu(const SpmvArgs a,
                                                                                           const SellUArgs u, int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    extern __shared__ double sellu_vd[];  // VD: value table [ncls][FL], then lengths [ncls]
    const double *svt = sellu_vd;
    const int32_t *svl = reinterpret_cast<const int32_t *>(sellu_vd + (VD == 1 ? u.ncls * FL : 0));
    if constexpr (VD == 1) {  // static data: staged before the PDL wait
        double *wv_ = sellu_vd;
        int32_t *wl_ = reinterpret_cast<int32_t *>(sellu_vd + u.ncls * FL);
        for (int i = threadIdx.x; i < u.ncls * FL; i += blockDim.x) wv_[i] = u.vtab[i];
        for (int i = threadIdx.x; i < u.ncls; i += blockDim.x) wl_[i] = u.vlen[i];
        __syncthreads();
    }
    if constexpr (VD == 2) {
        double *wv_ = sellu_vd;
        for (int i = threadIdx.x; i < u.ncls; i += blockDim.x) wv_[i] = u.vtab[i];
        __syncthreads();
    }
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int nthreads = gridDim.x * VEC_SPMV_THREADS;
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    const int W32 = 32 * u.W;
    double dacc = 0.0;
    int v = blockIdx.x * VEC_SPMV_THREADS + threadIdx.x;
    int c[FL];
    int len = 0, nrowid = 0, ncls_ = 0;
    auto fetch = [&](int r) {  // r: slot
        const int base = (r >> 5) * W32 + (r & 31);
        if constexpr (VD == 1) {
            ncls_ = __ldg(u.cls + r);
            len = svl[ncls_];
        } else {
            len = __ldg(u.len + r);
        }
        nrowid = (PLEN && u.perm) ? ((r & ~31) | (int)__ldg(u.perm + r)) : r;
#pragma unroll
        for (int k = 0; k < FL; ++k) c[k] = (k < (PLEN ? len : u.W)) ? __ldg(u.col + base + 32 * k) : 0;
    };
    if (v < nrows) fetch(vrow(a, v));
    for (; v < nrows; v += nthreads) {
        const int slot = vrow(a, v);
        const int row = nrowid;
        const int base = (slot >> 5) * W32 + (slot & 31);
        double p[FL];
        if constexpr (VD == 1) {
            const double *tv = svt + ncls_ * FL;
#pragma unroll
            for (int k = 0; k < FL; ++k) p[k] = (k < len) ? prod(tv[k], __ldg(x + c[k])) : 0.0;
        } else if constexpr (VD == 2) {
            int vi[FL];
#pragma unroll
            for (int k = 0; k < FL; ++k) vi[k] = (k < (PLEN ? len : u.W)) ? (int)__ldg(u.vid + base + 32 * k) : 0;
#pragma unroll
            for (int k = 0; k < FL; ++k) p[k] = (k < (PLEN ? len : u.W)) ? prod(svt[vi[k]], __ldg(x + c[k])) : 0.0;
        } else {
#pragma unroll
            for (int k = 0; k < FL; ++k)
                p[k] = (k < (PLEN ? len : u.W)) ? prod(__ldg(u.val + base + 32 * k), __ldg(x + c[k])) : 0.0;
        }
        const int clen = len;
        if (v + nthreads < nrows) fetch(vrow(a, v + nthreads));
        double bv = 0.0, wv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
        if (want_dot && !self_dot) wv = a.dotw[row];
        const double sum = ref_sum_fixed<FL>(p, clen);
        double yv;
        if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
        else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
        else yv = sum;
        a.y[row] = yv;
        if (want_dot) dacc = fma(yv, self_dot ? yv : wv, dacc);
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v2 = block_sum<VEC_SPMV_THREADS>(dacc, red);
        spmv_finalize<VEC_SPMV_THREADS>(v2, a);
    }
}

// ---------------------------------------------------------------- SpMV, sorted SELL-32 (SELL-C-sigma)

// Rows sorted by length (descending) inside windows of sigma rows, then cut
// into 32-row slices padded to their widest row: slice s holds W_s entries
// per lane, entry k of slot l at sbeg[s] + 32k + l, original row perm[32s+l].
// Slices of width <= 16 (most slices of the FSAI transposes) issue every
// value / column load at once, predicated on the warp-uniform W_s rather
// than on each row's length, then sum each row over its own length in the
// reference order; wider slices take the round-by-round path.  The slice
// metadata (offset, width) and the slot's row / length are fetched one slice
// ahead.
struct SellSArgs {
    const double *val;
    const int32_t *col;
    const int32_t *sbeg;   // per slice start
    const uint8_t *swid;   // per slice width
    const int32_t *perm;   // slot -> row
    const uint8_t *slen;   // per slot row length
    int nslots;            // rows of the matrix (slots beyond are empty)
};

template <int EPI, bool PLEN>
__global__ void __launch_bounds__(VEC_SPMV_THREADS, 4) spmv_sells(const SpmvArgs a, const SellSArgs q, int nrows)
{
    __shared__ double red[VEC_SPMV_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const int lane = threadIdx.x & 31;
    const int nslices = (nrows + 31) >> 5;  // virtual slices (row-range launches: whole windows)
    const int wstride = gridDim.x * (VEC_SPMV_THREADS / 32);
    const bool want_dot = a.dotw != nullptr;
    const bool self_dot = a.dotw == a.y;
    const double *__restrict__ x = a.x;
    double dacc = 0.0;
    int sl = blockIdx.x * (VEC_SPMV_THREADS / 32) + (threadIdx.x >> 5);
    int nsb = 0, nw = 0, nrow = -1, nlen = 0;
    auto meta = [&](int vs) {
        const int s = vrow(a, vs * 32) >> 5;
        nsb = __ldg(q.sbeg + s);
        nw = __ldg(q.swid + s);
        const int pos = s * 32 + lane;
        AMG_CHECK(s >= 0 && s * 32 < q.nslots);
        nrow = pos < q.nslots ? __ldg(q.perm + pos) : -1;
        nlen = pos < q.nslots ? __ldg(q.slen + pos) : 0;
    };
    if (sl < nslices) meta(sl);
    for (; sl < nslices; sl += wstride) {
        const int sb = nsb, W = nw, row = nrow, len = nlen;
        if (sl + wstride < nslices) meta(sl + wstride);
        const double *vb = q.val + sb + lane;
        const int32_t *cb = q.col + sb + lane;
        double sum;
        if (W <= 16) {
            double p[16];
#pragma unroll
            for (int k = 0; k < 16; ++k)  // PLEN: padding slots are not loaded (no bytes for padding)
                p[k] = (k < (PLEN ? len : W)) ? prod(__ldg(vb + 32 * k), __ldg(x + __ldg(cb + 32 * k))) : 0.0;
            sum = ref_sum_fixed<16>(p, len);
        } else {
            auto P = [&](int k) -> double { return prod(__ldg(vb + 32 * k), __ldg(x + __ldg(cb + 32 * k))); };
            sum = ref_row_sum<false>(P, len);
        }
        if (row >= 0) {
            double bv = 0.0;
            if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD) bv = a.b[row];
            double yv;
            if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sum);
            else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(a.omega, sum));
            else if constexpr (EPI == EPI_ADD) yv = add(bv, sum);
            else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(a.omega, sum);
            else yv = sum;
            a.y[row] = yv;
            if (want_dot) dacc = fma(yv, self_dot ? yv : a.dotw[row], dacc);
        }
    }
    if (want_dot || a.fin != FIN_NONE) {
        double v = block_sum<VEC_SPMV_THREADS>(dacc, red);
        spmv_finalize<VEC_SPMV_THREADS>(v, a);
    }
}

// ---------------------------------------------------------------- L2 prefetch of the coarse levels

// Launched on a side stream while the level above the cluster tail runs: pulls
// the tail's matrices (evicted by the fine-level sweeps) into L2, so the tail
// -- 16 SMs, latency-bound -- finds them there.  ranges: (ptr, bytes) pairs.
struct PrefetchRange {
    const char *p;
    long long bytes;
};

__global__ void __launch_bounds__(256) l2_prefetch(const PrefetchRange *__restrict__ r, int nr)
{
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nt = (long long)gridDim.x * blockDim.x;
    for (int k = 0; k < nr; ++k) {
        const PrefetchRange q = r[k];
        for (long long off = t * 128; off < q.bytes; off += nt * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(q.p + off));
    }
}

// ---------------------------------------------------------------- vectors

constexpr int VEC_THREADS = 256;

struct VecArgs {
    int64_t n;
    double *x;        // output / in-out
    double *r;        // second in-out (pcg_update)
    const double *p;  // inputs
    const double *q;
    const double *d;
    double omega;
    int mode;
    double *partials;
    unsigned *ticket;
    int fin;
    PcgCtl *ctl;
    const int *gate1;
    const int *gate2;
};

// x += alpha p ; r -= alpha q ; partial r.r      (krylov.py:73-75, 78)
__global__ void __launch_bounds__(VEC_THREADS) pcg_update(const VecArgs a)
{
    __shared__ double red[VEC_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const double alpha = a.ctl->alpha;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        a.x[i] = add(a.x[i], __dmul_rn(alpha, a.p[i]));
        double rv = __dsub_rn(a.r[i], __dmul_rn(alpha, a.q[i]));
        a.r[i] = rv;
        acc = fma(rv, rv, acc);
    }
    double v = block_sum<VEC_THREADS>(acc, red);
    grid_finalize<VEC_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
}

// p = z + beta p                                   (krylov.py:91)
__global__ void __launch_bounds__(VEC_THREADS) pcg_xpay(const VecArgs a)
{
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    const double beta = a.ctl->beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
        a.x[i] = add(a.p[i], __dmul_rn(beta, a.x[i]));
}

// mode 0: sum p.q ; finalize
__global__ void __launch_bounds__(VEC_THREADS) vec_dot(const VecArgs a)
{
    __shared__ double red[VEC_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
        acc = fma(a.p[i], a.q[i], acc);
    double v = block_sum<VEC_THREADS>(acc, red);
    grid_finalize<VEC_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
}

// Jacobi sweep (smoothers.py:47-49, 172): mode 0: x = w*(d*r) ; mode 1: x += w*(d*r)
// optional dot partial x.q
__global__ void __launch_bounds__(VEC_THREADS) jacobi_sweep(const VecArgs a)
{
    __shared__ double red[VEC_THREADS / 32];
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        double z = __dmul_rn(a.omega, __dmul_rn(a.d[i], a.p[i]));
        double xv = a.mode ? add(a.x[i], z) : z;
        a.x[i] = xv;
        if (a.q) acc = fma(xv, a.q[i], acc);
    }
    if (a.fin != FIN_NONE) {
        double v = block_sum<VEC_THREADS>(acc, red);
        grid_finalize<VEC_THREADS>(v, a.partials, a.ticket, a.fin, a.ctl);
    }
}

__global__ void __launch_bounds__(VEC_THREADS) vec_copy(const VecArgs a)
{
    pdl_launch();
    pdl_wait();
    if (!gate_open(a.gate1, a.gate2)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
        a.x[i] = a.p ? a.p[i] : 0.0;
}

// Multi-GPU: sum the all-gathered per-rank partials in rank order (the same
// on every rank, so every rank takes the same control-flow decisions).
__global__ void fin_ranks(PcgCtl *c, int fin, int nranks, const int *gate1)
{
    pdl_launch();
    pdl_wait();
    if (!gate_open(gate1, nullptr)) return;
    double v = 0.0;
    for (int r = 0; r < nranks; ++r) v += c->part_all[r];
    apply_fin(fin, v, c);
}

// Halo pack: buf[i] = x[idx[i]] (owned entries a peer needs).
__global__ void __launch_bounds__(VEC_THREADS) halo_pack(const double *x, const int32_t *idx, double *buf, int64_t n)
{
    pdl_launch();
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = x[idx[i]];
}

// BiCGstab vector updates (krylov.py:146-172), numpy's operation order:
// mode 0: p = r + beta * (p - omega * v)      x=p, p=r, q=v
// mode 1: s = r - alpha * v                   x=s, p=r, q=v
// mode 2: x = x + (alpha * phat + omega * shat)  x=x, p=phat, q=shat
// mode 3: r = s - omega * t                   x=r, p=s, q=t
// mode 4: x = x + alpha * phat                x=x, p=phat
struct BicgArgs {
    int64_t n;
    double *x;
    const double *p;
    const double *q;
    double alpha, beta, omega;
    int mode;
};

__global__ void __launch_bounds__(VEC_THREADS) bicg_update(const BicgArgs a)
{
    pdl_launch();
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        switch (a.mode) {
        case 0: a.x[i] = add(a.p[i], __dmul_rn(a.beta, __dsub_rn(a.x[i], __dmul_rn(a.omega, a.q[i])))); break;
        case 1: a.x[i] = __dsub_rn(a.p[i], __dmul_rn(a.alpha, a.q[i])); break;
        case 2: a.x[i] = add(a.x[i], add(__dmul_rn(a.alpha, a.p[i]), __dmul_rn(a.omega, a.q[i]))); break;
        case 3: a.x[i] = __dsub_rn(a.p[i], __dmul_rn(a.omega, a.q[i])); break;
        default: a.x[i] = add(a.x[i], __dmul_rn(a.alpha, a.p[i])); break;
        }
    }
}

// Loop continuation for the device while-loop graph.
__global__ void pcg_continue(PcgCtl *c, cudaGraphConditionalHandle handle, int use_handle)
{
    pdl_launch();
    pdl_wait();
    if (c->active && c->it >= c->max_iters) c->active = 0;
    if (use_handle) cudaGraphSetConditional(handle, c->active ? 1u : 0u);
}

// ---------------------------------------------------------------- coarse solve

// Cholesky: solve L y = b, then L^T z = y (dpotrs with uplo = 'L').
// L: packed lower triangle, row-major: row i holds L[i][0..i] at i(i+1)/2;
// dinv[i] = 1 / L[i][i] (OpenBLAS' trsm packs inverted diagonals too).
// One CTA, blocked by 32: warp 0 solves each 32x32 diagonal triangle with
// shuffles, then all warps apply the block to the remaining rows.  `v` (the
// right-hand side on entry, the solution on exit) lives in shared memory.
constexpr int COARSE_THREADS = 256;

__device__ __forceinline__ int64_t tri(int i) { return (int64_t)i * (i + 1) / 2; }

// Blocked forward / back substitution with the lower Cholesky factor.
// Diagonal 32x32 blocks are solved by warp 0 with the pre-scaled blocks
// Ms[r][c] = L[r][c] / L[c][c] (forward) and Ns[c][r] = L[c][r] / L[c][c]
// (backward, L^T), packed lower triangles computed at upload: one step of the
// substitution chain is then shuffle -> FMA, and the division by the
// diagonal is applied to the whole block at the end.  Rows below / above the
// block are updated as GEMVs (forward: one warp per row, conflict-free row
// segments; backward: along rows of L).
__device__ void chol_solve_cta(int n, const double *__restrict__ L, const double *__restrict__ dinv,
                               const double *__restrict__ MN, double *v)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int nblk = (n + 31) / 32;
    for (int bi = 0; bi < nblk; ++bi) {  // forward: L y = b
        const int jb = bi * 32, nb = min(32, n - jb);
        if (warp == 0 && MN == nullptr) {  // unscaled chain: vc = v_c / L_cc, then vi -= L_ic vc
            double vi = lane < nb ? v[jb + lane] : 0.0;
            const double di = lane < nb ? dinv[jb + lane] : 0.0;
            const double *Lr = L + tri(jb + lane) + jb;
            for (int c = 0; c < nb; ++c) {
                const double vc = __shfl_sync(0xffffffffu, vi * di, c);
                if (lane == c) vi = vc;
                if (lane > c && lane < nb) vi -= Lr[c] * vc;
            }
            if (lane < nb) v[jb + lane] = vi;
        } else if (warp == 0) {
            const double *Mr = MN + (size_t)bi * 1056 + lane * (lane + 1) / 2;  // row `lane` of Ms
            double vi = lane < nb ? v[jb + lane] : 0.0;
            if (nb == 32) {
#pragma unroll
                for (int c = 0; c < 31; ++c) {
                    const double vc = __shfl_sync(0xffffffffu, vi, c);
                    if (lane > c) vi = fma(-Mr[c], vc, vi);
                }
            } else {
                for (int c = 0; c + 1 < nb; ++c) {
                    const double vc = __shfl_sync(0xffffffffu, vi, c);
                    if (lane > c && lane < nb) vi = fma(-Mr[c], vc, vi);
                }
            }
            if (lane < nb) v[jb + lane] = vi * dinv[jb + lane];
        }
        __syncthreads();
        const double vb = lane < nb ? v[jb + lane] : 0.0;
        for (int i = jb + nb + warp; i < n; i += nwarps) {  // one warp per row: lanes read L[i][jb + lane]
            double t = lane < nb ? L[tri(i) + jb + lane] * vb : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) v[i] -= t;
        }
        __syncthreads();
    }
    for (int bi = nblk - 1; bi >= 0; --bi) {  // backward: L^T z = y
        const int jb = bi * 32, nb = min(32, n - jb);
        if (warp == 0 && MN == nullptr) {
            double vi = lane < nb ? v[jb + lane] : 0.0;
            const double di = lane < nb ? dinv[jb + lane] : 0.0;
            for (int c = nb - 1; c >= 0; --c) {
                const double zc = __shfl_sync(0xffffffffu, vi * di, c);
                if (lane == c) vi = zc;
                if (lane < c) vi -= L[tri(jb + c) + jb + lane] * zc;  // L^T[lane][c] = L[c][lane]
            }
            if (lane < nb) v[jb + lane] = vi;
        } else if (warp == 0) {
            const double *N = MN + (size_t)bi * 1056 + 528;
            double vi = lane < nb ? v[jb + lane] : 0.0;
            if (nb == 32) {
#pragma unroll
                for (int c = 31; c > 0; --c) {
                    const double vc = __shfl_sync(0xffffffffu, vi, c);
                    if (lane < c) vi = fma(-N[c * (c + 1) / 2 + lane], vc, vi);
                }
            } else {
                for (int c = nb - 1; c > 0; --c) {
                    const double vc = __shfl_sync(0xffffffffu, vi, c);
                    if (lane < c) vi = fma(-N[c * (c + 1) / 2 + lane], vc, vi);
                }
            }
            if (lane < nb) v[jb + lane] = vi * dinv[jb + lane];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < jb; i += blockDim.x) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (nb == 32) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    a0 = fma(L[tri(jb + c) + i], v[jb + c], a0);
                    a1 = fma(L[tri(jb + c + 1) + i], v[jb + c + 1], a1);
                    a2 = fma(L[tri(jb + c + 2) + i], v[jb + c + 2], a2);
                    a3 = fma(L[tri(jb + c + 3) + i], v[jb + c + 3], a3);
                }
            } else {
                for (int c = 0; c < nb; ++c) a0 = fma(L[tri(jb + c) + i], v[jb + c], a0);
            }
            v[i] -= (a0 + a1) + (a2 + a3);
        }
        __syncthreads();
    }
}

// Pipelined variant (n <= 32 * warps, <= 16 blocks): warp w owns rows
// [32w, 32w + 32).  Forward: it folds in the solved chunks 0..w-1 as each one
// is published (smem flag), then runs its own 32-step chain and publishes;
// backward mirrors it from the last chunk down.  The critical path is the
// chain of diagonal blocks alone (no CTA-wide barrier and GEMV between
// blocks): n = 188 takes ~1/3 of the blocked schedule.  Same arithmetic per
// entry (different association of the updates, as dtrsm's blocking differs
// from both).  `v` holds b on entry and z on exit; ends with __syncthreads.
__device__ __noinline__ void chol_solve_pipe(int n, const double *__restrict__ L, const double *__restrict__ dinv, double *v,
                                int nap = 0)
{
    __shared__ int s_done[2][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (n + 31) / 32;
    if (threadIdx.x < 32) {
        s_done[0][lane & 15] = 0;
        s_done[1][lane & 15] = 0;
    }
    __syncthreads();
    if (warp < nblk) {
        volatile int *fdone = s_done[0], *bdone = s_done[1];
        const int jb = warp * 32, nb = min(32, n - jb);
        const int i = jb + lane;
        const bool live = lane < nb;
        const double di = live ? dinv[i] : 0.0;
        const double *Li = L + tri(live ? i : jb);
        // the own diagonal block's row segment (forward) and column segment (backward) in
        // registers before any wait: the chains then run shuffle -> FMA only
        double Lr[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) Lr[c] = (c < lane && live) ? Li[jb + c] : 0.0;
        // forward: L y = b
        double vi = live ? v[i] : 0.0;
        for (int cb = 0; cb < warp; ++cb) {
            while (fdone[cb] == 0)
                if (nap) __nanosleep(nap);
            __syncwarp();
            const int c0 = cb * 32;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                a0 = fma(Li[c0 + c], v[c0 + c], a0);
                a1 = fma(Li[c0 + c + 1], v[c0 + c + 1], a1);
                a2 = fma(Li[c0 + c + 2], v[c0 + c + 2], a2);
                a3 = fma(Li[c0 + c + 3], v[c0 + c + 3], a3);
            }
            if (live) vi -= (a0 + a1) + (a2 + a3);
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {  // lanes >= nb are inert: no live lane reads them
            const double vc = __shfl_sync(0xffffffffu, vi * di, c);
            vi = (lane == c) ? vc : vi;
            vi = (lane > c) ? fma(-Lr[c], vc, vi) : vi;
        }
        if (live) v[i] = vi;
        __syncwarp();
        __threadfence_block();
        if (lane == 0) fdone[warp] = 1;
        double Lc[32];  // L^T[i][jb + c] = L[jb + c][i], loaded before the backward waits
#pragma unroll
        for (int c = 0; c < 32; ++c) Lc[c] = (c > lane && c < nb) ? L[tri(jb + c) + i] : 0.0;
        // backward: L^T z = y
        for (int cb = nblk - 1; cb > warp; --cb) {
            while (bdone[cb] == 0)
                if (nap) __nanosleep(nap);
            __syncwarp();
            const int c0 = cb * 32, cn = min(32, n - c0);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (cn == 32) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    a0 = fma(L[tri(c0 + c) + i], v[c0 + c], a0);
                    a1 = fma(L[tri(c0 + c + 1) + i], v[c0 + c + 1], a1);
                    a2 = fma(L[tri(c0 + c + 2) + i], v[c0 + c + 2], a2);
                    a3 = fma(L[tri(c0 + c + 3) + i], v[c0 + c + 3], a3);
                }
            } else {
                for (int c = 0; c < cn; ++c) a0 = fma(L[tri(c0 + c) + i], v[c0 + c], a0);
            }
            if (live) vi -= (a0 + a1) + (a2 + a3);
        }
#pragma unroll
        for (int c = 31; c >= 0; --c) {
            const double zc = __shfl_sync(0xffffffffu, vi * di, c);
            vi = (lane == c) ? zc : vi;
            vi = (lane < c) ? fma(-Lc[c], zc, vi) : vi;
        }
        if (live) v[i] = vi;
        __syncwarp();
        __threadfence_block();
        if (lane == 0) bdone[warp] = 1;
    }
    __syncthreads();
}

// LU (getrs, no transpose): b <- P b ; L (unit) y = b ; U z = y.  LU full n x n row-major.
__device__ void lu_solve_cta(int n, const double *__restrict__ LU, const int32_t *__restrict__ piv, double *v)
{
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            int p = piv[i];
            if (p != i) { double t = v[i]; v[i] = v[p]; v[p] = t; }
        }
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        const double yj = v[j];
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) v[i] -= LU[(int64_t)i * n + j] * yj;
        __syncthreads();
    }
    for (int j = n - 1; j >= 0; --j) {
        const double zj = v[j] / LU[(int64_t)j * n + j];
        __syncthreads();
        if (threadIdx.x == 0) v[j] = zj;
        for (int i = threadIdx.x; i < j; i += blockDim.x) v[i] -= LU[(int64_t)i * n + j] * zj;
        __syncthreads();
    }
}

struct CoarseArgs {
    int n;
    int kind;    // 0 cholesky, 1 lu
    int staged;  // packed factor + block inverses copied to shared memory
    const double *Lp;
    const double *mn;    // per diagonal block: Ms then Ns (2 x 528 doubles, packed lower)
    const double *dinv;
    const double *LU;
    const int32_t *piv;
    int prefetch;  // tail kernel: L2-prefetch the streamed matrices before waiting on the predecessor
    int pipe;      // Cholesky: pipelined per-warp substitution (chol_solve_pipe)
};

__global__ void __launch_bounds__(COARSE_THREADS) coarse_solve_k(const CoarseArgs c, const double *y, double *z,
                                                                  const int *gate1, double *partials,
                                                                  unsigned *ticket, int fin, PcgCtl *ctl,
                                                                  const double *dotw)
{
    extern __shared__ __align__(16) double sh[];
    __shared__ double red[COARSE_THREADS / 32];
    const int n = c.n;
    double *v = sh;
    double *tmp = sh + ((n + 1) & ~1);
    const double *L = c.Lp, *D = c.dinv, *MN = c.mn;
    if (c.kind == 0 && c.staged) {  // the factor is static: stage it before waiting on the producer
        double *Ds = tmp + 32;
        for (int i = threadIdx.x; i < n; i += blockDim.x) Ds[i] = c.dinv[i];
        double *MNs = Ds + ((n + 1) & ~1);
        const int nmn = ((n + 31) / 32) * 1056;
        for (int i = threadIdx.x; i < nmn; i += blockDim.x) MNs[i] = __ldg(c.mn + i);
        double *Ls = MNs + nmn;
        const int64_t np = tri(n);
#pragma unroll 8
        for (int64_t i = threadIdx.x; i < np; i += blockDim.x) Ls[i] = __ldg(c.Lp + i);
        L = Ls;
        D = Ds;
        MN = MNs;
    }
    pdl_launch();
    pdl_wait();
    if (!gate_open(gate1, nullptr)) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = y[i];
    __syncthreads();
    if (c.kind == 0 && c.pipe && n <= 32 * (int)(blockDim.x / 32) && n <= 512) chol_solve_pipe(n, L, D, v, c.pipe > 1 ? c.pipe : 0);
    else if (c.kind == 0) chol_solve_cta(n, L, D, MN, v);
    else lu_solve_cta(n, c.LU, c.piv, v);
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        z[i] = v[i];
        if (dotw) acc = fma(v[i], dotw[i], acc);
    }
    if (fin != FIN_NONE) {
        double s = block_sum<COARSE_THREADS>(acc, red);
        grid_finalize<COARSE_THREADS>(s, partials, ticket, fin, ctl);
    }
}

// ---------------------------------------------------------------- cluster tail

// The V-cycle below a size threshold runs as ONE kernel on one thread-block
// cluster: the operations of those levels (same sequence, same epilogues,
// same reference summation order as the per-op kernels) are executed in
// order with a cluster barrier between dependent operations, replacing
// kernel launches (~ microseconds each) by barriers (~0.2 us).  Every
// matrix block a CTA owns (rows balanced by stored entries) is staged in its
// shared memory once at kernel start -- before griddepcontrol.wait, so it
// overlaps the predecessor -- leaving one x-gather round trip per op.
enum TailKind { TAIL_SPMV = 0, TAIL_JACOBI = 1, TAIL_COARSE = 2 };

struct TailOp {
    int kind;
    int epi;
    int nrows;
    int mode;  // jacobi: 0 set, 1 accumulate
    int mat;   // SpMV: index into the staged-matrix table
    int xs, ys, bs;  // distributed-shared-memory slots of x / y / b (-1: global memory)
    const double *x;
    double *y;
    const double *b;
    const double *d;
    double omega;
};

// Level vectors of the tail held in distributed shared memory (option
// tail_dsm): element i of slot s lives in CTA i >> shift at byte offset
// off + 8 (i & (2^shift - 1)) of the cluster's shared windows; gathers are
// ld.shared::cluster (no L2 round trip), ordered by the cluster barriers.
constexpr int TAIL_MAX_VECS = 48;
struct TailVecs {
    const int2 *slot;  // {shift, byte offset} per slot
    int nslots;
    int pcap;          // product-buffer capacity (entries): streamed SpMVs run their rows in chunks
};

__device__ __forceinline__ double tv_ld(const double *g, int s, int i, const int2 *sv, const char *smem)
{
    if (s < 0) return __ldcg(g + i);
    const int2 d = sv[s];
    AMG_CHECK((unsigned)(i >> d.x) < 16u);
    const unsigned la = smem_u32(smem + d.y) + ((unsigned)(i & ((1 << d.x) - 1)) << 3);
    unsigned ra;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"((unsigned)(i >> d.x)));
    double v;
    asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
    return v;
}

__device__ __forceinline__ void tv_st(double *g, int s, int i, double v, const int2 *sv, const char *smem)
{
    if (s < 0) {
        g[i] = v;
        return;
    }
    const int2 d = sv[s];
    const unsigned la = smem_u32(smem + d.y) + ((unsigned)(i & ((1 << d.x) - 1)) << 3);
    unsigned ra;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"((unsigned)(i >> d.x)));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// A distinct matrix of the tail and where each CTA's block of it lives.
struct TailMat {
    const int32_t *off;
    const int32_t *col;
    const double *val;
    int split;     // (cluster + 1) row splits in the split table
    int staged;    // 1: block staged in smem at kernel start; 0: streamed from L2 per op
    int smem_off;  // byte offset of this matrix's region in every CTA's smem
    int rows_cap;  // region capacity: rows (offsets: rows_cap + 1 entries)
    int nnz_cap;   // region capacity: entries
};

__host__ __device__ inline int tail_region_bytes(int rows_cap, int nnz_cap)
{
    const int ob = ((rows_cap + 1) * 4 + 15) & ~15;
    const int cb = (nnz_cap * 4 + 15) & ~15;
    return ob + cb + nnz_cap * 8;
}

#ifndef AMG_TAIL_THREADS
#define AMG_TAIL_THREADS 512
#endif
constexpr int TAIL_THREADS = AMG_TAIL_THREADS;
constexpr int TAIL_MAX_OPS = 96;    // ops per tail (8 per level + coarse): up to 11 levels
constexpr int TAIL_MAX_MATS = 64;
constexpr int TAIL_MAX_DINV = 512;

__device__ __forceinline__ void cluster_barrier()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Grid-wide barrier of a cooperative (co-resident) tail grid: arrival count +
// generation word, release by the last CTA, acquire spin by the others.
__device__ __forceinline__ void grid_sync(unsigned *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        __threadfence();
        const unsigned a = atomicAdd(bar, 1u);
        if (a == gridDim.x - 1) {
            bar[0] = 0u;  // nobody arrives again before the generation flips
            __threadfence();
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
        } else {
            unsigned c;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(c) : "l"(bar + 1) : "memory");
            } while (c == g);
        }
        __threadfence();
    }
    __syncthreads();
}

// tail synchronisation: one cluster (barrier.cluster) or a cooperative grid (gbar)
__device__ __forceinline__ void tail_sync(unsigned *gbar)
{
    if (gbar) grid_sync(gbar);
    else cluster_barrier();
}

__device__ __forceinline__ unsigned cluster_rank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Streamed variant: the block's values / columns / offsets are read from
// global memory (L2) in the op itself (matrices that did not fit the smem
// budget); same phases and order as the staged variant.
template <int EPI>
__device__ __forceinline__ void tail_spmv_streamed_chunk(const TailOp &o, const TailMat &M, int r0, int r1, double *ps,
                                                         const int2 *tvs, const char *smem);

// rows [r0, r1) in chunks whose products fit the buffer (pcap entries)
template <int EPI>
__device__ __forceinline__ void tail_spmv_streamed(const TailOp &o, const TailMat &M, int r0, int r1, double *ps,
                                                   const int2 *tvs, const char *smem, int pcap)
{
    __shared__ int s_re;
    int rs = r0;
    while (rs < r1) {
        if (threadIdx.x == 0) {
            const int base = __ldg(M.off + rs);
            int lo = rs + 1, hi = r1;  // largest re in [rs + 1, r1] with off[re] - off[rs] <= pcap
            if (__ldg(M.off + hi) - base <= pcap) lo = hi;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (__ldg(M.off + mid) - base <= pcap) lo = mid;
                else hi = mid - 1;
            }
            s_re = lo;
        }
        __syncthreads();
        const int re = s_re;
        AMG_CHECK(re > rs && __ldg(M.off + re) - __ldg(M.off + rs) <= pcap);  // whole rows within the buffer
        tail_spmv_streamed_chunk<EPI>(o, M, rs, re, ps, tvs, smem);
        __syncthreads();
        rs = re;
    }
}

template <int EPI>
__device__ __forceinline__ void tail_spmv_streamed_chunk(const TailOp &o, const TailMat &M, int r0, int r1, double *ps,
                                                         const int2 *tvs, const char *smem)
{
    const int k0 = __ldg(M.off + r0);
    const int nk = __ldg(M.off + r1) - k0;
    AMG_CHECK(r0 <= r1);
    double bpre = 0.0;
    if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD)
        if (r0 + (int)threadIdx.x < r1) bpre = tv_ld(o.b, o.bs, r0 + threadIdx.x, tvs, smem);
    int lo = 0, hi = 0;
    if (r0 + (int)threadIdx.x < r1) {
        lo = __ldg(M.off + r0 + threadIdx.x) - k0;
        hi = __ldg(M.off + r0 + threadIdx.x + 1) - k0;
    }
#pragma unroll 8
    for (int k = threadIdx.x; k < nk; k += TAIL_THREADS)
        ps[k] = prod(__ldg(M.val + k0 + k), tv_ld(o.x, o.xs, __ldg(M.col + k0 + k), tvs, smem));
    __syncthreads();
    for (int rr = threadIdx.x; rr < r1 - r0; rr += TAIL_THREADS) {
        if (rr != (int)threadIdx.x) {
            lo = __ldg(M.off + r0 + rr) - k0;
            hi = __ldg(M.off + r0 + rr + 1) - k0;
        }
        const double sv = row_sum_staged<1>(ps, 0, lo, hi, 0, 0u);
        const int row = r0 + rr;
        double bv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD)
            bv = (rr == (int)threadIdx.x) ? bpre : tv_ld(o.b, o.bs, row, tvs, smem);
        double yv;
        if constexpr (EPI == EPI_PLAIN) yv = sv;
        else if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, sv);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(o.omega, sv));
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(o.omega, sv);
        else yv = add(bv, sv);
        tv_st(o.y, o.ys, row, yv, tvs, smem);
    }
}

template <int EPI>
__device__ __forceinline__ void tail_spmv(const TailOp &o, int r0, int r1, const int32_t *os, const int32_t *cs,
                                          const double *vs, double *ps, const int2 *tvs, const char *smem)
{
    if (r1 <= r0) return;  // no rows on this CTA (CTA 0 runs the coarsest solve; its smem holds the factor)
    const int nk = os[r1 - r0];
    // prefetch the epilogue operand of this thread's first row with the gathers
    double bpre = 0.0;
    if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD)
        if (r0 + (int)threadIdx.x < r1) bpre = tv_ld(o.b, o.bs, r0 + threadIdx.x, tvs, smem);
#pragma unroll 8
    for (int k = threadIdx.x; k < nk; k += TAIL_THREADS) ps[k] = prod(vs[k], tv_ld(o.x, o.xs, cs[k], tvs, smem));
    __syncthreads();
    for (int rr = threadIdx.x; rr < r1 - r0; rr += TAIL_THREADS) {
        const double s = row_sum_staged<1>(ps, 0, os[rr], os[rr + 1], 0, 0u);
        const int row = r0 + rr;
        double bv = 0.0;
        if constexpr (EPI == EPI_RESID || EPI == EPI_AXPYW || EPI == EPI_ADD)
            bv = (rr == (int)threadIdx.x) ? bpre : tv_ld(o.b, o.bs, row, tvs, smem);
        double yv;
        if constexpr (EPI == EPI_PLAIN) yv = s;
        else if constexpr (EPI == EPI_RESID) yv = __dsub_rn(bv, s);
        else if constexpr (EPI == EPI_AXPYW) yv = add(bv, __dmul_rn(o.omega, s));
        else if constexpr (EPI == EPI_SETW) yv = __dmul_rn(o.omega, s);
        else yv = add(bv, s);
        tv_st(o.y, o.ys, row, yv, tvs, smem);
    }
}

__global__ void __launch_bounds__(TAIL_THREADS) tail_vcycle(const TailOp *__restrict__ ops, int nops,
                                                             const TailMat *__restrict__ mats, int nmats,
                                                             const int32_t *__restrict__ splits, int prod_off,
                                                             const CoarseArgs c, const int *gate1,
                                                             unsigned long long *trace, const TailVecs tvv,
                                                             unsigned *gbar)
{
    __shared__ int2 s_vec[TAIL_MAX_VECS];
    for (int i = threadIdx.x; i < tvv.nslots; i += blockDim.x) s_vec[i] = tvv.slot[i];
    extern __shared__ __align__(16) double sh[];
    __shared__ TailOp s_ops[TAIL_MAX_OPS];
    __shared__ int s_split[TAIL_MAX_MATS][2];
    __shared__ int s_geo[TAIL_MAX_MATS][3];
    char *smem = reinterpret_cast<char *>(sh);
    double *ps = reinterpret_cast<double *>(smem + prod_off);  // product buffer
    const unsigned rank = gbar ? blockIdx.x : cluster_rank();
    // ---- stage static data (before waiting on the predecessor)
    const double *L = c.Lp, *D = c.dinv, *MN = c.mn;
    double *ctmp = sh + ((c.n + 1) & ~1);
    if (rank == 0 && c.kind == 0 && c.staged) {  // CTA 0 owns no SpMV rows: its smem is the coarse area
        double *Ds = ctmp + 32;
        for (int i = threadIdx.x; i < c.n; i += blockDim.x) Ds[i] = c.dinv[i];
        // the pre-scaled diagonal blocks stay in L2 here (their loads hoist off the chain);
        // a smaller footprint lets the cluster launch early
        double *Ls = Ds + ((c.n + 1) & ~1);
        const int64_t np = tri(c.n);
#pragma unroll 8
        for (int64_t i = threadIdx.x; i < np; i += blockDim.x) Ls[i] = __ldg(c.Lp + i);
        L = Ls;
        D = Ds;
    }
    {
        const int nw = nops * (int)(sizeof(TailOp) / 4);
        const int *src = reinterpret_cast<const int *>(ops);
        int *dst = reinterpret_cast<int *>(s_ops);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
        for (int m = threadIdx.x; m < nmats; m += blockDim.x) {
            s_split[m][0] = splits[mats[m].split + rank];
            s_split[m][1] = splits[mats[m].split + rank + 1];
            s_geo[m][0] = mats[m].staged ? mats[m].smem_off : -1;
            s_geo[m][1] = mats[m].rows_cap;
            s_geo[m][2] = mats[m].nnz_cap;
        }
    }
    for (int m = 0; m < nmats; ++m) {
        const TailMat M = mats[m];
        if (!M.staged) continue;
        const int r0 = splits[M.split + rank], r1 = splits[M.split + rank + 1];
        if (r1 <= r0) continue;  // no rows here: the region overlays the coarse area on CTA 0
        const int k0 = M.off[r0];
        int32_t *os = reinterpret_cast<int32_t *>(smem + M.smem_off);
        int32_t *cs = reinterpret_cast<int32_t *>(smem + M.smem_off + (((M.rows_cap + 1) * 4 + 15) & ~15));
        double *vs = reinterpret_cast<double *>(reinterpret_cast<char *>(cs) + ((M.nnz_cap * 4 + 15) & ~15));
        for (int r = threadIdx.x; r <= r1 - r0; r += blockDim.x) os[r] = M.off[r0 + r] - k0;
        const int nk = M.off[r1] - k0;
        for (int k = threadIdx.x; k < nk; k += blockDim.x) {
            cs[k] = M.col[k0 + k];
            vs[k] = M.val[k0 + k];
        }
    }
    if (c.prefetch) {
        // pull this CTA's share of the streamed matrices into L2 while the predecessor
        // drains: the level-0 sweeps evicted them, and 16 SMs alone fetch them from HBM slowly
        for (int m = 0; m < nmats; ++m) {
            const TailMat M = mats[m];
            if (M.staged) continue;
            const int r0 = splits[M.split + rank], r1 = splits[M.split + rank + 1];
            if (r1 <= r0) continue;
            const int k0 = M.off[r0], k1 = M.off[r1];
            const char *pv = reinterpret_cast<const char *>(M.val + k0);
            const char *pc = reinterpret_cast<const char *>(M.col + k0);
            const char *po = reinterpret_cast<const char *>(M.off + r0);
            for (int i = threadIdx.x * 128; i < (k1 - k0) * 8; i += blockDim.x * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pv + i));
            for (int i = threadIdx.x * 128; i < (k1 - k0) * 4; i += blockDim.x * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + i));
            for (int i = threadIdx.x * 128; i < (r1 - r0 + 1) * 4; i += blockDim.x * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(po + i));
        }
    }
    __syncthreads();
    pdl_launch();
    pdl_wait();
    if (!gate_open(gate1, nullptr)) return;  // uniform across the cluster
    const int t0 = rank * blockDim.x + threadIdx.x;
    const int nt = gridDim.x * blockDim.x;  // grid == one cluster
    if (trace && t0 == 0) trace[0] = globaltimer();
    for (int i = 0; i < nops; ++i) {
        const TailOp &o = s_ops[i];
        if (o.kind == TAIL_SPMV) {
            const int r0 = s_split[o.mat][0], r1 = s_split[o.mat][1];
            const int moff = s_geo[o.mat][0], rcap = s_geo[o.mat][1], kcap = s_geo[o.mat][2];
            if (moff < 0) {
                const TailMat M = mats[o.mat];
                switch (o.epi) {
                case EPI_PLAIN: tail_spmv_streamed<EPI_PLAIN>(o, M, r0, r1, ps, s_vec, smem, tvv.pcap); break;
                case EPI_RESID: tail_spmv_streamed<EPI_RESID>(o, M, r0, r1, ps, s_vec, smem, tvv.pcap); break;
                case EPI_AXPYW: tail_spmv_streamed<EPI_AXPYW>(o, M, r0, r1, ps, s_vec, smem, tvv.pcap); break;
                case EPI_SETW: tail_spmv_streamed<EPI_SETW>(o, M, r0, r1, ps, s_vec, smem, tvv.pcap); break;
                default: tail_spmv_streamed<EPI_ADD>(o, M, r0, r1, ps, s_vec, smem, tvv.pcap); break;
                }
                tail_sync(gbar);
                if (trace && t0 == 0) trace[i + 1] = globaltimer();
                continue;
            }
            const int32_t *os = reinterpret_cast<const int32_t *>(smem + moff);
            const int32_t *cs = reinterpret_cast<const int32_t *>(smem + moff + (((rcap + 1) * 4 + 15) & ~15));
            const double *vs = reinterpret_cast<const double *>(reinterpret_cast<const char *>(cs) + ((kcap * 4 + 15) & ~15));
            switch (o.epi) {
            case EPI_PLAIN: tail_spmv<EPI_PLAIN>(o, r0, r1, os, cs, vs, ps, s_vec, smem); break;
            case EPI_RESID: tail_spmv<EPI_RESID>(o, r0, r1, os, cs, vs, ps, s_vec, smem); break;
            case EPI_AXPYW: tail_spmv<EPI_AXPYW>(o, r0, r1, os, cs, vs, ps, s_vec, smem); break;
            case EPI_SETW: tail_spmv<EPI_SETW>(o, r0, r1, os, cs, vs, ps, s_vec, smem); break;
            default: tail_spmv<EPI_ADD>(o, r0, r1, os, cs, vs, ps, s_vec, smem); break;
            }
        } else if (o.kind == TAIL_JACOBI) {
            for (int r = t0; r < o.nrows; r += nt) {
                const double z = __dmul_rn(o.omega, __dmul_rn(__ldg(o.d + r), tv_ld(o.x, o.xs, r, s_vec, smem)));
                tv_st(o.y, o.ys, r, o.mode ? add(tv_ld(o.y, o.ys, r, s_vec, smem), z) : z, s_vec, smem);
            }
        } else if (rank == 0) {  // coarsest solve on CTA 0
            double *v = sh;
            for (int r = threadIdx.x; r < c.n; r += blockDim.x) v[r] = tv_ld(o.x, o.xs, r, s_vec, smem);
            __syncthreads();
            if (c.kind == 0 && c.pipe && c.n <= 32 * (int)(blockDim.x / 32) && c.n <= 512) chol_solve_pipe(c.n, L, D, v, c.pipe > 1 ? c.pipe : 0);
            else if (c.kind == 0) chol_solve_cta(c.n, L, D, c.staged ? nullptr : MN, v);
            else lu_solve_cta(c.n, c.LU, c.piv, v);
            for (int r = threadIdx.x; r < c.n; r += blockDim.x) tv_st(o.y, o.ys, r, v[r], s_vec, smem);
        }
        tail_sync(gbar);
        if (trace && t0 == 0) trace[i + 1] = globaltimer();
    }
}

}  // namespace amg
