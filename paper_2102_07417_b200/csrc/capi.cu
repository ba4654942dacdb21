// libamgb200: host runtime + C ABI of the B200-native PCG + AMG solve phase.
//
// Owns the device copy of the hierarchy (uploaded once from the reference's
// setup output), the tile schedules of every matrix, the work vectors of
// every level, the device-resident PCG state and the CUDA graph of one PCG
// iteration, which runs as a device-side while loop (conditional graph node)
// so a whole solve is a single graph launch with no host round trip.
//
// Reference behaviour each piece follows is cited at the entry points in
// include/amgb200.h; the per-level V-cycle sequence is hierarchy.py:294-312
// with smoothers.py:168-173 expanded as in SURVEY.md 8(a).
#include "amgb200.h"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <vector>

#include "halo.h"

using namespace amg;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

#define CK(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            return fail(AMG_E_CUDA, std::string(#call) + " failed: " + cudaGetErrorString(e_));      \
    } while (0)

#define TRY(expr)                \
    do {                         \
        int s_ = (expr);         \
        if (s_ != AMG_OK) return s_; \
    } while (0)

#include "setup.cuh"

namespace {

struct DevMat {
    bool present = false;
    int64_t nrows = 0, ncols = 0, nnz = 0;  // local rows; extended column space
    int64_t gncols = 0;                      // column-space size passed at upload
    int64_t n_own = 0;                       // owned columns (== gncols without a halo plan)
    int32_t *off = nullptr, *col = nullptr;
    double *val = nullptr;
    int32_t *sbeg = nullptr;     // SELL-32 layout (spmv_sell), nullptr if unused
    double *sval = nullptr;
    int32_t *scol = nullptr;
    uint8_t *slen = nullptr;
    int32_t *sperm = nullptr;    // SELL-sigma permutation (slice position -> row)
    int sell_grid = 0;
    uint8_t *pid = nullptr;      // stencil-pattern layout (spmv_pat): pattern id per row
    int32_t *prel = nullptr;     // concatenated relative offsets
    int32_t *pbeg = nullptr;     // pattern starts into prel
    int npat = 0, nrel = 0;
    double *uval = nullptr;      // symmetric stencil layout (spmv_symd), nullptr if unused
    int sym_slot = -1;           // its __constant__ pattern-start slot
    int sym_tab = -1, sym_ntab = 0, sym_classes = 1, sym_npad = 0;  // entry range in c_symd_tab; row classes
    double *uval_s = nullptr;    // uniform-width SELL-32 (spmv_sellu), nullptr if unused
    double *sv_s = nullptr;      // sorted SELL-32 (spmv_sells), nullptr if unused
    int32_t *sc_s = nullptr, *sb_s = nullptr, *sp_s = nullptr;
    uint8_t *sw_s = nullptr, *sl_s = nullptr;
    int s_grid = 0;
    int32_t *ucol_s = nullptr;
    uint8_t *ulen_s = nullptr;
    uint8_t *uperm_s = nullptr;  // PLEN layouts sorted inside each slice: slot -> row within the slice
    uint8_t *uvid_s = nullptr;   // value id per stored entry (VD == 2 kernels), nullptr if unused
    uint8_t *ucls_s = nullptr;   // value-tuple class per slot (VD kernels), nullptr if unused
    double *uvtab = nullptr;
    int32_t *uvlen = nullptr;
    int uncls = 0;
    int uW = 0, u_grid = 0, u_plen = 0;  // u_plen: padding slots skipped (short ragged rows)
    int nudiag = 0, sym_grid = 0, sym_fl = 0, symf_grid = 0, sym_blocked = 0;
    bool sym_fast_on = false;    // interior 27-entry pattern with parameter-bank offsets (spmv_symd27)
    SymFast sym_fast = {};
    int sym27_grid = 0;  // sym_fl: fixed-slot kernel width (0: none)
    int32_t *pstart = nullptr;   // padded-aligned layout (spmv_vec), nullptr if unused
    double *pval = nullptr;
    int32_t *pcol = nullptr;
    int pad_grid = 0;
    int lanes = 1;
    int grid = 0;
    int2 *leaf = nullptr;        // long-row leaves (spmv_leaves + spmv_leafsum), nullptr if unused
    int32_t *row_leaf = nullptr;
    double *lsum = nullptr;
    int nleaves = 0, leaf_grid = 0, leafsum_grid = 0;
    HaloPlan halo;  // exchange feeding this matrix's halo columns (nranks > 1)
    int64_t lbytes[16] = {};  // per layout: bytes its kernel must stream (values, indices, row metadata)
    int64_t int_lo = 0, int_hi = 0;  // interior rows [int_lo, int_hi): no halo column (overlap split), 128-aligned
    void *dcls = nullptr;     // row-class dictionary (spmv_dict): class id per row, nullptr if unused
    int32_t *dbeg = nullptr, *drel = nullptr;
    double *dval = nullptr;
    int dncls = 0, dnent = 0, dwide = 0, dfl = 0, dgrid = 0;
    int dmcls = -1, dmlen = 0;   // most frequent class (its entries travel as kernel parameters), -1: none
    int32_t dmrel[8] = {};
    double dmval[8] = {};
    int wcsr = 0, wcsr_grid = 0;  // warp-cooperative CSR (spmv_wcsr) on the uploaded arrays
};

struct LevelD {
    int64_t n = 0;   // local rows
    int64_t n0 = 0;  // first global row
    int64_t gn = 0;  // global rows
    int64_t cap = 0; // vector capacity: local + max halo
    std::vector<int64_t> starts;  // partition (nranks + 1)
    DevMat m[5];
    bool has_smoother = false;
    int sm_kind = AMG_SMOOTHER_FSAI;
    double omega = 1.0;
    double *inv_diag = nullptr;
    double *y = nullptr, *x = nullptr, *r = nullptr, *t = nullptr;
};

std::mutex g_alloc_mu;
std::unordered_map<const void *, size_t> g_alloc_size;  // allocation sizes (device memory accounting)

template <class T>
int dalloc(T **p, size_t count)
{
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc((void **)p, bytes);
    if (e != cudaSuccess) return fail(AMG_E_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    {
        std::lock_guard<std::mutex> g(g_alloc_mu);
        g_alloc_size[*p] = bytes;
    }
    e = cudaMemset(*p, 0, bytes);
    if (e != cudaSuccess) return fail(AMG_E_CUDA, cudaGetErrorString(e));
    return AMG_OK;
}

}  // namespace

// __constant__ pattern-table slots (kernels.cuh c_symd_*), per device, process-wide:
// handles on one device share the module's constant bank.
static std::mutex g_symd_mu;
static std::unordered_map<int, unsigned> g_symd_used;  // device -> slot bitmask

static int symd_slot_take(int device)
{
    std::lock_guard<std::mutex> g(g_symd_mu);
    unsigned &m = g_symd_used[device];
    for (int i = 0; i < SYMD_SLOTS; ++i)
        if (!(m & (1u << i))) {
            m |= 1u << i;
            return i;
        }
    return -1;
}

static std::unordered_map<int, std::vector<std::pair<int, int>>> g_symd_tab;  // device -> used [start, len)

static int symd_tab_take(int device, int len)
{
    std::lock_guard<std::mutex> g(g_symd_mu);
    auto &u = g_symd_tab[device];
    std::sort(u.begin(), u.end());
    int at = 0;
    for (auto &r : u) {
        if (r.first - at >= len) break;
        at = std::max(at, r.first + r.second);
    }
    if (at + len > SYMD_TAB) return -1;
    u.emplace_back(at, len);
    return at;
}

static void symd_tab_give(int device, int start, int len)
{
    if (start < 0) return;
    std::lock_guard<std::mutex> g(g_symd_mu);
    auto &u = g_symd_tab[device];
    for (size_t i = 0; i < u.size(); ++i)
        if (u[i].first == start && u[i].second == len) {
            u.erase(u.begin() + i);
            return;
        }
}

static void symd_slot_give(int device, int slot)
{
    if (slot < 0) return;
    std::lock_guard<std::mutex> g(g_symd_mu);
    g_symd_used[device] &= ~(1u << slot);
}

struct amg_handle {
    int device = 0, rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;           // side stream: L2 prefetch of the tail levels
    cudaStream_t comm_stream = nullptr;    // nranks > 1: halo send / recv, overlapped with interior rows
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    int overlap_test = 0;                  // nranks == 1 diagnostics: run the interior / boundary split anyway
    int nccl_selftest = 0;                 // nranks == 1 diagnostics: a one-rank NCCL communicator carries the dot
                                           // all-gathers and a self send / recv per split SpMV on the comm stream
    double *selftest_buf = nullptr;
    cudaEvent_t pf_fork = nullptr, pf_join = nullptr;
    PrefetchRange *pf_ranges = nullptr;    // device copy of the tail matrices' ranges
    int pf_n = 0;
    bool pf_pending = false;
    int sm_count = 148;
    std::vector<LevelD> lv;
    int nu1 = 1, nu2 = 1;
    // coarsest factor
    int nc = 0, coarse_kind = AMG_COARSE_CHOLESKY;
    double *Lp = nullptr, *LU = nullptr, *dinv = nullptr, *binv = nullptr;
    int32_t *piv = nullptr;
    int coarse_staged = 0;
    size_t coarse_smem = 0;
    bool finalized = false;
    bool container = false;
    // scratch
    double *partials = nullptr;
    unsigned *ticket = nullptr;
    int max_grid = 0;
    PcgCtl *ctl = nullptr;
    PcgCtl *ctl_h = nullptr;  // pinned mirror
    double *b = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double *tmp_in = nullptr, *tmp_out = nullptr;
    double *bicg[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // rs, v, phat, s, shat, t
    double *hist = nullptr;
    int hist_cap = 0;
    // options
    int force_graph = -1, batch = 8;
    int pad_min = 8;     // matrices averaging >= pad_min entries/row get the padded-aligned layout (0 = off)
    int long_avg = 128;           // rows averaging more entries run leaf by leaf (spmv_leaves); 0 = off
    int small_rows_per_sm = 128;  // below sm_count * this many rows a matrix counts as small
    int patterns = 1;             // stencil-pattern layout for square operators with few row patterns
    int symd_tsm = 0;             // round-by-round symmetric kernel: pattern table staged in smem instead of __constant__
    int symd_classes = 3;         // symmetric layout: try row classes r % K, K = 1..symd_classes
    int symd_blocked = 1;         // symmetric layout stored slice-blocked (32 rows x nu diagonals contiguous)
    int symd_gminb = 5;           // round-by-round symmetric kernel: min CTAs/SM 5, 6 or 8
    int symd_minb = 4;            // fixed-slot 32-wide kernel: min CTAs/SM (register budget) 3, 4 or 5
    int sells = 1;                // sorted SELL-32 (sigma window below) where natural slices pad > 10%
    int sells_sigma = 128;
    int sells_buckets = 0;        // > 0: matrices above sells_max_rows get rows partitioned by round count into
                                  // 1 + sells_buckets classes (order kept inside a class)
    int sells_plen = 1;           // sorted SELL: predicate slot loads on the row length (padding moves no bytes)
    int sells_max_pad = 60;       // % padding allowed for the sorted layout (padding slots are skipped with sells_plen)
    double sells_min_avg = 4.0;   // ... for matrices averaging at least this many entries per row
    int64_t sells_max_rows = 2000000;  // ... and at most this many rows (sorting costs fine-grid rows their gather
                                       // locality: config-2 G^T_0 85 -> 134 us; coarse A_1 18 -> 13 us)
    int rz_sep = 0;               // PCG: r.z in a separate dot kernel instead of the V-cycle's last SpMV
    int vec_minb = 4;             // padded-CSR kernel: min CTAs per SM (register budget) 4, 5 or 6
    int sellu_short = 1;          // ... and for rows of <= 8 entries at any padding, padding slots skipped
    int sellu_vdict = 1;          // skipped-padding uniform SELL: value-tuple classes (<= 255) instead of stored values
    int sellu_sort = 1;           // skipped-padding uniform SELL: rows sorted by length inside each slice
    int sellu = 1;                // uniform-width SELL-32 for rows of <= 16 entries padding <= 10% (e.g. FSAI G)
    int symd_chunked = 0;         // symmetric kernels: contiguous row chunk per CTA (measured slower than grid-stride)
    int symd_fixed = 1;           // fixed-slot symmetric kernel: 1 rows <= 8 entries (7-point), 2 also <= 32 (27-point:
                                  // measured slower than the round-by-round kernel on config 2), 0 off
    int symm = 1;                 // symmetric stencil layout (upper diagonals) for bitwise-symmetric pattern operators
    int symd_fast = 1;            // symmetric layout: interior 27-entry rows through spmv_symd27 (offsets as kernel parameters)
    int dict_main = 1;            // spmv_dict: warps whose rows all have the most frequent class take its entries from kernel parameters
    int dict = 1;                 // row-class dictionary layout for operators with few distinct rows
    int wcsr = 1;                 // large matrices averaging >= pad_min entries: warp-cooperative CSR instead of the padded copy
    int sell = 1;                 // SELL-32 slices where padding <= sell_pad %
    int gated_grid = 1;           // CTAs per SM for the rarely active gated residual SpMVs (0 = full grid)
    int grid_per_sm = 0;          // cap on SpMV CTAs per SM (0 = occupancy)
    int vec_per_sm = 0;           // cap on vector-kernel CTAs per SM (0 = 8)
    int sell_pad = 10;
    int sell_sigma = 0;           // SELL-sigma sort window (rows); <= 32 disables (measured slower on config 2)
    int direct_ctas = 0; // direct kernel CTAs per SM (0 = occupancy)
    int direct_per_sm = 8;
    int lanes_override = 0;
    int pdl = 1;  // programmatic dependent launch between consecutive kernels
    // cluster tail: levels >= tail_level run inside one cluster kernel
    int64_t tail_nnz = 300000;   // levels whose A_k has at most this many entries run in the cluster tail
    int tail_stage = 0;          // stage tail matrices in smem (measured slower on B200: the big smem
                                 // footprint delays the cluster launch; streamed from L2 by default)
    int cluster = 16;             // CTAs of the tail: one cluster, or (tail_grid) the cooperative grid
    int tail_grid = 0;            // tail on a cooperative grid of every SM (grid barriers) instead of one cluster
    unsigned *tail_gbar = nullptr;
    int coarse_pipe = 1;          // pipelined per-warp Cholesky substitution
    int side_prefetch = 1;        // side-stream L2 prefetch of the tail matrices during the level above it
    int tail_pcap = 16384;        // tail product buffer (entries); larger per-CTA blocks are processed in chunks
    int tail_pcap_used = 0;
    int tail_dsm = 0;             // tail level vectors in distributed shared memory
    int tail_prefetch = 1;        // tail kernel prefetches its streamed matrices into L2 before griddepcontrol.wait
    int tail_level = 0;  // 0 = disabled
    TailOp *tail_ops = nullptr;
    TailMat *tail_mats = nullptr;
    int2 *tail_vecs = nullptr;    // DSMEM slots of the tail's level vectors (tail_dsm)
    int tail_nvecs = 0;
    int tail_nmats = 0;
    int32_t *tail_splits = nullptr;
    int tail_prod_off = 0;
    int tail_nops = 0;
    size_t tail_smem = 0;
    std::vector<TailOp> *collect = nullptr;  // op collection mode (builds the tail)
    std::vector<const DevMat *> *collect_mats = nullptr;
    unsigned long long *trace = nullptr;     // AMGB200_TRACE: %globaltimer per tail op
    // graph
    cudaGraphExec_t gexec = nullptr;
    int graph_mode = 0;
    int64_t launches = 0;  // running launch counter
    int64_t launches_per_iter = 0;
    int64_t launches_last = 0;
    double solve_ms = 0.0, e2e_ms = 0.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    Comm comm;
    int agglom_level = -1;     // nranks > 1: first replicated level (-1: none declared)
    bool dist_dots = false;    // level-0 vectors are distributed: dots need a cross-rank sum
};

// ------------------------------------------------------------------ kernels dispatch

typedef void (*SpmvFn)(const SpmvArgs);

typedef void (*SpmvSellFn)(const SpmvArgs, const SellArgs, int);

static SpmvSellFn spmv_sell_fn(int epi, bool pat)
{
#define AMG_S(E) return pat ? spmv_sell<E, true> : spmv_sell<E, false>;
    switch (epi) {
    case EPI_PLAIN: AMG_S(EPI_PLAIN)
    case EPI_RESID: AMG_S(EPI_RESID)
    case EPI_AXPYW: AMG_S(EPI_AXPYW)
    case EPI_SETW: AMG_S(EPI_SETW)
    default: AMG_S(EPI_ADD)
    }
#undef AMG_S
}

typedef void (*SpmvSymFn)(const SpmvArgs, const SymArgs, int);

static SpmvSymFn spmv_symd_fn(int epi, int minb = 5, bool blk = false, bool tsm = false)
{
#define AMG_Y(E)                                                                                     \
    return (blk && tsm) ? spmv_symd<E, 5, true, true> : blk ? spmv_symd<E, 5, true>                   \
               : (minb >= 8 ? spmv_symd<E, 8, false> : minb == 6 ? spmv_symd<E, 6, false> : spmv_symd<E, 5, false>);
    switch (epi) {
    case EPI_PLAIN: AMG_Y(EPI_PLAIN)
    case EPI_RESID: AMG_Y(EPI_RESID)
    case EPI_AXPYW: AMG_Y(EPI_AXPYW)
    case EPI_SETW: AMG_Y(EPI_SETW)
    default: AMG_Y(EPI_ADD)
    }
#undef AMG_Y
}

typedef void (*SpmvSym27Fn)(const SpmvArgs, const SymArgs, const SymFast, int);

static SpmvSym27Fn spmv_symd27_fn(int epi)
{
    switch (epi) {
    case EPI_PLAIN: return spmv_symd27<EPI_PLAIN>;
    case EPI_RESID: return spmv_symd27<EPI_RESID>;
    case EPI_AXPYW: return spmv_symd27<EPI_AXPYW>;
    case EPI_SETW: return spmv_symd27<EPI_SETW>;
    default: return spmv_symd27<EPI_ADD>;
    }
}

static SpmvSymFn spmv_symd_fixed_fn(int epi, int fl, int minb = 0, bool blk = false)
{
#define AMG_F(E)                                                                                     \
    return fl <= 8 ? (blk ? spmv_symd_fixed<E, 8, 6, true> : spmv_symd_fixed<E, 8, 6, false>)          \
                   : blk ? spmv_symd_fixed<E, 32, 4, true>                                            \
                   : (minb == 3 ? spmv_symd_fixed<E, 32, 3, false>                                    \
                                : minb == 5 ? spmv_symd_fixed<E, 32, 5, false> : spmv_symd_fixed<E, 32, 4, false>);
    switch (epi) {
    case EPI_PLAIN: AMG_F(EPI_PLAIN)
    case EPI_RESID: AMG_F(EPI_RESID)
    case EPI_AXPYW: AMG_F(EPI_AXPYW)
    case EPI_SETW: AMG_F(EPI_SETW)
    default: AMG_F(EPI_ADD)
    }
#undef AMG_F
}

typedef void (*SpmvSellUFn)(const SpmvArgs, const SellUArgs, int);

static SpmvSellUFn spmv_sellu_fn(int epi, int W, bool plen = false, int vd = 0)
{
#define AMG_U(E)                                                                                        \
    if (plen && vd == 1) return W <= 4 ? spmv_sellu<E, 4, true, 1> : spmv_sellu<E, 8, true, 1>;           \
    if (!plen && vd == 1 && W <= 9) return W <= 4 ? spmv_sellu<E, 4, false, 1> : spmv_sellu<E, 9, false, 1>; \
    if (plen && vd == 2) return W <= 4 ? spmv_sellu<E, 4, true, 2> : spmv_sellu<E, 8, true, 2>;           \
    if (!plen && vd == 2 && W <= 9) return W <= 4 ? spmv_sellu<E, 4, false, 2> : spmv_sellu<E, 9, false, 2>; \
    return plen ? (W <= 4 ? spmv_sellu<E, 4, true> : spmv_sellu<E, 8, true>)                             \
                : (W <= 4 ? spmv_sellu<E, 4, false> : W <= 9 ? spmv_sellu<E, 9, false> : spmv_sellu<E, 16, false>);
    switch (epi) {
    case EPI_PLAIN: AMG_U(EPI_PLAIN)
    case EPI_RESID: AMG_U(EPI_RESID)
    case EPI_AXPYW: AMG_U(EPI_AXPYW)
    case EPI_SETW: AMG_U(EPI_SETW)
    default: AMG_U(EPI_ADD)
    }
#undef AMG_U
}

// dynamic shared memory of the value-class uniform SELL kernels: table [ncls][FL] + lengths
// slots per row of the spmv_sellu instantiation serving width W
static int sellu_fl(int W, bool plen) { return plen ? (W <= 4 ? 4 : 8) : (W <= 4 ? 4 : W <= 9 ? 9 : 16); }

static int sellu_vd_mode(const DevMat &M) { return M.ucls_s ? 1 : M.uvid_s ? 2 : 0; }

static size_t sellu_vd_bytes(const DevMat &M)
{
    if (M.uvid_s) return (size_t)M.uncls * sizeof(double);
    if (!M.ucls_s) return 0;
    const int fl = sellu_fl(M.uW, M.u_plen != 0);
    return (size_t)M.uncls * fl * sizeof(double) + (size_t)M.uncls * sizeof(int32_t);
}

typedef void (*SpmvWcsrFn)(const SpmvArgs, int);

static SpmvWcsrFn spmv_wcsr_fn(int epi)
{
    switch (epi) {
    case EPI_PLAIN: return spmv_wcsr<EPI_PLAIN>;
    case EPI_RESID: return spmv_wcsr<EPI_RESID>;
    case EPI_AXPYW: return spmv_wcsr<EPI_AXPYW>;
    case EPI_SETW: return spmv_wcsr<EPI_SETW>;
    default: return spmv_wcsr<EPI_ADD>;
    }
}

typedef void (*SpmvDictFn)(const SpmvArgs, const DictArgs, int);

static SpmvDictFn spmv_dict_fn(int epi, int fl, bool wide, int ml)
{
    // ml: entries of the most frequent class when it gets a compile-time interior path (3, 5, 7), else 0.
    // Two rows per thread and step were measured slower once the interior path was lean (stand-in A0
    // 31.7 vs 25.3 us, G0 19.7 vs 16.5 us): one row per thread, 5 CTAs / SM.
#define AMG_D(E)                                                                                                   \
    if (!wide && fl <= 4 && ml == 3) return spmv_dict<E, 4, false, 1, 3>;                                          \
    if (!wide && fl == 8 && ml == 5) return spmv_dict<E, 8, false, 1, 5>;                                          \
    if (!wide && fl == 8 && ml == 7) return spmv_dict<E, 8, false, 1, 7>;                                          \
    return wide ? (fl <= 8 ? spmv_dict<E, 8, true, 1> : fl <= 16 ? spmv_dict<E, 16, true, 1> : spmv_dict<E, 32, true, 1>) \
                : (fl <= 8 ? spmv_dict<E, 8, false, 1> : fl <= 16 ? spmv_dict<E, 16, false, 1> : spmv_dict<E, 32, false, 1>);
    switch (epi) {
    case EPI_PLAIN: AMG_D(EPI_PLAIN)
    case EPI_RESID: AMG_D(EPI_RESID)
    case EPI_AXPYW: AMG_D(EPI_AXPYW)
    case EPI_SETW: AMG_D(EPI_SETW)
    default: AMG_D(EPI_ADD)
    }
#undef AMG_D
}

typedef void (*SpmvSellSFn)(const SpmvArgs, const SellSArgs, int);

static SpmvSellSFn spmv_sells_fn(int epi, bool plen = false)
{
#define AMG_S2(E) return plen ? spmv_sells<E, true> : spmv_sells<E, false>;
    switch (epi) {
    case EPI_PLAIN: AMG_S2(EPI_PLAIN)
    case EPI_RESID: AMG_S2(EPI_RESID)
    case EPI_AXPYW: AMG_S2(EPI_AXPYW)
    case EPI_SETW: AMG_S2(EPI_SETW)
    default: AMG_S2(EPI_ADD)
    }
#undef AMG_S2
}

typedef void (*SpmvPatFn)(const SpmvArgs, const PatArgs, int);

static SpmvPatFn spmv_pat_fn(int epi)
{
    switch (epi) {
    case EPI_PLAIN: return spmv_pat<EPI_PLAIN>;
    case EPI_RESID: return spmv_pat<EPI_RESID>;
    case EPI_AXPYW: return spmv_pat<EPI_AXPYW>;
    case EPI_SETW: return spmv_pat<EPI_SETW>;
    default: return spmv_pat<EPI_ADD>;
    }
}

typedef void (*SpmvVecFn)(const SpmvArgs, const PadArgs, int);

static SpmvVecFn spmv_vec_fn(int epi, int vminb = 4)
{
#define AMG_V(E) return vminb >= 6 ? spmv_vec<E, 6> : vminb == 5 ? spmv_vec<E, 5> : spmv_vec<E, 4>;
    switch (epi) {
    case EPI_PLAIN: AMG_V(EPI_PLAIN)
    case EPI_RESID: AMG_V(EPI_RESID)
    case EPI_AXPYW: AMG_V(EPI_AXPYW)
    case EPI_SETW: AMG_V(EPI_SETW)
    default: AMG_V(EPI_ADD)
    }
#undef AMG_V
}

typedef void (*SpmvDirectFn)(const SpmvArgs, int);

static SpmvDirectFn spmv_direct_fn(int epi, int lanes)
{
#define AMG_L(E)                                               \
    switch (lanes) {                                           \
    case 1: return spmv_direct<E, 1>;                          \
    case 2: return spmv_direct<E, 2>;                          \
    case 4: return spmv_direct<E, 4>;                          \
    default: return spmv_direct<E, 8>;                         \
    }
    switch (epi) {
    case EPI_PLAIN: AMG_L(EPI_PLAIN)
    case EPI_RESID: AMG_L(EPI_RESID)
    case EPI_AXPYW: AMG_L(EPI_AXPYW)
    case EPI_SETW: AMG_L(EPI_SETW)
    default: AMG_L(EPI_ADD)
    }
#undef AMG_L
}

typedef void (*SpmvLeafsumFn)(const SpmvArgs, const LeafArgs, int);

static SpmvLeafsumFn spmv_leafsum_fn(int epi)
{
    switch (epi) {
    case EPI_PLAIN: return spmv_leafsum<EPI_PLAIN>;
    case EPI_RESID: return spmv_leafsum<EPI_RESID>;
    case EPI_AXPYW: return spmv_leafsum<EPI_AXPYW>;
    case EPI_SETW: return spmv_leafsum<EPI_SETW>;
    default: return spmv_leafsum<EPI_ADD>;
    }
}

// Every kernel goes through here: programmatic dependent launch lets a kernel
// start (stage static matrix tiles) while its predecessor drains.
template <typename... KArgs, typename... Args>
static int launch_k(amg_t *h, void (*kern)(KArgs...), int grid, int block, size_t smem, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (h->pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) return fail(AMG_E_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
    ++h->launches;
    return AMG_OK;
}

// Max-dynamic-smem caps are per-FUNCTION process state: raise them once to
// the device opt-in maximum so handles with different staging never clash.
static int raise_smem_caps(int device)
{
    static int done_for = -1;
    if (done_for == device) return AMG_OK;
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    auto cap = [&](const void *f) -> int {
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, f));
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
        return AMG_OK;
    };
    TRY(cap((const void *)coarse_solve_k));
    TRY(cap((const void *)tail_vcycle));
    CK(cudaFuncSetAttribute((const void *)tail_vcycle, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    done_for = device;
    return AMG_OK;
}

static int exchange(amg_t *h, const DevMat &M, double *x)
{
    if (h->nranks == 1 || M.halo.empty()) return AMG_OK;
    const HaloPlan &P = M.halo;
    NcclApi &api = nccl();
    if (P.n_send > 0) {
        int g = (int)std::min<int64_t>((P.n_send + VEC_THREADS - 1) / VEC_THREADS, (int64_t)h->sm_count * 4);
        TRY(launch_k(h, halo_pack, std::max(g, 1), VEC_THREADS, 0, (const double *)x, (const int32_t *)P.send_idx,
                     P.send_buf, P.n_send));
    }
    auto chk = [&](ncclResult_t r, const char *w) -> int {
        if (r != ncclSuccess) return fail(AMG_E_NCCL, std::string(w) + ": " + api.GetErrorString(r));
        return AMG_OK;
    };
    TRY(chk(api.GroupStart(), "ncclGroupStart"));
    int64_t roff = P.n_own;
    for (size_t i = 0; i < P.recv_peers.size(); ++i) {
        TRY(chk(api.Recv(x + roff, (size_t)P.recv_counts[i], ncclDouble, P.recv_peers[i], h->comm.comm, h->stream), "ncclRecv"));
        roff += P.recv_counts[i];
    }
    for (size_t i = 0; i < P.send_peers.size(); ++i)
        TRY(chk(api.Send(P.send_buf + P.send_displ[i], (size_t)P.send_counts[i], ncclDouble, P.send_peers[i],
                         h->comm.comm, h->stream), "ncclSend"));
    TRY(chk(api.GroupEnd(), "ncclGroupEnd"));
    return AMG_OK;
}

// Overlapped exchange: the pack kernel on the main stream, the grouped
// send / recv on the comm stream (after the pack), ev_halo marks arrival;
// exchange_end makes the main stream wait for it.  Captured into the
// iteration graph as a fork / join.
static int exchange_begin(amg_t *h, const DevMat &M, double *x)
{
    if (h->nranks == 1 && h->nccl_selftest && h->nccl_selftest != 2 && h->comm.comm) {  // one element to self
        NcclApi &api = nccl();
        // 4: p2p on the main stream (no fork / join); 5: fork / join with an empty side kernel, no NCCL
        cudaStream_t cs = h->nccl_selftest == 4 ? h->stream : h->comm_stream;
        if (h->nccl_selftest != 4) {
            CK(cudaEventRecord(h->ev_pack, h->stream));
            CK(cudaStreamWaitEvent(h->comm_stream, h->ev_pack, 0));
        }
        if (h->nccl_selftest == 5) {
            vec_copy<<<1, 32, 0, h->comm_stream>>>(VecArgs{});
            CK(cudaGetLastError());
        } else {
            ncclResult_t r = api.GroupStart();
            if (r == ncclSuccess) r = api.Recv(h->selftest_buf, 1, ncclDouble, 0, h->comm.comm, cs);
            if (r == ncclSuccess) r = api.Send(x, 1, ncclDouble, 0, h->comm.comm, cs);
            ncclResult_t r2 = api.GroupEnd();
            if (r != ncclSuccess || r2 != ncclSuccess)
                return fail(AMG_E_NCCL, std::string("self send/recv: ") + api.GetErrorString(r != ncclSuccess ? r : r2));
        }
        if (h->nccl_selftest != 4) CK(cudaEventRecord(h->ev_halo, h->comm_stream));
        return AMG_OK;
    }
    if (h->nranks == 1 || M.halo.empty()) return AMG_OK;
    const HaloPlan &P = M.halo;
    NcclApi &api = nccl();
    if (P.n_send > 0) {
        int g = (int)std::min<int64_t>((P.n_send + VEC_THREADS - 1) / VEC_THREADS, (int64_t)h->sm_count * 4);
        TRY(launch_k(h, halo_pack, std::max(g, 1), VEC_THREADS, 0, (const double *)x, (const int32_t *)P.send_idx,
                     P.send_buf, P.n_send));
    }
    CK(cudaEventRecord(h->ev_pack, h->stream));
    CK(cudaStreamWaitEvent(h->comm_stream, h->ev_pack, 0));
    auto chk = [&](ncclResult_t r, const char *w) -> int {
        if (r != ncclSuccess) return fail(AMG_E_NCCL, std::string(w) + ": " + api.GetErrorString(r));
        return AMG_OK;
    };
    TRY(chk(api.GroupStart(), "ncclGroupStart"));
    int64_t roff = P.n_own;
    for (size_t i = 0; i < P.recv_peers.size(); ++i) {
        TRY(chk(api.Recv(x + roff, (size_t)P.recv_counts[i], ncclDouble, P.recv_peers[i], h->comm.comm, h->comm_stream),
                "ncclRecv"));
        roff += P.recv_counts[i];
    }
    for (size_t i = 0; i < P.send_peers.size(); ++i)
        TRY(chk(api.Send(P.send_buf + P.send_displ[i], (size_t)P.send_counts[i], ncclDouble, P.send_peers[i],
                         h->comm.comm, h->comm_stream), "ncclSend"));
    TRY(chk(api.GroupEnd(), "ncclGroupEnd"));
    CK(cudaEventRecord(h->ev_halo, h->comm_stream));
    return AMG_OK;
}

static int exchange_end(amg_t *h, const DevMat &M)
{
    if (h->nranks == 1 && h->nccl_selftest && h->nccl_selftest != 2 && h->nccl_selftest != 4 && h->comm.comm) {
        CK(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
        return AMG_OK;
    }
    if (h->nranks == 1 || M.halo.empty()) return AMG_OK;
    CK(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
    return AMG_OK;
}

// Reductions: with distributed level-0 vectors a kernel's finalize stores the
// rank's partial; the partials are all-gathered and summed in rank order.
static int kfin(const amg_t *h, int fin) { return (h->dist_dots && fin != FIN_NONE) ? (int)FIN_LOCAL : fin; }

static int post_fin(amg_t *h, int fin, const int *g1)
{
    if (!h->dist_dots || fin == FIN_NONE) return AMG_OK;
    NcclApi &api = nccl();
    ncclResult_t r = api.AllGather(&h->ctl->part_local, h->ctl->part_all, 1, ncclDouble, h->comm.comm, h->stream);
    if (r != ncclSuccess) return fail(AMG_E_NCCL, std::string("ncclAllGather: ") + api.GetErrorString(r));
    TRY(launch_k(h, fin_ranks, 1, 1, 0, h->ctl, fin, h->nranks, g1));
    return AMG_OK;
}

// Agglomeration: every rank holds its piece of level k's vector at offset
// starts[rank]; grouped in-place broadcasts make the full vector everywhere.
static int allgather_level(amg_t *h, int k, double *y)
{
    NcclApi &api = nccl();
    const std::vector<int64_t> &s = h->lv[k].starts;
    ncclResult_t r = api.GroupStart();
    for (int q = 0; q < h->nranks && r == ncclSuccess; ++q)
        if (s[q + 1] > s[q]) r = api.Broadcast(y + s[q], y + s[q], (size_t)(s[q + 1] - s[q]), ncclDouble, q, h->comm.comm, h->stream);
    ncclResult_t r2 = api.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(AMG_E_NCCL, std::string("agglomeration broadcast: ") + api.GetErrorString(r != ncclSuccess ? r : r2));
    return AMG_OK;
}

// Halo exchange (nranks > 1): pack the owned entries each peer needs, then
// one grouped ncclSend/ncclRecv per peer into x[n_own ...] (plan order).
static int exchange(amg_t *h, const DevMat &M, double *x);

static int layout_of(const amg_t *h, const DevMat &M)
{
    // same precedence as launch_spmv
    return M.nrows == 0            ? AMG_LAYOUT_EMPTY
              : M.dcls                ? AMG_LAYOUT_DICT
              : (M.uval && h->symm)   ? AMG_LAYOUT_SYMD
              : (M.sv_s && h->sells)   ? AMG_LAYOUT_SELL_SORTED
              : (M.uval_s && h->sellu) ? AMG_LAYOUT_SELL_UNIFORM
              : M.sbeg                ? (M.scol ? AMG_LAYOUT_SELL : AMG_LAYOUT_SELL_PAT)
              : (M.pid && M.pstart)   ? AMG_LAYOUT_PATTERN
              : M.leaf                ? AMG_LAYOUT_LEAVES
              : M.wcsr                ? AMG_LAYOUT_WCSR
              : M.pstart              ? AMG_LAYOUT_PADDED
                                      : AMG_LAYOUT_CSR;
}

// Layouts whose kernels take row ranges (SpmvArgs rlo / rsplit / rgap).
static bool range_layout(int lay)
{
    return lay == AMG_LAYOUT_SELL_SORTED || lay == AMG_LAYOUT_SELL_UNIFORM || lay == AMG_LAYOUT_PADDED ||
           lay == AMG_LAYOUT_WCSR || lay == AMG_LAYOUT_CSR;
}

// One launch over `count` virtual rows (a.rlo / a.rsplit / a.rgap map them);
// *grid_used receives the grid (the partial slots this launch fills).
static int spmv_range(amg_t *h, const DevMat &M, int lay, const SpmvArgs &a, int epi, int count, int grid_cap,
                      int *grid_used)
{
    auto cap = [&](int g, int64_t need) {
        g = (int)std::max<int64_t>(1, std::min<int64_t>(g, need));
        return grid_cap ? std::min(g, grid_cap) : g;
    };
    int g = 1;
    if (lay == AMG_LAYOUT_SELL_SORTED) {
        SellSArgs qa{M.sv_s, M.sc_s, M.sb_s, M.sw_s, M.sp_s, M.sl_s, (int)M.nrows};
        g = cap(M.s_grid, ((count + 31) / 32 + 7) / 8);
        TRY(launch_k(h, spmv_sells_fn(epi, h->sells_plen), g, VEC_SPMV_THREADS, 0, a, qa, count));
    } else if (lay == AMG_LAYOUT_SELL_UNIFORM) {
        SellUArgs ua{M.uval_s, M.ucol_s, M.ulen_s, M.uW, M.uperm_s, M.ucls_s, M.uvtab, M.uvlen, M.uncls, M.uvid_s};
        g = cap(M.u_grid, (count + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS);
        TRY(launch_k(h, spmv_sellu_fn(epi, M.uW, M.u_plen, sellu_vd_mode(M)), g, VEC_SPMV_THREADS, sellu_vd_bytes(M), a, ua, count));
    } else if (lay == AMG_LAYOUT_WCSR) {
        g = cap(M.wcsr_grid, ((count + 31) / 32 + WCSR_THREADS / 32 - 1) / (WCSR_THREADS / 32));
        TRY(launch_k(h, spmv_wcsr_fn(epi), g, WCSR_THREADS, 0, a, count));
    } else if (lay == AMG_LAYOUT_PADDED) {
        PadArgs pa{M.pstart, M.pval, M.pcol};
        g = cap(M.pad_grid, (count + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS);
        TRY(launch_k(h, spmv_vec_fn(epi, h->vec_minb), g, VEC_SPMV_THREADS, 0, a, pa, count));
    } else if (lay == AMG_LAYOUT_CSR) {
        const int gpr = DIRECT_THREADS / M.lanes;
        g = cap(h->sm_count * h->direct_per_sm, (count + gpr - 1) / gpr);
        TRY(launch_k(h, spmv_direct_fn(epi, M.lanes), g, DIRECT_THREADS, 0, a, count));
    } else {
        return fail(AMG_E_STATE, "internal: row-range launch on a layout without range support");
    }
    if (grid_used) *grid_used = g;
    return AMG_OK;
}

static int launch_spmv(amg_t *h, const DevMat &M, const double *x, double *y, int epi, const double *b, double omega,
                       const double *dotw, int fin, const int *g1, const int *g2, int grid_cap = 0)
{
    if (h->collect) {
        if (dotw || fin != FIN_NONE) return fail(AMG_E_STATE, "internal: reduction inside the cluster tail");
        TailOp o{};
        o.kind = TAIL_SPMV;
        o.epi = epi;
        o.nrows = (int)M.nrows;
        o.mat = -1;
        h->collect_mats->push_back(&M);
        o.mode = (int)h->collect_mats->size() - 1;  // provisional: index into collect_mats
        o.x = x;
        o.y = y;
        o.b = b;
        o.omega = omega;
        h->collect->push_back(o);
        return AMG_OK;
    }
    if (h->grid_per_sm > 0) {  // global cap on CTAs per SM (tuning)
        const int c = h->grid_per_sm * h->sm_count;
        grid_cap = grid_cap ? std::min(grid_cap, c) : c;
    }
    const int ufin = fin;
    fin = kfin(h, fin);
    if (M.nrows == 0) {
        if (fin != FIN_NONE) {
            VecArgs v{};
            v.n = 0;
            v.partials = h->partials;
            v.ticket = h->ticket;
            v.fin = fin;
            v.ctl = h->ctl;
            v.gate1 = g1;
            v.gate2 = g2;
            TRY(launch_k(h, vec_dot, 1, VEC_THREADS, 0, v));
            TRY(post_fin(h, ufin, g1));
        }
        return AMG_OK;
    }
    SpmvArgs a{};
    a.off = M.off;
    a.col = M.col;
    a.val = M.val;
    a.x = x;
    a.y = y;
    a.b = b;
    a.omega = omega;
    a.dotw = dotw;
    a.partials = h->partials;
    a.ticket = h->ticket;
    a.fin = fin;
    a.ctl = h->ctl;
    a.gate1 = g1;
    a.gate2 = g2;
    a.rsplit = INT_MAX;
    a.pcap = 2 * h->max_grid;
    const int lay = layout_of(h, M);
    if (M.int_hi > M.int_lo && (h->nranks > 1 || h->overlap_test) && range_layout(lay)) {
        // interior / boundary split: the interior rows need no halo column, so they run
        // while the halo travels on the comm stream; the boundary rows (both ends of the
        // block) follow once it has arrived.  Every row is computed whole by one launch:
        // rows stay bit-identical; a fused dot folds both launches' partials in order.
        const bool red = dotw != nullptr || fin != FIN_NONE;
        TRY(exchange_begin(h, M, const_cast<double *>(x)));
        SpmvArgs ai = a;
        ai.rlo = (int)M.int_lo;
        ai.pmode = red ? 1 : 0;
        int gi = 0;
        TRY(spmv_range(h, M, lay, ai, epi, (int)(M.int_hi - M.int_lo), grid_cap, &gi));
        TRY(exchange_end(h, M));
        SpmvArgs ab = a;
        ab.rlo = 0;
        ab.rsplit = (int)M.int_lo;
        ab.rgap = (int)(M.int_hi - M.int_lo);
        ab.pmode = red ? 2 : 0;
        ab.pbase = gi;
        TRY(spmv_range(h, M, lay, ab, epi, (int)(M.nrows - (M.int_hi - M.int_lo)), grid_cap, nullptr));
        TRY(post_fin(h, ufin, g1));
        return AMG_OK;
    }
    TRY(exchange(h, M, const_cast<double *>(x)));
    if (M.dcls) {
        DictArgs da{M.dcls, M.dbeg, M.drel, M.dval, M.dncls, M.dnent, h->dict_main ? M.dmcls : -1, M.dmlen};
        for (int k = 0; k < 8; ++k) {
            da.mrel[k] = M.dmrel[k];
            da.moff[k] = (long long)M.dmrel[k] * 8;
            da.mval[k] = M.dmval[k];
        }
        const int dg = grid_cap ? std::min(grid_cap, M.dgrid) : M.dgrid;
        const size_t sm = (size_t)M.dnent * 12 + (size_t)(M.dncls + 1) * 4;
        TRY(launch_k(h, spmv_dict_fn(epi, M.dfl, M.dwide, (h->dict_main && M.dmcls >= 0) ? M.dmlen : 0), dg, VEC_SPMV_THREADS, sm, a, da, (int)M.nrows));
    } else if (M.uval && h->symm) {
        const bool fx = M.sym_fl && (h->symd_fixed >= 2 || (h->symd_fixed == 1 && M.sym_fl <= 8));
        int g = fx ? M.symf_grid : M.sym_grid;
        if (grid_cap) g = std::min(g, grid_cap);
        // contiguous row chunks per CTA (multiples of 256 rows) when the grid covers the matrix in >= 2 steps
        int chunk = 0;
        if (h->symd_chunked) {
            const int64_t c = ((M.nrows + g - 1) / g + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS * VEC_SPMV_THREADS;
            if (c >= 2 * VEC_SPMV_THREADS) {
                chunk = (int)c;
                g = (int)((M.nrows + c - 1) / c);
            }
        }
        SymArgs sa{M.uval, M.pid, M.sym_slot, chunk, M.sym_blocked ? 32 * M.nudiag : 0, M.sym_npad,
                   M.sym_tab, M.sym_ntab, M.npat};
        const bool tsm = h->symd_tsm && M.sym_blocked && !fx;
        const size_t tsm_bytes = tsm ? (size_t)M.sym_ntab * sizeof(int2) + (size_t)(M.npat + 1) * sizeof(int32_t) : 0;
        if (!fx && M.sym_fast_on && h->symd_fast && !tsm) {
            int g27 = M.sym27_grid;
            if (grid_cap) g27 = std::min(g27, grid_cap);
            SymArgs sb = sa;
            sb.chunk = 0;
            TRY(launch_k(h, spmv_symd27_fn(epi), g27, VEC_SPMV_THREADS, 0, a, sb, M.sym_fast, (int)M.nrows));
        } else if (fx)
            TRY(launch_k(h, spmv_symd_fixed_fn(epi, M.sym_fl, h->symd_minb, M.sym_blocked), g, VEC_SPMV_THREADS, 0, a, sa, (int)M.nrows));
        else
            TRY(launch_k(h, spmv_symd_fn(epi, h->symd_gminb, M.sym_blocked, tsm), g, VEC_SPMV_THREADS, tsm_bytes, a, sa,
                         (int)M.nrows));
    } else if (M.sv_s && h->sells) {
        SellSArgs qa{M.sv_s, M.sc_s, M.sb_s, M.sw_s, M.sp_s, M.sl_s, (int)M.nrows};
        TRY(launch_k(h, spmv_sells_fn(epi, h->sells_plen), grid_cap ? std::min(grid_cap, M.s_grid) : M.s_grid, VEC_SPMV_THREADS, 0, a,
                     qa, (int)M.nrows));
    } else if (M.uval_s && h->sellu) {
        SellUArgs ua{M.uval_s, M.ucol_s, M.ulen_s, M.uW, M.uperm_s, M.ucls_s, M.uvtab, M.uvlen, M.uncls, M.uvid_s};
        TRY(launch_k(h, spmv_sellu_fn(epi, M.uW, M.u_plen, sellu_vd_mode(M)), grid_cap ? std::min(grid_cap, M.u_grid) : M.u_grid, VEC_SPMV_THREADS, sellu_vd_bytes(M),
                     a, ua, (int)M.nrows));
    } else if (M.sbeg) {
        SellArgs sa{M.sbeg, M.sval, M.scol, M.slen, M.pid, M.prel, M.pbeg, M.npat, M.nrel, M.sperm};
        TRY(launch_k(h, spmv_sell_fn(epi, M.scol == nullptr), grid_cap ? std::min(grid_cap, M.sell_grid) : M.sell_grid,
                     VEC_SPMV_THREADS, 0, a, sa, (int)M.nrows));
    } else if (M.pid && M.pstart) {
        PatArgs pa{M.pstart, M.pval, M.pid, M.prel, M.pbeg, M.npat, M.nrel};
        TRY(launch_k(h, spmv_pat_fn(epi), grid_cap ? std::min(grid_cap, M.pad_grid) : M.pad_grid, VEC_SPMV_THREADS, 0, a,
                     pa, (int)M.nrows));
    } else if (M.leaf) {
        LeafArgs la{M.leaf, M.nleaves, M.lsum, M.row_leaf};
        SpmvArgs a1 = a;  // leaf pass: no reduction
        a1.dotw = nullptr;
        a1.fin = FIN_NONE;
        TRY(launch_k(h, spmv_leaves, grid_cap ? std::min(grid_cap, M.leaf_grid) : M.leaf_grid, DIRECT_THREADS, 0, a1, la));
        TRY(launch_k(h, spmv_leafsum_fn(epi), grid_cap ? std::min(grid_cap, M.leafsum_grid) : M.leafsum_grid,
                     DIRECT_THREADS, 0, a, la, (int)M.nrows));
    } else if (M.wcsr) {
        TRY(launch_k(h, spmv_wcsr_fn(epi), grid_cap ? std::min(grid_cap, M.wcsr_grid) : M.wcsr_grid, WCSR_THREADS, 0, a,
                     (int)M.nrows));
    } else if (M.pstart) {
        PadArgs pa{M.pstart, M.pval, M.pcol};
        TRY(launch_k(h, spmv_vec_fn(epi, h->vec_minb), grid_cap ? std::min(grid_cap, M.pad_grid) : M.pad_grid, VEC_SPMV_THREADS, 0, a,
                     pa, (int)M.nrows));
    } else {
        const int gpr = DIRECT_THREADS / M.lanes;  // row groups per CTA
        int g = (int)std::min<int64_t>((M.nrows + gpr - 1) / gpr, (int64_t)h->sm_count * h->direct_per_sm);
        if (grid_cap) g = std::min(g, grid_cap);
        TRY(launch_k(h, spmv_direct_fn(epi, M.lanes), std::max(g, 1), DIRECT_THREADS, 0, a, (int)M.nrows));
    }
    TRY(post_fin(h, ufin, g1));
    return AMG_OK;
}

static int vec_grid(const amg_t *h, int64_t n)
{
    int64_t g = (n + VEC_THREADS * 4 - 1) / (VEC_THREADS * 4);
    g = std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)h->sm_count * (h->vec_per_sm > 0 ? h->vec_per_sm : 8)));
    return (int)g;
}

static VecArgs vargs(amg_t *h, int64_t n, const int *g1, const int *g2)
{
    VecArgs v{};
    v.n = n;
    v.partials = h->partials;
    v.ticket = h->ticket;
    v.ctl = h->ctl;
    v.gate1 = g1;
    v.gate2 = g2;
    v.fin = FIN_NONE;
    return v;
}

static int launch_copy(amg_t *h, double *dst, const double *src, int64_t n, const int *g1)
{
    VecArgs v = vargs(h, n, g1, nullptr);
    v.x = dst;
    v.p = src;
    TRY(launch_k(h, vec_copy, vec_grid(h, n), VEC_THREADS, 0, v));
    return AMG_OK;
}

static int launch_dot(amg_t *h, const double *a, const double *b, int64_t n, int fin, const int *g1, const int *g2)
{
    VecArgs v = vargs(h, n, g1, g2);
    v.p = a;
    v.q = b;
    v.fin = kfin(h, fin);
    TRY(launch_k(h, vec_dot, vec_grid(h, n), VEC_THREADS, 0, v));
    TRY(post_fin(h, fin, g1));
    return AMG_OK;
}

static CoarseArgs coarse_args(const amg_t *h)
{
    CoarseArgs c{};
    c.n = h->nc;
    c.kind = h->coarse_kind == AMG_COARSE_CHOLESKY ? 0 : 1;
    c.staged = h->coarse_staged;
    c.Lp = h->Lp;
    c.mn = h->binv;
    c.dinv = h->dinv;
    c.LU = h->LU;
    c.piv = h->piv;
    c.prefetch = h->tail_prefetch;
    c.pipe = h->coarse_pipe;
    return c;
}

static int launch_coarse(amg_t *h, const double *y, double *z, const int *g1, int fin, const double *dotw)
{
    if (h->collect) {
        if (dotw || fin != FIN_NONE) return fail(AMG_E_STATE, "internal: reduction inside the cluster tail");
        TailOp o{};
        o.kind = TAIL_COARSE;
        o.nrows = h->nc;
        o.x = y;
        o.y = z;
        h->collect->push_back(o);
        return AMG_OK;
    }
    TRY(launch_k(h, coarse_solve_k, 1, COARSE_THREADS, h->coarse_smem, coarse_args(h), y, z, g1, h->partials,
                 h->ticket, fin, h->ctl, dotw));
    return AMG_OK;
}

static int launch_tail(amg_t *h, const int *g1)
{
    if (h->pf_pending) {  // the side-stream prefetch joins before the tail
        CK(cudaEventRecord(h->pf_join, h->side));
        CK(cudaStreamWaitEvent(h->stream, h->pf_join, 0));
        h->pf_pending = false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)h->cluster);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.dynamicSmemBytes = h->tail_smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[2];
    if (h->tail_grid) {  // every CTA co-resident: grid barriers inside
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    } else {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)h->cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    }
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = h->pdl ? 2 : 1;
    const TailVecs tv{h->tail_vecs, h->tail_nvecs, h->tail_pcap_used};
    cudaError_t e = cudaLaunchKernelEx(&cfg, tail_vcycle, (const TailOp *)h->tail_ops, h->tail_nops,
                                       (const TailMat *)h->tail_mats, h->tail_nmats, (const int32_t *)h->tail_splits,
                                       h->tail_prod_off, coarse_args(h), g1, h->trace, tv,
                                       h->tail_grid ? h->tail_gbar : (unsigned *)nullptr);
    if (e != cudaSuccess) return fail(AMG_E_CUDA, std::string("tail launch failed: ") + cudaGetErrorString(e));
    ++h->launches;
    return AMG_OK;
}

// x = apply_smoother(level k, b, x, steps) with x == 0 on entry when `from_zero`.
// The LAST operation carries (fin, dotw) when `tail` is set.
static int enqueue_smooth(amg_t *h, int k, const double *b, double *x, int steps, bool from_zero, const int *g1,
                          int fin, const double *dotw)
{
    LevelD &L = h->lv[k];
    for (int s = 0; s < steps; ++s) {
        const bool last = (s == steps - 1);
        const int f = last ? fin : FIN_NONE;
        const double *dw = last ? dotw : nullptr;
        const double *src = b;  // b - A*0 == b exactly (smoothers.py:172 with x0 = 0)
        if (!(from_zero && s == 0)) {
            TRY(launch_spmv(h, L.m[AMG_A], x, L.r, EPI_RESID, b, 0.0, nullptr, FIN_NONE, g1, nullptr));
            src = L.r;
        }
        const bool set = from_zero && s == 0;
        if (L.sm_kind == AMG_SMOOTHER_FSAI) {
            TRY(launch_spmv(h, L.m[AMG_G], src, L.t, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, g1, nullptr));
            TRY(launch_spmv(h, L.m[AMG_GT], L.t, x, set ? EPI_SETW : EPI_AXPYW, x, L.omega, dw, f, g1, nullptr));
        } else if (h->collect) {
            if (dw) return fail(AMG_E_STATE, "internal: reduction inside the cluster tail");
            TailOp o{};
            o.kind = TAIL_JACOBI;
            o.nrows = (int)L.n;
            o.mode = set ? 0 : 1;
            o.x = src;
            o.y = x;
            o.d = L.inv_diag;
            o.omega = L.omega;
            h->collect->push_back(o);
        } else {
            VecArgs v = vargs(h, L.n, g1, nullptr);
            v.x = x;
            v.p = src;
            v.d = L.inv_diag;
            v.omega = L.omega;
            v.mode = set ? 0 : 1;
            v.q = dw;
            v.fin = dw ? kfin(h, f) : FIN_NONE;
            TRY(launch_k(h, jacobi_sweep, vec_grid(h, L.n), VEC_THREADS, 0, v));
            if (dw) TRY(post_fin(h, f, g1));
        }
    }
    return AMG_OK;
}

// x = vcycle(h, y, level k) (hierarchy.py:294-312).  (fin, dotw) ride on the
// last operation of level 0 (e.g. r.z for PCG).
static int enqueue_vcycle(amg_t *h, int k, const double *y, double *x, const int *g1, int fin, const double *dotw)
{
    const int nl = (int)h->lv.size();
    if (!h->collect && h->tail_level > 0 && k == h->tail_level) return launch_tail(h, g1);
    if (k == nl - 1) return launch_coarse(h, y, x, g1, fin, dotw);
    LevelD &L = h->lv[k];
    LevelD &C = h->lv[k + 1];
    if (!h->collect && h->side_prefetch && h->pf_n > 0 && h->tail_level > 0 && k == h->tail_level - 1) {
        CK(cudaEventRecord(h->pf_fork, h->stream));
        CK(cudaStreamWaitEvent(h->side, h->pf_fork, 0));
        l2_prefetch<<<2 * h->sm_count, 256, 0, h->side>>>(h->pf_ranges, h->pf_n);
        CK(cudaGetLastError());
        ++h->launches;
        h->pf_pending = true;
    }
    const double *r = y;
    if (h->nu1 > 0) {
        TRY(enqueue_smooth(h, k, y, x, h->nu1, true, g1, FIN_NONE, nullptr));
        TRY(launch_spmv(h, L.m[AMG_A], x, L.r, EPI_RESID, y, 0.0, nullptr, FIN_NONE, g1, nullptr));
        r = L.r;
    }
    const bool agglom = h->nranks > 1 && (k + 1) == h->agglom_level;
    double *yc = agglom ? C.y + C.starts[h->rank] : C.y;  // this rank's piece of the replicated level
    TRY(launch_spmv(h, L.m[AMG_PT], r, yc, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, g1, nullptr));
    if (agglom) TRY(allgather_level(h, k + 1, C.y));
    TRY(enqueue_vcycle(h, k + 1, C.y, C.x, g1, FIN_NONE, nullptr));
    const bool tail_on_p = (h->nu2 == 0);
    TRY(launch_spmv(h, L.m[AMG_P], C.x, x, h->nu1 > 0 ? EPI_ADD : EPI_PLAIN, x, 0.0, tail_on_p ? dotw : nullptr,
                    tail_on_p ? fin : FIN_NONE, g1, nullptr));
    if (h->nu2 > 0) TRY(enqueue_smooth(h, k, y, x, h->nu2, false, g1, fin, dotw));
    return AMG_OK;
}

// One PCG iteration (krylov.py:66-91), every kernel gated on ctl->active.
static int enqueue_pcg_body(amg_t *h, cudaGraphConditionalHandle handle, int use_handle)
{
    LevelD &L0 = h->lv[0];
    const DevMat &A = L0.m[AMG_A];
    const int *act = &h->ctl->active;
    const int64_t n = L0.n;
    // q = A p ; curv = p.q ; alpha = rz / curv          (:66-73)
    TRY(launch_spmv(h, A, h->p, h->q, EPI_PLAIN, nullptr, 0.0, h->p, FIN_CURV, act, nullptr));
    // x += alpha p ; r -= alpha q ; ||r||               (:74-75, 78)
    {
        VecArgs v = vargs(h, n, act, nullptr);
        v.x = h->x;
        v.r = h->r;
        v.p = h->p;
        v.q = h->q;
        v.fin = kfin(h, FIN_UPDATE);
        TRY(launch_k(h, pcg_update, vec_grid(h, n), VEC_THREADS, 0, v));
        TRY(post_fin(h, FIN_UPDATE, act));
    }
    // every recompute_every iterations: r = b - A x     (:76-77)
    // (rarely active: launched one CTA per SM so the usual no-op costs little)
    const int gcap = h->gated_grid > 0 ? h->gated_grid * h->sm_count : 0;
    TRY(launch_spmv(h, A, h->x, h->r, EPI_RESID, h->b, 0.0, h->r, FIN_RECOMPUTE, act, &h->ctl->do_recompute, gcap));
    // relres <= rtol: true residual check              (:81-86)
    TRY(launch_spmv(h, A, h->x, h->r, EPI_RESID, h->b, 0.0, h->r, FIN_TRUE, act, &h->ctl->need_true, gcap));
    // z = M r ; rz_new = r.z ; beta                     (:87-90)
    if (h->rz_sep) {  // r.z as its own fixed-order dot after the V-cycle
        TRY(enqueue_vcycle(h, 0, h->r, h->z, act, FIN_NONE, nullptr));
        TRY(launch_dot(h, h->r, h->z, n, FIN_RZ, act, nullptr));
    } else {
        TRY(enqueue_vcycle(h, 0, h->r, h->z, act, FIN_RZ, h->r));
    }
    if (h->lv.size() == 1) {
        // the coarse kernel carried the dot already
    }
    // p = z + beta p                                    (:91)
    {
        VecArgs v = vargs(h, n, act, nullptr);
        v.x = h->p;
        v.p = h->z;
        TRY(launch_k(h, pcg_xpay, vec_grid(h, n), VEC_THREADS, 0, v));
    }
    TRY(launch_k(h, pcg_continue, 1, 1, 0, h->ctl, handle, use_handle));
    return AMG_OK;
}

static int build_graph(amg_t *h)
{
    if (h->gexec) return AMG_OK;
    const int64_t before = h->launches;
    int mode = (h->force_graph >= 0) ? h->force_graph : 2;
    if (mode == 2) {
        cudaGraph_t g = nullptr;
        cudaGraphConditionalHandle handle;
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess &&
                  cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
        cudaGraphNode_t node;
        cudaGraphNodeParams params = {cudaGraphNodeTypeConditional};
        if (ok) {
            params.conditional.handle = handle;
            params.conditional.type = cudaGraphCondTypeWhile;
            params.conditional.size = 1;
            ok = cudaGraphAddNode(&node, g, nullptr, 0, &params) == cudaSuccess;
        }
        if (ok) {
            cudaGraph_t body = params.conditional.phGraph_out[0];
            ok = cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                int s = enqueue_pcg_body(h, handle, 1);
                cudaGraph_t out = nullptr;
                cudaError_t e = cudaStreamEndCapture(h->stream, &out);
                ok = (s == AMG_OK) && e == cudaSuccess;
                if (!ok && getenv("AMGB200_DEBUG"))
                    fprintf(stderr, "amgb200: while-body capture failed: %s / %s\n", cudaGetErrorString(e),
                            s == AMG_OK ? "" : g_err.c_str());
            }
        }
        if (ok) {
            cudaError_t e = cudaGraphInstantiate(&h->gexec, g, 0);
            ok = e == cudaSuccess;
            if (!ok && getenv("AMGB200_DEBUG"))
                fprintf(stderr, "amgb200: while-graph instantiate failed: %s\n", cudaGetErrorString(e));
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        if (ok) {
            h->graph_mode = 2;
            h->launches_per_iter = h->launches - before;
            h->launches = before;
            return AMG_OK;
        }
        if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
        h->launches = before;
        mode = 1;
    }
    if (mode == 1) {
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        cudaGraphConditionalHandle dummy{};
        int s = enqueue_pcg_body(h, dummy, 0);
        cudaError_t e = cudaStreamEndCapture(h->stream, &g);
        if (s != AMG_OK) return s;
        if (e == cudaSuccess) {
            e = cudaGraphInstantiate(&h->gexec, g, 0);
            cudaGraphDestroy(g);
        }
        if (e != cudaSuccess) {  // e.g. a collective that cannot be captured here: launch eagerly
            cudaGetLastError();
            if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
            h->launches = before;
            h->graph_mode = 0;
            return AMG_OK;
        }
        h->graph_mode = 1;
        h->launches_per_iter = h->launches - before;
        h->launches = before;
        return AMG_OK;
    }
    h->graph_mode = 0;
    return AMG_OK;
}

// Choose the first level (>= 1) whose operator has at most tail_nnz stored
// entries (and every deeper level too), collect the ops of the V-cycle from
// there down, and upload them for the cluster tail kernel.
static int build_tail(amg_t *h)
{
    const int nl = (int)h->lv.size();
    h->tail_level = 0;
    if (h->tail_nnz <= 0 || nl < 2) return AMG_OK;
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    // CTA 0 of the tail stages v, tmp, 1/L_ii and the packed factor (not the pre-scaled blocks)
    const size_t coarse_bytes = (h->coarse_kind == AMG_COARSE_CHOLESKY && h->coarse_staged)
                                    ? (size_t)(2 * ((h->nc + 1) & ~1) + 32 + (int64_t)h->nc * (h->nc + 1) / 2) * sizeof(double)
                                    : (size_t)(((h->nc + 1) & ~1) + 32) * sizeof(double);
    const int budget = optin - (int)(TAIL_MAX_OPS * sizeof(TailOp) + TAIL_MAX_MATS * 5 * sizeof(int)) - 1024;  // static smem + slack
    // start level: the shallowest level (>= 1) from which every A_k has at most
    // tail_nnz entries; matrices are staged in smem coarsest-first while the
    // budget lasts, the rest are streamed from L2 inside their op
    int best = 0;
    std::vector<TailOp> best_ops;
    std::vector<TailMat> best_mats;
    std::vector<int32_t> best_splits;
    int best_prod_off = 0, best_smem = 0;
    int kstart = 0;
    for (int kt = nl - 1; kt >= 1; --kt) {
        if (h->lv[kt].m[AMG_A].nnz > h->tail_nnz) break;
        kstart = kt;
    }
    // multi-GPU: the tail holds replicated levels only (every rank runs the same
    // tail on its own full copy; no halo or collective inside the cluster kernel)
    if (h->nranks > 1) {
        if (h->agglom_level < 1 || kstart == 0) return AMG_OK;
        kstart = std::max(kstart, h->agglom_level);
        if (kstart >= nl) return AMG_OK;
    }
    for (int kt = kstart; kt >= 1 && kt < nl && best == 0; ++kt) {
        std::vector<TailOp> ops;
        std::vector<const DevMat *> mats_raw;
        h->collect = &ops;
        h->collect_mats = &mats_raw;
        int st = enqueue_vcycle(h, kt, h->lv[kt].y, h->lv[kt].x, nullptr, FIN_NONE, nullptr);
        h->collect = nullptr;
        h->collect_mats = nullptr;
        if (st != AMG_OK) return st;
        if ((int)ops.size() > TAIL_MAX_OPS) continue;
        std::vector<const DevMat *> uniq;
        std::vector<TailMat> mats;
        std::vector<int32_t> splits;
        std::vector<int> mat_level;
        int prod_cap = 0;
        int longest_row = 1;  // a streamed chunk holds at least one whole row
        for (auto &o : ops) {
            if (o.kind != TAIL_SPMV) continue;
            const DevMat *M = mats_raw[o.mode];
            o.mode = 0;
            int idx = -1;
            for (size_t u = 0; u < uniq.size(); ++u)
                if (uniq[u] == M) idx = (int)u;
            if (idx < 0) {
                std::vector<int32_t> off(M->nrows + 1);
                CK(cudaMemcpy(off.data(), M->off, (M->nrows + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
                TailMat T{};
                T.off = M->off;
                T.col = M->col;
                T.val = M->val;
                T.split = (int)splits.size();
                const int64_t nnz = off[M->nrows];
                for (int64_t q = 0; q < M->nrows; ++q) longest_row = std::max(longest_row, off[q + 1] - off[q]);
                // CTA 0 runs the coarsest solve and owns no SpMV rows; rows are
                // balanced by stored entries over CTAs 1..cluster-1
                const int workers = std::max(1, h->cluster - 1);
                int r = 0;
                splits.push_back(0);
                if (h->cluster > 1) splits.push_back(0);
                for (int c = 1; c < workers; ++c) {
                    const int64_t target = nnz * c / workers;
                    while (r < M->nrows && off[r] < target) ++r;
                    splits.push_back(r);
                }
                splits.push_back((int32_t)M->nrows);
                int rc = 0, kc = 0;
                for (int c = 0; c < h->cluster; ++c) {
                    rc = std::max(rc, splits[T.split + c + 1] - splits[T.split + c]);
                    kc = std::max(kc, off[splits[T.split + c + 1]] - off[splits[T.split + c]]);
                }
                T.rows_cap = rc;
                T.nnz_cap = kc;
                prod_cap = std::max(prod_cap, kc);
                idx = (int)uniq.size();
                uniq.push_back(M);
                mats.push_back(T);
                int lvl = 0;
                for (int k = 0; k < nl; ++k)
                    for (int w = 0; w < 5; ++w)
                        if (&h->lv[k].m[w] == M) lvl = k;
                mat_level.push_back(lvl);
            }
            o.mat = idx;
        }
        if ((int)mats.size() > TAIL_MAX_MATS) continue;
        // smem: CTA 0 = coarse area; CTAs >= 1 = [staged regions ...][products] (overlaid)
        const size_t base = (h->cluster > 1) ? 0 : ((coarse_bytes + 15) & ~(size_t)15);
        if (!h->tail_stage) prod_cap = std::min(prod_cap, h->tail_pcap);  // streamed SpMVs run in chunks
        prod_cap = std::max(prod_cap, longest_row);  // ... of whole rows: the chunk search assumes one row fits
        const size_t prod_bytes = (size_t)prod_cap * 8 + 16;
        if (base + prod_bytes > (size_t)budget || coarse_bytes > (size_t)budget) continue;
        std::vector<int> order(mats.size());
        for (size_t u = 0; u < order.size(); ++u) order[u] = (int)u;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return mat_level[a] > mat_level[b]; });
        size_t off_bytes = base;
        for (int u : order) {
            const size_t rb = tail_region_bytes(mats[u].rows_cap, mats[u].nnz_cap);
            if (h->tail_stage && off_bytes + rb + prod_bytes <= (size_t)budget) {
                mats[u].staged = 1;
                mats[u].smem_off = (int)off_bytes;
                off_bytes += rb;
            } else {
                mats[u].staged = 0;
                mats[u].smem_off = 0;
            }
        }
        const size_t prod_off = (off_bytes + 15) & ~(size_t)15;
        best = kt;
        best_ops = ops;
        best_mats = mats;
        best_splits = splits;
        best_prod_off = (int)prod_off;
        best_smem = (int)std::max(prod_off + prod_bytes, coarse_bytes);
        h->tail_pcap_used = prod_cap;
    }
    if (best == 0) return AMG_OK;
    TRY(raise_smem_caps(h->device));
    int nclusters = 0;
    if (h->tail_grid) {
        int nb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)tail_vcycle, TAIL_THREADS, best_smem));
        nclusters = (int64_t)nb * h->sm_count >= h->cluster ? 1 : 0;  // the whole grid co-resident
        if (nclusters) TRY(dalloc(&h->tail_gbar, 2));
        if (nclusters) CK(cudaMemset(h->tail_gbar, 0, 2 * sizeof(unsigned)));
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)h->cluster);
        cfg.blockDim = dim3(TAIL_THREADS);
        cfg.dynamicSmemBytes = best_smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)h->cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, (const void *)tail_vcycle, &cfg);
        if (e != cudaSuccess) { cudaGetLastError(); nclusters = 0; }
    }
    if (nclusters < 1) return AMG_OK;  // cluster shape not resident here: per-op kernels are used
    for (auto &o : best_ops) o.xs = o.ys = o.bs = -1;
    if (h->tail_dsm && !h->tail_grid) {
        // level vectors below the tail's entry / exit (y, x of its first level stay in global memory)
        struct V { const double *p; int shift; int off; };
        std::vector<V> vs;
        size_t off = ((size_t)best_smem + 15) & ~(size_t)15;
        auto add = [&](const double *p, int64_t n) {
            int64_t r = (n + h->cluster - 1) / h->cluster, sh = 0;
            while ((int64_t(1) << sh) < r) ++sh;
            vs.push_back({p, (int)sh, (int)off});
            off += ((size_t)8 << sh);
        };
        for (int k = best; k < nl; ++k) {
            LevelD &L = h->lv[k];
            if (k > best) {
                add(L.y, L.n);
                add(L.x, L.n);
            }
            add(L.r, L.n);
            add(L.t, L.n);
        }
        if ((int)vs.size() <= TAIL_MAX_VECS && off <= (size_t)(optin - 64 * 1024 / 8)) {
            auto slot = [&](const double *p) {
                for (size_t q = 0; q < vs.size(); ++q)
                    if (vs[q].p == p) return (int)q;
                return -1;
            };
            for (auto &o : best_ops) {
                o.xs = o.x ? slot(o.x) : -1;
                o.ys = o.y ? slot(o.y) : -1;
                o.bs = o.b ? slot(o.b) : -1;
            }
            std::vector<int2> tab(vs.size());
            for (size_t q = 0; q < vs.size(); ++q) tab[q] = make_int2(vs[q].shift, vs[q].off);
            TRY(dalloc(&h->tail_vecs, tab.size()));
            CK(cudaMemcpy(h->tail_vecs, tab.data(), tab.size() * sizeof(int2), cudaMemcpyHostToDevice));
            h->tail_nvecs = (int)tab.size();
            best_smem = (int)off;
        }
    }
    TRY(dalloc(&h->tail_ops, best_ops.size()));
    CK(cudaMemcpy(h->tail_ops, best_ops.data(), best_ops.size() * sizeof(TailOp), cudaMemcpyHostToDevice));
    TRY(dalloc(&h->tail_mats, best_mats.size()));
    if (!best_mats.empty()) CK(cudaMemcpy(h->tail_mats, best_mats.data(), best_mats.size() * sizeof(TailMat), cudaMemcpyHostToDevice));
    TRY(dalloc(&h->tail_splits, best_splits.size()));
    if (!best_splits.empty()) CK(cudaMemcpy(h->tail_splits, best_splits.data(), best_splits.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    h->tail_nops = (int)best_ops.size();
    h->tail_nmats = (int)best_mats.size();
    h->tail_smem = best_smem;
    h->tail_prod_off = best_prod_off;
    h->tail_level = best;
    if (getenv("AMGB200_TRACE")) TRY(dalloc(&h->trace, (size_t)h->tail_nops + 2));
    {   // L2 prefetch ranges for the side stream: every CSR array of the tail levels + the coarse factor
        std::vector<PrefetchRange> pr;
        for (int k = best; k < nl; ++k)
            for (int w = 0; w < 5; ++w) {
                const DevMat &M = h->lv[k].m[w];
                if (!M.present || M.nnz == 0) continue;
                pr.push_back({reinterpret_cast<const char *>(M.off), (long long)(M.nrows + 1) * 4});
                pr.push_back({reinterpret_cast<const char *>(M.col), (long long)M.nnz * 4});
                pr.push_back({reinterpret_cast<const char *>(M.val), (long long)M.nnz * 8});
            }
        if (h->Lp) pr.push_back({reinterpret_cast<const char *>(h->Lp), (long long)h->nc * (h->nc + 1) / 2 * 8});
        TRY(dalloc(&h->pf_ranges, pr.size()));
        if (!pr.empty()) CK(cudaMemcpy(h->pf_ranges, pr.data(), pr.size() * sizeof(PrefetchRange), cudaMemcpyHostToDevice));
        h->pf_n = (int)pr.size();
    }
    return AMG_OK;
}

// ------------------------------------------------------------------ C ABI

extern "C" {

int amg_get_version(void) { return 1; }

const char *amg_last_error(void) { return g_err.c_str(); }

int amg_create(int device, int rank, int nranks, const void *nccl_unique_id, amg_t **out)
{
    if (!out) return fail(AMG_E_ARG, "amg_create: out is NULL");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(AMG_E_ARG, "amg_create: bad rank / nranks");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(AMG_E_CUDA, std::string("amg_create: no CUDA device available (") + cudaGetErrorString(e) +
                                    "); amgb200 has no CPU fallback");
    if (device < 0 || device >= ndev) return fail(AMG_E_ARG, "amg_create: device ordinal out of range");
    CK(cudaSetDevice(device));
    amg_t *h = new amg_t();
    h->device = device;
    h->rank = rank;
    h->nranks = nranks;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    h->sm_count = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->pf_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->pf_join, cudaEventDisableTiming));
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    if (nranks > 1) {
        if (!nccl_unique_id) { delete h; return fail(AMG_E_ARG, "amg_create: nranks > 1 needs an ncclUniqueId"); }
        if (comm_init(h->comm, nccl_unique_id, rank, nranks) != 0) {
            std::string m = halo_error();
            delete h;
            return fail(AMG_E_NCCL, "amg_create: " + m);
        }
    }
    *out = h;
    return AMG_OK;
}

void amg_destroy(amg_t *h)
{
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    auto F = [](void *p) {
        if (!p) return;
        cudaFree(p);
        std::lock_guard<std::mutex> g(g_alloc_mu);
        g_alloc_size.erase(p);
    };
    for (auto &L : h->lv) {
        for (auto &M : L.m) {
            F(M.off); F(M.col); F(M.val); F(M.pstart); F(M.pval); F(M.pcol); F(M.pid); F(M.prel); F(M.pbeg); F(M.sbeg); F(M.sval); F(M.scol); F(M.slen); F(M.sperm); F(M.leaf); F(M.row_leaf); F(M.lsum); F(M.uval); F(M.uval_s); F(M.ucol_s); F(M.ulen_s); F(M.uperm_s); F(M.ucls_s); F(M.uvtab); F(M.uvlen); F(M.uvid_s); F(M.sv_s); F(M.sc_s); F(M.sb_s); F(M.sp_s); F(M.sw_s); F(M.sl_s); F(M.dcls); F(M.dbeg); F(M.drel); F(M.dval);
            symd_slot_give(h->device, M.sym_slot);
            M.sym_slot = -1;
            symd_tab_give(h->device, M.sym_tab, M.sym_ntab);
            M.sym_tab = -1;
            halo_free(M.halo);
        }
        F(L.inv_diag); F(L.y); F(L.x); F(L.r); F(L.t);
    }
    F(h->pf_ranges);
    F(h->selftest_buf);
    F(h->tail_gbar);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->ev_pack) cudaEventDestroy(h->ev_pack);
    if (h->ev_halo) cudaEventDestroy(h->ev_halo);
    if (h->pf_fork) cudaEventDestroy(h->pf_fork);
    if (h->pf_join) cudaEventDestroy(h->pf_join);
    F(h->Lp); F(h->LU); F(h->dinv); F(h->binv); F(h->tail_ops); F(h->tail_mats); F(h->tail_vecs); F(h->tail_splits); F(h->piv); F(h->partials); F(h->ticket); F(h->ctl);
    F(h->b); F(h->x); F(h->r); F(h->z); F(h->p); F(h->q); F(h->tmp_in); F(h->tmp_out); F(h->hist);
    for (auto *bp : h->bicg) F(bp);
    if (h->ctl_h) cudaFreeHost(h->ctl_h);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    comm_destroy(h->comm);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

int amg_set_option(amg_t *h, const char *key, int64_t value)
{
    if (!h || !key) return fail(AMG_E_ARG, "amg_set_option: NULL argument");
    std::string k(key);
    if (k == "graph") { h->force_graph = (int)value; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "batch") { h->batch = std::max<int>(1, (int)value); return AMG_OK; }
    if (k == "pdl") { h->pdl = value ? 1 : 0; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (h->finalized) return fail(AMG_E_STATE, "amg_set_option: '" + k + "' must be set before amg_finalize");
    if (k == "tail_nnz") { h->tail_nnz = value; return AMG_OK; }
    if (k == "tail_stage") { h->tail_stage = value ? 1 : 0; return AMG_OK; }
    if (k == "tail_grid") { h->tail_grid = value ? 1 : 0; return AMG_OK; }
    if (k == "cluster") { if (value != 8 && value != 16 && value != 4 && value != 2 && value != 1) return fail(AMG_E_ARG, "cluster must be 1,2,4,8,16"); h->cluster = (int)value; return AMG_OK; }
    if (k == "pad_min") { h->pad_min = (int)value; return AMG_OK; }
    if (k == "long_avg") { h->long_avg = (int)value; return AMG_OK; }
    if (k == "small_rows_per_sm") { h->small_rows_per_sm = (int)value; return AMG_OK; }
    if (k == "patterns") { h->patterns = value ? 1 : 0; return AMG_OK; }
    if (k == "symm") { h->symm = value ? 1 : 0; return AMG_OK; }
    if (k == "dict") { h->dict = value ? 1 : 0; return AMG_OK; }
    if (k == "symd_fast") { h->symd_fast = value ? 1 : 0; return AMG_OK; }
    if (k == "dict_main") { h->dict_main = value ? 1 : 0; return AMG_OK; }
    if (k == "wcsr") { h->wcsr = value ? 1 : 0; return AMG_OK; }
    if (k == "overlap_test") { h->overlap_test = value ? 1 : 0; return AMG_OK; }
    if (k == "nccl_selftest") { h->nccl_selftest = (int)value; return AMG_OK; }
    if (k == "sells") { h->sells = (int)value; return AMG_OK; }
    if (k == "sells_max_rows") { h->sells_max_rows = value; return AMG_OK; }
    if (k == "sells_buckets") { h->sells_buckets = (int)value; return AMG_OK; }
    if (k == "sells_plen") { h->sells_plen = value ? 1 : 0; return AMG_OK; }
    if (k == "sells_max_pad") { h->sells_max_pad = (int)value; return AMG_OK; }
    if (k == "sells_sigma") { h->sells_sigma = (int)value; return AMG_OK; }
    if (k == "sells_min_avg10") { h->sells_min_avg = value / 10.0; return AMG_OK; }
    if (k == "rz_sep") { h->rz_sep = value ? 1 : 0; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "vec_minb") { h->vec_minb = (int)value; return AMG_OK; }
    if (k == "sellu_short") { h->sellu_short = value ? 1 : 0; return AMG_OK; }
    if (k == "sellu") { h->sellu = value ? 1 : 0; return AMG_OK; }
    if (k == "sellu_vdict") { h->sellu_vdict = value ? 1 : 0; return AMG_OK; }
    if (k == "sellu_sort") { h->sellu_sort = value ? 1 : 0; return AMG_OK; }
    if (k == "symd_fixed") { h->symd_fixed = (int)value; return AMG_OK; }
    if (k == "symd_chunked") { h->symd_chunked = value ? 1 : 0; return AMG_OK; }
    if (k == "coarse_pipe") { h->coarse_pipe = (int)value; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "side_prefetch") { h->side_prefetch = value ? 1 : 0; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "tail_pcap") {
        if (value < 1 || value > (1 << 24)) return fail(AMG_E_ARG, "tail_pcap must be in [1, 2^24]");
        h->tail_pcap = (int)value;
        return AMG_OK;
    }
    if (k == "tail_dsm") { h->tail_dsm = value ? 1 : 0; return AMG_OK; }
    if (k == "tail_prefetch") { h->tail_prefetch = value ? 1 : 0; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "symd_tsm") { h->symd_tsm = value ? 1 : 0; return AMG_OK; }
    if (k == "symd_classes") { h->symd_classes = (int)value; return AMG_OK; }
    if (k == "symd_blocked") { h->symd_blocked = value ? 1 : 0; return AMG_OK; }
    if (k == "symd_gminb") { h->symd_gminb = (int)value; return AMG_OK; }
    if (k == "symd_minb") { h->symd_minb = (int)value; return AMG_OK; }
    if (k == "sell") { h->sell = value ? 1 : 0; return AMG_OK; }
    if (k == "grid_per_sm") { h->grid_per_sm = (int)value; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "vec_per_sm") {
        // the reduction partials scratch holds sm_count * 8 CTAs (max_grid)
        if (value < 0 || value > 8) return fail(AMG_E_ARG, "vec_per_sm must be in [0, 8]");
        h->vec_per_sm = (int)value; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "gated_grid") { h->gated_grid = (int)value; if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; } return AMG_OK; }
    if (k == "sell_pad") { h->sell_pad = (int)value; return AMG_OK; }
    if (k == "sell_sigma") { h->sell_sigma = (int)value; return AMG_OK; }
    if (k == "direct_ctas") { h->direct_ctas = (int)value; return AMG_OK; }
    if (k == "lanes") { if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8) return fail(AMG_E_ARG, "lanes must be 0,1,2,4,8"); h->lanes_override = (int)value; return AMG_OK; }
    return fail(AMG_E_ARG, "amg_set_option: unknown key '" + k + "'");
}

int amg_nccl_unique_id(void *out)
{
    if (!out) return fail(AMG_E_ARG, "amg_nccl_unique_id: NULL output");
    NcclApi &api = nccl();
    if (!api.loaded) return fail(AMG_E_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(AMG_E_NCCL, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
    memcpy(out, &id, sizeof(id));
    return AMG_OK;
}

int amg_set_halo(amg_t *h, int level, int which, int64_t n_own, int64_t n_halo, int n_recv, const int *recv_peers,
                 const int64_t *recv_counts, int n_send, const int *send_peers, const int64_t *send_counts,
                 const int32_t *send_idx)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (h->finalized) return fail(AMG_E_STATE, "amg_set_halo: already finalized");
    if (h->nranks == 1) return fail(AMG_E_ARG, "amg_set_halo: single-rank handle has no halos");
    if (level < 0 || level >= (int)h->lv.size() || which < 0 || which > 4) return fail(AMG_E_ARG, "amg_set_halo: bad level / slot");
    DevMat &M = h->lv[level].m[which];
    if (!M.present) return fail(AMG_E_STATE, "amg_set_halo: upload the matrix first");
    if (n_own < 0 || n_halo < 0 || n_own + n_halo != M.ncols) return fail(AMG_E_DIM, "amg_set_halo: n_own + n_halo must equal the local column count");
    HaloPlan &P = M.halo;
    halo_free(P);
    P = HaloPlan();
    P.n_own = n_own;
    P.n_halo = n_halo;
    M.n_own = n_own;
    int64_t tot = 0;
    for (int i = 0; i < n_recv; ++i) {
        if (recv_peers[i] < 0 || recv_peers[i] >= h->nranks || recv_peers[i] == h->rank) return fail(AMG_E_ARG, "amg_set_halo: bad recv peer");
        P.recv_peers.push_back(recv_peers[i]);
        P.recv_counts.push_back(recv_counts[i]);
        tot += recv_counts[i];
    }
    if (tot != n_halo) return fail(AMG_E_DIM, "amg_set_halo: receive counts do not add up to n_halo");
    int64_t ns = 0;
    for (int i = 0; i < n_send; ++i) {
        if (send_peers[i] < 0 || send_peers[i] >= h->nranks || send_peers[i] == h->rank) return fail(AMG_E_ARG, "amg_set_halo: bad send peer");
        P.send_peers.push_back(send_peers[i]);
        P.send_counts.push_back(send_counts[i]);
        P.send_displ.push_back(ns);
        ns += send_counts[i];
    }
    for (int64_t i = 0; i < ns; ++i)
        if (send_idx[i] < 0 || send_idx[i] >= n_own) return fail(AMG_E_ARG, "amg_set_halo: send index outside the owned range");
    P.n_send = ns;
    CK(cudaSetDevice(h->device));
    TRY(dalloc(&P.send_idx, (size_t)ns + 1));
    TRY(dalloc(&P.send_buf, (size_t)ns + 1));
    if (ns) CK(cudaMemcpy(P.send_idx, send_idx, ns * sizeof(int32_t), cudaMemcpyHostToDevice));
    return AMG_OK;
}

int amg_set_agglomeration(amg_t *h, int level)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (h->finalized) return fail(AMG_E_STATE, "amg_set_agglomeration: already finalized");
    if (level < 0 || level >= (int)h->lv.size()) return fail(AMG_E_ARG, "amg_set_agglomeration: bad level");
    h->agglom_level = level;
    return AMG_OK;
}

int amg_set_levels(amg_t *h, int n_levels)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (h->finalized) return fail(AMG_E_STATE, "amg_set_levels: already finalized");
    if (n_levels < 1 || n_levels > 64) return fail(AMG_E_ARG, "amg_set_levels: n_levels out of range");
    h->lv.assign(n_levels, LevelD());
    return AMG_OK;
}

int amg_set_partition(amg_t *h, int level, const int64_t *starts)
{
    if (!h || !starts) return fail(AMG_E_ARG, "amg_set_partition: NULL argument");
    if (level < 0 || level >= (int)h->lv.size()) return fail(AMG_E_ARG, "amg_set_partition: bad level");
    std::vector<int64_t> s(starts, starts + h->nranks + 1);
    if (s[0] != 0) return fail(AMG_E_ARG, "amg_set_partition: starts[0] must be 0");
    for (int i = 0; i < h->nranks; ++i)
        if (s[i + 1] < s[i]) return fail(AMG_E_ARG, "amg_set_partition: starts must be non-decreasing");
    h->lv[level].starts = s;
    return AMG_OK;
}

int64_t amg_local_rows(amg_t *h, int level)
{
    if (!h || level < 0 || level >= (int)h->lv.size()) return -1;
    return h->lv[level].n;
}

int amg_upload_matrix(amg_t *h, int level, int which, int64_t local_nrows, int64_t global_ncols,
                      const int64_t *offsets, const int32_t *cols, const double *vals)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (h->finalized) return fail(AMG_E_STATE, "amg_upload_matrix: already finalized");
    if (level < 0 || level >= (int)h->lv.size()) return fail(AMG_E_ARG, "amg_upload_matrix: bad level (call amg_set_levels first)");
    if (which < 0 || which > 4) return fail(AMG_E_ARG, "amg_upload_matrix: bad matrix slot");
    if (local_nrows < 0 || global_ncols < 0 || (!offsets && local_nrows >= 0))
        return fail(AMG_E_ARG, "amg_upload_matrix: bad sizes / NULL offsets");
    if (offsets[0] != 0) return fail(AMG_E_ARG, "amg_upload_matrix: offsets[0] must be 0");
    const int64_t nnz = offsets[local_nrows];
    if (nnz < 0 || nnz >= INT32_MAX - 64) return fail(AMG_E_ARG, "amg_upload_matrix: local nnz must fit int32 (partition across more GPUs)");
    if (nnz > 0 && (!cols || !vals)) return fail(AMG_E_ARG, "amg_upload_matrix: NULL cols / vals");
    if (global_ncols >= INT32_MAX) return fail(AMG_E_ARG, "amg_upload_matrix: too many columns for int32 indices");
    CK(cudaSetDevice(h->device));
    DevMat &M = h->lv[level].m[which];
    if (M.present) return fail(AMG_E_STATE, "amg_upload_matrix: slot already uploaded");
    std::vector<int32_t> off32(local_nrows + 1 + 8, (int32_t)nnz);
    for (int64_t i = 0; i <= local_nrows; ++i) {
        if (i > 0 && offsets[i] < offsets[i - 1]) return fail(AMG_E_ARG, "amg_upload_matrix: offsets must be non-decreasing");
        off32[i] = (int32_t)offsets[i];
    }
    for (int64_t k = 0; k < nnz; ++k)
        if (cols[k] < 0 || cols[k] >= global_ncols) return fail(AMG_E_ARG, "amg_upload_matrix: column index out of range");
    M.nrows = local_nrows;
    M.gncols = global_ncols;
    M.ncols = global_ncols;
    M.n_own = global_ncols;
    M.nnz = nnz;
    // Local column numbering: on one rank global == local.  With nranks > 1
    // the halo plan (built at finalize) renumbers non-owned columns.
    std::vector<int32_t> col_local(cols, cols + nnz);
    TRY(dalloc(&M.off, off32.size()));
    TRY(dalloc(&M.col, (size_t)nnz + 8));
    TRY(dalloc(&M.val, (size_t)nnz + 4));
    CK(cudaMemcpy(M.off, off32.data(), off32.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (nnz) {
        CK(cudaMemcpy(M.col, col_local.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(M.val, vals, nnz * sizeof(double), cudaMemcpyHostToDevice));
    }
    M.present = true;
    return AMG_OK;
}

int amg_set_smoother(amg_t *h, int level, int kind, double omega, const double *inv_diag, int64_t n)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (h->finalized) return fail(AMG_E_STATE, "amg_set_smoother: already finalized");
    if (level < 0 || level >= (int)h->lv.size()) return fail(AMG_E_ARG, "amg_set_smoother: bad level");
    LevelD &L = h->lv[level];
    if (kind != AMG_SMOOTHER_FSAI && kind != AMG_SMOOTHER_JACOBI) return fail(AMG_E_ARG, "amg_set_smoother: bad kind");
    L.has_smoother = true;
    L.sm_kind = kind;
    L.omega = omega;
    if (kind == AMG_SMOOTHER_JACOBI) {
        if (!inv_diag || n < 0) return fail(AMG_E_ARG, "amg_set_smoother: Jacobi needs inv_diag");
        CK(cudaSetDevice(h->device));
        if (L.inv_diag) cudaFree(L.inv_diag);
        TRY(dalloc(&L.inv_diag, (size_t)n + 2));
        CK(cudaMemcpy(L.inv_diag, inv_diag, n * sizeof(double), cudaMemcpyHostToDevice));
    }
    return AMG_OK;
}

int amg_upload_coarse(amg_t *h, int n, const double *factor, int kind, const int32_t *piv)
{
    if (!h || !factor) return fail(AMG_E_ARG, "amg_upload_coarse: NULL argument");
    if (h->finalized) return fail(AMG_E_STATE, "amg_upload_coarse: already finalized");
    if (n < 1) return fail(AMG_E_ARG, "amg_upload_coarse: n < 1");
    CK(cudaSetDevice(h->device));
    h->nc = n;
    h->coarse_kind = kind;
    if (kind == AMG_COARSE_CHOLESKY) {
        std::vector<double> packed((size_t)n * (n + 1) / 2);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j <= i; ++j) packed[(size_t)i * (i + 1) / 2 + j] = factor[(size_t)i * n + j];
        std::vector<double> dinv(n);
        for (int i = 0; i < n; ++i) {
            const double d = factor[(size_t)i * n + i];
            if (!(d > 0.0)) return fail(AMG_E_ARG, "amg_upload_coarse: Cholesky factor has a non-positive diagonal");
            dinv[i] = 1.0 / d;
        }
        // pre-scaled diagonal blocks: Ms[r][c] = L[r][c] / L[c][c], Ns[r][c] = L[r][c] / L[r][r] (r > c)
        const int nblk = (n + 31) / 32;
        std::vector<double> mn((size_t)nblk * 1056, 0.0);
        for (int b = 0; b < nblk; ++b) {
            const int jb = b * 32, nb = std::min(32, n - jb);
            for (int r = 0; r < nb; ++r)
                for (int c2 = 0; c2 < r; ++c2) {
                    const double l = factor[(size_t)(jb + r) * n + (jb + c2)];
                    mn[(size_t)b * 1056 + r * (r + 1) / 2 + c2] = l * dinv[jb + c2];
                    mn[(size_t)b * 1056 + 528 + r * (r + 1) / 2 + c2] = l * dinv[jb + r];
                }
        }
        TRY(dalloc(&h->binv, mn.size()));
        CK(cudaMemcpy(h->binv, mn.data(), mn.size() * sizeof(double), cudaMemcpyHostToDevice));
        TRY(dalloc(&h->Lp, packed.size()));
        TRY(dalloc(&h->dinv, (size_t)n));
        CK(cudaMemcpy(h->Lp, packed.data(), packed.size() * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->dinv, dinv.data(), n * sizeof(double), cudaMemcpyHostToDevice));
        const size_t vbytes = (size_t)(2 * ((n + 1) & ~1) + 32 + mn.size()) * sizeof(double);  // v, tmp, 1/L_ii, M/N
        const size_t lbytes = packed.size() * sizeof(double);
        if (vbytes + lbytes <= 200 * 1024) {
            h->coarse_staged = 1;
            h->coarse_smem = vbytes + lbytes;
        } else {
            h->coarse_staged = 0;
            h->coarse_smem = (size_t)(((n + 1) & ~1) + 32) * sizeof(double);  // v + tmp; factor read from L2
        }
    } else if (kind == AMG_COARSE_LU) {
        if (!piv) return fail(AMG_E_ARG, "amg_upload_coarse: LU needs pivots");
        for (int i = 0; i < n; ++i)
            if (piv[i] < 0 || piv[i] >= n) return fail(AMG_E_ARG, "amg_upload_coarse: pivot out of range");
        TRY(dalloc(&h->LU, (size_t)n * n));
        TRY(dalloc(&h->piv, (size_t)n));
        CK(cudaMemcpy(h->LU, factor, (size_t)n * n * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->piv, piv, (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice));
        h->coarse_staged = 0;
        h->coarse_smem = (size_t)((n + 1) & ~1) * sizeof(double);
    } else {
        return fail(AMG_E_ARG, "amg_upload_coarse: bad kind");
    }
    TRY(raise_smem_caps(h->device));
    return AMG_OK;
}

int amg_set_cycle(amg_t *h, int nu1, int nu2)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (nu1 < 0 || nu2 < 0) return fail(AMG_E_ARG, "smoothing step counts must be nonnegative");
    // the cluster tail's op list is fixed at amg_finalize: a later change would
    // reach the upper levels only
    if (h->finalized) return fail(AMG_E_STATE, "amg_set_cycle: already finalized");
    h->nu1 = nu1;
    h->nu2 = nu2;
    if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
    return AMG_OK;
}

// Row-class dictionary (spmv_dict): rows grouped by their exact (length, col - row
// offsets, value bits) tuple; used when at most DICT_MAX_CLS classes with at most
// DICT_MAX_ENT table entries in total cover every row of <= 32 entries.  Hash
// buckets hold candidate classes that are compared entry by entry, so equal
// hashes never merge different rows.  Gives up as soon as a limit is exceeded
// (irregular matrices cost a few thousand rows of hashing).
static constexpr int DICT_MAX_CLS = 1024;
static constexpr int DICT_MAX_ENT = 3072;

static int build_dict(amg_t *h, DevMat &M, const std::vector<int32_t> &off32)
{
    if (M.nrows <= 0 || M.nnz <= 0 || M.nrows >= INT32_MAX - 1) return AMG_OK;
    int maxlen = 0;
    for (int64_t r = 0; r < M.nrows; ++r) maxlen = std::max(maxlen, off32[r + 1] - off32[r]);
    if (maxlen > 32) return AMG_OK;
    std::vector<int32_t> col_h(M.nnz);
    std::vector<double> val_h(M.nnz);
    CK(cudaMemcpy(col_h.data(), M.col, M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(val_h.data(), M.val, M.nnz * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<int32_t> beg(1, 0), rel;
    std::vector<double> val;
    std::unordered_map<uint64_t, std::vector<int>> buckets;
    std::vector<uint16_t> cls(M.nrows);
    for (int64_t r = 0; r < M.nrows; ++r) {
        const int32_t s = off32[r], e = off32[r + 1];
        uint64_t hsh = 1469598103934665603ull ^ (uint64_t)(e - s);
        for (int32_t k = s; k < e; ++k) {
            uint64_t vb;
            memcpy(&vb, &val_h[k], 8);
            hsh = (hsh ^ (uint64_t)(uint32_t)(col_h[k] - (int32_t)r)) * 1099511628211ull;
            hsh = (hsh ^ vb) * 1099511628211ull;
        }
        auto &bk = buckets[hsh];
        int found = -1;
        for (int c : bk) {
            if (beg[c + 1] - beg[c] != e - s) continue;
            bool same = true;
            for (int32_t k = s; k < e && same; ++k) {
                const int q = beg[c] + (k - s);
                same = rel[q] == col_h[k] - (int32_t)r && memcmp(&val[q], &val_h[k], 8) == 0;
            }
            if (same) { found = c; break; }
        }
        if (found < 0) {
            found = (int)beg.size() - 1;
            if (found >= DICT_MAX_CLS || (int)rel.size() + (e - s) > DICT_MAX_ENT) return AMG_OK;
            for (int32_t k = s; k < e; ++k) {
                rel.push_back(col_h[k] - (int32_t)r);
                val.push_back(val_h[k]);
            }
            beg.push_back((int32_t)rel.size());
            bk.push_back(found);
        }
        cls[r] = (uint16_t)found;
    }
    M.dncls = (int)beg.size() - 1;
    M.dnent = (int)rel.size();
    {
        // the class most rows share (the interior stencil): rows of <= 8 entries only
        std::vector<int64_t> cnt(M.dncls, 0);
        for (int64_t r = 0; r < M.nrows; ++r) ++cnt[cls[r]];
        int best = -1;
        for (int c = 0; c < M.dncls; ++c)
            if (beg[c + 1] - beg[c] <= 8 && (best < 0 || cnt[c] > cnt[best])) best = c;
        M.dmcls = -1;
        if (best >= 0 && maxlen <= 8) {
            M.dmcls = best;
            M.dmlen = beg[best + 1] - beg[best];
            for (int k = 0; k < 8; ++k) {
                M.dmrel[k] = k < M.dmlen ? rel[beg[best] + k] : 0;
                M.dmval[k] = k < M.dmlen ? val[beg[best] + k] : 0.0;
            }
        }
    }
    M.dwide = M.dncls > 256 ? 1 : 0;
    M.dfl = maxlen <= 4 ? 4 : maxlen <= 8 ? 8 : maxlen <= 16 ? 16 : 32;
    if (M.dwide) {
        TRY(dalloc((uint16_t **)&M.dcls, (size_t)M.nrows));
        CK(cudaMemcpy(M.dcls, cls.data(), (size_t)M.nrows * 2, cudaMemcpyHostToDevice));
    } else {
        std::vector<uint8_t> c8(cls.begin(), cls.end());
        TRY(dalloc((uint8_t **)&M.dcls, (size_t)M.nrows));
        CK(cudaMemcpy(M.dcls, c8.data(), (size_t)M.nrows, cudaMemcpyHostToDevice));
    }
    TRY(dalloc(&M.dbeg, beg.size()));
    TRY(dalloc(&M.drel, std::max<size_t>(rel.size(), 1)));
    TRY(dalloc(&M.dval, std::max<size_t>(val.size(), 1)));
    CK(cudaMemcpy(M.dbeg, beg.data(), beg.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (!rel.empty()) {
        CK(cudaMemcpy(M.drel, rel.data(), rel.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(M.dval, val.data(), val.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    const size_t sm = (size_t)M.dnent * 12 + (size_t)(M.dncls + 1) * 4;
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)spmv_dict_fn(EPI_RESID, M.dfl, M.dwide, (h->dict_main && M.dmcls >= 0) ? M.dmlen : 0),
                                                     VEC_SPMV_THREADS, sm));
    M.dgrid = (int)std::max<int64_t>(1, std::min<int64_t>((M.nrows + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS,
                                                          (int64_t)h->sm_count * std::max(nb, 1)));
    h->max_grid = std::max(h->max_grid, M.dgrid);
    M.lbytes[AMG_LAYOUT_DICT] = M.nrows * (M.dwide ? 2 : 1) + (int64_t)sm;  // class ids + the table
    return AMG_OK;
}

// Stencil patterns: every row's (col - row) tuple from a dictionary of at most
// PAT_MAX patterns (PAT_MAX_REL offsets in total, rows <= 129 entries).
static bool pattern_dict(const DevMat &M, const std::vector<int32_t> &off32, const std::vector<int32_t> &col_h,
                         std::vector<uint8_t> &ids, std::vector<int32_t> &rel, std::vector<int32_t> &beg)
{
    std::unordered_map<std::string, int> dict;
    ids.assign(M.nrows, 0);
    rel.clear();
    beg.assign(1, 0);
    std::string key;
    for (int64_t r = 0; r < M.nrows; ++r) {
        const int32_t lo = off32[r], hi = off32[r + 1];
        key.resize((size_t)(hi - lo) * 4);
        for (int32_t k = lo; k < hi; ++k) {
            const int32_t d = col_h[k] - (int32_t)r;
            memcpy(&key[(size_t)(k - lo) * 4], &d, 4);
        }
        auto it = dict.find(key);
        int id;
        if (it == dict.end()) {
            id = (int)dict.size();
            if (id >= PAT_MAX || (int)rel.size() + (hi - lo) > PAT_MAX_REL || hi - lo > 129) return false;
            dict.emplace(key, id);
            for (int32_t k = lo; k < hi; ++k) rel.push_back(col_h[k] - (int32_t)r);
            beg.push_back((int32_t)rel.size());
        } else {
            id = it->second;
        }
        ids[r] = (uint8_t)id;
    }
    return !dict.empty();
}

// Symmetric stencil layout (spmv_symd): taken when the operator is square, its
// pattern dictionary exists, its relative offsets are closed under negation,
// every below-diagonal entry equals its mirror BIT FOR BIT, and storing the
// nu >= 0 diagonals densely costs at most 3/4 of the full value stream.
static int build_symd(amg_t *h, DevMat &M, const std::vector<int32_t> &off32, const std::vector<int32_t> &col_h,
                      const std::vector<double> &val_h, const std::vector<uint8_t> &ids,
                      const std::vector<int32_t> &rel, const std::vector<int32_t> &beg)
{
    const int64_t n = M.nrows;
    const int npat = (int)beg.size() - 1;
    if (npat < 1 || rel.size() > (size_t)SYMD_TAB || beg.size() > (size_t)SYMD_BEG_MAX) return AMG_OK;
    const int64_t npad = ((n + 31) / 32) * 32;
    int maxlen = 0;
    for (int p = 0; p < npat; ++p) maxlen = std::max(maxlen, beg[p + 1] - beg[p]);
    // Row classes: rows r with r % K == c share their set of stored diagonals D_c (d >= 0).
    // K = 1 for scalar stencils; K = 3 for node-major 3-dof systems (elasticity), whose
    // classes each use 41 of the 68 non-negative offsets.  A pattern must belong to one class.
    int K = 0;
    std::vector<std::vector<int32_t>> up;
    std::vector<int> pcls;
    for (int k : {1, 2, 3, 4}) {
        if (k > h->symd_classes) break;
        std::vector<int> cl(npat, -1);
        bool ok = true;
        for (int64_t r = 0; r < n && ok; ++r) {
            const int c = (int)(r % k), p = ids[r];
            if (cl[p] < 0) cl[p] = c;
            else if (cl[p] != c) ok = false;
        }
        if (!ok) continue;
        std::vector<std::vector<int32_t>> u(k);
        for (int p = 0; p < npat; ++p)
            if (cl[p] >= 0)
                for (int e = beg[p]; e < beg[p + 1]; ++e)
                    if (rel[e] >= 0) u[cl[p]].push_back(rel[e]);
        size_t nu = 0;
        for (auto &v : u) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            nu = std::max(nu, v.size());
        }
        if (nu == 0 || nu > 63 || (double)nu * (double)n > 0.75 * (double)M.nnz) continue;
        K = k;
        up = u;
        pcls = cl;
        break;
    }
    if (K == 0) return AMG_OK;
    int nu = 0;
    for (auto &v : up) nu = std::max(nu, (int)v.size());
    if ((int64_t)nu * npad + npad >= INT32_MAX - 64) return AMG_OK;
    auto jof = [&](int64_t r, int32_t d) -> int {  // stored diagonal index of a(r, r + d), d >= 0; -1 if none
        const auto &v = up[r % K];
        auto it = std::lower_bound(v.begin(), v.end(), d);
        return (it == v.end() || *it != d) ? -1 : (int)(it - v.begin());
    };
    // slice-blocked storage for the round-by-round kernel (27-point: 88 -> 81 us on config 2); the
    // fixed-slot 7-point kernel keeps one array per diagonal (config 4: 159 vs 171 us)
    const bool blk = h->symd_blocked && !(maxlen <= 8 && h->symd_fixed >= 1 && K == 1);
    auto sidx = [&](int64_t r, int j) -> size_t {  // storage index of stored diagonal j of row r
        return blk ? (size_t)((r >> 5) * 32 * nu + 32 * j + (r & 31)) : (size_t)j * npad + r;
    };
    std::vector<double> uv((size_t)nu * npad, 0.0);
    std::vector<uint8_t> have((size_t)nu * npad, 0);
    for (int64_t r = 0; r < n; ++r)  // upper entries (and the diagonal) first
        for (int32_t k = off32[r]; k < off32[r + 1]; ++k) {
            const int32_t d = col_h[k] - (int32_t)r;
            if (d < 0) continue;
            const size_t q = sidx(r, jof(r, d));
            uv[q] = val_h[k];
            have[q] = 1;
        }
    for (int64_t r = 0; r < n; ++r)  // every lower entry must be its mirror, bitwise
        for (int32_t k = off32[r]; k < off32[r + 1]; ++k) {
            const int32_t d = col_h[k] - (int32_t)r;
            if (d >= 0) continue;
            const int j = jof(r + d, -d);
            if (j < 0) return AMG_OK;
            const size_t q = sidx(r + d, j);
            if (!have[q] || memcmp(&uv[q], &val_h[k], sizeof(double)) != 0) return AMG_OK;
        }
    // pattern entries; a pattern's rows are all of class pcls[p], so the mirror row's class is known
    std::vector<int2> ent(rel.size());
    for (int p = 0; p < npat; ++p) {
        const int c = pcls[p] < 0 ? 0 : pcls[p];
        for (int e = beg[p]; e < beg[p + 1]; ++e) {
            const int32_t d = rel[e];
            if (std::abs((int64_t)d) >= (1 << 24)) return AMG_OK;
            const int64_t src = d >= 0 ? c : (((c + d) % K) + K) % K;  // class of the row holding the copy
            const int j = jof(src, d >= 0 ? d : -d);
            if (j < 0) return AMG_OK;
            const int64_t ds = d >= 0 ? 0 : d;  // row offset of the stored copy
            ent[e] = make_int2(d, blk ? (int)((ds << 6) | j) : (int)((int64_t)j * npad + ds));
        }
    }
    const int slot = symd_slot_take(h->device);
    if (slot < 0) return AMG_OK;  // every table slot of this device in use: keep the other layouts
    const int tbase = symd_tab_take(h->device, (int)ent.size());
    if (tbase < 0) {
        symd_slot_give(h->device, slot);
        return AMG_OK;
    }
    std::vector<int32_t> bg(SYMD_BEG_MAX, 0);
    for (size_t i = 0; i < beg.size(); ++i) bg[i] = tbase + beg[i];
    if (!ent.empty())
        CK(cudaMemcpyToSymbol(c_symd_tab, ent.data(), ent.size() * sizeof(int2), (size_t)tbase * sizeof(int2)));
    CK(cudaMemcpyToSymbol(c_symd_beg, bg.data(), bg.size() * sizeof(int32_t), (size_t)slot * SYMD_BEG_MAX * sizeof(int32_t)));
    M.sym_slot = slot;
    M.sym_tab = tbase;
    M.sym_ntab = (int)ent.size();
    M.sym_blocked = blk ? 1 : 0;
    M.sym_classes = K;
    M.sym_npad = (int)npad;
    TRY(dalloc(&M.uval, uv.size()));
    CK(cudaMemcpy(M.uval, uv.data(), uv.size() * sizeof(double), cudaMemcpyHostToDevice));
    M.lbytes[AMG_LAYOUT_SYMD] = (int64_t)uv.size() * 8 + n;  // stored diagonals + 1-byte pattern id per row
    M.nudiag = nu;
    int nb = 0;
    M.sym_fast_on = false;
    if (blk && K == 1 && n < INT32_MAX - 64) {
        // the pattern most rows have; 27 entries -> interior fast path with parameter-bank offsets
        std::vector<int64_t> cnt(npat, 0);
        for (int64_t r = 0; r < n; ++r) ++cnt[ids[r]];
        int mp = 0;
        for (int p2 = 1; p2 < npat; ++p2)
            if (cnt[p2] > cnt[mp]) mp = p2;
        if (beg[mp + 1] - beg[mp] == 27) {
            SymFast &F = M.sym_fast;
            F.pat = mp;
            const long long w32 = 32LL * nu;
            for (int k = 0; k < 27; ++k) {
                const int e = beg[mp] + k;
                const long long d = rel[e];
                const int j = ent[e].y & 63;
                F.xoff[k] = d * 8;
                if (d >= 0) {
                    F.thr[k] = 0;
                    F.voffA[k] = F.voffB[k] = 32LL * j * 8;
                } else {
                    const long long dd = -d, qA = -(dd / 32) - ((dd % 32) ? 0 : 0);
                    // row i = 32 s + l reads the copy in row i - dd: lane l - dd (mod 32) of slice s + floor((l - dd) / 32)
                    const long long t = dd % 32;
                    const long long qa = -(dd / 32);          // lanes l >= t
                    const long long qb = qa - 1;              // lanes l < t (t > 0)
                    (void)qA;
                    F.thr[k] = (int)t;
                    F.voffA[k] = (qa * (w32 - 32) + 32LL * j - dd) * 8;
                    F.voffB[k] = (qb * (w32 - 32) + 32LL * j - dd) * 8;
                }
            }
            M.sym_fast_on = true;
            int nb27 = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb27, (const void *)spmv_symd27_fn(EPI_RESID), VEC_SPMV_THREADS, 0));
            M.sym27_grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS,
                                                                       (int64_t)h->sm_count * std::max(nb27, 1)));
            h->max_grid = std::max(h->max_grid, M.sym27_grid);
        }
    }
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)spmv_symd_fn(EPI_RESID, h->symd_gminb, blk), VEC_SPMV_THREADS, 0));
    M.sym_grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS,
                                                             (int64_t)h->sm_count * std::max(nb, 1)));
    h->max_grid = std::max(h->max_grid, M.sym_grid);
    M.sym_fl = maxlen <= 8 ? 8 : maxlen <= 32 ? 32 : 0;
    if (M.sym_fl) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)spmv_symd_fixed_fn(EPI_RESID, M.sym_fl, h->symd_minb),
                                                         VEC_SPMV_THREADS, 0));
        M.symf_grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS,
                                                                  (int64_t)h->sm_count * std::max(nb, 1)));
        h->max_grid = std::max(h->max_grid, M.symf_grid);
    }
    return AMG_OK;
}

// Interior rows of a distributed matrix (no column in the halo segment): the
// rows below the last halo-touching row of the first half and above the first
// halo-touching row of the second half -- for a z-slab block, everything but
// its first and last planes.  Aligned inwards to 128 rows (slices / sorted
// windows map whole).  overlap_test (one rank): the middle half of every
// matrix, to exercise the split launches on one GPU.
static int interior_range(amg_t *h, DevMat &M, const std::vector<int32_t> &off32)
{
    M.int_lo = M.int_hi = 0;
    const int64_t n = M.nrows;
    int64_t lo_end = 0, hi_start = n;
    if (h->nranks > 1) {
        if (M.halo.empty() || M.nnz == 0) return AMG_OK;
        std::vector<int32_t> col_h(M.nnz);
        CK(cudaMemcpy(col_h.data(), M.col, M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (int64_t r = 0; r < n; ++r) {
            bool halo = false;
            for (int32_t k = off32[r]; k < off32[r + 1] && !halo; ++k) halo = col_h[k] >= M.n_own;
            if (!halo) continue;
            if (r < n / 2) lo_end = r + 1;
            else if (hi_start == n) hi_start = r;
        }
    } else if (h->overlap_test) {
        lo_end = n / 4;
        hi_start = 3 * n / 4;
    } else {
        return AMG_OK;
    }
    const int64_t a = (lo_end + 127) / 128 * 128, b = hi_start / 128 * 128;
    if (b - a >= 128 && b - a >= n / 8) {
        M.int_lo = a;
        M.int_hi = b;
    }
    return AMG_OK;
}

int amg_finalize(amg_t *h)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (h->finalized) return fail(AMG_E_STATE, "amg_finalize: already finalized");
    const int nl = (int)h->lv.size();
    if (nl < 1) return fail(AMG_E_STATE, "amg_finalize: no levels");
    CK(cudaSetDevice(h->device));
    // A handle without a coarsest factor is a plain matrix container (spmv only).
    const bool container = (h->nc == 0);
    if (h->nranks > 1 && !container) {
        if (h->agglom_level < 0 || h->agglom_level > nl - 1)
            return fail(AMG_E_STATE, "multi-GPU: amg_set_agglomeration must name a level <= the coarsest (replicated) level");
        h->dist_dots = h->agglom_level > 0;
    }
    if (h->nranks == 1 && h->nccl_selftest && !container) {
        // one-rank communicator: proves the NCCL calls of the multi-GPU path (dot
        // all-gathers, p2p on the comm stream with its fork / join) are captured
        // into the conditional WHILE body on this NCCL build
        NcclApi &api = nccl();
        if (!api.loaded) return fail(AMG_E_NCCL, "libnccl.so.2 could not be loaded");
        ncclUniqueId id;
        ncclResult_t r = api.GetUniqueId(&id);
        if (r != ncclSuccess) return fail(AMG_E_NCCL, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
        if (comm_init(h->comm, &id, 0, 1) != 0 || !h->comm.comm) {
            r = api.CommInitRank(&h->comm.comm, 1, id, 0);
            if (r != ncclSuccess) return fail(AMG_E_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
        }
        h->dist_dots = h->nccl_selftest != 3;  // 3: p2p only, 2: dots only, 1: both
        TRY(dalloc(&h->selftest_buf, 2));
    }
    // structural checks mirroring the Level / AmgHierarchy contract
    for (int k = 0; k < nl && !container; ++k) {
        LevelD &L = h->lv[k];
        if (!L.m[AMG_A].present) return fail(AMG_E_STATE, "level " + std::to_string(k) + ": operator A missing");
        L.n = L.m[AMG_A].nrows;
        if (h->nranks == 1) {
            L.gn = L.n;
            L.n0 = 0;
            if (L.m[AMG_A].gncols != L.n) return fail(AMG_E_DIM, "level " + std::to_string(k) + ": A is not square");
        } else if (k >= h->agglom_level) {  // replicated level: every rank holds all rows
            L.gn = L.n;
            L.n0 = 0;
            if (L.m[AMG_A].gncols != L.n) return fail(AMG_E_DIM, "level " + std::to_string(k) + ": replicated A is not square");
            if (k == h->agglom_level && k > 0 &&
                ((int)L.starts.size() != h->nranks + 1 || L.starts[h->nranks] != L.n))
                return fail(AMG_E_STATE, "level " + std::to_string(k) + ": agglomeration level needs its partition");
        } else {
            if ((int)L.starts.size() != h->nranks + 1) return fail(AMG_E_STATE, "level " + std::to_string(k) + ": partition missing");
            L.n0 = L.starts[h->rank];
            L.gn = L.starts[h->nranks];
            if (L.starts[h->rank + 1] - L.n0 != L.n) return fail(AMG_E_DIM, "level " + std::to_string(k) + ": local rows do not match the partition");
        }
        if (k < nl - 1) {
            if (!L.m[AMG_P].present || !L.m[AMG_PT].present) return fail(AMG_E_STATE, "level " + std::to_string(k) + ": P / Pt missing");
            if (!L.has_smoother) return fail(AMG_E_STATE, "level " + std::to_string(k) + ": smoother missing");
            if (L.sm_kind == AMG_SMOOTHER_FSAI && (!L.m[AMG_G].present || !L.m[AMG_GT].present))
                return fail(AMG_E_STATE, "level " + std::to_string(k) + ": FSAI factor G / Gt missing");
        }
    }
    for (int k = 0; k < nl; ++k) h->lv[k].n = h->lv[k].m[AMG_A].nrows;
    for (int k = 0; k < nl - 1 && !container; ++k) {
        LevelD &L = h->lv[k], &C = h->lv[k + 1];
        if (h->nranks == 1) {
            if (L.m[AMG_P].nrows != L.n || L.m[AMG_P].gncols != C.n)
                return fail(AMG_E_DIM, "level " + std::to_string(k) + ": P shape does not match the levels");
            if (L.m[AMG_PT].nrows != C.n) return fail(AMG_E_DIM, "level " + std::to_string(k) + ": Pt shape does not match");
        } else {
            const int64_t cown = (k + 1 >= h->agglom_level && k < h->agglom_level)
                                     ? C.starts[h->rank + 1] - C.starts[h->rank] : C.n;
            if (L.m[AMG_P].nrows != L.n) return fail(AMG_E_DIM, "level " + std::to_string(k) + ": P rows do not match");
            if (L.m[AMG_PT].nrows != cown) return fail(AMG_E_DIM, "level " + std::to_string(k) + ": Pt rows do not match the coarse partition");
        }
    }
    h->container = container;
    if (!container && h->nc != h->lv[nl - 1].gn) return fail(AMG_E_DIM, "coarsest factor size does not match the last level");
    TRY(raise_smem_caps(h->device));
    {
        int best = 1 << 30;
        for (int e = 0; e <= 4; ++e)
            for (int l : {1, 2, 4, 8}) {
                int nb = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)spmv_direct_fn(e, l), DIRECT_THREADS, 0));
                best = std::min(best, nb);
            }
        h->direct_per_sm = h->direct_ctas > 0 ? std::min(h->direct_ctas, best) : best;
        h->max_grid = std::max(h->max_grid, h->sm_count * h->direct_per_sm);
    }
    h->max_grid = h->sm_count * 8;
    // device layouts per matrix
    for (int k = 0; k < nl; ++k) {
        LevelD &L = h->lv[k];
        for (int w = 0; w < 5; ++w) {
            DevMat &M = L.m[w];
            if (!M.present) continue;
            std::vector<int32_t> off32(M.nrows + 1);
            CK(cudaMemcpy(off32.data(), M.off, (M.nrows + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
            TRY(interior_range(h, M, off32));
            // row-class dictionary first: where it applies no value / column stream is needed
            if (h->dict && h->nranks == 1 && !h->lanes_override && M.nrows >= (int64_t)h->sm_count * h->small_rows_per_sm)
                TRY(build_dict(h, M, off32));
            // rows averaging > long_avg entries: leaf list for spmv_leaves / spmv_leafsum
            const bool longrows = !M.dcls && h->long_avg > 0 && !h->lanes_override && M.nrows > 0 &&
                                  (double)M.nnz / (double)M.nrows > (double)h->long_avg;
            if (longrows) {
                std::vector<int2> lv;
                std::vector<int32_t> rl(M.nrows + 1);
                int sb[32], sm[32];
                for (int64_t r = 0; r < M.nrows; ++r) {
                    rl[r] = (int32_t)lv.size();
                    const int n = off32[r + 1] - off32[r] - 1;
                    if (n < 8) continue;
                    int sp = 1;
                    sb[0] = off32[r] + 1;
                    sm[0] = n;
                    while (sp > 0) {  // in-order leaves: pre-order walk, pending right children stacked
                        --sp;
                        int b = sb[sp], m = sm[sp];
                        while (m > 128) {
                            const int n2 = m / 2 - (m / 2) % 8;
                            sb[sp] = b + n2;
                            sm[sp] = m - n2;
                            ++sp;
                            m = n2;
                        }
                        lv.push_back(make_int2(b, m));
                    }
                }
                rl[M.nrows] = (int32_t)lv.size();
                M.nleaves = (int)lv.size();
                TRY(dalloc(&M.leaf, lv.size() + 1));
                TRY(dalloc(&M.row_leaf, rl.size()));
                TRY(dalloc(&M.lsum, lv.size() + 1));
                if (!lv.empty()) CK(cudaMemcpy(M.leaf, lv.data(), lv.size() * sizeof(int2), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(M.row_leaf, rl.data(), rl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                M.leaf_grid = (int)std::max<int64_t>(1, std::min<int64_t>((M.nleaves + 31) / 32,
                                                                         (int64_t)h->sm_count * h->direct_per_sm));
                M.leafsum_grid = (int)std::max<int64_t>(1, std::min<int64_t>((M.nrows + DIRECT_THREADS - 1) / DIRECT_THREADS,
                                                                            (int64_t)h->sm_count * 4));
                h->max_grid = std::max(h->max_grid, std::max(M.leaf_grid, M.leafsum_grid));
            }
            if (!M.dcls && !longrows && h->pad_min > 0 && M.nrows >= (int64_t)h->sm_count * h->small_rows_per_sm && !h->lanes_override &&
                (double)M.nnz / (double)M.nrows >= (double)h->pad_min) {
                // padded-aligned copy: row starts == 3 (mod 4) so entry 1 is 16-byte aligned
                std::vector<int32_t> col_h(M.nnz);
                std::vector<double> val_h(M.nnz);
                if (M.nnz) {
                    CK(cudaMemcpy(col_h.data(), M.col, M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
                    CK(cudaMemcpy(val_h.data(), M.val, M.nnz * sizeof(double), cudaMemcpyDeviceToHost));
                }
                if (h->wcsr) {
                    // warp-cooperative CSR on the uploaded arrays (no padded copy)
                    M.wcsr = 1;
                    int nbw = 0;
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbw, (const void *)spmv_wcsr<EPI_RESID>, WCSR_THREADS, 0));
                    M.wcsr_grid = (int)std::max<int64_t>(1, std::min<int64_t>((M.nrows + WCSR_THREADS - 1) / WCSR_THREADS,
                                                                             (int64_t)h->sm_count * std::max(nbw, 1)));
                    h->max_grid = std::max(h->max_grid, M.wcsr_grid);
                    M.lbytes[AMG_LAYOUT_WCSR] = M.nnz * 12 + (M.nrows + 1) * 4;
                } else {
                std::vector<int32_t> ps(M.nrows + 1);
                int64_t pos = 3;
                for (int64_t r = 0; r < M.nrows; ++r) {
                    ps[r] = (int32_t)pos;
                    const int64_t len = off32[r + 1] - off32[r];
                    pos += len;
                    pos += (3 - (pos % 4) + 4) % 4;  // next start == 3 (mod 4)
                    if (pos >= INT32_MAX - 64) return fail(AMG_E_ARG, "padded layout exceeds int32 indexing");
                }
                ps[M.nrows] = (int32_t)pos;
                const int64_t tot = pos + 16;  // vector over-read slack
                std::vector<int32_t> pc(tot, 0);
                std::vector<double> pv(tot, 0.0);
                for (int64_t r = 0; r < M.nrows; ++r)
                    for (int32_t k = off32[r]; k < off32[r + 1]; ++k) {
                        pc[ps[r] + (k - off32[r])] = col_h[k];
                        pv[ps[r] + (k - off32[r])] = val_h[k];
                    }
                TRY(dalloc(&M.pstart, ps.size()));
                TRY(dalloc(&M.pcol, pc.size()));
                TRY(dalloc(&M.pval, pv.size()));
                M.lbytes[AMG_LAYOUT_PADDED] = (int64_t)pv.size() * 12 + (int64_t)ps.size() * 4;
                CK(cudaMemcpy(M.pstart, ps.data(), ps.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(M.pcol, pc.data(), pc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(M.pval, pv.data(), pv.size() * sizeof(double), cudaMemcpyHostToDevice));
                }
                // stencil patterns: every row's (col - row) tuple from a small dictionary
                if (h->patterns && h->nranks == 1 && M.ncols == M.nrows) {
                    std::vector<int32_t> rel, beg;
                    std::vector<uint8_t> ids;
                    if (pattern_dict(M, off32, col_h, ids, rel, beg)) {
                        M.npat = (int)beg.size() - 1;
                        M.nrel = (int)rel.size();
                        TRY(dalloc(&M.pid, ids.size() + 16));
                        TRY(dalloc(&M.prel, rel.size()));
                        TRY(dalloc(&M.pbeg, beg.size()));
                        CK(cudaMemcpy(M.pid, ids.data(), ids.size(), cudaMemcpyHostToDevice));
                        CK(cudaMemcpy(M.prel, rel.data(), rel.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                        CK(cudaMemcpy(M.pbeg, beg.data(), beg.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                        if (h->symm) TRY(build_symd(h, M, off32, col_h, val_h, ids, rel, beg));
                    }
                }
                // SELL-32: coalesced slices where the padding stays small
                if (h->sell) {
                    const int64_t ns = (M.nrows + 31) / 32;
                    std::vector<int32_t> sb(ns + 1);
                    // slice order: natural, or (SELL-sigma) rows sorted by length inside windows of
                    // sigma rows when the natural slices pad too much; the pattern layout keeps order
                    std::vector<int32_t> order(M.nrows);
                    for (int64_t r = 0; r < M.nrows; ++r) order[r] = (int32_t)r;
                    auto slice_total = [&](int64_t *maxlen) {
                        int64_t tot = 0;
                        *maxlen = 0;
                        for (int64_t sl = 0; sl < ns; ++sl) {
                            int w = 0;
                            for (int64_t p = sl * 32; p < std::min<int64_t>(M.nrows, sl * 32 + 32); ++p)
                                w = std::max(w, off32[order[p] + 1] - off32[order[p]]);
                            sb[sl] = (int32_t)tot;
                            tot += (int64_t)w * 32;
                            *maxlen = std::max<int64_t>(*maxlen, w);
                        }
                        sb[ns] = (int32_t)tot;
                        return tot;
                    };
                    int64_t maxlen = 0;
                    int64_t tot = slice_total(&maxlen);
                    bool sorted = false;
                    if (tot > (int64_t)(M.nnz * (1.0 + h->sell_pad / 100.0)) && M.pid == nullptr && h->sell_sigma > 32) {
                        for (int64_t w0 = 0; w0 < M.nrows; w0 += h->sell_sigma) {
                            const int64_t w1 = std::min<int64_t>(M.nrows, w0 + h->sell_sigma);
                            std::stable_sort(order.begin() + w0, order.begin() + w1, [&](int32_t a, int32_t b) {
                                return off32[a + 1] - off32[a] > off32[b + 1] - off32[b];
                            });
                        }
                        tot = slice_total(&maxlen);
                        sorted = true;
                    }
                    if (maxlen <= 129 && tot <= (int64_t)(M.nnz * (1.0 + h->sell_pad / 100.0)) && tot < INT32_MAX - 64) {
                        std::vector<double> sv(tot + 32, 0.0);
                        const bool pat = M.pid != nullptr;
                        std::vector<int32_t> sc(pat ? 0 : tot + 32, 0);
                        std::vector<uint8_t> ln(M.nrows + 16, 0);
                        for (int64_t q = 0; q < M.nrows; ++q) {  // q = slice position, r = row
                            const int64_t r = order[q];
                            const int64_t sl = q / 32, l = q % 32;
                            ln[q] = (uint8_t)(off32[r + 1] - off32[r]);
                            for (int32_t k = off32[r]; k < off32[r + 1]; ++k) {
                                const int64_t dst = sb[sl] + (int64_t)(k - off32[r]) * 32 + l;
                                sv[dst] = val_h[k];
                                if (!pat) sc[dst] = col_h[k];
                            }
                        }
                        if (sorted) {
                            TRY(dalloc(&M.sperm, (size_t)M.nrows));
                            CK(cudaMemcpy(M.sperm, order.data(), (size_t)M.nrows * sizeof(int32_t), cudaMemcpyHostToDevice));
                        }
                        TRY(dalloc(&M.sbeg, sb.size()));
                        TRY(dalloc(&M.sval, sv.size()));
                        TRY(dalloc(&M.slen, ln.size()));
                        M.lbytes[pat ? AMG_LAYOUT_SELL_PAT : AMG_LAYOUT_SELL] =
                            (int64_t)sv.size() * (pat ? 8 : 12) + (int64_t)ln.size() + (int64_t)sb.size() * 4 +
                            (sorted ? M.nrows * 4 : 0) + (pat ? M.nrows : 0);
                        CK(cudaMemcpy(M.sbeg, sb.data(), sb.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                        CK(cudaMemcpy(M.sval, sv.data(), sv.size() * sizeof(double), cudaMemcpyHostToDevice));
                        CK(cudaMemcpy(M.slen, ln.data(), ln.size(), cudaMemcpyHostToDevice));
                        if (!pat) {
                            TRY(dalloc(&M.scol, sc.size()));
                            CK(cudaMemcpy(M.scol, sc.data(), sc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                        }
                        int nbs = 0;
                        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbs, (const void *)spmv_sell_fn(EPI_RESID, pat), VEC_SPMV_THREADS, 0));
                        M.sell_grid = (int)std::max<int64_t>(1, std::min<int64_t>((ns + 7) / 8, (int64_t)h->sm_count * std::max(nbs, 1)));
                        h->max_grid = std::max(h->max_grid, M.sell_grid);
                    }
                }
                int nb = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)spmv_vec_fn(EPI_RESID, h->vec_minb), VEC_SPMV_THREADS, 0));
                M.pad_grid = (int)std::max<int64_t>(1, std::min<int64_t>((M.nrows + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS,
                                                                        (int64_t)h->sm_count * std::max(nb, 1)));
                h->max_grid = std::max(h->max_grid, M.pad_grid);
            } else if (!M.dcls && !longrows && h->symm && h->patterns && h->nranks == 1 && M.ncols == M.nrows && !h->lanes_override &&
                       M.nrows >= (int64_t)h->sm_count * h->small_rows_per_sm) {
                // short-row stencil operators (7-point): the symmetric layout alone, pattern ids kept only with it
                std::vector<int32_t> col_h(M.nnz);
                std::vector<double> val_h(M.nnz);
                if (M.nnz) {
                    CK(cudaMemcpy(col_h.data(), M.col, M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
                    CK(cudaMemcpy(val_h.data(), M.val, M.nnz * sizeof(double), cudaMemcpyDeviceToHost));
                }
                std::vector<int32_t> rel, beg;
                std::vector<uint8_t> ids;
                if (pattern_dict(M, off32, col_h, ids, rel, beg)) {
                    M.npat = (int)beg.size() - 1;
                    M.nrel = (int)rel.size();
                    TRY(dalloc(&M.pid, ids.size() + 16));
                    CK(cudaMemcpy(M.pid, ids.data(), ids.size(), cudaMemcpyHostToDevice));
                    TRY(build_symd(h, M, off32, col_h, val_h, ids, rel, beg));
                    if (!M.uval) {
                        cudaFree(M.pid);
                        M.pid = nullptr;
                        M.npat = M.nrel = 0;
                    }
                }
            }
            if (!M.dcls && !M.uval && !longrows && !h->lanes_override && M.nrows >= (int64_t)h->sm_count * h->small_rows_per_sm) {
                // uniform-width SELL-32: rows of <= 16 entries, every slice as wide as the widest row
                int W = 0;
                for (int64_t r = 0; r < M.nrows; ++r) W = std::max(W, off32[r + 1] - off32[r]);
                const int64_t ns = (M.nrows + 31) / 32;
                const bool plen = h->sellu_short && W <= 8 && (double)ns * 32 * W > 1.10 * (double)M.nnz;
                if (W >= 1 && W <= 16 && ((double)ns * 32 * W <= 1.10 * (double)M.nnz || plen) && ns * 32 * W < INT32_MAX - 64) {
                    std::vector<int32_t> col_h(M.nnz);
                    std::vector<double> val_h(M.nnz);
                    if (M.nnz) {
                        CK(cudaMemcpy(col_h.data(), M.col, M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
                        CK(cudaMemcpy(val_h.data(), M.val, M.nnz * sizeof(double), cudaMemcpyDeviceToHost));
                    }
                    const size_t tot = (size_t)ns * 32 * W;
                    std::vector<double> sv(tot, 0.0);
                    std::vector<int32_t> sc(tot, 0);
                    std::vector<uint8_t> ln(ns * 32 + 16, 0);
                    // skipped padding (plen): rows sorted by length inside each slice, so the live
                    // lanes of a slot are a prefix and dead lanes cost no sectors
                    const bool sorted = plen && h->sellu_sort;
                    std::vector<uint8_t> pm(sorted ? ns * 32 + 16 : 0, 0);
                    for (int64_t sl = 0; sl < ns; ++sl) {
                      int ord[32];
                      for (int l = 0; l < 32; ++l) ord[l] = l;
                      auto rl = [&](int l) { return sl * 32 + l < M.nrows ? off32[sl * 32 + l + 1] - off32[sl * 32 + l] : -1; };
                      if (sorted) std::stable_sort(ord, ord + 32, [&](int x1, int x2) { return rl(x1) > rl(x2); });
                      for (int l = 0; l < 32; ++l) {
                        const int64_t r = sl * 32 + ord[l];   // row held by slot sl * 32 + l
                        if (sorted) pm[sl * 32 + l] = (uint8_t)ord[l];
                        if (r >= M.nrows) continue;
                        const int32_t len = off32[r + 1] - off32[r];
                        ln[sl * 32 + l] = (uint8_t)len;
                        const int64_t b0 = sl * 32 * W + l;
                        for (int32_t k = 0; k < W; ++k) {
                            const int64_t q = b0 + 32 * (int64_t)k;
                            if (k < len) {
                                sv[q] = val_h[off32[r] + k];
                                sc[q] = col_h[off32[r] + k];
                            } else {
                                sc[q] = (int32_t)std::min<int64_t>(r, M.ncols - 1);  // padding: any valid column
                            }
                        }
                      }
                    }
                    if (sorted) {
                        TRY(dalloc(&M.uperm_s, pm.size()));
                        CK(cudaMemcpy(M.uperm_s, pm.data(), pm.size(), cudaMemcpyHostToDevice));
                    }
                    bool vd = false, vd2 = false;
                    if ((plen || W <= 9) && h->sellu_vdict) {
                        // value-tuple classes: rows whose values (bit patterns, in order) coincide share a class
                        const int fl = sellu_fl(W, plen);
                        std::map<std::vector<uint64_t>, int> cmap;
                        std::vector<uint8_t> cl(ns * 32 + 16, 0);
                        std::vector<double> vt;
                        std::vector<int32_t> vl;
                        vd = true;
                        std::vector<uint64_t> key;
                        for (int64_t sl = 0; sl < ns && vd; ++sl)
                            for (int l = 0; l < 32; ++l) {
                                const int64_t r = sl * 32 + (sorted ? pm[sl * 32 + l] : l);
                                const int32_t len = r < M.nrows ? off32[r + 1] - off32[r] : 0;
                                key.assign((size_t)len, 0);
                                for (int32_t k2 = 0; k2 < len; ++k2) memcpy(&key[k2], &val_h[off32[r] + k2], 8);
                                auto it = cmap.find(key);
                                if (it == cmap.end()) {
                                    if (cmap.size() >= 255) { vd = false; break; }
                                    it = cmap.emplace(key, (int)cmap.size()).first;
                                    vl.push_back(len);
                                    for (int k2 = 0; k2 < fl; ++k2) vt.push_back(k2 < len ? val_h[off32[r] + k2] : 0.0);
                                }
                                cl[sl * 32 + l] = (uint8_t)it->second;
                            }
                        if (!vd) {
                            // too many tuples: <= 256 distinct values -> one value id per stored entry
                            std::map<uint64_t, int> vmap;
                            std::vector<double> tab;
                            std::vector<uint8_t> vi(tot + 16, 0);
                            bool ok = true;
                            for (size_t q2 = 0; q2 < tot && ok; ++q2) {
                                uint64_t bits;
                                memcpy(&bits, &sv[q2], 8);
                                auto it = vmap.find(bits);
                                if (it == vmap.end()) {
                                    if (vmap.size() >= 256) { ok = false; break; }
                                    it = vmap.emplace(bits, (int)vmap.size()).first;
                                    tab.push_back(sv[q2]);
                                }
                                vi[q2] = (uint8_t)it->second;
                            }
                            if (ok) {
                                vd2 = true;
                                M.uncls = (int)tab.size();
                                TRY(dalloc(&M.uvid_s, vi.size()));
                                TRY(dalloc(&M.uvtab, tab.size()));
                                CK(cudaMemcpy(M.uvid_s, vi.data(), vi.size(), cudaMemcpyHostToDevice));
                                CK(cudaMemcpy(M.uvtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
                            }
                        }
                        if (vd) {
                            M.uncls = (int)cmap.size();
                            TRY(dalloc(&M.ucls_s, cl.size()));
                            TRY(dalloc(&M.uvtab, vt.size()));
                            TRY(dalloc(&M.uvlen, vl.size()));
                            CK(cudaMemcpy(M.ucls_s, cl.data(), cl.size(), cudaMemcpyHostToDevice));
                            CK(cudaMemcpy(M.uvtab, vt.data(), vt.size() * sizeof(double), cudaMemcpyHostToDevice));
                            CK(cudaMemcpy(M.uvlen, vl.data(), vl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                        }
                    }
                    TRY(dalloc(&M.uval_s, tot));
                    TRY(dalloc(&M.ucol_s, tot));
                    TRY(dalloc(&M.ulen_s, ln.size()));
                    // padding slots are loaded unless skipped (plen)
                    M.lbytes[AMG_LAYOUT_SELL_UNIFORM] = vd2 ? (plen ? M.nnz : (int64_t)tot) * 5 + (int64_t)M.nrows * (sorted ? 2 : 1)  // columns + value ids + length (+ perm)
                                                          : vd ? (plen ? M.nnz : (int64_t)tot) * 4 + (int64_t)M.nrows * (sorted ? 2 : 1)  // columns + class (+ perm)
                                                          : (plen ? M.nnz : (int64_t)tot) * 12 + (int64_t)M.nrows * (sorted ? 2 : 1);
                    CK(cudaMemcpy(M.uval_s, sv.data(), tot * sizeof(double), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.ucol_s, sc.data(), tot * sizeof(int32_t), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.ulen_s, ln.data(), ln.size(), cudaMemcpyHostToDevice));
                    M.uW = W;
                    M.u_plen = plen ? 1 : 0;
                    int nbu = 0;
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbu, (const void *)spmv_sellu_fn(EPI_RESID, W, plen, vd ? 1 : vd2 ? 2 : 0),
                                                                     VEC_SPMV_THREADS, sellu_vd_bytes(M)));
                    M.u_grid = (int)std::max<int64_t>(1, std::min<int64_t>((M.nrows + VEC_SPMV_THREADS - 1) / VEC_SPMV_THREADS,
                                                                          (int64_t)h->sm_count * std::max(nbu, 1)));
                    h->max_grid = std::max(h->max_grid, M.u_grid);
                }
            }
            if (!M.dcls && !M.uval && !M.uval_s && h->sells && !longrows && !h->lanes_override && h->sells_sigma >= 32 &&
                M.nrows >= (int64_t)h->sm_count * h->small_rows_per_sm &&
                (M.nrows <= h->sells_max_rows || h->sells_buckets) &&
                (double)M.nnz >= h->sells_min_avg * (double)M.nrows) {
                // sorted SELL-32: taken where natural slices pad > 10% and sorted ones <= 10%
                const int64_t ns = (M.nrows + 31) / 32;
                int64_t nat = 0, maxlen = 0;
                for (int64_t sl = 0; sl < ns; ++sl) {
                    int w = 0;
                    for (int64_t r = sl * 32; r < std::min<int64_t>(M.nrows, sl * 32 + 32); ++r) w = std::max(w, off32[r + 1] - off32[r]);
                    nat += 32 * (int64_t)w;
                    maxlen = std::max<int64_t>(maxlen, w);
                }
                std::vector<int32_t> order(M.nrows);
                for (int64_t r = 0; r < M.nrows; ++r) order[r] = (int32_t)r;
                const bool bucket = M.nrows > h->sells_max_rows;
                if (bucket) {
                    // fine-level rows: stable partition by the number of 8-entry rounds the row needs
                    // (1 | 2 | 3 | more), rows keep their order inside a bucket, so lanes stay on
                    // neighbouring rows (the x gathers keep their locality) while a warp's rows need
                    // about the same number of rounds
                    auto bk = [&](int32_t r) {
                        const int n1 = off32[r + 1] - off32[r] - 1;
                        return n1 < 8 ? 0 : std::min(1 + (n1 - 8) / 8, h->sells_buckets);
                    };
                    std::stable_sort(order.begin(), order.end(), [&](int32_t x1, int32_t x2) { return bk(x1) < bk(x2); });
                }
                for (int64_t w0 = 0; w0 < M.nrows && !bucket; w0 += h->sells_sigma) {
                    const int64_t w1 = std::min<int64_t>(M.nrows, w0 + h->sells_sigma);
                    std::stable_sort(order.begin() + w0, order.begin() + w1, [&](int32_t x1, int32_t x2) {
                        return off32[x1 + 1] - off32[x1] > off32[x2 + 1] - off32[x2];
                    });
                }
                std::vector<int32_t> sb(ns + 1);
                std::vector<uint8_t> sw(ns + 1, 0);
                int64_t tot = 0;
                for (int64_t sl = 0; sl < ns; ++sl) {
                    int w = 0;
                    for (int64_t p = sl * 32; p < std::min<int64_t>(M.nrows, sl * 32 + 32); ++p)
                        w = std::max(w, off32[order[p] + 1] - off32[order[p]]);
                    sb[sl] = (int32_t)tot;
                    sw[sl] = (uint8_t)w;
                    tot += 32 * (int64_t)w;
                }
                sb[ns] = (int32_t)tot;
                if (maxlen <= 129 && nat > (int64_t)(1.10 * (double)M.nnz) &&
                    tot <= (int64_t)((1.0 + h->sells_max_pad / 100.0) * (double)M.nnz) &&
                    tot < INT32_MAX - 64) {
                    std::vector<int32_t> col_h(M.nnz);
                    std::vector<double> val_h(M.nnz);
                    if (M.nnz) {
                        CK(cudaMemcpy(col_h.data(), M.col, M.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
                        CK(cudaMemcpy(val_h.data(), M.val, M.nnz * sizeof(double), cudaMemcpyDeviceToHost));
                    }
                    std::vector<double> sv(tot + 32, 0.0);
                    std::vector<int32_t> sc(tot + 32, 0);
                    std::vector<uint8_t> ln(ns * 32 + 16, 0);
                    std::vector<int32_t> pm(ns * 32 + 16, 0);
                    for (int64_t p = 0; p < M.nrows; ++p) {
                        const int64_t r = order[p], sl = p / 32, l = p % 32;
                        const int32_t len = off32[r + 1] - off32[r];
                        ln[p] = (uint8_t)len;
                        pm[p] = (int32_t)r;
                        for (int32_t k = 0; k < sw[sl]; ++k) {
                            const int64_t q = sb[sl] + 32 * (int64_t)k + l;
                            if (k < len) {
                                sv[q] = val_h[off32[r] + k];
                                sc[q] = col_h[off32[r] + k];
                            } else {
                                sc[q] = (int32_t)std::min<int64_t>(r, M.ncols - 1);
                            }
                        }
                    }
                    TRY(dalloc(&M.sv_s, sv.size()));
                    TRY(dalloc(&M.sc_s, sc.size()));
                    // padding slots are never loaded: entries + slice starts/widths + row permutation + lengths
                    M.lbytes[AMG_LAYOUT_SELL_SORTED] = M.nnz * 12 + (int64_t)sb.size() * 4 + (int64_t)sw.size() +
                                                        (int64_t)pm.size() * 4 + (int64_t)ln.size();
                    TRY(dalloc(&M.sb_s, sb.size()));
                    TRY(dalloc(&M.sw_s, sw.size()));
                    TRY(dalloc(&M.sp_s, pm.size()));
                    TRY(dalloc(&M.sl_s, ln.size()));
                    CK(cudaMemcpy(M.sv_s, sv.data(), sv.size() * sizeof(double), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.sc_s, sc.data(), sc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.sb_s, sb.data(), sb.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.sw_s, sw.data(), sw.size(), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.sp_s, pm.data(), pm.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(M.sl_s, ln.data(), ln.size(), cudaMemcpyHostToDevice));
                    int nbs = 0;
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbs, (const void *)spmv_sells_fn(EPI_RESID, h->sells_plen),
                                                                     VEC_SPMV_THREADS, 0));
                    M.s_grid = (int)std::max<int64_t>(1, std::min<int64_t>((ns + 7) / 8, (int64_t)h->sm_count * std::max(nbs, 1)));
                    h->max_grid = std::max(h->max_grid, M.s_grid);
                }
            }
            const double avg = M.nrows ? (double)M.nnz / (double)M.nrows : 0.0;
            // direct kernel: one lane per row maximises rows in flight (measured on
            // B200: 27-pt A 3.5 TB/s at 1 lane vs 2.4 at 4); wide rows split over lanes
            // small matrices (fewer rows than ~2 CTAs/SM of one-lane rows) spread each row over
            // more lanes: the dependent load chain per lane shrinks and more SMs take part
            const bool small = M.nrows < (int64_t)h->sm_count * h->small_rows_per_sm;
            M.lanes = h->lanes_override ? h->lanes_override
                      : small ? (avg >= 16.0 ? 8 : avg >= 6.0 ? 4 : 2) : (avg < 48.0 ? 1 : avg < 96.0 ? 4 : 8);
        }
    }
    // vectors: capacity = local rows + the largest halo feeding a matrix on that level's column space
    int64_t nmax = 0;
    for (int k = 0; k < nl; ++k) {
        LevelD &L = h->lv[k];
        int64_t cap = L.n;
        for (int w = 0; w < 5; ++w)
            if (L.m[w].present && (w != AMG_P || container)) cap = std::max(cap, std::max(L.m[w].ncols, L.m[w].nrows));
        if (k > 0 && h->lv[k - 1].m[AMG_P].present) cap = std::max(cap, h->lv[k - 1].m[AMG_P].ncols);
        if (k == nl - 1) cap = std::max<int64_t>(cap, h->nc);
        L.cap = cap + 2;
        TRY(dalloc(&L.y, L.cap));
        TRY(dalloc(&L.x, L.cap));
        TRY(dalloc(&L.r, L.cap));
        TRY(dalloc(&L.t, L.cap));
        nmax = std::max(nmax, L.cap);
    }
    const int64_t c0 = h->lv[0].cap;
    TRY(dalloc(&h->b, c0));
    TRY(dalloc(&h->x, c0));
    TRY(dalloc(&h->r, c0));
    TRY(dalloc(&h->z, c0));
    TRY(dalloc(&h->p, c0));
    TRY(dalloc(&h->q, c0));
    TRY(dalloc(&h->tmp_in, nmax));
    TRY(dalloc(&h->tmp_out, nmax));
    TRY(dalloc(&h->partials, 2 * (size_t)h->max_grid));  // two-launch (interior / boundary) reductions
    TRY(dalloc(&h->ticket, 4));
    TRY(dalloc(&h->ctl, 1));
    CK(cudaMallocHost((void **)&h->ctl_h, sizeof(PcgCtl)));
    std::memset(h->ctl_h, 0, sizeof(PcgCtl));
    if (h->tail_grid) h->cluster = h->sm_count;  // one CTA per SM (512 threads x 128 registers fill an SM)
    if (!container) TRY(build_tail(h));
    h->finalized = true;
    CK(cudaDeviceSynchronize());
    return AMG_OK;
}

static int check_final(amg_t *h)
{
    if (!h) return fail(AMG_E_ARG, "NULL handle");
    if (!h->finalized) return fail(AMG_E_STATE, "handle is not finalized (call amg_finalize)");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return fail(AMG_E_CUDA, cudaGetErrorString(e));
    return AMG_OK;
}

static int to_dev(amg_t *h, double *dst, const double *src, int64_t n, int on_device)
{
    if (n == 0) return AMG_OK;
    CK(cudaMemcpyAsync(dst, src, n * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
    return AMG_OK;
}

static int from_dev(amg_t *h, double *dst, const double *src, int64_t n, int on_device)
{
    if (n == 0) return AMG_OK;
    CK(cudaMemcpyAsync(dst, src, n * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
    return AMG_OK;
}

static int sync_stream(amg_t *h)
{
    CK(cudaStreamSynchronize(h->stream));
    return AMG_OK;
}

int amg_spmv(amg_t *h, int level, int which, const double *x, double *y, int on_device)
{
    TRY(check_final(h));
    if (level < 0 || level >= (int)h->lv.size() || which < 0 || which > 4) return fail(AMG_E_ARG, "amg_spmv: bad level / slot");
    const DevMat &M = h->lv[level].m[which];
    if (!M.present) return fail(AMG_E_ARG, "amg_spmv: matrix slot is empty");
    if (!x || !y) return fail(AMG_E_ARG, "amg_spmv: NULL vector");
    const int64_t xn = M.n_own;  // owned column slice (all columns on one rank / replicated levels)
    TRY(to_dev(h, h->tmp_in, x, xn, on_device));
    TRY(launch_spmv(h, M, h->tmp_in, h->tmp_out, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, nullptr, nullptr));
    TRY(from_dev(h, y, h->tmp_out, M.nrows, on_device));
    return sync_stream(h);
}

int amg_smoother(amg_t *h, int level, const double *b, const double *x0, double *x, int steps, int on_device)
{
    TRY(check_final(h));
    if (h->container) return fail(AMG_E_STATE, "matrix container handle: no hierarchy uploaded");
    if (level < 0 || level >= (int)h->lv.size() - 1) return fail(AMG_E_ARG, "amg_smoother: level has no smoother");
    if (!b || !x || steps < 0) return fail(AMG_E_ARG, "amg_smoother: bad arguments");
    LevelD &L = h->lv[level];
    TRY(to_dev(h, h->tmp_in, b, L.n, on_device));
    if (x0) TRY(to_dev(h, h->tmp_out, x0, L.n, on_device));
    else CK(cudaMemsetAsync(h->tmp_out, 0, L.n * sizeof(double), h->stream));
    TRY(enqueue_smooth(h, level, h->tmp_in, h->tmp_out, steps, x0 == nullptr, nullptr, FIN_NONE, nullptr));
    TRY(from_dev(h, x, h->tmp_out, L.n, on_device));
    return sync_stream(h);
}

int amg_coarse_solve(amg_t *h, const double *y, double *z, int on_device)
{
    TRY(check_final(h));
    if (h->container) return fail(AMG_E_STATE, "matrix container handle: no hierarchy uploaded");
    if (!y || !z) return fail(AMG_E_ARG, "amg_coarse_solve: NULL vector");
    TRY(to_dev(h, h->tmp_in, y, h->nc, on_device));
    TRY(launch_coarse(h, h->tmp_in, h->tmp_out, nullptr, FIN_NONE, nullptr));
    TRY(from_dev(h, z, h->tmp_out, h->nc, on_device));
    return sync_stream(h);
}

int amg_vcycle(amg_t *h, const double *y, double *z, int on_device)
{
    TRY(check_final(h));
    if (h->container) return fail(AMG_E_STATE, "matrix container handle: no hierarchy uploaded");
    if (!y || !z) return fail(AMG_E_ARG, "amg_vcycle: NULL vector");
    const int64_t n = h->lv[0].n;
    TRY(to_dev(h, h->tmp_in, y, n, on_device));
    TRY(enqueue_vcycle(h, 0, h->tmp_in, h->tmp_out, nullptr, FIN_NONE, nullptr));
    TRY(from_dev(h, z, h->tmp_out, n, on_device));
    TRY(sync_stream(h));
    if (h->trace) {
        std::vector<unsigned long long> t(h->tail_nops + 1);
        CK(cudaMemcpy(t.data(), h->trace, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        std::vector<TailOp> ops(h->tail_nops);
        CK(cudaMemcpy(ops.data(), h->tail_ops, ops.size() * sizeof(TailOp), cudaMemcpyDeviceToHost));
        fprintf(stderr, "[amgb200 trace] tail from level %d, %d ops, cluster %d:", h->tail_level, h->tail_nops, h->cluster);
        for (int i = 0; i < h->tail_nops; ++i)
            fprintf(stderr, " %s%d/%d:%.2fus", ops[i].kind == TAIL_SPMV ? "spmv" : ops[i].kind == TAIL_JACOBI ? "jac" : "coarse",
                    ops[i].epi, ops[i].nrows, (t[i + 1] - t[i]) * 1e-3);
        fprintf(stderr, " total %.2fus\n", (t[h->tail_nops] - t[0]) * 1e-3);
    }
    return AMG_OK;
}

int amg_vcycle_level(amg_t *h, int level, const double *y, double *z, int on_device)
{
    TRY(check_final(h));
    if (h->container) return fail(AMG_E_STATE, "matrix container handle: no hierarchy uploaded");
    if (!y || !z) return fail(AMG_E_ARG, "amg_vcycle_level: NULL vector");
    const int nl = (int)h->lv.size();
    if (level < 0 || level >= nl) return fail(AMG_E_ARG, "amg_vcycle_level: level out of range");
    if (h->nranks > 1 && level > 0) return fail(AMG_E_STATE, "amg_vcycle_level: level > 0 needs a single-GPU handle");
    if (h->tail_level > 0 && level > h->tail_level)
        return fail(AMG_E_STATE, "amg_vcycle_level: levels below the first cluster-tail level run inside the tail kernel "
                                 "(start at or above it, or set option tail_nnz = 0)");
    const int64_t n = h->lv[level].n;
    if (h->tail_level > 0 && level == h->tail_level) {
        // the tail kernel works on the level's own vectors
        TRY(to_dev(h, h->lv[level].y, y, n, on_device));
        TRY(enqueue_vcycle(h, level, h->lv[level].y, h->lv[level].x, nullptr, FIN_NONE, nullptr));
        TRY(from_dev(h, z, h->lv[level].x, n, on_device));
    } else {
        TRY(to_dev(h, h->tmp_in, y, n, on_device));
        TRY(enqueue_vcycle(h, level, h->tmp_in, h->tmp_out, nullptr, FIN_NONE, nullptr));
        TRY(from_dev(h, z, h->tmp_out, n, on_device));
    }
    TRY(sync_stream(h));
    return AMG_OK;
}

int amg_pcg(amg_t *h, const double *b, const double *x0, double rtol, int max_iters, int recompute_every,
            double *x_out, int *n_iter, double *relres, int *converged, double *history, int *hist_len,
            double *curvature_at_fail, int on_device)
{
    auto t_start = std::chrono::steady_clock::now();
    TRY(check_final(h));
    if (h->container) return fail(AMG_E_STATE, "matrix container handle: no hierarchy uploaded");
    if (!b || !x_out || !n_iter || !relres || !converged) return fail(AMG_E_ARG, "amg_pcg: NULL argument");
    if (max_iters < 0 || recompute_every < 1) return fail(AMG_E_ARG, "amg_pcg: bad max_iters / recompute_every");
    const int64_t n = h->lv[0].n;
    const int64_t launches0 = h->launches;
    if (history) {
        if (h->hist_cap < max_iters + 1) {
            if (h->hist) cudaFree(h->hist);
            h->hist = nullptr;
            TRY(dalloc(&h->hist, (size_t)max_iters + 1));
            h->hist_cap = max_iters + 1;
        }
    }
    TRY(build_graph(h));
    PcgCtl c{};
    c.active = 1;
    c.max_iters = max_iters;
    c.recompute_every = recompute_every;
    c.record = history ? 1 : 0;
    c.rtol = rtol;
    c.hist = h->hist;
    *h->ctl_h = c;
    CK(cudaEventRecord(h->ev0, h->stream));
    CK(cudaMemcpyAsync(h->ctl, h->ctl_h, sizeof(PcgCtl), cudaMemcpyHostToDevice, h->stream));
    TRY(to_dev(h, h->b, b, n, on_device));
    if (x0) TRY(to_dev(h, h->x, x0, n, on_device));
    else CK(cudaMemsetAsync(h->x, 0, n * sizeof(double), h->stream));
    // bnorm = ||b||; b == 0 returns zeros (krylov.py:50-53)
    TRY(launch_dot(h, h->b, h->b, n, FIN_BNORM, nullptr, nullptr));
    CK(cudaMemcpyAsync(h->ctl_h, h->ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, h->stream));
    TRY(sync_stream(h));
    if (h->ctl_h->bnorm == 0.0) {
        CK(cudaMemsetAsync(h->x, 0, n * sizeof(double), h->stream));
        TRY(from_dev(h, x_out, h->x, n, on_device));
        TRY(sync_stream(h));
        *n_iter = 0;
        *relres = 0.0;
        *converged = 1;
        if (hist_len) *hist_len = 0;
        h->solve_ms = 0.0;
        return AMG_OK;
    }
    const LevelD &L0 = h->lv[0];
    const int *act = &h->ctl->active;
    // r = b - A x ; relres_0 ; z = M r ; rz = r.z ; p = z     (krylov.py:55-63)
    TRY(launch_spmv(h, L0.m[AMG_A], h->x, h->r, EPI_RESID, h->b, 0.0, h->r, FIN_INIT_RES, nullptr, nullptr));
    TRY(enqueue_vcycle(h, 0, h->r, h->z, nullptr, FIN_INIT_RZ, h->r));
    TRY(launch_copy(h, h->p, h->z, n, nullptr));
    (void)act;
    if (max_iters > 0) {
        if (h->graph_mode == 2) {
            CK(cudaGraphLaunch(h->gexec, h->stream));
            ++h->launches;
        } else {
            // batched launches of the iteration graph, host checks every `batch`
            for (;;) {
                for (int i = 0; i < h->batch; ++i) {
                    if (h->graph_mode == 1) CK(cudaGraphLaunch(h->gexec, h->stream));
                    else { cudaGraphConditionalHandle d{}; TRY(enqueue_pcg_body(h, d, 0)); }
                }
                CK(cudaMemcpyAsync(h->ctl_h, h->ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, h->stream));
                TRY(sync_stream(h));
                if (!h->ctl_h->active) break;
            }
        }
    }
    CK(cudaMemcpyAsync(h->ctl_h, h->ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    TRY(from_dev(h, x_out, h->x, n, on_device));
    TRY(sync_stream(h));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->solve_ms = ms;
    const PcgCtl &r = *h->ctl_h;
    int iters = r.it;
    if (h->graph_mode == 2) h->launches += (int64_t)std::max(iters, 1) * h->launches_per_iter;
    else if (h->graph_mode == 1) h->launches += (int64_t)std::max(iters, 1) * h->launches_per_iter;
    h->launches_last = h->launches - launches0;
    *n_iter = iters;
    *relres = r.relres;
    *converged = r.converged;
    if (history && hist_len) {
        int hl = r.record ? (iters + 1) : 0;
        if (r.status == 3) hl = iters;  // failing iteration appended nothing
        hl = std::min(hl, max_iters + 1);
        if (hl > 0) CK(cudaMemcpy(history, h->hist, hl * sizeof(double), cudaMemcpyDeviceToHost));
        *hist_len = hl;
    }
    h->e2e_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    if (r.status == 3) {
        if (curvature_at_fail) *curvature_at_fail = r.curv_fail;
        char buf[160];
        snprintf(buf, sizeof(buf), "iteration %d: direction with curvature %.3e; operator is not symmetric positive definite",
                 iters, r.curv_fail);
        return fail(AMG_E_NOT_SPD, buf);
    }
    return AMG_OK;
}

int amg_time_spmv(amg_t *h, int level, int which, int reps, double *ms_per_launch)
{
    TRY(check_final(h));
    if (level == -1 && reps >= 1 && ms_per_launch && !h->container) {  // diagnostics: the coarsest solve
        TRY(launch_coarse(h, h->tmp_in, h->tmp_out, nullptr, FIN_NONE, nullptr));
        CK(cudaEventRecord(h->ev0, h->stream));
        for (int i = 0; i < reps; ++i) TRY(launch_coarse(h, h->tmp_in, h->tmp_out, nullptr, FIN_NONE, nullptr));
        CK(cudaEventRecord(h->ev1, h->stream));
        TRY(sync_stream(h));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        *ms_per_launch = ms / reps;
        return AMG_OK;
    }
    if (which == 5 && level >= 0 && level + 1 < (int)h->lv.size() && reps >= 1 && ms_per_launch && !h->container) {
        // diagnostics: one smoother step from zero (x = w M^-1 b) at `level`
        TRY(enqueue_smooth(h, level, h->tmp_in, h->tmp_out, 1, true, nullptr, FIN_NONE, nullptr));
        CK(cudaEventRecord(h->ev0, h->stream));
        for (int i = 0; i < reps; ++i) TRY(enqueue_smooth(h, level, h->tmp_in, h->tmp_out, 1, true, nullptr, FIN_NONE, nullptr));
        CK(cudaEventRecord(h->ev1, h->stream));
        TRY(sync_stream(h));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        *ms_per_launch = ms / reps;
        return AMG_OK;
    }
    if (level < 0 || level >= (int)h->lv.size() || which < 0 || which > 4 || reps < 1 || !ms_per_launch)
        return fail(AMG_E_ARG, "amg_time_spmv: bad arguments");
    const DevMat &M = h->lv[level].m[which];
    if (!M.present) return fail(AMG_E_ARG, "amg_time_spmv: matrix slot is empty");
    TRY(launch_spmv(h, M, h->tmp_in, h->tmp_out, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, nullptr, nullptr));
    CK(cudaEventRecord(h->ev0, h->stream));
    for (int i = 0; i < reps; ++i)
        TRY(launch_spmv(h, M, h->tmp_in, h->tmp_out, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, nullptr, nullptr));
    CK(cudaEventRecord(h->ev1, h->stream));
    TRY(sync_stream(h));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    *ms_per_launch = ms / reps;
    return AMG_OK;
}

// ------------------------------------------------------------------ BiCGstab

static int dev_dot(amg_t *h, const double *a, const double *b, int64_t n, double *out)
{
    TRY(launch_dot(h, a, b, n, FIN_STORE, nullptr, nullptr));
    CK(cudaMemcpyAsync(&h->ctl_h->scratch, &h->ctl->scratch, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    TRY(sync_stream(h));
    *out = h->ctl_h->scratch;
    return AMG_OK;
}

static int bicg_op(amg_t *h, int mode, double *x, const double *p, const double *q, double alpha, double beta,
                   double omega)
{
    BicgArgs a{};
    a.n = h->lv[0].n;
    a.x = x;
    a.p = p;
    a.q = q;
    a.alpha = alpha;
    a.beta = beta;
    a.omega = omega;
    a.mode = mode;
    TRY(launch_k(h, bicg_update, vec_grid(h, a.n), VEC_THREADS, 0, a));
    return AMG_OK;
}

int amg_bicgstab(amg_t *h, const double *b, const double *x0, double rtol, int max_iters, int recompute_every,
                 double *x_out, int *n_iter, double *relres_out, int *converged, int *restarts_out,
                 double *history, int *hist_len, int on_device)
{
    auto t_start = std::chrono::steady_clock::now();
    TRY(check_final(h));
    if (h->container) return fail(AMG_E_STATE, "matrix container handle: no hierarchy uploaded");
    if (!b || !x_out || !n_iter || !relres_out || !converged) return fail(AMG_E_ARG, "amg_bicgstab: NULL argument");
    if (max_iters < 0 || recompute_every < 1) return fail(AMG_E_ARG, "amg_bicgstab: bad max_iters / recompute_every");
    const int64_t n = h->lv[0].n;
    const int64_t cap = h->lv[0].cap;
    for (auto *&bp : h->bicg)
        if (!bp) TRY(dalloc(&bp, cap));
    double *r = h->r, *x = h->x, *bb = h->b, *p = h->p;
    double *rs = h->bicg[0], *v = h->bicg[1], *phat = h->bicg[2], *sv = h->bicg[3], *shat = h->bicg[4],
           *t = h->bicg[5];
    const DevMat &A = h->lv[0].m[AMG_A];
    std::vector<double> hist;
    int hl = 0, restarts = 0;
    auto finish = [&](int its, double rr, int conv) -> int {
        TRY(from_dev(h, x_out, x, n, on_device));
        TRY(sync_stream(h));
        *n_iter = its;
        *relres_out = rr;
        *converged = conv;
        if (restarts_out) *restarts_out = restarts;
        if (history && hist_len) {
            hl = (int)std::min<size_t>(hist.size(), (size_t)max_iters + 1);
            for (int i = 0; i < hl; ++i) history[i] = hist[i];
            *hist_len = hl;
        }
        h->e2e_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        return AMG_OK;
    };
    auto resid = [&]() -> int {  // r = b - A x
        return launch_spmv(h, A, x, r, EPI_RESID, bb, 0.0, nullptr, FIN_NONE, nullptr, nullptr);
    };
    auto norm = [&](const double *a, double *out) -> int {
        double d = 0.0;
        TRY(dev_dot(h, a, a, n, &d));
        *out = std::sqrt(d);
        return AMG_OK;
    };
    TRY(to_dev(h, bb, b, n, on_device));
    if (x0) TRY(to_dev(h, x, x0, n, on_device));
    else CK(cudaMemsetAsync(x, 0, n * sizeof(double), h->stream));
    double bnorm = 0.0;
    TRY(norm(bb, &bnorm));
    if (bnorm == 0.0) {  // krylov.py:106-109
        CK(cudaMemsetAsync(x, 0, n * sizeof(double), h->stream));
        return finish(0, 0.0, 1);
    }
    TRY(resid());
    CK(cudaMemcpyAsync(rs, r, n * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    CK(cudaMemsetAsync(v, 0, n * sizeof(double), h->stream));
    CK(cudaMemsetAsync(p, 0, n * sizeof(double), h->stream));
    double nr = 0.0;
    TRY(norm(r, &nr));
    double relres = nr / bnorm;
    if (history) hist.push_back(relres);
    if (relres <= rtol) return finish(0, relres, 1);
    const double eps = 2.220446049250313e-16;
    const double eps_break = eps * eps;
    for (int it = 1; it <= max_iters; ++it) {
        double rho_new = 0.0;
        TRY(dev_dot(h, rs, r, n, &rho_new));
        if (std::fabs(rho_new) < eps_break * bnorm * bnorm) {  // krylov.py:125-143
            if (restarts >= 1) {
                TRY(finish(it, relres, 0));
                char buf[128];
                snprintf(buf, sizeof(buf), "iteration %d: shadow product vanished twice (rho=%.3e)", it, rho_new);
                return fail(AMG_E_BREAKDOWN, buf);
            }
            ++restarts;
            TRY(resid());
            TRY(norm(r, &nr));
            relres = nr / bnorm;
            if (relres <= rtol) return finish(it - 1, relres, 1);
            CK(cudaMemcpyAsync(rs, r, n * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
            rho = alpha = omega = 1.0;
            CK(cudaMemsetAsync(v, 0, n * sizeof(double), h->stream));
            CK(cudaMemsetAsync(p, 0, n * sizeof(double), h->stream));
            TRY(dev_dot(h, rs, r, n, &rho_new));
        }
        const double beta = (rho_new / rho) * (alpha / omega);
        rho = rho_new;
        TRY(bicg_op(h, 0, p, r, v, 0.0, beta, omega));                         // p = r + beta (p - omega v)
        TRY(enqueue_vcycle(h, 0, p, phat, nullptr, FIN_NONE, nullptr));        // phat = M p
        TRY(launch_spmv(h, A, phat, v, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, nullptr, nullptr));
        double denom = 0.0;
        TRY(dev_dot(h, rs, v, n, &denom));
        if (denom == 0.0) {
            TRY(finish(it, relres, 0));
            return fail(AMG_E_BREAKDOWN, "iteration " + std::to_string(it) + ": stagnated (shadow direction orthogonal)");
        }
        alpha = rho / denom;
        TRY(bicg_op(h, 1, sv, r, v, alpha, 0.0, 0.0));                         // s = r - alpha v
        double ns = 0.0;
        TRY(norm(sv, &ns));
        if (ns / bnorm <= rtol) {                                                // krylov.py:154-165
            TRY(bicg_op(h, 4, x, phat, nullptr, alpha, 0.0, 0.0));
            TRY(resid());
            TRY(norm(r, &nr));
            relres = nr / bnorm;
            if (history) hist.push_back(relres);
            if (relres <= rtol) return finish(it, relres, 1);
            continue;
        }
        TRY(enqueue_vcycle(h, 0, sv, shat, nullptr, FIN_NONE, nullptr));      // shat = M s
        TRY(launch_spmv(h, A, shat, t, EPI_PLAIN, nullptr, 0.0, nullptr, FIN_NONE, nullptr, nullptr));
        double tt = 0.0, ts = 0.0;
        TRY(dev_dot(h, t, t, n, &tt));
        if (tt == 0.0) {
            TRY(finish(it, relres, 0));
            return fail(AMG_E_BREAKDOWN, "iteration " + std::to_string(it) + ": t vanished");
        }
        TRY(dev_dot(h, t, sv, n, &ts));
        omega = ts / tt;
        TRY(bicg_op(h, 2, x, phat, shat, alpha, 0.0, omega));                  // x += alpha phat + omega shat
        TRY(bicg_op(h, 3, r, sv, t, 0.0, 0.0, omega));                         // r = s - omega t
        if (it % recompute_every == 0) TRY(resid());
        TRY(norm(r, &nr));
        relres = nr / bnorm;
        if (history) hist.push_back(relres);
        if (relres <= rtol) {
            TRY(resid());
            TRY(norm(r, &nr));
            relres = nr / bnorm;
            if (relres <= rtol) return finish(it, relres, 1);
        }
        if (omega == 0.0) {
            TRY(finish(it, relres, 0));
            return fail(AMG_E_BREAKDOWN, "iteration " + std::to_string(it) + ": omega vanished");
        }
    }
    return finish(max_iters, relres, 0);
}

int amg_matrix_layout(amg_t *h, int level, int which, int *layout)
{
    if (!h || !layout) return fail(AMG_E_ARG, "amg_matrix_layout: NULL argument");
    if (!h->finalized) return fail(AMG_E_STATE, "amg_matrix_layout: handle not finalized");
    if (level < 0 || level >= (int)h->lv.size() || which < 0 || which > 4)
        return fail(AMG_E_ARG, "amg_matrix_layout: level/which out of range");
    const DevMat &M = h->lv[level].m[which];
    if (!M.present) return fail(AMG_E_ARG, "amg_matrix_layout: matrix not uploaded");
    *layout = layout_of(h, M);
    return AMG_OK;
}

int amg_matrix_bytes(amg_t *h, int level, int which, int64_t *stored, int64_t *vectors)
{
    if (!h || !stored || !vectors) return fail(AMG_E_ARG, "amg_matrix_bytes: NULL argument");
    if (!h->finalized) return fail(AMG_E_STATE, "amg_matrix_bytes: handle not finalized");
    if (level < 0 || level >= (int)h->lv.size() || which < 0 || which > 4)
        return fail(AMG_E_ARG, "amg_matrix_bytes: level/which out of range");
    const DevMat &M = h->lv[level].m[which];
    if (!M.present) return fail(AMG_E_ARG, "amg_matrix_bytes: matrix not uploaded");
    const int lay = layout_of(h, M);
    *stored = (lay == AMG_LAYOUT_CSR || lay == AMG_LAYOUT_LEAVES || M.lbytes[lay] == 0)
                  ? M.nnz * 12 + (M.nrows + 1) * 4
                  : M.lbytes[lay];
    *vectors = 8 * (M.ncols + M.nrows);  // x read once, y written once
    return AMG_OK;
}


int amg_get_stats(amg_t *h, amg_stats_t *out)
{
    if (!h || !out) return fail(AMG_E_ARG, "amg_get_stats: NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->solve_ms = h->solve_ms;
    out->e2e_ms = h->e2e_ms;
    out->launches_per_iter = h->launches_per_iter;
    out->launches_last = h->launches_last;
    out->graph_mode = h->graph_mode;
    out->n_levels = (int)h->lv.size();
    out->tail_level = h->tail_level;
    out->cluster = h->cluster;
    return AMG_OK;
}


// ---------------------------------------------------------------- device setup operators (setup.cuh)

static int setup_device(int device)
{
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0)
        return fail(AMG_E_CUDA, "no CUDA device (there is no CPU fallback)");
    if (device < 0 || device >= count) return fail(AMG_E_ARG, "device index out of range");
    CK(cudaSetDevice(device));
    return AMG_OK;
}

int amg_device_galerkin(int device, int64_t n, int64_t m, const int64_t *a_offsets, const int32_t *a_cols,
                        const double *a_vals, const int64_t *p_offsets, const int32_t *p_cols, const double *p_vals,
                        int symmetrize, amg_csr_result_t **out)
{
    if (!out) return fail(AMG_E_ARG, "amg_device_galerkin: NULL output");
    *out = nullptr;
    TRY(setup_device(device));
    amg_csr_result *r = new amg_csr_result();
    r->device = device;
    const int st = amg_setup::galerkin(r, n, m, a_offsets, a_cols, a_vals, p_offsets, p_cols, p_vals, symmetrize);
    if (st != AMG_OK) {
        delete r;
        return st;
    }
    *out = r;
    return AMG_OK;
}

int amg_device_transpose(int device, int64_t nrows, int64_t ncols, const int64_t *offsets, const int32_t *cols,
                         const double *vals, amg_csr_result_t **out)
{
    if (!out) return fail(AMG_E_ARG, "amg_device_transpose: NULL output");
    *out = nullptr;
    TRY(setup_device(device));
    amg_csr_result *r = new amg_csr_result();
    r->device = device;
    const int st = amg_setup::transpose(r, nrows, ncols, offsets, cols, vals);
    if (st != AMG_OK) {
        delete r;
        return st;
    }
    *out = r;
    return AMG_OK;
}

int amg_csr_result_shape(const amg_csr_result_t *r, int64_t *nrows, int64_t *ncols, int64_t *nnz)
{
    if (!r || !nrows || !ncols || !nnz) return fail(AMG_E_ARG, "amg_csr_result_shape: NULL argument");
    *nrows = r->nrows;
    *ncols = r->ncols;
    *nnz = r->nnz;
    return AMG_OK;
}

int amg_csr_result_fetch(const amg_csr_result_t *r, int64_t *offsets, int32_t *cols, double *vals)
{
    if (!r || !offsets) return fail(AMG_E_ARG, "amg_csr_result_fetch: NULL argument");
    if (r->nnz > 0 && (!cols || !vals)) return fail(AMG_E_ARG, "amg_csr_result_fetch: NULL entry buffers");
    CK(cudaSetDevice(r->device));
    CK(cudaMemcpy(offsets, r->off.p, (r->nrows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (r->nnz) {
        CK(cudaMemcpy(cols, r->col.p, r->nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(vals, r->val.p, r->nnz * sizeof(double), cudaMemcpyDeviceToHost));
    }
    return AMG_OK;
}

void amg_csr_result_free(amg_csr_result_t *r)
{
    if (!r) return;
    cudaSetDevice(r->device);
    delete r;
}

}  // extern "C"
