// Device Galerkin product and transpose: the two setup
// operators a lean hierarchy cache replays on load -- A_{k+1} = P^T A P
// (amgkit/sparse.py:256-282, called at hierarchy.py:210) and P^T / G^T
// (sparse.py:220-224, hierarchy.py:216, smoothers.py:145) -- bit-identical
// to the reference's scipy calls.
//
// scipy's row-by-row SpGEMM (csr_matmat) adds the terms of an output entry
// one at a time, in the order it meets them, onto a zero-initialised
// accumulator, rounding the product first (no FMA), and drops sums that are
// exactly zero:
//   X = A P        : X_ic   = sum over j ascending (A's row i)      of a_ij p_jc
//   R = P^T X      : R_kc   = sum over i ascending (X's column c)   of x_ic p_ik
//                    (csc @ csr: scipy converts X to CSC -- a stable counting
//                    sort, rows ascending inside a column -- and runs the same
//                    kernel on the transposed problem)
//   S = (R + R^T) / 2 when symmetrising, zeros eliminated, canonical CSR.
// Here each product is EXPANDED into (key, term) pairs in exactly that meeting
// order, SORTED by key with a stable radix sort (equal keys keep their
// order), and COMPRESSED by one thread per key adding its terms left to
// right from 0.0 -- the same additions in the same order, in parallel over
// output entries.  Included by capi.cu (shares its error helpers).
#pragma once

#include <cub/cub.cuh>

namespace amg_setup {

template <class T>
struct Buf {
    T *p = nullptr;
    size_t n = 0;
    Buf() = default;
    Buf(const Buf &) = delete;
    Buf &operator=(const Buf &) = delete;
    ~Buf() { release(); }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count)
    {
        release();
        n = count;
        return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
    }
};

constexpr int TB = 256;
inline int blocks(int64_t n) { return (int)std::min<int64_t>((n + TB - 1) / TB, 1 << 20); }

// row id of every entry of a CSR matrix
__global__ void entry_rows(int64_t nrows, const int64_t *__restrict__ off, int32_t *__restrict__ rows)
{
    for (int64_t r = blockIdx.x * (int64_t)TB + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * TB)
        for (int64_t e = off[r]; e < off[r + 1]; ++e) rows[e] = (int32_t)r;
}

// products per left entry: the length of the right matrix's row `mid[e]`
__global__ void expand_counts(int64_t n, const int32_t *__restrict__ mid, const int64_t *__restrict__ boff,
                              int64_t *__restrict__ cnt)
{
    for (int64_t e = blockIdx.x * (int64_t)TB + threadIdx.x; e < n; e += (int64_t)gridDim.x * TB)
        cnt[e] = boff[mid[e] + 1] - boff[mid[e]];
}

// left entry e = (outer[e], mid[e], lv[e]) times every entry (mid[e], c, b) of the right matrix, in the
// right row's order: key = outer << 32 | c, term = lv * b (rounded product), written at pos[e] + t
__global__ void expand_products(int64_t n, const int32_t *__restrict__ outer, const int32_t *__restrict__ mid,
                                const double *__restrict__ lv, const int64_t *__restrict__ pos,
                                const int64_t *__restrict__ boff, const int32_t *__restrict__ bcol,
                                const double *__restrict__ bval, uint64_t *__restrict__ key, double *__restrict__ term)
{
    for (int64_t e = blockIdx.x * (int64_t)TB + threadIdx.x; e < n; e += (int64_t)gridDim.x * TB) {
        const int64_t b0 = boff[mid[e]], b1 = boff[mid[e] + 1];
        const uint64_t hi = (uint64_t)(uint32_t)outer[e] << 32;
        const double v = lv[e];
        int64_t q = pos[e];
        for (int64_t t = b0; t < b1; ++t, ++q) {
            key[q] = hi | (uint32_t)bcol[t];
            term[q] = __dmul_rn(v, bval[t]);
        }
    }
}

__global__ void head_flags(int64_t n, const uint64_t *__restrict__ key, int64_t *__restrict__ flag)
{
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB)
        flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// seg[i] = inclusive scan of the head flags: segment number + 1; heads record their start
__global__ void segment_starts(int64_t n, const uint64_t *__restrict__ key, const int64_t *__restrict__ seg,
                               int64_t *__restrict__ start)
{
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB)
        if (i == 0 || key[i] != key[i - 1]) start[seg[i] - 1] = i;
}

// one thread per key: terms added left to right onto 0.0 (scipy's accumulator), optionally scaled
__global__ void segment_sums(int64_t nseg, int64_t n, const int64_t *__restrict__ start, const uint64_t *__restrict__ key,
                             const double *__restrict__ term, double scale, uint64_t *__restrict__ okey,
                             double *__restrict__ oval, int64_t *__restrict__ keep)
{
    for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * TB) {
        const int64_t b = start[s], e = (s + 1 < nseg) ? start[s + 1] : n;
        double acc = 0.0;
        for (int64_t i = b; i < e; ++i) acc = __dadd_rn(acc, term[i]);
        acc = __dmul_rn(acc, scale);
        okey[s] = key[b];
        oval[s] = acc;
        keep[s] = acc != 0.0 ? 1 : 0;
    }
}

// compaction of the kept (key, value) pairs: pos = exclusive scan of keep
__global__ void compact_pairs(int64_t n, const int64_t *__restrict__ keep, const int64_t *__restrict__ pos,
                              const uint64_t *__restrict__ key, const double *__restrict__ val,
                              uint64_t *__restrict__ okey, double *__restrict__ oval)
{
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB)
        if (keep[i]) {
            okey[pos[i]] = key[i];
            oval[pos[i]] = val[i];
        }
}

__global__ void swap_halves(int64_t n, const uint64_t *__restrict__ in, uint64_t *__restrict__ out)
{
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB)
        out[i] = (in[i] << 32) | (in[i] >> 32);
}

__global__ void split_keys(int64_t n, const uint64_t *__restrict__ key, int32_t *__restrict__ hi, int32_t *__restrict__ lo)
{
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB) {
        if (hi) hi[i] = (int32_t)(key[i] >> 32);
        if (lo) lo[i] = (int32_t)(key[i] & 0xffffffffu);
    }
}

// CSR offsets of keys sorted by (row << 32 | col): off[r] = first key with row >= r
__global__ void offsets_from_keys(int64_t nrows, int64_t n, const uint64_t *__restrict__ key, int64_t *__restrict__ off)
{
    for (int64_t r = blockIdx.x * (int64_t)TB + threadIdx.x; r <= nrows; r += (int64_t)gridDim.x * TB) {
        const uint64_t want = (uint64_t)r << 32;
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t m = (lo + hi) >> 1;
            if (key[m] < want) lo = m + 1;
            else hi = m;
        }
        off[r] = lo;
    }
}

__global__ void csr_keys(int64_t n, const int32_t *__restrict__ rows, const int32_t *__restrict__ col, int transposed,
                         uint64_t *__restrict__ key)
{
    for (int64_t e = blockIdx.x * (int64_t)TB + threadIdx.x; e < n; e += (int64_t)gridDim.x * TB)
        key[e] = transposed ? ((uint64_t)(uint32_t)col[e] << 32) | (uint32_t)rows[e]
                            : ((uint64_t)(uint32_t)rows[e] << 32) | (uint32_t)col[e];
}

}  // namespace amg_setup

struct amg_csr_result {
    int device = 0;
    int64_t nrows = 0, ncols = 0, nnz = 0;
    amg_setup::Buf<int64_t> off;
    amg_setup::Buf<int32_t> col;
    amg_setup::Buf<double> val;
};

namespace amg_setup {

#define SCK(call)                                                                                     \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            return fail(AMG_E_CUDA, std::string(#call) + " failed: " + cudaGetErrorString(e_));      \
    } while (0)

static int scan_exclusive(const int64_t *in, int64_t *out, int64_t n)
{
    size_t tb = 0;
    SCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n));
    Buf<char> tmp;
    SCK(tmp.alloc(tb));
    SCK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n));
    return AMG_OK;
}

static int scan_inclusive(const int64_t *in, int64_t *out, int64_t n)
{
    size_t tb = 0;
    SCK(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, n));
    Buf<char> tmp;
    SCK(tmp.alloc(tb));
    SCK(cub::DeviceScan::InclusiveSum(tmp.p, tb, in, out, n));
    return AMG_OK;
}

// stable sort of (key, value) pairs on key bits [b0, b1); results replace key / val
static int sort_pairs(Buf<uint64_t> &key, Buf<double> &val, int64_t n, int b0, int b1)
{
    if (n <= 1) return AMG_OK;
    Buf<uint64_t> k2;
    Buf<double> v2;
    SCK(k2.alloc(n));
    SCK(v2.alloc(n));
    cub::DoubleBuffer<uint64_t> dk(key.p, k2.p);
    cub::DoubleBuffer<double> dv(val.p, v2.p);
    size_t tb = 0;
    SCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, b0, b1));
    Buf<char> tmp;
    SCK(tmp.alloc(tb));
    SCK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, n, b0, b1));
    SCK(cudaDeviceSynchronize());
    if (dk.Current() != key.p) std::swap(key.p, k2.p);
    if (dv.Current() != val.p) std::swap(val.p, v2.p);
    return AMG_OK;
}

static int read_i64(const int64_t *dev, int64_t *host)
{
    SCK(cudaMemcpy(host, dev, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return AMG_OK;
}

// keys sorted by the caller; equal keys summed in order, result scaled, zeros dropped
static int compress(Buf<uint64_t> &key, Buf<double> &term, int64_t n, double scale, Buf<uint64_t> &okey,
                    Buf<double> &oval, int64_t *nout)
{
    *nout = 0;
    if (n == 0) {
        SCK(okey.alloc(0));
        SCK(oval.alloc(0));
        return AMG_OK;
    }
    Buf<int64_t> flag, seg, start;
    SCK(flag.alloc(n));
    SCK(seg.alloc(n));
    head_flags<<<blocks(n), TB>>>(n, key.p, flag.p);
    TRY(scan_inclusive(flag.p, seg.p, n));
    int64_t nseg = 0;
    TRY(read_i64(seg.p + (n - 1), &nseg));
    SCK(start.alloc(nseg));
    segment_starts<<<blocks(n), TB>>>(n, key.p, seg.p, start.p);
    flag.release();
    seg.release();
    Buf<uint64_t> skey;
    Buf<double> sval;
    Buf<int64_t> keep, kpos;
    SCK(skey.alloc(nseg));
    SCK(sval.alloc(nseg));
    SCK(keep.alloc(nseg + 1));
    SCK(kpos.alloc(nseg + 1));
    SCK(cudaMemset(keep.p, 0, (nseg + 1) * sizeof(int64_t)));
    segment_sums<<<blocks(nseg), TB>>>(nseg, n, start.p, key.p, term.p, scale, skey.p, sval.p, keep.p);
    TRY(scan_exclusive(keep.p, kpos.p, nseg + 1));
    int64_t kept = 0;
    TRY(read_i64(kpos.p + nseg, &kept));
    SCK(okey.alloc(kept));
    SCK(oval.alloc(kept));
    compact_pairs<<<blocks(nseg), TB>>>(nseg, keep.p, kpos.p, skey.p, sval.p, okey.p, oval.p);
    SCK(cudaDeviceSynchronize());
    *nout = kept;
    return AMG_OK;
}

// left entries (outer, mid, lv) x rows of the right CSR matrix -> sorted, summed (outer, col) pairs
static int multiply(int64_t nleft, const int32_t *outer, const int32_t *mid, const double *lv, const int64_t *boff,
                    const int32_t *bcol, const double *bval, int key_bits_hi, Buf<uint64_t> &okey, Buf<double> &oval,
                    int64_t *nout)
{
    Buf<int64_t> cnt, pos;
    SCK(cnt.alloc(nleft + 1));
    SCK(pos.alloc(nleft + 1));
    SCK(cudaMemset(cnt.p, 0, (nleft + 1) * sizeof(int64_t)));
    if (nleft) expand_counts<<<blocks(nleft), TB>>>(nleft, mid, boff, cnt.p);
    TRY(scan_exclusive(cnt.p, pos.p, nleft + 1));
    int64_t total = 0;
    TRY(read_i64(pos.p + nleft, &total));
    cnt.release();
    Buf<uint64_t> key;
    Buf<double> term;
    SCK(key.alloc(total));
    SCK(term.alloc(total));
    if (nleft) expand_products<<<blocks(nleft), TB>>>(nleft, outer, mid, lv, pos.p, boff, bcol, bval, key.p, term.p);
    pos.release();
    TRY(sort_pairs(key, term, total, 0, 32 + key_bits_hi));
    TRY(compress(key, term, total, 1.0, okey, oval, nout));
    return AMG_OK;
}

static int bits_for(int64_t n)
{
    int b = 1;
    while (b < 32 && ((int64_t)1 << b) < n) ++b;
    return b;
}

struct DevCsrIn {
    Buf<int64_t> off;
    Buf<int32_t> col, rows;
    Buf<double> val;
    int64_t nrows = 0, ncols = 0, nnz = 0;
};

static int upload(DevCsrIn &d, int64_t nrows, int64_t ncols, const int64_t *off, const int32_t *col, const double *val,
                  bool want_rows)
{
    if (nrows < 0 || ncols < 0 || !off) return fail(AMG_E_ARG, "device setup: bad CSR arguments");
    if (nrows >= INT32_MAX || ncols >= INT32_MAX) return fail(AMG_E_ARG, "device setup: dimensions exceed int32");
    d.nrows = nrows;
    d.ncols = ncols;
    d.nnz = off[nrows];
    if (d.nnz > 0 && (!col || !val)) return fail(AMG_E_ARG, "device setup: NULL entries");
    SCK(d.off.alloc(nrows + 1));
    SCK(d.col.alloc(d.nnz));
    SCK(d.val.alloc(d.nnz));
    SCK(cudaMemcpy(d.off.p, off, (nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (d.nnz) {
        SCK(cudaMemcpy(d.col.p, col, d.nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
        SCK(cudaMemcpy(d.val.p, val, d.nnz * sizeof(double), cudaMemcpyHostToDevice));
    }
    if (want_rows) {
        SCK(d.rows.alloc(d.nnz));
        if (nrows) entry_rows<<<blocks(nrows), TB>>>(nrows, d.off.p, d.rows.p);
    }
    return AMG_OK;
}

// sorted (row << 32 | col) keys + values -> result CSR
static int finish(amg_csr_result *r, int64_t nrows, int64_t ncols, Buf<uint64_t> &key, Buf<double> &val, int64_t n)
{
    r->nrows = nrows;
    r->ncols = ncols;
    r->nnz = n;
    SCK(r->off.alloc(nrows + 1));
    SCK(r->col.alloc(n));
    offsets_from_keys<<<blocks(nrows + 1), TB>>>(nrows, n, key.p, r->off.p);
    if (n) split_keys<<<blocks(n), TB>>>(n, key.p, nullptr, r->col.p);
    SCK(cudaDeviceSynchronize());
    std::swap(r->val.p, val.p);
    std::swap(r->val.n, val.n);
    return AMG_OK;
}

static int galerkin(amg_csr_result *r, int64_t n, int64_t m, const int64_t *a_off, const int32_t *a_col,
                    const double *a_val, const int64_t *p_off, const int32_t *p_col, const double *p_val, int symmetrize)
{
    DevCsrIn A, P;
    TRY(upload(A, n, n, a_off, a_col, a_val, true));
    TRY(upload(P, n, m, p_off, p_col, p_val, false));
    const int cb = bits_for(m), rb = bits_for(n);
    // X = A P: left entries are A's (i, j, a_ij) in CSR order; keys (i, c)
    Buf<uint64_t> xkey;
    Buf<double> xval;
    int64_t nx = 0;
    TRY(multiply(A.nnz, A.rows.p, A.col.p, A.val.p, P.off.p, P.col.p, P.val.p, rb, xkey, xval, &nx));
    A.off.release();
    A.col.release();
    A.val.release();
    A.rows.release();
    // X's columns with rows ascending: a stable sort on the column half of the (i, c) keys
    TRY(sort_pairs(xkey, xval, nx, 0, 32));
    Buf<int32_t> xi, xc;
    SCK(xi.alloc(nx));
    SCK(xc.alloc(nx));
    if (nx) split_keys<<<blocks(nx), TB>>>(nx, xkey.p, xi.p, xc.p);
    xkey.release();
    // R^T = X^T P: left entries (c, i, x_ic) in that order; keys (c, k) hold R[k][c]
    Buf<uint64_t> rkey;
    Buf<double> rval;
    int64_t nr = 0;
    TRY(multiply(nx, xc.p, xi.p, xval.p, P.off.p, P.col.p, P.val.p, cb, rkey, rval, &nr));
    xi.release();
    xc.release();
    xval.release();
    // rows of R: keys (k, c)
    Buf<uint64_t> tkey;
    SCK(tkey.alloc(nr));
    if (nr) swap_halves<<<blocks(nr), TB>>>(nr, rkey.p, tkey.p);
    if (!symmetrize) {
        rkey.release();
        TRY(sort_pairs(tkey, rval, nr, 0, 32 + cb));
        return finish(r, m, m, tkey, rval, nr);
    }
    // (R + R^T) / 2: R's entries, then R^T's, merged by a stable sort; pairs summed in that order
    Buf<uint64_t> skey;
    Buf<double> sval;
    SCK(skey.alloc(2 * nr));
    SCK(sval.alloc(2 * nr));
    if (nr) {
        SCK(cudaMemcpy(skey.p, tkey.p, nr * sizeof(uint64_t), cudaMemcpyDeviceToDevice));
        SCK(cudaMemcpy(skey.p + nr, rkey.p, nr * sizeof(uint64_t), cudaMemcpyDeviceToDevice));
        SCK(cudaMemcpy(sval.p, rval.p, nr * sizeof(double), cudaMemcpyDeviceToDevice));
        SCK(cudaMemcpy(sval.p + nr, rval.p, nr * sizeof(double), cudaMemcpyDeviceToDevice));
    }
    tkey.release();
    rkey.release();
    rval.release();
    TRY(sort_pairs(skey, sval, 2 * nr, 0, 32 + cb));
    Buf<uint64_t> okey;
    Buf<double> oval;
    int64_t ns = 0;
    TRY(compress(skey, sval, 2 * nr, 0.5, okey, oval, &ns));
    return finish(r, m, m, okey, oval, ns);
}

static int transpose(amg_csr_result *r, int64_t nrows, int64_t ncols, const int64_t *off, const int32_t *col,
                     const double *val)
{
    DevCsrIn A;
    TRY(upload(A, nrows, ncols, off, col, val, true));
    Buf<uint64_t> key;
    SCK(key.alloc(A.nnz));
    if (A.nnz) csr_keys<<<blocks(A.nnz), TB>>>(A.nnz, A.rows.p, A.col.p, 1, key.p);
    TRY(sort_pairs(key, A.val, A.nnz, 0, 32 + bits_for(ncols)));
    return finish(r, ncols, nrows, key, A.val, A.nnz);
}

#undef SCK

}  // namespace amg_setup
