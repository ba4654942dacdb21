/* Plain-C restatement of the row-sum order of the reference SpMV
 * (TEST INFRASTRUCTURE ONLY -- the checker, never the product).
 *
 * amgkit's spmv (amgkit/sparse.py:203-217) multiplies values by the gathered
 * x entries (each product rounded: numpy does not contract to FMA) and sums
 * every row with np.add.reduceat (amgkit/sparse.py:28-48).  For one segment
 * p[0..L-1] numpy's reduce loop computes
 *
 *     p[0] + pairwise(p[1..L-1])
 *
 * where pairwise (numpy's pairwise_sum, un-vendored dependency numpy 2.3.5,
 * loops.c.src) is: n < 8 -> sequential from 0.0; n <= 128 -> eight strided
 * accumulators r[j] = p[j] + p[j+8] + ... over the largest multiple of 8,
 * combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail added
 * sequentially; n > 128 -> split at n2 = n/2 - (n/2) % 8 and recurse.
 * The CUDA kernels reproduce exactly this order (spmv.cu); tests pin this
 * file against np.add.reduceat bit for bit.
 */
#include <stdint.h>

static double pairwise(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

/* y[i] = sum over row i of vals[k] * x[cols[k]] in the reference order. */
void oracle_csr_spmv(int64_t nrows, const int64_t *offsets, const int32_t *cols,
                     const double *vals, const double *x, double *y, double *scratch)
{
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t lo = offsets[i], hi = offsets[i + 1];
        if (hi == lo) { y[i] = 0.0; continue; }
        for (int64_t k = lo; k < hi; ++k) {
            volatile double p = vals[k] * x[cols[k]]; /* rounded product */
            scratch[k - lo] = p;
        }
        y[i] = scratch[0] + pairwise(scratch + 1, hi - lo - 1);
    }
}

/* Segment sums of precomputed data (mirrors row_segment_sums). */
void oracle_segment_sums(int64_t nseg, const int64_t *offsets, const double *data, double *out)
{
    for (int64_t i = 0; i < nseg; ++i) {
        int64_t lo = offsets[i], hi = offsets[i + 1];
        out[i] = (hi == lo) ? 0.0 : data[lo] + pairwise(data + lo + 1, hi - lo - 1);
    }
}
