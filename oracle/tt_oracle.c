/*
 * tt_oracle.c -- CPU oracle for the out-of-place tensor permutation of
 * arXiv 1705.01598 (cuTT).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this file's
 * library.  It shares no code, header or constant with the CUDA path
 * (paper_1705_01598_b200/csrc), and it includes nothing from it.
 *
 * What it computes (Section 2, Eq. (1), with the stride
 * reading c(i,O) -- see DESIGN.md reading R2):
 *
 *   dims d[0..n-1], d[0] is the stride-1 dimension
 *   perm p: output dimension j is input dimension p[j]
 *   output extents e[j] = d[p[j]]
 *   input stride  c(i, I) = prod_{k<i} d[k]                 (ordering I)
 *   output stride c(j, O) = prod_{k<j} e[k]                 (ordering O)
 *
 *   for every coordinate x (0 <= x[i] < d[i]):
 *       out[ sum_j x[p[j]] * c(j,O) ] = in[ sum_i x[i] * c(i,I) ]
 *
 * Elements are opaque 4- or 8-byte words (never float types), so the copy is
 * bit-exact for NaN payloads, -0.0 and subnormals.
 *
 * Algorithm (plain and slow): walk the OUTPUT linearly with an odometer
 * y[0..n-1] over the output coordinates (y[0] fastest).  The element at output
 * coordinate y is the input element with x[p[j]] = y[j], whose input position
 * is off = sum_j y[j] * c(p[j], I).  The odometer keeps `off` incrementally:
 * incrementing y[j] adds c(p[j],I); wrapping y[j] to 0 subtracts
 * e[j]*c(p[j],I) and carries into y[j+1].
 *
 * A second, independent formulation (per-position division decode) is
 * oracle_permute_sample(), used for sampled checks at full benchmark sizes.
 */
#include <stdint.h>
#include <string.h>

#define ORACLE_MAX_RANK 64

/* Return codes. */
#define ORACLE_OK 0
#define ORACLE_BAD_ARG 1

static int check_args(int rank, const int64_t* dims, const int* perm, int esize) {
    if (rank < 1 || rank > ORACLE_MAX_RANK) return ORACLE_BAD_ARG;
    if (esize != 4 && esize != 8) return ORACLE_BAD_ARG;
    int seen[ORACLE_MAX_RANK];
    memset(seen, 0, sizeof(seen));
    for (int i = 0; i < rank; ++i) {
        if (dims[i] < 1) return ORACLE_BAD_ARG;
        if (perm[i] < 0 || perm[i] >= rank || seen[perm[i]]) return ORACLE_BAD_ARG;
        seen[perm[i]] = 1;
    }
    return ORACLE_OK;
}

/* Output elements [out_begin, out_end) of the permutation (gather form). */
int oracle_permute_range(int rank, const int64_t* dims, const int* perm, int esize,
                         const void* in, void* out, int64_t out_begin, int64_t out_end) {
    if (check_args(rank, dims, perm, esize) != ORACLE_OK) return ORACLE_BAD_ARG;
    int64_t cin[ORACLE_MAX_RANK];   /* c(i, I): input strides                 */
    int64_t e[ORACLE_MAX_RANK];     /* output extents e[j] = d[p[j]]          */
    int64_t step[ORACLE_MAX_RANK];  /* input stride of output dim j           */
    int64_t y[ORACLE_MAX_RANK];     /* output coordinate odometer             */
    int64_t vol = 1;
    for (int i = 0; i < rank; ++i) { cin[i] = vol; vol *= dims[i]; }
    for (int j = 0; j < rank; ++j) { e[j] = dims[perm[j]]; step[j] = cin[perm[j]]; }
    if (out_begin < 0) out_begin = 0;
    if (out_end > vol) out_end = vol;
    if (out_begin >= out_end) return ORACLE_OK;

    /* Starting coordinate: decode out_begin in output order. */
    int64_t rem = out_begin, off = 0;
    for (int j = 0; j < rank; ++j) {
        y[j] = rem % e[j];
        rem /= e[j];
        off += y[j] * step[j];
    }

    if (esize == 4) {
        const uint32_t* a = (const uint32_t*)in;
        uint32_t* b = (uint32_t*)out;
        for (int64_t q = out_begin; q < out_end; ++q) {
            b[q] = a[off];
            int j = 0;
            y[0] += 1; off += step[0];
            while (j < rank - 1 && y[j] == e[j]) {
                off -= e[j] * step[j]; y[j] = 0;
                ++j; y[j] += 1; off += step[j];
            }
        }
    } else {
        const uint64_t* a = (const uint64_t*)in;
        uint64_t* b = (uint64_t*)out;
        for (int64_t q = out_begin; q < out_end; ++q) {
            b[q] = a[off];
            int j = 0;
            y[0] += 1; off += step[0];
            while (j < rank - 1 && y[j] == e[j]) {
                off -= e[j] * step[j]; y[j] = 0;
                ++j; y[j] += 1; off += step[j];
            }
        }
    }
    return ORACLE_OK;
}

/* The whole permutation. */
int oracle_permute(int rank, const int64_t* dims, const int* perm, int esize,
                   const void* in, void* out) {
    int64_t vol = 1;
    if (check_args(rank, dims, perm, esize) != ORACLE_OK) return ORACLE_BAD_ARG;
    for (int i = 0; i < rank; ++i) vol *= dims[i];
    return oracle_permute_range(rank, dims, perm, esize, in, out, 0, vol);
}

/*
 * Sampled form: for each requested output position q, decode the output
 * coordinates y[j] = mod(floor(q / c(j,O)), e[j]) (P:L52 with ordering O),
 * form the input position sum_j y[j] * c(p[j], I) and copy that word.
 * values[s] receives out[positions[s]].
 */
int oracle_permute_sample(int rank, const int64_t* dims, const int* perm, int esize,
                          const void* in, const int64_t* positions, int64_t count,
                          void* values) {
    if (check_args(rank, dims, perm, esize) != ORACLE_OK) return ORACLE_BAD_ARG;
    int64_t cin[ORACLE_MAX_RANK], cout[ORACLE_MAX_RANK], e[ORACLE_MAX_RANK];
    int64_t vol = 1;
    for (int i = 0; i < rank; ++i) { cin[i] = vol; vol *= dims[i]; }
    int64_t acc = 1;
    for (int j = 0; j < rank; ++j) { e[j] = dims[perm[j]]; cout[j] = acc; acc *= e[j]; }
    for (int64_t s = 0; s < count; ++s) {
        int64_t q = positions[s];
        if (q < 0 || q >= vol) return ORACLE_BAD_ARG;
        int64_t src = 0;
        for (int j = 0; j < rank; ++j) {
            int64_t yj = (q / cout[j]) % e[j];
            src += yj * cin[perm[j]];
        }
        if (esize == 4) ((uint32_t*)values)[s] = ((const uint32_t*)in)[src];
        else            ((uint64_t*)values)[s] = ((const uint64_t*)in)[src];
    }
    return ORACLE_OK;
}

/*
 * Accumulate form (SURVEY f-3; Section 3.3: the TTC
 * comparison kernels "read input, read output, accumulate, write output"):
 *     out[q] = alpha * in[src(q)] + beta * out[q]
 * in float (esize 4) or double (esize 8) with alpha, beta converted to that
 * type; each multiply and the add rounded separately (this file is compiled
 * with -ffp-contract=off, no FMA); beta == 0 does not read out (BLAS
 * convention, reading R21).  src(q) by the P:L52 division decode.
 */
int oracle_permute_scaled(int rank, const int64_t* dims, const int* perm, int esize,
                          const void* in, void* out, double alpha, double beta) {
    if (check_args(rank, dims, perm, esize) != ORACLE_OK) return ORACLE_BAD_ARG;
    int64_t cin[ORACLE_MAX_RANK], cout[ORACLE_MAX_RANK], e[ORACLE_MAX_RANK];
    int64_t vol = 1;
    for (int i = 0; i < rank; ++i) { cin[i] = vol; vol *= dims[i]; }
    int64_t acc = 1;
    for (int j = 0; j < rank; ++j) { e[j] = dims[perm[j]]; cout[j] = acc; acc *= e[j]; }
    for (int64_t q = 0; q < vol; ++q) {
        int64_t src = 0;
        for (int j = 0; j < rank; ++j) src += ((q / cout[j]) % e[j]) * cin[perm[j]];
        if (esize == 4) {
            const float a = (float)alpha, b = (float)beta;
            float x, y, r;
            memcpy(&x, (const uint32_t*)in + src, 4);
            r = a * x;
            if (beta != 0.0) {
                memcpy(&y, (uint32_t*)out + q, 4);
                r = r + b * y;
            }
            memcpy((uint32_t*)out + q, &r, 4);
        } else {
            double x, y, r;
            memcpy(&x, (const uint64_t*)in + src, 8);
            r = alpha * x;
            if (beta != 0.0) {
                memcpy(&y, (uint64_t*)out + q, 8);
                r = r + beta * y;
            }
            memcpy((uint64_t*)out + q, &r, 8);
        }
    }
    return ORACLE_OK;
}

/*
 * Tensor contraction (Section 3.4; the contraction
 * "D = D + L . R" of P:L321, with scale factors):
 *
 *   D[y] = alpha * sum_z L[x_L(y, z)] * R[x_R(y, z)] + beta * D0[y]
 *
 * Every dimension carries an integer label; y runs over D's labels, z over
 * the contracted labels (in L and R, not in D); a tensor's element for a
 * labelled coordinate is at sum over its dims of coordinate * stride, with
 * column-major strides (dim 0 stride-1, as above).  Written out plainly: an
 * odometer over D's coordinates, and for each output an odometer over the
 * contracted coordinates, products and sums in double (float inputs are
 * converted exactly), in the order the odometers visit them.  No blocking,
 * no transposes, no GEMM.  D0 may be NULL (beta ignored).  Result in double.
 * Returns ORACLE_BAD_ARG for labels that do not form a contraction.
 */
#define ORACLE_MAX_LABELS 64
int oracle_contract(int rd, const int* md, int rl, const int64_t* dl, const int* ml, int rr,
                    const int64_t* dr, const int* mr, int esize, const void* L, const void* R,
                    const double* D0, double* D, double alpha, double beta) {
    if (rd < 0 || rl < 0 || rr < 0 || rd > ORACLE_MAX_LABELS || rl > ORACLE_MAX_LABELS ||
        rr > ORACLE_MAX_LABELS || (esize != 4 && esize != 8))
        return ORACLE_BAD_ARG;
    /* per D label: extent, stride in L, stride in R (0 when absent) */
    int64_t ye[ORACLE_MAX_LABELS], ysl[ORACLE_MAX_LABELS], ysr[ORACLE_MAX_LABELS];
    int64_t ze[ORACLE_MAX_LABELS], zsl[ORACLE_MAX_LABELS], zsr[ORACLE_MAX_LABELS];
    int64_t sl[ORACLE_MAX_LABELS], sr[ORACLE_MAX_LABELS];
    int64_t acc = 1;
    for (int i = 0; i < rl; ++i) { sl[i] = acc; acc *= dl[i]; }
    acc = 1;
    for (int i = 0; i < rr; ++i) { sr[i] = acc; acc *= dr[i]; }
    int nz = 0;
    for (int j = 0; j < rd; ++j) {
        int a = -1, b = -1;
        for (int i = 0; i < rl; ++i) if (ml[i] == md[j]) a = i;
        for (int i = 0; i < rr; ++i) if (mr[i] == md[j]) b = i;
        if ((a < 0) == (b < 0)) return ORACLE_BAD_ARG;   /* in exactly one input */
        ye[j] = a >= 0 ? dl[a] : dr[b];
        ysl[j] = a >= 0 ? sl[a] : 0;
        ysr[j] = b >= 0 ? sr[b] : 0;
    }
    for (int i = 0; i < rl; ++i) {
        int inD = 0, b = -1;
        for (int j = 0; j < rd; ++j) if (md[j] == ml[i]) inD = 1;
        if (inD) continue;
        for (int k = 0; k < rr; ++k) if (mr[k] == ml[i]) b = k;
        if (b < 0 || dr[b] != dl[i]) return ORACLE_BAD_ARG;
        ze[nz] = dl[i];
        zsl[nz] = sl[i];
        zsr[nz] = sr[b];
        ++nz;
    }
    for (int k = 0; k < rr; ++k) {          /* every label of R is in D or in L */
        int seen = 0;
        for (int j = 0; j < rd; ++j) if (md[j] == mr[k]) seen = 1;
        for (int i = 0; i < rl; ++i) if (ml[i] == mr[k]) seen = 1;
        if (!seen) return ORACLE_BAD_ARG;
    }
    int64_t y[ORACLE_MAX_LABELS], z[ORACLE_MAX_LABELS];
    int64_t volD = 1;
    for (int j = 0; j < rd; ++j) { volD *= ye[j]; y[j] = 0; }
    int64_t offL = 0, offR = 0;   /* of the current D coordinate y */
    for (int64_t pos = 0; pos < volD; ++pos) {
        double sum = 0.0;
        int64_t zl = offL, zr = offR;
        for (int k = 0; k < nz; ++k) z[k] = 0;
        for (;;) {
            double a, b;
            if (esize == 4) {
                a = (double)((const float*)L)[zl];
                b = (double)((const float*)R)[zr];
            } else {
                a = ((const double*)L)[zl];
                b = ((const double*)R)[zr];
            }
            sum += a * b;
            int k = 0;
            for (; k < nz; ++k) {           /* odometer over the contracted labels */
                if (++z[k] < ze[k]) { zl += zsl[k]; zr += zsr[k]; break; }
                zl -= (ze[k] - 1) * zsl[k];
                zr -= (ze[k] - 1) * zsr[k];
                z[k] = 0;
            }
            if (k == nz) break;
        }
        D[pos] = alpha * sum + (D0 ? beta * D0[pos] : 0.0);
        for (int j = 0; j < rd; ++j) {      /* odometer over D's coordinates */
            if (++y[j] < ye[j]) { offL += ysl[j]; offR += ysr[j]; break; }
            offL -= (ye[j] - 1) * ysl[j];
            offR -= (ye[j] - 1) * ysr[j];
            y[j] = 0;
        }
    }
    return 0;
}
