/*
 * exact.c -- EXACT REFERENCE (test infrastructure only; part of oracle/).
 *
 * Fixed-point long accumulator (Kulisch style) for the exact value of one entry
 * of C = AB (Eq. 1) over the reals, where every DD/QD input is the exact
 * sum of its words. It uses only integer arithmetic on the doubles' significands
 * and exponents (no DD/QD operation), so it pins the oracle and the GPU path
 * independently of docs/numerics.md.
 *
 * The accumulator holds X (two's complement, NL 64-bit limbs, little-endian);
 * the represented value is X * 2^-BIAS. Any term below 2^-BIAS or a result above
 * 2^(64*NL-BIAS-2) sets *status = 1 (window violated) instead of being dropped.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define NL 24
#define BIAS 1280

typedef struct { uint64_t v[NL]; } acc_t;

static void acc_add_shifted(acc_t *a, unsigned __int128 mag, int neg, int shift, int *status) {
    /* add (or subtract) mag * 2^shift to X */
    if (shift < 0) { *status = 1; return; }
    int q = shift / 64, r = shift % 64;
    uint64_t w[4] = { 0, 0, 0, 0 };
    uint64_t lo = (uint64_t)mag, hi = (uint64_t)(mag >> 64);
    if (r == 0) { w[0] = lo; w[1] = hi; }
    else {
        w[0] = lo << r;
        w[1] = (lo >> (64 - r)) | (hi << r);
        w[2] = hi >> (64 - r);
    }
    if (q + 3 >= NL) { *status = 1; return; }
    if (!neg) {
        unsigned __int128 carry = 0;
        for (int i = q; i < NL; i++) {
            unsigned __int128 s = (unsigned __int128)a->v[i] + (i - q < 4 ? w[i - q] : 0) + carry;
            a->v[i] = (uint64_t)s;
            carry = s >> 64;
            if (i - q >= 3 && carry == 0) break;
        }
    } else {
        uint64_t borrow = 0;
        for (int i = q; i < NL; i++) {
            uint64_t sub = (i - q < 4 ? w[i - q] : 0);
            uint64_t x = a->v[i];
            uint64_t d = x - sub - borrow;
            borrow = (x < sub) || (x - sub < borrow) ? 1 : 0;
            a->v[i] = d;
            if (i - q >= 3 && borrow == 0) break;
        }
    }
}

/* x = mant * 2^exp with |mant| < 2^53 integer */
static void decompose(double x, int64_t *mant, int *exp) {
    int e;
    double f = frexp(x, &e);          /* x = f * 2^e, 0.5 <= |f| < 1 */
    *mant = (int64_t)ldexp(f, 53);    /* exact */
    *exp = e - 53;
}

static void acc_add_prod(acc_t *a, double x, double y, int *status) {
    if (x == 0.0 || y == 0.0) return;
    if (!isfinite(x) || !isfinite(y)) { *status = 1; return; }
    int64_t mx, my;
    int ex, ey;
    decompose(x, &mx, &ex);
    decompose(y, &my, &ey);
    int neg = (mx < 0) != (my < 0);
    unsigned __int128 mag = (unsigned __int128)(uint64_t)(mx < 0 ? -mx : mx) * (uint64_t)(my < 0 ? -my : my);
    acc_add_shifted(a, mag, neg, ex + ey + BIAS, status);
}

static void acc_add_double(acc_t *a, double x, int neg, int *status) {
    if (x == 0.0) return;
    if (!isfinite(x)) { *status = 1; return; }
    int64_t mx;
    int ex;
    decompose(x, &mx, &ex);
    int n = (mx < 0) != (neg != 0);
    unsigned __int128 mag = (uint64_t)(mx < 0 ? -mx : mx);
    acc_add_shifted(a, mag, n, ex + BIAS, status);
}

/* value of X * 2^-BIAS rounded to double (truncation of bits below the top 64, then one rounding) */
static double acc_to_double(const acc_t *a0, int *status) {
    acc_t a = *a0;
    int neg = (a.v[NL - 1] >> 63) & 1;
    if (neg) { /* negate two's complement */
        uint64_t carry = 1;
        for (int i = 0; i < NL; i++) {
            uint64_t x = ~a.v[i];
            uint64_t s = x + carry;
            carry = (carry && s == 0) ? 1 : 0;
            a.v[i] = s;
        }
    }
    if (a.v[NL - 1] >> 62) *status = 1;
    int top = -1;
    for (int i = NL - 1; i >= 0; i--) if (a.v[i]) { top = i; break; }
    if (top < 0) return 0.0;
    int lz = __builtin_clzll(a.v[top]);
    int bitpos = top * 64 + (63 - lz);          /* index of the leading 1 */
    /* gather 64 bits starting at bitpos downward */
    int start = bitpos - 63;
    uint64_t bits = 0;
    for (int k = 0; k < 64; k++) {
        int b = start + k;
        if (b < 0) continue;
        if ((a.v[b / 64] >> (b % 64)) & 1) bits |= (uint64_t)1 << k;
    }
    /* sticky: any bit below start */
    int sticky = 0;
    for (int b = 0; b < start && !sticky; b++) if ((a.v[b / 64] >> (b % 64)) & 1) sticky = 1;
    if (sticky) bits |= 1;   /* keeps round-to-nearest correct for the 11 dropped bits */
    double r = ldexp((double)bits, start - BIAS);
    return neg ? -r : r;
}

/*
 * For each sampled entry (rows[t], cols[t]) of C = A B with A [W][m][l],
 * B [W][l][n], C [W][m][n] (planar contiguous):
 *   exact_out[t] = the exact entry rounded to double,
 *   err_out[t]   = (exact - sum of C's words) rounded to double.
 * Returns 0, or 1 if the fixed-point window was violated for any entry.
 */
int or_exact_entries(int W, int64_t m, int64_t l, int64_t n, const double *A, const double *B,
                     const double *C, int64_t count, const int64_t *rows, const int64_t *cols,
                     double *exact_out, double *err_out) {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
    for (int64_t t = 0; t < count; t++) {
        int status = 0;
        acc_t acc;
        memset(&acc, 0, sizeof(acc));
        int64_t i = rows[t], j = cols[t];
        for (int64_t k = 0; k < l; k++)
            for (int p = 0; p < W; p++) {
                double a = A[p * m * l + i * l + k];
                if (a == 0.0) continue;
                for (int q = 0; q < W; q++) acc_add_prod(&acc, a, B[q * l * n + k * n + j], &status);
            }
        exact_out[t] = acc_to_double(&acc, &status);
        for (int w = 0; w < W; w++) acc_add_double(&acc, C[w * m * n + i * n + j], 1, &status);
        err_out[t] = acc_to_double(&acc, &status);
        bad |= status;
    }
    return bad;
}

/* Exact sum of (x_w) - (y_w) words for arrays of W-word numbers (planar [W][count]); for pins. */
int or_exact_diff(int W, int64_t count, const double *x, const double *y, double *out) {
    int bad = 0;
    for (int64_t t = 0; t < count; t++) {
        int status = 0;
        acc_t acc;
        memset(&acc, 0, sizeof(acc));
        for (int w = 0; w < W; w++) {
            acc_add_double(&acc, x[w * count + t], 0, &status);
            acc_add_double(&acc, y[w * count + t], 1, &status);
        }
        out[t] = acc_to_double(&acc, &status);
        bad |= status;
    }
    return bad;
}
