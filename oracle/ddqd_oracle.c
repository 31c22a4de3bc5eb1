/*
 * ddqd_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * Plain, slow, obviously correct C implementation of what the B200 hot path
 * computes: DD/QD arithmetic, the Simple/Block GEMM of Eq. (1), the Strassen and
 * Winograd recursions, and the blocked right-looking LU with partial pivoting.
 * It follows docs/numerics.md step by step (section numbers cited below) and
 * shares NO code with paper_1510_08642_b200/csrc. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *   (no contraction: x*y+z must stay two roundings; fma() is the C99 correctly
 *    rounded fused multiply-add, used only where the contract says fma).
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n, BJ:n = BASELINE.json line n.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py (exact
 * rationals, closed forms, special cases, invariants, brute force on tiny inputs), and
 * tools/oracle_mutation_check.py shows that plausible mistakes in the EFTs, DD/QD ops,
 * the pivot orders and the solve's permutation each fail a pin. Which QD algorithm is
 * used (Hida-Li-Bailey "sloppy", reading R1) is a reading of P:58, not
 * something the paper's text fixes.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* numerics.md s.1: error-free transforms                           */
/* ------------------------------------------------------------------------- */
static void two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    double bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

static void fast_two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    *e = b - (ss - a);
    *s = ss;
}

static void two_prod(double a, double b, double *p, double *e) {
    double pp = a * b;
    *e = fma(a, b, -pp);
    *p = pp;
}

/* ------------------------------------------------------------------------- */
/* numerics.md s.2: double-double                             */
/* ------------------------------------------------------------------------- */
typedef struct { double hi, lo; } dd_t;

static dd_t dd_add(dd_t x, dd_t y) {            /* "sloppy" add */
    double s, e, t;
    dd_t r;
    two_sum(x.hi, y.hi, &s, &e);
    t = x.lo + y.lo;
    e = e + t;
    fast_two_sum(s, e, &r.hi, &r.lo);
    return r;
}

static dd_t dd_neg(dd_t x) { dd_t r = { -x.hi, -x.lo }; return r; }

static dd_t dd_sub(dd_t x, dd_t y) { return dd_add(x, dd_neg(y)); }

/* numerics.md s.2 accurate ("IEEE-style") add (variant DDQD_ADD_ACCURATE, SURVEY.md
 * s.8(f) row f3): both word pairs summed error-free, two renormalisations. 20 adds. */
static dd_t dd_add_acc(dd_t x, dd_t y) {
    double s1, s2, t1, t2;
    dd_t r;
    two_sum(x.hi, y.hi, &s1, &s2);
    two_sum(x.lo, y.lo, &t1, &t2);
    s2 = s2 + t1;
    fast_two_sum(s1, s2, &s1, &s2);
    s2 = s2 + t2;
    fast_two_sum(s1, s2, &r.hi, &r.lo);
    return r;
}

static dd_t dd_sub_acc(dd_t x, dd_t y) { return dd_add_acc(x, dd_neg(y)); }

static dd_t dd_mul(dd_t x, dd_t y) {
    double p, e, t;
    dd_t r;
    two_prod(x.hi, y.hi, &p, &e);
    t = (x.hi * y.lo) + (x.lo * y.hi);
    e = e + t;
    fast_two_sum(p, e, &r.hi, &r.lo);
    return r;
}

static dd_t dd_madd(dd_t c, dd_t a, dd_t b) { return dd_add(c, dd_mul(a, b)); }

/* numerics.md s.2 fused variant (DDQD_MADD_FUSED) */
static dd_t dd_madd_fused(dd_t c, dd_t a, dd_t b) {
    double p = a.hi * b.hi, e, s, t;
    dd_t r;
    e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, e);
    e = fma(a.lo, b.hi, e);
    two_sum(c.hi, p, &s, &t);
    t = t + (c.lo + e);
    fast_two_sum(s, t, &r.hi, &r.lo);
    return r;
}

/* arithmetic variant of a GEMM / LU call, set per call by or_gemm / or_lu from the algo
 * flags: 0 canonical, 1 fused DD madd (0x100), 2 accurate adds everywhere (0x200) */
static int g_variant = 0;

static dd_t dd_madd_acc(dd_t c, dd_t a, dd_t b) { return dd_add_acc(c, dd_mul(a, b)); }

static dd_t dd_madd_v(dd_t c, dd_t a, dd_t b) {
    if (g_variant == 1) return dd_madd_fused(c, a, b);
    if (g_variant == 2) return dd_madd_acc(c, a, b);
    return dd_madd(c, a, b);
}
static dd_t dd_add_v(dd_t x, dd_t y) { return g_variant == 2 ? dd_add_acc(x, y) : dd_add(x, y); }
static dd_t dd_sub_v(dd_t x, dd_t y) { return g_variant == 2 ? dd_sub_acc(x, y) : dd_sub(x, y); }

static dd_t dd_div(dd_t x, dd_t y) {
    dd_t q1d, r, out;
    double q1 = x.hi / y.hi, q2;
    q1d.hi = q1; q1d.lo = 0.0;
    r = dd_sub(x, dd_mul(y, q1d));
    q2 = r.hi / y.hi;
    fast_two_sum(q1, q2, &out.hi, &out.lo);
    return out;
}

/* |x| > |y| in the DD magnitude order of numerics.md s.2 */
static int dd_abs_gt(dd_t x, dd_t y) {
    dd_t ax = x.hi >= 0.0 ? x : dd_neg(x);
    dd_t ay = y.hi >= 0.0 ? y : dd_neg(y);
    if (ax.hi != ay.hi) return ax.hi > ay.hi;
    return ax.lo > ay.lo;
}

/* ------------------------------------------------------------------------- */
/* numerics.md s.3: quad-double, Hida-Li-Bailey "sloppy"      */
/* ------------------------------------------------------------------------- */
typedef struct { double w[4]; } qd_t;

static void three_sum(double *a, double *b, double *c) {
    double t1, t2, t3;
    two_sum(*a, *b, &t1, &t2);
    two_sum(*c, t1, a, &t3);
    two_sum(t2, t3, b, c);
}

static void three_sum2(double *a, double *b, double *c) {
    double t1, t2, t3;
    two_sum(*a, *b, &t1, &t2);
    two_sum(*c, t1, a, &t3);
    *b = t2 + t3;
}

static qd_t qd_renorm(double c0, double c1, double c2, double c3, double c4) {
    double s, t0, t1, t2, t3, t4, s0, s1, s2, s3;
    qd_t r;
    fast_two_sum(c3, c4, &s, &t4);
    fast_two_sum(c2, s, &s, &t3);
    fast_two_sum(c1, s, &s, &t2);
    fast_two_sum(c0, s, &t0, &t1);
    s0 = t0; s1 = t1; s2 = 0.0; s3 = 0.0;
    if (s1 != 0.0) {
        fast_two_sum(s1, t2, &s1, &s2);
        if (s2 != 0.0) {
            fast_two_sum(s2, t3, &s2, &s3);
            if (s3 != 0.0) s3 = s3 + t4;
            else           s2 = s2 + t4;
        } else {
            fast_two_sum(s1, t3, &s1, &s2);
            if (s2 != 0.0) fast_two_sum(s2, t4, &s2, &s3);
            else           fast_two_sum(s1, t4, &s1, &s2);
        }
    } else {
        fast_two_sum(s0, t2, &s0, &s1);
        if (s1 != 0.0) {
            fast_two_sum(s1, t3, &s1, &s2);
            if (s2 != 0.0) fast_two_sum(s2, t4, &s2, &s3);
            else           fast_two_sum(s1, t4, &s1, &s2);
        } else {
            fast_two_sum(s0, t3, &s0, &s1);
            if (s1 != 0.0) fast_two_sum(s1, t4, &s1, &s2);
            else           fast_two_sum(s0, t4, &s0, &s1);
        }
    }
    r.w[0] = s0; r.w[1] = s1; r.w[2] = s2; r.w[3] = s3;
    return r;
}

static qd_t qd_add(qd_t a, qd_t b) {
    double s0, s1, s2, s3, t0, t1, t2, t3;
    two_sum(a.w[0], b.w[0], &s0, &t0);
    two_sum(a.w[1], b.w[1], &s1, &t1);
    two_sum(a.w[2], b.w[2], &s2, &t2);
    two_sum(a.w[3], b.w[3], &s3, &t3);
    two_sum(s1, t0, &s1, &t0);
    three_sum(&s2, &t0, &t1);
    three_sum2(&s3, &t0, &t2);
    t0 = (t0 + t1) + t3;
    return qd_renorm(s0, s1, s2, s3, t0);
}

static qd_t qd_neg(qd_t a) {
    qd_t r;
    for (int i = 0; i < 4; i++) r.w[i] = -a.w[i];
    return r;
}

static qd_t qd_sub(qd_t a, qd_t b) { return qd_add(a, qd_neg(b)); }

static qd_t qd_mul(qd_t a, qd_t b) {
    double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5;
    double s0, s1, s2, t0, t1, tail;
    two_prod(a.w[0], b.w[0], &p0, &q0);
    two_prod(a.w[0], b.w[1], &p1, &q1);
    two_prod(a.w[1], b.w[0], &p2, &q2);
    two_prod(a.w[0], b.w[2], &p3, &q3);
    two_prod(a.w[1], b.w[1], &p4, &q4);
    two_prod(a.w[2], b.w[0], &p5, &q5);
    three_sum(&p1, &p2, &q0);
    three_sum(&p2, &q1, &q2);
    three_sum(&p3, &p4, &p5);
    two_sum(p2, p3, &s0, &t0);
    two_sum(q1, p4, &s1, &t1);
    s2 = q2 + p5;
    two_sum(s1, t0, &s1, &t0);
    s2 = s2 + (t0 + t1);
    tail = a.w[0] * b.w[3];
    tail = tail + a.w[1] * b.w[2];
    tail = tail + a.w[2] * b.w[1];
    tail = tail + a.w[3] * b.w[0];
    tail = tail + q0;
    tail = tail + q3;
    tail = tail + q4;
    tail = tail + q5;
    s1 = s1 + tail;
    return qd_renorm(p0, p1, s0, s1, s2);
}

static qd_t qd_madd(qd_t c, qd_t a, qd_t b) { return qd_add(c, qd_mul(a, b)); }

/* numerics.md s.3 fused QD multiply-add (variant DDQD_MADD_FUSED):
 * the product's five-term expansion (p0, p1, s0, s1, s2) of qd_mul is added to c by the
 * qd_add network without renormalising it first (s2 joins the final tail). */
static qd_t qd_madd_fused(qd_t c, qd_t a, qd_t b) {
    double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5;
    double s0, s1, s2, t0, t1, tail;
    double u0, u1, u2, u3, v0, v1, v2, v3;
    two_prod(a.w[0], b.w[0], &p0, &q0);
    two_prod(a.w[0], b.w[1], &p1, &q1);
    two_prod(a.w[1], b.w[0], &p2, &q2);
    two_prod(a.w[0], b.w[2], &p3, &q3);
    two_prod(a.w[1], b.w[1], &p4, &q4);
    two_prod(a.w[2], b.w[0], &p5, &q5);
    three_sum(&p1, &p2, &q0);
    three_sum(&p2, &q1, &q2);
    three_sum(&p3, &p4, &p5);
    two_sum(p2, p3, &s0, &t0);
    two_sum(q1, p4, &s1, &t1);
    s2 = q2 + p5;
    two_sum(s1, t0, &s1, &t0);
    s2 = s2 + (t0 + t1);
    tail = a.w[0] * b.w[3];
    tail = tail + a.w[1] * b.w[2];
    tail = tail + a.w[2] * b.w[1];
    tail = tail + a.w[3] * b.w[0];
    tail = tail + q0;
    tail = tail + q3;
    tail = tail + q4;
    tail = tail + q5;
    s1 = s1 + tail;
    two_sum(c.w[0], p0, &u0, &v0);
    two_sum(c.w[1], p1, &u1, &v1);
    two_sum(c.w[2], s0, &u2, &v2);
    two_sum(c.w[3], s1, &u3, &v3);
    two_sum(u1, v0, &u1, &v0);
    three_sum(&u2, &v0, &v1);
    three_sum2(&u3, &v0, &v2);
    v0 = ((v0 + v1) + v3) + s2;
    return qd_renorm(u0, u1, u2, u3, v0);
}

/* numerics.md s.3 ThreeAccum: adds t into the two-word accumulator (u, v); returns the
 * word that has become complete (or 0 when none has) */
static double three_accum(double *u, double *v, double t) {
    double s, e0, e1;
    two_sum(*v, t, &s, &e1);
    two_sum(*u, s, &s, &e0);
    if (e0 != 0.0 && e1 != 0.0) { *u = e0; *v = e1; return s; }
    if (e1 == 0.0) { *u = s; *v = e0; return 0.0; }
    *u = s; *v = e1;
    return 0.0;
}

/* numerics.md s.3 accurate ("IEEE-style") QD add (variant DDQD_ADD_ACCURATE): the eight
 * words merged by decreasing magnitude, accumulated word by word, then renormalised. */
static qd_t qd_add_acc(qd_t a, qd_t b) {
    double m[8], x[4] = { 0.0, 0.0, 0.0, 0.0 }, u, v;
    int i = 0, j = 0, k = 0, q;
    for (q = 0; q < 8; q++) {
        if (j >= 4 || (i < 4 && fabs(a.w[i]) > fabs(b.w[j]))) m[q] = a.w[i++];
        else m[q] = b.w[j++];
    }
    fast_two_sum(m[0], m[1], &u, &v);
    q = 2;
    while (k < 4) {
        if (q == 8) {
            x[k] = u;
            if (k < 3) x[k + 1] = v;
            break;
        }
        double s = three_accum(&u, &v, m[q++]);
        if (s != 0.0) x[k++] = s;
    }
    for (; q < 8; q++) x[3] = x[3] + m[q];
    return qd_renorm(x[0], x[1], x[2], x[3], 0.0);
}

static qd_t qd_sub_acc(qd_t a, qd_t b) { return qd_add_acc(a, qd_neg(b)); }
static qd_t qd_madd_acc(qd_t c, qd_t a, qd_t b) { return qd_add_acc(c, qd_mul(a, b)); }
static qd_t qd_madd_v(qd_t c, qd_t a, qd_t b) {
    if (g_variant == 1) return qd_madd_fused(c, a, b);
    if (g_variant == 2) return qd_madd_acc(c, a, b);
    return qd_madd(c, a, b);
}
static qd_t qd_add_v(qd_t x, qd_t y) { return g_variant == 2 ? qd_add_acc(x, y) : qd_add(x, y); }
static qd_t qd_sub_v(qd_t x, qd_t y) { return g_variant == 2 ? qd_sub_acc(x, y) : qd_sub(x, y); }

/* ------------------------------------------------------------------------- */
/* Scalar entry points for the pins (arrays, planar [W][n])                   */
/* ------------------------------------------------------------------------- */
void or_two_sum(int64_t n, const double *a, const double *b, double *s, double *e) {
    for (int64_t i = 0; i < n; i++) two_sum(a[i], b[i], &s[i], &e[i]);
}
void or_fast_two_sum(int64_t n, const double *a, const double *b, double *s, double *e) {
    for (int64_t i = 0; i < n; i++) fast_two_sum(a[i], b[i], &s[i], &e[i]);
}
void or_two_prod(int64_t n, const double *a, const double *b, double *p, double *e) {
    for (int64_t i = 0; i < n; i++) two_prod(a[i], b[i], &p[i], &e[i]);
}

/* op: 0 add, 1 sub, 2 mul, 3 div (DD only), 4 madd z = x + y*w, 5 fused madd (DD only),
 * 6 accurate add, 7 accurate sub, 8 accurate madd (z = x + y*w with the accurate add) */
void or_dd_op(int op, int64_t n, const double *x, const double *y, const double *w, double *z) {
    for (int64_t i = 0; i < n; i++) {
        dd_t a = { x[i], x[n + i] }, b = { y[i], y[n + i] }, r;
        switch (op) {
        case 0: r = dd_add(a, b); break;
        case 1: r = dd_sub(a, b); break;
        case 2: r = dd_mul(a, b); break;
        case 3: r = dd_div(a, b); break;
        case 5: { dd_t c = { w[i], w[n + i] }; r = dd_madd_fused(a, b, c); break; }
        case 6: r = dd_add_acc(a, b); break;
        case 7: r = dd_sub_acc(a, b); break;
        case 8: { dd_t c = { w[i], w[n + i] }; r = dd_madd_acc(a, b, c); break; }
        default: { dd_t c = { w[i], w[n + i] }; r = dd_madd(a, b, c); }
        }
        z[i] = r.hi; z[n + i] = r.lo;
    }
}

void or_qd_op(int op, int64_t n, const double *x, const double *y, const double *w, double *z) {
    for (int64_t i = 0; i < n; i++) {
        qd_t a, b, r;
        for (int k = 0; k < 4; k++) { a.w[k] = x[k * n + i]; b.w[k] = y[k * n + i]; }
        switch (op) {
        case 0: r = qd_add(a, b); break;
        case 1: r = qd_sub(a, b); break;
        case 2: r = qd_mul(a, b); break;
        case 6: r = qd_add_acc(a, b); break;
        case 7: r = qd_sub_acc(a, b); break;
        default: {
            qd_t c;
            for (int k = 0; k < 4; k++) c.w[k] = w[k * n + i];
            r = op == 8 ? qd_madd_acc(a, b, c) : op == 5 ? qd_madd_fused(a, b, c) : qd_madd(a, b, c);
        }
        }
        for (int k = 0; k < 4; k++) z[k * n + i] = r.w[k];
    }
}

void or_qd_renorm(int64_t n, const double *c, double *out) {
    for (int64_t i = 0; i < n; i++) {
        qd_t r = qd_renorm(c[i], c[n + i], c[2 * n + i], c[3 * n + i], c[4 * n + i]);
        for (int k = 0; k < 4; k++) out[k * n + i] = r.w[k];
    }
}

int or_dd_abs_gt(const double *x, const double *y) {
    dd_t a = { x[0], x[1] }, b = { y[0], y[1] };
    return dd_abs_gt(a, b);
}

/* ------------------------------------------------------------------------- */
/* Matrices: planar row-major view, W words per element                       */
/* element (i,j) word w at p[w*ps + i*ld + j]                                  */
/* ------------------------------------------------------------------------- */
typedef struct {
    int W;
    int64_t rows, cols, ld, ps;
    double *p;
} mat_t;

static int64_t g_leaf_madds = 0;   /* instrumented counters (count law) */
static int64_t g_block_adds = 0;

int64_t or_counter_madds(void) { return g_leaf_madds; }
int64_t or_counter_block_adds(void) { return g_block_adds; }
void or_counter_reset(void) { g_leaf_madds = 0; g_block_adds = 0; }

static mat_t mat_alloc(int W, int64_t rows, int64_t cols) {
    mat_t m;
    m.W = W; m.rows = rows; m.cols = cols; m.ld = cols; m.ps = rows * cols;
    m.p = (double *)calloc((size_t)(W * rows * cols > 0 ? W * rows * cols : 1), sizeof(double));
    return m;
}

static double get_w(const mat_t *m, int w, int64_t i, int64_t j) { return m->p[w * m->ps + i * m->ld + j]; }
static void set_w(mat_t *m, int w, int64_t i, int64_t j, double v) { m->p[w * m->ps + i * m->ld + j] = v; }

/* Zero-padded copy of the sub-block [r0, r0+rows) x [c0, c0+cols) of src
 * (rows/cols beyond src are exact zeros: numerics.md s.4 halving and padding). */
static mat_t mat_quadrant(const mat_t *src, int64_t r0, int64_t c0, int64_t rows, int64_t cols) {
    mat_t q = mat_alloc(src->W, rows, cols);
    for (int w = 0; w < src->W; w++)
        for (int64_t i = 0; i < rows; i++)
            for (int64_t j = 0; j < cols; j++)
                if (r0 + i < src->rows && c0 + j < src->cols)
                    set_w(&q, w, i, j, get_w(src, w, r0 + i, c0 + j));
    return q;
}

/* Elementwise z = x (+|-) y in DD/QD (numerics.md s.4: dd_add/dd_sub, qd_add/qd_sub). */
static mat_t mat_addsub(const mat_t *x, const mat_t *y, int sub) {
    mat_t z = mat_alloc(x->W, x->rows, x->cols);
    g_block_adds++;
    for (int64_t i = 0; i < x->rows; i++)
        for (int64_t j = 0; j < x->cols; j++) {
            if (x->W == 2) {
                dd_t a = { get_w(x, 0, i, j), get_w(x, 1, i, j) };
                dd_t b = { get_w(y, 0, i, j), get_w(y, 1, i, j) };
                dd_t r = sub ? dd_sub_v(a, b) : dd_add_v(a, b);
                set_w(&z, 0, i, j, r.hi); set_w(&z, 1, i, j, r.lo);
            } else {
                qd_t a, b, r;
                for (int w = 0; w < 4; w++) { a.w[w] = get_w(x, w, i, j); b.w[w] = get_w(y, w, i, j); }
                r = sub ? qd_sub_v(a, b) : qd_add_v(a, b);
                for (int w = 0; w < 4; w++) set_w(&z, w, i, j, r.w[w]);
            }
        }
    return z;
}

static mat_t mat_add(const mat_t *x, const mat_t *y) { return mat_addsub(x, y, 0); }
static mat_t mat_sub(const mat_t *x, const mat_t *y) { return mat_addsub(x, y, 1); }

/* Simple (Eq. 1): c_ij := +0; for k ascending c_ij := madd(c_ij, a_ik, b_kj).
 * The i-k-j loop keeps every element's k order (numerics.md s.4). */
static void gemm_simple(const mat_t *A, const mat_t *B, mat_t *C) {
    int64_t m = A->rows, l = A->cols, n = B->cols;
    int W = A->W;
    g_leaf_madds += m * l * n;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; i++) {
        double *acc = (double *)calloc((size_t)(W * (n > 0 ? n : 1)), sizeof(double));
        for (int64_t k = 0; k < l; k++) {
            if (W == 2) {
                dd_t a = { get_w(A, 0, i, k), get_w(A, 1, i, k) };
                for (int64_t j = 0; j < n; j++) {
                    dd_t c = { acc[j], acc[n + j] };
                    dd_t b = { get_w(B, 0, k, j), get_w(B, 1, k, j) };
                    c = dd_madd_v(c, a, b);
                    acc[j] = c.hi; acc[n + j] = c.lo;
                }
            } else {
                qd_t a;
                for (int w = 0; w < 4; w++) a.w[w] = get_w(A, w, i, k);
                for (int64_t j = 0; j < n; j++) {
                    qd_t b, c;
                    for (int w = 0; w < 4; w++) { c.w[w] = acc[w * n + j]; b.w[w] = get_w(B, w, k, j); }
                    c = qd_madd_v(c, a, b);
                    for (int w = 0; w < 4; w++) acc[w * n + j] = c.w[w];
                }
            }
        }
        for (int w = 0; w < W; w++)
            for (int64_t j = 0; j < n; j++) set_w(C, w, i, j, acc[w * n + j]);
        free(acc);
    }
}

static mat_t view(int W, int64_t rows, int64_t cols, int64_t ld, int64_t ps, const double *p);
static mat_t mat_alloc(int W, int64_t rows, int64_t cols);
static void mat_free(mat_t *m);

/* numerics.md s.4 split-k leaf (variant DDQD_SPLITK(s)): the k range
 * is cut into s contiguous slices of ceil(l/s) (the last ragged, possibly empty); each slice's
 * partial product is the Simple sum from +0 over its k ascending; the s partials are combined
 * by the fixed pairwise tree ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7)) with the (variant's) add. */
static int g_split = 1;

static void gemm_splitk(const mat_t *A, const mat_t *B, mat_t *C, int s) {
    int64_t m = A->rows, l = A->cols, n = B->cols, L = (l + s - 1) / s;
    int W = A->W;
    mat_t P[8];
    for (int q = 0; q < s; q++) {
        int64_t k0 = q * L < l ? q * L : l, k1 = (q + 1) * L < l ? (q + 1) * L : l;
        P[q] = mat_alloc(W, m, n);
        mat_t a = view(W, m, k1 - k0, A->ld, A->ps, A->p + k0);
        mat_t b = view(W, k1 - k0, n, B->ld, B->ps, B->p + k0 * B->ld);
        gemm_simple(&a, &b, &P[q]);   /* k1 == k0: all +0 */
    }
    for (int stride = 1; stride < s; stride *= 2)
        for (int q = 0; q + stride < s; q += 2 * stride) {
            mat_t t = mat_addsub(&P[q], &P[q + stride], 0);
            g_block_adds--;   /* the split tree is not a Strassen/Winograd block addition */
            mat_free(&P[q]);
            P[q] = t;
        }
    for (int w = 0; w < W; w++)
        for (int64_t i = 0; i < m; i++)
            for (int64_t j = 0; j < n; j++) set_w(C, w, i, j, get_w(&P[0], w, i, j));
    for (int q = 0; q < s; q++) if (P[q].p) mat_free(&P[q]);
}

/* the leaf of every algorithm: Simple, or its split-k variant */
static void gemm_leaf(const mat_t *A, const mat_t *B, mat_t *C) {
    if (g_split > 1) gemm_splitk(A, B, C, g_split);
    else gemm_simple(A, B, C);
}

/* Block(bs): C_ij := sum_k A_ik B_kj over bs x bs pieces, k-blocks ascending,
 * accumulating into C in place, so each element still sees k ascending from +0. */
static void gemm_block(const mat_t *A, const mat_t *B, mat_t *C, int64_t bs) {
    int64_t m = A->rows, l = A->cols, n = B->cols;
    int W = A->W;
    g_leaf_madds += m * l * n;
    for (int w = 0; w < W; w++)
        for (int64_t i = 0; i < m; i++)
            for (int64_t j = 0; j < n; j++) set_w(C, w, i, j, 0.0);
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int64_t i0 = 0; i0 < m; i0 += bs)
        for (int64_t j0 = 0; j0 < n; j0 += bs)
            for (int64_t k0 = 0; k0 < l; k0 += bs)
                for (int64_t i = i0; i < i0 + bs && i < m; i++)
                    for (int64_t k = k0; k < k0 + bs && k < l; k++)
                        for (int64_t j = j0; j < j0 + bs && j < n; j++) {
                            if (W == 2) {
                                dd_t a = { get_w(A, 0, i, k), get_w(A, 1, i, k) };
                                dd_t b = { get_w(B, 0, k, j), get_w(B, 1, k, j) };
                                dd_t c = { get_w(C, 0, i, j), get_w(C, 1, i, j) };
                                c = dd_madd_v(c, a, b);
                                set_w(C, 0, i, j, c.hi); set_w(C, 1, i, j, c.lo);
                            } else {
                                qd_t a, b, c;
                                for (int w = 0; w < 4; w++) {
                                    a.w[w] = get_w(A, w, i, k); b.w[w] = get_w(B, w, k, j); c.w[w] = get_w(C, w, i, j);
                                }
                                c = qd_madd_v(c, a, b);
                                for (int w = 0; w < 4; w++) set_w(C, w, i, j, c.w[w]);
                            }
                        }
}

static void mat_free(mat_t *m) { free(m->p); m->p = NULL; }

/* Copy the (rows x cols) top-left of src into dst at (r0, c0), cropping to dst. */
static void mat_place(mat_t *dst, const mat_t *src, int64_t r0, int64_t c0) {
    for (int w = 0; w < dst->W; w++)
        for (int64_t i = 0; i < src->rows && r0 + i < dst->rows; i++)
            for (int64_t j = 0; j < src->cols && c0 + j < dst->cols; j++)
                set_w(dst, w, r0 + i, c0 + j, get_w(src, w, i, j));
}

/* Forced recursion depth (DDQD_DEPTH(d), reading R21): recurse exactly d levels
 * instead of applying the stop rule -- the recursion tree of a larger problem restricted to
 * a row/column band of it (the multi-GPU band schedule). -1 = the P:52 stop rule. */
static int g_fdepth = -1;

/* Strassen / Winograd with stop rule min(m,l,n) <= T and
 * explicit zero padding to (ceil(m/2), ceil(l/2), ceil(n/2)) per level. */
static void gemm_rec(int algo, int64_t T, int dep, const mat_t *A, const mat_t *B, mat_t *C) {
    int64_t m = A->rows, l = A->cols, n = B->cols;
    int64_t mn = m < l ? m : l;
    if (n < mn) mn = n;
    if (g_fdepth >= 0 ? dep >= g_fdepth : mn <= T) { gemm_leaf(A, B, C); return; }
    int64_t hm = (m + 1) / 2, hl = (l + 1) / 2, hn = (n + 1) / 2;
    mat_t A11 = mat_quadrant(A, 0, 0, hm, hl), A12 = mat_quadrant(A, 0, hl, hm, hl);
    mat_t A21 = mat_quadrant(A, hm, 0, hm, hl), A22 = mat_quadrant(A, hm, hl, hm, hl);
    mat_t B11 = mat_quadrant(B, 0, 0, hl, hn), B12 = mat_quadrant(B, 0, hn, hl, hn);
    mat_t B21 = mat_quadrant(B, hl, 0, hl, hn), B22 = mat_quadrant(B, hl, hn, hl, hn);
    mat_t P[7];
    for (int i = 0; i < 7; i++) P[i] = mat_alloc(A->W, hm, hn);
    mat_t C11, C12, C21, C22;
    if (algo == 1) {
        /* Strassen: P1..P7 */
        mat_t X, Y, t1, t2;
        X = mat_add(&A11, &A22); Y = mat_add(&B11, &B22); gemm_rec(algo, T, dep + 1, &X, &Y, &P[0]); mat_free(&X); mat_free(&Y);
        X = mat_add(&A21, &A22); gemm_rec(algo, T, dep + 1, &X, &B11, &P[1]); mat_free(&X);
        Y = mat_sub(&B12, &B22); gemm_rec(algo, T, dep + 1, &A11, &Y, &P[2]); mat_free(&Y);
        Y = mat_sub(&B21, &B11); gemm_rec(algo, T, dep + 1, &A22, &Y, &P[3]); mat_free(&Y);
        X = mat_add(&A11, &A12); gemm_rec(algo, T, dep + 1, &X, &B22, &P[4]); mat_free(&X);
        X = mat_sub(&A21, &A11); Y = mat_add(&B11, &B12); gemm_rec(algo, T, dep + 1, &X, &Y, &P[5]); mat_free(&X); mat_free(&Y);
        X = mat_sub(&A12, &A22); Y = mat_add(&B21, &B22); gemm_rec(algo, T, dep + 1, &X, &Y, &P[6]); mat_free(&X); mat_free(&Y);
        /* C11 = ((P1+P4)-P5)+P7, C12 = P3+P5, C21 = P2+P4, C22 = ((P1-P2)+P3)+P6 */
        t1 = mat_add(&P[0], &P[3]); t2 = mat_sub(&t1, &P[4]); C11 = mat_add(&t2, &P[6]); mat_free(&t1); mat_free(&t2);
        C12 = mat_add(&P[2], &P[4]);
        C21 = mat_add(&P[1], &P[3]);
        t1 = mat_sub(&P[0], &P[1]); t2 = mat_add(&t1, &P[2]); C22 = mat_add(&t2, &P[5]); mat_free(&t1); mat_free(&t2);
    } else {
        /* Winograd: S1..S4, T1..T4, M1..M7, U1..U7 */
        mat_t S1 = mat_add(&A21, &A22), S2 = mat_sub(&S1, &A11), S3 = mat_sub(&A11, &A21), S4 = mat_sub(&A12, &S2);
        mat_t T1 = mat_sub(&B12, &B11), T2 = mat_sub(&B22, &T1), T3 = mat_sub(&B22, &B12), T4 = mat_sub(&T2, &B21);
        gemm_rec(algo, T, dep + 1, &A11, &B11, &P[0]);
        gemm_rec(algo, T, dep + 1, &A12, &B21, &P[1]);
        gemm_rec(algo, T, dep + 1, &S4, &B22, &P[2]);
        gemm_rec(algo, T, dep + 1, &A22, &T4, &P[3]);
        gemm_rec(algo, T, dep + 1, &S1, &T1, &P[4]);
        gemm_rec(algo, T, dep + 1, &S2, &T2, &P[5]);
        gemm_rec(algo, T, dep + 1, &S3, &T3, &P[6]);
        mat_free(&S1); mat_free(&S2); mat_free(&S3); mat_free(&S4);
        mat_free(&T1); mat_free(&T2); mat_free(&T3); mat_free(&T4);
        mat_t U2 = mat_add(&P[0], &P[5]);
        mat_t U3 = mat_add(&U2, &P[6]);
        mat_t U4 = mat_add(&U2, &P[4]);
        C11 = mat_add(&P[0], &P[1]);          /* U1 */
        C12 = mat_add(&U4, &P[2]);            /* U5 */
        C21 = mat_sub(&U3, &P[3]);            /* U6 */
        C22 = mat_add(&U3, &P[4]);            /* U7 */
        mat_free(&U2); mat_free(&U3); mat_free(&U4);
    }
    mat_place(C, &C11, 0, 0);
    mat_place(C, &C12, 0, hn);
    mat_place(C, &C21, hm, 0);
    mat_place(C, &C22, hm, hn);
    mat_free(&C11); mat_free(&C12); mat_free(&C21); mat_free(&C22);
    for (int i = 0; i < 7; i++) mat_free(&P[i]);
    mat_free(&A11); mat_free(&A12); mat_free(&A21); mat_free(&A22);
    mat_free(&B11); mat_free(&B12); mat_free(&B21); mat_free(&B22);
}

static mat_t view(int W, int64_t rows, int64_t cols, int64_t ld, int64_t ps, const double *p) {
    mat_t m;
    m.W = W; m.rows = rows; m.cols = cols; m.ld = ld; m.ps = ps; m.p = (double *)p;
    return m;
}

static void gemm_any(int algo, int64_t T, const mat_t *A, const mat_t *B, mat_t *C) {
    if (algo == 0) gemm_leaf(A, B, C);
    else gemm_rec(algo, T, 0, A, B, C);
}

/* C := A B, planar contiguous [W][m][l] x [W][l][n] -> [W][m][n].
 * algo: 0 Block (== Simple bitwise), 1 Strassen, 2 Winograd; T = n_min.
 * bs > 0 selects the explicitly tiled Block(bs) loop nest (for the Block == Simple pin). */
int or_gemm(int W, int algo, int64_t T, int64_t bs, int64_t m, int64_t l, int64_t n,
            const double *A, const double *B, double *C, int nthreads) {
    if ((algo & 0x100) && (algo & 0x200)) return -1;
    if (algo & ~0xff33ff) return -1;
    g_variant = (algo & 0x100) ? 1 : (algo & 0x200) ? 2 : 0;
    g_fdepth = ((algo >> 16) & 0xff) - 1;        /* DDQD_DEPTH(d): d + 1 in bits 16-23 */
    g_split = 1 << ((algo >> 12) & 3);           /* DDQD_SPLITK: 1, 2, 4 or 8 */
    algo &= 0xff;
    if ((W != 2 && W != 4) || algo < 0 || algo > 2 || m < 0 || l < 0 || n < 0) return -1;
    if (algo != 0 && T < 1) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    mat_t a = view(W, m, l, l, m * l, A), b = view(W, l, n, n, l * n, B), c = view(W, m, n, n, m * n, C);
    if (algo == 0 && bs > 0) gemm_block(&a, &b, &c, bs);
    else gemm_any(algo, T, &a, &b, &c);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* numerics.md s.3: qd_div and the QD magnitude order (LU) */
/* ------------------------------------------------------------------------- */
static qd_t qd_div(qd_t a, qd_t b) {
    qd_t r = a, t;
    double q[4];
    for (int i = 0; i < 3; i++) {
        q[i] = r.w[0] / b.w[0];
        t.w[0] = q[i]; t.w[1] = 0.0; t.w[2] = 0.0; t.w[3] = 0.0;
        r = qd_sub(r, qd_mul(b, t));
    }
    q[3] = r.w[0] / b.w[0];
    return qd_renorm(q[0], q[1], q[2], q[3], 0.0);
}

static int qd_abs_gt(qd_t x, qd_t y) {
    qd_t ax = x.w[0] >= 0.0 ? x : qd_neg(x);
    qd_t ay = y.w[0] >= 0.0 ? y : qd_neg(y);
    for (int i = 0; i < 4; i++)
        if (ax.w[i] != ay.w[i]) return ax.w[i] > ay.w[i];
    return 0;
}

int or_qd_abs_gt(const double *x, const double *y) {
    qd_t a, b;
    for (int k = 0; k < 4; k++) { a.w[k] = x[k]; b.w[k] = y[k]; }
    return qd_abs_gt(a, b);
}

void or_qd_div(int64_t n, const double *x, const double *y, double *z) {
    for (int64_t i = 0; i < n; i++) {
        qd_t a, b, r;
        for (int k = 0; k < 4; k++) { a.w[k] = x[k * n + i]; b.w[k] = y[k * n + i]; }
        r = qd_div(a, b);
        for (int k = 0; k < 4; k++) z[k * n + i] = r.w[k];
    }
}

/* A W-word scalar for the LU (DD when W = 2, QD when W = 4). */
typedef struct { double w[4]; } sc_t;

static sc_t sc_from_dd(dd_t v) { sc_t r = { { v.hi, v.lo, 0.0, 0.0 } }; return r; }
static dd_t sc_dd(sc_t v) { dd_t r = { v.w[0], v.w[1] }; return r; }
static qd_t sc_qd(sc_t v) { qd_t r; for (int i = 0; i < 4; i++) r.w[i] = v.w[i]; return r; }
static sc_t sc_from_qd(qd_t v) { sc_t r; for (int i = 0; i < 4; i++) r.w[i] = v.w[i]; return r; }

static sc_t sc_sub(int W, sc_t x, sc_t y) {
    return W == 2 ? sc_from_dd(dd_sub(sc_dd(x), sc_dd(y))) : sc_from_qd(qd_sub(sc_qd(x), sc_qd(y)));
}
static sc_t sc_mul(int W, sc_t x, sc_t y) {
    return W == 2 ? sc_from_dd(dd_mul(sc_dd(x), sc_dd(y))) : sc_from_qd(qd_mul(sc_qd(x), sc_qd(y)));
}
static sc_t sc_div(int W, sc_t x, sc_t y) {
    return W == 2 ? sc_from_dd(dd_div(sc_dd(x), sc_dd(y))) : sc_from_qd(qd_div(sc_qd(x), sc_qd(y)));
}
static int sc_abs_gt(int W, sc_t x, sc_t y) {
    return W == 2 ? dd_abs_gt(sc_dd(x), sc_dd(y)) : qd_abs_gt(sc_qd(x), sc_qd(y));
}
static sc_t sc_one(void) { sc_t r = { { 1.0, 0.0, 0.0, 0.0 } }; return r; }

/* element (i,j) of a planar [W][n][n] matrix */
static sc_t ld_sc(int W, const double *A, int64_t n, int64_t i, int64_t j) {
    sc_t r = { { 0.0, 0.0, 0.0, 0.0 } };
    for (int w = 0; w < W; w++) r.w[w] = A[w * n * n + i * n + j];
    return r;
}
static void st_sc(int W, double *A, int64_t n, int64_t i, int64_t j, sc_t v) {
    for (int w = 0; w < W; w++) A[w * n * n + i * n + j] = v.w[w];
}

/* ------------------------------------------------------------------------- */
/* Steps 1-2 for the panel of columns [p, p+kb) (numerics.md s.5): column-by-column
 * factorisation with full-row interchanges, then U12 by forward substitution. Returns the
 * first k+1 whose pivot is exactly zero within this panel, else 0. */
int or_lu_panel(int W, int pivot, int64_t n, double *A, int64_t *ipiv, int64_t p, int64_t kb) {
    int info = 0;
    for (int64_t k = p; k < p + kb; k++) {
        int64_t r = k;
        if (pivot) {
            sc_t best = ld_sc(W, A, n, k, k);
            for (int64_t i = k + 1; i < n; i++) {
                sc_t v = ld_sc(W, A, n, i, k);
                if (sc_abs_gt(W, v, best)) { best = v; r = i; }
            }
        }
        ipiv[k] = r;
        if (r != k)
            for (int64_t j = 0; j < n; j++) {
                sc_t t = ld_sc(W, A, n, k, j);
                st_sc(W, A, n, k, j, ld_sc(W, A, n, r, j));
                st_sc(W, A, n, r, j, t);
            }
        sc_t piv = ld_sc(W, A, n, k, k);
        if (piv.w[0] == 0.0) { if (!info) info = (int)(k + 1); continue; }
        sc_t rinv = sc_div(W, sc_one(), piv);
#pragma omp parallel for schedule(static)
        for (int64_t i = k + 1; i < n; i++) {
            sc_t lik = sc_mul(W, ld_sc(W, A, n, i, k), rinv);
            st_sc(W, A, n, i, k, lik);
            for (int64_t j = k + 1; j < p + kb; j++)
                st_sc(W, A, n, i, j, sc_sub(W, ld_sc(W, A, n, i, j), sc_mul(W, lik, ld_sc(W, A, n, k, j))));
        }
    }
    /* step 2: U12 := L11^{-1} A12 (unit lower, forward substitution in row order) */
    for (int64_t i = p; i < p + kb; i++)
#pragma omp parallel for schedule(static)
        for (int64_t r = i + 1; r < p + kb; r++) {
            sc_t lri = ld_sc(W, A, n, r, i);
            for (int64_t j = p + kb; j < n; j++)
                st_sc(W, A, n, r, j, sc_sub(W, ld_sc(W, A, n, r, j), sc_mul(W, lri, ld_sc(W, A, n, i, j))));
        }
    return info;
}

/* ------------------------------------------------------------------------- */
/* numerics.md s.5: blocked right-looking LU (P:121-133 steps 1-3); partial  */
/* pivoting per BJ:11 (pivot = 1) or the paper's pivot-free LU (pivot = 0,   */
/* P:121). A is n x n planar [W][n][n], overwritten by L\U; ipiv[k] = pivot  */
/* row. Returns info: 0, or k+1 for the first exactly-zero pivot.            */
/* ------------------------------------------------------------------------- */
int or_lu(int W, int pivot, int64_t n, double *A, int64_t *ipiv, int64_t K, int algo, int64_t T,
          int nthreads) {
    int info = 0;
    /* the accurate-add variant is a GEMM variant; the LU's own panel, TRSM and solve
     * arithmetic is the canonical one, so an accurate LU is not defined (rejected) */
    if (algo & 0x200) return -1;
    g_variant = (algo & 0x100) ? 1 : 0;
    g_fdepth = -1;                               /* the LU's updates use the P:52 stop rule */
    g_split = 1 << ((algo >> 12) & 3);
    algo &= 0xff;
    if ((W != 2 && W != 4) || n < 0 || K < 1) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    for (int64_t p = 0; p < n; p += K) {
        int64_t kb = (n - p < K) ? n - p : K;
        /* steps 1-2 */
        int pinfo = or_lu_panel(W, pivot, n, A, ipiv, p, kb);
        if (!info) info = pinfo;
        int64_t n2 = n - p - kb;
        if (n2 <= 0) continue;
        /* step 3: A22 := A22 - L21 U12, T := gemm(L21, U12) first (the underlined term) */
        mat_t L21 = mat_alloc(W, n2, kb), U12 = mat_alloc(W, kb, n2), Tm = mat_alloc(W, n2, n2);
        for (int w = 0; w < W; w++) {
            for (int64_t i = 0; i < n2; i++)
                for (int64_t j = 0; j < kb; j++) set_w(&L21, w, i, j, A[w * n * n + (p + kb + i) * n + p + j]);
            for (int64_t i = 0; i < kb; i++)
                for (int64_t j = 0; j < n2; j++) set_w(&U12, w, i, j, A[w * n * n + (p + i) * n + p + kb + j]);
        }
        gemm_any(algo, T, &L21, &U12, &Tm);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n2; i++)
            for (int64_t j = 0; j < n2; j++) {
                sc_t t = { { 0.0, 0.0, 0.0, 0.0 } };
                for (int w = 0; w < W; w++) t.w[w] = get_w(&Tm, w, i, j);
                int64_t gi = p + kb + i, gj = p + kb + j;
                st_sc(W, A, n, gi, gj, sc_sub(W, ld_sc(W, A, n, gi, gj), t));
            }
        mat_free(&L21); mat_free(&U12); mat_free(&Tm);
    }
    return info;
}

/* Solve with the factors of or_lu (numerics.md s.5): y := P b; forward (unit L,
 * j ascending); backward (j descending, x_j = div(y_j, u_jj)). b, x: [W][n]. */
void or_lu_solve(int W, int64_t n, const double *LU, const int64_t *ipiv, const double *b, double *x) {
    double *y = (double *)malloc((size_t)(W * (n > 0 ? n : 1)) * sizeof(double));
    for (int64_t i = 0; i < W * n; i++) y[i] = b[i];
    for (int64_t k = 0; k < n; k++) {
        int64_t r = ipiv[k];
        if (r != k)
            for (int w = 0; w < W; w++) {
                double t = y[w * n + k];
                y[w * n + k] = y[w * n + r];
                y[w * n + r] = t;
            }
    }
#define YV(i) ({ sc_t v_ = { { 0.0, 0.0, 0.0, 0.0 } }; for (int w_ = 0; w_ < W; w_++) v_.w[w_] = y[w_ * n + (i)]; v_; })
#define YS(i, v) do { sc_t s_ = (v); for (int w_ = 0; w_ < W; w_++) y[w_ * n + (i)] = s_.w[w_]; } while (0)
    for (int64_t j = 0; j < n; j++) {
        sc_t yj = YV(j);
        for (int64_t i = j + 1; i < n; i++) YS(i, sc_sub(W, YV(i), sc_mul(W, ld_sc(W, LU, n, i, j), yj)));
    }
    for (int64_t j = n - 1; j >= 0; j--) {
        sc_t xj = sc_div(W, YV(j), ld_sc(W, LU, n, j, j));
        for (int w = 0; w < W; w++) x[w * n + j] = xj.w[w];
        for (int64_t i = 0; i < j; i++) YS(i, sc_sub(W, YV(i), sc_mul(W, ld_sc(W, LU, n, i, j), xj)));
    }
#undef YV
#undef YS
    free(y);
}
