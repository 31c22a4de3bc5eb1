// ddqd_arith.cuh -- DD/QD device arithmetic (north_star subsystem (1)).
//
// Every operation is the sequence fixed in docs/numerics.md s.1-3, written with the
// correctly-rounded intrinsics __dadd_rn/__dsub_rn/__dmul_rn/__fma_rn so that nvcc can
// neither contract nor reassociate them (the library is also built with --fmad=false).
// All of it runs on the FP64 pipe (DADD/DMUL/DFMA); tensor cores cannot provide the
// exact FMA the error-free transforms need (BJ:5).
#pragma once
#include <cstdint>

namespace ddqd {

// ---- s.1 error-free transforms ------------------------------------------
__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void fast_two_sum(double a, double b, double &s, double &e) {
    s = __dadd_rn(a, b);
    e = __dsub_rn(b, __dsub_rn(s, a));
}
__device__ __forceinline__ void two_prod(double a, double b, double &p, double &e) {
    p = __dmul_rn(a, b);
    e = __fma_rn(a, b, -p);
}

// ---- s.2 double-double --------------------------------------------------------
struct dd { double hi, lo; };

__device__ __forceinline__ dd dd_add(dd x, dd y) {
    double s, e;
    two_sum(x.hi, y.hi, s, e);
    double t = __dadd_rn(x.lo, y.lo);
    e = __dadd_rn(e, t);
    dd r;
    fast_two_sum(s, e, r.hi, r.lo);
    return r;
}
__device__ __forceinline__ dd dd_neg(dd x) { return dd{-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    double p, e;
    two_prod(x.hi, y.hi, p, e);
    double t = __dadd_rn(__dmul_rn(x.hi, y.lo), __dmul_rn(x.lo, y.hi));
    e = __dadd_rn(e, t);
    dd r;
    fast_two_sum(p, e, r.hi, r.lo);
    return r;
}
// 20 FP64 instructions: 3 DMUL + 1 DFMA + 16 DADD.
__device__ __forceinline__ dd dd_madd(dd c, dd a, dd b) { return dd_add(c, dd_mul(a, b)); }
// Fused variant (numerics.md s.2, NEXT row f3): the product's error terms are folded with
// FMAs and added to c without renormalising the product first. 15 FP64 instructions:
// 1 DMUL + 3 DFMA + 11 DADD.
__device__ __forceinline__ dd dd_madd_fused(dd c, dd a, dd b) {
    const double p = __dmul_rn(a.hi, b.hi);
    double e = __fma_rn(a.hi, b.hi, -p);
    e = __fma_rn(a.hi, b.lo, e);
    e = __fma_rn(a.lo, b.hi, e);
    double s, t;
    two_sum(c.hi, p, s, t);
    t = __dadd_rn(t, __dadd_rn(c.lo, e));
    dd r;
    fast_two_sum(s, t, r.hi, r.lo);
    return r;
}
// Accurate ("IEEE-style") add (numerics.md s.2, variant DDQD_ADD_ACCURATE, SURVEY.md s.8(f)
// row f3): both word pairs error-free, two renormalisations; 20 DADD.
__device__ __forceinline__ dd dd_add_acc(dd x, dd y) {
    double s1, s2, t1, t2;
    two_sum(x.hi, y.hi, s1, s2);
    two_sum(x.lo, y.lo, t1, t2);
    s2 = __dadd_rn(s2, t1);
    fast_two_sum(s1, s2, s1, s2);
    s2 = __dadd_rn(s2, t2);
    dd r;
    fast_two_sum(s1, s2, r.hi, r.lo);
    return r;
}
__device__ __forceinline__ dd dd_sub_acc(dd x, dd y) { return dd_add_acc(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_madd_acc(dd c, dd a, dd b) { return dd_add_acc(c, dd_mul(a, b)); }
__device__ __forceinline__ dd dd_div(dd x, dd y) {
    double q1 = __ddiv_rn(x.hi, y.hi);
    dd r = dd_sub(x, dd_mul(y, dd{q1, 0.0}));
    double q2 = __ddiv_rn(r.hi, y.hi);
    dd out;
    fast_two_sum(q1, q2, out.hi, out.lo);
    return out;
}
// |x| > |y| in the DD magnitude order (numerics.md s.2).
__device__ __forceinline__ bool dd_abs_gt(dd x, dd y) {
    dd ax = x.hi >= 0.0 ? x : dd_neg(x);
    dd ay = y.hi >= 0.0 ? y : dd_neg(y);
    if (ax.hi != ay.hi) return ax.hi > ay.hi;
    return ax.lo > ay.lo;
}

// ---- s.3 quad-double (Hida-Li-Bailey "sloppy" algorithms) ---------------------------
struct qd { double w[4]; };

__device__ __forceinline__ void three_sum(double &a, double &b, double &c) {
    double t1, t2, t3;
    two_sum(a, b, t1, t2);
    two_sum(c, t1, a, t3);
    two_sum(t2, t3, b, c);
}
__device__ __forceinline__ void three_sum2(double &a, double &b, double c) {
    double t1, t2, t3;
    two_sum(a, b, t1, t2);
    two_sum(c, t1, a, t3);
    b = __dadd_rn(t2, t3);
}
// IEEE "x != 0" on the bit pattern (-0 == 0). The move goes through inline PTX so nvcc
// cannot fold it back into a DSETP: the test runs on the integer pipe, not the FP64 pipe.
__device__ __forceinline__ bool nz(double x) {
    unsigned long long u;
    asm("mov.b64 %0, %1;" : "=l"(u) : "d"(x));
    return (u << 1) != 0ull;
}

__device__ __forceinline__ qd qd_renorm(double c0, double c1, double c2, double c3, double c4) {
    double s, t0, t1, t2, t3, t4;
    fast_two_sum(c3, c4, s, t4);
    fast_two_sum(c2, s, s, t3);
    fast_two_sum(c1, s, s, t2);
    fast_two_sum(c0, s, t0, t1);
    double s0 = t0, s1 = t1, s2 = 0.0, s3 = 0.0;
    if (nz(s1)) {
        fast_two_sum(s1, t2, s1, s2);
        if (nz(s2)) {
            fast_two_sum(s2, t3, s2, s3);
            if (nz(s3)) s3 = __dadd_rn(s3, t4);
            else        s2 = __dadd_rn(s2, t4);
        } else {
            fast_two_sum(s1, t3, s1, s2);
            if (nz(s2)) fast_two_sum(s2, t4, s2, s3);
            else        fast_two_sum(s1, t4, s1, s2);
        }
    } else {
        fast_two_sum(s0, t2, s0, s1);
        if (nz(s1)) {
            fast_two_sum(s1, t3, s1, s2);
            if (nz(s2)) fast_two_sum(s2, t4, s2, s3);
            else        fast_two_sum(s1, t4, s1, s2);
        } else {
            fast_two_sum(s0, t3, s0, s1);
            if (nz(s1)) fast_two_sum(s1, t4, s1, s2);
            else        fast_two_sum(s0, t4, s0, s1);
        }
    }
    qd r;
    r.w[0] = s0; r.w[1] = s1; r.w[2] = s2; r.w[3] = s3;
    return r;
}

__device__ __forceinline__ qd qd_add(const qd &a, const qd &b) {
    double s0, s1, s2, s3, t0, t1, t2, t3;
    two_sum(a.w[0], b.w[0], s0, t0);
    two_sum(a.w[1], b.w[1], s1, t1);
    two_sum(a.w[2], b.w[2], s2, t2);
    two_sum(a.w[3], b.w[3], s3, t3);
    two_sum(s1, t0, s1, t0);
    three_sum(s2, t0, t1);
    three_sum2(s3, t0, t2);
    t0 = __dadd_rn(__dadd_rn(t0, t1), t3);
    return qd_renorm(s0, s1, s2, s3, t0);
}
__device__ __forceinline__ qd qd_neg(const qd &a) {
    qd r;
#pragma unroll
    for (int i = 0; i < 4; i++) r.w[i] = -a.w[i];
    return r;
}
__device__ __forceinline__ qd qd_sub(const qd &a, const qd &b) { return qd_add(a, qd_neg(b)); }

__device__ __forceinline__ qd qd_mul(const qd &a, const qd &b) {
    double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5;
    two_prod(a.w[0], b.w[0], p0, q0);
    two_prod(a.w[0], b.w[1], p1, q1);
    two_prod(a.w[1], b.w[0], p2, q2);
    two_prod(a.w[0], b.w[2], p3, q3);
    two_prod(a.w[1], b.w[1], p4, q4);
    two_prod(a.w[2], b.w[0], p5, q5);
    three_sum(p1, p2, q0);
    three_sum(p2, q1, q2);
    three_sum(p3, p4, p5);
    double s0, s1, s2, t0, t1;
    two_sum(p2, p3, s0, t0);
    two_sum(q1, p4, s1, t1);
    s2 = __dadd_rn(q2, p5);
    two_sum(s1, t0, s1, t0);
    s2 = __dadd_rn(s2, __dadd_rn(t0, t1));
    double tail = __dmul_rn(a.w[0], b.w[3]);
    tail = __dadd_rn(tail, __dmul_rn(a.w[1], b.w[2]));
    tail = __dadd_rn(tail, __dmul_rn(a.w[2], b.w[1]));
    tail = __dadd_rn(tail, __dmul_rn(a.w[3], b.w[0]));
    tail = __dadd_rn(tail, q0);
    tail = __dadd_rn(tail, q3);
    tail = __dadd_rn(tail, q4);
    tail = __dadd_rn(tail, q5);
    s1 = __dadd_rn(s1, tail);
    return qd_renorm(p0, p1, s0, s1, s2);
}
__device__ __forceinline__ qd qd_madd(const qd &c, const qd &a, const qd &b) {
    return qd_add(c, qd_mul(a, b));
}

// |x| > |y| for finite doubles on the integer pipe (sign bit cleared, unsigned compare)
__device__ __forceinline__ bool abs_gt_bits(double x, double y) {
    unsigned long long ux, uy;
    asm("mov.b64 %0, %1;" : "=l"(ux) : "d"(x));
    asm("mov.b64 %0, %1;" : "=l"(uy) : "d"(y));
    return (ux << 1) > (uy << 1);
}
__device__ __forceinline__ double word_at(const qd &a, int i) {   // 0 past the last word
    return i == 0 ? a.w[0] : i == 1 ? a.w[1] : i == 2 ? a.w[2] : i == 3 ? a.w[3] : 0.0;
}
// ThreeAccum (numerics.md s.3): t into the two-word accumulator (u, v); returns the completed
// word, or 0 when none completed
__device__ __forceinline__ double three_accum(double &u, double &v, double t) {
    double s, e0, e1;
    two_sum(v, t, s, e1);
    two_sum(u, s, s, e0);
    if (nz(e0) && nz(e1)) { u = e0; v = e1; return s; }
    if (!nz(e1)) { u = s; v = e0; return 0.0; }
    u = s; v = e1;
    return 0.0;
}
// Accurate QD add (numerics.md s.3, variant DDQD_ADD_ACCURATE): the eight words merged by
// decreasing magnitude, accumulated with ThreeAccum, leftovers folded into the last word,
// renormalised. Written branch-light with static register indices (fully unrolled).
__device__ __forceinline__ qd qd_add_acc(const qd &a, const qd &b) {
    double m[8];
    int i = 0, j = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        const double ai = word_at(a, i), bj = word_at(b, j);
        const bool ta = j >= 4 || (i < 4 && abs_gt_bits(ai, bj));
        m[q] = ta ? ai : bj;
        i += ta ? 1 : 0;
        j += ta ? 0 : 1;
    }
    double u, v;
    fast_two_sum(m[0], m[1], u, v);
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
    int k = 0, qend = 8;
#pragma unroll
    for (int q = 2; q < 8; q++) {
        if (k < 4) {
            const double s = three_accum(u, v, m[q]);
            if (nz(s)) {
                if (k == 0) x0 = s; else if (k == 1) x1 = s; else if (k == 2) x2 = s; else x3 = s;
                k++;
                if (k == 4) qend = q + 1;
            }
        }
    }
    if (k < 4) {
        if (k == 0) { x0 = u; x1 = v; }
        else if (k == 1) { x1 = u; x2 = v; }
        else if (k == 2) { x2 = u; x3 = v; }
        else x3 = u;
    } else {
#pragma unroll
        for (int q = 2; q < 8; q++)
            if (q >= qend) x3 = __dadd_rn(x3, m[q]);
    }
    return qd_renorm(x0, x1, x2, x3, 0.0);
}
__device__ __forceinline__ qd qd_sub_acc(const qd &a, const qd &b) { return qd_add_acc(a, qd_neg(b)); }
__device__ __forceinline__ qd qd_madd_acc(const qd &c, const qd &a, const qd &b) {
    return qd_add_acc(c, qd_mul(a, b));
}

// Fused QD multiply-add (numerics.md s.3, variant DDQD_MADD_FUSED): qd_mul's five-term
// product expansion is added to c by the qd_add network without renormalising it first.
__device__ __forceinline__ qd qd_madd_fused(const qd &c, const qd &a, const qd &b) {
    double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5;
    two_prod(a.w[0], b.w[0], p0, q0);
    two_prod(a.w[0], b.w[1], p1, q1);
    two_prod(a.w[1], b.w[0], p2, q2);
    two_prod(a.w[0], b.w[2], p3, q3);
    two_prod(a.w[1], b.w[1], p4, q4);
    two_prod(a.w[2], b.w[0], p5, q5);
    three_sum(p1, p2, q0);
    three_sum(p2, q1, q2);
    three_sum(p3, p4, p5);
    double s0, s1, s2, t0, t1;
    two_sum(p2, p3, s0, t0);
    two_sum(q1, p4, s1, t1);
    s2 = __dadd_rn(q2, p5);
    two_sum(s1, t0, s1, t0);
    s2 = __dadd_rn(s2, __dadd_rn(t0, t1));
    double tail = __dmul_rn(a.w[0], b.w[3]);
    tail = __dadd_rn(tail, __dmul_rn(a.w[1], b.w[2]));
    tail = __dadd_rn(tail, __dmul_rn(a.w[2], b.w[1]));
    tail = __dadd_rn(tail, __dmul_rn(a.w[3], b.w[0]));
    tail = __dadd_rn(tail, q0);
    tail = __dadd_rn(tail, q3);
    tail = __dadd_rn(tail, q4);
    tail = __dadd_rn(tail, q5);
    s1 = __dadd_rn(s1, tail);
    double u0, u1, u2, u3, v0, v1, v2, v3;
    two_sum(c.w[0], p0, u0, v0);
    two_sum(c.w[1], p1, u1, v1);
    two_sum(c.w[2], s0, u2, v2);
    two_sum(c.w[3], s1, u3, v3);
    two_sum(u1, v0, u1, v0);
    three_sum(u2, v0, v1);
    three_sum2(u3, v0, v2);
    v0 = __dadd_rn(__dadd_rn(__dadd_rn(v0, v1), v3), s2);
    return qd_renorm(u0, u1, u2, u3, v0);
}

// qd_div (numerics.md s.3): long division with three correction steps, then renorm.
__device__ __forceinline__ qd qd_div(const qd &a, const qd &b) {
    qd r = a, t;
    double q[4];
#pragma unroll
    for (int i = 0; i < 3; i++) {
        q[i] = __ddiv_rn(r.w[0], b.w[0]);
        t.w[0] = q[i]; t.w[1] = 0.0; t.w[2] = 0.0; t.w[3] = 0.0;
        r = qd_sub(r, qd_mul(b, t));
    }
    q[3] = __ddiv_rn(r.w[0], b.w[0]);
    return qd_renorm(q[0], q[1], q[2], q[3], 0.0);
}
// |x| > |y| in the QD magnitude order (words compared lexicographically after the sign fold)
__device__ __forceinline__ bool qd_abs_gt(const qd &x, const qd &y) {
    const qd ax = x.w[0] >= 0.0 ? x : qd_neg(x);
    const qd ay = y.w[0] >= 0.0 ? y : qd_neg(y);
#pragma unroll
    for (int i = 0; i < 4; i++)
        if (ax.w[i] != ay.w[i]) return ax.w[i] > ay.w[i];
    return false;
}

// ---- width-generic element type: W = 2 (DD) or 4 (QD) -----------------------------
template <int W> struct elem;
template <> struct elem<2> {
    using T = dd;
    static __device__ __forceinline__ T zero() { return dd{0.0, 0.0}; }
    static __device__ __forceinline__ T add(T x, T y) { return dd_add(x, y); }
    static __device__ __forceinline__ T sub(T x, T y) { return dd_sub(x, y); }
    static __device__ __forceinline__ T madd(T c, T a, T b) { return dd_madd(c, a, b); }
    static __device__ __forceinline__ T madd_fused(T c, T a, T b) { return dd_madd_fused(c, a, b); }
    static __device__ __forceinline__ T add_acc(T x, T y) { return dd_add_acc(x, y); }
    static __device__ __forceinline__ T sub_acc(T x, T y) { return dd_sub_acc(x, y); }
    static __device__ __forceinline__ T madd_acc(T c, T a, T b) { return dd_madd_acc(c, a, b); }
    static __device__ __forceinline__ T load(const double *p, int64_t ps) { return dd{p[0], p[ps]}; }
    static __device__ __forceinline__ void store(double *p, int64_t ps, T v) { p[0] = v.hi; p[ps] = v.lo; }
    static __device__ __forceinline__ double word(const T &v, int w) { return w == 0 ? v.hi : v.lo; }
    static __device__ __forceinline__ void set_word(T &v, int w, double x) { if (w == 0) v.hi = x; else v.lo = x; }
    static __device__ __forceinline__ T one() { return dd{1.0, 0.0}; }
    static __device__ __forceinline__ T mul(T x, T y) { return dd_mul(x, y); }
    static __device__ __forceinline__ T div(T x, T y) { return dd_div(x, y); }
    static __device__ __forceinline__ bool abs_gt(T x, T y) { return dd_abs_gt(x, y); }
};
template <> struct elem<4> {
    using T = qd;
    static __device__ __forceinline__ T zero() { qd r; r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0.0; return r; }
    static __device__ __forceinline__ T add(const T &x, const T &y) { return qd_add(x, y); }
    static __device__ __forceinline__ T sub(const T &x, const T &y) { return qd_sub(x, y); }
    static __device__ __forceinline__ T madd(const T &c, const T &a, const T &b) { return qd_madd(c, a, b); }
    static __device__ __forceinline__ T madd_fused(const T &c, const T &a, const T &b) { return qd_madd_fused(c, a, b); }
    static __device__ __forceinline__ T add_acc(const T &x, const T &y) { return qd_add_acc(x, y); }
    static __device__ __forceinline__ T sub_acc(const T &x, const T &y) { return qd_sub_acc(x, y); }
    static __device__ __forceinline__ T madd_acc(const T &c, const T &a, const T &b) { return qd_madd_acc(c, a, b); }
    static __device__ __forceinline__ T load(const double *p, int64_t ps) {
        qd r; r.w[0] = p[0]; r.w[1] = p[ps]; r.w[2] = p[2 * ps]; r.w[3] = p[3 * ps]; return r;
    }
    static __device__ __forceinline__ void store(double *p, int64_t ps, const T &v) {
        p[0] = v.w[0]; p[ps] = v.w[1]; p[2 * ps] = v.w[2]; p[3 * ps] = v.w[3];
    }
    static __device__ __forceinline__ double word(const T &v, int w) { return v.w[w]; }
    static __device__ __forceinline__ void set_word(T &v, int w, double x) { v.w[w] = x; }
    static __device__ __forceinline__ T one() { qd r; r.w[0] = 1.0; r.w[1] = r.w[2] = r.w[3] = 0.0; return r; }
    static __device__ __forceinline__ T mul(const T &x, const T &y) { return qd_mul(x, y); }
    static __device__ __forceinline__ T div(const T &x, const T &y) { return qd_div(x, y); }
    static __device__ __forceinline__ bool abs_gt(const T &x, const T &y) { return qd_abs_gt(x, y); }
};

// Arithmetic variant of a GEMM (the algo flags): V = 0 canonical, 1 fused DD madd
// (DDQD_MADD_FUSED), 2 accurate adds everywhere (DDQD_ADD_ACCURATE). Kernels take
// E = arith<W, V> and call E::add / E::sub / E::madd.
template <int W, int V> struct arith : elem<W> {
    using B = elem<W>;
    using T = typename B::T;
    static __device__ __forceinline__ T add(const T &x, const T &y) { return V == 2 ? B::add_acc(x, y) : B::add(x, y); }
    static __device__ __forceinline__ T sub(const T &x, const T &y) { return V == 2 ? B::sub_acc(x, y) : B::sub(x, y); }
    static __device__ __forceinline__ T madd(const T &c, const T &a, const T &b) {
        return V == 1 ? B::madd_fused(c, a, b) : V == 2 ? B::madd_acc(c, a, b) : B::madd(c, a, b);
    }
};

}  // namespace ddqd
