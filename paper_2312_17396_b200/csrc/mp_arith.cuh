// Multiword floating-point arithmetic for sm_100a: error-free transforms (EFTs)
// built from DFMA/DADD, double-double (dd, ~106 bits) and quad-double
// (qd, ~212 bits) values, and the fused multiply-accumulate chains used by
// the GEMM main loops.
//
// The reference rounds every scalar op at p = ceil(d*log2 10) bits through
// MPFR (pkg/src/mpps/precision.py:160-184).  The B200 lattice replaces those
// contexts by hardware formats: d<=7 -> fp32, d<=15 -> fp64, d<=31 -> dd,
// d<=63 -> qd.  Every EFT below uses the *_rn
// intrinsics so nvcc cannot contract or reassociate them.
#pragma once
#include <cuda_runtime.h>

// Programmatic dependent launch: first statement of every kernel the host
// launches with programmaticStreamSerialization (mpps_capi.cu launch_k).  The
// wait returns once the preceding kernel in the stream has completed and its
// writes are visible (a no-op for an ordinary launch), so nothing of the
// predecessor is read or overwritten early; the trigger lets the next kernel's
// CTAs be placed on SMs freed by this grid's last wave.
#define MPPS_PDL_ENTER() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

#include <stdint.h>

#define MP_INLINE __device__ __forceinline__

namespace mp {

// ---------------------------------------------------------------- EFTs
MP_INLINE double add(double a, double b) { return __dadd_rn(a, b); }
MP_INLINE double sub(double a, double b) { return __dsub_rn(a, b); }
MP_INLINE double mul(double a, double b) { return __dmul_rn(a, b); }
MP_INLINE double fma(double a, double b, double c) { return __fma_rn(a, b, c); }

// Knuth TwoSum: s + e == a + b exactly (6 FP64-pipe ops, no branch).
MP_INLINE void two_sum(double a, double b, double &s, double &e) {
  s = add(a, b);
  double v = sub(s, a);
  e = add(sub(a, sub(s, v)), sub(b, v));
}
// Dekker FastTwoSum, requires exponent(a) >= exponent(b) (3 ops).
MP_INLINE void quick_two_sum(double a, double b, double &s, double &e) {
  s = add(a, b);
  e = sub(b, sub(s, a));
}
// TwoProd via FMA: p + e == a * b exactly (2 ops).
MP_INLINE void two_prod(double a, double b, double &p, double &e) {
  p = mul(a, b);
  e = fma(a, b, -p);
}

// ---------------------------------------------------------------- dd
struct dd { double hi, lo; };

MP_INLINE dd dd_make(double h, double l) { dd r; r.hi = h; r.lo = l; return r; }

// Accurate dd + dd (two TwoSums; relative error ~ 2^-106 even under
// cancellation).
MP_INLINE dd dd_add(dd a, dd b) {
  double s, e, t, f;
  two_sum(a.hi, b.hi, s, e);
  two_sum(a.lo, b.lo, t, f);
  e = add(e, t);
  quick_two_sum(s, e, s, e);
  e = add(e, f);
  quick_two_sum(s, e, s, e);
  return dd_make(s, e);
}
// "Sloppy" dd add: one TwoSum on the high words (error <= ~2^-106 (|a|+|b|),
// normwise; 11 FP64 instructions instead of 20).
MP_INLINE dd dd_add_sloppy(dd a, dd b) {
  double s, e;
  two_sum(a.hi, b.hi, s, e);
  e = add(e, add(a.lo, b.lo));
  quick_two_sum(s, e, s, e);
  return dd_make(s, e);
}
MP_INLINE dd dd_add_d(dd a, double b) {
  double s, e;
  two_sum(a.hi, b, s, e);
  e = add(e, a.lo);
  quick_two_sum(s, e, s, e);
  return dd_make(s, e);
}
MP_INLINE dd dd_mul(dd a, dd b) {
  double p, e;
  two_prod(a.hi, b.hi, p, e);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  quick_two_sum(p, e, p, e);
  return dd_make(p, e);
}
MP_INLINE dd dd_neg(dd a) { return dd_make(-a.hi, -a.lo); }
MP_INLINE dd dd_ldexp(dd a, int k) {
  // exact power-of-two multiply when 2^k is a normal double (same rounding
  // as ldexp, which is much longer in SASS)
  if (k >= -1022 && k <= 1023) {
    const double p = __longlong_as_double((long long)(k + 1023) << 52);
    return dd_make(a.hi * p, a.lo * p);
  }
  return dd_make(ldexp(a.hi, k), ldexp(a.lo, k));
}

// Correctly rounded dd -> fp32.  If hi is not an fp32 midpoint, hi+lo
// rounds like hi (|lo| <= ulp_double(hi)/2 < distance to the midpoint);
// if hi is exactly a midpoint the sign of lo breaks the tie.
MP_INLINE float dd_to_float(double hi, double lo) {
  float f = __double2float_rn(hi);
  double back = (double)f;
  double d = sub(hi, back);
  if (d != 0.0 && lo != 0.0 && isfinite(f)) {
    float up = nextafterf(f, d > 0 ? INFINITY : -INFINITY);
    double half = 0.5 * sub((double)up, back);
    if (d == half && ((lo > 0) == (half > 0))) f = up;
  }
  return f;
}

// ---------------------------------------------------------------- qd
struct qd { double x[4]; };

MP_INLINE qd qd_make(double a, double b, double c, double d) {
  qd r; r.x[0] = a; r.x[1] = b; r.x[2] = c; r.x[3] = d; return r;
}

// One exact VecSum sweep (bottom-up): the running sum flows into c[0], the
// rounding errors stay behind.  sum(c) is invariant.
template <int N>
MP_INLINE void vecsum_sweep(double (&c)[N]) {
#pragma unroll
  for (int i = N - 1; i >= 1; --i) two_sum(c[i - 1], c[i], c[i - 1], c[i]);
}

// Renormalise a 4-level expansion (level k ~ eps^k, possibly overlapping or
// cancelling) into a non-overlapping qd: three exact sweeps, branch free.
MP_INLINE qd qd_renorm(double c0, double c1, double c2, double c3) {
  double c[4] = {c0, c1, c2, c3};
  vecsum_sweep(c);
  vecsum_sweep(c);
  vecsum_sweep(c);
  return qd_make(c[0], c[1], c[2], c[3]);
}

// qd + qd by magnitude levels: exact TwoSums on levels 0-2, plain sum on
// level 3 (error ~eps^4 max(|a|,|b|)), then renormalise.
MP_INLINE qd qd_add(const qd &a, const qd &b) {
  double s0, t0, s1, t1, s2, t2, x, y1, y2;
  two_sum(a.x[0], b.x[0], s0, t0);
  two_sum(a.x[1], b.x[1], s1, t1);
  two_sum(a.x[2], b.x[2], s2, t2);
  double s3 = add(a.x[3], b.x[3]);
  two_sum(s1, t0, s1, x);
  two_sum(s2, t1, s2, y1);
  two_sum(s2, x, s2, y2);
  s3 = add(add(s3, t2), add(y1, y2));
  return qd_renorm(s0, s1, s2, s3);
}

MP_INLINE qd qd_from_dd(dd a) { return qd_make(a.hi, a.lo, 0.0, 0.0); }
MP_INLINE qd qd_from_d(double a) { return qd_make(a, 0.0, 0.0, 0.0); }
MP_INLINE qd qd_ldexp(const qd &a, int k) {
  return qd_make(ldexp(a.x[0], k), ldexp(a.x[1], k), ldexp(a.x[2], k), ldexp(a.x[3], k));
}
MP_INLINE qd qd_neg(const qd &a) { return qd_make(-a.x[0], -a.x[1], -a.x[2], -a.x[3]); }
// qd -> dd (nearest, up to ties at 2^-106 that cannot matter here).
MP_INLINE dd qd_to_dd(const qd &a) {
  double s, e;
  quick_two_sum(a.x[0], add(a.x[1], add(a.x[2], a.x[3])), s, e);
  return dd_make(s, e);
}

// ------------------------------------------------- GEMM accumulators
// dd accumulation of a*b into an unnormalised (ch, cl) pair.  12 FP64-pipe
// instructions per MAC: 1 DMUL + 3 DFMA (exact hi*hi error and the two cross
// terms) + TwoSum(6) + 2 DADD.  The low word is renormalised once per K-tile
// (dd_acc_renorm), which bounds |cl| <= BK * u * max|partial sum| and keeps the
// accumulated error at ~BK*n*u^2 |A||B| (u = 2^-53), well below the dd
// tolerance 10*r*n*10^-31 used by the parity tests.
MP_INLINE void dd_mac(double ah, double al, double bh, double bl, double &ch, double &cl) {
  double p = mul(ah, bh);
  double e = fma(ah, bh, -p);
  e = fma(ah, bl, e);
  e = fma(al, bh, e);
  double s = add(ch, p);
  double v = sub(s, ch);
  double t = add(sub(ch, sub(s, v)), sub(p, v));
  cl = add(cl, add(t, e));
  ch = s;
}
// 9-FP64-instruction variant: the hi-word sum uses Dekker's FastTwoSum on
// magnitude-ordered operands (exact for |big| >= |small|), the ordering done
// with integer compares/selects on the ALU pipe; the cross terms are folded
// into cl by FMA.  FP64 pipe: DMUL + 3 DFMA + 3 DADD + 2 DADD.
MP_INLINE void dd_mac9(double ah, double al, double bh, double bl, double &ch, double &cl) {
  double p = mul(ah, bh);
  double e = fma(ah, bh, -p);
  cl = fma(ah, bl, cl);
  cl = fma(al, bh, cl);
  double s = add(ch, p);
  // |ch| >= |p| as unsigned compare of the magnitude bit patterns
  unsigned long long mc = (unsigned long long)__double_as_longlong(ch) & 0x7fffffffffffffffULL;
  unsigned long long mp_ = (unsigned long long)__double_as_longlong(p) & 0x7fffffffffffffffULL;
  bool cbig = mc >= mp_;
  double big = cbig ? ch : p;
  double small = cbig ? p : ch;
  double t = sub(small, sub(s, big));
  cl = add(cl, add(t, e));
  ch = s;
}
MP_INLINE void dd_acc_renorm(double &ch, double &cl) {
  double s, e;
  two_sum(ch, cl, s, e);
  ch = s; cl = e;
}

// qd accumulation into magnitude levels c0..c3 (level k ~ eps^k |c0|).
// Level-0..2 items are added with exact TwoSums whose errors carry to the
// next level; level 3 is a plain sum (its rounding error is ~eps^4).
MP_INLINE void qd_mac(const double a[4], const double b[4], double c[4]) {
  double p00, e00, p01, e01, p10, e10, p02, e02, p11, e11, p20, e20;
  two_prod(a[0], b[0], p00, e00);
  two_prod(a[0], b[1], p01, e01);
  two_prod(a[1], b[0], p10, e10);
  two_prod(a[0], b[2], p02, e02);
  two_prod(a[1], b[1], p11, e11);
  two_prod(a[2], b[0], p20, e20);
  double l3 = mul(a[0], b[3]);
  l3 = fma(a[1], b[2], l3);
  l3 = fma(a[2], b[1], l3);
  l3 = fma(a[3], b[0], l3);
  l3 = add(l3, add(add(e02, e11), e20));
  // level 0
  double r0;
  two_sum(c[0], p00, c[0], r0);
  // level 1: r0, e00, p01, p10
  double x1, x2, x3, x4;
  two_sum(c[1], r0, c[1], x1);
  two_sum(c[1], e00, c[1], x2);
  two_sum(c[1], p01, c[1], x3);
  two_sum(c[1], p10, c[1], x4);
  // level 2: x1..x4, e01, e10, p02, p11, p20 (exact), errors -> level 3
  double y, acc3 = l3;
  two_sum(c[2], x1, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], x2, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], x3, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], x4, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], e01, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], e10, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], p02, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], p11, c[2], y); acc3 = add(acc3, y);
  two_sum(c[2], p20, c[2], y); acc3 = add(acc3, y);
  c[3] = add(c[3], acc3);
}
MP_INLINE void qd_acc_renorm(double c[4]) {
  qd q = qd_renorm(c[0], c[1], c[2], c[3]);
  c[0] = q.x[0]; c[1] = q.x[1]; c[2] = q.x[2]; c[3] = q.x[3];
}

// qd * qd through the same level cascade as the GEMM MAC.
MP_INLINE qd qd_mul(const qd &a, const qd &b) {
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  qd_mac(a.x, b.x, c);
  return qd_renorm(c[0], c[1], c[2], c[3]);
}

}  // namespace mp
