// Lattice formats and the element-level helpers shared by every kernel of
// the library: word-plane matrix references (SoA planes, batch stride, row
// stride), exact loads into a quad-double value, the rounding store into a
// lattice format with an exact power-of-two scaling (fp32 levels live inside
// the fp32 exponent range; the reference's MPFR exponents are unbounded,
// SPEC.md:84) and the Horner add B_{j-1} + T of engine.py:249-251 formed in
// the output format's working type.
//
// (Round 1 also had a tiled SIMT DFMA / FFMA GEMM here behind an engine
// switch; it was retired in round 2 -- every product of the path runs on the
// INT8 tensor cores, ozaki.cuh.)
#pragma once
#include "mp_arith.cuh"

namespace mpps {

enum Fmt { F32 = 0, F64 = 1, DD = 2, QD = 3 };

template <int F> struct FmtT;
template <> struct FmtT<F32> { static constexpr int W = 1; using word = float; };
template <> struct FmtT<F64> { static constexpr int W = 1; using word = double; };
template <> struct FmtT<DD>  { static constexpr int W = 2; using word = double; };
template <> struct FmtT<QD>  { static constexpr int W = 4; using word = double; };

struct MatRef {
  void *data;
  long long plane;   // elements between word planes
  long long bstride; // elements between matrices of the batch
  int ld;
  int words;         // number of planes actually stored (1, 2 or 4)
};

struct HornerEpi {
  MatRef Bprev;        // working-format block B_{j-1} (words = 1, 2 or 4, double)
  const int *exp_y;    // per batch index (may be null -> 0)
  const int *exp_in;
  const int *exp_out;
};

// cp.async with zero fill (src-size 0 when out of bounds: ragged tiles).
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void *smem, const void *gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int src = pred ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES), "r"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ----------------------------------------------------- value load / store
__device__ __forceinline__ mp::qd load_qd(const MatRef &m, long long off) {
  const double *p = (const double *)m.data + off;
  double w0 = p[0];
  double w1 = m.words > 1 ? p[m.plane] : 0.0;
  double w2 = m.words > 2 ? p[2 * m.plane] : 0.0;
  double w3 = m.words > 3 ? p[3 * m.plane] : 0.0;
  return mp::qd_make(w0, w1, w2, w3);
}

// Round v (exact value held as a qd) into format FO and store it scaled by
// 2^e.  fp32 rounding happens after the scaling, so with e chosen by the host
// (see engine.py mirror) the stored fp32 word is the 24-bit rounding of the
// unbounded-exponent value.
template <int FO>
__device__ __forceinline__ void store_fmt(const MatRef &m, long long off, const mp::qd &v, int e) {
  if constexpr (FO == F32) {
    mp::dd d = mp::qd_to_dd(v);
    if (e) d = mp::dd_ldexp(d, e);
    ((float *)m.data)[off] = mp::dd_to_float(d.hi, d.lo);
  } else if constexpr (FO == F64) {
    mp::dd d = mp::qd_to_dd(v);
    ((double *)m.data)[off] = e ? mp::dd_ldexp(d, e).hi : d.hi;
  } else if constexpr (FO == DD) {
    mp::dd d = mp::qd_to_dd(v);
    if (e) d = mp::dd_ldexp(d, e);
    double *p = (double *)m.data + off;
    p[0] = d.hi; p[m.plane] = d.lo;
  } else {
    mp::qd q = e ? mp::qd_ldexp(v, e) : v;
    double *p = (double *)m.data + off;
    p[0] = q.x[0]; p[m.plane] = q.x[1]; p[2 * m.plane] = q.x[2]; p[3 * m.plane] = q.x[3];
  }
}

// B + T evaluated in format FO's working type (single rounding into FO for
// fp32/fp64 outputs: the sum is formed in dd first).
template <int FO>
__device__ __forceinline__ mp::qd horner_add(const mp::qd &B, const mp::qd &T) {
  if constexpr (FO == QD) {
    return mp::qd_add(B, T);
  } else {
    mp::dd s = mp::dd_add(mp::qd_to_dd(B), mp::qd_to_dd(T));
    return mp::qd_make(s.hi, s.lo, 0.0, 0.0);
  }
}

}  // namespace mpps
