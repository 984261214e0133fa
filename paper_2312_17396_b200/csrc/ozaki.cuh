// Multiword GEMMs on the INT8 tensor cores (tcgen05.mma kind::i8) by exact
// operand splitting (Ozaki scheme I).
//
//   A (rows scaled by 2^-ea_i) = sum_{s<S} a_s 2^-(6+7s),   a_s int8 in [-65, 65]
//   B (cols scaled by 2^-eb_j) = sum_{t<S} b_t 2^-(6+7t)
//   A B = 2^(ea_i+eb_j) sum_{d<S} 2^-(12+7d) D_d,   D_d = sum_{s+t=d} a_s b_t
//
// Every D_d is an exact int32 accumulation over K on the tensor cores (one
// TMEM accumulator per diagonal d, all (s,t) pairs of the diagonal issued into
// it); pairs with s+t >= S are dropped (their weight is below 2^-(12+7S),
// i.e. below the target format's unit roundoff for S = 8 / 16 / 31 slices
// -> fp64 / dd / qd).  The epilogue recombines the diagonals exactly (groups
// of three fit a double), sums them in the target format, applies the
// power-of-two row/column scales and then the same store / fused Horner
// epilogue helpers (formats.cuh).
//
// Slices are stored K-major ([S][batch][rows_pad][K_pad] int8, rows_pad a
// multiple of the tile, K_pad of 32, padding zero), B transposed (its columns
// are the rows of the slice arrays).  Shared-memory operand tiles use the
// canonical no-swizzle K-major UMMA layout: 8-row x 16-byte core matrices,
// LBO = 128 B between the two 16-byte K chunks of one MMA-K step, SBO = 256 B
// between 8-row groups.
#pragma once
#include <cuda.h>
#include <cooperative_groups.h>
#include "formats.cuh"

namespace mpps {
namespace oz {

constexpr int kTileM = 128;
constexpr int kKStep = 32;      // int8 MMA K per instruction (32 bytes)
constexpr int kThreadsEpi = 256;   // TMA/ring kernels: 8 warps (producer, MMA issuer, 8 epilogue)

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;              // descriptor version (Blackwell)
  d |= (uint64_t)(layout & 7) << 61;   // 0 = SWIZZLE_NONE, 6 = SWIZZLE_32B
  return d;                            // base offset 0
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes) : "memory");
}

// 3-D TMA tile load into shared memory, completion counted on an mbarrier.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}

// kind::i8 instruction descriptor: D s32, A/B signed int8, K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(mbar), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mbar) : "memory");
}
// named barrier among the `n` threads of the epilogue warps (id 1; 0 is __syncthreads)
__device__ __forceinline__ void epi_bar_sync(int n) { asm volatile("bar.sync 1, %0;\n" ::"r"(n) : "memory"); }

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(dst_smem), "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// 8 consecutive 32-bit columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, int32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

__host__ __device__ constexpr int tmem_cols_for(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// ------------------------------------------------------------- slicing
struct SliceRef {
  int8_t *digits;   // [S][batch][rpad][kpad]
  int *exps;        // [batch][rpad]
  int S, batch, rpad, kpad;
  int db;           // digit bits: 7 (digits in [-65, 65]) or 8 ([-128, 127]); first digit 6 bits
  int row0 = 0;     // column splits: first slice row written (mpps_slice_into)
  int nrows = 1 << 30;   // and the number of rows written (default: through rpad)
  int given = 0;    // exps already hold the row / column exponents (mpps_slice_ex mode 2)
  __host__ __device__ long long plane() const { return (long long)batch * rpad * kpad; }
};

// Digit width of a tensor-core product: S = 14 / 28 planes exist only as
// 8-bit digits, 16 / 31 only as 7-bit ones; 4 and 8 planes are prefixes of
// either split (the operands' SliceRef.db, equal for A and B).
template <int S>
__host__ __device__ constexpr bool oz_has7() {   // a 7-bit variant exists
  return !(S == 14 || S == 28 || S == 2 || S == 3 || S == 5 || S == 6 || S == 10 || S == 12);
}
template <int S>
__device__ __forceinline__ int oz_db_of(int db) {
  // 14 / 28 and the per-level plane counts of the 8-bit split (2, 3, 5, 6,
  // 10, 12) exist only with 8-bit digits
  if constexpr (S == 14 || S == 28 || S == 2 || S == 3 || S == 5 || S == 6 || S == 10 || S == 12) return 8;
  else if constexpr (S == 16 || S == 31) return 7;
  else return db == 8 ? 8 : 7;
}

// Split one exact value (W words, |v| < 1 after scaling) into S signed
// digits: first 6 bits, then db = 7 or 8 bits each.  The residual is kept exactly
// (scaling by 2^k and subtracting the nearest integer are exact; the words
// are renormalised with TwoSums), so sum_s d_s 2^-(6+7s) is the value
// truncated after S digits.
// 2^e as a double (exact); e within the normal range.
__device__ __forceinline__ double pow2i(int e) {
  if (e >= -1022 && e <= 1023) return __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(1.0, e);
}

// v * 2^k on the first W words (exact power-of-two multiply; ldexp only
// outside the normal range of 2^k)
template <int W>
__device__ __forceinline__ mp::qd scale_words(mp::qd v, int k) {
  if (k >= -1022 && k <= 1023) {
    const double p = __longlong_as_double((long long)(k + 1023) << 52);
#pragma unroll
    for (int w = 0; w < W; ++w) v.x[w] *= p;
    return v;
  }
  return mp::qd_ldexp(v, k);
}

template <int W, int S, int DB>
__device__ __forceinline__ void split_digits_wi(const mp::qd &v, int (&dg)[S]) {
  // Digit s is the nearest integer to the running residual times 2^6 (s = 0)
  // or 2^7.  Rounding uses the 1.5*2^52 shifter fused into the scaling FMA
  // (FP64 pipe only; the digit is the low word of the shifted value), and
  // the residual update x0 = x0*2^k - d is exact.  Lower words are carried
  // lazily: they are rescaled and folded into x0 every kFold digits (exact
  // two-sum chain), which keeps |x0| <= 0.5 + 2^-25 between folds, so every
  // digit stays in [-65, 65] and sum_s d_s 2^-(6+7s) + residual == v exactly.
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
  constexpr int kFold = 4;
  double x[W];
#pragma unroll
  for (int w = 0; w < W; ++w) x[w] = v.x[w];
  double pend = 1.0;  // scale owed to the lower words since the last fold
  constexpr double scd = DB == 8 ? 256.0 : 128.0;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const double sc = (s == 0) ? 64.0 : scd;
    if constexpr (W > 1) {
      pend *= sc;
      if (s > 0 && s % kFold == 0) {
#pragma unroll
        for (int w = 1; w < W; ++w) x[w] *= pend / sc;  // lower words to x0's scale
        double c = x[0];
#pragma unroll
        for (int w = 1; w < W; ++w) {
          double t, e;
          mp::two_sum(c, x[w], t, e);
          x[w - 1] = t;
          c = e;
        }
        x[W - 1] = c;
        pend = sc;
      }
    }
    const double t = fma(x[0], sc, kShift);
    const double d = t - kShift;
    x[0] = fma(x[0], sc, -d);  // exact
    dg[s] = __double2loint(t);  // low byte = the digit (two's complement)
  }
  if constexpr (DB == 8) {
    // nearest-integer base-256 digits lie in [-128, 128]; carry the +128s
    // (and anything outside int8) into the next more significant digit,
    // bottom up -- the value is unchanged, every digit lands in [-128, 127]
    // and the 6-bit first digit in [-65, 65]
#pragma unroll
    for (int s = S - 1; s >= 1; --s) {   // digits >= -128 always; only +128 / +129 carry
      const int c = dg[s] > 127;
      dg[s] -= c << 8;
      dg[s - 1] += c;
    }
  }
}

template <int W, int S, int DB>
__device__ __forceinline__ void split_digits_w(const mp::qd &v, int8_t (&dg)[S]) {
  int di[S];
  split_digits_wi<W, S, DB>(v, di);
#pragma unroll
  for (int s = 0; s < S; ++s) dg[s] = (int8_t)di[s];
}

// Non-finite entries: a NaN or Inf in a row (column) must not come back as
// finite digits.  AbsMax reports such a row (column) maximum as +Inf (fmax
// alone drops NaNs), and row_exponent answers Inf with kExpNonFinite: every product entry of that
// row (column) is then scaled by 2^kExpNonFinite = Inf in the GEMM epilogues
// (pow2i), i.e. comes out Inf or NaN as mat_mul's would (precision.py:160-184),
// and the block norms carry it to the planner, which raises.
constexpr int kExpNonFinite = 1 << 20;
// running maximum of |v| taken on the bit patterns: for non-negative doubles
// the integer order is the numeric order and Inf / NaN are the largest
// patterns, so a non-finite entry stays (fmax drops NaNs) at the cost of the
// integer compare-and-select that replaces fmax's DSETP + selects
struct AbsMax {
  long long m = 0;
  __device__ __forceinline__ void add(double v) { m = max(m, __double_as_longlong(v) & 0x7fffffffffffffffll); }
  __device__ __forceinline__ double value() const {
    return m >= 0x7ff0000000000000ll ? __longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double(m);
  }
};
__device__ __forceinline__ int row_exponent(double mx) {
  int e = 0;
  if (!(mx < __longlong_as_double(0x7ff0000000000000ll))) return kExpNonFinite;
  if (mx > 0.0) {
    frexp(mx, &e);  // mx in [2^(e-1), 2^e)
    // a multiword value may exceed its leading word by half an ulp: one bit
    // of headroom when the maximum sits just below a power of two
    if (ldexp(mx, -e) > 0.9999999999) e += 1;
  }
  return e;
}

// 8-bit digits by exact fixed-point arithmetic (W <= 2 words, S <= 14):
// V = round(v 2^(F - e)), F = 6 + 8 (S-1) <= 110 fractional bits, formed
// with 16 guard bits in an int128 (words shifted into place by their
// exponents; bits below the guard bits are dropped, so V is the nearest
// integer up to a 2^-16 ulp tie window).  The balanced base-256 digits are
// then carry-free: the bytes of Y = V + 0x80..80 (S-1 bytes) are d_s + 128,
// i.e. d_s = byte ^ 0x80 read as int8 for s >= 1, and the top digit d_0 is
// the (signed) byte S-1 of Y.  No FP64 work and no carry pass.
template <int S>
__host__ __device__ constexpr unsigned long long fixed_cmask_lo() {
  unsigned long long c = 0;
  for (int k = 0; k < S - 1 && k < 8; ++k) c |= 0x80ull << (8 * k);
  return c;
}
template <int S>
__host__ __device__ constexpr unsigned long long fixed_cmask_hi() {
  unsigned long long c = 0;
  for (int k = 8; k < S - 1; ++k) c |= 0x80ull << (8 * (k - 8));
  return c;
}

template <int W, int S>
__device__ __forceinline__ unsigned __int128 fixed_biased(const mp::qd &v, int e) {
  constexpr int F = 6 + 8 * (S - 1);
  constexpr int G = 16;
  static_assert(W <= 2 && F + G <= 126, "fixed-point split: at most 2 words and 14 planes");
  __int128 acc = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const long long bits = __double_as_longlong(v.x[w]);
    const int ex = (int)((bits >> 52) & 0x7ff);
    const long long mant = bits & 0xfffffffffffffLL;
    const long long m = ex ? (mant | 0x10000000000000LL) : mant;   // subnormals: no implicit bit
    const int sh = (ex ? ex : 1) - 1075 + F + G - e;                // |v| < 2^e  =>  sh < F + G - 52
    __int128 t = 0;
    if (sh >= 0) t = (__int128)m << sh;
    else if (sh > -64) t = (__int128)(m >> (-sh));
    acc += bits < 0 ? -t : t;
  }
  const __int128 V = (acc + ((__int128)1 << (G - 1))) >> G;
  const unsigned __int128 C = ((unsigned __int128)fixed_cmask_hi<S>() << 64) | fixed_cmask_lo<S>();
  return (unsigned __int128)V + C;
}

// Same V (up to the rounding of the low word, |V - v 2^(F-e)| <= 1) with
// explicit 64-bit limbs instead of generic variable 128-bit shifts
// (~3x fewer integer instructions per entry; the split is issue-bound):
// hi = m_h 2^x_h with |hi| < 2^e gives s = x_h + F - e <= F - 53, i.e.
// s < 64 for S <= 14, so m_h << s needs one funnel step; lo (<= half an ulp
// of hi) lands at s - 53 <= 4 and is added as a rounded signed 64-bit value.
// the W stored words of a W-word source (W from the format: no run-time word count)
template <int W>
__device__ __forceinline__ mp::qd load_w(const MatRef &m, long long off) {
  const double *p = (const double *)m.data + off;
  return mp::qd_make(p[0], W > 1 ? p[m.plane] : 0.0, W > 2 ? p[2 * m.plane] : 0.0, W > 3 ? p[3 * m.plane] : 0.0);
}
__device__ __forceinline__ void dbl_int_parts(double x, long long &m, int &ex) {
  const long long bits = __double_as_longlong(x);
  const int eb = (int)((bits >> 52) & 0x7ff);
  const long long mant = bits & 0xfffffffffffffLL;
  const long long mm = eb ? (mant | 0x10000000000000LL) : mant;
  m = bits < 0 ? -mm : mm;
  ex = (eb ? eb : 1) - 1075;
}
// round(m 2^s) for s <= 4 (signed 64-bit; s < 0 rounds half up)
__device__ __forceinline__ long long shift_round64(long long m, int s) {
  const int t = min(max(-s, 1), 62);
  const long long down = (m + (1LL << (t - 1))) >> t;
  return s >= 0 ? (m << (s & 63)) : down;
}
template <int W, int S>
__device__ __forceinline__ unsigned __int128 fixed_biased_fast(const mp::qd &v, int e) {
  constexpr int F = 6 + 8 * (S - 1);
  static_assert(W <= 2 && F - 53 < 64, "fixed-point split: at most 2 words and 14 planes");
  long long mh;
  int xh;
  dbl_int_parts(v.x[0], mh, xh);
  const int sh = xh + F - e;
  unsigned long long L;
  long long H;
  {                                    // m_h << sh (sh <= F - 53 < 64) or rounded m_h 2^sh
    const int sp = sh & 63;
    const long long r = shift_round64(mh, sh);
    const long long hs = sp ? (mh >> (64 - sp)) : (mh >> 63);
    L = sh >= 0 ? ((unsigned long long)mh << sp) : (unsigned long long)r;
    H = sh >= 0 ? hs : (r >> 63);
  }
  if constexpr (W == 2) {
    long long ml;
    int xl;
    dbl_int_parts(v.x[1], ml, xl);
    const long long w = shift_round64(ml, xl + F - e);      // ml = 0 -> 0
    const unsigned long long L2 = L + (unsigned long long)w;
    H += (w >> 63) + (L2 < L ? 1 : 0);
    L = L2;
  }
  const unsigned __int128 V = ((unsigned __int128)(unsigned long long)H << 64) | L;
  const unsigned __int128 C = ((unsigned __int128)fixed_cmask_hi<S>() << 64) | fixed_cmask_lo<S>();
  return V + C;
}

// The same V as fixed_biased_fast, with the alignment done on the FP64 pipe
// (the split is ALU-bound: ncu on slice_rows_kernel<2,14> at cfg2 showed the
// ALU pipe 73 % busy at ~150 instructions per entry, ~100 of them integer
// shifts/selects of the 128-bit alignment above).  The row's 2^(F-e) comes
// as two normal factors p1 p2 (F - e spans [-1015, 1183]); w 2^(F-e) is then
// exact wherever it can round to a nonzero integer (an intermediate below
// 2^-1022 only arises when the result is < 2^-1022 as well), the half-up
// rounding is floor(a + 1/2) below 2^52 (exact there; above, a is already an
// integer), and the 128-bit two's complement comes from |r| = q 2^64 + rem
// (q, rem exact doubles) converted with F2I and negated.
__device__ __forceinline__ double pow2_normal(int k) {   // k in [-1022, 1023]
  return __longlong_as_double((long long)(k + 1023) << 52);
}
template <int S>
__device__ __forceinline__ void fixed_scale(int e, double &p1, double &p2) {
  constexpr int F = 6 + 8 * (S - 1);
  const int k = F - e, k1 = k >> 1;
  p1 = pow2_normal(k1);
  p2 = pow2_normal(k - k1);
}
__device__ __forceinline__ double round_half_up_scaled(double w, double p1, double p2) {
  const double a = __dmul_rn(__dmul_rn(w, p1), p2);
  return fabs(a) < 0x1p52 ? floor(__dadd_rn(a, 0.5)) : a;
}
template <int W, int S>
__device__ __forceinline__ unsigned __int128 fixed_biased_fp(double h, double l, double p1, double p2) {
  static_assert(W <= 2 && 6 + 8 * (S - 1) - 53 < 64, "fixed-point split: at most 2 words and 14 planes");
  const double r = round_half_up_scaled(h, p1, p2);
  const double m = fabs(r);
  const double q = trunc(__dmul_rn(m, 0x1p-64));
  const double rem = __fma_rn(-q, 0x1p64, m);
  unsigned long long L = __double2ull_rz(rem);
  unsigned long long H = __double2ull_rz(q);
  {                                    // branch-free 128-bit negate for r < 0
    const bool neg = r < 0.0;
    const unsigned long long nH = ~H + (L == 0ull ? 1ull : 0ull), nL = 0ull - L;
    H = neg ? nH : H;
    L = neg ? nL : L;
  }
  if constexpr (W == 2) {
    const long long w = __double2ll_rz(round_half_up_scaled(l, p1, p2));
    const unsigned long long L2 = L + (unsigned long long)w;
    H += (unsigned long long)(w >> 63) + (L2 < L ? 1ull : 0ull);
    L = L2;
  }
  const unsigned __int128 V = ((unsigned __int128)H << 64) | L;
  const unsigned __int128 C = ((unsigned __int128)fixed_cmask_hi<S>() << 64) | fixed_cmask_lo<S>();
  return V + C;
}

// byte k of the 128-bit Y as the low byte of an int
__device__ __forceinline__ uint32_t fixed_word(const unsigned __int128 &Y, int j) {
  return (uint32_t)(Y >> (32 * j));
}

// The S plane words of four consecutive entries (digit s = byte S-1-s of Y;
// bytes below the top one are offset by 0x80) stored at k0 of each plane.
template <int S>
__device__ __forceinline__ void store_plane_words(const unsigned __int128 (&Y)[4], int8_t *o, long long plane, int k0) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int kb = S - 1 - s, j = kb >> 2, bsel = kb & 3;
    const uint32_t lo = __byte_perm(fixed_word(Y[0], j), fixed_word(Y[1], j), bsel | ((bsel + 4) << 4));
    const uint32_t hi = __byte_perm(fixed_word(Y[2], j), fixed_word(Y[3], j), bsel | ((bsel + 4) << 4));
    uint32_t wv = __byte_perm(lo, hi, 0x5410);
    if (s > 0) wv ^= 0x80808080u;
    *reinterpret_cast<uint32_t *>(o + s * plane + k0) = wv;
  }
}

// Register-resident row split for rows of 128 or 256 fp64/dd entries (the
// cfg2 shapes): every lane loads its entries' words (4 consecutive per 128
// columns, 16-byte loads) before the row maximum, so one DRAM latency covers
// the row instead of a max pass followed by a second, dependent load pass.
template <int W, int S>
__device__ __forceinline__ void slice_rows_regs(const MatRef &A, long long base, int cols, int fi, const SliceRef &out,
                                                int b, int i, int lane) {
  constexpr int NIT = 2;
  double h[NIT][4], l[NIT][4];
  const double *p = (const double *)A.data + base + 4 * lane;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    if (W == 1 && fi == F32 && it * 128 < cols) {     // fp32 source: one 16-byte load, exact widening
      const float4 a = *reinterpret_cast<const float4 *>((const float *)A.data + base + 4 * lane + 128 * it);
      h[it][0] = a.x; h[it][1] = a.y; h[it][2] = a.z; h[it][3] = a.w;
#pragma unroll
      for (int q = 0; q < 4; ++q) l[it][q] = 0.0;
    } else if (it * 128 < cols) {
      const double2 a0 = *reinterpret_cast<const double2 *>(p + 128 * it);
      const double2 a1 = *reinterpret_cast<const double2 *>(p + 128 * it + 2);
      h[it][0] = a0.x; h[it][1] = a0.y; h[it][2] = a1.x; h[it][3] = a1.y;
      if constexpr (W > 1) {
        const double2 b0 = *reinterpret_cast<const double2 *>(p + A.plane + 128 * it);
        const double2 b1 = *reinterpret_cast<const double2 *>(p + A.plane + 128 * it + 2);
        l[it][0] = b0.x; l[it][1] = b0.y; l[it][2] = b1.x; l[it][3] = b1.y;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) l[it][q] = 0.0;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) h[it][q] = l[it][q] = 0.0;
    }
  }
  AbsMax am;
#pragma unroll
  for (int it = 0; it < NIT; ++it)
#pragma unroll
    for (int q = 0; q < 4; ++q) am.add(h[it][q]);
  double mx = am.value();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = row_exponent(mx);
  if (lane == 0) out.exps[(long long)b * out.rpad + i] = e;
  double p1, p2;
  fixed_scale<S>(e, p1, p2);
  const long long plane = out.plane();
  int8_t *o = out.digits + ((long long)b * out.rpad + i) * out.kpad;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    if (it * 128 < cols) {
      unsigned __int128 Y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) Y[q] = fixed_biased_fp<W, S>(h[it][q], l[it][q], p1, p2);
      store_plane_words<S>(Y, o, plane, 4 * lane + 128 * it);
    }
  }
}

// Side A: rows scaled by their own max exponent; output [S][b][i][k].
// One warp per row; each lane splits 4 consecutive entries and stores the 4
// digits of a plane as one 32-bit word.
template <int W, int S, int DB>
__device__ __forceinline__ void slice_rows_body(const MatRef &A, int rows, int cols, int fi, const SliceRef &out,
                                                const int *sel) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int bz = blockIdx.y;
  const int b = sel ? sel[bz] : bz;
  const int i = warp;
  if (i >= out.rpad) return;
  const long long base = (long long)b * A.bstride + (long long)i * A.ld;
  if constexpr (DB == 8 && W <= 2 && S <= 14) {
    // warp-uniform: the whole row is interior and 16-byte aligned
    const bool f32 = fi == F32;
    if (!out.given && i < rows && (W == 1 || !f32) && cols == out.kpad && (cols == 128 || cols == 256) && (f32 || (A.plane & 1) == 0) &&
        ((f32 ? reinterpret_cast<uintptr_t>((const float *)A.data + base)
              : reinterpret_cast<uintptr_t>((const double *)A.data + base)) & 15) == 0) {
      slice_rows_regs<W, S>(A, base, cols, fi, out, b, i, lane);
      return;
    }
  }
  int e;
  if (out.given) {
    // the row exponent of the whole panel row (SUMMA: max over the process
    // row), so this block's digits are exactly those of the gathered panel
    e = out.exps[(long long)b * out.rpad + i];
  } else {
    AbsMax am;
    if (i < rows) {
#pragma unroll 4
      for (int k = lane; k < cols; k += 32) {
        double v = fi == F32 ? (double)((const float *)A.data)[base + k] : ((const double *)A.data)[base + k];
        am.add(v);
      }
    }
    double mx = am.value();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    e = row_exponent(mx);
    if (lane == 0) out.exps[(long long)b * out.rpad + i] = e;
  }
  double p1 = 1.0, p2 = 1.0;
  if constexpr (DB == 8 && W <= 2 && S <= 14) fixed_scale<S>(e, p1, p2);
  const long long plane = out.plane();
  int8_t *o = out.digits + ((long long)b * out.rpad + i) * out.kpad;
  for (int k0 = 4 * lane; k0 < out.kpad; k0 += 128) {
    if constexpr (DB == 8 && W <= 2 && S <= 14) {
      // 8-bit digits from the exact fixed-point value (carry-free bytes)
      unsigned __int128 Y[4];
      if (i < rows && k0 + 3 < cols && fi != F32) {
        // interior: W words of four entries, no per-entry guards or format checks
        const double *p = (const double *)A.data + base + k0;
        double w0[4], w1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w0[q] = p[q];
#pragma unroll
        for (int q = 0; q < 4; ++q) w1[q] = W > 1 ? p[A.plane + q] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) Y[q] = fixed_biased_fp<W, S>(w0[q], w1[q], p1, p2);
      } else if (W == 1 && i < rows && k0 + 3 < cols) {
        // interior of an fp32 source (one word; widening to fp64 is exact)
        const float *p = (const float *)A.data + base + k0;
        float w0[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w0[q] = p[q];
#pragma unroll
        for (int q = 0; q < 4; ++q) Y[q] = fixed_biased_fp<1, S>((double)w0[q], 0.0, p1, p2);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + q;
          mp::qd v = mp::qd_make(0.0, 0.0, 0.0, 0.0);
          if (i < rows && k < cols)
            v = fi == F32 ? mp::qd_from_d((double)((const float *)A.data)[base + k]) : load_qd(A, base + k);
          Y[q] = fixed_biased_fast<W, S>(v, e);
        }
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int kb = S - 1 - s;                       // byte of Y holding digit s
        const int j = kb >> 2, bsel = kb & 3;
        const uint32_t lo = __byte_perm(fixed_word(Y[0], j), fixed_word(Y[1], j), bsel | ((bsel + 4) << 4));
        const uint32_t hi = __byte_perm(fixed_word(Y[2], j), fixed_word(Y[3], j), bsel | ((bsel + 4) << 4));
        uint32_t wv = __byte_perm(lo, hi, 0x5410);
        if (s > 0) wv ^= 0x80808080u;
        *reinterpret_cast<uint32_t *>(o + s * plane + k0) = wv;
      }
    } else if constexpr (DB == 8) {
      // 8-bit digits are final only after the bottom-up carry pass over the
      // whole entry, so the four entries are split one after another and
      // their digits inserted byte by byte into the plane words (S digits +
      // S words live instead of 4 S digits)
      uint32_t wd[S];
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + q;
        mp::qd v = mp::qd_make(0.0, 0.0, 0.0, 0.0);
        if (i < rows && k < cols) {
          v = fi == F32 ? mp::qd_from_d((double)((const float *)A.data)[base + k]) : load_qd(A, base + k);
          v = scale_words<W>(v, -e);
        }
        int dg[S];
        split_digits_wi<W, S, DB>(v, dg);
        // byte 0 of dg[s] -> byte q of wd[s] (selector nibble q = 4, others keep wd)
        const uint32_t sel = 0x3210u + ((4u - q) << (4 * q));
#pragma unroll
        for (int s = 0; s < S; ++s) wd[s] = __byte_perm(q == 0 ? 0u : wd[s], (uint32_t)dg[s], sel);
      }
#pragma unroll
      for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t *>(o + s * plane + k0) = wd[s];
    } else {
      int dq[4][S];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + q;
        mp::qd v = mp::qd_make(0.0, 0.0, 0.0, 0.0);
        if (i < rows && k < cols) {
          v = fi == F32 ? mp::qd_from_d((double)((const float *)A.data)[base + k]) : load_qd(A, base + k);
          v = scale_words<W>(v, -e);
        }
        split_digits_wi<W, S, DB>(v, dq[q]);
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {  // bytes 0 of the four digits -> one word
        const uint32_t lo = __byte_perm(dq[0][s], dq[1][s], 0x0040);
        const uint32_t hi = __byte_perm(dq[2][s], dq[3][s], 0x0040);
        *reinterpret_cast<uint32_t *>(o + s * plane + k0) = __byte_perm(lo, hi, 0x5410);
      }
    }
  }
}

template <int W, int S>
__global__ void __launch_bounds__(256, (W <= 2 && S <= 14) ? 3 : 1) slice_rows_kernel(MatRef A, int rows, int cols, int fi, SliceRef out, const int *sel) {
  MPPS_PDL_ENTER();
  if (oz_db_of<S>(out.db) == 8) {
    if constexpr (S != 16 && S != 31) slice_rows_body<W, S, 8>(A, rows, cols, fi, out, sel);
  } else {
    if constexpr (oz_has7<S>()) slice_rows_body<W, S, 7>(A, rows, cols, fi, out, sel);
  }
}

// Side A exponents only (mpps_slice_ex mode 1): one warp per row.
__global__ void row_exps_kernel(MatRef A, int rows, int cols, int fi, SliceRef out, const int *sel) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int b = sel ? sel[blockIdx.y] : (int)blockIdx.y;
  if (i >= out.rpad) return;
  AbsMax am;
  const long long base = (long long)b * A.bstride + (long long)i * A.ld;
  if (i < rows) {
#pragma unroll 4
    for (int k = lane; k < cols; k += 32) {
      double v = fi == F32 ? (double)((const float *)A.data)[base + k] : ((const double *)A.data)[base + k];
      am.add(v);
    }
  }
  double mx = am.value();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) out.exps[(long long)b * out.rpad + i] = row_exponent(mx);
}

// Side B: column exponents.  Block = 32 columns x 8 row groups; each thread
// scans every 8th row of its column (coalesced across the warp), then a
// shared-memory max over the 8 groups.
__global__ void col_exps_kernel(MatRef B, int rows, int cols, int fi, SliceRef out, const int *sel) {
  MPPS_PDL_ENTER();
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  const int bz = blockIdx.y;
  const int b = sel ? sel[bz] : bz;
  AbsMax am;
  if (j < cols) {
#pragma unroll 4
    for (int k = ty; k < rows; k += 8) {
      const long long off = (long long)b * B.bstride + (long long)k * B.ld + j;
      double v = fi == F32 ? (double)((const float *)B.data)[off] : ((const double *)B.data)[off];
      am.add(v);
    }
  }
  double mx = am.value();
  red[ty][tx] = mx;
  __syncthreads();
  if (ty == 0 && out.row0 + j < out.rpad && j < out.nrows) {
#pragma unroll
    for (int g = 1; g < 8; ++g) mx = fmax(mx, red[g][tx]);
    out.exps[(long long)b * out.rpad + out.row0 + j] = row_exponent(mx);
  }
}

// Side B digits, transposed through shared memory: tile of 32 k x 32 j.
template <int W, int S, int DB>
__device__ __forceinline__ void slice_cols_body(const MatRef &B, int rows, int cols, int fi, const SliceRef &out,
                                                const int *sel, int8_t (*tile)[32][36], int k0, int bz,
                                                const int *ecs = nullptr) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int j0 = blockIdx.x * 32;
  const int b = sel ? sel[bz] : bz;
  if constexpr (DB == 8 && W <= 2 && S <= 14) {
    // fixed-point path: each thread splits 4 consecutive k (rows 4 ty .. 4 ty + 3,
    // coalesced over the warp's 32 columns) of column j0 + tx and packs each
    // plane's 4 digits into one word (3 PRMT), staged as words in the tile
    // (one STS per plane instead of four byte stores)
    uint32_t(*tw)[32][9] = reinterpret_cast<uint32_t(*)[32][9]>(tile);
    const int j = j0 + tx, kb0 = k0 + 4 * ty;
    int ecol = 0;
    if (j < cols) ecol = ecs ? ecs[tx] : out.exps[(long long)b * out.rpad + out.row0 + j];
    double p1, p2;
    fixed_scale<S>(ecol, p1, p2);
    unsigned __int128 Y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = kb0 + q;
      double h = 0.0, l = 0.0;
      if (k < rows && j < cols) {
        const long long off = (long long)b * B.bstride + (long long)k * B.ld + j;
        if (fi == F32) {
          h = (double)((const float *)B.data)[off];
        } else {
          h = ((const double *)B.data)[off];
          if constexpr (W > 1) l = ((const double *)B.data)[off + B.plane];
        }
      }
      Y[q] = fixed_biased_fp<W, S>(h, l, p1, p2);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int kb = S - 1 - s, wj = kb >> 2, bsel = kb & 3;
      const uint32_t lo = __byte_perm(fixed_word(Y[0], wj), fixed_word(Y[1], wj), bsel | ((bsel + 4) << 4));
      const uint32_t hi = __byte_perm(fixed_word(Y[2], wj), fixed_word(Y[3], wj), bsel | ((bsel + 4) << 4));
      uint32_t wv = __byte_perm(lo, hi, 0x5410);
      if (s > 0) wv ^= 0x80808080u;
      tw[s][tx][ty] = wv;
    }
    __syncthreads();
    const long long plane = out.plane();
    const int jj = threadIdx.x >> 3, kq = threadIdx.x & 7;
    const int jo = j0 + jj;
    if (out.row0 + jo < out.rpad && jo < out.nrows && k0 + 4 * kq < out.kpad)
#pragma unroll
      for (int s = 0; s < S; ++s)
        *reinterpret_cast<uint32_t *>(out.digits + s * plane + ((long long)b * out.rpad + out.row0 + jo) * out.kpad +
                                      k0 + 4 * kq) = tw[s][jj][kq];
    return;
  }
  for (int kk = ty; kk < 32; kk += 8) {
    const int k = k0 + kk, j = j0 + tx;
    mp::qd v = mp::qd_make(0.0, 0.0, 0.0, 0.0);
    constexpr bool FIXED = DB == 8 && W <= 2 && S <= 14;
    int ecol = 0;
    if (k < rows && j < cols) {
      const long long off = (long long)b * B.bstride + (long long)k * B.ld + j;
      v = fi == F32 ? mp::qd_from_d((double)((const float *)B.data)[off]) : load_w<W>(B, off);
      ecol = ecs ? ecs[tx] : out.exps[(long long)b * out.rpad + out.row0 + j];
      if constexpr (!FIXED) v = scale_words<W>(v, -ecol);
    }
    const mp::qd vraw = v;
    int8_t dg[S];
    if constexpr (FIXED) {
      // fixed-point path on the unscaled words (the column exponent enters
      // the shift)
      double p1, p2;
      fixed_scale<S>(ecol, p1, p2);
      const unsigned __int128 Y = fixed_biased_fp<W, S>(vraw.x[0], W > 1 ? vraw.x[1] : 0.0, p1, p2);
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) {
        const int kb = S - 1 - s2;
        const int byte = (int)((Y >> (8 * kb)) & 0xff);
        dg[s2] = (int8_t)(s2 > 0 ? (byte ^ 0x80) : byte);
      }
    } else {
      split_digits_w<W, S, DB>(v, dg);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) tile[s][tx][kk] = dg[s];
  }
  __syncthreads();
  const long long plane = out.plane();
  // each thread writes 4 consecutive k of one column j as a 32-bit word
  const int jj = threadIdx.x >> 3, kq = (threadIdx.x & 7) * 4;
  const int j = j0 + jj;
  if (out.row0 + j < out.rpad && j < out.nrows && k0 + kq < out.kpad)
#pragma unroll
    for (int s = 0; s < S; ++s)
      *reinterpret_cast<uint32_t *>(out.digits + s * plane + ((long long)b * out.rpad + out.row0 + j) * out.kpad +
                                    k0 + kq) = *reinterpret_cast<const uint32_t *>(&tile[s][jj][kq]);
}

// Fixed-point column split (8-bit digits, <= 14 planes), 32 columns x 64 k per
// CTA: each thread splits 2 x 4 consecutive k of its column (8 loads in
// flight), packs plane words and stages them in a [S][32 j][16 k-words] tile
// for coalesced 32-byte row segments.  Column exponents from col_exps_kernel.
template <int W, int S>
__global__ void __launch_bounds__(256) slice_cols_fixed_kernel(MatRef B, int rows, int cols, int fi, SliceRef out,
                                                               const int *sel) {
  MPPS_PDL_ENTER();
  static_assert(W <= 2 && S <= 14, "fixed-point column split");
  __shared__ __align__(16) uint32_t tw[S][32][17];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j0 = blockIdx.x * 32, j = j0 + tx;
  const int k0 = blockIdx.y * 64;
  const int b = sel ? sel[blockIdx.z] : (int)blockIdx.z;
  int ecol = 0;
  if (j < cols) ecol = out.exps[(long long)b * out.rpad + out.row0 + j];
  double h[2][4], l[2][4];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = k0 + 32 * hf + 4 * ty + q;
      h[hf][q] = 0.0;
      l[hf][q] = 0.0;
      if (k < rows && j < cols) {
        const long long off = (long long)b * B.bstride + (long long)k * B.ld + j;
        if (fi == F32) {
          h[hf][q] = (double)((const float *)B.data)[off];
        } else {
          h[hf][q] = ((const double *)B.data)[off];
          if constexpr (W > 1) l[hf][q] = ((const double *)B.data)[off + B.plane];
        }
      }
    }
  double p1, p2;
  fixed_scale<S>(ecol, p1, p2);
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    unsigned __int128 Y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) Y[q] = fixed_biased_fp<W, S>(h[hf][q], l[hf][q], p1, p2);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int kb = S - 1 - s, wj = kb >> 2, bsel = kb & 3;
      const uint32_t lo = __byte_perm(fixed_word(Y[0], wj), fixed_word(Y[1], wj), bsel | ((bsel + 4) << 4));
      const uint32_t hi = __byte_perm(fixed_word(Y[2], wj), fixed_word(Y[3], wj), bsel | ((bsel + 4) << 4));
      uint32_t wv = __byte_perm(lo, hi, 0x5410);
      if (s > 0) wv ^= 0x80808080u;
      tw[s][tx][8 * hf + ty] = wv;
    }
  }
  __syncthreads();
  const long long plane = out.plane();
  // 16 words (64 k) per column: thread -> (column jj, word kq), two passes of 16 columns
#pragma unroll
  for (int ps = 0; ps < 2; ++ps) {
    const int jj = 16 * ps + (threadIdx.x >> 4), kq = threadIdx.x & 15;
    const int jo = j0 + jj;
    if (out.row0 + jo < out.rpad && jo < out.nrows && k0 + 4 * kq < out.kpad)
#pragma unroll
      for (int s = 0; s < S; ++s)
        *reinterpret_cast<uint32_t *>(out.digits + s * plane + ((long long)b * out.rpad + out.row0 + jo) * out.kpad +
                                      k0 + 4 * kq) = tw[s][jj][kq];
  }
}

template <int W, int S>
__global__ void slice_cols_kernel(MatRef B, int rows, int cols, int fi, SliceRef out, const int *sel) {
  MPPS_PDL_ENTER();
  __shared__ __align__(16) int8_t tile[S][32][36];
  if (oz_db_of<S>(out.db) == 8) {
    if constexpr (S != 16 && S != 31)
      slice_cols_body<W, S, 8>(B, rows, cols, fi, out, sel, tile, blockIdx.y * 32, blockIdx.z);
  } else {
    if constexpr (oz_has7<S>())
      slice_cols_body<W, S, 7>(B, rows, cols, fi, out, sel, tile, blockIdx.y * 32, blockIdx.z);
  }
}

// -------------------------------------------------------------- GEMM
struct OzArgs {
  SliceRef A, B;   // A: rows = M (row-scaled); B: rows = N (transposed B, col-scaled)
  int M, N, K;     // logical sizes
  int S;           // slices used (<= A.S, B.S)
  MatRef C;
  const int *sel;
  HornerEpi epi;
};

// Smem per stage: S slices of A (128 x 32 B) + S slices of B (NT x 32 B).
template <int S, int NT>
__host__ __device__ constexpr size_t oz_stage_bytes() { return (size_t)S * (kTileM + NT) * kKStep; }

// sum_d D_d 2^-(12+DB d) as a qd (dd-width sums for S <= 16)
template <int S, int DB>
__device__ __forceinline__ mp::qd combine_qd(const int32_t *D);
template <int S, int DB>
__device__ __forceinline__ mp::dd combine_dd(const int32_t *D);
template <int S, int DB = 7>
__device__ __forceinline__ mp::qd combine_diagonals(const int32_t *D) {
  if constexpr (S > 16) return combine_qd<S, DB>(D);
  else return mp::qd_from_dd(combine_dd<S, DB>(D));
}

// ------------------------------------------------------ shared epilogue
__host__ __device__ constexpr double pow2c(int e) {  // compile-time 2^e
  double r = 1.0;
  if (e >= 0) for (int i = 0; i < e; ++i) r *= 2.0;
  else for (int i = 0; i < -e; ++i) r *= 0.5;
  return r;
}

// m * 2^-q for an integer 0 <= m < 2^52, exactly: m dropped into the mantissa
// of 2^(52-q) (one logic op on the high word) minus that power of two (one
// DADD) -- no I2F.  `bias` is subtracted as well (signed values enter as
// m = v + 2^51 with bias 2^(51-q)).
template <int Q>
__device__ __forceinline__ double u52_scaled(unsigned long long m, double bias = 0.0) {
  constexpr unsigned long long EXPO = (unsigned long long)(1075 - Q) << 52;
  constexpr double BASE = pow2c(52 - Q);
  return __longlong_as_double((long long)(EXPO | m)) - (BASE + bias);
}

// sum_d D_d 2^-(12+DB d) for S <= 16 as a dd, through integer carries (the
// epilogue's FP64 work: ~10 DADD; a chain of dd additions of the exact
// three-digit groups cost ~40 DADD + 5 I2F.S64 per output).  The groups of three digits,
// weights 2^(3 DB) apart, are carry-normalised into base-2^(3 DB) digits
// (top signed, the rest in [0, 2^(3 DB))); pairs of digits are exact doubles
// P0 > P1 > ... that do not overlap, so FastTwoSum(P0, P1), one add of the
// tail and a final FastTwoSum give the normalised dd of the exact sum
// (one rounding of the low word, relative error <= 2^-105).
template <int S, int DB = 7>
__device__ __forceinline__ mp::dd combine_dd(const int32_t *D) {
  constexpr int NG = (S + 2) / 3;
  constexpr int WB = 3 * DB;
  long long G[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int d0 = 3 * g;
    G[g] = (long long)D[d0] << (2 * DB);
    if (d0 + 1 < S) G[g] += (long long)D[d0 + 1] << DB;
    if (d0 + 2 < S) G[g] += (long long)D[d0 + 2];
  }
  if constexpr (NG == 1) {
    return mp::dd_make((double)G[0] * pow2c(-(12 + DB * 2)), 0.0);
  } else {
    unsigned long long dig[NG];
    long long c = 0;
#pragma unroll
    for (int g = NG - 1; g >= 1; --g) {
      const long long t = G[g] + c;
      dig[g] = (unsigned long long)t & ((1ull << WB) - 1ull);
      c = t >> WB;
    }
    // |top| < 2^(31 + 2 DB + 1) <= 2^48
    const unsigned long long top = (unsigned long long)(G[0] + c + (1ll << 51));
    const double p0 = u52_scaled<12 + DB * 2>(top, pow2c(51 - (12 + DB * 2)));
    // pairs (1,2), (3,4), ...; a last single digit keeps its own weight
    constexpr int NP = (NG - 1 + 1) / 2;
    double p[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int a = 1 + 2 * k;
      if (a + 1 < NG) {
        const unsigned long long m = (dig[a] << WB) | dig[a + 1];
        p[k] = k == 0 ? u52_scaled<12 + DB * (3 * 2 + 2)>(m)
             : k == 1 ? u52_scaled<12 + DB * (3 * 4 + 2)>(m)
                      : u52_scaled<12 + DB * (3 * 6 + 2)>(m);
      } else {
        p[k] = k == 0 ? u52_scaled<12 + DB * (3 * 1 + 2)>(dig[a])
             : k == 1 ? u52_scaled<12 + DB * (3 * 3 + 2)>(dig[a])
                      : u52_scaled<12 + DB * (3 * 5 + 2)>(dig[a]);
      }
    }
    static_assert(NP <= 3, "combine_dd: S <= 16");
    const double s = p0 + p[0];
    double lo = p[0] - (s - p0);          // FastTwoSum: |p0| >= |p[0]| or p0 == 0
    if constexpr (NP == 2) lo += p[1];
    if constexpr (NP == 3) lo += p[1] + p[2];
    const double hi = s + lo;             // |s| >= |lo| or s == 0
    return mp::dd_make(hi, lo - (hi - s));
  }
}

// The same for qd outputs (S <= 31 planes: up to 11 groups).  The carry-
// normalised digits pair up into at most six exact, non-overlapping doubles
// P0 > P1 > ...; three VecSum sweeps (exact TwoSums; the first with
// FastTwoSum, its operands are ordered) leave the leading three qd words, the
// fourth takes the rounded rest (relative error <= 2^-205; zero words are
// moved behind the value).  ~75 DADD per output instead of ~950 for the chain
// of qd additions.
template <int S, int DB>
__device__ __forceinline__ mp::qd combine_qd(const int32_t *D) {
  constexpr int NG = (S + 2) / 3;
  constexpr int WB = 3 * DB;
  static_assert(NG >= 4 && NG <= 11, "combine_qd: 10..31 planes");
  long long G[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int d0 = 3 * g;
    G[g] = (long long)D[d0] << (2 * DB);
    if (d0 + 1 < S) G[g] += (long long)D[d0 + 1] << DB;
    if (d0 + 2 < S) G[g] += (long long)D[d0 + 2];
  }
  unsigned long long dig[NG];
  long long c = 0;
#pragma unroll
  for (int g = NG - 1; g >= 1; --g) {
    const long long t = G[g] + c;
    dig[g] = (unsigned long long)t & ((1ull << WB) - 1ull);
    c = t >> WB;
  }
  constexpr int NP = 1 + NG / 2;   // P0 and the pairs (1,2), (3,4), ... (a last single digit alone)
  double p[NP];
  p[0] = u52_scaled<12 + DB * 2>((unsigned long long)(G[0] + c + (1ll << 51)), pow2c(51 - (12 + DB * 2)));
#define MPPS_QD_TERM(K)                                                                             \
  if constexpr (K < NP) {                                                                           \
    constexpr int a = 2 * K - 1;                                                                    \
    if constexpr (a + 1 < NG) p[K] = u52_scaled<12 + DB * (3 * (a + 1) + 2)>((dig[a] << WB) | dig[a + 1]); \
    else p[K] = u52_scaled<12 + DB * (3 * a + 2)>(dig[a]);                                          \
  }
  MPPS_QD_TERM(1) MPPS_QD_TERM(2) MPPS_QD_TERM(3) MPPS_QD_TERM(4) MPPS_QD_TERM(5)
#undef MPPS_QD_TERM
  // sweep 1 (bottom-up): |p[i-1]| >= |sum below| or p[i-1] == 0, so FastTwoSum is exact
#pragma unroll
  for (int i = NP - 1; i >= 1; --i) {
    const double sum = p[i - 1] + p[i];
    p[i] = p[i] - (sum - p[i - 1]);
    p[i - 1] = sum;
  }
#pragma unroll
  for (int k = 1; k <= 2; ++k)   // two more whole sweeps, as mp::qd_renorm
#pragma unroll
    for (int i = NP - 1; i >= 1; --i) mp::two_sum(p[i - 1], p[i], p[i - 1], p[i]);
  double q[4] = {p[0], p[1], p[2], 0.0};
#pragma unroll
  for (int i = NP - 1; i >= 3; --i) q[3] += p[i];
  // heavy cancellation (the leading digits summing to almost nothing) leaves
  // zero words in front of the value: move them behind it, so that word 0 is
  // the leading word (the digit splits take row / column maxima from it)
#pragma unroll
  for (int pass = 0; pass < 3; ++pass)
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (q[i] == 0.0) { q[i] = q[i + 1]; q[i + 1] = 0.0; }
  return mp::qd_make(q[0], q[1], q[2], q[3]);
}

// fp64 value of the recombined diagonals (one rounding per group beyond the
// first; for fp32 / fp64 outputs)
template <int S, int DB>
__device__ __forceinline__ double combine_d(const int32_t *D) {
  double acc = 0.0;
#pragma unroll
  for (int g = 0; g < (S + 2) / 3; ++g) {
    const int d0 = 3 * g;
    long long G = (long long)D[d0] << (2 * DB);
    if (d0 + 1 < S) G += (long long)D[d0 + 1] << DB;
    if (d0 + 2 < S) G += (long long)D[d0 + 2];
    acc = fma((double)G, pow2c(-(12 + DB * (d0 + 2))), acc);
  }
  return acc;
}

// Column split of the epilogue: warps w and w+4 share TMEM lane quarter
// w % 4; the first takes columns [0, HALF), the second [HALF, NT).
template <int S, int NT>
struct EpiCols {
  static constexpr int CW = (S > 16) ? 4 : 8;                      // columns per TMEM load
  static constexpr int HALF = ((NT / 2 + CW - 1) / CW) * CW;
  static constexpr int MAXC = (NT - HALF > HALF) ? NT - HALF : HALF;
};

// Operands of the epilogue that do not depend on the MMAs (column
// exponents; for the fused Horner step the previous block B_prev), loaded
// by the epilogue warps while the mainloop runs instead of one dependent
// global load per column afterwards.
template <int S, int NT, int FO, int MODE>
struct EpiPre {
  static constexpr int MAXC = EpiCols<S, NT>::MAXC;
  static constexpr bool BP = (MODE == 1) && (S <= 16) && (FO != QD);  // dd-width B_prev
  int eb[MAXC];
  double bp[BP ? MAXC : 1][2];
};

template <int S, int NT, int FO, int MODE, typename Args>
__device__ __forceinline__ void oz_epi_prefetch(const Args &args, EpiPre<S, NT, FO, MODE> &pre, int quarter,
                                                int c_begin, int c_end, int b, int m0, int n0, int lane) {
  using P = EpiPre<S, NT, FO, MODE>;
  const int row = m0 + quarter * 32 + lane;
#pragma unroll
  for (int i = 0; i < P::MAXC; ++i) {
    const int col = n0 + c_begin + i;
    const bool ok = (c_begin + i < c_end) && col < args.N;
    pre.eb[i] = ok ? args.B.exps[(long long)b * args.B.rpad + col] : 0;
    if constexpr (P::BP) {
      pre.bp[i][0] = pre.bp[i][1] = 0.0;
      if (ok && row < args.M) {
        const MatRef &Bp = args.epi.Bprev;
        const double *bp = (const double *)Bp.data + (long long)b * Bp.bstride + (long long)row * Bp.ld + col;
        pre.bp[i][0] = bp[0];
        if (Bp.words > 1) pre.bp[i][1] = bp[Bp.plane];
      }
    }
  }
}

// Drain the S diagonal accumulators of this thread's TMEM lane for columns
// [c_begin, c_end) and run the store / fused Horner epilogue (DB: digit bits).
template <int S, int NT, int FO, int MODE, int DB, typename Args>
__device__ __forceinline__ void oz_epilogue(const Args &args, const EpiPre<S, NT, FO, MODE> &pre, uint32_t tmem,
                                            int quarter, int c_begin, int c_end, int b, int m0, int n0, int lane) {
  using P = EpiPre<S, NT, FO, MODE>;
  const int row = m0 + quarter * 32 + lane;
  const int ea = args.A.exps[(long long)b * args.A.rpad + row];
  const MatRef &C = args.C;
  int ey = 0, ei = 0, eo = 0;
  if constexpr (MODE == 1) {
    if (args.epi.exp_y) ey = args.epi.exp_y[b];
    if (args.epi.exp_in) ei = args.epi.exp_in[b];
    if (args.epi.exp_out) eo = args.epi.exp_out[b];
  }
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
  constexpr int CW = EpiCols<S, NT>::CW;
#pragma unroll
  for (int i0 = 0; i0 < P::MAXC; i0 += CW) {
    const int c0 = c_begin + i0;
    if (c0 >= c_end) break;
    int32_t D[S][CW];
#pragma unroll
    for (int d = 0; d < S; ++d) {
      if constexpr (CW == 8) tmem_ld8(lane_base + (uint32_t)(d * NT + c0), D[d]);
      else tmem_ld4(lane_base + (uint32_t)(d * NT + c0), D[d]);
    }
    tmem_ld_wait();
#pragma unroll
    for (int jj = 0; jj < CW; ++jj) {
      const int col = n0 + c0 + jj;
      if (row >= args.M || col >= args.N) continue;
      int32_t Dj[S];
#pragma unroll
      for (int d = 0; d < S; ++d) Dj[d] = D[d][jj];
      const int eb = pre.eb[i0 + jj];
      const long long off = (long long)b * C.bstride + (long long)row * C.ld + col;
      if constexpr (S <= 16 && FO != QD) {
        // dd-width epilogue (fp32 / fp64 / dd outputs)
        mp::dd v = combine_dd<S, DB>(Dj);
        const double sc = pow2i(ea + eb - (MODE == 1 ? (ey + ei) : 0));
        v = mp::dd_make(v.hi * sc, v.lo * sc);
        if constexpr (MODE == 1) v = mp::dd_add(mp::dd_make(pre.bp[i0 + jj][0], pre.bp[i0 + jj][1]), v);
        if constexpr (FO == DD) {
          if (eo) { const double so = pow2i(eo); v = mp::dd_make(v.hi * so, v.lo * so); }
          double *p = (double *)C.data + off;
          p[0] = v.hi;
          p[C.plane] = v.lo;
        } else if constexpr (FO == F64) {
          ((double *)C.data)[off] = eo ? v.hi * pow2i(eo) : v.hi;
        } else {
          if (eo) { const double so = pow2i(eo); v = mp::dd_make(v.hi * so, v.lo * so); }
          ((float *)C.data)[off] = mp::dd_to_float(v.hi, v.lo);
        }
      } else {
        mp::qd v = combine_diagonals<S, DB>(Dj);
        v = mp::qd_ldexp(v, ea + eb);
        // a non-finite operand row / column (row_exponent): ldexp leaves a zero sum zero
        if (ea + eb >= kExpNonFinite / 2) v = mp::qd_make(__longlong_as_double(0x7ff8000000000000ll), 0.0, 0.0, 0.0);
        if constexpr (MODE == 0) {
          store_fmt<FO>(C, off, v, 0);
        } else {
          const int sh = -(ey + ei);
          if (sh) v = mp::qd_ldexp(v, sh);
          mp::qd bv = load_qd(args.epi.Bprev, (long long)b * args.epi.Bprev.bstride + (long long)row * args.epi.Bprev.ld + col);
          store_fmt<FO>(C, off, horner_add<FO>(bv, v), eo);
        }
      }
    }
  }
}

template <int S, int NT, int FO, int MODE, typename Args>
__device__ __forceinline__ void oz_epilogue_db(const Args &args, const EpiPre<S, NT, FO, MODE> &pre, uint32_t tmem,
                                               int quarter, int c_begin, int c_end, int b, int m0, int n0, int lane) {
  if (oz_db_of<S>(args.A.db) == 8) {
    if constexpr (S != 16 && S != 31)
      oz_epilogue<S, NT, FO, MODE, 8>(args, pre, tmem, quarter, c_begin, c_end, b, m0, n0, lane);
  } else {
    if constexpr (oz_has7<S>())
      oz_epilogue<S, NT, FO, MODE, 7>(args, pre, tmem, quarter, c_begin, c_end, b, m0, n0, lane);
  }
}


// All MMAs of one K step, fully unrolled: A_s x [B_0 .. B_{S-1-s}] (the B
// planes are stacked along N) lands in diagonals s .. S-1 (TMEM column
// offset s*NT), split at the 256-column instruction limit.  Descriptors are
// compile-time offsets on two base descriptors (the 14-bit start-address
// field cannot carry: shared addresses < 228 KB), so the issuing thread
// spends a few instructions per MMA instead of ~150 cycles of descriptor
// and loop arithmetic (which left the tensor pipe idle between MMAs).
// acc0: accumulate flag of the K step's first write to every diagonal.
// More than 256 columns are issued as equal chunks (multiples of 16 columns)
// instead of 256 + remainder: a kind::i8 MMA costs ~0.55 clk per column down
// to N = 112 but never less than ~60 clk (tools/mma_probe_n.py), so 288
// columns cost 141 + 60 clk as 256 + 32 and 2 x 80 as 144 + 144 (dd, 14
// planes: 2011 -> 1938 clk of MMAs per K step).
__host__ __device__ constexpr int oz_chunk_w(int ncols) {
  const int nc = (ncols + 255) / 256;
  return ((ncols + nc - 1) / nc + 15) / 16 * 16;
}
template <int S, int NT, uint32_t A_SLICE, uint32_t B_SLICE>
__device__ __forceinline__ void oz_issue_kstep(uint32_t tmem, uint64_t ad0, uint64_t bd0, uint32_t acc0) {
  constexpr uint32_t B_ROW = B_SLICE / NT;   // bytes per B row
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int ncols = (S - s) * NT, cw = oz_chunk_w(ncols);
#pragma unroll
    for (int c0 = 0; c0 < ncols; c0 += cw) {
      const int nn = ncols - c0 > cw ? cw : ncols - c0;
      mma_i8(tmem + (uint32_t)(s * NT + c0), ad0 + (uint64_t)((s * A_SLICE) >> 4),
             bd0 + (uint64_t)((c0 * B_ROW) >> 4), idesc_i8(kTileM, nn), s > 0 ? 1u : acc0);
    }
  }
}

// ------------------------------------------------- TMA-fed pipeline
// Digit planes [S][batch][rpad][kpad] viewed by TMA as a 3-D tensor
// (k, row, slice); one box = 32 B of K x R rows x all S planes, written
// with the 32-byte swizzle that the UMMA SWIZZLE_32B K-major layout expects
// (8-row groups every 256 B; plane s of A at +s*R*32 B; the B planes are
// contiguous rows, so the concatenated-B MMAs see one N = (S-t0)*NT tile).
struct OzTmaArgs {
  CUtensorMap mapA;   // box {32, 128, S}
  CUtensorMap mapB;   // box {32, NT, S}
  SliceRef A, B;
  int M, N, K, S;
  MatRef C;
  const int *sel;
  HornerEpi epi;
  unsigned long long *trace;  // diagnostics (mpps_debug_oz_trace): per-CTA phase timestamps or null
  int dbg;                     // diagnostics: bit 0 skip MMAs (feed only), bit 1 skip TMA (MMA only)
  int mtiles, ntiles, group;   // tile raster: blockIdx.x walks `group` M tiles fastest, then N
  int nbatch;                  // persistent kernels: batch members (tiles = nbatch * mtiles * ntiles)
};

// Grouped raster: consecutive CTAs cover a group of up to `group` M tiles
// (fastest) times successive N tiles, so a wave shares both its A row
// panels and its B column panels in L2 (an N-fastest raster streams all of
// B from DRAM once per M-tile row: 34x the operand bytes at n = 8192).
__device__ __forceinline__ void oz_tile_at(const OzTmaArgs &a, int id, int nt, int &m0, int &n0) {
  const int per_group = a.group * a.ntiles;
  const int g = id / per_group;
  const int first_m = g * a.group;
  const int gm = min(a.group, a.mtiles - first_m);
  const int r = id - g * per_group;
  m0 = (first_m + r % gm) * kTileM;
  n0 = (r / gm) * nt;
}
__device__ __forceinline__ void oz_tile_of(const OzTmaArgs &a, int nt, int &m0, int &n0) {
  oz_tile_at(a, blockIdx.x, nt, m0, n0);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// Epilogue staging tile for the fused Horner step (dd-width outputs,
// NT = 32): 2 words x 128 rows x NT columns of fp64, swizzled so that both
// the per-row (thread = row) and the per-column (lane = column, coalesced
// global access) passes are conflict-free.  B_prev is copied into it with
// coalesced cp.async during the mainloop (a per-thread row-wise prefetch
// competes with the TMA feed and slows the mainloop ~2.5x).
template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr bool oz_staged() {
  return S <= 16 && FO != QD && (NT == 32 || (NT == 64 && S <= 8)) && MODE == 1;
}
// NT = 128 tiles for the few-plane Horner levels at large K (8-bit S <= 4:
// fp32 levels, S * 128 <= 512 TMEM columns): 4x fewer A-plane re-reads and
// N = 256 MMAs; the epilogue stages 32-column chunks of the tile in turn.
template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr bool oz_chunked() {
  return ((NT == 128 && S <= 4) || (NT == 64 && S <= 8)) && FO != QD && MODE == 1;
}
constexpr int kEpiChunk = 32;
template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr uint32_t oz_ebuf_bytes() {
  return oz_chunked<S, NT, FO, MODE>() ? 2u * kTileM * kEpiChunk * 8u
         : oz_staged<S, NT, FO, MODE>() ? 2u * kTileM * NT * 8u : 0u;
}
// Co-resident CTAs per SM: one CTA's epilogue overlaps the other's
// mainloop.  Needs <= 256 TMEM columns (S <= 8) and shared memory for two.
// NT = 64 (fp32 / fp64 Horner levels: half the A-plane re-reads) runs one
// CTA per SM: its 128 KB staging tile leaves no room for a second.
template <int S, int MODE, int NT = 32>
__host__ __device__ constexpr int oz_ctas_per_sm() { return NT == 32 && (MODE == 0 ? S <= 8 : S <= 4) ? 2 : 1; }
template <int S, int NT, int FO = DD, int MODE = 0>
__host__ __device__ constexpr int oz_tma_stages() {
  constexpr size_t cap = (oz_ctas_per_sm<S, MODE, NT>() == 2 ? (size_t)113 : (size_t)226) * 1024;
  constexpr size_t ring = cap - oz_ebuf_bytes<S, NT, FO, MODE>() - 2048;
  return (int)(ring / oz_stage_bytes<S, NT>()) >= 4 ? 4 : (int)(ring / oz_stage_bytes<S, NT>());
}
template <int S, int NT, int FO = DD, int MODE = 0>
__host__ __device__ constexpr size_t oz_tma_smem_bytes() {
  return oz_tma_stages<S, NT, FO, MODE>() * oz_stage_bytes<S, NT>() + oz_ebuf_bytes<S, NT, FO, MODE>() + 2048;
}
// The streamed-plane ring kernel also stages the plain dd GEMM's epilogue
// (coalesced stores instead of one 64-byte row segment per thread)
template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr bool oz_ring_staged() {
  return oz_staged<S, NT, FO, MODE>() || (MODE == 0 && FO == DD && NT == 32 && S >= 14 && S <= 16);
}
template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr uint32_t oz_ring_ebuf() {
  return oz_ring_staged<S, NT, FO, MODE>() ? 2u * kTileM * NT * 8u : 0u;
}
template <int NT = 32>
__device__ __forceinline__ int ebuf_idx(int w, int r, int c) { return (w * kTileM + r) * NT + (c ^ (r & 15)); }

// Staged epilogue, phase 1 (epilogue warps 2..7, during the mainloop):
// column exponents and, for the fused Horner step, the B_prev tile are
// copied into shared memory with coalesced cp.async (lane = column).
template <int S, int NT, int FO, int MODE, typename Args>
__device__ __forceinline__ void oz_stage_load(const Args &args, double *ebuf, int *ebs, int b, int m0, int n0,
                                              int wid, int nw, int lane) {
  if (wid == 0)
#pragma unroll
    for (int c = lane; c < NT; c += 32) ebs[c] = n0 + c < args.N ? args.B.exps[(long long)b * args.B.rpad + n0 + c] : 0;
  if constexpr (MODE == 1) {
    const MatRef &Bp = args.epi.Bprev;
    const bool two = Bp.words > 1;
    const double *base = (const double *)Bp.data + (long long)b * Bp.bstride;
#pragma unroll 4
    for (int r = wid; r < kTileM; r += nw) {
      const int row = m0 + r;
#pragma unroll
      for (int c = lane; c < NT; c += 32) {
        const int col = n0 + c;
        const bool ok = row < args.M && col < args.N;
        const double *src = ok ? base + (long long)row * Bp.ld + col : base;
        cp_async_zfill<8>(ebuf + ebuf_idx<NT>(0, r, c), src, ok);
        cp_async_zfill<8>(ebuf + ebuf_idx<NT>(1, r, c), ok && two ? src + Bp.plane : base, ok && two);
      }
    }
    cp_async_commit();
  }
}

// Phase 2 (all 8 warps, after the MMAs): thread = row; its columns are
// combined from TMEM, the B_prev words read from (and the dd-width result
// written back to) the staging tile.
template <int S, int NT, int FO, int MODE, int DB, int CW = 8, int TS = NT, typename Args>
__device__ __forceinline__ void oz_stage_compute(const Args &args, double *ebuf, const int *ebs, uint32_t tmem,
                                                 int quarter, int c_begin, int c_end, int b, int m0, int lane,
                                                 int toff = 0) {
  const int r = quarter * 32 + lane;
  const int row = m0 + r;
  const int ea = row < args.M ? args.A.exps[(long long)b * args.A.rpad + row] : 0;
  int ey = 0, ei = 0, eo = 0;
  if constexpr (MODE == 1) {
    if (args.epi.exp_y) ey = args.epi.exp_y[b];
    if (args.epi.exp_in) ei = args.epi.exp_in[b];
    if (args.epi.exp_out) eo = args.epi.exp_out[b];
  }
  const double so = pow2i(eo);
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
  for (int i0 = 0; i0 < NT / 2; i0 += CW) {
    const int c0 = c_begin + i0;
    if (c0 >= c_end) break;
    int32_t D[S][CW];
#pragma unroll
    for (int d = 0; d < S; ++d) {
      if constexpr (CW == 8) tmem_ld8(lane_base + (uint32_t)(d * TS + toff + c0), D[d]);
      else tmem_ld4(lane_base + (uint32_t)(d * TS + toff + c0), D[d]);
    }
    tmem_ld_wait();
#pragma unroll
    for (int jj = 0; jj < CW; ++jj) {
      const int c = c0 + jj;
      int32_t Dj[S];
#pragma unroll
      for (int d = 0; d < S; ++d) Dj[d] = D[d][jj];
      const double sc = pow2i(ea + ebs[c] - (MODE == 1 ? (ey + ei) : 0));
      const int i0w = ebuf_idx<NT>(0, r, c), i1w = ebuf_idx<NT>(1, r, c);
      if constexpr (FO != DD && S <= 8) {
        // fp32 / fp64 outputs: the sum in fp64 (relative error ~2^-52
        // before the final rounding to the output format) instead of dd
        double v = combine_d<S, DB>(Dj) * sc;
        if constexpr (MODE == 1) v = (ebuf[i0w] + v) + ebuf[i1w];
        if (eo) v *= so;
        ebuf[i0w] = FO == F64 ? v : (double)__double2float_rn(v);
        continue;
      }
      mp::dd v = combine_dd<S, DB>(Dj);
      v = mp::dd_make(v.hi * sc, v.lo * sc);
      if constexpr (MODE == 1) v = mp::dd_add(mp::dd_make(ebuf[i0w], ebuf[i1w]), v);
      if (eo) v = mp::dd_make(v.hi * so, v.lo * so);
      if constexpr (FO == DD) {
        ebuf[i0w] = v.hi;
        ebuf[i1w] = v.lo;
      } else if constexpr (FO == F64) {
        ebuf[i0w] = v.hi;
      } else {
        ebuf[i0w] = (double)mp::dd_to_float(v.hi, v.lo);
      }
    }
  }
}

// Phase 3 (all 8 warps): coalesced stores of the tile, lane = column.
template <int FO, int NT = 32, int EW = 8>
__device__ __forceinline__ void oz_stage_store(const MatRef &C, const double *ebuf, int M, int N, int b, int m0,
                                               int n0, int warp, int lane) {
#pragma unroll
  for (int c = lane; c < NT; c += 32) {
    const int col = n0 + c;
    if (col >= N) return;
#pragma unroll 4
    for (int r = warp; r < kTileM; r += EW) {
      const int row = m0 + r;
      if (row >= M) break;
      const long long off = (long long)b * C.bstride + (long long)row * C.ld + col;
      const double w0 = ebuf[ebuf_idx<NT>(0, r, c)];
      if constexpr (FO == DD) {
        double *p = (double *)C.data + off;
        p[0] = w0;
        p[C.plane] = ebuf[ebuf_idx<NT>(1, r, c)];
      } else if constexpr (FO == F64) {
        ((double *)C.data)[off] = w0;
      } else {
        ((float *)C.data)[off] = (float)w0;  // exact: w0 holds an fp32 value
      }
    }
  }
}


// Epilogue of the TMA / ring kernels (all 8 warps): operands that do not
// depend on the MMAs are loaded while the mainloop runs (staged B_prev via
// coalesced cp.async, or per-thread register prefetch), then the TMEM
// diagonals are combined and stored.  Ends with every thread past its
// TMEM reads (the caller deallocates).
template <int S, int NT, int FO, int MODE, bool STAGED, int EW = 8>
__device__ __forceinline__ void oz_kernel_epilogue(const OzTmaArgs &args, double *ebuf, int *ebs, uint32_t tmem,
                                                   uint64_t *done, int warp, int lane, int b, int m0, int n0,
                                                   unsigned long long *tr) {
  // warps w, w+4, ... share TMEM lane quarter w % 4 and split the columns
  // (EW = 16, staged only: four column parts of NT/4, 4-column TMEM loads)
  static_assert(EW == 8 || (EW == 16 && STAGED), "16 epilogue warps need the staged epilogue");
  const int quarter = warp & 3, half = warp >> 2;
  const int cb = EW == 16 ? half * (NT / 4) : (half ? EpiCols<S, NT>::HALF : 0);
  const int ce = EW == 16 ? cb + NT / 4 : (half ? NT : EpiCols<S, NT>::HALF);
  if constexpr (STAGED) {
    if (warp >= 2) {
      oz_stage_load<S, NT, FO, MODE>(args, ebuf, ebs, b, m0, n0, warp - 2, EW - 2, lane);
      if constexpr (MODE == 1) cp_async_wait<0>();
    }
    __syncwarp();
    mbar_wait(smem_u32(done), 0);
    fence_after();
    if (tr) tr[2] = globaltimer();
    __syncthreads();  // staged B_prev / exponents visible to every warp
    fence_after();
    constexpr int SCW = EW == 16 ? 4 : 8;
    if (oz_db_of<S>(args.A.db) == 8) {
      if constexpr (S != 16 && S != 31)
        oz_stage_compute<S, NT, FO, MODE, 8, SCW>(args, ebuf, ebs, tmem, quarter, cb, ce, b, m0, lane);
    } else {
      if constexpr (oz_has7<S>())
        oz_stage_compute<S, NT, FO, MODE, 7, SCW>(args, ebuf, ebs, tmem, quarter, cb, ce, b, m0, lane);
    }
    if (tr) tr[5] = globaltimer();
    __syncthreads();
    if (tr) tr[6] = globaltimer();
    oz_stage_store<FO, NT, EW>(args.C, ebuf, args.M, args.N, b, m0, n0, warp, lane);
    if (tr) tr[7] = globaltimer();
  } else {
    EpiPre<S, NT, FO, MODE> pre;
    oz_epi_prefetch<S, NT, FO, MODE>(args, pre, quarter, cb, ce, b, m0, n0, lane);
    __syncwarp();
    mbar_wait(smem_u32(done), 0);
    fence_after();
    if (tr) tr[2] = globaltimer();
    oz_epilogue_db<S, NT, FO, MODE>(args, pre, tmem, quarter, cb, ce, b, m0, n0, lane);
  }
  fence_before();
  __syncthreads();
  if (tr) tr[3] = globaltimer();
}

// Epilogue of the NT = 128 few-plane Horner tiles: the tile's columns are
// staged, combined and stored in 32-column chunks through one 64 KB staging
// tile (B_prev of chunk 0 is copied during the mainloop, the later chunks'
// after it); TMEM diagonal d of column c sits at d * NT + c.
template <int S, int NT, int FO, int MODE, int EW = 8>
__device__ __forceinline__ void oz_kernel_epilogue_chunked(const OzTmaArgs &args, double *ebuf, int *ebs,
                                                           uint32_t tmem, uint64_t *done, int warp, int lane, int b,
                                                           int m0, int n0, unsigned long long *tr) {
  static_assert(EW == 8, "chunked epilogue: 8 warps");
  constexpr int C = kEpiChunk;
  const int quarter = warp & 3, half = warp >> 2;
  const int cb = half ? EpiCols<S, C>::HALF : 0, ce = half ? C : EpiCols<S, C>::HALF;
  if (warp >= 2) oz_stage_load<S, C, FO, MODE>(args, ebuf, ebs, b, m0, n0, warp - 2, EW - 2, lane);
  __syncwarp();
  mbar_wait(smem_u32(done), 0);
  fence_after();
  if (tr) tr[2] = globaltimer();
#pragma unroll 1
  for (int q = 0; q < NT / C; ++q) {
    const int nq = n0 + q * C;
    if (q > 0) {
      if (nq >= args.N) break;
      oz_stage_load<S, C, FO, MODE>(args, ebuf, ebs, b, m0, nq, warp, EW, lane);
    }
    cp_async_wait<0>();
    __syncthreads();  // staged B_prev / exponents visible to every warp
    fence_after();
    if (oz_db_of<S>(args.A.db) == 8) {
      if constexpr (S != 16 && S != 31)
        oz_stage_compute<S, C, FO, MODE, 8, 8, NT>(args, ebuf, ebs, tmem, quarter, cb, ce, b, m0, lane, q * C);
    } else {
      if constexpr (oz_has7<S>())
        oz_stage_compute<S, C, FO, MODE, 7, 8, NT>(args, ebuf, ebs, tmem, quarter, cb, ce, b, m0, lane, q * C);
    }
    __syncthreads();
    oz_stage_store<FO, C, EW>(args.C, ebuf, args.M, args.N, b, m0, nq, warp, lane);
    __syncthreads();  // the staging tile is refilled by the next chunk
  }
  fence_before();
  __syncthreads();
  if (tr) tr[3] = globaltimer();
}

__device__ __forceinline__ unsigned long long *oz_trace_begin(const OzTmaArgs &args) {
  if (!args.trace || threadIdx.x != 64) return nullptr;
  unsigned long long *tr =
      args.trace + 8ull * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
  tr[0] = globaltimer();
  tr[4] = smid();
  return tr;
}

template <int S, int NT, int FO, int MODE, int EW = 8>
__global__ void __launch_bounds__(32 * EW, EW == 8 ? oz_ctas_per_sm<S, MODE, NT>() : 1) oz_gemm_tma_kernel(const __grid_constant__ OzTmaArgs args) {
  MPPS_PDL_ENTER();
  constexpr int STAGES = oz_tma_stages<S, NT, FO, MODE>();
  static_assert(STAGES >= 1, "stage ring does not fit");
  constexpr uint32_t STAGE = (uint32_t)oz_stage_bytes<S, NT>();
  constexpr uint32_t A_SLICE = kTileM * kKStep;   // 4 KB
  constexpr uint32_t B_SLICE = NT * kKStep;
  constexpr int TCOLS = tmem_cols_for(S * NT);

  constexpr bool STAGED = oz_staged<S, NT, FO, MODE>();
  constexpr uint32_t EBUF = oz_ebuf_bytes<S, NT, FO, MODE>();

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB aligned stage ring (swizzle atoms must not straddle)
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  double *ebuf = reinterpret_cast<double *>(smem + STAGES * STAGE);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE + EBUF);
  uint64_t *empty = full + STAGES;
  uint64_t *done = empty + STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);
  int *ebs = reinterpret_cast<int *>(tmem_slot + 4);  // NT column exponents

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bz = blockIdx.z;
  const int b = args.sel ? args.sel[bz] : bz;
  int m0, n0;
  oz_tile_of(args, NT, m0, n0);
  const int ksteps = args.A.kpad / kKStep;
  unsigned long long *tr = oz_trace_begin(args);

  if (warp == 0) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  const int rowA = b * args.A.rpad + m0, rowB = b * args.B.rpad + n0;
  if (tr) tr[1] = globaltimer();

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    for (int kb = 0; kb < ksteps; ++kb) {
      const int st = kb % STAGES;
      if (kb >= STAGES) mbar_wait(smem_u32(&empty[st]), ((kb / STAGES) - 1) & 1);
      const uint32_t sa = sbase + st * STAGE;
      if (args.dbg & 2) {
        mbar_expect_tx(smem_u32(&full[st]), 0);
      } else {
        mbar_expect_tx(smem_u32(&full[st]), STAGE);
        tma_load_3d(sa, &args.mapA, kb * kKStep, rowA, 0, smem_u32(&full[st]));
        tma_load_3d(sa + S * A_SLICE, &args.mapB, kb * kKStep, rowB, 0, smem_u32(&full[st]));
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    for (int kb = 0; kb < ksteps; ++kb) {
      const int st = kb % STAGES;
      mbar_wait(smem_u32(&full[st]), (kb / STAGES) & 1);
      fence_after();
      const uint32_t sa = sbase + st * STAGE;
      const uint32_t sb = sa + S * A_SLICE;
      if (!(args.dbg & 1))
        oz_issue_kstep<S, NT, A_SLICE, B_SLICE>(tmem, umma_desc(sa, 16, 256, 6), umma_desc(sb, 16, 256, 6),
                                                kb > 0 ? 1u : 0u);
      mma_commit(smem_u32(&empty[st]));
    }
    mma_commit(smem_u32(done));
  }
  if constexpr (oz_chunked<S, NT, FO, MODE>())
    oz_kernel_epilogue_chunked<S, NT, FO, MODE, EW>(args, ebuf, ebs, tmem, done, warp, lane, b, m0, n0, tr);
  else
    oz_kernel_epilogue<S, NT, FO, MODE, STAGED, EW>(args, ebuf, ebs, tmem, done, warp, lane, b, m0, n0, tr);
  if (warp == 0) tmem_dealloc<TCOLS>(tmem);
}

// ----------------------------------------- TMA pipeline, streamed A planes
// B (all S planes of one 32-byte K step, 16 KB for dd) sits in a 2-deep
// ring; A planes stream through a deeper ring in groups of SG planes
// (16 KB), so many loads are in flight while the wide MMAs of earlier
// groups run.  Same MMA sequence and epilogue as oz_gemm_tma_kernel.

// The MMAs of planes s0 .. s0+SG-1 of one K step (A planes of a ring group
// at ad0 + (s - s0) * A_SLICE), fully unrolled like oz_issue_kstep.
template <int S, int NT, uint32_t A_SLICE, uint32_t B_SLICE, int S0, int SG>
__device__ __forceinline__ void oz_issue_planes(uint32_t tmem, uint64_t ad0, uint64_t bd0, uint32_t acc0) {
  constexpr uint32_t B_ROW = B_SLICE / NT;   // bytes per B row
#pragma unroll
  for (int s = S0; s < S0 + SG && s < S; ++s) {
    const int ncols = (S - s) * NT, cw = oz_chunk_w(ncols);
#pragma unroll
    for (int c0 = 0; c0 < ncols; c0 += cw) {
      const int nn = ncols - c0 > cw ? cw : ncols - c0;
      mma_i8(tmem + (uint32_t)(s * NT + c0), ad0 + (uint64_t)(((s - S0) * A_SLICE) >> 4),
             bd0 + (uint64_t)((c0 * B_ROW) >> 4), idesc_i8(kTileM, nn), s > 0 ? 1u : acc0);
    }
  }
}

template <int S, int NT, uint32_t A_SLICE, uint32_t B_SLICE, int SG, int G = 0>
__device__ __forceinline__ void oz_ring_groups(uint32_t tmem, uint64_t bd0, uint32_t acc0, int &ai, uint8_t *aring,
                                               uint64_t *a_full, uint64_t *a_empty, int nas, uint32_t a_bytes) {
  if constexpr (G * SG < S) {
    const int ast = ai % nas;
    mbar_wait(smem_u32(&a_full[ast]), (ai / nas) & 1);
    fence_after();
    oz_issue_planes<S, NT, A_SLICE, B_SLICE, G * SG, SG>(tmem, umma_desc(smem_u32(aring + ast * a_bytes), 16, 256, 6),
                                                         bd0, acc0);
    mma_commit(smem_u32(&a_empty[ast]));
    ++ai;
    oz_ring_groups<S, NT, A_SLICE, B_SLICE, SG, G + 1>(tmem, bd0, acc0, ai, aring, a_full, a_empty, nas, a_bytes);
  }
}

// Ring sizes (160 KB of stages next to the epilogue staging tile).  Larger
// rings (4 B steps, 9-12 A groups, 210 KB) measured no faster: the feed
// is not bound by the bytes in flight.
template <int S, int NT, uint32_t EBUF = 0>
struct OzRing {
  // planes per A stage: groups of 4 (16 KB); 14 planes (8-bit dd) in two
  // groups of 7 so that no stage carries out-of-range planes
  static constexpr int SG = S < 4 ? S : (S == 14 ? 7 : 4);
  static constexpr int NG = (S + SG - 1) / SG;                   // A stages per K step
  static constexpr uint32_t A_BYTES = SG * kTileM * kKStep;      // 16 KB
  static constexpr uint32_t B_BYTES = S * NT * kKStep;
  static constexpr int NBS = 2;
  static constexpr int NAS = (int)((160u * 1024u - NBS * ((B_BYTES + 1023) / 1024 * 1024)) / A_BYTES) > 8
                                 ? 8
                                 : (int)((160u * 1024u - NBS * ((B_BYTES + 1023) / 1024 * 1024)) / A_BYTES);
  static constexpr uint32_t B_STRIDE = (B_BYTES + 1023) / 1024 * 1024;
  static constexpr size_t SMEM = (size_t)NBS * B_STRIDE + (size_t)NAS * A_BYTES + 2048;
};
template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr size_t oz_ring_smem_bytes() {
  return OzRing<S, NT, oz_ring_ebuf<S, NT, FO, MODE>()>::SMEM + oz_ring_ebuf<S, NT, FO, MODE>();
}

template <int S, int NT, int FO, int MODE, int EW = 8>
__global__ void __launch_bounds__(32 * EW, 1) oz_gemm_ring_kernel(const __grid_constant__ OzTmaArgs args) {
  MPPS_PDL_ENTER();
  constexpr uint32_t EBUF = oz_ring_ebuf<S, NT, FO, MODE>();
  using R = OzRing<S, NT, EBUF>;
  constexpr uint32_t A_SLICE = kTileM * kKStep;
  constexpr uint32_t B_SLICE = NT * kKStep;
  constexpr int TCOLS = tmem_cols_for(S * NT);

  constexpr bool STAGED = oz_ring_staged<S, NT, FO, MODE>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *bring = smem;
  uint8_t *aring = smem + R::NBS * R::B_STRIDE;
  double *ebuf = reinterpret_cast<double *>(aring + R::NAS * R::A_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(aring + R::NAS * R::A_BYTES + EBUF);
  uint64_t *b_full = bar, *b_empty = bar + R::NBS;
  uint64_t *a_full = bar + 2 * R::NBS, *a_empty = a_full + R::NAS;
  uint64_t *done = a_empty + R::NAS;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);
  int *ebs = reinterpret_cast<int *>(tmem_slot + 4);  // NT column exponents

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bz = blockIdx.z;
  const int b = args.sel ? args.sel[bz] : bz;
  int m0, n0;
  oz_tile_of(args, NT, m0, n0);
  const int ksteps = args.A.kpad / kKStep;
  unsigned long long *tr = oz_trace_begin(args);

  if (warp == 0) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < R::NBS; ++i) { mbar_init(smem_u32(&b_full[i]), 1); mbar_init(smem_u32(&b_empty[i]), 1); }
    for (int i = 0; i < R::NAS; ++i) { mbar_init(smem_u32(&a_full[i]), 1); mbar_init(smem_u32(&a_empty[i]), 1); }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rowA = b * args.A.rpad + m0, rowB = b * args.B.rpad + n0;
  if (tr) tr[1] = globaltimer();

  if (warp == 0 && lane == 0) {
    // ---- TMA producer: B step, then the A plane groups of that step
    int ai = 0;
    for (int kb = 0; kb < ksteps; ++kb) {
      const int bst = kb % R::NBS;
      if (kb >= R::NBS) mbar_wait(smem_u32(&b_empty[bst]), ((kb / R::NBS) - 1) & 1);
      const bool feed = !(args.dbg & 2);   // diagnostics: MMA-only run (no loads)
      mbar_expect_tx(smem_u32(&b_full[bst]), feed ? R::B_BYTES : 0);
      if (feed)
        tma_load_3d(smem_u32(bring + bst * R::B_STRIDE), &args.mapB, kb * kKStep, rowB, 0, smem_u32(&b_full[bst]));
      for (int g = 0; g < R::NG; ++g, ++ai) {
        const int ast = ai % R::NAS;
        if (ai >= R::NAS) mbar_wait(smem_u32(&a_empty[ast]), ((ai / R::NAS) - 1) & 1);
        mbar_expect_tx(smem_u32(&a_full[ast]), feed ? R::A_BYTES : 0);
        if (feed)
          tma_load_3d(smem_u32(aring + ast * R::A_BYTES), &args.mapA, kb * kKStep, rowA, g * R::SG,
                      smem_u32(&a_full[ast]));
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    int ai = 0;
    for (int kb = 0; kb < ksteps; ++kb) {
      const int bst = kb % R::NBS;
      mbar_wait(smem_u32(&b_full[bst]), (kb / R::NBS) & 1);
      const uint32_t sb = smem_u32(bring + bst * R::B_STRIDE);
      if (args.dbg & 1) {                  // diagnostics: feed-only run (no MMAs)
        for (int g = 0; g < R::NG; ++g, ++ai) {
          mbar_wait(smem_u32(&a_full[ai % R::NAS]), (ai / R::NAS) & 1);
          mma_commit(smem_u32(&a_empty[ai % R::NAS]));
        }
      } else
      oz_ring_groups<S, NT, A_SLICE, B_SLICE, R::SG>(tmem, umma_desc(sb, 16, 256, 6), kb > 0 ? 1u : 0u, ai, aring,
                                                      a_full, a_empty, R::NAS, R::A_BYTES);
      mma_commit(smem_u32(&b_empty[bst]));
    }
    mma_commit(smem_u32(done));
  }
  oz_kernel_epilogue<S, NT, FO, MODE, STAGED, EW>(args, ebuf, ebs, tmem, done, warp, lane, b, m0, n0, tr);
  if (warp == 0) tmem_dealloc<TCOLS>(tmem);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                               uint32_t mbar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint32_t mbar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(mbar),
      "h"(mask)
      : "memory");
}

// ------------------------------------------- 128-byte K boxes (wide feed)
// The 32-byte K boxes of the kernels above move one 32-byte sector per
// tile row per TMA request, and the feed saturates at ~45-60 GB/s per SM
// (the kernels run as fast with the MMAs switched off).  Here every TMA
// box row is 128 bytes (4 MMA K steps; SWIZZLE_128B, the UMMA K-major
// 128-byte-swizzle layout: 8-row x 128-byte atoms, SBO = 1024 B, the k-th
// 32-byte K step selected by +32 B on the descriptor start address).
// B: all S planes of NT rows x 128 B per stage (2 stages); A: one plane of
// 128 rows x 128 B per ring slot, its 4 K steps of MMAs issued back to back.
// A ring slots hold SG = 2 planes for even S >= 14 (the pair (j, S-1-j) of
// the issue order below, two TMA loads on one barrier): half the barrier
// waits, fences and tcgen05.commit of the issuing thread, which costs ~70 clk
// per instruction.
#ifndef MPPS_OZ_SLOT_PLANES
#define MPPS_OZ_SLOT_PLANES 2
#endif
template <int S>
__host__ __device__ constexpr int oz_slot_planes() { return (MPPS_OZ_SLOT_PLANES == 2 && S % 2 == 0 && S >= 14) ? 2 : 1; }
template <int S, int NT, int SGP = oz_slot_planes<S>()>
struct OzWide {
  static constexpr int KB = 128;                                  // K bytes per stage
  static constexpr int SG = SGP;
  static constexpr int NSLOT = S / SG;                            // ring slots per stage
  static constexpr uint32_t A_PLANE = kTileM * KB;                // 16 KB: one plane
  static constexpr uint32_t A_BYTES = SG * A_PLANE;
  static constexpr uint32_t B_PLANE = NT * KB;                    // bytes per B plane
  static constexpr uint32_t B_BYTES = S * B_PLANE;
  static constexpr uint32_t B_STRIDE = (B_BYTES + 1023) / 1024 * 1024;
  static constexpr int NBS = 2;
  template <uint32_t EBUF>
  __host__ __device__ static constexpr int nas() {
    constexpr long long room = 225ll * 1024 - 2048 - (long long)EBUF - NBS * (long long)B_STRIDE;
    return room / A_BYTES > 8 / SG ? 8 / SG : (int)(room / A_BYTES);
  }
};

// MMAs of plane s for K step kk of a stage: A_s x [B_0 .. B_{S-1-s}]
template <int S, int NT, int s>
__device__ __forceinline__ void oz_wide_plane(uint32_t tmem, uint64_t ad, uint64_t bd0, uint32_t acc) {
  constexpr uint32_t B_ROW = OzWide<S, NT>::KB;   // bytes per B row (128-byte swizzle atoms of 8 rows)
  constexpr int ncols = (S - s) * NT, cw = oz_chunk_w(ncols);
#pragma unroll
  for (int c0 = 0; c0 < ncols; c0 += cw) {
    const int nn = ncols - c0 > cw ? cw : ncols - c0;
    mma_i8(tmem + (uint32_t)(s * NT + c0), ad, bd0 + (uint64_t)((c0 * B_ROW) >> 4), idesc_i8(kTileM, nn),
           s > 0 ? 1u : acc);
  }
}

// Order in which the A planes of a stage are loaded and issued: low and high
// planes alternate (0, S-1, 1, S-2, ...).  One thread issues every MMA and
// spends ~70 clk per tcgen05.mma / tcgen05.commit whatever the shape
// (tools/mma_probe_n.py: two issuing threads reach 42 clk at N = 32), so a
// run of narrow planes (s >= S-4: N <= 128 columns, 42-71 clk of tensor
// pipe each) leaves the pipe idle; next to a wide plane (N = 448: 247 clk)
// the issue time of the narrow one hides behind the queued wide MMAs.
// Plane 0 stays first (it initialises every accumulator of a tile).
#ifndef MPPS_OZ_INTERLEAVE
#define MPPS_OZ_INTERLEAVE 1
#endif
template <int S>
__host__ __device__ constexpr int oz_plane_at(int i) {
  return MPPS_OZ_INTERLEAVE ? ((i & 1) ? S - 1 - i / 2 : i / 2) : i;
}

template <int S, int NT, int CL = 1, int j = 0, int SGP = oz_slot_planes<S>()>
__device__ __forceinline__ void oz_wide_stage(uint32_t tmem, uint32_t sb, int nk, uint32_t acc0, int &ai,
                                              uint8_t *aring, uint64_t *a_full, uint64_t *a_empty, int nas) {
  using W = OzWide<S, NT, SGP>;
  if constexpr (j < W::NSLOT) {
    constexpr int s0 = oz_plane_at<S>(j * W::SG), s1 = oz_plane_at<S>(j * W::SG + W::SG - 1);
    const int ast = ai % nas;
    mbar_wait(smem_u32(&a_full[ast]), (ai / nas) & 1);
    fence_after();
    const uint32_t sa = smem_u32(aring + ast * W::A_BYTES);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      if (kk < nk) {
        oz_wide_plane<S, NT, s0>(tmem, umma_desc(sa + kk * 32, 16, 1024, 2), umma_desc(sb + kk * 32, 16, 1024, 2),
                                 kk > 0 ? 1u : acc0);
        if constexpr (W::SG == 2)
          oz_wide_plane<S, NT, s1>(tmem, umma_desc(sa + W::A_PLANE + kk * 32, 16, 1024, 2),
                                   umma_desc(sb + kk * 32, 16, 1024, 2), kk > 0 ? 1u : acc0);
      }
    // the slot is refilled by a multicast into every CTA of the pair: it is
    // free only when all of their MMAs have read it
    if constexpr (CL == 1) mma_commit(smem_u32(&a_empty[ast]));
    else mma_commit_mc(smem_u32(&a_empty[ast]), (uint16_t)((1u << CL) - 1u));
    ++ai;
    oz_wide_stage<S, NT, CL, j + 1, SGP>(tmem, sb, nk, acc0, ai, aring, a_full, a_empty, nas);
  }
}

template <int S, int NT, int FO, int MODE>
__host__ __device__ constexpr size_t oz_wide_smem_bytes() {
  using W = OzWide<S, NT>;
  constexpr uint32_t EBUF = oz_ebuf_bytes<S, NT, FO, MODE>();
  return (size_t)W::NBS * W::B_STRIDE + (size_t)W::template nas<EBUF>() * W::A_BYTES + EBUF + 2048;
}

// CL = 2: a 2-CTA cluster takes two adjacent N tiles of one M tile; both
// need the same A planes, so plane s is loaded by CTA s % 2 and multicast
// into both CTAs' rings (L2 -> SM traffic of A, ~80 % of the feed at
// NT = 32, halves); B stays per CTA.
template <int S, int NT, int FO, int MODE, int CL = 1>
__global__ void __launch_bounds__(kThreadsEpi, 1) oz_gemm_wide_kernel(const __grid_constant__ OzTmaArgs args) {
  using W = OzWide<S, NT>;
  constexpr int TCOLS = tmem_cols_for(S * NT);
  constexpr bool STAGED = oz_staged<S, NT, FO, MODE>();
  constexpr uint32_t EBUF = oz_ebuf_bytes<S, NT, FO, MODE>();
  constexpr int NAS = W::template nas<EBUF>();
  static_assert(NAS >= 2, "A ring does not fit");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *bring = smem;
  uint8_t *aring = smem + W::NBS * W::B_STRIDE;
  double *ebuf = reinterpret_cast<double *>(aring + NAS * W::A_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(aring + NAS * W::A_BYTES + EBUF);
  uint64_t *b_full = bar, *b_empty = bar + W::NBS;
  uint64_t *a_full = bar + 2 * W::NBS, *a_empty = a_full + NAS;
  uint64_t *done = a_empty + NAS;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);
  int *ebs = reinterpret_cast<int *>(tmem_slot + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bz = blockIdx.z;
  const int b = args.sel ? args.sel[bz] : bz;
  int m0, n0;
  const int rank = CL > 1 ? (int)cluster_rank() : 0;
  if constexpr (CL == 1) {
    oz_tile_of(args, NT, m0, n0);
  } else {
    OzTmaArgs g = args;
    g.ntiles = args.ntiles / CL;             // the launch guarantees ntiles % CL == 0
    oz_tile_at(g, blockIdx.x / CL, NT * CL, m0, n0);
    n0 += rank * NT;
  }
  const int kpad = args.A.kpad;
  const int kstages = (kpad + W::KB - 1) / W::KB;
  unsigned long long *tr = oz_trace_begin(args);

  if (warp == 0) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < W::NBS; ++i) { mbar_init(smem_u32(&b_full[i]), 1); mbar_init(smem_u32(&b_empty[i]), 1); }
    for (int i = 0; i < NAS; ++i) { mbar_init(smem_u32(&a_full[i]), 1); mbar_init(smem_u32(&a_empty[i]), CL); }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  if constexpr (CL > 1) cluster_sync();   // the peer's barriers exist before any multicast
  else __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rowA = b * args.A.rpad + m0, rowB = b * args.B.rpad + n0;
  if (tr) tr[1] = globaltimer();

  if (warp == 0 && lane == 0) {
    // ---- TMA producer: B stage (all planes), then the S A planes of that stage
    int ai = 0;
    for (int kb = 0; kb < kstages; ++kb) {
      const int bst = kb % W::NBS;
      if (kb >= W::NBS) mbar_wait(smem_u32(&b_empty[bst]), ((kb / W::NBS) - 1) & 1);
      mbar_expect_tx(smem_u32(&b_full[bst]), W::B_BYTES);
      tma_load_3d(smem_u32(bring + bst * W::B_STRIDE), &args.mapB, kb * W::KB, rowB, 0, smem_u32(&b_full[bst]));
      for (int j = 0; j < W::NSLOT; ++j, ++ai) {
        const int ast = ai % NAS;
        if (ai >= NAS) mbar_wait(smem_u32(&a_empty[ast]), ((ai / NAS) - 1) & 1);
        mbar_expect_tx(smem_u32(&a_full[ast]), W::A_BYTES);
#pragma unroll
        for (int q = 0; q < W::SG; ++q) {
          const int pl = oz_plane_at<S>(j * W::SG + q);
          const uint32_t dst = smem_u32(aring + ast * W::A_BYTES + q * W::A_PLANE);
          if constexpr (CL == 1)
            tma_load_3d(dst, &args.mapA, kb * W::KB, rowA, pl, smem_u32(&a_full[ast]));
          else if (j % CL == rank)
            tma_load_3d_mc(dst, &args.mapA, kb * W::KB, rowA, pl, smem_u32(&a_full[ast]), (uint16_t)((1u << CL) - 1u));
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    int ai = 0;
    for (int kb = 0; kb < kstages; ++kb) {
      const int bst = kb % W::NBS;
      mbar_wait(smem_u32(&b_full[bst]), (kb / W::NBS) & 1);
      fence_after();
      const int left = (kpad - kb * W::KB) / kKStep;
      const int nk = left < 4 ? left : 4;
      oz_wide_stage<S, NT, CL>(tmem, smem_u32(bring + bst * W::B_STRIDE), nk, kb > 0 ? 1u : 0u, ai, aring, a_full,
                               a_empty, NAS);
      mma_commit(smem_u32(&b_empty[bst]));
    }
    mma_commit(smem_u32(done));
  }
  if constexpr (oz_chunked<S, NT, FO, MODE>())
    oz_kernel_epilogue_chunked<S, NT, FO, MODE>(args, ebuf, ebs, tmem, done, warp, lane, b, m0, n0, tr);
  else
    oz_kernel_epilogue<S, NT, FO, MODE, STAGED>(args, ebuf, ebs, tmem, done, warp, lane, b, m0, n0, tr);
  if constexpr (CL > 1) {
    // no CTA leaves while its peer may still multicast into its ring or
    // arrive on its barriers
    fence_before();
    cluster_sync();
    fence_after();
  }
  if (warp == 0) tmem_dealloc<TCOLS>(tmem);
}

// ------------------------------------------------ persistent kernels
// tile t of a CL-CTA group: (batch member, M offset, N offset of this CTA)
template <int CL>
__device__ __forceinline__ void oz_pers_tile(const OzTmaArgs &a, int t, int nt, int rank, int &bz, int &m0, int &n0) {
  const int npairs = (a.ntiles + CL - 1) / CL;
  const int per = a.mtiles * npairs;
  bz = t / per;
  OzTmaArgs g = a;
  g.ntiles = npairs;
  oz_tile_at(g, t - bz * per, nt * CL, m0, n0);
  n0 += rank * nt;
}

// INT8 tensor-pipe peak probe: one CTA per SM issues back-to-back
// 128x256x32 kind::i8 MMAs (operands: 40 KB of zeroed shared memory) into a
// 256-column TMEM accumulator.  2*128*256*32 ops per MMA.
__global__ void __launch_bounds__(128, 1) i8_mma_probe_kernel(int iters, int *out, int n = 256, int nacc = 1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t *done = reinterpret_cast<uint64_t *>(smem + 40960);
  uint32_t *slot = reinterpret_cast<uint32_t *>(done + 1);
  // pseudo-random operand bytes (a zero operand draws little power, so a
  // sustained run with it would never meet the power cap real data meets)
  for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
    reinterpret_cast<uint32_t *>(smem)[i] = x;
  }
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(slot));
  // nacc < 0: -nacc issuing threads (lane 0 of warps 0..), one accumulator each
  const int nissue = nacc < 0 ? -nacc : 1;
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(done), nissue);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  if (nacc < 0) {
    if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < nissue) {
      const uint32_t sa = smem_u32(smem), sb = sa + 4096;
      const uint64_t ad = umma_desc(sa, 16, 256, 6), bd = umma_desc(sb, 16, 256, 6);
      const uint32_t idesc = idesc_i8(128, n);
      const uint32_t acc = tmem + (uint32_t)((threadIdx.x >> 5) * n);
      for (int i = 0; i < iters; ++i) mma_i8(acc, ad, bd, idesc, i > 0 ? 1u : 0u);
      mma_commit(smem_u32(done));
    }
  } else if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 4096;
    const uint64_t ad = umma_desc(sa, 16, 256, 6), bd = umma_desc(sb, 16, 256, 6);
    const uint32_t idesc = idesc_i8(128, n);
    // nacc > 1: consecutive MMAs rotate over nacc independent accumulators
    int a = 0;
    for (int i = 0; i < iters; ++i) {
      mma_i8(tmem + (uint32_t)(a * n), ad, bd, idesc, i >= nacc ? 1u : 0u);
      a = a + 1 == nacc ? 0 : a + 1;
    }
    mma_commit(smem_u32(done));
  }
  __syncwarp();
  mbar_wait(smem_u32(done), 0);
  fence_after();
  if (threadIdx.x == 0 && iters < 0) out[0] = 1;
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

// 256-bit global accesses (sm_100: LDG/STG.256): a row-per-thread epilogue
// touches one line per lane and instruction, so its cost is the number of
// instructions -- 4 doubles each instead of 2.
__device__ __forceinline__ void ldg256(const double *p, double &a, double &b, double &c, double &d) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void stg256(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void stg256f(float *p, const double *v) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"l"(p), "f"((float)v[0]), "f"((float)v[1]),
               "f"((float)v[2]), "f"((float)v[3]), "f"((float)v[4]), "f"((float)v[5]), "f"((float)v[6]), "f"((float)v[7])
               : "memory");
}

// ------------- persistent, 128-byte K boxes, one accumulator set, 16 epilogue warps
// The dd products of the power chain at small and medium K (cfg2: K = 256,
// cfg3: K = 1024).  Per 128 x 32 tile the 32-byte-box ring kernel spends
// 0.2 us of set-up, a mainloop bound by its feed (12.4 us at K = 256 where
// the MMAs alone take 9), 3.9 us of epilogue and 1.15 us until the SM's next
// CTA starts (tools/cta_timeline.py).  Here one CTA per SM walks the tiles:
// the producer streams the next tile's planes (128-byte boxes) while the
// epilogue drains the accumulators, so a tile's MMAs start on a full ring;
// the 14 x 32 accumulators fill TMEM, so the MMAs of tile i+1 wait for the
// epilogue's last TMEM load of tile i (signalled before its arithmetic and
// stores of the last columns).  Warp 0: TMA producer, warp 1: MMA issuer,
// warps 2..17: epilogue (TMEM lane quarter = warp % 4, 8 columns each).
constexpr int kThreadsPw16 = 576;

template <int S, int NT, int SGP>
struct OzPw16 {
  using W = OzWide<S, NT, SGP>;
  static constexpr int NBS = 2;
  static constexpr int NAS_FIT = (int)((226ll * 1024 - 2048 - NBS * (long long)W::B_STRIDE) / W::A_BYTES);
  static constexpr int NAS = NAS_FIT > 8 / W::SG ? 8 / W::SG : NAS_FIT;
  static constexpr int ACC = S * NT;
  static_assert(ACC <= 512 && NT == 32, "one accumulator set of S x 32 columns");
  static constexpr int NACC = (2 * ACC <= 512) ? 2 : 1;
  static constexpr size_t SMEM = (size_t)NBS * W::B_STRIDE + (size_t)NAS * W::A_BYTES + 2048;
};

// SGP: planes per A ring slot -- 2 halves the issuing thread's barrier work
// (16 x 1024^3: 1114 -> 1081 us) but at K = 256 a tile has only two stages
// and the coarser ring stalls the feed (64 x 256^3: 105 -> 118 us): 1 there.
// FO / MODE: MODE 1 is the fused Horner level C = RN_FO(A B 2^-(ey+ei) + B_prev)
// 2^eo for dd-width outputs (B_prev: 1 or 2 fp64 words, read straight into the
// registers of its row's thread before the accumulators are awaited).  Plane
// counts with 2 S NT <= 512 get two accumulator sets: the epilogue of tile i
// then runs under the MMAs of tile i+1 and is the critical path -- bound by
// the latency of its row-wise B_prev loads (64 KB in flight per SM; a variant
// staging B_prev and C through one or two shared-memory tiles with coalesced
// cp.async measured no faster: 80.6 vs 81.9 us at S = 5, slower at S = 2).
template <int S, int NT, int DB, int SGP, int FO = DD, int MODE = 0>
__global__ void __launch_bounds__(kThreadsPw16, 1) oz_gemm_pw16_kernel(const __grid_constant__ OzTmaArgs args) {
  MPPS_PDL_ENTER();
  using W = OzWide<S, NT, SGP>;
  using P = OzPw16<S, NT, SGP>;
  constexpr int NAS = P::NAS;
  constexpr int NACC = P::NACC;
  static_assert(NAS * W::SG >= 4, "A ring does not fit");
  static_assert(FO != QD, "dd-width outputs");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *bring = smem;
  uint8_t *aring = smem + P::NBS * W::B_STRIDE;
  uint64_t *bar = reinterpret_cast<uint64_t *>(aring + NAS * W::A_BYTES);
  uint64_t *b_full = bar, *b_empty = bar + P::NBS;
  uint64_t *a_full = bar + 2 * P::NBS, *a_empty = a_full + NAS;
  uint64_t *acc_full = a_empty + NAS, *acc_empty = acc_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kpad = args.A.kpad;
  const int kstages = (kpad + W::KB - 1) / W::KB;
  const int total = args.nbatch * args.mtiles * args.ntiles;

  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < P::NBS; ++i) { mbar_init(smem_u32(&b_full[i]), 1); mbar_init(smem_u32(&b_empty[i]), 1); }
    for (int i = 0; i < NAS; ++i) { mbar_init(smem_u32(&a_full[i]), 1); mbar_init(smem_u32(&a_empty[i]), 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(smem_u32(&acc_full[i]), 1); mbar_init(smem_u32(&acc_empty[i]), 16); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (ring positions continue across tiles)
      int kg = 0, ai = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int bz, m0, n0;
        oz_pers_tile<1>(args, t, NT, 0, bz, m0, n0);
        const int b = args.sel ? args.sel[bz] : bz;
        const int rowA = b * args.A.rpad + m0, rowB = b * args.B.rpad + n0;
        for (int kb = 0; kb < kstages; ++kb, ++kg) {
          const int bst = kg % P::NBS;
          if (kg >= P::NBS) mbar_wait(smem_u32(&b_empty[bst]), ((kg / P::NBS) - 1) & 1);
          mbar_expect_tx(smem_u32(&b_full[bst]), W::B_BYTES);
          tma_load_3d(smem_u32(bring + bst * W::B_STRIDE), &args.mapB, kb * W::KB, rowB, 0, smem_u32(&b_full[bst]));
          for (int j = 0; j < W::NSLOT; ++j, ++ai) {
            const int ast = ai % NAS;
            if (ai >= NAS) mbar_wait(smem_u32(&a_empty[ast]), ((ai / NAS) - 1) & 1);
            mbar_expect_tx(smem_u32(&a_full[ast]), W::A_BYTES);
#pragma unroll
            for (int q = 0; q < W::SG; ++q)
              tma_load_3d(smem_u32(aring + ast * W::A_BYTES + q * W::A_PLANE), &args.mapA, kb * W::KB, rowA,
                          oz_plane_at<S>(j * W::SG + q), smem_u32(&a_full[ast]));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: tile i accumulates into set i % NACC
      int kg = 0, ai = 0, i = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
        const int buf = i % NACC;
        // the epilogue has read tile i - NACC out of this accumulator set
        if (i >= NACC) mbar_wait(smem_u32(&acc_empty[buf]), ((i / NACC) - 1) & 1);
        fence_after();
        const uint32_t tacc = tmem + (uint32_t)(buf * P::ACC);
        if (args.trace) args.trace[8ull * t + 0] = globaltimer();
        for (int kb = 0; kb < kstages; ++kb, ++kg) {
          const int bst = kg % P::NBS;
          mbar_wait(smem_u32(&b_full[bst]), (kg / P::NBS) & 1);
          fence_after();
          const int left = (kpad - kb * W::KB) / kKStep;
          const int nk = left < 4 ? left : 4;
          oz_wide_stage<S, NT, 1, 0, SGP>(tacc, smem_u32(bring + bst * W::B_STRIDE), nk, kb > 0 ? 1u : 0u, ai, aring,
                                          a_full, a_empty, NAS);
          mma_commit(smem_u32(&b_empty[bst]));
        }
        mma_commit(smem_u32(&acc_full[buf]));
        if (args.trace) args.trace[8ull * t + 1] = globaltimer();
      }
    }
  } else {
    // ---- epilogue warps: thread = tile row, 8 columns in two loads of 4
    const int quarter = warp & 3, cb = ((warp - 2) >> 2) * 8;
    const MatRef &C = args.C;
    int i = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
      int bz, m0, n0;
      oz_pers_tile<1>(args, t, NT, 0, bz, m0, n0);
      const int b = args.sel ? args.sel[bz] : bz;
      const int buf = i % NACC;
      const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * P::ACC);
      const int row = m0 + quarter * 32 + lane;
      const int col0 = n0 + cb;
      const bool full = col0 + 8 <= args.N;
      const int ea = row < args.M ? args.A.exps[(long long)b * args.A.rpad + row] : 0;
      int eb[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) eb[j] = col0 + j < args.N ? args.B.exps[(long long)b * args.B.rpad + col0 + j] : 0;
      // outputs; for the Horner step they first hold B_prev
      double hi[8], lo[8];
      int esh = 0, eo = 0;
      if constexpr (MODE == 1) {
        if (args.epi.exp_y) esh += args.epi.exp_y[b];
        if (args.epi.exp_in) esh += args.epi.exp_in[b];
        if (args.epi.exp_out) eo = args.epi.exp_out[b];
        const MatRef &Bp = args.epi.Bprev;
        const double *bp = (const double *)Bp.data + (long long)b * Bp.bstride + (long long)row * Bp.ld + col0;
        const bool two = Bp.words > 1;
#pragma unroll
        for (int j = 0; j < 8; ++j) hi[j] = lo[j] = 0.0;
        if (row < args.M) {
          if (full && ((reinterpret_cast<uintptr_t>(bp) | reinterpret_cast<uintptr_t>(bp + Bp.plane)) & 31) == 0) {
#pragma unroll
            for (int j = 0; j < 8; j += 4) {
              ldg256(bp + j, hi[j], hi[j + 1], hi[j + 2], hi[j + 3]);
              if (two) ldg256(bp + Bp.plane + j, lo[j], lo[j + 1], lo[j + 2], lo[j + 3]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (col0 + j < args.N) { hi[j] = bp[j]; if (two) lo[j] = bp[Bp.plane + j]; }
          }
        }
      }
      mbar_wait(smem_u32(&acc_full[buf]), (i / NACC) & 1);
      fence_after();
      unsigned long long *tr = (args.trace && tid == 64) ? args.trace + 8ull * t : nullptr;
      if (tr) { tr[2] = globaltimer(); tr[5] = smid(); }
      const double so = pow2i(eo);
#pragma unroll
      for (int i0 = 0; i0 < 8; i0 += 4) {
        int32_t D[S][4];
#pragma unroll
        for (int d = 0; d < S; ++d) tmem_ld4(lane_base + (uint32_t)(d * NT + cb + i0), D[d]);
        tmem_ld_wait();
        if (i0 == 4) {
          // every accumulator of this warp's part is in registers: the MMAs
          // of tile i + NACC may overwrite them while the last columns are combined
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&acc_empty[buf]));
          if (tr) tr[3] = globaltimer();
        }
        if (args.dbg & 4) {    // diagnostics: no recombination
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) hi[i0 + jj] = lo[i0 + jj] = (double)D[0][jj];
          continue;
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          int32_t Dj[S];
#pragma unroll
          for (int d = 0; d < S; ++d) Dj[d] = D[d][jj];
          const double sc = pow2i(ea + eb[i0 + jj] - esh);
          if constexpr (FO != DD && S <= 8) {
            // fp32 / fp64 outputs of few planes: the sum in fp64 (as the
            // staged epilogue of the tile-per-CTA kernels)
            double v = combine_d<S, DB>(Dj) * sc;
            if constexpr (MODE == 1) v = (hi[i0 + jj] + v) + lo[i0 + jj];
            if (eo) v *= so;
            hi[i0 + jj] = FO == F64 ? v : (double)__double2float_rn(v);
          } else {
            mp::dd v = combine_dd<S, DB>(Dj);
            v = mp::dd_make(v.hi * sc, v.lo * sc);
            if constexpr (MODE == 1) {
              v = mp::dd_add(mp::dd_make(hi[i0 + jj], lo[i0 + jj]), v);
              if (eo) v = mp::dd_make(v.hi * so, v.lo * so);
            }
            if constexpr (FO == DD) { hi[i0 + jj] = v.hi; lo[i0 + jj] = v.lo; }
            else if constexpr (FO == F64) hi[i0 + jj] = v.hi;
            else hi[i0 + jj] = (double)mp::dd_to_float(v.hi, v.lo);
          }
        }
      }
      if (row < args.M && !(args.dbg & 8)) {
        const long long off = (long long)b * C.bstride + (long long)row * C.ld + col0;
        if constexpr (FO == F32) {
          float *p = (float *)C.data + off;
          if (full && (reinterpret_cast<uintptr_t>(p) & 31) == 0) {
            stg256f(p, hi);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (col0 + j < args.N) p[j] = (float)hi[j];
          }
        } else {
          double *p = (double *)C.data + off;
          double *q = p + C.plane;
          if (full && ((reinterpret_cast<uintptr_t>(p) | (FO == DD ? reinterpret_cast<uintptr_t>(q) : 0)) & 31) == 0) {
#pragma unroll
            for (int j = 0; j < 8; j += 4) {
              stg256(p + j, hi[j], hi[j + 1], hi[j + 2], hi[j + 3]);
              if constexpr (FO == DD) stg256(q + j, lo[j], lo[j + 1], lo[j + 2], lo[j + 3]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (col0 + j < args.N) {
                p[j] = hi[j];
                if constexpr (FO == DD) q[j] = lo[j];
              }
          }
        }
      }
      if (tr) tr[4] = globaltimer();
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// Global -> shared ingest probe: one CTA per SM streams 16 KB bulk copies
// (the TMA engine, 8 in flight) from an L2-resident buffer; the tensor-core
// GEMMs are bound by this per-SM fill rate (~25 B/clk with every SM
// loading), not by the MMAs (DESIGN 5.1).
__global__ void __launch_bounds__(32, 1) ingest_probe_kernel(const uint8_t *src, long long span, int iters) {
  constexpr int CH = 16384, NB = 8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NB * CH);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NB; ++i) mbar_init(smem_u32(&bar[i]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  const long long nchunks = span / CH;
  const long long base = ((long long)blockIdx.x * 7919) % nchunks;
  for (int it = 0; it < iters; ++it) {
    const int st = it % NB;
    if (it >= NB) mbar_wait(smem_u32(&bar[st]), ((it / NB) - 1) & 1);
    mbar_expect_tx(smem_u32(&bar[st]), CH);
    const uint8_t *g = src + ((base + it) % nchunks) * CH;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(sm + st * CH)),
                 "l"(g), "r"(CH), "r"(smem_u32(&bar[st]))
                 : "memory");
  }
  for (int it = iters > NB ? iters - NB : 0; it < iters; ++it) mbar_wait(smem_u32(&bar[it % NB]), (it / NB) & 1);
}

}  // namespace oz
}  // namespace mpps
