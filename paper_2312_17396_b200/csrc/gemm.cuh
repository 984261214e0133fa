// Tiled SIMT GEMM for the four lattice formats (fp32 FFMA, fp64 DFMA,
// double-double and quad-double DFMA error-free transforms) with the fused
// matrix-Horner epilogue of engine.py:249-251:
//
//     phi_{j-1} = RN_out( 2^e_out * ( B_{j-1} + 2^-(e_y+e_in) * (Y~ . phi~_j) ) )
//
// The GEMM runs in the level-j format (the operands Y~ and phi~_j are already
// stored in it); the epilogue widens the accumulator exactly, adds the
// working-precision block B_{j-1}, rounds once into the level-(j-1) format and
// applies the exact power-of-two scaling that keeps fp32 levels inside the
// fp32 exponent range (the reference's MPFR exponents are unbounded,
// SPEC.md:84).  No separate elementwise kernel runs for the Horner add.
//
// Layout: every operand is a batch of row-major matrices whose W words are
// stored as separate planes (SoA).  CTA tile BM x BN, K-tile BK, each thread
// owns a TM x TN register tile.  Tiles are staged global -> registers -> shared
// (k-major) with a two-slot ring so the next tile's loads overlap the current
// tile's FP64 work (one __syncthreads per K-tile).
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

struct GemmArgs {
  int M, N, K;
  MatRef A, B, C;
  const int *sel;      // batch indices (null -> blockIdx.z)
  HornerEpi epi;
};

template <int F> struct Tile;
//                                   BM   BN  BK TM TN
template <> struct Tile<F32> { enum { BM = 128, BN = 128, BK = 8,  TM = 8, TN = 8 }; };
template <> struct Tile<F64> { enum { BM = 64,  BN = 64,  BK = 16, TM = 4, TN = 4 }; };
template <> struct Tile<DD>  { enum { BM = 64,  BN = 64,  BK = 16, TM = 4, TN = 4 }; };
template <> struct Tile<QD>  { enum { BM = 32,  BN = 32,  BK = 8,  TM = 2, TN = 2 }; };

constexpr int kThreads = 256;

// Dynamic shared memory of gemm_kernel<F, ...>: two ring slots of the A and
// B tiles, all word planes.
constexpr int kStages = 3;

template <int F> struct SmemGeom {
  using T = typename FmtT<F>::word;
  static constexpr int W = FmtT<F>::W;
  static constexpr int APAD = 1;                          // odd A row stride: conflict-free column reads
  static constexpr int BPAD = (sizeof(T) == 8) ? 2 : 4;   // 16-byte aligned B rows (vector reads)
  static constexpr int AROW = Tile<F>::BK + APAD;
  static constexpr int BROW = Tile<F>::BN + BPAD;
  static constexpr size_t A_STAGE = (size_t)W * Tile<F>::BM * AROW;   // elements
  static constexpr size_t B_STAGE = (size_t)W * Tile<F>::BK * BROW;
};

template <int F>
constexpr size_t gemm_smem_bytes() {
  using G = SmemGeom<F>;
  return sizeof(typename G::T) * kStages * (G::A_STAGE + G::B_STAGE);
}

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

// ------------------------------------------------------------ accumulators
template <int F> struct Acc;
template <> struct Acc<F32> {
  float c;
  __device__ __forceinline__ void zero() { c = 0.f; }
  __device__ __forceinline__ void mac(const float *a, const float *b) { c = __fmaf_rn(a[0], b[0], c); }
  __device__ __forceinline__ void renorm() {}
  __device__ __forceinline__ mp::qd as_qd() const { return mp::qd_from_d((double)c); }
};
template <> struct Acc<F64> {
  double c;
  __device__ __forceinline__ void zero() { c = 0.0; }
  __device__ __forceinline__ void mac(const double *a, const double *b) { c = __fma_rn(a[0], b[0], c); }
  __device__ __forceinline__ void renorm() {}
  __device__ __forceinline__ mp::qd as_qd() const { return mp::qd_from_d(c); }
};
template <> struct Acc<DD> {
  double h, l;
  __device__ __forceinline__ void zero() { h = 0.0; l = 0.0; }
  // 12-instruction MAC (TwoSum).  The 9-instruction magnitude-select
  // FastTwoSum variant (mp::dd_mac9) measured 12-17 % slower on B200: its
  // integer compare/selects cost more issue slots than the 3 DADDs saved.
#ifdef MPPS_DD_MAC9
  __device__ __forceinline__ void mac(const double *a, const double *b) { mp::dd_mac9(a[0], a[1], b[0], b[1], h, l); }
#else
  __device__ __forceinline__ void mac(const double *a, const double *b) { mp::dd_mac(a[0], a[1], b[0], b[1], h, l); }
#endif
  __device__ __forceinline__ void renorm() { mp::dd_acc_renorm(h, l); }
  __device__ __forceinline__ mp::qd as_qd() const { return mp::qd_make(h, l, 0.0, 0.0); }
};
template <> struct Acc<QD> {
  double c[4];
  __device__ __forceinline__ void zero() { c[0] = c[1] = c[2] = c[3] = 0.0; }
  __device__ __forceinline__ void mac(const double *a, const double *b) { mp::qd_mac(a, b, c); }
  __device__ __forceinline__ void renorm() { mp::qd_acc_renorm(c); }
  __device__ __forceinline__ mp::qd as_qd() const { return mp::qd_make(c[0], c[1], c[2], c[3]); }
};

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

// ---------------------------------------------------------------- kernel
// MODE 0: C = A*B stored in format F.  MODE 1: fused Horner epilogue into FO.
template <int F> struct MinBlocks { enum { value = 2 }; };
template <> struct MinBlocks<F32> { enum { value = 1 }; };

template <int F, int FO, int MODE>
__global__ void __launch_bounds__(kThreads, MinBlocks<F>::value)
gemm_kernel(const GemmArgs args) {
  using G = SmemGeom<F>;
  using T = typename FmtT<F>::word;
  constexpr int W = FmtT<F>::W;
  constexpr int BM = Tile<F>::BM, BN = Tile<F>::BN, BK = Tile<F>::BK;
  constexpr int TM = Tile<F>::TM, TN = Tile<F>::TN;
  constexpr int A_PER = BM * BK / kThreads;  // A elements per thread per plane
  constexpr int B_PER = BK * BN / kThreads;
  constexpr int TX = BN / TN;                // threads along N
  static_assert((BM / TM) * (BN / TN) == kThreads, "thread tile mismatch");
  static_assert(A_PER >= 1 && B_PER >= 1, "tile too small");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *As = reinterpret_cast<T *>(smem_raw);                      // [stage][w][BM][AROW]
  T *Bs = As + kStages * G::A_STAGE;                            // [stage][w][BK][BROW]

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int bidx = args.sel ? args.sel[blockIdx.z] : (int)blockIdx.z;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = args.M, N = args.N, K = args.K;

  const T *Ag = (const T *)args.A.data + (long long)bidx * args.A.bstride;
  const T *Bg = (const T *)args.B.data + (long long)bidx * args.B.bstride;
  const long long ap = args.A.plane, bp = args.B.plane;
  const int lda = args.A.ld, ldb = args.B.ld;

  auto load_tile = [&](int stage, int k0) {
    T *as = As + stage * G::A_STAGE;
    T *bs = Bs + stage * G::B_STAGE;
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      const int e = tid + i * kThreads;
      const int row = e / BK, col = e % BK;
      const int gr = m0 + row, gc = k0 + col;
      const bool ok = gr < M && gc < K;
      const long long off = ok ? (long long)gr * lda + gc : 0;
#pragma unroll
      for (int w = 0; w < W; ++w)
        cp_async_zfill<sizeof(T)>(as + (w * BM + row) * G::AROW + col, Ag + off + w * ap, ok);
    }
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      const int e = tid + i * kThreads;
      const int row = e / BN, col = e % BN;
      const int gr = k0 + row, gc = n0 + col;
      const bool ok = gr < K && gc < N;
      const long long off = ok ? (long long)gr * ldb + gc : 0;
#pragma unroll
      for (int w = 0; w < W; ++w)
        cp_async_zfill<sizeof(T)>(bs + (w * BK + row) * G::BROW + col, Bg + off + w * bp, ok);
    }
  };

  Acc<F> acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j].zero();

  const int ktiles = (K + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < ktiles) load_tile(st, st * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nk = kt + kStages - 1;
      if (nk < ktiles) load_tile(nk % kStages, nk * BK);
      cp_async_commit();
    }
    const T *as = As + (kt % kStages) * G::A_STAGE;
    const T *bs = Bs + (kt % kStages) * G::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM][W], b[TN][W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i][w] = as[(w * BM + ty * TM + i) * G::AROW + kk];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j][w] = bs[(w * BK + kk) * G::BROW + tx * TN + j];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j].mac(a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j].renorm();
  }
  cp_async_wait<0>();

  // ---------------------------------------------------------- epilogue
  const MatRef &C = args.C;
  const long long cbase = (long long)bidx * C.bstride;
  int ey = 0, ei = 0, eo = 0;
  if constexpr (MODE == 1) {
    if (args.epi.exp_y) ey = args.epi.exp_y[bidx];
    if (args.epi.exp_in) ei = args.epi.exp_in[bidx];
    if (args.epi.exp_out) eo = args.epi.exp_out[bidx];
  }
  const long long bbase = (MODE == 1) ? (long long)bidx * args.epi.Bprev.bstride : 0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gr = m0 + ty * TM + i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gc = n0 + tx * TN + j;
      if (gc >= N) continue;
      const long long off = cbase + (long long)gr * C.ld + gc;
      if constexpr (MODE == 0) {
        T *Cg = (T *)C.data;
        if constexpr (F == F32) Cg[off] = acc[i][j].c;
        else if constexpr (F == F64) Cg[off] = acc[i][j].c;
        else if constexpr (F == DD) {
          double s, e;
          mp::quick_two_sum(acc[i][j].h, acc[i][j].l, s, e);
          Cg[off] = s; Cg[off + C.plane] = e;
        } else {
          Cg[off] = acc[i][j].c[0]; Cg[off + C.plane] = acc[i][j].c[1];
          Cg[off + 2 * C.plane] = acc[i][j].c[2]; Cg[off + 3 * C.plane] = acc[i][j].c[3];
        }
      } else {
        mp::qd t = acc[i][j].as_qd();
        const int sh = -(ey + ei);
        if (sh) t = mp::qd_ldexp(t, sh);
        mp::qd bv = load_qd(args.epi.Bprev, bbase + (long long)gr * args.epi.Bprev.ld + gc);
        store_fmt<FO>(C, off, horner_add<FO>(bv, t), eo);
      }
    }
  }
}

}  // namespace mpps
