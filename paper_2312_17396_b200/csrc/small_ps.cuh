// K5: the whole mixed-precision Paterson-Stockmeyer evaluation
// of small matrices (n <= 32, fp64 working format -- config 1) in two
// kernels around the host planner, one CTA per matrix with every operand
// resident in shared memory.  The evaluation is latency bound at this size
// (a 32^3 product is 32K FMAs), so the ~40 launches of the general pipeline
// (splits, tensor-core GEMMs, assembly, norms, Horner levels) become two.
//
//   small_prepare_kernel  X, X^2 .. X^s   (engine.py:141-154, X^{k+1} = X^k X)
//                         B_0 .. B_r      (engine.py:127-138: acc = b_{si} I,
//                                          acc = RN(RN(b_{si+j} X^j) + acc))
//                         ||B_i||, ||Y||  (precision.py:235-249: column
//                                          abs-sums in row order, max)
//   (host)                planner on the norms (engine.py:157-215)
//   small_horner_kernel   phi = B_r (or RN_top(b_m Y) + B_{r-1} when B_r =
//                         b_m I, engine.py:132); phi_{j-1} = RN_{j-1}(B_{j-1}
//                         + Y phi_j), j = r..1 (engine.py:243-252), the
//                         level formats per matrix (fp32 levels: 24-bit
//                         roundings with an unbounded exponent, as the
//                         tensor-core path stores them)
//
// Products are fp64 FMA chains (one rounding per step instead of the
// reference's two; within the c n u tolerance, like every GPU product).
#pragma once
#include "formats.cuh"

namespace mpps {
namespace small {

constexpr int kMaxN = 32;
constexpr int kMaxS = 8;
constexpr int kMaxBlocks = 9;      // r + 1 with m <= 64 (s = ceil(sqrt m) <= 8)
constexpr int kMaxCoef = 65;
constexpr int kThreads = 256;

struct PrepArgs {
  const double *X;      // (B, n, n) fp64, row stride ldx, batch stride xbs
  long long xbs;
  int ldx;
  int n, m, s, r, top_scalar;
  double coef[kMaxCoef];  // RN_p(b_k) (fp64 working: one word each)
  double *blocks;       // (r+1, B, n, n); block r is not stored when top_scalar
  double *Y;            // (B, n, n)
  double *norms;        // (B, r+2): ||B_0..B_r||, ||Y||
  int batch;
};

constexpr int kInlineFmt = 4096;   // level formats carried in the kernel parameters

struct HornerArgs {
  const double *Y, *blocks;
  const signed char *fmt;   // (B, r+1) device copy when they do not fit inline
  double *out;              // (B, n, n) fp64
  double bm;                // b_m (top_scalar)
  int n, r, top_scalar, batch;
  signed char fmt_inline[kInlineFmt];   // (B, r+1): 0 fp32, 1 fp64 per level (level 0 = working fp64)
};

// RN to 24 significant bits with an unbounded exponent (Veltkamp split)
__device__ __forceinline__ double rn24(double v) {
  const double c = v * 536870913.0;  // 2^29 + 1
  return c - (c - v);
}
__device__ __forceinline__ double rn_level(double v, int f) { return f == 0 ? rn24(v) : v; }

// C = A B for n x n row-major tiles in shared memory (fp64 FMA chains)
__device__ __forceinline__ void mat_mul_smem(const double *A, const double *B, double *C, int n) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double acc = A[i * n] * B[j];
    for (int t = 1; t < n; ++t) acc = fma(A[i * n + t], B[t * n + j], acc);
    C[e] = acc;
  }
}

// one warp per matrix: lane = column (n <= 32), rows summed in order, then
// the max over columns
__device__ __forceinline__ double one_norm_warp(const double *M, int n, int lane) {
  double s = 0.0;
  if (lane < n)
    for (int i = 0; i < n; ++i) s += fabs(M[i * n + lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {   // a NaN column sum stays (fmax would drop it)
    const double t = __shfl_xor_sync(0xffffffffu, s, o);
    s = (t > s || t != t) ? t : s;
  }
  return s;
}

__global__ void __launch_bounds__(kThreads) small_prepare_kernel(const PrepArgs a) {
  MPPS_PDL_ENTER();
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, nn = n * n, s = a.s, r = a.r, b = blockIdx.x;
  double *P = sm;                  // s matrices: X^1 .. X^s
  double *Bk = sm + s * nn;        // r + 1 blocks
  const double *xg = a.X + (long long)b * a.xbs;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    P[e] = xg[(long long)i * a.ldx + j];
  }
  __syncthreads();
  for (int k = 1; k < s; ++k) {
    mat_mul_smem(P + (k - 1) * nn, P, P + k * nn, n);
    __syncthreads();
  }
  const int full = a.m / s;
  for (int i = 0; i <= r; ++i) {
    if (i == r && a.top_scalar) break;
    const int hi = (i < full) ? s - 1 : a.m - s * full;
    double *Bi = Bk + i * nn;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int row = e / n, col = e - row * n;
      double acc = row == col ? a.coef[s * i] : 0.0;
      for (int j = 1; j <= hi; ++j) acc = __dadd_rn(__dmul_rn(a.coef[s * i + j], P[(j - 1) * nn + e]), acc);
      Bi[e] = acc;
      a.blocks[((long long)i * a.batch + b) * nn + e] = acc;
    }
  }
  for (int e = threadIdx.x; e < nn; e += blockDim.x) a.Y[(long long)b * nn + e] = P[(s - 1) * nn + e];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k <= r + 1; k += blockDim.x >> 5) {
    double v;
    if (k == r + 1) v = one_norm_warp(P + (s - 1) * nn, n, lane);
    else if (k == r && a.top_scalar) v = fabs(a.coef[a.m]);        // ||b_m I||
    else v = one_norm_warp(Bk + k * nn, n, lane);
    if (lane == 0) a.norms[(long long)b * (r + 2) + k] = v;
  }
}

__global__ void __launch_bounds__(kThreads) small_horner_kernel(const __grid_constant__ HornerArgs a) {
  MPPS_PDL_ENTER();
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, nn = n * n, r = a.r, b = blockIdx.x;
  double *Ys = sm, *phi = sm + nn, *nxt = sm + 2 * nn;
  const signed char *fm = (a.fmt ? a.fmt : a.fmt_inline) + (long long)b * (r + 1);
  const double *yg = a.Y + (long long)b * nn;
  auto blk = [&](int i) { return a.blocks + ((long long)i * a.batch + b) * nn; };
  for (int e = threadIdx.x; e < nn; e += blockDim.x) Ys[e] = yg[e];
  int j0;
  if (a.top_scalar) {
    // level r: B_r = b_m I, so Y phi_r = b_m Y (K3, no product)
    const double *bp = blk(r - 1);
    for (int e = threadIdx.x; e < nn; e += blockDim.x)
      phi[e] = rn_level(bp[e] + rn_level(a.bm * Ys[e], fm[r]), fm[r - 1]);
    j0 = r - 1;
  } else {
    const double *br = blk(r);
    for (int e = threadIdx.x; e < nn; e += blockDim.x) phi[e] = rn_level(br[e], fm[r]);
    j0 = r;
  }
  __syncthreads();
  for (int j = j0; j >= 1; --j) {
    const double *bp = blk(j - 1);
    const int fo = fm[j - 1];
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int i = e / n, c = e - i * n;
      double acc = Ys[i * n] * phi[c];
      for (int t = 1; t < n; ++t) acc = fma(Ys[i * n + t], phi[t * n + c], acc);
      nxt[e] = rn_level(bp[e] + acc, fo);
    }
    __syncthreads();
    double *t = phi; phi = nxt; nxt = t;
  }
  double *og = a.out + (long long)b * nn;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) og[e] = phi[e];
}

}  // namespace small
}  // namespace mpps
