// K5: the whole mixed-precision Paterson-Stockmeyer evaluation
// of small matrices (n <= 32, fp64 working format -- config 1), one CTA per
// matrix with every operand resident in shared memory.  The evaluation is
// latency bound at this size (a 32^3 product is 32K FMAs), so the ~40
// launches of the general pipeline (splits, tensor-core GEMMs, assembly,
// norms, Horner levels) become ONE (small_fused_kernel, below: prepare, the
// digit rule on the device, Horner; the host reads norms and plan from pinned
// memory while the Horner chains still run) -- or the two kernels it is made
// of around the exact host planner when the certified rule declines:
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

// powers, blocks and norms of matrix b in shared memory (P: s matrices X^1 .. X^s, Bk: r + 1
// blocks) and in global memory (a.blocks, a.Y, a.norms); nrm (shared, r + 2 doubles) when given
__device__ __forceinline__ void small_prepare_body(const PrepArgs &a, double *P, double *Bk, double *nrm) {
  const int n = a.n, nn = n * n, s = a.s, r = a.r, b = blockIdx.x;
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
    if (lane == 0) {
      a.norms[(long long)b * (r + 2) + k] = v;
      if (nrm) nrm[k] = v;
    }
  }
}

__global__ void __launch_bounds__(kThreads) small_prepare_kernel(const PrepArgs a) {
  MPPS_PDL_ENTER();
  extern __shared__ __align__(16) double sm[];
  small_prepare_body(a, sm, sm + a.s * a.n * a.n, nullptr);
}

// the mixed Horner chain of matrix b: Ys = Y in shared memory, blk(i) = block i (shared or
// global), fm = its level formats, phi / nxt = two n x n shared buffers; result to og
template <typename Blk, typename Fmt>
__device__ __forceinline__ void small_horner_body(int n, int r, int top_scalar, double bm, const double *Ys, Blk blk,
                                                  Fmt fm, double *phi, double *nxt, double *og) {
  const int nn = n * n;
  int j0;
  if (top_scalar) {
    // level r: B_r = b_m I, so Y phi_r = b_m Y (K3, no product)
    const double *bp = blk(r - 1);
    for (int e = threadIdx.x; e < nn; e += blockDim.x)
      phi[e] = rn_level(bp[e] + rn_level(bm * Ys[e], fm[r]), fm[r - 1]);
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
  for (int e = threadIdx.x; e < nn; e += blockDim.x) og[e] = phi[e];
}

__global__ void __launch_bounds__(kThreads) small_horner_kernel(const __grid_constant__ HornerArgs a) {
  MPPS_PDL_ENTER();
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, nn = n * n, r = a.r, b = blockIdx.x;
  double *Ys = sm, *phi = sm + nn, *nxt = sm + 2 * nn;
  const signed char *fm = (a.fmt ? a.fmt : a.fmt_inline) + (long long)b * (r + 1);
  const double *yg = a.Y + (long long)b * nn;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) Ys[e] = yg[e];
  small_horner_body(n, r, a.top_scalar, a.bm, Ys,
                    [&](int i) { return a.blocks + ((long long)i * a.batch + b) * nn; }, fm, phi, nxt,
                    a.out + (long long)b * nn);
}

// ------------------------------------------------ one launch per evaluation
// The planner's digit rule (engine.py:184-215) in certified float64, as
// small_plan_row on the host (mpps_capi.cu): exact digits unless some e_i
// lies within 1e-8 of an integer or of the delta threshold (the float64
// evaluation is within ~1e-11 of the exact value whichever libm computes
// log10) -- then 1, and the host plans exactly.
__device__ __forceinline__ int small_plan_dev(const double *nb, double y, int r, int d, double delta, int apply_switch,
                                              int *digits, int *nu_out) {
  const double M = 1e-8, lim = d - log10(delta);
  if (y == 0.0) {
    for (int i = 0; i < r; ++i) digits[i] = 1;
    *nu_out = 1;
    return 0;
  }
  if (!isfinite(y)) return 1;
  for (int i = 0; i <= r; ++i)
    if (!isfinite(nb[i])) return 1;
  const double lb0 = nb[0] > 0 ? log10(nb[0]) : 0.0, ly = log10(y);
  unsigned qual = 0;
  for (int i = 1; i <= r; ++i) {
    if (nb[i] == 0.0 || nb[0] == 0.0) {
      digits[i - 1] = 1;
      qual |= 1u << (i - 1);
      continue;
    }
    const double e = (d - lb0) + (log10(nb[i]) + i * ly) + 1e-9;
    if (fabs(e - nearbyint(e)) < M || fabs(e - lim) < M) return 1;
    const int di = (int)floor(e);
    digits[i - 1] = di < 1 ? 1 : (di > d ? d : di);
    if (e <= lim) qual |= 1u << (i - 1);
  }
  int nu = r + 1;
  for (int i = 1; i <= r; ++i)
    if (qual >> (i - 1) & 1u) { nu = i; break; }
  if (apply_switch)
    for (int i = 1; i < nu; ++i) digits[i - 1] = d;
  for (int i = r - 2; i >= 0; --i)
    if (digits[i + 1] > digits[i]) digits[i] = digits[i + 1];
  *nu_out = nu;
  return 0;
}

struct FusedArgs {
  PrepArgs p;
  double *out;          // (B, n, n) fp64
  double *host;         // pinned, device-mapped: per matrix (r + 2) norms, r digits, nu, 1 when the rule declined
  unsigned *arrived;    // pinned: matrices whose norms and plan are in `host`
  double delta;
  int d, apply_switch, fixed;
};

// prepare -> plan -> Horner for one matrix per CTA without leaving the SM:
// the blocks and Y stay in shared memory (they also go to global memory for
// the host-planned fallback), thread 0 plans.  Same operations in the same
// order as the two kernels above, hence the same bits.
__global__ void __launch_bounds__(kThreads) small_fused_kernel(const __grid_constant__ FusedArgs a) {
  MPPS_PDL_ENTER();
  extern __shared__ __align__(16) double sm[];
  const int n = a.p.n, nn = n * n, s = a.p.s, r = a.p.r, b = blockIdx.x;
  double *P = sm, *Bk = sm + s * nn, *phi = Bk + (r + 1) * nn, *nxt = phi + nn, *nrm = nxt + nn;
  signed char *fm = reinterpret_cast<signed char *>(nrm + r + 2);
  __shared__ int declined;
  small_prepare_body(a.p, P, Bk, nrm);
  __syncthreads();
  if (threadIdx.x == 0) {
    int dg[kMaxBlocks], nu = r + 1, un = 0;
    if (a.fixed) {
      for (int i = 0; i < r; ++i) dg[i] = a.d;
    } else {
      un = small_plan_dev(nrm, nrm[r + 1], r, a.d, a.delta, a.apply_switch, dg, &nu);
    }
    double *pl = a.host + (long long)b * (2 * (r + 2));
    for (int k = 0; k < r + 2; ++k) pl[k] = nrm[k];
    for (int i = 0; i < r; ++i) pl[r + 2 + i] = un ? 0.0 : (double)dg[i];
    pl[2 * r + 2] = (double)nu;
    pl[2 * r + 3] = (double)un;
    __threadfence_system();
    atomicAdd_system(a.arrived, 1u);
    fm[0] = 1;                                   // level 0: the fp64 working format
    for (int i = 0; i < r; ++i) fm[1 + i] = dg[i] <= 7 ? 0 : 1;
    declined = un;
  }
  __syncthreads();
  if (declined) return;
  small_horner_body(n, r, a.p.top_scalar, a.p.coef[a.p.m], P + (s - 1) * nn, [&](int i) { return Bk + i * nn; }, fm, phi,
                    nxt, a.out + (long long)b * nn);
}

}  // namespace small
}  // namespace mpps
