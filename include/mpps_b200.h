/*
 * mpps_b200.h -- C-ABI of the B200-native mixed-precision Paterson-Stockmeyer
 * hot path (arXiv 2312.17396).  Plain pointers and sizes only; no torch types.
 *
 * The reference (pkg/src/mpps, pure Python over gmpy2) has no FFI of its own:
 * its operator seam is the per-op precision-context layer of precision.py
 * (round_to / mat_mul / mat_axpy / mat_add / one_norm) driven by engine.py.
 * Each entry point below replaces one reference operator or one fused group
 * of them; the reference interface it replaces is cited beside it.  The
 * Python mirror of the reference API (paper_2312_17396_b200/engine.py) is the
 * only in-tree caller; INTEGRATION.md shows the ctypes stub a maintainer of
 * the reference would add.
 *
 * Conventions
 *  - Matrices are batches of row-major real matrices; multiword formats are
 *    stored as separate word planes (SoA): word w of matrix b, entry (i,j) is
 *    ((T*)data)[w*plane_stride + b*batch_stride + i*ld + j].  fp32 uses float
 *    words, every other format double words.
 *  - A format is named by its lattice digits: 7 = fp32, 15 = fp64, 31 = dd
 *    (double-double), 63 = qd (quad-double) (engine.py:218-240).
 *  - Every call is asynchronous and stream-ordered on the handle's stream;
 *    buffers are caller-owned device memory.  A handle is not thread-safe;
 *    use one handle per host thread.  There is no hidden global state.
 *  - "sel" arrays (device int32, length nsel) select which batch members a
 *    call processes (grouped launches for heterogeneous plans); pass NULL to
 *    process the whole batch.  "exp" arrays (device int32, indexed by batch
 *    member) give exact power-of-two scalings 2^exp (NULL = 0).
 *  - Return codes: MPPS_OK; MPPS_EINVAL mirrors the reference's
 *    DimensionError / ValueError (precision.py:25-26, engine.py:55-63);
 *    MPPS_EFMT an unsupported format; MPPS_ECUDA a CUDA launch error.  The
 *    message is available from mpps_last_error().
 */
#ifndef MPPS_B200_H
#define MPPS_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define MPPS_OK 0
#define MPPS_EINVAL 1
#define MPPS_EFMT 2
#define MPPS_ECUDA 3

#define MPPS_FP32 7
#define MPPS_FP64 15
#define MPPS_DD 31
#define MPPS_QD 63

/* Maximum PS blocks per evaluation supported by the fused assembly kernel
 * (r + 1 <= MPPS_MAX_BLOCKS; covers Table 1's m = 182, s = 14, r = 13). */
#define MPPS_MAX_BLOCKS 16

typedef struct mpps_handle mpps_handle;

typedef struct {
  void *data;              /* device pointer: word 0 of matrix 0           */
  long long plane_stride;  /* elements between word planes                  */
  long long batch_stride;  /* elements between matrices of the batch        */
  int rows, cols, ld;      /* row-major, ld >= cols                         */
  int batch;               /* number of matrices                            */
  int fmt;                 /* MPPS_FP32 / MPPS_FP64 / MPPS_DD / MPPS_QD     */
} mpps_mat;

/* ABI version (major*100 + minor). */
int mpps_version(void);

/* Handle lifecycle.  stream is a cudaStream_t (NULL = legacy default). */
int mpps_create(int device, void *stream, mpps_handle **out);
int mpps_destroy(mpps_handle *h);
int mpps_set_stream(mpps_handle *h, void *stream);
const char *mpps_last_error(const mpps_handle *h);
/* Number of kernels this handle has launched (evidence counter). */
long long mpps_launch_count(const mpps_handle *h);

/* round_to (precision.py:153-157) and format conversion:
 * dst = RN_dst(2^exp[b] * src).  Widening is exact. */
int mpps_convert(mpps_handle *h, const mpps_mat *src, mpps_mat *dst,
                 const int *sel, int nsel, const int *exp);

/* mat_mul (precision.py:160-184): C = RN_fmt(A * B), A, B, C in one format;
 * A is rows x k, B is k x cols, C is rows x cols (SUMMA blocks may be
 * rectangular). */
int mpps_gemm(mpps_handle *h, const mpps_mat *A, const mpps_mat *B,
              mpps_mat *C, const int *sel, int nsel);

/* mat_axpy (precision.py:187-197): C = RN(RN(alpha*A) + B) at C's format;
 * alpha is given as 4 host doubles whose exact sum is the coefficient. */
int mpps_axpy(mpps_handle *h, const double *alpha_words, const mpps_mat *A,
              const mpps_mat *B, mpps_mat *C);

/* form_powers / eval_b0_and_power power chain (engine.py:118-124, 141-154):
 * powers[0] must already hold X at the working format; fills powers[1..s-1]
 * with X^2..X^s, powers[k] = RN(powers[k-1] * X). */
int mpps_powers(mpps_handle *h, mpps_mat *powers, int s);

/* The same with the coefficient words on the HOST ((m+1) x 4 doubles),
 * passed in the kernel's parameter space (compile-time coefficient
 * offsets, no shared-memory coefficient traffic).  flags bit 0: when
 * m mod s == 0, B_r = b_m I is not stored (blocks[r] may be unallocated;
 * the K3 Horner step mpps_horner_scalar_top uses b_m directly) -- its norm
 * is still written.  Supported shapes: mpps_assemble_hc_supported(fmt, s, m)
 * (others: MPPS_EFMT, use mpps_assemble_blocks). */
int mpps_assemble_blocks_hc(mpps_handle *h, const mpps_mat *powers, int s, int m,
                            const double *coeff_host, mpps_mat *blocks, double *norms, int flags);
int mpps_assemble_hc_supported(int fmt, int s, int m);
/* Two-pass block assembly (B200 extension of the same reference operators,
 * engine.py:127-138 + precision.py:235-249): blocks[0..nblocks-1] only, at
 * the blocks' formats: a prefix of dd blocks (full dd accumulation, the
 * levels the plan keeps at dd), then fp64 blocks made from the high words
 * of the dd powers (the planner's norms and the blocks of fp32/fp64 Horner
 * levels).  Compiled mixes: all dd (nblocks <= 4), all fp64, or B_0, B_1 dd
 * + fp64 (mpps_assemble_hc_n_supported, block_fmt -1).
 * norms ([batch][nblocks+1], the last one ||Y||) may be NULL.  nblocks = r+1
 * with m mod s = 0 is refused (B_r = b_m I). */
int mpps_assemble_blocks_hc_n(mpps_handle *h, const mpps_mat *powers, int s, int m, const double *coeff_host,
                              mpps_mat *blocks, int nblocks, double *norms);
int mpps_assemble_hc_n_supported(int block_fmt, int s, int m, int nblocks);

/* assemble_block for i = 0..r plus one_norm of every block and of Y
 * (engine.py:127-138, 141-154; precision.py:235-249), fused into one pass
 * over the powers:  B_i = b_{si} I + sum_{j=1..hi_i} b_{si+j} X^j,
 * accumulated in index order at the working format.  powers holds X^1..X^s
 * (s entries, powers[s-1] = Y).  coeff_words: device, (m+1) x 4 doubles, the
 * coefficients already rounded at the working precision.  norms: device,
 * batch x (r+2) doubles, [b][i] = ||B_i||_1 (i <= r), [b][r+1] = ||Y||_1
 * (deterministic column-sum order). */
int mpps_assemble_blocks(mpps_handle *h, const mpps_mat *powers, int s, int m,
                         const double *coeff_words, mpps_mat *blocks,
                         double *norms);

/* Distributed variant for a local block (rows x cols) of 2-D block-distributed
 * matrices (SUMMA, cfg5): the identity of b_{si} I is placed where
 * row0 + i == col0 + j (global indices), and instead of norms the kernel
 * writes the local column abs-sums colsums[b][i][j] (i = 0..r blocks, r+1 =
 * Y), summed over the local rows in a fixed order; the caller all-reduces
 * them along the process column and applies mpps_colmax. */
int mpps_assemble_blocks_dist(mpps_handle *h, const mpps_mat *powers, int s,
                              int m, const double *coeff_words,
                              mpps_mat *blocks, double *colsums, int row0,
                              int col0);

/* out[b][i] = max_j colsums[b][i][j] (the column max of one_norm). */
int mpps_colmax(mpps_handle *h, const double *colsums, int nvec, int cols,
                int batch, double *out);

/* one_norm (precision.py:235-249) of every batch member: norms[b]. */
int mpps_one_norm(mpps_handle *h, const mpps_mat *A, double *norms);

/* Exact power-of-two scalings of fp32 Horner levels from the planner norms
 * (device, no host round trip): norms is [batch][r+2]
 * (||B_0..B_r||, ||Y||); e = -rint(log2 norm) (0 for zero / non-finite);
 * exps[j][b] = e for the levels j whose bit is set in fp32_mask, else 0;
 * exp_y[b] = e of ||Y||.  r + 2 <= 64. */
int mpps_level_exps(mpps_handle *h, const double *norms, int batch, int r, unsigned long long fp32_mask,
                    int *exps, int *exp_y);

/* The planner's inputs to the host without the copy engine: n doubles from
 * device memory src stored by a kernel into dst, a pinned (device-mapped)
 * host buffer; visible to the host once the stream has reached this point.
 * The reference's planner reads ||B_i|| and ||X^s|| on the host between the
 * block assembly and the Horner recurrence (engine.py:467-470); a memcpy of
 * these few hundred bytes queues behind the previous result's download on
 * the device-to-host copy engine and stalls the planner for its whole
 * duration (cfg2 host stream: 1.63 instead of 1.09 ms per step). */
int mpps_store_host(mpps_handle *h, const double *src, double *dst_pinned, long long n);

/* one_norm of complex matrices (precision.py:235-249 with mpc_abs, the
 * reference's native element type, precision.py:78-105): A holds the real
 * embeddings [[Re, -Im], [Im, Re]] (2nc x 2nc) on which the evaluators run
 * complex inputs; norms[b * stride] = max_j sum_i |z_ij|, |z| = hypot(Re, Im). */
int mpps_one_norm_complex(mpps_handle *h, const mpps_mat *A, int nc, double *norms, int stride);

/* One fused matrix-Horner step of horner_mixed (engine.py:249-251):
 *   out = RN_out( 2^eo ( Bprev + 2^-(ey+ei) * RN_fmt(Y * phi) ) )
 * Y and phi share the level-j format, Bprev is the working-format block and
 * out is in the level-(j-1) format (>= level j's).  Shapes: Y is M x K, phi
 * K x N, Bprev and out M x N (K = n; M, N < n for SUMMA blocks). */
int mpps_horner_step(mpps_handle *h, const mpps_mat *Y, const mpps_mat *phi,
                     const mpps_mat *Bprev, mpps_mat *out, const int *sel,
                     int nsel, const int *exp_y, const int *exp_in,
                     const int *exp_out);

/* Top Horner step when B_r = b_m I (m mod s == 0, engine.py:132): the
 * reference's Y * (b_m I) equals RN_j(b_m * Y) entrywise, so no GEMM runs:
 *   out = RN_out( 2^eo ( Bprev + RN_{fmt_top}(b_m * Y) ) ).
 * Y is at the working format; fmt_top is the level-r format. */
int mpps_horner_scalar_top(mpps_handle *h, const double *bm_words, int fmt_top,
                           const mpps_mat *Y, const mpps_mat *Bprev,
                           mpps_mat *out, const int *sel, int nsel,
                           const int *exp_out);

/* ------------------------------------------------------------------
 * Tensor-core path (INT8 tcgen05 MMA, exact operand splitting).
 * A multiword operand is split into signed 8-bit digit planes with one
 * power-of-two scale per row (side 0, the left operand) or per column
 * (side 1, the right operand, stored transposed); C = A B is then a sum of
 * exact int32 tensor-core products recombined in the target format.
 * Slices used per format: fp64 8, dd 16 (14 with 8-bit digits), qd 31 (28)
 * (first digits of a finer split are a valid coarser split, so one slicing
 * serves every level).
 */
typedef struct {
  void *digits;      /* device int8 [nslices][batch][rpad][kpad]            */
  int *exps;         /* device int32 [batch][rpad] (row/column exponents)   */
  int nslices, batch;
  int rpad;          /* padded rows (side 0) / columns (side 1), % 128 == 0 */
  int kpad;          /* padded inner dimension, % 32 == 0                   */
  int digit_bits;    /* 7: digits in [-65, 65]; 8: [-128, 127] (first digit
                        6 bits either way); 0 means 7.  Both operands of a
                        product must use the same width.                    */
} mpps_slices;

/* Split src (side 0: by rows, side 1: by columns) into out->nslices digit
 * planes (padding written as zero). */
int mpps_slice(mpps_handle *h, const mpps_mat *src, int side, mpps_slices *out,
               const int *sel, int nsel);
/* mpps_slice in two halves, for operands whose row / column scales span
 * more than the caller's block (the SUMMA driver splits its own block and
 * gathers digit planes): mode 1 writes only out->exps (each row's -- side 0
 * -- or column's -- side 1 -- power-of-two scale); mode 2 splits with the
 * scales already in out->exps (which may be larger than the block's own, e.g.
 * the max over a process row), giving exactly the digits the split of the
 * whole panel would give; mode 0 = mpps_slice. */
int mpps_slice_ex(mpps_handle *h, const mpps_mat *src, int side, mpps_slices *out,
                  const int *sel, int nsel, int mode);
/* Column split of src into slice rows [row0, row0 + src->cols) of out: the
 * right operand [P_0 | P_1] of one GEMM over several matrices (the power
 * chain's [X | X^2]); other rows are untouched. */
int mpps_slice_into(mpps_handle *h, const mpps_mat *src, mpps_slices *out, int row0, const int *sel, int nsel);

/* mat_mul (precision.py:160-184) on the tensor cores: C (M x N, format of C)
 * = A (sliced by rows) * B (sliced by columns), using nslices digit planes. */
int mpps_gemm_sliced(mpps_handle *h, const mpps_slices *A, const mpps_slices *B,
                     int nslices, int M, int N, int K, mpps_mat *C,
                     const int *sel, int nsel);

/* horner_mixed level (engine.py:249-251) on the tensor cores; same epilogue
 * as mpps_horner_step. */
int mpps_horner_step_sliced(mpps_handle *h, const mpps_slices *Y,
                            const mpps_slices *phi, int nslices,
                            const mpps_mat *Bprev, mpps_mat *out,
                            const int *sel, int nsel, const int *exp_y,
                            const int *exp_in, const int *exp_out);

/* Digit planes the tensor-core path uses for a format (-1: not supported):
 * 7-bit digits fp32 4, fp64 8, dd 16, qd 31 (mpps_oz_slices_for); 8-bit
 * digits fp32 4, fp64 8, dd 14, qd 28 (mpps_oz_slices_for_bits(fmt, 8)). */
int mpps_oz_slices_for(int fmt);
int mpps_oz_slices_for_bits(int fmt, int digit_bits);

/* Largest inner dimension K for which 8-bit digits keep every int32
 * diagonal accumulator exact at any format (qd: 28 planes). */
int mpps_oz_max_k_8bit(void);
/* Largest inner dimension K for which a product of format fmt's full plane
 * count with digit_bits-bit digits keeps its int32 diagonal accumulators
 * exact (dd: 10070 with 8-bit digits, 31770 with 7-bit; qd: 4851 / 16443). */
int mpps_oz_max_k(int fmt, int digit_bits);

/* K5: the whole mixed PS evaluation of small matrices (n <= 32, fp64
 * working format) in two launches around the host planner, one
 * CTA per matrix, operands in shared memory.
 *   mpps_small_ps_prepare: powers X^2..X^s, blocks B_0..B_r and the planner
 *     norms (eval_b0_and_power + assemble_block + one_norm, engine.py:127-154,
 *     467-468).  coeff: m+1 fp64 RN_p(b_k); blocks: device (r+1, B, n, n)
 *     fp64 (block r not written when m mod s == 0: B_r = b_m I); Y: device
 *     (B, n, n); norms: device (B, r+2) = ||B_0..B_r||, ||Y||.
 *   mpps_small_ps_horner: horner_mixed (engine.py:243-252) with per-matrix
 *     level formats level_fmt: HOST (B, r+1) int8, 0 = fp32, 1 = fp64 (copied
 *     into the launch; the call returns once it is enqueued);
 *     out: contiguous fp64 (B, n, n).  bm = RN_p(b_m). */
int mpps_small_ps_supported(int n, int m, int fmt);
int mpps_small_ps_prepare(mpps_handle *h, const mpps_mat *X, int m, int s, const double *coeff,
                          double *blocks, double *Y, double *norms);
int mpps_small_ps_horner(mpps_handle *h, const double *Y, const double *blocks, const signed char *level_fmt,
                         int m, int s, double bm, mpps_mat *out);
/* The whole small evaluation (engine.py:390-482 for one matrix per CTA) in
 * one call and one launch: prepare, the planner's digit rule in certified
 * float64 on the device (digits_host (B, r), nu_host (B); fixed != 0: all
 * levels at d), Horner from the blocks still in shared memory.  The norms
 * (norms_host, (B, r+2)) and the plan reach the host through pinned memory;
 * the call returns when every matrix is planned, the Horner chains may still
 * be running on the handle's stream.  Returns 4 (MPPS_NEED_PLAN) when some e_i
 * lies within 1e-8 of a digit boundary (those matrices' Horner chains are not
 * run): the caller then plans exactly and calls mpps_small_ps_horner on the
 * blocks, Y and norms this call left in place. */
#define MPPS_NEED_PLAN 4
int mpps_small_ps_eval(mpps_handle *h, const mpps_mat *X, int m, int s, const double *coeff, int d, double delta,
                       int apply_switch, int fixed, double *blocks, double *Y, double *norms_dev,
                       double *norms_host, int *digits_host, int *nu_host, mpps_mat *out);

/* Diagnostic: pipe-peak probe used by bench.py for the per-precision
 * roofline denominators (not a reference operator).  Launches `blocks`
 * CTAs x 256 threads, each running 8 independent FMA chains of `iters`
 * steps in fmt (MPPS_FP32 / MPPS_FP64): 16 * iters flops per thread. */
int mpps_probe_fma(mpps_handle *h, int fmt, int blocks, int iters, void *scratch);

/* Diagnostic: INT8 tensor-pipe peak probe (tcgen05 kind::i8, 128x256x32
 * MMAs back to back, one CTA per SM): 2*128*256*32*iters ops per CTA. */
int mpps_probe_i8mma(mpps_handle *h, int blocks, int iters, void *scratch);

/* Diagnostic: while `buf` (device, 5 x uint64 per CTA) is set, the TMA-fed
 * tensor-core GEMMs record per-CTA %globaltimer stamps (start, after
 * setup, MMAs done, end) and the SM id; NULL turns it off.  Process-wide;
 * for tools/cta_timeline.py only. */
void mpps_debug_oz_trace(void *buf);

/* Diagnostic: bit 0 skips the MMAs (operand feed only), bit 1 skips the
 * TMA loads (MMAs on stale shared memory) of the TMA-fed GEMMs (results
 * are garbage while set); bits 8.. override the tile-raster group size
 * (0 = default / MPPS_OZ_GROUP).  For tools/ only. */
void mpps_debug_oz_flags(int flags);

/* Peak probe: global -> shared ingest.  `blocks` CTAs (one per SM) each
 * stream iters x 16 KB bulk copies (TMA engine, 8 in flight) from src
 * (span_bytes, keep it L2-resident); bytes = blocks * iters * 16384. */
int mpps_probe_ingest(mpps_handle *h, int blocks, int iters, const void *src, long long span_bytes);

/* Diagnostic: mpps_probe_i8mma with M = 128, N = n (16..256, multiple of
 * 16), K = 32 MMAs back to back. */
int mpps_debug_probe_i8mma_n(mpps_handle *h, int blocks, int iters, int n, void *scratch);

#ifdef __cplusplus
}
#endif
#endif /* MPPS_B200_H */
