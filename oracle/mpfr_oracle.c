/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle of the B200 mixed-precision
 * Paterson-Stockmeyer hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library;
 * the product path (paper_2312_17396_b200/) never links or calls it.
 *
 * A plain-C restatement of the reference's arithmetic (pkg/src/mpps, pure
 * Python over gmpy2 -> MPFR/MPC).  The reference's hot path rounds every
 * scalar op at p = ceil(d*log2 10) bits, round-to-nearest-even, in a fixed
 * sequential order.  This file performs the same MPFR calls in the same
 * order, so for real inputs it reproduces the reference bit for bit
 * (mpc ops with zero imaginary parts equal MPFR real ops):
 *
 *   orc_matmul / mat_mul      precision.py:160-184  acc = RN(a_i0 b_0j);
 *                                                   acc = RN(acc + RN(a_ik b_kj))
 *   axpy                      precision.py:187-197  RN(RN(alpha a) + b)
 *   add                       precision.py:200-207
 *   one_norm                  precision.py:235-249  54-bit sequential column sums
 *   orc_prepare               engine.py:141-154 (eval_b0_and_power),
 *                             engine.py:127-138 (assemble_block), 467-468 (norms)
 *   orc_horner                engine.py:243-252 (horner_mixed)
 *   orc_plan                  engine.py:184-215 (the digit rule of plan_precisions)
 *   orc_poly_cols             Tier C of SURVEY 8(c): sampled columns of p(X) (or
 *                             p(X^2)) by matrix-vector Horner at high precision --
 *                             the ground truth of harness.py:105-109 (reference_eval,
 *                             2x digits) for sizes whose n^3 MPFR GEMMs cannot finish
 *   orc_matpow_cols           sampled columns of P^k (the squaring phase of cfg3)
 *
 * MPFR 4.2.1 is present as a runtime library only (no headers), so the few
 * prototypes needed are declared here against the documented ABI
 * (__mpfr_struct = {prec, sign, exp, limb*}).  Row loops of the GEMM run
 * under OpenMP (each output entry is still the reference's sequential sum).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef struct {
  mpfr_prec_t _mpfr_prec;
  mpfr_sign_t _mpfr_sign;
  mpfr_exp_t _mpfr_exp;
  unsigned long *_mpfr_d;
} mpfr_struct;
typedef mpfr_struct *mpfr_ptr;
typedef const mpfr_struct *mpfr_srcptr;
enum { RNDN = 0 };

extern void mpfr_init2(mpfr_ptr, mpfr_prec_t);
extern void mpfr_clear(mpfr_ptr);
extern void mpfr_set_prec(mpfr_ptr, mpfr_prec_t);
extern int mpfr_set(mpfr_ptr, mpfr_srcptr, int);
extern int mpfr_set_d(mpfr_ptr, double, int);
extern int mpfr_set_si(mpfr_ptr, long, int);
extern int mpfr_set_str(mpfr_ptr, const char *, int, int);
extern double mpfr_get_d(mpfr_srcptr, int);
extern int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, int);
extern int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, int);
extern int mpfr_sub(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, int);
extern int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, int);
extern int mpfr_abs(mpfr_ptr, mpfr_srcptr, int);
extern int mpfr_log10(mpfr_ptr, mpfr_srcptr, int);
extern int mpfr_cmp(mpfr_srcptr, mpfr_srcptr);
extern int mpfr_sgn(mpfr_srcptr);
extern int mpfr_zero_p(mpfr_srcptr);
extern int mpfr_mul_d(mpfr_ptr, mpfr_srcptr, double, int);

#define NORM_BITS 54  /* NORM_CTX = 16 digits (precision.py:72) */
#define BOUND_BITS 107 /* BOUND_CTX = 32 digits (precision.py:75) */
#define WIDE_BITS 1024

typedef struct {
  int n;
  mpfr_struct *v; /* n*n, row-major */
} mat;

static mat mat_new(int n, long bits) {
  mat A;
  A.n = n;
  A.v = (mpfr_struct *)malloc(sizeof(mpfr_struct) * (size_t)n * n);
  for (long i = 0; i < (long)n * n; ++i) {
    mpfr_init2(&A.v[i], bits);
    mpfr_set_si(&A.v[i], 0, RNDN);
  }
  return A;
}
static void mat_free(mat *A) {
  if (!A->v) return;
  for (long i = 0; i < (long)A->n * A->n; ++i) mpfr_clear(&A->v[i]);
  free(A->v);
  A->v = NULL;
}
static void mat_set_prec(mat *A, long bits) {
  for (long i = 0; i < (long)A->n * A->n; ++i) mpfr_set_prec(&A->v[i], bits);
}

/* C = RN_bits(A * B), sequential inner product, separate mul/add roundings
 * (precision.py:176-181). */
static void mat_mul(const mat *A, const mat *B, mat *C, long bits) {
  int n = A->n;
  mat_set_prec(C, bits);
#pragma omp parallel
  {
    mpfr_struct t;
    mpfr_init2(&t, bits);
#pragma omp for schedule(dynamic, 1)
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) {
        mpfr_ptr acc = &C->v[(long)i * n + j];
        mpfr_mul(acc, &A->v[(long)i * n], &B->v[j], RNDN);
        for (int k = 1; k < n; ++k) {
          mpfr_mul(&t, &A->v[(long)i * n + k], &B->v[(long)k * n + j], RNDN);
          mpfr_add(acc, acc, &t, RNDN);
        }
      }
    }
    mpfr_clear(&t);
  }
}

/* B = RN(RN(alpha*A) + B) in place, B already at `bits` (precision.py:194-196:
 * add(mul(a, x), y); the exact sum is commutative, so operand order is moot). */
static void mat_axpy_inplace(mpfr_srcptr alpha, const mat *A, mat *B, long bits) {
  long nn = (long)A->n * A->n;
  mpfr_struct t;
  mpfr_init2(&t, bits);
  for (long i = 0; i < nn; ++i) {
    mpfr_mul(&t, alpha, &A->v[i], RNDN);
    mpfr_add(&B->v[i], &t, &B->v[i], RNDN);
  }
  mpfr_clear(&t);
}

/* C = RN(A + B) at bits; C may alias neither. */
static void mat_add(const mat *A, const mat *B, mat *C, long bits) {
  long nn = (long)A->n * A->n;
  mat_set_prec(C, bits);
  for (long i = 0; i < nn; ++i) mpfr_add(&C->v[i], &A->v[i], &B->v[i], RNDN);
}

/* one_norm at 54 bits (precision.py:235-249). */
static void one_norm(const mat *A, mpfr_ptr best) {
  int n = A->n;
  mpfr_struct s, a;
  mpfr_init2(&s, NORM_BITS);
  mpfr_init2(&a, NORM_BITS);
  mpfr_set_prec(best, NORM_BITS);
  mpfr_set_si(best, 0, RNDN);
  for (int j = 0; j < n; ++j) {
    mpfr_set_si(&s, 0, RNDN);
    for (int i = 0; i < n; ++i) {
      mpfr_abs(&a, &A->v[(long)i * n + j], RNDN);
      mpfr_add(&s, &s, &a, RNDN);
    }
    if (mpfr_cmp(&s, best) > 0) mpfr_set(best, &s, RNDN);
  }
  mpfr_clear(&s);
  mpfr_clear(&a);
}

/* exact split of an MPFR value into nw doubles (greedy nearest) */
static void split(mpfr_srcptr x, double *out, int nw, long stride) {
  mpfr_struct r;
  mpfr_init2(&r, WIDE_BITS);
  mpfr_set(&r, x, RNDN);
  for (int w = 0; w < nw; ++w) {
    double d = mpfr_get_d(&r, RNDN);
    out[w * stride] = d;
    mpfr_struct dd;
    mpfr_init2(&dd, 64);
    mpfr_set_d(&dd, d, RNDN);
    mpfr_sub(&r, &r, &dd, RNDN);
    mpfr_clear(&dd);
  }
  mpfr_clear(&r);
}

/* value = sum of nw word planes (exact at WIDE_BITS) rounded to bits */
static void set_words(mpfr_ptr x, const double *w, int nw, long stride, long bits) {
  mpfr_struct acc, t;
  mpfr_init2(&acc, WIDE_BITS);
  mpfr_init2(&t, 64);
  mpfr_set_si(&acc, 0, RNDN);
  for (int k = 0; k < nw; ++k) {
    mpfr_set_d(&t, w[k * stride], RNDN);
    mpfr_add(&acc, &acc, &t, RNDN);
  }
  mpfr_set_prec(x, bits);
  mpfr_set(x, &acc, RNDN);
  mpfr_clear(&acc);
  mpfr_clear(&t);
}

/* correctly rounded num/den at bits (coefficients.py:87-89) */
static void set_rational(mpfr_ptr x, const char *num, const char *den, long bits) {
  mpfr_struct a, b;
  long na = (long)strlen(num) * 4 + 16, nb = (long)strlen(den) * 4 + 16;
  mpfr_init2(&a, na);
  mpfr_init2(&b, nb);
  mpfr_set_str(&a, num, 10, RNDN); /* exact: precision > log2(10)*digits */
  mpfr_set_str(&b, den, 10, RNDN);
  mpfr_set_prec(x, bits);
  mpfr_div(x, &a, &b, RNDN);
  mpfr_clear(&a);
  mpfr_clear(&b);
}

/* ------------------------------------------------------------ PS state */
typedef struct {
  int n, m, s, r, have_result;
  long wbits;
  mat *powers;      /* s+1: I, X, ..., X^s (index 0 unused) */
  mat *blocks;      /* r+1 */
  mpfr_struct *coef;/* m+1 at wbits */
  mat result;
} orc_ps;

orc_ps *orc_new(int n) {
  orc_ps *p = (orc_ps *)calloc(1, sizeof(orc_ps));
  p->n = n;
  return p;
}

static void free_state(orc_ps *p) {
  if (p->powers) {
    for (int k = 0; k <= p->s; ++k) mat_free(&p->powers[k]);
    free(p->powers);
    p->powers = NULL;
  }
  if (p->blocks) {
    for (int k = 0; k <= p->r; ++k) mat_free(&p->blocks[k]);
    free(p->blocks);
    p->blocks = NULL;
  }
  if (p->coef) {
    for (int k = 0; k <= p->m; ++k) mpfr_clear(&p->coef[k]);
    free(p->coef);
    p->coef = NULL;
  }
  if (p->have_result) mat_free(&p->result);
  p->have_result = 0;
}

void orc_free(orc_ps *p) {
  if (!p) return;
  free_state(p);
  free(p);
}

/* eval_b0_and_power + assemble_block(i>=1) + norms, at wbits.
 *   X: xwords planes of n*n doubles (exact sum = the argument), rounded at
 *      wbits (round_to, engine.py:147);
 *   nums/dens: m+1 decimal strings of the exact coefficients;
 *   norms_out: (r+2) x 2 doubles, exact (hi, lo) of the 54-bit norms
 *      ||B_0..B_r|| then ||Y||.
 * explicit_b0_first: when nonzero, B_0 is assembled with assemble_block as
 * in ps_fixed (engine.py:328) instead of interleaved -- identical math. */
int orc_prepare(orc_ps *p, const double *X, int xwords, int m, int s, long wbits, const char **nums,
                const char **dens, double *norms_out) {
  int n = p->n;
  if (s < 1 || s > m) return 1;
  free_state(p);
  p->m = m;
  p->s = s;
  p->r = m / s;
  p->wbits = wbits;
  p->coef = (mpfr_struct *)malloc(sizeof(mpfr_struct) * (m + 1));
  for (int k = 0; k <= m; ++k) {
    mpfr_init2(&p->coef[k], wbits);
    set_rational(&p->coef[k], nums[k], dens[k], wbits);
  }
  p->powers = (mat *)calloc(s + 1, sizeof(mat));
  for (int k = 1; k <= s; ++k) p->powers[k] = mat_new(n, wbits);
  for (long i = 0; i < (long)n * n; ++i) set_words(&p->powers[1].v[i], X + i, xwords, (long)n * n, wbits);
  /* interleaved power formation (engine.py:151-153) */
  for (int j = 1; j < s; ++j) mat_mul(&p->powers[j], &p->powers[1], &p->powers[j + 1], wbits);
  /* blocks (engine.py:127-138): acc = b_{si} I; acc = RN(RN(b X^j) + acc) */
  int r = p->r, full = m / s;
  p->blocks = (mat *)calloc(r + 1, sizeof(mat));
  for (int i = 0; i <= r; ++i) {
    int hi = (i < full) ? s - 1 : m - s * full;
    mat *B = &p->blocks[i];
    *B = mat_new(n, wbits);
    for (int d = 0; d < n; ++d) mpfr_set(&B->v[(long)d * n + d], &p->coef[s * i], RNDN);
    for (int j = 1; j <= hi; ++j) mat_axpy_inplace(&p->coef[s * i + j], &p->powers[j], B, wbits);
  }
  mpfr_struct nrm, t;
  mpfr_init2(&nrm, NORM_BITS);
  mpfr_init2(&t, WIDE_BITS);
  for (int i = 0; i <= r + 1; ++i) {
    one_norm(i <= r ? &p->blocks[i] : &p->powers[s], &nrm);
    split(&nrm, norms_out + 2 * i, 2, 1);
  }
  mpfr_clear(&nrm);
  mpfr_clear(&t);
  return 0;
}

/* horner_mixed (engine.py:243-252): level_bits[0] = working, [j] = level j. */
int orc_horner(orc_ps *p, const long *level_bits) {
  int n = p->n, r = p->r;
  if (!p->blocks) return 1;
  if (p->have_result) mat_free(&p->result);
  mat phi = mat_new(n, level_bits[r]);
  for (long i = 0; i < (long)n * n; ++i) {
    mpfr_set_prec(&phi.v[i], p->blocks[r].v[i]._mpfr_prec);
    mpfr_set(&phi.v[i], &p->blocks[r].v[i], RNDN);
  }
  mat tmp = mat_new(n, 2);
  for (int j = r; j >= 1; --j) {
    mat_mul(&p->powers[p->s], &phi, &tmp, level_bits[j]);
    mat_add(&p->blocks[j - 1], &tmp, &phi, level_bits[j - 1]);
  }
  mat_free(&tmp);
  p->result = phi;
  p->have_result = 1;
  return 0;
}

/* result entries as nw exact word planes (n*n each) */
int orc_result_words(const orc_ps *p, double *out, int nw) {
  if (!p->have_result) return 1;
  long nn = (long)p->n * p->n;
  for (long i = 0; i < nn; ++i) split(&p->result.v[i], out + i, nw, nn);
  return 0;
}

/* block / power entries as 4 word planes: which = 0..r blocks, r+1+k = X^k */
int orc_matrix_words(const orc_ps *p, int which, double *out) {
  long nn = (long)p->n * p->n;
  const mat *A;
  if (which <= p->r) A = &p->blocks[which];
  else if (which - p->r - 1 >= 1 && which - p->r - 1 <= p->s) A = &p->powers[which - p->r - 1];
  else return 1;
  for (long i = 0; i < nn; ++i) split(&A->v[i], out + i, 4, nn);
  return 0;
}

/* ||G - R||_1 and ||R||_1 (R = oracle result), the difference taken at
 * WIDE_BITS so it measures the operands (harness.py:112-121). */
int orc_compare(const orc_ps *p, const double *g, int gw, double *diff, double *refn) {
  if (!p->have_result) return 1;
  int n = p->n;
  long nn = (long)n * n;
  mat D = mat_new(n, WIDE_BITS);
  mpfr_struct gv;
  mpfr_init2(&gv, WIDE_BITS);
  for (long i = 0; i < nn; ++i) {
    set_words(&gv, g + i, gw, nn, WIDE_BITS);
    mpfr_sub(&D.v[i], &gv, &p->result.v[i], RNDN);
  }
  mpfr_clear(&gv);
  /* norms at WIDE_BITS (not 54) so tiny differences are resolved */
  mpfr_struct s, a, best;
  mpfr_init2(&s, WIDE_BITS);
  mpfr_init2(&a, WIDE_BITS);
  mpfr_init2(&best, WIDE_BITS);
  for (int pass = 0; pass < 2; ++pass) {
    const mat *A = pass == 0 ? &D : &p->result;
    mpfr_set_si(&best, 0, RNDN);
    for (int j = 0; j < n; ++j) {
      mpfr_set_si(&s, 0, RNDN);
      for (int i = 0; i < n; ++i) {
        mpfr_abs(&a, &A->v[(long)i * n + j], RNDN);
        mpfr_add(&s, &s, &a, RNDN);
      }
      if (mpfr_cmp(&s, &best) > 0) mpfr_set(&best, &s, RNDN);
    }
    if (pass == 0) *diff = mpfr_get_d(&best, RNDN);
    else *refn = mpfr_get_d(&best, RNDN);
  }
  mpfr_clear(&s);
  mpfr_clear(&a);
  mpfr_clear(&best);
  mat_free(&D);
  return 0;
}

/* Plain mat_mul for operator-level parity: A, B given as aw / bw word planes,
 * C returned as 4 word planes. */
int orc_matmul(int n, const double *A, int aw, const double *B, int bw, long bits, double *C4) {
  long nn = (long)n * n;
  mat a = mat_new(n, WIDE_BITS), b = mat_new(n, WIDE_BITS), c = mat_new(n, bits);
  for (long i = 0; i < nn; ++i) {
    set_words(&a.v[i], A + i, aw, nn, WIDE_BITS);
    set_words(&b.v[i], B + i, bw, nn, WIDE_BITS);
  }
  mat_mul(&a, &b, &c, bits);
  for (long i = 0; i < nn; ++i) split(&c.v[i], C4 + i, 4, nn);
  mat_free(&a);
  mat_free(&b);
  mat_free(&c);
  return 0;
}

/* The digit rule of plan_precisions (engine.py:184-215) on exact norms
 * given as (hi, lo) word pairs: first mpfr(b, 64) (engine.py:170-171), then
 * e_i at 107 bits, + mpfr("1e-9") (53 bits), float(), floor, clamp, delta
 * switch, running max.  Returns 1 for the nilpotent plan (norm_y == 0). */
int orc_plan(const double *norm_bs2, const double *norm_y2, int r, int d, double delta, int apply_switch,
             int *digits, int *nu_out, double *e_out) {
  mpfr_struct nb[64], ny, lb0, ly, e, t, u, onee9;
  if (r + 1 > 64) return -1;
  for (int i = 0; i <= r; ++i) {
    mpfr_init2(&nb[i], 64);
    set_words(&nb[i], norm_bs2 + 2 * i, 2, 1, 64);
  }
  mpfr_init2(&ny, 64);
  set_words(&ny, norm_y2, 2, 1, 64);
  int rc = 0;
  if (mpfr_zero_p(&ny)) {
    for (int i = 0; i < r; ++i) digits[i] = 1;
    *nu_out = 1;
    rc = 1;
    goto done;
  }
  mpfr_init2(&lb0, BOUND_BITS);
  mpfr_init2(&ly, BOUND_BITS);
  mpfr_init2(&e, BOUND_BITS);
  mpfr_init2(&t, BOUND_BITS);
  mpfr_init2(&u, BOUND_BITS);
  mpfr_init2(&onee9, 53);
  mpfr_set_str(&onee9, "1e-9", 10, RNDN);
  if (mpfr_sgn(&nb[0]) > 0) mpfr_log10(&lb0, &nb[0], RNDN);
  else mpfr_set_si(&lb0, 0, RNDN);
  mpfr_log10(&ly, &ny, RNDN);
  int qual[64];
  double lim = d - log10(delta);
  for (int i = 1; i <= r; ++i) {
    if (mpfr_zero_p(&nb[i]) || mpfr_zero_p(&nb[0])) {
      digits[i - 1] = 1;
      qual[i - 1] = 1;
      e_out[i - 1] = NAN;
      continue;
    }
    mpfr_struct dd;
    mpfr_init2(&dd, 64);
    mpfr_set_si(&dd, d, RNDN);
    mpfr_sub(&e, &dd, &lb0, RNDN);         /* RN(d - log_b0) */
    mpfr_log10(&t, &nb[i], RNDN);          /* RN(log10 b_i) */
    mpfr_set_si(&dd, i, RNDN);
    mpfr_mul(&u, &dd, &ly, RNDN);          /* RN(i * log_y) */
    mpfr_add(&t, &t, &u, RNDN);
    mpfr_add(&e, &e, &t, RNDN);
    mpfr_add(&e, &e, &onee9, RNDN);
    double ef = mpfr_get_d(&e, RNDN);
    e_out[i - 1] = ef;
    int di = (int)floor(ef);
    if (di > d) di = d;
    if (di < 1) di = 1;
    digits[i - 1] = di;
    qual[i - 1] = ef <= lim;
    mpfr_clear(&dd);
  }
  {
    int nu = r + 1;
    for (int i = 1; i <= r; ++i)
      if (qual[i - 1]) { nu = i; break; }
    if (apply_switch)
      for (int i = 1; i < nu; ++i) digits[i - 1] = d;
    for (int i = r - 2; i >= 0; --i)
      if (digits[i + 1] > digits[i]) digits[i] = digits[i + 1];
    *nu_out = nu;
  }
  mpfr_clear(&lb0);
  mpfr_clear(&ly);
  mpfr_clear(&e);
  mpfr_clear(&t);
  mpfr_clear(&u);
  mpfr_clear(&onee9);
done:
  for (int i = 0; i <= r; ++i) mpfr_clear(&nb[i]);
  mpfr_clear(&ny);
  return rc;
}

/* nilpotent plan (engine.py:378-379, 473-474): the result is B_0 itself */
int orc_result_from_block(orc_ps *p, int which) {
  if (!p->blocks || which < 0 || which > p->r) return 1;
  if (p->have_result) mat_free(&p->result);
  int n = p->n;
  p->result = mat_new(n, 2);
  for (long i = 0; i < (long)n * n; ++i) {
    mpfr_set_prec(&p->result.v[i], p->blocks[which].v[i]._mpfr_prec);
    mpfr_set(&p->result.v[i], &p->blocks[which].v[i], RNDN);
  }
  p->have_result = 1;
  return 0;
}

/* ---------------------------------------------------------------- Tier C
 * y = RN_bits(A w) for a dense A given as aw word planes of n*n doubles (the
 * exact sum of the planes is the matrix): per row, acc = sum_k sum_w
 * RN(a_ik^(w) w_k) added sequentially at `bits`.  At twice the working digits
 * this is far below the parity tolerance (c n u_work), like reference_eval. */
static void matvec_words(int n, const double *A, int aw, const mpfr_struct *w, mpfr_struct *y, long bits) {
  long nn = (long)n * n;
#pragma omp parallel
  {
    mpfr_struct t;
    mpfr_init2(&t, bits);
#pragma omp for schedule(static)
    for (int i = 0; i < n; ++i) {
      mpfr_ptr acc = &y[i];
      mpfr_set_si(acc, 0, RNDN);
      for (int k = 0; k < n; ++k) {
        for (int q = 0; q < aw; ++q) {
          double a = A[q * nn + (long)i * n + k];
          if (a == 0.0) continue;
          mpfr_mul_d(&t, &w[k], a, RNDN);
          mpfr_add(acc, acc, &t, RNDN);
        }
      }
    }
    mpfr_clear(&t);
  }
}

static mpfr_struct *vec_new(int n, long bits) {
  mpfr_struct *v = (mpfr_struct *)malloc(sizeof(mpfr_struct) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    mpfr_init2(&v[i], bits);
    mpfr_set_si(&v[i], 0, RNDN);
  }
  return v;
}
static void vec_free(mpfr_struct *v, int n) {
  for (int i = 0; i < n; ++i) mpfr_clear(&v[i]);
  free(v);
}

/* Columns cols[0..ncols) of p(A), A = X (squares = 0) or A = X X (squares =
 * 1, the cosine's Z, harness.py:100-101, applied as X (X w)), p = sum_k b_k
 * A^k with b_k = RN_bits(nums[k]/dens[k]): w = b_m e_j, then
 * w = A w + b_k e_j for k = m-1..0.  out: (4, ncols, n) exact word planes. */
int orc_poly_cols(int n, const double *X, int xw, int m, const char **nums, const char **dens, long bits,
                  int squares, const int *cols, int ncols, double *out) {
  mpfr_struct *coef = (mpfr_struct *)malloc(sizeof(mpfr_struct) * (m + 1));
  for (int k = 0; k <= m; ++k) {
    mpfr_init2(&coef[k], bits);
    set_rational(&coef[k], nums[k], dens[k], bits);
  }
  mpfr_struct *w = vec_new(n, bits), *y = vec_new(n, bits);
  long plane = (long)ncols * n;
  for (int c = 0; c < ncols; ++c) {
    int j = cols[c];
    if (j < 0 || j >= n) return 1;
    for (int i = 0; i < n; ++i) mpfr_set_si(&w[i], 0, RNDN);
    mpfr_set(&w[j], &coef[m], RNDN);
    for (int k = m - 1; k >= 0; --k) {
      matvec_words(n, X, xw, w, y, bits);
      if (squares) {
        mpfr_struct *tmp = w; w = y; y = tmp;
        matvec_words(n, X, xw, w, y, bits);
      }
      mpfr_add(&y[j], &y[j], &coef[k], RNDN);
      mpfr_struct *tmp = w; w = y; y = tmp;
    }
    for (int i = 0; i < n; ++i) split(&w[i], out + (long)c * n + i, 4, plane);
  }
  vec_free(w, n);
  vec_free(y, n);
  for (int k = 0; k <= m; ++k) mpfr_clear(&coef[k]);
  free(coef);
  return 0;
}

/* Columns of P^count (P given as pw word planes) at `bits`: out (4, ncols, n). */
int orc_matpow_cols(int n, const double *P, int pw, int count, long bits, const int *cols, int ncols,
                    double *out) {
  mpfr_struct *w = vec_new(n, bits), *y = vec_new(n, bits);
  long plane = (long)ncols * n;
  for (int c = 0; c < ncols; ++c) {
    int j = cols[c];
    if (j < 0 || j >= n) return 1;
    for (int i = 0; i < n; ++i) mpfr_set_si(&w[i], i == j ? 1 : 0, RNDN);
    for (int k = 0; k < count; ++k) {
      matvec_words(n, P, pw, w, y, bits);
      mpfr_struct *tmp = w; w = y; y = tmp;
    }
    for (int i = 0; i < n; ++i) split(&w[i], out + (long)c * n + i, 4, plane);
  }
  vec_free(w, n);
  vec_free(y, n);
  return 0;
}
