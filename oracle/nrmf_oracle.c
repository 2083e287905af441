/*
 * oracle/nrmf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded C implementation of what the xNRMF hot path
 * computes, written from the paper (arXiv 2509.06220, /root/reference/PAPER.md,
 * cited below as P:<line>).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this code.  It shares no code,
 * header, table or constant with the CUDA path (paper_2509_06220_b200/csrc) and
 * must never be called by the product path.
 *
 * Build (see __graft_entry__.build / oracle/__init__.py):
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *       -o oracle/liboracle.so oracle/nrmf_oracle.c -lm
 * -ffp-contract=off: no multiply-add is ever fused except the explicit fma()
 * of Listing 2; x86-64 uses SSE2 scalar arithmetic (no x87 double rounding);
 * gradual underflow is the default (no FTZ/DAZ).
 *
 * Contents
 *   1. v1_hypot / v1_hypotf        -- Listing 2, statement by statement.
 *   2. R_H / R_Hf                  -- Listing 1, literally (recursive,
 *                                     ceil split p = ceil(n/2)).
 *   3. oracle_nrmf_[sd]            -- the frozen tile-lane tree (DESIGN.md §3,
 *                                     SURVEY.md Appendix A): tile transpose, zero
 *                                     padding, then R_H (= BAL on power-of-two
 *                                     lengths) over the whole padded array.
 *   4. oracle_nrmf_cols_[sd]       -- per-column trees + BAL over column norms
 *                                     (e:F: the inner sum is over rows).
 *   5. exact_nrm_[sd]              -- RN(sqrt(sum x_i^2)) computed EXACTLY: an
 *                                     integer fixed-point superaccumulator plus a
 *                                     correctly rounded integer square root; the
 *                                     "exact" ||x||'_F of P:727-731 (reading R7).
 *
 * Parity pins: every function above is pinned by tests/test_oracle_*.py against
 * things that do not come from this file (closed forms, Python exact-rational
 * arithmetic, the paper's Table 3, worked examples).  See DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* 1. v1_hypot -- Listing 2.  Each statement is one IEEE-754 RN   */
/*    operation.  fmin/fmax return the non-NaN operand.              */
/* ------------------------------------------------------------------------- */
double oracle_v1_hypot_d(double x, double y)
{
    const double X = fabs(x);          /* X = |x| */
    const double Y = fabs(y);          /* Y = |y| */
    const double m = fmin(X, Y);       /* m = min{X,Y} */
    const double M = fmax(X, Y);       /* M = max{X,Y} */
    const double q = (m / M);          /* may be NaN if m = M = 0 */
    const double Q = fmax(q, 0.0);     /* ... Q is not a NaN */
    const double S = fma(Q, Q, 1.0);   /* S = fma(Q,Q,1), one rounding P:629 */
    const double s = sqrt(S);          /* s = sqrt(S) */
    return (M * s);                    /* M*sqrt(1+(m/M)^2) */
}

/* Listing 2 applied to n pairs (a convenience loop for large pin sets). */
void oracle_v1_hypot_array_d(int64_t n, const double *x, const double *y, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_v1_hypot_d(x[i], y[i]);
}

/* R_S substitutions double->float, fabs->fabsf, hypot->hypotf. */
float oracle_v1_hypot_s(float x, float y)
{
    const float X = fabsf(x);
    const float Y = fabsf(y);
    const float m = fminf(X, Y);
    const float M = fmaxf(X, Y);
    const float q = (m / M);
    const float Q = fmaxf(q, 0.0f);
    const float S = fmaf(Q, Q, 1.0f);
    const float s = sqrtf(S);
    return (M * s);
}

void oracle_v1_hypot_array_s(int64_t n, const float *x, const float *y, float *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_v1_hypot_s(x[i], y[i]);
}

/* ------------------------------------------------------------------------- */
/* 2. Listing 1, H variant (hypot = v1_hypot).         */
/* ------------------------------------------------------------------------- */
double oracle_R_H_d(int64_t n, const double *x)
{
    if (n == 1) return fabs(*x);
    if (n == 2) return oracle_v1_hypot_d(x[0], x[1]);
    const int64_t p = ((n >> 1) + (n & 1));               /* p = ceil(n/2) P:593 */
    const int64_t q = (n - p);                            /* q = n - p */
    const double fp = oracle_R_H_d(p, x);
    const double fq = oracle_R_H_d(q, x + p);
    return oracle_v1_hypot_d(fp, fq);
}

float oracle_R_H_s(int64_t n, const float *x)
{
    if (n == 1) return fabsf(*x);
    if (n == 2) return oracle_v1_hypot_s(x[0], x[1]);
    const int64_t p = ((n >> 1) + (n & 1));
    const int64_t q = (n - p);
    const float fp = oracle_R_H_s(p, x);
    const float fq = oracle_R_H_s(q, x + p);
    return oracle_v1_hypot_s(fp, fq);
}

/* ------------------------------------------------------------------------- */
/* 2b. cr_hypot ("correctly rounded hypotenuse functions") and the   */
/*     A variant of Listing 1 (A_x = R with cr_hypot).  The plain    */
/*     definition written out: RN(sqrt(x^2 + y^2)) computed exactly by the     */
/*     exact reference of section 5; IEEE 754 hypot specials: +inf if either   */
/*     operand is infinite (even with a NaN), else NaN if either is NaN.        */
/* ------------------------------------------------------------------------- */
double exact_nrm_d(const double *x, int64_t n);
float exact_nrm_s(const float *x, int64_t n);

double oracle_cr_hypot_d(double x, double y)
{
    if (isinf(x) || isinf(y)) return INFINITY;
    if (isnan(x) || isnan(y)) return NAN;
    const double v[2] = {x, y};
    return exact_nrm_d(v, 2);
}

float oracle_cr_hypot_s(float x, float y)
{
    if (isinf(x) || isinf(y)) return INFINITY;
    if (isnan(x) || isnan(y)) return NAN;
    const float v[2] = {x, y};
    return exact_nrm_s(v, 2);
}

void oracle_cr_hypot_array_d(int64_t n, const double *x, const double *y, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_cr_hypot_d(x[i], y[i]);
}

void oracle_cr_hypot_array_s(int64_t n, const float *x, const float *y, float *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_cr_hypot_s(x[i], y[i]);
}

double oracle_R_A_d(int64_t n, const double *x)
{
    if (n == 1) return fabs(*x);
    if (n == 2) return oracle_cr_hypot_d(x[0], x[1]);
    const int64_t p = ((n >> 1) + (n & 1));
    const int64_t q = (n - p);
    const double fp = oracle_R_A_d(p, x);
    const double fq = oracle_R_A_d(q, x + p);
    return oracle_cr_hypot_d(fp, fq);
}

float oracle_R_A_s(int64_t n, const float *x)
{
    if (n == 1) return fabsf(*x);
    if (n == 2) return oracle_cr_hypot_s(x[0], x[1]);
    const int64_t p = ((n >> 1) + (n & 1));
    const int64_t q = (n - p);
    const float fp = oracle_R_A_s(p, x);
    const float fq = oracle_R_A_s(q, x + p);
    return oracle_cr_hypot_s(fp, fq);
}

/* ------------------------------------------------------------------------- */
/* 3. The tile-lane tree (DESIGN.md §3 / SURVEY Appendix A).                  */
/*                                                                           */
/*   lanes = number of lanes p (fp64 production: 64, fp32: 128)               */
/*   J     = elements per lane per tile (fp64: 64, fp32: 32)                  */
/*   T     = lanes*J (tile length; must be a power of two)                    */
/*   NT    = ceil(n/T) tiles, P2 = smallest power of two >= max(NT, p2_min)   */
/*   x~_i  = x_i for i < n, +0 otherwise (the paper's masked tail) */
/*   y[tau*T + l*J + j] = x~[tau*T + j*lanes + l]   (lane l of tile tau holds  */
/*                        the strided subsequence, as lanes do in Z)*/
/*   result = R_H(P2*T, y)  -- Listing 1 over y.  On a power-of-two length the */
/*            ceil split is exact halving, so this is the balanced tree.      */
/*                                                                           */
/* Listing 1 splits a power-of-two length at tile boundaries first, so R_H   */
/* over y equals R_H over the P2 tile values, each tile value being R_H over  */
/* its own T entries of y.  We evaluate it in that (identical) way to avoid  */
/* materialising y for 2^30-element inputs.  A tile made only of padding has */
/* value +0 (v1_hypot(+0,+0) = +0, pinned in tests), so it is not evaluated.  */
/* ------------------------------------------------------------------------- */
static int64_t pow2_ceil(int64_t v)
{
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

/* Tile value tau of x (length n): R_H over the transposed, zero-padded tile. */
double oracle_tile_d(const double *x, int64_t n, int64_t lanes, int64_t J,
                     int64_t tau, double *scratch /* T entries */)
{
    const int64_t T = lanes * J;
    for (int64_t l = 0; l < lanes; ++l)
        for (int64_t j = 0; j < J; ++j) {
            const int64_t i = tau * T + j * lanes + l;
            scratch[l * J + j] = (i < n) ? x[i] : 0.0;
        }
    return oracle_R_H_d(T, scratch);
}

float oracle_tile_s(const float *x, int64_t n, int64_t lanes, int64_t J,
                    int64_t tau, float *scratch)
{
    const int64_t T = lanes * J;
    for (int64_t l = 0; l < lanes; ++l)
        for (int64_t j = 0; j < J; ++j) {
            const int64_t i = tau * T + j * lanes + l;
            scratch[l * J + j] = (i < n) ? x[i] : 0.0f;
        }
    return oracle_R_H_s(T, scratch);
}

/* Tree over n elements padded to P2 = pow2_ceil(max(ceil(n/T), p2_min))     */
/* tiles.  p2_min = 1 gives the canonical tree; a larger p2_min evaluates the */
/* same tree as an aligned subtree of a bigger one (used by the shard tests). */
/* Returns -1 status through *ok = 0 on allocation failure.                   */
double oracle_nrmf_tree_d(const double *x, int64_t n, int64_t lanes, int64_t J,
                          int64_t p2_min, int top_cr, int *ok)
{
    *ok = 1;
    if (n == 0 && p2_min <= 1) return 0.0;               /* n = 0 -> +0 (R5) */
    const int64_t T = lanes * J;
    const int64_t NT = (n + T - 1) / T;
    const int64_t P2 = pow2_ceil(NT > p2_min ? NT : p2_min);
    double *tiles = (double *)calloc((size_t)P2, sizeof(double));
    double *scratch = (double *)malloc((size_t)T * sizeof(double));
    if (!tiles || !scratch) { free(tiles); free(scratch); *ok = 0; return 0.0; }
    for (int64_t tau = 0; tau < NT; ++tau)
        tiles[tau] = oracle_tile_d(x, n, lanes, J, tau, scratch);
    /* top levels (above the tiles): v1_hypot, or cr_hypot for the A-style
       final reduction (R1 / SURVEY f1) */
    const double r = top_cr ? oracle_R_A_d(P2, tiles) : oracle_R_H_d(P2, tiles);
    free(tiles); free(scratch);
    return r;
}

float oracle_nrmf_tree_s(const float *x, int64_t n, int64_t lanes, int64_t J,
                         int64_t p2_min, int top_cr, int *ok)
{
    *ok = 1;
    if (n == 0 && p2_min <= 1) return 0.0f;
    const int64_t T = lanes * J;
    const int64_t NT = (n + T - 1) / T;
    const int64_t P2 = pow2_ceil(NT > p2_min ? NT : p2_min);
    float *tiles = (float *)calloc((size_t)P2, sizeof(float));
    float *scratch = (float *)malloc((size_t)T * sizeof(float));
    if (!tiles || !scratch) { free(tiles); free(scratch); *ok = 0; return 0.0f; }
    for (int64_t tau = 0; tau < NT; ++tau)
        tiles[tau] = oracle_tile_s(x, n, lanes, J, tau, scratch);
    const float r = top_cr ? oracle_R_A_s(P2, tiles) : oracle_R_H_s(P2, tiles);
    free(tiles); free(scratch);
    return r;
}

/* All tile values (for sampled parity at full size): out[k] = tile tau0+k.  */
int oracle_tiles_d(const double *x, int64_t n, int64_t lanes, int64_t J,
                   int64_t tau0, int64_t count, double *out)
{
    double *scratch = (double *)malloc((size_t)(lanes * J) * sizeof(double));
    if (!scratch) return 0;
    for (int64_t k = 0; k < count; ++k)
        out[k] = oracle_tile_d(x, n, lanes, J, tau0 + k, scratch);
    free(scratch);
    return 1;
}

int oracle_tiles_s(const float *x, int64_t n, int64_t lanes, int64_t J,
                   int64_t tau0, int64_t count, float *out)
{
    float *scratch = (float *)malloc((size_t)(lanes * J) * sizeof(float));
    if (!scratch) return 0;
    for (int64_t k = 0; k < count; ++k)
        out[k] = oracle_tile_s(x, n, lanes, J, tau0 + k, scratch);
    free(scratch);
    return 1;
}

/* ------------------------------------------------------------------------- */
/* 4. Columns (e:F).  Column j (at A + j*ld, r rows) gets the tree   */
/*    of a length-r vector; frob = R_H over the c column norms padded with +0 */
/*    to a power of two.                                                      */
/* ------------------------------------------------------------------------- */
int oracle_nrmf_cols_d(int64_t r, int64_t c, int64_t ld, const double *A,
                       int64_t lanes, int64_t J, int top_cr, double *col_norms, double *frob)
{
    int ok = 1;
    for (int64_t j = 0; j < c; ++j) {
        col_norms[j] = oracle_nrmf_tree_d(A + j * ld, r, lanes, J, 1, top_cr, &ok);
        if (!ok) return 0;
    }
    if (frob) {
        if (c == 0) { *frob = 0.0; return 1; }
        const int64_t P = pow2_ceil(c);
        double *v = (double *)calloc((size_t)P, sizeof(double));
        if (!v) return 0;
        memcpy(v, col_norms, (size_t)c * sizeof(double));
        *frob = top_cr ? oracle_R_A_d(P, v) : oracle_R_H_d(P, v);
        free(v);
    }
    return 1;
}

int oracle_nrmf_cols_s(int64_t r, int64_t c, int64_t ld, const float *A,
                       int64_t lanes, int64_t J, int top_cr, float *col_norms, float *frob)
{
    int ok = 1;
    for (int64_t j = 0; j < c; ++j) {
        col_norms[j] = oracle_nrmf_tree_s(A + j * ld, r, lanes, J, 1, top_cr, &ok);
        if (!ok) return 0;
    }
    if (frob) {
        if (c == 0) { *frob = 0.0f; return 1; }
        const int64_t P = pow2_ceil(c);
        float *v = (float *)calloc((size_t)P, sizeof(float));
        if (!v) return 0;
        memcpy(v, col_norms, (size_t)c * sizeof(float));
        *frob = top_cr ? oracle_R_A_s(P, v) : oracle_R_H_s(P, v);
        free(v);
    }
    return 1;
}

/* ------------------------------------------------------------------------- */
/* 5. Exact reference ||x||'_F = RN(sqrt(sum_i x_i^2))  (e:relerr  */
/*    P:737-743), computed exactly.                                          */
/*                                                                           */
/* Every finite x is M*2^E with M an integer (< 2^53, resp. 2^24) and        */
/* E >= Emin (-1074, resp. -149).  x^2 = M^2 * 2^(2E) is an integer multiple  */
/* of 2^(2*Emin), so sum x_i^2 = S * 2^(2*Emin) with S a non-negative integer */
/* held exactly in a little-endian array of 64-bit words.  sqrt(S*2^(2Emin))  */
/* = sqrt(S) * 2^Emin, rounded to nearest-even with an integer square root    */
/* of S scaled by an even power of two plus a sticky bit.                     */
/* Non-finite input: NaN if any NaN, else +inf if any inf.                    */
/* ------------------------------------------------------------------------- */
#define ACC_WORDS_D 70   /* 4480 bits >= 2048 + 2148 + 31 headroom + carry */
#define ACC_WORDS_S 12   /*  768 bits >=  256 +  298 + 31 headroom + carry */

typedef unsigned __int128 u128;

static void acc_add_shifted(uint64_t *acc, int words, u128 v, int shift)
{
    int w = shift >> 6, o = shift & 63;
    uint64_t parts[3];
    parts[0] = (uint64_t)(v << o);
    parts[1] = (uint64_t)((o ? (v >> (64 - o)) : (v >> 64)) & 0xFFFFFFFFFFFFFFFFULL);
    parts[2] = o ? (uint64_t)(v >> (128 - o)) : 0;
    /* v < 2^106 so parts fit; propagate the carry through higher words. */
    uint64_t carry = 0;
    for (int k = 0; k < 3 || carry; ++k) {
        if (w + k >= words) break;   /* cannot happen with the headroom above */
        uint64_t add = (k < 3) ? parts[k] : 0;
        u128 s = (u128)acc[w + k] + add + carry;
        acc[w + k] = (uint64_t)s;
        carry = (uint64_t)(s >> 64);
    }
}

static int acc_bitlen(const uint64_t *acc, int words)
{
    for (int k = words - 1; k >= 0; --k)
        if (acc[k]) return 64 * k + (64 - __builtin_clzll(acc[k]));
    return 0;
}

/* bits [lo, lo+128) of acc as a u128 (bits beyond the array read as 0). */
static u128 acc_bits(const uint64_t *acc, int words, int lo)
{
    u128 r = 0;
    for (int b = 0; b < 128; ++b) {
        int bit = lo + b;
        if (bit < 0) continue;
        int w = bit >> 6;
        if (w >= words) break;
        if ((acc[w] >> (bit & 63)) & 1) r |= ((u128)1) << b;
    }
    return r;
}

static int acc_any_below(const uint64_t *acc, int words, int lo)
{
    for (int bit = 0; bit < lo; ++bit) {
        int w = bit >> 6;
        if (w >= words) break;
        if ((acc[w] >> (bit & 63)) & 1) return 1;
    }
    return 0;
}

static u128 isqrt128(u128 v)   /* floor(sqrt(v)), bit by bit */
{
    u128 res = 0, bit = ((u128)1) << 126;
    while (bit > v) bit >>= 2;
    while (bit) {
        if (v >= res + bit) { v -= res + bit; res = (res >> 1) + bit; }
        else res >>= 1;
        bit >>= 2;
    }
    return res;
}

/* RN(sqrt(S) * 2^emin) to a binary format with `prec` significand bits,    */
/* smallest quantum 2^emin and overflow threshold 2^emax_plus1.               */
static double round_sqrt_acc(const uint64_t *acc, int words, int emin, int prec,
                             int emax_plus1, int *is_inf)
{
    *is_inf = 0;
    const int b = acc_bitlen(acc, words);
    if (b == 0) return 0.0;
    /* Choose k (possibly negative) so that S' = S / 4^k has 114 or 115 bits; */
    /* then r = floor(sqrt(S')) = floor(sqrt(S) / 2^k) has 57 or 58 bits.    */
    int k = 0;
    while (b - 2 * k > 115) ++k;
    while (b - 2 * k < 114) --k;
    u128 Sp;
    int sticky;
    if (k >= 0) {
        Sp = acc_bits(acc, words, 2 * k);           /* floor(S / 4^k) */
        sticky = acc_any_below(acc, words, 2 * k);  /* S / 4^k not an integer */
    } else {
        Sp = acc_bits(acc, words, 0) << (-2 * k);   /* b < 114: fits */
        sticky = 0;
    }
    const u128 r = isqrt128(Sp);
    if (r * r != Sp) sticky = 1;
    /* sqrt(S) * 2^emin = (r + f) * 2^(k + emin), f in [0,1), f > 0 iff sticky */
    int rb = 0;
    for (u128 t = r; t; t >>= 1) ++rb;
    const int e = rb - 1 + k + emin;               /* value in [2^e, 2^(e+1)) */
    int qe = e - (prec - 1);                       /* quantum of the result */
    if (qe < emin) qe = emin;                      /* subnormal range */
    const int d = qe - (k + emin);                 /* bits of r below the quantum */
    u128 mant = r >> d;
    const int guard = (int)((r >> (d - 1)) & 1);
    const u128 rest_mask = (((u128)1) << (d - 1)) - 1;
    const int rest = ((r & rest_mask) != 0) || sticky;
    if (guard && (rest || (mant & 1))) mant += 1;  /* round half to even */
    int mb = 0;
    for (u128 t = mant; t; t >>= 1) ++mb;
    if (mb + qe > emax_plus1) { *is_inf = 1; return INFINITY; }
    return ldexp((double)(uint64_t)mant, qe);      /* exact: mant <= 2^prec */
}

/* Accumulate sum x_i^2 of x[0..n) into acc (ACC_WORDS_D words, exact);
 * flags |= 1 for a NaN, |= 2 for an infinity.  Exact integer addition is
 * associative, so disjoint chunks may be accumulated separately and their
 * accumulators added (used to spread large inputs over host threads).      */
void exact_acc_d(const double *x, int64_t n, uint64_t *acc, int *flags)
{
    for (int64_t i = 0; i < n; ++i) {
        uint64_t u;
        memcpy(&u, &x[i], 8);
        const int ef = (int)((u >> 52) & 0x7FF);
        const uint64_t fr = u & 0xFFFFFFFFFFFFFULL;
        if (ef == 0x7FF) { *flags |= fr ? 1 : 2; continue; }
        const uint64_t M = ef ? (fr | (1ULL << 52)) : fr;
        if (!M) continue;
        /* x = M * 2^E, E = ef - 1075 (normal) or -1074 (subnormal);
           x^2 = M^2 * 2^(2E) = M^2 * 2^(shift) * 2^(-2148). */
        const int E = ef ? (ef - 1075) : -1074;
        acc_add_shifted(acc, ACC_WORDS_D, (u128)M * M, 2 * E + 2148);
    }
}

void exact_acc_s(const float *x, int64_t n, uint64_t *acc, int *flags)
{
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u;
        memcpy(&u, &x[i], 4);
        const int ef = (int)((u >> 23) & 0xFF);
        const uint32_t fr = u & 0x7FFFFFu;
        if (ef == 0xFF) { *flags |= fr ? 1 : 2; continue; }
        const uint64_t M = ef ? (fr | (1u << 23)) : fr;
        if (!M) continue;
        const int E = ef ? (ef - 150) : -149;
        acc_add_shifted(acc, ACC_WORDS_S, (u128)M * M, 2 * E + 298);
    }
}

/* acc += other (both `words` long) */
void exact_acc_merge(uint64_t *acc, const uint64_t *other, int words)
{
    uint64_t carry = 0;
    for (int k = 0; k < words; ++k) {
        u128 s = (u128)acc[k] + other[k] + carry;
        acc[k] = (uint64_t)s;
        carry = (uint64_t)(s >> 64);
    }
}

double exact_round_d(const uint64_t *acc, int flags)
{
    if (flags & 1) return NAN;
    if (flags & 2) return INFINITY;
    int inf;
    return round_sqrt_acc(acc, ACC_WORDS_D, -1074, 53, 1024, &inf);
}

float exact_round_s(const uint64_t *acc, int flags)
{
    if (flags & 1) return NAN;
    if (flags & 2) return INFINITY;
    int inf;
    double r = round_sqrt_acc(acc, ACC_WORDS_S, -149, 24, 128, &inf);
    return inf ? INFINITY : (float)r;   /* r is already a float value: exact */
}

int exact_acc_words_d(void) { return ACC_WORDS_D; }
int exact_acc_words_s(void) { return ACC_WORDS_S; }

double exact_nrm_d(const double *x, int64_t n)
{
    uint64_t acc[ACC_WORDS_D];
    memset(acc, 0, sizeof acc);
    int flags = 0;
    exact_acc_d(x, n, acc, &flags);
    return exact_round_d(acc, flags);
}

float exact_nrm_s(const float *x, int64_t n)
{
    uint64_t acc[ACC_WORDS_S];
    memset(acc, 0, sizeof acc);
    int flags = 0;
    exact_acc_s(x, n, acc, &flags);
    return exact_round_s(acc, flags);
}
