/*
 * nrmf_inputs/gen.c -- seeded, counter-based, index-addressable input
 * generators shared by the tests, the bench and the oracle runs.
 *
 * This module holds NO arithmetic of the method (no hypot, no tree, no norm):
 * it only turns (seed, stream, index) into input values, so that the oracle,
 * one GPU and every rank of a sharded run see identical bits for element i no
 * matter how the array is split ("input recipe").
 *
 * Base draw: k(i) = SplitMix64 finaliser of (key + (i+1) * golden), with
 * key = SplitMix64 finaliser of (seed ^ (stream * golden)).  All conversions
 * below are exact (integer -> float with <= 53 / 24 significant bits, and
 * ldexp by in-range powers of two) except the Box-Muller normal, which uses
 * the host libm (log, cos, sqrt); normals are therefore generated on the host
 * only, and every rank of a sharded run generates its own shard with the same
 * code on the same image.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared -o nrmf_inputs/libnrmf_gen.so gen.c -lm
 */
#include <math.h>
#include <stdint.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t gen_key(uint64_t seed, uint64_t stream)
{
    return mix64(seed ^ (stream * GOLDEN) ^ 0x5DEECE66DULL);
}

static inline uint64_t draw(uint64_t key, uint64_t i)
{
    return mix64(key + (i + 1) * GOLDEN);
}

/* raw 64-bit draws (used by tests to check the distributions / indexing) */
void gen_u64(uint64_t seed, uint64_t stream, int64_t off, int64_t cnt, uint64_t *out)
{
    const uint64_t key = gen_key(seed, stream);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) out[i] = draw(key, (uint64_t)(off + i));
}

/* C1: fp64 uniform in [-1, 1): (k >> 11) * 2^-52 - 1, exact. */
void gen_uniform_pm1_d(uint64_t seed, int64_t off, int64_t cnt, double *out)
{
    const uint64_t key = gen_key(seed, 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        const uint64_t k = draw(key, (uint64_t)(off + i));
        out[i] = ldexp((double)(k >> 11), -52) - 1.0;
    }
}

/* fp32 uniform in [-1, 1): (k >> 40) * 2^-23 - 1, exact. */
void gen_uniform_pm1_s(uint64_t seed, int64_t off, int64_t cnt, float *out)
{
    const uint64_t key = gen_key(seed, 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        const uint64_t k = draw(key, (uint64_t)(off + i));
        out[i] = ldexpf((float)(k >> 40), -23) - 1.0f;
    }
}

/* C2: fp32 x = s * m * 2^e, s = +-1 (bit 0), m = 1 + f * 2^-23 with f the 23
 * bits above bit 0, e uniform integer in [elo, ehi] from the top 32 bits.   */
void gen_sme_s(uint64_t seed, int64_t off, int64_t cnt, int elo, int ehi, float *out)
{
    const uint64_t key = gen_key(seed, 2);
    const uint64_t span = (uint64_t)(ehi - elo + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        const uint64_t k = draw(key, (uint64_t)(off + i));
        const float m = 1.0f + ldexpf((float)((k >> 1) & 0x7FFFFFu), -23);
        const int e = elo + (int)(((k >> 32) * span) >> 32);
        const float v = ldexpf(m, e);
        out[i] = (k & 1) ? -v : v;
    }
}

/* fp64 variant of C2 (same recipe, 52-bit mantissa). */
void gen_sme_d(uint64_t seed, int64_t off, int64_t cnt, int elo, int ehi, double *out)
{
    const uint64_t key = gen_key(seed, 2);
    const uint64_t span = (uint64_t)(ehi - elo + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        const uint64_t k = draw(key, (uint64_t)(off + i));
        const uint64_t k2 = draw(key ^ GOLDEN, (uint64_t)(off + i));
        const double m = 1.0 + ldexp((double)(k2 >> 12), -52);
        const int e = elo + (int)(((k >> 32) * span) >> 32);
        const double v = ldexp(m, e);
        out[i] = (k & 1) ? -v : v;
    }
}

/* C3: standard normal by Box-Muller on the host: element i uses draws 2i and
 * 2i+1: u1 = ((k0 >> 11) + 1) * 2^-53 in (0,1], u2 = (k1 >> 11) * 2^-53,
 * z = sqrt(-2 ln u1) * cos(2 pi u2).                                         */
static inline double normal_at(uint64_t key, uint64_t i)
{
    const uint64_t k0 = draw(key, 2 * i), k1 = draw(key, 2 * i + 1);
    const double u1 = ldexp((double)((k0 >> 11) + 1), -53);
    const double u2 = ldexp((double)(k1 >> 11), -53);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void gen_normal_d(uint64_t seed, int64_t off, int64_t cnt, double *out)
{
    const uint64_t key = gen_key(seed, 3);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) out[i] = normal_at(key, (uint64_t)(off + i));
}

void gen_normal_s(uint64_t seed, int64_t off, int64_t cnt, float *out)
{
    const uint64_t key = gen_key(seed, 3);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) out[i] = (float)normal_at(key, (uint64_t)(off + i));
}

/* C4: column-major r x c (leading dimension ld >= r), A_ij = z_ij * 2^k_j with
 * z_ij the normal at linear index j*r + i (independent of ld) and k_j uniform
 * integer in [klo, khi] from a separate stream.  Columns [c0, c0+cc) only;
 * out points at column c0.  Entries i in [r, ld) are left untouched.         */
void gen_colscaled_normal_d(uint64_t seed, int64_t r, int64_t ld, int64_t c0, int64_t cc,
                            int klo, int khi, double *out)
{
    const uint64_t key = gen_key(seed, 3);
    const uint64_t kkey = gen_key(seed, 4);
    const uint64_t span = (uint64_t)(khi - klo + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t jj = 0; jj < cc; ++jj) {
        const int64_t j = c0 + jj;
        const int kj = klo + (int)(((draw(kkey, (uint64_t)j) >> 32) * span) >> 32);
        for (int64_t i = 0; i < r; ++i)
            out[jj * ld + i] = ldexp(normal_at(key, (uint64_t)(j * r + i)), kj);
    }
}

void gen_colscaled_normal_s(uint64_t seed, int64_t r, int64_t ld, int64_t c0, int64_t cc,
                            int klo, int khi, float *out)
{
    const uint64_t key = gen_key(seed, 3);
    const uint64_t kkey = gen_key(seed, 4);
    const uint64_t span = (uint64_t)(khi - klo + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t jj = 0; jj < cc; ++jj) {
        const int64_t j = c0 + jj;
        const int kj = klo + (int)(((draw(kkey, (uint64_t)j) >> 32) * span) >> 32);
        for (int64_t i = 0; i < r; ++i)
            out[jj * ld + i] = ldexpf((float)normal_at(key, (uint64_t)(j * r + i)), kj);
    }
}

/* C5: extreme range fp64.  Unbiased exponent E uniform integer in
 * [-1074, emax]; for E >= -1022 the value is (1 + f*2^-52) * 2^E with 52
 * random fraction bits f; for E < -1022 it is a subnormal in [2^E, 2^(E+1))
 * (leading bit at 2^E, random bits below it down to 2^-1074).  Random sign.
 * Magnitudes above vmax are replaced by vmax (the "up to 0.99*DBL_MAX" cap).
 * plant_index >= 0 puts +-vmax at that index (E-fin reading, R9).  */
void gen_extreme_d(uint64_t seed, int64_t off, int64_t cnt, int emax, double vmax,
                   int64_t plant_index, double *out)
{
    const uint64_t key = gen_key(seed, 5);
    const uint64_t span = (uint64_t)(emax + 1074 + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        const uint64_t gi = (uint64_t)(off + i);
        const uint64_t k = draw(key, gi);
        const uint64_t k2 = draw(key ^ GOLDEN, gi);
        const int E = -1074 + (int)(((k >> 32) * span) >> 32);
        double v;
        if (E >= -1022) {
            v = ldexp(1.0 + ldexp((double)(k2 >> 12), -52), E);
        } else {
            /* bits below the leading one: positions -1074 .. E-1 */
            const int nb = E + 1074;                  /* 0..51 */
            const uint64_t frac = nb ? ((k2 >> 12) >> (52 - nb)) : 0;
            v = ldexp((double)((1ULL << nb) | frac), -1074);
        }
        if (v > vmax) v = vmax;
        if ((int64_t)gi == plant_index) v = vmax;
        out[i] = (k & 1) ? -v : v;
    }
}
