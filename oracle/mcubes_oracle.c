/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this; the product never does.
 *
 * A plain-C restatement of the reference m-Cubes iteration, written from the
 * reference's algorithm (file:line citations are relative to
 * /root/reference/proj/include/mcubes/).  It is pinned bit for bit against the
 * compiled reference (oracle/_ref/libmcubes_ref.so, built from the reference's
 * own headers) and the reference's golden vectors by tests/test_oracle.py.
 * Must be compiled with -ffp-contract=off (the reference's
 * CMakeLists.txt:14-19 flag), otherwise FMA contraction changes the bits.
 *
 * Exact sums use the same exchange format as the GPU path
 * (include/mcubes_b200.h, "superaccumulator words"): MCB_XWORDS unsigned 64-bit
 * words per accumulator, word w holding an unnormalised sum of radix-2^32
 * digits of weight 2^(32 w - 1074).  This is a different representation from
 * the reference's 34-limb ExactSum (exact_sum.hpp:98-150) but denotes the same
 * exact integer, so RN() of it is the same double.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#define XW 67 /* words per accumulator: 2098 value bits + carry headroom */

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ---------------- keyed RNG: rng.hpp:26-68 ---------------- */
static const uint64_t kGamma = 0x9e3779b97f4a7c15ull;
static inline uint64_t avalanche(uint64_t z) { /* rng.hpp:29-33 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline uint64_t feed(uint64_t h, uint64_t v) { return avalanche(h + kGamma + v); } /* :37-39 */
static inline double to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }   /* :41-43 */
uint64_t orc_iteration_root(uint64_t seed, uint64_t it) { return feed(feed(0, seed), it); } /* :47-50 */
double orc_uniform01(uint64_t seed, uint64_t it, uint64_t cube, uint64_t k, uint64_t axis) { /* :63-68 */
  return to_unit(feed(feed(feed(orc_iteration_root(seed, it), cube), k), axis));
}

/* ---------------- exact accumulation (exact_sum.hpp semantics) ---------------- */
typedef struct { uint64_t w[XW]; } xacc;

/* add |v| (finite, v != 0 allowed) as radix-2^32 digits; no carries needed
 * while fewer than 2^32 addends touch a word. */
static inline void xacc_add_mag(xacc* a, double v) {
  uint64_t bits;
  memcpy(&bits, &v, 8);
  bits &= 0x7fffffffffffffffull;
  if (!bits) return;
  const uint32_t be = (uint32_t)(bits >> 52);
  const uint64_t mant = (bits & 0xfffffffffffffull) | (be ? (1ull << 52) : 0);
  const uint32_t pos = be ? be - 1 : 0; /* exact_sum.hpp:108-110 */
  const uint32_t w = pos >> 5, off = pos & 31;
  const unsigned __int128 sh = (unsigned __int128)mant << off;
  a->w[w] += (uint32_t)sh;
  a->w[w + 1] += (uint32_t)(sh >> 32);
  a->w[w + 2] += (uint32_t)(sh >> 64);
}
static void xacc_merge(xacc* a, const xacc* b) {
  for (int i = 0; i < XW; ++i) a->w[i] += b->w[i];
}

/* normalise words into 32-bit digits (little endian), returns digits */
static void normalise(const uint64_t* w, uint32_t* dig) {
  unsigned __int128 c = 0;
  for (int i = 0; i < XW; ++i) {
    c += w[i];
    dig[i] = (uint32_t)c;
    c >>= 32;
  }
}

/* RN-even of the exact integer (pos - neg) * 2^-1074: exact_sum.hpp:67-109 */
static double round_digits(uint32_t* mag, int neg) {
  int top = -1;
  for (int i = XW - 1; i >= 0; --i)
    if (mag[i]) { top = 32 * i + 31 - __builtin_clz(mag[i]); break; }
  if (top < 0) return 0.0;
#define BIT(p) ((mag[(p) >> 5] >> ((p) & 31)) & 1u)
  if (top <= 52) {
    uint64_t v = (uint64_t)mag[0] | ((uint64_t)mag[1] << 32);
    double r = ldexp((double)v, -1074);
    return neg ? -r : r;
  }
  uint64_t mant = 0;
  for (int p = top; p >= top - 52; --p) mant = (mant << 1) | BIT(p);
  const int gpos = top - 53;
  const int guard = BIT(gpos);
  int sticky = 0;
  for (int p = gpos - 1; p >= 0 && !sticky; --p) sticky = BIT(p);
#undef BIT
  int e = top - 52 - 1074;
  if (guard && (sticky || (mant & 1))) {
    if (++mant == (1ull << 53)) { mant >>= 1; ++e; }
  }
  double r = ldexp((double)mant, e);
  return neg ? -r : r;
}

/* value of pos - neg, both given as unnormalised words */
double orc_words_value(const uint64_t* pos, const uint64_t* neg) {
  uint32_t a[XW], b[XW];
  normalise(pos, a);
  if (neg) normalise(neg, b); else memset(b, 0, sizeof b);
  int cmp = 0;
  for (int i = XW - 1; i >= 0 && !cmp; --i) cmp = a[i] < b[i] ? -1 : (a[i] > b[i] ? 1 : 0);
  uint32_t* big = cmp >= 0 ? a : b;
  uint32_t* small = cmp >= 0 ? b : a;
  int64_t br = 0;
  for (int i = 0; i < XW; ++i) {
    int64_t d = (int64_t)big[i] - small[i] - br;
    br = d < 0;
    big[i] = (uint32_t)(d + (br ? (1ll << 32) : 0));
  }
  return round_digits(big, cmp < 0);
}

double orc_exact_sum(const double* v, uint64_t n) {
  xacc p, q;
  memset(&p, 0, sizeof p);
  memset(&q, 0, sizeof q);
  for (uint64_t i = 0; i < n; ++i) {
    if (!isfinite(v[i])) return NAN; /* exact_sum.hpp:104 throws */
    if (v[i] < 0) xacc_add_mag(&q, v[i]); else xacc_add_mag(&p, v[i]);
  }
  return orc_words_value(p.w, q.w);
}

/* ---------------- integrands: integrands.hpp:107-215 ---------------- */
typedef struct {
  int id;
  uint32_t d;
  const double* params;
  uint32_t nparams;
  double fb_norm;
} orc_fn;

static double eval_fn(const orc_fn* f, const double* x) {
  const uint32_t d = f->d;
  double s, prod;
  switch (f->id) {
    case 1: /* :119-126 */
      s = 0.0;
      for (uint32_t i = 0; i < d; ++i) s += (double)(i + 1) * x[i];
      return cos(s);
    case 2: /* :127-136 */
      prod = 1.0;
      for (uint32_t i = 0; i < d; ++i) {
        const double t = x[i] - 0.5;
        prod *= 1.0 / (1.0 / 2500.0 + t * t);
      }
      return prod;
    case 3: /* :137-144 */
      s = 1.0;
      for (uint32_t i = 0; i < d; ++i) s += (double)(i + 1) * x[i];
      return pow(s, -(double)d - 1.0);
    case 4: /* :145-154 */
      s = 0.0;
      for (uint32_t i = 0; i < d; ++i) {
        const double t = x[i] - 0.5;
        s += t * t;
      }
      return exp(-625.0 * s);
    case 5: /* :155-161 */
      s = 0.0;
      for (uint32_t i = 0; i < d; ++i) s += fabs(x[i] - 0.5);
      return exp(-10.0 * s);
    case 6: /* :162-172 */
      s = 0.0;
      for (uint32_t i = 0; i < d; ++i) {
        const double bound = (3.0 + (double)(i + 1)) / 10.0;
        if (!(x[i] < bound)) return 0.0;
        s += ((double)(i + 1) + 4.0) * x[i];
      }
      return exp(s);
    case 7: /* fA :181-196 */
      s = 0.0;
      for (uint32_t i = 0; i < d; ++i) s += x[i];
      return sin(s);
    case 8: /* fB :200-215 */
      s = 0.0;
      for (uint32_t i = 0; i < d; ++i) s += x[i] * x[i];
      return f->fb_norm * exp(-s / (2.0 * 0.01));
    case 9: { /* table integrand (BASELINE config 4; CPU twin, see include/mcubes_b200.h) */
      const uint32_t n = (uint32_t)f->params[0];
      const double* lo = f->params + 1;
      const double* inv_h = f->params + 1 + d;
      const double* tab = f->params + 1 + 2 * d;
      prod = 1.0;
      for (uint32_t j = 0; j < d; ++j) {
        const double t = (x[j] - lo[j]) * inv_h[j];
        uint32_t k = 0;
        if (t >= (double)(n - 1)) k = n - 2;
        else if (t > 0.0) k = (uint32_t)t;
        if (k > n - 2) k = n - 2;
        const double* row = tab + (size_t)j * n;
        const double frac = t - (double)k;
        prod *= row[k] + frac * (row[k + 1] - row[k]);
      }
      return prod;
    }
    case 32: return x[0];
    case 33: return f->nparams ? f->params[0] : 0.0;
    case 34: return x[0] * x[0] + 0.5;
    case 35: return x[0] > 0.0 ? INFINITY : 1.0;
    case 36: return INFINITY;
    case 37: return 0.0;
    case 38: {  /* inf_near_origin: +inf if every x_j < c (a failure inside one corner cube) */
      const double c = f->nparams ? f->params[0] : 0.0;
      for (uint32_t j = 0; j < d; ++j)
        if (!(x[j] < c)) return 1.0;
      return INFINITY;
    }
  }
  return NAN;
}

static int make_fn(orc_fn* f, int id, const double* params, uint32_t nparams, uint32_t d) {
  f->id = id;
  f->d = d;
  f->params = params;
  f->nparams = nparams;
  f->fb_norm = pow(2.0 * 3.141592653589793 * 0.01, -4.5); /* integrands.hpp:207 */
  if ((id >= 1 && id <= 9) || (id >= 32 && id <= 37)) {
    if (id == 9) {
      if (nparams < 1) return fail(-1, "table integrand needs params");
      const uint32_t n = (uint32_t)params[0];
      if (n < 2 || nparams != 1 + 2 * d + (size_t)n * d) return fail(-1, "table integrand: bad params");
    }
    return 0;
  }
  return fail(-1, "unknown integrand id");
}

int orc_eval(int id, const double* params, uint32_t nparams, uint32_t d, const double* x, double* out) {
  orc_fn f;
  int rc = make_fn(&f, id, params, nparams, d);
  if (rc) return rc;
  *out = eval_fn(&f, x);
  return 0;
}

/* ---------------- grid: grid.hpp:30-50, 61-67, 204-224, 232-297 ---------------- */
typedef struct {
  uint32_t d, nb;
  const double* lower;
  const double* upper;
  const double* edges; /* d x nb row-major right edges (grid.hpp:303) */
} orc_grid;

void orc_grid_uniform(uint32_t d, uint32_t nb, const double* lower, const double* upper, double* edges) {
  for (uint32_t j = 0; j < d; ++j) { /* grid.hpp:44-49 */
    double* row = edges + (size_t)j * nb;
    const double width = (upper[j] - lower[j]) / (double)nb;
    for (uint32_t i = 0; i + 1 < nb; ++i) row[i] = lower[j] + (double)(i + 1) * width;
    row[nb - 1] = upper[j];
  }
}

static inline double transform(const orc_grid* g, const double* u, double* x, uint32_t* bins) {
  double jac = 1.0; /* grid.hpp:204-224 */
  const double nbd = (double)g->nb;
  for (uint32_t j = 0; j < g->d; ++j) {
    const double z = u[j] * nbd;
    uint32_t i = 0;
    if (z >= nbd) i = g->nb - 1;
    else if (z > 0.0) i = (uint32_t)z;
    const double* row = g->edges + (size_t)j * g->nb;
    const double left = i == 0 ? g->lower[j] : row[i - 1];
    const double width = row[i] - left;
    x[j] = left + (z - (double)i) * width;
    jac *= nbd * width;
    if (bins) bins[j] = i;
  }
  return jac;
}

int orc_transform(uint32_t d, uint32_t nb, const double* lower, const double* upper,
                  const double* edges, const double* u, double* x, uint32_t* bins, double* jac) {
  orc_grid g = {d, nb, lower, upper, edges};
  *jac = transform(&g, u, x, bins);
  return 0;
}

/* grid.hpp:232-297 (adjust_axis) */
static int adjust_axis(double* edges, double lo, double hi, const double* contrib, uint32_t n,
                       double alpha) {
  int any = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (contrib[i] < 0.0 || !isfinite(contrib[i])) return fail(-1, "Grid: contributions must be finite and >= 0");
    any |= contrib[i] != 0.0;
  }
  if (!any || n == 1) return 0;
  double* smooth = malloc(sizeof(double) * n * 3);
  double* imp = smooth + n;
  double* out = smooth + 2 * n;
  smooth[0] = 0.5 * (contrib[0] + contrib[1]);
  for (uint32_t i = 1; i + 1 < n; ++i) smooth[i] = (contrib[i - 1] + contrib[i] + contrib[i + 1]) / 3.0;
  smooth[n - 1] = 0.5 * (contrib[n - 2] + contrib[n - 1]);
  double total = 0.0;
  for (uint32_t i = 0; i < n; ++i) total += smooth[i];
  double rtot = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    const double c = smooth[i] / total;
    double r = 0.0;
    if (c == 1.0) r = 1.0;
    else if (c > 0.0) r = pow((c - 1.0) / log(c), alpha);
    imp[i] = r;
    rtot += r;
  }
  const double share = rtot / (double)n;
  out[n - 1] = hi;
  double target = 0.0, cum = 0.0;
  uint32_t k = 0;
  for (uint32_t i = 0; i + 1 < n; ++i) {
    target += share;
    while (k + 1 < n && (imp[k] == 0.0 || cum + imp[k] < target)) {
      cum += imp[k];
      ++k;
    }
    const double left = k == 0 ? lo : edges[k - 1];
    const double width = edges[k] - left;
    out[i] = left + width * ((target - cum) / imp[k]);
  }
  double prev = lo;
  for (uint32_t i = 0; i + 1 < n; ++i) {
    if (!(out[i] > prev)) out[i] = nextafter(prev, INFINITY);
    prev = out[i];
  }
  double next = hi;
  for (uint32_t i = n - 1; i-- > 0;) {
    if (!(out[i] < next)) out[i] = nextafter(next, -INFINITY);
    next = out[i];
  }
  memcpy(edges, out, sizeof(double) * n);
  free(smooth);
  return 0;
}

static int valid_alpha(double a) { return a >= 0.0 && isfinite(a); }

/* grid.hpp:104-114 and 122-146 */
int orc_grid_adjust(uint32_t d, uint32_t nb, const double* lower, const double* upper,
                    const double* edges, const double* contrib, double alpha, int symmetric, double* out) {
  if (!valid_alpha(alpha)) return fail(-1, "Grid: damping exponent alpha must be finite and >= 0");
  memcpy(out, edges, sizeof(double) * d * nb);
  if (!symmetric) {
    for (uint32_t j = 0; j < d; ++j) {
      int rc = adjust_axis(out + (size_t)j * nb, lower[j], upper[j], contrib + (size_t)j * nb, nb, alpha);
      if (rc) return rc;
    }
    return 0;
  }
  int rc = adjust_axis(out, lower[0], upper[0], contrib, nb, alpha);
  if (rc) return rc;
  for (uint32_t j = 1; j < d; ++j) {
    double* row = out + (size_t)j * nb;
    if (lower[j] == lower[0] && upper[j] == upper[0]) {
      memcpy(row, out, sizeof(double) * nb);
    } else {
      const double range0 = upper[0] - lower[0];
      const double range = upper[j] - lower[j];
      for (uint32_t i = 0; i + 1 < nb; ++i) row[i] = lower[j] + ((out[i] - lower[0]) / range0) * range;
      row[nb - 1] = upper[j];
    }
  }
  return 0;
}

/* ---------------- sampling: sampler.hpp:147-197, 285-295 ---------------- */
static uint64_t exact_root(uint64_t m, uint32_t d) { /* sampler.hpp:184-197 */
  const uint64_t guess = (uint64_t)llround(pow((double)m, 1.0 / (double)d));
  for (uint64_t g = guess > 2 ? guess - 2 : 1; g <= guess + 2; ++g) {
    uint64_t acc = 1;
    int overflow = 0;
    for (uint32_t i = 0; i < d && !overflow; ++i) {
      if (acc > m / g) overflow = 1;
      else acc *= g;
    }
    if (!overflow && acc == m) return g;
  }
  return 0;
}

typedef struct {
  xacc est_pos, est_neg, var;
  xacc* bins; /* bin_axes * nb */
  uint64_t writes;
  /* first non-finite sample in cube order (the serial oracle's throw) */
  int bad;
  double bad_fx;
  double bad_x[64];
} partial;

/* Host threads of orc_sample_partial (1 = the serial loop).  Threads take
 * contiguous cube ranges and their exact partials are merged word-wise, so
 * the result is the same for any thread count (the reference's own
 * invariance, sampler.hpp:213-278); the first non-finite sample in cube order
 * is the lowest range's. */
static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

/* run_cube (sampler.hpp:147-181), accumulating straight into exact words */
static void run_cube(const orc_fn* f, const orc_grid* g, uint64_t t, uint64_t gi, uint64_t p,
                     uint64_t iter_root, double scale, uint32_t bin_axes, int kbins, partial* acc) {
  const uint32_t d = g->d;
  double digit[64], u[64], x[64];
  uint32_t bin[64];
  uint64_t tt = t;
  for (uint32_t j = 0; j < d; ++j) {
    digit[j] = (double)(tt % gi);
    tt /= gi;
  }
  const double gd = (double)gi;
  const uint64_t croot = feed(iter_root, t);
  double sum_scaled = 0.0, mean = 0.0, m2 = 0.0;
  uint64_t n = 0;
  for (uint64_t k = 0; k < p; ++k) {
    const uint64_t proot = feed(croot, k);
    for (uint32_t j = 0; j < d; ++j) u[j] = (digit[j] + to_unit(feed(proot, j))) / gd;
    const double jac = transform(g, u, x, bin);
    const double fx = eval_fn(f, x);
    const double fj = fx * jac;
    if (!isfinite(fj)) {
      if (!acc->bad) {
        acc->bad = 1;
        acc->bad_fx = fx;
        memcpy(acc->bad_x, x, sizeof(double) * d);
      }
      return;
    }
    sum_scaled += fj * scale;
    ++n; /* Welford, sampler.hpp:98-103 */
    const double dd = fj - mean;
    mean += dd / (double)n;
    m2 += dd * (fj - mean);
    if (kbins) {
      const double sq = fj * fj;
      for (uint32_t j = 0; j < bin_axes; ++j) xacc_add_mag(&acc->bins[(size_t)j * g->nb + bin[j]], sq);
      acc->writes += bin_axes;
    }
  }
  double var = m2 / ((double)p * (double)(p - 1));
  if (!(var > 0.0)) var = 0.0;
  xacc_add_mag(sum_scaled < 0 ? &acc->est_neg : &acc->est_pos, sum_scaled);
  xacc_add_mag(&acc->var, var);
}

static int g_rng = 0; /* 0 = the reference stream, 1 = the Philox path twin (r24 bins), 2 = Philox, exact bins */
void orc_set_rng(int rng) { g_rng = rng; }

/* ---------------- Philox path twin (NOT the reference) ----------------
 * The B200 north-star stream (include/mcubes_b200/sampler.cuh,
 * sample_point_fast): Philox4x32-10 keyed by the iteration root with counter
 * (cube lo, cube hi, sample, block of 4 axes), 32-bit uniforms, FMA-contracted
 * transform and Welford.  The reference has no such mode; this restatement
 * lets tests check the GPU Philox path bit for bit on integrands built from + - * and /, while
 * its agreement with the reference itself is statistical (3 combined sigma). */
static void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

static void run_cube_philox(const orc_fn* f, const orc_grid* g, uint64_t t, uint64_t gi, uint64_t p,
                            uint64_t key, double scale, uint32_t bin_axes, int kbins, partial* acc) {
  const uint32_t d = g->d, nb = g->nb;
  const double nbg = (double)nb / (double)gi, cs = nbg * 0x1.0p-32;
  double nbpow = 1.0;
  for (uint32_t j = 0; j < d; ++j) nbpow *= (double)nb;
  double base[64], x[64];
  uint64_t dig[64];
  uint32_t bin[64], r[68];
  uint64_t tt = t;
  for (uint32_t j = 0; j < d; ++j) {
    dig[j] = tt % gi;
    base[j] = (double)dig[j] * nbg;
    tt /= gi;
  }
  double sum = 0.0, mean = 0.0, m2 = 0.0;
  for (uint64_t k = 0; k < p; ++k) {
    for (uint32_t q = 0; q < (d + 3) / 4; ++q) {
      uint32_t c[4] = {(uint32_t)t, (uint32_t)(t >> 32), (uint32_t)k, q};
      philox4x32_10(c, (uint32_t)key, (uint32_t)(key >> 32));
      memcpy(r + 4 * q, c, sizeof c);
    }
    double jw = 1.0;
    for (uint32_t j = 0; j < d; ++j) {
      /* d >= 3: 32-bit digits, z = RN((digit 2^32 + r) * cs) from the exact
       * 64-bit integer; d <= 2: z = fma(r, cs, RN(digit * nb / g)) */
      const double z = d >= 3 ? (double)((dig[j] << 32) | r[j]) * cs : fma((double)r[j], cs, base[j]);
      uint32_t i = (uint32_t)z;
      if (i > nb - 1) i = nb - 1;
      const double* row = g->edges + (size_t)j * nb;
      const double left = i == 0 ? g->lower[j] : row[i - 1];
      const double w = row[i] - left;
      const double A = fma(-(double)i, w, left);
      x[j] = fma(z, w, A);
      jw = j == 0 ? w : jw * w;
      bin[j] = i;
    }
    const double fx = eval_fn(f, x);
    const double fj = fx * (jw * nbpow);
    if (!isfinite(fj)) {
      if (!acc->bad) {
        acc->bad = 1;
        acc->bad_fx = fx;
        memcpy(acc->bad_x, x, sizeof(double) * d);
      }
      return;
    }
    sum += fj;
    const double dd = fj - mean;
    const uint64_t nk = k + 1;
    mean = fma(dd, 1.0 / (double)nk, mean);
    m2 = fma(dd, fj - mean, m2);
    if (kbins) { /* (f J)^2, rounded half-up to 24 significant bits on the r24 path (exact.cuh
                  * split_r24; orc_set_rng(1)), exact with orc_set_rng(2) (philox_exact) */
      double sq = fj * fj;
      if (g_rng == 1) {
        uint64_t b;
        memcpy(&b, &sq, 8);
        b = (b + (1ull << 28)) & ~((1ull << 29) - 1);
        memcpy(&sq, &b, 8);
      }
      for (uint32_t j = 0; j < bin_axes; ++j) xacc_add_mag(&acc->bins[(size_t)j * nb + bin[j]], sq);
      acc->writes += bin_axes;
    }
  }
  sum = sum * scale;
  double var = m2 * (1.0 / ((double)p * (double)(p - 1)));
  if (!(var > 0.0)) var = 0.0;
  xacc_add_mag(sum < 0 ? &acc->est_neg : &acc->est_pos, sum);
  xacc_add_mag(&acc->var, var);
}


/* one thread's contiguous cube range [t0, t1) (sample_all_cubes' batches) */
typedef struct {
  const orc_fn* f;
  const orc_grid* g;
  uint64_t gi, p, root, t0, t1;
  double scale;
  uint32_t bin_axes;
  int kbins;
  partial acc;
} range_job;

static void* range_worker(void* arg) {
  range_job* jb = (range_job*)arg;
  for (uint64_t t = jb->t0; t < jb->t1; ++t) {
    if (g_rng) run_cube_philox(jb->f, jb->g, t, jb->gi, jb->p, jb->root, jb->scale, jb->bin_axes, jb->kbins, &jb->acc);
    else run_cube(jb->f, jb->g, t, jb->gi, jb->p, jb->root, jb->scale, jb->bin_axes, jb->kbins, &jb->acc);
    if (jb->acc.bad) break;
  }
  return NULL;
}

/* Exact partial over cubes [c0, c1) in the GPU exchange format: out_words
 * receives (3 + bin_axes*nb) accumulators of XW words:
 * [est_pos, est_neg, var, bins...].  This is what one rank contributes before
 * the cross-rank sum (tests/test_dist_gloo.py). */
int orc_sample_partial(int id, const double* params, uint32_t nparams, uint32_t d, uint32_t nb,
                       const double* lower, const double* upper, const double* edges, uint64_t m,
                       uint64_t p, uint64_t seed, uint64_t iteration, int bin_mode, int kbins,
                       uint64_t c0, uint64_t c1, uint64_t* out_words, uint64_t* writes,
                       double* err_x, double* err_fx) {
  orc_fn f;
  int rc = make_fn(&f, id, params, nparams, d);
  if (rc) return rc;
  if (m == 0) return fail(-1, "v_sample: m must be >= 1");
  if (p < 2) return fail(-1, "v_sample: p must be >= 2");
  if (d > 64) return fail(-1, "oracle supports d <= 64");
  const uint64_t gi = exact_root(m, d);
  if (!gi) return fail(-1, "v_sample: m must be a perfect d-th power of the cube count");
  const double scale = 1.0 / ((double)m * (double)p);
  const uint32_t bin_axes = bin_mode == 0 ? d : 1;
  orc_grid g = {d, nb, lower, upper, edges};
  const uint64_t iter_root = orc_iteration_root(seed, iteration);
  if (c1 > m) c1 = m;
  if (c0 > c1) c0 = c1;
  const uint64_t span = c1 - c0;
  int nth = g_threads;
  if ((uint64_t)nth > span / 64 + 1) nth = (int)(span / 64 + 1);
  range_job* jobs = calloc((size_t)nth, sizeof(range_job));
  pthread_t* tids = calloc((size_t)nth, sizeof(pthread_t));
  for (int i = 0; i < nth; ++i) {
    range_job* jb = &jobs[i];
    jb->f = &f;
    jb->g = &g;
    jb->gi = gi;
    jb->p = p;
    jb->root = iter_root;
    jb->scale = scale;
    jb->bin_axes = bin_axes;
    jb->kbins = kbins;
    jb->t0 = c0 + span * (uint64_t)i / (uint64_t)nth;
    jb->t1 = c0 + span * (uint64_t)(i + 1) / (uint64_t)nth;
    jb->acc.bins = calloc((size_t)bin_axes * nb, sizeof(xacc));
    if (nth > 1) pthread_create(&tids[i], NULL, range_worker, jb);
    else range_worker(jb);
  }
  partial acc;
  memset(&acc, 0, sizeof acc);
  acc.bins = jobs[0].acc.bins;
  for (int i = 0; i < nth; ++i) {
    if (nth > 1) pthread_join(tids[i], NULL);
    partial* q = &jobs[i].acc;
    if (q->bad && !acc.bad) {
      acc.bad = 1;
      acc.bad_fx = q->bad_fx;
      memcpy(acc.bad_x, q->bad_x, sizeof acc.bad_x);
    }
    if (i == 0) {
      acc.est_pos = q->est_pos;
      acc.est_neg = q->est_neg;
      acc.var = q->var;
      acc.writes = q->writes;
      continue;
    }
    xacc_merge(&acc.est_pos, &q->est_pos);
    xacc_merge(&acc.est_neg, &q->est_neg);
    xacc_merge(&acc.var, &q->var);
    for (size_t c = 0; c < (size_t)bin_axes * nb; ++c) xacc_merge(&acc.bins[c], &q->bins[c]);
    acc.writes += q->writes;
    free(q->bins);
  }
  free(jobs);
  free(tids);
  if (acc.bad) {
    if (err_x) memcpy(err_x, acc.bad_x, sizeof(double) * d);
    if (err_fx) *err_fx = acc.bad_fx;
    free(acc.bins);
    return fail(-2, "integrand produced non-finite value");
  }
  const size_t nacc = 3 + (size_t)bin_axes * nb;
  memset(out_words, 0, sizeof(uint64_t) * XW * nacc);
  memcpy(out_words + 0 * XW, acc.est_pos.w, sizeof acc.est_pos.w);
  memcpy(out_words + 1 * XW, acc.est_neg.w, sizeof acc.est_neg.w);
  memcpy(out_words + 2 * XW, acc.var.w, sizeof acc.var.w);
  if (kbins) memcpy(out_words + 3 * XW, acc.bins, sizeof(xacc) * bin_axes * nb);
  if (writes) *writes = acc.writes;
  free(acc.bins);
  return 0;
}

/* Round a (possibly cross-rank-summed) partial into the v_sample outputs
 * (sampler.hpp:322-332). */
int orc_round_partial(const uint64_t* words, uint32_t d, uint32_t nb, uint64_t m, int bin_mode,
                      int kbins, double* est, double* var, double* contrib) {
  *est = orc_words_value(words + 0 * XW, words + 1 * XW);
  const double md = (double)m;
  *var = orc_words_value(words + 2 * XW, NULL) / (md * md);
  if (kbins && contrib) {
    const uint32_t bin_axes = bin_mode == 0 ? d : 1;
    memset(contrib, 0, sizeof(double) * d * nb);
    for (uint32_t c = 0; c < bin_axes * nb; ++c) contrib[c] = orc_words_value(words + (3 + (size_t)c) * XW, NULL);
  }
  return 0;
}

uint32_t orc_xwords(void) { return XW; }

/* v_sample / v_sample_no_adjust / vegas_serial_iteration semantics in one:
 * sampler.hpp:312-349, oracle.hpp:21-50.  kbins=0 is the frozen iteration. */
int orc_v_sample(int id, const double* params, uint32_t nparams, uint32_t d, uint32_t nb,
                 const double* lower, const double* upper, const double* edges, uint64_t m,
                 uint64_t s, uint64_t p, uint64_t seed, uint64_t iteration, int bin_mode, int kbins,
                 double* est, double* var, double* contrib, uint64_t* writes, double* err_x,
                 double* err_fx) {
  if (s == 0) return fail(-1, "v_sample: batch size must be >= 1");
  const uint32_t bin_axes = bin_mode == 0 ? d : 1;
  const size_t nacc = 3 + (size_t)bin_axes * nb;
  uint64_t* w = malloc(sizeof(uint64_t) * XW * nacc);
  int rc = orc_sample_partial(id, params, nparams, d, nb, lower, upper, edges, m, p, seed, iteration,
                              bin_mode, kbins, 0, m, w, writes, err_x, err_fx);
  if (!rc) orc_round_partial(w, d, nb, m, bin_mode, kbins, est, var, contrib);
  free(w);
  return rc;
}

/* ---------------- driver: driver.hpp:52-123, 146-178, 215-258 ---------------- */
static int validate(uint32_t d, uint32_t nb, uint64_t maxcalls, uint32_t itmax, uint32_t ita,
                    double tau, double alpha, double chi2max, const double* lower, const double* upper) {
  if (d < 1) return fail(-1, "RunConfig: dims must be >= 1");
  if (nb < 2) return fail(-1, "RunConfig: n_bins must be >= 2");
  if (d >= 63 || maxcalls < (2ull << d)) return fail(-1, "RunConfig: maxcalls must be >= 2*2^dims");
  if (!(tau > 0.0) || !(tau < 1.0)) return fail(-1, "RunConfig: tau_rel must lie in (0, 1)");
  if (itmax < 1) return fail(-1, "RunConfig: itmax must be >= 1");
  if (ita > itmax) return fail(-1, "RunConfig: ita must not exceed itmax");
  if (!(alpha >= 0.0) || !isfinite(alpha)) return fail(-1, "RunConfig: alpha must be finite and >= 0");
  if (!(chi2max > 0.0)) return fail(-1, "RunConfig: chi2_dof_max must be positive");
  for (uint32_t j = 0; j < d; ++j)
    if (!isfinite(lower[j]) || !isfinite(upper[j]) || !(lower[j] < upper[j]))
      return fail(-1, "RunConfig: requires finite lower < upper on every axis");
  return 0;
}

static int fits(uint64_t g, uint64_t maxcalls, uint32_t d) {
  unsigned __int128 acc = 2;
  for (uint32_t i = 0; i < d; ++i) {
    acc *= g;
    if (acc > maxcalls) return 0;
  }
  return 1;
}

int orc_setup(uint32_t d, uint32_t nb, uint64_t maxcalls, uint32_t itmax, uint32_t ita, double tau,
              double alpha, double chi2max, const double* lower, const double* upper,
              unsigned workers, uint64_t* out4) {
  int rc = validate(d, nb, maxcalls, itmax, ita, tau, alpha, chi2max, lower, upper);
  if (rc) return rc;
  uint64_t g = (uint64_t)floor(pow((double)maxcalls / 2.0, 1.0 / (double)d)); /* driver.hpp:102-106 */
  if (g < 1) g = 1;
  while (!fits(g, maxcalls, d) && g > 1) --g;
  while (fits(g + 1, maxcalls, d)) ++g;
  uint64_t m = 1;
  for (uint32_t i = 0; i < d; ++i) m *= g;
  uint64_t p = maxcalls / m;
  if (p < 2) p = 2;
  if (workers == 0) workers = 1;
  const uint64_t per = (uint64_t)workers * 32; /* driver.hpp:82-87 */
  uint64_t s = (m + per - 1) / per;
  if (s < 1) s = 1;
  out4[0] = g; out4[1] = m; out4[2] = p; out4[3] = s;
  return 0;
}

int orc_weighted_estimate(uint32_t n, const double* est, const double* var, double* out3) {
  if (n == 0) return fail(-1, "weighted_estimate: history must be non-empty");
  for (uint32_t i = 0; i < n; ++i) { /* driver.hpp:149-153 */
    if (!(var[i] >= 0.0)) return fail(-1, "weighted_estimate: negative variance");
    if (var[i] == 0.0) { out3[0] = est[i]; out3[1] = 0.0; out3[2] = 0.0; return 0; }
  }
  double sum_w = 0.0, sum_wi = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    const double w = 1.0 / var[i];
    sum_w += w;
    sum_wi += w * est[i];
  }
  const double mean = sum_wi / sum_w;
  double chi2 = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    const double dd = est[i] - mean;
    chi2 += dd * dd / var[i];
  }
  const double dof = (double)(n > 1 ? n - 1 : 1);
  out3[0] = mean;
  out3[1] = 1.0 / sqrt(sum_w);
  out3[2] = chi2 / dof;
  return 0;
}

int orc_check_convergence(double est, double sigma, double chi2, double tau, double chi2max) {
  const double sc = fabs(est); /* driver.hpp:173-178 */
  const int ok = sc < 1e-300 ? sigma <= tau : sigma / sc <= tau;
  return ok && chi2 <= chi2max;
}

/* integrate (driver.hpp:215-258).  res8 = {estimate, sigma, chi2_dof,
 * iterations_used, converged, total_samples, bin_writes, 0}; sp4 = {g,m,p,s}.
 * grids_out (nullable): per iteration, the grid after that iteration's
 * adjustment (itmax*d*nb). */
int orc_integrate(int id, const double* params, uint32_t nparams, uint32_t d, uint32_t nb,
                  uint64_t maxcalls, uint32_t itmax, uint32_t ita, double tau, double alpha,
                  double chi2max, uint64_t seed, int variant, const double* lower, const double* upper,
                  double* res8, uint64_t* sp4, double* hist_est, double* hist_var, uint32_t cap,
                  double* grids_out, uint64_t* writes_out, double* err_x, double* err_fx) {
  int rc = orc_setup(d, nb, maxcalls, itmax, ita, tau, alpha, chi2max, lower, upper, 1, sp4);
  if (rc) return rc;
  const uint64_t m = sp4[1], p = sp4[2];
  double* edges = malloc(sizeof(double) * d * nb * 2);
  double* next = edges + (size_t)d * nb;
  double* contrib = malloc(sizeof(double) * d * nb);
  double* he = malloc(sizeof(double) * itmax);
  double* hv = malloc(sizeof(double) * itmax);
  orc_grid_uniform(d, nb, lower, upper, edges);
  memset(res8, 0, sizeof(double) * 8);
  const int bin_mode = variant ? 1 : 0;
  double total_samples = 0, bin_writes = 0;
  for (uint32_t it = 1; it <= itmax; ++it) {
    const int adjusting = it <= ita;
    uint64_t writes = 0;
    double est, var;
    rc = orc_v_sample(id, params, nparams, d, nb, lower, upper, edges, m, 1, p, seed, it, bin_mode,
                      adjusting, &est, &var, contrib, &writes, err_x, err_fx);
    if (rc) break;
    if (adjusting) {
      rc = orc_grid_adjust(d, nb, lower, upper, edges, contrib, alpha, variant, next);
      if (rc) break;
      memcpy(edges, next, sizeof(double) * d * nb);
    }
    he[it - 1] = est;
    hv[it - 1] = var;
    if (it - 1 < cap) { hist_est[it - 1] = est; hist_var[it - 1] = var; }
    bin_writes += (double)writes;
    total_samples += (double)(m * p);
    res8[3] = it;
    double c[3];
    rc = orc_weighted_estimate(it, he, hv, c);
    if (rc) break;
    res8[0] = c[0]; res8[1] = c[1]; res8[2] = c[2];
    if (grids_out) memcpy(grids_out + (size_t)(it - 1) * d * nb, edges, sizeof(double) * d * nb);
    if (writes_out) writes_out[it - 1] = writes;
    if (orc_check_convergence(c[0], c[1], c[2], tau, chi2max)) { res8[4] = 1.0; break; }
  }
  res8[5] = total_samples;
  res8[6] = bin_writes;
  free(edges); free(contrib); free(he); free(hv);
  return rc;
}
