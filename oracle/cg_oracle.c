/* oracle/cg_oracle.c -- TEST INFRASTRUCTURE (checker only; see cg_oracle.h).
 *
 * Plain-C FP64 restatement of the reference hot path.  Every function cites
 * the reference file:line it follows (paths under /root/reference/proj).
 * The restatement is pinned in tests/test_oracle.py against the reference
 * library itself (oracle/_ref/libcgmimo_ref.so built by oracle/Makefile) and
 * against the committed fixtures in tests/golden/.
 */
#define _GNU_SOURCE
#include "cg_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cx;

/* ------------------------------------------------------------------ RNG */
/* src/rng.cpp:12-19 */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;
static uint64_t mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t key, counter;
  int have_cached;
  double cached;
} rng_t;

static rng_t rng_make(uint64_t key) { rng_t r = {key, 0, 0, 0.0}; return r; }
/* src/rng.cpp:23-25 */
static rng_t rng_fork(const rng_t* r, uint64_t stream) {
  return rng_make(mix64(mix64(r->key ^ 0x8BB84B93962EACC9ull) + stream));
}
/* src/rng.cpp:27 */
static uint64_t rng_u64(rng_t* r) { return mix64(r->key + kGolden * ++r->counter); }
/* src/rng.cpp:29-31 */
static double rng_unit(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
/* src/rng.cpp:33-45 (Box-Muller, second variate cached) */
static double rng_gauss(rng_t* r) {
  if (r->have_cached) { r->have_cached = 0; return r->cached; }
  const double u1 = 1.0 - rng_unit(r);
  const double u2 = rng_unit(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * M_PI * u2;
  r->cached = radius * sin(angle);
  r->have_cached = 1;
  return radius * cos(angle);
}
/* src/rng.cpp:47-52 */
static cx rng_cgauss(rng_t* r, double variance) {
  const double sd = sqrt(0.5 * variance);
  const double re = rng_gauss(r);
  const double im = rng_gauss(r);
  return sd * re + I * (sd * im);
}

static rng_t rng_path(uint64_t key, const uint64_t* forks, int n_forks) {
  rng_t r = rng_make(key);
  for (int i = 0; i < n_forks; ++i) r = rng_fork(&r, forks[i]);
  return r;
}

void orc_rng_u64(uint64_t key, const uint64_t* forks, int n_forks, long n, uint64_t* out) {
  rng_t r = rng_path(key, forks, n_forks);
  for (long i = 0; i < n; ++i) out[i] = rng_u64(&r);
}

void orc_rng_cgaussian(uint64_t key, const uint64_t* forks, int n_forks, double variance,
                       long n, double* out) {
  rng_t r = rng_path(key, forks, n_forks);
  for (long i = 0; i < n; ++i) {
    const cx z = rng_cgauss(&r, variance);
    out[2 * i] = creal(z);
    out[2 * i + 1] = cimag(z);
  }
}

/* src/channel.cpp:10-17: B x U, drawn row-major */
void orc_rayleigh(uint64_t key, const uint64_t* forks, int n_forks, int B, int U, double* out) {
  rng_t r = rng_path(key, forks, n_forks);
  for (long i = 0; i < (long)B * U; ++i) {
    const cx z = rng_cgauss(&r, 1.0);
    out[2 * i] = creal(z);
    out[2 * i + 1] = cimag(z);
  }
}

/* -------------------------------------------------------- constellation */
/* src/constellation.cpp:29-34 */
static unsigned gray_decode(unsigned g) {
  unsigned m = g;
  for (unsigned s = g >> 1; s != 0; s >>= 1) m ^= s;
  return m;
}

typedef struct {
  int bits, axis_bits, per; /* per = amplitudes per subset */
  double axis0[3][4], axis1[3][4];
  cx points[64];
} constel_t;

/* src/constellation.cpp:37-86 */
static int constel_make(int bits, constel_t* c) {
  if (bits != 2 && bits != 4 && bits != 6) return 2;
  const int half = bits / 2;
  const unsigned levels = 1u << half, count = 1u << bits;
  const double axis_power = ((double)levels * levels - 1.0) / 3.0;
  const double scale = 1.0 / sqrt(2.0 * axis_power);
  c->bits = bits;
  c->axis_bits = half;
  c->per = (int)levels / 2;
  for (unsigned label = 0; label < count; ++label) {
    const unsigned gi = label >> half, gq = label & (levels - 1);
    const double ai = 2.0 * gray_decode(gi) - (levels - 1.0);
    const double aq = 2.0 * gray_decode(gq) - (levels - 1.0);
    c->points[label] = ai * scale + I * (aq * scale);
  }
  int n0[3] = {0, 0, 0}, n1[3] = {0, 0, 0};
  for (unsigned g = 0; g < levels; ++g) {
    const double amp = (2.0 * gray_decode(g) - (levels - 1.0)) * scale;
    for (int p = 0; p < half; ++p) {
      if ((g >> (half - 1 - p)) & 1u) c->axis1[p][n1[p]++] = amp;
      else c->axis0[p][n0[p]++] = amp;
    }
  }
  return 0;
}

int orc_constellation(int qam_bits, double* points, double* axis0, double* axis1) {
  constel_t c;
  if (constel_make(qam_bits, &c)) return 2;
  for (int l = 0; l < (1 << qam_bits); ++l) {
    points[2 * l] = creal(c.points[l]);
    points[2 * l + 1] = cimag(c.points[l]);
  }
  for (int p = 0; p < c.axis_bits; ++p)
    for (int k = 0; k < c.per; ++k) {
      axis0[p * c.per + k] = c.axis0[p][k];
      axis1[p * c.per + k] = c.axis1[p][k];
    }
  return 0;
}

/* ------------------------------------------------------------------ LLR */
/* include/cgmimo/detect.hpp:23-26 */
static const double kLlrMax = 64.0, kGainFloor = 1e-12;

/* src/detect.cpp:24 */
static double clip_llr(double v) { return v < -kLlrMax ? -kLlrMax : (v > kLlrMax ? kLlrMax : v); }
/* src/detect.cpp:26-29 */
static double safe_rho(double mu, double nu2) { return nu2 < 1e-300 ? 0.0 : mu * mu / nu2; }

/* src/detect.cpp:57-64 */
static double axis_min_sq(double z, const double* amps, int n) {
  double best = INFINITY;
  for (int k = 0; k < n; ++k) {
    const double d = z - amps[k];
    if (d * d < best) best = d * d;
  }
  return best;
}

/* src/detect.cpp:68-86: erasure below the gain floor, rho<0 -> 0, z = xhat/mu,
 * I-axis bits first then Q-axis bits, positive favours bit 1, clip +-64. */
static void llrs_one(cx xhat, double mu, double rho, const constel_t* c, double* out) {
  for (int b = 0; b < c->bits; ++b) out[b] = 0.0;
  if (fabs(mu) < kGainFloor) return;
  if (rho < 0.0) rho = 0.0;
  const cx z = xhat / mu;
  for (int p = 0; p < c->axis_bits; ++p) {
    const double d0 = axis_min_sq(creal(z), c->axis0[p], c->per);
    const double d1 = axis_min_sq(creal(z), c->axis1[p], c->per);
    out[p] = clip_llr(rho * (d0 - d1));
  }
  for (int p = 0; p < c->axis_bits; ++p) {
    const double d0 = axis_min_sq(cimag(z), c->axis0[p], c->per);
    const double d1 = axis_min_sq(cimag(z), c->axis1[p], c->per);
    out[c->axis_bits + p] = clip_llr(rho * (d0 - d1));
  }
}

int orc_compute_llrs(double xr, double xi, double mu, double rho, int qam_bits, double* out) {
  constel_t c;
  if (constel_make(qam_bits, &c)) return 2;
  llrs_one(xr + I * xi, mu, rho, &c, out);
  return 0;
}

/* --------------------------------------------------------------- linalg */
/* src/linalg.cpp:59-101.  Full U x U storage (row-major) of the Hermitian
 * result; the lower triangle is computed, the upper mirrored by conjugation
 * (linalg.hpp:50-52), the diagonal is real.  col(i)[t] is h(t,i) uplink and
 * conj(h(i,t)) downlink. */
static void gram(const cx* h, int B, int U, int downlink, double rho_inv, cx* a) {
  for (int i = 0; i < U; ++i) {
    for (int j = 0; j <= i; ++j) {
      double sr = 0.0, si = 0.0;
      for (int t = 0; t < B; ++t) {
        const cx vi = downlink ? conj(h[(long)i * B + t]) : h[(long)t * U + i];
        const cx vj = downlink ? conj(h[(long)j * B + t]) : h[(long)t * U + j];
        sr += creal(vi) * creal(vj) + cimag(vi) * cimag(vj);
        si += creal(vi) * cimag(vj) - cimag(vi) * creal(vj);
      }
      if (i == j) {
        a[(long)i * U + i] = sr + rho_inv;
      } else {
        a[(long)i * U + j] = sr + I * si;
        a[(long)j * U + i] = sr - I * si;
      }
    }
  }
}

/* src/linalg.cpp:128-139 */
static void hmatvec(const cx* a, int n, const cx* v, cx* y) {
  for (int i = 0; i < n; ++i) {
    cx s = 0.0;
    for (int j = 0; j < n; ++j) s += a[(long)i * n + j] * v[j];
    y[i] = s;
  }
}

/* src/linalg.cpp:141-154 (square case) */
static void matmul(const cx* a, const cx* b, int n, cx* c) {
  memset(c, 0, sizeof(cx) * n * n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const cx aik = a[(long)i * n + k];
      for (int j = 0; j < n; ++j) c[(long)i * n + j] += aik * b[(long)k * n + j];
    }
}

static double norm2_sq(const cx* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += creal(v[i]) * creal(v[i]) + cimag(v[i]) * cimag(v[i]);
  return s;
}

/* ---------------------------------------------------------------- CG */
/* Tracker state: src/detect.cpp:330-368 (exact), :397-433 (approx);
 * histories start at alpha = 1, beta = 0 (detect.hpp:97-98). */
typedef struct {
  int U, k, exact;
  cx *f, *f1, *f2;      /* exact: U x U filters L_k, L_{k-1}, L_{k-2} */
  double *d, *d1, *d2;  /* approx: diagonals */
  double am1, am2, bm1, bm2;
  cx *tmp_d1, *tmp_d2, *tmp_ad;
} tracker_t;

static void tracker_step(tracker_t* t, const cx* a, double alpha, double beta) {
  const int U = t->U;
  ++t->k;
  if (t->exact) {
    if (t->k == 1) {
      cx* nf = t->f2;  /* rotate buffers: f2 <- f1 <- f <- new */
      t->f2 = t->f1; t->f1 = t->f; t->f = nf;
      memset(t->f, 0, sizeof(cx) * U * U);
      for (int i = 0; i < U; ++i) t->f[(long)i * U + i] = alpha;
    } else {
      const double c1 = alpha * (1.0 + t->bm1) / t->am1;
      const double c2 = alpha * t->bm2 / t->am2;
      for (long e = 0; e < (long)U * U; ++e) {
        t->tmp_d1[e] = t->f[e] - t->f1[e];
        t->tmp_d2[e] = t->f1[e] - t->f2[e];
      }
      matmul(a, t->tmp_d1, U, t->tmp_ad);
      cx* nf = t->f2;
      for (long e = 0; e < (long)U * U; ++e)
        nf[e] = t->f[e] + c1 * t->tmp_d1[e] - alpha * t->tmp_ad[e] - c2 * t->tmp_d2[e];
      t->f2 = t->f1; t->f1 = t->f; t->f = nf;
    }
  } else {
    if (t->k == 1) {
      double* nd = t->d2;
      t->d2 = t->d1; t->d1 = t->d; t->d = nd;
      for (int i = 0; i < U; ++i) t->d[i] = alpha;
    } else {
      const double c1 = alpha * (1.0 + t->bm1) / t->am1;
      const double c2 = alpha * t->bm2 / t->am2;
      double* nd = t->d2;
      for (int i = 0; i < U; ++i) {
        const double d1 = t->d[i] - t->d1[i];
        const double d2 = t->d1[i] - t->d2[i];
        nd[i] = t->d[i] + (c1 - alpha * creal(a[(long)i * U + i])) * d1 - c2 * d2;
      }
      t->d2 = t->d1; t->d1 = t->d; t->d = nd;
    }
  }
  t->am2 = t->am1; t->am1 = alpha;
  t->bm2 = t->bm1; t->bm1 = beta;
}

/* src/solvers.cpp:17-27,37-72: exactly K iterations from v = 0, freeze at
 * ||r||^2 <= 1e-28 ||r0||^2 (alpha = 1, beta = 0 still reported), breakdown
 * when p^H A p < 1e-30.  The 1e-9 imaginary-part check (:29-35) can only fire
 * for a non-Hermitian A, which gram() cannot produce.  Returns 1 on breakdown. */
static int cg_run(const cx* a, const cx* b, int U, int K, cx* v, tracker_t* trk,
                  cx* r, cx* p, cx* e) {
  for (int i = 0; i < U; ++i) { v[i] = 0.0; r[i] = b[i]; p[i] = b[i]; }
  double rn = norm2_sq(r, U);
  const double rn0 = rn;
  for (int k = 1; k <= K; ++k) {
    double alpha = 1.0, beta = 0.0;
    if (!(rn <= 1e-28 * rn0)) {
      hmatvec(a, U, p, e);
      cx q = 0.0;
      for (int i = 0; i < U; ++i) q += conj(p[i]) * e[i];
      const double curv = creal(q);
      if (curv < 1e-30) return 1;
      alpha = rn / curv;
      for (int i = 0; i < U; ++i) v[i] += alpha * p[i];
      for (int i = 0; i < U; ++i) r[i] -= alpha * e[i];
      const double rn_next = norm2_sq(r, U);
      beta = rn_next / rn;
      rn = rn_next;
      for (int i = 0; i < U; ++i) p[i] = r[i] + beta * p[i];
    }
    if (trk) tracker_step(trk, a, alpha, beta);
  }
  return 0;
}

/* src/detect.cpp:370-395 with G = A - rho^-1 I (unregularized, :32-39) */
static void exact_extract(const cx* filt, const cx* g, int U, double es, double n0,
                          double* mu, double* nu2, cx* bmat) {
  matmul(filt, g, U, bmat);
  for (int i = 0; i < U; ++i) {
    mu[i] = creal(bmat[(long)i * U + i]);
    double interference = 0.0;
    cx cii = 0.0;
    for (int j = 0; j < U; ++j) {
      const cx bij = bmat[(long)i * U + j];
      if (j != i) interference += creal(bij) * creal(bij) + cimag(bij) * cimag(bij);
      cii += bij * conj(filt[(long)i * U + j]);
    }
    nu2[i] = interference * es + creal(cii) * n0;
  }
}

static void* xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz); }

static void load_cx(const double* p, long n, cx* out) {
  for (long i = 0; i < n; ++i) out[i] = p[2 * i] + I * p[2 * i + 1];
}
static void store_cx(const cx* v, long n, double* p) {
  for (long i = 0; i < n; ++i) { p[2 * i] = creal(v[i]); p[2 * i + 1] = cimag(v[i]); }
}

/* src/detect.cpp:182-237 (detect_cg), per (sc, s) instance */
int orc_detect_cg(int B, int U, long n_sc, int S, const double* H, const double* Y,
                  double rho_u, double n0, double es, int qam_bits, int K, int tracker,
                  double* xhat, double* mu, double* rho, double* llr, uint8_t* status) {
  constel_t c;
  if (constel_make(qam_bits, &c)) return 2;
  const int bad = !(rho_u > 0.0 && n0 > 0.0 && es > 0.0) || K < 1;
  const double rho_inv = 1.0 / rho_u;
  cx* h = xcalloc((size_t)B * U, sizeof(cx));
  cx* y = xcalloc(B, sizeof(cx));
  cx* a = xcalloc((size_t)U * U, sizeof(cx));
  cx* g = xcalloc((size_t)U * U, sizeof(cx));
  cx* bv = xcalloc(U, sizeof(cx));
  cx *v = xcalloc(U, sizeof(cx)), *r = xcalloc(U, sizeof(cx));
  cx *p = xcalloc(U, sizeof(cx)), *e = xcalloc(U, sizeof(cx));
  cx* fbuf = xcalloc((size_t)6 * U * U, sizeof(cx));
  double* dbuf = xcalloc((size_t)3 * U, sizeof(double));
  double* nu2 = xcalloc(U, sizeof(double));
  for (long sc = 0; sc < n_sc; ++sc) {
    load_cx(H + 2 * sc * B * U, (long)B * U, h);
    gram(h, B, U, 0, rho_inv, a);
    memcpy(g, a, sizeof(cx) * U * U);
    for (int i = 0; i < U; ++i) g[(long)i * U + i] = creal(a[(long)i * U + i]) - rho_inv;
    for (int s = 0; s < S; ++s) {
      const long inst = sc * S + s;
      double* xo = xhat + 2 * inst * U;
      double* mo = mu + inst * U;
      double* ro = rho + inst * U;
      double* lo = llr + inst * U * qam_bits;
      status[inst] = 0;
      if (bad) { status[inst] = 4; goto zero; }
      load_cx(Y + 2 * inst * B, B, y);
      /* matched filter H^H y (linalg.cpp:116-126) */
      for (int u = 0; u < U; ++u) bv[u] = 0.0;
      for (int t = 0; t < B; ++t)
        for (int u = 0; u < U; ++u) bv[u] += conj(h[(long)t * U + u]) * y[t];
      tracker_t trk;
      memset(&trk, 0, sizeof trk);
      trk.U = U; trk.exact = tracker == 0;
      trk.am1 = trk.am2 = 1.0; trk.bm1 = trk.bm2 = 0.0;
      trk.f = fbuf; trk.f1 = fbuf + (long)U * U; trk.f2 = fbuf + 2L * U * U;
      trk.tmp_d1 = fbuf + 3L * U * U; trk.tmp_d2 = fbuf + 4L * U * U;
      trk.tmp_ad = fbuf + 5L * U * U;
      memset(fbuf, 0, sizeof(cx) * 3 * U * U);
      trk.d = dbuf; trk.d1 = dbuf + U; trk.d2 = dbuf + 2 * U;
      memset(dbuf, 0, sizeof(double) * 3 * U);
      if (cg_run(a, bv, U, K, v, &trk, r, p, e)) { status[inst] = 1; goto zero; }
      if (trk.exact) {
        exact_extract(trk.f, g, U, es, n0, mo, nu2, trk.tmp_ad);
        for (int i = 0; i < U; ++i) ro[i] = safe_rho(mo[i], nu2[i]);
      } else { /* detect.cpp:435-441 */
        for (int i = 0; i < U; ++i) {
          const double gd = creal(g[(long)i * U + i]);
          mo[i] = trk.d[i] * gd;
          ro[i] = n0 > 0.0 ? gd / n0 : 0.0;
        }
      }
      store_cx(v, U, xo);
      for (int i = 0; i < U; ++i) llrs_one(v[i], mo[i], ro[i], &c, lo + (long)i * qam_bits);
      continue;
    zero:
      memset(xo, 0, sizeof(double) * 2 * U);
      memset(mo, 0, sizeof(double) * U);
      memset(ro, 0, sizeof(double) * U);
      memset(lo, 0, sizeof(double) * U * qam_bits);
    }
  }
  free(h); free(y); free(a); free(g); free(bv); free(v); free(r); free(p); free(e);
  free(fbuf); free(dbuf); free(nu2);
  return 0;
}

/* Inverse of a Hermitian positive-definite matrix through its Cholesky
 * factor A = M M^H (solvers.cpp:237-320).  Returns 1 if not PD. */
static int chol_inverse(const cx* a, int n, cx* inv, cx* m, cx* col) {
  memset(m, 0, sizeof(cx) * n * n);
  for (int j = 0; j < n; ++j) {
    double d = creal(a[(long)j * n + j]);
    for (int k = 0; k < j; ++k) {
      const cx vv = m[(long)j * n + k];
      d -= creal(vv) * creal(vv) + cimag(vv) * cimag(vv);
    }
    if (!(d > 0.0)) return 1;
    const double piv = sqrt(d);
    m[(long)j * n + j] = piv;
    for (int i = j + 1; i < n; ++i) {
      cx s = a[(long)i * n + j];
      for (int k = 0; k < j; ++k) s -= m[(long)i * n + k] * conj(m[(long)j * n + k]);
      m[(long)i * n + j] = s / piv;
    }
  }
  for (int cc = 0; cc < n; ++cc) {
    for (int i = 0; i < cc; ++i) col[i] = 0.0;
    col[cc] = 1.0 / creal(m[(long)cc * n + cc]);
    for (int i = cc + 1; i < n; ++i) {
      cx s = 0.0;
      for (int k = cc; k < i; ++k) s -= m[(long)i * n + k] * col[k];
      col[i] = s / creal(m[(long)i * n + i]);
    }
    for (int ii = n - 1; ii >= 0; --ii) {
      cx s = col[ii];
      for (int k = ii + 1; k < n; ++k) s -= conj(m[(long)k * n + ii]) * col[k];
      col[ii] = s / creal(m[(long)ii * n + ii]);
    }
    for (int i = 0; i < n; ++i) inv[(long)i * n + cc] = col[i];
  }
  return 0;
}

/* src/detect.cpp:88-126: W = inv(A) H^H, xhat = W y, mu_i = Re (WH)_ii,
 * nu_i^2 = Es sum_{j!=i} |(WH)_ij|^2 + N0 ||w_i||^2. */
int orc_detect_explicit(int B, int U, long n_sc, int S, const double* H, const double* Y,
                        double rho_u, double n0, double es, int qam_bits, double* xhat,
                        double* mu, double* rho, double* llr, uint8_t* status) {
  constel_t c;
  if (constel_make(qam_bits, &c)) return 2;
  const int bad = !(rho_u > 0.0 && n0 > 0.0 && es > 0.0);
  cx* h = xcalloc((size_t)B * U, sizeof(cx));
  cx* y = xcalloc(B, sizeof(cx));
  cx* a = xcalloc((size_t)U * U, sizeof(cx));
  cx* inv = xcalloc((size_t)U * U, sizeof(cx));
  cx* m = xcalloc((size_t)U * U, sizeof(cx));
  cx* col = xcalloc(U, sizeof(cx));
  cx* w = xcalloc((size_t)U * B, sizeof(cx));
  cx* wh = xcalloc((size_t)U * U, sizeof(cx));
  cx* xh = xcalloc(U, sizeof(cx));
  for (long sc = 0; sc < n_sc; ++sc) {
    load_cx(H + 2 * sc * B * U, (long)B * U, h);
    int notpd = 0;
    if (!bad) {
      gram(h, B, U, 0, 1.0 / rho_u, a);
      notpd = chol_inverse(a, U, inv, m, col);
      for (int i = 0; i < U; ++i)
        for (int t = 0; t < B; ++t) {
          cx s = 0.0;
          for (int k = 0; k < U; ++k) s += inv[(long)i * U + k] * conj(h[(long)t * U + k]);
          w[(long)i * B + t] = s;
        }
      for (int i = 0; i < U; ++i)
        for (int j = 0; j < U; ++j) {
          cx s = 0.0;
          for (int t = 0; t < B; ++t) s += w[(long)i * B + t] * h[(long)t * U + j];
          wh[(long)i * U + j] = s;
        }
    }
    for (int s = 0; s < S; ++s) {
      const long inst = sc * S + s;
      double* xo = xhat + 2 * inst * U;
      double* mo = mu + inst * U;
      double* ro = rho + inst * U;
      double* lo = llr + inst * U * qam_bits;
      status[inst] = (bad || notpd) ? 4 : 0;
      if (status[inst]) {
        memset(xo, 0, sizeof(double) * 2 * U); memset(mo, 0, sizeof(double) * U);
        memset(ro, 0, sizeof(double) * U); memset(lo, 0, sizeof(double) * U * qam_bits);
        continue;
      }
      load_cx(Y + 2 * inst * B, B, y);
      for (int i = 0; i < U; ++i) {
        cx acc = 0.0;
        for (int t = 0; t < B; ++t) acc += w[(long)i * B + t] * y[t];
        xh[i] = acc;
        mo[i] = creal(wh[(long)i * U + i]);
        double interference = 0.0, wn = 0.0;
        for (int j = 0; j < U; ++j)
          if (j != i) {
            const cx q = wh[(long)i * U + j];
            interference += creal(q) * creal(q) + cimag(q) * cimag(q);
          }
        for (int t = 0; t < B; ++t) {
          const cx q = w[(long)i * B + t];
          wn += creal(q) * creal(q) + cimag(q) * cimag(q);
        }
        ro[i] = safe_rho(mo[i], interference * es + wn * n0);
      }
      store_cx(xh, U, xo);
      for (int i = 0; i < U; ++i) llrs_one(xh[i], mo[i], ro[i], &c, lo + (long)i * qam_bits);
    }
  }
  free(h); free(y); free(a); free(inv); free(m); free(col); free(w); free(wh); free(xh);
  return 0;
}

/* solvers.cpp:323-359: Sum = D^-1 + T D^-1 + T^2 D^-1 + ..., T = -D^-1 E;
 * from the third term on, one triangle (j >= i) and its mirror.  Returns 1
 * on a zero diagonal entry (std::domain_error). */
static int neumann_inverse(const cx* a, int n, int terms, cx* sum, cx* t, cx* term, cx* next,
                           double* inv_d) {
  for (int i = 0; i < n; ++i) {
    const double d = creal(a[(long)i * n + i]);
    if (fabs(d) < 1e-300) return 1;
    inv_d[i] = 1.0 / d;
  }
  memset(sum, 0, sizeof(cx) * n * n);
  for (int i = 0; i < n; ++i) sum[(long)i * n + i] = inv_d[i];
  if (terms == 1) return 0;
  memset(t, 0, sizeof(cx) * n * n);
  memset(term, 0, sizeof(cx) * n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      t[(long)i * n + j] = -inv_d[i] * a[(long)i * n + j];
      term[(long)i * n + j] = t[(long)i * n + j] * inv_d[j];
    }
  for (long e = 0; e < (long)n * n; ++e) sum[e] += term[e];
  for (int extra = 2; extra < terms; ++extra) {
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j) {
        cx acc = 0.0;
        for (int k = 0; k < n; ++k) acc += t[(long)i * n + k] * term[(long)k * n + j];
        next[(long)i * n + j] = acc;
        if (j != i) next[(long)j * n + i] = conj(acc);
      }
    for (long e = 0; e < (long)n * n; ++e) sum[e] += next[e];
    memcpy(term, next, sizeof(cx) * n * n);
  }
  return 0;
}

/* detect_cholesky (detect.cpp:122-181, method 0), detect_cgls (:238-272,
 * method 2: cgls_solve_regularized solvers.cpp:141-194 over cgls_core
 * :87-139 with the approximate tracker), detect_neumann (:274-326, method 3) */
static int detect_alt(int method, int B, int U, long n_sc, int S, const double* H,
                      const double* Y, double rho_u, double n0, double es, int qam_bits, int K,
                      double* xhat, double* mu, double* rho, double* llr, uint8_t* status) {
  constel_t c;
  if (constel_make(qam_bits, &c)) return 2;
  const int bad = !(rho_u > 0.0 && n0 > 0.0 && es > 0.0) || (method != 0 && K < 1);
  const double rho_inv = 1.0 / rho_u;
  const int UU = U * U;
  cx* h = xcalloc((size_t)B * U, sizeof(cx));
  cx* y = xcalloc((size_t)B + U, sizeof(cx));
  cx *a = xcalloc(UU, sizeof(cx)), *inv = xcalloc(UU, sizeof(cx)), *m = xcalloc(UU, sizeof(cx));
  cx *t = xcalloc(UU, sizeof(cx)), *term = xcalloc(UU, sizeof(cx)), *nx = xcalloc(UU, sizeof(cx));
  cx *col = xcalloc(U, sizeof(cx)), *bv = xcalloc(U, sizeof(cx)), *xh = xcalloc(U, sizeof(cx));
  cx *sv = xcalloc(U, sizeof(cx)), *dv = xcalloc(U, sizeof(cx)), *qv = xcalloc((size_t)B + U, sizeof(cx));
  double *gd = xcalloc(U, sizeof(double)), *ad = xcalloc(U, sizeof(double)), *dinv = xcalloc(U, sizeof(double));
  double *f = xcalloc(U, sizeof(double)), *f1 = xcalloc(U, sizeof(double)), *f2 = xcalloc(U, sizeof(double));
  double *mus = xcalloc(U, sizeof(double)), *rhos = xcalloc(U, sizeof(double));
  for (long sc = 0; sc < n_sc; ++sc) {
    load_cx(H + 2 * sc * B * U, (long)B * U, h);
    int fail = bad;
    if (!fail && method != 2) {
      gram(h, B, U, 0, rho_inv, a);
      fail = method == 0 ? chol_inverse(a, U, inv, m, col)
                         : neumann_inverse(a, U, K, inv, t, term, nx, dinv);
    }
    if (!fail && method == 0) { /* detect.cpp:154-178, channel only */
      for (int i = 0; i < U; ++i) {
        const cx vii = inv[(long)i * U + i];
        mus[i] = 1.0 - rho_inv * creal(vii);
        double interference = 0.0, colnorm2 = 0.0;
        for (int j = 0; j < U; ++j) {
          const cx v = inv[(long)i * U + j];
          if (j != i) {
            const double er = -rho_inv * creal(v), ei = -rho_inv * cimag(v);
            interference += er * er + ei * ei;
          }
          const cx w = inv[(long)j * U + i];
          colnorm2 += creal(w) * creal(w) + cimag(w) * cimag(w);
        }
        const double noise = n0 * (creal(vii) - rho_inv * colnorm2);
        rhos[i] = safe_rho(mus[i], es * interference + noise);
      }
    }
    if (!fail && method == 3) { /* detect.cpp:299-323 */
      for (int i = 0; i < U; ++i) {
        if (K == 1) {
          mus[i] = creal(inv[(long)i * U + i]) * (creal(a[(long)i * U + i]) - rho_inv);
        } else {
          cx dg = 0.0;
          for (int j = 0; j < U; ++j) {
            const cx gji = j == i ? creal(a[(long)j * U + j]) - rho_inv : a[(long)j * U + i];
            dg += inv[(long)i * U + j] * gji;
          }
          mus[i] = creal(dg);
        }
        double nu2 = es * (mus[i] - mus[i] * mus[i]);
        if (nu2 < 1e-12) nu2 = 1e-12;
        rhos[i] = safe_rho(mus[i], nu2);
      }
    }
    if (!fail && method == 2) {
      for (int i = 0; i < U; ++i) {
        double d = 0.0;
        for (int b = 0; b < B; ++b) {
          const cx v = h[(long)b * U + i];
          d += creal(v) * creal(v) + cimag(v) * cimag(v);
        }
        gd[i] = d;
        ad[i] = d + rho_inv;
      }
    }
    for (int s = 0; s < S; ++s) {
      const long inst = sc * S + s;
      double* xo = xhat + 2 * inst * U;
      double* mo = mu + inst * U;
      double* ro = rho + inst * U;
      double* lo = llr + inst * U * qam_bits;
      status[inst] = fail ? 4 : 0;
      if (fail) goto zero;
      load_cx(Y + 2 * inst * B, B, y);
      if (method != 2) {
        for (int u = 0; u < U; ++u) bv[u] = 0.0;
        for (int b = 0; b < B; ++b)
          for (int u = 0; u < U; ++u) bv[u] += conj(h[(long)b * U + u]) * y[b];
        if (method == 3 && K == 1) {
          for (int i = 0; i < U; ++i) xh[i] = creal(inv[(long)i * U + i]) * bv[i];
        } else {
          hmatvec(inv, U, bv, xh);
        }
        for (int i = 0; i < U; ++i) { mo[i] = mus[i]; ro[i] = rhos[i]; }
      } else {
        /* residual-space vectors carry B + U entries; y_aug = [y; 0] */
        const double aug = sqrt(rho_inv);
        for (int i = 0; i < U; ++i) y[B + i] = 0.0;
        for (int i = 0; i < U; ++i) { xh[i] = 0.0; f[i] = f1[i] = f2[i] = 0.0; }
        for (int u = 0; u < U; ++u) sv[u] = 0.0;
        for (int b = 0; b < B; ++b)
          for (int u = 0; u < U; ++u) sv[u] += conj(h[(long)b * U + u]) * y[b];
        memcpy(dv, sv, sizeof(cx) * U);
        double gamma = norm2_sq(sv, U);
        const double gamma0 = gamma;
        double am1 = 1.0, am2 = 1.0, bm1 = 0.0, bm2 = 0.0;
        int broke = 0;
        for (int k = 1; k <= K; ++k) {
          double alpha = 1.0, beta = 0.0;
          if (!(gamma <= 1e-28 * gamma0)) {
            for (int b = 0; b < B; ++b) {
              cx acc = 0.0;
              for (int j = 0; j < U; ++j) acc += h[(long)b * U + j] * dv[j];
              qv[b] = acc;
            }
            for (int j = 0; j < U; ++j) qv[B + j] = aug * dv[j];
            const double qn2 = norm2_sq(qv, B + U);
            if (qn2 < 1e-30) { broke = 1; break; }
            alpha = gamma / qn2;
            for (int j = 0; j < U; ++j) xh[j] += alpha * dv[j];
            for (int b = 0; b < B + U; ++b) y[b] -= alpha * qv[b];
            for (int u = 0; u < U; ++u) sv[u] = 0.0;
            for (int b = 0; b < B; ++b)
              for (int u = 0; u < U; ++u) sv[u] += conj(h[(long)b * U + u]) * y[b];
            for (int u = 0; u < U; ++u) sv[u] += aug * y[B + u];
            const double gn = norm2_sq(sv, U);
            beta = gn / gamma;
            gamma = gn;
            for (int u = 0; u < U; ++u) dv[u] = sv[u] + beta * dv[u];
          }
          /* ApproxSinrTracker::step (detect.cpp:400-428) */
          for (int i = 0; i < U; ++i) {
            double nxv;
            if (k == 1) {
              nxv = alpha;
            } else {
              const double c1 = alpha * (1.0 + bm1) / am1, c2 = alpha * bm2 / am2;
              nxv = f[i] + (c1 - alpha * ad[i]) * (f[i] - f1[i]) - c2 * (f1[i] - f2[i]);
            }
            f2[i] = f1[i];
            f1[i] = f[i];
            f[i] = nxv;
          }
          am2 = am1; am1 = alpha; bm2 = bm1; bm1 = beta;
        }
        if (broke) { status[inst] = 1; goto zero; }
        for (int i = 0; i < U; ++i) { /* detect.cpp:430-441 */
          mo[i] = f[i] * gd[i];
          ro[i] = n0 > 0.0 ? gd[i] / n0 : 0.0;
        }
      }
      store_cx(xh, U, xo);
      for (int i = 0; i < U; ++i) llrs_one(xh[i], mo[i], ro[i], &c, lo + (long)i * qam_bits);
      continue;
    zero:
      memset(xo, 0, sizeof(double) * 2 * U);
      memset(mo, 0, sizeof(double) * U);
      memset(ro, 0, sizeof(double) * U);
      memset(lo, 0, sizeof(double) * U * qam_bits);
    }
  }
  free(h); free(y); free(a); free(inv); free(m); free(t); free(term); free(nx); free(col);
  free(bv); free(xh); free(sv); free(dv); free(qv); free(gd); free(ad); free(dinv);
  free(f); free(f1); free(f2); free(mus); free(rhos);
  return 0;
}

int orc_detect_cholesky(int B, int U, long n_sc, int S, const double* H, const double* Y,
                        double rho_u, double n0, double es, int qam_bits, double* xhat,
                        double* mu, double* rho, double* llr, uint8_t* status) {
  return detect_alt(0, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, 1, xhat, mu, rho, llr, status);
}
int orc_detect_cgls(int B, int U, long n_sc, int S, const double* H, const double* Y,
                    double rho_u, double n0, double es, int qam_bits, int K, double* xhat,
                    double* mu, double* rho, double* llr, uint8_t* status) {
  return detect_alt(2, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, K, xhat, mu, rho, llr, status);
}
int orc_detect_neumann(int B, int U, long n_sc, int S, const double* H, const double* Y,
                       double rho_u, double n0, double es, int qam_bits, int K, double* xhat,
                       double* mu, double* rho, double* llr, uint8_t* status) {
  return detect_alt(3, B, U, n_sc, S, H, Y, rho_u, n0, es, qam_bits, K, xhat, mu, rho, llr, status);
}

/* src/precode.cpp:22-36 normalize: s = q/||q||, zero_input when ||q|| < 1e-300 */
static uint8_t normalize(const cx* q, int B, double* qo, double* so, double* gain) {
  const double g = sqrt(norm2_sq(q, B));
  store_cx(q, B, qo);
  if (g < 1e-300) {
    if (so) memset(so, 0, sizeof(double) * 2 * B);
    *gain = 0.0;
    return 2;
  }
  if (so) {
    const double inv = 1.0 / g;
    for (int i = 0; i < B; ++i) { so[2 * i] = creal(q[i]) * inv; so[2 * i + 1] = cimag(q[i]) * inv; }
  }
  *gain = g;
  return 0;
}

/* src/precode.cpp:38-71: A_d = H_d H_d^H + rho_d^-1 I, CG on t, q = H_d^H v
 * (mode 0), or v = inv(A_d) t (mode 1, precode.cpp:45-54), v = Neumann
 * series of A_d applied to t (mode 3, precode.cpp:84-93); mode 2 is
 * precode_cgls (precode.cpp:73-82): min-norm CGLS (solvers.cpp:196-235)
 * accumulating q = H_d^H inner directly. */
static int precode_common(int mode, int B, int U, long n_sc, int S, const double* Hd,
                          const double* T, double rho_d, int K, double* q, double* s_out,
                          double* gain, uint8_t* status) {
  const int bad = !(rho_d > 0.0) || (mode != 1 && K < 1);
  cx* h = xcalloc((size_t)U * B, sizeof(cx));
  cx *nt = xcalloc((size_t)U * U, sizeof(cx)), *nterm = xcalloc((size_t)U * U, sizeof(cx));
  cx *nnext = xcalloc((size_t)U * U, sizeof(cx)), *wv = xcalloc(B, sizeof(cx));
  double* dinv = xcalloc(U, sizeof(double));
  cx* a = xcalloc((size_t)U * U, sizeof(cx));
  cx* inv = xcalloc((size_t)U * U, sizeof(cx));
  cx* m = xcalloc((size_t)U * U, sizeof(cx));
  cx* col = xcalloc(U, sizeof(cx));
  cx *t = xcalloc(U, sizeof(cx)), *v = xcalloc(U, sizeof(cx));
  cx *r = xcalloc(U, sizeof(cx)), *p = xcalloc(U, sizeof(cx)), *e = xcalloc(U, sizeof(cx));
  cx* qv = xcalloc(B, sizeof(cx));
  for (long sc = 0; sc < n_sc; ++sc) {
    load_cx(Hd + 2 * sc * U * B, (long)U * B, h);
    int notpd = 0;
    if (!bad) {
      gram(h, B, U, 1, 1.0 / rho_d, a);
      if (mode == 1) notpd = chol_inverse(a, U, inv, m, col);
      if (mode == 3) notpd = neumann_inverse(a, U, K, inv, nt, nterm, nnext, dinv);
    }
    for (int s = 0; s < S; ++s) {
      const long inst = sc * S + s;
      double* qo = q + 2 * inst * B;
      double* so = s_out ? s_out + 2 * inst * B : NULL;
      uint8_t st = (bad || notpd) ? 4 : 0;
      if (!st) {
        load_cx(T + 2 * inst * U, U, t);
        if (mode == 0) {
          if (cg_run(a, t, U, K, v, NULL, r, p, e)) st = 1;
        } else if (mode == 2) {
          const double rho_inv = 1.0 / rho_d;
          for (int b = 0; b < B; ++b) qv[b] = 0.0;
          memcpy(r, t, sizeof(cx) * U);
          memcpy(p, t, sizeof(cx) * U);
          double rn2 = norm2_sq(r, U);
          const double rn0 = rn2;
          for (int k = 1; k <= K && !st; ++k) {
            if (rn2 <= 1e-28 * rn0) continue;
            for (int b = 0; b < B; ++b) { /* w = H_d^H p */
              cx acc = 0.0;
              for (int u = 0; u < U; ++u) acc += conj(h[(long)u * B + b]) * p[u];
              wv[b] = acc;
            }
            double curv = 0.0;
            for (int u = 0; u < U; ++u) { /* e = H_d w + rho^-1 p */
              cx acc = 0.0;
              for (int b = 0; b < B; ++b) acc += h[(long)u * B + b] * wv[b];
              e[u] = acc + rho_inv * p[u];
              curv += creal(conj(p[u]) * e[u]);
            }
            if (curv < 1e-30) { st = 1; break; }
            const double alpha = rn2 / curv;
            for (int b = 0; b < B; ++b) qv[b] += alpha * wv[b];
            for (int u = 0; u < U; ++u) r[u] -= alpha * e[u];
            const double rn = norm2_sq(r, U);
            const double beta = rn / rn2;
            rn2 = rn;
            for (int u = 0; u < U; ++u) p[u] = r[u] + beta * p[u];
          }
        } else {
          hmatvec(inv, U, t, v);
        }
      }
      if (st) {
        memset(qo, 0, sizeof(double) * 2 * B);
        if (so) memset(so, 0, sizeof(double) * 2 * B);
        gain[inst] = 0.0;
        status[inst] = st;
        continue;
      }
      /* q = H_d^H v (linalg.cpp:116-126) */
      if (mode != 2) {
        for (int b = 0; b < B; ++b) qv[b] = 0.0;
        for (int u = 0; u < U; ++u)
          for (int b = 0; b < B; ++b) qv[b] += conj(h[(long)u * B + b]) * v[u];
      }
      status[inst] = normalize(qv, B, qo, so, gain + inst);
    }
  }
  free(h); free(a); free(inv); free(m); free(col); free(t); free(v); free(r); free(p);
  free(e); free(qv); free(nt); free(nterm); free(nnext); free(wv); free(dinv);
  return 0;
}

int orc_precode_cg(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                   double rho_d, int K, double* q, double* s, double* gain, uint8_t* status) {
  return precode_common(0, B, U, n_sc, S, Hd, T, rho_d, K, q, s, gain, status);
}

int orc_precode_explicit(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                         double rho_d, double* q, double* s, double* gain, uint8_t* status) {
  return precode_common(1, B, U, n_sc, S, Hd, T, rho_d, 1, q, s, gain, status);
}

int orc_precode_cgls(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                     double rho_d, int K, double* q, double* s, double* gain, uint8_t* status) {
  return precode_common(2, B, U, n_sc, S, Hd, T, rho_d, K, q, s, gain, status);
}

int orc_precode_neumann(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                        double rho_d, int K, double* q, double* s, double* gain, uint8_t* status) {
  return precode_common(3, B, U, n_sc, S, Hd, T, rho_d, K, q, s, gain, status);
}

/* --------------------------------------------------------------- coding */
/* K = 7 (133, 171)_8 mother code, puncture period 5 to rate 5/6, 6-bit tail
 * (coding.cpp:14-58).  State = last 6 inputs, newest in bit 5; the encoder
 * register word is (u << 6) | state. */
enum { kMemory = 6, kNStates = 64, kPeriod = 5 };
static const int kPunctA[kPeriod] = {1, 1, 0, 1, 0};
static const int kPunctB[kPeriod] = {1, 0, 1, 0, 1};

static unsigned par(unsigned w) {
  w ^= w >> 16; w ^= w >> 8; w ^= w >> 4; w ^= w >> 2; w ^= w >> 1;
  return w & 1u;
}
static void branch(unsigned s, unsigned u, unsigned* a, unsigned* b, unsigned* next) {
  const unsigned word = (u << kMemory) | s;
  *a = par(word & 0133u);
  *b = par(word & 0171u);
  *next = (u << (kMemory - 1)) | (s >> 1);
}

/* coding.cpp:65-84 */
long orc_conv_encode(const uint8_t* info, long n, uint8_t* out) {
  const long total = n + kMemory;
  if (n < 0 || total % kPeriod != 0) return -1;
  long pos = 0;
  unsigned s = 0;
  for (long t = 0; t < total; ++t) {
    unsigned a, b, nx;
    branch(s, t < n ? (info[t] & 1u) : 0u, &a, &b, &nx);
    if (kPunctA[t % kPeriod]) out[pos++] = (uint8_t)a;
    if (kPunctB[t % kPeriod]) out[pos++] = (uint8_t)b;
    s = nx;
  }
  return pos;
}

/* coding.cpp:86-147: depuncture, max-log ACS in FP64 visiting states and
 * inputs in ascending order with a strict '>' (ties keep the first), tail
 * forces u = 0, traceback from state 0 */
long orc_viterbi_decode(const double* llrs, long n, uint8_t* out) {
  if (n % 6 != 0 || n / 6 * kPeriod <= kMemory) return -1;
  const long total = n / 6 * kPeriod, info_len = total - kMemory;
  double* la = xcalloc((size_t)total, sizeof(double));
  double* lb = xcalloc((size_t)total, sizeof(double));
  uint8_t* dec = xcalloc((size_t)total * kNStates, 1);
  long pos = 0;
  for (long t = 0; t < total; ++t) {
    if (kPunctA[t % kPeriod]) la[t] = llrs[pos++];
    if (kPunctB[t % kPeriod]) lb[t] = llrs[pos++];
  }
  double m[kNStates], nm[kNStates];
  for (int s = 0; s < kNStates; ++s) m[s] = -INFINITY;
  m[0] = 0.0;
  for (long t = 0; t < total; ++t) {
    const double bm[4] = {-la[t] - lb[t], -la[t] + lb[t], la[t] - lb[t], la[t] + lb[t]};
    for (int s = 0; s < kNStates; ++s) nm[s] = -INFINITY;
    const unsigned umax = t < info_len ? 2u : 1u;
    for (unsigned s = 0; s < kNStates; ++s) {
      if (m[s] == -INFINITY) continue;
      for (unsigned u = 0; u < umax; ++u) {
        unsigned a, b, nx;
        branch(s, u, &a, &b, &nx);
        const double v = m[s] + bm[(a << 1) | b];
        if (v > nm[nx]) {
          nm[nx] = v;
          dec[t * kNStates + nx] = (uint8_t)((u << 6) | s);
        }
      }
    }
    memcpy(m, nm, sizeof m);
  }
  unsigned s = 0;
  for (long t = total; t-- > 0;) {
    const uint8_t d = dec[t * kNStates + s];
    if (t < info_len) out[t] = (uint8_t)(d >> 6);
    s = d & (kNStates - 1);
  }
  free(la);
  free(lb);
  free(dec);
  return info_len;
}

/* coding.cpp:149-157: Fisher-Yates from the top with next_unit */
void orc_make_interleaver(uint64_t key, const uint64_t* forks, int n_forks, long n, int64_t* perm) {
  rng_t r = rng_path(key, forks, n_forks);
  for (long i = 0; i < n; ++i) perm[i] = i;
  for (long i = n; i-- > 1;) {
    long j = (long)(rng_unit(&r) * (double)(i + 1));
    if (j > i) j = i;
    const int64_t x = perm[i];
    perm[i] = perm[j];
    perm[j] = x;
  }
}
