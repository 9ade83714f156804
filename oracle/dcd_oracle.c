/*
 * TEST INFRASTRUCTURE ONLY — CPU checker for the CUDA hot path; see
 * dcd_oracle.h for the contract and the parity pin.  Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * Compiled with -ffp-contract=off and no FMA so the arithmetic matches the
 * reference's scalar backend operation for operation.
 */
#define _GNU_SOURCE
#include "dcd_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* errors                                                                    */
/* ------------------------------------------------------------------------ */
static __thread char g_err[512];

const char* dcdo_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
#define EINVAL_ 1
#define ERUNTIME_ 2

/* complex helpers: z = (re, im) pairs stored in double[2] */
typedef struct { double re, im; } cplx;

static inline cplx cmul(cplx a, cplx b) {  /* GCC std::complex operator* */
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cplx conjz(cplx a) { cplx r = {a.re, -a.im}; return r; }
static inline double normz(cplx a) { return a.re * a.re + a.im * a.im; }  /* std::norm */
static inline cplx ld(const double* p, size_t i) { cplx r = {p[2 * i], p[2 * i + 1]}; return r; }
static inline void st(double* p, size_t i, cplx v) { p[2 * i] = v.re; p[2 * i + 1] = v.im; }

/* ------------------------------------------------------------------------ */
/* vector kernels — src/kernels/kernels_scalar.cpp                           */
/* ------------------------------------------------------------------------ */
/* kernels_scalar.cpp:9-20 */
void dcdo_cdotc(const double* pa, const double* pb, int n, double* out) {
  double re = 0.0, im = 0.0;
  for (int i = 0; i < n; ++i) {
    const double ar = pa[2 * i], ai = pa[2 * i + 1];
    const double br = pb[2 * i], bi = pb[2 * i + 1];
    re += ar * br + ai * bi;
    im += ar * bi - ai * br;
  }
  out[0] = re;
  out[1] = im;
}
static cplx cdotc(const double* a, const double* b, int n) {
  double o[2];
  dcdo_cdotc(a, b, n, o);
  cplx r = {o[0], o[1]};
  return r;
}

/* kernels_scalar.cpp:22-31 */
void dcdo_caxpy(double ar, double ai, const double* px, double* py, int n) {
  for (int i = 0; i < n; ++i) {
    const double xr = px[2 * i], xi = px[2 * i + 1];
    py[2 * i] += ar * xr - ai * xi;
    py[2 * i + 1] += ar * xi + ai * xr;
  }
}

/* kernels_scalar.cpp:33-41 */
double dcdo_norm2sq(const double* pa, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double re = pa[2 * i], im = pa[2 * i + 1];
    acc += re * re + im * im;
  }
  return acc;
}

/* kernels_scalar.cpp:43-74 */
uint16_t dcdo_f64_to_f16_bits(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  const uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
  const int biased = (int)((u >> 52) & 0x7ff);
  const uint64_t man = u & 0xfffffffffffffULL;
  if (biased == 0x7ff) {
    if (man == 0) return (uint16_t)(sign | 0x7c00u);
    return (uint16_t)(sign | 0x7e00u);
  }
  if (biased == 0) return sign;
  const int e = biased - 1023;
  if (e >= 16) return (uint16_t)(sign | 0x7c00u);
  const uint64_t sig = man | (1ULL << 52);
  int shift = (e >= -14) ? 42 : 42 + (-14 - e);
  if (shift > 62) shift = 62;
  const uint64_t half = 1ULL << (shift - 1);
  const uint64_t rem = sig & ((1ULL << shift) - 1);
  const uint16_t keep = (uint16_t)(sig >> shift);
  uint16_t h = (e >= -14) ? (uint16_t)(((e + 14) << 10) + keep) : keep;
  if (rem > half || (rem == half && (h & 1u))) ++h;
  return (uint16_t)(sign | h);
}

/* kernels_scalar.cpp:76-90 */
double dcdo_f16_bits_to_f64(uint16_t h) {
  const int sign = h >> 15;
  const int e = (h >> 10) & 0x1f;
  const int man = h & 0x3ff;
  double v;
  if (e == 0x1f) v = man ? NAN : INFINITY;
  else if (e == 0) v = ldexp((double)man, -24);
  else v = ldexp((double)(man | 0x400), e - 25);
  return sign ? -v : v;
}

/* precision.cpp:43-72 with kernels_scalar.cpp:92-98 */
void dcdo_round_precision(double* p, int n, int fmt) {
  if (fmt == DCDO_FP32) {
    for (int i = 0; i < n; ++i) p[i] = (double)(float)p[i];
  } else if (fmt == DCDO_FP16) {
    for (int i = 0; i < n; ++i) p[i] = dcdo_f16_bits_to_f64(dcdo_f64_to_f16_bits(p[i]));
  }
}
static cplx round_z(cplx z, int fmt) {
  double t[2] = {z.re, z.im};
  dcdo_round_precision(t, 2, fmt);
  cplx r = {t[0], t[1]};
  return r;
}

/* ------------------------------------------------------------------------ */
/* numerics — src/numerics.cpp                                               */
/* ------------------------------------------------------------------------ */
/* numerics.cpp:31-79 (Cholesky, no pivoting). a: n x n column-major. */
int dcdo_hermitian_solve(const double* a, int n, const double* b, double* x) {
  if (n <= 0) return fail(EINVAL_, "hermitian_solve: matrix must be square and nonempty");
  double max_abs = 0.0, max_diag = 0.0;
  for (int j = 0; j < n; ++j) {
    const cplx d = ld(a, (size_t)j * n + j);
    const double ad = hypot(d.re, d.im);
    if (ad > max_diag) max_diag = ad;
    for (int i = 0; i < n; ++i) {
      const cplx z = ld(a, (size_t)j * n + i);
      const double az = hypot(z.re, z.im);
      if (az > max_abs) max_abs = az;
    }
  }
  const double herm_tol = 1e-10 * (1.0 + max_abs);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) {
      const cplx aij = ld(a, (size_t)j * n + i), aji = ld(a, (size_t)i * n + j);
      if (hypot(aij.re - aji.re, aij.im + aji.im) > herm_tol)
        return fail(EINVAL_, "hermitian_solve: matrix is not hermitian");
    }
  double* l = (double*)malloc(sizeof(double) * 2 * (size_t)n * n);
  memcpy(l, a, sizeof(double) * 2 * (size_t)n * n);
#define L(i, j) ((size_t)(j) * n + (i))
  const double pivot_floor = 1e-14 * max_diag;
  for (int j = 0; j < n; ++j) {
    double d = ld(l, L(j, j)).re;
    for (int k = 0; k < j; ++k) d -= normz(ld(l, L(j, k)));
    if (!(d > pivot_floor)) {
      free(l);
      return fail(ERUNTIME_, "hermitian_solve: matrix is numerically singular");
    }
    const double ljj = sqrt(d);
    cplx dj = {ljj, 0.0};
    st(l, L(j, j), dj);
    for (int i = j + 1; i < n; ++i) {
      cplx s = ld(l, L(i, j));
      for (int k = 0; k < j; ++k) {
        const cplx p = cmul(ld(l, L(i, k)), conjz(ld(l, L(j, k))));
        s.re -= p.re;
        s.im -= p.im;
      }
      s.re /= ljj;
      s.im /= ljj;
      st(l, L(i, j), s);
    }
  }
  double* xx = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  memcpy(xx, b, sizeof(double) * 2 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    cplx s = ld(xx, i);
    for (int k = 0; k < i; ++k) {
      const cplx p = cmul(ld(l, L(i, k)), ld(xx, k));
      s.re -= p.re;
      s.im -= p.im;
    }
    const double di = ld(l, L(i, i)).re;
    s.re /= di;
    s.im /= di;
    st(xx, i, s);
  }
  for (int ii = n; ii-- > 0;) {
    cplx s = ld(xx, ii);
    for (int k = ii + 1; k < n; ++k) {
      const cplx p = cmul(conjz(ld(l, L(k, ii))), ld(xx, k));
      s.re -= p.re;
      s.im -= p.im;
    }
    const double di = ld(l, L(ii, ii)).re;
    s.re /= di;
    s.im /= di;
    st(xx, ii, s);
  }
#undef L
  memcpy(x, xx, sizeof(double) * 2 * (size_t)n);
  free(xx);
  free(l);
  return 0;
}

/* detect.cpp:21-28 */
static double* gram(const double* h, int b, int u) {
  double* g = (double*)malloc(sizeof(double) * 2 * (size_t)u * u);
  for (int j = 0; j < u; ++j)
    for (int i = 0; i < u; ++i) {
      const cplx z = cdotc(h + 2 * (size_t)i * b, h + 2 * (size_t)j * b, b);
      st(g, (size_t)j * u + i, z);
    }
  return g;
}

/* ------------------------------------------------------------------------ */
/* uplink — src/detect.cpp                                                   */
/* ------------------------------------------------------------------------ */
/* detect.cpp:12-19 */
static int check_system(int b, int u, int ylen, double n0, double ex) {
  if (b == 0 || u == 0) return fail(EINVAL_, "detector: empty channel matrix");
  if (ylen != b) return fail(EINVAL_, "detector: observation length must match antenna count");
  if (n0 < 0.0 || !(ex > 0.0)) return fail(EINVAL_, "detector: need N0 >= 0 and E_x > 0");
  return 0;
}

/* detect.cpp:67-110 */
int dcdo_cd_detect(const double* h, int b, int u, const double* y, double n0, double ex,
                   unsigned t_max, int fmt, int scope, double* x_out) {
  int rc = check_system(b, u, b, n0, ex);
  if (rc) return rc;
  if (t_max == 0) return fail(EINVAL_, "cd_detect: need at least one sweep");
  const int store_rounded = fmt != DCDO_FP64 && scope == DCDO_FULL_STORAGE;
  const size_t hn = (size_t)b * u;
  double* hs = (double*)malloc(sizeof(double) * 2 * hn);
  double* r = (double*)malloc(sizeof(double) * 2 * (size_t)b);
  double* m = (double*)malloc(sizeof(double) * (size_t)u);
  double* nn = (double*)malloc(sizeof(double) * (size_t)u);
  double* x = (double*)calloc(2 * (size_t)u, sizeof(double));
  memcpy(hs, h, sizeof(double) * 2 * hn);
  memcpy(r, y, sizeof(double) * 2 * (size_t)b);
  if (store_rounded) {
    dcdo_round_precision(hs, 2 * (int)hn, fmt);
    dcdo_round_precision(r, 2 * b, fmt);
  }
  const double kappa = n0 / ex;
  for (int j = 0; j < u; ++j) {
    const double e = dcdo_norm2sq(hs + 2 * (size_t)j * b, b);
    m[j] = 1.0 / (e + kappa);
    nn[j] = m[j] * e;
  }
  if (store_rounded) {
    dcdo_round_precision(m, u, fmt);
    dcdo_round_precision(nn, u, fmt);
  }
  for (unsigned t = 0; t < t_max; ++t) {
    for (int j = 0; j < u; ++j) {
      const double* hj = hs + 2 * (size_t)j * b;
      const cplx d = cdotc(hj, r, b);
      const cplx xo = ld(x, j);
      cplx xj = {m[j] * d.re + nn[j] * xo.re, m[j] * d.im + nn[j] * xo.im};
      if (store_rounded) xj = round_z(xj, fmt);
      const cplx dx = {xj.re - xo.re, xj.im - xo.im};
      st(x, j, xj);
      dcdo_caxpy(-dx.re, -dx.im, hj, r, b);
      if (store_rounded) dcdo_round_precision(r, 2 * b, fmt);
    }
  }
  memcpy(x_out, x, sizeof(double) * 2 * (size_t)u);
  free(hs); free(r); free(m); free(nn); free(x);
  return 0;
}

/* detect.cpp:54-65 */
int dcdo_lmmse_exact(const double* h, int b, int u, const double* y, double n0, double ex,
                     double* x_out) {
  int rc = check_system(b, u, b, n0, ex);
  if (rc) return rc;
  double* a = gram(h, b, u);
  const double kappa = n0 / ex;
  for (int j = 0; j < u; ++j) a[2 * ((size_t)j * u + j)] += kappa;
  double* bb = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  for (int j = 0; j < u; ++j) st(bb, j, cdotc(h + 2 * (size_t)j * b, y, b));
  rc = dcdo_hermitian_solve(a, u, bb, x_out);
  free(a); free(bb);
  return rc;
}

/* detect.cpp:112-130 */
int dcdo_post_eq_variance(const double* h, int b, int u, double n0, double ex, double* out) {
  if (b == 0 || u == 0) return fail(EINVAL_, "post_eq_variance: empty channel block");
  if (!(n0 > 0.0) || !(ex > 0.0)) return fail(EINVAL_, "post_eq_variance: need N0 > 0 and E_x > 0");
  double* a = gram(h, b, u);
  const double g = ex / n0;
  for (int j = 0; j < u; ++j)
    for (int i = 0; i < u; ++i) {
      const size_t k = (size_t)j * u + i;
      a[2 * k] = (i == j ? 1.0 : 0.0) + g * a[2 * k];
      a[2 * k + 1] = g * a[2 * k + 1];
    }
  double tr = 0.0;
  double* e = (double*)calloc(2 * (size_t)u, sizeof(double));
  double* sol = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  int rc = 0;
  for (int j = 0; j < u && !rc; ++j) {
    e[2 * j] = 1.0;
    rc = dcdo_hermitian_solve(a, u, e, sol);
    if (!rc) tr += sol[2 * j];
    e[2 * j] = 0.0;
  }
  free(a); free(e); free(sol);
  if (rc) return rc;
  *out = ex / (double)u * tr;
  return 0;
}

/* detect.cpp:132-145 */
int dcdo_fusion_weights(const double* s2, int c, double* w) {
  if (c == 0) return fail(EINVAL_, "fusion_weights: no clusters");
  double total = 0.0;
  for (int k = 0; k < c; ++k) {
    if (!(s2[k] > 0.0) || !isfinite(s2[k]))
      return fail(EINVAL_, "fusion_weights: variances must be positive and finite");
    w[k] = 1.0 / s2[k];
    total += w[k];
  }
  for (int k = 0; k < c; ++k) w[k] /= total;
  return 0;
}

/* detect.cpp:227-242 */
int dcdo_mmse_bias_factors(const double* h, int b, int u, double n0, double ex, double* beta) {
  int rc = check_system(b, u, b, n0, ex);
  if (rc) return rc;
  for (int j = 0; j < u; ++j) beta[j] = 1.0;
  const double kappa = n0 / ex;
  if (kappa == 0.0) return 0;
  double* a = gram(h, b, u);
  for (int j = 0; j < u; ++j) a[2 * ((size_t)j * u + j)] += kappa;
  double* e = (double*)calloc(2 * (size_t)u, sizeof(double));
  double* sol = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  for (int j = 0; j < u && !rc; ++j) {
    e[2 * j] = 1.0;
    rc = dcdo_hermitian_solve(a, u, e, sol);
    if (!rc) beta[j] = 1.0 - kappa * sol[2 * j];
    e[2 * j] = 0.0;
  }
  free(a); free(e); free(sol);
  return rc;
}

/* detect.cpp:147-189 (sequential worker order; the reference's concurrent
 * mode is bitwise identical, test_detect.cpp:361-379) */
int dcdo_decentralized_cd_detect(int nc, const int* bc, int u, const double* h_tiles,
                                 const double* y, double n0, double ex, unsigned t_max,
                                 int fusion, int fmt, int scope, double* xhat, double* local,
                                 double* sigma2, double* weights) {
  if (nc == 0) return fail(EINVAL_, "decentralized_cd_detect: no clusters");
  const int optimal = fusion == DCDO_FUSION_OPTIMAL;
  double* loc = (double*)malloc(sizeof(double) * 2 * (size_t)nc * u);
  double* s2 = (double*)calloc((size_t)nc, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (size_t)nc);
  size_t ho = 0, yo = 0;
  int rc = 0;
  for (int c = 0; c < nc && !rc; ++c) {
    double* est = loc + 2 * (size_t)c * u;
    rc = dcdo_cd_detect(h_tiles + 2 * ho, bc[c], u, y + 2 * yo, n0, ex, t_max, fmt, scope, est);
    if (!rc && optimal) rc = dcdo_post_eq_variance(h_tiles + 2 * ho, bc[c], u, n0, ex, &s2[c]);
    if (!rc && fmt != DCDO_FP64) {
      dcdo_round_precision(est, 2 * u, fmt);
      if (optimal) dcdo_round_precision(&s2[c], 1, fmt);
    }
    ho += (size_t)bc[c] * u;
    yo += (size_t)bc[c];
  }
  if (!rc) {
    if (optimal) rc = dcdo_fusion_weights(s2, nc, w);
    else
      for (int c = 0; c < nc; ++c) w[c] = 1.0 / (double)nc;
  }
  if (!rc) {
    for (int j = 0; j < u; ++j) {
      xhat[2 * j] = w[0] * loc[2 * j];
      xhat[2 * j + 1] = w[0] * loc[2 * j + 1];
    }
    for (int c = 1; c < nc; ++c)
      for (int j = 0; j < u; ++j) {
        xhat[2 * j] += w[c] * loc[2 * ((size_t)c * u + j)];
        xhat[2 * j + 1] += w[c] * loc[2 * ((size_t)c * u + j) + 1];
      }
    if (local) memcpy(local, loc, sizeof(double) * 2 * (size_t)nc * u);
    if (sigma2 && optimal) memcpy(sigma2, s2, sizeof(double) * (size_t)nc);
    if (weights) memcpy(weights, w, sizeof(double) * (size_t)nc);
  }
  free(loc); free(s2); free(w);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* downlink — src/precode.cpp                                                */
/* ------------------------------------------------------------------------ */
/* precode.cpp:52-99 (rows = conj_rows(h_dl), precode.cpp:19-27) */
int dcdo_cd_precode(const double* h_dl, int u, int b, const double* s, unsigned t_max,
                    int fmt, int scope, double* x_out) {
  if (u == 0 || b == 0) return fail(EINVAL_, "precoder: empty channel matrix");
  if (t_max == 0) return fail(EINVAL_, "cd_precode: need at least one sweep");
  const int store_rounded = fmt != DCDO_FP64 && scope == DCDO_FULL_STORAGE;
  const size_t hn = (size_t)u * b;
  double* hs = (double*)malloc(sizeof(double) * 2 * hn);
  double* sb = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  double* rows = (double*)malloc(sizeof(double) * 2 * hn); /* [u][b] */
  double* p = (double*)malloc(sizeof(double) * (size_t)u);
  double* x = (double*)calloc(2 * (size_t)b, sizeof(double));
  memcpy(hs, h_dl, sizeof(double) * 2 * hn);
  memcpy(sb, s, sizeof(double) * 2 * (size_t)u);
  if (store_rounded) {
    dcdo_round_precision(hs, 2 * (int)hn, fmt);
    dcdo_round_precision(sb, 2 * u, fmt);
  }
  for (int j = 0; j < b; ++j)
    for (int i = 0; i < u; ++i) st(rows, (size_t)i * b + j, conjz(ld(hs, (size_t)j * u + i)));
  int rc = 0;
  for (int i = 0; i < u; ++i) {
    const double e = dcdo_norm2sq(rows + 2 * (size_t)i * b, b);
    if (e == 0.0) {
      rc = fail(ERUNTIME_, "cd_precode: user %d has an all-zero channel row", i);
      break;
    }
    p[i] = 1.0 / sqrt(e);
  }
  if (!rc) {
    if (store_rounded) dcdo_round_precision(p, u, fmt);
    for (int i = 0; i < u; ++i) {
      double* ri = rows + 2 * (size_t)i * b;
      for (int j = 0; j < 2 * b; ++j) ri[j] *= p[i];
      sb[2 * i] *= p[i];
      sb[2 * i + 1] *= p[i];
      if (store_rounded) {
        dcdo_round_precision(ri, 2 * b, fmt);
        dcdo_round_precision(sb + 2 * i, 2, fmt);
      }
    }
    for (unsigned t = 0; t < t_max; ++t)
      for (int i = 0; i < u; ++i) {
        const double* ri = rows + 2 * (size_t)i * b;
        const cplx d = cdotc(ri, x, b);
        const cplx resid = {d.re - sb[2 * i], d.im - sb[2 * i + 1]};
        dcdo_caxpy(-resid.re, -resid.im, ri, x, b);
        if (store_rounded) dcdo_round_precision(x, 2 * b, fmt);
      }
    memcpy(x_out, x, sizeof(double) * 2 * (size_t)b);
  }
  free(hs); free(sb); free(rows); free(p); free(x);
  return rc;
}

/* precode.cpp:31-50 */
int dcdo_zf_exact(const double* h_dl, int u, int b, const double* s, double* x_out) {
  if (u == 0 || b == 0) return fail(EINVAL_, "precoder: empty channel matrix");
  double* rows = (double*)malloc(sizeof(double) * 2 * (size_t)u * b);
  for (int j = 0; j < b; ++j)
    for (int i = 0; i < u; ++i) st(rows, (size_t)i * b + j, conjz(ld(h_dl, (size_t)j * u + i)));
  double* a = (double*)malloc(sizeof(double) * 2 * (size_t)u * u);
  for (int j = 0; j < u; ++j)
    for (int i = 0; i < u; ++i)
      st(a, (size_t)j * u + i, cdotc(rows + 2 * (size_t)i * b, rows + 2 * (size_t)j * b, b));
  double* z = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  int rc = dcdo_hermitian_solve(a, u, s, z);
  if (rc == ERUNTIME_) rc = fail(ERUNTIME_, "zf_exact: channel rows are rank deficient");
  if (!rc)
    for (int j = 0; j < b; ++j) st(x_out, j, cdotc(h_dl + 2 * (size_t)j * u, z, u));
  free(rows); free(a); free(z);
  return rc;
}

/* precode.cpp:101-111 */
int dcdo_power_scale(double* x, int n, double rho) {
  if (!(rho > 0.0)) return fail(EINVAL_, "power_scale: amplitude must be positive");
  if (n == 0) return fail(EINVAL_, "power_scale: empty beamformer");
  const double n2 = dcdo_norm2sq(x, n);
  if (n2 == 0.0) return fail(ERUNTIME_, "power_scale: zero beamformer cannot be scaled");
  const double g = rho / sqrt(n2);
  for (int i = 0; i < 2 * n; ++i) x[i] *= g;
  return 0;
}

/* precode.cpp:136-169 + assemble_blocks precode.cpp:115-132 */
int dcdo_decentralized_cd_precode(int nc, const int* bc, int u, const double* hdl_tiles,
                                  const double* s, double rho, unsigned t_max, int fmt,
                                  int scope, double* x, double* gain) {
  if (nc == 0) return fail(EINVAL_, "decentralized_cd_precode: no clusters");
  for (int c = 0; c < nc; ++c)
    if (bc[c] < u)
      return fail(EINVAL_,
                  "decentralized_cd_precode: cluster %d has %d antennas for %d users; local "
                  "zero-forcing needs B_c >= U",
                  c, bc[c], u);
  const double rho_c = rho / sqrt((double)nc);
  double* s_msg = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  memcpy(s_msg, s, sizeof(double) * 2 * (size_t)u);
  if (fmt != DCDO_FP64) dcdo_round_precision(s_msg, 2 * u, fmt);
  double* combined = (double*)calloc(2 * (size_t)u, sizeof(double));
  size_t ho = 0, xo = 0;
  int rc = 0;
  for (int c = 0; c < nc && !rc; ++c) {
    double* xc = x + 2 * xo;
    const double* hc = hdl_tiles + 2 * ho;
    rc = dcdo_cd_precode(hc, u, bc[c], s_msg, t_max, fmt, scope, xc);
    if (!rc) rc = dcdo_power_scale(xc, bc[c], rho_c);
    if (!rc) {
      /* matvec (numerics.cpp:21-28): y += x_j * col_j in ascending j */
      double* yc = (double*)calloc(2 * (size_t)u, sizeof(double));
      for (int j = 0; j < bc[c]; ++j) dcdo_caxpy(xc[2 * j], xc[2 * j + 1], hc + 2 * (size_t)j * u, yc, u);
      for (int i = 0; i < 2 * u; ++i) combined[i] += yc[i];
      free(yc);
    }
    ho += (size_t)bc[c] * u;
    xo += (size_t)bc[c];
  }
  if (!rc && gain) {
    const double se = dcdo_norm2sq(s, u);
    *gain = 0.0;
    if (se > 0.0) *gain = cdotc(s, combined, u).re / se;
  }
  free(s_msg); free(combined);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* batched helpers over the device batch layout                              */
/* ------------------------------------------------------------------------ */
int dcdo_ul_detect_batch(int S, int C, int bc, int u, const double* h_tiles, const double* y,
                         double n0, double ex, unsigned t_max, int fusion, int fmt, int scope,
                         double* xhat, double* local, double* sigma2) {
  int* sizes = (int*)malloc(sizeof(int) * (size_t)C);
  for (int c = 0; c < C; ++c) sizes[c] = bc;
  const size_t tile = (size_t)bc * u;
  int rc = 0;
  for (int s = 0; s < S && !rc; ++s)
    rc = dcdo_decentralized_cd_detect(C, sizes, u, h_tiles + 2 * tile * C * s,
                                      y + 2 * (size_t)bc * C * s, n0, ex, t_max, fusion, fmt,
                                      scope, xhat + 2 * (size_t)u * s,
                                      local ? local + 2 * (size_t)u * C * s : NULL,
                                      sigma2 ? sigma2 + (size_t)C * s : NULL, NULL);
  free(sizes);
  return rc;
}

int dcdo_dl_precode_batch(int S, int C, int bc, int u, const double* h_tiles, const double* sym,
                          double rho, unsigned t_max, int fmt, int scope, double* x_dl,
                          double* gain) {
  int* sizes = (int*)malloc(sizeof(int) * (size_t)C);
  for (int c = 0; c < C; ++c) sizes[c] = bc;
  const size_t tile = (size_t)bc * u;
  double* hdl = (double*)malloc(sizeof(double) * 2 * tile * C);
  int rc = 0;
  for (int s = 0; s < S && !rc; ++s) {
    /* reciprocity: H_dl,c = H_ul,c^H (src/cluster.cpp:246-248) */
    for (int c = 0; c < C; ++c) {
      const double* t = h_tiles + 2 * tile * ((size_t)C * s + c);
      double* d = hdl + 2 * tile * c;
      for (int j = 0; j < u; ++j)
        for (int i = 0; i < bc; ++i) st(d, (size_t)i * u + j, conjz(ld(t, (size_t)j * bc + i)));
    }
    double g = 0.0;
    rc = dcdo_decentralized_cd_precode(C, sizes, u, hdl, sym + 2 * (size_t)u * s, rho, t_max, fmt,
                                       scope, x_dl + 2 * (size_t)bc * C * s, &g);
    if (gain) gain[s] = g;
  }
  free(hdl);
  free(sizes);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* RNG — src/rng.cpp (std::mt19937_64 + splitmix64 keys + Box-Muller)        */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int has_spare;
  uint64_t bit_buffer;
  int bits_left;
} rng_t;

static void mt_seed(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->has_spare = 0;
  r->spare = 0.0;
  r->bit_buffer = 0;
  r->bits_left = 0;
}

static uint64_t mt_next(rng_t* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.cpp:8-13 */
uint64_t dcdo_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.cpp:15-17 */
uint64_t dcdo_derive_seed(uint64_t master, uint64_t purpose, uint64_t index) {
  return dcdo_mix64(dcdo_mix64(dcdo_mix64(master) ^ purpose) ^ index);
}

/* rng.cpp:19-21 */
static double uniform01(rng_t* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* rng.cpp:23-36 */
static double gaussian(rng_t* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = uniform01(r);
  const double u2 = uniform01(r);
  if (u1 < 0x1.0p-100) u1 = 0x1.0p-100;
  const double rr = sqrt(-2.0 * log(u1));
  const double t = 2.0 * 3.141592653589793238462643383279502884 * u2;
  r->spare = rr * sin(t);
  r->has_spare = 1;
  return rr * cos(t);
}

/* rng.cpp:38-43 */
static cplx cgaussian(rng_t* r, double var) {
  const double s = sqrt(var / 2.0);
  const double re = gaussian(r);
  const double im = gaussian(r);
  cplx z = {s * re, s * im};
  return z;
}

/* rng.cpp:45-54 */
static unsigned rbit(rng_t* r) {
  if (r->bits_left == 0) {
    r->bit_buffer = mt_next(r);
    r->bits_left = 64;
  }
  const unsigned b = (unsigned)(r->bit_buffer & 1u);
  r->bit_buffer >>= 1;
  --r->bits_left;
  return b;
}

void dcdo_rng_draw(uint64_t seed, int kind, int n, double* out) {
  rng_t r;
  mt_seed(&r, seed);
  for (int i = 0; i < n; ++i)
    out[i] = kind == 0 ? uniform01(&r) : kind == 1 ? gaussian(&r) : (double)rbit(&r);
}

/* ------------------------------------------------------------------------ */
/* system model — src/mimo.cpp, src/cluster.cpp                              */
/* ------------------------------------------------------------------------ */
enum { P_CHANNEL = 1, P_NOISE = 2, P_BITS = 3, P_GENERIC = 4 }; /* rng.hpp:20-25 */

/* mimo.cpp:64-109 */
int dcdo_qam_points(unsigned order, double ex, double* pts) {
  if (order != 4 && order != 16 && order != 64)
    return fail(EINVAL_, "Constellation::qam: order must be 4, 16 or 64");
  if (!(ex > 0.0)) return fail(EINVAL_, "Constellation::qam: symbol energy must be positive");
  unsigned levels = 2, bits = 2;
  while (levels * levels < order) {
    levels <<= 1;
    bits += 2;
  }
  const unsigned axis_bits = bits / 2;
  const double scale = sqrt(3.0 * ex / (2.0 * (levels * levels - 1.0)));
  double level_of_label[8];
  for (unsigned pos = 0; pos < levels; ++pos)
    level_of_label[pos ^ (pos >> 1)] = scale * (2.0 * pos - (levels - 1.0));
  for (unsigned idx = 0; idx < order; ++idx) {
    pts[2 * idx] = level_of_label[idx >> axis_bits];
    pts[2 * idx + 1] = level_of_label[idx & (levels - 1)];
  }
  return 0;
}

/* mimo.cpp:111-122: nearest point, ties to the lowest index */
int dcdo_slice(unsigned order, double ex, const double* y, int n, unsigned* labels) {
  double pts[128];
  int rc = dcdo_qam_points(order, ex, pts);
  if (rc) return rc;
  for (int k = 0; k < n; ++k) {
    const double yr = y[2 * k], yi = y[2 * k + 1];
    unsigned best = 0;
    double dr = yr - pts[0], di = yi - pts[1];
    double best_d = dr * dr + di * di;
    for (unsigned i = 1; i < order; ++i) {
      dr = yr - pts[2 * i];
      di = yi - pts[2 * i + 1];
      const double d = dr * dr + di * di;
      if (d < best_d) {
        best_d = d;
        best = i;
      }
    }
    labels[k] = best;
  }
  return 0;
}

static unsigned bits_per_symbol(unsigned order) { return order == 4 ? 2 : order == 16 ? 4 : 6; }

/* cluster.cpp:80-105 with gen_rayleigh mimo.cpp:16-26 (uniform layout) */
int dcdo_make_batch(int nc, int bc, int u, unsigned qam, int count, uint64_t seed,
                    uint64_t first_trial, double* h_out, uint8_t* bits_out) {
  const int b = nc * bc;
  if (nc == 0 || b == 0) return fail(EINVAL_, "make_batch: empty layout");
  if (u == 0 || b < u) return fail(EINVAL_, "make_batch: need B >= U >= 1");
  if (qam != 4 && qam != 16 && qam != 64)
    return fail(EINVAL_, "Constellation::qam: order must be 4, 16 or 64");
  const unsigned bps = bits_per_symbol(qam);
  const size_t hb = (size_t)b * u;
  rng_t r;
  for (int s = 0; s < count; ++s) {
    const uint64_t trial = first_trial + (uint64_t)s;
    const uint64_t hseed = dcdo_derive_seed(seed, P_GENERIC, trial);
    mt_seed(&r, dcdo_derive_seed(hseed, P_CHANNEL, 0));
    double* h = h_out + 2 * hb * s;
    for (size_t k = 0; k < hb; ++k) st(h, k, cgaussian(&r, 1.0));
    mt_seed(&r, dcdo_derive_seed(seed, P_BITS, trial));
    for (unsigned k = 0; k < (unsigned)u * bps; ++k) bits_out[(size_t)u * bps * s + k] = (uint8_t)rbit(&r);
  }
  return 0;
}

/* cluster.cpp:152-155: y = awgn(matvec(H, modulate(bits)), n0, (seed, noise, trial)) */
int dcdo_uplink_observe(const double* h, int b, int u, const uint8_t* bits, unsigned qam,
                        double n0, uint64_t seed, uint64_t trial, double* y_out,
                        double* x_true_out) {
  double pts[128];
  int rc = dcdo_qam_points(qam, 1.0, pts);
  if (rc) return rc;
  if (n0 < 0.0) return fail(EINVAL_, "awgn: noise power must be nonnegative");
  const unsigned bps = bits_per_symbol(qam);
  double* x = (double*)malloc(sizeof(double) * 2 * (size_t)u);
  for (int k = 0; k < u; ++k) {
    unsigned label = 0;
    for (unsigned q = 0; q < bps; ++q) label = (label << 1) | bits[(size_t)k * bps + q];
    x[2 * k] = pts[2 * label];
    x[2 * k + 1] = pts[2 * label + 1];
  }
  memset(y_out, 0, sizeof(double) * 2 * (size_t)b);
  for (int j = 0; j < u; ++j) dcdo_caxpy(x[2 * j], x[2 * j + 1], h + 2 * (size_t)j * b, y_out, b);
  if (n0 != 0.0) {
    rng_t r;
    mt_seed(&r, dcdo_derive_seed(seed, P_NOISE, trial));
    for (int i = 0; i < b; ++i) {
      const cplx z = cgaussian(&r, n0);
      y_out[2 * i] += z.re;
      y_out[2 * i + 1] += z.im;
    }
  }
  if (x_true_out) memcpy(x_true_out, x, sizeof(double) * 2 * (size_t)u);
  free(x);
  return 0;
}

/* mimo.cpp:165-169 */
double dcdo_snr_to_n0(double snr_db, int users, double ex) {
  return (double)users * ex / pow(10.0, snr_db / 10.0);
}

/* mf_detect, detect.cpp:191-218 (messages in fp64: no rounding). Tiles back to
 * back, tile c is bc[c] x u column-major; ys concatenated. */
int dcdo_mf_detect(int nc, const int* bc, int u, const double* h_tiles, const double* ys, double* x_out) {
  if (nc == 0) return fail(EINVAL_, "mf_detect: no clusters");
  double* corr = (double*)calloc(2 * (size_t)u, sizeof(double));
  double* energy = (double*)calloc((size_t)u, sizeof(double));
  size_t ho = 0, yo = 0;
  for (int c = 0; c < nc; ++c) {
    for (int j = 0; j < u; ++j) {
      double pc[2];
      const double* col = h_tiles + 2 * (ho + (size_t)j * bc[c]);
      dcdo_cdotc(col, ys + 2 * yo, bc[c], pc);
      const double pe = dcdo_norm2sq(col, bc[c]);
      corr[2 * j] += pc[0];
      corr[2 * j + 1] += pc[1];
      energy[j] += pe;
    }
    ho += (size_t)bc[c] * u;
    yo += (size_t)bc[c];
  }
  int rc = 0;
  for (int j = 0; j < u && !rc; ++j) {
    if (energy[j] == 0.0) {
      rc = fail(ERUNTIME_, "mf_detect: user %d has zero channel energy", j);
      break;
    }
    x_out[2 * j] = corr[2 * j] / energy[j];
    x_out[2 * j + 1] = corr[2 * j + 1] / energy[j];
  }
  free(corr);
  free(energy);
  return rc;
}

/* mf_precode, precode.cpp:171-202 (fp64): x_c[j] = cdotc(h_dl,c col j, s),
 * power_scale(x_c, rho/sqrt(C)). Downlink tiles u x bc[c] column-major. */
int dcdo_mf_precode(int nc, const int* bc, int u, const double* hdl_tiles, const double* s, double rho, double* x) {
  if (nc == 0) return fail(EINVAL_, "mf_precode: no clusters");
  const double rho_c = rho / sqrt((double)nc);
  size_t ho = 0, xo = 0;
  for (int c = 0; c < nc; ++c) {
    double* xc = x + 2 * xo;
    for (int j = 0; j < bc[c]; ++j) dcdo_cdotc(hdl_tiles + 2 * (ho + (size_t)j * u), s, u, xc + 2 * j);
    if (dcdo_power_scale(xc, bc[c], rho_c)) return fail(ERUNTIME_, "mf_precode: cluster %d produced a zero beamformer", c);
    ho += (size_t)bc[c] * u;
    xo += (size_t)bc[c];
  }
  return 0;
}
