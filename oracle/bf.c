/* oracle/bf.c -- brute-force periodic potential sums (oracle step O12), plain C + OpenMP, fp64.
 * TEST INFRASTRUCTURE ONLY: called from oracle/bf.py, which only tests/, smoke() and bench.py's
 * cpu_baseline / reference legs may import.  Shares no code with the CUDA library.
 *
 *   u_t = sum_{s : t - s != 0} q_s G_p(t - s)                      (Eq. hms_d2)
 *
 * G_p is the static periodic Green's function of P:179-188 (Eq. 2 with k0 = 0), written as the
 * Ewald sums of SURVEY.md App. B with the normalisation of DESIGN.md reading R3 -- the same
 * formulas oracle/pgf.py evaluates in NumPy, restated here in C so that the O(N' x rows) pair
 * sums of the AIM-vs-brute-force checks (north_star: "the oracle's AIM must match brute force to
 * <= 1e-3") finish in seconds.  tests/test_oracle_bf.py pins this file against oracle/pgf.py and
 * against the closed forms (Madelung constants, 1D digamma form) directly.
 *
 *   real part (all dims): sum_n erfc(a|d + R_n|) / |d + R_n|
 *   3D: + (4 pi / V) sum_{k != 0} e^{-k^2/4a^2} / k^2 cos(k.d) - pi / (a^2 V)
 *   2D: + (pi / A) sum_{k != 0} cos(k.rho)/k [e^{kz} erfc(k/2a + az) + e^{-kz} erfc(k/2a - az)]
 *       - (2 pi / A) [z erf(az) + e^{-a^2 z^2} / (a sqrt(pi))]
 *   1D: + (2 / L) sum_{m >= 1} cos(k_m x) I(k_m^2/4a^2, rho^2 k_m^2/4)
 *       - (1 / L) [Ein(a^2 rho^2) - 2 ln(2 a L) + gamma],   I(a,b) = int_a^inf e^{-u - b/u} du/u
 * The 3D reciprocal part is summed through structure factors S(k) = sum_s q_s e^{i k.s} (the same
 * sum, reordered); 1D/2D reciprocal terms depend on the pair's free coordinates and are summed
 * pair by pair.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EULER_GAMMA 0.57721566490153286061
#define PI 3.14159265358979323846

typedef struct {
  int dim;          /* number of periodic axes (1, 2, 3) */
  int ax[3];        /* periodic axes first, then the free axes */
  double L[3];      /* periods of ax[0..dim-1] */
  double alpha;
  int nreal[3];     /* real-space image range per periodic axis */
  int mrec[3];      /* reciprocal range per periodic axis */
} bf_spec;

/* Gauss-Legendre nodes/weights on [-1, 1] (Newton on the Legendre recurrence) */
static void gauss_legendre(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = cos(PI * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 1; j <= n; ++j) {
        const double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
      }
      pp = n * (z * p0 - p1) / (z * z - 1.0);
      const double dz = p0 / pp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    x[i] = -z;
    w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

static double GL_X[64], GL_W[64];
static int gl_ready = 0;
static void gl_init(void) {
  if (!gl_ready) { gauss_legendre(64, GL_X, GL_W); gl_ready = 1; }
}

/* Ein(x) = int_0^x (1 - e^{-t}) / t dt = E1(x) + ln x + gamma (entire); series for x < 1,
 * 64-point Gauss-Legendre of the smooth integrand on [0, x] for 1 <= x <= 60, asymptote beyond */
static double ein(double x) {
  if (x < 1.0) {
    double term = 1.0, acc = 0.0;
    for (int k = 1; k < 40; ++k) {
      term *= x / k;
      acc += ((k & 1) ? 1.0 : -1.0) * term / k;
    }
    return acc;
  }
  if (x > 60.0) return log(x) + EULER_GAMMA;   /* E1(60) < 1e-28 */
  double acc = 0.0;
  for (int i = 0; i < 64; ++i) {
    const double t = 0.5 * x * (GL_X[i] + 1.0);
    acc += GL_W[i] * (1.0 - exp(-t)) / t;
  }
  return 0.5 * x * acc;
}

/* I(a, b) = int_a^inf exp(-u - b/u) du/u: u = a e^s, 64-point Gauss-Legendre on s in [0, S],
 * a e^S = 60 (the integrand is < e^-60 beyond) */
static double incomplete_bessel(double a, double b) {
  double S = log(60.0 / a);
  if (S < 0.5) S = 0.5;
  double acc = 0.0;
  for (int i = 0; i < 64; ++i) {
    const double s = 0.5 * S * (GL_X[i] + 1.0);
    const double u = a * exp(s);
    acc += GL_W[i] * exp(-u - b / u);
  }
  return 0.5 * S * acc;
}

/* e^{sgn k z} erfc(k/2a + sgn a z), overflow-safe: for w >= 0 through erfcx(w) e^{-k^2/4a^2 - a^2 z^2} */
static double erfcx_pos(double w) {   /* exp(w^2) erfc(w), w >= 0 */
  if (w < 25.0) return exp(w * w) * erfc(w);
  const double iw2 = 1.0 / (w * w);    /* asymptotic series, |error| < 1e-16 at w >= 25 */
  return (1.0 - 0.5 * iw2 * (1.0 - 1.5 * iw2 * (1.0 - 2.5 * iw2 * (1.0 - 3.5 * iw2)))) / (w * sqrt(PI));
}
static double bracket_term(double k, double z, double a, double sgn) {
  const double w = k / (2 * a) + sgn * a * z;
  if (w >= 0) return erfcx_pos(w) * exp(-k * k / (4 * a * a) - a * a * z * z);
  return exp(sgn * k * z) * erfc(w);
}

static double wrap_half(double x, double L) { return x - L * floor(x / L + 0.5); }

/* real-space image list: lattice vectors whose lower bound distance from a wrapped point is
 * within the cutoff rc = 6.2 / a (erfc(6.2) < 1e-17) */
typedef struct { int n; double* R; } img_list;
static img_list make_images(const bf_spec* s) {
  const double rc = 6.2 / s->alpha;
  int nr[3] = {0, 0, 0};
  for (int i = 0; i < s->dim; ++i) nr[i] = s->nreal[i];
  const int cnt = (2 * nr[0] + 1) * (2 * nr[1] + 1) * (2 * nr[2] + 1);
  img_list L;
  L.R = (double*)malloc(sizeof(double) * 3 * cnt);
  L.n = 0;
  for (int a = -nr[0]; a <= nr[0]; ++a)
    for (int b = -nr[1]; b <= nr[1]; ++b)
      for (int c = -nr[2]; c <= nr[2]; ++c) {
        const int n[3] = {a, b, c};
        double lb = 0.0;
        for (int i = 0; i < s->dim; ++i) {
          const double t = fabs((double)n[i]) - 0.5;
          if (t > 0) lb += t * t * s->L[i] * s->L[i];
        }
        if (lb > rc * rc) continue;
        for (int i = 0; i < 3; ++i) L.R[3 * L.n + i] = (i < s->dim) ? n[i] * s->L[i] : 0.0;
        ++L.n;
      }
  return L;
}

/* G_p(d) minus nothing, for d != 0 given in (periodic comps wrapped, free comps) order */
static double g_pair(const bf_spec* s, const img_list* im, const double* dp, const double* df, int with_recip3) {
  const double a = s->alpha;
  double out = 0.0;
  double f2 = 0.0;
  for (int i = 0; i < 3 - s->dim; ++i) f2 += df[i] * df[i];
  for (int j = 0; j < im->n; ++j) {
    double d2 = f2;
    for (int i = 0; i < s->dim; ++i) {
      const double t = dp[i] + im->R[3 * j + i];
      d2 += t * t;
    }
    if (d2 > 0.0) {
      const double r = sqrt(d2);
      out += erfc(a * r) / r;
    }
  }
  if (s->dim == 3) {
    (void)with_recip3;   /* 3D reciprocal part is added through structure factors */
  } else if (s->dim == 2) {
    const double A = s->L[0] * s->L[1], z = df[0];
    double acc = 0.0;
    for (int i = -s->mrec[0]; i <= s->mrec[0]; ++i)
      for (int j = -s->mrec[1]; j <= s->mrec[1]; ++j) {
        if (i == 0 && j == 0) continue;
        const double kx = 2 * PI * i / s->L[0], ky = 2 * PI * j / s->L[1];
        const double k = hypot(kx, ky);
        acc += cos(kx * dp[0] + ky * dp[1]) / k * (bracket_term(k, z, a, 1.0) + bracket_term(k, z, a, -1.0));
      }
    out += (PI / A) * acc;
    out += -(2 * PI / A) * (z * erf(a * z) + exp(-a * a * z * z) / (a * sqrt(PI)));
  } else {
    const double L = s->L[0];
    const double rho2 = f2, x = dp[0];
    double acc = 0.0;
    for (int m = 1; m <= s->mrec[0]; ++m) {
      const double km = 2 * PI * m / L;
      acc += cos(km * x) * incomplete_bessel(km * km / (4 * a * a), rho2 * km * km / 4.0);
    }
    out += (2.0 / L) * acc;
    out += -(1.0 / L) * (ein(a * a * rho2) - 2.0 * log(2 * a * L) + EULER_GAMMA);
  }
  return out;
}

static void split(const bf_spec* s, const double* t, const double* src, double* dp, double* df) {
  for (int i = 0; i < s->dim; ++i) dp[i] = wrap_half(t[s->ax[i]] - src[s->ax[i]], s->L[i]);
  for (int i = s->dim; i < 3; ++i) df[i - s->dim] = t[s->ax[i]] - src[s->ax[i]];
}

/* Single-point evaluation G_p(r), r != 0 (pins against oracle/pgf.py and closed forms).
 * self_term = 1: the regularised self value G_p^reg(0) = lim [G_p(r) - 1/r] (r ignored). */
int bf_pgf_points(const bf_spec* s, int64_t n, const double* r, int self_term, double* out) {
  gl_init();
  img_list im = make_images(s);
  const double a = s->alpha;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t p = 0; p < n; ++p) {
    double dp[3] = {0, 0, 0}, df[3] = {0, 0, 0};
    const double zero[3] = {0, 0, 0};
    split(s, self_term ? zero : &r[3 * p], zero, dp, df);
    double v = g_pair(s, &im, dp, df, 0);      /* d = 0 skips the n = 0 image in the real part */
    if (self_term) v += -2.0 * a / sqrt(PI);
    if (s->dim == 3) {
      const double V = s->L[0] * s->L[1] * s->L[2];
      double acc = 0.0;
      for (int i = -s->mrec[0]; i <= s->mrec[0]; ++i)
        for (int j = -s->mrec[1]; j <= s->mrec[1]; ++j)
          for (int k = -s->mrec[2]; k <= s->mrec[2]; ++k) {
            if (!i && !j && !k) continue;
            const double kx = 2 * PI * i / s->L[0], ky = 2 * PI * j / s->L[1], kz = 2 * PI * k / s->L[2];
            const double k2 = kx * kx + ky * ky + kz * kz;
            acc += exp(-k2 / (4 * a * a)) / k2 * cos(kx * dp[0] + ky * dp[1] + kz * dp[2]);
          }
      v += (4 * PI / V) * acc - PI / (a * a * V);
    }
    out[p] = v;
  }
  free(im.R);
  return 0;
}

/* u_t = sum_{s : t != s} q_s G_p(t - s) for nt targets and ns sources ([n][3] fp64, cm). */
int bf_potential(const bf_spec* s, int64_t nt, const double* targets, int64_t ns, const double* sources,
                 const double* q, double* out) {
  gl_init();
  img_list im = make_images(s);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < nt; ++t) {
    const double* tp = &targets[3 * t];
    double acc = 0.0;
    for (int64_t k = 0; k < ns; ++k) {
      const double* sp = &sources[3 * k];
      if (tp[0] == sp[0] && tp[1] == sp[1] && tp[2] == sp[2]) continue;
      double dp[3], df[3];
      split(s, tp, sp, dp, df);
      acc += q[k] * g_pair(s, &im, dp, df, 0);
    }
    out[t] = acc;
  }
  free(im.R);
  if (s->dim != 3) return 0;
  /* 3D reciprocal part: (4 pi / V) sum_k c_k Re[e^{i k.t} conj(S(k))] - pi/(a^2 V) sum q,
   * S(k) = sum_s q_s e^{i k.s}; pairs with t == s are removed afterwards */
  const double a = s->alpha, V = s->L[0] * s->L[1] * s->L[2];
  const int M0 = s->mrec[0], M1 = s->mrec[1], M2 = s->mrec[2];
  const int W0 = 2 * M0 + 1, W1 = 2 * M1 + 1, W2 = 2 * M2 + 1;
  if (W0 > 64 || W1 > 64 || W2 > 64) return 1;
  const int64_t K = (int64_t)W0 * W1 * W2;
  double* Sre = (double*)calloc(K, sizeof(double));
  double* Sim = (double*)calloc(K, sizeof(double));
#pragma omp parallel
  {
    double* lre = (double*)calloc(K, sizeof(double));
    double* lim = (double*)calloc(K, sizeof(double));
    double ex[2][64], ey[2][64], ez[2][64];
#pragma omp for schedule(static)
    for (int64_t k = 0; k < ns; ++k) {
      const double* sp = &sources[3 * k];
      for (int i = 0; i < W0; ++i) { const double ph = 2 * PI * (i - M0) / s->L[0] * sp[0]; ex[0][i] = cos(ph); ex[1][i] = sin(ph); }
      for (int i = 0; i < W1; ++i) { const double ph = 2 * PI * (i - M1) / s->L[1] * sp[1]; ey[0][i] = cos(ph); ey[1][i] = sin(ph); }
      for (int i = 0; i < W2; ++i) { const double ph = 2 * PI * (i - M2) / s->L[2] * sp[2]; ez[0][i] = cos(ph); ez[1][i] = sin(ph); }
      for (int i = 0; i < W0; ++i)
        for (int j = 0; j < W1; ++j) {
          const double xr = ex[0][i] * ey[0][j] - ex[1][i] * ey[1][j];
          const double xi = ex[0][i] * ey[1][j] + ex[1][i] * ey[0][j];
          const int64_t b = ((int64_t)i * W1 + j) * W2;
          for (int l = 0; l < W2; ++l) {
            lre[b + l] += q[k] * (xr * ez[0][l] - xi * ez[1][l]);
            lim[b + l] += q[k] * (xr * ez[1][l] + xi * ez[0][l]);
          }
        }
    }
#pragma omp critical
    for (int64_t i = 0; i < K; ++i) { Sre[i] += lre[i]; Sim[i] += lim[i]; }
    free(lre); free(lim);
  }
  double* coef = (double*)calloc(K, sizeof(double));
  double csum = 0.0, qsum = 0.0;
  for (int i = 0; i < W0; ++i)
    for (int j = 0; j < W1; ++j)
      for (int l = 0; l < W2; ++l) {
        if (i == M0 && j == M1 && l == M2) continue;
        const double kx = 2 * PI * (i - M0) / s->L[0], ky = 2 * PI * (j - M1) / s->L[1], kz = 2 * PI * (l - M2) / s->L[2];
        const double k2 = kx * kx + ky * ky + kz * kz;
        const double c = (4 * PI / V) * exp(-k2 / (4 * a * a)) / k2;
        coef[((int64_t)i * W1 + j) * W2 + l] = c;
        csum += c;
      }
  for (int64_t k = 0; k < ns; ++k) qsum += q[k];
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < nt; ++t) {
    const double* tp = &targets[3 * t];
    double acc = 0.0;
    for (int i = 0; i < W0; ++i)
      for (int j = 0; j < W1; ++j)
        for (int l = 0; l < W2; ++l) {
          const int64_t b = ((int64_t)i * W1 + j) * W2 + l;
          if (coef[b] == 0.0) continue;
          const double ph = 2 * PI * ((i - M0) / s->L[0] * tp[0] + (j - M1) / s->L[1] * tp[1] + (l - M2) / s->L[2] * tp[2]);
          /* Re[e^{i k.t} conj(S)] = cos(ph) Sre + sin(ph) Sim */
          acc += coef[b] * (cos(ph) * Sre[b] + sin(ph) * Sim[b]);
        }
    acc += -PI / (a * a * V) * qsum;
    /* remove the pairs t == s (they belong to the self term) */
    double qs = 0.0;
    for (int64_t k = 0; k < ns; ++k) {
      const double* sp = &sources[3 * k];
      if (tp[0] == sp[0] && tp[1] == sp[1] && tp[2] == sp[2]) qs += q[k];
    }
    acc -= qs * (csum - PI / (a * a * V));
    out[t] += acc;
  }
  free(Sre); free(Sim); free(coef);
  return 0;
}
