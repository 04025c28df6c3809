// Host side of the PGF build: Ewald parameters, Gauss-Legendre nodes, and (host-only
// contexts) the fp64 kernel table + spectrum with a plain radix-2 FFT.  Device contexts build
// the same table on the GPU (device.cu: k_pgf_table + fp64 FFT passes).
//   P:179-188 Eq. 2 (k0 = 0); P:204 K on grid displacements; P:214 G0 -> G_p in step 2.
#include <algorithm>
#include <cmath>
#include <complex>
#include <omp.h>
#include "pmfem_internal.h"
#include "pgf.cuh"

namespace pmfem {

void gauss_legendre01(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1, p1 = z;
      for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      dp = n * (z * p1 - p0) / (z * z - 1);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1, p1 = z;
    for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
    dp = n * (z * p1 - p0) / (z * z - 1);
    x[i] = 0.5 * (1 - z);
    w[i] = 1.0 / ((1 - z * z) * dp * dp);
  }
}

PgfParams make_pgf_params(const int periodic[3], const double L[3], double target) {
  PgfParams P{};
  int k = 0;
  for (int a = 0; a < 3; ++a)
    if (periodic[a]) { P.ax[k] = a; P.L[k] = L[a]; ++k; }
  P.dim = k;
  for (int a = 0; a < 3; ++a)
    if (!periodic[a]) P.ax[k++] = a;
  double Lmin = 1e300;
  for (int i = 0; i < P.dim; ++i) Lmin = std::min(Lmin, P.L[i]);
  P.alpha = P.dim > 0 ? std::sqrt(M_PI) / Lmin : 1.0;   // dim 0: free space, alpha unused
  const double tol = 1e-2 * std::min(std::max(target, 1e-16), 1e-2);
  P.xr = 1.0;
  while (std::erfc(P.xr) > tol && P.xr < 7.0) P.xr += 0.05;
  const double kmax = 2.0 * P.alpha * std::sqrt(-std::log(tol)) * 1.1;
  for (int i = 0; i < 3; ++i) {
    if (i < P.dim) {
      P.nreal[i] = (int)std::ceil(P.xr / (P.alpha * P.L[i]) + 1.0);
      P.mrec[i] = (int)std::ceil(kmax * P.L[i] / (2 * M_PI)) + 1;
    } else {
      P.nreal[i] = 0;
      P.mrec[i] = 0;
    }
  }
  return P;
}

static PgfDev to_dev(const PgfParams& P) {
  PgfDev d{};
  d.dim = P.dim;
  for (int i = 0; i < 3; ++i) { d.ax[i] = P.ax[i]; d.L[i] = P.L[i]; d.nreal[i] = P.nreal[i]; d.mrec[i] = P.mrec[i]; }
  d.alpha = P.alpha;
  d.xr = P.xr;
  gauss_legendre01(64, d.gl_x, d.gl_w);
  return d;
}

double pgf_truncation_error(const HostSetup& S, const PgfParams& P) {
  if (P.dim == 0) return 0.0;
  PgfParams Q = P;                     // enlarged cutoffs: +1.5 in alpha r_c, +2 shells each way
  Q.xr = P.xr + 1.5;
  for (int i = 0; i < P.dim; ++i) {
    Q.nreal[i] = (int)std::ceil(Q.xr / (Q.alpha * Q.L[i]) + 1.0);
    Q.mrec[i] = P.mrec[i] + 2 + P.mrec[i] / 2;
  }
  const PgfDev a = to_dev(P), b = to_dev(Q);
  // probes: the self value and 63 grid displacements j = (u_a (N_a - 1)) on a scrambled
  // lattice of fractions u in (0, 1) (Weyl sequence), covering near and far displacements
  double dmax = 0.0, kmax = 0.0;
  for (int t = 0; t < 64; ++t) {
    double r[3];
    for (int x = 0; x < 3; ++x) {
      const double u = std::fmod(0.5 + t * (x == 0 ? 0.7548776662 : x == 1 ? 0.5698402910 : 0.3319573700), 1.0);
      const int j = (int)std::floor(u * S.grid_n[x]);
      r[x] = j * S.delta[x];
    }
    const bool self = t == 0;
    if (!self && r[0] == 0 && r[1] == 0 && r[2] == 0) continue;
    const double ka = pgf_eval(a, r, self), kb = pgf_eval(b, r, self);
    dmax = std::max(dmax, std::fabs(ka - kb));
    kmax = std::max(kmax, std::fabs(kb));
  }
  // nothing is resolved below the fp64 unit roundoff: report at least DBL_EPSILON
  return std::max(kmax > 0 ? dmax / kmax : 0.0, 2.220446049250313e-16);
}

void host_kernel_table(const HostSetup& S, const PgfParams& P, std::vector<double>& K) {
  const PgfDev pd = to_dev(P);
  const int P0 = S.fft_n[0], P1 = S.fft_n[1], P2 = S.fft_n[2];
  const int64_t tot = (int64_t)P0 * P1 * P2;
  K.assign(tot, 0.0);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t idx = 0; idx < tot; ++idx) {
    int j[3] = {(int)(idx % P0), (int)((idx / P0) % P1), (int)(idx / ((int64_t)P0 * P1))};
    bool skip = false;
    double r[3];
    for (int a = 0; a < 3; ++a) {
      if (!S.periodic[a] && j[a] == S.grid_n[a]) skip = true;
      int jj = S.periodic[a] ? j[a] : (j[a] < S.grid_n[a] ? j[a] : j[a] - S.fft_n[a]);
      r[a] = jj * S.delta[a];
    }
    if (skip) continue;
    bool self = (j[0] == 0 && j[1] == 0 && j[2] == 0);
    K[idx] = pgf_eval(pd, r, self);
  }
}

void fft1d(std::complex<double>* x, int n, int stride) {
  // iterative radix-2 DIT, forward (exp(-2 pi i k j / n))
  int logn = 0;
  while ((1 << logn) < n) ++logn;
  for (int i = 0, j = 0; i < n; ++i) {
    if (i < j) std::swap(x[i * stride], x[j * stride]);
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
  }
  for (int len = 2; len <= n; len <<= 1) {
    double ang = -2 * M_PI / len;
    for (int i = 0; i < n; i += len)
      for (int k = 0; k < len / 2; ++k) {
        std::complex<double> w(std::cos(ang * k), std::sin(ang * k));
        std::complex<double> u = x[(i + k) * stride], v = w * x[(i + k + len / 2) * stride];
        x[(i + k) * stride] = u + v;
        x[(i + k + len / 2) * stride] = u - v;
      }
  }
}

void host_fft_spectrum(const HostSetup& S, const std::vector<double>& K, std::vector<double>& Ghat) {
  const int P0 = S.fft_n[0], P1 = S.fft_n[1], P2 = S.fft_n[2];
  const int64_t tot = (int64_t)P0 * P1 * P2;
  std::vector<std::complex<double>> c(K.begin(), K.end());
#pragma omp parallel for
  for (int64_t r = 0; r < (int64_t)P1 * P2; ++r) fft1d(&c[r * P0], P0, 1);
#pragma omp parallel for
  for (int64_t r = 0; r < (int64_t)P0 * P2; ++r) {
    int64_t i2 = r / P0, i0 = r % P0;
    fft1d(&c[i2 * P0 * P1 + i0], P1, P0);
  }
#pragma omp parallel for
  for (int64_t r = 0; r < (int64_t)P0 * P1; ++r) fft1d(&c[r], P2, P0 * P1);
  const int H0 = P0 / 2 + 1;
  Ghat.assign((int64_t)H0 * P1 * P2, 0.0);
  for (int64_t i2 = 0; i2 < P2; ++i2)
    for (int64_t i1 = 0; i1 < P1; ++i1)
      for (int64_t i0 = 0; i0 < H0; ++i0)
        Ghat[(i2 * P1 + i1) * H0 + i0] = c[(i2 * P1 + i1) * P0 + i0].real() / (double)tot;
  Ghat[0] = 0.0;
}

}  // namespace pmfem

namespace pmfem {

// NEXT-4: the modulated Bloch kernel exp(j k0.r) G(r; k0) at every padded grid displacement
// (the same index -> displacement map as host_kernel_table), and its full complex spectrum
// (the kernel is not even: no half-spectrum) divided by the number of FFT points.
void bloch_grid_points(const HostSetup& S, int64_t idx, double r[3], bool& skip, bool& self) {
  const int P0 = S.fft_n[0], P1 = S.fft_n[1];
  const int j[3] = {(int)(idx % P0), (int)((idx / P0) % P1), (int)(idx / ((int64_t)P0 * P1))};
  skip = false;
  for (int a = 0; a < 3; ++a) {
    if (!S.periodic[a] && j[a] == S.grid_n[a]) skip = true;
    const int jj = S.periodic[a] ? j[a] : (j[a] < S.grid_n[a] ? j[a] : j[a] - S.fft_n[a]);
    r[a] = jj * S.delta[a];
  }
  self = j[0] == 0 && j[1] == 0 && j[2] == 0;
}

void host_bloch_table(const HostSetup& S, const PgfParams& P, const double k0[3], std::vector<double>& K) {
  const PgfDev pd = to_dev(P);
  const int64_t tot = (int64_t)S.fft_n[0] * S.fft_n[1] * S.fft_n[2];
  K.assign(2 * tot, 0.0);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t idx = 0; idx < tot; ++idx) {
    double r[3];
    bool skip, self;
    bloch_grid_points(S, idx, r, skip, self);
    if (skip) continue;
    const Cplx v = pgf_eval_bloch(pd, k0, r, self);
    K[2 * idx] = v.re;
    K[2 * idx + 1] = v.im;
  }
}

void host_bloch_spectrum(const HostSetup& S, const std::vector<double>& K, std::vector<double>& Gh) {
  const int P0 = S.fft_n[0], P1 = S.fft_n[1], P2 = S.fft_n[2];
  const int64_t tot = (int64_t)P0 * P1 * P2;
  std::vector<std::complex<double>> c(tot);
  for (int64_t i = 0; i < tot; ++i) c[i] = {K[2 * i], K[2 * i + 1]};
#pragma omp parallel for
  for (int64_t r = 0; r < (int64_t)P1 * P2; ++r) fft1d(&c[r * P0], P0, 1);
#pragma omp parallel for
  for (int64_t r = 0; r < (int64_t)P0 * P2; ++r) fft1d(&c[(r / P0) * P0 * P1 + r % P0], P1, P0);
#pragma omp parallel for
  for (int64_t r = 0; r < (int64_t)P0 * P1; ++r) fft1d(&c[r], P2, P0 * P1);
  Gh.assign(2 * tot, 0.0);
  for (int64_t i = 0; i < tot; ++i) { Gh[2 * i] = c[i].real() / (double)tot; Gh[2 * i + 1] = c[i].imag() / (double)tot; }
}

}  // namespace pmfem
