// Periodic Green's function G_p(r) = sum_images 1/|r - R| (Eq. 2, k0 = 0) by Ewald
// sums ("exponentially rapidly convergent sums"), fp64, host + device.
// Normalisation (reading R3): 3D zero cell mean (k = 0 dropped); 2D G + 2 pi |z|/A -> 0;
// 1D renormalised so that G_reg(0) = 0.  Self value G_reg(0) = lim_{r->0} G(r) - 1/r.
#pragma once
#include <cmath>

#ifdef __CUDACC__
#define PM_HD __host__ __device__
#else
#define PM_HD
#endif

namespace pmfem {

struct PgfDev {
  int dim;
  int ax[3];          // periodic axes first, then free axes
  double L[3];        // periods along ax[0..dim-1]
  double alpha;
  int nreal[3];       // real-space image range per periodic axis
  int mrec[3];        // reciprocal range per periodic axis
  double xr;          // real-space cutoff alpha * r_c (erfc(xr) below the truncation target)
  double gl_x[64], gl_w[64];   // Gauss-Legendre on [0,1] for the incomplete Bessel integral
};

PM_HD inline double pm_erfcx(double w) {
#ifdef __CUDA_ARCH__
  return erfcx(w);
#else
  if (w < 2.0) return std::exp(w * w) * std::erfc(w);
  // Laplace continued fraction: erfcx(w) = (1/sqrt(pi)) / (w + (1/2)/(w + 1/(w + (3/2)/(w + ...))))
  double f = w;
  for (int k = 60; k >= 1; --k) f = w + 0.5 * k / f;
  return 0.5641895835477563 / f;
#endif
}

// Ein(x) = E1(x) + ln x + gamma = sum_{k>=1} (-1)^{k+1} x^k / (k k!)
PM_HD inline double pm_ein(double x) {
  const double gamma_e = 0.57721566490153286061;
  if (x < 2.0) {
    double term = 1.0, acc = 0.0;
    for (int k = 1; k < 60; ++k) {
      term *= x / k;
      acc += ((k & 1) ? 1.0 : -1.0) * term / k;
      if (term < 1e-18 * fabs(acc)) break;
    }
    return acc;
  }
  // E1(x) by the continued fraction e^{-x} / (x + 1/(1 + 1/(x + 2/(1 + 2/(x + ...)))))  (Lentz)
  double b = x + 1.0, c = 1e300, d = 1.0 / b, h = d;
  for (int i = 1; i < 200; ++i) {
    double an = -(double)i * i;
    b += 2.0;
    d = 1.0 / (an * d + b);
    c = b + an / c;
    double del = c * d;
    h *= del;
    if (fabs(del - 1.0) < 1e-16) break;
  }
  double e1 = h * exp(-x);
  return e1 + log(x) + gamma_e;
}

// I(a,b) = int_a^inf exp(-u - b/u) du/u ; u = a e^s, s in [0, S], a e^S = 60
PM_HD inline double pm_incbessel(const PgfDev& P, double a, double b) {
  double S = log(60.0 / a);
  if (S < 0.5) S = 0.5;
  double acc = 0.0;
  for (int i = 0; i < 64; ++i) {
    double s = S * P.gl_x[i];
    double u = a * exp(s);
    acc += P.gl_w[i] * exp(-u - b / u);
  }
  return acc * S;
}

// r given in cartesian components; self = true returns G_reg(0) (r ignored).
PM_HD inline double pgf_eval(const PgfDev& P, const double r_in[3], bool self) {
  const double pi = 3.14159265358979323846;
  if (P.dim == 0)   // non-periodic mode (NEXT-3): G0 = 1/|r|, regularised self value 0
    return self ? 0.0 : 1.0 / sqrt(r_in[0] * r_in[0] + r_in[1] * r_in[1] + r_in[2] * r_in[2]);
  const double a = P.alpha;
  double rp[3] = {0, 0, 0}, rf[2] = {0, 0};
  for (int i = 0; i < P.dim; ++i) {
    double x = self ? 0.0 : r_in[P.ax[i]];
    double L = P.L[i];
    rp[i] = x - L * floor(x / L + 0.5);      // wrap into [-L/2, L/2)
  }
  for (int i = P.dim; i < 3; ++i) rf[i - P.dim] = self ? 0.0 : r_in[P.ax[i]];
  const double rf2 = rf[0] * rf[0] + rf[1] * rf[1];
  const double rc = P.xr / a;
  // real-space sum over pruned images
  double real = 0.0;
  int n0 = P.nreal[0], n1 = P.dim > 1 ? P.nreal[1] : 0, n2 = P.dim > 2 ? P.nreal[2] : 0;
  for (int i = -n0; i <= n0; ++i) {
    double lbi = fmax(0.0, fabs((double)i) - 0.5) * P.L[0];
    for (int j = -n1; j <= n1; ++j) {
      double lbj = P.dim > 1 ? fmax(0.0, fabs((double)j) - 0.5) * P.L[1] : 0.0;
      for (int k = -n2; k <= n2; ++k) {
        double lbk = P.dim > 2 ? fmax(0.0, fabs((double)k) - 0.5) * P.L[2] : 0.0;
        if (lbi * lbi + lbj * lbj + lbk * lbk > rc * rc) continue;
        if (self && i == 0 && j == 0 && k == 0) continue;
        double x = rp[0] + i * P.L[0];
        double y = rp[1] + (P.dim > 1 ? j * P.L[1] : 0.0);
        double z = rp[2] + (P.dim > 2 ? k * P.L[2] : 0.0);
        double d = sqrt(x * x + y * y + z * z + rf2);
        if (d > 0) real += erfc(a * d) / d;
      }
    }
  }
  double out = real;
  if (self) out += -2.0 * a / sqrt(pi);
  if (P.dim == 3) {
    const double V = P.L[0] * P.L[1] * P.L[2];
    double rec = 0.0;
    // half space: (mz > 0) or (mz == 0, my > 0) or (mz == my == 0, mx > 0); doubled
    for (int mz = 0; mz <= P.mrec[2]; ++mz) {
      double kz = 2 * pi * mz / P.L[2];
      for (int my = (mz == 0 ? 0 : -P.mrec[1]); my <= P.mrec[1]; ++my) {
        double ky = 2 * pi * my / P.L[1];
        for (int mx = ((mz == 0 && my == 0) ? 1 : -P.mrec[0]); mx <= P.mrec[0]; ++mx) {
          double kx = 2 * pi * mx / P.L[0];
          double k2 = kx * kx + ky * ky + kz * kz;
          double e = exp(-k2 / (4 * a * a));
          if (e < 1e-300) continue;
          rec += e / k2 * cos(kx * rp[0] + ky * rp[1] + kz * rp[2]);
        }
      }
    }
    out += 2.0 * rec * 4 * pi / V - pi / (a * a * V);
  } else if (P.dim == 2) {
    const double A = P.L[0] * P.L[1];
    const double z = rf[0];
    double rec = 0.0;
    for (int my = 0; my <= P.mrec[1]; ++my) {
      double ky = 2 * pi * my / P.L[1];
      for (int mx = (my == 0 ? 1 : -P.mrec[0]); mx <= P.mrec[0]; ++mx) {
        double kx = 2 * pi * mx / P.L[0];
        double k = sqrt(kx * kx + ky * ky);
        double br = 0.0;
        for (int sg = -1; sg <= 1; sg += 2) {
          double w = k / (2 * a) + sg * a * z;
          if (w >= 0) br += pm_erfcx(w) * exp(-k * k / (4 * a * a) - a * a * z * z);
          else br += exp(sg * k * z) * erfc(w);
        }
        rec += cos(kx * rp[0] + ky * rp[1]) / k * br;
      }
    }
    out += 2.0 * rec * pi / A;
    out += -(2 * pi / A) * (z * erf(a * z) + exp(-a * a * z * z) / (a * sqrt(pi)));
  } else {
    const double L = P.L[0];
    const double gamma_e = 0.57721566490153286061;
    double rec = 0.0;
    for (int m = 1; m <= P.mrec[0]; ++m) {
      double km = 2 * pi * m / L;
      double am = km * km / (4 * a * a);
      if (am > 700) break;
      rec += cos(km * rp[0]) * pm_incbessel(P, am, rf2 * km * km / 4.0);
    }
    out += (2.0 / L) * rec;
    out += -(1.0 / L) * (pm_ein(a * a * rf2) - 2.0 * log(2 * a * L) + gamma_e);
  }
  return out;
}

}  // namespace pmfem

namespace pmfem {

// ---- NEXT-4: Bloch-phase PGF (Eq. 2 with k0 != 0):
//   G(r; k0) = sum_i exp(-j k0.R_i) / |r - R_i|
// Ewald split with the G = 0 reciprocal term kept (k0 off the reciprocal lattice):
//   real: sum_i exp(-j k0.R_i) erfc(a |r - R_i|) / |r - R_i|
//   3D: (4 pi / V) sum_G exp(-|q|^2/4a^2) / |q|^2 exp(-j q.r),      q = G + k0
//   2D: (1 / A) sum_G (pi/|q|) [e^{|q|z} erfc(|q|/2a + az) + e^{-|q|z} erfc(|q|/2a - az)] exp(-j q.rho)
//   1D: (1 / L) sum_m I(q^2/4a^2, rho^2 q^2/4) exp(-j q x)
// The point is first wrapped into the unit cell, r = r_w + n L, and G(r) = exp(-j k0.nL) G(r_w).
// Returns the MODULATED kernel exp(+j k0.r) G(r; k0), which is periodic (the AIM grid convolves
// quasi-periodic data through it).  self = true: lim [G(r) - 1/r] at r = 0.
struct Cplx { double re, im; };

PM_HD inline Cplx pgf_eval_bloch(const PgfDev& P, const double k0_in[3], const double r_in[3], bool self) {
  const double pi = 3.14159265358979323846;
  const double a = P.alpha;
  double rw[3] = {0, 0, 0}, rf[2] = {0, 0}, k0[3] = {0, 0, 0};
  double ph_wrap = 0.0;                     // k0 . (n L) of the wrap
  double kr = 0.0;                          // k0 . r (modulation)
  for (int i = 0; i < P.dim; ++i) {
    const double x = self ? 0.0 : r_in[P.ax[i]];
    const double L = P.L[i];
    const double nw = floor(x / L + 0.5);
    rw[i] = x - nw * L;
    k0[i] = k0_in[P.ax[i]];
    ph_wrap += k0[i] * nw * L;
    kr += k0[i] * x;
  }
  for (int i = P.dim; i < 3; ++i) rf[i - P.dim] = self ? 0.0 : r_in[P.ax[i]];
  const double rf2 = rf[0] * rf[0] + rf[1] * rf[1];
  double gre = 0.0, gim = 0.0;
  // real space (images of the wrapped point)
  const double rc = P.xr / a;
  const int n0 = P.nreal[0] + 1, n1 = P.dim > 1 ? P.nreal[1] + 1 : 0, n2 = P.dim > 2 ? P.nreal[2] + 1 : 0;
  for (int i = -n0; i <= n0; ++i)
    for (int j = -n1; j <= n1; ++j)
      for (int k = -n2; k <= n2; ++k) {
        if (self && i == 0 && j == 0 && k == 0) continue;
        const double Rx = i * P.L[0], Ry = P.dim > 1 ? j * P.L[1] : 0.0, Rz = P.dim > 2 ? k * P.L[2] : 0.0;
        const double x = rw[0] - Rx, y = rw[1] - Ry, z = rw[2] - Rz;
        const double d = sqrt(x * x + y * y + z * z + rf2);
        if (d == 0.0 || d > rc + 1e-300) continue;
        const double e = erfc(a * d) / d, ph = -(k0[0] * Rx + k0[1] * Ry + k0[2] * Rz);
        gre += e * cos(ph); gim += e * sin(ph);
      }
  if (self) gre += -2.0 * a / sqrt(pi);
  // reciprocal space, q = G + k0 (index ranges grown by the shift)
  int mr[3] = {0, 0, 0};
  for (int i = 0; i < P.dim; ++i) mr[i] = P.mrec[i] + 1 + (int)ceil(fabs(k0[i]) * P.L[i] / (2 * pi));
  if (P.dim == 3) {
    const double V = P.L[0] * P.L[1] * P.L[2];
    for (int i = -mr[0]; i <= mr[0]; ++i)
      for (int j = -mr[1]; j <= mr[1]; ++j)
        for (int k = -mr[2]; k <= mr[2]; ++k) {
          const double qx = 2 * pi * i / P.L[0] + k0[0], qy = 2 * pi * j / P.L[1] + k0[1], qz = 2 * pi * k / P.L[2] + k0[2];
          const double q2 = qx * qx + qy * qy + qz * qz;
          if (q2 == 0.0) continue;
          const double e = 4 * pi / V * exp(-q2 / (4 * a * a)) / q2;
          if (e < 1e-300) continue;
          const double ph = -(qx * rw[0] + qy * rw[1] + qz * rw[2]);
          gre += e * cos(ph); gim += e * sin(ph);
        }
  } else if (P.dim == 2) {
    const double A = P.L[0] * P.L[1], z = rf[0];
    for (int i = -mr[0]; i <= mr[0]; ++i)
      for (int j = -mr[1]; j <= mr[1]; ++j) {
        const double qx = 2 * pi * i / P.L[0] + k0[0], qy = 2 * pi * j / P.L[1] + k0[1];
        const double q = sqrt(qx * qx + qy * qy);
        if (q == 0.0) continue;
        double br = 0.0;
        for (int sg = -1; sg <= 1; sg += 2) {
          const double w = q / (2 * a) + sg * a * z;
          if (w >= 0) br += pm_erfcx(w) * exp(-q * q / (4 * a * a) - a * a * z * z);
          else br += exp(sg * q * z) * erfc(w);
        }
        const double e = pi / (A * q) * br, ph = -(qx * rw[0] + qy * rw[1]);
        gre += e * cos(ph); gim += e * sin(ph);
      }
  } else {
    const double L = P.L[0];
    for (int m = -mr[0]; m <= mr[0]; ++m) {
      const double q = 2 * pi * m / L + k0[0];
      if (q == 0.0) continue;
      const double am = q * q / (4 * a * a);
      if (am > 700) continue;
      const double e = pm_incbessel(P, am, rf2 * q * q / 4.0) / L, ph = -q * rw[0];
      gre += e * cos(ph); gim += e * sin(ph);
    }
  }
  // undo the wrap (G(r) = e^{-j k0.nL} G(r_w)) and modulate by e^{+j k0.r}: net phase k0.r - k0.nL
  const double ph = kr - ph_wrap;
  Cplx out;
  out.re = gre * cos(ph) - gim * sin(ph);
  out.im = gre * sin(ph) + gim * cos(ph);
  return out;
}

}  // namespace pmfem
