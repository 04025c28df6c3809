// Host setup, BAIM geometry (fp64): wrapped coordinates, grid, Lagrange stencils, the
// precorrection matrix C_box and the internal (box-sorted) node order.
//   P:193-200  Cartesian grid (Eq. grid; reading R6: periodic Delta = L/N)
//   P:202/206  projection / interpolation (reading R7: Lagrange = AIM moment matching, P^T)
//   P:208-218  step 4 precorrection; only G0 is subtracted and added back
//   P:220-232  near region Omega~_n^ER over periodic images (Eq. new_er; readings R8, R9),
//              "searching boxes ... box index pre-tabulated"
//   P:236-245  protruding cells: positions are used modulo L for BAIM (reading R16)
#include <algorithm>
#include <cmath>
#include <numeric>
#include <omp.h>
#include "pmfem_internal.h"

namespace pmfem {

namespace {
bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

void lagrange(double t, int s, int p, double* w) {
  for (int j = 0; j <= p; ++j) {
    double v = 1.0;
    for (int i = 0; i <= p; ++i)
      if (i != j) v *= (t - (s + i)) / double(j - i);
    w[j] = v;
  }
}
}  // namespace

// Host C_box rows (K8/K9): near pairs by a box list on the wrapped coordinates (box size
// r_ER); with kb the Bloch-modulated values exp(j k0 . d) G0*(d) - sum w w exp(j k0 . d_g) G0*(d_g)
void host_cbox_rows(const HostSetup& S, const double* kb, std::vector<std::vector<int32_t>>& rcol,
                    std::vector<std::vector<double>>& rval) {
  const int p = S.order;
  const int64_t Np = S.Np;
  const double rer = S.rer_scale * std::max(S.delta[0], std::max(S.delta[1], S.delta[2]));
  // near pairs (K8) by a box list on the wrapped coordinates, box size r_ER
  int64_t nb[3];
  double blo[3];
  for (int a = 0; a < 3; ++a) {
    double lo = 1e300, hi = -1e300;
    for (int64_t n = 0; n < Np; ++n) { lo = std::min(lo, S.xw[3 * n + a]); hi = std::max(hi, S.xw[3 * n + a]); }
    if (S.periodic[a]) { blo[a] = 0; nb[a] = std::max<int64_t>(1, (int64_t)std::floor(S.L[a] / rer)); }
    else { blo[a] = lo; nb[a] = (int64_t)std::floor((hi - lo) / rer) + 1; }
  }
  auto box_of = [&](int64_t n, int a) {
    double bs = S.periodic[a] ? S.L[a] / nb[a] : rer;
    int64_t b = (int64_t)std::floor((S.xw[3 * n + a] - blo[a]) / bs);
    return std::min<int64_t>(std::max<int64_t>(b, 0), nb[a] - 1);
  };
  std::vector<int64_t> bkey(Np), border(Np);
  for (int64_t n = 0; n < Np; ++n) bkey[n] = (box_of(n, 0) * nb[1] + box_of(n, 1)) * nb[2] + box_of(n, 2);
  std::iota(border.begin(), border.end(), 0);
  std::sort(border.begin(), border.end(), [&](int64_t x, int64_t y) { return bkey[x] < bkey[y]; });
  int64_t nbox = nb[0] * nb[1] * nb[2];
  std::vector<int64_t> bptr(nbox + 1, 0);
  for (int64_t n = 0; n < Np; ++n) bptr[bkey[n] + 1]++;
  for (int64_t b = 0; b < nbox; ++b) bptr[b + 1] += bptr[b];

  const int p1 = p + 1;
  const int W = 2 * p + 1;
  rcol.assign(Np, {});
  rval.assign(Np, {});
#pragma omp parallel
  {
    std::vector<std::pair<int64_t, int>> cand;    // (k, image code)
#pragma omp for schedule(dynamic, 512)
    for (int64_t n = 0; n < Np; ++n) {
      cand.clear();
      int64_t bn[3] = {box_of(n, 0), box_of(n, 1), box_of(n, 2)};
      // box reach: boxes have size >= r_ER so +-1 box suffices
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dz = -1; dz <= 1; ++dz) {
            int64_t bb[3] = {bn[0] + dx, bn[1] + dy, bn[2] + dz};
            bool ok = true;
            for (int a = 0; a < 3; ++a) {
              if (S.periodic[a]) bb[a] = ((bb[a] % nb[a]) + nb[a]) % nb[a];
              else ok &= (bb[a] >= 0 && bb[a] < nb[a]);
            }
            if (!ok) continue;
            int64_t b = (bb[0] * nb[1] + bb[1]) * nb[2] + bb[2];
            for (int64_t i = bptr[b]; i < bptr[b + 1]; ++i) {
              int64_t k = border[i];
              int img[3] = {0, 0, 0};
              bool in = true;
              for (int a = 0; a < 3; ++a) {
                double d = S.xw[3 * n + a] - S.xw[3 * k + a];
                if (S.periodic[a]) { img[a] = (int)std::nearbyint(d / S.L[a]); d -= img[a] * S.L[a]; }
                in &= std::fabs(d) <= rer;
              }
              if (in) cand.push_back({k, ((img[0] + 1) * 3 + (img[1] + 1)) * 3 + (img[2] + 1)});
            }
          }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      std::vector<int32_t> cols;
      std::vector<double> vals;
      double wn[3][4];
      for (int a = 0; a < 3; ++a) lagrange(S.st_t[3 * n + a], 0, p, wn[a]);
      for (auto& c : cand) {
        int64_t k = c.first;
        int img[3] = {c.second / 9 - 1, (c.second / 3) % 3 - 1, c.second % 3 - 1};
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = S.xw[3 * n + a] - S.xw[3 * k + a] - img[a] * S.L[a];
        double r = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        double val = r > 0 ? 1.0 / r : 0.0;
        double vim = 0.0;
        if (kb) {                      // Bloch: exp(j k0 . d) G0*(d)
          const double ph = kb[0] * d[0] + kb[1] * d[1] + kb[2] * d[2];
          vim = val * std::sin(ph);
          val *= std::cos(ph);
        }
        // grid-mediated G0: sum_{a in st(n), b in st(k)} w_na w_kb G0*((a - b - img N) o Delta)
        // per axis combine weights by index difference delta = (s_n + i) - (s_k + j) - img N
        double wk[3][4];
        for (int a = 0; a < 3; ++a) lagrange(S.st_t[3 * k + a], 0, p, wk[a]);
        double cw[3][7];
        int base[3];
        for (int a = 0; a < 3; ++a) {
          base[a] = S.st_s[3 * n + a] - S.st_s[3 * k + a] - img[a] * S.grid_n[a] - p;
          for (int e = 0; e < W; ++e) cw[a][e] = 0;
          for (int i = 0; i < p1; ++i)
            for (int j = 0; j < p1; ++j) cw[a][i - j + p] += wn[a][i] * wk[a][j];
        }
        if (!kb) {
          double gm = 0;
          for (int ex = 0; ex < W; ++ex) {
            double dx = (base[0] + ex) * S.delta[0];
            for (int ey = 0; ey < W; ++ey) {
              double dy = (base[1] + ey) * S.delta[1];
              double wxy = cw[0][ex] * cw[1][ey];
              for (int ez = 0; ez < W; ++ez) {
                double dz = (base[2] + ez) * S.delta[2];
                double rr = dx * dx + dy * dy + dz * dz;
                if (rr > 0) gm += wxy * cw[2][ez] / std::sqrt(rr);
              }
            }
          }
          cols.push_back((int32_t)k);
          vals.push_back(val - gm);
          continue;
        }
        // Bloch: the modulation exp(j k0 . d_g) of the grid separation is separable per axis
        double cr[3][7], ci[3][7];
        for (int a = 0; a < 3; ++a)
          for (int e = 0; e < W; ++e) {
            const double ph = kb[a] * (base[a] + e) * S.delta[a];
            cr[a][e] = cw[a][e] * std::cos(ph);
            ci[a][e] = cw[a][e] * std::sin(ph);
          }
        double gr = 0, gi = 0;
        for (int ex = 0; ex < W; ++ex) {
          double dx = (base[0] + ex) * S.delta[0];
          for (int ey = 0; ey < W; ++ey) {
            double dy = (base[1] + ey) * S.delta[1];
            const double xr = cr[0][ex] * cr[1][ey] - ci[0][ex] * ci[1][ey];
            const double xi = cr[0][ex] * ci[1][ey] + ci[0][ex] * cr[1][ey];
            for (int ez = 0; ez < W; ++ez) {
              double dz = (base[2] + ez) * S.delta[2];
              double rr = dx * dx + dy * dy + dz * dz;
              if (rr > 0) {
                const double ir = 1.0 / std::sqrt(rr);
                gr += (xr * cr[2][ez] - xi * ci[2][ez]) * ir;
                gi += (xr * ci[2][ez] + xi * cr[2][ez]) * ir;
              }
            }
          }
        }
        cols.push_back((int32_t)k);
        vals.push_back(val - gr);
        vals.push_back(vim - gi);
      }
      rcol[n] = std::move(cols);
      rval[n] = std::move(vals);
    }
  }
}

void setup_aim(HostSetup& S, const pmfem_grid* g) {
  require(g != nullptr, PMFEM_E_INVALID_ARG, "NULL grid");
  require(g->order >= 1 && g->order <= 3, PMFEM_E_INVALID_ARG, "stencil order must be 1, 2 or 3");
  require(g->rer_scale > 0, PMFEM_E_INVALID_ARG, "rer_scale must be positive");
  require(g->z0_ring == 0 || g->z0_ring == 1, PMFEM_E_INVALID_ARG, "z0_ring must be 0 or 1");
  S.order = g->order;
  S.rer_scale = g->rer_scale;
  S.z0_ring = g->z0_ring;
  const int p = S.order;
  const int64_t Np = S.Np;
  // wrapped parent coordinates (R16): w = x - L floor(x/L); w >= L -> w - L; w < 0 -> 0
  S.xw.resize(3 * Np);
  for (int64_t n = 0; n < Np; ++n)
    for (int a = 0; a < 3; ++a) {
      double x = S.xyz[3 * S.parent[n] + a];
      if (S.periodic[a]) {
        double L = S.L[a];
        double w = x - L * std::floor(x / L);
        if (w >= L) w -= L;
        if (w < 0) w = 0;
        x = w;
      }
      S.xw[3 * n + a] = x;
    }
  for (int a = 0; a < 3; ++a) {
    S.grid_n[a] = g->n[a];
    require(g->n[a] >= (S.periodic[a] ? 2 * (p + 1) : p + 1), PMFEM_E_INVALID_ARG,
            "grid too small for the stencil order");
    if (S.periodic[a]) {
      S.delta[a] = S.L[a] / g->n[a];
      S.origin[a] = 0.0;
      S.fft_n[a] = g->n[a];
    } else {
      double lo = 1e300, hi = -1e300;
      for (int64_t n = 0; n < Np; ++n) { lo = std::min(lo, S.xw[3 * n + a]); hi = std::max(hi, S.xw[3 * n + a]); }
      require(hi > lo, PMFEM_E_INVALID_ARG, "zero extent on a non-periodic axis");
      S.origin[a] = lo;
      S.delta[a] = (hi - lo) / (g->n[a] - 1);
      S.fft_n[a] = 2 * g->n[a];
    }
    require(is_pow2(S.fft_n[a]), PMFEM_E_INVALID_ARG, "FFT length must be a power of two on every axis");
  }
  // shared-memory limits of the FFT passes (device.cu): the fp64 PGF transform stages 16 lines of
  // P complex doubles per CTA along axes 1 and 2 (P <= 512 in 227 KB), the x pass <= 4096
  // complex per line
  require(S.fft_n[1] <= 512 && S.fft_n[2] <= 512 && S.fft_n[0] <= 8192, PMFEM_E_INVALID_ARG,
          "FFT lengths above the shared-memory limits (axis 0 <= 8192, axes 1, 2 <= 512)");
  // r_ER = s * max(Delta) on every axis (R8); validity on periodic axes (K8)
  const double rer = S.rer_scale * std::max(S.delta[0], std::max(S.delta[1], S.delta[2]));
  for (int a = 0; a < 3; ++a)
    if (S.periodic[a])
      require(rer < S.L[a] / 2 && rer / S.delta[a] + p + 1 < S.grid_n[a] / 2.0, PMFEM_E_RER_TOO_LARGE,
              "r_ER too large on periodic axis " + std::to_string(a));

  // stencils (K5): t = (x - x0)/Delta; p odd: s = floor(t) - (p-1)/2; p even: s = floor(t+1/2) - p/2;
  // non-periodic axes clamp s to [0, N-1-p]
  S.st_s.resize(3 * Np);
  S.st_t.resize(3 * Np);
  for (int64_t n = 0; n < Np; ++n)
    for (int a = 0; a < 3; ++a) {
      double t = (S.xw[3 * n + a] - S.origin[a]) / S.delta[a];
      // the grid spans the node extent, so only corrupted coordinates leave it
      require(std::isfinite(t) && (S.periodic[a] ? (t >= 0.0 && t < S.grid_n[a] + 1e-9)
                                                 : (t >= -1e-9 && t <= S.grid_n[a] - 1 + 1e-9)),
              PMFEM_E_OUTSIDE_GRID, "node outside the AIM grid on axis " + std::to_string(a));
      int64_t s = (p % 2) ? (int64_t)std::floor(t) - (p - 1) / 2 : (int64_t)std::floor(t + 0.5) - p / 2;
      if (!S.periodic[a]) s = std::min<int64_t>(std::max<int64_t>(s, 0), S.grid_n[a] - 1 - p);
      S.st_s[3 * n + a] = (int32_t)s;
      S.st_t[3 * n + a] = t - (double)s;
    }

  if (S.cbox_device) {            // device contexts: C_box is built on the GPU (cbox_gpu.cu)
    S.cbox = Csr();
    return;
  }
  std::vector<std::vector<int32_t>> rcol;
  std::vector<std::vector<double>> rval;
  host_cbox_rows(S, nullptr, rcol, rval);
  Csr& C = S.cbox;
  C.n_rows = Np;
  C.nv = 1;
  C.rowptr.assign(Np + 1, 0);
  for (int64_t n = 0; n < Np; ++n) C.rowptr[n + 1] = C.rowptr[n] + (int64_t)rcol[n].size();
  C.col.resize(C.rowptr[Np]);
  C.val.resize(C.rowptr[Np]);
#pragma omp parallel for
  for (int64_t n = 0; n < Np; ++n) {
    std::copy(rcol[n].begin(), rcol[n].end(), C.col.begin() + C.rowptr[n]);
    std::copy(rval[n].begin(), rval[n].end(), C.val.begin() + C.rowptr[n]);
  }
}

// Internal order: parents sorted by their wrapped stencil anchor box, x fastest (the grid's
// memory order), ties by user index -- consecutive rows touch the same grid lines.
void setup_order(HostSetup& S) {
  const int64_t Np = S.Np;
  std::vector<int64_t> key(Np);
  for (int64_t n = 0; n < Np; ++n) {
    int64_t s[3];
    for (int a = 0; a < 3; ++a) {
      int64_t v = S.st_s[3 * n + a];
      if (S.periodic[a]) v = ((v % S.grid_n[a]) + S.grid_n[a]) % S.grid_n[a];
      s[a] = v;
    }
    key[n] = (s[2] * S.grid_n[1] + s[1]) * S.grid_n[0] + s[0];
  }
  S.perm.resize(Np);
  std::iota(S.perm.begin(), S.perm.end(), 0);
  std::stable_sort(S.perm.begin(), S.perm.end(), [&](int64_t x, int64_t y) { return key[x] < key[y]; });
  S.iperm.resize(Np);
  for (int64_t i = 0; i < Np; ++i) S.iperm[S.perm[i]] = i;
}

}  // namespace pmfem
