// Host setup of the NEXT-4 complex field path (fp64): the Bloch-phased operators.
//   P:183-185  G_p(r) = sum_i exp(-j k0.R_i) G_0(r - R_i)  (Eq. 2): the unit-cell kernel of a
//              Bloch-periodic charge rho(r + R) = exp(-j k0.R) rho(r); the magnetisation
//              amplitudes obey the same condition, m(r + R) = exp(-j k0.R) m(r) (reading R27)
//   P:117-157, P:170-177  folded local operators: a tet entry between copies a (row) and b
//              (column) with lattice shifts s_a, s_b carries exp(j k0.L(s_a - s_b))
//   P:173, P:190, P:234   Z0: element image (t, s) seen from r_n -- vertex v carries
//              exp(-j k0.L(shift_v + s)); the point-charge term of near source (p, ell)
//              carries exp(-j k0.L ell)
//   P:193-232  AIM on modulated charges q~ = exp(j k0.r) q with the L-periodic kernel
//              G~(r) = exp(j k0.r) G_p(r); C~ (host_cbox_rows with kb) and the half spectra of
//              Re G~ (even, real spectrum) and Im G~ (odd, imaginary spectrum)
// The oracle (oracle/bloch_heff.py) implements the same readings independently.
#include <algorithm>
#include <cmath>
#include <complex>
#include <omp.h>
#include "pmfem_internal.h"
#include "z0_cone.cuh"

namespace pmfem {

namespace {
using cd = std::complex<double>;

inline cd phase(const double k[3], const int s[3], const double L[3]) {
  const double ph = k[0] * s[0] * L[0] + k[1] * s[1] * L[1] + k[2] * s[2] * L[2];
  return {std::cos(ph), std::sin(ph)};
}

void pack_rows(Csr& R, int nv, int64_t Np, std::vector<std::vector<int32_t>>& rcol,
               std::vector<std::vector<double>>& rval) {
  R.n_rows = Np;
  R.nv = nv;
  R.rowptr.assign(Np + 1, 0);
  for (int64_t n = 0; n < Np; ++n) R.rowptr[n + 1] = R.rowptr[n] + (int64_t)rcol[n].size();
  R.col.resize(R.rowptr[Np]);
  R.val.resize((size_t)nv * R.rowptr[Np]);
#pragma omp parallel for
  for (int64_t n = 0; n < Np; ++n) {
    std::copy(rcol[n].begin(), rcol[n].end(), R.col.begin() + R.rowptr[n]);
    std::copy(rval[n].begin(), rval[n].end(), R.val.begin() + (size_t)nv * R.rowptr[n]);
  }
}
}  // namespace

void setup_bloch_ops(const HostSetup& S, const double k0[3], BlochHost& B) {
  const int64_t Np = S.Np;
  for (int a = 0; a < 3; ++a) B.k0[a] = S.periodic[a] ? k0[a] : 0.0;
  const double* k = B.k0;
  // ---- modulation exp(j k0 . r_n)
  B.mod.resize(2 * Np);
  for (int64_t n = 0; n < Np; ++n) {
    const double* r = &S.xyz[3 * S.parent[n]];
    const double ph = k[0] * r[0] + k[1] * r[1] + k[2] * r[2];
    B.mod[2 * n] = std::cos(ph);
    B.mod[2 * n + 1] = std::sin(ph);
  }
  // ---- ring-1 operators L, D, G (diagonal included)
  {
    std::vector<std::vector<int32_t>> rcol(Np);
    std::vector<std::vector<double>> rval(Np);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t n = 0; n < Np; ++n) {
      std::vector<int32_t> cols;
      std::vector<cd> acc;                       // 7 per column
      for (int64_t ci = S.copies_ptr[n]; ci < S.copies_ptr[n + 1]; ++ci) {
        const int64_t c = S.copies[ci];
        for (int64_t ti = S.ntet_ptr[c]; ti < S.ntet_ptr[c + 1]; ++ti) {
          const int64_t t = S.ntet[ti];
          const int32_t* tv = &S.tets[4 * t];
          int a = 0;
          while (tv[a] != c) ++a;
          const double* g = &S.grads[12 * t];
          const double V = S.vol[t];
          const double coef = 2.0 * S.Aex_tet[t] / S.Ms_tet[t];
          for (int b = 0; b < 4; ++b) {
            const int32_t col = S.pid[tv[b]];
            int ds[3];
            for (int x = 0; x < 3; ++x) ds[x] = S.shift[3 * c + x] - S.shift[3 * tv[b] + x];
            const cd ph = phase(k, ds, S.L);
            double v[7];
            v[0] = coef * V * (g[3 * a] * g[3 * b] + g[3 * a + 1] * g[3 * b + 1] + g[3 * a + 2] * g[3 * b + 2]);
            for (int x = 0; x < 3; ++x) {
              v[1 + x] = S.Ms_tet[t] * V / 4.0 * g[3 * a + x];
              v[4 + x] = V / 4.0 * g[3 * b + x];
            }
            size_t j = 0;
            while (j < cols.size() && cols[j] != col) ++j;
            if (j == cols.size()) { cols.push_back(col); acc.insert(acc.end(), 7, cd(0, 0)); }
            for (int x = 0; x < 7; ++x) acc[7 * j + x] += ph * v[x];
          }
        }
      }
      std::vector<int> ord(cols.size());
      for (size_t j = 0; j < ord.size(); ++j) ord[j] = (int)j;
      std::sort(ord.begin(), ord.end(), [&](int x, int y) { return cols[x] < cols[y]; });
      const double iv = 1.0 / S.Vt[n];
      std::vector<int32_t>& c2 = rcol[n];
      std::vector<double>& v2 = rval[n];
      for (int j : ord) {
        c2.push_back(cols[j]);
        const cd* s = &acc[7 * j];
        const cd out[7] = {-s[0] * iv, s[1], s[2], s[3], s[4] * iv, s[5] * iv, s[6] * iv};
        for (int x = 0; x < 7; ++x) { v2.push_back(out[x].real()); v2.push_back(out[x].imag()); }
      }
    }
    pack_rows(B.r1, 14, Np, rcol, rval);
  }
  // ---- Z0 (host element integrals, z0_cone.cuh)
  {
    static TriRules rules;
    build_tri_rules(rules);
    std::vector<std::vector<int32_t>> rcol(Np);
    std::vector<std::vector<double>> rval(Np);
    std::string err;
#pragma omp parallel
    {
      ConeIntegrator I;
      I.R = &rules;
      Z0RowEnum W;
#pragma omp for schedule(dynamic, 16)
      for (int64_t n = 0; n < Np; ++n) {
        try {
          z0_enumerate_row(S, n, W);
          std::vector<int32_t> cols;
          for (auto& it : W.its) {
            const int32_t* tv = &S.tets[4 * (it.key / Z0_NC)];
            for (int j = 0; j < 4; ++j) cols.push_back(S.pid[tv[j]]);
          }
          for (auto& pr : W.near)
            for (int64_t e = B.r1.rowptr[pr.first]; e < B.r1.rowptr[pr.first + 1]; ++e) cols.push_back(B.r1.col[e]);
          std::sort(cols.begin(), cols.end());
          cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
          auto slot = [&](int32_t c) { return (int)(std::lower_bound(cols.begin(), cols.end(), c) - cols.begin()); };
          std::vector<cd> acc(3 * cols.size(), cd(0, 0));
          const double* xn = &S.xyz[3 * S.parent[n]];
          for (auto& it : W.its) {
            const int64_t t = it.key / Z0_NC;
            const int32_t* tv = &S.tets[4 * t];
            int s[3];
            z0_unpack_shift((int)(it.key % Z0_NC), s);
            for (int j = 0; j < 4; ++j)
              for (int x = 0; x < 3; ++x) {
                I.P[j][x] = S.xyz[3 * tv[j] + x] + s[x] * S.L[x];
                I.g[j][x] = S.grads[12 * t + 3 * j + x];
              }
            for (int x = 0; x < 3; ++x) I.o[x] = xn[x];
            I.run(it.va);
            const double Ms = S.Ms_tet[t];
            for (int m = 0; m < 4; ++m) {
              int sv[3];
              for (int x = 0; x < 3; ++x) sv[x] = -(S.shift[3 * tv[m] + x] + s[x]);
              const cd ph = phase(k, sv, S.L);
              const int p = slot(S.pid[tv[m]]);
              for (int kk = 0; kk < 4; ++kk) {
                if (!(it.flags & (1u << kk))) continue;
                for (int x = 0; x < 3; ++x) acc[3 * p + x] += ph * (Ms * (I.B[kk][m][x] + I.g[kk][x] * I.A[m]));
              }
            }
          }
          // minus the point-charge value of each near source: -exp(-j k0.L ell) G0*(d) q_p
          for (auto& pr : W.near) {
            const int64_t p = pr.first;
            int ell[3];
            z0_unpack_shift(pr.second, ell);
            const double* xp = &S.xyz[3 * S.parent[p]];
            double d[3];
            for (int x = 0; x < 3; ++x) d[x] = xn[x] - xp[x] - ell[x] * S.L[x];
            const double r = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            if (r == 0.0) continue;
            int ml[3] = {-ell[0], -ell[1], -ell[2]};
            const cd gi = phase(k, ml, S.L) / r;
            for (int64_t e = B.r1.rowptr[p]; e < B.r1.rowptr[p + 1]; ++e) {
              const int sp = slot(B.r1.col[e]);
              const double* v = &B.r1.val[14 * e];
              for (int x = 0; x < 3; ++x) acc[3 * sp + x] -= gi * cd(v[2 + 2 * x], v[3 + 2 * x]);
            }
          }
          rcol[n] = std::move(cols);
          std::vector<double>& v2 = rval[n];
          v2.resize(2 * acc.size());
          for (size_t j = 0; j < acc.size(); ++j) { v2[2 * j] = acc[j].real(); v2[2 * j + 1] = acc[j].imag(); }
        } catch (const std::exception& e) {
#pragma omp critical
          err = e.what();
        }
      }
    }
    require(err.empty(), PMFEM_E_MESH, err);
    pack_rows(B.z0, 6, Np, rcol, rval);
  }
  // ---- modulated precorrection C~
  {
    std::vector<std::vector<int32_t>> rcol;
    std::vector<std::vector<double>> rval;
    host_cbox_rows(S, k, rcol, rval);
    pack_rows(B.cbox, 2, Np, rcol, rval);
  }
  // ---- half spectra of Re G~ and Im G~ from the full complex spectrum (S.spectrum_bloch,
  // [P2][P1][P0], already / #points): FFT(Re G~)(f) = (G^(f) + conj G^(-f)) / 2 is real,
  // FFT(Im G~)(f) = (G^(f) - conj G^(-f)) / 2j is imaginary (Re G~ even, Im G~ odd: G~(-r) =
  // conj G~(r)); fb stores its imaginary part
  {
    const int P0 = S.fft_n[0], P1 = S.fft_n[1], P2 = S.fft_n[2], H0 = P0 / 2 + 1;
    require((int64_t)S.spectrum_bloch.size() == 2LL * P0 * P1 * P2, PMFEM_E_STATE, "Bloch spectrum missing");
    B.fa.assign((size_t)H0 * P1 * P2, 0.0);
    B.fb.assign((size_t)H0 * P1 * P2, 0.0);
    for (int z = 0; z < P2; ++z)
      for (int y = 0; y < P1; ++y)
        for (int x = 0; x < H0; ++x) {
          const int64_t i = ((int64_t)z * P1 + y) * P0 + x;
          const int64_t j = ((int64_t)((P2 - z) % P2) * P1 + (P1 - y) % P1) * P0 + (P0 - x) % P0;
          const cd g(S.spectrum_bloch[2 * i], S.spectrum_bloch[2 * i + 1]);
          const cd gm(S.spectrum_bloch[2 * j], -S.spectrum_bloch[2 * j + 1]);   // conj G^(-f)
          const int64_t h = ((int64_t)z * P1 + y) * H0 + x;
          B.fa[h] = 0.5 * (g + gm).real();
          B.fb[h] = (0.5 * (g - gm) / cd(0, 1)).imag();
        }
  }
}

}  // namespace pmfem
