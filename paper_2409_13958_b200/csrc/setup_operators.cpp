// Host setup, local operators (fp64): lumped volume, folded exchange Laplacian, charge and
// gradient operators on the periodic 1-ring.
//   P:117-123  H_ex = (2A/Ms^2) lap M  ->  H_ex,n = sum_{m in Omega_n} w_mn M_m   (Eqs. hex, lapl)
//   P:125-157  T-PBC Cases 1-3 (Eqs. lapl_1, shift, dedup, lapl_2): realised as
//              "assemble over every tet touching any copy of n, remap columns to their LCA"
//   P:171      q_n = sum_k w^q_kn M(r_LCA(k))            (Eq. hms_d1)
//   P:174      H_ms,n = -sum_k w^grad_kn u(r_LCA(k))     (Eq. hms_d3)
//   P:177      charge / gradient operators "modified similarly" under T-PBC
// Row n gathers the tets of every copy c of parent n (the region union Omega_n U {Omega_n'} of
// Case 3); each tet is visited once per row, so the dedup of Eq. dedup is automatic.
// Readings: R1 q_n = int grad(phi_n).M dV; R14 lumped-mass gradient; R15 lumped
// exchange with 2A/Ms folded in.  Stored in off-diagonal ("difference") form:
//   sum_m X_nm v_m = sum_{m != n} X_nm (v_m - v_n) + (sum_m X_nm) v_n,
// with sum_m L_nm = sum_m G_nm = 0 exactly (sum_b grad phi_b = 0 per tet).
#include <algorithm>
#include <cmath>
#include <omp.h>
#include "pmfem_internal.h"

namespace pmfem {

void setup_operators(HostSetup& S) {
  const int64_t Np = S.Np;
  // lumped volume Vt_n = sum_{T ∋ copy of n} V_T / 4
  S.Vt.assign(Np, 0.0);
  for (int64_t t = 0; t < S.T; ++t)
    for (int k = 0; k < 4; ++k) S.Vt[S.pid[S.tets[4 * t + k]]] += S.vol[t] / 4.0;
  for (int64_t n = 0; n < Np; ++n)
    require(S.Vt[n] > 0, PMFEM_E_MESH, "zero lumped volume at parent " + std::to_string(n));

  const int NV = 7;   // L, Dx, Dy, Dz, Gx, Gy, Gz
  std::vector<std::vector<int32_t>> rcol(Np);
  std::vector<std::vector<double>> rval(Np);
  S.rowsumD.assign(3 * Np, 0.0);
  S.diagD.assign(3 * Np, 0.0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t n = 0; n < Np; ++n) {
    std::vector<int32_t> cols;
    std::vector<double> vals;
    double diagL = 0, diag[7] = {0};
    for (int64_t ci = S.copies_ptr[n]; ci < S.copies_ptr[n + 1]; ++ci) {
      int64_t c = S.copies[ci];
      for (int64_t ti = S.ntet_ptr[c]; ti < S.ntet_ptr[c + 1]; ++ti) {
        int64_t t = S.ntet[ti];
        const int32_t* tv = &S.tets[4 * t];
        int a = 0;
        while (tv[a] != c) ++a;
        const double* g = &S.grads[12 * t];
        const double V = S.vol[t];
        const double coef = 2.0 * S.Aex_tet[t] / S.Ms_tet[t];
        for (int b = 0; b < 4; ++b) {
          int32_t col = S.pid[tv[b]];
          double v[7];
          v[0] = coef * V * (g[3 * a] * g[3 * b] + g[3 * a + 1] * g[3 * b + 1] + g[3 * a + 2] * g[3 * b + 2]);
          for (int x = 0; x < 3; ++x) {
            v[1 + x] = S.Ms_tet[t] * V / 4.0 * g[3 * a + x];
            v[4 + x] = V / 4.0 * g[3 * b + x];
          }
          if (col == n) {
            for (int x = 0; x < 7; ++x) diag[x] += v[x];
            continue;
          }
          size_t j = 0;
          while (j < cols.size() && cols[j] != col) ++j;
          if (j == cols.size()) { cols.push_back(col); vals.insert(vals.end(), 7, 0.0); }
          for (int x = 0; x < 7; ++x) vals[NV * j + x] += v[x];
        }
      }
    }
    (void)diagL;
    // sort by column
    std::vector<int> ord(cols.size());
    for (size_t j = 0; j < ord.size(); ++j) ord[j] = (int)j;
    std::sort(ord.begin(), ord.end(), [&](int x, int y) { return cols[x] < cols[y]; });
    std::vector<int32_t> c2(cols.size());
    std::vector<double> v2(vals.size());
    double rs[3] = {diag[1], diag[2], diag[3]};
    const double iv = 1.0 / S.Vt[n];
    for (size_t j = 0; j < ord.size(); ++j) {
      c2[j] = cols[ord[j]];
      const double* s = &vals[NV * ord[j]];
      v2[NV * j + 0] = -s[0] * iv;                      // L = -S / Vt
      for (int x = 0; x < 3; ++x) {
        v2[NV * j + 1 + x] = s[1 + x];                  // D
        v2[NV * j + 4 + x] = s[4 + x] * iv;             // G
        rs[x] += s[1 + x];
      }
    }
    for (int x = 0; x < 3; ++x) { S.rowsumD[3 * n + x] = rs[x]; S.diagD[3 * n + x] = diag[1 + x]; }
    rcol[n] = std::move(c2);
    rval[n] = std::move(v2);
  }
  Csr& R = S.ring1;
  R.n_rows = Np;
  R.nv = NV;
  R.rowptr.assign(Np + 1, 0);
  for (int64_t n = 0; n < Np; ++n) R.rowptr[n + 1] = R.rowptr[n] + (int64_t)rcol[n].size();
  R.col.resize(R.rowptr[Np]);
  R.val.resize(NV * R.rowptr[Np]);
#pragma omp parallel for
  for (int64_t n = 0; n < Np; ++n) {
    std::copy(rcol[n].begin(), rcol[n].end(), R.col.begin() + R.rowptr[n]);
    std::copy(rval[n].begin(), rval[n].end(), R.val.begin() + NV * R.rowptr[n]);
  }
}

}  // namespace pmfem
