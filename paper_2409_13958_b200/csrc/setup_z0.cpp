// Host setup: exact near-field correction matrix Z0 (fp64).
//   P:173  u(r_n) = u~(r_n) + sum_{k in near(n)} w^near_kn M(r_k)          (Eq. hms_d2b)
//   P:190  "The correction sparse matrix elements are found through exact integrals of
//          Eq. (hms_d2) performed over the relevant elements (tetrahedrons in our case)"
//   P:234  range = "the average edge length", region expanded over periodic images (Eq. new_er)
// Reading R10/R12: the exact potential at r_n of node k's charge piece
// phi_k (rho + sigma delta_S) is, after integration by parts, the volume integral
//   E_{n<-(k,img)} = int_{supp phi_k + img L} [phi_k grad'G0(r_n - r') + G0(r_n - r') grad phi_k] . M_h dV'
// and (Z0 m)_n = sum_{(k,img) in near(n)} E_{n<-(k,img)} - G0*(r_n - r_k - img L) q_k.
//
// Integration method (independent of the oracle's Duffy/Gauss scheme): the signed cone
// decomposition from the observer o,
//   int_T g dV = sum_F h_F int_F dA(y) int_0^1 t^2 g(o + t (y - o)) dt,
// h_F = signed distance from o to the plane of face F (positive on the inner side).  For the
// two kernels needed here the t-integral is done in closed form (the integrands are
// polynomials in t once the 1/R and 1/R^2 singularities cancel against t^2), leaving smooth
// face integrals evaluated with adaptively subdivided collapsed Gauss rules.
#include <algorithm>
#include <cmath>
#include <omp.h>
#include "pmfem_internal.h"

namespace pmfem {

namespace {

struct GaussRule {
  std::vector<double> x, w;   // on [0,1]
  explicit GaussRule(int n) : x(n), w(n) {
    for (int i = 0; i < n; ++i) {
      double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
      for (int it = 0; it < 100; ++it) {
        double p0 = 1, p1 = z;
        for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
        double dp = n * (z * p1 - p0) / (z * z - 1);
        double dz = p1 / dp;
        z -= dz;
        if (std::fabs(dz) < 1e-16) break;
      }
      double p0 = 1, p1 = z;
      for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      double dp = n * (z * p1 - p0) / (z * z - 1);
      x[i] = 0.5 * (1 - z);
      w[i] = 1.0 / ((1 - z * z) * dp * dp);   // = 0.5 * 2/((1-z^2) dp^2)
    }
  }
};

struct TriRule {               // collapsed n x n Gauss on the reference triangle
  std::vector<double> l0, l1, l2, w;   // barycentrics and weights (sum w = 1/2)
  explicit TriRule(int n) {
    GaussRule g(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double u = g.x[i], v = g.x[j];
        l0.push_back(1 - u); l1.push_back(u * (1 - v)); l2.push_back(u * v);
        w.push_back(g.w[i] * g.w[j] * u);
      }
  }
};

inline double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

struct ConeIntegrator {
  // tet data
  double P[4][3], g[4][3], c[4];     // phi_i(r) = c_i + g_i . r
  double o[3], a[4];                 // observer, phi_i(o)
  double A[4], B[4][4][3];
  const TriRule* rules[3];          // n = 4, 6, 8 collapsed Gauss
  double eta;
  int maxdepth;

  double phi(int i, const double* r) const { return c[i] + dot3(g[i], r); }

  void face(const double* V0, const double* V1, const double* V2, double h, int depth) {
    double cen[3], e01[3], e02[3], e12[3];
    for (int x = 0; x < 3; ++x) {
      cen[x] = (V0[x] + V1[x] + V2[x]) / 3.0;
      e01[x] = V1[x] - V0[x]; e02[x] = V2[x] - V0[x]; e12[x] = V2[x] - V1[x];
    }
    double size = std::sqrt(std::max(dot3(e01, e01), std::max(dot3(e02, e02), dot3(e12, e12))));
    double rc = 0;
    for (const double* V : {V0, V1, V2}) {
      double d[3] = {V[0] - cen[0], V[1] - cen[1], V[2] - cen[2]};
      rc = std::max(rc, std::sqrt(dot3(d, d)));
    }
    double dc[3] = {cen[0] - o[0], cen[1] - o[1], cen[2] - o[2]};
    double dest = std::max(std::fabs(h), std::sqrt(dot3(dc, dc)) - rc);
    if (size > eta * dest && depth < maxdepth) {
      double m01[3], m02[3], m12[3];
      for (int x = 0; x < 3; ++x) {
        m01[x] = 0.5 * (V0[x] + V1[x]); m02[x] = 0.5 * (V0[x] + V2[x]); m12[x] = 0.5 * (V1[x] + V2[x]);
      }
      face(V0, m01, m02, h, depth + 1);
      face(m01, V1, m12, h, depth + 1);
      face(m02, m12, V2, h, depth + 1);
      face(m12, m02, m01, h, depth + 1);
      return;
    }
    double cr[3] = {e01[1] * e02[2] - e01[2] * e02[1], e01[2] * e02[0] - e01[0] * e02[2],
                    e01[0] * e02[1] - e01[1] * e02[0]};
    double area2 = std::sqrt(dot3(cr, cr));
    // rule by distance ratio: the error of an n-point Gauss rule on a kernel whose nearest
    // singularity is at relative distance d/size decays like rho^-2n (Bernstein ellipse)
    const double ratio = size / dest;
    const TriRule& R = ratio <= 0.3 ? *rules[0] : (ratio <= 0.6 ? *rules[1] : *rules[2]);
    for (size_t q = 0; q < R.w.size(); ++q) {
      double y[3];
      for (int x = 0; x < 3; ++x) y[x] = R.l0[q] * V0[x] + R.l1[q] * V1[x] + R.l2[q] * V2[x];
      double Rv[3] = {y[0] - o[0], y[1] - o[1], y[2] - o[2]};
      double r2 = dot3(Rv, Rv);
      double inv = 1.0 / std::sqrt(r2);
      double inv3 = inv * inv * inv;
      double w = R.w[q] * area2 * h;
      double py[4], b[4];
      for (int i = 0; i < 4; ++i) { py[i] = phi(i, y); b[i] = py[i] - a[i]; }
      // A_m += h w (a_m/6 + phi_m(y)/3) / |y-o|
      for (int m = 0; m < 4; ++m) A[m] += w * (a[m] / 6.0 + py[m] / 3.0) * inv;
      // B_km += -h w (a_k a_m + (a_k b_m + a_m b_k)/2 + b_k b_m/3) (y-o)/|y-o|^3
      for (int k = 0; k < 4; ++k)
        for (int m = k; m < 4; ++m) {
          double s = -w * (a[k] * a[m] + 0.5 * (a[k] * b[m] + a[m] * b[k]) + b[k] * b[m] / 3.0) * inv3;
          for (int x = 0; x < 3; ++x) B[k][m][x] += s * Rv[x];
        }
    }
  }

  // va >= 0: o is vertex va (only the opposite face has h != 0)
  void run(int va) {
    for (int i = 0; i < 4; ++i) {
      A[i] = 0;
      for (int j = 0; j < 4; ++j)
        for (int x = 0; x < 3; ++x) B[i][j][x] = 0;
    }
    for (int i = 0; i < 4; ++i) c[i] = 1.0 - dot3(g[i], P[i]);
    for (int i = 0; i < 4; ++i) a[i] = (va >= 0) ? (i == va ? 1.0 : 0.0) : phi(i, o);
    for (int j = 0; j < 4; ++j) {
      if (va >= 0 && j != va) continue;
      double gn = std::sqrt(dot3(g[j], g[j]));
      double h = a[j] / gn;            // phi_j(o) = |g_j| h_j
      if (std::fabs(h) * gn < 1e-14) continue;
      const double* V0 = P[(j + 1) % 4];
      const double* V1 = P[(j + 2) % 4];
      const double* V2 = P[(j + 3) % 4];
      face(V0, V1, V2, h, 0);
    }
    for (int k = 0; k < 4; ++k)
      for (int m = 0; m < k; ++m)
        for (int x = 0; x < 3; ++x) B[k][m][x] = B[m][k][x];
  }
};

inline int pack_shift(const int s[3]) {
  for (int a = 0; a < 3; ++a)
    require(s[a] >= -8 && s[a] <= 8, PMFEM_E_MESH, "lattice shift out of range in Z0 near set");
  return ((s[0] + 8) * 17 + (s[1] + 8)) * 17 + (s[2] + 8);
}
inline void unpack_shift(int code, int s[3]) {
  s[2] = code % 17 - 8; code /= 17;
  s[1] = code % 17 - 8; code /= 17;
  s[0] = code - 8;
}

}  // namespace

void setup_z0(HostSetup& S) {
  const int64_t Np = S.Np;
  const int NC = 17 * 17 * 17;
  static const TriRule rule4(4), rule6(6), rule8(8);
  std::vector<std::vector<int32_t>> rcol(Np);
  std::vector<std::vector<double>> rval(Np);
  S.rowsumZ.assign(3 * Np, 0.0);
  std::string err;
#pragma omp parallel
  {
    ConeIntegrator I;
    I.rules[0] = &rule4; I.rules[1] = &rule6; I.rules[2] = &rule8;
    I.eta = 1.0;
    I.maxdepth = 7;
    std::vector<std::pair<int64_t, int>> near;   // (parent, shift code)
    std::vector<int64_t> U;                       // tet * NC + code
    std::vector<int32_t> cols;
    std::vector<double> vals;
#pragma omp for schedule(dynamic, 16)
    for (int64_t n = 0; n < Np; ++n) {
      try {
        near.clear(); U.clear(); cols.clear(); vals.clear();
        const int zero_code = ((8 * 17) + 8) * 17 + 8;
        if (S.z0_ring == 0) {
          near.push_back({n, zero_code});
        } else {
          for (int64_t ci = S.copies_ptr[n]; ci < S.copies_ptr[n + 1]; ++ci) {
            int64_t c = S.copies[ci];
            for (int64_t ti = S.ntet_ptr[c]; ti < S.ntet_ptr[c + 1]; ++ti) {
              int64_t t = S.ntet[ti];
              for (int b = 0; b < 4; ++b) {
                int32_t v = S.tets[4 * t + b];
                int s[3];
                for (int x = 0; x < 3; ++x) s[x] = S.shift[3 * v + x] - S.shift[3 * c + x];
                near.push_back({S.pid[v], pack_shift(s)});
              }
            }
          }
          std::sort(near.begin(), near.end());
          near.erase(std::unique(near.begin(), near.end()), near.end());
        }
        for (auto& pr : near) {
          int ell[3];
          unpack_shift(pr.second, ell);
          for (int64_t ci = S.copies_ptr[pr.first]; ci < S.copies_ptr[pr.first + 1]; ++ci) {
            int64_t c = S.copies[ci];
            int s[3];
            for (int x = 0; x < 3; ++x) s[x] = ell[x] - S.shift[3 * c + x];
            int code = pack_shift(s);
            for (int64_t ti = S.ntet_ptr[c]; ti < S.ntet_ptr[c + 1]; ++ti) U.push_back(S.ntet[ti] * NC + code);
          }
        }
        std::sort(U.begin(), U.end());
        U.erase(std::unique(U.begin(), U.end()), U.end());
        const double* o = &S.xyz[3 * S.parent[n]];
        auto add = [&](int32_t col, const double* w) {
          size_t j = 0;
          while (j < cols.size() && cols[j] != col) ++j;
          if (j == cols.size()) { cols.push_back(col); vals.insert(vals.end(), 3, 0.0); }
          for (int x = 0; x < 3; ++x) vals[3 * j + x] += w[x];
        };
        for (int64_t key : U) {
          int64_t t = key / NC;
          int s[3];
          unpack_shift((int)(key % NC), s);
          const int32_t* tv = &S.tets[4 * t];
          bool flag[4];
          int va = -1, nflag = 0;
          for (int j = 0; j < 4; ++j) {
            int sv[3];
            for (int x = 0; x < 3; ++x) sv[x] = S.shift[3 * tv[j] + x] + s[x];
            std::pair<int64_t, int> k2 = {S.pid[tv[j]], pack_shift(sv)};
            flag[j] = std::binary_search(near.begin(), near.end(), k2);
            nflag += flag[j];
            if (S.pid[tv[j]] == n && sv[0] == 0 && sv[1] == 0 && sv[2] == 0) va = j;
          }
          if (!nflag) continue;
          for (int j = 0; j < 4; ++j)
            for (int x = 0; x < 3; ++x) {
              I.P[j][x] = S.xyz[3 * tv[j] + x] + s[x] * S.L[x];
              I.g[j][x] = S.grads[12 * t + 3 * j + x];
            }
          for (int x = 0; x < 3; ++x) I.o[x] = o[x];
          I.run(va);
          const double Ms = S.Ms_tet[t];
          for (int k = 0; k < 4; ++k) {
            if (!flag[k]) continue;
            for (int m = 0; m < 4; ++m) {
              double w[3];
              for (int x = 0; x < 3; ++x) w[x] = Ms * (I.B[k][m][x] + I.g[k][x] * I.A[m]);
              add(S.pid[tv[m]], w);
            }
          }
        }
        // minus the point-charge value of each near source: -G0*(d) q_p, q_p = D_p . m
        const double* xn = &S.xyz[3 * S.parent[n]];
        for (auto& pr : near) {
          int64_t p = pr.first;
          int ell[3];
          unpack_shift(pr.second, ell);
          const double* xp = &S.xyz[3 * S.parent[p]];
          double d[3];
          for (int x = 0; x < 3; ++x) d[x] = xn[x] - xp[x] - ell[x] * S.L[x];
          double r = std::sqrt(dot3(d, d));
          if (r == 0.0) continue;
          double gi = 1.0 / r;
          double w[3];
          for (int x = 0; x < 3; ++x) w[x] = -gi * S.diagD[3 * p + x];
          add((int32_t)p, w);
          for (int64_t e = S.ring1.rowptr[p]; e < S.ring1.rowptr[p + 1]; ++e) {
            for (int x = 0; x < 3; ++x) w[x] = -gi * S.ring1.val[7 * e + 1 + x];
            add(S.ring1.col[e], w);
          }
        }
        // split into diagonal (kept only in the row sum) and sorted off-diagonals
        std::vector<int> ord;
        double rs[3] = {0, 0, 0};
        for (size_t j = 0; j < cols.size(); ++j) {
          for (int x = 0; x < 3; ++x) rs[x] += vals[3 * j + x];
          if (cols[j] != n) ord.push_back((int)j);
        }
        std::sort(ord.begin(), ord.end(), [&](int x, int y) { return cols[x] < cols[y]; });
        std::vector<int32_t> c2(ord.size());
        std::vector<double> v2(3 * ord.size());
        for (size_t j = 0; j < ord.size(); ++j) {
          c2[j] = cols[ord[j]];
          for (int x = 0; x < 3; ++x) v2[3 * j + x] = vals[3 * ord[j] + x];
        }
        for (int x = 0; x < 3; ++x) S.rowsumZ[3 * n + x] = rs[x];
        rcol[n] = std::move(c2);
        rval[n] = std::move(v2);
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    }
  }
  require(err.empty(), PMFEM_E_MESH, err);
  Csr& R = S.z0;
  R.n_rows = Np;
  R.nv = 3;
  R.rowptr.assign(Np + 1, 0);
  for (int64_t n = 0; n < Np; ++n) R.rowptr[n + 1] = R.rowptr[n] + (int64_t)rcol[n].size();
  R.col.resize(R.rowptr[Np]);
  R.val.resize(3 * R.rowptr[Np]);
#pragma omp parallel for
  for (int64_t n = 0; n < Np; ++n) {
    std::copy(rcol[n].begin(), rcol[n].end(), R.col.begin() + R.rowptr[n]);
    std::copy(rval[n].begin(), rval[n].end(), R.val.begin() + 3 * R.rowptr[n]);
  }
}

}  // namespace pmfem
