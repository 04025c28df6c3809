// Host setup, mesh layer: validation, orientation, T-PBC pair detection by spatial hashing,
// union-find LCA folding, lattice shifts, classification, element geometry.
//   P:44   T-PBC: "one of its periodic images ... can still be found within the 0th unit cell"
//   P:96   PBC pairs merged "to their lowest common ancestors (LCA) by the union-find algorithm";
//          N' = N - N_PBC unknowns
//   P:80-84 linear tetrahedral basis phi_n
#include <algorithm>
#include <array>
#include <cmath>
#include <numeric>
#include <omp.h>
#include "pmfem_internal.h"

namespace pmfem {

namespace {

struct CellHash {
  double lo[3], cell;
  int64_t dim[3];
  std::vector<std::pair<int64_t, int64_t>> keys;   // (cell key, node)

  int64_t key_of(const int64_t c[3]) const { return (c[0] * dim[1] + c[1]) * dim[2] + c[2]; }

  void build(const std::vector<double>& xyz, int64_t n, double cell_size) {
    cell = cell_size;
    double hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = 1e300; hi[a] = -1e300; }
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], xyz[3 * i + a]); hi[a] = std::max(hi[a], xyz[3 * i + a]); }
    for (int a = 0; a < 3; ++a) dim[a] = (int64_t)std::floor((hi[a] - lo[a]) / cell) + 1;
    keys.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      int64_t c[3];
      for (int a = 0; a < 3; ++a) c[a] = (int64_t)std::floor((xyz[3 * i + a] - lo[a]) / cell);
      keys[i] = {key_of(c), i};
    }
    std::sort(keys.begin(), keys.end());
  }

  // all nodes within tol (Euclidean) of point p
  template <class F>
  void query(const double p[3], const std::vector<double>& xyz, double tol, F&& f) const {
    int64_t c[3];
    int lo_o[3], hi_o[3];
    for (int a = 0; a < 3; ++a) {
      const double u = (p[a] - lo[a]) / cell;
      c[a] = (int64_t)std::floor(u);
      // only the neighbouring cells the tol-ball reaches (tol << cell: almost always one cell)
      const double f = (u - (double)c[a]) * cell;
      lo_o[a] = (f <= tol) ? -1 : 0;
      hi_o[a] = (cell - f <= tol) ? 1 : 0;
    }
    for (int dx = lo_o[0]; dx <= hi_o[0]; ++dx)
      for (int dy = lo_o[1]; dy <= hi_o[1]; ++dy)
        for (int dz = lo_o[2]; dz <= hi_o[2]; ++dz) {
          int64_t cc[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
          bool ok = true;
          for (int a = 0; a < 3; ++a) ok &= (cc[a] >= 0 && cc[a] < dim[a]);
          if (!ok) continue;
          int64_t k = key_of(cc);
          auto it = std::lower_bound(keys.begin(), keys.end(), std::make_pair(k, (int64_t)-1));
          for (; it != keys.end() && it->first == k; ++it) {
            int64_t j = it->second;
            double d2 = 0;
            for (int a = 0; a < 3; ++a) { double d = xyz[3 * j + a] - p[a]; d2 += d * d; }
            if (d2 <= tol * tol) f(j);
          }
        }
  }
};

int64_t uf_find(std::vector<int64_t>& par, int64_t i) {
  int64_t r = i;
  while (par[r] != r) r = par[r];
  while (par[i] != r) { int64_t nx = par[i]; par[i] = r; i = nx; }
  return r;
}

}  // namespace

void setup_mesh(HostSetup& S, const pmfem_mesh* mesh, const pmfem_periodicity* per) {
  require(mesh && per && mesh->xyz && mesh->tets, PMFEM_E_INVALID_ARG, "NULL mesh/periodicity/array");
  require(mesh->n_nodes > 0 && mesh->n_tets > 0, PMFEM_E_INVALID_ARG, "empty mesh");
  require(mesh->n_regions >= 1 && mesh->Ms && mesh->Aex, PMFEM_E_INVALID_ARG, "materials missing");
  require(mesh->n_nodes < (int64_t(1) << 31), PMFEM_E_INVALID_ARG, "n_nodes must fit int32");
  S.N = mesh->n_nodes;
  S.T = mesh->n_tets;
  S.xyz.assign(mesh->xyz, mesh->xyz + 3 * S.N);
  S.tets.assign(mesh->tets, mesh->tets + 4 * S.T);
  int nper = 0;
  // lattice vectors: rows of lattice[3][3]; P:36-43 writes them L_x x^, L_y y^, L_z z^, so they
  // must be diagonal (the grid, stencils and FFT are axis-aligned)
  double lmax = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) lmax = std::max(lmax, std::fabs(per->lattice[a][b]));
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      if (a != b)
        require(std::fabs(per->lattice[a][b]) <= 1e-12 * lmax, PMFEM_E_INVALID_ARG,
                "non-diagonal lattice vectors (P:36 uses L_x x, L_y y, L_z z)");
  for (int a = 0; a < 3; ++a) {
    S.periodic[a] = per->periodic[a] ? 1 : 0;
    S.L[a] = S.periodic[a] ? per->lattice[a][a] : 0.0;
    if (S.periodic[a]) require(S.L[a] > 0, PMFEM_E_INVALID_ARG, "non-positive period");
    nper += S.periodic[a];
  }
  (void)nper;   // nper == 0: non-periodic mode, free-space kernel, 2N padding on every axis

  // materials per tet
  S.Ms_tet.resize(S.T);
  S.Aex_tet.resize(S.T);
  for (int64_t t = 0; t < S.T; ++t) {
    int r = mesh->region ? mesh->region[t] : 0;
    require(r >= 0 && r < mesh->n_regions, PMFEM_E_MESH, "region id out of range at tet " + std::to_string(t));
    S.Ms_tet[t] = mesh->Ms[r];
    S.Aex_tet[t] = mesh->Aex[r];
    require(S.Ms_tet[t] > 0, PMFEM_E_INVALID_ARG, "Ms must be positive");
  }

  // orientation + degenerate check
  S.vol.resize(S.T);
  S.grads.resize(12 * S.T);
  double sumv = 0;
  int64_t bad_index = -1;
#pragma omp parallel for reduction(+ : sumv) reduction(max : bad_index)
  for (int64_t t = 0; t < S.T; ++t) {
    int32_t* v = &S.tets[4 * t];
    bool ok = true;
    for (int k = 0; k < 4; ++k) ok &= v[k] >= 0 && v[k] < S.N;
    if (!ok) { bad_index = std::max(bad_index, t); continue; }
    const double* p0 = &S.xyz[3 * v[0]];
    double e[3][3];
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) e[k][a] = S.xyz[3 * v[k + 1] + a] - p0[a];
    double c23[3] = {e[1][1] * e[2][2] - e[1][2] * e[2][1], e[1][2] * e[2][0] - e[1][0] * e[2][2],
                     e[1][0] * e[2][1] - e[1][1] * e[2][0]};
    double det = e[0][0] * c23[0] + e[0][1] * c23[1] + e[0][2] * c23[2];
    if (det < 0) std::swap(v[1], v[2]);
    S.vol[t] = std::fabs(det) / 6.0;
    sumv += S.vol[t];
  }
  require(bad_index < 0, PMFEM_E_MESH, "tet index out of range at tet " + std::to_string(bad_index));
  double meanv = sumv / S.T;
  int64_t degenerate = -1;
#pragma omp parallel for reduction(max : degenerate)
  for (int64_t t = 0; t < S.T; ++t)
    if (!(S.vol[t] >= 1e-12 * meanv)) degenerate = std::max(degenerate, t);
  require(degenerate < 0, PMFEM_E_MESH, "degenerate tetrahedron " + std::to_string(degenerate));

  // element gradients grad(phi_i) = rows of J^-1 (J columns = P_i - P_0), phi_0 = 1 - sum
  double min_edge2 = 1e300;
#pragma omp parallel for reduction(min : min_edge2)
  for (int64_t t = 0; t < S.T; ++t) {
    const int32_t* v = &S.tets[4 * t];
    double P[4][3];
    for (int k = 0; k < 4; ++k)
      for (int a = 0; a < 3; ++a) P[k][a] = S.xyz[3 * v[k] + a];
    double e[3][3];
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) e[k][a] = P[k + 1][a] - P[0][a];
    auto cross = [](const double* x, const double* y, double* z) {
      z[0] = x[1] * y[2] - x[2] * y[1]; z[1] = x[2] * y[0] - x[0] * y[2]; z[2] = x[0] * y[1] - x[1] * y[0];
    };
    double g[4][3];
    cross(e[1], e[2], g[1]);
    cross(e[2], e[0], g[2]);
    cross(e[0], e[1], g[3]);
    double det = e[0][0] * g[1][0] + e[0][1] * g[1][1] + e[0][2] * g[1][2];
    for (int k = 1; k < 4; ++k)
      for (int a = 0; a < 3; ++a) g[k][a] /= det;
    for (int a = 0; a < 3; ++a) g[0][a] = -(g[1][a] + g[2][a] + g[3][a]);
    for (int k = 0; k < 4; ++k)
      for (int a = 0; a < 3; ++a) S.grads[12 * t + 3 * k + a] = g[k][a];
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j) {
        double d2 = 0;
        for (int a = 0; a < 3; ++a) d2 += (P[i][a] - P[j][a]) * (P[i][a] - P[j][a]);
        min_edge2 = std::min(min_edge2, d2);
      }
  }
  double min_edge = std::sqrt(min_edge2);
  S.match_tol = per->match_tol > 0 ? per->match_tol : 1e-6 * min_edge;
  const double tol = S.match_tol;

  // T-PBC pairs by hashing translated coordinates; union-find with min root
  std::vector<int64_t> uf(S.N);
  std::iota(uf.begin(), uf.end(), 0);
  CellHash H;
  H.build(S.xyz, S.N, std::max(0.5 * min_edge, 4 * tol));
  std::vector<std::array<int, 3>> offs;
  for (int gx = -1; gx <= 1; ++gx)
    for (int gy = -1; gy <= 1; ++gy)
      for (int gz = -1; gz <= 1; ++gz) {
        int o[3] = {gx, gy, gz};
        bool ok = (gx || gy || gz);
        for (int a = 0; a < 3; ++a) ok &= (S.periodic[a] || o[a] == 0);
        if (ok) offs.push_back({gx, gy, gz});
      }
  std::vector<std::pair<int64_t, int64_t>> pairs;
  std::string err;
#pragma omp parallel
  {
    std::vector<std::pair<int64_t, int64_t>> local;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < S.N; ++i) {
      for (auto& o : offs) {
        double p[3];
        for (int a = 0; a < 3; ++a) p[a] = S.xyz[3 * i + a] + o[a] * S.L[a];
        int64_t found = -1, cnt = 0;
        H.query(p, S.xyz, tol, [&](int64_t j) { if (j != i) { ++cnt; if (found < 0 || j < found) found = j; } });
        if (cnt > 1) {
#pragma omp critical
          err = "PBC ambiguous: node " + std::to_string(i) + " has " + std::to_string(cnt) + " image candidates";
        }
        if (found >= 0 && found > i) local.push_back({i, found});
      }
    }
#pragma omp critical
    pairs.insert(pairs.end(), local.begin(), local.end());
  }
  require(err.empty(), PMFEM_E_PBC_AMBIGUOUS, err);
  for (auto& pr : pairs) {
    int64_t a = uf_find(uf, pr.first), b = uf_find(uf, pr.second);
    if (a != b) { if (a < b) uf[b] = a; else uf[a] = b; }
  }
  S.lca.resize(S.N);
  for (int64_t i = 0; i < S.N; ++i) S.lca[i] = uf_find(uf, i);

  // parents numbered by increasing original index (user order)
  S.pid.assign(S.N, -1);
  S.parent.clear();
  for (int64_t i = 0; i < S.N; ++i)
    if (S.lca[i] == i) { S.pid[i] = (int32_t)S.parent.size(); S.parent.push_back(i); }
  S.Np = (int64_t)S.parent.size();
  for (int64_t i = 0; i < S.N; ++i) S.pid[i] = S.pid[S.lca[i]];

  // lattice shifts + consistency
  S.shift.assign(3 * S.N, 0);
  for (int64_t i = 0; i < S.N; ++i) {
    int64_t r = S.lca[i];
    for (int a = 0; a < 3; ++a) {
      double d = S.xyz[3 * i + a] - S.xyz[3 * r + a];
      if (S.periodic[a]) {
        double k = std::nearbyint(d / S.L[a]);
        require(std::fabs(d - k * S.L[a]) <= tol, PMFEM_E_PBC_INCONSISTENT,
                "PBC component of node " + std::to_string(i) + " is not a period translate");
        S.shift[3 * i + a] = (int32_t)k;
      } else {
        require(std::fabs(d) <= tol, PMFEM_E_PBC_INCONSISTENT,
                "PBC component of node " + std::to_string(i) + " differs on a non-periodic axis");
      }
    }
  }

  // classification
  S.touching = S.Np < S.N;
  S.protruding = 0;
  for (int a = 0; a < 3; ++a) {
    double lo = 1e300, hi = -1e300;
    for (int64_t i = 0; i < S.N; ++i) { lo = std::min(lo, S.xyz[3 * i + a]); hi = std::max(hi, S.xyz[3 * i + a]); }
    if (S.periodic[a] && hi - lo > S.L[a] + tol) S.protruding = 1;
  }

  // copies (parent -> nodes) and node -> tets
  S.copies_ptr.assign(S.Np + 1, 0);
  for (int64_t i = 0; i < S.N; ++i) S.copies_ptr[S.pid[i] + 1]++;
  for (int64_t p = 0; p < S.Np; ++p) S.copies_ptr[p + 1] += S.copies_ptr[p];
  S.copies.resize(S.N);
  {
    std::vector<int64_t> fill(S.copies_ptr.begin(), S.copies_ptr.end() - 1);
    for (int64_t i = 0; i < S.N; ++i) S.copies[fill[S.pid[i]]++] = i;
  }
  S.ntet_ptr.assign(S.N + 1, 0);
  for (int64_t t = 0; t < S.T; ++t)
    for (int k = 0; k < 4; ++k) S.ntet_ptr[S.tets[4 * t + k] + 1]++;
  for (int64_t i = 0; i < S.N; ++i) S.ntet_ptr[i + 1] += S.ntet_ptr[i];
  S.ntet.resize(4 * S.T);
  {
    std::vector<int64_t> fill(S.ntet_ptr.begin(), S.ntet_ptr.end() - 1);
    for (int64_t t = 0; t < S.T; ++t)
      for (int k = 0; k < 4; ++k) S.ntet[fill[S.tets[4 * t + k]]++] = t;
  }
}

}  // namespace pmfem
