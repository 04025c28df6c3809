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
// Per row n the host enumerates near(n) (self, or the periodic 1-ring), the deduplicated set
// U(n) of tetrahedron images in the supports of the near sources (Eq. dedup) and
// the row's column list.  The element integrals (z0_cone.cuh, signed cone decomposition --
// independent of the oracle's Duffy/Gauss scheme) run on the host for host-only contexts and
// on the GPU (z0_gpu.cu, one thread per (row, element image)) for device contexts.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <omp.h>
#include "pmfem_internal.h"
#include "z0_cone.cuh"

namespace pmfem {

void build_tri_rules(TriRules& R) {
  // subdivision / rule-selection parameters (PMFEM_Z0_SPLIT, PMFEM_Z0_THR0/1/2 for
  // accuracy-vs-cost studies; defaults measured against the oracle in DESIGN.md)
  auto envd = [](const char* k, double d) { return std::getenv(k) ? std::atof(std::getenv(k)) : d; };
  R.split = envd("PMFEM_Z0_SPLIT", 1.0);
  R.thr0 = envd("PMFEM_Z0_THR0", 0.3);
  R.thr1 = envd("PMFEM_Z0_THR1", 0.6);
  R.thr2 = envd("PMFEM_Z0_THR2", 1e30);
  int off = 0;
  const int ns[4] = {4, 6, 8, 12};
  for (int r = 0; r < 4; ++r) {
    const int n = ns[r];
    double x[12], w[12];
    gauss_legendre01(n, x, w);
    R.off[r] = off;
    R.cnt[r] = n * n;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double u = x[i], v = x[j];
        R.l0[off] = 1 - u; R.l1[off] = u * (1 - v); R.l2[off] = u * v;
        R.w[off] = w[i] * w[j] * u;
        ++off;
      }
  }
}

namespace {

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

// open-addressing set of a row's columns (~65 unique among ~1000 candidates): insertion without
// sorting the candidates, then O(1) slot lookups
struct ColSet {
  static constexpr int CAP = 1024;
  int32_t key[CAP];
  int32_t val[CAP];
  int n = 0;
  void clear() { std::memset(key, 0xff, sizeof(key)); n = 0; }
  int find_pos(int32_t c) const {
    unsigned h = ((unsigned)c * 2654435761u) & (CAP - 1);
    while (key[h] != -1 && key[h] != c) h = (h + 1) & (CAP - 1);
    return (int)h;
  }
  bool insert(int32_t c) {               // false when the set is too full (caller falls back)
    const int h = find_pos(c);
    if (key[h] == c) return true;
    if (n >= CAP / 2) return false;
    key[h] = c;
    ++n;
    return true;
  }
  int& slot(int32_t c) { return val[find_pos(c)]; }
};

struct RowWork {
  Z0RowEnum e;
  ColSet cs;
};

}  // namespace

void z0_unpack_shift(int code, int s[3]) { unpack_shift(code, s); }

// near(n) (self, or the periodic 1-ring: every (LCA(v), relative shift) of the tets of every
// copy of n) and the deduplicated element images U(n) of the near sources' supports
// (Eq. dedup), with per image the near-source vertex flags and the observer vertex
void z0_enumerate_row(const HostSetup& S, int64_t n, Z0RowEnum& W) {
  const int NC = Z0_NC;
  auto& near = W.near;
  auto& U = W.U;
  near.clear(); U.clear(); W.its.clear();
  const int zero_code = ((8 * 17) + 8) * 17 + 8;
  if (S.z0_ring == 0) {
    near.push_back({n, zero_code});
  } else {
    for (int64_t ci = S.copies_ptr[n]; ci < S.copies_ptr[n + 1]; ++ci) {
      const int64_t c = S.copies[ci];
      for (int64_t ti = S.ntet_ptr[c]; ti < S.ntet_ptr[c + 1]; ++ti) {
        const int64_t t = S.ntet[ti];
        for (int b = 0; b < 4; ++b) {
          const int32_t v = S.tets[4 * t + b];
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
      const int64_t c = S.copies[ci];
      int s[3];
      for (int x = 0; x < 3; ++x) s[x] = ell[x] - S.shift[3 * c + x];
      const int code = pack_shift(s);
      for (int64_t ti = S.ntet_ptr[c]; ti < S.ntet_ptr[c + 1]; ++ti) U.push_back(S.ntet[ti] * NC + code);
    }
  }
  std::sort(U.begin(), U.end());
  U.erase(std::unique(U.begin(), U.end()), U.end());
  for (int64_t key : U) {
    const int64_t t = key / NC;
    int s[3];
    unpack_shift((int)(key % NC), s);
    const int32_t* tv = &S.tets[4 * t];
    unsigned flags = 0;
    int va = -1;
    for (int j = 0; j < 4; ++j) {
      int sv[3];
      for (int x = 0; x < 3; ++x) sv[x] = S.shift[3 * tv[j] + x] + s[x];
      std::pair<int64_t, int> k2 = {S.pid[tv[j]], pack_shift(sv)};
      if (std::binary_search(near.begin(), near.end(), k2)) flags |= 1u << j;
      if (S.pid[tv[j]] == n && sv[0] == 0 && sv[1] == 0 && sv[2] == 0) va = j;
    }
    if (!flags) continue;
    W.its.push_back({key, va, flags});
  }
}

void setup_z0(HostSetup& S) {
  const int64_t Np = S.Np;
  const int NC = 17 * 17 * 17;
  static TriRules rules;
  build_tri_rules(rules);
  std::vector<std::vector<int32_t>> rcol(Np);
  std::vector<std::vector<double>> rval(Np);
  S.rowsumZ.assign(3 * Np, 0.0);
  const bool on_device = S.z0_device >= 0;
  const int64_t chunk = on_device ? 250000 : Np;
  // rows to integrate (user parent ids): all, or a rank's own rows (distributed device contexts)
  std::vector<int64_t> rows_all;
  if (S.z0_rows.empty()) {
    rows_all.resize(Np);
    for (int64_t n = 0; n < Np; ++n) rows_all[n] = n;
  }
  const std::vector<int64_t>& rows = S.z0_rows.empty() ? rows_all : S.z0_rows;
  const int64_t nrows_tot = (int64_t)rows.size();
  std::string err;
  const bool verbose = std::getenv("PMFEM_VERBOSE") != nullptr;
  if (on_device) z0_device_begin(S, rules);
  // on an exception the device pipeline is released (z0_device_end) before it propagates
  struct PipeGuard {
    bool on; std::vector<std::vector<double>>* rv;
    ~PipeGuard() { if (on) { try { z0_device_end(*rv); } catch (...) {} } }
  } guard_pipe{on_device, &rval};
  for (int64_t c0 = 0; c0 < nrows_tot && err.empty(); c0 += chunk) {
    const double t_chunk = omp_get_wtime();
    const int64_t c1 = std::min(nrows_tot, c0 + chunk);
    long long host_pts = 0;
    std::vector<std::vector<Z0Item>> titems(omp_get_max_threads());
#pragma omp parallel reduction(+ : host_pts)
    {
      ConeIntegrator I;
      I.R = &rules;
      RowWork W;
      std::vector<Z0Item>& items = titems[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 16)
      for (int64_t j = c0; j < c1; ++j) {
        const int64_t n = rows[j];
        try {
          z0_enumerate_row(S, n, W.e);
          auto& near = W.e.near;
          // column list: every vertex of every contributing element image + the D rows of the
          // near sources (point-charge subtraction)
          std::vector<int32_t>& cols = rcol[n];
          cols.clear();
          W.cs.clear();
          bool cs_ok = true;
          auto add_col = [&](int32_t c) {
            if (cs_ok && !W.cs.insert(c)) cs_ok = false;
            cols.push_back(c);
          };
          auto& its = W.e.its;
          for (auto& it : its) {
            const int32_t* tv = &S.tets[4 * (it.key / NC)];
            for (int j = 0; j < 4; ++j) add_col(S.pid[tv[j]]);
          }
          const double* xn = &S.xyz[3 * S.parent[n]];
          for (auto& pr : near) {
            int ell[3];
            unpack_shift(pr.second, ell);
            const double* xp = &S.xyz[3 * S.parent[pr.first]];
            double d[3];
            for (int x = 0; x < 3; ++x) d[x] = xn[x] - xp[x] - ell[x] * S.L[x];
            if (d[0] == 0 && d[1] == 0 && d[2] == 0) continue;
            add_col((int32_t)pr.first);
            for (int64_t e = S.ring1.rowptr[pr.first]; e < S.ring1.rowptr[pr.first + 1]; ++e) add_col(S.ring1.col[e]);
          }
          if (cs_ok) {                     // the set's unique columns, sorted; slots from the set
            cols.clear();
            for (int h = 0; h < ColSet::CAP; ++h)
              if (W.cs.key[h] != -1) cols.push_back(W.cs.key[h]);
            std::sort(cols.begin(), cols.end());
            for (size_t i = 0; i < cols.size(); ++i) W.cs.slot(cols[i]) = (int)i;
          } else {
            std::sort(cols.begin(), cols.end());
            cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
          }
          std::vector<double>& vals = rval[n];
          vals.assign(3 * cols.size(), 0.0);
          auto slot = [&](int32_t col) {
            if (cs_ok) return W.cs.slot(col);
            return (int)(std::lower_bound(cols.begin(), cols.end(), col) - cols.begin());
          };
          for (auto& it : its) {
            const int64_t t = it.key / NC;
            const int32_t* tv = &S.tets[4 * t];
            if (on_device) {
              Z0Item z;
              z.row = n;
              z.slot = (int32_t)(j - c0);
              z.tet = (int32_t)t;
              z.code = (int16_t)(it.key % NC);
              z.va = (int8_t)it.va;
              z.flags = (uint8_t)it.flags;
              for (int m = 0; m < 4; ++m) z.pos[m] = (int16_t)slot(S.pid[tv[m]]);
              items.push_back(z);
              continue;
            }
            int s[3];
            unpack_shift((int)(it.key % NC), s);
            for (int j = 0; j < 4; ++j)
              for (int x = 0; x < 3; ++x) {
                I.P[j][x] = S.xyz[3 * tv[j] + x] + s[x] * S.L[x];
                I.g[j][x] = S.grads[12 * t + 3 * j + x];
              }
            for (int x = 0; x < 3; ++x) I.o[x] = xn[x];
            I.run(it.va);
            const double Ms = S.Ms_tet[t];
            for (int k = 0; k < 4; ++k) {
              if (!(it.flags & (1u << k))) continue;
              for (int m = 0; m < 4; ++m) {
                const int p = slot(S.pid[tv[m]]);
                for (int x = 0; x < 3; ++x) vals[3 * p + x] += Ms * (I.B[k][m][x] + I.g[k][x] * I.A[m]);
              }
            }
          }
          // minus the point-charge value of each near source: -G0*(d) q_p, q_p = D_p . m
          for (auto& pr : near) {
            const int64_t p = pr.first;
            int ell[3];
            unpack_shift(pr.second, ell);
            const double* xp = &S.xyz[3 * S.parent[p]];
            double d[3];
            for (int x = 0; x < 3; ++x) d[x] = xn[x] - xp[x] - ell[x] * S.L[x];
            const double r = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            if (r == 0.0) continue;
            const double gi = 1.0 / r;
            int sp = slot((int32_t)p);
            for (int x = 0; x < 3; ++x) vals[3 * sp + x] -= gi * S.diagD[3 * p + x];
            for (int64_t e = S.ring1.rowptr[p]; e < S.ring1.rowptr[p + 1]; ++e) {
              sp = slot(S.ring1.col[e]);
              for (int x = 0; x < 3; ++x) vals[3 * sp + x] -= gi * S.ring1.val[7 * e + 1 + x];
            }
          }
        } catch (const std::exception& e) {
#pragma omp critical
          err = e.what();
        }
      }
      host_pts += I.npts;
    }
    const double t_enum = omp_get_wtime();
    if (on_device && err.empty()) z0_device_integrate(S, titems, rcol, rval, rules, rows.data() + c0, c1 - c0);
    if (verbose)
      std::fprintf(stderr, "[pmfem]   z0 rows %lld-%lld: enumerate %.2f s, integrate %.2f s (host quadrature points %lld)\n",
                   (long long)c0, (long long)c1, t_enum - t_chunk, omp_get_wtime() - t_enum, host_pts);
  }
  if (on_device) { guard_pipe.on = false; z0_device_end(rval); }   // the last chunks' values
  require(err.empty(), PMFEM_E_MESH, err);
  // split diagonal (kept only in the row sum) from the off-diagonal entries
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t n = 0; n < Np; ++n) {
    std::vector<int32_t> c2;
    std::vector<double> v2;
    double rs[3] = {0, 0, 0};
    for (size_t j = 0; j < rcol[n].size(); ++j) {
      for (int x = 0; x < 3; ++x) rs[x] += rval[n][3 * j + x];
      if (rcol[n][j] == n) continue;
      c2.push_back(rcol[n][j]);
      for (int x = 0; x < 3; ++x) v2.push_back(rval[n][3 * j + x]);
    }
    for (int x = 0; x < 3; ++x) S.rowsumZ[3 * n + x] = rs[x];
    rcol[n] = std::move(c2);
    rval[n] = std::move(v2);
  }
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
