// Host setup, multi-GPU plan: the internal rows (box-sorted, z slowest) are
// partitioned at anchor-z-plane boundaries = the z slabs of the FFT (slab-aligned mesh
// partition), and the halo exchange lists of the evaluation are built:
//   M: m at the own rows' local-operator columns (K1: ring-1 + Z0)
//   Q: q of the rows anchored in the planes bordering the slab (K2 stencils, C_box columns)
//   U: u at the ring-1 columns (K5), plus the U ghost planes K4's stencils read
// Every rank runs the same deterministic setup on the full mesh, so each rank computes every
// peer's needs locally: no coordination is required to build the plan.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <omp.h>
#include "pmfem_internal.h"

namespace pmfem {

namespace {
// stored (wrapped / clamped) anchor z plane of internal row i
inline int anchor_z(const HostSetup& S, int64_t i) {
  int v = S.st_s[3 * S.perm[i] + 2];
  if (S.periodic[2]) v = ((v % S.grid_n[2]) + S.grid_n[2]) % S.grid_n[2];
  return v;
}
}  // namespace

int slab_granularity(const HostSetup& S, int world) {
  // planes per K2 tile along z: a power of two <= 8 leaving >= 1 granule per rank
  int gz = 8;
  while (gz > 1 && (S.grid_n[2] % gz != 0 || S.grid_n[2] / gz < world)) gz >>= 1;
  return gz;
}

std::vector<int32_t> slab_planes(const HostSetup& S, int world, int gz) {
  const int n2 = S.grid_n[2];
  require(n2 / gz >= world, PMFEM_E_INVALID_ARG, "fewer z planes than ranks: no slab decomposition");
  std::vector<int64_t> cnt(n2 + 1, 0);                  // rows anchored below plane z
  for (int64_t i = 0; i < S.Np; ++i) cnt[anchor_z(S, i) + 1]++;
  for (int z = 0; z < n2; ++z) cnt[z + 1] += cnt[z];
  std::vector<int32_t> Z(world + 1, 0);
  Z[world] = n2;
  for (int w = 1; w < world; ++w) {
    const double target = (double)S.Np * w / world;
    int best = Z[w - 1] + gz;
    double bd = 1e300;
    for (int z = Z[w - 1] + gz; z <= n2 - (world - w) * gz; z += gz) {
      const double d = std::fabs((double)cnt[z] - target);
      if (d < bd) { bd = d; best = z; }
    }
    Z[w] = best;
  }
  return Z;
}

// Partition: the internal rows are box-sorted with z slowest, so the rows anchored
// in the z planes [Z_r, Z_r+1) are contiguous; the plane boundaries balance the row counts and are
// the z slabs of the FFT.  Needs setup_order.
void setup_dist(HostSetup& S, int rank, int world) {
  require(world >= 1 && rank >= 0 && rank < world, PMFEM_E_INVALID_ARG, "bad rank / world");
  DistPlan& D = S.dist;
  D.rank = rank;
  D.world = world;
  const int64_t Np = S.Np;
  const int n2 = S.grid_n[2];
  if (world == 1) {
    D.bounds = {0, Np};
    D.planes = {0, n2};
    return;
  }
  D.planes = slab_planes(S, world, slab_granularity(S, world));
  D.bounds.assign(world + 1, 0);
  D.bounds[world] = Np;
  for (int w = 1; w < world; ++w) {
    int64_t i = D.bounds[w - 1];
    while (i < Np && anchor_z(S, i) < D.planes[w]) ++i;
    D.bounds[w] = i;
  }
  // q halo bands: K2's stencils reach p planes below the slab; C_box columns lie within
  // R_z = ceil(r_ER / Delta_z + 1) - 1 anchor planes (+1 plane of rounding margin) either way
  const double rer = S.rer_scale * std::max(S.delta[0], std::max(S.delta[1], S.delta[2]));
  const int Rz = (int)std::ceil(rer / S.delta[2] + 1.0) - 1 + 1;
  D.qband_lo = std::max(Rz, S.order);
  D.qband_hi = Rz;
  // the own rows' Z0 (the setup's dominant cost) is built on this rank only
  S.z0_rows.clear();
  for (int64_t i = D.lo(); i < D.hi(); ++i) S.z0_rows.push_back(S.perm[i]);
  std::sort(S.z0_rows.begin(), S.z0_rows.end());
}

// Halo lists (after Z0): per peer, the rows of my gathered vectors they need / I need from them
//   M: m at the own rows' local-operator columns (K1: ring-1 + Z0)
//   Q: q of every row anchored within the q bands around the own slab (K2 + C_box)
//   U: u at the ring-1 columns (K5)
// and the U ghost planes K4 reads above the own slab.  Every rank derives every peer's plan.
void setup_dist_halos(HostSetup& S) {
  DistPlan& D = S.dist;
  const int world = D.world, rank = D.rank;
  if (world == 1) {
    for (int k = 0; k < 3; ++k) {
      D.send_ptr[k].assign(2, 0); D.recv_ptr[k].assign(2, 0);
      D.send_idx[k].clear(); D.recv_idx[k].clear();
    }
    return;
  }
  const int64_t Np = S.Np;
  const int n2 = S.grid_n[2];
  auto owner = [&](int64_t i) {
    return (int)(std::upper_bound(D.bounds.begin(), D.bounds.end(), i) - D.bounds.begin()) - 1;
  };
  std::vector<int> az(Np);
  for (int64_t i = 0; i < Np; ++i) az[i] = anchor_z(S, i);
  const Csr* ops[3][2] = {{&S.ring1, &S.z0}, {nullptr, nullptr}, {&S.ring1, nullptr}};
  std::vector<std::vector<int32_t>> need[3];
  for (int k = 0; k < 3; ++k) need[k].resize(world);
  // rows of peer p's halo in plane terms: z within [Z_p - lo, Z_p+1 + hi) (wrapped when periodic)
  auto in_band = [&](int z, int p) {
    const int Z0 = D.planes[p], Z1 = D.planes[p + 1];
    for (int d = 1; d <= D.qband_lo; ++d) {
      int zz = Z0 - d;
      if (S.periodic[2]) zz = ((zz % n2) + n2) % n2;
      if (zz == z) return true;
    }
    for (int d = 0; d < D.qband_hi; ++d) {
      int zz = Z1 + d;
      if (S.periodic[2]) zz = ((zz % n2) + n2) % n2;
      if (zz == z) return true;
    }
    return false;
  };
#pragma omp parallel for schedule(dynamic)
  for (int p = 0; p < world; ++p) {
    std::vector<char> band(n2, 0);
    for (int z = 0; z < n2; ++z) band[z] = in_band(z, p) && !(z >= D.planes[p] && z < D.planes[p + 1]);
    std::vector<int32_t> v;
    for (int64_t i = 0; i < Np; ++i)
      if (band[az[i]] && (i < D.bounds[p] || i >= D.bounds[p + 1])) v.push_back((int32_t)i);
    need[1][p] = std::move(v);
  }
  // M: K1's columns are the ring-1 (L, D) and the Z0 columns; Z0's lie in the periodic 2-ring
  // (near sources = 1-ring, their support elements' vertices and D rows = 2-ring).  A rank builds
  // Z0 for its own rows only, so every rank uses the 2-ring (ring1 o ring1, known for all rows)
  // to derive every peer's needs.  U: K5's ring-1 columns.
  (void)ops;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int k = 0; k < 3; k += 2)
    for (int p = 0; p < world; ++p) {
      std::vector<int32_t> v;
      const Csr& A = S.ring1;
      for (int64_t i = D.bounds[p]; i < D.bounds[p + 1]; ++i) {
        const int64_t r = S.perm[i];
        for (int64_t e = A.rowptr[r]; e < A.rowptr[r + 1]; ++e) {
          const int64_t c = S.iperm[A.col[e]];
          if (c < D.bounds[p] || c >= D.bounds[p + 1]) v.push_back((int32_t)c);
          if (k == 0) {
            const int64_t rc = A.col[e];
            for (int64_t f = A.rowptr[rc]; f < A.rowptr[rc + 1]; ++f) {
              const int64_t c2 = S.iperm[A.col[f]];
              if (c2 < D.bounds[p] || c2 >= D.bounds[p + 1]) v.push_back((int32_t)c2);
            }
          }
        }
      }
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      need[k][p] = std::move(v);
    }
  for (int k = 0; k < 3; ++k) {
    D.send_ptr[k].assign(world + 1, 0);
    D.recv_ptr[k].assign(world + 1, 0);
    D.send_idx[k].clear();
    D.recv_idx[k].clear();
    for (int p = 0; p < world; ++p) {
      if (p != rank)
        for (int32_t c : need[k][p])
          if (owner(c) == rank) D.send_idx[k].push_back(c);
      D.send_ptr[k][p + 1] = (int64_t)D.send_idx[k].size();
      if (p != rank)
        for (int32_t c : need[k][rank])
          if (owner(c) == p) D.recv_idx[k].push_back(c);
      D.recv_ptr[k][p + 1] = (int64_t)D.recv_idx[k].size();
    }
  }
  // U ghost planes: rank r's K4 reads planes up to Z_r+1 - 1 + p (anchors + stencil; periodic z
  // wraps, non-periodic anchors are clamped so the reach stays < n2)
  auto ghost = [&](int r) {
    std::vector<int> g;
    for (int d = 0; d < S.order; ++d) {
      int z = D.planes[r + 1] + d;
      if (S.periodic[2]) z %= n2;
      else if (z >= n2) continue;
      if (!(z >= D.planes[r] && z < D.planes[r + 1])) g.push_back(z);
    }
    return g;
  };
  auto ranges = [&](const std::vector<int>& zs, int p, std::vector<int32_t>* out) {
    // planes of zs owned by p, as up to two contiguous (plane0, count) ranges
    std::vector<int> mine;
    for (int z : zs)
      if (z >= D.planes[p] && z < D.planes[p + 1]) mine.push_back(z);
    std::sort(mine.begin(), mine.end());
    int nr = 0;
    for (size_t i = 0; i < mine.size();) {
      size_t j = i + 1;
      while (j < mine.size() && mine[j] == mine[j - 1] + 1) ++j;
      require(nr < 2, PMFEM_E_STATE, "ghost planes in more than two ranges");
      out[nr].push_back(mine[i]);
      out[nr].push_back((int)(j - i));
      ++nr;
      i = j;
    }
    for (; nr < 2; ++nr) { out[nr].push_back(0); out[nr].push_back(0); }
  };
  for (int k = 0; k < 2; ++k) { D.gsend[k].clear(); D.grecv[k].clear(); }
  const std::vector<int> mine = ghost(rank);
  for (int p = 0; p < world; ++p) {
    ranges(p == rank ? std::vector<int>() : ghost(p), rank, D.gsend);   // my planes p needs
    ranges(p == rank ? std::vector<int>() : mine, p, D.grecv);         // p's planes I need
  }
}

}  // namespace pmfem
