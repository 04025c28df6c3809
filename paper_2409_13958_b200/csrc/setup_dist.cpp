// Host setup, multi-GPU plan: contiguous row partition of the internal
// (box-sorted, z-slowest) order = slab-aligned mesh partition, and the halo exchange lists
// for the three gathered vectors of the evaluation:
//   M: m at the shared local-operator columns (K1: ring-1 + Z0)
//   Q: q at the C_box columns (K4)
//   U: u at the ring-1 columns (K5)
// Every rank runs the same deterministic setup on the full mesh, so each rank computes every
// peer's needs locally: no coordination is required to build the plan.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <omp.h>
#include "pmfem_internal.h"

namespace pmfem {

void setup_dist(HostSetup& S, int rank, int world) {
  require(world >= 1 && rank >= 0 && rank < world, PMFEM_E_INVALID_ARG, "bad rank / world");
  DistPlan& D = S.dist;
  D.rank = rank;
  D.world = world;
  const int64_t Np = S.Np;
  // per-row cost in bytes of the streamed operators (balanced partition)
  // (a device-built C_box is not on the host: its per-row cost is then taken as uniform)
  const bool have_cbox = !S.cbox.rowptr.empty();
  std::vector<double> cost(Np);
  for (int64_t i = 0; i < Np; ++i) {
    const int64_t r = S.perm[i];
    cost[i] = 64.0 + 20.0 * (S.ring1.rowptr[r + 1] - S.ring1.rowptr[r]) + 16.0 * (S.z0.rowptr[r + 1] - S.z0.rowptr[r]) +
              (have_cbox ? 8.0 * (S.cbox.rowptr[r + 1] - S.cbox.rowptr[r]) : 0.0);
  }
  std::vector<double> pre(Np + 1, 0.0);
  for (int64_t i = 0; i < Np; ++i) pre[i + 1] = pre[i] + cost[i];
  D.bounds.assign(world + 1, 0);
  D.bounds[world] = Np;
  for (int w = 1; w < world; ++w) {
    const double target = pre[Np] * w / world;
    int64_t i = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
    i = (i + 16) / 32 * 32;                              // SELL slices never straddle ranks
    D.bounds[w] = std::min<int64_t>(std::max<int64_t>(i, D.bounds[w - 1]), Np);
  }
  auto owner = [&](int64_t i) {
    return (int)(std::upper_bound(D.bounds.begin(), D.bounds.end(), i) - D.bounds.begin()) - 1;
  };
  // needed external rows of rank p for kind k
  const Csr* ops[3][2] = {{&S.ring1, &S.z0}, {&S.cbox, nullptr}, {&S.ring1, nullptr}};
  std::vector<std::vector<int32_t>> need[3];
  for (int k = 0; k < 3; ++k) need[k].resize(world);
  // C_box built on the device: q halo = every foreign node in the r_ER boxes (edge >= r_ER)
  // adjacent to a box holding an owned node -- a superset of the C_box columns
  // (PMFEM_GEOMETRIC_QHALO=1 forces this path on host-only contexts so the CPU tests cover it)
  const bool geometric_q = S.cbox.rowptr.empty() || std::getenv("PMFEM_GEOMETRIC_QHALO") != nullptr;
  std::vector<int64_t> bkey;
  int64_t nb[3] = {1, 1, 1};
  if (geometric_q && world > 1) {
    const double rer = S.rer_scale * std::max(S.delta[0], std::max(S.delta[1], S.delta[2]));
    double blo[3], bs[3];
    for (int a = 0; a < 3; ++a) {
      double lo = 1e300, hi = -1e300;
      for (int64_t n = 0; n < Np; ++n) { lo = std::min(lo, S.xw[3 * n + a]); hi = std::max(hi, S.xw[3 * n + a]); }
      if (S.periodic[a]) { blo[a] = 0; nb[a] = std::max<int64_t>(1, (int64_t)std::floor(S.L[a] / rer)); bs[a] = S.L[a] / nb[a]; }
      else { blo[a] = lo; nb[a] = (int64_t)std::floor((hi - lo) / rer) + 1; bs[a] = rer; }
    }
    bkey.resize(Np);
    for (int64_t i = 0; i < Np; ++i) {
      const int64_t r = S.perm[i];
      int64_t b[3];
      for (int a = 0; a < 3; ++a)
        b[a] = std::min<int64_t>(std::max<int64_t>((int64_t)std::floor((S.xw[3 * r + a] - blo[a]) / bs[a]), 0), nb[a] - 1);
      bkey[i] = (b[0] * nb[1] + b[1]) * nb[2] + b[2];
    }
    const int64_t nbox = nb[0] * nb[1] * nb[2];
    std::vector<std::vector<int32_t>> box_nodes(nbox);
    for (int64_t i = 0; i < Np; ++i) box_nodes[bkey[i]].push_back((int32_t)i);
    for (int p = 0; p < world; ++p) {
      std::vector<char> mark(nbox, 0);
      for (int64_t i = D.bounds[p]; i < D.bounds[p + 1]; ++i) {
        const int64_t b = bkey[i];
        const int64_t b0 = b / (nb[1] * nb[2]), b1 = (b / nb[2]) % nb[1], b2 = b % nb[2];
        for (int dx = -1; dx <= 1; ++dx)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz) {
              int64_t c[3] = {b0 + dx, b1 + dy, b2 + dz};
              bool ok = true;
              for (int a = 0; a < 3; ++a) {
                if (S.periodic[a]) c[a] = ((c[a] % nb[a]) + nb[a]) % nb[a];
                else ok &= (c[a] >= 0 && c[a] < nb[a]);
              }
              if (ok) mark[(c[0] * nb[1] + c[1]) * nb[2] + c[2]] = 1;
            }
      }
      std::vector<int32_t> v;
      for (int64_t b = 0; b < nbox; ++b)
        if (mark[b])
          for (int32_t i : box_nodes[b])
            if (i < D.bounds[p] || i >= D.bounds[p + 1]) v.push_back(i);
      std::sort(v.begin(), v.end());
      need[1][p] = std::move(v);
    }
  }
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int k = 0; k < 3; ++k)
    for (int p = 0; p < world; ++p) {
      if (k == 1 && geometric_q) continue;
      std::vector<int32_t> v;
      for (int64_t i = D.bounds[p]; i < D.bounds[p + 1]; ++i) {
        const int64_t r = S.perm[i];
        for (int o = 0; o < 2; ++o) {
          const Csr* A = ops[k][o];
          if (!A) continue;
          for (int64_t e = A->rowptr[r]; e < A->rowptr[r + 1]; ++e) {
            const int64_t c = S.iperm[A->col[e]];
            if (c < D.bounds[p] || c >= D.bounds[p + 1]) v.push_back((int32_t)c);
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
      // what peer p needs from me
      if (p != rank)
        for (int32_t c : need[k][p])
          if (owner(c) == rank) D.send_idx[k].push_back(c);
      D.send_ptr[k][p + 1] = (int64_t)D.send_idx[k].size();
      // what I need from peer p
      if (p != rank)
        for (int32_t c : need[k][rank])
          if (owner(c) == p) D.recv_idx[k].push_back(c);
      D.recv_ptr[k][p + 1] = (int64_t)D.recv_idx[k].size();
    }
  }
}

}  // namespace pmfem
