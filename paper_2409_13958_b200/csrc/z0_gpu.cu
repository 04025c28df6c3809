// GPU integration of the Z0 element integrals: the (row, element image) tasks
// enumerated by setup_z0.cpp, the same signed-cone quadrature (z0_cone.cuh: the same adaptive
// face subdivision, the same collapsed Gauss rules) as the host path, in fp64; contributions are
// accumulated with fp64 atomics into the row's value slots.
//
// k_z0_warp (default): ONE WARP PER TASK.  Lane 0 runs the adaptive subdivision of a face on a
// shared-memory stack and emits leaf triangles into a shared-memory buffer; all 32 lanes then
// share the leaves' quadrature points (flattened over the batch), each lane accumulating the 34
// moments (A[4], B[10][3]) in registers; a butterfly reduction at the end of the task gives every
// lane the totals and lanes scatter the 48 (k, m, axis) contributions.  No divergence inside
// the point loop and no per-thread local-memory stack (the thread-per-task kernel k_z0_items,
// PMFEM_Z0_THREAD=1, spilled its 24-triangle stack and diverged on the adaptive depth).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include <omp.h>
#include "pmfem_internal.h"
#include "z0_cone.cuh"

namespace pmfem {

namespace {

#define CKZ(x)                                                                                  \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) throw Error(PMFEM_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
T* up(const T* src, size_t n) {
  T* p = nullptr;
  CKZ(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  if (n) CKZ(cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

struct Lat { double L[3]; };

__global__ void k_z0_items(const Z0Item* __restrict__ items, int64_t nitems, const double* __restrict__ xyz,
                           const int32_t* __restrict__ tets, const int64_t* __restrict__ parent,
                           const double* __restrict__ Ms_tet, Lat lat, const TriRules* __restrict__ rules,
                           const int64_t* __restrict__ rowbase, int64_t r0, double* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nitems) return;
  const Z0Item it = items[i];
  int code = it.code;
  int s[3];
  s[2] = code % 17 - 8; code /= 17;
  s[1] = code % 17 - 8; code /= 17;
  s[0] = code - 8;
  ConeIntegrator I;
  I.R = rules;
  const int32_t* tv = tets + 4 * (int64_t)it.tet;
  for (int j = 0; j < 4; ++j)
    for (int x = 0; x < 3; ++x) I.P[j][x] = xyz[3 * (int64_t)tv[j] + x] + s[x] * lat.L[x];
  tet_grads(I.P, I.g);
  const int64_t pn = parent[it.row];
  for (int x = 0; x < 3; ++x) I.o[x] = xyz[3 * pn + x];
  I.run(it.va);
  const double Ms = Ms_tet[it.tet];
  double* v = vals + rowbase[it.slot];
  for (int k = 0; k < 4; ++k) {
    if (!(it.flags & (1u << k))) continue;
    for (int m = 0; m < 4; ++m)
      for (int x = 0; x < 3; ++x) atomicAdd(v + 3 * it.pos[m] + x, Ms * (I.B[k][m][x] + I.g[k][x] * I.A[m]));
  }
}

// ---- one warp per task
constexpr int Z0W_WARPS = 4;           // warps per CTA
constexpr int Z0W_LEAVES = 48;         // leaf buffer per warp (flushed when full)
// POP: sub-triangles examined per step (one per lane 0..POP-1); the stack holds
// >= 1 + 7 levels x 4 POP entries and never overflows (see below).  POP = 8 (default) halves the
// stack and, with at most 102 registers (5 CTAs per SM), doubles the resident warps: the kernel
// is latency-bound (ncu C5: 18 % warps active at POP = 16 / 168 registers, fp64 pipe 26 %);
// PMFEM_Z0_POP=16 selects the round-2 configuration.
template <int POP> struct Z0Stack { static constexpr int N = ((1 + 7 * 4 * POP) + 31) / 32 * 32; };

struct Z0Leaf { double v[9]; double wf; int rule; };
template <int POP>
struct Z0Warp {
  Z0Leaf leaf[Z0W_LEAVES];
  DTri stack[Z0Stack<POP>::N];
  double g[4][3], c[4], a[4], o[3];
  int start[Z0W_LEAVES + 1];
};

// The task's faces are subdivided by the whole warp: each step pops up to Z0W_POP sub-triangles
// from the top of a shared stack (lanes 0..15 measure one each, ConeIntegrator's rule: split
// while size > split * dest and depth < 7), pushes the children of the splitting ones (<= 64) and
// appends the others to the leaf buffer.  Depths on the stack never decrease towards the top and
// each push is one group of <= 64 of the next depth, so the stack holds <= 1 + 7 x 64 entries.
// The leaf SET equals the host's depth-first one (the split test does not depend on the order);
// the quadrature of the leaves is shared by all 32 lanes.
template <int POP, int MINB>
__global__ void __launch_bounds__(32 * Z0W_WARPS, MINB) k_z0_warp(
    const Z0Item* __restrict__ items, int64_t nitems, const double* __restrict__ xyz, const int32_t* __restrict__ tets,
    const int64_t* __restrict__ parent, const double* __restrict__ Ms_tet, Lat lat, const TriRules* __restrict__ rules,
    const int64_t* __restrict__ rowbase, int64_t r0, double* __restrict__ vals) {
  constexpr int Z0W_POP = POP;
  extern __shared__ __align__(16) unsigned char z0w_smem[];
  TriRules& R = *reinterpret_cast<TriRules*>(z0w_smem);
  Z0Warp<POP>* W = reinterpret_cast<Z0Warp<POP>*>(z0w_smem + ((sizeof(TriRules) + 15) / 16) * 16);
  for (int i = threadIdx.x; i < (int)(sizeof(TriRules) / sizeof(double)); i += blockDim.x)
    reinterpret_cast<double*>(&R)[i] = reinterpret_cast<const double*>(rules)[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  Z0Warp<POP>& w = W[wid];
  for (int64_t it_i = (int64_t)blockIdx.x * Z0W_WARPS + wid; it_i < nitems; it_i += (int64_t)gridDim.x * Z0W_WARPS) {
    const Z0Item it = items[it_i];
    int code = it.code;
    int sh[3];
    sh[2] = code % 17 - 8; code /= 17;
    sh[1] = code % 17 - 8; code /= 17;
    sh[0] = code - 8;
    const int32_t* tv = tets + 4 * (int64_t)it.tet;
    double P[4][3];
    for (int j = 0; j < 4; ++j)
      for (int x = 0; x < 3; ++x) P[j][x] = xyz[3 * (int64_t)tv[j] + x] + sh[x] * lat.L[x];
    const int64_t pn = parent[it.row];
    if (lane == 0) {
      double g[4][3];
      tet_grads(P, g);
      for (int i = 0; i < 4; ++i) {
        for (int x = 0; x < 3; ++x) w.g[i][x] = g[i][x];
        w.c[i] = 1.0 - zc_dot(g[i], P[i]);
      }
      for (int x = 0; x < 3; ++x) w.o[x] = xyz[3 * pn + x];
      for (int i = 0; i < 4; ++i)
        w.a[i] = (it.va >= 0) ? (i == it.va ? 1.0 : 0.0) : w.c[i] + zc_dot(w.g[i], w.o);
    }
    __syncwarp();
    // 23 face moments summed over the task's faces (the per-task coefficients a, g are common to
    // all of them): S0 = sum w/R, S1 = sum w Rv/R, T1 = sum w Rv/R^3, T2 = sum w Rv Rv/R^3 (6),
    // T3 = sum w Rv Rv Rv/R^3 (10), Rv = y - o, w = rule weight * area2 * h
    double Mo[23];
#pragma unroll
    for (int i = 0; i < 23; ++i) Mo[i] = 0.0;
    int nleaf = 0;
    // quadrature of the buffered leaves: their points flattened over the 32 lanes
    auto flush = [&]() {
      if (lane == 0) {
        int acc = 0;
        for (int l = 0; l < nleaf; ++l) { w.start[l] = acc; acc += R.cnt[w.leaf[l].rule]; }
        w.start[nleaf] = acc;
      }
      __syncwarp();
      const int npts = w.start[nleaf];
      int l = 0;
      for (int gq = lane; gq < npts; gq += 32) {
        while (gq >= w.start[l + 1]) ++l;
        const Z0Leaf& L = w.leaf[l];
        const int q = R.off[L.rule] + (gq - w.start[l]);
        double y[3], Rv[3];
        for (int x = 0; x < 3; ++x) {
          y[x] = R.l0[q] * L.v[x] + R.l1[q] * L.v[3 + x] + R.l2[q] * L.v[6 + x];
          Rv[x] = y[x] - w.o[x];
        }
        const double inv = rsqrt(zc_dot(Rv, Rv));
        const double wt = R.w[q] * L.wf;
        const double wi = wt * inv, w3 = wi * inv * inv;
        const double x = Rv[0], yy = Rv[1], z = Rv[2];
        Mo[0] += wi;
        Mo[1] += wi * x; Mo[2] += wi * yy; Mo[3] += wi * z;
        Mo[4] += w3 * x; Mo[5] += w3 * yy; Mo[6] += w3 * z;
        const double xx = w3 * x * x, xy = w3 * x * yy, xz = w3 * x * z, yv = w3 * yy * yy, yz = w3 * yy * z,
                     zz = w3 * z * z;
        Mo[7] += xx; Mo[8] += xy; Mo[9] += xz; Mo[10] += yv; Mo[11] += yz; Mo[12] += zz;
        Mo[13] += xx * x; Mo[14] += xx * yy; Mo[15] += xx * z; Mo[16] += xy * yy; Mo[17] += xy * z;
        Mo[18] += xz * z; Mo[19] += yv * yy; Mo[20] += yv * z; Mo[21] += yz * z; Mo[22] += zz * z;
      }
      __syncwarp();
      nleaf = 0;
    };
    for (int j = 0; j < 4; ++j) {
      if (it.va >= 0 && j != it.va) continue;                 // warp-uniform
      const double gn = sqrt(zc_dot(w.g[j], w.g[j]));
      const double h = w.a[j] / gn;                            // phi_j(o) = |g_j| h_j
      if (fabs(h) * gn < 1e-14) continue;
      const int f0 = (j + 1) % 4, f1 = (j + 2) % 4, f2 = (j + 3) % 4;
      double F0[3], E1[3], E2[3];
      for (int x = 0; x < 3; ++x) { F0[x] = P[f0][x]; E1[x] = P[f1][x] - P[f0][x]; E2[x] = P[f2][x] - P[f0][x]; }
      if (lane == 0) w.stack[0] = dtri_root();
      int top = 1;
      __syncwarp();
      while (top > 0) {
        const int np = top < Z0W_POP ? top : Z0W_POP;
        const int base = top - np;
        const bool act = lane < np;
        DTri T = dtri_root();
        double V[3][3], size = 0.0, dest = 1.0;
        bool split = false;
        if (act) {
          T = w.stack[base + lane];
          dtri_vertices(F0, E1, E2, T, V);
          dtri_measure(V, w.o, h, size, dest);
          split = size > R.split * dest && T.depth < 7;
        }
        const unsigned bs = __ballot_sync(0xffffffffu, split), bl = __ballot_sync(0xffffffffu, act && !split);
        __syncwarp();                                          // every lane has read its entry
        const int nl = __popc(bl);
        if (nleaf + nl > Z0W_LEAVES) flush();
        if (act && !split) {
          double e01[3], e02[3];
          for (int x = 0; x < 3; ++x) { e01[x] = V[1][x] - V[0][x]; e02[x] = V[2][x] - V[0][x]; }
          const double cr[3] = {e01[1] * e02[2] - e01[2] * e02[1], e01[2] * e02[0] - e01[0] * e02[2],
                                e01[0] * e02[1] - e01[1] * e02[0]};
          Z0Leaf& L = w.leaf[nleaf + __popc(bl & lt)];
          for (int k = 0; k < 3; ++k)
            for (int x = 0; x < 3; ++x) L.v[3 * k + x] = V[k][x];
          L.wf = sqrt(zc_dot(cr, cr)) * h;
          L.rule = tri_rule(R, size / dest);
        }
        if (split) dtri_children(T, &w.stack[base + 4 * __popc(bs & lt)]);
        nleaf += nl;
        top = base + 4 * __popc(bs);
        __syncwarp();
      }
    }
    if (nleaf > 0) flush();
    // butterfly: every lane gets the task's moments
#pragma unroll
    for (int i = 0; i < 23; ++i)
      for (int o = 16; o > 0; o >>= 1) Mo[i] += __shfl_xor_sync(0xffffffffu, Mo[i], o);
    // A_m = a_m S0 / 2 + g_m . S1 / 3;
    // B_km,x = -(a_k a_m T1_x + (a_k g_m + a_m g_k) . T2_(.x) / 2 + g_k^T T3_(..x) g_m / 3)
    // (the per-point formulas of ConeIntegrator::quad with phi(y) = a + g . (y - o), regrouped)
    const double Ms = Ms_tet[it.tet];
    double* v = vals + rowbase[it.slot];
    for (int t = lane; t < 48; t += 32) {
      const int k = t / 12, m = (t / 3) % 4, x = t % 3;
      if (!(it.flags & (1u << k))) continue;
      const double* gk = w.g[k];
      const double* gm = w.g[m];
      const double ak = w.a[k], am = w.a[m];
      const double Am = 0.5 * am * Mo[0] + (gm[0] * Mo[1] + gm[1] * Mo[2] + gm[2] * Mo[3]) / 3.0;
      // T2 column x, T3 slice x as 3x3 (symmetric index maps)
      double t2[3], t3[3][3];
      const int i2[3][3] = {{7, 8, 9}, {8, 10, 11}, {9, 11, 12}};
      const int i3[3][3][3] = {{{13, 14, 15}, {14, 16, 17}, {15, 17, 18}},
                               {{14, 16, 17}, {16, 19, 20}, {17, 20, 21}},
                               {{15, 17, 18}, {17, 20, 21}, {18, 21, 22}}};
      double bv = ak * am * (x == 0 ? Mo[4] : x == 1 ? Mo[5] : Mo[6]);
      for (int i = 0; i < 3; ++i) {
        double c2 = 0.0;
        for (int j = 0; j < 23; ++j)
          if (j == i2[i][x]) c2 = Mo[j];
        t2[i] = c2;
        for (int l = 0; l < 3; ++l) {
          double c3 = 0.0;
          for (int j = 0; j < 23; ++j)
            if (j == i3[i][l][x]) c3 = Mo[j];
          t3[i][l] = c3;
        }
      }
      for (int i = 0; i < 3; ++i) bv += 0.5 * (ak * gm[i] + am * gk[i]) * t2[i];
      double q3 = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int l = 0; l < 3; ++l) q3 += gk[i] * gm[l] * t3[i][l];
      bv = -(bv + q3 / 3.0);
      atomicAdd(v + 3 * it.pos[m] + x, Ms * (bv + gk[x] * Am));
    }
    __syncwarp();
  }
}

}  // namespace

// Chunked, pipelined driver: the mesh arrays are uploaded once (z0_device_begin); each chunk's
// tasks are uploaded and integrated asynchronously on a private stream and its values copied
// back into pinned memory, while the host enumerates the next chunk; a chunk's values are
// accumulated into rval when the NEXT chunk has been launched (or at z0_device_end).
struct Z0Pipe {
  int dev = -1;
  cudaStream_t st = nullptr;
  double* xyz = nullptr;
  int32_t* tets = nullptr;
  int64_t* parent = nullptr;
  double* ms = nullptr;
  TriRules* rules = nullptr;
  struct Chunk {
    bool busy = false;
    std::vector<int64_t> rows;     // user parent ids of the chunk's rows
    std::vector<int64_t> rowbase;
    Z0Item* items = nullptr;
    int64_t* base = nullptr;
    double* vals = nullptr;
    size_t items_cap = 0, base_cap = 0, vals_cap = 0;
    double* hvals = nullptr;       // pinned
    size_t hcap = 0;
    Z0Item* hitems = nullptr;      // pinned staging of the chunk's tasks
    size_t hicap = 0;
    cudaEvent_t done = nullptr;
  } ch[2];
  int cur = 0;
};

static Z0Pipe g_z0;

void z0_device_begin(const HostSetup& S, const TriRules& rules) {
  Z0Pipe& P = g_z0;
  P.dev = S.z0_device;
  CKZ(cudaSetDevice(P.dev));
  CKZ(cudaStreamCreateWithFlags(&P.st, cudaStreamNonBlocking));
  P.xyz = up(S.xyz.data(), S.xyz.size());
  P.tets = up(S.tets.data(), S.tets.size());
  P.parent = up(S.parent.data(), S.parent.size());
  P.ms = up(S.Ms_tet.data(), S.Ms_tet.size());
  P.rules = up(&rules, 1);
  for (auto& c : P.ch) CKZ(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
  P.cur = 0;
}

static void z0_finish_chunk(Z0Pipe::Chunk& c, std::vector<std::vector<double>>& rval) {
  if (!c.busy) return;
  CKZ(cudaEventSynchronize(c.done));
#pragma omp parallel for schedule(static)
  for (size_t j = 0; j < c.rows.size(); ++j) {
    const double* src = c.hvals + c.rowbase[j];
    std::vector<double>& dst = rval[c.rows[j]];
    for (size_t e = 0; e < dst.size(); ++e) dst[e] += src[e];
  }
  c.busy = false;            // the slot's device buffers are kept (cudaFree would synchronise the device)
}

// grow-only device buffer of a pipeline slot (freed at z0_device_end)
template <class T>
static T* slot_buf(T*& p, size_t& cap, size_t n) {
  n = std::max<size_t>(n, 1);
  if (n > cap) {
    if (p) CKZ(cudaFree(p));
    CKZ(cudaMalloc(&p, n * sizeof(T)));
    cap = n;
  }
  return p;
}

void z0_device_integrate(const HostSetup& S, std::vector<std::vector<Z0Item>>& titems,
                         const std::vector<std::vector<int32_t>>& rcol, std::vector<std::vector<double>>& rval,
                         const TriRules& rules, const int64_t* rows, int64_t nrows) {
  (void)rules;
  Z0Pipe& P = g_z0;
  CKZ(cudaSetDevice(P.dev));
  Z0Pipe::Chunk& c = P.ch[P.cur];
  z0_finish_chunk(c, rval);                       // the chunk two launches ago (normally done)
  // the threads' task lists are gathered in parallel into the slot's pinned staging buffer, so
  // the upload is a true async copy (a serial concatenation + pageable copy of ~1 GB per chunk
  // was ~1 s of host time per 250k rows at C4)
  std::vector<size_t> toff(titems.size() + 1, 0);
  for (size_t i = 0; i < titems.size(); ++i) toff[i + 1] = toff[i] + titems[i].size();
  const size_t tot = toff.back();
  if (tot > c.hicap) {
    if (c.hitems) CKZ(cudaFreeHost(c.hitems));
    c.hicap = tot + tot / 4;
    CKZ(cudaMallocHost(&c.hitems, c.hicap * sizeof(Z0Item)));
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (size_t i = 0; i < titems.size(); ++i) {
    if (!titems[i].empty()) std::memcpy(c.hitems + toff[i], titems[i].data(), titems[i].size() * sizeof(Z0Item));
    std::vector<Z0Item>().swap(titems[i]);
  }
  c.rows.assign(rows, rows + nrows);
  c.rowbase.assign(nrows + 1, 0);
  for (int64_t j = 0; j < nrows; ++j) c.rowbase[j + 1] = c.rowbase[j] + 3 * (int64_t)rcol[rows[j]].size();
  const int64_t nvals = c.rowbase[nrows];
  slot_buf(c.items, c.items_cap, tot);
  slot_buf(c.base, c.base_cap, c.rowbase.size());
  slot_buf(c.vals, c.vals_cap, (size_t)std::max<int64_t>(nvals, 1));
  // the private non-blocking stream orders the copies before the kernel without synchronising
  // the device (rowbase is pageable: staged, small)
  if (tot) CKZ(cudaMemcpyAsync(c.items, c.hitems, tot * sizeof(Z0Item), cudaMemcpyHostToDevice, P.st));
  CKZ(cudaMemcpyAsync(c.base, c.rowbase.data(), c.rowbase.size() * sizeof(int64_t), cudaMemcpyHostToDevice, P.st));
  CKZ(cudaMemsetAsync(c.vals, 0, std::max<int64_t>(nvals, 1) * sizeof(double), P.st));
  if ((size_t)nvals > c.hcap) {
    if (c.hvals) cudaFreeHost(c.hvals);
    c.hcap = (size_t)std::max<int64_t>(nvals, 1);
    CKZ(cudaMallocHost(&c.hvals, c.hcap * sizeof(double)));
  }
  Lat lat{{S.L[0], S.L[1], S.L[2]}};
  const int64_t n = (int64_t)tot;
  static const bool thread_per_task = std::getenv("PMFEM_Z0_THREAD") != nullptr;
  if (n && thread_per_task) {
    k_z0_items<<<(unsigned)((n + 127) / 128), 128, 0, P.st>>>(c.items, n, P.xyz, P.tets, P.parent, P.ms, lat, P.rules,
                                                               c.base, 0, c.vals);
    CKZ(cudaGetLastError());
  } else if (n) {
    static const bool pop16 = std::getenv("PMFEM_Z0_POP") && std::atoi(std::getenv("PMFEM_Z0_POP")) == 16;
    int nsm = 148;
    CKZ(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P.dev));
    const int64_t want = (n + Z0W_WARPS - 1) / Z0W_WARPS;
    const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)nsm * 32);
    const size_t rb = ((sizeof(TriRules) + 15) / 16) * 16;
    if (pop16) {
      const size_t smem = rb + Z0W_WARPS * sizeof(Z0Warp<16>);
      CKZ(cudaFuncSetAttribute(k_z0_warp<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_z0_warp<16, 1><<<blocks, 32 * Z0W_WARPS, smem, P.st>>>(c.items, n, P.xyz, P.tets, P.parent, P.ms, lat, P.rules,
                                                               c.base, 0, c.vals);
    } else {
      const size_t smem = rb + Z0W_WARPS * sizeof(Z0Warp<8>);
      CKZ(cudaFuncSetAttribute(k_z0_warp<8, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_z0_warp<8, 5><<<blocks, 32 * Z0W_WARPS, smem, P.st>>>(c.items, n, P.xyz, P.tets, P.parent, P.ms, lat, P.rules,
                                                              c.base, 0, c.vals);
    }
    CKZ(cudaGetLastError());
  }
  if (nvals) CKZ(cudaMemcpyAsync(c.hvals, c.vals, nvals * sizeof(double), cudaMemcpyDeviceToHost, P.st));
  CKZ(cudaEventRecord(c.done, P.st));
  c.busy = true;
  P.cur ^= 1;
}

void z0_device_end(std::vector<std::vector<double>>& rval) {
  Z0Pipe& P = g_z0;
  if (P.dev < 0) return;
  CKZ(cudaSetDevice(P.dev));
  for (int k = 0; k < 2; ++k) z0_finish_chunk(P.ch[(P.cur + k) & 1], rval);
  for (auto& c : P.ch) {
    if (c.hvals) cudaFreeHost(c.hvals);
    c.hvals = nullptr; c.hcap = 0;
    if (c.hitems) cudaFreeHost(c.hitems);
    c.hitems = nullptr; c.hicap = 0;
    cudaFree(c.items); cudaFree(c.base); cudaFree(c.vals);
    c.items = nullptr; c.base = nullptr; c.vals = nullptr;
    c.items_cap = c.base_cap = c.vals_cap = 0;
    cudaEventDestroy(c.done);
  }
  cudaFree(P.xyz); cudaFree(P.tets); cudaFree(P.parent); cudaFree(P.ms); cudaFree(P.rules);
  cudaStreamDestroy(P.st);
  P = Z0Pipe();
}

}  // namespace pmfem
