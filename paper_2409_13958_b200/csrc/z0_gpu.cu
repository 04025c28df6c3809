// GPU integration of the Z0 element integrals: one thread per (row, element
// image) task enumerated by setup_z0.cpp; the same ConeIntegrator (z0_cone.cuh) as the host
// path, in fp64; contributions are accumulated with fp64 atomics into the row's value slots.
#include <cstring>
#include <string>
#include <vector>
#include <cuda_runtime.h>
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
  double* v = vals + rowbase[it.row - r0];
  for (int k = 0; k < 4; ++k) {
    if (!(it.flags & (1u << k))) continue;
    for (int m = 0; m < 4; ++m)
      for (int x = 0; x < 3; ++x) atomicAdd(v + 3 * it.pos[m] + x, Ms * (I.B[k][m][x] + I.g[k][x] * I.A[m]));
  }
}

}  // namespace

void z0_device_integrate(const HostSetup& S, std::vector<std::vector<Z0Item>>& titems,
                         const std::vector<std::vector<int32_t>>& rcol, std::vector<std::vector<double>>& rval,
                         const TriRules& rules, int64_t r0, int64_t r1) {
  CKZ(cudaSetDevice(S.z0_device));
  std::vector<Z0Item> items;
  size_t tot = 0;
  for (auto& v : titems) tot += v.size();
  items.reserve(tot);
  for (auto& v : titems) { items.insert(items.end(), v.begin(), v.end()); std::vector<Z0Item>().swap(v); }
  std::vector<int64_t> rowbase(r1 - r0 + 1, 0);
  for (int64_t n = r0; n < r1; ++n) rowbase[n - r0 + 1] = rowbase[n - r0] + 3 * (int64_t)rcol[n].size();
  const int64_t nvals = rowbase[r1 - r0];
  Z0Item* d_items = up(items.data(), items.size());
  double* d_xyz = up(S.xyz.data(), S.xyz.size());
  int32_t* d_tets = up(S.tets.data(), S.tets.size());
  int64_t* d_parent = up(S.parent.data(), S.parent.size());
  double* d_ms = up(S.Ms_tet.data(), S.Ms_tet.size());
  TriRules* d_rules = up(&rules, 1);
  int64_t* d_base = up(rowbase.data(), rowbase.size());
  double* d_vals = nullptr;
  CKZ(cudaMalloc(&d_vals, std::max<int64_t>(nvals, 1) * sizeof(double)));
  CKZ(cudaMemset(d_vals, 0, std::max<int64_t>(nvals, 1) * sizeof(double)));
  Lat lat{{S.L[0], S.L[1], S.L[2]}};
  const int64_t n = (int64_t)items.size();
  if (n) {
    k_z0_items<<<(unsigned)((n + 127) / 128), 128>>>(d_items, n, d_xyz, d_tets, d_parent, d_ms, lat, d_rules, d_base,
                                                     r0, d_vals);
    CKZ(cudaGetLastError());
    CKZ(cudaDeviceSynchronize());
  }
  std::vector<double> vals(nvals);
  if (nvals) CKZ(cudaMemcpy(vals.data(), d_vals, nvals * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t r = r0; r < r1; ++r) {
    const double* src = &vals[rowbase[r - r0]];
    std::vector<double>& dst = rval[r];
    for (size_t j = 0; j < dst.size(); ++j) dst[j] += src[j];
  }
  cudaFree(d_items); cudaFree(d_xyz); cudaFree(d_tets); cudaFree(d_parent); cudaFree(d_ms);
  cudaFree(d_rules); cudaFree(d_base); cudaFree(d_vals);
}

}  // namespace pmfem
