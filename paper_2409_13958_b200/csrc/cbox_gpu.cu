// Device-side construction of the precorrection matrix C_box (BAIM step 4, P:208-232;
// contract K8/K9, readings R8/R9) directly in internal order, fp64 arithmetic, fp32 storage.
//   near set : all (n, k, img) with |x_n - x_k - img L| <= r_ER on every axis (closed),
//              min image on periodic axes (unique because r_ER < L/2)
//   entry    : G0*(d) - sum_{a in st(n), b in st(k)} w_na w_kb G0*((a - b - img N) o Delta)
// The host computes the same thing in setup_aim.cpp (used by host-only contexts and as the
// reference of the GPU test); device contexts build C_box here in seconds instead of minutes.
// Pass 1 counts the near pairs of every row, the host scans (rows padded to a multiple of 4
// for K4's 16-byte loads), pass 2 writes columns and values.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>
#include "device.cuh"

namespace pmfem {

namespace {

#define CKC(x)                                                                                  \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) throw Error(PMFEM_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct CboxGeom {
  int per[3];
  int n[3];
  int p;
  double L[3], delta[3], rer;
  long long nb[3];       // boxes per axis (box edge >= r_ER)
  double blo[3], bs[3];  // box origin and edge per axis
};

__device__ __forceinline__ long long box_of(const CboxGeom& c, double x, int a) {
  long long b = (long long)floor((x - c.blo[a]) / c.bs[a]);
  return b < 0 ? 0 : (b >= c.nb[a] ? c.nb[a] - 1 : b);
}

__device__ __forceinline__ void lagr_d(double t, int p, double* w) {
  for (int j = 0; j <= p; ++j) {
    double v = 1.0;
    for (int i = 0; i <= p; ++i)
      if (i != j) v *= (t - i) / double(j - i);
    w[j] = v;
  }
}

// visit every near pair (k, img) of row n; distinct neighbour boxes (periodic axes with fewer
// than 3 boxes visit each box once)
template <class F>
__device__ void for_near(const CboxGeom& c, const double* __restrict__ xw, const long long* __restrict__ bptr,
                         const int* __restrict__ bnode, long long n, F&& f) {
  const double xn[3] = {xw[3 * n], xw[3 * n + 1], xw[3 * n + 2]};
  long long bn[3];
  int lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    bn[a] = box_of(c, xn[a], a);
    if (c.per[a] && c.nb[a] < 3) { lo[a] = 0; hi[a] = (int)c.nb[a] - 1; bn[a] = 0; }
    else { lo[a] = -1; hi[a] = 1; }
  }
  for (int dx = lo[0]; dx <= hi[0]; ++dx)
    for (int dy = lo[1]; dy <= hi[1]; ++dy)
      for (int dz = lo[2]; dz <= hi[2]; ++dz) {
        long long bb[3] = {bn[0] + dx, bn[1] + dy, bn[2] + dz};
        bool ok = true;
        for (int a = 0; a < 3; ++a) {
          if (c.per[a]) bb[a] = ((bb[a] % c.nb[a]) + c.nb[a]) % c.nb[a];
          else ok &= (bb[a] >= 0 && bb[a] < c.nb[a]);
        }
        if (!ok) continue;
        const long long b = (bb[0] * c.nb[1] + bb[1]) * c.nb[2] + bb[2];
        for (long long i = bptr[b]; i < bptr[b + 1]; ++i) {
          const int k = bnode[i];
          double d[3];
          int img[3] = {0, 0, 0};
          bool in = true;
          for (int a = 0; a < 3; ++a) {
            d[a] = xn[a] - xw[3 * (long long)k + a];
            if (c.per[a]) { img[a] = (int)rint(d[a] / c.L[a]); d[a] -= img[a] * c.L[a]; }
            in &= fabs(d[a]) <= c.rer;
          }
          if (in) f(k, d, img);
        }
      }
}

__global__ void k_cbox_count(CboxGeom c, long long Np, const double* __restrict__ xw, const long long* __restrict__ bptr,
                             const int* __restrict__ bnode, int* __restrict__ cnt) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  int k_cnt = 0;
  for_near(c, xw, bptr, bnode, n, [&](int, const double*, const int*) { ++k_cnt; });
  cnt[n] = k_cnt;
}

__global__ void k_cbox_fill(CboxGeom c, long long Np, const double* __restrict__ xw, const long long* __restrict__ bptr,
                            const int* __restrict__ bnode, const int* __restrict__ s_unw, const double* __restrict__ t_loc,
                            const long long* __restrict__ rowptr, int* __restrict__ col, float* __restrict__ val) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  const int p = c.p, p1 = p + 1, W = 2 * p + 1;
  double wn[3][4];
  for (int a = 0; a < 3; ++a) lagr_d(t_loc[3 * n + a], p, wn[a]);
  long long o = rowptr[n];
  for_near(c, xw, bptr, bnode, n, [&](int k, const double* d, const int* img) {
    const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double v = r > 0 ? 1.0 / r : 0.0;
    double wk[3][4], cw[3][7];
    int base[3];
    for (int a = 0; a < 3; ++a) {
      lagr_d(t_loc[3 * (long long)k + a], p, wk[a]);
      base[a] = s_unw[3 * n + a] - s_unw[3 * (long long)k + a] - img[a] * c.n[a] - p;
      for (int e = 0; e < W; ++e) cw[a][e] = 0.0;
      for (int i = 0; i < p1; ++i)
        for (int j = 0; j < p1; ++j) cw[a][i - j + p] += wn[a][i] * wk[a][j];
    }
    double gm = 0.0;
    for (int ex = 0; ex < W; ++ex) {
      const double dx = (base[0] + ex) * c.delta[0];
      for (int ey = 0; ey < W; ++ey) {
        const double dy = (base[1] + ey) * c.delta[1];
        const double wxy = cw[0][ex] * cw[1][ey];
        for (int ez = 0; ez < W; ++ez) {
          const double dz = (base[2] + ez) * c.delta[2];
          const double rr = dx * dx + dy * dy + dz * dz;
          if (rr > 0) gm += wxy * cw[2][ez] / sqrt(rr);
        }
      }
    }
    col[o] = k;
    val[o] = (float)(v - gm);
    ++o;
  });
  for (; o < rowptr[n + 1]; ++o) { col[o] = (int)n; val[o] = 0.f; }   // padding to 4
}

template <class T>
T* dalloc_c(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) throw Error(PMFEM_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return p;
}
template <class T>
T* dup_c(const std::vector<T>& v) {
  T* p = dalloc_c<T>(v.size());
  if (!v.empty()) CKC(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

}  // namespace

// Builds D.c_ptr / D.c_col / D.c_val (internal order) on the device.  Returns the number of
// (unpadded) entries.
int64_t device_build_cbox(DeviceState& D, const HostSetup& S) {
  CKC(cudaSetDevice(D.device));
  const int64_t Np = S.Np;
  const int p = S.order;
  const double rer = S.rer_scale * std::max(S.delta[0], std::max(S.delta[1], S.delta[2]));
  CboxGeom c{};
  c.p = p;
  c.rer = rer;
  std::vector<double> xw(3 * Np), tl(3 * Np);
  std::vector<int> su(3 * Np);
  for (int64_t i = 0; i < Np; ++i) {
    const int64_t r = S.perm[i];
    for (int a = 0; a < 3; ++a) {
      xw[3 * i + a] = S.xw[3 * r + a];
      tl[3 * i + a] = S.st_t[3 * r + a];
      su[3 * i + a] = S.st_s[3 * r + a];
    }
  }
  for (int a = 0; a < 3; ++a) {
    c.per[a] = S.periodic[a];
    c.n[a] = S.grid_n[a];
    c.L[a] = S.L[a];
    c.delta[a] = S.delta[a];
    double lo = 1e300, hi = -1e300;
    for (int64_t i = 0; i < Np; ++i) { lo = std::min(lo, xw[3 * i + a]); hi = std::max(hi, xw[3 * i + a]); }
    if (S.periodic[a]) { c.blo[a] = 0; c.nb[a] = std::max<long long>(1, (long long)std::floor(S.L[a] / rer)); c.bs[a] = S.L[a] / c.nb[a]; }
    else { c.blo[a] = lo; c.nb[a] = (long long)std::floor((hi - lo) / rer) + 1; c.bs[a] = rer; }
  }
  // box lists (same box rule as the host's setup_aim)
  const long long nbox = c.nb[0] * c.nb[1] * c.nb[2];
  std::vector<long long> key(Np), bptr(nbox + 1, 0);
  for (int64_t i = 0; i < Np; ++i) {
    long long bb[3];
    for (int a = 0; a < 3; ++a) {
      long long b = (long long)std::floor((xw[3 * i + a] - c.blo[a]) / c.bs[a]);
      bb[a] = std::min<long long>(std::max<long long>(b, 0), c.nb[a] - 1);
    }
    key[i] = (bb[0] * c.nb[1] + bb[1]) * c.nb[2] + bb[2];
    bptr[key[i] + 1]++;
  }
  for (long long b = 0; b < nbox; ++b) bptr[b + 1] += bptr[b];
  std::vector<int> bnode(Np);
  {
    std::vector<long long> fill(bptr.begin(), bptr.end() - 1);
    for (int64_t i = 0; i < Np; ++i) bnode[fill[key[i]]++] = (int)i;
  }
  double* d_xw = dup_c(xw);
  double* d_tl = dup_c(tl);
  int* d_su = dup_c(su);
  long long* d_bptr = dup_c(bptr);
  int* d_bnode = dup_c(bnode);
  int* d_cnt = dalloc_c<int>(Np);
  const unsigned blocks = (unsigned)((Np + 127) / 128);
  k_cbox_count<<<blocks, 128>>>(c, Np, d_xw, d_bptr, d_bnode, d_cnt);
  CKC(cudaGetLastError());
  std::vector<int> cnt(Np);
  CKC(cudaMemcpy(cnt.data(), d_cnt, sizeof(int) * Np, cudaMemcpyDeviceToHost));
  std::vector<long long> ptr(Np + 1, 0);
  int64_t nnz = 0;
  for (int64_t i = 0; i < Np; ++i) { ptr[i + 1] = ptr[i] + (cnt[i] + 3) / 4 * 4; nnz += cnt[i]; }
  long long* d_ptr = dup_c(ptr);
  int* d_col = dalloc_c<int>(ptr[Np]);
  float* d_val = dalloc_c<float>(ptr[Np]);
  k_cbox_fill<<<blocks, 128>>>(c, Np, d_xw, d_bptr, d_bnode, d_su, d_tl, d_ptr, d_col, d_val);
  CKC(cudaGetLastError());
  CKC(cudaDeviceSynchronize());
  cudaFree(d_xw); cudaFree(d_tl); cudaFree(d_su); cudaFree(d_bptr); cudaFree(d_bnode); cudaFree(d_cnt);
  D.c_ptr = reinterpret_cast<int64_t*>(d_ptr);
  D.c_col = d_col;
  D.c_val = d_val;
  D.cbox_nnz = nnz;
  return nnz;
}

}  // namespace pmfem
