// Device path of libpmfem (sm_100a): upload, fp64 PGF build, and the fp32 H_eff hot path.
//
//   K1  local_in      q = D m, u_loc = Z0 m, H_ex = L m
//   K2  anterpolate   Q = P q                                     (P:202 BAIM step 1)
//   K3  FFT conv      U = F^-1(G_hat . F Q)                       (P:204, P:214 step 2)
//   K4  interp_corr   u = P^T U + C_box q + u_loc                 (P:206-218 steps 3-4)
//   K5  grad_sum      H = H_ex - G u
//
// Every sparse operator is stored off-diagonal with its row sum ("difference form"):
//   sum_m X_nm v_m = sum_{m != n} X_nm (v_m - v_n) + (sum_m X_nm) v_n,
// so uniform m gives exactly zero charge and exchange field in fp32 (L, G have zero row sums).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include "device.cuh"
#include "fft.cuh"
#include "pgf.cuh"

namespace pmfem {

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) throw Error(PMFEM_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

template <class T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) throw Error(PMFEM_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return p;
}
template <class T>
T* dupload(const std::vector<T>& v) {
  T* p = dalloc<T>(v.size());
  if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}
int ilog2(int v) { int l = 0; while ((1 << l) < v) ++l; return l; }

// ------------------------------------------------------------------ K1 local_in
// One warp per row.  Reads m (12 B/node, gathered), the ring-1 row (col + 16 B), the Z0 row
// (col + 16 B); writes q, u_loc (4 B each) and H_ex (12 B, optional).
__global__ void __launch_bounds__(256) k1_local_in(
    int64_t Np, const float* __restrict__ m, const int64_t* __restrict__ r1_ptr, const int32_t* __restrict__ r1_col,
    const float4* __restrict__ r1_LD, const float4* __restrict__ rowsumD, const int64_t* __restrict__ z_ptr,
    const int32_t* __restrict__ z_col, const float4* __restrict__ z_val, const float4* __restrict__ rowsumZ,
    float* __restrict__ q, float* __restrict__ uloc, float* __restrict__ H, int write_hex) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= Np) return;
  const float mx = m[3 * n], my = m[3 * n + 1], mz = m[3 * n + 2];
  float hx = 0, hy = 0, hz = 0, qq = 0, ul = 0;
  for (int64_t e = r1_ptr[n] + lane; e < r1_ptr[n + 1]; e += 32) {
    const int32_t c = r1_col[e];
    const float4 w = r1_LD[e];
    const float dx = m[3 * c] - mx, dy = m[3 * c + 1] - my, dz = m[3 * c + 2] - mz;
    hx += w.x * dx; hy += w.x * dy; hz += w.x * dz;
    qq += w.y * dx + w.z * dy + w.w * dz;
  }
  for (int64_t e = z_ptr[n] + lane; e < z_ptr[n + 1]; e += 32) {
    const int32_t c = z_col[e];
    const float4 w = z_val[e];
    ul += w.x * (m[3 * c] - mx) + w.y * (m[3 * c + 1] - my) + w.z * (m[3 * c + 2] - mz);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hx += __shfl_xor_sync(0xffffffffu, hx, o);
    hy += __shfl_xor_sync(0xffffffffu, hy, o);
    hz += __shfl_xor_sync(0xffffffffu, hz, o);
    qq += __shfl_xor_sync(0xffffffffu, qq, o);
    ul += __shfl_xor_sync(0xffffffffu, ul, o);
  }
  if (lane == 0) {
    const float4 rd = rowsumD[n], rz = rowsumZ[n];
    q[n] = qq + rd.x * mx + rd.y * my + rd.z * mz;
    uloc[n] = ul + rz.x * mx + rz.y * my + rz.z * mz;
    if (write_hex) { H[3 * n] = hx; H[3 * n + 1] = hy; H[3 * n + 2] = hz; }
  }
}

// exchange only: H = L m
__global__ void __launch_bounds__(256) k_exchange(int64_t Np, const float* __restrict__ m,
                                                  const int64_t* __restrict__ r1_ptr, const int32_t* __restrict__ r1_col,
                                                  const float4* __restrict__ r1_LD, float* __restrict__ H) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= Np) return;
  const float mx = m[3 * n], my = m[3 * n + 1], mz = m[3 * n + 2];
  float hx = 0, hy = 0, hz = 0;
  for (int64_t e = r1_ptr[n] + lane; e < r1_ptr[n + 1]; e += 32) {
    const int32_t c = r1_col[e];
    const float L = r1_LD[e].x;
    hx += L * (m[3 * c] - mx); hy += L * (m[3 * c + 1] - my); hz += L * (m[3 * c + 2] - mz);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hx += __shfl_xor_sync(0xffffffffu, hx, o);
    hy += __shfl_xor_sync(0xffffffffu, hy, o);
    hz += __shfl_xor_sync(0xffffffffu, hz, o);
  }
  if (lane == 0) { H[3 * n] = hx; H[3 * n + 1] = hy; H[3 * n + 2] = hz; }
}

// Lagrange weights on nodes 0..P at local coordinate t
template <int P>
__device__ __forceinline__ void lagr(float t, float* w) {
#pragma unroll
  for (int j = 0; j <= P; ++j) {
    float v = 1.f;
#pragma unroll
    for (int i = 0; i <= P; ++i)
      if (i != j) v *= (t - (float)i) / (float)(j - i);
    w[j] = v;
  }
}

struct GridDims { int n0, n1, n2; int per0, per1, per2; };

__device__ __forceinline__ int wrapi(int i, int n, int per) { return per ? (i >= n ? i - n : i) : i; }

// ------------------------------------------------------------------ K2 anterpolation
template <int P>
__global__ void __launch_bounds__(256) k2_anterp(int64_t Np, const float* __restrict__ q, const int4* __restrict__ st_s,
                                                 const float4* __restrict__ st_t, GridDims g, float* __restrict__ Q) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  const int4 s = st_s[n];
  const float4 t = st_t[n];
  const float qn = q[n];
  float wx[P + 1], wy[P + 1], wz[P + 1];
  lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    const int iz = wrapi(s.z + k, g.n2, g.per2);
#pragma unroll
    for (int j = 0; j <= P; ++j) {
      const int iy = wrapi(s.y + j, g.n1, g.per1);
      const float wzy = qn * wz[k] * wy[j];
      float* row = Q + ((int64_t)iz * g.n1 + iy) * g.n0;
#pragma unroll
      for (int i = 0; i <= P; ++i) atomicAdd(row + wrapi(s.x + i, g.n0, g.per0), wzy * wx[i]);
    }
  }
}

// ------------------------------------------------------------------ K4 interpolation + precorrection
template <int P>
__global__ void __launch_bounds__(256) k4_interp_corr(int64_t Np, const float* __restrict__ U, const int4* __restrict__ st_s,
                                                      const float4* __restrict__ st_t, GridDims g,
                                                      const int64_t* __restrict__ c_ptr, const int32_t* __restrict__ c_col,
                                                      const float* __restrict__ c_val, const float* __restrict__ q,
                                                      const float* __restrict__ uloc, float* __restrict__ u) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= Np) return;
  float acc = 0.f;
  for (int64_t e = c_ptr[n] + lane; e < c_ptr[n + 1]; e += 32) acc += c_val[e] * q[c_col[e]];
  constexpr int NS = (P + 1) * (P + 1) * (P + 1);
  const int4 s = st_s[n];
  const float4 t = st_t[n];
  float wx[P + 1], wy[P + 1], wz[P + 1];
  lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
  for (int k = lane; k < NS; k += 32) {
    const int i = k % (P + 1), j = (k / (P + 1)) % (P + 1), l = k / ((P + 1) * (P + 1));
    const int ix = wrapi(s.x + i, g.n0, g.per0), iy = wrapi(s.y + j, g.n1, g.per1), iz = wrapi(s.z + l, g.n2, g.per2);
    float wi = 0, wj = 0, wl = 0;
#pragma unroll
    for (int a = 0; a <= P; ++a) { if (a == i) wi = wx[a]; if (a == j) wj = wy[a]; if (a == l) wl = wz[a]; }
    acc += wi * wj * wl * U[((int64_t)iz * g.n1 + iy) * g.n0 + ix];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) u[n] = acc + uloc[n];
}

// ------------------------------------------------------------------ K5 gradient + sum
__global__ void __launch_bounds__(256) k5_grad_sum(int64_t Np, const float* __restrict__ u, const int64_t* __restrict__ r1_ptr,
                                                   const int32_t* __restrict__ r1_col, const float4* __restrict__ r1_G,
                                                   float* __restrict__ H, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= Np) return;
  const float un = u[n];
  float gx = 0, gy = 0, gz = 0;
  for (int64_t e = r1_ptr[n] + lane; e < r1_ptr[n + 1]; e += 32) {
    const float4 w = r1_G[e];
    const float du = u[r1_col[e]] - un;
    gx += w.x * du; gy += w.y * du; gz += w.z * du;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gx += __shfl_xor_sync(0xffffffffu, gx, o);
    gy += __shfl_xor_sync(0xffffffffu, gy, o);
    gz += __shfl_xor_sync(0xffffffffu, gz, o);
  }
  if (lane == 0) {
    if (accumulate) { H[3 * n] -= gx; H[3 * n + 1] -= gy; H[3 * n + 2] -= gz; }
    else { H[3 * n] = -gx; H[3 * n + 1] = -gy; H[3 * n + 2] = -gz; }
  }
}

// ------------------------------------------------------------------ PGF table (fp64)
__global__ void k_pgf_table(PgfDev pd, int P0, int P1, int P2, int n0, int n1, int n2, int per0, int per1, int per2,
                            double d0, double d1, double d2, double* __restrict__ K) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)P0 * P1 * P2;
  if (idx >= tot) return;
  const int j0 = (int)(idx % P0), j1 = (int)((idx / P0) % P1), j2 = (int)(idx / ((int64_t)P0 * P1));
  // K6: periodic j -> j Delta ; non-periodic j < n -> j Delta, j > n -> (j - 2n) Delta, j = n -> 0
  if ((!per0 && j0 == n0) || (!per1 && j1 == n1) || (!per2 && j2 == n2)) { K[idx] = 0.0; return; }
  double r[3];
  r[0] = (per0 ? j0 : (j0 < n0 ? j0 : j0 - P0)) * d0;
  r[1] = (per1 ? j1 : (j1 < n1 ? j1 : j1 - P1)) * d1;
  r[2] = (per2 ? j2 : (j2 < n2 ? j2 : j2 - P2)) * d2;
  const bool self = (j0 == 0 && j1 == 0 && j2 == 0);
  K[idx] = pgf_eval(pd, r, self);
}

__global__ void k_spec_finish(const double2* __restrict__ C, float* __restrict__ spec, int64_t tot, double scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tot) return;
  spec[i] = (i == 0) ? 0.f : (float)(C[i].x * scale);   // K7: G_hat at the zero frequency := 0
}

template <class T>
void twiddles(int P, std::vector<typename Cx<T>::t>& tw) {
  tw.resize(std::max(1, P / 2));
  for (int k = 0; k < P / 2; ++k) {
    double a = -2.0 * M_PI * k / P;
    tw[k].x = (T)std::cos(a);
    tw[k].y = (T)std::sin(a);
  }
}

// 3D transform driver shared by the fp32 hot path and the fp64 spectrum build
template <class T>
struct FftDims {
  int n[3], P[3], H0;
};

template <class T>
size_t x_smem_lines(int P0) {
  int M = P0 / 2;
  int nl = std::max(1, 4096 / std::max(M, 1));
  return (size_t)nl;
}

constexpr int TILE = 16;

template <class T>
void launch_strided(typename Cx<T>::t* data, int P, long long es, int ncol, int nplanes, long long plane_stride,
                    int nin, int nout, int mode, const T* spec, long long spec_es, long long spec_ps,
                    const typename Cx<T>::t* tw, cudaStream_t st) {
  using C = typename Cx<T>::t;
  size_t smem = (size_t)P * TILE * sizeof(C);
  auto kern = fft_strided<T, TILE>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((ncol + TILE - 1) / TILE, nplanes);
  kern<<<grid, 256, smem, st>>>(data, P, ilog2(P), es, ncol, plane_stride, nin, nout, mode, spec, spec_es, spec_ps, tw);
  CK(cudaGetLastError());
}

template <class T>
void launch_x(bool fwd, const T* rin, typename Cx<T>::t* cio, T* rout, int nrows, int n0, int P0, int n1, int P1,
              const typename Cx<T>::t* tw, cudaStream_t st) {
  using C = typename Cx<T>::t;
  int M = P0 / 2;
  int nl = (int)x_smem_lines<T>(P0);
  size_t smem = (size_t)nl * M * sizeof(C);
  RowMap rm{n1, P1};
  int blocks = (nrows + nl - 1) / nl;
  if (fwd) {
    auto kern = fft_x_forward<T>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, 256, smem, st>>>(rin, cio, nrows, n0, P0, ilog2(M), rm, tw, nl);
  } else {
    auto kern = fft_x_inverse<T>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, 256, smem, st>>>(cio, rout, nrows, n0, P0, ilog2(M), rm, tw, nl);
  }
  CK(cudaGetLastError());
}

}  // namespace

void device_upload(DeviceState& D, const HostSetup& S) {
  CK(cudaSetDevice(D.device));
  const int64_t Np = S.Np;
  D.Np = Np;
  D.order = S.order;
  for (int a = 0; a < 3; ++a) { D.periodic[a] = S.periodic[a]; D.n[a] = S.grid_n[a]; D.P[a] = S.fft_n[a]; }
  D.H0 = D.P[0] / 2 + 1;
  // permute rows and columns to internal order
  auto perm_csr = [&](const Csr& A, std::vector<int64_t>& ptr, std::vector<int32_t>& col, std::vector<int64_t>& src) {
    ptr.assign(Np + 1, 0);
    for (int64_t i = 0; i < Np; ++i) {
      int64_t r = S.perm[i];
      ptr[i + 1] = ptr[i] + (A.rowptr[r + 1] - A.rowptr[r]);
    }
    col.resize(ptr[Np]);
    src.resize(ptr[Np]);
    for (int64_t i = 0; i < Np; ++i) {
      int64_t r = S.perm[i];
      int64_t o = ptr[i];
      // sort the row by internal column for locality
      std::vector<std::pair<int32_t, int64_t>> tmp;
      for (int64_t e = A.rowptr[r]; e < A.rowptr[r + 1]; ++e) tmp.push_back({(int32_t)S.iperm[A.col[e]], e});
      std::sort(tmp.begin(), tmp.end());
      for (auto& pr : tmp) { col[o] = pr.first; src[o] = pr.second; ++o; }
    }
  };
  {
    std::vector<int64_t> ptr, src;
    std::vector<int32_t> col;
    perm_csr(S.ring1, ptr, col, src);
    std::vector<float4> LD(col.size()), G(col.size());
    for (size_t e = 0; e < col.size(); ++e) {
      const double* v = &S.ring1.val[7 * src[e]];
      LD[e] = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
      G[e] = make_float4((float)v[4], (float)v[5], (float)v[6], 0.f);
    }
    D.r1_ptr = dupload(ptr); D.r1_col = dupload(col); D.r1_LD = dupload(LD); D.r1_G = dupload(G);
  }
  {
    std::vector<int64_t> ptr, src;
    std::vector<int32_t> col;
    perm_csr(S.z0, ptr, col, src);
    std::vector<float4> Z(col.size());
    for (size_t e = 0; e < col.size(); ++e) {
      const double* v = &S.z0.val[3 * src[e]];
      Z[e] = make_float4((float)v[0], (float)v[1], (float)v[2], 0.f);
    }
    D.z_ptr = dupload(ptr); D.z_col = dupload(col); D.z_val = dupload(Z);
  }
  {
    std::vector<int64_t> ptr, src;
    std::vector<int32_t> col;
    perm_csr(S.cbox, ptr, col, src);
    std::vector<float> V(col.size());
    for (size_t e = 0; e < col.size(); ++e) V[e] = (float)S.cbox.val[src[e]];
    D.c_ptr = dupload(ptr); D.c_col = dupload(col); D.c_val = dupload(V);
  }
  std::vector<float4> rD(Np), rZ(Np), stt(Np);
  std::vector<int4> sts(Np);
  for (int64_t i = 0; i < Np; ++i) {
    int64_t r = S.perm[i];
    rD[i] = make_float4((float)S.rowsumD[3 * r], (float)S.rowsumD[3 * r + 1], (float)S.rowsumD[3 * r + 2], 0.f);
    rZ[i] = make_float4((float)S.rowsumZ[3 * r], (float)S.rowsumZ[3 * r + 1], (float)S.rowsumZ[3 * r + 2], 0.f);
    int s[3];
    for (int a = 0; a < 3; ++a) {
      int v = S.st_s[3 * r + a];
      if (S.periodic[a]) v = ((v % S.grid_n[a]) + S.grid_n[a]) % S.grid_n[a];
      s[a] = v;
    }
    sts[i] = make_int4(s[0], s[1], s[2], 0);
    stt[i] = make_float4((float)S.st_t[3 * r], (float)S.st_t[3 * r + 1], (float)S.st_t[3 * r + 2], 0.f);
  }
  D.rowsumD = dupload(rD); D.rowsumZ = dupload(rZ); D.st_s = dupload(sts); D.st_t = dupload(stt);
  for (int a = 0; a < 3; ++a) {
    std::vector<float2> t32; std::vector<double2> t64;
    twiddles<float>(D.P[a], t32); twiddles<double>(D.P[a], t64);
    D.tw32[a] = dupload(t32); D.tw64[a] = dupload(t64);
  }
  D.q = dalloc<float>(Np); D.uloc = dalloc<float>(Np); D.u = dalloc<float>(Np);
  D.Q = dalloc<float>((size_t)D.n[0] * D.n[1] * D.n[2]);
  D.C = dalloc<float2>((size_t)D.H0 * D.P[1] * D.P[2]);
  D.spec = dalloc<float>((size_t)D.H0 * D.P[1] * D.P[2]);
  for (int i = 0; i < 8; ++i) CK(cudaEventCreate(&D.ev[i]));
  // algorithmic bytes per launch (DESIGN.md byte model; fp32 values, int32 columns, int64 row ptrs)
  const double nnz1 = (double)S.ring1.nnz(), nnzz = (double)S.z0.nnz(), nnzc = (double)S.cbox.nnz();
  const double G = (double)D.n[0] * D.n[1] * D.n[2];
  const int ns = (S.order + 1) * (S.order + 1) * (S.order + 1);
  D.kernel_bytes[0] = Np * (12.0 + 16 + 16 + 8 + 8 + 4 + 4 + 12) + nnz1 * (4 + 16) + nnzz * (4 + 16);
  D.kernel_bytes[1] = Np * (4.0 + 16 + 16) + G * 4.0 * 2;                 // read q + stencil, grid RMW
  {
    double Hc = (double)D.H0;
    double bx = G * 4 + (double)D.n[1] * D.n[2] * Hc * 8;                   // X fwd: read real, write cplx
    double by = 2.0 * (double)D.n[2] * Hc * D.P[1] * 8;                     // Y fwd read+write (pruned in)
    double bz = 2.0 * Hc * D.P[1] * D.P[2] * 8 + Hc * D.P[1] * D.P[2] * 4;  // Z fused + spectrum
    double by2 = 2.0 * (double)D.n[2] * Hc * D.P[1] * 8;
    double bx2 = (double)D.n[1] * D.n[2] * Hc * 8 + G * 4;
    (void)by2;
    D.kernel_bytes[2] = bx + by + bz + by + bx2;
  }
  D.kernel_bytes[3] = Np * (16.0 + 16 + 8 + 4 + 4) + nnzc * (4 + 4 + 4) + Np * ns * 4.0;
  D.kernel_bytes[4] = Np * (4.0 + 8 + 12 + 12) + nnz1 * (4 + 16 + 4);
}

void device_build_pgf(DeviceState& D, const HostSetup& S, const PgfParams& Pp) {
  CK(cudaSetDevice(D.device));
  PgfDev pd;
  std::memset(&pd, 0, sizeof(pd));
  pd.dim = Pp.dim;
  for (int i = 0; i < 3; ++i) { pd.ax[i] = Pp.ax[i]; pd.L[i] = Pp.L[i]; pd.nreal[i] = Pp.nreal[i]; pd.mrec[i] = Pp.mrec[i]; }
  pd.alpha = Pp.alpha;
  gauss_legendre01(64, pd.gl_x, pd.gl_w);
  const int P0 = D.P[0], P1 = D.P[1], P2 = D.P[2];
  const int64_t tot = (int64_t)P0 * P1 * P2;
  double* K = dalloc<double>(tot);
  k_pgf_table<<<(unsigned)((tot + 127) / 128), 128>>>(pd, P0, P1, P2, D.n[0], D.n[1], D.n[2], D.periodic[0],
                                                      D.periodic[1], D.periodic[2], S.delta[0], S.delta[1], S.delta[2], K);
  CK(cudaGetLastError());
  // fp64 forward transform of the full padded table (no pruning)
  const int H0 = D.H0;
  double2* C = dalloc<double2>((size_t)H0 * P1 * P2);
  launch_x<double>(true, K, C, nullptr, P1 * P2, P0, P0, P1, P1, D.tw64[0], 0);
  launch_strided<double>(C, P1, H0, H0, P2, (long long)P1 * H0, P1, P1, 0, nullptr, 0, 0, D.tw64[1], 0);
  launch_strided<double>(C, P2, (long long)P1 * H0, H0, P1, H0, P2, P2, 0, nullptr, 0, 0, D.tw64[2], 0);
  const int64_t nspec = (int64_t)H0 * P1 * P2;
  k_spec_finish<<<(unsigned)((nspec + 255) / 256), 256>>>(C, D.spec, nspec, 1.0 / (double)tot);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaFree(K);
  cudaFree(C);
  D.pgf_ready = true;
}

void device_free(DeviceState& D) {
  if (D.device < 0) return;
  cudaSetDevice(D.device);
  void* ptrs[] = {D.r1_ptr, D.r1_col, D.r1_LD, D.r1_G, D.rowsumD, D.z_ptr, D.z_col, D.z_val, D.rowsumZ,
                  D.c_ptr, D.c_col, D.c_val, D.st_s, D.st_t, D.spec, D.q, D.uloc, D.u, D.Q, D.C,
                  D.m_stage, D.H_stage, D.tw32[0], D.tw32[1], D.tw32[2], D.tw64[0], D.tw64[1], D.tw64[2]};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int i = 0; i < 8; ++i)
    if (D.ev[i]) cudaEventDestroy(D.ev[i]);
}

void device_eval(DeviceState& D, const float* m, float* H, cudaStream_t st, EvalMode mode) {
  const int64_t Np = D.Np;
  const int WPB = 8;                       // warps per block (256 threads)
  const unsigned rows_blocks = (unsigned)((Np + WPB - 1) / WPB);
  const unsigned node_blocks = (unsigned)((Np + 255) / 256);
  if (mode == EVAL_EXCHANGE) {
    k_exchange<<<rows_blocks, 256, 0, st>>>(Np, m, D.r1_ptr, D.r1_col, D.r1_LD, H);
    CK(cudaGetLastError());
    return;
  }
  if (!D.pgf_ready) throw Error(PMFEM_E_STATE, "pmfem_build_pgf has not been called");
  auto mark = [&](int i) { if (D.timing) CK(cudaEventRecord(D.ev[i], st)); };
  GridDims g{D.n[0], D.n[1], D.n[2], D.periodic[0], D.periodic[1], D.periodic[2]};
  mark(0);
  k1_local_in<<<rows_blocks, 256, 0, st>>>(Np, m, D.r1_ptr, D.r1_col, D.r1_LD, D.rowsumD, D.z_ptr, D.z_col, D.z_val,
                                           D.rowsumZ, D.q, D.uloc, H, mode == EVAL_HEFF ? 1 : 0);
  CK(cudaGetLastError());
  mark(1);
  CK(cudaMemsetAsync(D.Q, 0, sizeof(float) * (size_t)D.n[0] * D.n[1] * D.n[2], st));
  switch (D.order) {
    case 1: k2_anterp<1><<<node_blocks, 256, 0, st>>>(Np, D.q, D.st_s, D.st_t, g, D.Q); break;
    case 2: k2_anterp<2><<<node_blocks, 256, 0, st>>>(Np, D.q, D.st_s, D.st_t, g, D.Q); break;
    default: k2_anterp<3><<<node_blocks, 256, 0, st>>>(Np, D.q, D.st_s, D.st_t, g, D.Q); break;
  }
  CK(cudaGetLastError());
  mark(2);
  {
    const int n0 = D.n[0], n1 = D.n[1], n2 = D.n[2], P0 = D.P[0], P1 = D.P[1], P2 = D.P[2], H0 = D.H0;
    launch_x<float>(true, D.Q, D.C, nullptr, n1 * n2, n0, P0, n1, P1, D.tw32[0], st);
    launch_strided<float>(D.C, P1, H0, H0, n2, (long long)P1 * H0, n1, P1, 0, nullptr, 0, 0, D.tw32[1], st);
    launch_strided<float>(D.C, P2, (long long)P1 * H0, H0, P1, H0, n2, n2, 2, D.spec, (long long)P1 * H0, H0,
                          D.tw32[2], st);
    launch_strided<float>(D.C, P1, H0, H0, n2, (long long)P1 * H0, P1, n1, 1, nullptr, 0, 0, D.tw32[1], st);
    launch_x<float>(false, nullptr, D.C, D.Q, n1 * n2, n0, P0, n1, P1, D.tw32[0], st);
  }
  mark(3);
  switch (D.order) {
    case 1: k4_interp_corr<1><<<rows_blocks, 256, 0, st>>>(Np, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_col, D.c_val, D.q, D.uloc, D.u); break;
    case 2: k4_interp_corr<2><<<rows_blocks, 256, 0, st>>>(Np, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_col, D.c_val, D.q, D.uloc, D.u); break;
    default: k4_interp_corr<3><<<rows_blocks, 256, 0, st>>>(Np, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_col, D.c_val, D.q, D.uloc, D.u); break;
  }
  CK(cudaGetLastError());
  mark(4);
  k5_grad_sum<<<rows_blocks, 256, 0, st>>>(Np, D.u, D.r1_ptr, D.r1_col, D.r1_G, H, mode == EVAL_HEFF ? 1 : 0);
  CK(cudaGetLastError());
  mark(5);
}

}  // namespace pmfem
