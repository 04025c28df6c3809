// Hand-written shared-memory FFT passes for the BAIM step-2 convolution:
//   U = F^-1( G_hat . F Q ) on the padded grid (periodic axes circular, no padding, P:340;
//   non-periodic axes zero-padded to 2N).
// Layout: real grid [n2][n1][n0] (x fastest); complex half spectrum [P2][P1][H0], H0 = P0/2+1.
// Plan (5 sweeps of the data, pruned on padded axes):
//   X  forward real->complex along x  (rows i1 < n1, i2 < n2 only; padding never read)
//   Y  forward C2C along y            (planes i2 < n2; input rows >= n1 are zero)
//   Z  forward C2C along z, * G_hat, inverse C2C along z, keep i2 < n2   (fused, one sweep)
//   Y' inverse C2C along y, keep i1 < n1
//   X' inverse complex->real along x, keep i0 < n0
// Each CTA stages a tile of lines in shared memory, runs an in-place radix-2 DIT FFT there
// (bit-reversed load, log2 P butterfly stages) and writes back with coalesced accesses.
// Templated on the real type: float for the hot path, double for the PGF spectrum build.
#pragma once
#include <cuda_runtime.h>

namespace pmfem {

template <class T> struct Cx;
template <> struct Cx<float> { using t = float2; };
template <> struct Cx<double> { using t = double2; };

template <class C> __device__ __forceinline__ C cmul(C a, C b) {
  C r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r;
}
template <class C> __device__ __forceinline__ C cconj(C a) { a.y = -a.y; return a; }

__device__ __forceinline__ int bitrev(int v, int logn) { return __brev(v) >> (32 - logn); }

// In-place radix-2 DIT on `nl` lines in smem: element e of line l at buf[l*ls + e*es].
// Input must be in bit-reversed order.  tw[k] = exp(-2 pi i k / Pt) for k < Pt/2 with
// Pt = P * tw_stride (so the P-point twiddle j is tw[j * tw_stride]).  inv -> conj twiddles.
template <class C>
__device__ void smem_fft(C* buf, int P, int logP, int nl, int ls, int es, const C* __restrict__ tw,
                         int tw_stride, bool inv) {
  const int nb = P >> 1;
  for (int s = 0; s < logP; ++s) {
    const int half = 1 << s;
    const int tstep = (nb >> s) * tw_stride;
    for (int idx = threadIdx.x; idx < nl * nb; idx += blockDim.x) {
      // tile layout (es > 1, lines contiguous): line fastest; row layout (es == 1): butterfly
      // fastest -- either way consecutive threads touch consecutive banks
      int l, b;
      if (es == 1) { b = idx % nb; l = idx / nb; } else { l = idx % nl; b = idx / nl; }
      int j = b & (half - 1);
      int i0 = ((b >> s) << (s + 1)) + j;
      int i1 = i0 + half;
      C w = tw[j * tstep];
      if (inv) w.y = -w.y;
      C* p0 = buf + l * ls + i0 * es;
      C* p1 = buf + l * ls + i1 * es;
      C a = *p0, bb = *p1;
      C t = cmul(w, bb);
      p0->x = a.x + t.x; p0->y = a.y + t.y;
      p1->x = a.x - t.x; p1->y = a.y - t.y;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- X pass (contiguous lines)
// forward: real rows (length n0 valid, P0 padded) -> H0 complex.  One CTA handles `nl` rows.
// Row r in [0, nrows): real source offset r * in_row_stride, complex dest offset r * H0 (rows
// are mapped (i1,i2) -> complex row index i2*P1 + i1 by the caller via row_map()).
struct RowMap {
  int n1, P1;        // real rows are r = i2*n1 + i1 ; complex rows are i2*P1 + i1
  __device__ __forceinline__ long long crow(int r) const { int i2 = r / n1, i1 = r - i2 * n1; return (long long)i2 * P1 + i1; }
};

template <class T>
__global__ void fft_x_forward(const T* __restrict__ in, typename Cx<T>::t* __restrict__ out, int nrows, int n0,
                              int P0, int logM, RowMap rm, const typename Cx<T>::t* __restrict__ tw, int nl) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int M = P0 >> 1, H0 = M + 1;
  const int r0 = blockIdx.x * nl;
  const int nlines = min(nl, nrows - r0);
  // load z_j = x_2j + i x_2j+1 in bit-reversed position
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    int l = idx / M, j = idx - l * M;
    const T* row = in + (long long)(r0 + l) * n0;
    C z;
    z.x = (2 * j < n0) ? row[2 * j] : T(0);
    z.y = (2 * j + 1 < n0) ? row[2 * j + 1] : T(0);
    buf[l * M + bitrev(j, logM)] = z;
  }
  __syncthreads();
  smem_fft<C>(buf, M, logM, nlines, M, 1, tw, 2, false);
  // X_k = A_k + W^k B_k, A = (Z_k + conj Z_{M-k})/2, B = (Z_k - conj Z_{M-k})/(2i)
  for (int idx = threadIdx.x; idx < nlines * H0; idx += blockDim.x) {
    int l = idx / H0, k = idx - l * H0;
    C zk = buf[l * M + (k % M)];
    C zm = cconj(buf[l * M + ((M - k) % M)]);
    C A, B;
    A.x = T(0.5) * (zk.x + zm.x); A.y = T(0.5) * (zk.y + zm.y);
    // (zk - zm)/(2i) = ( (zk-zm).y/2 , -(zk-zm).x/2 )
    B.x = T(0.5) * (zk.y - zm.y); B.y = -T(0.5) * (zk.x - zm.x);
    C w;
    if (k < M) w = tw[k]; else { w.x = T(-1); w.y = T(0); }
    C t = cmul(w, B);
    C X; X.x = A.x + t.x; X.y = A.y + t.y;
    out[rm.crow(r0 + l) * H0 + k] = X;
  }
}

// inverse: H0 complex -> real row, keep i0 < n0 (unnormalised: returns P0 * x)
template <class T>
__global__ void fft_x_inverse(const typename Cx<T>::t* __restrict__ in, T* __restrict__ out, int nrows, int n0,
                              int P0, int logM, RowMap rm, const typename Cx<T>::t* __restrict__ tw, int nl) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int M = P0 >> 1, H0 = M + 1;
  const int r0 = blockIdx.x * nl;
  const int nlines = min(nl, nrows - r0);
  // Z_k = (X_k + conj X_{M-k}) + i W^{-k} (X_k - conj X_{M-k}),  k < M
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    int l = idx / M, k = idx - l * M;
    const C* row = in + rm.crow(r0 + l) * H0;
    C xk = row[k];
    C xm = cconj(row[M - k]);
    C E; E.x = xk.x + xm.x; E.y = xk.y + xm.y;
    C D; D.x = xk.x - xm.x; D.y = xk.y - xm.y;
    C w = cconj(tw[k]);
    C O = cmul(w, D);
    C Z; Z.x = E.x - O.y; Z.y = E.y + O.x;     // E + i O
    buf[l * M + bitrev(k, logM)] = Z;
  }
  __syncthreads();
  smem_fft<C>(buf, M, logM, nlines, M, 1, tw, 2, true);
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    int l = idx / M, j = idx - l * M;
    C z = buf[l * M + j];
    T* row = out + (long long)(r0 + l) * n0;
    if (2 * j < n0) row[2 * j] = z.x;
    if (2 * j + 1 < n0) row[2 * j + 1] = z.y;
  }
}

// ---------------------------------------------------------------- strided C2C passes
// Lines along an axis with element stride `es` (in complex elements); a CTA takes TILE
// consecutive columns (contiguous in memory) of one "plane" so every global access is a
// TILE-wide contiguous segment.  Line element e of column c is at base + e*es + c.
//   nin  : input elements 0..nin-1 are read, the rest are zero (pruning)
//   nout : outputs 0..nout-1 are written
//   mode : 0 forward, 1 inverse, 2 forward * spec * inverse (fused, spec real [P][ncol] at
//          spec_base + e*spec_es + c)
template <class T, int TILE>
__global__ void fft_strided(typename Cx<T>::t* __restrict__ data, int P, int logP, long long es, int ncol,
                            long long plane_stride, int nin, int nout, int mode,
                            const T* __restrict__ spec, long long spec_es, long long spec_plane_stride,
                            const typename Cx<T>::t* __restrict__ tw) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);       // [P][TILE]
  const int c0 = blockIdx.x * TILE;
  const int nc = min(TILE, ncol - c0);
  C* base = data + (long long)blockIdx.y * plane_stride + c0;
  for (int idx = threadIdx.x; idx < P * TILE; idx += blockDim.x) {
    int e = idx / TILE, c = idx - e * TILE;
    C v; v.x = T(0); v.y = T(0);
    if (e < nin && c < nc) v = base[e * es + c];
    buf[bitrev(e, logP) * TILE + c] = v;
  }
  __syncthreads();
  smem_fft<C>(buf, P, logP, TILE, 1, TILE, tw, 1, mode == 1);
  if (mode == 2) {
    const T* sp = spec + (long long)blockIdx.y * spec_plane_stride + c0;
    // multiply (natural order) and re-load bit-reversed for the inverse
    for (int idx = threadIdx.x; idx < P * TILE; idx += blockDim.x) {
      int e = idx / TILE, c = idx - e * TILE;
      T g = (c < nc) ? sp[e * spec_es + c] : T(0);
      C v = buf[e * TILE + c];
      v.x *= g; v.y *= g;
      buf[e * TILE + c] = v;
    }
    __syncthreads();
    // bit-reverse permutation in place (swap pairs)
    for (int idx = threadIdx.x; idx < P * TILE; idx += blockDim.x) {
      int e = idx / TILE, c = idx - e * TILE;
      int r = bitrev(e, logP);
      if (r > e) { C a = buf[e * TILE + c]; buf[e * TILE + c] = buf[r * TILE + c]; buf[r * TILE + c] = a; }
    }
    __syncthreads();
    smem_fft<C>(buf, P, logP, TILE, 1, TILE, tw, 1, true);
  }
  for (int idx = threadIdx.x; idx < nout * TILE; idx += blockDim.x) {
    int e = idx / TILE, c = idx - e * TILE;
    if (c < nc) base[e * es + c] = buf[e * TILE + c];
  }
}

}  // namespace pmfem
