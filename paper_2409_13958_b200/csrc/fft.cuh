// Hand-written shared-memory FFT passes for the BAIM step-2 convolution:
//   U = F^-1( G_hat . F Q ) on the padded grid (periodic axes circular, no padding, P:340;
//   non-periodic axes zero-padded to 2N).
// Layout: real grid [n2][n1][n0] (x fastest); complex half spectrum [P2][P1][H0], H0 = P0/2+1.
// Plans (pruned on padded axes: zero halves are never read, unneeded outputs never written):
//   fused (yz plane of TILE columns fits in shared memory -- C1, C2, C3, C5):
//     X  : real->complex along x for the n1*n2 data rows
//     YZ : per column tile: FFT_y (n2 data planes) -> FFT_z -> * G_hat -> IFFT_z (keep n2)
//          -> IFFT_y (keep n1), all in shared memory (one read + one write of the spectrum)
//     X' : complex->real along x, keep n0
//   split (C4, 256^2 planes): X, Y, Z(* G_hat, fused fwd/inv), Y', X'.
// Line transforms: Stockham autosort passes of radix 8 (plus one radix-2/4 pass when log2 P is
// not a multiple of 3) -- natural order in and out, no bit reversal.  In a pass every thread
// reads its R-point groups into registers, the CTA synchronises, then each thread twiddles,
// does the R-point DFT in registers and writes back in place; a thread holds up to 32 float2
// (16 double2) per pass, so a CTA transforms up to 32 x blockDim complex values at once.
// Zero inputs beyond nin are never loaded; outputs beyond nout are never stored.
// Twiddles come from a shared-memory table W_N^m, m < N.
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
template <class C> __device__ __forceinline__ C cadd(C a, C b) { a.x += b.x; a.y += b.y; return a; }
template <class C> __device__ __forceinline__ C csub(C a, C b) { a.x -= b.x; a.y -= b.y; return a; }
// multiply by -i (forward) or +i (inverse)
template <class C> __device__ __forceinline__ C cmi(C a, bool inv) {
  C r;
  if (inv) { r.x = -a.y; r.y = a.x; } else { r.x = a.y; r.y = -a.x; }
  return r;
}

// complex values a thread holds per pass
template <class C> struct FftBudget { static constexpr int V = sizeof(C) == 8 ? 32 : 16; };

// ---------------------------------------------------------------- in-register DFTs
template <class C> __device__ __forceinline__ void dft2(C& a, C& b) { C t = a; a = cadd(t, b); b = csub(t, b); }

template <class C> __device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3, bool inv) {
  const C t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = cmi(csub(a1, a3), inv);
  a0 = cadd(t0, t2); a2 = csub(t0, t2); a1 = cadd(t1, t3); a3 = csub(t1, t3);
}

template <class C, int R> struct Dft;
template <class C> struct Dft<C, 2> {
  static __device__ __forceinline__ void run(C* v, bool) { dft2(v[0], v[1]); }
};
template <class C> struct Dft<C, 4> {
  static __device__ __forceinline__ void run(C* v, bool inv) { dft4(v[0], v[1], v[2], v[3], inv); }
};
template <class C> struct Dft<C, 8> {
  // X_k = U_k + W8^k V_k, X_{k+4} = U_k - W8^k V_k with U, V the DFT4 of the even / odd inputs
  static __device__ __forceinline__ void run(C* v, bool inv) {
    using T = decltype(v[0].x);
    C u0 = v[0], u1 = v[2], u2 = v[4], u3 = v[6];
    C w0 = v[1], w1 = v[3], w2 = v[5], w3 = v[7];
    dft4(u0, u1, u2, u3, inv);
    dft4(w0, w1, w2, w3, inv);
    const T c = T(0.70710678118654752440);
    C t;
    // W8^1 = (c, -c) forward, (c, c) inverse
    t.x = c * (w1.x + (inv ? -w1.y : w1.y)); t.y = c * (w1.y + (inv ? w1.x : -w1.x)); w1 = t;
    w2 = cmi(w2, inv);
    // W8^3 = (-c, -c) forward, (-c, c) inverse
    t.x = c * (-w3.x + (inv ? -w3.y : w3.y)); t.y = c * (-w3.y + (inv ? w3.x : -w3.x)); w3 = t;
    v[0] = cadd(u0, w0); v[4] = csub(u0, w0);
    v[1] = cadd(u1, w1); v[5] = csub(u1, w1);
    v[2] = cadd(u2, w2); v[6] = csub(u2, w2);
    v[3] = cadd(u3, w3); v[7] = csub(u3, w3);
  }
};

template <int R> struct Log2;
template <> struct Log2<2> { static constexpr int v = 1; };
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };

// One in-place Stockham pass of radix R over nl lines of length P (element stride es, line
// base base(l)), Ns = product of the earlier radices.  tw[m] = W_{P << tws}^m.
// LF: consecutive threads take consecutive lines (strided layouts), else consecutive groups
// of one line (contiguous lines).
template <class C, int R, bool LF, class Base>
__device__ __forceinline__ void sk_pass(C* buf, int P, int logP, int logNs, int nl, Base base, int es, const C* tw,
                                        int tws, bool inv, int nin, int nout) {
  constexpr int IT = FftBudget<C>::V / R;
  constexpr int LR = Log2<R>::v;
  const int logT = logP - LR, T = 1 << logT;
  const int items = nl << logT;
  const int Ns = 1 << logNs;
  const int lnl = (nl & (nl - 1)) == 0 ? __ffs(nl) - 1 : -1;       // log2(nl) if a power of two
  C v[IT][R];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int w = threadIdx.x + it * blockDim.x;
    if (w < items) {
      int l, j;
      if (LF) {
        if (lnl >= 0) { l = w & (nl - 1); j = w >> lnl; } else { l = w % nl; j = w / nl; }
      } else { j = w & (T - 1); l = w >> logT; }
      const C* p = buf + base(l);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int idx = j + (r << logT);
        if (idx < nin) v[it][r] = p[idx * es];
        else { v[it][r].x = 0; v[it][r].y = 0; }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int w = threadIdx.x + it * blockDim.x;
    if (w < items) {
      int l, j;
      if (LF) {
        if (lnl >= 0) { l = w & (nl - 1); j = w >> lnl; } else { l = w % nl; j = w / nl; }
      } else { j = w & (T - 1); l = w >> logT; }
      const int k = j & (Ns - 1);
      if (logNs > 0) {
        // W_{Ns R}^{r k} = W_P^{r k P / (Ns R)}
        const int sh = logP - logNs - LR + tws;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          C wv = tw[(r * k) << sh];
          if (inv) wv.y = -wv.y;
          v[it][r] = cmul(v[it][r], wv);
        }
      }
      Dft<C, R>::run(v[it], inv);
      C* p = buf + base(l);
      const int d = ((j - k) << LR) + k;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int o = d + r * Ns;
        if (o < nout) p[o * es] = v[it][r];
      }
    }
  }
  __syncthreads();
}

// Full line transform (natural order in and out): radix-8 passes, then one radix-2/4 pass.
template <class C, bool LF, class Base>
__device__ void sk_fft(C* buf, int P, int logP, int nl, Base base, int es, const C* tw, int tws, bool inv, int nin,
                       int nout) {
  int logNs = 0, left = logP;
  while (left >= 3) {
    sk_pass<C, 8, LF>(buf, P, logP, logNs, nl, base, es, tw, tws, inv, logNs == 0 ? nin : P, left == 3 ? nout : P);
    logNs += 3;
    left -= 3;
  }
  if (left == 2) sk_pass<C, 4, LF>(buf, P, logP, logNs, nl, base, es, tw, tws, inv, logNs == 0 ? nin : P, nout);
  else if (left == 1) sk_pass<C, 2, LF>(buf, P, logP, logNs, nl, base, es, tw, tws, inv, logNs == 0 ? nin : P, nout);
}

// shared twiddle table tw[m] = W_N^m, m < N, from the global half table twg[k] = W_N^k, k < N/2
template <class C>
__device__ __forceinline__ void load_twiddles(C* tw, const C* __restrict__ twg, int N) {
  const int h = N >> 1;
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    C w;
    if (h == 0) { w.x = 1; w.y = 0; }
    else if (m < h) w = twg[m];
    else { w = twg[m - h]; w.x = -w.x; w.y = -w.y; }
    tw[m] = w;
  }
}

struct RowMap {   // real rows r = i2*n1 + i1  ->  complex rows i2*P1 + i1
  int n1, P1;
  __device__ __forceinline__ long long crow(int r) const { int i2 = r / n1, i1 = r - i2 * n1; return (long long)i2 * P1 + i1; }
};

struct RowBase {
  int M;
  __device__ __forceinline__ int operator()(int l) const { return l * M; }
};

struct TileBase {
  __device__ __forceinline__ int operator()(int l) const { return l; }
};

// ---------------------------------------------------------------- X pass (contiguous lines)
// A real line of P0 points is transformed as M = P0/2 complex points z_j = x_2j + i x_2j+1.
// smem: nl lines of M values at row stride M+1 (line-fast passes are bank-conflict free),
// then the M-entry twiddle table of W_M.
template <class T>
__global__ void fft_x_forward(const T* __restrict__ in, typename Cx<T>::t* __restrict__ out, int nrows, int n0,
                              int P0, int logM, RowMap rm, const typename Cx<T>::t* __restrict__ tw, int nl) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int M = P0 >> 1, H0 = M + 1;
  const int MS = M + 1;
  C* stw = buf + nl * MS;
  const int r0 = blockIdx.x * nl;
  const int nlines = min(nl, nrows - r0);
  const int nin = (n0 + 1) >> 1;                 // z_j = 0 for 2j >= n0
  // W_M^m = W_P0^{2m}
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const int e = 2 * m;
    C w;
    if (e < M) w = tw[e]; else { w = tw[e - M]; w.x = -w.x; w.y = -w.y; }
    stw[m] = w;
  }
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    const int l = idx >> logM, j = idx & (M - 1);
    if (j >= nin) continue;
    const T* row = in + (long long)(r0 + l) * n0;
    C z;
    z.x = row[2 * j];
    z.y = (2 * j + 1 < n0) ? row[2 * j + 1] : T(0);
    buf[l * MS + j] = z;
  }
  __syncthreads();
  sk_fft<C, true>(buf, M, logM, nlines, RowBase{MS}, 1, stw, 0, false, nin, M);
  // X_k = A_k + W^k B_k, A = (Z_k + conj Z_{M-k})/2, B = (Z_k - conj Z_{M-k})/(2i)
  for (int idx = threadIdx.x; idx < nlines * H0; idx += blockDim.x) {
    const int l = idx / H0, k = idx - l * H0;
    C zk = buf[l * MS + (k % M)];
    C zm = cconj(buf[l * MS + ((M - k) % M)]);
    C A, B;
    A.x = T(0.5) * (zk.x + zm.x); A.y = T(0.5) * (zk.y + zm.y);
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
  const int MS = M + 1;
  C* stw = buf + nl * MS;
  const int r0 = blockIdx.x * nl;
  const int nlines = min(nl, nrows - r0);
  const int nout = (n0 + 1) >> 1;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const int e = 2 * m;
    C w;
    if (e < M) w = tw[e]; else { w = tw[e - M]; w.x = -w.x; w.y = -w.y; }
    stw[m] = w;
  }
  // Z_k = (X_k + conj X_{M-k}) + i W^{-k} (X_k - conj X_{M-k}),  k < M
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    const int l = idx >> logM, k = idx & (M - 1);
    const C* row = in + rm.crow(r0 + l) * H0;
    C xk = row[k];
    C xm = cconj(row[M - k]);
    C E; E.x = xk.x + xm.x; E.y = xk.y + xm.y;
    C D; D.x = xk.x - xm.x; D.y = xk.y - xm.y;
    C O = cmul(cconj(tw[k]), D);
    C Z; Z.x = E.x - O.y; Z.y = E.y + O.x;     // E + i O
    buf[l * MS + k] = Z;
  }
  __syncthreads();
  sk_fft<C, true>(buf, M, logM, nlines, RowBase{MS}, 1, stw, 0, true, M, nout);
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    const int l = idx >> logM, j = idx & (M - 1);
    if (j >= nout) continue;
    C z = buf[l * MS + j];
    T* row = out + (long long)(r0 + l) * n0;
    row[2 * j] = z.x;
    if (2 * j + 1 < n0) row[2 * j + 1] = z.y;
  }
}

// ---------------------------------------------------------------- strided C2C pass (split plan)
// Lines along an axis with element stride es; a CTA takes TILE consecutive columns of one
// plane.  mode 0 forward, 1 inverse, 2 forward * spec * inverse.  smem: [P][TILE] + P twiddles.
template <class T, int TILE>
__global__ void fft_strided(typename Cx<T>::t* __restrict__ data, int P, int logP, long long es, int ncol,
                            long long plane_stride, int nin, int nout, int mode,
                            const T* __restrict__ spec, long long spec_es, long long spec_plane_stride,
                            const typename Cx<T>::t* __restrict__ tw) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);       // [P][TILE]
  C* stw = buf + P * TILE;
  const int c0 = blockIdx.x * TILE;
  const int nc = min(TILE, ncol - c0);
  C* base = data + (long long)blockIdx.y * plane_stride + c0;
  load_twiddles(stw, tw, P);
  for (int idx = threadIdx.x; idx < nin * TILE; idx += blockDim.x) {
    const int e = idx / TILE, c = idx - e * TILE;
    C v; v.x = T(0); v.y = T(0);
    if (c < nc) v = base[e * es + c];
    buf[idx] = v;
  }
  __syncthreads();
  if (mode == 2) {
    sk_fft<C, true>(buf, P, logP, TILE, TileBase{}, TILE, stw, 0, false, nin, P);
    const T* sp = spec + (long long)blockIdx.y * spec_plane_stride + c0;
    constexpr int SB = 8;
    for (int b0 = threadIdx.x; b0 < P * TILE; b0 += SB * blockDim.x) {
      T gv[SB];
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int idx = b0 + b * blockDim.x;
        const int e = idx / TILE, c = idx - e * TILE;
        gv[b] = (idx < P * TILE && c < nc) ? __ldg(sp + e * spec_es + c) : T(0);
      }
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int idx = b0 + b * blockDim.x;
        if (idx < P * TILE) {
          C v = buf[idx];
          v.x *= gv[b]; v.y *= gv[b];
          buf[idx] = v;
        }
      }
    }
    __syncthreads();
    sk_fft<C, true>(buf, P, logP, TILE, TileBase{}, TILE, stw, 0, true, P, nout);
  } else {
    sk_fft<C, true>(buf, P, logP, TILE, TileBase{}, TILE, stw, 0, mode == 1, nin, nout);
  }
  for (int idx = threadIdx.x; idx < nout * TILE; idx += blockDim.x) {
    const int e = idx / TILE, c = idx - e * TILE;
    if (c < nc) base[e * es + c] = buf[idx];
  }
}

// ---------------------------------------------------------------- fused YZ pass (fused plan)
struct PlaneBase {   // line l = (plane l / tile, column l % tile)
  int ltile, plane, tile;
  __device__ __forceinline__ int operator()(int l) const { return (l >> ltile) * plane + (l & (tile - 1)); }
};

// smem [P2][pl] planes (pl = P1*tile + 1: consecutive y lines of different planes fall in
// different banks), tile columns contiguous, then the twiddle table of W_{max(P1,P2)}.
template <class T>
__global__ void fft_yz_fused(typename Cx<T>::t* __restrict__ data, int n1, int P1, int logP1, int n2, int P2,
                             int logP2, int H0, int tile, const T* __restrict__ spec,
                             const typename Cx<T>::t* __restrict__ tw1, const typename Cx<T>::t* __restrict__ tw2) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int c0 = blockIdx.x * tile;
  const int nc = min(tile, H0 - c0);
  const int nzl = P1 * tile;                                  // z lines per CTA
  const int pl = nzl + 1;                                     // plane stride in smem
  const int ltile = __ffs(tile) - 1, ln1 = __ffs(n1) - 1;     // tile, n1 powers of two
  // twiddle table for the longer axis; the other indexes it with a stride
  const bool ybig = P1 >= P2;
  const int PN = ybig ? P1 : P2;
  C* stw = buf + P2 * pl;
  load_twiddles(stw, ybig ? tw1 : tw2, PN);
  const int tws1 = ybig ? 0 : logP2 - logP1, tws2 = ybig ? logP1 - logP2 : 0;
  for (int idx = threadIdx.x; idx < n2 * n1 * tile; idx += blockDim.x) {
    const int c = idx & (tile - 1), r = idx >> ltile, i1 = r & (n1 - 1), i2 = r >> ln1;
    C v; v.x = T(0); v.y = T(0);
    if (c < nc) v = data[((long long)i2 * P1 + i1) * H0 + c0 + c];
    buf[i2 * pl + i1 * tile + c] = v;
  }
  __syncthreads();
  // forward y on the n2 data planes: line (i2, c), stride tile
  const PlaneBase yb{ltile, pl, tile};
  sk_fft<C, true>(buf, P1, logP1, n2 * tile, yb, tile, stw, tws1, false, n1, P1);
  // forward z on every (k1, c): base = k1*tile + c, stride pl
  sk_fft<C, true>(buf, P2, logP2, nzl, TileBase{}, pl, stw, tws2, false, n2, P2);
  // multiply by the real spectrum G_hat[k2][k1][k0]; the spectrum loads are issued 8 at a
  // time per thread so their latency overlaps
  constexpr int SB = 8;
  for (int b0 = threadIdx.x; b0 < P2 * nzl; b0 += SB * blockDim.x) {
    T gv[SB];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int idx = b0 + b * blockDim.x;
      const int c = idx & (tile - 1), r = idx >> ltile, k1 = r & (P1 - 1), k2 = r >> logP1;
      gv[b] = (idx < P2 * nzl && c < nc) ? __ldg(spec + ((long long)k2 * P1 + k1) * H0 + c0 + c) : T(0);
    }
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int idx = b0 + b * blockDim.x;
      if (idx < P2 * nzl) {
        const int c = idx & (tile - 1), r = idx >> ltile, k1 = r & (P1 - 1), k2 = r >> logP1;
        C* pv = buf + k2 * pl + k1 * tile + c;
        C v = *pv;
        v.x *= gv[b]; v.y *= gv[b];
        *pv = v;
      }
    }
  }
  __syncthreads();
  // inverse z, keep planes i2 < n2; inverse y on them, keep rows i1 < n1
  sk_fft<C, true>(buf, P2, logP2, nzl, TileBase{}, pl, stw, tws2, true, P2, n2);
  sk_fft<C, true>(buf, P1, logP1, n2 * tile, yb, tile, stw, tws1, true, P1, n1);
  for (int idx = threadIdx.x; idx < n2 * n1 * tile; idx += blockDim.x) {
    const int c = idx & (tile - 1), r = idx >> ltile, i1 = r & (n1 - 1), i2 = r >> ln1;
    if (c < nc) data[((long long)i2 * P1 + i1) * H0 + c0 + c] = buf[i2 * pl + i1 * tile + c];
  }
}

}  // namespace pmfem
