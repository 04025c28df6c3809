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
// In-place radix-2 DIT in shared memory (bit-reversed load, log2 P butterfly stages).
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

__device__ __forceinline__ int bitrev(int v, int logn) { return logn ? (int)(__brev((unsigned)v) >> (32 - logn)) : 0; }

// In-place radix-2 DIT on nl lines in smem; element e of line l is at base(l) + e*es.
// Input in bit-reversed order, output natural.  tw[k] = exp(-2 pi i k / (P*tw_stride)).
// line_fast: consecutive threads take consecutive lines (tile layouts, es > 1).
template <class C, class Base>
__device__ void smem_fft(C* buf, int P, int logP, int nl, Base base, int es, const C* __restrict__ tw,
                         int tw_stride, bool inv, bool line_fast) {
  const int nb = P >> 1;
  const bool pow2_nl = (nl & (nl - 1)) == 0;
  const int lnl = __ffs(nl) - 1;
  // pairs of radix-2 stages (s, s+1) fused into one radix-4 pass: each thread loads 4
  // elements, does both butterfly levels in registers -> half the syncs and smem traffic
  int s = 0;
  const int nq = P >> 2;
  for (; s + 1 < logP; s += 2) {
    const int h = 1 << s;
    const int t1 = (nb >> s) * tw_stride;          // W_{2h}^j   = tw[j * t1]
    const int t2 = (nb >> (s + 1)) * tw_stride;    // W_{4h}^j   = tw[j * t2]
    for (int idx = threadIdx.x; idx < nl * nq; idx += blockDim.x) {
      int l, b;
      if (line_fast) {
        if (pow2_nl) { l = idx & (nl - 1); b = idx >> lnl; } else { l = idx % nl; b = idx / nl; }
      } else {
        b = idx & (nq - 1); l = idx >> (logP - 2);
      }
      const int j = b & (h - 1);
      const int i0 = ((b >> s) << (s + 2)) + j;
      C w1 = tw[j * t1], w2a = tw[j * t2], w2b = tw[(j + h) * t2];
      if (inv) { w1.y = -w1.y; w2a.y = -w2a.y; w2b.y = -w2b.y; }
      C* p = buf + base(l) + i0 * es;
      const int hs = h * es;
      const C a0 = p[0], a1 = p[hs], a2 = p[2 * hs], a3 = p[3 * hs];
      C t = cmul(w1, a1);
      C b0, b1, b2, b3;
      b0.x = a0.x + t.x; b0.y = a0.y + t.y; b1.x = a0.x - t.x; b1.y = a0.y - t.y;
      t = cmul(w1, a3);
      b2.x = a2.x + t.x; b2.y = a2.y + t.y; b3.x = a2.x - t.x; b3.y = a2.y - t.y;
      t = cmul(w2a, b2);
      p[0].x = b0.x + t.x; p[0].y = b0.y + t.y; p[2 * hs].x = b0.x - t.x; p[2 * hs].y = b0.y - t.y;
      t = cmul(w2b, b3);
      p[hs].x = b1.x + t.x; p[hs].y = b1.y + t.y; p[3 * hs].x = b1.x - t.x; p[3 * hs].y = b1.y - t.y;
    }
    __syncthreads();
  }
  for (; s < logP; ++s) {
    const int half = 1 << s;
    const int tstep = (nb >> s) * tw_stride;
    for (int idx = threadIdx.x; idx < nl * nb; idx += blockDim.x) {
      int l, b;
      // power-of-two line counts (every line-fast call site) use shifts, not integer division
      if (line_fast) {
        if (pow2_nl) { l = idx & (nl - 1); b = idx >> lnl; } else { l = idx % nl; b = idx / nl; }
      } else {
        b = idx & (nb - 1); l = idx >> (logP - 1);
      }
      const int j = b & (half - 1);
      const int i0 = ((b >> s) << (s + 1)) + j;
      C w = tw[j * tstep];
      if (inv) w.y = -w.y;
      C* p0 = buf + base(l) + i0 * es;
      C* p1 = p0 + half * es;
      C a = *p0, bb = *p1;
      C t = cmul(w, bb);
      p0->x = a.x + t.x; p0->y = a.y + t.y;
      p1->x = a.x - t.x; p1->y = a.y - t.y;
    }
    __syncthreads();
  }
}

// bit-reversal permutation of nl lines in place
template <class C, class Base>
__device__ void smem_bitrev(C* buf, int P, int logP, int nl, Base base, int es) {
  for (int idx = threadIdx.x; idx < nl * P; idx += blockDim.x) {
    // es == 1: element fastest (consecutive banks); else line fastest (lines are contiguous)
    // P and (at every call site) nl are powers of two
    const int l = (es == 1) ? (idx >> logP) : (idx & (nl - 1));
    const int e = (es == 1) ? (idx & (P - 1)) : (idx >> (__ffs(nl) - 1));
    const int r = bitrev(e, logP);
    if (r > e) {
      C* p = buf + base(l);
      C a = p[e * es]; p[e * es] = p[r * es]; p[r * es] = a;
    }
  }
  __syncthreads();
}

struct RowMap {   // real rows r = i2*n1 + i1  ->  complex rows i2*P1 + i1
  int n1, P1;
  __device__ __forceinline__ long long crow(int r) const { int i2 = r / n1, i1 = r - i2 * n1; return (long long)i2 * P1 + i1; }
};

struct RowBase {
  int M;
  __device__ __forceinline__ int operator()(int l) const { return l * M; }
};

// ---------------------------------------------------------------- X pass (contiguous lines)
template <class T>
__global__ void fft_x_forward(const T* __restrict__ in, typename Cx<T>::t* __restrict__ out, int nrows, int n0,
                              int P0, int logM, RowMap rm, const typename Cx<T>::t* __restrict__ tw, int nl) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int M = P0 >> 1, H0 = M + 1;
  const int r0 = blockIdx.x * nl;
  const int nlines = min(nl, nrows - r0);
  // global loads issued LB at a time per thread (latency: one pass streams the whole grid)
  constexpr int LB = 8;
  for (int i0 = threadIdx.x; i0 < nlines * M; i0 += LB * blockDim.x) {
    C z[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, l = idx >> logM, j = idx & (M - 1);
      z[b].x = T(0); z[b].y = T(0);
      if (idx < nlines * M) {
        const T* row = in + (long long)(r0 + l) * n0;
        if (2 * j < n0) z[b].x = row[2 * j];
        if (2 * j + 1 < n0) z[b].y = row[2 * j + 1];
      }
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, l = idx >> logM, j = idx & (M - 1);
      if (idx < nlines * M) buf[l * M + bitrev(j, logM)] = z[b];
    }
  }
  __syncthreads();
  smem_fft<C>(buf, M, logM, nlines, RowBase{M}, 1, tw, 2, false, false);
  // X_k = A_k + W^k B_k, A = (Z_k + conj Z_{M-k})/2, B = (Z_k - conj Z_{M-k})/(2i)
  for (int idx = threadIdx.x; idx < nlines * H0; idx += blockDim.x) {
    const int l = idx / H0, k = idx - l * H0;
    C zk = buf[l * M + (k % M)];
    C zm = cconj(buf[l * M + ((M - k) % M)]);
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
  const int r0 = blockIdx.x * nl;
  const int nlines = min(nl, nrows - r0);
  // Z_k = (X_k + conj X_{M-k}) + i W^{-k} (X_k - conj X_{M-k}),  k < M
  constexpr int LB = 4;
  for (int i0 = threadIdx.x; i0 < nlines * M; i0 += LB * blockDim.x) {
    C xa[LB], xb[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, l = idx >> logM, k = idx & (M - 1);
      if (idx < nlines * M) {
        const C* row = in + rm.crow(r0 + l) * H0;
        xa[b] = row[k]; xb[b] = row[M - k];
      }
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
    const int idx = i0 + b * blockDim.x, l = idx >> logM, k = idx & (M - 1);
    if (idx >= nlines * M) break;
    C xk = xa[b];
    C xm = cconj(xb[b]);
    C E; E.x = xk.x + xm.x; E.y = xk.y + xm.y;
    C D; D.x = xk.x - xm.x; D.y = xk.y - xm.y;
    C O = cmul(cconj(tw[k]), D);
    C Z; Z.x = E.x - O.y; Z.y = E.y + O.x;     // E + i O
    buf[l * M + bitrev(k, logM)] = Z;
    }
  }
  __syncthreads();
  smem_fft<C>(buf, M, logM, nlines, RowBase{M}, 1, tw, 2, true, false);
  for (int idx = threadIdx.x; idx < nlines * M; idx += blockDim.x) {
    const int l = idx >> logM, j = idx & (M - 1);
    C z = buf[l * M + j];
    T* row = out + (long long)(r0 + l) * n0;
    if (2 * j < n0) row[2 * j] = z.x;
    if (2 * j + 1 < n0) row[2 * j + 1] = z.y;
  }
}

// ---------------------------------------------------------------- strided C2C pass (split plan)
// Lines along an axis with element stride es; a CTA takes TILE consecutive columns of one
// plane.  mode 0 forward, 1 inverse, 2 forward * spec * inverse.
struct TileBase {
  __device__ __forceinline__ int operator()(int l) const { return l; }
};

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
  constexpr int LB = 8;
  for (int i0 = threadIdx.x; i0 < P * TILE; i0 += LB * blockDim.x) {
    C v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, e = idx / TILE, c = idx - e * TILE;
      v[b].x = T(0); v[b].y = T(0);
      if (idx < P * TILE && e < nin && c < nc) v[b] = base[e * es + c];
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, e = idx / TILE, c = idx - e * TILE;
      if (idx < P * TILE) buf[bitrev(e, logP) * TILE + c] = v[b];
    }
  }
  __syncthreads();
  smem_fft<C>(buf, P, logP, TILE, TileBase{}, TILE, tw, 1, mode == 1, true);
  if (mode == 2) {
    const T* sp = spec + (long long)blockIdx.y * spec_plane_stride + c0;
    constexpr int SB = 8;
    for (int base = threadIdx.x; base < P * TILE; base += SB * blockDim.x) {
      T gv[SB];
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int idx = base + b * blockDim.x;
        const int e = idx / TILE, c = idx - e * TILE;
        gv[b] = (idx < P * TILE && c < nc) ? __ldg(sp + e * spec_es + c) : T(0);
      }
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int idx = base + b * blockDim.x;
        if (idx < P * TILE) {
          C v = buf[idx];
          v.x *= gv[b]; v.y *= gv[b];
          buf[idx] = v;
        }
      }
    }
    __syncthreads();
    smem_bitrev<C>(buf, P, logP, TILE, TileBase{}, TILE);
    smem_fft<C>(buf, P, logP, TILE, TileBase{}, TILE, tw, 1, true, true);
  }
  for (int idx = threadIdx.x; idx < nout * TILE; idx += blockDim.x) {
    const int e = idx / TILE, c = idx - e * TILE;
    if (c < nc) base[e * es + c] = buf[e * TILE + c];
  }
}

// ---------------------------------------------------------------- fused YZ pass (fused plan)
struct PlaneBase {   // line l = (plane index l / tile, column l % tile); logP2 = 0: natural order
  int tile, plane, logP2;
  __device__ __forceinline__ int operator()(int l) const {
    const int p = l >> (__ffs(tile) - 1);        // tile is a power of two
    return (logP2 ? bitrev(p, logP2) : p) * plane + (l & (tile - 1));
  }
};

// smem [P2][P1][tile] (tile columns contiguous).  Planes are stored at bit-reversed z
// positions so the y transforms of the n2 data planes leave the z lines in DIT input order.
template <class T>
__global__ void __launch_bounds__(1024) fft_yz_fused(typename Cx<T>::t* __restrict__ data, int n1, int P1, int logP1, int n2, int P2,
                             int logP2, int H0, int tile, const T* __restrict__ spec,
                             const typename Cx<T>::t* __restrict__ tw1, const typename Cx<T>::t* __restrict__ tw2) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int c0 = blockIdx.x * tile;
  const int nc = min(tile, H0 - c0);
  // plane stride padded by one element when tile == 1: consecutive threads then take
  // consecutive y lines (line-fast) at a stride of P1+1 elements -> no bank conflicts
  const int nzl = P1 * tile;                                  // z lines per CTA
  const int pl = nzl + (tile == 1 ? 1 : 0);                   // plane stride in smem
  const int ltile = __ffs(tile) - 1, ln1 = __ffs(n1) - 1;     // tile, n1 powers of two
  // zero the whole tile (padded planes / rows must read as zero), then load the data block
  for (int idx = threadIdx.x; idx < P2 * pl; idx += blockDim.x) { C z; z.x = T(0); z.y = T(0); buf[idx] = z; }
  __syncthreads();
  // iterate over the destination y slots (slot = bit-reversed row, every (P1/n1)-th slot holds
  // data) so consecutive threads store to nearby shared addresses; the global reads of one
  // column are strided either way
  const int sstep = P1 / n1;
  constexpr int LB = 8;
  for (int i0 = threadIdx.x; i0 < n2 * n1 * tile; i0 += LB * blockDim.x) {
    C v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x;
      const int c = idx & (tile - 1), r = idx >> ltile, slot = (r & (n1 - 1)) * sstep, i2 = r >> ln1;
      if (idx < n2 * n1 * tile && c < nc) v[b] = data[((long long)i2 * P1 + bitrev(slot, logP1)) * H0 + c0 + c];
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x;
      const int c = idx & (tile - 1), r = idx >> ltile, slot = (r & (n1 - 1)) * sstep, i2 = r >> ln1;
      if (idx < n2 * n1 * tile && c < nc) buf[bitrev(i2, logP2) * pl + slot * tile + c] = v[b];
    }
  }
  __syncthreads();
  // forward y on the n2 data planes: line (i2, c) base = bitrev(i2)*pl + c, stride tile
  const PlaneBase ybase{tile, pl, logP2};
  // (one column per CTA: element-fast -- line-fast would put consecutive threads on planes at
  // bit-reversed offsets, i.e. in the same banks)
  smem_fft<C>(buf, P1, logP1, n2 * tile, ybase, tile, tw1, 1, false, tile > 1);
  // forward z on every (k1, c): base = k1*tile + c, stride pl
  const TileBase zbase{};
  smem_fft<C>(buf, P2, logP2, nzl, zbase, pl, tw2, 1, false, true);
  // multiply by the real spectrum G_hat[k2][k1][k0] (natural order now); the spectrum loads
  // are issued 8 at a time per thread so their latency overlaps
  constexpr int SB = 8;
  for (int base = threadIdx.x; base < P2 * nzl; base += SB * blockDim.x) {
    T gv[SB];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int idx = base + b * blockDim.x;
      const int c = idx & (tile - 1), r = idx >> ltile, k1 = r & (P1 - 1), k2 = r >> logP1;
      gv[b] = (idx < P2 * nzl && c < nc) ? __ldg(spec + ((long long)k2 * P1 + k1) * H0 + c0 + c) : T(0);
    }
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int idx = base + b * blockDim.x;
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
  // inverse z (bit-reverse first); only planes i2 < n2 are needed afterwards
  smem_bitrev<C>(buf, P2, logP2, nzl, zbase, pl);
  smem_fft<C>(buf, P2, logP2, nzl, zbase, pl, tw2, 1, true, true);
  // inverse y on planes i2 < n2 (natural z order now)
  const PlaneBase ybase2{tile, pl, 0};
  smem_bitrev<C>(buf, P1, logP1, n2 * tile, ybase2, tile);
  smem_fft<C>(buf, P1, logP1, n2 * tile, ybase2, tile, tw1, 1, true, tile > 1);
  for (int idx = threadIdx.x; idx < n2 * n1 * tile; idx += blockDim.x) {
    const int c = idx & (tile - 1), r = idx >> ltile, i1 = r & (n1 - 1), i2 = r >> ln1;
    if (c < nc) data[((long long)i2 * P1 + i1) * H0 + c0 + c] = buf[i2 * pl + i1 * tile + c];
  }
}

// ---------------------------------------------------------------- fused YZ, zero-padded z
// One column per CTA (tile 1) when z is zero-padded (P2 = 2 n2).  The length-P2 z transform of
// a line with n2 data values splits into two length-n2 transforms (w = exp(-2 pi i / P2)):
//   X[2k] = DFT_n2(x)[k],   X[2k+1] = DFT_n2(x_j w^j)[k],
// and the n2 kept outputs of the (unnormalised) inverse are
//   y_j = IDFT_n2(Y_even)_j + w^-j IDFT_n2(Y_odd)_j,
// so shared memory holds only the n2 data planes [n2][P1 + 1] plus scratch for `chunk` z lines
// (even and odd halves, line stride n2 + 1): about half the footprint of fft_yz_fused, i.e. two
// CTAs per SM at P1 = P2 = 128 (C3) instead of one.
template <class T>
__global__ void __launch_bounds__(512, 2) fft_yz_fused_zhalf(typename Cx<T>::t* __restrict__ data, int n1, int P1,
                                                             int logP1, int n2, int logn2, int H0, int chunk,
                                                             const T* __restrict__ spec,
                                                             const typename Cx<T>::t* __restrict__ tw1,
                                                             const typename Cx<T>::t* __restrict__ tw2) {
  using C = typename Cx<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  const int pl = P1 + 1, ls = n2 + 1;
  C* scr = buf + n2 * pl;
  const int c0 = blockIdx.x;
  const int ln1 = __ffs(n1) - 1, lch = __ffs(chunk) - 1;
  for (int idx = threadIdx.x; idx < n2 * pl; idx += blockDim.x) { C z; z.x = T(0); z.y = T(0); buf[idx] = z; }
  __syncthreads();
  // data rows i1 < n1 go to their bit-reversed y slots (every (P1/n1)-th slot)
  const int sstep = P1 / n1;
  constexpr int LB = 8;
  for (int i0 = threadIdx.x; i0 < n2 * n1; i0 += LB * blockDim.x) {
    C v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, slot = (idx & (n1 - 1)) * sstep, i2 = idx >> ln1;
      if (idx < n2 * n1) v[b] = data[((long long)i2 * P1 + bitrev(slot, logP1)) * H0 + c0];
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * blockDim.x, slot = (idx & (n1 - 1)) * sstep, i2 = idx >> ln1;
      if (idx < n2 * n1) buf[i2 * pl + slot] = v[b];
    }
  }
  __syncthreads();
  const PlaneBase yb{1, pl, 0};
  smem_fft<C>(buf, P1, logP1, n2, yb, 1, tw1, 1, false, false);
  const RowBase zb{ls};
  for (int k1a = 0; k1a < P1; k1a += chunk) {
    // z lines k1a .. k1a+chunk: even half x_j, odd half x_j w^j, both bit-reversed (DIT input)
    for (int idx = threadIdx.x; idx < chunk * n2; idx += blockDim.x) {
      const int l = idx & (chunk - 1), j = idx >> lch, r = bitrev(j, logn2);
      const C x = buf[j * pl + k1a + l];
      scr[l * ls + r] = x;
      scr[(chunk + l) * ls + r] = cmul(x, tw2[j]);
    }
    __syncthreads();
    smem_fft<C>(scr, n2, logn2, 2 * chunk, zb, 1, tw2, 2, false, false);
    // x G_hat[k2][k1]: k2 = 2k (even half), 2k + 1 (odd half); loads batched for latency
    constexpr int SB = 8;
    const int tot = 2 * chunk * n2;
    for (int base = threadIdx.x; base < tot; base += SB * blockDim.x) {
      T gv[SB];
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int idx = base + b * blockDim.x;
        const int k = idx & (n2 - 1), l = idx >> logn2, half = l >= chunk ? 1 : 0, k1 = k1a + l - half * chunk;
        gv[b] = idx < tot ? __ldg(spec + ((long long)(2 * k + half) * P1 + k1) * H0 + c0) : T(0);
      }
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int idx = base + b * blockDim.x;
        if (idx < tot) {
          C* pv = scr + (idx >> logn2) * ls + (idx & (n2 - 1));
          C v = *pv;
          v.x *= gv[b]; v.y *= gv[b];
          *pv = v;
        }
      }
    }
    __syncthreads();
    smem_bitrev<C>(scr, n2, logn2, 2 * chunk, zb, 1);
    smem_fft<C>(scr, n2, logn2, 2 * chunk, zb, 1, tw2, 2, true, false);
    for (int idx = threadIdx.x; idx < chunk * n2; idx += blockDim.x) {
      const int l = idx & (chunk - 1), j = idx >> lch;
      const C e = scr[l * ls + j], o = cmul(cconj(tw2[j]), scr[(chunk + l) * ls + j]);
      C y; y.x = e.x + o.x; y.y = e.y + o.y;
      buf[j * pl + k1a + l] = y;
    }
    __syncthreads();
  }
  smem_bitrev<C>(buf, P1, logP1, n2, yb, 1);
  smem_fft<C>(buf, P1, logP1, n2, yb, 1, tw1, 1, true, false);
  for (int idx = threadIdx.x; idx < n2 * n1; idx += blockDim.x) {
    const int i1 = idx & (n1 - 1), i2 = idx >> ln1;
    data[((long long)i2 * P1 + i1) * H0 + c0] = buf[i2 * pl + i1];
  }
}

}  // namespace pmfem
