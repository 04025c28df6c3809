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
//
// Formats: the local operators (L, D, G on the periodic 1-ring and Z0 on the 1-/2-ring) share
// one column list per row and are stored SELL-32 (slices of 32 rows, column-major inside a
// slice): K1 and K5 run one thread per row with fully coalesced streaming loads and many
// independent loads in flight.  C_box (~10^2-10^3 entries per row) is CSR with rows padded to
// a multiple of 4 and is read by one warp per row with 16-byte vector loads.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include "device.cuh"
#include "fft.cuh"
#include "pgf.cuh"
#include <nccl.h>

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
float __int_as_float_host(int32_t c) { float f; std::memcpy(&f, &c, 4); return f; }

// Rows [row0, row1) of the internal order are processed; per-row outputs H are stored at
// n - hoff (hoff = row0 for the rank-local H of a distributed context, 0 otherwise).
struct RowRange {
  int64_t row0, row1, hoff;
  int c0, c1, c2;          // user component of internal axis 0, 1, 2 (axis permutation of m, H)
  int64_t ncol;            // columns (all rows, N') -- bounds of the gathered vectors (checked build)
};

// halo pack / unpack: buf[i*w + c] <-> v[idx[i]*w + c]
__global__ void k_pack(const float* __restrict__ v, const int32_t* __restrict__ idx, int64_t n, int w,
                       float* __restrict__ buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  const int64_t i = t / w;
  buf[t] = v[(int64_t)idx[i] * w + (t - i * w)];
}
__global__ void k_unpack(const float* __restrict__ buf, const int32_t* __restrict__ idx, int64_t n, int w,
                         float* __restrict__ v) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * w) return;
  const int64_t i = t / w;
  v[(int64_t)idx[i] * w + (t - i * w)] = buf[t];
}

// ------------------------------------------------------------------ K1 local_in
// One thread per row (SELL-32).  Per shared entry one 16-byte load (Zx, Zy, Zz, col) and one
// 16-byte gather of m (float4 copy); on the ring-1 prefix one more 16-byte load (L, Dx, Dy, Dz).
__device__ __forceinline__ int colof(float4 v) { return __float_as_int(v.w); }

// operator streams of K1/K5 are read once per evaluation: loaded with the evict-first
// (cache-streaming) hint so L1/L2 keep the gathered m / u vectors (measured: K1 at C2 0.067 ->
// 0.059 ms, C5 -5 %; K4's C_box stream measured neutral-to-worse with it (C3 +3 %) and keeps
// __ldg).  PMFEM_NO_STREAM_CS builds the plain __ldg variant for A/B.
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
#ifndef PMFEM_NO_STREAM_CS
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

__global__ void k_to_m4(RowRange rr, const float* __restrict__ m, float4* __restrict__ m4) {
  const int64_t n = rr.row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= rr.row1) return;
  const int64_t h = n - rr.hoff;
  m4[n] = make_float4(m[3 * h + rr.c0], m[3 * h + rr.c1], m[3 * h + rr.c2], 0.f);
}

// SPLIT = 2 (small meshes, < ~1M rows): two threads per row, lanes 0-15 of a warp take the
// even SELL columns of 16 rows and lanes 16-31 the odd ones (each half still reads 256
// contiguous bytes per column), partial sums combined with one shuffle -- twice the loads in
// flight when the row count alone cannot fill the GPU.
template <int SPLIT>
__global__ void __launch_bounds__(256) k1_local_in(
    RowRange rr, const float4* __restrict__ m4, const int64_t* __restrict__ sl_off, const int64_t* __restrict__ sl1_off,
    const float4* __restrict__ s_zc, const float4* __restrict__ s_LD, const float4* __restrict__ rowsum,
    float* __restrict__ q, float* __restrict__ uloc, float* __restrict__ H, int write_hex) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t n;
  int part;
  if (SPLIT == 1) { n = rr.row0 + gid; part = 0; }
  else { n = rr.row0 + (gid >> 6) * 32 + ((gid >> 5) & 1) * 16 + (threadIdx.x & 15); part = (threadIdx.x >> 4) & 1; }
  const bool valid = n < rr.row1;
  if (SPLIT == 1 && !valid) return;
  const int64_t s = (n - rr.row0) >> 5;                 // slices are relative to the own rows
  const int l = (int)((n - rr.row0) & 31);
  int64_t o = 0, o1 = 0;
  int w = 0, w1 = 0;
  float4 mn = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
    o = sl_off[s]; o1 = sl1_off[s];
    w = (int)((sl_off[s + 1] - o) >> 5); w1 = (int)((sl1_off[s + 1] - o1) >> 5);
    mn = m4[n];
  }
  float hx = 0.f, hy = 0.f, hz = 0.f, qq = 0.f, ul = 0.f;
  int64_t e = o + l + 32 * part, e1 = o1 + l + 32 * part;
  int j = part;
#pragma unroll 4
  for (; j < w1; j += SPLIT, e += 32 * SPLIT, e1 += 32 * SPLIT) {
    const float4 zc = ld_stream(s_zc + e);
    const float4 LD = ld_stream(s_LD + e1);
    DCHECK(colof(zc) >= 0 && colof(zc) < rr.ncol);
    const float4 mc = m4[colof(zc)];
    const float dx = mc.x - mn.x, dy = mc.y - mn.y, dz = mc.z - mn.z;
    hx = fmaf(LD.x, dx, hx); hy = fmaf(LD.x, dy, hy); hz = fmaf(LD.x, dz, hz);
    qq = fmaf(LD.y, dx, fmaf(LD.z, dy, fmaf(LD.w, dz, qq)));
    ul = fmaf(zc.x, dx, fmaf(zc.y, dy, fmaf(zc.z, dz, ul)));
  }
#pragma unroll 4
  for (; j < w; j += SPLIT, e += 32 * SPLIT) {
    const float4 zc = ld_stream(s_zc + e);
    DCHECK(colof(zc) >= 0 && colof(zc) < rr.ncol);
    const float4 mc = m4[colof(zc)];
    ul = fmaf(zc.x, mc.x - mn.x, fmaf(zc.y, mc.y - mn.y, fmaf(zc.z, mc.z - mn.z, ul)));
  }
  if (SPLIT == 2) {
    hx += __shfl_xor_sync(0xffffffffu, hx, 16); hy += __shfl_xor_sync(0xffffffffu, hy, 16);
    hz += __shfl_xor_sync(0xffffffffu, hz, 16); qq += __shfl_xor_sync(0xffffffffu, qq, 16);
    ul += __shfl_xor_sync(0xffffffffu, ul, 16);
    if (part) return;
  }
  if (!valid) return;
  const float4 rd = rowsum[2 * n], rz = rowsum[2 * n + 1];
  q[n] = qq + rd.x * mn.x + rd.y * mn.y + rd.z * mn.z;
  uloc[n] = ul + rz.x * mn.x + rz.y * mn.y + rz.z * mn.z;
  if (write_hex) { H[3 * (n - rr.hoff) + rr.c0] = hx; H[3 * (n - rr.hoff) + rr.c1] = hy; H[3 * (n - rr.hoff) + rr.c2] = hz; }
}

// exchange only: H = L m
__global__ void __launch_bounds__(256) k_exchange(RowRange rr, const float4* __restrict__ m4,
                                                  const int64_t* __restrict__ sl_off, const int64_t* __restrict__ sl1_off,
                                                  const float4* __restrict__ s_zc, const float4* __restrict__ s_LD,
                                                  float* __restrict__ H) {
  const int64_t n = rr.row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= rr.row1) return;
  const int64_t s = (n - rr.row0) >> 5;
  const int l = (int)((n - rr.row0) & 31);
  const int64_t o = sl_off[s], o1 = sl1_off[s];
  const int w1 = (int)((sl1_off[s + 1] - o1) >> 5);
  const float4 mn = m4[n];
  float hx = 0.f, hy = 0.f, hz = 0.f;
  int64_t e = o + l, e1 = o1 + l;
#pragma unroll 4
  for (int j = 0; j < w1; ++j, e += 32, e1 += 32) {
    const float4 mc = m4[colof(ld_stream(s_zc + e))];
    const float L = __ldg(&s_LD[e1].x);
    hx = fmaf(L, mc.x - mn.x, hx); hy = fmaf(L, mc.y - mn.y, hy); hz = fmaf(L, mc.z - mn.z, hz);
  }
  H[3 * (n - rr.hoff) + rr.c0] = hx; H[3 * (n - rr.hoff) + rr.c1] = hy; H[3 * (n - rr.hoff) + rr.c2] = hz;
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
// Tiled particle-to-grid: one CTA owns a T0 x T1 x T2 tile of the grid (the tiles partition
// it, so every grid point is written exactly once -- no memset, no global atomics).  The nodes
// whose (P+1)^3 stencil can reach the tile are those anchored in [tile - P, tile_end) per axis;
// rows are sorted by anchor box (x fastest), so they are the contiguous row ranges of the
// tile's (T2+P) x (T1+P) anchor lines, read through box_ptr.  A warp takes one line at a time,
// lanes take its nodes.  Shared-memory fp32 atomics are CAS loops on sm_100 (ATOMS.CAST.SPIN),
// so the tile accumulates in 32-bit fixed point with the native integer ATOMS.ADD: a first
// sweep finds max|q| of the tile's halo; with m_b the largest anchor-box population of the mesh
// (D.box_max, a global bound) every partial sum is bounded by 2 m_b (P+1)^3 max|q| (|Lagrange weight| <= 1 on the stencil interval,
// x2 margin); the scale is the power of two that maps that bound to 2^30 (no overflow), so a
// contribution is rounded to ~1e-7 of max|q| -- the level of fp32 accumulation -- and the sum is
// order-independent (deterministic).  Each node is read by up to prod_a (T_a+P)/T_a tiles.
// Rows outside [lo, hi) belong to other ranks (their contributions arrive with the Q reduction).
struct TileDims { int t0, t1, t2; };

// distinct anchors whose stencil can touch [a0, a0+T): up to two ranges [r0,r1],[r2,r3]
__device__ __forceinline__ int anchor_ranges(int a0, int T, int n, int per, int P, int* r) {
  if (per) {
    if (T + P >= n) { r[0] = 0; r[1] = n - 1; return 1; }
    if (a0 - P >= 0) { r[0] = a0 - P; r[1] = a0 + T - 1; return 1; }
    r[0] = 0; r[1] = a0 + T - 1; r[2] = n + a0 - P; r[3] = n - 1; return 2;
  }
  r[0] = max(a0 - P, 0); r[1] = min(a0 + T - 1, n - 1 - P);
  return r[0] <= r[1] ? 1 : 0;
}

// dynamic shared memory of k2_tile: the int tile, then per candidate segment (anchor line x
// x range) its first row and the exclusive prefix of the segment sizes, then the row map
// (2 x tile volume entries)
__host__ __device__ __forceinline__ int k2_nseg(int t1, int t2, int P) { return 2 * (t1 + P) * (t2 + P); }

template <int P>
__global__ void __launch_bounds__(256) k2_tile(GridDims g, TileDims td, const int32_t* __restrict__ box_ptr,
                                               const int4* __restrict__ st_s, const float4* __restrict__ st_t,
                                               const float* __restrict__ q, int64_t lo, int64_t hi, int box_max,
                                               int bz0, float* __restrict__ Q) {
  extern __shared__ int tile[];
  __shared__ int red_q;
  __shared__ int wsum[8];
  const int T0 = td.t0, T1 = td.t1, T2 = td.t2, vol = T0 * T1 * T2;
  int* seg_beg = tile + vol;
  int* seg_cum = seg_beg + k2_nseg(T1, T2, P);
  const int nt0 = g.n0 / T0, nt1 = g.n1 / T1;
  const int bx = blockIdx.x % nt0, by = (blockIdx.x / nt0) % nt1, bz = bz0 + blockIdx.x / (nt0 * nt1);
  const int x0 = bx * T0, y0 = by * T1, z0 = bz * T2;
  for (int i = threadIdx.x; i < vol; i += blockDim.x) tile[i] = 0;
  if (threadIdx.x == 0) red_q = 0;
  int rz[4], ry[4], rx[4];
  const int nz = anchor_ranges(z0, T2, g.n2, g.per2, P, rz);
  const int ny = anchor_ranges(y0, T1, g.n1, g.per1, P, ry);
  const int nx = anchor_ranges(x0, T0, g.n0, g.per0, P, rx);
  const int cz = nz == 0 ? 0 : (rz[1] - rz[0] + 1) + (nz == 2 ? rz[3] - rz[2] + 1 : 0);
  const int cy = ny == 0 ? 0 : (ry[1] - ry[0] + 1) + (ny == 2 ? ry[3] - ry[2] + 1 : 0);
  const int nseg = cz * cy * nx;
  DCHECK(nseg <= 256 * 8 && nseg <= k2_nseg(T1, T2, P));
  // segment table: rows [box_ptr(line + xa), box_ptr(line + xb + 1)) clipped to [lo, hi)
  constexpr int PER = 8;                                   // segments per thread in the scan
  int cnt[PER];
  int mysum = 0;
  const int s0 = threadIdx.x * PER;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int sg = s0 + u;
    cnt[u] = 0;
    if (sg < nseg) {
      const int line = sg / nx, r = sg - line * nx;
      const int iz = line / cy, iy = line - iz * cy;
      const int sz = iz <= rz[1] - rz[0] ? rz[0] + iz : rz[2] + iz - (rz[1] - rz[0] + 1);
      const int sy = iy <= ry[1] - ry[0] ? ry[0] + iy : ry[2] + iy - (ry[1] - ry[0] + 1);
      const int64_t lb = ((int64_t)sz * g.n1 + sy) * g.n0;
      const int64_t i0 = max((int64_t)__ldg(box_ptr + lb + rx[2 * r]), lo);
      const int64_t i1 = min((int64_t)__ldg(box_ptr + lb + rx[2 * r + 1] + 1), hi);
      seg_beg[sg] = (int)i0;
      cnt[u] = i1 > i0 ? (int)(i1 - i0) : 0;
    }
    mysum += cnt[u];
  }
  // block exclusive scan of the per-thread sums
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int incl = mysum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int woff = 0, total = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const int v = wsum[w]; if (w < warp) woff += v; total += v; }
  int run = woff + incl - mysum;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int sg = s0 + u;
    if (sg < nseg) seg_cum[sg] = run;
    run += cnt[u];
  }
  if (threadIdx.x == 0) seg_cum[nseg] = total;
  __syncthreads();
  // flattened node f -> row: a shared row map when it fits (2 x tile volume entries), filled
  // by a warp per segment; otherwise a binary search in seg_cum
  int* rows = seg_cum + nseg + 1;
  const bool mapped = total <= 2 * vol;
  if (mapped) {
    for (int sg = warp; sg < nseg; sg += (int)(blockDim.x >> 5)) {
      const int c0 = seg_cum[sg], cn = seg_cum[sg + 1] - c0, b0 = seg_beg[sg];
      for (int k = lane; k < cn; k += 32) rows[c0 + k] = b0 + k;
    }
    __syncthreads();
  }
  auto row_of = [&](int f) -> int64_t {
    if (mapped) return rows[f];
    int a = 0, b = nseg;                                   // seg_cum[a] <= f < seg_cum[b]
    while (b - a > 1) { const int m = (a + b) >> 1; if (seg_cum[m] <= f) a = m; else b = m; }
    return (int64_t)seg_beg[a] + (f - seg_cum[a]);
  };
  // sweep 1: max |q| over the halo nodes
  float qm = 0.f;
  for (int f = threadIdx.x; f < total; f += blockDim.x) qm = fmaxf(qm, fabsf(__ldg(q + row_of(f))));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
  if (lane == 0) atomicMax(&red_q, __float_as_int(qm));
  __syncthreads();
  const float qmax = __int_as_float(red_q);
  const int P3 = (P + 1) * (P + 1) * (P + 1);
  // power-of-two scale: 2 box_max (P+1)^3 qmax * scale <= 2^30
  const float scale = qmax > 0.f ? exp2f(floorf(log2f(1073741824.f / (2.f * (float)box_max * (float)P3 * qmax)))) : 0.f;
  // sweep 2: fixed-point scatter into the tile
  if (qmax > 0.f) {
    for (int f = threadIdx.x; f < total; f += blockDim.x) {
      const int64_t i = row_of(f);
      DCHECK(i >= lo && i < hi);
      const int4 s = __ldg(st_s + i);
      const float4 t = __ldg(st_t + i);
      const float qn = __ldg(q + i) * scale;
      float wx[P + 1], wy[P + 1], wz[P + 1];
      lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
      int lx[P + 1], ly[P + 1], lz[P + 1];
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        int a = wrapi(s.x + k, g.n0, g.per0) - x0; lx[k] = (a >= 0 && a < T0) ? a : -1;
        a = wrapi(s.y + k, g.n1, g.per1) - y0;     ly[k] = (a >= 0 && a < T1) ? a : -1;
        a = wrapi(s.z + k, g.n2, g.per2) - z0;     lz[k] = (a >= 0 && a < T2) ? a : -1;
      }
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        if (lz[k] < 0) continue;
#pragma unroll
        for (int j = 0; j <= P; ++j) {
          if (ly[j] < 0) continue;
          const float wzy = qn * wz[k] * wy[j];
          int* row = tile + (lz[k] * T1 + ly[j]) * T0;
#pragma unroll
          for (int l = 0; l <= P; ++l)
            if (lx[l] >= 0) atomicAdd(row + lx[l], __float2int_rn(wzy * wx[l]));
        }
      }
    }
  }
  __syncthreads();
  const float inv = qmax > 0.f ? 1.f / scale : 0.f;
  for (int i = threadIdx.x; i < vol; i += blockDim.x) {
    const int ix = i % T0, r = i / T0, iy = r % T1, iz = r / T1;
    Q[((int64_t)(z0 + iz) * g.n1 + (y0 + iy)) * g.n0 + x0 + ix] = (float)tile[i] * inv;
  }
}

// ------------------------------------------------------------------ K4 interpolation + precorrection
// G lanes per row (8, 16 or 32, chosen from the mean C_box row length so every lane has
// several loads in flight); the (P+1)^3 grid gathers are spread over the same lanes.  C_box
// is streamed in the C4x format (cbox_gpu.cu): per chunk one 16-byte value load and one
// 8-byte header (base column + three 12-bit deltas) -- consecutive lanes take consecutive
// chunks, so the q gathers of a lane group mostly hit the same few lines.
// F = 1: B4 blocks instead -- one 4-byte block index, one 16-byte value load and ONE aligned
// 16-byte q gather per block of 4 consecutive columns.
template <int P, int G, int F>
__global__ void __launch_bounds__(256) k4_interp_corr(RowRange rr, const float* __restrict__ U, const int4* __restrict__ st_s,
                                                      const float4* __restrict__ st_t, GridDims g,
                                                      const int64_t* __restrict__ c_ptr, const unsigned long long* __restrict__ c_hdr,
                                                      const int* __restrict__ c_bidx,
                                                      const float4* __restrict__ c_val4, const float* __restrict__ q,
                                                      const float* __restrict__ uloc, float* __restrict__ u, int64_t q4s) {
  const int lane = threadIdx.x & (G - 1);
  const int64_t n = rr.row0 + (int64_t)blockIdx.x * (blockDim.x / G) + (threadIdx.x / G);
  const bool valid = n < rr.row1;          // no early return: the group reduction needs every lane
  float acc = 0.f;
  const int64_t b = valid ? c_ptr[n - rr.row0] : 0, e_end = valid ? c_ptr[n - rr.row0 + 1] : 0;
  const float ul = (valid && lane == 0) ? uloc[n] : 0.f;
  // interpolation first (its stencil and grid loads overlap the C_box stream below): lane
  // r < (P+1)^2 takes one (y, z) stencil row and its P+1 x-consecutive grid values
  constexpr int NR = (P + 1) * (P + 1);
  if (valid && lane < NR) {
    const int4 s = st_s[n];
    const float4 t = st_t[n];
    float wx[P + 1], wy[P + 1], wz[P + 1];
    lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
    int ix[P + 1];
#pragma unroll
    for (int i = 0; i <= P; ++i) ix[i] = wrapi(s.x + i, g.n0, g.per0);
    for (int r = lane; r < NR; r += G) {
      const int jy = r % (P + 1), jz = r / (P + 1);
      float wyz = 0.f;
#pragma unroll
      for (int a = 0; a <= P; ++a)
#pragma unroll
        for (int b = 0; b <= P; ++b)
          if (a == jy && b == jz) wyz = wy[a] * wz[b];
      DCHECK(wrapi(s.z + jz, g.n2, g.per2) < g.n2 && wrapi(s.y + jy, g.n1, g.per1) < g.n1 && ix[0] >= 0 && ix[P] < g.n0);
      const float* row = U + ((int64_t)wrapi(s.z + jz, g.n2, g.per2) * g.n1 + wrapi(s.y + jy, g.n1, g.per1)) * g.n0;
      float v = 0.f;
#pragma unroll
      for (int i = 0; i <= P; ++i) v = fmaf(wx[i], __ldg(row + ix[i]), v);
      acc = fmaf(wyz, v, acc);
    }
  }
  if (F == 1 || F == 3) {
    // B4: block index b, q4 = q viewed as float4 (aligned [4b, 4b+4)); U4: start column c, q4 =
    // the per-evaluation shifted copies q4x (passed in place of q), word (c & 3) * q4s + (c >> 2)
    const float4* q4 = reinterpret_cast<const float4*>(q);
    // explicitly batched: the U block indices and values of KB blocks per lane are loaded first
    // (independent), then their KB q gathers -- the gather depends on its index, so without the
    // batching every block paid two dependent memory round trips (ncu: 80 % long-scoreboard)
    constexpr int KB = 4;
    for (int64_t base = b + lane; base < e_end; base += KB * G) {
      int bi[KB];
      float4 vv[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int64_t e = base + (int64_t)j * G;
        const bool ok = e < e_end;
        bi[j] = ok ? __ldg(c_bidx + e) : 0;
        vv[j] = ok ? __ldg(c_val4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        DCHECK(bi[j] >= 0 && (F == 3 ? bi[j] < rr.ncol : 4 * (int64_t)bi[j] < rr.ncol + 4));
        const float4 qq = __ldg(q4 + (F == 3 ? (int64_t)(bi[j] & 3) * q4s + (bi[j] >> 2) : (int64_t)bi[j]));
        acc = fmaf(vv[j].x, qq.x, fmaf(vv[j].y, qq.y, fmaf(vv[j].z, qq.z, fmaf(vv[j].w, qq.w, acc))));
      }
    }
  } else if (F == 2) {
    // C4x with vector gathers for run chunks (deltas 1,1,1): the 4 consecutive q values come
    // from one or two aligned 16-byte loads instead of four scalar ones
    const float4* q4 = reinterpret_cast<const float4*>(q);
#pragma unroll 2
    for (int64_t e = b + lane; e < e_end; e += G) {
      const unsigned long long h = __ldg(c_hdr + e);
      const float4 vv = __ldg(c_val4 + e);
      const int k0 = (int)(h & 0xFFFFFFFull);
      float a0, a1, a2, a3;
      if ((h >> 28) == 0x001001001ull) {
        const int o = k0 & 3;
        const float4 lo = __ldg(q4 + (k0 >> 2));
        float4 hi = lo;
        if (o) hi = __ldg(q4 + (k0 >> 2) + 1);
        a0 = o == 0 ? lo.x : o == 1 ? lo.y : o == 2 ? lo.z : lo.w;
        a1 = o == 0 ? lo.y : o == 1 ? lo.z : o == 2 ? lo.w : hi.x;
        a2 = o == 0 ? lo.z : o == 1 ? lo.w : o == 2 ? hi.x : hi.y;
        a3 = o == 0 ? lo.w : o == 1 ? hi.x : o == 2 ? hi.y : hi.z;
      } else {
        const int k1 = k0 + (int)((h >> 28) & 0xFFF);
        const int k2 = k1 + (int)((h >> 40) & 0xFFF);
        const int k3 = k2 + (int)(h >> 52);
        a0 = __ldg(q + k0); a1 = __ldg(q + k1); a2 = __ldg(q + k2); a3 = __ldg(q + k3);
      }
      acc = fmaf(vv.x, a0, fmaf(vv.y, a1, fmaf(vv.z, a2, fmaf(vv.w, a3, acc))));
    }
  } else {
    // C4x, batched like B4/U4: KB headers + values first, then their 4 KB scalar gathers
    // (F = 4: KB = 4, the default since round 2 call 29 -- fewer dependent round trips per row; PMFEM_K4_KB=2 for F = 0)
    constexpr int KB = F == 4 ? 4 : 2;
    for (int64_t base = b + lane; base < e_end; base += KB * G) {
      unsigned long long h[KB];
      float4 vv[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int64_t e = base + (int64_t)j * G;
        const bool ok = e < e_end;
        h[j] = ok ? __ldg(c_hdr + e) : 0ull;
        vv[j] = ok ? __ldg(c_val4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k0 = (int)(h[j] & 0xFFFFFFFull);
        const int k1 = k0 + (int)((h[j] >> 28) & 0xFFF);
        const int k2 = k1 + (int)((h[j] >> 40) & 0xFFF);
        const int k3 = k2 + (int)(h[j] >> 52);
        DCHECK(k0 >= 0 && k3 < rr.ncol && k0 <= k1 && k1 <= k2 && k2 <= k3);
        acc = fmaf(vv[j].x, __ldg(q + k0), acc);
        acc = fmaf(vv[j].y, __ldg(q + k1), acc);
        acc = fmaf(vv[j].z, __ldg(q + k2), acc);
        acc = fmaf(vv[j].w, __ldg(q + k3), acc);
      }
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (valid && lane == 0) u[n] = acc + ul;
}

// K4 over the W4 C_box (cbox_format 5, cbox_gpu.cu): ONE CTA PER TILE of consecutive rows of
// one anchor line.  Staged once per tile in shared memory:
//  * the q window -- the rows of every anchor box within the candidate reach of the tile, as
//    runs of consecutive internal rows (a warp per run);
//  * the U sub-grid of the tile's stencils -- the rows share the (y, z) anchor, so their
//    (P+1)^3 stencils lie in (P+1)^2 grid lines over x in [xa, xb + P] (xa, xb the first and
//    last row's x anchor), stored with an odd line pitch (distinct banks across the lines).
// The C_box chunks (float4 values + ushort4 window-local indices, 24 bytes per 4 entries) then
// stream from HBM and every gather -- q and U -- hits shared memory: the global-index formats
// were L1-request bound (ncu C4 C4x: L1 hit 77 %, DRAM 49-61 % of peak), and the (P+1)^2
// scattered U line gathers per row were as many L1 wavefronts as the q gathers.  G lanes per
// row as k4_interp_corr; rows of the tile in passes of 256 / G.
template <int P, int G, int KB>
__global__ void __launch_bounds__(256) k4_win(RowRange rr, const float* __restrict__ U, const int4* __restrict__ st_s,
                                              const float4* __restrict__ st_t, GridDims g,
                                              const int64_t* __restrict__ tile_row, const int* __restrict__ run_ptr,
                                              const int* __restrict__ run_start, const int* __restrict__ run_len,
                                              const int* __restrict__ run_loc, const int64_t* __restrict__ c_ptr,
                                              const float4* __restrict__ c_val4, const ushort4* __restrict__ c_idx,
                                              const float* __restrict__ q, const float* __restrict__ uloc,
                                              float* __restrict__ u, int wmax, int umax) {
  extern __shared__ float qs[];
  float* us = qs + wmax;
  __shared__ int64_t cp[W4_TMAX + 1];     // the tile's chunk offsets (no dependent load per row)
  constexpr int NR = (P + 1) * (P + 1);
  const int t = blockIdx.x;
  const int64_t row0 = tile_row[t], row1 = tile_row[t + 1];
  DCHECK(row1 - row0 <= W4_TMAX);
  for (int i = threadIdx.x; i <= (int)(row1 - row0); i += blockDim.x) cp[i] = c_ptr[row0 - rr.row0 + i];
  const int4 sa = st_s[row0];
  const int xa = sa.x, nxs = st_s[row1 - 1].x - xa + P + 1, pitch = nxs | 1;
  DCHECK(pitch * NR <= umax);
  {
    // a warp per run (measured faster than a flattened copy with a per-element run search, and
    // than staging every per-row operand in shared memory: both cost registers / occupancy)
    const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
    for (int r = run_ptr[t] + warp; r < run_ptr[t + 1]; r += blockDim.x >> 5) {
      const int s0 = run_start[r], len = run_len[r], loc = run_loc[r];
      DCHECK(loc >= 0 && loc + len <= wmax && s0 >= 0 && s0 + len <= rr.ncol);
      for (int j = l32; j < len; j += 32) qs[loc + j] = __ldg(q + s0 + j);
    }
    for (int i = threadIdx.x; i < nxs * NR; i += blockDim.x) {
      const int ix = i % nxs, l = i / nxs, jy = l % (P + 1), jz = l / (P + 1);
      us[l * pitch + ix] = __ldg(U + ((int64_t)wrapi(sa.z + jz, g.n2, g.per2) * g.n1 + wrapi(sa.y + jy, g.n1, g.per1)) * g.n0 +
                                wrapi(xa + ix, g.n0, g.per0));
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & (G - 1);
  for (int64_t base = row0; base < row1; base += 256 / G) {
    const int64_t n = base + (threadIdx.x / G);
    const bool valid = n < row1;
    float acc = 0.f;
    const int64_t b = valid ? cp[n - row0] : 0, e_end = valid ? cp[n - row0 + 1] : 0;
    const float ul = (valid && lane == 0) ? uloc[n] : 0.f;
    if (valid && lane < NR) {
      const int sx = st_s[n].x - xa;
      const float4 tt = st_t[n];
      float wx[P + 1], wy[P + 1], wz[P + 1];
      lagr<P>(tt.x, wx); lagr<P>(tt.y, wy); lagr<P>(tt.z, wz);
      for (int r = lane; r < NR; r += G) {
        const int jy = r % (P + 1), jz = r / (P + 1);
        float wyz = 0.f;
#pragma unroll
        for (int a = 0; a <= P; ++a)
#pragma unroll
          for (int c = 0; c <= P; ++c)
            if (a == jy && c == jz) wyz = wy[a] * wz[c];
        const float* row = us + r * pitch + sx;
        float v = 0.f;
#pragma unroll
        for (int i = 0; i <= P; ++i) v = fmaf(wx[i], row[i], v);
        acc = fmaf(wyz, v, acc);
      }
    }
    // KB chunks per lane in flight: the whole row's loads at once for rows of <= KB * G chunks
    for (int64_t e0 = b + lane; e0 < e_end; e0 += KB * G) {
      ushort4 id[KB];
      float4 vv[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int64_t e = e0 + (int64_t)j * G;
        const bool ok = e < e_end;
        id[j] = ok ? __ldcs(c_idx + e) : make_ushort4(0, 0, 0, 0);
        vv[j] = ok ? __ldcs(c_val4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        DCHECK(id[j].x < wmax && id[j].y < wmax && id[j].z < wmax && id[j].w < wmax);
        acc = fmaf(vv[j].x, qs[id[j].x], fmaf(vv[j].y, qs[id[j].y], fmaf(vv[j].z, qs[id[j].z], fmaf(vv[j].w, qs[id[j].w], acc))));
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (valid && lane == 0) u[n] = acc + ul;
  }
}

// W4 with the tile's whole chunk block (values and indices, <= W4_CCAP chunks) copied into shared
// memory by the bulk-copy engine (cp.async.bulk, one mbarrier with the byte count): the HBM stream
// no longer waits on any per-row dependency -- the copy is issued first, the q window and the U
// sub-grid are staged by the threads meanwhile, and the rows then read everything from shared
// memory (PMFEM_W4_TMA=1).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(phase) : "memory");
  }
}

template <int P, int G>
__global__ void __launch_bounds__(256) k4_win_tma(RowRange rr, const float* __restrict__ U, const int4* __restrict__ st_s,
                                                  const float4* __restrict__ st_t, GridDims g,
                                                  const int64_t* __restrict__ tile_row, const int* __restrict__ run_ptr,
                                                  const int* __restrict__ run_start, const int* __restrict__ run_len,
                                                  const int* __restrict__ run_loc, const int64_t* __restrict__ c_ptr,
                                                  const float4* __restrict__ c_val4, const ushort4* __restrict__ c_idx,
                                                  const float* __restrict__ q, const float* __restrict__ uloc,
                                                  float* __restrict__ u, int wmax, int umax) {
  extern __shared__ __align__(16) unsigned char w4t_smem[];
  float4* vs = reinterpret_cast<float4*>(w4t_smem);                       // [W4_CCAP]
  ushort4* is = reinterpret_cast<ushort4*>(vs + W4_CCAP);                 // [W4_CCAP]
  float* qs = reinterpret_cast<float*>(is + W4_CCAP);                     // [wmax]
  float* us = qs + wmax;                                                  // [umax]
  __shared__ __align__(8) uint64_t bar;
  __shared__ int64_t cp[W4_TMAX + 1];
  constexpr int NR = (P + 1) * (P + 1);
  const int t = blockIdx.x;
  const int64_t row0 = tile_row[t], row1 = tile_row[t + 1];
  const int64_t ce0 = c_ptr[row0 - rr.row0] & ~(int64_t)1;               // even: 16-byte aligned index block
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t ce1 = c_ptr[row1 - rr.row0];
    const unsigned nch = (unsigned)((ce1 - ce0 + 1) & ~(int64_t)1);
    DCHECK(nch <= W4_CCAP);
    mbar_expect_tx(&bar, nch * 24u);
    bulk_g2s(vs, c_val4 + ce0, nch * 16u, &bar);
    bulk_g2s(is, c_idx + ce0, nch * 8u, &bar);
  }
  for (int i = threadIdx.x; i <= (int)(row1 - row0); i += blockDim.x) cp[i] = c_ptr[row0 - rr.row0 + i] - ce0;
  const int4 sa = st_s[row0];
  const int xa = sa.x, nxs = st_s[row1 - 1].x - xa + P + 1, pitch = nxs | 1;
  DCHECK(pitch * NR <= umax);
  {
    const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
    for (int r = run_ptr[t] + warp; r < run_ptr[t + 1]; r += blockDim.x >> 5) {
      const int s0 = run_start[r], len = run_len[r], loc = run_loc[r];
      DCHECK(loc >= 0 && loc + len <= wmax && s0 >= 0 && s0 + len <= rr.ncol);
      for (int j = l32; j < len; j += 32) qs[loc + j] = __ldg(q + s0 + j);
    }
    for (int i = threadIdx.x; i < nxs * NR; i += blockDim.x) {
      const int ix = i % nxs, l = i / nxs, jy = l % (P + 1), jz = l / (P + 1);
      us[l * pitch + ix] = __ldg(U + ((int64_t)wrapi(sa.z + jz, g.n2, g.per2) * g.n1 + wrapi(sa.y + jy, g.n1, g.per1)) * g.n0 +
                                wrapi(xa + ix, g.n0, g.per0));
    }
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int lane = threadIdx.x & (G - 1);
  for (int64_t base = row0; base < row1; base += 256 / G) {
    const int64_t n = base + (threadIdx.x / G);
    const bool valid = n < row1;
    float acc = 0.f;
    const int b = valid ? (int)cp[n - row0] : 0, e_end = valid ? (int)cp[n - row0 + 1] : 0;
    const float ul = (valid && lane == 0) ? uloc[n] : 0.f;
    if (valid && lane < NR) {
      const int sx = st_s[n].x - xa;
      const float4 tt = st_t[n];
      float wx[P + 1], wy[P + 1], wz[P + 1];
      lagr<P>(tt.x, wx); lagr<P>(tt.y, wy); lagr<P>(tt.z, wz);
      for (int r = lane; r < NR; r += G) {
        const int jy = r % (P + 1), jz = r / (P + 1);
        float wyz = 0.f;
#pragma unroll
        for (int a = 0; a <= P; ++a)
#pragma unroll
          for (int c = 0; c <= P; ++c)
            if (a == jy && c == jz) wyz = wy[a] * wz[c];
        const float* row = us + r * pitch + sx;
        float v = 0.f;
#pragma unroll
        for (int i = 0; i <= P; ++i) v = fmaf(wx[i], row[i], v);
        acc = fmaf(wyz, v, acc);
      }
    }
#pragma unroll 4
    for (int e = b + lane; e < e_end; e += G) {
      const ushort4 id = is[e];
      const float4 vv = vs[e];
      DCHECK(id.x < wmax && id.y < wmax && id.z < wmax && id.w < wmax);
      acc = fmaf(vv.x, qs[id.x], fmaf(vv.y, qs[id.y], fmaf(vv.z, qs[id.z], fmaf(vv.w, qs[id.w], acc))));
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (valid && lane == 0) u[n] = acc + ul;
  }
}

// K4 "stream" variant for the block formats (B4: F = 1, U4: F = 3), PMFEM_K4_STREAM=1: a warp
// owns RPW consecutive rows and streams their C_box blocks as ONE contiguous range
// [c_ptr[r0], c_ptr[r0 + RPW]) -- 32 consecutive blocks per step, KB steps of index/value loads
// issued before their gathers -- regardless of where the rows break.  Each lane finds its block's
// row with a cursor over c_ptr (rows hold ~100-300 blocks, so it rarely moves); per step the
// lanes' block partials are reduced by row with a segmented warp scan (rows are non-decreasing
// across the lanes) and the tail lane of each segment adds the sum to the row's shared-memory
// accumulator (one writer per row per step: no atomics).  Then the interpolation P^T U of the
// warp's rows, 32 / LR rows at a time (LR = lanes per row >= (P+1)^2 stencil rows).
template <int P, int F>
__global__ void __launch_bounds__(256) k4_stream(RowRange rr, const float* __restrict__ U, const int4* __restrict__ st_s,
                                                 const float4* __restrict__ st_t, GridDims g,
                                                 const int64_t* __restrict__ c_ptr, const int* __restrict__ c_bidx,
                                                 const float4* __restrict__ c_val4, const float* __restrict__ q,
                                                 const float* __restrict__ uloc, float* __restrict__ u, int64_t q4s) {
  constexpr int RPW = 64, KB = 4;
  constexpr int NR = (P + 1) * (P + 1);
  constexpr int LR = NR <= 4 ? 4 : (NR <= 8 ? 8 : (NR <= 16 ? 16 : 32));
  __shared__ float sacc[8][RPW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r0 = rr.row0 + ((int64_t)blockIdx.x * 8 + wid) * RPW;
  if (r0 >= rr.row1) return;                               // whole warp: uniform
  const int nr = (int)(rr.row1 - r0 < RPW ? rr.row1 - r0 : RPW);
  for (int i = lane; i < RPW; i += 32) sacc[wid][i] = 0.f;
  __syncwarp();
  const int64_t* cp = c_ptr + (r0 - rr.row0);
  const int64_t e0 = cp[0], e1 = cp[nr];
  const float4* q4 = reinterpret_cast<const float4*>(q);
  int row = 0;                                             // local row of the lane's current block
  for (int64_t base = e0; base < e1; base += 32 * KB) {
    int bi[KB];
    float4 vv[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int64_t e = base + (int64_t)j * 32 + lane;
      const bool ok = e < e1;
      bi[j] = ok ? __ldg(c_bidx + e) : 0;
      vv[j] = ok ? __ldg(c_val4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int64_t e = base + (int64_t)j * 32 + lane;
      const bool ok = e < e1;
      DCHECK(!ok || (bi[j] >= 0 && (F == 3 ? bi[j] < rr.ncol : 4 * (int64_t)bi[j] < rr.ncol + 4)));
      const float4 qq = ok ? __ldg(q4 + (F == 3 ? (int64_t)(bi[j] & 3) * q4s + (bi[j] >> 2) : (int64_t)bi[j]))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      float p = vv[j].x * qq.x + vv[j].y * qq.y + vv[j].z * qq.z + vv[j].w * qq.w;
      if (ok) while (cp[row + 1] <= e) ++row;
      const int key = ok ? row : RPW;                      // out-of-range lanes form their own segment
      // segmented inclusive scan by row (rows non-decreasing across lanes)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float pu = __shfl_up_sync(0xffffffffu, p, o);
        const int ku = __shfl_up_sync(0xffffffffu, key, o);
        if (lane >= o && ku == key) p += pu;
      }
      const int kn = __shfl_down_sync(0xffffffffu, key, 1);
      if (key < RPW && (lane == 31 || kn != key)) sacc[wid][key] += p;
    }
  }
  __syncwarp();
  // interpolation + u_loc + store, 32 / LR rows at a time
  const int sub = lane / LR, sl = lane % LR;
  for (int rb = 0; rb < nr; rb += 32 / LR) {
    const int lr = rb + sub;
    const bool valid = lr < nr;
    const int64_t n = r0 + lr;
    float acc = 0.f;
    if (valid && sl < NR) {
      const int4 s = st_s[n];
      const float4 t = st_t[n];
      float wx[P + 1], wy[P + 1], wz[P + 1];
      lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
      const int jy = sl % (P + 1), jz = sl / (P + 1);
      float wyz = 0.f;
#pragma unroll
      for (int a = 0; a <= P; ++a)
#pragma unroll
        for (int c = 0; c <= P; ++c)
          if (a == jy && c == jz) wyz = wy[a] * wz[c];
      const float* rowp = U + ((int64_t)wrapi(s.z + jz, g.n2, g.per2) * g.n1 + wrapi(s.y + jy, g.n1, g.per1)) * g.n0;
      float v = 0.f;
#pragma unroll
      for (int i = 0; i <= P; ++i) v = fmaf(wx[i], __ldg(rowp + wrapi(s.x + i, g.n0, g.per0)), v);
      acc = wyz * v;
    }
#pragma unroll
    for (int o = LR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (valid && sl == 0) u[n] = acc + sacc[wid][lr] + uloc[n];
  }
}

// K4 over the SEG C_box (cbox_format 2, device.cuh): G lanes per row.  The lanes first build the
// row's table of column runs in shared memory -- one run per (z, y) candidate anchor line and x
// subrange, [box_ptr(line + xa), box_ptr(line + xb + 1)) -- with an exclusive scan of the run
// lengths; then per 32-candidate mask word each lane takes candidates sub * G + lane: a set bit
// selects the next stored value (rank = popcount of the lower bits) and q at the candidate's
// column, found by a per-lane cursor over the runs (candidates are visited in increasing order).
// No column indices are streamed and the q reads walk contiguous runs.
template <int P, int G>
__global__ void __launch_bounds__(256) k4_seg(RowRange rr, const float* __restrict__ U, const int4* __restrict__ st_s,
                                              const float4* __restrict__ st_t, GridDims g, SegGeom sg, int maxseg,
                                              const int* __restrict__ box_ptr, const int64_t* __restrict__ moff,
                                              const int64_t* __restrict__ voff, const uint32_t* __restrict__ mask,
                                              const float* __restrict__ val, const float* __restrict__ q,
                                              const float* __restrict__ uloc, float* __restrict__ u) {
  extern __shared__ int k4s_smem[];
  const int lane = threadIdx.x & (G - 1);
  const int grp = threadIdx.x / G;
  int* beg = k4s_smem + grp * (2 * maxseg + 2);
  int* cum = beg + maxseg;                    // maxseg + 1 entries
  const int64_t n = rr.row0 + (int64_t)blockIdx.x * (blockDim.x / G) + grp;
  const bool valid = n < rr.row1;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1) << ((threadIdx.x & 31) & ~(G - 1)));
  float acc = 0.f;
  int4 s = make_int4(0, 0, 0, 0);
  if (valid) s = st_s[n];
  // ---- runs of candidate columns
  int rz[4], ry[4], rx[4];
  const int nz = seg_axis(sg, 2, s.z, rz), ny = seg_axis(sg, 1, s.y, ry), nx = seg_axis(sg, 0, s.x, rx);
  const int lz = seg_len(rz, nz), ly = seg_len(ry, ny);
  const int nseg = valid ? lz * ly * nx : 0;
  int carry = 0;
  for (int b0 = 0; b0 < nseg; b0 += G) {
    const int sgi = b0 + lane;
    int len = 0;
    if (sgi < nseg) {
      const int xi = sgi % nx, li = sgi / nx;
      const int z = seg_at(rz, li / ly), y = seg_at(ry, li - (li / ly) * ly);
      const int64_t line = ((int64_t)z * g.n1 + y) * g.n0;
      const int k0 = __ldg(box_ptr + line + rx[2 * xi]), k1 = __ldg(box_ptr + line + rx[2 * xi + 1] + 1);
      beg[sgi] = k0;
      len = k1 - k0;
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int v = __shfl_up_sync(gmask, incl, o, G);
      if (lane >= o) incl += v;
    }
    if (sgi < nseg) cum[sgi] = carry + incl - len;
    carry += __shfl_sync(gmask, incl, G - 1, G);
  }
  if (lane == 0) cum[nseg] = carry;
  __syncwarp();
  const int ncand = carry;
  // ---- masked candidate loop
  if (valid && ncand > 0) {
    const uint32_t* M = mask + moff[n - rr.row0];
    const float* V = val + voff[n - rr.row0];
    const int nwords = (ncand + 31) >> 5;
    int base = 0, sidx = 0;
    for (int w = 0; w < nwords; ++w) {
      const uint32_t word = __ldg(M + w);
#pragma unroll
      for (int sub = 0; sub < 32 / G; ++sub) {
        const int bp = sub * G + lane;
        if ((word >> bp) & 1u) {
          const int c = (w << 5) + bp;
          while (cum[sidx + 1] <= c) ++sidx;
          const int k = beg[sidx] + (c - cum[sidx]);
          acc = fmaf(__ldg(V + base + __popc(word & ((1u << bp) - 1u))), __ldg(q + k), acc);
        }
      }
      base += __popc(word);
    }
  }
  // ---- interpolation P^T U (as k4_interp_corr)
  constexpr int NR = (P + 1) * (P + 1);
  if (valid) {
    const float4 t = st_t[n];
    float wx[P + 1], wy[P + 1], wz[P + 1];
    lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
    int ix[P + 1];
#pragma unroll
    for (int i = 0; i <= P; ++i) ix[i] = wrapi(s.x + i, g.n0, g.per0);
    for (int r = lane; r < NR; r += G) {
      const int jy = r % (P + 1), jz = r / (P + 1);
      float wyz = 0.f;
#pragma unroll
      for (int a = 0; a <= P; ++a)
#pragma unroll
        for (int b = 0; b <= P; ++b)
          if (a == jy && b == jz) wyz = wy[a] * wz[b];
      const float* row = U + ((int64_t)wrapi(s.z + jz, g.n2, g.per2) * g.n1 + wrapi(s.y + jy, g.n1, g.per1)) * g.n0;
      float v = 0.f;
#pragma unroll
      for (int i = 0; i <= P; ++i) v = fmaf(wx[i], __ldg(row + ix[i]), v);
      acc = fmaf(wyz, v, acc);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (valid && lane == 0) u[n] = acc + uloc[n];
}

// U4 C_box: four shifted float4 copies of q, q4x[r * S + k] = (q[4k+r], .., q[4k+r+3]), so the
// q of the block starting at column c is q4x[(c & 3) * S + (c >> 2)] and consecutive blocks of a
// run of columns (c, c+4, ..) read consecutive 16-byte words -- as dense as B4's aligned gathers
// (a single copy q4[c] would put them 64 bytes apart).  q carries 16 trailing zeros.
__global__ void k_q4(int64_t S, const float* __restrict__ q, float4* __restrict__ q4x) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * S) return;
  const int64_t r = t / S, k = t - r * S, i = 4 * k + r;
  q4x[t] = make_float4(q[i], q[i + 1], q[i + 2], q[i + 3]);
}

// ------------------------------------------------------------------ K5 gradient + sum
template <int SPLIT>
__global__ void __launch_bounds__(256) k5_grad_sum(RowRange rr, const float* __restrict__ u, const int64_t* __restrict__ sl1_off,
                                                   const float4* __restrict__ s_Gc, float* __restrict__ H, int accumulate) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t n;
  int part;
  if (SPLIT == 1) { n = rr.row0 + gid; part = 0; }
  else { n = rr.row0 + (gid >> 6) * 32 + ((gid >> 5) & 1) * 16 + (threadIdx.x & 15); part = (threadIdx.x >> 4) & 1; }
  const bool valid = n < rr.row1;
  if (SPLIT == 1 && !valid) return;
  const int64_t s = (n - rr.row0) >> 5;
  const int l = (int)((n - rr.row0) & 31);
  int64_t o1 = 0;
  int w1 = 0;
  float un = 0.f;
  if (valid) { o1 = sl1_off[s]; w1 = (int)((sl1_off[s + 1] - o1) >> 5); un = u[n]; }
  float gx = 0.f, gy = 0.f, gz = 0.f;
  int64_t e1 = o1 + l + 32 * part;
#pragma unroll 4
  for (int j = part; j < w1; j += SPLIT, e1 += 32 * SPLIT) {
    const float4 gc = ld_stream(s_Gc + e1);
    DCHECK(colof(gc) >= 0 && colof(gc) < rr.ncol);
    const float du = u[colof(gc)] - un;
    gx = fmaf(gc.x, du, gx); gy = fmaf(gc.y, du, gy); gz = fmaf(gc.z, du, gz);
  }
  if (SPLIT == 2) {
    gx += __shfl_xor_sync(0xffffffffu, gx, 16); gy += __shfl_xor_sync(0xffffffffu, gy, 16);
    gz += __shfl_xor_sync(0xffffffffu, gz, 16);
    if (part) return;
  }
  if (!valid) return;
  if (accumulate) {
    H[3 * (n - rr.hoff) + rr.c0] -= gx; H[3 * (n - rr.hoff) + rr.c1] -= gy; H[3 * (n - rr.hoff) + rr.c2] -= gz;
  } else {
    H[3 * (n - rr.hoff) + rr.c0] = -gx; H[3 * (n - rr.hoff) + rr.c1] = -gy; H[3 * (n - rr.hoff) + rr.c2] = -gz;
  }
}

// ------------------------------------------------------------------ LLG RK4 stage (NEXT-2)
// dm/dt = -g [ m x H + alpha m x (m x H) ], g = gamma / (1 + alpha^2)   (Eq. llg)
// Stage s of classical RK4: k = f(ms, H + H_ap + H_an(ms)); acc (+)= w_s dt k; next stage state
// m0 + c_{s+1} dt k, or (last stage) m0 <- normalize(m0 + acc).  Rank-local rows.
struct Anis { int kind; float hk; float ux, uy, uz; };   // hk = 2 K / Ms (NEXT-2)

// H_an of the unit vector (sx, sy, sz) (oracle/llg.py anisotropy_field): uniaxial (2K/Ms)(m.u)u,
// cubic -(2K/Ms)(mx(my^2+mz^2), my(mz^2+mx^2), mz(mx^2+my^2))
__device__ __forceinline__ void anis_field(const Anis& a, float sx, float sy, float sz, float& hx, float& hy, float& hz) {
  if (a.kind == 1) {
    const float d = a.hk * (sx * a.ux + sy * a.uy + sz * a.uz);
    hx += d * a.ux; hy += d * a.uy; hz += d * a.uz;
  } else if (a.kind == 2) {
    const float x2 = sx * sx, y2 = sy * sy, z2 = sz * sz;
    hx -= a.hk * sx * (y2 + z2); hy -= a.hk * sy * (z2 + x2); hz -= a.hk * sz * (x2 + y2);
  }
}

// dm/dt = -g [m x H + alpha m x (m x H)]
__device__ __forceinline__ void llg_f(float sx, float sy, float sz, float Hx, float Hy, float Hz, float g, float alpha,
                                      float& kx, float& ky, float& kz) {
  const float cx = sy * Hz - sz * Hy, cy = sz * Hx - sx * Hz, cz = sx * Hy - sy * Hx;        // m x H
  const float dx = sy * cz - sz * cy, dy = sz * cx - sx * cz, dz = sx * cy - sy * cx;        // m x (m x H)
  kx = -g * (cx + alpha * dx); ky = -g * (cy + alpha * dy); kz = -g * (cz + alpha * dz);
}

__global__ void k_llg_stage(int64_t n, float* __restrict__ m0, const float* __restrict__ ms,
                            const float* __restrict__ H, float hx, float hy, float hz, Anis an, float g, float alpha,
                            float wdt, float cnext_dt, float* __restrict__ acc, float* __restrict__ mnext,
                            int first, int last) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float sx = ms[3 * i], sy = ms[3 * i + 1], sz = ms[3 * i + 2];
  float Hx = H[3 * i] + hx, Hy = H[3 * i + 1] + hy, Hz = H[3 * i + 2] + hz;
  anis_field(an, sx, sy, sz, Hx, Hy, Hz);
  float kx, ky, kz;
  llg_f(sx, sy, sz, Hx, Hy, Hz, g, alpha, kx, ky, kz);
  float ax = wdt * kx, ay = wdt * ky, az = wdt * kz;
  if (!first) { ax += acc[3 * i]; ay += acc[3 * i + 1]; az += acc[3 * i + 2]; }
  const float m0x = m0[3 * i], m0y = m0[3 * i + 1], m0z = m0[3 * i + 2];
  if (!last) {
    acc[3 * i] = ax; acc[3 * i + 1] = ay; acc[3 * i + 2] = az;
    mnext[3 * i] = m0x + cnext_dt * kx; mnext[3 * i + 1] = m0y + cnext_dt * ky; mnext[3 * i + 2] = m0z + cnext_dt * kz;
  } else {
    const float nx = m0x + ax, ny = m0y + ay, nz = m0z + az;
    const float inv = rsqrtf(nx * nx + ny * ny + nz * nz);
    m0[3 * i] = nx * inv; m0[3 * i + 1] = ny * inv; m0[3 * i + 2] = nz * inv;
  }
}

// ---- AM2 predictor-corrector (oracle/llg.py am2_step)
// f = dm/dt at (m, H + H_ap + H_an(m))
__global__ void k_llg_rhs(int64_t n, const float* __restrict__ m, const float* __restrict__ H, float hx, float hy,
                          float hz, Anis an, float g, float alpha, float* __restrict__ f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float sx = m[3 * i], sy = m[3 * i + 1], sz = m[3 * i + 2];
  float Hx = H[3 * i] + hx, Hy = H[3 * i + 1] + hy, Hz = H[3 * i + 2] + hz;
  anis_field(an, sx, sy, sz, Hx, Hy, Hz);
  llg_f(sx, sy, sz, Hx, Hy, Hz, g, alpha, f[3 * i], f[3 * i + 1], f[3 * i + 2]);
}
// predictor m_p = m + dt [(1 + r/2) f_n - (r/2) f_prev]  (r = 0: forward Euler)
__global__ void k_am2_pred(int64_t n, const float* __restrict__ m, const float* __restrict__ fn,
                           const float* __restrict__ fprev, float dt, float r, float* __restrict__ mp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  mp[i] = m[i] + dt * ((1.f + 0.5f * r) * fn[i] - (r > 0.f ? 0.5f * r * fprev[i] : 0.f));
}
// corrector m_c = m + dt/2 (f_n + f_p), normalised into mc; err = max |m_c - m_p| / 6 (float bits)
__global__ void k_am2_corr(int64_t n, const float* __restrict__ m, const float* __restrict__ fn,
                           const float* __restrict__ fp, const float* __restrict__ mp, float dt,
                           float* __restrict__ mc, unsigned* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float e = 0.f;
  if (i < n) {
    float c[3];
    for (int k = 0; k < 3; ++k) c[k] = m[3 * i + k] + 0.5f * dt * (fn[3 * i + k] + fp[3 * i + k]);
    const float ex = c[0] - mp[3 * i], ey = c[1] - mp[3 * i + 1], ez = c[2] - mp[3 * i + 2];
    e = sqrtf(ex * ex + ey * ey + ez * ez) / 6.f;
    const float inv = rsqrtf(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    for (int k = 0; k < 3; ++k) mc[3 * i + k] = c[k] * inv;
  }
  for (int o = 16; o > 0; o >>= 1) e = fmaxf(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0) atomicMax(err, __float_as_uint(e));   // e >= 0: bit order = value order
}

// ------------------------------------------------------------------ PGF table (fp64)
// One thread per point of the octant j_a in [0, P_a/2]; the value is written to every mirror
// position j_a and P_a - j_a (K is even on each axis: lattice reflection symmetry + periodicity
// on periodic axes, K(2N - j) = G(-(2N - j) Delta) on padded axes), so K is exactly symmetric
// and its spectrum exactly real.
__global__ void k_pgf_table(PgfDev pd, int P0, int P1, int P2, int n0, int n1, int n2, int per0, int per1, int per2,
                            double d0, double d1, double d2, double* __restrict__ K) {
  const int Q0 = P0 / 2 + 1, Q1 = P1 / 2 + 1, Q2 = P2 / 2 + 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)Q0 * Q1 * Q2) return;
  const int j0 = (int)(idx % Q0), j1 = (int)((idx / Q0) % Q1), j2 = (int)(idx / ((int64_t)Q0 * Q1));
  double v;
  // K6: j -> j Delta (j <= P/2 here); on a padded axis j = n -> value 0 (never used)
  if ((!per0 && j0 == n0) || (!per1 && j1 == n1) || (!per2 && j2 == n2)) {
    v = 0.0;
  } else {
    const double r[3] = {j0 * d0, j1 * d1, j2 * d2};
    v = pgf_eval(pd, r, j0 == 0 && j1 == 0 && j2 == 0);
  }
  const int a0[2] = {j0, P0 - j0}, a1[2] = {j1, P1 - j1}, a2[2] = {j2, P2 - j2};
  for (int z = 0; z < ((j2 > 0 && P2 - j2 != j2) ? 2 : 1); ++z)
    for (int y = 0; y < ((j1 > 0 && P1 - j1 != j1) ? 2 : 1); ++y)
      for (int x = 0; x < ((j0 > 0 && P0 - j0 != j0) ? 2 : 1); ++x)
        K[((int64_t)a2[z] * P1 + a1[y]) * P0 + a0[x]] = v;
}

// NEXT-4: modulated Bloch kernel exp(j k0.r) G(r; k0) (pgf.cuh pgf_eval_bloch) at every padded
// grid displacement, fp64 complex interleaved; one thread per point (no mirror symmetry)
struct K0v { double k[3]; };
__global__ void k_pgf_table_bloch(PgfDev pd, K0v k0, int P0, int P1, int P2, int n0, int n1, int n2, int per0,
                                  int per1, int per2, double d0, double d1, double d2, double* __restrict__ K) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)P0 * P1 * P2) return;
  const int j[3] = {(int)(idx % P0), (int)((idx / P0) % P1), (int)(idx / ((int64_t)P0 * P1))};
  const int n[3] = {n0, n1, n2}, P[3] = {P0, P1, P2}, per[3] = {per0, per1, per2};
  const double d[3] = {d0, d1, d2};
  double r[3];
  bool skip = false;
  for (int a = 0; a < 3; ++a) {
    if (!per[a] && j[a] == n[a]) skip = true;
    const int jj = per[a] ? j[a] : (j[a] < n[a] ? j[a] : j[a] - P[a]);
    r[a] = jj * d[a];
  }
  Cplx v{0.0, 0.0};
  if (!skip) v = pgf_eval_bloch(pd, k0.k, r, j[0] == 0 && j[1] == 0 && j[2] == 0);
  K[2 * idx] = v.re;
  K[2 * idx + 1] = v.im;
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
  const int M = P0 / 2;
  // lines per CTA: enough CTAs to cover 2 waves of 148 SMs, at most 4096 complex per CTA
  int nl = std::max(1, std::min(4096 / std::max(M, 1), nrows / 296));
  size_t smem = (size_t)nl * M * sizeof(C);
  RowMap rm{n1, P1};
  int blocks = (nrows + nl - 1) / nl;
  int threads = std::min(256, std::max(64, nl * M / 2));
  threads = (threads + 31) / 32 * 32;
  if (fwd) {
    auto kern = fft_x_forward<T>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, threads, smem, st>>>(rin, cio, nrows, n0, P0, ilog2(M), rm, tw, nl);
  } else {
    auto kern = fft_x_inverse<T>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, threads, smem, st>>>(cio, rout, nrows, n0, P0, ilog2(M), rm, tw, nl);
  }
  CK(cudaGetLastError());
}

// ---------------------------------------------------------------- slab-decomposed convolution
// (SURVEY 8(e)): rank r owns the z planes [r nzl, (r+1) nzl) of the grid for the X and Y
// passes and the k0 columns [h_r, h_r + H_r) of the half spectrum for the Z pass; two
// all-to-all transposes move the spectrum between the two layouts.
//   z-slab layout Cz [nzl][P1][H0]   x-slab layout Cx [P2][P1][H_r]
// Block (r -> p) = Cz_r[:, :, h_p : h_p + H_p] packed as [nzl][P1][H_p]; it lands in Cx_p at
// plane offset r nzl (contiguous), so only the sender packs and only the return path unpacks.
// slab_h0 / slab_hn: device.cuh

// pack (dir 0): Cz[rows][H0] cols [h_p, h_p+H_p) -> buf + p*rows*(h_p) ... contiguous [rows][H_p] blocks
// unpack (dir 1): the reverse.  blockIdx.y = peer p.
__global__ void k_slab_pack(float2* __restrict__ cz, float2* __restrict__ buf, int64_t rows, int H0, int W, int dir) {
  const int p = blockIdx.y;
  const int h = slab_h0(p, H0, W), hn = slab_hn(p, H0, W);
  float2* blk = buf + rows * (int64_t)h;                  // blocks are stored back to back
  const int64_t tot = rows * hn;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / hn;
    const int c = (int)(i - r * hn);
    if (dir == 0) blk[i] = cz[r * H0 + h + c];
    else cz[r * H0 + h + c] = blk[i];
  }
}

// spectrum slice for rank r: spec [P2 P1][H0] cols [h_r, h_r+H_r) -> [P2 P1][H_r]
__global__ void k_spec_slice(const float* __restrict__ spec, float* __restrict__ out, int64_t rows, int H0, int h, int hn) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * hn) return;
  const int64_t r = i / hn;
  out[i] = spec[r * H0 + h + (int)(i - r * hn)];
}

void launch_yz_fused(const DeviceState& D, cudaStream_t st) {
  const int tile = D.fused_tile, P1 = D.P[1], P2 = D.P[2];
  if (D.yz_half) {   // tile 1, zero-padded z: half the shared memory (fft_yz_fused_zhalf)
    const int n2 = D.n[2], chunk = std::min(32, P1);
    const size_t smem = ((size_t)n2 * (P1 + 1) + (size_t)2 * chunk * (n2 + 1)) * sizeof(float2);
    auto kh = fft_yz_fused_zhalf<float>;
    CK(cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kh<<<D.H0, 512, smem, st>>>(D.C, D.n[1], P1, ilog2(P1), n2, ilog2(n2), D.H0, chunk, D.spec, D.tw32[1], D.tw32[2]);
    CK(cudaGetLastError());
    return;
  }
  size_t smem = (size_t)P2 * (P1 * tile + (tile == 1 ? 1 : 0)) * sizeof(float2);   // padded planes
  auto kern = fft_yz_fused<float>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // up to 1024 threads: at the C3 plane size (129 KB) one CTA fills an SM, and its passes are
  // latency-bound (measured C3 FFT 0.156 -> 0.151 ms vs 512); PMFEM_YZ_THREADS overrides
  static const int cap = std::getenv("PMFEM_YZ_THREADS") ? std::atoi(std::getenv("PMFEM_YZ_THREADS")) : 1024;
  int threads = std::min(cap, std::max(128, P1 * P2 * tile / 4));
  threads = (threads + 31) / 32 * 32;
  kern<<<(D.H0 + tile - 1) / tile, threads, smem, st>>>(D.C, D.n[1], P1, ilog2(P1), D.n[2], P2, ilog2(P2), D.H0,
                                                         tile, D.spec, D.tw32[1], D.tw32[2]);
  CK(cudaGetLastError());
}

}  // namespace

void device_upload(DeviceState& D, const HostSetup& S) {
  CK(cudaSetDevice(D.device));
  static const bool verbose = std::getenv("PMFEM_VERBOSE") != nullptr;
  auto t_up0 = std::chrono::steady_clock::now();
  auto upload_stage = [&](const char* what) {
    if (!verbose) return;
    CK(cudaDeviceSynchronize());
    std::fprintf(stderr, "[pmfem]   upload %-18s %8.2f s\n", what,
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t_up0).count());
  };
  const int64_t Np = S.Np;
  D.Np = Np;
  D.order = S.order;
  for (int a = 0; a < 3; ++a) { D.periodic[a] = S.periodic[a]; D.n[a] = S.grid_n[a]; D.P[a] = S.fft_n[a]; }
  D.H0 = D.P[0] / 2 + 1;
  D.rank = S.dist.rank;
  D.world = S.dist.world;
  for (int a = 0; a < 3; ++a) D.axperm[a] = S.axperm[a];
  D.lo = S.dist.lo();
  D.hi = S.dist.hi();

  // ---- shared local operator in SELL-32, internal order; a rank stores its own rows [lo, hi)
  // only (slices relative to lo)
  const int64_t lo = D.lo, nloc = D.hi - D.lo;
  const int64_t ns = (nloc + 31) / 32;
  D.nslices = ns;
  std::vector<int64_t> sl_off(ns + 1, 0), sl1_off(ns + 1, 0);
  // per own internal row: ring-1 cols (user ids) + Z0-only cols, with values
  std::vector<int> len1(nloc), lenz(nloc);
  std::vector<std::vector<int32_t>> rcols(nloc);
  std::vector<std::vector<float>> rz(nloc), rld(nloc), rg(nloc);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < nloc; ++i) {
    const int64_t r = S.perm[lo + i];
    std::vector<std::pair<int32_t, int64_t>> r1, rzl;
    for (int64_t e = S.ring1.rowptr[r]; e < S.ring1.rowptr[r + 1]; ++e) r1.push_back({(int32_t)S.iperm[S.ring1.col[e]], e});
    for (int64_t e = S.z0.rowptr[r]; e < S.z0.rowptr[r + 1]; ++e) rzl.push_back({(int32_t)S.iperm[S.z0.col[e]], e});
    std::sort(r1.begin(), r1.end());
    std::sort(rzl.begin(), rzl.end());
    std::vector<int32_t>& cols = rcols[i];
    std::vector<float>& z = rz[i];
    for (auto& pr : r1) {
      cols.push_back(pr.first);
      const double* v = &S.ring1.val[7 * pr.second];
      for (int x = 0; x < 4; ++x) rld[i].push_back((float)v[x]);
      for (int x = 0; x < 3; ++x) rg[i].push_back((float)v[4 + x]);
      // Z0 value for this column (0 if Z0 has no entry there)
      auto it = std::lower_bound(rzl.begin(), rzl.end(), std::make_pair(pr.first, (int64_t)-1));
      for (int x = 0; x < 3; ++x)
        z.push_back((it != rzl.end() && it->first == pr.first) ? (float)S.z0.val[3 * it->second + x] : 0.f);
    }
    for (auto& pr : rzl) {
      auto it = std::lower_bound(r1.begin(), r1.end(), std::make_pair(pr.first, (int64_t)-1));
      if (it != r1.end() && it->first == pr.first) continue;
      cols.push_back(pr.first);
      for (int x = 0; x < 3; ++x) z.push_back((float)S.z0.val[3 * pr.second + x]);
    }
    len1[i] = (int)r1.size();
    lenz[i] = (int)cols.size();
  }
  for (int64_t s = 0; s < ns; ++s) {
    int w = 0, w1 = 0;
    for (int64_t i = 32 * s; i < std::min(nloc, 32 * s + 32); ++i) { w = std::max(w, lenz[i]); w1 = std::max(w1, len1[i]); }
    sl_off[s + 1] = sl_off[s] + 32 * (int64_t)w;
    sl1_off[s + 1] = sl1_off[s] + 32 * (int64_t)w1;
  }
  const int64_t zt = sl_off[ns], gt = sl1_off[ns];
  D.zt = zt;
  D.gt = gt;
  std::vector<float4> s_zc(zt), s_Gc(gt), s_LD(gt, make_float4(0, 0, 0, 0));
  auto pack = [](float x, float y, float z, int32_t c) { return make_float4(x, y, z, __int_as_float_host(c)); };
#pragma omp parallel for
  for (int64_t s = 0; s < ns; ++s) {
    const int w = (int)((sl_off[s + 1] - sl_off[s]) / 32), w1 = (int)((sl1_off[s + 1] - sl1_off[s]) / 32);
    for (int l = 0; l < 32; ++l) {
      const int64_t i = 32 * s + l;                                      // local row
      const int32_t self = (int32_t)(lo + std::min<int64_t>(i, nloc - 1));   // padding: the row itself, weight 0
      for (int j = 0; j < w; ++j) {
        const int64_t e = sl_off[s] + 32 * j + l;
        if (i < nloc && j < lenz[i]) s_zc[e] = pack(rz[i][3 * j], rz[i][3 * j + 1], rz[i][3 * j + 2], rcols[i][j]);
        else s_zc[e] = pack(0.f, 0.f, 0.f, self);
      }
      for (int j = 0; j < w1; ++j) {
        const int64_t e1 = sl1_off[s] + 32 * j + l;
        if (i < nloc && j < len1[i]) {
          s_LD[e1] = make_float4(rld[i][4 * j], rld[i][4 * j + 1], rld[i][4 * j + 2], rld[i][4 * j + 3]);
          s_Gc[e1] = pack(rg[i][3 * j], rg[i][3 * j + 1], rg[i][3 * j + 2], rcols[i][j]);
        } else {
          s_Gc[e1] = pack(0.f, 0.f, 0.f, self);
        }
      }
    }
  }
  D.sl_off = dupload(sl_off); D.sl1_off = dupload(sl1_off);
  D.s_zc = dupload(s_zc); D.s_LD = dupload(s_LD); D.s_Gc = dupload(s_Gc);
  D.m4 = dalloc<float4>(Np);
  CK(cudaMemset(D.m4, 0, sizeof(float4) * (size_t)Np));

  std::vector<float4> rsum(2 * Np), stt(Np);
  std::vector<int4> sts(Np);
  for (int64_t i = 0; i < Np; ++i) {
    int64_t r = S.perm[i];
    rsum[2 * i] = make_float4((float)S.rowsumD[3 * r], (float)S.rowsumD[3 * r + 1], (float)S.rowsumD[3 * r + 2], 0.f);
    rsum[2 * i + 1] = make_float4((float)S.rowsumZ[3 * r], (float)S.rowsumZ[3 * r + 1], (float)S.rowsumZ[3 * r + 2], 0.f);
    int s[3];
    for (int a = 0; a < 3; ++a) {
      int v = S.st_s[3 * r + a];
      if (S.periodic[a]) v = ((v % S.grid_n[a]) + S.grid_n[a]) % S.grid_n[a];
      s[a] = v;
    }
    sts[i] = make_int4(s[0], s[1], s[2], 0);
    // .w carries the wrapped anchor x (bit pattern) for the gather anterpolation
    stt[i] = make_float4((float)S.st_t[3 * r], (float)S.st_t[3 * r + 1], (float)S.st_t[3 * r + 2],
                         __int_as_float_host(s[0]));
  }
  D.rowsum = dupload(rsum); D.st_s = dupload(sts); D.st_t = dupload(stt);
  upload_stage("SELL + stencils");
  // K2 reads the rows of each anchor line through box_ptr: rows must be sorted by anchor box
  {
    const int64_t Gb = (int64_t)D.n[0] * D.n[1] * D.n[2];
    std::vector<int32_t> bp(Gb + 1, 0);
    for (int64_t i = 0; i < Np; ++i) {
      const int64_t key = ((int64_t)sts[i].z * D.n[1] + sts[i].y) * D.n[0] + sts[i].x;
      if (i > 0) {
        const int64_t k0 = ((int64_t)sts[i - 1].z * D.n[1] + sts[i - 1].y) * D.n[0] + sts[i - 1].x;
        if (key < k0) throw Error(PMFEM_E_STATE, "internal rows are not sorted by anchor box");
      }
      bp[key + 1]++;
    }
    D.box_max = 1;
    for (int64_t b = 0; b < Gb; ++b) { D.box_max = std::max(D.box_max, bp[b + 1]); bp[b + 1] += bp[b]; }
    D.box_ptr = dupload(bp);
    // K2 tile: ~G/600 points (>= 4 CTAs per SM), 256..4096 points, grown by doubling the
    // shortest axis (x first on ties) so the tile stays compact; PMFEM_K2_TILE=t0,t1,t2 overrides
    int64_t target = 256;
    while (target < 4096 && target * 2 * 600 <= Gb) target *= 2;
    int t[3] = {1, 1, 1};
    // the kernel's segment scan holds k2_nseg(t1, t2, P) <= 256 threads x 8 segments
    auto nseg_ok = [&](int a) {
      return k2_nseg(a == 1 ? 2 * t[1] : t[1], a == 2 ? 2 * t[2] : t[2], D.order) <= 2048;
    };
    while ((int64_t)t[0] * t[1] * t[2] < target) {
      int best = -1;
      for (int a = 0; a < 3; ++a)
        if (t[a] < D.n[a] && nseg_ok(a) && (best < 0 || t[a] < t[best])) best = a;
      if (best < 0) break;
      t[best] *= 2;
    }
    if (const char* e = std::getenv("PMFEM_K2_TILE")) {
      int a0, a1, a2;
      if (std::sscanf(e, "%d,%d,%d", &a0, &a1, &a2) == 3 && a0 > 0 && a1 > 0 && a2 > 0 && D.n[0] % a0 == 0 &&
          D.n[1] % a1 == 0 && D.n[2] % a2 == 0 && a0 * a1 * a2 <= 12288 && k2_nseg(a1, a2, D.order) <= 2048) {
        t[0] = a0; t[1] = a1; t[2] = a2;
      }
    }
    for (int a = 0; a < 3; ++a) D.k2_tile[a] = t[a];
    if (k2_nseg(t[1], t[2], D.order) > 2048) throw Error(PMFEM_E_STATE, "K2 tile exceeds the segment scan capacity");
  }
  // ---- C_box: built on the device in internal order, stored in the chunked C4x format
  if (!S.cbox_device) throw Error(PMFEM_E_STATE, "device contexts build C_box on the device");
  device_build_cbox(D, S);
  upload_stage("C_box");
  for (int a = 0; a < 3; ++a) {
    std::vector<float2> t32; std::vector<double2> t64;
    twiddles<float>(D.P[a], t32); twiddles<double>(D.P[a], t64);
    D.tw32[a] = dupload(t32); D.tw64[a] = dupload(t64);
  }
  // q: + 4 zero floats so B4's aligned 4-column gathers stay in bounds
  // q: + 16 zero floats so B4's aligned and U4's shifted 4-column gathers stay in bounds
  D.q = dalloc<float>(Np + 16); D.uloc = dalloc<float>(Np); D.u = dalloc<float>(Np);
  if (D.cbox_format == 3) {
    D.q4s = (Np + 3) / 4 + 1;
    D.q4 = dalloc<float4>(4 * D.q4s);
  }
  CK(cudaMemset(D.q, 0, sizeof(float) * (size_t)(Np + 16)));
  D.Q = dalloc<float>((size_t)D.n[0] * D.n[1] * D.n[2]);
  D.C = dalloc<float2>((size_t)D.H0 * D.P[1] * D.P[2]);
  D.spec = dalloc<float>((size_t)D.H0 * D.P[1] * D.P[2]);
  for (int i = 0; i < 8; ++i) CK(cudaEventCreate(&D.ev[i]));
  // FFT plan: fused YZ when a yz plane of `tile` columns fits in shared memory
  {
    const size_t plane_bytes = (size_t)(D.P[1] + 1) * D.P[2] * sizeof(float2);
    D.fused_tile = 0;
    // PMFEM_FFT_SPLIT=1 forces the split plan (tests exercise it on small grids)
    if (plane_bytes <= 200 * 1024 && std::getenv("PMFEM_FFT_SPLIT") == nullptr) {
      int tile = 1;
      while (tile < 4 && plane_bytes * tile * 2 <= 96 * 1024 && (D.H0 + 2 * tile - 1) / (2 * tile) >= 148) tile *= 2;
      // PMFEM_YZ_TILE=1|2|4|8 forces the column tile when its planes fit (tests run tile > 1 on
      // small grids: the production tile-4 plan of C5 has H0 = 1025)
      if (const char* e = std::getenv("PMFEM_YZ_TILE")) {
        const int tv = std::atoi(e);
        if ((tv == 1 || tv == 2 || tv == 4 || tv == 8) && (size_t)D.P[1] * D.P[2] * tv * sizeof(float2) <= 200 * 1024)
          tile = tv;
      }
      D.fused_tile = tile;
      // PMFEM_YZ_HALF=1: the split-z fused kernel for tile-1 columns with a zero-padded z axis
      // (opt-in: measured slower, C3 FFT 0.156 -> 0.182 ms -- more barriers per column)
      const char* yh = std::getenv("PMFEM_YZ_HALF");
      D.yz_half = tile == 1 && D.P[2] == 2 * D.n[2] && D.n[2] >= 2 && yh != nullptr && std::atoi(yh) == 1;
    }
  }
  D.launches_per_eval = 5 + (D.fused_tile ? 3 : 5) + (D.cbox_format == 3 ? 1 : 0);   // m4, K1, K2, FFT, (q4), K4, K5
  D.k4_vec = std::getenv("PMFEM_K4_VEC") != nullptr && std::atoi(std::getenv("PMFEM_K4_VEC")) == 1;
  // K4 variants read per context (tests switch them between contexts of one process)
  D.k4_stream = std::getenv("PMFEM_K4_STREAM") != nullptr && std::atoi(std::getenv("PMFEM_K4_STREAM")) == 1;
  // C4x: 4 batched chunks per lane by default (call 29, 8 lanes per row: C4 K4 8.18 -> 7.86 ms);
  // PMFEM_K4_KB=2 selects 2
  D.k4_kb4 = !(std::getenv("PMFEM_K4_KB") != nullptr && std::atoi(std::getenv("PMFEM_K4_KB")) == 2);
  D.row_split = 1;            // 2 measured slower on C2 (K1 0.067 -> 0.070 ms); kept for PMFEM_ROW_SPLIT=2
  if (const char* e = std::getenv("PMFEM_ROW_SPLIT")) {
    const int v = std::atoi(e);
    if (v == 1 || v == 2) D.row_split = v;
  }
  // slab-decomposed convolution: NCCL ranks (z slabs = the row partition's planes), or simulated
  // ranks on one device (tests, PMFEM_SLAB_SIM=W: the same plane rule for W ranks)
  {
    int W = 1;
    if (D.world > 1) {
      if (D.H0 >= D.world && std::getenv("PMFEM_NO_SLAB") == nullptr) W = D.world;
    } else if (const char* e = std::getenv("PMFEM_SLAB_SIM")) {
      const int w = std::atoi(e);
      if (w > 1 && D.H0 >= w && D.n[2] >= w) W = w;
    }
    D.slab_world = W;
    if (W > 1) {
      if (D.world > 1) {
        D.zpl.assign(S.dist.planes.begin(), S.dist.planes.end());
        for (int k = 0; k < 2; ++k) { D.gsend[k] = S.dist.gsend[k]; D.grecv[k] = S.dist.grecv[k]; }
      } else {
        const std::vector<int32_t> z = slab_planes(S, W, slab_granularity(S, W));
        D.zpl.assign(z.begin(), z.end());
      }
      int nzmax = 0;
      for (int r = 0; r < W; ++r) nzmax = std::max(nzmax, D.zpl[r + 1] - D.zpl[r]);
      const int64_t plane = (int64_t)D.P[1];
      const int64_t Hr = D.world > 1 ? slab_hn(D.rank, D.H0, W) : D.H0;
      D.slab_cx = dalloc<float2>((size_t)D.P[2] * plane * Hr);
      D.slab_spec = dalloc<float>((size_t)D.P[2] * plane * Hr);
      D.slab_buf = dalloc<float2>((size_t)(D.world > 1 ? nzmax : D.n[2]) * plane * D.H0);
      D.fused_tile = 0;
      // per rank: X, Y, pack, Z, unpack, Y', X' (+ W-1 sends/receives and the copies in NCCL)
      D.launches_per_eval = 5 + 7 * (D.world > 1 ? 1 : W) + (D.cbox_format == 3 ? 1 : 0);
    }
  }
  // K2 tiles must not straddle a z-slab boundary: the z tile divides every slab's planes
  if (D.slab_world > 1) {
    int t2 = D.k2_tile[2];
    auto ok = [&](int t) { for (int b : D.zpl) if (b % t) return false; return true; };
    while (t2 > 1 && !ok(t2)) t2 >>= 1;
    D.k2_tile[2] = t2;
  }
  // compulsory bytes per launch: every array read or written once (gathered m, q, u once),
  // actual entries only (SELL padding is overhead, not algorithmic traffic)
  const double G = (double)D.n[0] * D.n[1] * D.n[2];
  double nsh = 0, n1e = 0;
  for (int64_t i = 0; i < nloc; ++i) { nsh += lenz[i]; n1e += len1[i]; }
  // K1 window = m -> float4 copy (12 + 16) + K1 (m4 16, row sums 32, slice offsets ~0, q, u_loc, H_ex)
  D.kernel_bytes[0] = nloc * (12.0 + 16 + 16 + 32 + 4 + 4 + 12) + nsh * 16 + n1e * 16;
  // q + anchors + local t of the rows read (own + halo band), box_ptr, Q write of the own planes
  const double Gl = G * (double)(S.dist.planes[S.dist.rank + 1] - S.dist.planes[S.dist.rank]) / D.n[2];
  D.kernel_bytes[1] = (double)std::min<int64_t>(Np, nloc + (int64_t)S.dist.recv_idx[1].size()) * (4.0 + 16 + 16) + Gl * 4.0 * 2;
  {
    const double Hc = (double)D.H0;
    const double spec_b = Hc * D.P[1] * D.P[2] * 4;
    if (D.fused_tile) {
      D.kernel_bytes[2] = (G * 4 + (double)D.n[1] * D.n[2] * Hc * 8)        // X
                          + 2.0 * (double)D.n[1] * D.n[2] * Hc * 8 + spec_b   // YZ: data block in + out
                          + ((double)D.n[1] * D.n[2] * Hc * 8 + G * 4);       // X'
    } else {
      D.kernel_bytes[2] = (G * 4 + (double)D.n[1] * D.n[2] * Hc * 8) + 2.0 * (double)D.n[2] * Hc * D.P[1] * 8 +
                          2.0 * Hc * D.P[1] * D.P[2] * 8 + spec_b + 2.0 * (double)D.n[2] * Hc * D.P[1] * 8 +
                          ((double)D.n[1] * D.n[2] * Hc * 8 + G * 4);
    }
  }
  const int64_t cnnz = D.cbox_nnz;
  {
    // K4 group size: ~4+ chunks per lane; PMFEM_K4_GROUP overrides (tests)
    const double row4 = (double)D.cbox_chunks / std::max<int64_t>(Np, 1);
    D.k4_group = row4 >= 96 ? 32 : (row4 >= 40 ? 16 : 8);
    if (D.cbox_format == 2) D.k4_group = 16;   // SEG: mask words per row (A/B: PMFEM_K4_GROUP)
    // global-index formats (C4x, B4, U4): 8 lanes per row -- four rows per warp keep four
    // independent header -> gather chains in flight (call 25: C4 K4 9.98 ms at 32 lanes, 8.80 at
    // 16, 8.25 at 8, 8.54 at 4; C3 0.89 / 0.53 / 0.47 / 0.49 ms); W4 keeps the row-length rule
    // (its gathers hit shared memory: C5 1.89 ms at 32 lanes vs 2.21 at 8)
    if (D.cbox_format == 0 || D.cbox_format == 1 || D.cbox_format == 3) D.k4_group = 8;
    if (const char* e = std::getenv("PMFEM_K4_GROUP")) {
      const int gsel = std::atoi(e);
      if (gsel == 4 || gsel == 8 || gsel == 16 || gsel == 32) D.k4_group = gsel;
    }
  }
  // C_box per near pair: C4x 4-byte value + 2 bytes of chunk header, B4 4-byte value + 1 byte
  // of block index (chunk padding / empty block slots are format overhead, not counted)
  // SEG: 4-byte value per near pair + the candidate bitmask words + two 8-byte row offsets
  if (D.cbox_format == 2)
    D.kernel_bytes[3] = nloc * (16.0 + 16 + 16 + 4 + 4 + 4) + (double)cnnz * 4 + (double)D.seg_mask_words * 4 + Gl * 4.0;
  else if (D.cbox_format == 3)   // + the q4 copy (4-byte read, 16-byte write per row)
    D.kernel_bytes[3] = nloc * (16.0 + 16 + 8 + 4 + 4 + 4) + Np * 20.0 + (double)cnnz * 5 + Gl * 4.0;
  else   // C4x and W4: 4-byte value + 2 bytes of chunk header / window index per near pair
    D.kernel_bytes[3] = nloc * (16.0 + 16 + 8 + 4 + 4 + 4) + (double)cnnz * (D.cbox_format == 1 ? 5 : 6) + Gl * 4.0;
  D.kernel_bytes[4] = nloc * (4.0 + 12 + 12) + n1e * 16;        // u, H read+write, (G, col)
}

void device_build_pgf(DeviceState& D, const HostSetup& S, const PgfParams& Pp) {
  CK(cudaSetDevice(D.device));
  PgfDev pd;
  std::memset(&pd, 0, sizeof(pd));
  pd.dim = Pp.dim;
  for (int i = 0; i < 3; ++i) { pd.ax[i] = Pp.ax[i]; pd.L[i] = Pp.L[i]; pd.nreal[i] = Pp.nreal[i]; pd.mrec[i] = Pp.mrec[i]; }
  pd.alpha = Pp.alpha;
  pd.xr = Pp.xr;
  gauss_legendre01(64, pd.gl_x, pd.gl_w);
  const int P0 = D.P[0], P1 = D.P[1], P2 = D.P[2];
  const int64_t tot = (int64_t)P0 * P1 * P2;
  double* K = dalloc<double>(tot);
  const int64_t oct = (int64_t)(P0 / 2 + 1) * (P1 / 2 + 1) * (P2 / 2 + 1);
  k_pgf_table<<<(unsigned)((oct + 63) / 64), 64>>>(pd, P0, P1, P2, D.n[0], D.n[1], D.n[2], D.periodic[0],
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
  if (D.slab_world > 1) {   // spectrum slices of the x-slab layout
    const int W = D.slab_world;
    const int64_t rows = (int64_t)P1 * P2;
    for (int p = 0; p < W; ++p) {
      if (D.world > 1 && p != D.rank) continue;
      const int h = slab_h0(p, H0, W), hn = slab_hn(p, H0, W);
      float* out = D.slab_spec + (D.world > 1 ? 0 : rows * h);
      k_spec_slice<<<(unsigned)((rows * hn + 255) / 256), 256>>>(D.spec, out, rows, H0, h, hn);
      CK(cudaGetLastError());
    }
  }
  CK(cudaDeviceSynchronize());
  cudaFree(K);
  cudaFree(C);
  D.pgf_ready = true;
}

void device_bloch_table(DeviceState& D, const HostSetup& S, const PgfParams& Pp, const double k0[3],
                        std::vector<double>& K) {
  CK(cudaSetDevice(D.device));
  PgfDev pd;
  std::memset(&pd, 0, sizeof(pd));
  pd.dim = Pp.dim;
  for (int i = 0; i < 3; ++i) { pd.ax[i] = Pp.ax[i]; pd.L[i] = Pp.L[i]; pd.nreal[i] = Pp.nreal[i]; pd.mrec[i] = Pp.mrec[i]; }
  pd.alpha = Pp.alpha;
  pd.xr = Pp.xr;
  gauss_legendre01(64, pd.gl_x, pd.gl_w);
  const int64_t tot = (int64_t)D.P[0] * D.P[1] * D.P[2];
  double* dK = dalloc<double>(2 * tot);
  K0v kv{{k0[0], k0[1], k0[2]}};
  k_pgf_table_bloch<<<(unsigned)((tot + 63) / 64), 64>>>(pd, kv, D.P[0], D.P[1], D.P[2], D.n[0], D.n[1], D.n[2],
                                                           D.periodic[0], D.periodic[1], D.periodic[2], S.delta[0],
                                                           S.delta[1], S.delta[2], dK);
  CK(cudaGetLastError());
  K.resize(2 * tot);
  CK(cudaMemcpy(K.data(), dK, sizeof(double) * 2 * tot, cudaMemcpyDeviceToHost));
  cudaFree(dK);
}

void device_free(DeviceState& D) {
  if (D.device < 0) return;
  cudaSetDevice(D.device);
  device_bloch_free(D);
  void* ptrs[] = {D.sl_off, D.sl1_off, D.s_zc, D.s_LD, D.s_Gc, D.m4, D.rowsum, D.c_ptr, D.c_hdr, D.c_bidx, D.c_val,
                  D.seg_moff, D.seg_mask, D.q4, D.w_trow, D.w_rptr, D.w_rstart, D.w_rlen, D.w_rloc, D.w_idx,
                  D.st_s, D.st_t, D.box_ptr, D.spec, D.q, D.uloc, D.u, D.Q, D.C, D.m_stage, D.H_stage,
                  D.tw32[0], D.tw32[1], D.tw32[2], D.tw64[0], D.tw64[1], D.tw64[2],
                  D.send_buf, D.recv_buf, D.slab_cx, D.slab_buf, D.slab_spec, D.send_idx[0], D.send_idx[1], D.send_idx[2],
                  D.recv_idx[0], D.recv_idx[1], D.recv_idx[2]};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int i = 0; i < 8; ++i)
    if (D.ev[i]) cudaEventDestroy(D.ev[i]);
  for (auto& g : D.graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (D.llg_exec) cudaGraphExecDestroy(D.llg_exec);
  for (void* p : {(void*)D.llg_ms, (void*)D.llg_H, (void*)D.llg_acc})
    if (p) cudaFree(p);
  if (D.comm) ncclCommDestroy((ncclComm_t)D.comm);
}

#define NCK(x)                                                                                  \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) throw Error(PMFEM_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

void device_init_comm(DeviceState& D, const HostSetup& S, const void* nccl_id) {
  CK(cudaSetDevice(D.device));
  const DistPlan& P = S.dist;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t comm;
  NCK(ncclCommInitRank(&comm, P.world, id, P.rank));
  D.comm = comm;
  int64_t sbuf = 0, rbuf = 0;
  const int width[3] = {4, 1, 1};   // m travels as the float4 copy
  // grid traffic per rank: the two spectrum transposes and the U ghost planes (slab FFT), or a
  // ring all-reduce of Q (replicated FFT)
  const double plane_b = 4.0 * (double)D.n[0] * D.n[1];
  if (D.slab_world > 1) {
    const int nz = D.zpl[P.rank + 1] - D.zpl[P.rank];
    const int hn = slab_hn(P.rank, D.H0, P.world);
    D.comm_bytes_per_eval = 2.0 * 8.0 * (double)nz * D.P[1] * (D.H0 - hn) +
                            2.0 * 8.0 * (double)(D.n[2] - nz) * D.P[1] * hn;
    for (int p = 0; p < P.world; ++p)
      for (int k = 0; k < 2; ++k)
        D.comm_bytes_per_eval += plane_b * (P.gsend[k][2 * p + 1] + P.grecv[k][2 * p + 1]);
  } else {
    D.comm_bytes_per_eval = 2.0 * 4.0 * (double)D.n[0] * D.n[1] * D.n[2] * (P.world - 1) / P.world;
  }
  for (int k = 0; k < 3; ++k) {
    D.send_ptr[k] = P.send_ptr[k];
    D.recv_ptr[k] = P.recv_ptr[k];
    D.send_idx[k] = dupload(P.send_idx[k]);
    D.recv_idx[k] = dupload(P.recv_idx[k]);
    sbuf = std::max<int64_t>(sbuf, (int64_t)P.send_idx[k].size() * width[k]);
    rbuf = std::max<int64_t>(rbuf, (int64_t)P.recv_idx[k].size() * width[k]);
    D.comm_bytes_per_eval += 4.0 * width[k] * (double)(P.send_idx[k].size() + P.recv_idx[k].size());
    D.launches_per_eval += (P.send_idx[k].empty() ? 0 : 1) + (P.recv_idx[k].empty() ? 0 : 1);   // pack/unpack
  }
  D.send_buf = dalloc<float>(sbuf);
  D.recv_buf = dalloc<float>(rbuf);
}

namespace {
// halo exchange of vector v (width w floats per row) for plan kind k: pack my rows that peers
// need, grouped NCCL send/recv with every peer, unpack the received rows in place
void halo(DeviceState& D, int k, float* v, int w, cudaStream_t st) {
  if (D.world <= 1) return;
  const int64_t ns = D.send_ptr[k][D.world], nr = D.recv_ptr[k][D.world];
  if (ns) {
    k_pack<<<(unsigned)((ns * w + 255) / 256), 256, 0, st>>>(v, D.send_idx[k], ns, w, D.send_buf);
    CK(cudaGetLastError());
  }
  ncclComm_t comm = (ncclComm_t)D.comm;
  NCK(ncclGroupStart());
  for (int p = 0; p < D.world; ++p) {
    const int64_t sc = D.send_ptr[k][p + 1] - D.send_ptr[k][p];
    const int64_t rc = D.recv_ptr[k][p + 1] - D.recv_ptr[k][p];
    if (sc) NCK(ncclSend(D.send_buf + D.send_ptr[k][p] * w, (size_t)(sc * w), ncclFloat, p, comm, st));
    if (rc) NCK(ncclRecv(D.recv_buf + D.recv_ptr[k][p] * w, (size_t)(rc * w), ncclFloat, p, comm, st));
  }
  NCK(ncclGroupEnd());
  if (nr) {
    k_unpack<<<(unsigned)((nr * w + 255) / 256), 256, 0, st>>>(D.recv_buf, D.recv_idx[k], nr, w, v);
    CK(cudaGetLastError());
  }
}

// ---- slab-decomposed FFT convolution; D.slab_world > 1.  Rank r owns the z planes
// [Z_r, Z_r+1) (D.zpl, variable thickness) for the X and Y passes and the k0 columns
// [h_r, h_r + H_r) for the Z pass; block (r -> p) = Cz_r[:, :, h_p : h_p + H_p] packed as
// [nz_r][P1][H_p] lands in Cx_p at plane offset Z_r (contiguous).
// per-rank phases, shared by the NCCL path and the single-device simulation (PMFEM_SLAB_SIM)
void slab_phase_fwd(const DeviceState& D, int r, const float* Qs, float2* Cz, float2* sbuf, cudaStream_t st) {
  const int W = D.slab_world, n0 = D.n[0], n1 = D.n[1], nz = D.zpl[r + 1] - D.zpl[r], P0 = D.P[0], P1 = D.P[1],
            H0 = D.H0;
  if (nz == 0) return;
  launch_x<float>(true, Qs, Cz, nullptr, nz * n1, n0, P0, n1, P1, D.tw32[0], st);
  launch_strided<float>(Cz, P1, H0, H0, nz, (long long)P1 * H0, n1, P1, 0, nullptr, 0, 0, D.tw32[1], st);
  const int64_t rows = (int64_t)nz * P1;
  k_slab_pack<<<dim3((unsigned)std::min<int64_t>(1024, (rows * (H0 / W + 1) + 255) / 256), W), 256, 0, st>>>(Cz, sbuf, rows, H0, W, 0);
  CK(cudaGetLastError());
}
void slab_phase_z(const DeviceState& D, float2* Cx, const float* spec_r, int Hr, cudaStream_t st) {
  const int P1 = D.P[1];
  launch_strided<float>(Cx, D.P[2], (long long)P1 * Hr, Hr, P1, Hr, D.n[2], D.n[2], 2, spec_r, (long long)P1 * Hr, Hr,
                        D.tw32[2], st);
}
void slab_phase_inv(const DeviceState& D, int r, float2* rbuf, float2* Cz, float* Us, cudaStream_t st) {
  const int W = D.slab_world, n0 = D.n[0], n1 = D.n[1], nz = D.zpl[r + 1] - D.zpl[r], P0 = D.P[0], P1 = D.P[1],
            H0 = D.H0;
  if (nz == 0) return;
  const int64_t rows = (int64_t)nz * P1;
  k_slab_pack<<<dim3((unsigned)std::min<int64_t>(1024, (rows * (H0 / W + 1) + 255) / 256), W), 256, 0, st>>>(Cz, rbuf, rows, H0, W, 1);
  CK(cudaGetLastError());
  launch_strided<float>(Cz, P1, H0, H0, nz, (long long)P1 * H0, P1, n1, 1, nullptr, 0, 0, D.tw32[1], st);
  launch_x<float>(false, nullptr, Cz, Us, nz * n1, n0, P0, n1, P1, D.tw32[0], st);
}

// NCCL path: Q holds this rank's z planes [Z_r, Z_r+1) of the anterpolated grid (K2 computed
// them completely from own + halo rows: no reduction); on return Q holds U on those planes.
// X, Y -> all-to-all -> Z*G -> all-to-all -> Y', X'.
void slab_conv_nccl(DeviceState& D, cudaStream_t st) {
  const int W = D.world, r = D.rank, H0 = D.H0, P1 = D.P[1];
  const size_t plane = (size_t)D.n[1] * D.n[0];
  ncclComm_t comm = (ncclComm_t)D.comm;
  float* Qr = D.Q + (size_t)D.zpl[r] * plane;
  slab_phase_fwd(D, r, Qr, D.C, D.slab_buf, st);
  const int Hr = slab_hn(r, H0, W);
  const int64_t rows_r = (int64_t)(D.zpl[r + 1] - D.zpl[r]) * P1;
  NCK(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    if (p == r) continue;
    const int64_t rows_p = (int64_t)(D.zpl[p + 1] - D.zpl[p]) * P1;
    if (rows_r) NCK(ncclSend(D.slab_buf + rows_r * slab_h0(p, H0, W), (size_t)(rows_r * slab_hn(p, H0, W) * 2), ncclFloat, p, comm, st));
    if (rows_p) NCK(ncclRecv(D.slab_cx + (int64_t)D.zpl[p] * P1 * Hr, (size_t)(rows_p * Hr * 2), ncclFloat, p, comm, st));
  }
  NCK(ncclGroupEnd());
  if (rows_r)
    CK(cudaMemcpyAsync(D.slab_cx + (int64_t)D.zpl[r] * P1 * Hr, D.slab_buf + rows_r * slab_h0(r, H0, W),
                       sizeof(float2) * rows_r * Hr, cudaMemcpyDeviceToDevice, st));
  slab_phase_z(D, D.slab_cx, D.slab_spec, Hr, st);
  NCK(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    if (p == r) continue;
    const int64_t rows_p = (int64_t)(D.zpl[p + 1] - D.zpl[p]) * P1;
    if (rows_p) NCK(ncclSend(D.slab_cx + (int64_t)D.zpl[p] * P1 * Hr, (size_t)(rows_p * Hr * 2), ncclFloat, p, comm, st));
    if (rows_r) NCK(ncclRecv(D.slab_buf + rows_r * slab_h0(p, H0, W), (size_t)(rows_r * slab_hn(p, H0, W) * 2), ncclFloat, p, comm, st));
  }
  NCK(ncclGroupEnd());
  if (rows_r)
    CK(cudaMemcpyAsync(D.slab_buf + rows_r * slab_h0(r, H0, W), D.slab_cx + (int64_t)D.zpl[r] * P1 * Hr,
                       sizeof(float2) * rows_r * Hr, cudaMemcpyDeviceToDevice, st));
  slab_phase_inv(D, r, D.slab_buf, D.C, Qr, st);
  // U ghost planes: K4's stencils read p planes above the slab (DistPlan gsend / grecv)
  NCK(ncclGroupStart());
  for (int p = 0; p < W; ++p)
    for (int k = 0; k < 2; ++k) {
      const int sz0 = D.gsend[k][2 * p], sn = D.gsend[k][2 * p + 1];
      const int rz0 = D.grecv[k][2 * p], rn = D.grecv[k][2 * p + 1];
      if (sn) NCK(ncclSend(D.Q + (size_t)sz0 * plane, (size_t)sn * plane, ncclFloat, p, comm, st));
      if (rn) NCK(ncclRecv(D.Q + (size_t)rz0 * plane, (size_t)rn * plane, ncclFloat, p, comm, st));
    }
  NCK(ncclGroupEnd());
}

// The same decomposition with W simulated ranks on this device (test mode, PMFEM_SLAB_SIM=W):
// every rank's phase runs in turn and the transposes are device copies of exactly the blocks the
// NCCL path sends.  Q holds the full anterpolated grid; each rank's U planes land in place.
void slab_conv_sim(DeviceState& D, cudaStream_t st) {
  const int W = D.slab_world, H0 = D.H0, P1 = D.P[1], P2 = D.P[2];
  const size_t plane = (size_t)D.n[1] * D.n[0];
  // rank r's z-slab blocks live at plane offset Z_r of C / slab_buf ([n2][P1][H0] in total)
  auto rows_of = [&](int r) { return (int64_t)(D.zpl[r + 1] - D.zpl[r]) * P1; };
  auto off = [&](int r) { return (int64_t)D.zpl[r] * P1 * H0; };
  for (int r = 0; r < W; ++r) slab_phase_fwd(D, r, D.Q + D.zpl[r] * plane, D.C + off(r), D.slab_buf + off(r), st);
  for (int r = 0; r < W; ++r)
    for (int p = 0; p < W; ++p) {
      const int64_t hp = slab_h0(p, H0, W), np = slab_hn(p, H0, W);
      if (rows_of(r))
        CK(cudaMemcpyAsync(D.slab_cx + (int64_t)P2 * P1 * hp + (int64_t)D.zpl[r] * P1 * np,
                           D.slab_buf + off(r) + rows_of(r) * hp, sizeof(float2) * rows_of(r) * np,
                           cudaMemcpyDeviceToDevice, st));
    }
  for (int p = 0; p < W; ++p) {
    const int64_t hp = slab_h0(p, H0, W);
    slab_phase_z(D, D.slab_cx + (int64_t)P2 * P1 * hp, D.slab_spec + (int64_t)P2 * P1 * hp, slab_hn(p, H0, W), st);
  }
  for (int r = 0; r < W; ++r)
    for (int p = 0; p < W; ++p) {
      const int64_t hp = slab_h0(p, H0, W), np = slab_hn(p, H0, W);
      if (rows_of(r))
        CK(cudaMemcpyAsync(D.slab_buf + off(r) + rows_of(r) * hp,
                           D.slab_cx + (int64_t)P2 * P1 * hp + (int64_t)D.zpl[r] * P1 * np,
                           sizeof(float2) * rows_of(r) * np, cudaMemcpyDeviceToDevice, st));
    }
  for (int r = 0; r < W; ++r) slab_phase_inv(D, r, D.slab_buf + off(r), D.C + off(r), D.Q + D.zpl[r] * plane, st);
}
}  // namespace

// m, H: [hi-lo][3] rank-local rows (the full [N'][3] on a single GPU)
void device_eval(DeviceState& D, const float* m, float* H, cudaStream_t st, EvalMode mode) {
  const RowRange rr{D.lo, D.hi, D.lo, D.axperm[0], D.axperm[1], D.axperm[2], D.Np};
  const int64_t nrows = D.hi - D.lo;
  // a rank without rows (thin slab) still takes part in every collective: only its row kernels
  // are skipped (launch grids of zero blocks are invalid)
  if (nrows <= 0 && D.world == 1) return;
  const unsigned thr_blocks = (unsigned)std::max<int64_t>(1, (nrows + 255) / 256);   // thread per row
  // external records: inside a captured graph a plain cudaEventRecord would only become an
  // internal dependency, not a timestamp readable with cudaEventElapsedTime
  auto mark = [&](int i) { if (D.timing) CK(cudaEventRecordWithFlags(D.ev[i], st, cudaEventRecordExternal)); };
  mark(0);
  k_to_m4<<<thr_blocks, 256, 0, st>>>(rr, m, D.m4);
  CK(cudaGetLastError());
  halo(D, 0, reinterpret_cast<float*>(D.m4), 4, st);
  if (mode == EVAL_EXCHANGE) {
    k_exchange<<<thr_blocks, 256, 0, st>>>(rr, D.m4, D.sl_off, D.sl1_off, D.s_zc, D.s_LD, H);
    CK(cudaGetLastError());
    return;
  }
  if (!D.pgf_ready) throw Error(PMFEM_E_STATE, "pmfem_build_pgf has not been called");
  GridDims g{D.n[0], D.n[1], D.n[2], D.periodic[0], D.periodic[1], D.periodic[2]};
  // two threads per row when the rows alone cannot fill the GPU (PMFEM_ROW_SPLIT=1|2 overrides)
  const bool split = D.row_split == 2;
  const unsigned split_blocks = (unsigned)std::max<int64_t>(1, (2 * ((nrows + 31) / 32 * 32) + 255) / 256);
  if (split)
    k1_local_in<2><<<split_blocks, 256, 0, st>>>(rr, D.m4, D.sl_off, D.sl1_off, D.s_zc, D.s_LD, D.rowsum, D.q, D.uloc, H,
                                                 mode == EVAL_HEFF ? 1 : 0);
  else
    k1_local_in<1><<<thr_blocks, 256, 0, st>>>(rr, D.m4, D.sl_off, D.sl1_off, D.s_zc, D.s_LD, D.rowsum, D.q, D.uloc, H,
                                               mode == EVAL_HEFF ? 1 : 0);
  CK(cudaGetLastError());
  // q of the rows anchored in the planes bordering the own slab (K2's stencils, C_box columns)
  halo(D, 1, D.q, 1, st);
  mark(1);
  const size_t G = (size_t)D.n[0] * D.n[1] * D.n[2];
  {
    // slab NCCL path: tiles of the own z planes only, reading own + halo rows (no row clip, no
    // reduction); otherwise tiles of the whole grid over the rows [lo, hi)
    const bool own_planes = D.world > 1 && D.slab_world > 1;
    const TileDims td{D.k2_tile[0], D.k2_tile[1], D.k2_tile[2]};
    const int z0p = own_planes ? D.zpl[D.rank] : 0, z1p = own_planes ? D.zpl[D.rank + 1] : D.n[2];
    const unsigned nt = (unsigned)(((size_t)D.n[0] / td.t0) * (D.n[1] / td.t1) * ((z1p - z0p) / td.t2));
    const int64_t klo = own_planes ? 0 : D.lo, khi = own_planes ? D.Np : D.hi;
    const size_t smem = sizeof(int) * ((size_t)3 * td.t0 * td.t1 * td.t2 + 2 * k2_nseg(td.t1, td.t2, D.order) + 1);
#define K2_LAUNCH(PP)                                                                                 \
  do {                                                                                                \
    CK(cudaFuncSetAttribute(k2_tile<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));    \
    if (nt) k2_tile<PP><<<nt, 256, smem, st>>>(g, td, D.box_ptr, D.st_s, D.st_t, D.q, klo, khi, D.box_max, \
                                               z0p / td.t2, D.Q);                                    \
  } while (0)
    switch (D.order) {
      case 1: K2_LAUNCH(1); break;
      case 2: K2_LAUNCH(2); break;
      default: K2_LAUNCH(3); break;
    }
#undef K2_LAUNCH
  }
  CK(cudaGetLastError());
  if (D.world > 1 && D.slab_world <= 1) NCK(ncclAllReduce(D.Q, D.Q, G, ncclFloat, ncclSum, (ncclComm_t)D.comm, st));
  mark(2);
  if (D.slab_world > 1) {
    if (D.world > 1) slab_conv_nccl(D, st);
    else slab_conv_sim(D, st);
  } else {
    const int n0 = D.n[0], n1 = D.n[1], n2 = D.n[2], P0 = D.P[0], P1 = D.P[1], P2 = D.P[2], H0 = D.H0;
    launch_x<float>(true, D.Q, D.C, nullptr, n1 * n2, n0, P0, n1, P1, D.tw32[0], st);
    if (D.fused_tile) {
      launch_yz_fused(D, st);
    } else {
      launch_strided<float>(D.C, P1, H0, H0, n2, (long long)P1 * H0, n1, P1, 0, nullptr, 0, 0, D.tw32[1], st);
      launch_strided<float>(D.C, P2, (long long)P1 * H0, H0, P1, H0, n2, n2, 2, D.spec, (long long)P1 * H0, H0,
                            D.tw32[2], st);
      launch_strided<float>(D.C, P1, H0, H0, n2, (long long)P1 * H0, P1, n1, 1, nullptr, 0, 0, D.tw32[1], st);
    }
    launch_x<float>(false, nullptr, D.C, D.Q, n1 * n2, n0, P0, n1, P1, D.tw32[0], st);
  }
  mark(3);
  const float4* v4 = reinterpret_cast<const float4*>(D.c_val);
  if (D.cbox_format == 3) {
    k_q4<<<(unsigned)((4 * D.q4s + 255) / 256), 256, 0, st>>>(D.q4s, D.q, D.q4);
    CK(cudaGetLastError());
  }
  const bool k4_stream_on = D.k4_stream;
  if (k4_stream_on && (D.cbox_format == 1 || D.cbox_format == 3)) {
    const unsigned blocks = (unsigned)std::max<int64_t>(1, (nrows + 8 * 64 - 1) / (8 * 64));
    const float* qv = D.cbox_format == 3 ? reinterpret_cast<const float*>(D.q4) : D.q;
#define K4T_LAUNCH(PP)                                                                                      \
    (D.cbox_format == 3                                                                                     \
         ? k4_stream<PP, 3><<<blocks, 256, 0, st>>>(rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_bidx, v4, qv, D.uloc, D.u, D.q4s) \
         : k4_stream<PP, 1><<<blocks, 256, 0, st>>>(rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_bidx, v4, qv, D.uloc, D.u, D.q4s))
    switch (D.order) {
      case 1: K4T_LAUNCH(1); break;
      case 2: K4T_LAUNCH(2); break;
      default: K4T_LAUNCH(3); break;
    }
#undef K4T_LAUNCH
  } else if (D.cbox_format == 5) {
    const size_t smem = sizeof(float) * ((size_t)D.w_max + D.w_umax);
#define K4W_LAUNCH(PP, GG)                                                                                  \
  do {                                                                                                      \
    CK(cudaFuncSetAttribute(k4_win<PP, GG, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));    \
    k4_win<PP, GG, 6><<<(unsigned)D.w_ntiles, 256, smem, st>>>(rr, D.Q, D.st_s, D.st_t, g, D.w_trow, D.w_rptr, \
                                                            D.w_rstart, D.w_rlen, D.w_rloc, D.c_ptr, v4,      \
                                                            D.w_idx, D.q, D.uloc, D.u, D.w_max, D.w_umax);  \
  } while (0)
#define K4W_BY_G(PP) \
  if (D.k4_group == 4) K4W_LAUNCH(PP, 4); else if (D.k4_group == 8) K4W_LAUNCH(PP, 8);                   \
  else if (D.k4_group == 16) K4W_LAUNCH(PP, 16); else K4W_LAUNCH(PP, 32)
    if (D.w_ntiles > 0 && D.w_tma) {
      const size_t smem_t = (size_t)W4_CCAP * 24 + sizeof(float) * ((size_t)D.w_max + D.w_umax);
#define K4WT_LAUNCH(PP, GG)                                                                                 \
  do {                                                                                                      \
    CK(cudaFuncSetAttribute(k4_win_tma<PP, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t)); \
    k4_win_tma<PP, GG><<<(unsigned)D.w_ntiles, 256, smem_t, st>>>(rr, D.Q, D.st_s, D.st_t, g, D.w_trow,       \
                                                                 D.w_rptr, D.w_rstart, D.w_rlen, D.w_rloc,    \
                                                                 D.c_ptr, v4, D.w_idx, D.q, D.uloc, D.u,      \
                                                                 D.w_max, D.w_umax);                          \
  } while (0)
#define K4WT_BY_G(PP) \
  if (D.k4_group <= 8) K4WT_LAUNCH(PP, 8); else if (D.k4_group == 16) K4WT_LAUNCH(PP, 16); else K4WT_LAUNCH(PP, 32)
      switch (D.order) {
        case 1: K4WT_BY_G(1); break;
        case 2: K4WT_BY_G(2); break;
        default: K4WT_BY_G(3); break;
      }
#undef K4WT_BY_G
#undef K4WT_LAUNCH
    } else if (D.w_ntiles > 0) {
      switch (D.order) {
        case 1: K4W_BY_G(1); break;
        case 2: K4W_BY_G(2); break;
        default: K4W_BY_G(3); break;
      }
    }
#undef K4W_BY_G
#undef K4W_LAUNCH
  } else if (D.cbox_format == 2) {
    const int G = D.k4_group;
    const size_t smem = sizeof(int) * (size_t)(256 / G) * (2 * D.seg_maxseg + 2);
    const unsigned blocks = (unsigned)std::max<int64_t>(1, (nrows * G + 255) / 256);
#define K4S_LAUNCH(PP, GG)                                                                                 \
  do {                                                                                                     \
    CK(cudaFuncSetAttribute(k4_seg<PP, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
    k4_seg<PP, GG><<<blocks, 256, smem, st>>>(rr, D.Q, D.st_s, D.st_t, g, D.seg, D.seg_maxseg, D.box_ptr,    \
                                              D.seg_moff, D.c_ptr, D.seg_mask, D.c_val, D.q, D.uloc, D.u); \
  } while (0)
#define K4S_BY_G(PP) \
  if (G <= 8) K4S_LAUNCH(PP, 8); else if (G == 16) K4S_LAUNCH(PP, 16); else K4S_LAUNCH(PP, 32)
    switch (D.order) {
      case 1: K4S_BY_G(1); break;
      case 2: K4S_BY_G(2); break;
      default: K4S_BY_G(3); break;
    }
#undef K4S_BY_G
#undef K4S_LAUNCH
  } else {
  const bool k4_kb4 = D.k4_kb4;
  switch (D.order) {
#define K4_LAUNCH(PP, GG)                                                                               \
  (D.cbox_format == 3                                                                                   \
       ? k4_interp_corr<PP, GG, 3><<<(unsigned)std::max<int64_t>(1, (nrows * GG + 255) / 256), 256, 0, st>>>(                \
             rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_hdr, D.c_bidx, v4,                                \
             reinterpret_cast<const float*>(D.q4), D.uloc, D.u, D.q4s)                                  \
   : D.cbox_format == 1                                                                                 \
       ? k4_interp_corr<PP, GG, 1><<<(unsigned)std::max<int64_t>(1, (nrows * GG + 255) / 256), 256, 0, st>>>(                \
             rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_hdr, D.c_bidx, v4, D.q, D.uloc, D.u, (int64_t)0)   \
   : D.k4_vec                                                                                           \
       ? k4_interp_corr<PP, GG, 2><<<(unsigned)std::max<int64_t>(1, (nrows * GG + 255) / 256), 256, 0, st>>>(                \
             rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_hdr, D.c_bidx, v4, D.q, D.uloc, D.u, (int64_t)0)   \
   : k4_kb4                                                                                             \
       ? k4_interp_corr<PP, GG, 4><<<(unsigned)std::max<int64_t>(1, (nrows * GG + 255) / 256), 256, 0, st>>>(                \
             rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_hdr, D.c_bidx, v4, D.q, D.uloc, D.u, (int64_t)0)   \
       : k4_interp_corr<PP, GG, 0><<<(unsigned)std::max<int64_t>(1, (nrows * GG + 255) / 256), 256, 0, st>>>(                \
             rr, D.Q, D.st_s, D.st_t, g, D.c_ptr, D.c_hdr, D.c_bidx, v4, D.q, D.uloc, D.u, (int64_t)0))
#define K4_BY_G(PP)                                                                                     \
  (D.k4_group == 4 ? K4_LAUNCH(PP, 4) : D.k4_group == 8 ? K4_LAUNCH(PP, 8) :                           \
   D.k4_group == 16 ? K4_LAUNCH(PP, 16) : K4_LAUNCH(PP, 32))
    case 1: K4_BY_G(1); break;
    case 2: K4_BY_G(2); break;
    default: K4_BY_G(3); break;
#undef K4_BY_G
#undef K4_LAUNCH
  }
  }
  CK(cudaGetLastError());
  halo(D, 2, D.u, 1, st);
  mark(4);
  if (split) k5_grad_sum<2><<<split_blocks, 256, 0, st>>>(rr, D.u, D.sl1_off, D.s_Gc, H, mode == EVAL_HEFF ? 1 : 0);
  else k5_grad_sum<1><<<thr_blocks, 256, 0, st>>>(rr, D.u, D.sl1_off, D.s_Gc, H, mode == EVAL_HEFF ? 1 : 0);
  CK(cudaGetLastError());
  mark(5);
}

}  // namespace pmfem

namespace pmfem {

// One classical RK4 step of the LLG equation on the rank-local rows of m (in place):
// 4 H_eff evaluations + 4 fused stage kernels (k_llg_stage).
static Anis anis_of(const DeviceState& D) {
  Anis a{D.anis_kind, (float)(2.0 * D.anis_K / D.anis_Ms), (float)D.anis_u[0], (float)D.anis_u[1], (float)D.anis_u[2]};
  return a;
}

static void llg_scratch(DeviceState& D, int64_t n) {
  if (!D.llg_ms) {
    D.llg_ms = dalloc<float>(3 * (size_t)std::max<int64_t>(n, 1));
    D.llg_H = dalloc<float>(3 * (size_t)std::max<int64_t>(n, 1));
    D.llg_acc = dalloc<float>(3 * (size_t)std::max<int64_t>(n, 1));
  }
}

void device_llg_rk4_step(DeviceState& D, float* m, cudaStream_t st, double dt, double alpha, double gamma,
                         const double Hap[3]) {
  const int64_t n = D.hi - D.lo;
  if (n <= 0 && D.world == 1) return;     // a row-less rank still joins the evaluations' collectives
  llg_scratch(D, n);
  const float g = (float)(gamma / (1.0 + alpha * alpha));
  const unsigned blocks = (unsigned)((n + 255) / 256);
  const float w[4] = {(float)(dt / 6), (float)(dt / 3), (float)(dt / 3), (float)(dt / 6)};
  const float c[4] = {(float)(dt / 2), (float)(dt / 2), (float)dt, 0.f};
  const Anis an = anis_of(D);
  for (int s = 0; s < 4; ++s) {
    const float* ms = (s == 0) ? m : D.llg_ms;
    device_eval(D, ms, D.llg_H, st, EVAL_HEFF);
    if (n > 0)
    k_llg_stage<<<blocks, 256, 0, st>>>(n, m, ms, D.llg_H, (float)Hap[0], (float)Hap[1], (float)Hap[2], an, g,
                                        (float)alpha, w[s], c[s], D.llg_acc, D.llg_ms, s == 0, s == 3);
    CK(cudaGetLastError());
  }
}

// Adaptive AM2 integration from t = 0 to t_end (oracle/llg.py am2_integrate): per attempt one
// predictor, one H_eff evaluation, one corrector with the error reduction (read back by the host
// to accept / reject), and on acceptance one more evaluation for f_{n+1}.  N > 1: the error is
// max-reduced over the ranks.
void device_llg_am2(DeviceState& D, float* m, cudaStream_t st, double t_end, double dt0, double tol, double alpha,
                    double gamma, const double Hap[3], double dt_max, int64_t* acc_out, int64_t* rej_out) {
  const int64_t n = D.hi - D.lo;
  llg_scratch(D, n);
  const size_t b = 3 * (size_t)std::max<int64_t>(n, 1) * sizeof(float);
  float *fn = nullptr, *fprev = nullptr, *mp = nullptr, *fp = nullptr;
  unsigned* err = nullptr;
  CK(cudaMalloc(&fn, b)); CK(cudaMalloc(&fprev, b)); CK(cudaMalloc(&mp, b)); CK(cudaMalloc(&fp, b));
  CK(cudaMalloc(&err, sizeof(unsigned)));
  struct Free { void* p[5]; ~Free() { for (void* x : p) cudaFree(x); } } fr{{fn, fprev, mp, fp, err}};
  const float g = (float)(gamma / (1.0 + alpha * alpha));
  const unsigned blocks = (unsigned)std::max<int64_t>(1, (n + 255) / 256), blocks3 = (unsigned)std::max<int64_t>(1, (3 * n + 255) / 256);
  const Anis an = anis_of(D);
  auto rhs = [&](const float* x, float* f) {
    device_eval(D, x, D.llg_H, st, EVAL_HEFF);
    if (n > 0) k_llg_rhs<<<blocks, 256, 0, st>>>(n, x, D.llg_H, (float)Hap[0], (float)Hap[1], (float)Hap[2], an, g, (float)alpha, f);
    CK(cudaGetLastError());
  };
  rhs(m, fn);
  double t = 0.0, dt = dt0, dt_prev = 0.0;
  int64_t acc = 0, rej = 0;
  while (t < t_end * (1 - 1e-12)) {
    dt = std::min(dt, t_end - t);
    if (dt_max > 0) dt = std::min(dt, dt_max);
    const double r = dt_prev > 0 ? dt / dt_prev : 0.0;
    if (n > 0) k_am2_pred<<<blocks3, 256, 0, st>>>(n, m, fn, fprev, (float)dt, (float)r, mp);
    CK(cudaGetLastError());
    rhs(mp, fp);
    CK(cudaMemsetAsync(err, 0, sizeof(unsigned), st));
    if (n > 0) k_am2_corr<<<blocks, 256, 0, st>>>(n, m, fn, fp, mp, (float)dt, D.llg_ms, err);
    CK(cudaGetLastError());
    if (D.world > 1) {
      ncclComm_t comm = (ncclComm_t)D.comm;
      NCK(ncclAllReduce(err, err, 1, ncclUint32, ncclMax, comm, st));
    }
    unsigned eb = 0;
    CK(cudaMemcpyAsync(&eb, err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ef;
    std::memcpy(&ef, &eb, sizeof(float));
    const double e = ef;
    const double fac = e == 0.0 ? 2.0 : std::min(2.0, std::max(0.2, 0.9 * std::cbrt(tol / e)));
    if (e <= tol) {
      t += dt;
      if (n > 0) CK(cudaMemcpyAsync(m, D.llg_ms, 3 * (size_t)n * sizeof(float), cudaMemcpyDeviceToDevice, st));
      std::swap(fprev, fn);
      rhs(m, fn);
      dt_prev = dt;
      ++acc;
    } else {
      ++rej;
    }
    dt *= fac;
    fr.p[0] = fn; fr.p[1] = fprev;
  }
  *acc_out = acc;
  *rej_out = rej;
}

}  // namespace pmfem

// ====================================================================================== NEXT-4
// Complex Bloch field path (host operators: setup_bloch.cpp, reading R27).
// m(r + R) = exp(-j k0.R) m(r) enters as two fp32 planes (re, im) in user order; internally
// every vector is complex (float2) in the box-sorted internal order.  The AIM grid part runs on
// the MODULATED charges q~ = exp(j k0.r) q with the L-periodic kernel G~ = exp(j k0.r) G_p:
// G~ = A + jB with A = Re G~ even and B = Im G~ odd, so both real grids Qr, Qi go through the
// real-to-complex FFT of the static path (K2 and the X/Y/Z passes reused unchanged) and meet in
// one pointwise 2x2 product of the half spectra,
//   Ur^ = A^ Qr^ - B^ Qi^,   Ui^ = A^ Qi^ + B^ Qr^   (A^ real, B^ = j fb imaginary).
namespace pmfem {

struct BlochDev {
  int64_t* r1_ptr = nullptr; int32_t* r1_col = nullptr; float2* r1_val = nullptr;   // 7 complex / entry
  int64_t* z_ptr = nullptr;  int32_t* z_col = nullptr;  float2* z_val = nullptr;    // 3 complex / entry
  int64_t* c_ptr = nullptr;  int32_t* c_col = nullptr;  float2* c_val = nullptr;    // 1 complex / entry
  float2* mod = nullptr;     // exp(j k0 . r_n), internal order
  float* fa = nullptr;       // half spectrum of Re G~ (real)
  float* fb = nullptr;       // half spectrum of Im G~ (imaginary part)
  float2* m = nullptr;       // [N'][3] internal
  float* qr = nullptr;       // modulated charges, re / im (K2 inputs, N' + 16 padded)
  float* qi = nullptr;
  float2* uloc = nullptr;    // Z0 potential
  float2* u = nullptr;       // total potential
  float* Q2 = nullptr;       // second real grid (Qi, then Ui)
  float2* C2 = nullptr;      // second half spectrum
  int64_t nnz[3] = {0, 0, 0};
};

namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, c.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, c.y)));
}

__global__ void kb_gather(int64_t Np, const float* __restrict__ mre, const float* __restrict__ mim,
                          float2* __restrict__ m) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * Np) return;
  m[i] = make_float2(mre[i], mim[i]);
}

// K1 (complex): q~ = exp(j k0.r) (D m), u_loc = Z0 m, H_ex = L m (into H) -- thread per row
__global__ void __launch_bounds__(256) kb_local(int64_t Np, const int64_t* __restrict__ r1_ptr,
                                                const int32_t* __restrict__ r1_col, const float2* __restrict__ r1_val,
                                                const int64_t* __restrict__ z_ptr, const int32_t* __restrict__ z_col,
                                                const float2* __restrict__ z_val, const float2* __restrict__ m,
                                                const float2* __restrict__ mod, float* __restrict__ qr, float* __restrict__ qi,
                                                float2* __restrict__ uloc, float* __restrict__ Hre,
                                                float* __restrict__ Him, int mode) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  float2 q = make_float2(0.f, 0.f), h[3] = {q, q, q};
  for (int64_t e = r1_ptr[n]; e < r1_ptr[n + 1]; ++e) {
    const int64_t c = r1_col[e];
    DCHECK(c >= 0 && c < Np);
    const float2* v = r1_val + 7 * e;
    const float2 mx = m[3 * c], my = m[3 * c + 1], mz = m[3 * c + 2];
    q = cfma(v[1], mx, cfma(v[2], my, cfma(v[3], mz, q)));
    h[0] = cfma(v[0], mx, h[0]); h[1] = cfma(v[0], my, h[1]); h[2] = cfma(v[0], mz, h[2]);
  }
  if (mode == EVAL_EXCHANGE || mode == EVAL_HEFF) {
    for (int x = 0; x < 3; ++x) { Hre[3 * n + x] = h[x].x; Him[3 * n + x] = h[x].y; }
  }
  if (mode == EVAL_EXCHANGE) return;
  float2 ul = make_float2(0.f, 0.f);
  for (int64_t e = z_ptr[n]; e < z_ptr[n + 1]; ++e) {
    const int64_t c = z_col[e];
    DCHECK(c >= 0 && c < Np);
    const float2* v = z_val + 3 * e;
    ul = cfma(v[0], m[3 * c], cfma(v[1], m[3 * c + 1], cfma(v[2], m[3 * c + 2], ul)));
  }
  uloc[n] = ul;
  const float2 qt = cmul(mod[n], q);
  qr[n] = qt.x;
  qi[n] = qt.y;
}

// pointwise product of the two half spectra with A^ (real) and B^ = j fb
__global__ void kb_spec_mul(int64_t tot, float2* __restrict__ Cr, float2* __restrict__ Ci,
                            const float* __restrict__ fa, const float* __restrict__ fb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tot) return;
  const float2 X = Cr[i], Y = Ci[i];
  const float a = fa[i], b = fb[i];
  Cr[i] = make_float2(fmaf(a, X.x, b * Y.y), fmaf(a, X.y, -b * Y.x));
  Ci[i] = make_float2(fmaf(a, Y.x, -b * X.y), fmaf(a, Y.y, b * X.x));
}

// K4 (complex): u = exp(-j k0.r) (P^T U + C~ q~) + u_loc -- thread per row
template <int P>
__global__ void __launch_bounds__(256) kb_interp_corr(int64_t Np, const float* __restrict__ Ur,
                                                      const float* __restrict__ Ui, const int4* __restrict__ st_s,
                                                      const float4* __restrict__ st_t, GridDims g,
                                                      const int64_t* __restrict__ c_ptr, const int32_t* __restrict__ c_col,
                                                      const float2* __restrict__ c_val, const float* __restrict__ qr,
                                                      const float* __restrict__ qi, const float2* __restrict__ mod,
                                                      const float2* __restrict__ uloc, float2* __restrict__ u) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  const int4 s = st_s[n];
  const float4 t = st_t[n];
  float wx[P + 1], wy[P + 1], wz[P + 1];
  lagr<P>(t.x, wx); lagr<P>(t.y, wy); lagr<P>(t.z, wz);
  float2 acc = make_float2(0.f, 0.f);
  for (int jz = 0; jz <= P; ++jz)
    for (int jy = 0; jy <= P; ++jy) {
      const int64_t row = ((int64_t)wrapi(s.z + jz, g.n2, g.per2) * g.n1 + wrapi(s.y + jy, g.n1, g.per1)) * g.n0;
      const float w = wy[jy] * wz[jz];
#pragma unroll
      for (int i = 0; i <= P; ++i) {
        const int64_t gi = row + wrapi(s.x + i, g.n0, g.per0);
        acc.x = fmaf(w * wx[i], Ur[gi], acc.x);
        acc.y = fmaf(w * wx[i], Ui[gi], acc.y);
      }
    }
  for (int64_t e = c_ptr[n]; e < c_ptr[n + 1]; ++e) {
    const int64_t c = c_col[e];
    DCHECK(c >= 0 && c < Np);
    acc = cfma(c_val[e], make_float2(qr[c], qi[c]), acc);
  }
  const float2 md = mod[n];
  const float2 ul = uloc[n];
  u[n] = make_float2(fmaf(md.x, acc.x, fmaf(md.y, acc.y, ul.x)), fmaf(md.x, acc.y, fmaf(-md.y, acc.x, ul.y)));
}

// K5 (complex): H = -G u (+ H_ex already in H for H_eff)
__global__ void __launch_bounds__(256) kb_grad(int64_t Np, const int64_t* __restrict__ r1_ptr,
                                               const int32_t* __restrict__ r1_col, const float2* __restrict__ r1_val,
                                               const float2* __restrict__ u, float* __restrict__ Hre, float* __restrict__ Him, int add) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  float2 h[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (int64_t e = r1_ptr[n]; e < r1_ptr[n + 1]; ++e) {
    const float2 uc = u[r1_col[e]];
    const float2* v = r1_val + 7 * e;
    h[0] = cfma(v[4], uc, h[0]); h[1] = cfma(v[5], uc, h[1]); h[2] = cfma(v[6], uc, h[2]);
  }
  for (int x = 0; x < 3; ++x) {
    const float ar = add ? Hre[3 * n + x] : 0.f, ai = add ? Him[3 * n + x] : 0.f;
    Hre[3 * n + x] = ar - h[x].x;
    Him[3 * n + x] = ai - h[x].y;
  }
}

// user-order complex CSR -> internal order, fp32
void csr_internal(const HostSetup& S, const Csr& R, int ncplx, int64_t*& ptr, int32_t*& col, float2*& val) {
  const int64_t Np = S.Np;
  std::vector<int64_t> p(Np + 1, 0);
  for (int64_t i = 0; i < Np; ++i) {
    const int64_t n = S.perm[i];
    p[i + 1] = p[i] + (R.rowptr[n + 1] - R.rowptr[n]);
  }
  std::vector<int32_t> c(p[Np]);
  std::vector<float2> v((size_t)ncplx * p[Np]);
#pragma omp parallel for
  for (int64_t i = 0; i < Np; ++i) {
    const int64_t n = S.perm[i];
    int64_t o = p[i];
    for (int64_t e = R.rowptr[n]; e < R.rowptr[n + 1]; ++e, ++o) {
      c[o] = (int32_t)S.iperm[R.col[e]];
      for (int k = 0; k < ncplx; ++k)
        v[(size_t)ncplx * o + k] = make_float2((float)R.val[2 * (ncplx * e + k)], (float)R.val[2 * (ncplx * e + k) + 1]);
    }
  }
  ptr = dupload(p);
  col = dupload(c);
  val = dupload(v);
}

}  // namespace

void device_bloch_free(DeviceState& D) {
  if (!D.bloch) return;
  BlochDev& B = *D.bloch;
  void* ptrs[] = {B.r1_ptr, B.r1_col, B.r1_val, B.z_ptr, B.z_col, B.z_val, B.c_ptr, B.c_col, B.c_val, B.mod,
                  B.fa, B.fb, B.m, B.qr, B.qi, B.uloc, B.u, B.Q2, B.C2};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete D.bloch;
  D.bloch = nullptr;
}

void device_bloch_upload(DeviceState& D, const HostSetup& S, const BlochHost& H) {
  CK(cudaSetDevice(D.device));
  device_bloch_free(D);
  D.bloch = new BlochDev();
  BlochDev& B = *D.bloch;
  const int64_t Np = S.Np;
  csr_internal(S, H.r1, 7, B.r1_ptr, B.r1_col, B.r1_val);
  csr_internal(S, H.z0, 3, B.z_ptr, B.z_col, B.z_val);
  csr_internal(S, H.cbox, 1, B.c_ptr, B.c_col, B.c_val);
  B.nnz[0] = H.r1.nnz(); B.nnz[1] = H.z0.nnz(); B.nnz[2] = H.cbox.nnz();
  std::vector<float2> md(Np);
  for (int64_t i = 0; i < Np; ++i) md[i] = make_float2((float)H.mod[2 * S.perm[i]], (float)H.mod[2 * S.perm[i] + 1]);
  B.mod = dupload(md);
  std::vector<float> fa(H.fa.begin(), H.fa.end()), fb(H.fb.begin(), H.fb.end());
  B.fa = dupload(fa);
  B.fb = dupload(fb);
  B.m = dalloc<float2>(3 * (size_t)Np);
  B.qr = dalloc<float>(Np + 16);
  B.qi = dalloc<float>(Np + 16);
  CK(cudaMemset(B.qr, 0, sizeof(float) * (Np + 16)));
  CK(cudaMemset(B.qi, 0, sizeof(float) * (Np + 16)));
  B.uloc = dalloc<float2>(Np);
  B.u = dalloc<float2>(Np);
  B.Q2 = dalloc<float>((size_t)D.n[0] * D.n[1] * D.n[2]);
  B.C2 = dalloc<float2>((size_t)D.H0 * D.P[1] * D.P[2]);
  CK(cudaDeviceSynchronize());
}

void device_bloch_eval(DeviceState& D, const float* m_re, const float* m_im, float* H_re, float* H_im,
                       cudaStream_t st, EvalMode mode) {
  require(D.bloch != nullptr, PMFEM_E_STATE, "pmfem_build_bloch has not been called");
  require(D.world == 1 && D.slab_world <= 1, PMFEM_E_STATE, "the Bloch field path is single-device");
  BlochDev& B = *D.bloch;
  const int64_t Np = D.Np;
  if (Np <= 0) return;
  const unsigned rb = (unsigned)((Np + 255) / 256);
  kb_gather<<<(unsigned)((3 * Np + 255) / 256), 256, 0, st>>>(Np, m_re, m_im, B.m);
  kb_local<<<rb, 256, 0, st>>>(Np, B.r1_ptr, B.r1_col, B.r1_val, B.z_ptr, B.z_col, B.z_val, B.m, B.mod, B.qr, B.qi, B.uloc, H_re, H_im, (int)mode);
  CK(cudaGetLastError());
  if (mode == EVAL_EXCHANGE) return;
  GridDims g{D.n[0], D.n[1], D.n[2], D.periodic[0], D.periodic[1], D.periodic[2]};
  {
    const TileDims td{D.k2_tile[0], D.k2_tile[1], D.k2_tile[2]};
    const unsigned nt = (unsigned)(((size_t)D.n[0] / td.t0) * (D.n[1] / td.t1) * (D.n[2] / td.t2));
    const size_t smem = sizeof(int) * ((size_t)3 * td.t0 * td.t1 * td.t2 + 2 * k2_nseg(td.t1, td.t2, D.order) + 1);
#define KB2_LAUNCH(PP)                                                                                          \
  do {                                                                                                          \
    CK(cudaFuncSetAttribute(k2_tile<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));              \
    k2_tile<PP><<<nt, 256, smem, st>>>(g, td, D.box_ptr, D.st_s, D.st_t, B.qr, 0, Np, D.box_max, 0, D.Q);      \
    k2_tile<PP><<<nt, 256, smem, st>>>(g, td, D.box_ptr, D.st_s, D.st_t, B.qi, 0, Np, D.box_max, 0, B.Q2);     \
  } while (0)
    switch (D.order) {
      case 1: KB2_LAUNCH(1); break;
      case 2: KB2_LAUNCH(2); break;
      default: KB2_LAUNCH(3); break;
    }
#undef KB2_LAUNCH
    CK(cudaGetLastError());
  }
  {
    const int n0 = D.n[0], n1 = D.n[1], n2 = D.n[2], P0 = D.P[0], P1 = D.P[1], P2 = D.P[2], H0 = D.H0;
    float* Qs[2] = {D.Q, B.Q2};
    float2* Cs[2] = {D.C, B.C2};
    for (int k = 0; k < 2; ++k) {
      launch_x<float>(true, Qs[k], Cs[k], nullptr, n1 * n2, n0, P0, n1, P1, D.tw32[0], st);
      launch_strided<float>(Cs[k], P1, H0, H0, n2, (long long)P1 * H0, n1, P1, 0, nullptr, 0, 0, D.tw32[1], st);
      launch_strided<float>(Cs[k], P2, (long long)P1 * H0, H0, P1, H0, n2, P2, 0, nullptr, 0, 0, D.tw32[2], st);
    }
    const int64_t tot = (int64_t)P2 * P1 * H0;
    kb_spec_mul<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tot, D.C, B.C2, B.fa, B.fb);
    CK(cudaGetLastError());
    for (int k = 0; k < 2; ++k) {
      launch_strided<float>(Cs[k], P2, (long long)P1 * H0, H0, P1, H0, P2, n2, 1, nullptr, 0, 0, D.tw32[2], st);
      launch_strided<float>(Cs[k], P1, H0, H0, n2, (long long)P1 * H0, P1, n1, 1, nullptr, 0, 0, D.tw32[1], st);
      launch_x<float>(false, nullptr, Cs[k], Qs[k], n1 * n2, n0, P0, n1, P1, D.tw32[0], st);
    }
  }
  switch (D.order) {
    case 1: kb_interp_corr<1><<<rb, 256, 0, st>>>(Np, D.Q, B.Q2, D.st_s, D.st_t, g, B.c_ptr, B.c_col, B.c_val, B.qr, B.qi,
                                                   B.mod, B.uloc, B.u); break;
    case 2: kb_interp_corr<2><<<rb, 256, 0, st>>>(Np, D.Q, B.Q2, D.st_s, D.st_t, g, B.c_ptr, B.c_col, B.c_val, B.qr, B.qi,
                                                   B.mod, B.uloc, B.u); break;
    default: kb_interp_corr<3><<<rb, 256, 0, st>>>(Np, D.Q, B.Q2, D.st_s, D.st_t, g, B.c_ptr, B.c_col, B.c_val, B.qr,
                                                    B.qi, B.mod, B.uloc, B.u); break;
  }
  CK(cudaGetLastError());
  kb_grad<<<rb, 256, 0, st>>>(Np, B.r1_ptr, B.r1_col, B.r1_val, B.u, H_re, H_im, mode == EVAL_HEFF ? 1 : 0);
  CK(cudaGetLastError());
}

}  // namespace pmfem
