// Device-side construction of the precorrection matrix C_box (BAIM step 4, P:208-232;
// contract K8/K9, readings R8/R9) directly in internal order, fp64 arithmetic, fp32 storage.
//   near set : all (n, k, img) with |x_n - x_k - img L| <= r_ER on every axis (closed),
//              min image on periodic axes (unique because r_ER < L/2)
//   entry    : G0*(d) - sum_{a in st(n), b in st(k)} w_na w_kb G0*((a - b - img N) o Delta)
// The host computes the same thing in setup_aim.cpp (used by host-only contexts and as the
// reference of the GPU test); device contexts build C_box here in seconds instead of minutes.
// Pass 1 counts the near pairs of every row, the host scans, pass 2 writes columns (in
// increasing order, by construction) and values; the rows are then packed into the C4x
// chunk format K4 streams (6 bytes per entry instead of 8 for a column + value CSR).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
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
  double L[3], delta[3], origin[3], rer;
};

__device__ __forceinline__ void lagr_d(double t, int p, double* w) {
  for (int j = 0; j <= p; ++j) {
    double v = 1.0;
    for (int i = 0; i <= p; ++i)
      if (i != j) v *= (t - i) / double(j - i);
    w[j] = v;
  }
}

// unclamped, unwrapped stencil anchor of coordinate x on axis a (contract K5)
__device__ __forceinline__ int anchor_of(const CboxGeom& c, double x, int a) {
  const double t = (x - c.origin[a]) / c.delta[a];
  return (c.p & 1) ? (int)floor(t) - (c.p - 1) / 2 : (int)floor(t + 0.5) - c.p / 2;
}

// Distinct stored anchors (wrapped on periodic axes, clamped otherwise) of every node whose
// coordinate can lie within r_ER of x on axis a, as up to two increasing ranges.  The margin
// of one anchor on each side covers the rounding of (x + img L) / Delta.
__device__ int cand_ranges(const CboxGeom& c, double x, int a, int* r) {
  int lo = anchor_of(c, x - c.rer, a) - 1, hi = anchor_of(c, x + c.rer, a) + 1;
  const int N = c.n[a];
  if (!c.per[a]) {
    lo = max(lo, 0); hi = min(hi, N - 1 - c.p);
    if (lo > hi) return 0;
    r[0] = lo; r[1] = hi; return 1;
  }
  if (hi - lo + 1 >= N) { r[0] = 0; r[1] = N - 1; return 1; }
  const int wl = ((lo % N) + N) % N, wh = ((hi % N) + N) % N;
  if (wl <= wh) { r[0] = wl; r[1] = wh; return 1; }
  r[0] = 0; r[1] = wh; r[2] = wl; r[3] = N - 1; return 2;
}

// Visit every near pair (k, img) of row n in increasing internal column order: internal rows
// are sorted by stored anchor box (x fastest) and box_ptr gives each box's row range, so
// candidate anchor lines (z, then y increasing) with their x ranges (increasing) enumerate
// the candidates in column order; the exact near test (K8) then selects the pairs.
template <class F>
__device__ void for_near(const CboxGeom& c, const double* __restrict__ xw, const int* __restrict__ box_ptr,
                         long long n, F&& f) {
  const double xn[3] = {xw[3 * n], xw[3 * n + 1], xw[3 * n + 2]};
  int rx[4], ry[4], rz[4];
  const int nx = cand_ranges(c, xn[0], 0, rx), ny = cand_ranges(c, xn[1], 1, ry), nz = cand_ranges(c, xn[2], 2, rz);
  for (int iz = 0; iz < nz; ++iz)
    for (int z = rz[2 * iz]; z <= rz[2 * iz + 1]; ++z)
      for (int iy = 0; iy < ny; ++iy)
        for (int y = ry[2 * iy]; y <= ry[2 * iy + 1]; ++y) {
          const long long line = ((long long)z * c.n[1] + y) * c.n[0];
          for (int ix = 0; ix < nx; ++ix) {
            const int k0 = box_ptr[line + rx[2 * ix]], k1 = box_ptr[line + rx[2 * ix + 1] + 1];
            for (int k = k0; k < k1; ++k) {
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
}

// rows r0 + [0, Np) (a rank's own rows); per-row outputs are indexed locally
__global__ void k_cbox_count(CboxGeom c, long long Np, long long r0, const double* __restrict__ xw,
                             const int* __restrict__ box_ptr, int* __restrict__ cnt) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Np) return;
  int k_cnt = 0;
  for_near(c, xw, box_ptr, r0 + i, [&](int, const double*, const int*) { ++k_cnt; });
  cnt[i] = k_cnt;
}

// C_box entry (K9) of the near pair (n, k, img): G0*(d) - sum_{a,b} w_na w_kb G0*((a - b - img N) o Delta),
// the double stencil sum regrouped per axis into the (2p+1)-point convolution cw of the two
// weight vectors (exact algebraic regrouping)
__device__ __forceinline__ double cbox_entry(const CboxGeom& c, const double (*wn)[4], const double* __restrict__ t_loc,
                                             const int* __restrict__ s_unw, long long n, int k, const double* d,
                                             const int* img) {
  const int p = c.p, p1 = p + 1, W = 2 * p + 1;
  const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  const double v = r > 0 ? 1.0 / r : 0.0;
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
  return v - gm;
}

__global__ void k_cbox_fill(CboxGeom c, long long Np, long long r0, const double* __restrict__ xw,
                            const int* __restrict__ box_ptr, const int* __restrict__ s_unw,
                            const double* __restrict__ t_loc, const long long* __restrict__ rowptr,
                            int* __restrict__ col, float* __restrict__ val) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Np) return;
  const long long n = r0 + i;
  double wn[3][4];
  for (int a = 0; a < 3; ++a) lagr_d(t_loc[3 * n + a], c.p, wn[a]);
  long long o = rowptr[i];
  for_near(c, xw, box_ptr, n, [&](int k, const double* d, const int* img) {
    col[o] = k;
    val[o] = (float)cbox_entry(c, wn, t_loc, s_unw, n, k, d, img);
    ++o;
  });
}

// ---- SEG: candidate enumeration (device.cuh seg_axis) shared by the builder and K4
template <class F>
__device__ void for_cand(const SegGeom& G, const int* __restrict__ box_ptr, int4 s, F&& f) {
  int rz[4], ry[4], rx[4];
  const int nz = seg_axis(G, 2, s.z, rz), ny = seg_axis(G, 1, s.y, ry), nx = seg_axis(G, 0, s.x, rx);
  const int lz = seg_len(rz, nz), ly = seg_len(ry, ny);
  int c = 0;
  for (int iz = 0; iz < lz; ++iz) {
    const int z = seg_at(rz, iz);
    for (int iy = 0; iy < ly; ++iy) {
      const long long line = ((long long)z * G.n[1] + seg_at(ry, iy)) * G.n[0];
      for (int ix = 0; ix < nx; ++ix) {
        const int k0 = box_ptr[line + rx[2 * ix]], k1 = box_ptr[line + rx[2 * ix + 1] + 1];
        for (int k = k0; k < k1; ++k) f(k, c++);
      }
    }
  }
}

// K8 near test of the candidate pair (n, k) with its minimum image (as for_near)
__device__ __forceinline__ bool near_pair(const CboxGeom& c, const double* xn, const double* __restrict__ xw, int k,
                                          double* d, int* img) {
  bool in = true;
  for (int a = 0; a < 3; ++a) {
    d[a] = xn[a] - xw[3 * (long long)k + a];
    img[a] = 0;
    if (c.per[a]) { img[a] = (int)rint(d[a] / c.L[a]); d[a] -= img[a] * c.L[a]; }
    in &= fabs(d[a]) <= c.rer;
  }
  return in;
}

// per row: near pairs among the candidates, candidate count, number of column runs
__global__ void k_seg_count(CboxGeom c, SegGeom G, long long Np, const double* __restrict__ xw,
                            const int* __restrict__ box_ptr, const int4* __restrict__ st, int* __restrict__ nnear,
                            int* __restrict__ ncand, int* __restrict__ nseg) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  const double xn[3] = {xw[3 * n], xw[3 * n + 1], xw[3 * n + 2]};
  int cnt = 0, cc = 0;
  for_cand(G, box_ptr, st[n], [&](int k, int) {
    double d[3];
    int img[3];
    cnt += near_pair(c, xn, xw, k, d, img);
    ++cc;
  });
  int rz[4], ry[4], rx[4];
  const int4 s = st[n];
  const int nz = seg_axis(G, 2, s.z, rz), ny = seg_axis(G, 1, s.y, ry), nx = seg_axis(G, 0, s.x, rx);
  nnear[n] = cnt;
  ncand[n] = cc;
  nseg[n] = seg_len(rz, nz) * seg_len(ry, ny) * nx;
}

__global__ void k_seg_fill(CboxGeom c, SegGeom G, long long Np, const double* __restrict__ xw,
                           const int* __restrict__ box_ptr, const int4* __restrict__ st, const int* __restrict__ s_unw,
                           const double* __restrict__ t_loc, const long long* __restrict__ moff,
                           const long long* __restrict__ voff, uint32_t* __restrict__ mask, float* __restrict__ val) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  const double xn[3] = {xw[3 * n], xw[3 * n + 1], xw[3 * n + 2]};
  double wn[3][4];
  for (int a = 0; a < 3; ++a) lagr_d(t_loc[3 * n + a], c.p, wn[a]);
  uint32_t bits = 0;
  long long o = voff[n];
  int last = -1;
  for_cand(G, box_ptr, st[n], [&](int k, int ci) {
    double d[3];
    int img[3];
    if (near_pair(c, xn, xw, k, d, img)) {
      bits |= 1u << (ci & 31);
      val[o++] = (float)cbox_entry(c, wn, t_loc, s_unw, n, k, d, img);
    }
    if ((ci & 31) == 31) { mask[moff[n] + (ci >> 5)] = bits; bits = 0; }
    last = ci;
  });
  if (last >= 0 && (last & 31) != 31) mask[moff[n] + (last >> 5)] = bits;
}

// expand SEG rows to (column, value) lists (pmfem_export of the device C_box, tests)
__global__ void k_seg_decode(SegGeom G, long long Np, const int* __restrict__ box_ptr, const int4* __restrict__ st,
                             const long long* __restrict__ moff, const long long* __restrict__ voff,
                             const uint32_t* __restrict__ mask, int* __restrict__ col) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long o = voff[n];
  for_cand(G, box_ptr, st[n], [&](int k, int ci) {
    if ((mask[moff[n] + (ci >> 5)] >> (ci & 31)) & 1u) col[o++] = k;
  });
}

// ---- C4x: chunks of 4 consecutive entries of a (column-sorted) row, per chunk a float4 of
// values and a 64-bit header = base column (28 bits) + three 12-bit column deltas.  A delta
// above 4095 (a jump to the next anchor plane) closes the chunk early; unused slots repeat
// the previous column (delta 0) with value 0, so every gathered q is one of the row's own.
constexpr int C4X_DBITS = 12;
constexpr long long C4X_DMAX = (1 << C4X_DBITS) - 1;

__global__ void k_c4x_count(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                            long long* __restrict__ nch) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long chunks = 0;
  int pos = 4, prev = 0;
  for (long long e = rowptr[n]; e < rowptr[n + 1]; ++e) {
    const int k = col[e];
    if (pos == 4 || k - prev > C4X_DMAX) { ++chunks; pos = 0; }
    ++pos; prev = k;
  }
  nch[n] = chunks;
}

__global__ void k_c4x_fill(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                           const float* __restrict__ val, const long long* __restrict__ cptr,
                           unsigned long long* __restrict__ hdr, float* __restrict__ cval) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long ch = cptr[n] - 1;
  int pos = 4, prev = 0;
  unsigned long long h = 0;
  for (long long e = rowptr[n]; e < rowptr[n + 1]; ++e) {
    const int k = col[e];
    if (pos == 4 || k - prev > C4X_DMAX) {
      if (ch >= cptr[n]) { for (; pos < 4; ++pos) cval[4 * ch + pos] = 0.f; hdr[ch] = h; }
      ++ch; pos = 0; h = (unsigned long long)k;
    } else {
      h |= (unsigned long long)(k - prev) << (28 + C4X_DBITS * (pos - 1));
    }
    cval[4 * ch + pos] = val[e];
    ++pos; prev = k;
  }
  if (ch >= cptr[n]) { for (; pos < 4; ++pos) cval[4 * ch + pos] = 0.f; hdr[ch] = h; }
}

// ---- B4: aligned blocks of 4 consecutive columns [4b, 4b+4) of a (column-sorted) row, per
// block a float4 of values (0 for columns outside the near set) and the int32 block index b.
// K4 then gathers q for a whole block with one aligned 16-byte load.  Chosen over C4x when
// the rows' near columns fill their blocks densely (long runs of consecutive columns).
__global__ void k_b4_count(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                           long long* __restrict__ nb) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long blocks = 0;
  int prev = -1;
  for (long long e = rowptr[n]; e < rowptr[n + 1]; ++e) {
    const int b = col[e] >> 2;
    if (b != prev) { ++blocks; prev = b; }
  }
  nb[n] = blocks;
}

__global__ void k_b4_fill(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                          const float* __restrict__ val, const long long* __restrict__ bptr,
                          int* __restrict__ bidx, float* __restrict__ bval) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long o = bptr[n] - 1;
  int prev = -1;
  for (long long e = rowptr[n]; e < rowptr[n + 1]; ++e) {
    const int b = col[e] >> 2;
    if (b != prev) {
      ++o; prev = b;
      bidx[o] = b;
      for (int j = 0; j < 4; ++j) bval[4 * o + j] = 0.f;
    }
    bval[4 * o + (col[e] & 3)] = val[e];
  }
}

// ---- U4: blocks of 4 consecutive columns [c, c+4) starting at ANY column c (greedy from the
// first uncovered entry of a column-sorted row: the fewest length-4 windows covering the row),
// per block a float4 of values (0 for columns outside the near set) and the int32 start c.  K4
// gathers q for a block with one 16-byte load of the per-evaluation array q4[c] = (q[c..c+3]),
// so blocks need no alignment and only run ends leave empty slots (B4 also wastes the slots
// before a run's first aligned boundary).
__global__ void k_u4_count(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                           long long* __restrict__ nb) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long blocks = 0;
  long long end = -1;                 // last column covered by the current block
  for (long long e = rowptr[n]; e < rowptr[n + 1]; ++e) {
    if (col[e] > end) { ++blocks; end = (long long)col[e] + 3; }
  }
  nb[n] = blocks;
}

__global__ void k_u4_fill(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                          const float* __restrict__ val, const long long* __restrict__ bptr,
                          int* __restrict__ bstart, float* __restrict__ bval) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Np) return;
  long long o = bptr[n] - 1;
  long long end = -1;
  int start = 0;
  for (long long e = rowptr[n]; e < rowptr[n + 1]; ++e) {
    if (col[e] > end) {
      ++o;
      start = col[e];
      end = (long long)start + 3;
      bstart[o] = start;
      for (int j = 0; j < 4; ++j) bval[4 * o + j] = 0.f;
    }
    bval[4 * o + (col[e] - start)] = val[e];
  }
}

// ---- W4: per own row, the CSR entries as nch = ceil(m/4) chunks of 4 with window-local
// indices: the run of the row's tile containing column k (runs of a tile sorted by first row;
// binary search) gives loc = run_loc + k - run_start.  Quarter-transposed: entry e of the row goes
// to chunk e mod nch, slot e / nch, so the 32 lanes of a K4 group reading chunks c..c+31 gather
// 32 CONSECUTIVE entries per slot -- consecutive window indices along a run, i.e. distinct
// shared-memory banks (with 4 consecutive entries per chunk the lanes' indices were 4 apart: a
// 4-way bank conflict on every gather).  Padding slots: value 0 at the row's first index.
// Columns outside the window are counted in *miss (the build then falls back to another format).
__global__ void k_w4_fill(long long Np, const long long* __restrict__ rowptr, const int* __restrict__ col,
                          const float* __restrict__ val, const int* __restrict__ tile_of, const int* __restrict__ rptr,
                          const int* __restrict__ rstart, const int* __restrict__ rlen, const int* __restrict__ rloc,
                          const long long* __restrict__ cptr, float* __restrict__ cval, unsigned short* __restrict__ cidx,
                          unsigned long long* __restrict__ miss) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Np) return;
  const int t = tile_of[i];
  const int r0 = rptr[t], r1 = rptr[t + 1];
  const long long c0 = cptr[i], nch = cptr[i + 1] - c0, m = rowptr[i + 1] - rowptr[i];
  unsigned short first = 0;
  for (long long j = 0; j < m; ++j) {
    const int k = col[rowptr[i] + j];
    int lo = r0, hi = r1 - 1;           // last run with start <= k
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rstart[mid] <= k) lo = mid; else hi = mid - 1;
    }
    unsigned short loc = 0;
    if (rstart[lo] <= k && k < rstart[lo] + rlen[lo]) loc = (unsigned short)(rloc[lo] + (k - rstart[lo]));
    else atomicAdd(miss, 1ull);
    if (j == 0) first = loc;
    const long long o = 4 * (c0 + j % nch) + j / nch;
    cidx[o] = loc;
    cval[o] = val[rowptr[i] + j];
  }
  for (long long j = m; j < 4 * nch; ++j) {
    const long long o = 4 * (c0 + j % nch) + j / nch;
    cidx[o] = first;
    cval[o] = 0.f;
  }
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

// Builds the C4x arrays D.c_ptr (chunk offsets) / D.c_hdr / D.c_val in internal order on the
// device.  Needs D.box_ptr (anchor-box row pointers of the internal order).  Returns the number
// of near pairs.
// SEG rows expanded to column lists (tests): col[voff[n] + j] for the j-th near pair of row n
void device_seg_decode(const DeviceState& D, int* d_col) {
  const unsigned blocks = (unsigned)((D.Np + 127) / 128);
  k_seg_decode<<<blocks, 128>>>(D.seg, D.Np, D.box_ptr, reinterpret_cast<const int4*>(D.st_s),
                                reinterpret_cast<const long long*>(D.seg_moff), reinterpret_cast<const long long*>(D.c_ptr),
                                D.seg_mask, d_col);
  CKC(cudaGetLastError());
  CKC(cudaDeviceSynchronize());
}

int64_t device_build_cbox(DeviceState& D, const HostSetup& S) {
  CKC(cudaSetDevice(D.device));
  const int64_t Nall = S.Np;
  const int64_t r0 = D.lo, Np = D.hi - D.lo;          // this rank's own rows
  if (Nall >= (int64_t(1) << 28)) throw Error(PMFEM_E_INVALID_ARG, "C4x column base holds 28 bits: N' < 2^28 required");
  const int p = S.order;
  CboxGeom c{};
  c.p = p;
  c.rer = S.rer_scale * std::max(S.delta[0], std::max(S.delta[1], S.delta[2]));
  std::vector<double> xw(3 * Nall), tl(3 * Nall);
  std::vector<int> su(3 * Nall);
  for (int64_t i = 0; i < Nall; ++i) {
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
    c.origin[a] = S.origin[a];
  }
  double* d_xw = dup_c(xw);
  double* d_tl = dup_c(tl);
  int* d_su = dup_c(su);
  int* d_cnt = dalloc_c<int>(Np);
  const unsigned blocks = (unsigned)((Np + 127) / 128);
  k_cbox_count<<<blocks, 128>>>(c, Np, r0, d_xw, D.box_ptr, d_cnt);
  CKC(cudaGetLastError());
  std::vector<int> cnt(Np);
  CKC(cudaMemcpy(cnt.data(), d_cnt, sizeof(int) * Np, cudaMemcpyDeviceToHost));
  std::vector<long long> ptr(Np + 1, 0);
  for (int64_t i = 0; i < Np; ++i) ptr[i + 1] = ptr[i] + cnt[i];
  const int64_t nnz = ptr[Np];
  // ---- SEG (opt-in, PMFEM_CBOX_FORMAT=seg; measured slower: per-row run tables and a serial
  // mask walk are latency-bound, profiles/ab/r02_*): candidate reach R_a = ceil(rho_a + 1) - 1, rho_a = r_ER / Delta_a; usable
  // when every row's near set (the for_near count above) is found among its candidates
  const char* fmt_env = std::getenv("PMFEM_CBOX_FORMAT");
  const std::string fmt = fmt_env ? std::string(fmt_env) : std::string("auto");
  if (fmt == "seg" && D.world == 1) {
    SegGeom G{};
    for (int a = 0; a < 3; ++a) {
      const double rho = c.rer / c.delta[a];
      G.R[a] = (int)std::ceil(rho + 1.0) - 1;
      G.n[a] = c.n[a];
      G.per[a] = c.per[a];
      G.lim[a] = c.per[a] ? c.n[a] - 1 : c.n[a] - 1 - p;
    }
    int* d_near = dalloc_c<int>(Np);
    int* d_cand = dalloc_c<int>(Np);
    int* d_nseg = dalloc_c<int>(Np);
    const int4* d_st = reinterpret_cast<const int4*>(D.st_s);
    k_seg_count<<<blocks, 128>>>(c, G, Np, d_xw, D.box_ptr, d_st, d_near, d_cand, d_nseg);
    CKC(cudaGetLastError());
    std::vector<int> nnear(Np), ncand(Np), nseg(Np);
    CKC(cudaMemcpy(nnear.data(), d_near, sizeof(int) * Np, cudaMemcpyDeviceToHost));
    CKC(cudaMemcpy(ncand.data(), d_cand, sizeof(int) * Np, cudaMemcpyDeviceToHost));
    CKC(cudaMemcpy(nseg.data(), d_nseg, sizeof(int) * Np, cudaMemcpyDeviceToHost));
    bool ok = true;
    int maxseg = 0;
    for (int64_t i = 0; i < Np && ok; ++i) {
      ok = nnear[i] == cnt[i];
      maxseg = std::max(maxseg, nseg[i]);
    }
    if (ok && maxseg <= SEG_MAXSEG) {
      std::vector<long long> moff(Np + 1, 0), voff(Np + 1, 0);
      for (int64_t i = 0; i < Np; ++i) {
        moff[i + 1] = moff[i] + (ncand[i] + 31) / 32;
        voff[i + 1] = voff[i] + nnear[i];
      }
      long long* d_moff = dup_c(moff);
      long long* d_voff = dup_c(voff);
      uint32_t* d_mask = dalloc_c<uint32_t>(moff[Np]);
      float* d_val = dalloc_c<float>(voff[Np] + 4);
      CKC(cudaMemset(d_mask, 0, sizeof(uint32_t) * std::max<long long>(moff[Np], 1)));
      CKC(cudaMemset(d_val, 0, sizeof(float) * (voff[Np] + 4)));
      k_seg_fill<<<blocks, 128>>>(c, G, Np, d_xw, D.box_ptr, d_st, d_su, d_tl, d_moff, d_voff, d_mask, d_val);
      CKC(cudaGetLastError());
      CKC(cudaDeviceSynchronize());
      D.c_ptr = reinterpret_cast<int64_t*>(d_voff);
      D.seg_moff = reinterpret_cast<int64_t*>(d_moff);
      D.seg_mask = d_mask;
      D.c_val = d_val;
      D.seg = G;
      D.seg_maxseg = maxseg;
      D.seg_mask_words = moff[Np];
      D.cbox_chunks = moff[Np];
      D.cbox_format = 2;
      D.cbox_nnz = nnz;
      cudaFree(d_near); cudaFree(d_cand); cudaFree(d_nseg);
      cudaFree(d_xw); cudaFree(d_tl); cudaFree(d_su); cudaFree(d_cnt);
      return nnz;
    }
    cudaFree(d_near); cudaFree(d_cand); cudaFree(d_nseg);
    if (std::getenv("PMFEM_VERBOSE"))
      std::fprintf(stderr, "[pmfem] SEG C_box not usable (near sets %s, max runs %d): packed format\n",
                   ok ? "covered" : "NOT covered", maxseg);
  }
  long long* d_ptr = dup_c(ptr);
  int* d_col = dalloc_c<int>(nnz);
  float* d_val = dalloc_c<float>(nnz);
  k_cbox_fill<<<blocks, 128>>>(c, Np, r0, d_xw, D.box_ptr, d_su, d_tl, d_ptr, d_col, d_val);
  CKC(cudaGetLastError());
  // sizes of both packed formats: C4x chunks (24 B) and B4 blocks (20 B)
  long long* d_nch = dalloc_c<long long>(Np);
  k_c4x_count<<<blocks, 128>>>(Np, d_ptr, d_col, d_nch);
  CKC(cudaGetLastError());
  std::vector<long long> nch(Np), cptr(Np + 1, 0), nbk(Np), bptr(Np + 1, 0);
  CKC(cudaMemcpy(nch.data(), d_nch, sizeof(long long) * Np, cudaMemcpyDeviceToHost));
  k_b4_count<<<blocks, 128>>>(Np, d_ptr, d_col, d_nch);
  CKC(cudaGetLastError());
  CKC(cudaMemcpy(nbk.data(), d_nch, sizeof(long long) * Np, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < Np; ++i) { cptr[i + 1] = cptr[i] + nch[i]; bptr[i + 1] = bptr[i] + nbk[i]; }
  // U4: never more blocks than B4 (greedy unaligned covering), one 16-byte gather per block from
  // four shifted copies of q (4x q's footprint).  Measured (round 2, p = 3, s = 4, batched
  // gathers; profiles/ab): U4 wins where the near columns form long runs and q is dense in the
  // boxes (C4 9.64 vs C4x 9.87 ms, C5 2.03 vs B4 2.21 ms), C4x where the runs are short and
  // sparse (C3, 0.74 nodes per box: 0.53 vs U4 0.73 ms).  Default: U4 when the mesh has >= 1
  // node per grid box and U4 blocks hold >= 3.1 of their 4 slots, else C4x;
  // PMFEM_CBOX_FORMAT=c4x|b4|u4|seg forces a format (tests, A/B)
  std::vector<long long> nu(Np), uptr(Np + 1, 0);
  k_u4_count<<<blocks, 128>>>(Np, d_ptr, d_col, d_nch);
  CKC(cudaGetLastError());
  CKC(cudaMemcpy(nu.data(), d_nch, sizeof(long long) * Np, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < Np; ++i) uptr[i + 1] = uptr[i] + nu[i];
  // ---- W4 (windowed, format 5): tiles of consecutive own rows of one anchor (y, z) line; the
  // window of a tile = the rows of the anchor boxes within the candidate reach R_a (as SEG:
  // R_a = ceil(r_ER / Delta_a + 1) - 1, stored anchors) of the tile's boxes, as runs of internal
  // rows; a tile is halved until its window fits W4_WMAX floats of shared memory.  Every near
  // column must fall in its row's window (checked: otherwise another format is used).
  // W4 by default on dense meshes (>= 1 node per grid box: C2, C5 -- measured K4 0.24 vs 0.27 ms
  // and 1.79 vs 2.34 ms against U4); sparse ones (C3 0.74, C4 0.61 nodes per box) keep C4x
  // (W4 measured 0.59-0.80 vs 0.53 ms at C3, 9.4-10.7 vs 10.0-10.1 ms at C4: their tiles hold
  // fewer rows per window)
  const double per_box_w = (double)Nall / ((double)c.n[0] * c.n[1] * c.n[2]);
  if (fmt == "w4" || (fmt == "auto" && D.world == 1 && per_box_w >= 1.0)) {
    const int W4_WMAX = std::getenv("PMFEM_W4_WMAX") ? std::atoi(std::getenv("PMFEM_W4_WMAX")) : 6144;
    const bool w4_tma = std::getenv("PMFEM_W4_TMA") != nullptr && std::atoi(std::getenv("PMFEM_W4_TMA")) == 1;
    int R[3], lim[3];
    for (int a = 0; a < 3; ++a) {
      R[a] = (int)std::ceil(c.rer / c.delta[a] + 1.0) - 1;
      lim[a] = c.per[a] ? c.n[a] - 1 : c.n[a] - 1 - p;
    }
    // stored anchors (wrapped / clamped) of the internal rows and the anchor-box row pointers
    std::vector<int> an(3 * Nall);
    for (int64_t i = 0; i < Nall; ++i)
      for (int a = 0; a < 3; ++a) {
        int v = su[3 * i + a];
        if (c.per[a]) v = ((v % c.n[a]) + c.n[a]) % c.n[a];
        an[3 * i + a] = v;
      }
    const int64_t nbox = (int64_t)c.n[0] * c.n[1] * c.n[2];
    std::vector<int64_t> bp(nbox + 1, 0);
    for (int64_t i = 0; i < Nall; ++i) bp[((int64_t)an[3 * i + 2] * c.n[1] + an[3 * i + 1]) * c.n[0] + an[3 * i] + 1]++;
    for (int64_t b = 0; b < nbox; ++b) bp[b + 1] += bp[b];
    // anchor ranges of axis a around [lo, hi] (stored anchors), up to two increasing ranges
    auto ranges = [&](int a, int lo, int hi, int* r) {
      const int N = c.n[a];
      lo -= R[a]; hi += R[a];
      if (!c.per[a]) { r[0] = std::max(lo, 0); r[1] = std::min(hi, lim[a]); return r[0] <= r[1] ? 1 : 0; }
      if (hi - lo + 1 >= N) { r[0] = 0; r[1] = N - 1; return 1; }
      const int wl = ((lo % N) + N) % N, wh = ((hi % N) + N) % N;
      if (wl <= wh) { r[0] = wl; r[1] = wh; return 1; }
      r[0] = 0; r[1] = wh; r[2] = wl; r[3] = N - 1; return 2;
    };
    std::vector<int64_t> trow;
    std::vector<int> rptr(1, 0), rstart, rlen, rloc, tile_of(Np);
    std::vector<std::pair<int64_t, int64_t>> runs;
    auto window = [&](int64_t i0, int64_t i1) {      // runs of the window of own rows [i0, i1)
      runs.clear();
      const int y = an[3 * i0 + 1], z = an[3 * i0 + 2];
      int xa = an[3 * i0], xb = an[3 * (i1 - 1)];
      int rx[4], ry[4], rz[4];
      const int nx = ranges(0, xa, xb, rx), ny = ranges(1, y, y, ry), nz = ranges(2, z, z, rz);
      int64_t tot = 0;
      for (int iz = 0; iz < nz; ++iz)
        for (int zz = rz[2 * iz]; zz <= rz[2 * iz + 1]; ++zz)
          for (int iy = 0; iy < ny; ++iy)
            for (int yy = ry[2 * iy]; yy <= ry[2 * iy + 1]; ++yy) {
              const int64_t line = ((int64_t)zz * c.n[1] + yy) * c.n[0];
              for (int ix = 0; ix < nx; ++ix) {
                const int64_t k0 = bp[line + rx[2 * ix]], k1 = bp[line + rx[2 * ix + 1] + 1];
                if (k1 > k0) { runs.push_back({k0, k1 - k0}); tot += k1 - k0; }
              }
            }
      return tot;
    };
    int wmax = 0, umax = 0;
    bool fits = true;
    for (int64_t i = r0; i < r0 + Np && fits;) {
      int64_t j = i + 1;
      while (j < r0 + Np && j - i < W4_TMAX && an[3 * j + 1] == an[3 * i + 1] && an[3 * j + 2] == an[3 * i + 2]) ++j;
      // TMA variant: the tile's chunk block must fit the shared-memory stage (W4_CCAP chunks)
      if (w4_tma) {
        int64_t ch = 0, k = i;
        for (; k < j; ++k) {
          const int64_t ck = (cnt[k - r0] + 3) / 4;
          if (k > i && ch + ck > W4_CCAP - 2) break;
          ch += ck;
        }
        j = k;
      }
      int64_t w = window(i, j);
      while ((w > W4_WMAX || runs.size() > (size_t)W4_RMAX) && j - i > 1) { j = i + (j - i) / 2; w = window(i, j); }
      if (w > W4_WMAX || w > 65535 || runs.size() > (size_t)W4_RMAX) { fits = false; break; }
      std::sort(runs.begin(), runs.end());
      int loc = 0;
      for (auto& rn : runs) { rstart.push_back((int)rn.first); rlen.push_back((int)rn.second); rloc.push_back(loc); loc += (int)rn.second; }
      rptr.push_back((int)rstart.size());
      for (int64_t k = i; k < j; ++k) tile_of[k - r0] = (int)trow.size();
      trow.push_back(i);
      wmax = std::max<int>(wmax, (int)w);
      umax = std::max<int>(umax, ((an[3 * (j - 1)] - an[3 * i] + p + 1) | 1) * (p + 1) * (p + 1));
      i = j;
    }
    trow.push_back(r0 + Np);
    if (fits) {
      std::vector<long long> wptr(Np + 1, 0);
      for (int64_t i = 0; i < Np; ++i) wptr[i + 1] = wptr[i] + (cnt[i] + 3) / 4;
      long long* d_wptr = dup_c(wptr);
      int* d_tof = dup_c(tile_of);
      int* d_rptr = dup_c(rptr);
      int* d_rs = dup_c(rstart);
      int* d_rl = dup_c(rlen);
      int* d_rc = dup_c(rloc);
      // + 2 chunks: the TMA variant copies from an even chunk index in whole 16-byte units
      float* d_wval = dalloc_c<float>(4 * ((size_t)wptr[Np] + 2));
      unsigned short* d_widx = dalloc_c<unsigned short>(4 * ((size_t)wptr[Np] + 2));
      CKC(cudaMemset(d_wval + 4 * (size_t)wptr[Np], 0, 8 * sizeof(float)));
      CKC(cudaMemset(d_widx + 4 * (size_t)wptr[Np], 0, 8 * sizeof(unsigned short)));
      unsigned long long* d_miss = dalloc_c<unsigned long long>(1);
      CKC(cudaMemset(d_miss, 0, sizeof(unsigned long long)));
      k_w4_fill<<<blocks, 128>>>(Np, d_ptr, d_col, d_val, d_tof, d_rptr, d_rs, d_rl, d_rc, d_wptr, d_wval, d_widx, d_miss);
      CKC(cudaGetLastError());
      unsigned long long miss = 0;
      CKC(cudaMemcpy(&miss, d_miss, sizeof(miss), cudaMemcpyDeviceToHost));
      cudaFree(d_miss); cudaFree(d_tof);
      if (miss == 0) {
        D.c_ptr = reinterpret_cast<int64_t*>(d_wptr);
        D.c_val = d_wval;
        D.w_idx = reinterpret_cast<ushort4*>(d_widx);
        D.w_trow = dup_c(trow);
        D.w_rptr = d_rptr; D.w_rstart = d_rs; D.w_rlen = d_rl; D.w_rloc = d_rc;
        D.w_ntiles = (int64_t)trow.size() - 1;
        D.w_max = std::max(wmax, 1);
        D.w_umax = umax;
        D.w_tma = w4_tma;
        D.cbox_chunks = wptr[Np];
        D.cbox_format = 5;
        if (std::getenv("PMFEM_VERBOSE"))
          std::fprintf(stderr, "[pmfem] W4 C_box: %lld tiles, %zu runs, largest window %d rows\n",
                       (long long)D.w_ntiles, rstart.size(), wmax);
        CKC(cudaDeviceSynchronize());
        cudaFree(d_xw); cudaFree(d_tl); cudaFree(d_su); cudaFree(d_cnt); cudaFree(d_nch);
        cudaFree(d_ptr); cudaFree(d_col); cudaFree(d_val);
        D.cbox_nnz = nnz;
        return nnz;
      }
      cudaFree(d_wptr); cudaFree(d_rptr); cudaFree(d_rs); cudaFree(d_rl); cudaFree(d_rc); cudaFree(d_wval);
      cudaFree(d_widx);
    }
    if (std::getenv("PMFEM_VERBOSE"))
      std::fprintf(stderr, "[pmfem] W4 C_box not usable (%s): packed format\n", fits ? "near columns outside a window" : "window too large");
  }
  const double per_box = (double)Nall / ((double)c.n[0] * c.n[1] * c.n[2]);
  const double u4_fill = uptr[Np] ? (double)nnz / (double)uptr[Np] : 4.0;
  bool use_b4 = fmt == "b4";
  bool use_c4x = fmt == "c4x";
  if (fmt != "b4" && fmt != "c4x" && fmt != "u4") use_c4x = !(per_box >= 1.0 && u4_fill >= 3.1);
  if (!use_b4 && !use_c4x) {
    long long* d_uptr = dup_c(uptr);
    int* d_ustart = dalloc_c<int>(uptr[Np]);
    float* d_uval = dalloc_c<float>(4 * uptr[Np]);
    k_u4_fill<<<blocks, 128>>>(Np, d_ptr, d_col, d_val, d_uptr, d_ustart, d_uval);
    CKC(cudaGetLastError());
    D.c_ptr = reinterpret_cast<int64_t*>(d_uptr);
    D.c_bidx = d_ustart;
    D.c_val = d_uval;
    D.cbox_chunks = uptr[Np];
    D.cbox_format = 3;
  } else if (use_b4) {
    long long* d_bptr = dup_c(bptr);
    int* d_bidx = dalloc_c<int>(bptr[Np]);
    float* d_bval = dalloc_c<float>(4 * bptr[Np]);
    k_b4_fill<<<blocks, 128>>>(Np, d_ptr, d_col, d_val, d_bptr, d_bidx, d_bval);
    CKC(cudaGetLastError());
    D.c_ptr = reinterpret_cast<int64_t*>(d_bptr);
    D.c_bidx = d_bidx;
    D.c_val = d_bval;
    D.cbox_chunks = bptr[Np];
    D.cbox_format = 1;
  } else {
    long long* d_cptr = dup_c(cptr);
    unsigned long long* d_hdr = dalloc_c<unsigned long long>(cptr[Np]);
    float* d_cval = dalloc_c<float>(4 * cptr[Np]);
    k_c4x_fill<<<blocks, 128>>>(Np, d_ptr, d_col, d_val, d_cptr, d_hdr, d_cval);
    CKC(cudaGetLastError());
    D.c_ptr = reinterpret_cast<int64_t*>(d_cptr);
    D.c_hdr = d_hdr;
    D.c_val = d_cval;
    D.cbox_chunks = cptr[Np];
    D.cbox_format = 0;
  }
  CKC(cudaDeviceSynchronize());
  cudaFree(d_xw); cudaFree(d_tl); cudaFree(d_su); cudaFree(d_cnt); cudaFree(d_nch);
  cudaFree(d_ptr); cudaFree(d_col); cudaFree(d_val);
  D.cbox_nnz = nnz;
  return nnz;
}

}  // namespace pmfem
