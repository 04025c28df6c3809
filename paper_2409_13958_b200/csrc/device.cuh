// Device-side state of a context: fp32 operators in internal (box-sorted) order, the PGF
// spectrum, FFT twiddles and scratch.
#pragma once
#include <cassert>
#include <cuda_runtime.h>

// device-side bounds checks of the hot kernels, compiled in only for the checked build
// (build.py --checked, PMFEM_LIB=checked): the memory-safety evidence in place of
// compute-sanitizer, which is closed on the GPU pool
#ifdef PMFEM_DEVICE_CHECKS
#define DCHECK(c) assert(c)
#else
#define DCHECK(c) ((void)0)
#endif
#include <cstdint>
#include <vector>
#include "pmfem_internal.h"

namespace pmfem {

// slab-decomposed FFT: rank p owns the k0 columns [slab_h0, slab_h0 + slab_hn) of
// the H0-column half spectrum (uneven splits: the first H0 % W ranks get one more column)
__host__ __device__ __forceinline__ int slab_h0(int p, int H0, int W) { return p * (H0 / W) + (p < H0 % W ? p : H0 % W); }
__host__ __device__ __forceinline__ int slab_hn(int p, int H0, int W) { return H0 / W + (p < H0 % W ? 1 : 0); }

// ---- SEG C_box format (cbox_format 2): per row, the candidate columns are every node of the
// anchor boxes within +-R_a anchors of the row's own stored anchor on each axis (wrapped on
// periodic axes, clamped to [0, N-1-p] on non-periodic ones) -- a superset of the K8 near set,
// proven per row at build time.  Candidates are enumerated z-major, then y, then the x
// subranges of each (z, y) anchor line; rows are box-sorted, so each line contributes one or two
// CONTIGUOUS runs of columns [box_ptr(line + xa), box_ptr(line + xb + 1)).  A per-row bitmask over
// the candidates marks the near pairs; their values are stored contiguously in candidate order.
// No column indices are stored: K4 reads q along contiguous runs.
constexpr int SEG_MAXSEG = 512;
struct SegGeom {
  int R[3];      // candidate reach in anchors per axis
  int n[3];      // grid points per axis
  int per[3];    // periodic flags
  int lim[3];    // largest stored anchor per axis (N-1 periodic, N-1-p non-periodic)
};
// candidate anchor subranges of axis a for stored anchor s, in enumeration order: up to two
// [lo, hi] pairs in r (returns their number, >= 1)
__host__ __device__ __forceinline__ int seg_axis(const SegGeom& G, int a, int s, int* r) {
  const int N = G.n[a], R = G.R[a];
  if (G.per[a]) {
    if (2 * R + 1 >= N) { r[0] = 0; r[1] = N - 1; return 1; }
    const int lo = s - R, hi = s + R;
    if (lo < 0) { r[0] = lo + N; r[1] = N - 1; r[2] = 0; r[3] = hi; return 2; }
    if (hi >= N) { r[0] = lo; r[1] = N - 1; r[2] = 0; r[3] = hi - N; return 2; }
    r[0] = lo; r[1] = hi; return 1;
  }
  r[0] = s - R < 0 ? 0 : s - R;
  r[1] = s + R > G.lim[a] ? G.lim[a] : s + R;
  return 1;
}
__host__ __device__ __forceinline__ int seg_len(const int* r, int nr) {
  return (r[1] - r[0] + 1) + (nr == 2 ? r[3] - r[2] + 1 : 0);
}
// i-th anchor of the subranges r (i < seg_len)
__host__ __device__ __forceinline__ int seg_at(const int* r, int i) {
  const int l0 = r[1] - r[0] + 1;
  return i < l0 ? r[0] + i : r[2] + (i - l0);
}

constexpr int W4_TMAX = 128;   // W4 C_box: rows per tile (cbox_gpu.cu builder, K4 k4_win)
constexpr int W4_RMAX = 512;   // W4 C_box: runs per tile (the builder splits tiles above it)
constexpr int W4_CCAP = 2048;  // W4 TMA variant: chunks per tile (the tile's block staged in shared memory)

struct DeviceState {
  int device = -1;
  int64_t Np = 0;
  int order = 1;
  int periodic[3] = {0, 0, 0};
  int n[3] = {0, 0, 0}, P[3] = {0, 0, 0}, H0 = 0;
  // Local operators in SELL-32 (32 rows per slice, column-major inside a slice).  One shared
  // column list per row: the ring-1 columns first, then the Z0-only columns (2-ring at ring 1).
  int64_t nslices = 0;
  int64_t zt = 0, gt = 0;      // total SELL entries of the shared / ring-1 arrays (SoA plane strides)
  int64_t* sl_off = nullptr;   // [nslices+1] entry offsets of the shared col / Z arrays
  int64_t* sl1_off = nullptr;  // [nslices+1] entry offsets of the ring-1 value arrays
  float4* s_zc = nullptr;      // (Zx, Zy, Zz, column bits) per shared entry (padding: the row itself, 0)
  float4* s_LD = nullptr;      // (L, Dx, Dy, Dz) for the first sl1 width entries
  float4* s_Gc = nullptr;      // (Gx, Gy, Gz, column bits) for the first sl1 width entries
  float4* m4 = nullptr;        // [N'] internal float4 copy of m (one 16-byte gather per entry)
  float4* rowsum = nullptr;    // [N'][2] (sum_m D_nm, 0), (sum_m Z_nm, 0)
  // C_box in the C4x format (cbox_gpu.cu): per row a range of chunks of 4 column-sorted
  // entries; per chunk 4 fp32 values + a 64-bit header (base column, three 12-bit deltas)
  int64_t* c_ptr = nullptr;           // [N'+1] chunk offsets
  unsigned long long* c_hdr = nullptr;
  float* c_val = nullptr;             // [chunks][4]
  int64_t cbox_nnz = 0;               // near pairs (entries without chunk padding)
  int64_t cbox_chunks = 0;             // C4x chunks or B4 blocks
  int cbox_format = 0;                // 0: C4x, 1: B4 (aligned 4-column blocks, c_bidx + c_val), 2: SEG,
                                      // 3: U4 (unaligned 4-column blocks, start in c_bidx, q4 gathers)
  float4* q4 = nullptr;               // U4: per evaluation 4 shifted float4 copies of q (k_q4)
  int64_t q4s = 0;                    // U4: words per copy
  SegGeom seg{};                      // SEG: candidate geometry
  int seg_maxseg = 0;                 // SEG: largest number of column runs of a row
  int64_t* seg_moff = nullptr;        // SEG: [N'+1] mask word offsets (c_ptr holds the value offsets)
  uint32_t* seg_mask = nullptr;       // SEG: candidate bitmasks
  int64_t seg_mask_words = 0;
  int* c_bidx = nullptr;              // B4 block index (column >> 2) per block
  // W4 (cbox_format 5): tiles of consecutive own rows of one anchor line; per tile the runs of
  // internal rows forming its q window (staged in shared memory by K4) and per chunk the
  // window-local indices of its 4 entries
  int64_t w_ntiles = 0;
  int w_max = 0;                      // largest window (floats of shared memory)
  int w_umax = 0;                     // largest U sub-grid of a tile (odd line pitch x (P+1)^2 floats)
  bool w_tma = false;                 // PMFEM_W4_TMA=1: k4_win_tma (the tile's chunk block by cp.async.bulk)
  int64_t* w_trow = nullptr;          // [ntiles+1] first internal row of each tile
  int* w_rptr = nullptr;              // [ntiles+1] run offsets
  int* w_rstart = nullptr;            // run first internal row
  int* w_rlen = nullptr;              // run length
  int* w_rloc = nullptr;              // run offset in the window
  ushort4* w_idx = nullptr;           // [chunks] window-local indices
  int k4_group = 32;          // lanes per row in K4 (8/16/32 from the mean padded row length)
  // stencils
  int4* st_s = nullptr;       // wrapped (periodic) / clamped anchors
  int32_t* box_ptr = nullptr; // [G+1] first internal row of each anchor box (rows are box-sorted)
  int k2_tile[3] = {8, 8, 8}; // K2 grid tile per axis (divides n)
  int box_max = 1;            // largest anchor-box population (K2 fixed-point bound)
  int row_split = 1;          // K1/K5 threads per row (2 for small meshes)
  bool yz_half = false;       // fused YZ FFT with the z axis split into even/odd halves (PMFEM_YZ_HALF=1)
  bool k4_vec = false;        // C4x: vector q gathers for run chunks (PMFEM_K4_VEC=1)
  bool k4_stream = false;     // B4/U4: row-range streaming kernel (PMFEM_K4_STREAM=1)
  bool k4_kb4 = true;         // C4x: 4 batched chunks per lane (default; PMFEM_K4_KB=2 for 2)

  float4* st_t = nullptr;     // local coordinates t - s
  // PGF spectrum [P2][P1][H0] / (P0 P1 P2), fp32
  float* spec = nullptr;
  bool pgf_ready = false;
  // FFT plan + twiddles per axis (fp32 and fp64)
  int fused_tile = 0;          // > 0: fused YZ plan with this column tile
  float2* tw32[3] = {nullptr, nullptr, nullptr};
  double2* tw64[3] = {nullptr, nullptr, nullptr};
  // scratch
  float* q = nullptr;
  float* uloc = nullptr;
  float* u = nullptr;
  float* Q = nullptr;         // real grid [n2][n1][n0] (also holds U after the inverse)
  float2* C = nullptr;        // complex half spectrum [P2][P1][H0]
  float* m_stage = nullptr;   // pmfem_heff_host staging
  // slab-decomposed convolution (world > 1, or PMFEM_SLAB_SIM=W simulated ranks on one device)
  int slab_world = 1;
  std::vector<int> zpl;       // [slab_world+1] z-slab plane boundaries (variable thickness; the
                              // row partition's planes on N > 1, the same rule for the simulation)
  std::vector<int32_t> gsend[2], grecv[2];   // U ghost planes per peer (DistPlan)
  float2* slab_cx = nullptr;  // x-slab spectrum [P2][P1][H_r] (simulation: all ranks back to back)
  float2* slab_buf = nullptr; // transpose send / receive blocks [nzl][P1][H0]
  float* slab_spec = nullptr; // spectrum slice [P2][P1][H_r]
  float* H_stage = nullptr;
  // timing
  bool timing = false;
  bool timing_pending = false;
  cudaEvent_t ev[8] = {};
  float last_ms[8] = {0};
  double kernel_bytes[8] = {0};
  int launches_per_eval = 0;
  // multi-GPU (world > 1): this rank owns internal rows [lo, hi); gathered vectors are kept
  // full length (global column indices) and filled at owned + halo rows; the anterpolated
  // grid is all-reduced and the FFT convolution is replicated on every rank.
  int rank = 0, world = 1;
  int axperm[3] = {0, 1, 2};  // user axis of internal axis i (m / H components are permuted)
  int64_t lo = 0, hi = 0;
  void* comm = nullptr;                         // ncclComm_t
  std::vector<int64_t> send_ptr[3], recv_ptr[3];
  int32_t* send_idx[3] = {nullptr, nullptr, nullptr};
  int32_t* recv_idx[3] = {nullptr, nullptr, nullptr};
  float* send_buf = nullptr;
  float* recv_buf = nullptr;
  double comm_bytes_per_eval = 0;
  // captured evaluation graphs (pmfem_api.cu eval_graph)
  struct GraphSlot {
    const float* m = nullptr;
    float* H = nullptr;
    cudaStream_t st = nullptr;
    int mode = -1;
    bool timing = false;
    cudaGraphExec_t exec = nullptr;
  };
  GraphSlot graphs[4];
  int graph_next = 0;
  // LLG RK4 scratch (rank-local rows) and the captured RK4 step
  int anis_kind = 0;          // NEXT-2 anisotropy: 0 none, 1 uniaxial, 2 cubic (pmfem_set_anisotropy)
  double anis_K = 0, anis_Ms = 1, anis_u[3] = {0, 0, 1};
  float* llg_ms = nullptr;
  float* llg_H = nullptr;
  float* llg_acc = nullptr;
  cudaGraphExec_t llg_exec = nullptr;
  const float* llg_key_m = nullptr;
  cudaStream_t llg_key_st = nullptr;
  double llg_key[6] = {0, 0, 0, 0, 0, 0};
  struct BlochDev* bloch = nullptr;   // NEXT-4 complex field path (device_bloch_upload)
};

void device_llg_rk4_step(DeviceState& D, float* m, cudaStream_t st, double dt, double alpha, double gamma,
                         const double Hap[3]);
void device_llg_am2(DeviceState& D, float* m, cudaStream_t st, double t_end, double dt0, double tol, double alpha,
                    double gamma, const double Hap[3], double dt_max, int64_t* acc_out, int64_t* rej_out);

void device_init_comm(DeviceState& D, const HostSetup& S, const void* nccl_id);
int64_t device_build_cbox(DeviceState& D, const HostSetup& S);
void device_seg_decode(const DeviceState& D, int* d_col);

void device_upload(DeviceState& D, const HostSetup& S);
void device_build_pgf(DeviceState& D, const HostSetup& S, const PgfParams& P);
void device_bloch_table(DeviceState& D, const HostSetup& S, const PgfParams& P, const double k0[3],
                        std::vector<double>& K);
void device_free(DeviceState& D);
enum EvalMode { EVAL_HEFF = 0, EVAL_DEMAG = 1, EVAL_EXCHANGE = 2 };
// NEXT-4 complex Bloch field path (single device): operators from setup_bloch_ops, then
// H_re + j H_im = H(m_re + j m_im) for Bloch amplitudes m(r + R) = exp(-j k0.R) m(r)
void device_bloch_upload(DeviceState& D, const HostSetup& S, const BlochHost& B);
void device_bloch_eval(DeviceState& D, const float* m_re, const float* m_im, float* H_re, float* H_im,
                       cudaStream_t st, EvalMode mode);
void device_bloch_free(DeviceState& D);
void device_eval(DeviceState& D, const float* m, float* H, cudaStream_t st, EvalMode mode);

}  // namespace pmfem
