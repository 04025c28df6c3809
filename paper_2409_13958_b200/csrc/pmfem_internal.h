// Internal declarations of libpmfem (host setup in fp64, device path in fp32).
#pragma once
#include <cstdint>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>
#include "../../include/pmfem.h"

namespace pmfem {

struct Error : std::runtime_error {
  pmfem_status code;
  Error(pmfem_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void require(bool ok, pmfem_status code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// Sparse row-compressed matrix with a fixed number of fp64 values per entry.
struct Csr {
  int64_t n_rows = 0;
  int nv = 1;                       // values per entry
  std::vector<int64_t> rowptr;      // [n_rows+1]
  std::vector<int32_t> col;         // [nnz]
  std::vector<double> val;          // [nnz*nv]
  int64_t nnz() const { return (int64_t)col.size(); }
};

// One (row, element image) Z0 integration task for the GPU (z0_gpu.cu).
struct Z0Item {
  int64_t row;        // observer parent n
  int32_t tet;        // element id
  int32_t slot;       // position of row n in the integration chunk (value block)
  int16_t code;       // packed lattice shift of the element image
  int8_t va;          // local vertex that coincides with the observer, or -1
  uint8_t flags;      // bit j: local vertex j is a near source of row n
  int16_t pos[4];     // row-relative column slot of each local vertex
};

// Z0 near-set enumeration of one observer row (setup_z0.cpp; shared by the static and the Bloch
// operator builds): near(n) as (parent, packed lattice shift) pairs and the element images
// (key = tet * Z0_NC + packed shift) with the near-source vertex flags and the observer vertex.
constexpr int Z0_NC = 17 * 17 * 17;
struct Z0RowEnum {
  struct It { int64_t key; int va; unsigned flags; };
  std::vector<std::pair<int64_t, int>> near;
  std::vector<int64_t> U;           // scratch
  std::vector<It> its;
};

// Multi-GPU plan: contiguous internal-row ranges per rank and halo exchange index lists
// (internal row indices) for the gathered vectors M (m), Q (q), U (u).
struct DistPlan {
  int rank = 0, world = 1;
  std::vector<int64_t> bounds{0, 0};           // [world+1] internal row boundaries
  std::vector<int32_t> planes{0, 0};           // [world+1] slab boundaries (anchor z planes) of the
                                               // rows = the FFT's z slabs
  int qband_lo = 0, qband_hi = 0;              // q halo: rows anchored within these many planes
                                               // below / above the own slab (K2 stencils, C_box)
  // U ghost planes (K4's stencils reach p planes above the own slab): per peer, the contiguous
  // plane ranges (first plane, count) to send / receive; up to 2 ranges per peer (z wrap)
  std::vector<int32_t> gsend[2], grecv[2];     // [world] x (plane0, count) for range 0 / 1
  std::vector<int64_t> send_ptr[3], recv_ptr[3];  // [world+1] per peer
  std::vector<int32_t> send_idx[3], recv_idx[3];  // my rows to send / peer rows to receive
  int64_t lo() const { return bounds[rank]; }
  int64_t hi() const { return bounds[rank + 1]; }
};

// Host setup products (all in fp64, rows/cols in USER parent order [0, N')).
struct HostSetup {
  // inputs
  int64_t N = 0, T = 0;
  std::vector<double> xyz;          // [N][3]
  std::vector<int32_t> tets;        // [T][4] (oriented)
  std::vector<double> Ms_tet, Aex_tet;
  int periodic[3] = {0, 0, 0};
  double L[3] = {0, 0, 0};
  double match_tol = 0;
  int axperm[3] = {0, 1, 2};        // internal axis i = user axis axperm[i] (N > 1: the slab axis,
                                    // the longest grid axis, becomes internal z); every setup
                                    // artifact is in the internal frame, m / H in the user frame
  int touching = 0, protruding = 0;
  // PBC / LCA
  int64_t Np = 0;
  std::vector<int64_t> lca;         // [N] original index of the component root (min index)
  std::vector<int32_t> pid;         // [N] parent id
  std::vector<int64_t> parent;      // [Np] original node index of parent p
  std::vector<int32_t> shift;       // [N][3] integer lattice shift r_i = r_parent + shift*L
  std::vector<int64_t> copies_ptr;  // [Np+1] parent -> its copies (nodes), CSR
  std::vector<int64_t> copies;      // [N]
  std::vector<int64_t> ntet_ptr;    // [N+1] node -> incident tets, CSR
  std::vector<int64_t> ntet;        // [4T]
  // element data
  std::vector<double> vol;          // [T]
  std::vector<double> grads;        // [T][4][3]
  std::vector<double> Vt;           // [Np] lumped volume
  // operators (off-diagonal CSR + per-row sums), user parent order
  Csr ring1;                        // values: L, Dx, Dy, Dz, Gx, Gy, Gz   (nv = 7)
  std::vector<double> rowsumD;      // [Np][3] sum_m D_nm (non-zero on surfaces)
  std::vector<double> diagD;        // [Np][3] D_nn
  Csr z0;                           // values: Zx, Zy, Zz (nv = 3), off-diagonal
  std::vector<double> rowsumZ;      // [Np][3]
  // AIM
  int grid_n[3] = {0, 0, 0}, fft_n[3] = {0, 0, 0};
  double origin[3] = {0, 0, 0}, delta[3] = {0, 0, 0};
  int order = 1;
  double rer_scale = 2.0;
  int z0_ring = 1;
  int z0_device = -1;               // >= 0: Z0 element integrals run on this CUDA device
  std::vector<int64_t> z0_rows;     // rows (user parent ids) whose Z0 is built; empty = all rows
  std::vector<double> xw;           // [Np][3] wrapped parent coordinates
  std::vector<int32_t> st_s;        // [Np][3] unwrapped stencil start index
  std::vector<double> st_t;         // [Np][3] t - s (local coordinate in grid units)
  Csr cbox;                         // nv = 1 (empty when built on the device, cbox_device)
  bool cbox_device = false;         // device contexts build C_box on the GPU (cbox_gpu.cu)
  // internal order
  std::vector<int64_t> perm;        // internal row i -> user parent id
  std::vector<int64_t> iperm;       // user parent id -> internal row
  // PGF
  std::vector<double> kernel;       // host-only contexts: K table [fft2][fft1][fft0]
  std::vector<double> spectrum;     // host-only: G_hat half spectrum [fft2][fft1][fft0/2+1]
  std::vector<double> kernel_bloch, spectrum_bloch;   // NEXT-4 (complex interleaved, full grid)
  double k0[3] = {0, 0, 0};
  double setup_seconds = 0, pgf_seconds = 0;
  double pgf_achieved_rel_err = 0;
  DistPlan dist;
};

void setup_mesh(HostSetup& S, const pmfem_mesh* mesh, const pmfem_periodicity* per);
void setup_operators(HostSetup& S);
void setup_z0(HostSetup& S);
void z0_enumerate_row(const HostSetup& S, int64_t n, Z0RowEnum& W);
void z0_unpack_shift(int code, int s[3]);
// host C_box rows (K8/K9, fp64): nv = 1 static; with kb (internal-frame k0) nv = 2, the
// modulated Bloch precorrection (re, im)
void host_cbox_rows(const HostSetup& S, const double* kb, std::vector<std::vector<int32_t>>& rcol,
                    std::vector<std::vector<double>>& rval);
// NEXT-4 complex field path: Bloch-phased operators in USER parent order (setup_bloch.cpp)
struct BlochHost {
  double k0[3] = {0, 0, 0};         // internal frame
  Csr r1;                           // nv = 14: complex L, Dx, Dy, Dz, Gx, Gy, Gz (re, im), diagonal included
  Csr z0;                           // nv = 6: complex Zx, Zy, Zz, diagonal included
  Csr cbox;                         // nv = 2: complex modulated C~
  std::vector<double> mod;          // [Np][2] exp(j k0 . r_n), r_n the unwrapped parent coordinate
  std::vector<double> fa, fb;       // half spectra [P2][P1][H0] / #points of Re G~ (real) and Im G~ (imag part)
};
void setup_bloch_ops(const HostSetup& S, const double k0[3], BlochHost& B);
void setup_aim(HostSetup& S, const pmfem_grid* g);
void setup_order(HostSetup& S);
void setup_dist(HostSetup& S, int rank, int world);          // partition (needs setup_order)
void setup_dist_halos(HostSetup& S);                         // halo lists (needs Z0 of the own rows)
// slab boundaries (anchor z planes, multiples of gz) balancing the internal rows over `world`
// ranks; shared with the single-device slab simulation
std::vector<int32_t> slab_planes(const HostSetup& S, int world, int gz);
int slab_granularity(const HostSetup& S, int world);
struct TriRules;
void z0_device_begin(const HostSetup& S, const TriRules& rules);
void z0_device_end(std::vector<std::vector<double>>& rval);
void z0_device_integrate(const HostSetup& S, std::vector<std::vector<Z0Item>>& items,
                         const std::vector<std::vector<int32_t>>& rcol, std::vector<std::vector<double>>& rval,
                         const TriRules& rules, const int64_t* rows, int64_t nrows);

// Periodic Green's function (Ewald) -- host/device fp64, defined in pgf.cuh.
struct PgfParams {
  int dim;                // 1, 2, 3
  int ax[3];              // periodic axes first, then free axes
  double L[3];            // periods of the periodic axes (ax[0..dim-1])
  double alpha;
  int nreal[3];
  int mrec[3];
  double xr;              // real-space cutoff alpha * r_c
};
// Ewald parameters for a truncation target (clamped to [1e-16, 1e-2]): erfc(xr) and
// exp(-kmax^2 / 4 alpha^2) at 1e-2 x target
PgfParams make_pgf_params(const int periodic[3], const double L[3], double target = 1e-15);
// measured truncation error of P: max |K_P - K_P'| / max |K_P'| over probe displacements of the
// AIM grid, P' = P with enlarged cutoffs (0 in free space)
double pgf_truncation_error(const HostSetup& S, const PgfParams& P);
void gauss_legendre01(int n, double* x, double* w);
void host_kernel_table(const HostSetup& S, const PgfParams& P, std::vector<double>& K);
void host_fft_spectrum(const HostSetup& S, const std::vector<double>& K, std::vector<double>& Ghat);
// NEXT-4 Bloch-phase PGF: modulated kernel exp(j k0.r) G(r; k0) on the padded grid (complex,
// interleaved) and its full complex spectrum / #points
void bloch_grid_points(const HostSetup& S, int64_t idx, double r[3], bool& skip, bool& self);
void host_bloch_table(const HostSetup& S, const PgfParams& P, const double k0[3], std::vector<double>& K);
void host_bloch_spectrum(const HostSetup& S, const std::vector<double>& K, std::vector<double>& Gh);

}  // namespace pmfem
