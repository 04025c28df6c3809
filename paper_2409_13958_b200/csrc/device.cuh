// Device-side state of a context: fp32 operators in internal (box-sorted) order, the PGF
// spectrum, FFT twiddles and scratch.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>
#include "pmfem_internal.h"

namespace pmfem {

struct DeviceState {
  int device = -1;
  int64_t Np = 0;
  int order = 1;
  int periodic[3] = {0, 0, 0};
  int n[3] = {0, 0, 0}, P[3] = {0, 0, 0}, H0 = 0;
  // ring-1 operators (off-diagonal, difference form)
  int64_t* r1_ptr = nullptr;  int32_t* r1_col = nullptr;
  float4* r1_LD = nullptr;    // (L, Dx, Dy, Dz)
  float4* r1_G = nullptr;     // (Gx, Gy, Gz, 0)
  float4* rowsumD = nullptr;  // (sum_m D_nm, 0)
  // Z0 (off-diagonal) + row sums
  int64_t* z_ptr = nullptr;   int32_t* z_col = nullptr;
  float4* z_val = nullptr;    // (Zx, Zy, Zz, 0)
  float4* rowsumZ = nullptr;
  // C_box
  int64_t* c_ptr = nullptr;   int32_t* c_col = nullptr;
  float* c_val = nullptr;
  // stencils
  int4* st_s = nullptr;       // wrapped (periodic) / clamped anchors
  float4* st_t = nullptr;     // local coordinates t - s
  // PGF spectrum [P2][P1][H0] / (P0 P1 P2), fp32
  float* spec = nullptr;
  bool pgf_ready = false;
  // FFT twiddles per axis (fp32 and fp64)
  float2* tw32[3] = {nullptr, nullptr, nullptr};
  double2* tw64[3] = {nullptr, nullptr, nullptr};
  // scratch
  float* q = nullptr;
  float* uloc = nullptr;
  float* u = nullptr;
  float* Q = nullptr;         // real grid [n2][n1][n0] (also holds U after the inverse)
  float2* C = nullptr;        // complex half spectrum [P2][P1][H0]
  float* m_stage = nullptr;   // pmfem_heff_host staging
  float* H_stage = nullptr;
  // timing
  bool timing = false;
  bool timing_pending = false;
  cudaEvent_t ev[8] = {};
  float last_ms[8] = {0};
  double kernel_bytes[8] = {0};
};

void device_upload(DeviceState& D, const HostSetup& S);
void device_build_pgf(DeviceState& D, const HostSetup& S, const PgfParams& P);
void device_free(DeviceState& D);
enum EvalMode { EVAL_HEFF = 0, EVAL_DEMAG = 1, EVAL_EXCHANGE = 2 };
void device_eval(DeviceState& D, const float* m, float* H, cudaStream_t st, EvalMode mode);

}  // namespace pmfem
