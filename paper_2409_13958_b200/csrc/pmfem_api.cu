// extern "C" entry points of libpmfem (include/pmfem.h).  No exception crosses the ABI.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <nccl.h>
#include "device.cuh"
#include "pmfem_internal.h"

struct pmfem_ctx_s {
  pmfem::HostSetup S;
  pmfem::DeviceState D;
  std::string err;
  bool host_only = true;
  pmfem::BlochHost bloch;       // NEXT-4 phased operators (kept on host-only contexts, for export)
};

namespace {
thread_local std::string g_setup_err;

template <class F>
pmfem_status guard(pmfem_ctx ctx, F&& f) {
  try {
    f();
    return PMFEM_OK;
  } catch (const pmfem::Error& e) {
    if (ctx) ctx->err = e.what(); else g_setup_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed"; else g_setup_err = "host allocation failed";
    return PMFEM_E_OOM;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what(); else g_setup_err = e.what();
    return PMFEM_E_INVALID_ARG;
  }
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void check_eval(pmfem_ctx ctx, const float* m, float* H) {
  pmfem::require(!ctx->host_only, PMFEM_E_STATE, "host-only context (cuda_device = -1) cannot evaluate fields");
  pmfem::require(m != nullptr && H != nullptr, PMFEM_E_INVALID_ARG, "NULL m or H");
  pmfem::require((const void*)m != (const void*)H, PMFEM_E_INVALID_ARG, "H must not alias m");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(e));
  cudaSetDevice(ctx->D.device);
}

void record_timing(pmfem_ctx ctx, cudaStream_t st) {
  (void)st;   // events were recorded on the stream; read back lazily in pmfem_get_timing
  if (ctx->D.timing) ctx->D.timing_pending = true;
}
}  // namespace

extern "C" {

static pmfem_status setup_impl(pmfem_ctx* out, const pmfem_mesh* mesh, const pmfem_periodicity* per,
                               const pmfem_grid* grid, int cuda_device, const void* nccl_id, int rank, int world) {
  if (!out) { g_setup_err = "NULL out"; return PMFEM_E_INVALID_ARG; }
  *out = nullptr;
  pmfem_ctx ctx = nullptr;
  try {
    ctx = new pmfem_ctx_s();
  } catch (...) {
    g_setup_err = "host allocation failed";
    return PMFEM_E_OOM;
  }
  pmfem_status st = guard(nullptr, [&] {
    double t0 = now();
    static const bool verbose = std::getenv("PMFEM_VERBOSE") != nullptr;
    auto stage = [&](const char* what) {
      if (verbose) {
        std::fprintf(stderr, "[pmfem] %-16s %8.2f s  (cuda: %s)\n", what, now() - t0,
                     cudaGetErrorString(cudaPeekAtLastError()));
        std::fflush(stderr);
      }
    };
    pmfem::HostSetup& S = ctx->S;
    pmfem::require(grid != nullptr && mesh != nullptr && per != nullptr, PMFEM_E_INVALID_ARG, "NULL argument");
    // axis permutation: on N > 1 the slab axis -- the longest grid axis, z on ties --
    // becomes the internal z (slowest) axis, so thin films and wires split along their length;
    // PMFEM_AXIS_PERM=a,b,c forces one (tests run permuted frames on one GPU).  The setup then
    // runs on permuted copies of the coordinates, periodicity and grid.
    int ap[3] = {0, 1, 2};
    if (world > 1) {
      int sa = 2;
      for (int a = 1; a >= 0; --a)
        if (grid->n[a] > grid->n[sa]) sa = a;
      if (sa != 2) { ap[sa] = 2; ap[2] = sa; }
    }
    if (const char* e = std::getenv("PMFEM_AXIS_PERM")) {
      int a0, a1, a2;
      if (std::sscanf(e, "%d,%d,%d", &a0, &a1, &a2) == 3 && a0 + a1 + a2 == 3 && a0 != a1 && a1 != a2 && a0 != a2 &&
          a0 >= 0 && a1 >= 0 && a2 >= 0 && a0 < 3 && a1 < 3 && a2 < 3) { ap[0] = a0; ap[1] = a1; ap[2] = a2; }
    }
    std::vector<double> xyz_p;
    pmfem_mesh mesh_p = *mesh;
    pmfem_periodicity per_p = *per;
    pmfem_grid grid_p = *grid;
    if (!(ap[0] == 0 && ap[1] == 1 && ap[2] == 2)) {
      pmfem::require(mesh->xyz != nullptr && mesh->n_nodes >= 0, PMFEM_E_INVALID_ARG, "NULL coordinates");
      xyz_p.resize(3 * (size_t)mesh->n_nodes);
      for (int64_t i = 0; i < mesh->n_nodes; ++i)
        for (int a = 0; a < 3; ++a) xyz_p[3 * i + a] = mesh->xyz[3 * i + ap[a]];
      mesh_p.xyz = xyz_p.data();
      for (int a = 0; a < 3; ++a) {
        per_p.periodic[a] = per->periodic[ap[a]];
        grid_p.n[a] = grid->n[ap[a]];
        for (int b = 0; b < 3; ++b) per_p.lattice[a][b] = per->lattice[ap[a]][ap[b]];
      }
      mesh = &mesh_p; per = &per_p; grid = &grid_p;
    }
    for (int a = 0; a < 3; ++a) S.axperm[a] = ap[a];
    pmfem::setup_mesh(S, mesh, per);
    stage("mesh/pbc");
    pmfem::setup_operators(S);
    stage("operators");
    S.z0_ring = grid ? grid->z0_ring : 1;
    pmfem::require(grid != nullptr, PMFEM_E_INVALID_ARG, "NULL grid");
    pmfem::require(grid->z0_ring == 0 || grid->z0_ring == 1, PMFEM_E_INVALID_ARG, "z0_ring must be 0 or 1");
    S.z0_device = cuda_device;            // device contexts integrate Z0 on the GPU
    S.cbox_device = cuda_device >= 0;     // device contexts build C_box on the GPU
    pmfem::setup_aim(S, grid);
    stage("aim");
    pmfem::setup_order(S);
    pmfem::setup_dist(S, rank, world);    // slab partition; a rank builds Z0 for its own rows
    stage("order/dist");
    pmfem::setup_z0(S);
    stage("z0");
    pmfem::setup_dist_halos(S);
    stage("halos");
    S.setup_seconds = now() - t0;
    if (cuda_device >= 0) {
      ctx->host_only = false;
      ctx->D.device = cuda_device;
      pmfem::device_upload(ctx->D, S);
      stage("device upload");
      if (world > 1) {
        pmfem::require(nccl_id != nullptr, PMFEM_E_INVALID_ARG, "NULL NCCL unique id");
        pmfem::device_init_comm(ctx->D, S, nccl_id);
      }
    }
  });
  if (st != PMFEM_OK) {
    if (!ctx->host_only) pmfem::device_free(ctx->D);
    delete ctx;
    return st;
  }
  *out = ctx;
  return PMFEM_OK;
}

pmfem_status pmfem_setup(pmfem_ctx* out, const pmfem_mesh* mesh, const pmfem_periodicity* per,
                         const pmfem_grid* grid, int cuda_device) {
  return setup_impl(out, mesh, per, grid, cuda_device, nullptr, 0, 1);
}

pmfem_status pmfem_setup_dist(pmfem_ctx* out, const pmfem_mesh* mesh, const pmfem_periodicity* per,
                              const pmfem_grid* grid, int cuda_device, const void* nccl_unique_id, int rank,
                              int world) {
  if (world < 1 || rank < 0 || rank >= world) { g_setup_err = "bad rank/world"; return PMFEM_E_INVALID_ARG; }
  return setup_impl(out, mesh, per, grid, cuda_device, nccl_unique_id, rank, world);
}

pmfem_status pmfem_nccl_unique_id(void* out128) {
  if (!out128) return PMFEM_E_INVALID_ARG;
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) { g_setup_err = ncclGetErrorString(r); return PMFEM_E_NCCL; }
  std::memcpy(out128, &id, sizeof(id));
  return PMFEM_OK;
}

pmfem_status pmfem_build_pgf(pmfem_ctx ctx, double target_rel_err) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    pmfem::require(target_rel_err > 0 && std::isfinite(target_rel_err), PMFEM_E_INVALID_ARG,
                   "target_rel_err must be positive");
    double t0 = now();
    // Ewald cutoffs from the target, then the truncation error measured with enlarged cutoffs;
    // tightened up to 4 times (report the achieved error, fail if the target is missed)
    double tgt = target_rel_err;
    pmfem::PgfParams P = pmfem::make_pgf_params(ctx->S.periodic, ctx->S.L, tgt);
    double achieved = pmfem::pgf_truncation_error(ctx->S, P);
    for (int it = 0; it < 4 && achieved > target_rel_err; ++it) {
      tgt *= 1e-2;
      P = pmfem::make_pgf_params(ctx->S.periodic, ctx->S.L, tgt);
      achieved = pmfem::pgf_truncation_error(ctx->S, P);
    }
    ctx->S.pgf_achieved_rel_err = achieved;
    if (achieved > target_rel_err) {
      char buf[160];
      std::snprintf(buf, sizeof(buf), "PGF truncation error %.3e above target %.3e", achieved, target_rel_err);
      throw pmfem::Error(PMFEM_E_PGF_NOT_CONVERGED, buf);
    }
    if (ctx->host_only) {
      pmfem::host_kernel_table(ctx->S, P, ctx->S.kernel);
      pmfem::host_fft_spectrum(ctx->S, ctx->S.kernel, ctx->S.spectrum);
    } else {
      pmfem::device_build_pgf(ctx->D, ctx->S, P);
    }
    ctx->S.pgf_seconds = now() - t0;
    if (std::getenv("PMFEM_VERBOSE")) {
      std::fprintf(stderr, "[pmfem] build_pgf        %8.2f s  (cuda: %s)\n", ctx->S.pgf_seconds,
                   cudaGetErrorString(cudaPeekAtLastError()));
      std::fflush(stderr);
    }
  });
}

// Bloch kernel table + full complex spectrum of k0 (user frame) into S.kernel_bloch /
// S.spectrum_bloch; S.k0 = k0 in the internal frame
static void bloch_kernel(pmfem_ctx ctx, const double* k0, double target_rel_err) {
  pmfem::HostSetup& S = ctx->S;
  pmfem::require(k0 != nullptr && target_rel_err > 0, PMFEM_E_INVALID_ARG, "NULL k0 or bad target");
  double kin[3];
  for (int a = 0; a < 3; ++a) {
    kin[a] = k0[S.axperm[a]];          // internal frame
    pmfem::require(std::isfinite(kin[a]), PMFEM_E_INVALID_ARG, "k0 must be finite");
    pmfem::require(S.periodic[a] || kin[a] == 0.0, PMFEM_E_INVALID_ARG, "k0 must vanish on non-periodic axes");
  }
  bool off = false;                    // k0 on the reciprocal lattice is the static kernel
  for (int a = 0; a < 3; ++a)
    if (S.periodic[a]) {
      const double f = kin[a] * S.L[a] / (2 * M_PI);
      off |= std::fabs(f - std::round(f)) > 1e-12;
    }
  pmfem::require(off, PMFEM_E_INVALID_ARG, "k0 on the reciprocal lattice: use pmfem_build_pgf");
  pmfem::PgfParams P = pmfem::make_pgf_params(S.periodic, S.L, target_rel_err);
  if (ctx->host_only) pmfem::host_bloch_table(S, P, kin, S.kernel_bloch);
  else pmfem::device_bloch_table(ctx->D, S, P, kin, S.kernel_bloch);
  pmfem::host_bloch_spectrum(S, S.kernel_bloch, S.spectrum_bloch);
  for (int a = 0; a < 3; ++a) S.k0[a] = kin[a];
}

pmfem_status pmfem_build_pgf_bloch(pmfem_ctx ctx, const double* k0, double target_rel_err) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] { bloch_kernel(ctx, k0, target_rel_err); });
}

pmfem_status pmfem_build_bloch(pmfem_ctx ctx, const double* k0, double target_rel_err) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    pmfem::require(ctx->host_only || ctx->D.world == 1, PMFEM_E_STATE,
                   "the Bloch field path is single-device (world = 1)");
    const double t0 = now();
    bloch_kernel(ctx, k0, target_rel_err);
    pmfem::BlochHost B;
    pmfem::setup_bloch_ops(ctx->S, ctx->S.k0, B);
    if (!ctx->host_only) pmfem::device_bloch_upload(ctx->D, ctx->S, B);
    else ctx->bloch = std::move(B);      // host-only: kept for pmfem_export (setup parity tests)
    if (std::getenv("PMFEM_VERBOSE")) {
      std::fprintf(stderr, "[pmfem] build_bloch      %8.2f s\n", now() - t0);
      std::fflush(stderr);
    }
  });
}

static pmfem_status eval_bloch(pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im,
                               void* stream, pmfem::EvalMode mode) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    check_eval(ctx, m_re, H_re);
    pmfem::require(m_im != nullptr && H_im != nullptr, PMFEM_E_INVALID_ARG, "NULL m_im or H_im");
    const void* outs[2] = {H_re, H_im};
    const void* ins[2] = {m_re, m_im};
    for (const void* o : outs)
      for (const void* i : ins) pmfem::require(o != i, PMFEM_E_INVALID_ARG, "H must not alias m");
    pmfem::require((const void*)H_re != (const void*)H_im, PMFEM_E_INVALID_ARG, "H_re must not alias H_im");
    pmfem::device_bloch_eval(ctx->D, m_re, m_im, H_re, H_im, (cudaStream_t)stream, mode);
  });
}

pmfem_status pmfem_demag_bloch(pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im, void* s) {
  return eval_bloch(ctx, m_re, m_im, H_re, H_im, s, pmfem::EVAL_DEMAG);
}
pmfem_status pmfem_exchange_bloch(pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im, void* s) {
  return eval_bloch(ctx, m_re, m_im, H_re, H_im, s, pmfem::EVAL_EXCHANGE);
}
pmfem_status pmfem_heff_bloch(pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im, void* s) {
  return eval_bloch(ctx, m_re, m_im, H_re, H_im, s, pmfem::EVAL_HEFF);
}

// One evaluation = ~9 kernel launches (+ NCCL calls on N>1).  On a non-default stream the
// sequence is captured once per (m, H, stream, mode, timing) into a CUDA graph and replayed
// (launch overhead paid once); PMFEM_NO_GRAPH=1 disables it.  The legacy default stream cannot
// be captured, so calls on it launch the kernels directly.
static void eval_graph(pmfem_ctx ctx, const float* m, float* H, cudaStream_t st, pmfem::EvalMode mode) {
  pmfem::DeviceState& D = ctx->D;
  static const bool no_graph = std::getenv("PMFEM_NO_GRAPH") != nullptr;
  if (no_graph || st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) {
    pmfem::device_eval(D, m, H, st, mode);
    return;
  }
  for (auto& g : D.graphs)
    if (g.exec && g.m == m && g.H == H && g.st == st && g.mode == (int)mode && g.timing == D.timing) {
      if (cudaGraphLaunch(g.exec, st) != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, "cudaGraphLaunch failed");
      return;
    }
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    throw pmfem::Error(PMFEM_E_CUDA, "cudaStreamBeginCapture failed");
  try {
    pmfem::device_eval(D, m, H, st, mode);
  } catch (...) {
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  if (cudaStreamEndCapture(st, &graph) != cudaSuccess || !graph)
    throw pmfem::Error(PMFEM_E_CUDA, "cudaStreamEndCapture failed");
  cudaGraphExec_t exec = nullptr;
  cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  // replace the least recently inserted slot
  pmfem::DeviceState::GraphSlot& slot = D.graphs[D.graph_next];
  D.graph_next = (D.graph_next + 1) % (int)(sizeof(D.graphs) / sizeof(D.graphs[0]));
  if (slot.exec) cudaGraphExecDestroy(slot.exec);
  slot = pmfem::DeviceState::GraphSlot{m, H, st, (int)mode, D.timing, exec};
  if (cudaGraphLaunch(exec, st) != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, "cudaGraphLaunch failed");
}

static pmfem_status eval(pmfem_ctx ctx, const float* m, float* H, void* stream, pmfem::EvalMode mode) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    check_eval(ctx, m, H);
    cudaStream_t st = (cudaStream_t)stream;
    eval_graph(ctx, m, H, st, mode);
    record_timing(ctx, st);
  });
}

pmfem_status pmfem_set_anisotropy(pmfem_ctx ctx, int kind, double K, const double* axis) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    pmfem::require(kind >= 0 && kind <= 2 && std::isfinite(K), PMFEM_E_INVALID_ARG, "anisotropy kind 0, 1 or 2");
    double u[3] = {0, 0, 1};
    if (kind == 1) {
      pmfem::require(axis != nullptr, PMFEM_E_INVALID_ARG, "NULL uniaxial axis");
      const double nrm = std::sqrt(axis[0] * axis[0] + axis[1] * axis[1] + axis[2] * axis[2]);
      pmfem::require(nrm > 0, PMFEM_E_INVALID_ARG, "zero uniaxial axis");
      for (int a = 0; a < 3; ++a) u[a] = axis[a] / nrm;
    }
    pmfem::DeviceState& D = ctx->D;
    D.anis_kind = kind;
    D.anis_K = K;
    D.anis_Ms = ctx->S.Ms_tet.empty() ? 1.0 : ctx->S.Ms_tet[0];
    for (int a = 0; a < 3; ++a) D.anis_u[a] = u[a];
    if (D.llg_exec) { cudaGraphExecDestroy(D.llg_exec); D.llg_exec = nullptr; }   // recapture
  });
}

pmfem_status pmfem_llg_am2(pmfem_ctx ctx, float* m, double t_end, double dt0, double tol, double alpha, double gamma,
                           const double* H_applied, double dt_max, void* stream, int64_t* steps_accepted,
                           int64_t* steps_rejected) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    pmfem::require(!ctx->host_only, PMFEM_E_STATE, "host-only context (cuda_device = -1) cannot integrate");
    pmfem::require(m != nullptr, PMFEM_E_INVALID_ARG, "NULL m");
    pmfem::require(ctx->D.pgf_ready, PMFEM_E_STATE, "pmfem_build_pgf has not been called");
    pmfem::require(t_end >= 0 && dt0 > 0 && tol > 0 && alpha >= 0 && gamma > 0, PMFEM_E_INVALID_ARG,
                   "bad LLG parameters");
    cudaSetDevice(ctx->D.device);
    const double zero[3] = {0, 0, 0};
    int64_t a = 0, r = 0;
    pmfem::device_llg_am2(ctx->D, m, (cudaStream_t)stream, t_end, dt0, tol, alpha, gamma,
                          H_applied ? H_applied : zero, dt_max, &a, &r);
    if (steps_accepted) *steps_accepted = a;
    if (steps_rejected) *steps_rejected = r;
  });
}

pmfem_status pmfem_llg_rk4(pmfem_ctx ctx, float* m, int64_t steps, double dt, double alpha, double gamma,
                           const double* H_applied, void* stream) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    pmfem::require(!ctx->host_only, PMFEM_E_STATE, "host-only context (cuda_device = -1) cannot integrate");
    pmfem::require(m != nullptr, PMFEM_E_INVALID_ARG, "NULL m");
    pmfem::require(ctx->D.pgf_ready, PMFEM_E_STATE, "pmfem_build_pgf has not been called");
    cudaSetDevice(ctx->D.device);
    pmfem::require(steps >= 0 && dt > 0 && alpha >= 0 && gamma > 0, PMFEM_E_INVALID_ARG, "bad LLG parameters");
    const double zero[3] = {0, 0, 0};
    const double* hap = H_applied ? H_applied : zero;
    pmfem::DeviceState& D = ctx->D;
    cudaStream_t st = (cudaStream_t)stream;
    static const bool no_graph = std::getenv("PMFEM_NO_GRAPH") != nullptr;
    if (no_graph || st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) {
      for (int64_t s = 0; s < steps; ++s) pmfem::device_llg_rk4_step(D, m, st, dt, alpha, gamma, hap);
      return;
    }
    const double key[6] = {dt, alpha, gamma, hap[0], hap[1], hap[2]};
    bool hit = D.llg_exec && D.llg_key_m == m && D.llg_key_st == st && !D.timing;
    for (int i = 0; i < 6 && hit; ++i) hit = D.llg_key[i] == key[i];
    if (!hit && steps > 0) {
      if (D.llg_exec) { cudaGraphExecDestroy(D.llg_exec); D.llg_exec = nullptr; }
      if (!D.llg_ms) pmfem::device_llg_rk4_step(D, m, st, dt, alpha, gamma, hap), --steps;   // allocates scratch
      cudaGraph_t graph = nullptr;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        throw pmfem::Error(PMFEM_E_CUDA, "cudaStreamBeginCapture failed");
      try {
        pmfem::device_llg_rk4_step(D, m, st, dt, alpha, gamma, hap);
      } catch (...) {
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      if (cudaStreamEndCapture(st, &graph) != cudaSuccess || !graph)
        throw pmfem::Error(PMFEM_E_CUDA, "cudaStreamEndCapture failed");
      cudaError_t e = cudaGraphInstantiate(&D.llg_exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, "cudaGraphInstantiate failed");
      D.llg_key_m = m;
      D.llg_key_st = st;
      for (int i = 0; i < 6; ++i) D.llg_key[i] = key[i];
    }
    for (int64_t s = 0; s < steps; ++s)
      if (cudaGraphLaunch(D.llg_exec, st) != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, "cudaGraphLaunch failed");
  });
}

pmfem_status pmfem_demag(pmfem_ctx ctx, const float* m, float* H, void* s) { return eval(ctx, m, H, s, pmfem::EVAL_DEMAG); }
pmfem_status pmfem_exchange(pmfem_ctx ctx, const float* m, float* H, void* s) { return eval(ctx, m, H, s, pmfem::EVAL_EXCHANGE); }
pmfem_status pmfem_heff(pmfem_ctx ctx, const float* m, float* H, void* s) { return eval(ctx, m, H, s, pmfem::EVAL_HEFF); }

pmfem_status pmfem_heff_host(pmfem_ctx ctx, const float* m_host, float* H_host, void* stream) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    pmfem::require(!ctx->host_only, PMFEM_E_STATE, "host-only context");
    pmfem::require(m_host && H_host, PMFEM_E_INVALID_ARG, "NULL host buffer");
    cudaSetDevice(ctx->D.device);
    const size_t bytes = sizeof(float) * 3 * (size_t)(ctx->D.hi - ctx->D.lo);   // rank-local rows
    if (!ctx->D.m_stage) {
      if (cudaMalloc(&ctx->D.m_stage, bytes) != cudaSuccess || cudaMalloc(&ctx->D.H_stage, bytes) != cudaSuccess)
        throw pmfem::Error(PMFEM_E_OOM, "staging allocation failed");
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemcpyAsync(ctx->D.m_stage, m_host, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
      throw pmfem::Error(PMFEM_E_CUDA, "H2D copy failed");
    pmfem::device_eval(ctx->D, ctx->D.m_stage, ctx->D.H_stage, st, pmfem::EVAL_HEFF);
    if (cudaMemcpyAsync(H_host, ctx->D.H_stage, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      throw pmfem::Error(PMFEM_E_CUDA, "D2H copy failed");
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw pmfem::Error(PMFEM_E_CUDA, cudaGetErrorString(e));
  });
}

pmfem_status pmfem_query(pmfem_ctx ctx, pmfem_info* out) {
  if (!ctx || !out) return PMFEM_E_INVALID_ARG;
  const pmfem::HostSetup& S = ctx->S;
  std::memset(out, 0, sizeof(*out));
  out->n_nodes = S.N;
  out->n_parents = S.Np;
  out->n_parents_local = S.dist.hi() - S.dist.lo();
  out->periodic_dims = S.periodic[0] + S.periodic[1] + S.periodic[2];
  out->touching = S.touching;
  out->protruding = S.protruding;
  for (int a = 0; a < 3; ++a) { out->grid[a] = S.grid_n[a]; out->fft[a] = S.fft_n[a]; }
  out->nnz_ring1 = S.ring1.nnz();
  out->nnz_z0 = S.z0.nnz();
  out->nnz_cbox = S.cbox_device ? ctx->D.cbox_nnz : S.cbox.nnz();
  double tot = 0;
  for (int i = 0; i < 5; ++i) { out->kernel_bytes[i] = ctx->D.kernel_bytes[i]; tot += ctx->D.kernel_bytes[i]; }
  out->bytes_per_eval_algorithmic = tot;
  out->launches_per_eval = ctx->D.launches_per_eval;
  out->fft_fused = ctx->D.fused_tile > 0;
  for (int a = 0; a < 3; ++a) out->k2_tile[a] = ctx->D.k2_tile[a];
  out->slab_world = ctx->D.slab_world;
  out->cbox_format = ctx->D.cbox_format;
  out->cbox_packed_units = ctx->D.cbox_chunks;
  out->pgf_achieved_rel_err = ctx->S.pgf_achieved_rel_err;
  out->comm_bytes_per_eval = ctx->D.comm_bytes_per_eval;
  out->setup_seconds = S.setup_seconds;
  out->pgf_seconds = S.pgf_seconds;
  return PMFEM_OK;
}

pmfem_status pmfem_get_order(pmfem_ctx ctx, int64_t* internal_to_user) {
  if (!ctx || !internal_to_user) return PMFEM_E_INVALID_ARG;
  const pmfem::HostSetup& S = ctx->S;
  for (int64_t i = S.dist.lo(); i < S.dist.hi(); ++i) internal_to_user[i - S.dist.lo()] = S.parent[S.perm[i]];
  return PMFEM_OK;
}

pmfem_status pmfem_export(pmfem_ctx ctx, const char* name, void* dst, int64_t* count) {
  if (!ctx || !name || !count) return PMFEM_E_INVALID_ARG;
  return guard(ctx, [&] {
    const pmfem::HostSetup& S = ctx->S;
    std::string n(name);
    auto put = [&](const void* src, int64_t cnt, size_t esz) {
      *count = cnt;
      if (dst && cnt) std::memcpy(dst, src, (size_t)cnt * esz);
    };
    if (n == "parent") put(S.parent.data(), S.Np, 8);
    else if (n == "lca") put(S.lca.data(), S.N, 8);
    else if (n == "shift") put(S.shift.data(), 3 * S.N, 4);
    else if (n == "Vt") put(S.Vt.data(), S.Np, 8);
    else if (n == "ring1_rowptr") put(S.ring1.rowptr.data(), S.Np + 1, 8);
    else if (n == "ring1_col") put(S.ring1.col.data(), S.ring1.nnz(), 4);
    else if (n == "ring1_val") put(S.ring1.val.data(), 7 * S.ring1.nnz(), 8);
    else if (n == "rowsumD") put(S.rowsumD.data(), 3 * S.Np, 8);
    else if (n == "z0_rowptr") put(S.z0.rowptr.data(), S.Np + 1, 8);
    else if (n == "z0_col") put(S.z0.col.data(), S.z0.nnz(), 4);
    else if (n == "z0_val") put(S.z0.val.data(), 3 * S.z0.nnz(), 8);
    else if (n == "rowsumZ") put(S.rowsumZ.data(), 3 * S.Np, 8);
    else if (n == "cbox_rowptr") put(S.cbox.rowptr.data(), S.Np + 1, 8);
    else if (n == "cbox_col") put(S.cbox.col.data(), S.cbox.nnz(), 4);
    else if (n == "cbox_val") put(S.cbox.val.data(), S.cbox.nnz(), 8);
    else if (n == "xw") put(S.xw.data(), 3 * S.Np, 8);
    else if (n == "stencil_s") put(S.st_s.data(), 3 * S.Np, 4);
    else if (n == "stencil_t") put(S.st_t.data(), 3 * S.Np, 8);
    else if (n == "grid_delta") put(S.delta, 3, 8);
    else if (n == "grid_origin") put(S.origin, 3, 8);
    else if (n == "perm") put(S.perm.data(), S.Np, 8);
    else if (n == "dist_bounds") put(S.dist.bounds.data(), (int64_t)S.dist.bounds.size(), 8);
    else if (n == "axis_perm") {
      const int64_t a[3] = {S.axperm[0], S.axperm[1], S.axperm[2]};
      put(a, 3, 8);
    }
    else if (n == "dist_planes") {
      // z-slab plane boundaries [world+1] of the row partition = the FFT's z slabs
      std::vector<int64_t> z(S.dist.planes.begin(), S.dist.planes.end());
      put(z.data(), (int64_t)z.size(), 8);
    }
    else if (n == "dist_ghost") {
      // U ghost planes per peer: [world][send r0 (z0, n), send r1, recv r0, recv r1] (8 values)
      const int W = S.dist.world;
      std::vector<int64_t> g(8 * W, 0);
      if (W > 1)
        for (int p = 0; p < W; ++p)
          for (int k = 0; k < 2; ++k) {
            g[8 * p + 2 * k] = S.dist.gsend[k][2 * p]; g[8 * p + 2 * k + 1] = S.dist.gsend[k][2 * p + 1];
            g[8 * p + 4 + 2 * k] = S.dist.grecv[k][2 * p]; g[8 * p + 4 + 2 * k + 1] = S.dist.grecv[k][2 * p + 1];
          }
      put(g.data(), (int64_t)g.size(), 8);
    }
    else if (n == "slab_kranges") {
      // per rank (first k0 column, count) of the slab-decomposed FFT's x slabs, world = this
      // context's world (the z slabs are n2 / world planes each)
      const int W = S.dist.world, H0 = S.fft_n[0] / 2 + 1;
      std::vector<int64_t> r(2 * W);
      for (int p = 0; p < W; ++p) { r[2 * p] = pmfem::slab_h0(p, H0, W); r[2 * p + 1] = pmfem::slab_hn(p, H0, W); }
      put(r.data(), 2 * W, 8);
    }
    else if (n.rfind("cbox_device_", 0) == 0) {
      // the device-built C_box (internal order), decoded from its C4x chunks / B4 blocks for
      // tests: every slot is returned (C4x padding repeats the previous column with value 0; B4
      // empty slots are the block's other columns with value 0)
      pmfem::require(!ctx->host_only && S.cbox_device, PMFEM_E_STATE, "C_box was not built on the device");
      const pmfem::DeviceState& D = ctx->D;
      const int64_t nr = D.hi - D.lo;                // the rank's own rows
      std::vector<int64_t> ptr(nr + 1);
      cudaMemcpy(ptr.data(), D.c_ptr, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost);
      const std::string tail = n.substr(12);
      const int64_t nch = ptr[nr];
      if (D.cbox_format == 2 && (tail == "rowptr" || tail == "col" || tail == "val")) {
        // SEG: value offsets, the near columns decoded from the candidate bitmasks, the values
        if (tail == "rowptr") put(ptr.data(), nr + 1, 8);
        else {
          *count = nch;
          if (dst && nch) {
            if (tail == "val") {
              cudaMemcpy(dst, D.c_val, sizeof(float) * (size_t)nch, cudaMemcpyDeviceToHost);
            } else {
              int* d_col = nullptr;
              if (cudaMalloc(&d_col, sizeof(int) * (size_t)nch) != cudaSuccess)
                throw pmfem::Error(PMFEM_E_OOM, "cudaMalloc (SEG decode)");
              pmfem::device_seg_decode(D, d_col);
              cudaMemcpy(dst, d_col, sizeof(int) * (size_t)nch, cudaMemcpyDeviceToHost);
              cudaFree(d_col);
            }
          }
        }
      } else if (tail == "rowptr") {
        for (auto& v : ptr) v *= 4;
        put(ptr.data(), nr + 1, 8);
      } else if (tail == "val") {
        *count = 4 * nch;
        if (dst && nch) cudaMemcpy(dst, D.c_val, sizeof(float) * 4 * (size_t)nch, cudaMemcpyDeviceToHost);
      } else if (tail == "col" && D.cbox_format == 5) {
        // W4: window-local index -> run (runs of a tile sorted by first row, window offsets
        // increasing with it) -> internal row
        *count = 4 * nch;
        if (dst && nch) {
          const int64_t nt = D.w_ntiles;
          std::vector<int64_t> trow(nt + 1);
          std::vector<int> rptr(nt + 1);
          cudaMemcpy(trow.data(), D.w_trow, sizeof(int64_t) * (nt + 1), cudaMemcpyDeviceToHost);
          cudaMemcpy(rptr.data(), D.w_rptr, sizeof(int) * (nt + 1), cudaMemcpyDeviceToHost);
          std::vector<int> rs(rptr[nt]), rc(rptr[nt]);
          cudaMemcpy(rs.data(), D.w_rstart, sizeof(int) * rs.size(), cudaMemcpyDeviceToHost);
          cudaMemcpy(rc.data(), D.w_rloc, sizeof(int) * rc.size(), cudaMemcpyDeviceToHost);
          std::vector<uint16_t> id(4 * (size_t)nch);
          cudaMemcpy(id.data(), D.w_idx, sizeof(uint16_t) * id.size(), cudaMemcpyDeviceToHost);
          int32_t* c = static_cast<int32_t*>(dst);
          // (slot order inside a row is quarter-transposed; the export lists the slots as stored)
          for (int64_t t = 0; t < nt; ++t)
            for (int64_t e = 4 * ptr[trow[t] - D.lo]; e < 4 * ptr[trow[t + 1] - D.lo]; ++e) {
              const int* b = rc.data() + rptr[t];
              const int* en = rc.data() + rptr[t + 1];
              const int* f = std::upper_bound(b, en, (int)id[e]);
              const int r = (int)(f - b) - 1 + rptr[t];
              c[e] = rs[r] + ((int)id[e] - rc[r]);
            }
        }
      } else if (tail == "col" && (D.cbox_format == 1 || D.cbox_format == 3)) {
        // B4: aligned block index b -> columns 4b..4b+3; U4: start column c -> c..c+3
        *count = 4 * nch;
        if (dst && nch) {
          std::vector<int32_t> b(nch);
          cudaMemcpy(b.data(), D.c_bidx, sizeof(int32_t) * (size_t)nch, cudaMemcpyDeviceToHost);
          int32_t* c = static_cast<int32_t*>(dst);
          const int32_t mul = D.cbox_format == 1 ? 4 : 1;
          for (int64_t i = 0; i < nch; ++i)
            for (int j = 0; j < 4; ++j) c[4 * i + j] = mul * b[i] + j;
        }
      } else if (tail == "col") {
        *count = 4 * nch;
        if (dst && nch) {
          std::vector<unsigned long long> h(nch);
          cudaMemcpy(h.data(), D.c_hdr, sizeof(unsigned long long) * (size_t)nch, cudaMemcpyDeviceToHost);
          int32_t* c = static_cast<int32_t*>(dst);
          for (int64_t i = 0; i < nch; ++i) {
            int32_t k = (int32_t)(h[i] & 0xFFFFFFFull);
            c[4 * i] = k;
            for (int j = 0; j < 3; ++j) { k += (int32_t)((h[i] >> (28 + 12 * j)) & 0xFFF); c[4 * i + 1 + j] = k; }
          }
        }
      } else if (tail == "chunks") {
        put(&D.cbox_chunks, 1, 8);
      } else if (tail == "format") {
        const int64_t f = D.cbox_format;
        put(&f, 1, 8);
      } else throw pmfem::Error(PMFEM_E_INVALID_ARG, "unknown export name '" + n + "'");
    }
    else if (n.rfind("send_", 0) == 0 || n.rfind("recv_", 0) == 0) {
      const std::string kinds = "mqu";
      const bool snd = n[0] == 's';
      const size_t kpos = kinds.find(n[5]);
      if (kpos == std::string::npos || n.size() < 8) throw pmfem::Error(PMFEM_E_INVALID_ARG, "unknown export name '" + n + "'");
      const int k = (int)kpos;
      const std::string tail = n.substr(7);
      if (tail == "ptr") put(snd ? S.dist.send_ptr[k].data() : S.dist.recv_ptr[k].data(), S.dist.world + 1, 8);
      else if (tail == "idx") {
        const auto& v = snd ? S.dist.send_idx[k] : S.dist.recv_idx[k];
        put(v.data(), (int64_t)v.size(), 4);
      } else throw pmfem::Error(PMFEM_E_INVALID_ARG, "unknown export name '" + n + "'");
    }
    else if (n == "spectrum_device") {
      // the fp32 spectrum the device evaluation multiplies by ([P2][P1][H0], / #FFT points)
      pmfem::require(!ctx->host_only && ctx->D.pgf_ready, PMFEM_E_STATE, "no device spectrum (build_pgf first)");
      const int64_t cnt = (int64_t)ctx->D.H0 * ctx->D.P[1] * ctx->D.P[2];
      *count = cnt;
      if (dst) {
        std::vector<float> f(cnt);
        cudaMemcpy(f.data(), ctx->D.spec, sizeof(float) * cnt, cudaMemcpyDeviceToHost);
        double* o = static_cast<double*>(dst);
        for (int64_t i = 0; i < cnt; ++i) o[i] = f[i];
      }
    }
    else if (n == "kernel_bloch") put(S.kernel_bloch.data(), (int64_t)S.kernel_bloch.size(), 8);
    else if (n == "spectrum_bloch") put(S.spectrum_bloch.data(), (int64_t)S.spectrum_bloch.size(), 8);
    else if (n.rfind("bloch_", 0) == 0) {     // host-only contexts after pmfem_build_bloch
      const pmfem::BlochHost& B = ctx->bloch;
      const pmfem::Csr* R = n.rfind("bloch_r1_", 0) == 0 ? &B.r1 : n.rfind("bloch_z0_", 0) == 0 ? &B.z0
                            : n.rfind("bloch_cbox_", 0) == 0 ? &B.cbox : nullptr;
      const std::string f = R ? n.substr(n.find('_', 6) + 1) : "";
      if (R && f == "rowptr") put(R->rowptr.data(), (int64_t)R->rowptr.size(), 8);
      else if (R && f == "col") put(R->col.data(), R->nnz(), 4);
      else if (R && f == "val") put(R->val.data(), (int64_t)R->val.size(), 8);
      else if (n == "bloch_mod") put(B.mod.data(), (int64_t)B.mod.size(), 8);
      else if (n == "bloch_fa") put(B.fa.data(), (int64_t)B.fa.size(), 8);
      else if (n == "bloch_fb") put(B.fb.data(), (int64_t)B.fb.size(), 8);
      else throw pmfem::Error(PMFEM_E_INVALID_ARG, "unknown export name '" + n + "'");
    }
    else if (n == "kernel") put(S.kernel.data(), (int64_t)S.kernel.size(), 8);
    else if (n == "spectrum") put(S.spectrum.data(), (int64_t)S.spectrum.size(), 8);
    else throw pmfem::Error(PMFEM_E_INVALID_ARG, "unknown export name '" + n + "'");
  });
}

pmfem_status pmfem_set_timing(pmfem_ctx ctx, int enable) {
  if (!ctx) return PMFEM_E_INVALID_ARG;
  ctx->D.timing = enable != 0;
  return PMFEM_OK;
}

pmfem_status pmfem_get_timing(pmfem_ctx ctx, float* ms) {
  if (!ctx || !ms) return PMFEM_E_INVALID_ARG;
  if (ctx->D.timing_pending) {
    cudaEventSynchronize(ctx->D.ev[5]);
    for (int i = 0; i < 5; ++i)
      if (cudaEventElapsedTime(&ctx->D.last_ms[i], ctx->D.ev[i], ctx->D.ev[i + 1]) != cudaSuccess)
        ctx->D.last_ms[i] = -1.f;
    (void)cudaGetLastError();   // never leave a timing failure pending for the next evaluation
    ctx->D.timing_pending = false;
  }
  for (int i = 0; i < 8; ++i) ms[i] = ctx->D.last_ms[i];
  return PMFEM_OK;
}

const char* pmfem_last_error(pmfem_ctx ctx) { return ctx ? ctx->err.c_str() : g_setup_err.c_str(); }

void pmfem_destroy(pmfem_ctx ctx) {
  if (!ctx) return;
  if (!ctx->host_only) pmfem::device_free(ctx->D);
  delete ctx;
}

}  // extern "C"
