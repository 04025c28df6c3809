/*
 * pmfem.h -- C ABI of the B200-native PM-FEM periodic H_eff library (libpmfem.so).
 *
 * Implements the data-parallel hot path of "Periodic micromagnetic finite element method"
 * (Ai, Duan, Lomakin; arXiv 2409.13958; /root/reference/PAPER.md cited as P:<line>):
 *
 *   q     = D (Ms m)                       periodized divergence + surface charge (P:171 Eq. hms_d1)
 *   u_loc = Z0 m                           exact near-field correction            (P:173 Eq. hms_d2b)
 *   Q     = P q                            AIM anterpolation onto the grid        (P:202 BAIM step 1)
 *   U     = F^-1( G_hat . F Q )            FFT convolution with the periodic GF   (P:204, P:214 step 2)
 *   u     = P^T U + C_box q + u_loc        interpolation + precorrection          (P:206-218 steps 3-4, Eq. new_er)
 *   H_ms  = -G u                           periodized gradient                    (P:174 Eq. hms_d3)
 *   H_ex  = -(2A/Ms) Vt^-1 S m             periodic exchange Laplacian            (P:117-157 Eqs. hex, lapl, lapl_1, lapl_2)
 *   H_eff = H_ms + H_ex                                                           (P:73 Eq. heff)
 *
 * Units are CGS: positions in cm, Ms in emu/cm^3, Aex in erg/cm, fields in Oe, m is a unit
 * vector.  G_0 = 1/|r|.  The discrete conventions (grid, stencils, PGF normalisation,
 * near-set rules) are the contract K1-K11 of SURVEY.md 8(c) with the readings listed in
 * DESIGN.md.
 *
 * Threading: a context is not thread-safe; calls on one context must be serialised by the
 * caller.  No entry point throws; every one returns a pmfem_status and, on failure, stores a
 * message retrievable with pmfem_last_error(ctx).
 */
#ifndef PMFEM_H
#define PMFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmfem_ctx_s* pmfem_ctx;   /* opaque; owns every host and device buffer it allocates */

typedef enum {
  PMFEM_OK = 0,
  PMFEM_E_INVALID_ARG = 1,      /* NULL pointer, bad size, non-positive period, non-diagonal lattice
                                   vectors, grid not a power of two, stencil order not in 1..3,
                                   N_i < 2(p+1)                                                    */
  PMFEM_E_MESH = 2,             /* tet index out of range, degenerate tet (|V| < 1e-12 mean |V|),
                                   zero lumped volume                                              */
  PMFEM_E_PBC_AMBIGUOUS = 3,    /* two nodes within match_tol of one periodic image        */
  PMFEM_E_PBC_INCONSISTENT = 4, /* an LCA component whose members are not period translates*/
  PMFEM_E_OUTSIDE_GRID = 5,     /* a node's stencil anchor falls outside [0, N_i - 1 - p] on a
                                   non-periodic axis (fp64 rounding of the grid built from the node
                                   extent); the grid is built to cover the mesh, so this
                                   signals corrupted coordinates (NaN / Inf)                        */
  PMFEM_E_RER_TOO_LARGE = 6,    /* r_ER >= L/2 or r_ER/Delta + p + 1 >= N/2 on a periodic axis     */
  PMFEM_E_PGF_NOT_CONVERGED = 7,/* pmfem_build_pgf: the Ewald truncation error measured with enlarged
                                   cutoffs stays above target_rel_err after 4 refinements;
                                   the achieved value is in the message and pmfem_info            */
  PMFEM_E_STATE = 8,            /* call order (field evaluation before pmfem_build_pgf, host-only ctx)*/
  PMFEM_E_CUDA = 9,             /* a CUDA runtime error (message holds cudaGetErrorString)         */
  PMFEM_E_NCCL = 10,            /* a NCCL error (distributed contexts)                              */
  PMFEM_E_OOM = 11              /* host or device allocation failure                                */
} pmfem_status;

/* Tetrahedral mesh.  Host arrays, borrowed for the duration of pmfem_setup only. */
typedef struct {
  int64_t        n_nodes;   /* N                                                              */
  const double*  xyz;       /* [n_nodes][3] node coordinates, cm                               */
  int64_t        n_tets;    /* T                                                              */
  const int32_t* tets;      /* [n_tets][4] 0-based node indices; orientation fixed by the lib  */
  const int32_t* region;    /* [n_tets] region id per tet, or NULL for a single region 0       */
  int32_t        n_regions; /* number of entries in Ms / Aex (>= 1)                            */
  const double*  Ms;        /* [n_regions] saturation magnetisation, emu/cm^3                  */
  const double*  Aex;       /* [n_regions] exchange stiffness, erg/cm                          */
} pmfem_mesh;

/* Periodicity (P:36-43 Eq. pm_cont; 1D, 2D or 3D along any axes; P:277 uses z). */
typedef struct {
  int32_t periodic[3];      /* 1 = axis is periodic; none periodic = non-periodic mode (NEXT-3) */
  double  lattice[3][3];    /* rows = lattice vectors (cm).  P:36-43 writes them L_x x^, L_y y^,
                               L_z z^: they must be diagonal (|off-diagonal| <= 1e-12 x max |L_i|,
                               else PMFEM_E_INVALID_ARG); lattice[i][i] = L_i > 0 on periodic axes,
                               ignored on non-periodic axes                                      */
  double  match_tol;        /* T-PBC pair tolerance (cm); 0 -> 1e-6 x shortest edge */
} pmfem_periodicity;

/* AIM grid and near-field parameters. */
typedef struct {
  int32_t n[3];             /* grid points per axis.  periodic: Delta = L/n; non-periodic:
                               Delta = (max-min)/(n-1) over the nodes (Eq. grid).
                               FFT lengths n (periodic) / 2n (non-periodic) must be powers of 2 */
  int32_t order;            /* Lagrange stencil order p in {1,2,3} ((p+1)^3 points per node)    */
  double  rer_scale;        /* s: r_ER = s * max(Delta_x,Delta_y,Delta_z) (reading R8)   */
  int32_t z0_ring;          /* 0: exact self term only; 1: exact periodic 1-ring        */
} pmfem_grid;

typedef struct {
  int64_t n_nodes, n_parents, n_parents_local;    /* N, N', N' owned by this rank             */
  int32_t periodic_dims, touching, protruding;    /* classification                    */
  int32_t grid[3], fft[3];                        /* AIM grid and padded FFT lengths          */
  int64_t nnz_ring1, nnz_z0, nnz_cbox;            /* off-diagonal nnz of L/D/G, Z0, C_box     */
  double  bytes_per_eval_algorithmic;             /* DESIGN.md byte model with the real nnz   */
  double  setup_seconds, pgf_seconds;             /* host wall time of setup / build_pgf      */
  double  kernel_bytes[8];                        /* algorithmic bytes per launch of K1..K5 (index
                                                     0 K1, 1 K2, 2 K3 (all FFT passes), 3 K4, 4 K5) */
  int32_t launches_per_eval;                      /* library kernels launched by one pmfem_heff   */
  int32_t fft_fused;                              /* 1: fused YZ FFT plan, 0: split plan          */
  double  comm_bytes_per_eval;                    /* bytes this rank sends+receives per evaluation */
  int32_t k2_tile[3];                             /* K2 anterpolation grid tile (points per axis) */
  int32_t slab_world;                             /* > 1: slab-decomposed FFT over this many ranks
                                                     (SURVEY 8(e)); 1: FFT on the full grid      */
  int32_t cbox_format;                            /* packed C_box streamed by K4: 0 = C4x chunks
                                                     (4 entries + 64-bit column header), 1 = B4
                                                     (aligned 4-column blocks + 32-bit block id)  */
  int64_t cbox_packed_units;                      /* C4x chunks or B4 blocks                     */
  double  pgf_achieved_rel_err;                   /* pmfem_build_pgf: max |K(cutoffs) - K(enlarged
                                                     cutoffs)| / max |K| over probe displacements
                                                     (0 before build_pgf and in free space)      */
} pmfem_info;

/* Build a context: validate, orient, detect T-PBC pairs and fold them to LCAs,
 * assemble the folded operators, the exact near field Z0, the AIM
 * grid, stencils and precorrection C_box.  cuda_device >= 0 uploads the fp32
 * operators to that device; cuda_device = -1 builds a host-only context (setup artifacts can
 * be exported with pmfem_export, no field evaluation).  On failure *out is NULL and the
 * message is returned by pmfem_last_error(NULL) (thread-local). */
pmfem_status pmfem_setup(pmfem_ctx* out, const pmfem_mesh* mesh, const pmfem_periodicity* per,
                         const pmfem_grid* grid, int cuda_device);

/* Multi-GPU context: every rank passes the FULL mesh; the library runs the
 * same deterministic host setup and derives every peer's plan without coordination:
 *  - slab axis: the longest grid axis (z on ties) becomes the internal z (slowest) axis by an axis
 *    permutation of the coordinates, periodicity and grid; m and H stay in the user frame, every
 *    exported setup artifact and pmfem_info.grid/fft are in the internal frame (export "axis_perm");
 *  - partition: rank r owns the rows anchored in the z planes [Z_r, Z_r+1) (export "dist_planes";
 *    variable thickness balancing the row counts) = its z slab of the FFT; it builds Z0, the local
 *    operators and C_box for its own rows only (setup time and operator memory ~1/world);
 *  - per evaluation: grouped ncclSend/ncclRecv halos of m (the own rows' 2-ring), q (the rows
 *    anchored within the anterpolation stencil / r_ER planes around the slab) and u (ring 1); K2
 *    computes the own planes completely (no grid reduction); slab FFT: X, Y on the own planes, an
 *    all-to-all into k0 columns [h_r, h_r + H_r) (export "slab_kranges"), Z x G_hat, the
 *    all-to-all back, Y', X'; then the p U "ghost" planes above the slab that K4's stencils read
 *    come from their owners (export "dist_ghost").
 * The slab axis needs at least one plane per rank (else PMFEM_E_INVALID_ARG).  With fewer k0
 * columns than ranks (or PMFEM_NO_SLAB set) the anterpolated grid is all-reduced and the FFT
 * replicated instead.  nccl_unique_id: 128 bytes from
 * pmfem_nccl_unique_id on rank 0, broadcast by the caller (e.g. torch.distributed).
 * cuda_device = -1 builds the host-only plan (exportable: dist_bounds, dist_planes, dist_ghost,
 * axis_perm, send_/recv_{m,q,u}_{ptr,idx}).  world = 1 is identical to pmfem_setup. */
pmfem_status pmfem_setup_dist(pmfem_ctx* out, const pmfem_mesh* mesh, const pmfem_periodicity* per,
                              const pmfem_grid* grid, int cuda_device, const void* nccl_unique_id,
                              int rank, int world);
pmfem_status pmfem_nccl_unique_id(void* out128);

/* Tabulate the periodic Green's function K on the padded grid with Ewald sums in fp64
 * (Eq. 2 with k0 = 0; "exponentially rapidly convergent sums"; normalisation
 * R3), K(0) = G_p^reg(0), and store G_hat = real(FFT(K)) / (#FFT points), G_hat[0] = 0, as fp32
 * (P:204).  On a device context the tabulation and fp64 FFT run on the GPU.
 * target_rel_err (clamped to [1e-16, 1e-2]) sets the Ewald cutoffs (erfc(x_r) and
 * exp(-k_max^2/4 alpha^2) at 1e-2 x target); the truncation error is then MEASURED as
 * max |K - K'| / max |K| over 64 probe displacements, K' with enlarged cutoffs, and the cutoffs
 * are tightened (x 1e-2, up to 4 times) until it is <= target; otherwise
 * PMFEM_E_PGF_NOT_CONVERGED.  The reported error is at least DBL_EPSILON (2.2e-16): targets
 * below fp64 resolution cannot be met.  The achieved value is reported in pmfem_info. */
pmfem_status pmfem_build_pgf(pmfem_ctx ctx, double target_rel_err);

/* NEXT-4: the Bloch-phase periodic Green's function of Eq. 2 with k0 != 0
 * (P:183-185), G(r; k0) = sum_i exp(-j k0.R_i) / |r - R_i|, by Ewald sums in fp64 (the static
 * formulas with cos(k.r) -> exp(-j (G + k0).r) and the G = 0 term kept; no renormalisation is
 * needed off the reciprocal lattice).  Tabulates the MODULATED kernel exp(j k0.r) G(r; k0) --
 * L-periodic, so the AIM grid convolution of quasi-periodic data runs through it -- at every
 * padded grid displacement (on the GPU for device contexts, on the host otherwise) and its full
 * complex spectrum / #FFT points (host fp64 FFT); exports "kernel_bloch" and "spectrum_bloch"
 * ([P2][P1][P0] complex, interleaved re/im).  k0[3] in rad/cm, user frame; must vanish on
 * non-periodic axes and must not be a reciprocal lattice vector (PMFEM_E_INVALID_ARG).
 * The complex field path is pmfem_build_bloch / pmfem_*_bloch below. */
pmfem_status pmfem_build_pgf_bloch(pmfem_ctx ctx, const double* k0, double target_rel_err);

/* NEXT-4 complex field path.  Magnetisation amplitudes that are Bloch-periodic with the phase
 * of Eq. 2, m(r + R) = exp(-j k0.R) m(r), have the potential
 * u(r_n) = sum_m G_p(r_n - r_m; k0) q_m + Z0 terms, and everything in the static path carries
 * over with phases (reading R27): folded local operators weight a tet entry between
 * copies with lattice shifts s_a (row), s_b (column) by exp(j k0.L(s_a - s_b)); Z0 weights an
 * element image by the shifts of its vertices; the AIM grid part runs on the modulated charges
 * exp(j k0.r_n) q_n with the L-periodic kernel exp(j k0.r) G_p(r) (complex spectrum, nothing
 * removed: k0 is off the reciprocal lattice) and the modulated precorrection.
 * pmfem_build_bloch builds the Bloch kernel (as pmfem_build_pgf_bloch) and the phased operators
 * (host fp64: ring-1 L/D/G, Z0 with host element integrals, C~) and uploads them; world = 1 only
 * (PMFEM_E_STATE otherwise); k0 as in pmfem_build_pgf_bloch.  Replaces any previous Bloch build;
 * the static path is unaffected.  On a host-only context the operators are kept for
 * pmfem_export ("bloch_{r1,z0,cbox}_{rowptr,col,val}" in user parent order, complex values
 * interleaved re/im -- r1: L, Dx, Dy, Dz, Gx, Gy, Gz with the diagonal; z0: Zx, Zy, Zz; cbox: C~
 * -- and "bloch_mod", "bloch_fa", "bloch_fb") and no field can be evaluated.
 * pmfem_{demag,exchange,heff}_bloch: m_re, m_im, H_re, H_im device pointers [N'][3] fp32 in
 * internal node order as for pmfem_demag (the real and imaginary planes of m and H);
 * H written, not accumulated; no output may alias an input or the other output
 * (PMFEM_E_INVALID_ARG); PMFEM_E_STATE before pmfem_build_bloch.  Asynchronous on cuda_stream
 * (plain launches, no graph capture). */
pmfem_status pmfem_build_bloch(pmfem_ctx ctx, const double* k0, double target_rel_err);
pmfem_status pmfem_demag_bloch   (pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im,
                                  void* cuda_stream);
pmfem_status pmfem_exchange_bloch(pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im,
                                  void* cuda_stream);
pmfem_status pmfem_heff_bloch    (pmfem_ctx ctx, const float* m_re, const float* m_im, float* H_re, float* H_im,
                                  void* cuda_stream);

/* Field evaluations.  m: device pointer [N'_local][3] fp32 (internal node order, unit vectors);
 * H: device pointer [N'][3] fp32, written (not accumulated); must not alias m.
 * cuda_stream: a cudaStream_t or NULL for the legacy default stream.  Asynchronous: nothing
 * synchronises the host; kernel faults surface as PMFEM_E_CUDA on a later call. */
pmfem_status pmfem_demag   (pmfem_ctx ctx, const float* m, float* H, void* cuda_stream);  /* H := H_ms        */
pmfem_status pmfem_exchange(pmfem_ctx ctx, const float* m, float* H, void* cuda_stream);  /* H := H_ex        */
pmfem_status pmfem_heff    (pmfem_ctx ctx, const float* m, float* H, void* cuda_stream);  /* H := H_ms + H_ex */

/* Same as pmfem_heff but m and H are HOST buffers [N'][3] fp32 (pinned or pageable); the
 * host->device copy of m, the evaluation and the device->host copy of H are enqueued on the
 * stream and the call returns after the stream is synchronised (end-to-end path). */
pmfem_status pmfem_heff_host(pmfem_ctx ctx, const float* m_host, float* H_host, void* cuda_stream);

/* NEXT-2: `steps` classical RK4 steps of the LLG equation (P:67-71, P:101-105,
 * Eq. llg; reading R18) dm/dt = -gamma/(1+alpha^2) [m x H + alpha m x (m x H)],
 * H = H_ms + H_ex + H_an + H_applied (uniform, Oe; H_an from pmfem_set_anisotropy), |m|
 * renormalised to 1 after every step.
 * m: device pointer [n_parents_local][3] fp32, updated in place.  dt in s, gamma in rad/(s Oe)
 * (1.7595e7 for electrons).  Each step = 4 pmfem_heff evaluations + 4 fused stage kernels; on a
 * non-default stream the step is captured once into a CUDA graph and replayed `steps` times.
 * H_applied may be NULL (zero).  Asynchronous like the field calls. */
pmfem_status pmfem_llg_rk4(pmfem_ctx ctx, float* m, int64_t steps, double dt, double alpha, double gamma,
                           const double* H_applied, void* cuda_stream);

/* NEXT-2: the local anisotropy field H_an of Eq. heff ("local ... straightforward")
 * added by the LLG integrators (not by pmfem_heff, whose H_eff is H_ms + H_ex):
 *   kind 0: none;  1: uniaxial, energy -K (m.u)^2, H = (2K/Ms) (m.u) u, axis u (normalised);
 *   kind 2: cubic (crystal axes = x, y, z), energy K (mx^2 my^2 + my^2 mz^2 + mz^2 mx^2),
 *           H = -(2K/Ms) (mx (my^2 + mz^2), my (mz^2 + mx^2), mz (mx^2 + my^2)).
 * K in erg/cm^3, Ms of material region 0 (single-material meshes), axis in the user frame
 * (may be NULL for kinds 0 and 2). */
pmfem_status pmfem_set_anisotropy(pmfem_ctx ctx, int kind, double K, const double* axis);

/* NEXT-2: the paper's adaptive second-order Adams predictor-corrector ("predictor-corrector
 * schemes based on explicit second order Adams-Moulton (midpoint) approach"), t = 0 .. t_end:
 * variable-step AB2 predictor (forward Euler on the first step), one H_eff evaluation, AM2
 * (trapezoidal) corrector, |m| renormalised; Milne error estimate err = max_n |m_c - m_p| / 6
 * (max over ranks on N > 1), accepted when err <= tol, next dt = dt min(2, max(0.2,
 * 0.9 (tol/err)^(1/3))), capped by dt_max when dt_max > 0.  Two H_eff evaluations per accepted
 * step.  The host reads the error after every attempt (the call synchronises the stream).
 * m: device pointer [n_parents_local][3], updated in place; the step counts may be NULL. */
pmfem_status pmfem_llg_am2(pmfem_ctx ctx, float* m, double t_end, double dt0, double tol, double alpha,
                           double gamma, const double* H_applied, double dt_max, void* cuda_stream,
                           int64_t* steps_accepted, int64_t* steps_rejected);

pmfem_status pmfem_query(pmfem_ctx ctx, pmfem_info* out);

/* internal_to_user[i] = original (user) node index of the parent stored in internal row i. */
pmfem_status pmfem_get_order(pmfem_ctx ctx, int64_t* internal_to_user);

/* Copy a named fp64/int setup artifact to host memory (tests and diagnostics).  Call with
 * dst = NULL to get the element count in *count.  Names and types are listed in DESIGN.md
 * ("Export names"); unknown name -> PMFEM_E_INVALID_ARG. */
pmfem_status pmfem_export(pmfem_ctx ctx, const char* name, void* dst, int64_t* count);

/* Device time (ms) of each kernel class in the last evaluation when timing is enabled with
 * pmfem_set_timing(ctx, 1) (CUDA events on the evaluation stream; adds event records only). */
pmfem_status pmfem_set_timing(pmfem_ctx ctx, int enable);
pmfem_status pmfem_get_timing(pmfem_ctx ctx, float* ms_per_kernel /* [8] as kernel_bytes */);

const char*  pmfem_last_error(pmfem_ctx ctx);
void         pmfem_destroy(pmfem_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* PMFEM_H */
