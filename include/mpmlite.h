/*
 * mpmlite.h — C ABI of the B200-native MPM Lite solve-time hot path (libmpmlite.so).
 *
 * The calls follow the paper's statement of one time step (Alg. 1):
 *   set particles + materials (Alg. 1 "Require")
 *   -> resample to quadrature: Unload (Alg. 2) + stretch bases (Alg. 3 lines 4-7)
 *   -> energy / gradient / Hessian-vector product of the incremental potential
 *      (Eq. incpot-rotfree; App. B)
 *   -> Newton / Jacobi-PCG minimisation (Alg. 3 line 8; "matrix-free PCG" P:495)
 *   -> transfer back to particles: Load (Alg. 4).
 * Readings of passages the paper leaves open are listed in DESIGN.md §2 (amb-1..amb-21).
 *
 * Conventions
 *  - Every call returns mpl_status (MPL_OK == 0).  No C++ exception crosses the ABI.  On error
 *    mpl_last_error(ctx) returns a message naming the offending particle / cell where relevant.
 *  - Precision: a context computes in fp32 or fp64 (mpl_config.precision = 32 | 64).  Every
 *    floating-point buffer passed to or returned from a context is `float` or `double`
 *    accordingly ("real" below).  Accumulations of dot products and energies are fp64.
 *  - Memory: buffers may live on the host or on the device (any pointer cudaMemcpyDefault accepts:
 *    pageable or pinned host memory, or device memory of the context's GPU).  The caller owns every
 *    buffer; the library copies inputs and never retains caller pointers after a call returns.
 *  - Streams: all work is ordered on the context's stream (its own stream unless mpl_set_stream);
 *    every call is synchronous with respect to the host at return.
 *  - Node-vector order ("canonical order"): the active nodes (m_i > 0) ordered by 4^3 node block
 *    (blocks sorted by x-major block id (bx*NBy + by)*NBz + bz), then x-major within the block.
 *    mpl_get_nodes exports the (i,j,k) of each entry; compare by key, never by position.
 *  - Quadrature order: cells of the structural stencil set (every cell touched by some particle's
 *    2^3 stencil), same block-major order; mpl_get_quadrature exports (i,j,k).
 *  - Grid: N0 x N1 x N2 cells of size dx; node (i,j,k) at origin + dx (i,j,k); cell centre at
 *    origin + dx (i+1/2, j+1/2, k+1/2).  Blocks are 4^3 cells.  Every particle's base
 *    cell b = floor((x - origin)/dx - 1/2) must satisfy 0 <= b <= N-2 per axis (stencil inside the
 *    grid), else MPL_ERR_OUT_OF_DOMAIN.
 *  - Threading: one context per host thread.  A failing call leaves particle state unchanged;
 *    after a failure inside mpl_resample / mpl_newton_step, mpl_resample is required again.
 */
#ifndef MPMLITE_H
#define MPMLITE_H

#include <stdint.h>

#if defined(__GNUC__)
#define MPL_API __attribute__((visibility("default")))
#else
#define MPL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpl_ctx_s *mpl_ctx;
/* An in-process group of slab ranks (one host thread per rank, one process): the loopback transport
 * used to run the multi-GPU decomposition on one GPU (tests).  Production runs use NCCL instead. */
typedef struct mpl_group_s *mpl_group;

typedef enum {
    MPL_OK = 0,
    MPL_ERR_INVALID_ARG = 1,
    MPL_ERR_STATE = 2,            /* call order: e.g. mpl_hvp before mpl_linearize            */
    MPL_ERR_OUT_OF_DOMAIN = 3,    /* a particle stencil leaves the grid                */
    MPL_ERR_INVERTED = 4,         /* det F_p <= 0 at unload                    */
    MPL_ERR_INVERSION_DOMAIN = 5, /* stress -> stretch inversion failed               */
    MPL_ERR_NONFINITE = 6,        /* NaN / Inf produced                        */
    MPL_ERR_OOM = 7,
    MPL_ERR_CUDA = 8,
    MPL_ERR_NCCL = 9,
    MPL_ERR_UNSUPPORTED = 10
} mpl_status;

typedef struct {
    int32_t n[3];     /* cells per axis                                   */
    double dx;        /* cell size                                        */
    double origin[3]; /* position of node (0,0,0)                         */
} mpl_grid;

typedef struct {
    int32_t kind; /* 0 = StVK with Hencky strain (amb-1); 1 = split Neo-Hookean
                     (P:229-285); 2 = J-based water (kappa = E)          */
    double E, nu; /* Young's modulus, Poisson ratio -> 3D Lame (amb-2) */
    double rho;   /* density: m_p = rho * V_p                          */
    double yield_stress; /* von Mises sigma_y > 0: fixed-point plasticity (kind 0 only; 0 = elastic).
                            P:658-663: at every Newton iterate the trial deformation A(v) S_base of
                            each slot is return-mapped in Hencky space, the slot's base
                            becomes S = S_base P (A(v) S = F^E) and is held through that iteration's
                            PCG (elasticity only) and line search; Load return-maps F_p too.   */
} mpl_material;

typedef struct {
    int32_t precision; /* 32 or 64                                              */
    int32_t device;    /* CUDA device ordinal                                   */
    int32_t rank, nranks; /* slab decomposition rank / size (1 process per GPU) */
    const uint8_t *nccl_unique_id; /* 128 bytes from mpl_nccl_unique_id on rank 0; NULL if nranks==1 */
    mpl_group loopback;            /* non-NULL: ranks are threads of this process (mpl_group_create);
                                      every collective then meets at a host barrier (no NCCL)        */
} mpl_config;

typedef struct {
    double lo[3], hi[3]; /* nodes with lo <= x_i <= hi (all axes) are prescribed (amb-9) */
    double velocity[3];  /* prescribed velocity                                          */
} mpl_dirichlet_box;

typedef struct {
    int32_t newton_max;   /* Newton iteration cap (amb-6)                                */
    int32_t cg_max;       /* PCG iteration cap per Newton iteration                      */
    double newton_rtol;   /* stop when ||g_free|| <= newton_rtol ||g_free(v^0)||          */
    double cg_rtol;       /* stop when ||r|| <= cg_rtol ||r_0|| (amb-7)                   */
    double armijo_c;      /* Armijo constant (1e-4)                                      */
    int32_t ls_max;       /* maximum halvings (30)                                       */
    double ls_slack;      /* accept when Phi_new <= Phi + c a g.p + ls_slack |Phi| (amb-6) */
    int32_t fixed_newton_iters;        /* >0: run exactly this many Newton iterations (parity replay) */
    const int32_t *fixed_cg_iters;     /* NULL or per-Newton-iteration PCG counts (parity replay)    */
    const int32_t *fixed_ls_halvings;  /* NULL or per-Newton-iteration halvings (parity replay)      */
    int32_t psd_project;  /* 0: exact Hessian, PCG stops at negative curvature (amb-6);
                             1: per-cell PSD projection of the cached tangent, K_c -> Q max(Lambda, 0) Q^T
                             (for indefinite compressed states, e.g. cfg5's plate contact).
                             Energy and gradient are unchanged; the Jacobi diagonal follows K_c.      */
} mpl_solver_cfg;

#define MPL_MAX_NEWTON_LOG 64
typedef struct {
    int32_t newton_iters, cg_iters_total, ls_halvings, converged, neg_curvature;
    int32_t n_inverted_trials; /* line-search trials rejected for det(I + dt G) <= 0 (amb-21) */
    double grad_norm0, grad_norm, energy;
    int32_t cg_iters[MPL_MAX_NEWTON_LOG];
    int32_t ls_iters[MPL_MAX_NEWTON_LOG];
    int32_t n_hvp;        /* HVPs executed in this call (= PCG iterations; launches past convergence exit at once) */
    double hvp_ms;        /* device time of those HVP launches (CUDA events around every 4th launch, scaled) */
    double ms_phase[8];   /* 0 resample, 1 PCG vector kernels (MPL_VEC_EVENTS=1), 2 explicit update, 3 linearize, 4 PCG, 5 line search, 6 G2P, 7 total (ms) */
    int64_t n_cells, n_nodes, n_free_nodes; /* quadrature points, active nodes, free (non-Dirichlet) nodes */
    int64_t n_launches;   /* CUDA kernels launched by the library during this call                */
    double grad_norms[MPL_MAX_NEWTON_LOG]; /* ||g_free|| at the start of Newton iteration k (k < newton_iters),
                                              then at the returned iterate (index newton_iters) if measured */
    double alphas[MPL_MAX_NEWTON_LOG];     /* accepted line-search step of Newton iteration k            */
    int32_t tangent_format;               /* cached tangent of the last linearisation: 0 = 45 numbers per
                                             quadrature point, 1 = compressed (28: SVD-frame blocks)     */
    int32_t pad_;
} mpl_solve_stats;

/* ---- context ------------------------------------------------------------------------------ */
/* Create a context on cfg->device.  precision must be 32 or 64; nranks > 1 needs NCCL support. */
MPL_API mpl_status mpl_create(const mpl_config *cfg, const mpl_grid *grid, mpl_ctx *out);
MPL_API void mpl_destroy(mpl_ctx ctx);
MPL_API const char *mpl_last_error(mpl_ctx ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = own stream. */
MPL_API mpl_status mpl_set_stream(mpl_ctx ctx, void *cuda_stream);
/* Library version string and the compute capability it was built for ("sm_100a"). */
MPL_API const char *mpl_version(void);
/* rank 0 only: 128-byte NCCL unique id to broadcast to the other ranks before mpl_create. */
MPL_API mpl_status mpl_nccl_unique_id(uint8_t out[128]);

/* ---- slab decomposition ---------------------------------------
 * With nranks > 1 every call below marked "collective" must be made by every rank, in the same
 * order.  Rank r owns the 4-cell blocks [cuts[r], cuts[r+1]) along x: their quadrature points, the
 * particles whose base cell lies there, and the nodes those cells touch.  The node plane at the
 * cut is held by both neighbours with identical values (partial sums completed by a neighbour
 * exchange after C2N, every gradient and every HVP); dot products and Phi count it once.  Each
 * step particles that left the slab migrate to the neighbour (more than one slab per step is
 * MPL_ERR_OUT_OF_DOMAIN) and the last owned cell plane is copied to the upper neighbour as ghosts.
 * A failing collective returns an error on every rank. */
/* One-rank self-test of the NCCL transport on `device` (unique id, communicator, allreduce, grouped
 * send / receive); *out_sum = 8.0 on success.  MPL_ERR_NCCL if libnccl.so.2 cannot be used. */
MPL_API mpl_status mpl_nccl_selftest(int32_t device, double *out_sum);
MPL_API mpl_status mpl_group_create(int32_t nranks, mpl_group *out);
MPL_API void mpl_group_destroy(mpl_group g);
/* cuts: nranks + 1 strictly increasing cell-block x indices, cuts[0] = 0, cuts[nranks] =
 * ceil(n[0] / 4).  Default: equal widths.  Call before mpl_set_particles. */
MPL_API mpl_status mpl_set_slabs(mpl_ctx ctx, const int32_t *cuts);
/* Host-only helper (no GPU needed): cuts balancing a per-plane weight (e.g. particles per cell-block
 * plane); cuts[r] is the first plane whose prefix weight reaches r / nranks of the total, kept
 * strictly increasing.  weight may be NULL (equal widths). */
MPL_API mpl_status mpl_balance_slabs(int32_t nplanes, const int64_t *weight, int32_t nranks, int32_t *cuts);
/* Global particle ids (int32 >= 0) of the particles last passed to mpl_set_particles on this rank
 * (slab ranks only; default: input index).  Exports of a slab rank (mpl_get_particles,
 * mpl_get_particle_cells, mpl_get_particle_ids) list its owned particles in ascending id. */
MPL_API mpl_status mpl_set_particle_ids(mpl_ctx ctx, const int32_t *ids);
MPL_API mpl_status mpl_get_particle_ids(mpl_ctx ctx, int32_t *ids);
/* per active node (canonical order): 1 if this rank's copy is the counted one (n_nodes bytes). */
MPL_API mpl_status mpl_get_node_owner(mpl_ctx ctx, uint8_t *owned);

/* ---- scene -------------------------------------------------------------------------------- */
/* n <= 8 materials; kind 0 (StVK-Hencky) or 1 (split Neo-Hookean, bulk modulus kappa = 2/3 mu + lam,
 * P:250): require mu > 0 and lam > -2 mu / 3.  Kind 2 (J-based water, §4.5):
 * psi = kappa/2 (J - 1)^2 with kappa = E > 0 (nu ignored); a water particle carries only
 * J_p = det F_p: its stress is kappa J (J - 1) I, its slot's base stretch J_base^{1/3} I
 * (J_base = (1 + sqrt(1 + 4 pi_c / kappa)) / 2), and Load sets F_p = J_p^{1/3} I with
 * J_p^{n+1} = (1 + dt tr G_p) J_p^n.  Each material slot of a quadrature point keeps its own
 * law; solids and water may share cells. */
MPL_API mpl_status mpl_set_materials(mpl_ctx ctx, int32_t n, const mpl_material *mats);
/* gravity acceleration g (inertia target vhat = v^n + dt g, amb-4); default (0, -9.81, 0). */
MPL_API mpl_status mpl_set_gravity(mpl_ctx ctx, const double g[3]);
/* n <= 8 boxes; a node inside several boxes takes the first one's velocity. */
MPL_API mpl_status mpl_set_dirichlet(mpl_ctx ctx, int32_t n, const mpl_dirichlet_box *boxes);
/* Particle state (Alg. 1 "Require"): x (n*3), v (n*3), F (n*9 row-major), G (n*9 row-major,
 * the APIC velocity gradient G_p), vol (n, rest volume V_p), mat (n, material id int32).
 * on_device is advisory (any cudaMemcpyDefault pointer works). */
MPL_API mpl_status mpl_set_particles(mpl_ctx ctx, int64_t n, const void *x, const void *v, const void *F,
                             const void *G, const void *vol, const int32_t *mat, int32_t on_device);
/* Particle state in the order it was given to mpl_set_particles (one rank; slab ranks: owned
 * particles in ascending global id, mpl_num_particles of them).  Any pointer may be NULL. */
MPL_API mpl_status mpl_get_particles(mpl_ctx ctx, void *x, void *v, void *F, void *G, int32_t on_device);
MPL_API int64_t mpl_num_particles(mpl_ctx ctx);

/* ---- resample: Alg. 2 + Alg. 3 lines 4-7 ------------------------ */
/* Bins particles, activates blocks / cells / nodes, scatters particle state to the cell-centre
 * quadrature (Eqs. p2c-mV, p2c-mv-affine, p2c-A-sum, vtau), gathers it to the nodes,
 * reconstructs the rotation-free stretch S_{c,k} per material slot (Eqs. hencky-trace..sigmai),
 * forms vhat = v^n + dt g and the Newton start v^0 (Dirichlet values on prescribed nodes).
 * Outputs the counts of quadrature cells, active nodes and active 4^3 cell blocks (NULL allowed). */
MPL_API mpl_status mpl_resample(mpl_ctx ctx, double dt, int64_t *n_cells, int64_t *n_nodes, int64_t *n_blocks);
/* active nodes in canonical order: ijk (n_nodes*3 int32), lumped mass m_i, v^n_i (n_nodes*3),
 * free flag (uint8: 1 = free DOF, 0 = prescribed).  NULL pointers are skipped. */
MPL_API mpl_status mpl_get_nodes(mpl_ctx ctx, int32_t *ijk, void *m, void *v_n, uint8_t *free_dof);
/* sorted x-major linear ids (bx*NBy + by)*NBz + bz of the 4^3 cell blocks touched by any particle
 * stencil (structural; bit-exact).  n_blocks entries. */
MPL_API mpl_status mpl_get_active_blocks(mpl_ctx ctx, int64_t *ids);
/* per-particle base cell floor((x - origin)/dx - 1/2) the last mpl_resample binned each particle into
 * (n*3 int32, input order; bit-exact).  Valid between mpl_resample and mpl_transfer_to_particles (which
 * moves the particles): MPL_ERR_STATE otherwise. */
MPL_API mpl_status mpl_get_particle_cells(mpl_ctx ctx, int32_t *base_ijk);
/* quadrature state (n_cells entries, canonical cell order): ijk (n*3), m_c, v_c (n*3), G_c (n*9),
 * and per material k: V_{c,k} (nmat*n), tau_{c,k} (nmat*n*9), S_{c,k} (nmat*n*9).  NULL skips. */
MPL_API mpl_status mpl_get_quadrature(mpl_ctx ctx, int32_t *ijk, void *m_c, void *v_c, void *G_c, void *V_ck,
                              void *tau_ck, void *S_ck);

/* ---- the incremental potential ------------------------------- */
/* Phi(v) = sum_i 1/2 m_i |v_i - vhat_i|^2 + sum_{c,k} V_ck psi_k((I + dt G_c(v)) S_ck)
 * (Eq. incpot-rotfree).  v: n_nodes*3 canonical order.  phi = +inf if some
 * det(I + dt G_c) <= 0 (amb-21). */
MPL_API mpl_status mpl_energy(mpl_ctx ctx, const void *v, double *phi);
/* g_i = dPhi/dv_i (unprojected; App. B Eq. residual with the sign of amb-3).  phi may be NULL. */
MPL_API mpl_status mpl_gradient(mpl_ctx ctx, const void *v, void *g, double *phi);
/* Linearise at v: caches the per-quadrature tangent K_c (45 numbers, the 9x9 symmetric
 * d^2(sum_k V_ck psi_k)/dG^2) and the Jacobi diagonal.  Required before mpl_hvp. */
MPL_API mpl_status mpl_linearize(mpl_ctx ctx, const void *v);
/* Tangent used by mpl_linearize / mpl_hvp / mpl_get_diag: 0 = exact (default), 1 = per-cell PSD projection
 * (as mpl_solver_cfg.psd_project; mpl_newton_step follows its cfg instead). */
MPL_API mpl_status mpl_set_psd_projection(mpl_ctx ctx, int32_t on);
/* Jacobi diagonal D_ia = (H)_{ia,ia} at the last linearisation point (n_nodes*3). */
MPL_API mpl_status mpl_get_diag(mpl_ctx ctx, void *D);
/* Matrix-free Hessian-vector product at the last linearisation point (unprojected):
 * (Hu)_i = m_i u_i + sum_c (K_c : dG_c(u)) grad w_ic, dG_c(u) = sum_j u_j (x) grad w_jc. */
MPL_API mpl_status mpl_hvp(mpl_ctx ctx, const void *u, void *Hu);
/* Benchmark of the HVP kernel: `reps` back-to-back launches on u (canonical order, any memory),
 * mean device time per launch from CUDA events on the context stream (kernel only: no zeroing of Hu,
 * no slab halo exchange); then one complete product written to Hu (may be NULL). */
MPL_API mpl_status mpl_hvp_bench(mpl_ctx ctx, const void *u_dev, void *Hu_dev, int32_t reps, double *ms_per_hvp);

/* ---- the implicit solve ---------------------------------------- */
/* Newton with Jacobi-PCG and Armijo backtracking from v^0 (amb-6, amb-7, amb-8); stores v^{n+1}. */
MPL_API mpl_status mpl_newton_step(mpl_ctx ctx, const mpl_solver_cfg *cfg, mpl_solve_stats *stats);
/* v^{n+1} after mpl_newton_step (or v^0 before it), n_nodes*3 canonical order. */
MPL_API mpl_status mpl_get_velocity(mpl_ctx ctx, void *v);
/* replace the current iterate (n_nodes*3 canonical order) — e.g. to restart from a given v. */
MPL_API mpl_status mpl_set_velocity(mpl_ctx ctx, const void *v);

/* ---- load ------------------------------------------------------------ */
/* Alg. 4: v_c = sum w_ic v_i, G_c = sum v_i (x) grad w_ic (cells with m_c > 0); v_p = sum w_cp v_c,
 * G_p = sum w_cp G_c (weights at x_p^n); x_p += dt v_p; F_p <- (I + dt G_p) F_p. */
MPL_API mpl_status mpl_transfer_to_particles(mpl_ctx ctx, double dt);

/* ---- explicit integration (Eq. explicitforce; Alg. 3 lines 1-3) -- */
/* After mpl_resample: f_i = -sum_{c,k} V_ck tau_ck grad w_ic and v^{n+1} = v^n + dt (g + f_i / m_i) on
 * free nodes (prescribed nodes keep their Dirichlet value); v^{n+1} is then read by
 * mpl_get_velocity / mpl_transfer_to_particles.  Collective on slab ranks (force halo sum). */
MPL_API mpl_status mpl_explicit_velocity(mpl_ctx ctx);
/* One explicit step: resample -> explicit velocity -> transfer.  stats (may be NULL): ms_phase[0]
 * resample, [2] explicit update, [6] transfer, [7] total; counts as for mpl_step. */
MPL_API mpl_status mpl_explicit_step(mpl_ctx ctx, double dt, mpl_solve_stats *stats);

/* ---- pipelined particle I/O (end-to-end stepping with host-resident particle state) ---------- */
/* mpl_stage_particles: like mpl_set_particles, but asynchronous: the host arrays (pinned memory for
 * real overlap) are copied on the context's H2D copy stream into a staging set, which the next
 * mpl_resample adopts (it waits for the copy; the staged set becomes the particle state by a buffer
 * swap).  May be called while the previous step computes, after that step's resample; one staged set
 * at a time (MPL_ERR_STATE otherwise).  The host arrays must stay valid and unchanged until that
 * adoption completes (mpl_stage_wait).  Single-rank contexts (MPL_ERR_UNSUPPORTED on slab ranks).
 * mpl_get_particles_async: like mpl_get_particles (input order), but only enqueues: the reorder runs
 * on the compute stream after the last enqueued work, the D2H copies on a second copy stream, so they
 * overlap the next step; the host arrays are complete after mpl_stage_wait.
 * mpl_stage_wait: blocks until every enqueued stage / readback copy and the compute stream are done. */
MPL_API mpl_status mpl_stage_particles(mpl_ctx ctx, int64_t n, const void *x, const void *v, const void *F,
                                       const void *G, const void *vol, const int32_t *mat);
MPL_API mpl_status mpl_get_particles_async(mpl_ctx ctx, void *x, void *v, void *F, void *G);
MPL_API mpl_status mpl_stage_wait(mpl_ctx ctx);

/* One full step: resample -> newton -> transfer (Alg. 1). */
MPL_API mpl_status mpl_step(mpl_ctx ctx, double dt, const mpl_solver_cfg *cfg, mpl_solve_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* MPMLITE_H */
