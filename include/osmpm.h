/*
 * osmpm.h -- C ABI of the B200-native (sm_100a) OS-MPM hot path.
 *
 * OS-MPM = overlapping Schwarz space-time refinement for the implicit Material Point Method
 * (Luo, Li, Jiang, arXiv 2605.09097; /root/reference/PAPER.md, cited as PAPER.md:line).
 * The library implements, as hand-written CUDA kernels, one fine-subdomain implicit sub-step
 * of the paper (Alg. 1) and the operators it is built from:
 *   - quadratic-B-spline APIC P2G of mass, momentum and stress
 *   - the matrix-free Hessian-vector product inside Newton-PCG
 *   - G2P with the deformation-gradient update and advection
 *   - the coarse<->fine transmission Pi_{S->B}, I_{B->S} and T_m
 *
 * General conventions (apply to every call unless stated otherwise)
 *   * Every function returns osmpm_status; OSMPM_OK == 0.  On failure osmpm_last_error() returns
 *     a thread-local message naming the particle / node / iteration involved.  No exception
 *     crosses the ABI and the library never calls exit().
 *   * Handles are opaque; the caller creates and destroys them.  A subdomain belongs to the ctx
 *     it was created with; all its work is enqueued on that ctx's CUDA stream.
 *   * Input pointers are BORROWED for the duration of the call only; the library copies what it
 *     keeps into library-owned device memory.  Output buffers are caller-owned.
 *   * osmpm_memspace says whether a caller pointer is host memory or device memory of the ctx's
 *     device (e.g. a torch tensor's data_ptr()).  Host buffers are copied synchronously.
 *   * All caller-visible floating-point arrays are IEEE fp64, whatever the subdomain's internal
 *     precision.  Particle arrays are in CREATION order, particle-major, components innermost:
 *       x, v:   n*d;   F, B: n*d*d (row-major d x d per particle);   m, V0: n.
 *   * Node ("grid") vectors at the ABI are dense over the subdomain's node box `dims`
 *     (osmpm_grid_desc), C order with axis 0 slowest, components innermost:
 *       value(node (k0,k1,k2), component a) at [((k0*dims[1] + k1)*dims[2] + k2)*d + a]
 *     (2D: dims[2] == 1).  Node (k0,k1,k2) sits at x = origin + dx*k.
 *     Nodes never touched by a particle stencil read as 0.
 *   * Asynchrony: calls returning device results are asynchronous on the ctx stream, except
 *     osmpm_implicit_solve, osmpm_schwarz_substep, osmpm_schwarz_step, osmpm_p2g (which read back
 *     a few scalars) and any call given host buffers.  Device-side errors (out-of-domain particle,
 *     inverted F) are latched and surface at the next synchronising call or osmpm_sync().
 *   * Reproducibility: node sums that several tiles contribute to meet in fp64 atomics, so results
 *     may differ run to run in the last bits.  With the environment variable OSMPM_DETERMINISTIC=1
 *     (read at every launch) the P2G, Newton-gradient / Jacobi-diagonal and HVP scatters store
 *     per-tile node blocks summed in a fixed tile order instead: bitwise reproducible, ~4 % slower.
 */
#ifndef OSMPM_H
#define OSMPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OSMPM_OK = 0,
    OSMPM_E_INVALID_ARG = 1,
    OSMPM_E_OUT_OF_DOMAIN = 2,          /* a particle stencil leaves the node box     */
    OSMPM_E_INVERTED_F = 3,             /* det F_p <= 0 after G2P                    */
    OSMPM_E_NEWTON_NOT_CONVERGED = 4,   /* Newton iteration cap reached              */
    OSMPM_E_LINESEARCH_STAGNATION = 5,  /* line-search step below ls_min_alpha       */
    OSMPM_E_SCHWARZ_NOT_CONVERGED = 6,  /* k_max Schwarz iterations without convergence           */
    OSMPM_E_COUPLING_CONFIG = 7,        /* inconsistent coarse/fine pair       */
    OSMPM_E_CUDA = 8,
    OSMPM_E_NCCL = 9,
    OSMPM_E_OOM = 10,
    OSMPM_E_STATE = 11                  /* call out of order (e.g. HVP before a gradient call)     */
} osmpm_status;

typedef enum { OSMPM_F64 = 0, OSMPM_F32 = 1 } osmpm_precision;
typedef enum { OSMPM_HOST = 0, OSMPM_DEVICE = 1 } osmpm_memspace;
typedef enum { OSMPM_COARSE_TO_FINE = 0, OSMPM_FINE_TO_COARSE = 1 } osmpm_direction;

typedef struct osmpm_ctx osmpm_ctx;
typedef struct osmpm_subdomain osmpm_subdomain;
typedef struct osmpm_coupler osmpm_coupler;

/* Structured node box of one subdomain: node k at origin + dx*k, k in [0, dims).  dim in {2,3}. */
typedef struct {
    int32_t dim;
    double origin[3];
    double dx;
    int64_t dims[3];
} osmpm_grid_desc;

/* Neo-Hookean material (Psi per DESIGN.md R2): Young's modulus E, Poisson nu. */
typedef struct {
    double E, nu;
} osmpm_material;

/* Particle set in creation order ("mass m_p, position x_p, velocity v_p, deformation
 * gradient F_p"; affine matrix B_p; initial volume V0_p).
 * material: per-particle index into the material table (NULL -> all 0).
 * is_boundary: the P^∂ markers of PAPER.md:281 (NULL -> none). */
typedef struct {
    int64_t n;
    osmpm_memspace space;
    const double *x, *v, *F, *B, *m, *V0;
    const int32_t* material;
    const uint8_t* is_boundary;
} osmpm_particles_view;

/* Newton-PCG settings (readings DESIGN.md R5-R8 = SURVEY.md Z6-Z10).
 *   max_newton, max_cg   iteration caps (per solve / per Newton iteration)
 *   fixed_iters          1: run exactly max_newton x max_cg (timing mode); 0: stop on tolerances
 *   guess                0: xhat^(0) = xtilde (u = dt v^n); 1: xhat^(0) = x^n (u = 0)
 *   newton_rtol/atol     stop when ||g_free|| <= max(rtol*||g_free^(0)||, atol)
 *   cg_rtol              PCG stops when ||r|| <= cg_rtol * ||g_free||
 *   ls_min_alpha         line search fails below this step (2^-20)
 *   energy_noise_rtol    accept a step whose energy change is within this fraction of the
 *                        energy's absolute scale (round-off floor, R8)            */
typedef struct {
    int32_t max_newton, max_cg, fixed_iters, guess;
    double newton_rtol, newton_atol, cg_rtol, ls_min_alpha, energy_noise_rtol;
    int32_t cg_variant;  /* 0: standard Jacobi PCG (two reductions per iteration); 1: single-reduction
                            PCG (Chronopoulos-Gear, R22: the same iterates in exact arithmetic,
                            one reduction -- one all-reduce across ranks -- per iteration) */
    int32_t psd;         /* PSD projection of the per-particle tangent blocks (R23):
                            0 never (the timed path), 1 in a second PCG solve when the Newton direction
                            fails the descent check g . dx < 0, 2 always.  Projected solves run the
                            standard PCG with per-particle scatter kernels (not bitwise reproducible). */
} osmpm_newton_settings;

/* Outcome of one implicit solve.  Besides the counts, three events that change what the solve
 * returns are reported (R7, R8), identically in the oracle:
 *   negcurv       PCG solves stopped by non-positive curvature p^T H p <= 0 (the Newton step is the
 *                 iterate reached, or -diag^-1 g if it was the first PCG iteration)
 *   ls_failures   fixed_iters only: Newton iterations whose line search found no decrease down to
 *                 ls_min_alpha; alpha = 0 is taken (u unchanged) and the solve goes on, so the work
 *                 of a timed solve stays fixed
 *   floor_accept  tolerance mode only: 1 if the solve was accepted as converged at the round-off
 *                 floor of E_h (||g|| <= sqrt(newton_rtol) * g_ref while no decrease was resolvable)
 *                 rather than at newton_rtol */
typedef struct {
    int32_t newton_iters, cg_iters, ls_halvings, status;
    double grad_norm0, grad_norm, energy;
    int32_t negcurv, ls_failures, floor_accept;
    int32_t psd_solves;  /* PCG solves run with the PSD-projected tangent (settings.psd) */
} osmpm_solve_stats;

/* Schwarz coupling settings (R10-R16).
 *   eps_conv     interface residual tolerance (1e-5)
 *   eps_tol      projection regularisation epsilon_tol; < 0 -> 1e-12 * fine mass
 *   tau_gamma_rel  tau_Gamma = tau_gamma_rel * median particle mass of each subdomain (1e-6)
 *   k_max        Schwarz iteration cap
 *   M            sub-cycling ratio dT/dt (integer >= 1)
 *   parity_fixed_k  > 0: run exactly this many Schwarz iterations (parity mode)            */
typedef struct {
    double eps_conv, eps_tol, tau_gamma_rel;
    int32_t k_max, M, parity_fixed_k;
    osmpm_newton_settings coarse, fine;
} osmpm_schwarz_settings;

typedef struct {
    int32_t iters, fine_substeps, converged, n_recv_B, n_recv_S;
    double r_B[256], r_S[256];
} osmpm_schwarz_report;

/* ----------------------------------------------------------------------------------------------
 * Context
 * ----------------------------------------------------------------------------------------------*/
const char* osmpm_last_error(void);
const char* osmpm_version(void);

/* device: CUDA ordinal; cuda_stream: the cudaStream_t all work is enqueued on (e.g.
 * torch.cuda.current_stream().cuda_stream; pass cudaStreamLegacy for the legacy default stream),
 * or NULL for a library-created non-blocking stream.  The ctx never destroys a caller-supplied
 * stream. */
osmpm_status osmpm_ctx_create(int device, void* cuda_stream, osmpm_ctx** out);
void osmpm_ctx_destroy(osmpm_ctx* ctx);

/* Kernel timing (CUDA events on the ctx stream around each launch of the named kernel family:
 * "hvp", "grad", "energy", "p2g", "g2p", "sort", "cg", "transmit").  enable != 0 starts recording;
 * osmpm_kernel_time synchronises and returns the launch count and summed device milliseconds
 * since the last reset. */
osmpm_status osmpm_profile_enable(osmpm_ctx* ctx, int enable);
osmpm_status osmpm_profile_reset(osmpm_ctx* ctx);
osmpm_status osmpm_kernel_time(osmpm_ctx* ctx, const char* family, int64_t* launches, double* ms);
/* Number of CUDA kernels the library has launched on this ctx since creation (all families). */
osmpm_status osmpm_launch_count(osmpm_ctx* ctx, int64_t* launches);

/* ----------------------------------------------------------------------------------------------
 * Slab decomposition of a fine subdomain (the paper's method is serial on one CPU,
 * PAPER.md:508, and names scalable parallel implementations as future work).
 * One process per GPU: rank 0 calls osmpm_comm_unique_id and shares the 128 bytes (e.g. with
 * torch.distributed); every rank then calls osmpm_ctx_init_comm (ncclCommInitRank over NVLink /
 * NVSwitch).  Subdomains created afterwards with decompose != 0 are split into x-slabs: each rank
 * keeps the particles whose base node lies in its slabs, ghost node planes are exchanged after every
 * scatter, reductions are all-reduced, and particles migrate across the cuts after G2P.
 * osmpm_ctx_set_local_slabs splits each rank's share further into n slabs ON THE SAME DEVICE (halo
 * exchange by device copies): the same decomposition testable on one GPU.  nranks == 1 also creates
 * a (one-rank) communicator: the ctx's decomposed subdomains then run the multi-rank code path, every
 * all-reduce / all-gather / broadcast through NCCL, neighbour exchanges finding no neighbour.
 * Reads of a decomposed subdomain fill only this rank's particles / owned nodes (others untouched
 * for particles, zero for dense node vectors); sum over ranks to assemble.
 * Errors: INVALID_ARG (rank / nranks out of range, a second init on one ctx), NCCL (init failed). */
osmpm_status osmpm_comm_unique_id(uint8_t id[128]);
osmpm_status osmpm_ctx_init_comm(osmpm_ctx* ctx, int rank, int nranks, const uint8_t id[128]);
osmpm_status osmpm_ctx_set_local_slabs(osmpm_ctx* ctx, int n);
/* Host-only (no GPU needed): the slab cuts the decomposition uses for particles with base nodes
 * base_x[n] along x: nslab - 1 increasing cell indices, on the lattice of `tile`-cell columns from the
 * lowest base node, each at the column boundary whose prefix particle count is nearest k n / nslab
 * (at least one column per slab).  INVALID_ARG if fewer columns than slabs. */
osmpm_status osmpm_slab_cuts(const int32_t* base_x, int64_t n, int32_t nslab, int32_t tile, int32_t* cuts);
/* slabs_total, slabs_local, first_slab (this rank's first global slab), n_local (particles on this
 * rank now), cuts[slabs_total - 1] (cell index along x where slab k+1 starts; may be NULL). */
osmpm_status osmpm_subdomain_decomp(osmpm_subdomain* sub, int32_t* slabs_total, int32_t* slabs_local,
                                    int32_t* first_slab, int64_t* n_local, int32_t* cuts);

/* ----------------------------------------------------------------------------------------------
 * Subdomain (§3.1: each subdomain owns a grid (dx, dt) and its particles)
 * ----------------------------------------------------------------------------------------------*/
/* Copies the particles into library-owned device SoA (sorted internally; reads return creation
 * order).  mats[n_mats]: material table; gravity[3]: body acceleration g.
 * Errors: INVALID_ARG (bad dims/dx/dt, n < 0, material index out of range),
 * OUT_OF_DOMAIN (a particle outside the safe interior base >= 0, base + 2 <= dims - 1). */
osmpm_status osmpm_subdomain_create(osmpm_ctx* ctx, const osmpm_grid_desc* grid, double dt,
                                    const osmpm_particles_view* particles,
                                    const osmpm_material* mats, int32_t n_mats,
                                    const double gravity[3], osmpm_precision prec,
                                    osmpm_subdomain** out);
/* As osmpm_subdomain_create; decompose = 0 keeps the subdomain whole on this GPU even when the ctx
 * has a process group or local slabs (e.g. the small coarse subdomain, replicated on every rank). */
osmpm_status osmpm_subdomain_create_ex(osmpm_ctx* ctx, const osmpm_grid_desc* grid, double dt,
                                       const osmpm_particles_view* particles,
                                       const osmpm_material* mats, int32_t n_mats,
                                       const double gravity[3], osmpm_precision prec, int32_t decompose,
                                       osmpm_subdomain** out);
void osmpm_subdomain_destroy(osmpm_subdomain* sub);

osmpm_status osmpm_set_gravity(osmpm_subdomain* sub, const double gravity[3]);
osmpm_status osmpm_set_dt(osmpm_subdomain* sub, double dt);
/* Overwrite the particle state in place (same n, creation order): the per-step host upload of the
 * end-to-end benchmark.  Any of the pointers may be NULL (field kept). */
osmpm_status osmpm_set_particles(osmpm_subdomain* sub, const double* x, const double* v,
                                 const double* F, const double* B, osmpm_memspace space);

/* Dirichlet set ("subject to v_Gamma = ..."; R9): n entries with
 * node_idx = linear index in the dense node box, comp_mask bit a = component a constrained,
 * vel = prescribed velocity (n*d).  Replaces the previous user set.  Constrained DOFs are
 * eliminated from the Newton unknowns; the Schwarz receivers are added on top by the coupler. */
osmpm_status osmpm_set_dirichlet(osmpm_subdomain* sub, int64_t n, const int64_t* node_idx,
                                 const uint8_t* comp_mask, const double* vel, osmpm_memspace space);

/* a1 + a2: sort particles into grid blocks (tile-major radix sort), then APIC P2G of mass,
 * momentum and stress (PAPER.md:171 Eq. p2g_transfer, 178, 183), nodal velocity v^n = (mv)/m on
 * active nodes (m_i > 1e-12 median m_p, R4).  Synchronising (reads the node box). */
osmpm_status osmpm_p2g(osmpm_subdomain* sub);

/* Dense reads of the last P2G (any pointer may be NULL): m (nn), p = (mv) (nn*d), v^n (nn*d),
 * f_ext = m g (nn*d), f^sigma = -sum V0 P F^T grad N (nn*d), active (nn, uint8). */
osmpm_status osmpm_read_grid(osmpm_subdomain* sub, double* m, double* p, double* v, double* f_ext,
                             double* f_sigma, uint8_t* active, osmpm_memspace space);

/* a4: Newton gradient of the incremental potential E_h (Eq. discrete_energy) at the
 * displacement-like unknown u = xhat - x^n (dense, nn*d), for ALL node DOFs (no Dirichlet
 * elimination):  g_i = m_i/dt^2 (u_i - dt v_i^n) - f_ext,i + sum_p V0 P(F_p(u)) F_p^nT grad N_ip
 * with F_p(u) = (I + sum_i u_i grad N_ip^T) F_p^n.  *E receives E_h(u) without the
 * constant -sum x_i^n . f_ext,i (R3).  Sets the linearisation point of newton_hvp /
 * newton_diag.  g or E may be NULL. */
osmpm_status osmpm_newton_gradient(osmpm_subdomain* sub, const double* u, double* g, double* E,
                                   osmpm_memspace space);
/* a5: y = H d with H = M/dt^2 + K(u), K the Hessian of the elastic potential at the
 * point set by the last newton_gradient, for ALL node DOFs (dense d, y: nn*d). */
osmpm_status osmpm_newton_hvp(osmpm_subdomain* sub, const double* d, double* y, osmpm_memspace space);
/* Jacobi diagonal diag_{i,a} = e_{i,a}^T H e_{i,a} at the same point (dense nn*d). */
osmpm_status osmpm_newton_diag(osmpm_subdomain* sub, double* diag, osmpm_memspace space);

/* a3-a7: backward-Euler Newton with Jacobi-PCG and backtracking line search
 * from the last P2G, Dirichlet DOFs fixed at dt*v_D.  Stores v^{n+1} = u/dt for osmpm_g2p.
 * Synchronising.  Errors: NEWTON_NOT_CONVERGED, LINESEARCH_STAGNATION (stats filled anyway). */
osmpm_status osmpm_implicit_solve(osmpm_subdomain* sub, const osmpm_newton_settings* settings,
                                  osmpm_solve_stats* stats);
/* Dense read / write of the solved grid velocity v^{n+1} (nn*d).  Writing replaces the solve's
 * result (used to drive osmpm_g2p from a given grid field).  After osmpm_g2p the read still returns the
 * velocity the particles were advanced with, until the next osmpm_p2g / osmpm_restore /
 * osmpm_set_particles (e.g. a coupler frame's last fine sub-step). */
osmpm_status osmpm_read_grid_velocity(osmpm_subdomain* sub, double* v, osmpm_memspace space);
osmpm_status osmpm_set_grid_velocity(osmpm_subdomain* sub, const double* v, osmpm_memspace space);

/* a8: APIC G2P + F update + advection with v^{n+1}:
 * v_p = sum N v_i; B_p = sum N v_i (x_i - x_p)^T; F_p <- (I + dt sum v_i grad N^T) F_p;
 * x_p <- x_p + dt v_p.  Latches INVERTED_F / OUT_OF_DOMAIN. */
osmpm_status osmpm_g2p(osmpm_subdomain* sub);

/* Particle state in creation order (any pointer may be NULL). */
osmpm_status osmpm_read_particles(osmpm_subdomain* sub, double* x, double* v, double* F, double* B,
                                  osmpm_memspace space);
/* n particles, dims of the current internal node box and its offset in the dense box. */
osmpm_status osmpm_subdomain_info(osmpm_subdomain* sub, int64_t* n_particles, int64_t box_lo[3],
                                  int64_t box_dims[3]);

/* a9 / a10: transmission between a coarse and a fine subdomain.
 * FINE_TO_COARSE (src = fine, dst = coarse): Pi_{S->B}: for every coarse target node I
 *     v_I = sum_j m_S,j v_S,j N_B,I(x_S,j) / (sum_j m_S,j N_B,I(x_S,j) + eps_tol)
 *   over the ACTIVE fine nodes j of src's last P2G, using src's v^n (alpha == 0) or its solved
 *   v^{n+1} (alpha == 1); Eq. spatial_projection.
 * COARSE_TO_FINE (src = coarse, dst = fine): I_{B->S} then T_m (Eqs. interp_BtoS, temporal_interp):
 *     v_j = (1 - alpha) sum_I v_B,I^n N_B,I(x_S,j) + alpha sum_I v_B,I^{n+1} N_B,I(x_S,j)
 *   with v_B^n from src's last P2G and v_B^{n+1} its solved / set grid velocity; alpha in [0,1].
 * targets: n_targets linear node indices of dst's dense box (NULL: all nodes of dst's box,
 *   n_targets must then equal dst's node count); v_out: n_targets*d.  eps_tol only for Pi.
 * Coarse stencil nodes outside the coarse box contribute / receive nothing (R9).
 * Errors: INVALID_ARG for alpha outside [0, 1] (FINE_TO_COARSE: alpha not 0 or 1), n_targets < 0,
 *   targets == NULL with n_targets != dst node count, or a HOST target outside dst's dense box (checked
 *   before any work).  A DEVICE target outside the box is skipped (its output row is 0) and latched:
 *   INVALID_ARG with its position in `targets` at the next synchronising call / osmpm_sync of the
 *   coarse subdomain.  STATE if src has no grid (no osmpm_p2g) or alpha > 0 without a solved velocity.
 * Pi is evaluated as a gather (fixed-order sums, no atomics): bitwise reproducible. */
osmpm_status osmpm_transmit(osmpm_subdomain* src, osmpm_subdomain* dst, osmpm_direction dir,
                            double alpha, double eps_tol, int64_t n_targets, const int64_t* targets,
                            double* v_out, osmpm_memspace space);

/* ----------------------------------------------------------------------------------------------
 * Schwarz coupler (Alg. 1)
 * ----------------------------------------------------------------------------------------------*/
osmpm_status osmpm_coupler_create(osmpm_subdomain* coarse, osmpm_subdomain* fine,
                                  const osmpm_schwarz_settings* settings, osmpm_coupler** out);
void osmpm_coupler_destroy(osmpm_coupler* cpl);
/* Host only (no GPU): the coupler's receiver decision for one fine node box -- the whole fine subdomain,
 * or one slab of it with its two ghost planes (R21) -- exposed so that the distributed
 * arbitration can be tested without GPUs.  Gamma_S candidates are the box nodes with active_s and
 * mb_s > tau_s (Eq. boundary_grid_set); a candidate coinciding with a coarse node
 * flagged in gamma_b is arbitrated by raw nodal mass, ties to B (Eq. overlap_donor):
 * if B donates, drop_b[that coarse box node] is set to 1 (the fine side receives), else the candidate is
 * dropped; a remaining candidate is a fine receiver if every coarse stencil node with N > 0 is active
 * (R13).  Boxes: node k = lo + l, box-local index (l0 * dims1 + l1) * dims2 + l2 (2D: dims[2]
 * ignored); all per-node arrays are over the box.  recv (capacity n_cap; NULL: count only) receives the
 * dense fine node indices of the receivers, ascending; owned[q] = 1 if its box-local index is < nown
 * (the slab owns it; ghost-plane nodes come after the owned ones).  Errors: INVALID_ARG (NULL, dims,
 * capacity). */
osmpm_status osmpm_schwarz_receivers_host(const osmpm_grid_desc* coarse, const int64_t coarse_lo[3],
                                          const int64_t coarse_dims[3], const double* m_b, const uint8_t* gamma_b,
                                          const uint8_t* active_b, const osmpm_grid_desc* fine,
                                          const int64_t fine_lo[3], const int64_t fine_dims[3], int64_t nown,
                                          const double* m_s, const double* mb_s, const uint8_t* active_s,
                                          double tau_s, uint8_t* drop_b, int64_t n_cap, int64_t* recv,
                                          uint8_t* owned, int64_t* n_recv);

/* Step 0 of Alg. 1: store fine particles, P2G both, Gamma_B, Gamma_S,
 * arbitration, receivers, v_Gamma_B^(0) = Pi(v_S^n).  Called by schwarz_step; exposed so a caller
 * can drive sub-steps itself. */
osmpm_status osmpm_schwarz_prepare(osmpm_coupler* cpl);
/* One fine sub-step m (1..M) of Alg. 1: T_m BCs on the fine receivers, implicit
 * solve, G2P + advection, P2G.  Uses the coarse endpoint fields of the current iteration. */
osmpm_status osmpm_schwarz_substep(osmpm_coupler* cpl, int32_t m, osmpm_solve_stats* stats);
/* Whole frame t_n -> t_n+1 (Alg. 1). */
osmpm_status osmpm_schwarz_step(osmpm_coupler* cpl, osmpm_schwarz_report* report);

/* CUDA-core FMA throughput of the ctx's device in TFLOP/s (fp64 or fp32 by `prec`): 8 independent FMA
 * chains per thread on 8 CTAs of 256 threads per SM, best of 5 event-timed launches.  The measured
 * denominator of bench.py's `roofline.fp_pipe` (MEASURED_PEAKS.json has no CUDA-core
 * peak).  Synchronising. */
osmpm_status osmpm_measure_fma_peak(osmpm_ctx* ctx, osmpm_precision prec, double* tflops);

/* a1 building block, exposed for testing: stable LSD radix sort (8 bits per pass) of n (key, value)
 * pairs on the low nbits bits of the keys, in place; equal keys keep their input order.  This is the
 * sort osmpm_p2g runs on the particles' tile-major cell keys every step (north_star: "block-level
 * radix sort").  keys, vals: n entries each, host or device memory per `space`.  Synchronising.
 * Errors: INVALID_ARG (n outside [0, 2^31), nbits outside [0, 32], NULL arrays), OOM. */
osmpm_status osmpm_sort_pairs(osmpm_ctx* ctx, uint32_t* keys, int32_t* vals, int64_t n, int32_t nbits,
                              osmpm_memspace space);

/* a11 (PAPER.md:376-379 Eq. store_states, 455 Alg. 1 "reset"): osmpm_checkpoint stores the whole
 * particle state {x, v, F, B, m, V0, material, P^∂ flag, id} -- per slab, with its particle count,
 * for a decomposed subdomain -- in library-owned device memory (one copy per subdomain; a second
 * call overwrites it); osmpm_restore copies it back, so the next osmpm_p2g starts from exactly the
 * stored state.  Device-to-device copies on the ctx stream, asynchronous.  Errors: STATE (restore
 * without a checkpoint), OOM. */
osmpm_status osmpm_checkpoint(osmpm_subdomain* sub);
osmpm_status osmpm_restore(osmpm_subdomain* sub);

/* Block until all work of the ctx is done; surfaces latched device errors. */
osmpm_status osmpm_sync(osmpm_subdomain* sub);

#ifdef __cplusplus
}
#endif
#endif /* OSMPM_H */
