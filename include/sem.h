/*
 * sem.h -- C ABI of libsem: one explicit leapfrog time step of the coupled PMUT-array /
 * DG-SEM acoustic model of arxiv 2603.06267, in FP64 on NVIDIA B200 (sm_100a).
 *
 * Citations are PAPER.md lines (P:L<n>), equations in the paper's LaTeX order, and the
 * readings R<n> listed in DESIGN.md.  All quantities are SI.
 *
 * Problem (Eqs. 9-12):   M p'' + K p + C p' = f(q'')      (acoustic, DG-SEM)
 *                                     q'' + W q = g(p, phi)            (PMUT modal ROM)
 * advanced by Algorithm 1 (Newmark gamma = 1/2, beta = 0 == leapfrog) with the
 * coupling time level of reading R2 (default: the PMUT solve consumes the acoustic predictor).
 *
 * Conventions (all entry points):
 *  - Host arrays passed in are owned by the caller and copied before the call returns.
 *  - The context owns every device allocation it makes (cudaMalloc on ctx->device).
 *  - Every call returns a sem_status; no C++ exception crosses the ABI.  On error the
 *    context's message is available from sem_last_error(ctx) (NULL-safe).
 *  - sem_step only enqueues work on the context stream; asynchronous CUDA errors surface at
 *    the next synchronising call (sem_read_*, sem_sync, sem_query).
 *  - One context per rank / device; a context is not thread-safe.
 *  - Node layout of every acoustic field (input and output): per box, lexicographic over the
 *    GLL lattice, x fastest:  id = gx + NX (gy + NY gz),  NX = N nel_x + 1 (P:L413-420,
 *    continuous inside a box, discontinuous across the DG interface).
 */
#ifndef SEM_H
#define SEM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sem_ctx sem_ctx;   /* opaque: device state of one rank */

typedef enum {
    SEM_OK = 0,
    SEM_E_ARG = -1,        /* invalid argument (degree outside 1..8, overlapping membranes, C <= 0, ...) */
    SEM_E_CUDA = -2,       /* CUDA runtime error (message holds cudaGetErrorString) */
    SEM_E_NCCL = -3,       /* NCCL error in the slab halo exchange */
    SEM_E_STATE = -4,      /* call out of order (e.g. interface built twice, step before setup) */
    SEM_E_NONFINITE = -5,  /* NaN/Inf detected (SEM_F_NAN_CHECK); message names the step */
    SEM_E_PARTITION = -6,  /* slab cut not element- / 2:1- / membrane-aligned */
    SEM_E_UNMATCHED = -7,  /* interface quadrature point without a coarse owner */
    SEM_E_OOM = -8         /* device allocation failed */
} sem_status;

/* Boundary condition of each box face, order -x, +x, -y, +y, -z, +z. */
typedef enum {
    SEM_BC_RIGID = 0,      /* hard wall, homogeneous Neumann (natural; no work)               */
    SEM_BC_ABSORBING = 1,  /* first-order ABC, d(w, v) = int_F c w v (Eq. 8)      */
    SEM_BC_INTERFACE = 2   /* DG interface Gamma_I, set up by sem_dg_interface_build (Eq. 7)  */
} sem_bc;

/* Coupling time level of the PMUT solve (reading R2). */
enum {
    SEM_F_COUPLING_LITERAL = 1 << 0, /* g(p^n, phi^n) exactly as printed (unstable at cfg masses)  */
    SEM_F_NAN_CHECK = 1 << 1,        /* check p for NaN/Inf after every sem_step call              */
    SEM_F_NO_GRAPH = 1 << 2,         /* launch kernels directly instead of a captured CUDA graph   */
    SEM_F_EMULATE_SLABS = 1 << 3     /* world > 1 in ONE context on one device: every y-slab of the
                                        decomposition lives here and the per-step exchange is a
                                        device copy instead of NCCL (verifies the slab path on 1 GPU) */
};

/* One axis-aligned box of hexahedral GLL elements of degree `degree` (1..8). */
typedef struct {
    double origin[3];      /* lower corner [m]                                      */
    double extent[3];      /* edge lengths [m]                                      */
    int nel[3];            /* elements per axis (>= 1)                              */
    int degree;            /* GLL degree N (1..8); (N+1)^3 nodes per element        */
    double c;              /* sound speed [m/s] (> 0)                               */
    double rho;            /* density [kg/m^3] (>= 0); kappa = rho c^2     */
    int bc[6];             /* sem_bc per face                                       */
} sem_box_desc;

typedef struct {
    int n_boxes;                 /* 1 or 2                                               */
    const sem_box_desc* boxes;   /* [n_boxes]                                            */
    double dt;                   /* time step [s], caller-computed (reading R8)          */
    int device;                  /* CUDA device ordinal                                  */
    void* stream;                /* cudaStream_t to enqueue on; NULL -> library stream   */
    int rank, world;             /* y-slab decomposition: rank r's slab = box-0 elements
                                    [slab_y0[r], slab_y0[r+1]) along y and the same y range of every
                                    other box (see slab_y0)                                      */
    const void* nccl_unique_id;  /* ncclUniqueId (128 bytes) when world > 1, else NULL  */
    int flags;                   /* SEM_F_*                                              */
    /* Optional caller allocator for every persistent device array of the context (e.g. the torch
     * caching allocator, so the library shares the caller's memory pool); NULL -> cudaMalloc /
     * cudaFree.  dev_alloc(bytes, alloc_user) returns device memory (>= 256-byte aligned) on
     * `device` or NULL (-> SEM_E_OOM); dev_free(ptr, alloc_user) is called from sem_destroy. */
    void* (*dev_alloc)(size_t bytes, void* user);
    void (*dev_free)(void* ptr, void* user);
    void* alloc_user;
    /* Optional slab plan [world + 1]: box-0 element y index where each slab starts (0 first, nel_y
     * last, increasing; from sem_slab_plan).  NULL -> equal slabs (nel_y divisible by world).  Every
     * cut must be an element boundary of every box (so the cuts of a 2:1 interface sit on coarse
     * elements) -> SEM_E_PARTITION otherwise; cuts crossing a membrane are rejected by
     * sem_pmut_attach (SEM_E_PARTITION). */
    const long long* slab_y0;
} sem_mesh_desc;

/* Create the context: validates boxes, builds the 1D GLL tables and allocates p (two time
 * levels), w = p' + dt/2 p'' (one level) per box (this rank's y-slab), zero-initialised
 * (P:L609-610).  The structured step keeps only the two p levels current (w^n = (p^{n+1} - p^n)/dt
 * is recomputed); w serves the element-scatter boxes.  With world > 1 (and no
 * SEM_F_EMULATE_SLABS) every rank calls it with the same global boxes, the same slab plan and the
 * ncclUniqueId from sem_nccl_unique_id on rank 0; each step then exchanges one cut plane per box with
 * each y-neighbour.
 * Errors: SEM_E_ARG (bad descriptor), SEM_E_PARTITION (no slab_y0 and nel_y not divisible by world,
 * or a slab_y0 cut that is not an element boundary of every box), SEM_E_NCCL, SEM_E_CUDA /
 * SEM_E_OOM.  *out is NULL on error. */
sem_status sem_mesh_create(const sem_mesh_desc* desc, sem_ctx** out);

/* 128-byte ncclUniqueId for world > 1 (rank 0 calls it and broadcasts the bytes).
 * NCCL is loaded with dlopen("libnccl.so.2"); SEM_E_NCCL if it is unavailable. */
sem_status sem_nccl_unique_id(void* out128);

/* PMUT array on face `face` (only 4 = -z) of box `box` (Eqs. 2-3, 5, 11-12).
 * Mode shapes S_{k,m}(x,y) = sin(m pi x'/a) sin(n pi y'/a) on the square membrane of side a
 * centred at center[k] (reading R19); U.n = -S (reading R4).  Modal ODE (reading R3):
 *   q'' = -w^2 q - 2 zeta w q'* + (int_gamma_k p U.n + eta phi) / M_m,   w = 2 pi freq_hz.
 * phi_k = TX Hann burst amp_v sin(2 pi f0 t')(1 - cos(2 pi f0 t'/n_cycles))/2, t' = t - delay_s[k]
 * in [0, n_cycles/f0] (reading R10) for t <= t_switch; (1/C) sum_m eta_m q_m after (Eq. 3).
 * Arrays: center [n_pmut*2] (x, y), mode_mn [n_modes*2], freq_hz [n_pmut*n_modes] (k-major),
 * modal_mass / damping_ratio / eta [n_modes], delay_s [n_pmut].  n_modes <= 8.
 * The box may be a structured box, an affine obstacle box (sem_box_set_obstacle, called first) or a
 * curved box (sem_box_set_vertices, called first): there the coupling is tabulated per membrane node,
 * B_{k,m,j} = sum_F w_a w_b |J_s| S_{k,m}(x_j) with the trilinear face's |J_s| and physical node
 * positions (not separable), and the force enters the box's assembled residual.
 * Caller-defined mode shapes (the paper's U_{k,m} are the eigenmodes of a 3D FEM model of the
 * membrane, so any shape must be admissible -- e.g. the circular membranes of P:L1097, reading
 * R33): with shape_fn != NULL the table uses S_{k,m}(x_j) = shape_fn(k, m, x_j - center_x, y_j -
 * center_y, shape_user) instead of the square sines; it is called on the host during this call only,
 * for the face nodes inside the membrane's bounding square of side `side` (S = 0 outside it; a disc's
 * shape returns 0 beyond its radius); mode_mn is then only a label.  Needs the tabulated coupling, i.e.
 * a curved box (sem_box_set_vertices, possibly with the affine lattice): SEM_E_ARG on any other box.
 * Errors: SEM_E_ARG (membranes overlapping or off the face, zero-node membrane, membrane on a solid
 * element's face, rx with C <= 0, a non-finite shape value), SEM_E_STATE (already attached). */
typedef double (*sem_shape_fn)(int k, int m, double x_rel, double y_rel, void* user);
typedef struct {
    int box, face;
    int n_pmut, n_modes;
    const double* center;
    double side;
    const int* mode_mn;
    const double* freq_hz;
    const double* modal_mass;
    const double* damping_ratio;
    const double* eta;
    int rx;                       /* 1: open-circuit RX feedback for t > t_switch        */
    double t_switch;              /* t_bar [s]; +inf for pure TX                */
    double capacitance;           /* C [F]                                               */
    double amp_v, f0_hz;          /* TX burst amplitude [V] and carrier [Hz]             */
    int n_cycles;
    const double* delay_s;
    sem_shape_fn shape_fn;        /* NULL: the square sines of mode_mn (reading R19)     */
    void* shape_user;
} sem_pmut_desc;
sem_status sem_pmut_attach(sem_ctx* ctx, const sem_pmut_desc* pm);

/* Host-only (no device touched): the y-slab plan of `world` slabs for these global boxes and (optional)
 * PMUT array.  slab_y0[world+1] receives the box-0 element y index where each slab starts: equal slabs
 * when they are admissible, else the admissible cuts nearest to the equal ones (uneven slabs): every cut
 * on an element boundary of every box (so a 2:1 interface's face pairs stay slab-local) and in a gap
 * between membranes (the paper's membrane-preserving partition).  SEM_E_PARTITION if
 * no admissible plan exists. */
sem_status sem_slab_plan(const sem_box_desc* boxes, int n_boxes, int world, const sem_pmut_desc* pm,
                         long long* slab_y0);

/* Non-conforming SIPG interface between the +z face of `fine_box` and the -z face of
 * `coarse_box` (Eq. 7's three Gamma_I sums), gamma_F = penalty_alpha cbar^2
 * max(N+, N-)^2 / min(h+, h-) with cbar the harmonic mean of c (reading R7).
 * quad_rule 0 = the fine faces' (N+ + 1)^2 GLL nodes (reading R9, collocated with the fine trace);
 * quad_rule 1 = their (N+ + 1)^2 Gauss-Legendre points (R9's flag, Fig. 7's "LG" nodes):
 * the fine trace is interpolated to the points and the fine side's terms projected back onto the
 * fine face nodes; single slab only (world 1, no emulation: SEM_E_PARTITION otherwise).
 * Requires matching lateral extents; h_coarse = R h_fine for an integer R >= 1 gives the lattice kernel,
 * otherwise (lattices that do not nest, e.g. 6 : 4 elements) both boxes move to the element-scatter
 * path with their affine vertex lattices and take the general interface below (single slab, GLL rule,
 * no PML / plane wave on them: SEM_E_UNMATCHED otherwise).
 * Curved boxes (sem_box_set_vertices / sem_box_set_obstacle on BOTH boxes, before this call): the
 * general non-conforming interface -- any trilinear face sets that tile the same surface, lattices that
 * need not nest.  Algorithm 3 (sem_face_match) gives every
 * fine-face GLL node its coarse owner and x_hat^- at setup; per step one kernel evaluates the face terms
 * of Eq. 7 at those points (J = p+ - p-(x_hat^-), A = {c^2 d_n p}, n = n+ of the fine face) and adds them
 * to both boxes' assembled residuals.  GLL rule only, world 1 only (SEM_E_PARTITION), SEM_E_STATE if only
 * one of the boxes is curved, SEM_E_UNMATCHED if a quadrature node has no owner.
 * Errors: SEM_E_ARG (geometry), SEM_E_UNMATCHED (lattices do not nest), SEM_E_STATE. */
sem_status sem_dg_interface_build(sem_ctx* ctx, int fine_box, int coarse_box, double penalty_alpha,
                                  int quad_rule);

/* Curved box (trilinear maps X_K of P:L415-416): replace the affine geometry of
 * `box` by the vertex lattice verts[n_verts][3], n_verts = (nel_x+1)(nel_y+1)(nel_z+1), x fastest
 * (element (ex,ey,ez) vertex v = i + 2j + 4k is lattice vertex (ex+i, ey+j, ez+k)); connectivity stays
 * the box's lattice.  The box then uses the element-scatter path: K p element by element with the
 * metric terms w_q c^2 |J| J^-1 J^-T recomputed from the 8 vertices at every GLL point (nothing
 * stored per quadrature point), FP64 atomics into an assembled residual, and a nodal kick-drift with
 * the assembled lumped mass and ABC diagonal (computed here on the host).  Call right after
 * sem_mesh_create: curved boxes carry no PML (SEM_E_STATE); PMUTs (tabulated coupling), a plane wave and
 * an interface between two curved boxes (the general one of sem_dg_interface_build) are attached
 * afterwards; world 1 only (SEM_E_PARTITION).  Caller owns `verts` (copied).  Errors: SEM_E_ARG (size, non-positive
 * Jacobian at a GLL point), SEM_E_STATE, SEM_E_OOM. */
sem_status sem_box_set_vertices(sem_ctx* ctx, int box, const double* verts, size_t n_verts);

/* Rigid obstacle inside box `box` ("obstacle Neumann surfaces"): solid[n_el],
 * n_el = nel_x nel_y nel_z, element (ex,ey,ez) at index ex + nel_x (ey + nel_y ez); solid[e] != 0
 * removes element e from the fluid domain Omega.  The faces it shares with fluid elements become
 * Neumann (rigid) surfaces -- the natural boundary condition of the weak form, Eq. (4) with no
 * boundary term there -- so nothing is assembled for them: the element's stiffness, mass and
 * absorbing-face terms are skipped.  Nodes of no fluid element (obstacle interiors) are held at 0
 * (sem_read_pressure returns 0 there after the first step).  The box moves to the element-scatter
 * path of sem_box_set_vertices (with its own affine vertex lattice unless vertices are set, before or
 * after this call) and carries the same restrictions (no PML / plane wave: SEM_E_STATE; a general
 * interface only with another curved / obstacle box;
 * world 1 only: SEM_E_PARTITION) except one: an affine obstacle box (no vertices set) may carry the
 * PMUT array (the paper's Section 6.2 scenario, a PMUT transmitting to an obstacle and receiving its
 * echo): the modal kernel is unchanged and the nodal update adds f = kappa B^T qdd on
 * the z = 0 face.  Call it before sem_pmut_attach (SEM_E_STATE otherwise); a membrane on the face of
 * a solid element is rejected by sem_pmut_attach (SEM_E_ARG).  Caller owns `solid` (copied).
 * Errors: SEM_E_ARG (size, every element solid), SEM_E_STATE (already set), SEM_E_OOM. */
sem_status sem_box_set_obstacle(sem_ctx* ctx, int box, const unsigned char* solid, size_t n_el);

/* Perfectly matched layer (Eq. 1 lines 1-3; coefficients P:L271-277; profile P:L280-289)
 * inside box `box`: thickness[f] [m] for faces f = -x,+x,-y,+y,-z,+z (0 = no layer) is the slab of the
 * box next to face f; z_d(d) = zt (d/l - sin(2 pi d/l)/(2 pi)), d = depth into the layer,
 * zt = (c/l) log(1/R), 0 < R < 1 (the paper uses R in [1e-5, 1e-4]).  The faces keep their own
 * boundary condition (the paper's Gamma_ABC behind the layer: tag them SEM_BC_ABSORBING).
 * Discretisation (readings R23-R25): psi continuous nodal, Phi element-local, div Phi in weak
 * form, psi/Phi at half steps (Crank-Nicolson on Z1), PML terms at the predictor velocity.
 * Under y-slabs (world > 1, NCCL or emulated) the profiles come from the global box and the PML
 * accelerations of the cut-plane nodes travel with the cut exchange (reading R31).
 * Caller owns `thickness` (copied).  Errors: SEM_E_ARG (negative thickness, overlapping layers, R
 * outside (0, 1)), SEM_E_STATE (already attached, curved box), SEM_E_OOM.  Resets the dynamic state
 * like sem_pmut_attach. */
sem_status sem_pml_attach(sem_ctx* ctx, int box, const double* thickness, double R);

/* Algorithm 3 (face matching on the non-conforming interface) on GPU `device`: for every
 * quadrature node x_q = X_{K+}(xhat_q+) of every fine face (the face's GLL nodes of `degree`, reading R9;
 * node q = a + (degree+1) b, a along the face's first tangential axis) find the coarse face dK- that
 * contains it: opposite normals |n+ + n-| < normal_tol (centre normals), one-vertex radius filter
 * |V_{K-} - x_q| < max(diam dK-, diam dK+) + eps, Newton-Raphson xhat_q- = X_{K-}^{-1}(x_q), accept if
 * xhat_q- in [-1,1]^3 (1e-9 tolerance); the lowest coarse index wins (reading R26).  A uniform grid of
 * the coarse faces' first vertices (cell = the largest filter radius) supplies the candidates.
 * Face sets (host, caller-owned, copied): verts [n][8][3] of the trilinear elements (vertex v = i + 2j
 * + 4k at reference corner (2i-1, 2j-1, 2k-1)), face [n] local face 0..5 (-x,+x,-y,+y,-z,+z).
 * Outputs (host, caller-owned): owner [n_fine (degree+1)^2] coarse face index or -1, xi_minus [..][3];
 * elapsed_ms (optional) = device time of the matching kernels.  Self-contained (no sem_ctx).
 * Errors: SEM_E_ARG, SEM_E_CUDA, SEM_E_OOM; SEM_E_UNMATCHED if some node has no owner (outputs filled). */
typedef struct {
    int n;
    const double* verts;
    const int* face;
} sem_face_set;
sem_status sem_face_match(int device, const sem_face_set* fine, const sem_face_set* coarse, int degree,
                          double normal_tol, long long* owner, double* xi_minus, double* elapsed_ms);

/* Incident plane wave entering through absorbing face `face` (only 5 = +z) of `box`
 * (reading R13): p_inc = amp s(t - k.(x - x_ref)/c), s(u) = exp(-(u-t0)^2/(2 sigma^2))
 * sin(2 pi f0 (u-t0)), imposed as total-field first-order ABC data
 * b_j = int c amp s'(tau) (1 - n.k) psi_j.  dir is the unit propagation direction k.
 * On a curved box (sem_box_set_vertices first; every box of the context on the element-scatter path,
 * SEM_E_STATE otherwise) the load is tabulated per face node with the trilinear faces' weights
 * w_a w_b |J_s| and physical node positions; the +z face must be planar (SEM_E_ARG), x_ref is the
 * first-hit corner of its bounding rectangle.
 * Errors: SEM_E_ARG (face, non-absorbing face, parameters), SEM_E_STATE. */
sem_status sem_plane_wave_source(sem_ctx* ctx, int box, int face, double amp_pa, double f0_hz,
                                 double sigma_s, double t0_s, const double dir[3]);

/* Advance n_steps iterations of Algorithm 1 (async on the context stream). */
sem_status sem_step(sem_ctx* ctx, int n_steps);

/* Block until all enqueued work finished; reports asynchronous errors. */
sem_status sem_sync(sem_ctx* ctx);

/* p^S of box `box` after S steps into host[n] (n must equal the box's global node count).
 * Synchronising.  Shared DG interface nodes are reported once per side.  With world > 1 this is
 * collective: every rank calls it, rank 0 receives the assembled field (host may be NULL elsewhere). */
sem_status sem_read_pressure(sem_ctx* ctx, int box, double* host, size_t n);

/* p^S at n sampled global node ids (layout above) of `box` into out[n] (host).  Synchronising.
 * Single-process only (world 1 or SEM_F_EMULATE_SLABS): SEM_E_STATE under NCCL. */
sem_status sem_read_pressure_at(sem_ctx* ctx, int box, const long long* ids, size_t n, double* out);

/* q^S, q'^S [n_pmut*n_modes] and phi_k(t^S) [n_pmut] (received voltage for RX, drive for TX), in
 * the global PMUT order.  n must equal n_pmut*n_modes.  Any pointer may be NULL.  Synchronising;
 * collective with world > 1 (rank 0 receives). */
sem_status sem_read_modal(sem_ctx* ctx, double* q, double* qdot, double* v_rx, size_t n);

/* Test hook: set p^0, p'^0 of `box` from host arrays [n] (p''^0 = 0; reading R20),
 * modal state and step counter reset to zero for every box's first call. */
sem_status sem_write_state(sem_ctx* ctx, int box, const double* p, const double* pdot, size_t n);

/* Test hook: fill p^0 = p_scale u(seed, box, 0, id), p'^0 = v_scale u(seed, box, 1, id) on the
 * device with the counter-based generator u in [-1, 1) documented in DESIGN.md (splitmix64);
 * p''^0 = 0, modal state and step counter reset. */
sem_status sem_fill_random_state(sem_ctx* ctx, int box, unsigned long long seed, double p_scale,
                                 double v_scale);

/* Total acoustic node count over all boxes of this rank, steps taken, and t = steps * dt. */
sem_status sem_query(sem_ctx* ctx, long long* n_dof, long long* step, double* t);

/* Per-kernel device time [ms] accumulated since the last reset while SEM_F_NO_GRAPH profiling
 * is enabled (sem_set_profiling).  which: 0 = volume (all boxes), 1 = interface, 2 = modal,
 * 3 = PML element kernel.
 * n_launches receives the number of launches timed. */
sem_status sem_set_profiling(sem_ctx* ctx, int on);
sem_status sem_kernel_time(sem_ctx* ctx, int which, double* ms, long long* n_launches);

/* Number of kernel launches issued by the last sem_step call (graph nodes counted). */
sem_status sem_last_launch_count(sem_ctx* ctx, long long* n);

const char* sem_last_error(const sem_ctx* ctx);
void sem_destroy(sem_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SEM_H */
