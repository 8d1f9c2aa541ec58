// Internal declarations of libsem (host setup <-> kernels).  Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/sem.h"

// Device-side bounds checks of the debug build (libsem_debug.so, -DSEM_DEBUG_CHECKS): the stand-in for
// compute-sanitizer memcheck, which this pool does not offer.  A failed check prints the condition and
// traps (the next sync call reports the CUDA error).
#ifdef SEM_DEBUG_CHECKS
#include <cstdio>
#define SEM_CHECK(cond)                                                                                    \
    do {                                                                                                   \
        if (!(cond)) {                                                                                     \
            printf("libsem debug check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);                  \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
#define SEM_CHECK(cond) \
    do {                \
    } while (0)
#endif

namespace sem {

// Two-level time stepping of the structured volume kernel: the state is p^{n+1},
// p^n; the half-step velocity w^n = (p^{n+1} - p^n) / dt is recomputed per node instead of stored, so a
// step reads p^{n+1} (with the stencil halo) and p^n and writes p^{n+2} over p^n: 24 B per DOF-step
// instead of 32 (p, w read and written).  The element-scatter (curved / obstacle) update does the same
// (56 instead of 64 B per node).
#ifndef SEM_TWO_LEVEL
#define SEM_TWO_LEVEL 1
#endif

constexpr int kMaxN = 8;          // supported GLL degrees 1..8
constexpr int kRows = kMaxN + 3;  // row classes per direction: R[0..N-1], L, B0, BN
constexpr int kMaxModes = 8;
#ifndef SEM_KPREF
#define SEM_KPREF 16
#endif
constexpr int kPref = SEM_KPREF;  // volume kernel: planes prefetched beyond the z-stencil window

// Volume kernel tile geometry for degree N: one warp spans a row of
// TXE = N floor(31/N) computed nodes (whole elements); lane 31 is the "virtual left neighbour"
// that evaluates the left-element row of lane 0's shared node from the halo.
// TMA box x-starts must be 16 B aligned: TXE is even and the x halo is NH = N rounded up to even.
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int vol_txe(int N) { return (N * (31 / N)) % 2 ? N * (31 / N) - N : N * (31 / N); }
__host__ __device__ constexpr int vol_nh(int N) { return N + (N & 1); }
__host__ __device__ constexpr int vol_pbox_w(int N) { return vol_txe(N) + 2 * vol_nh(N); }
// W tile: TXE + 1 nodes (the last x tile of a box also takes the box's last node, so NX = k TXE + 1
// needs k tiles, not k + 1), rounded up to an even count (TMA boxes are 16-byte multiples)
__host__ __device__ constexpr int vol_wbox_w(int N) { return ((vol_txe(N) + 2) / 2) * 2; }
// slot = [P tile | pad to 128 B | W tile | pad to 128 B]: TMA destinations must be 128 B aligned
__host__ __device__ constexpr int vol_pbytes_aligned(int N, int TY) {
    return ((vol_pbox_w(N) * (TY + 2 * N) * 8 + 127) / 128) * 128;
}
__host__ __device__ constexpr int vol_slot_bytes(int N, int TY) {
    return vol_pbytes_aligned(N, TY) + ((vol_wbox_w(N) * TY * 8 + 127) / 128) * 128;
}
// ring depth: the z window (N + 1 planes) + 1 + kPref planes of prefetch, capped by shared memory
// (227 KB per CTA; per slot: the tiles, two mbarriers and a tile header)
constexpr int kSmemMax = 227 * 1024;
__host__ __device__ constexpr int vol_depth_for_slot(int N, int slot) {
    return (N + 2 + kPref) * (slot + 20) + 128 <= kSmemMax ? N + 2 + kPref : (kSmemMax - 128) / (slot + 20);
}
__host__ __device__ constexpr int vol_depth(int N, int TY) { return vol_depth_for_slot(N, vol_slot_bytes(N, TY)); }

// Row-class indices inside a direction table.
//   R[a]  interior node with local index a (a = 0: shared, right element), base = i - a
//   L     interior shared node (a = 0), left element, base = i - N
//   B0    box lower boundary node (i = 0), right element only
//   BN    box upper boundary node (i = N nel), left element only
__host__ __device__ constexpr int row_L(int N) { return N; }
__host__ __device__ constexpr int row_B0(int N) { return N + 1; }
__host__ __device__ constexpr int row_BN(int N) { return N + 2; }

// Per-box coefficient tables, passed by value inside VolParams (kernel parameter constant bank,
// per launch: contexts never share them).
struct BoxTables {
    // G[d][row][b] = c^2 (2/h_d)^2 A_hat[a][b] / w_asm(a)   (M^-1 K restricted to direction d)
    double G[3][kRows][kMaxN + 1];
    // interface layer coefficients: a -= tau * ktau[c] + sigma * ksig[c] on the element layer
    // adjacent to the interface (c = local index across that layer, 0..N)
    double ksig[kMaxN + 1];
    double ktau[kMaxN + 1];
};

struct VolParams {
    CUtensorMap tmP;                // TMA map of p^{n+1} (3D: NX, NY, NZ; row pitch PX)
    CUtensorMap tmW;                // TMA map of w^n (two-level: of p^n, the same box shape)
    BoxTables tab;
    double* __restrict__ Pn;        // p^{n+2} (output)
    double* __restrict__ W;         // w^n in, w^{n+1} out (in place)
    long long NX, NY, NZ;           // node counts of the (local) box
    long long PX;                   // row pitch (doubles) of the device layout
    int N;                          // GLL degree of the box
    double sdir[3];                 // s_d = c^2 (2/h_d)^2: scale of the compile-time reference rows
    int nelz;
    double dt;
    double inv_dt;
    // lumped ABC: C_ii / M_ii at boundary nodes of absorbing faces (0 if rigid)
    double damp[6];
    // PMUT forcing plane on z = 0 (F = kappa sum_m qdd S), scaled by kF = 1 / m_z(0)
    const double* __restrict__ F;
    double kF;
    // slab cuts (multi-GPU): this slab's -x / +x face is an internal cut, not a box face
    int cutL, cutR;                 // this slab's -y / +y face is an internal cut (y-slabs)
    // DG interface layer: side = +1 (this box's +z face is Gamma_I, fine side),
    // -1 (its -z face, coarse side), 0 none; tau / sigma on the face lattice [NX*NY]
    int iface_side;
    const double* __restrict__ tau;
    const double* __restrict__ sig;
    // plane-wave boundary source on the +z face (reading R13)
    int pw_on;
    double pw_fac;                  // c A (1 - n.k) / m_z(top)
    double pw_k[3], pw_xref[3], pw_c, pw_t0, pw_sigma, pw_om, pw_ztop;
    const double* __restrict__ xc; // node x coordinates [NX]
    const double* __restrict__ yc; // node y coordinates [NY]
    // device step counter: t^{n+1} = (step + 1) dt (read by the plane-wave source)
    const long long* step;
    // fine side of the structured interface (iface_side > 0), one GPU, no PML on the box: the kernel also
    // writes d_z p^{n+2} at the top face, dzf[iy NX + ix] = sum_c dzc[c] p^{n+2}(top - N + c) (the
    // next step's interface reads it instead of the top element's N + 1 planes); nullptr otherwise
    double* dzf;
    double dzc[kMaxN + 1];
};

// One persistent volume launch: one or two boxes (box[1] of degree N1 != N0 shares the launch so
// that a single plane stream per SM covers the whole step; see vol_kernel).
struct VolLaunch {
    VolParams box[2];
    int nbox;                       // 1 or 2
    unsigned ntx[2];                // tiles along x per box (filled by launch_volume)
    unsigned nty[2];                // tiles along y per box
    unsigned ntiles[2];             // tiles per box
    unsigned int* sched;            // [0] next tile, [1] finished CTAs; reset by the launch's last CTA
    long long* step;                // device step counter, bumped by the last CTA if bump_step
    int bump_step;                  // 1 for the last volume launch of a step
    int reserve_sms;                // SMs kept free (NCCL exchange running beside the launch)
    int ty;                         // consumer rows per tile (volume_tile_y of the context)
};

struct ModalParams {
    int n_pmut, n_modes, lmax;      // lmax = stride of the per-pmut 1D tables
    int literal;
    double dt;
    const double* __restrict__ P;   // plane z = 0 of the PMUT box (p^{n+1} or p^n if literal)
    long long NX, PX;               // F is compact [NY][NX]; P has row pitch PX
    const int* __restrict__ rect;   // [k][4] = i0, j0, ni, nj
    const double* __restrict__ sx;  // [k][m][lmax] S factors along x (unweighted)
    const double* __restrict__ sy;
    const double* __restrict__ wx;  // [k][lmax] face mass factors m_x(i)
    const double* __restrict__ wy;
    const double* __restrict__ omega2;   // [k][m]
    const double* __restrict__ twozw;    // [k][m]  2 zeta omega
    const double* __restrict__ invmass;  // [m]
    const double* __restrict__ eta;      // [m]
    const double* __restrict__ delay;    // [k]
    double amp, om0, ncyc, t_end, t_switch, invC;
    int rx;
    double kappa;
    double* __restrict__ q;
    double* __restrict__ qd;
    double* __restrict__ qdd;
    double* __restrict__ phi;       // phi_k(t^{n+1}, q^{n+1}) for readout
    double* __restrict__ F;         // force plane [NX*NY]
    const long long* step;
    // tabulated coupling (curved boxes: B_{k,m,j} = sum_F w_a w_b |J_s| S_{k,m}(x_j), not separable):
    // PMUT k's face nodes tidx[toff[k] .. toff[k+1]) (pitched indices into P's plane z = 0) with B[j][m];
    // the force f = kappa B^T qdd goes straight into the box's assembled residual res (r -= f)
    const int* __restrict__ toff;
    const long long* __restrict__ tidx;
    const double* __restrict__ tB;
    double* res;
    long long NY_dbg;                   // node rows of the PMUT box (debug-build bounds checks)
};

struct IfaceParams {
    const double* __restrict__ Pf;  // fine box p^{n+1}
    const double* __restrict__ Pc;  // coarse box p^{n+1}
    long long NXf, NYf, NZf, NXc, NYc;
    long long PXf, PXc;             // row pitches of the pitched volume layouts
    int Nf, Nc, R, nelcx, nelcy;
    double gamma, cf2, cc2;
    double dfT[kMaxN + 1];          // (2/h_f) D_f[N_f][c]: d/dz at the fine top face
    double dcB[kMaxN + 1];          // (2/h_c) D_c[0][c]: d/dz at the coarse bottom face
    const double* __restrict__ I;   // [(Nf R + 1)][(Nc + 1)] coarse basis at fine lattice points
    const double* __restrict__ mxf; // [NXf] fine face mass factors
    const double* __restrict__ myf;
    const double* __restrict__ mxc; // [NXc]
    const double* __restrict__ myc;
    double* trc; double* drc;       // coarse trace / normal derivative [NXc*NYc]
    double* tauf; double* sigf;     // fine outputs [NXf*NYf]
    double* h1; double* h2;         // [NYc][NXf] after the y gather
    double* tauc; double* sigc;     // coarse outputs [NXc*NYc]
    int skip_iy0;                   // slab with a lower cut: the shared fine cut line belongs to the lower slab
    const double* __restrict__ dzf; // d_z p+ at the fine face [NXf*NYf] written by the previous volume launch
                                    // (or iface_dz_init), or nullptr: the fused kernel reads the N_f + 1 planes
    // Gauss-Legendre quadrature on the fine faces (quad_rule 1, R9's flag): nq = Nf + 1 points per
    // direction and fine face, none shared; the fine side's terms are projected back onto the fine
    // face nodes (collocated-equivalent tau / sigma, so vol_kernel is unchanged)
    int lg;
    int nelfx, nelfy;               // fine faces along x / y
    long long NXq, NYq;             // LG point lattice: nelf * nq
    const double* __restrict__ Lf;  // [nq][Nf+1] fine GLL basis at the LG points
    const double* __restrict__ ILG; // [R nq][Nc+1] coarse basis at the fine LG points of a coarse element
    double wqx[kMaxN + 1], wqy[kMaxN + 1];   // (h_f/2) w_LG per direction
    double* g1; double* g2;         // [NYq][NXq] weighted coarse-side terms at the LG points
    double* tacc; double* sacc;     // [NYf][NXf] fine-node accumulators (atomics), cleared by the normaliser
    double* q1; double* q2;         // [NYc][NXq] after the y gather
};

// PML auxiliaries of one box (readings R23-R25).  Phi is element-local
// (3 components per element GLL node, PML elements only), psi a pitched nodal field (double
// buffered: psi^{n+1/2} in, psi^{n+3/2} out), da the PML part of the acceleration at region nodes
// (accumulated by pml_element_kernel, applied and cleared by pml_fixup_kernel).
struct PmlParams {
    int N;
    long long NX, NY, NZ, PX;
    int nelx, nely, nelz;
    const int* __restrict__ elems;      // [n_el][3] element coordinates (ex, ey, ez)
    int n_el;
    const double* __restrict__ P;       // p^{n+1}
    const double* __restrict__ W;       // w^n (the predictor velocity pdot^{n+1})
    double* Pn;                         // p^{n+2} (fix-up)
    double* Wn;                         // w^{n+1} (fix-up, same array as W)
    const double* __restrict__ psi_old; // psi^{n+1/2}
    double* psi_new;                    // psi^{n+3/2}
    double* phi;                        // [n_el][3][(N+1)^3] Phi^{n+1/2} in, Phi^{n+3/2} out
    double* da;                         // pitched [nalloc]: PML acceleration, accumulated with atomics
    // per-axis node tables [n_d][4]: z_d, (1 - dt z_d/2)/(1 + dt z_d/2), dt/(1 + dt z_d/2), 1/m_d with
    // m_d the assembled 1D lumped mass (h/2) w_asm (no division in the kernel)
    const double* __restrict__ tx;
    const double* __restrict__ ty;
    const double* __restrict__ tz;
    double D[kMaxN + 1][kMaxN + 1];     // GLL differentiation matrix D[i][j] = l_j'(x_i)
    double w[kMaxN + 1];                // GLL weights
    double s2h[3];                      // 2 / h_d
    double jac;                         // |J| = h_x h_y h_z / 8
    double c2, dt, inv_dt;
    int cutL;                           // y-slab with a lower cut (multi-GPU): its row 0 is the cut plane
    // the PML region (nodes of PML elements) as contiguous lattice-row segments [start, start + len)
    // of the pitched layout, each node once (the fix-up sweeps them coalesced, no atomics)
    const long long* __restrict__ seg_start;
    const int* __restrict__ seg_len;
    long long n_seg;
};

// Curved box: element-by-element K p with the geometric factors recomputed from
// the 8 vertices at every GLL point (no stored metric terms), scatter-add, then a nodal update.
struct CurvedParams {
    int N;
    long long NX, NY, NZ, PX;
    int nelx, nely, nelz;
    int grid;                        // persistent residual-kernel blocks (curved_grid)
    const unsigned char* __restrict__ solid;   // [nel] obstacle elements (skipped), or nullptr
    const double* __restrict__ vlat;
    const double* __restrict__ P;    // p^{n+1}
    double* res;
    double* W;                       // w^n in, w^{n+1} out
    double* Pn;                      // p^{n+2}
    const double* __restrict__ minv;
    const double* __restrict__ cdamp;
    double D[kMaxN + 1][kMaxN + 1];  // D[i][j] = l_j'(x_i)
    double x[kMaxN + 1], w[kMaxN + 1];
    double c2, dt, inv_dt;
    // PMUT forcing on the z = 0 face of an affine element-scatter (obstacle) box: the update subtracts
    // F m_x m_y (F = kappa sum_m qdd S, face weights m_x m_y) from the residual of the face nodes
    const double* __restrict__ F;    // [NY][NX] or nullptr
    const double* __restrict__ fmx;  // [NX] face mass factors
    const double* __restrict__ fmy;  // [NY]
    // incident plane wave on the planar +z face (reading R13): the update subtracts b_j(t^{n+1}) =
    // pwf_j s'(t^{n+1} - pwd_j - t0) from the residual of the top-plane nodes; pwf_j = c A (1 - n.k) W_j
    // (W_j the assembled face weight w_a w_b |J_s|), pwd_j = k.(x_j - x_ref)/c (host tables)
    const double* __restrict__ pwd;  // [NY][NX] or nullptr
    const double* __restrict__ pwf;  // [NY][NX]
    const long long* __restrict__ step;
    double pw_t0, pw_is2, pw_om;
};

// General non-conforming SIPG interface between two element-scatter boxes (curved vertex lattices):
// per fine-face quadrature point (the fine face's GLL nodes, reading R9) the owner coarse element and
// x_hat^- come from Algorithm 3 (sem_face_match) at setup; the kernel adds the face terms of Eq. 7 into
// both boxes' assembled residuals (atomics).
struct GIfaceParams {
    int Nf, Nc;
    long long nqp;                          // quadrature points (fine faces x (Nf+1)^2)
    const double* __restrict__ Pf;          // p^{n+1} of the fine / coarse box (pitched)
    const double* __restrict__ Pc;
    double* resF;                           // assembled residuals (K p), consumed by the curved update
    double* resC;
    long long PXf, NYf, PXc, NYc;           // node (ix, iy, iz) at (iz NY + iy) PX + ix
    const long long* __restrict__ fbase;    // [nqp] pitched index of the fine element's node (0,0,0)
    const long long* __restrict__ cbase;    // [nqp] same for the owner coarse element
    const double* __restrict__ geo;         // [nqp][7]: W_q = w_a w_b |J_s|, J_F^-1 n+, J_C(x_hat^-)^-1 n+
    const double* __restrict__ bas;         // [nqp][6][Nc+1]: l, l' of the coarse basis at x_hat^- per axis
    double Df[kMaxN + 1][kMaxN + 1];        // fine GLL differentiation matrix D[i][j] = l_j'(x_i)
    double gamma, cf2, cc2;
    long long NZf_dbg;                      // fine box node count along z (debug-build bounds checks)
};

// One side of one slab cut for one box (partial rows before, fix-up after the exchange).
struct CutParams {
    int side;                       // 0: cut at iy = 0 (neighbour below in y), 1: at iy = NY-1
    int N;
    long long NX, NY, NZ, PX;
    const double* P;                // p^{n+1} (partial)
    double* Pn;                     // p^{n+2}, w^{n+1} (fix-up)
    double* W;
    double row[kMaxN + 1];          // R0 (side 0) or L (side 1), scaled by c^2 (2/h_y)^2
    double dt;
    // coarse box of an interface: SIPG partials at the cut column (NYt > 0)
    long long NXt, NYt;
    const double* tau;
    const double* sig;
    double ktau[kMaxN + 1], ksig[kMaxN + 1];
    // PML box: its acceleration da at the cut plane travels with the message (the neighbour's PML
    // elements touching the shared nodes), applied by the fix-up like the partial rows
    const double* pda;              // PML da of this box (pitched) or nullptr
    double* out;                    // send buffer: [NX*NZ plane][NXt tau][NXt sigma][NX*NZ PML da]
    const double* in;               // receive buffer, same layout
};

// all cut (side, box) pairs of one slab, handled by one launch per phase
struct CutBatch {
    CutParams c[4];
    int n;
};

struct Box {
    sem_box_desc d{};
    int N = 0;
    long long NX = 0, NY = 0, NZ = 0;
    long long PX = 0;       // device row pitch (doubles): NX rounded up to 8 (TMA needs 16 B strides)
    double h[3] = {0, 0, 0};
    CUtensorMap tmP[2], tmW;
    CUtensorMap tmPw[2];            // p levels with the W tile's box shape (two-level: p^n tile)
    double* P[2] = {nullptr, nullptr};
    double* W = nullptr;
    double* xc = nullptr;
    double* yc = nullptr;
    double* mx = nullptr;  // face mass factors along x [NX] = (h_x/2) w_asm
    double* my = nullptr;
    BoxTables tab{};
    std::vector<double> xh, yh, mxh, myh, mzh;  // host copies (global-lattice values for slab nodes)
    long long gy0 = 0;      // global lattice y index of local iy = 0 (slab decomposition)
    long long NYg = 0;      // global lattice NY of the box
    bool cutL = false, cutR = false;  // -y / +y face of this slab is an internal cut
    int iface_side = 0;
    double* tau = nullptr;  // interface outputs on this box's face lattice
    double* sig = nullptr;
    // curved (trilinear vertex-lattice) box: element-scatter path (curved_residual/update kernels)
    bool curved = false;
    double* vlat = nullptr;   // vertex lattice [(nelx+1)(nely+1)(nelz+1)][3]
    double* minv = nullptr;   // pitched: inverse assembled lumped mass
    double* cdamp = nullptr;  // pitched: C_ii / M_ii on absorbing faces, 0 elsewhere
    double* res = nullptr;    // pitched: assembled K p residual (atomics), cleared by the update
    unsigned char* solid = nullptr;            // [nel] obstacle elements (nullptr: none)
    double* pwd = nullptr;    // plane wave on a curved box: per top-face node delay and factor
    double* pwf = nullptr;
    std::vector<double> vlat_h;                // host copy of the vertex lattice
    bool verts_set = false;                    // sem_box_set_vertices called (else affine lattice)
    std::vector<unsigned char> solid_h;        // host copy of the obstacle mask (empty: none)
    long long ndof() const { return NX * NY * NZ; }
    long long nalloc() const { return PX * NY * NZ; }
};

struct PmlBox {
    bool on = false;
    int box = 0;
    int n_el = 0;
    int* elems = nullptr;
    double* phi = nullptr;
    double* psi[2] = {nullptr, nullptr};
    double* da = nullptr;
    double* tab[3] = {nullptr, nullptr, nullptr};   // per-axis node tables (PmlParams::tx)
    long long* seg_start = nullptr;                  // PML region row segments (PmlParams::seg_start)
    int* seg_len = nullptr;
    long long n_seg = 0;
    std::vector<double> D, w;
};

struct Pmut {
    bool on = false;
    int box = 0, n_pmut = 0, n_modes = 0, lmax = 0;
    int* rect = nullptr;
    double *sx = nullptr, *sy = nullptr, *wx = nullptr, *wy = nullptr;
    double *omega2 = nullptr, *twozw = nullptr, *invmass = nullptr, *eta = nullptr, *delay = nullptr;
    double *q = nullptr, *qd = nullptr, *qdd = nullptr, *phi = nullptr, *F = nullptr;
    double amp = 0, om0 = 0, ncyc = 1, t_end = 0, t_switch = 0, invC = 0, kappa = 0;
    int rx = 0;
    int* toff = nullptr;             // tabulated coupling of a curved box (ModalParams::toff)
    long long* tidx = nullptr;
    double* tB = nullptr;
};

struct Iface {
    bool on = false;
    int fine = 0, coarse = 1;
    IfaceParams prm{};
    bool general = false;          // curved boxes: table-driven kernel on Algorithm 3's matching
    GIfaceParams gprm{};
    std::vector<void*> allocs;
    double* dzf = nullptr;         // d_z p at the fine face, kept by the volume kernel (dzf_active)
};

struct PlaneWave {
    bool on = false;
    int box = 0;
    double amp = 0, f0 = 0, sigma = 0, t0 = 0, k[3] = {0, 0, 0}, xref[3] = {0, 0, 0};
};

}  // namespace sem

namespace sem {
// One y-slab of the decomposition (one rank; all slabs live in one context under emulation).
struct Part {
    int slab = 0;
    std::vector<Box> boxes;
    Pmut pm;
    std::vector<int> pm_global;   // global PMUT index of each local PMUT
    Iface itf;
    PmlBox pml;
    bool cutL = false, cutR = false;
    double* send[2] = {nullptr, nullptr};   // [0] to the left neighbour, [1] to the right
    double* recv[2] = {nullptr, nullptr};
    long long xcount = 0;                   // doubles per neighbour message
    std::vector<long long> xoff;            // offset of box b's block in a message
};
}  // namespace sem

struct sem_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t comm = nullptr;   // NCCL stream (world > 1, not emulated)
    bool own_stream = false;
    int flags = 0;
    int rank = 0, world = 1;
    bool emulate = false;          // all slabs in this context, exchange by device copies
    double dt = 0;
    void* (*dev_alloc)(size_t, void*) = nullptr;   // caller allocator (sem_mesh_desc), or cudaMalloc
    void (*dev_free)(void*, void*) = nullptr;
    void* alloc_user = nullptr;
    std::vector<sem_box_desc> gdesc;               // global boxes as given
    std::vector<long long> gNX, gNY, gNZ;          // global lattice sizes
    std::vector<sem::Part> parts;
    std::vector<long long> cuts;                   // slab plan: box-0 element y index of each slab start [world+1]
    int n_pmut = 0, n_modes = 0;                   // global PMUT array
    std::vector<std::vector<int>> pm_lists;        // global PMUT indices per slab
    bool itf_on = false;
    sem::PlaneWave pw;
    double pw_xref_curved[3] = {0, 0, 0};   // x_ref of a plane wave on a curved box (set by curved_plane_wave)
    int cur = 0;                 // P[cur] = p^{step+1}, P[1-cur] = p^{step}
    long long step = 0;          // host mirror of the device counter
    long long* d_step = nullptr;
    unsigned int* d_sched = nullptr;  // tile scheduler pairs, one per volume launch of a step
    int vol_ty = 0;                   // consumer rows per volume tile (sem::volume_tile_y)
    static constexpr int kSchedPairs = 64;
    unsigned long long* d_flag = nullptr;
    cudaGraphExec_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [parity][1 or 2 steps]
    long long graph_launches[2][2] = {{0, 0}, {0, 0}};
    long long last_launches = 0;
    bool profiling = false;
    bool graph_failed = false;   // stream capture refused (NCCL without capture support): direct launches
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
    double kt_ms[4] = {0, 0, 0, 0};   // kernel groups: 0 volume, 1 interface, 2 modal, 3 PML
    long long kt_n[4] = {0, 0, 0, 0};
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_mfork = nullptr, ev_mjoin = nullptr;   // modal kernel on `aux`, beside the interface
    cudaStream_t aux = nullptr;
    void* nccl = nullptr;        // ncclComm_t
    std::string err;
    std::vector<void*> allocs;
};

namespace sem {
// kernels.cu
void launch_volume(VolLaunch L, cudaStream_t s);
bool volume_pair_supported(int N0, int N1);
void volume_pair_prepare(int N0, int N1, int ty);
void launch_modal(const ModalParams& p, cudaStream_t s);
int launch_iface(const IfaceParams& p, cudaStream_t s);   // returns the number of kernel launches
bool iface_uses_dzf(int Nf, int Nc, int R, int lg);       // the interface path that reads IfaceParams::dzf
void launch_iface_dz_init(const IfaceParams& p, double* dzf, cudaStream_t s);
void iface_prepare(int Nf, int Nc, int R);
void launch_fill_random(double* p, double* w, double* pn, long long NX, long long PX, long long NY, long long NZ,
                        long long gy0, long long NYg, unsigned long long seed, int box, double ps, double vs,
                        double dt, cudaStream_t s);
void launch_cut_partial(const CutBatch& B, cudaStream_t s);
void launch_pml_elements(const PmlParams& p, cudaStream_t s);
void launch_curved(const CurvedParams& p, cudaStream_t s);
void launch_iface_general(const GIfaceParams& p, cudaStream_t s);
int curved_grid(int N, int nel);   // resident blocks of the curved residual kernel on this device
void launch_step_bump(long long* step, cudaStream_t s);
void launch_pml_fixup(const PmlParams& p, cudaStream_t s);
void launch_cut_fixup(const CutBatch& B, cudaStream_t s);
void launch_zero_inactive(double* p0, double* p1, double* w, const double* minv, long long NX, long long PX,
                          long long rows, cudaStream_t s);
void launch_set_state(const double* pprev, double* pcur, const double* w, long long NX, long long PX, long long rows,
                      double dt, cudaStream_t s);
void launch_gather(const double* src, const long long* idx, long long n, double* out, cudaStream_t s);
void launch_nonfinite(const double* p, long long NX, long long PX, long long rows, unsigned long long* flag,
                      cudaStream_t s);
int volume_smem_bytes(int N);
int volume_tile_y(bool slabs);
void volume_prepare(int N, int ty);
}  // namespace sem
