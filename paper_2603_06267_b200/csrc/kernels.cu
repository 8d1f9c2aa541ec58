// sm_100a FP64 kernels of one leapfrog step (Algorithm 1) of the DG-SEM / PMUT model.
//
//  vol_kernel     volume stiffness (Eq. 7 first sum) in 1D-stiffness sum-factorised form on affine
//                 GLL elements, CG assembly in registers / shared memory (owner computes), fused with
//                 the ABC (Eq. 8), the PMUT forcing (Eq. 11), the SIPG layer terms (Eq. 7) and the
//                 kick-drift update.  One CTA owns a (TXE x TY) column of nodes and marches over z:
//                 TMA streams each z-plane of p (with an N-node halo, zero-filled outside the box) and
//                 of w into a D-deep shared-memory ring guarded by mbarriers; the z-stencil lives in a
//                 register window, the x / y stencils read the shared plane.
//  modal_kernel   one warp per PMUT: pressure projection (Eq. 12), modal predictor / solve / corrector
//                 (Eq. 10), force plane f = kappa B^T qdd (Eq. 11).
//  iface_*        SIPG flux of Eq. 7 on the 2:1 non-conforming face, quadrature at the fine-face GLL
//                 lattice (reading R9).
// DESIGN.md derives every coefficient and gives the byte budget of each kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gll_constexpr.h"
#include "sem_internal.h"

// Volume-kernel tiling (tuned on B200, see profiles/): consumer rows per CTA and minimum CTAs per SM.

#ifndef SEM_MINB
#define SEM_MINB 1
#endif
#ifndef SEM_XSPLIT
#define SEM_XSPLIT 0
#endif
#ifndef SEM_PSLEEP
#define SEM_PSLEEP 64   // producer back-off (ns) while the slot it refills is still in use
#endif
#ifndef SEM_BATCH_WAIT
#define SEM_BATCH_WAIT 1   // window slide: the N full-barrier tests issued back to back
#endif
#ifndef SEM_BW_TEST
#define SEM_BW_TEST mbar_test_wait
#endif
// SEM_WG 1: warp-specialised warpgroups -- TY (a multiple of 4) consumer warps in TY/4 warpgroups that
// grow their register budget with setmaxnreg, and one producer warpgroup (one active warp) that shrinks
// its own to 24, so that 16 row warps get 112 registers (the register file is split per SM sub-partition:
// 17 warps of one kernel-wide budget would allow only 96)
#ifndef SEM_WG
#define SEM_WG 1
#endif
#ifndef SEM_KTY
#define SEM_KTY (SEM_WG ? 16 : 11)   // consumer rows per CTA: 16 in four warpgroups, or 11 + a producer warp
#endif
#ifndef SEM_KTY_SLAB
#define SEM_KTY_SLAB (SEM_WG ? 12 : 11)   // rows per CTA in y-slab contexts (fewer tiles per slab: smaller tail)
#endif
// setmaxnreg budgets per thread: 16 row warps (65536 - 128 * 24) / 512 -> 112 and 24; 12 row warps 160 and 32
template <int TY>
constexpr int wg_cons_regs() { return TY >= 16 ? 112 : 160; }
template <int TY>
constexpr int wg_prod_regs() { return TY >= 16 ? 24 : 32; }
#define SEM_VOL_WARPS(TY) ((TY) + (SEM_WG ? 4 : 1))
#define SEM_VOL_BOUNDS(TY) __launch_bounds__(32 * SEM_VOL_WARPS(TY), SEM_MINB)

namespace sem {

// ------------------------------------------------------------------------------------------------
// mbarrier / TMA helpers (inline PTX)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// non-blocking test of a phase (no suspension: several tests can be in flight back to back)
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
// ------------------------------------------------------------------------------------------------
// Volume + update kernel (persistent, one launch for both boxes of a step)
// ------------------------------------------------------------------------------------------------
template <int N, int TY>
struct VolGeo {
    static constexpr int TXE = vol_txe(N);
    static constexpr int NH = vol_nh(N);         // x halo width in the shared plane (even)
    static constexpr int SW = vol_pbox_w(N);     // shared P plane pitch (doubles)
    static constexpr int WW = vol_wbox_w(N);     // shared W plane pitch
    static constexpr int SH = TY + 2 * N;
    static constexpr int PBYTES = SW * SH * 8;
    static constexpr int POFF = vol_pbytes_aligned(N, TY);   // W tile offset inside a slot
    static constexpr int WBYTES = WW * TY * 8;
};

// Ring geometry of a launch: depth and slot stride are those of the most demanding box, so that the
// plane stream of a persistent CTA runs on without a break across tiles and across the two boxes.
template <int D_, int SLOT_>
struct Ring {
    static constexpr int D = D_;
    static constexpr int SLOT = SLOT_;
};

template <int N, int TY, class RG>
__device__ __forceinline__ void vol_issue(const VolParams& p, unsigned char* ring, uint32_t bars, int slot, int z,
                                          int tx0, int ty0) {
    using G = VolGeo<N, TY>;
    unsigned char* s = ring + slot * RG::SLOT;
    const uint32_t bar = bars + 8u * slot;
    mbar_expect_tx(bar, G::PBYTES + G::WBYTES);
    tma_load_3d(smem_u32(s), &p.tmP, tx0 - G::NH, ty0 - N, z, bar);
    tma_load_3d(smem_u32(s + G::POFF), &p.tmW, tx0, ty0, z, bar);
}

// Output stores of the volume kernel: default write-back policy (measured faster than streaming .cs)
__device__ __forceinline__ void st_out(double* p, double v) { *p = v; }

// Per-thread state of the volume kernel (one tile).
template <int N>
struct VolThread {
    double cR[N + 1];     // x row of this lane's node (right element, or B0), scaled; zeros if none
    double cyR[N + 1];    // y row of this warp's node row (right element or B0), scaled; zeros if none
    double fL;            // s_x * factor on the left-element x row received from lane-1 (0, 1, or 2 at BN)
    double yLs;           // s_y * factor on the left-element y row (0, 1, or 2 at BN), warp-uniform
    double dxy;           // lateral ABC C_ii / M_ii
    int fc;               // face-lattice index iy NX + ix (edge-layer inputs are loaded on demand)
    int xb;               // smem column of the right element's first node (lane 31: left element of lane 0)
    int own;              // smem offset of the own node in the P plane
    int wown;             // smem offset in the W plane
    int yb;               // smem offset of the right element's first row (x col of the own node)
    int yl;               // smem offset of the left element's first row
    bool valid;
};

// Ring position of a plane: slot = g mod D and the parity of its fill, advanced incrementally
// (g counts the planes a CTA has streamed since the launch began).
struct RingPos {
    int slot;
    uint32_t par;
    template <int D>
    __device__ __forceinline__ static RingPos at(unsigned g) {
        return RingPos{(int)(g % D), (uint32_t)((g / D) & 1u)};
    }
    template <int D>
    __device__ __forceinline__ void advance() {
        if (++slot == D) {
            slot = 0;
            par ^= 1u;
        }
    }
};

// compile-time reference rows, materialised as device constants (folded for constant indices)
template <int N>
__device__ constexpr gllc::Tables<N> kRef = gllc::make_tables<N>();

// Layer kinds (compile time): bit 0 = first element layer (z = 0 face), bit 1 = last (z = N nel_z face).
constexpr int kFirst = 1, kLast = 2;

// One plane: a = -(M^-1 K p)_i - C_ii/M_ii w_i + extras;  w <- w + dt a;  p <- p + dt w.
// Returns the new (w, p) of this thread's node; the caller stores them.
template <int N, int TY, int C, int F>
__device__ __forceinline__ void vol_plane(const VolParams& p, const VolThread<N>& t, const double* __restrict__ sP,
                                          const double* __restrict__ sW, const double (&zw)[N + 2], int ez,
                                          double& wn_out, double& pn_out) {
    using G = VolGeo<N, TY>;
    const BoxTables& T = p.tab;
#ifdef SEM_MEMONLY   // diagnostic build: same data movement, no stencil arithmetic
    {
        const double wv = sW[t.wown];
        wn_out = wv;
        pn_out = fma(p.dt, wv, zw[C]);
        return;
    }
#endif
    // ---- x: right-element row with per-lane (scaled) coefficients; the left-element row of a shared
    //      node (the compile-time reference row L) is evaluated by lane-1, then shuffled
    const auto& RT = kRef<N>;
    double v[N + 1];
#pragma unroll
    for (int b = 0; b <= N; ++b) v[b] = sP[t.xb + b];
    double xr = 0.0, xl = 0.0;
#if SEM_XSPLIT   // two accumulation chains per x row (shorter fma dependency chains)
    {
        double xr1 = 0.0, xl1 = 0.0;
#pragma unroll
        for (int b = 0; b <= N; b += 2) {
            xr = fma(t.cR[b], v[b], xr);
            xl = fma(RT.L[b], v[b], xl);
        }
#pragma unroll
        for (int b = 1; b <= N; b += 2) {
            xr1 = fma(t.cR[b], v[b], xr1);
            xl1 = fma(RT.L[b], v[b], xl1);
        }
        xr += xr1;
        xl += xl1;
    }
#else
#pragma unroll
    for (int b = 0; b <= N; ++b) {
        xr = fma(t.cR[b], v[b], xr);
        xl = fma(RT.L[b], v[b], xl);
    }
#endif
    const double xlr = __shfl_sync(0xffffffffu, xl, (threadIdx.x + 31) & 31);
    // ---- y: per-warp row (registers, scaled); left row of a shared node: row L
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int b = 0; b <= N; b += 2) y0 = fma(t.cyR[b], sP[t.yb + b * G::SW], y0);
#pragma unroll
    for (int b = 1; b <= N; b += 2) y1 = fma(t.cyR[b], sP[t.yb + b * G::SW], y1);
    double acc = fma(t.fL, xlr, xr) + (y0 + y1);
    if (t.yLs != 0.0) {
        double yl = 0.0;
#pragma unroll
        for (int b = 0; b <= N; ++b) yl = fma(RT.L[b], sP[t.yl + b * G::SW], yl);
        acc = fma(t.yLs, yl, acc);
    }
    // ---- z: register window zw[b] = p(z0 + b), b = 0..N (this element's planes); zw[N + 1] = the
    //      previous element's L row applied to its planes (the left part of the shared plane z0),
    //      accumulated when that element's window slid out (vol_layer); rows by compile-time plane class
    double z0 = 0.0, z1 = 0.0;
    if constexpr (C == N) {   // top boundary plane: left element only, BN = 2 L
#pragma unroll
        for (int b = 0; b <= N; b += 2) z0 = fma(2.0 * RT.L[b], zw[b], z0);
#pragma unroll
        for (int b = 1; b <= N; b += 2) z1 = fma(2.0 * RT.L[b], zw[b], z1);
    } else if constexpr (C == 0 && (F & kFirst)) {   // bottom boundary plane: B0 = 2 R0
#pragma unroll
        for (int b = 0; b <= N; b += 2) z0 = fma(2.0 * RT.R[0][b], zw[b], z0);
#pragma unroll
        for (int b = 1; b <= N; b += 2) z1 = fma(2.0 * RT.R[0][b], zw[b], z1);
    } else if constexpr (C == 0) {
#pragma unroll
        for (int b = 0; b <= N; ++b) z0 = fma(RT.R[0][b], zw[b], z0);
        z1 = zw[N + 1];
    } else {
#pragma unroll
        for (int b = 0; b <= N; b += 2) z0 = fma(RT.R[C][b], zw[b], z0);
#pragma unroll
        for (int b = 1; b <= N; b += 2) z1 = fma(RT.R[C][b], zw[b], z1);
    }
    acc = fma(p.sdir[2], z0 + z1, acc);
    double a = -acc;
    const double pv = zw[C];
#if SEM_TWO_LEVEL   // w^n = (p^{n+1} - p^n) / dt from the p^n tile
    const double wv = (pv - sW[t.wown]) * p.inv_dt;
#else
    const double wv = sW[t.wown];
#endif
    double damp = t.dxy;
    if constexpr ((F & kFirst) && C == 0) {      // z = 0 face: ABC and PMUT forcing (Eq. 11)
        damp += p.damp[4];
        if (p.F && t.valid) a = fma(p.kF, __ldg(p.F + t.fc), a);
    }
    if constexpr ((F & kLast) && C == N) {       // z = top face: ABC and incident plane wave (R13)
        damp += p.damp[5];
        if (p.pw_on && t.valid) {
            const int ixp = t.fc % (int)p.NX, iyp = t.fc / (int)p.NX;
            const double t1 = (double)(__ldcg(p.step) + 1) * p.dt;
            const double tau = t1 - (p.pw_k[0] * (__ldg(p.xc + ixp) - p.pw_xref[0]) +
                                     p.pw_k[1] * (__ldg(p.yc + iyp) - p.pw_xref[1]) +
                                     p.pw_k[2] * (p.pw_ztop - p.pw_xref[2])) / p.pw_c;
            const double u = tau - p.pw_t0;
            const double is2 = 1.0 / (p.pw_sigma * p.pw_sigma);
            double sn, cs;
            sincos(p.pw_om * u, &sn, &cs);
            a += p.pw_fac * (exp(-0.5 * u * u * is2) * (-u * is2 * sn + p.pw_om * cs));
        }
    }
    // SIPG layer terms (Eq. 7): fine side on the last element layer, coarse side on the first
    if constexpr (F & kLast) {
        if (p.iface_side > 0 && t.valid) {
            a -= __ldg(p.sig + t.fc) * T.ksig[C];
            if constexpr (C == N) a -= __ldg(p.tau + t.fc) * T.ktau[N];
        }
    }
    if constexpr (F & kFirst) {
        if (p.iface_side < 0 && t.valid) {
            a -= __ldg(p.sig + t.fc) * T.ksig[C];
            if constexpr (C == 0) a -= __ldg(p.tau + t.fc) * T.ktau[0];
        }
    } else if constexpr (C == 0) {
        if (p.iface_side < 0 && ez == 1 && t.valid)
            a -= __ldg(p.sig + t.fc) * T.ksig[N];   // shared plane z = N of the first layer
    }
    a = fma(-damp, wv, a);
    wn_out = fma(p.dt, a, wv);
    pn_out = fma(p.dt, wn_out, pv);
}

// One element layer: planes z0 .. z0+N-1 (plus the top plane N nel_z on the last layer), unrolled by
// compile-time recursion over the local plane index C so that every z row and window index is a
// constant.  cur tracks the ring position of plane iz.  With SEM_PAIR, two planes are evaluated
// together (independent dependency chains interleave: twice the ILP per consumer warp) before their
// stores and slot releases.
#ifndef SEM_PAIR
#define SEM_PAIR (SEM_WG ? 0 : 1)   // with 12 row warps (warpgroups) the single-plane order is faster
#endif
template <int N, int TY, class RG, int F, int C>
__device__ __forceinline__ void vol_layer_step(const VolParams& p, const VolThread<N>& t, unsigned char* ring,
                                               uint32_t bars, int ez, const double (&zw)[N + 2],
                                               double*& outP, double*& outW, RingPos& cur, double& dz) {
    constexpr int NP = (F & kLast) ? N + 1 : N;   // planes of this layer
    if constexpr (C < NP) {
        using G = VolGeo<N, TY>;
        const long long PS = p.PX * p.NY;
        if constexpr (SEM_PAIR && C + 1 < NP) {
            RingPos nxt = cur;
            nxt.template advance<RG::D>();
            const unsigned char* s0 = ring + cur.slot * RG::SLOT;
            const unsigned char* s1 = ring + nxt.slot * RG::SLOT;
            double w0, p0, w1, p1;
            vol_plane<N, TY, C, F>(p, t, reinterpret_cast<const double*>(s0),
                                   reinterpret_cast<const double*>(s0 + G::POFF), zw, ez, w0, p0);
            vol_plane<N, TY, C + 1, F>(p, t, reinterpret_cast<const double*>(s1),
                                       reinterpret_cast<const double*>(s1 + G::POFF), zw, ez, w1, p1);
            if (t.valid) {
                if (!SEM_TWO_LEVEL) st_out(outW, w0);
                st_out(outP, p0);
                if (!SEM_TWO_LEVEL) st_out(outW + PS, w1);
                st_out(outP + PS, p1);
            }
            if constexpr (F & kLast) {   // d_z p^{n+2} at the top face for the next step's interface
                if (p.dzf) {
                    dz = fma(p.dzc[C], p0, dz);
                    dz = fma(p.dzc[C + 1], p1, dz);
                    if constexpr (C + 1 == N)
                        if (t.valid) p.dzf[t.fc] = dz;
                }
            }
            outP += 2 * PS;
            outW += 2 * PS;
            __syncwarp();
            if (threadIdx.x == 0) {
                mbar_arrive(bars + 8u * (RG::D + cur.slot));
                mbar_arrive(bars + 8u * (RG::D + nxt.slot));
            }
            nxt.template advance<RG::D>();
            cur = nxt;
            vol_layer_step<N, TY, RG, F, C + 2>(p, t, ring, bars, ez, zw, outP, outW, cur, dz);
        } else {
            const unsigned char* s0 = ring + cur.slot * RG::SLOT;
            double w0, p0;
            vol_plane<N, TY, C, F>(p, t, reinterpret_cast<const double*>(s0),
                                   reinterpret_cast<const double*>(s0 + G::POFF), zw, ez, w0, p0);
            if (t.valid) {
                if (!SEM_TWO_LEVEL) st_out(outW, w0);
                st_out(outP, p0);
            }
            if constexpr (F & kLast) {
                if (p.dzf) {
                    dz = fma(p.dzc[C], p0, dz);
                    if constexpr (C == N)
                        if (t.valid) p.dzf[t.fc] = dz;
                }
            }
            outP += PS;
            outW += PS;
            // release the slot: one arrival per consumer warp on its "empty" barrier (no block-wide
            // barrier: warps drift across planes and hide each other's latency; the producer warp refills)
            __syncwarp();
            if (threadIdx.x == 0) mbar_arrive(bars + 8u * (RG::D + cur.slot));
            cur.template advance<RG::D>();
            vol_layer_step<N, TY, RG, F, C + 1>(p, t, ring, bars, ez, zw, outP, outW, cur, dz);
        }
    }
}

// Layer, then slide the window to the next element: zw[N + 1] <- L row of this element (the left part of
// the next shared plane), zw[0] <- plane z0 + N, zw[1..N] <- planes z0 + N + 1 .. z0 + 2N (read from the
// ring; plane z0+N+1+j is resident because slots are only refilled after their own plane has been
// processed).  N + 2 window registers instead of 2N + 1.
template <int N, int TY, class RG, int F>
__device__ __forceinline__ void vol_layer(const VolParams& p, const VolThread<N>& t, unsigned char* ring,
                                          uint32_t bars, int ez, double (&zw)[N + 2],
                                          double*& outP, double*& outW, RingPos& cur, RingPos& nx) {
    double dz = 0.0;   // top layer: d_z p^{n+2} at the top face (same fma order as the interface's)
    vol_layer_step<N, TY, RG, F, 0>(p, t, ring, bars, ez, zw, outP, outW, cur, dz);
    if constexpr (!(F & kLast)) {
        const auto& RT = kRef<N>;
        double zl = 0.0;
#pragma unroll
        for (int b = 0; b <= N; ++b) zl = fma(RT.L[b], zw[b], zl);
        zw[N + 1] = zl;
        zw[0] = zw[N];
        // planes z0 + N + 1 .. z0 + 2N exist (this is not the last layer: N ez + 2N <= NZ - 1).  The N
        // full-barrier tests are issued back to back so that their latencies overlap (a try_wait on a
        // completed phase still takes ~90 cycles), then the laggards are waited for, then the loads.
#if SEM_BATCH_WAIT
        RingPos q = nx;
        uint32_t ok = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            ok |= (uint32_t)SEM_BW_TEST(bars + 8u * q.slot, q.par) << j;
            q.template advance<RG::D>();
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (!((ok >> j) & 1u)) mbar_wait(bars + 8u * nx.slot, nx.par);
            zw[1 + j] = reinterpret_cast<const double*>(ring + nx.slot * RG::SLOT)[t.own];
            nx.template advance<RG::D>();
        }
#else
#pragma unroll
        for (int j = 0; j < N; ++j) {
            mbar_wait(bars + 8u * nx.slot, nx.par);
            zw[1 + j] = reinterpret_cast<const double*>(ring + nx.slot * RG::SLOT)[t.own];
            nx.template advance<RG::D>();
        }
#endif
    }
}

// Consumer side of one tile (TXE x TY node column, all z): planes g0 .. g0 + NZ - 1 of the ring.
template <int N, int TY, class RG>
__device__ __forceinline__ void vol_tile(const VolParams& p, unsigned char* ring, uint32_t bars, int tx0, int ty0,
                                         unsigned g0) {
    using G = VolGeo<N, TY>;
    const int lane = threadIdx.x, ly = threadIdx.y;
    const long long NX = p.NX, NY = p.NY;
    const int NZ = (int)p.NZ;
    const BoxTables& T = p.tab;
    VolThread<N> t;
    const long long ix = tx0 + lane, iy = ty0 + ly;
    // node lanes: TXE per tile; the last tile in x takes one more node when that ends the box
    const int txe_t = (NX - tx0 <= G::TXE + 1) ? (int)(NX - tx0) : G::TXE;
    const bool node_lane = lane < txe_t;
    t.valid = node_lane && ix < NX && iy < NY;
    const int a = lane % N;
    int rxR = -1;
    t.fL = 0.0;
    if (t.valid) {   // box faces: B0 = 2 R0 / BN = 2 L
        if (ix == 0) rxR = row_B0(N);
        else if (ix < NX - 1) rxR = a;
        if (a == 0 && ix > 0) t.fL = (ix == NX - 1) ? 2.0 : 1.0;
    }
    // the extra last node (lane TXE, a = 0, no right element: its x row is zero) reads its left element
    // so that every shared-memory read stays inside the row
    t.xb = (ly + N) * G::SW + (!node_lane ? G::NH - N : (lane == G::TXE ? lane - N + G::NH : lane - a + G::NH));
    const int ay = (int)(iy % N);
    int ryR = -1;
    t.yLs = 0.0;
    if (iy < NY) {
        // box faces: B0 = 2 R0 / BN = 2 L; slab cuts (multi-GPU, y-slabs): the shared node keeps its
        // interior rows R0 (upper side) / L (lower side) and the other side's part is added by
        // cut_fixup_kernel after the exchange
        if (iy == 0) ryR = p.cutL ? 0 : row_B0(N);
        else if (iy < NY - 1) ryR = ay;
        if (ay == 0 && iy > 0) t.yLs = (iy == NY - 1 && !p.cutR) ? 2.0 * p.sdir[1] : p.sdir[1];
    }
    t.fL *= p.sdir[0];
#pragma unroll
    for (int b = 0; b <= N; ++b) {
        t.cR[b] = rxR >= 0 ? T.G[0][rxR][b] : 0.0;
        t.cyR[b] = ryR >= 0 ? T.G[1][ryR][b] : 0.0;
    }
    const int col = node_lane ? lane + G::NH : 0;
    t.own = (ly + N) * G::SW + col;
    t.wown = ly * G::WW + (node_lane ? lane : 0);
    t.yb = (ly + N - ay) * G::SW + col;
    t.yl = ly * G::SW + col;
    t.dxy = 0.0;
    t.fc = t.valid ? (int)(iy * NX + ix) : 0;
    if (t.valid) {
        if (ix == 0) t.dxy += p.damp[0];
        if (ix == NX - 1) t.dxy += p.damp[1];
        if (iy == 0) t.dxy += p.damp[2];
        if (iy == NY - 1) t.dxy += p.damp[3];
    }
    const long long off = t.valid ? iy * p.PX + ix : 0;
    double* outP = p.Pn + off;
    double* outW = p.W + off;

    // ---- register window zw[b] = p(b), b = 0..N: planes 0..N from the ring (zw[N + 1] is not read on
    //      the first layer: its bottom plane is a box face)
    double zw[N + 2];
    zw[N + 1] = 0.0;
    RingPos w = RingPos::at<RG::D>(g0);
#pragma unroll
    for (int k = 0; k <= N; ++k) {
        zw[k] = 0.0;
        if (k < NZ) {
            mbar_wait(bars + 8u * w.slot, w.par);
            zw[k] = reinterpret_cast<const double*>(ring + w.slot * RG::SLOT)[t.own];
        }
        w.template advance<RG::D>();
    }

    const int nelz = p.nelz;
    RingPos cur = RingPos::at<RG::D>(g0), nx = RingPos::at<RG::D>(g0 + N + 1);
    if (nelz == 1) {
        vol_layer<N, TY, RG, kFirst | kLast>(p, t, ring, bars, 0, zw, outP, outW, cur, nx);
    } else {
        vol_layer<N, TY, RG, kFirst>(p, t, ring, bars, 0, zw, outP, outW, cur, nx);
        for (int ez = 1; ez < nelz - 1; ++ez)
            vol_layer<N, TY, RG, 0>(p, t, ring, bars, ez, zw, outP, outW, cur, nx);
        vol_layer<N, TY, RG, kLast>(p, t, ring, bars, nelz - 1, zw, outP, outW, cur, nx);
    }
}

// Tile order inside a box: row-major (tx fastest).  Tiles are handed out in this order, so a tile's x
// neighbours (which re-read its halo columns of p) run at the same time, and the concurrently streamed
// region spans long contiguous x rows (DRAM page locality).  (Strip and band orders that keep the y
// neighbours closer were measured slower: profiles/README.md.)
__device__ __forceinline__ void tile_xy(unsigned lt, unsigned ntx, unsigned /*nty*/, int& tx, int& ty) {
    tx = (int)(lt % ntx);
    ty = (int)(lt / ntx);
}

// Launch-wide ring of a (N0, N1) pair (N1 = 0: one box).
template <int N0, int N1, int TY>
struct PairRing {
    static constexpr int SLOT = cmax(vol_slot_bytes(N0, TY), N1 ? vol_slot_bytes(N1, TY) : 0);
    static constexpr int D = cmax(vol_depth_for_slot(N0, SLOT), N1 ? vol_depth_for_slot(N1, SLOT) : 0);
    static_assert(D >= cmax(N0, N1) + 2, "ring too shallow for the z window (it holds N + 1 planes)");
    using RG = Ring<D, SLOT>;
};

// Persistent CTAs (one per SM): TY consumer warps (one tile row each) + 1 producer warp
// (threadIdx.y == TY).  The producer takes tiles from a launch-wide counter (the boxes' tiles in one
// list, the larger tiles of box 1 first) and streams every plane of each with TMA into the ring as soon
// as all consumer warps released a slot; the tile index travels with the first plane of its tile (a
// per-slot header, published by the mbarrier arrive).  The stream never stops at a tile boundary, so
// the next tile's first planes are already in flight while the consumers finish the current one.
template <int N0, int N1, int TY>
__global__ void SEM_VOL_BOUNDS(TY) vol_kernel(const __grid_constant__ VolLaunch L) {
    using RG = typename PairRing<N0, N1, TY>::RG;
    constexpr int D = RG::D;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* ring = smem_raw;   // direct indexing keeps the shared address space (LDS, not generic LD)
    const uint32_t bars = smem_u32(ring + D * RG::SLOT);
    volatile int* tileq = reinterpret_cast<volatile int*>(ring + D * RG::SLOT + 2 * D * 8);
    const int lane = threadIdx.x, ly = threadIdx.y;
    const unsigned n1 = N1 ? L.ntiles[1] : 0u;
    const unsigned ntot = n1 + L.ntiles[0];

    if (lane == 0 && ly == 0) {
        for (int s = 0; s < D; ++s) {
            mbar_init(bars + 8u * s, 1);               // full: TMA transaction bytes (or the end marker)
            mbar_init(bars + 8u * (D + s), TY);        // empty: one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
#if SEM_WG
    static_assert(TY % 4 == 0, "warpgroup mode needs whole consumer warpgroups");
    if (ly >= TY) {   // producer warpgroup: give registers back; its first warp streams the planes
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(wg_prod_regs<TY>()));
        if (ly > TY) return;
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(wg_cons_regs<TY>()));
    }
#endif
    if (ly == TY) {   // producer warp
        if (lane == 0) {
            unsigned g = 0;
            for (;;) {
                const unsigned tile = atomicAdd(L.sched, 1u);
                const int box = (N1 > 0 && tile < n1) ? 1 : (tile < ntot ? 0 : -1);
                if (box < 0) {   // end marker: a header of -1 on the next slot, completed without data
                    const int slot = (int)(g % D);
                    if (g >= (unsigned)D)
                        while (!mbar_try_wait(bars + 8u * (D + slot), ((g / D) - 1u) & 1u)) __nanosleep(SEM_PSLEEP);
                    tileq[slot] = -1;
                    mbar_arrive(bars + 8u * slot);
                    break;
                }
                const unsigned lt = box ? tile : tile - n1;
                const VolParams& p = L.box[box];
                const int NZ = (int)p.NZ;
                int tx, ty;
                tile_xy(lt, L.ntx[box], L.nty[box], tx, ty);
                const int tx0 = tx * (box ? vol_txe(N1 ? N1 : 1) : vol_txe(N0));
                const int ty0 = ty * TY;
                for (int z = 0; z < NZ; ++z, ++g) {   // plane g reuses the slot of plane g - D
                    const int slot = (int)(g % D);
                    if (g >= (unsigned)D)
                        while (!mbar_try_wait(bars + 8u * (D + slot), ((g / D) - 1u) & 1u)) __nanosleep(SEM_PSLEEP);
                    if (z == 0) tileq[slot] = (int)tile;
                    if constexpr (N1 > 0) {
                        if (box) vol_issue<N1, TY, RG>(L.box[1], ring, bars, slot, z, tx0, ty0);
                        else vol_issue<N0, TY, RG>(L.box[0], ring, bars, slot, z, tx0, ty0);
                    } else {
                        vol_issue<N0, TY, RG>(L.box[0], ring, bars, slot, z, tx0, ty0);
                    }
                }
            }
        }
        return;
    }

    // consumers: follow the tiles in the order the producer streams them
    unsigned g = 0;
    for (;;) {
        const RingPos h = RingPos::at<D>(g);
        mbar_wait(bars + 8u * h.slot, h.par);
        const int tile = tileq[h.slot];
        if (tile < 0) break;
        if (N1 > 0 && (unsigned)tile < n1) {
            if constexpr (N1 > 0) {
                const VolParams& p = L.box[1];
                const unsigned lt = (unsigned)tile;
                int tx, ty;
                tile_xy(lt, L.ntx[1], L.nty[1], tx, ty);
                vol_tile<N1, TY, RG>(p, ring, bars, tx * vol_txe(N1), ty * TY, g);
                g += (unsigned)p.NZ;
            }
        } else {
            const VolParams& p = L.box[0];
            const unsigned lt = (unsigned)tile - n1;
            int tx, ty;
            tile_xy(lt, L.ntx[0], L.nty[0], tx, ty);
            vol_tile<N0, TY, RG>(p, ring, bars, tx * vol_txe(N0), ty * TY, g);
            g += (unsigned)p.NZ;
        }
    }

    // end of the launch: the last CTA resets the tile scheduler and (last launch of the step) bumps the
    // device step counter.  The named barrier keeps every consumer warp of this CTA (which may still
    // read the step counter in its last plane) ahead of the bump.
    asm volatile("bar.sync 1, %0;" ::"r"(32 * TY) : "memory");
    if (lane == 0 && ly == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(L.sched + 1, 1u);
        if (prev == gridDim.x - 1) {
            L.sched[0] = 0u;
            L.sched[1] = 0u;
            if (L.bump_step) *L.step += 1;
            __threadfence();
        }
    }
}

constexpr int kTY = SEM_KTY;        // consumer rows per CTA, one GPU
constexpr int kTYs = SEM_KTY_SLAB;  // consumer rows per CTA, y-slab contexts

template <int N0, int N1, int TY>
struct VolInst {
    static int smem() {
        using R = PairRing<N0, N1, TY>;
        return R::D * R::SLOT + 2 * R::D * 8 + R::D * 4 + 128;
    }
    static int ctas_per_sm() {   // resident CTAs per SM (occupancy), cached
        static int occ = -1;
        if (occ < 0) {
            cudaFuncSetAttribute(vol_kernel<N0, N1, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem());
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vol_kernel<N0, N1, TY>, 32 * SEM_VOL_WARPS(TY),
                                                              smem()) != cudaSuccess || occ < 1)
                occ = 1;
        }
        return occ;
    }
    static void launch(const VolLaunch& L, cudaStream_t s) {
        static int nsm = 0;
        if (!nsm) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        }
        const unsigned ntot = L.ntiles[0] + (N1 ? L.ntiles[1] : 0u);
        // SMs left free for a concurrent NCCL exchange (its kernel could not co-reside with a volume CTA)
        const int nsm_use = nsm - L.reserve_sms > 1 ? nsm - L.reserve_sms : 1;
        unsigned grid = (unsigned)(nsm_use * ctas_per_sm());
        if (grid > ntot) grid = ntot;
        vol_kernel<N0, N1, TY><<<grid, dim3(32, SEM_VOL_WARPS(TY)), smem(), s>>>(L);
    }
};

template <int TY>
static void volume_prepare_t(int N) {
    switch (N) {
        case 1: VolInst<1, 0, TY>::ctas_per_sm(); break;
        case 2: VolInst<2, 0, TY>::ctas_per_sm(); break;
        case 3: VolInst<3, 0, TY>::ctas_per_sm(); break;
        case 4: VolInst<4, 0, TY>::ctas_per_sm(); break;
        case 5: VolInst<5, 0, TY>::ctas_per_sm(); break;
        case 6: VolInst<6, 0, TY>::ctas_per_sm(); break;
        case 7: VolInst<7, 0, TY>::ctas_per_sm(); break;
        case 8: VolInst<8, 0, TY>::ctas_per_sm(); break;
        default: break;
    }
}
void volume_prepare(int N, int ty) {
    if (ty == kTYs) volume_prepare_t<kTYs>(N);
    else volume_prepare_t<kTY>(N);
}

bool volume_pair_supported(int N0, int N1) { return N0 == 5 && N1 == 3; }

void volume_pair_prepare(int N0, int N1, int ty) {
    if (N0 == 5 && N1 == 3) {
        if (ty == kTYs) VolInst<5, 3, kTYs>::ctas_per_sm();
        else VolInst<5, 3, kTY>::ctas_per_sm();
    }
}

void fill_tiles(VolLaunch& L) {
    for (int b = 0; b < L.nbox; ++b) {
        const VolParams& p = L.box[b];
        const int txe = vol_txe(p.N);
        L.ntx[b] = (unsigned)((p.NX - 1 + txe - 1) / txe);   // the last tile may take TXE + 1 nodes
        L.nty[b] = (unsigned)((p.NY + L.ty - 1) / L.ty);
        L.ntiles[b] = L.ntx[b] * L.nty[b];
    }
}

template <int TY>
static void launch_volume_t(const VolLaunch& L, cudaStream_t s) {
    if (L.nbox == 2) {
        if (L.box[0].N == 5 && L.box[1].N == 3) VolInst<5, 3, TY>::launch(L, s);
        return;
    }
    switch (L.box[0].N) {
        case 1: VolInst<1, 0, TY>::launch(L, s); break;
        case 2: VolInst<2, 0, TY>::launch(L, s); break;
        case 3: VolInst<3, 0, TY>::launch(L, s); break;
        case 4: VolInst<4, 0, TY>::launch(L, s); break;
        case 5: VolInst<5, 0, TY>::launch(L, s); break;
        case 6: VolInst<6, 0, TY>::launch(L, s); break;
        case 7: VolInst<7, 0, TY>::launch(L, s); break;
        case 8: VolInst<8, 0, TY>::launch(L, s); break;
        default: break;
    }
}

void launch_volume(VolLaunch L, cudaStream_t s) {
    if (L.ty != kTYs) L.ty = kTY;
    fill_tiles(L);
    if (L.ty == kTYs) launch_volume_t<kTYs>(L, s);
    else launch_volume_t<kTY>(L, s);
}

int volume_smem_bytes(int N) {
    switch (N) {
        case 1: return VolInst<1, 0, kTY>::smem();
        case 2: return VolInst<2, 0, kTY>::smem();
        case 3: return VolInst<3, 0, kTY>::smem();
        case 4: return VolInst<4, 0, kTY>::smem();
        case 5: return VolInst<5, 0, kTY>::smem();
        case 6: return VolInst<6, 0, kTY>::smem();
        case 7: return VolInst<7, 0, kTY>::smem();
        case 8: return VolInst<8, 0, kTY>::smem();
        default: return 0;
    }
}
// consumer rows per volume tile: one GPU, or y-slab contexts (more, smaller launches: a smaller tail)
int volume_tile_y(bool slabs) { return slabs ? kTYs : kTY; }

// ------------------------------------------------------------------------------------------------
// Modal kernel: one warp per PMUT
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double drive_tx(const ModalParams& p, double tp) {
    if (tp < 0.0 || tp > p.t_end) return 0.0;
    return p.amp * sin(p.om0 * tp) * 0.5 * (1.0 - cos(p.om0 * tp / p.ncyc));
}

// One block of kModalWarps warps per PMUT (see modal_kernel).
constexpr int kModalWarps = 4;

// Modal ODE of PMUT k (warp 0, lane m = mode m): predictor / solve / corrector with the
// projection G_m = sum over the block's partial sums red[w][m]; q'' of every mode into qv_s.
__device__ __forceinline__ void modal_ode(const ModalParams& p, int k, const double (*red)[kMaxModes], double* qv_s,
                                          int lane) {
    const unsigned FULL = 0xffffffffu;
    const int M = p.n_modes;
    const double dt = p.dt;
    {
        const long long n = __ldcg(p.step);
        const double t1 = (double)(n + 1) * dt, t0 = (double)n * dt;
        double G = 0.0;
        if (lane < kMaxModes)
#pragma unroll
            for (int w = 0; w < kModalWarps; ++w) G += red[w][lane];
        const bool act = lane < M;
        const size_t km = (size_t)k * M + lane;
        double q = 0, qd = 0, qdd = 0;
        if (act) { q = p.q[km]; qd = p.qd[km]; qdd = p.qdd[km]; }
        const double q1 = q + dt * qd + 0.5 * dt * dt * qdd;
        double qd1 = qd + 0.5 * dt * qdd;
        const double etam = act ? p.eta[lane] : 0.0;
        // phi at the coupling time level (R2): predicted -> (t^{n+1}, q^{n+1}); literal -> (t^n, q^n)
        const double tu = p.literal ? t0 : t1;
        double s = etam * (p.literal ? q : q1);
        double s1 = etam * q1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(FULL, s, o);
            s1 += __shfl_xor_sync(FULL, s1, o);
        }
        const double tp_delay = p.delay[k];
        const double phi = (p.rx && tu > p.t_switch) ? s * p.invC : drive_tx(p, tu - tp_delay);
        const double phi1 = (p.rx && t1 > p.t_switch) ? s1 * p.invC : drive_tx(p, t1 - tp_delay);
        double qdd1 = 0.0;
        if (act) {
            qdd1 = -p.omega2[km] * q1 - p.twozw[km] * qd1 + (-G + etam * phi) * p.invmass[lane];
            qd1 = qd1 + 0.5 * dt * qdd1;
            p.q[km] = q1;
            p.qd[km] = qd1;
            p.qdd[km] = qdd1;
        }
        if (lane == 0) p.phi[k] = phi1;
        if (lane < kMaxModes) qv_s[lane] = qdd1;
    }
}

// One block of kModalWarps warps per PMUT: the warps share the membrane's rows (projection and force
// plane), warp 0 advances the modes.  (One warp per PMUT left the grid at < 1 block per SM for the
// 512 PMUTs of a cfg-3 slab: latency-bound.)

__global__ void __launch_bounds__(32 * kModalWarps) modal_kernel(const __grid_constant__ ModalParams p) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x;
    const unsigned FULL = 0xffffffffu;
    const int M = p.n_modes;
    const int i0 = p.rect[4 * k], j0 = p.rect[4 * k + 1], ni = p.rect[4 * k + 2], nj = p.rect[4 * k + 3];
    const int L = p.lmax, nn = ni * nj;
    __shared__ double red[kModalWarps][kMaxModes];
    __shared__ double qv_s[kMaxModes];
    // this PMUT's separable tables, staged once: sx[m][i], sy[m][j] and the face mass factors wx, wy
    extern __shared__ double mtab[];
    double* const tsx = mtab;
    double* const tsy = tsx + M * L;
    double* const twx = tsy + M * L;
    double* const twy = twx + L;
    {
        const double* sxk = p.sx + (size_t)k * M * L;
        const double* syk = p.sy + (size_t)k * M * L;
        for (int q = threadIdx.x; q < M * L; q += blockDim.x) {
            tsx[q] = __ldg(sxk + q);
            tsy[q] = __ldg(syk + q);
        }
        for (int q = threadIdx.x; q < L; q += blockDim.x) {
            twx[q] = __ldg(p.wx + (size_t)k * L + q);
            twy[q] = __ldg(p.wy + (size_t)k * L + q);
        }
    }
    __syncthreads();
    // pressure projection G_m = sum_ij m_x(i) S_x(i) m_y(j) S_y(j) p_ij   (Eq. 12: int p U.n = -G); the
    // membrane's nodes are spread over the block, several loads in flight per thread
    double acc[kMaxModes];
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) acc[m] = 0.0;
#pragma unroll 4
    for (int q = threadIdx.x; q < nn; q += blockDim.x) {
        const int j = q / ni, i = q - j * ni;
        const double val = p.P[(long long)(j0 + j) * p.PX + i0 + i] * twx[i] * twy[j];
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m)
            if (m < M) acc[m] = fma(tsx[m * L + i] * tsy[m * L + j], val, acc[m]);
    }
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[m] += __shfl_xor_sync(FULL, acc[m], o);
    }
    if (lane == 0)
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m) red[warp][m] = acc[m];
    __syncthreads();

    if (warp == 0) modal_ode(p, k, red, qv_s, lane);
    __syncthreads();
    double qv[kMaxModes];
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) qv[m] = qv_s[m];
    // force plane F = kappa sum_m qdd_m S_m  (Eq. 11; the 1/M factor is applied in vol_kernel)
    for (int q = threadIdx.x; q < nn; q += blockDim.x) {
        const int j = q / ni, i = q - j * ni;
        double f = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m)
            if (m < M) f = fma(qv[m], tsx[m * L + i] * tsy[m * L + j], f);
        SEM_CHECK(i0 + i < p.NX);
        p.F[(long long)(j0 + j) * p.NX + i0 + i] = p.kappa * f;
    }
}

// Tabulated coupling (curved boxes): one block per PMUT over its face-node list; projection
// G_m = sum_j B[j][m] p_j (Eq. 12), the same modal ODE, then r_j -= kappa sum_m qdd_m B[j][m] (Eq. 11)
// into the box's assembled residual (membranes are disjoint: no two blocks touch a node).
__global__ void __launch_bounds__(32 * kModalWarps) modal_table_kernel(const __grid_constant__ ModalParams p) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x, M = p.n_modes;
    const int j0 = p.toff[k], j1 = p.toff[k + 1];
    __shared__ double red[kModalWarps][kMaxModes];
    __shared__ double qv_s[kMaxModes];
    double acc[kMaxModes];
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) acc[m] = 0.0;
    SEM_CHECK(j0 >= 0 && j1 >= j0);
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        SEM_CHECK(p.tidx[j] >= 0 && p.tidx[j] < p.PX * p.NY_dbg);
        const double v = p.P[p.tidx[j]];
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m)
            if (m < M) acc[m] = fma(p.tB[(long long)j * M + m], v, acc[m]);
    }
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[m] += __shfl_xor_sync(0xffffffffu, acc[m], o);
    }
    if (lane == 0)
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m) red[warp][m] = acc[m];
    __syncthreads();
    if (warp == 0) modal_ode(p, k, red, qv_s, lane);
    __syncthreads();
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        double f = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m)
            if (m < M) f = fma(qv_s[m], p.tB[(long long)j * M + m], f);
        atomicAdd(p.res + p.tidx[j], -p.kappa * f);   // (other kernels may add to the residual concurrently)
    }
}

void launch_modal(const ModalParams& p, cudaStream_t s) {
    if (p.n_pmut <= 0) return;
    if (p.toff) modal_table_kernel<<<p.n_pmut, 32 * kModalWarps, 0, s>>>(p);
    else modal_kernel<<<p.n_pmut, 32 * kModalWarps, (size_t)8 * (2 * p.n_modes * p.lmax + 2 * p.lmax), s>>>(p);
}

// ------------------------------------------------------------------------------------------------
// Interface (SIPG, Eq. 7) on the 2:1 face, fine-face GLL lattice as quadrature (reading R9)
// ------------------------------------------------------------------------------------------------
__global__ void iface_coarse_trace(const __grid_constant__ IfaceParams p) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (int)(p.NXc * p.NYc)) return;
    const int NXc = (int)p.NXc;
    const int jx = id % NXc, jy = id / NXc;
    const long long S = p.PXc * p.NYc;
    const double* col = p.Pc + (long long)jy * p.PXc + jx;
    double d = 0.0;
    for (int c = 0; c <= p.Nc; ++c) d = fma(p.dcB[c], col[c * S], d);
    p.trc[id] = col[0];
    p.drc[id] = d;
}


// Fine side of the SIPG flux at the fine-face GLL lattice (reading R9): jump J = p+ - p-(x_q) and
// average flux A = 1/2 (c+^2 d_n p+ + c-^2 d_n p-) with p-, d_n p- interpolated from the coarse face
// lattice (tensor product of the 1D tables I).  Writes tau = gamma J - A and sigma = -1/2 c+^2 J (the
// fine side's layer terms); the coarse side's weighted terms are derived from them in iface_gather_y.
// Template arguments NF, NC, R fix the degrees and the ratio at compile time (0: read from p).
template <int NF, int NC, int R>
__global__ void __launch_bounds__(256) iface_fine(const __grid_constant__ IfaceParams p) {
    const int Nf = NF ? NF : p.Nf, Nc = NC ? NC : p.Nc, NfR = Nf * (R ? R : p.R);
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int NXf = (int)p.NXf;
    if (id >= NXf * (int)p.NYf) return;
    const int ix = id % NXf, iy = id / NXf;
    const long long S = p.PXf * p.NYf;
    const double* top = p.Pf + (p.NZf - 1) * S + (long long)iy * p.PXf + ix;
    // coarse element and local fine index along x and y
    int ex = ix / NfR, ey = iy / NfR;
    if (ex > p.nelcx - 1) ex = p.nelcx - 1;
    if (ey > p.nelcy - 1) ey = p.nelcy - 1;
    const int qx = ix - ex * NfR, qy = iy - ey * NfR;
    const int NXc = (int)p.NXc;
    const int c0 = ey * Nc * NXc + ex * Nc;
    SEM_CHECK(c0 + Nc * NXc + Nc < NXc * (int)p.NYc && p.NZf > Nf);
    // fine trace and normal derivative (n+ = +e_z): the top element layer of the fine box
    const double pp = __ldg(top);
    double dpp = 0.0;
#pragma unroll
    for (int c = 0; c <= (NF ? NF : kMaxN); ++c)
        if (NF || c <= Nf) dpp = fma(p.dfT[c], __ldg(top - (long long)(Nf - c) * S), dpp);
    double pm = 0.0, dpm = 0.0;
#pragma unroll
    for (int b = 0; b <= (NC ? NC : kMaxN); ++b) {
        if (!NC && b > Nc) break;
        const double wy = __ldg(p.I + qy * (Nc + 1) + b);
        const int row = c0 + b * NXc;
        double rt = 0.0, rd = 0.0;
#pragma unroll
        for (int a = 0; a <= (NC ? NC : kMaxN); ++a) {
            if (!NC && a > Nc) break;
            const double wx = __ldg(p.I + qx * (Nc + 1) + a);
            rt = fma(wx, __ldg(p.trc + row + a), rt);
            rd = fma(wx, __ldg(p.drc + row + a), rd);
        }
        pm = fma(wy, rt, pm);
        dpm = fma(wy, rd, dpm);
    }
    const double J = pp - pm;                              // [[p]].n+
    const double A = 0.5 * (p.cf2 * dpp + p.cc2 * dpm);     // {c^2 grad p}.n+
    p.tauf[id] = p.gamma * J - A;
    p.sigf[id] = -0.5 * p.cf2 * J;
}

// Transposed interpolation along one lattice direction: out(j) = sum_i psi_j(x_i) in(i), where fine
// lattice index i lies in coarse element e = min(i / NfR, nelc - 1) at local index q = i - e NfR and
// psi_j(x_i) = I[q][j - e Nc] if 0 <= j - e Nc <= Nc.  Coarse node j = e Nc + b touches the fine
// nodes of element e (and of e - 1 if b = 0): at most 2 NfR + 1 of them, from lo = (e or e-1) NfR.
template <int NF, int NC, int R>
__device__ __forceinline__ void gather_1d(const IfaceParams& p, int j, int nelc, int nf, const double* __restrict__ in1,
                                          const double* __restrict__ in2, int stride, const double* __restrict__ wi,
                                          int skip0, double& s1, double& s2) {
    const int Nc = NC ? NC : p.Nc, NfR = (NF ? NF : p.Nf) * (R ? R : p.R);
    int e = j / Nc;
    int b = j - e * Nc;
    if (e > nelc - 1) {   // last coarse node: b = Nc of the last element
        e = nelc - 1;
        b = Nc;
    }
    s1 = 0.0;
    s2 = 0.0;
    // own element e: fine nodes e NfR + q, q = 0..NfR (q = NfR only for the last element)
    const int qend = (e == nelc - 1) ? NfR : NfR - 1;
#pragma unroll 4
    for (int q = 0; q <= qend; ++q) {
        const int i = e * NfR + q;
        SEM_CHECK(i < nf);
        if (skip0 && i == 0) continue;
        double w = __ldg(p.I + q * (Nc + 1) + b);
        if (wi) w *= __ldg(wi + i);
        s1 = fma(w, __ldg(in1 + i * stride), s1);
        s2 = fma(w, __ldg(in2 + i * stride), s2);
    }
    if (b == 0 && e > 0) {   // left element e - 1 (its q = 0 node has weight I[0][Nc] = 0; q = NfR is in e)
#pragma unroll 4
        for (int q = 1; q < NfR; ++q) {
            const int i = (e - 1) * NfR + q;
            double w = __ldg(p.I + q * (Nc + 1) + Nc);
            if (wi) w *= __ldg(wi + i);
            s1 = fma(w, __ldg(in1 + i * stride), s1);
            s2 = fma(w, __ldg(in2 + i * stride), s2);
        }
    }
}

// y pass of the coarse-side gather.  The weighted fine terms are g1 = W_q (A - gamma J) = -W_q tau and
// g2 = W_q (-1/2 c-^2 J) = W_q (c-^2 / c+^2) sigma, W_q = m_x(ix) m_y(iy) the assembled fine-face weights.
template <int NF, int NC, int R>
__global__ void __launch_bounds__(256) iface_gather_y(const __grid_constant__ IfaceParams p) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int NXf = (int)p.NXf;
    if (id >= NXf * (int)p.NYc) return;
    const int ix = id % NXf, jy = id / NXf;
    double s1, s2;
    // the fine cut line iy = 0 of a slab with a lower cut is counted by the lower slab only
    gather_1d<NF, NC, R>(p, jy, p.nelcy, (int)p.NYf, p.tauf + ix, p.sigf + ix, NXf, p.myf, p.skip_iy0, s1, s2);
    const double mx = __ldg(p.mxf + ix);
    p.h1[id] = -mx * s1;
    p.h2[id] = (p.cc2 / p.cf2) * mx * s2;
}

template <int NF, int NC, int R>
__global__ void __launch_bounds__(256) iface_gather_x(const __grid_constant__ IfaceParams p) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int NXc = (int)p.NXc, NXf = (int)p.NXf;
    if (id >= NXc * (int)p.NYc) return;
    const int jx = id % NXc, jy = id / NXc;
    double s1, s2;
    gather_1d<NF, NC, R>(p, jx, p.nelcx, NXf, p.h1 + jy * NXf, p.h2 + jy * NXf, 1, nullptr, 0, s1, s2);
    const double inv = 1.0 / (p.mxc[jx] * p.myc[jy]);
    p.tauc[id] = s1 * inv;
    p.sigc[id] = s2 * inv;
}

// ---- Gauss-Legendre variant (quad_rule 1).  A block holds FPB = 256 / (Nf+1)^2 fine faces, one
// thread per face node / LG point; the 2D interpolations are done as two 1D passes through shared
// memory.  (1) node (a, b): trace p+ and d_n p+.  (2) LG point (kx, ky): p+, d_n p+ by the fine basis
// at the LG points, p-, d_n p- by the coarse basis (ILG); T = gamma J - A, S = -1/2 c+^2 J weighted by
// W_q; the coarse side's terms g1 = -W T, g2 = W (c-^2/c+^2) S go to the LG lattice.  (3) node
// (a, b): sum_q W_q T_q l_a l_b (and S) accumulated into the fine nodes (atomics: face edges are shared).
__global__ void __launch_bounds__(256) iface_fine_lg(const __grid_constant__ IfaceParams p) {
    const int Nf = p.Nf, Nc = p.Nc, n1 = Nf + 1, n2 = n1 * n1, R = p.R, nq = n1;
    const int FPB = blockDim.x / n2;
    extern __shared__ double lg_smem[];
    double* const sL = lg_smem;                           // Lf [nq][n1]
    const int fl = threadIdx.x / n2, t = threadIdx.x - fl * n2;
    double* const base = lg_smem + n2 + (size_t)(fl < FPB ? fl : 0) * 6 * n2;
    double* const sPp = base;            // trace at the nodes, then T at the LG points
    double* const sDp = base + n2;       // d_n p+ at the nodes, then S
    double* const t1 = base + 2 * n2;    // first-pass buffers
    double* const t2 = base + 3 * n2;
    double* const sT = base + 4 * n2;
    double* const sS = base + 5 * n2;
    for (int q = threadIdx.x; q < n2; q += blockDim.x) sL[q] = p.Lf[q];
    const int f = blockIdx.x * FPB + fl;
    const bool act = fl < FPB && f < p.nelfx * p.nelfy;
    const int fx = act ? f % p.nelfx : 0, fy = act ? f / p.nelfx : 0;
    const int a = t % n1, b = t / n1;   // node (a, b) or LG point (kx, ky) = (a, b)
    const long long S = p.PXf * p.NYf;
    const int ix = fx * Nf + a, iy = fy * Nf + b;
    if (act) {
        const double* top = p.Pf + (p.NZf - 1) * S + (long long)iy * p.PXf + ix;
        double d = 0.0;
        for (int c = 0; c <= Nf; ++c) d = fma(p.dfT[c], __ldg(top - (long long)(Nf - c) * S), d);
        sPp[t] = __ldg(top);
        sDp[t] = d;
    }
    __syncthreads();
    if (act) {   // x pass: t1(kx, b) = sum_aa l_aa(xq_kx) P(aa, b)
        const int kx = a;
        double r1 = 0.0, r2 = 0.0;
        for (int aa = 0; aa <= Nf; ++aa) {
            const double l = sL[kx * n1 + aa];
            r1 = fma(l, sPp[aa + n1 * b], r1);
            r2 = fma(l, sDp[aa + n1 * b], r2);
        }
        t1[t] = r1;
        t2[t] = r2;
    }
    __syncthreads();
    if (act) {   // y pass and the flux at LG point (kx, ky)
        const int kx = a, ky = b;
        double pp = 0.0, dpp = 0.0;
        for (int bb = 0; bb <= Nf; ++bb) {
            const double l = sL[ky * n1 + bb];
            pp = fma(l, t1[kx + n1 * bb], pp);
            dpp = fma(l, t2[kx + n1 * bb], dpp);
        }
        const int ecx = fx / R, ecy = fy / R;
        const int qx = (fx - ecx * R) * nq + kx, qy = (fy - ecy * R) * nq + ky;
        const int NXc = (int)p.NXc;
        const int c0 = ecy * Nc * NXc + ecx * Nc;
        double pm = 0.0, dpm = 0.0;
        for (int bb = 0; bb <= Nc; ++bb) {
            double rt = 0.0, rd = 0.0;
            for (int aa = 0; aa <= Nc; ++aa) {
                const double wx = __ldg(p.ILG + qx * (Nc + 1) + aa);
                rt = fma(wx, __ldg(p.trc + c0 + bb * NXc + aa), rt);
                rd = fma(wx, __ldg(p.drc + c0 + bb * NXc + aa), rd);
            }
            const double wy = __ldg(p.ILG + qy * (Nc + 1) + bb);
            pm = fma(wy, rt, pm);
            dpm = fma(wy, rd, dpm);
        }
        const double J = pp - pm;
        const double A = 0.5 * (p.cf2 * dpp + p.cc2 * dpm);
        const double W = p.wqx[kx] * p.wqy[ky];
        const double T = W * (p.gamma * J - A), Sg = W * (-0.5 * p.cf2 * J);
        sT[t] = T;
        sS[t] = Sg;
        const long long gq = (long long)(fy * nq + ky) * p.NXq + fx * nq + kx;
        SEM_CHECK(gq < p.NXq * p.NYq && c0 + Nc * NXc + Nc < NXc * (int)p.NYc);
        p.g1[gq] = -T;
        p.g2[gq] = (p.cc2 / p.cf2) * Sg;
    }
    __syncthreads();
    if (act) {   // projection, x pass: t1(a, ky) = sum_kx l_a(xq_kx) T(kx, ky)
        const int ky = b;
        double r1 = 0.0, r2 = 0.0;
        for (int kx = 0; kx < nq; ++kx) {
            const double l = sL[kx * n1 + a];
            r1 = fma(l, sT[kx + n1 * ky], r1);
            r2 = fma(l, sS[kx + n1 * ky], r2);
        }
        t1[t] = r1;
        t2[t] = r2;
    }
    __syncthreads();
    if (act) {   // y pass and accumulation at node (a, b)
        double ts = 0.0, ss = 0.0;
        for (int ky = 0; ky < nq; ++ky) {
            const double l = sL[ky * n1 + b];
            ts = fma(l, t1[a + n1 * ky], ts);
            ss = fma(l, t2[a + n1 * ky], ss);
        }
        const long long g = (long long)iy * p.NXf + ix;
        SEM_CHECK(ix < p.NXf && iy < p.NYf);
        atomicAdd(p.tacc + g, ts);
        atomicAdd(p.sacc + g, ss);
    }
}

// collocated-equivalent fine values tau = acc / (m_x m_y) (vol_kernel divides by m_z); clears acc
__global__ void iface_lg_normalise(const __grid_constant__ IfaceParams p) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int NXf = (int)p.NXf;
    if (id >= NXf * (int)p.NYf) return;
    const int ix = id % NXf, iy = id / NXf;
    const double inv = 1.0 / (p.mxf[ix] * p.myf[iy]);
    p.tauf[id] = p.tacc[id] * inv;
    p.sigf[id] = p.sacc[id] * inv;
    p.tacc[id] = 0.0;
    p.sacc[id] = 0.0;
}

// transposed coarse interpolation over the LG lattice along one direction: coarse node j = e Nc + b
// collects the RQ = R nq points of element e (weight ILG[k][b]) and, for b = 0, those of e - 1
// (weight ILG[k][Nc]); no point is shared between elements
__device__ __forceinline__ void gather_1d_lg(const IfaceParams& p, int j, int nelc, const double* __restrict__ in1,
                                             const double* __restrict__ in2, long long stride, double& s1, double& s2) {
    const int Nc = p.Nc, RQ = p.R * (p.Nf + 1);
    int e = j / Nc, b = j - e * Nc;
    if (e > nelc - 1) {
        e = nelc - 1;
        b = Nc;
    }
    s1 = 0.0;
    s2 = 0.0;
    for (int k = 0; k < RQ; ++k) {
        const long long i = (long long)(e * RQ + k) * stride;
        const double w = __ldg(p.ILG + k * (Nc + 1) + b);
        s1 = fma(w, __ldg(in1 + i), s1);
        s2 = fma(w, __ldg(in2 + i), s2);
    }
    if (b == 0 && e > 0) {
        for (int k = 0; k < RQ; ++k) {
            const long long i = (long long)((e - 1) * RQ + k) * stride;
            const double w = __ldg(p.ILG + k * (Nc + 1) + Nc);
            s1 = fma(w, __ldg(in1 + i), s1);
            s2 = fma(w, __ldg(in2 + i), s2);
        }
    }
}

__global__ void iface_gather_y_lg(const __grid_constant__ IfaceParams p) {
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= p.NXq * p.NYc) return;
    const long long qx = id % p.NXq, jy = id / p.NXq;
    double s1, s2;
    gather_1d_lg(p, (int)jy, p.nelcy, p.g1 + qx, p.g2 + qx, p.NXq, s1, s2);
    p.q1[id] = s1;
    p.q2[id] = s2;
}

__global__ void iface_gather_x_lg(const __grid_constant__ IfaceParams p) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int NXc = (int)p.NXc;
    if (id >= NXc * (int)p.NYc) return;
    const int jx = id % NXc, jy = id / NXc;
    double s1, s2;
    gather_1d_lg(p, jx, p.nelcx, p.q1 + (long long)jy * p.NXq, p.q2 + (long long)jy * p.NXq, 1, s1, s2);
    const double inv = 1.0 / (p.mxc[jx] * p.myc[jy]);
    p.tauc[id] = s1 * inv;
    p.sigc[id] = s2 * inv;
}

static void launch_iface_lg(const IfaceParams& p, cudaStream_t s) {
    const int T = 256;
    const long long nc = p.NXc * p.NYc, nf = p.NXf * p.NYf, nfaces = (long long)p.nelfx * p.nelfy;
    iface_coarse_trace<<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(p);
    const int n2 = (p.Nf + 1) * (p.Nf + 1), fpb = 256 / n2;
    const size_t smem = sizeof(double) * (size_t)n2 * (1 + 6 * fpb);
    iface_fine_lg<<<(unsigned)((nfaces + fpb - 1) / fpb), fpb * n2, smem, s>>>(p);
    iface_lg_normalise<<<(unsigned)((nf + T - 1) / T), T, 0, s>>>(p);
    iface_gather_y_lg<<<(unsigned)((p.NXq * p.NYc + T - 1) / T), T, 0, s>>>(p);
    iface_gather_x_lg<<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(p);
}

// Fused SIPG flux on the 2:1 face lattice for compile-time (NF, NC, R) (configs 2-4: 5, 3, 2): one block
// per TC x TC tile of coarse elements does what iface_coarse_trace -> iface_fine -> iface_gather_y ->
// iface_gather_x do, with the intermediate face arrays in shared memory.  The tile's footprint extends
// one coarse element below it in x and y (the coarse nodes on its lower edges also collect the fine
// points of that element), so every coarse node it owns gets its complete sum: the halo element's fine
// flux is recomputed (L2-resident inputs) instead of exchanged.
//   (1) coarse trace p- and d_n p- at the footprint's coarse face nodes (bottom element layer);
//   (2) fine flux at the footprint's fine face nodes: J = p+ - p-(x_q), A = 1/2 (c+^2 d_n p+ + c-^2 d_n p-),
//       tau = gamma J - A, sigma = -1/2 c+^2 J (written for the fine nodes the tile owns) and the weighted
//       coarse-side terms g1 = -W tau, g2 = W (c-^2/c+^2) sigma (W = m_x m_y) in shared memory;
//   (3) transposed interpolation along y, then (4) along x, divided by the coarse face masses.
#ifndef SEM_IF_TC
#define SEM_IF_TC 4
#endif
constexpr int kIfTC = SEM_IF_TC;   // coarse elements per tile edge
template <int NF, int NC, int R>
struct IfFused {
    static constexpr int NFR = NF * R;                 // fine nodes per coarse element edge
    static constexpr int FW = (kIfTC + 1) * NFR + 1;   // fine footprint nodes per direction
    static constexpr int CW = (kIfTC + 1) * NC + 1;    // coarse footprint nodes per direction
    static constexpr int CO = kIfTC * NC + 1;          // owned coarse rows (the last tile: + the box's last)
    // shared memory: coarse trace [2][CW][CW] | weighted fine terms [2][FW][FW] | a union of the
    // x-interpolated coarse trace [2][CW][FW] (phase 2) and the y-gathered terms [2][CO][FW] (phases 3-4)
    static constexpr int UNION = (CW > CO ? CW : CO) * FW;
    static constexpr int SMEM = 8 * (2 * CW * CW + 2 * FW * FW + 2 * UNION);
};

template <int NF, int NC, int R>
#ifndef SEM_IF_THREADS
#define SEM_IF_THREADS 512
#endif
__global__ void __launch_bounds__(SEM_IF_THREADS) iface_fused(const __grid_constant__ IfaceParams p) {
    using G = IfFused<NF, NC, R>;
    constexpr int NFR = G::NFR, FW = G::FW, CW = G::CW, CO = G::CO, TC = kIfTC;
    extern __shared__ double ifs[];
    double* const st = ifs;                 // [CW][CW] coarse trace
    double* const sd = st + CW * CW;        // [CW][CW] coarse normal derivative
    double* const g1 = sd + CW * CW;        // [FW][FW] weighted fine terms (row = y)
    double* const g2 = g1 + FW * FW;
    double* const h1 = g2 + FW * FW;        // [CO][FW] after the y pass
    double* const h2 = h1 + G::UNION;
    double* const xt = h1;                  // [CW][FW] coarse trace interpolated along x (phase 2 only)
    double* const xd = h2;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int ex0 = (int)blockIdx.x * TC - 1, ey0 = (int)blockIdx.y * TC - 1;   // footprint's first element
    const long long NXf = p.NXf, NYf = p.NYf, NXc = p.NXc, NYc = p.NYc;
    const int nelcx = p.nelcx, nelcy = p.nelcy;
    // (1) coarse trace
    const long long Sc = p.PXc * NYc;
    for (int k = tid; k < CW * CW; k += nth) {
        const int i = k % CW, j = k / CW;
        const long long jx = (long long)ex0 * NC + i, jy = (long long)ey0 * NC + j;
        double t = 0.0, d = 0.0;
        if (jx >= 0 && jx < NXc && jy >= 0 && jy < NYc) {
            const double* col = p.Pc + jy * p.PXc + jx;
            t = __ldg(col);
#pragma unroll
            for (int c = 0; c <= NC; ++c) d = fma(p.dcB[c], __ldg(col + c * Sc), d);
        }
        st[k] = t;
        sd[k] = d;
    }
    __syncthreads();
    // (1b) the coarse trace interpolated along x at every fine column of the footprint (separable: the
    //      fine flux then needs N_c + 1 values per node instead of (N_c + 1)^2)
    for (int k = tid; k < CW * FW; k += nth) {
        const int i = k % FW, j = k / FW;
        const int elx = i / NFR < TC ? i / NFR : TC, qx = i - elx * NFR;
        double rt = 0.0, rd = 0.0;
#pragma unroll
        for (int a = 0; a <= NC; ++a) {
            const double wx = __ldg(p.I + qx * (NC + 1) + a);
            rt = fma(wx, st[j * CW + elx * NC + a], rt);
            rd = fma(wx, sd[j * CW + elx * NC + a], rd);
        }
        xt[k] = rt;
        xd[k] = rd;
    }
    __syncthreads();
    // (2) fine flux
    const long long Sf = p.PXf * NYf;
    const double* top = p.Pf + (p.NZf - 1) * Sf;
    const long long ox = (long long)blockIdx.x * TC * NFR, oy = (long long)blockIdx.y * TC * NFR;   // owned start
    const double crat = p.cc2 / p.cf2;
    for (int k = tid; k < FW * FW; k += nth) {
        const int i = k % FW, j = k / FW;
        const long long ix = (long long)ex0 * NFR + i, iy = (long long)ey0 * NFR + j;
        double v1 = 0.0, v2 = 0.0;
        if (ix >= 0 && ix < NXf && iy >= 0 && iy < NYf) {
            const double* node = top + iy * p.PXf + ix;
            const double pp = __ldg(node);
            double dpp = 0.0;
            if (p.dzf) {   // written by the previous volume launch (the same sum in the same order)
                dpp = __ldg(p.dzf + iy * NXf + ix);
            } else {
#pragma unroll
                for (int c = 0; c <= NF; ++c) dpp = fma(p.dfT[c], __ldg(node - (long long)(NF - c) * Sf), dpp);
            }
            // coarse element row (footprint-local) and local fine index of this node in it along y
            const int ely = j / NFR < TC ? j / NFR : TC, qy = j - ely * NFR;
            double pm = 0.0, dpm = 0.0;
#pragma unroll
            for (int b = 0; b <= NC; ++b) {
                const double wy = __ldg(p.I + qy * (NC + 1) + b);
                pm = fma(wy, xt[(ely * NC + b) * FW + i], pm);
                dpm = fma(wy, xd[(ely * NC + b) * FW + i], dpm);
            }
            const double J = pp - pm;
            const double A = 0.5 * (p.cf2 * dpp + p.cc2 * dpm);
            const double tau = p.gamma * J - A, sig = -0.5 * p.cf2 * J;
            const bool own = ix >= ox && (ix < ox + TC * NFR || ix == NXf - 1) && iy >= oy &&
                             (iy < oy + TC * NFR || iy == NYf - 1);
            if (own) {
                SEM_CHECK(ix < NXf && iy < NYf);
                p.tauf[iy * NXf + ix] = tau;
                p.sigf[iy * NXf + ix] = sig;
            }
            if (!(p.skip_iy0 && iy == 0)) {   // the fine cut line of a slab belongs to the lower slab
                const double W = __ldg(p.mxf + ix) * __ldg(p.myf + iy);
                v1 = -W * tau;
                v2 = crat * W * sig;
            }
        }
        g1[k] = v1;
        g2[k] = v2;
    }
    __syncthreads();
    // coarse node (footprint-local index jl) -> element el and local index b as in gather_1d
    auto split = [](int jl, int e0, int nelc, int& el, int& b) {
        el = jl / NC;
        b = jl - el * NC;
        if (e0 + el > nelc - 1) {   // the box's last coarse node: b = NC of the last element
            el -= 1;
            b = NC;
        }
    };
    // owned coarse rows / columns: footprint-local jl in [NC, NC + CO), global j < n, and j in the tile's
    // range (the box's last node belongs to the last tile)
    auto owned = [](long long j, long long j0, long long n) { return j < n && (j < j0 + TC * NC || j == n - 1); };
    const long long jx0 = (long long)blockIdx.x * TC * NC, jy0 = (long long)blockIdx.y * TC * NC;
    // (3) y pass: h[jr][i] = sum_q psi_b(x_q) g[q][i] over the fine rows of the coarse row's support
    for (int k = tid; k < CO * FW; k += nth) {
        const int i = k % FW, jr = k / FW, jl = NC + jr;
        const long long jy = (long long)ey0 * NC + jl;
        double s1 = 0.0, s2 = 0.0;
        if (owned(jy, jy0, NYc)) {
            int el, b;
            split(jl, ey0, nelcy, el, b);
            const int qend = (ey0 + el == nelcy - 1) ? NFR : NFR - 1;
            for (int q = 0; q <= qend; ++q) {
                const double w = __ldg(p.I + q * (NC + 1) + b);
                s1 = fma(w, g1[(el * NFR + q) * FW + i], s1);
                s2 = fma(w, g2[(el * NFR + q) * FW + i], s2);
            }
            if (b == 0 && el > 0) {   // the element below (its q = 0 node has weight I[0][NC] = 0)
                for (int q = 1; q < NFR; ++q) {
                    const double w = __ldg(p.I + q * (NC + 1) + NC);
                    s1 = fma(w, g1[((el - 1) * NFR + q) * FW + i], s1);
                    s2 = fma(w, g2[((el - 1) * NFR + q) * FW + i], s2);
                }
            }
        }
        h1[k] = s1;
        h2[k] = s2;
    }
    __syncthreads();
    // (4) x pass and the coarse face masses
    for (int k = tid; k < CO * CO; k += nth) {
        const int ir = k % CO, jr = k / CO, il = NC + ir;
        const long long jx = (long long)ex0 * NC + il, jy = (long long)ey0 * NC + NC + jr;
        if (!owned(jx, jx0, NXc) || !owned(jy, jy0, NYc)) continue;
        int el, b;
        split(il, ex0, nelcx, el, b);
        const int qend = (ex0 + el == nelcx - 1) ? NFR : NFR - 1;
        double s1 = 0.0, s2 = 0.0;
        for (int q = 0; q <= qend; ++q) {
            const double w = __ldg(p.I + q * (NC + 1) + b);
            s1 = fma(w, h1[jr * FW + el * NFR + q], s1);
            s2 = fma(w, h2[jr * FW + el * NFR + q], s2);
        }
        if (b == 0 && el > 0) {
            for (int q = 1; q < NFR; ++q) {
                const double w = __ldg(p.I + q * (NC + 1) + NC);
                s1 = fma(w, h1[jr * FW + (el - 1) * NFR + q], s1);
                s2 = fma(w, h2[jr * FW + (el - 1) * NFR + q], s2);
            }
        }
        SEM_CHECK(jx >= 0 && jx < NXc && jy >= 0 && jy < NYc);
        const double inv = 1.0 / (__ldg(p.mxc + jx) * __ldg(p.myc + jy));
        p.tauc[jy * NXc + jx] = s1 * inv;
        p.sigc[jy * NXc + jx] = s2 * inv;
    }
}

template <int NF, int NC, int R>
static int launch_iface_fused(const IfaceParams& p, cudaStream_t s) {
    using G = IfFused<NF, NC, R>;
    const dim3 grid((unsigned)((p.nelcx + kIfTC - 1) / kIfTC), (unsigned)((p.nelcy + kIfTC - 1) / kIfTC));
    iface_fused<NF, NC, R><<<grid, SEM_IF_THREADS, G::SMEM, s>>>(p);
    return 1;
}

template <int NF, int NC, int R>
static void launch_iface_t(const IfaceParams& p, cudaStream_t s) {
    const int T = 256;
    const long long nc = p.NXc * p.NYc, nf = p.NXf * p.NYf, nh = p.NXf * p.NYc;
    iface_coarse_trace<<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(p);
    iface_fine<NF, NC, R><<<(unsigned)((nf + T - 1) / T), T, 0, s>>>(p);
    iface_gather_y<NF, NC, R><<<(unsigned)((nh + T - 1) / T), T, 0, s>>>(p);
    iface_gather_x<NF, NC, R><<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(p);
}

#ifndef SEM_IFACE_FUSED
#define SEM_IFACE_FUSED 1
#endif
// d_z p at the fine face from the current state (after sem_write_state / sem_fill_random_state / the
// interface build): the value the volume kernel keeps up to date from then on (VolParams::dzf)
__global__ void iface_dz_init(const __grid_constant__ IfaceParams p, double* dzf) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.NXf * p.NYf) return;
    const long long ix = k % p.NXf, iy = k / p.NXf;
    const long long Sf = p.PXf * p.NYf;
    const double* node = p.Pf + (p.NZf - 1) * Sf + iy * p.PXf + ix;
    double d = 0.0;
    for (int c = 0; c <= p.Nf; ++c) d = fma(p.dfT[c], node[-(long long)(p.Nf - c) * Sf], d);
    dzf[k] = d;
}

void launch_iface_dz_init(const IfaceParams& p, double* dzf, cudaStream_t s) {
    const long long n = p.NXf * p.NYf;
    iface_dz_init<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, dzf);
}

bool iface_uses_dzf(int Nf, int Nc, int R, int lg) { return SEM_IFACE_FUSED && !lg && Nf == 5 && Nc == 3 && R == 2; }


void iface_prepare(int Nf, int Nc, int R) {   // outside any stream capture (function attributes)
    if (SEM_IFACE_FUSED && Nf == 5 && Nc == 3 && R == 2)
        cudaFuncSetAttribute(iface_fused<5, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, IfFused<5, 3, 2>::SMEM);
}

int launch_iface(const IfaceParams& p, cudaStream_t s) {
    if (p.lg) {
        launch_iface_lg(p, s);
        return 5;
    }
    if (p.Nf == 5 && p.Nc == 3 && p.R == 2) {   // configs 2-4
        if (SEM_IFACE_FUSED) return launch_iface_fused<5, 3, 2>(p, s);
        launch_iface_t<5, 3, 2>(p, s);
        return 4;
    }
    launch_iface_t<0, 0, 0>(p, s);
    return 4;
}

// ------------------------------------------------------------------------------------------------
// State / test-hook kernels (pitched device layout: element (ix, r) at r * PX + ix, r = iy + NY iz)
// ------------------------------------------------------------------------------------------------
// Counter-based generator: splitmix64 finaliser of
// key = seed * 0xD1B54A32D192ED03 + box * 0x8CB92BA72F3D8DD7 + field * 0x9E3779B97F4A7C15
// advanced by (id + 1) * 0x9E3779B97F4A7C15; u = 2 (z >> 11) 2^-53 - 1 in [-1, 1); id is the
// lexicographic node id of the ABI layout.
__device__ __forceinline__ double cb_uniform(unsigned long long seed, int box, int field, long long id) {
    unsigned long long z = seed * 0xD1B54A32D192ED03ull + (unsigned long long)box * 0x8CB92BA72F3D8DD7ull +
                           (unsigned long long)field * 0x9E3779B97F4A7C15ull;
    z += ((unsigned long long)id + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}

__global__ void fill_random_kernel(double* pprev, double* w, double* pcur, long long NX, long long PX, long long NY,
                                   long long NZ, long long gy0, long long NYg, unsigned long long seed, int box,
                                   double ps, double vs, double dt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= NX * NY * NZ) return;
    const long long ix = i % NX, r = i / NX, iy = r % NY, iz = r / NY, d = r * PX + ix;
    const long long gid = ix + NX * ((iy + gy0) + NYg * iz);   // global lexicographic id (slab-independent field)
    const double p0 = ps * cb_uniform(seed, box, 0, gid);
    const double v0 = vs * cb_uniform(seed, box, 1, gid);
    pprev[d] = p0;
    w[d] = v0;
    pcur[d] = p0 + dt * v0;     // p^1 = p^0 + dt p'^0 (+ dt^2/2 p''^0 = 0)
}

void launch_fill_random(double* pprev, double* w, double* pcur, long long NX, long long PX, long long NY, long long NZ,
                        long long gy0, long long NYg, unsigned long long seed, int box, double ps, double vs, double dt,
                        cudaStream_t s) {
    const long long n = NX * NY * NZ;
    fill_random_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pprev, w, pcur, NX, PX, NY, NZ, gy0, NYg, seed,
                                                                   box, ps, vs, dt);
}

// ------------------------------------------------------------------------------------------------
// Slab decomposition along y (multi-GPU): partial rows at the cut planes and the fix-up after the
// exchange.  A shared cut node's x row is R0 (right slab) + L (left slab); each
// slab evaluates its own part inside vol_kernel and sends it to the neighbour, which adds it here.
// ------------------------------------------------------------------------------------------------
// One launch per phase for all (side, box) pairs of a slab: blockIdx.y selects the CutParams.  The cut
// plane iy = const is, per z-plane, a contiguous lattice row: one thread per (ix, iz), coalesced.
__global__ void cut_partial_kernel(const __grid_constant__ CutBatch B) {
    const CutParams& c = B.c[blockIdx.y];
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = c.NX * c.NZ;
    if (i < n) {
        const long long ix = i % c.NX, iz = i / c.NX;
        const long long y0 = c.side ? c.NY - 1 - c.N : 0;
        const double* col = c.P + (iz * c.NY + y0) * c.PX + ix;
        double s = 0.0;
        for (int b = 0; b <= c.N; ++b) s = fma(c.row[b], col[(long long)b * c.PX], s);
        c.out[i] = s;
        if (c.pda)   // PML acceleration of this slab's elements at the cut node
            c.out[n + 2 * c.NXt + i] = c.pda[(iz * c.NY + (c.side ? c.NY - 1 : 0)) * c.PX + ix];
    } else if (i < n + c.NXt) {   // coarse SIPG partial sums at the cut row of the face lattice
        const long long jx = i - n;
        const long long jy = c.side ? c.NYt - 1 : 0;
        c.out[n + jx] = c.tau[jy * c.NXt + jx];
        c.out[n + c.NXt + jx] = c.sig[jy * c.NXt + jx];
    }
}

__global__ void cut_fixup_kernel(const __grid_constant__ CutBatch B) {
    const CutParams& c = B.c[blockIdx.y];
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = c.NX * c.NZ;
    if (i >= n) return;
    const long long ix = i % c.NX, iz = i / c.NX;
    double da = -c.in[i];
    if (c.NXt > 0 && iz <= c.N)   // coarse-side SIPG layer terms of the neighbour's fine points
        da -= c.in[n + ix] * c.ktau[iz] + c.in[n + c.NXt + ix] * c.ksig[iz];
    if (c.pda) da += c.in[n + 2 * c.NXt + i];   // the neighbour's PML acceleration
    const long long d = (iz * c.NY + (c.side ? c.NY - 1 : 0)) * c.PX + ix;
    const double dw = c.dt * da;
    if (!SEM_TWO_LEVEL) c.W[d] += dw;
    c.Pn[d] = fma(c.dt, dw, c.Pn[d]);
}

static unsigned cut_blocks(const CutBatch& B, bool partial) {
    long long m = 0;
    for (int k = 0; k < B.n; ++k) {
        const long long n = B.c[k].NX * B.c[k].NZ + (partial ? B.c[k].NXt : 0);
        if (n > m) m = n;
    }
    return (unsigned)((m + 255) / 256);
}

void launch_cut_partial(const CutBatch& B, cudaStream_t s) {
    if (B.n > 0) cut_partial_kernel<<<dim3(cut_blocks(B, true), B.n), 256, 0, s>>>(B);
}

void launch_cut_fixup(const CutBatch& B, cudaStream_t s) {
    if (B.n > 0) cut_fixup_kernel<<<dim3(cut_blocks(B, false), B.n), 256, 0, s>>>(B);
}

// 8-byte asynchronous global -> shared copies (LDGSTS), used to stage element data
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------------------------------------------
// PML (Eq. 1; readings R23-R25): one block per PML element, one thread per
// element GLL node.  psi^{n+3/2} = psi^{n+1/2} + dt p^{n+1}; element-local grad p^{n+1}, grad psi^{n+1};
// Crank-Nicolson update of Phi; weak divergence sum_q w_q |J| Phi^{n+1}(q) . grad phi_i(x_q) and the
// nodal terms alpha pdot + beta p + gamma psi accumulate (atomics) into the PML acceleration da.
// ------------------------------------------------------------------------------------------------
// elements per block of the PML kernels (blocks of ~256 threads: small elements share a block)
template <int N>
constexpr int pml_epb() { return (N + 1) * (N + 1) * (N + 1) >= 256 ? 1 : 256 / ((N + 1) * (N + 1) * (N + 1)); }

// resident blocks per SM the element kernel is compiled for (register budget): more blocks hide the
// latency of its short, barrier-separated phases (N = 3: 339 vs 458 us per cfg-3 PML step); the larger
// elements would spill
#ifndef SEM_PML_MINB3
#define SEM_PML_MINB3 4
#endif
template <int N>
constexpr int pml_minb() { return N <= 3 ? SEM_PML_MINB3 : (N <= 5 ? 3 : (N == 6 ? 2 : 1)); }

template <int N>
__global__ void __launch_bounds__(pml_epb<N>() * (N + 1) * (N + 1) * (N + 1), pml_minb<N>()) pml_element_kernel(const __grid_constant__ PmlParams p) {
    constexpr int n1 = N + 1, nl = n1 * n1 * n1, EPB = pml_epb<N>();
    __shared__ double sp_[EPB][nl], ss_[EPB][nl], sf_[EPB][3][nl], Ds[n1 * n1], DWs[n1 * n1], Ws[n1];
    const int el = threadIdx.x / nl, t = threadIdx.x - el * nl;
    // D[i][j] and w_i D[i][j] in shared memory: lane-dependent indices into the parameter bank would
    // serialise (one constant-cache access per distinct address)
    for (int q = threadIdx.x; q < n1 * n1; q += blockDim.x) {
        Ds[q] = p.D[q / n1][q % n1];
        DWs[q] = p.w[q / n1] * p.D[q / n1][q % n1];
        if (q < n1) Ws[q] = p.w[q];
    }
    double* sp = sp_[el];
    double* ss = ss_[el];
    double (&sf)[3][nl] = sf_[el];
    const int a = t % n1, b = (t / n1) % n1, c = t / (n1 * n1);
    const int kraw = blockIdx.x * EPB + el;
    const bool active = kraw < p.n_el;
    const int k = active ? kraw : p.n_el - 1;   // idle threads mirror the last element (no writes)
    const int ex = p.elems[3 * k], ey = p.elems[3 * k + 1], ez = p.elems[3 * k + 2];
    const int gx = N * ex + a, gy = N * ey + b, gz = N * ez + c;
    const long long g = ((long long)gz * p.NY + gy) * p.PX + gx;
    SEM_CHECK(k >= 0 && k < p.n_el && gx < p.NX && gy < p.NY && gz < p.NZ);
    // every global load first (memory-level parallelism): nodal p, psi, w, the element-local Phi and the
    // per-axis tables
    const double pv = p.P[g];
    const double so = p.psi_old[g];
    // (a y-slab with a lower cut leaves its cut-plane nodes' nodal terms to the slab below, whose last
    //  element owns them: the exchanged PML accelerations then count them once)
    const bool own = (a < N || ex == p.nelx - 1) && (b < N || ey == p.nely - 1) && (c < N || ez == p.nelz - 1) &&
                     !(p.cutL && gy == 0);
#if SEM_TWO_LEVEL   // predictor velocity w^n = (p^{n+1} - p^n) / dt (p^n still in Pn before the volume kernel)
    const double wv = own ? (pv - p.Pn[g]) * p.inv_dt : 0.0;
#else
    const double wv = own ? p.W[g] : 0.0;
#endif
    double* ph = p.phi + (size_t)k * 3 * nl;
    const double phold[3] = {ph[t], ph[nl + t], ph[2 * nl + t]};
    const double* __restrict__ Tx = p.tx + 4 * gx;
    const double* __restrict__ Ty = p.ty + 4 * gy;
    const double* __restrict__ Tz = p.tz + 4 * gz;
    const double z[3] = {Tx[0], Ty[0], Tz[0]};
    const double cA[3] = {Tx[1], Ty[1], Tz[1]}, cB[3] = {Tx[2], Ty[2], Tz[2]};
    const double minv = Tx[3] * Ty[3] * Tz[3];
    const double sn = fma(p.dt, pv, so);
    if (active) p.psi_new[g] = sn;   // a node shared by several PML elements gets the same value from each
    const double sm = 0.5 * (so + sn);
    sp[t] = pv;
    ss[t] = sm;
    __syncthreads();
    // element-local gradients at the own node (reference derivative rows, scaled by 2/h)
    double gp[3] = {0.0, 0.0, 0.0}, gs[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j <= N; ++j) {
        const int ix = j + n1 * (b + n1 * c), iy = a + n1 * (j + n1 * c), iz = a + n1 * (b + n1 * j);
        const double dx = Ds[a * n1 + j], dy = Ds[b * n1 + j], dz = Ds[c * n1 + j];
        gp[0] = fma(dx, sp[ix], gp[0]);
        gs[0] = fma(dx, ss[ix], gs[0]);
        gp[1] = fma(dy, sp[iy], gp[1]);
        gs[1] = fma(dy, ss[iy], gs[1]);
        gp[2] = fma(dz, sp[iz], gp[2]);
        gs[2] = fma(dz, ss[iz], gs[2]);
    }
    const double alpha = z[0] + z[1] + z[2];
    const double beta = z[0] * z[1] + z[1] * z[2] + z[2] * z[0];
    const double gamma = z[0] * z[1] * z[2];
    const double Z3[3] = {z[1] * z[2], z[2] * z[0], z[0] * z[1]};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double old = phold[d];
        const double rhs = p.c2 * p.s2h[d] * ((alpha - 2.0 * z[d]) * gp[d] + Z3[d] * gs[d]);
        const double nw = fma(cA[d], old, cB[d] * rhs);   // Crank-Nicolson on Z1 = -z_d
        if (active) ph[d * nl + t] = nw;
        sf[d][t] = 0.5 * (old + nw);
    }
    __syncthreads();
    // weak divergence at the own node
    double rx = 0.0, ry = 0.0, rz = 0.0;
#pragma unroll
    for (int j = 0; j <= N; ++j) {
        rx = fma(DWs[j * n1 + a], sf[0][j + n1 * (b + n1 * c)], rx);
        ry = fma(DWs[j * n1 + b], sf[1][a + n1 * (j + n1 * c)], ry);
        rz = fma(DWs[j * n1 + c], sf[2][a + n1 * (b + n1 * j)], rz);
    }
    const double wa = Ws[a], wb = Ws[b], wc = Ws[c];
    const double r = p.jac * (p.s2h[0] * wb * wc * rx + p.s2h[1] * wa * wc * ry + p.s2h[2] * wa * wb * rz);
    double da = -r * minv;
    // nodal terms once per node: by the element that owns it (lowest element index containing the node;
    // a non-PML owner only occurs where all z vanish)
    if (own) da -= alpha * wv + beta * pv + gamma * sm;
    if (active) atomicAdd(p.da + g, da);
}

// After the volume kernel: w^{n+1} += dt da, p^{n+2} += dt^2 da (the update is linear in the
// acceleration), and clear da for the next step.  Every node of every PML element is visited; the
// atomic exchange hands each node's value to exactly one thread.
template <int N>
__global__ void __launch_bounds__(pml_epb<N>() * (N + 1) * (N + 1) * (N + 1)) pml_fixup_kernel(const __grid_constant__ PmlParams p) {
    constexpr int n1 = N + 1, nl = n1 * n1 * n1, EPB = pml_epb<N>();
    const int el = threadIdx.x / nl, t = threadIdx.x - el * nl;
    const int a = t % n1, b = (t / n1) % n1, c = t / (n1 * n1);
    const int k = blockIdx.x * EPB + el;
    if (k >= p.n_el) return;
    const int gx = N * p.elems[3 * k] + a, gy = N * p.elems[3 * k + 1] + b, gz = N * p.elems[3 * k + 2] + c;
    const long long g = ((long long)gz * p.NY + gy) * p.PX + gx;
    SEM_CHECK(gx < p.NX && gy < p.NY && gz < p.NZ);
    const unsigned long long bits = atomicExch(reinterpret_cast<unsigned long long*>(p.da + g), 0ull);
    if (bits) {
        const double v = __longlong_as_double((long long)bits);
        const double dw = p.dt * v;
        if (!SEM_TWO_LEVEL) p.Wn[g] += dw;
        p.Pn[g] = fma(p.dt, dw, p.Pn[g]);
    }
}

void launch_pml_elements(const PmlParams& p, cudaStream_t s) {
    if (p.n_el <= 0) return;
    switch (p.N) {
#define SEM_PML_CASE(n) case n: pml_element_kernel<n><<<(p.n_el + pml_epb<n>() - 1) / pml_epb<n>(), pml_epb<n>() * (n + 1) * (n + 1) * (n + 1), 0, s>>>(p); break;
        SEM_PML_CASE(1) SEM_PML_CASE(2) SEM_PML_CASE(3) SEM_PML_CASE(4)
        SEM_PML_CASE(5) SEM_PML_CASE(6) SEM_PML_CASE(7) SEM_PML_CASE(8)
#undef SEM_PML_CASE
        default: break;
    }
}

// Row-segment sweep of the PML region (one warp per segment, coalesced): w += dt da, p += dt^2 da,
// da = 0.  Each region node lies in exactly one segment, so no atomics are needed.
__global__ void __launch_bounds__(256) pml_fixup_rows_kernel(const __grid_constant__ PmlParams p) {
    const int lane = threadIdx.x & 31;
    const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long sg = wid; sg < p.n_seg; sg += nw) {
        const long long g0 = p.seg_start[sg];
        const int len = p.seg_len[sg];
        SEM_CHECK(g0 >= 0 && len > 0 && len <= p.NX && g0 + len <= p.PX * p.NY * p.NZ);
        // da and p^{n+2} are loaded together (one memory round trip per pass, not two dependent ones)
        for (int i = lane; i < len; i += 32) {
            const long long g = g0 + i;
            const double v = p.da[g];
            const double pn = p.Pn[g];
            if (v != 0.0) {
                const double dw = p.dt * v;
                if (!SEM_TWO_LEVEL) p.Wn[g] += dw;
                p.Pn[g] = fma(p.dt, dw, pn);
                p.da[g] = 0.0;
            }
        }
    }
}

void launch_pml_fixup(const PmlParams& p, cudaStream_t s) {
    if (p.n_el <= 0) return;
    if (p.n_seg > 0) {
        const long long warps = p.n_seg < 148LL * 64 ? p.n_seg : 148LL * 64;
        pml_fixup_rows_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(p);
        return;
    }
    switch (p.N) {
#define SEM_PML_CASE(n) case n: pml_fixup_kernel<n><<<(p.n_el + pml_epb<n>() - 1) / pml_epb<n>(), pml_epb<n>() * (n + 1) * (n + 1) * (n + 1), 0, s>>>(p); break;
        SEM_PML_CASE(1) SEM_PML_CASE(2) SEM_PML_CASE(3) SEM_PML_CASE(4)
        SEM_PML_CASE(5) SEM_PML_CASE(6) SEM_PML_CASE(7) SEM_PML_CASE(8)
#undef SEM_PML_CASE
        default: break;
    }
}

// ------------------------------------------------------------------------------------------------
// Curved boxes (trilinear vertex lattice): element scatter with the metric
// recomputed.  A persistent grid of blocks; a block holds EPB elements and one thread per element
// x-line (b, c), so the x index a of the line's nodes is a compile-time loop index: the x derivative
// and its transpose use compile-time D entries on the line's own registers; the y and z derivatives
// read the other lines from shared memory.  The next element group's lines and vertices are
// prefetched into registers while the current group computes.
//   grad_hat p  ->  flux = w_q c^2 |J| J^-1 J^-T grad_hat p  (adj(J) adj(J)^T / det J, J recomputed
//   from the 8 vertices: dx/dxi is constant along an x-line and dx/deta, dx/dzeta are affine in xi)
//   ->  r_i = sum_q grad_hat phi_i(q) . flux(q)  ->  scatter-add; then a nodal kick-drift.
// ------------------------------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ long long curved_node(const CurvedParams& p, int e, int a, int b, int c) {
    const int ex = e % p.nelx, ey = (e / p.nelx) % p.nely, ez = e / (p.nelx * p.nely);
    return ((long long)(N * ez + c) * p.NY + (N * ey + b)) * p.PX + (N * ex + a);
}

// elements per block: up to 256 threads; dynamic shared memory: two staging buffers of the element
// pressures, two flux arrays, two vertex buffers and D
#ifndef SEM_CV_EPB
#define SEM_CV_EPB 256   // threads per block the element count aims at
#endif
template <int N>
constexpr int curved_epb() {
    constexpr int by_threads = SEM_CV_EPB / ((N + 1) * (N + 1));
    constexpr int by_smem = 100000 / (32 * (N + 1) * (N + 1) * (N + 1) + 384);
    constexpr int e = by_threads < by_smem ? by_threads : by_smem;
    return e > 1 ? e : 1;
}
template <int N>
constexpr int curved_threads() { return curved_epb<N>() * (N + 1) * (N + 1); }
template <int N>
constexpr int curved_smem() { return 8 * (curved_epb<N>() * (4 * (N + 1) * (N + 1) * (N + 1) + 48) + (N + 1) * (N + 1)); }
#ifndef SEM_CV_MINB
#define SEM_CV_MINB 2
#endif
#ifndef SEM_CV_LINES
#define SEM_CV_LINES 1   // y / z derivatives and their transposes by line passes (0: every x-line reads
#endif                   // its y- and z-neighbour lines from shared memory, the round-1 form)


template <int N>
__global__ void __launch_bounds__(curved_threads<N>(), SEM_CV_MINB) curved_residual_kernel(const __grid_constant__ CurvedParams p) {
    constexpr int n1 = N + 1, NL = n1 * n1, nl = n1 * NL, EPB = curved_epb<N>();
    const auto& RT = kRef<N>;
    extern __shared__ __align__(16) double cv_smem[];
    double* const spb = cv_smem;                          // [2][EPB][nl] staged pressures
    double* const sf1 = spb + 2 * EPB * nl;               // [EPB][nl] eta flux
    double* const sf2 = sf1 + EPB * nl;                   // [EPB][nl] zeta flux
    double* const Xvb = sf2 + EPB * nl;                   // [2][EPB][24] vertices
    double* const Ds = Xvb + 2 * EPB * 24;                // [n1][n1]
    const int t = threadIdx.x;
    const int el = t / NL, ln = t - el * NL, b = ln % n1, c = ln / n1;
    const int nel = p.nelx * p.nely * p.nelz;
    const int ngroups = (nel + EPB - 1) / EPB;
    for (int q = t; q < NL; q += blockDim.x) Ds[q] = p.D[q / n1][q % n1];
    const double xb = p.x[b], xc = p.x[c];
    const double wbc = p.w[b] * p.w[c] * p.c2;
    const double ly0 = 0.5 * (1.0 - xb), ly1 = 0.5 * (1.0 + xb);
    const double lz0 = 0.5 * (1.0 - xc), lz1 = 0.5 * (1.0 + xc);
    // stage group g's line of this thread and its element's vertices into buffer k (async)
    auto stage = [&](int g, int k) -> long long {
        const int e = g * EPB + el;
        if (g >= ngroups || e >= nel) return -1;
        if (p.solid && p.solid[e]) return -1;   // obstacle element: no contribution
        const long long g0 = curved_node<N>(p, e, 0, b, c);
        SEM_CHECK(g0 >= 0 && g0 + N < p.PX * p.NY * p.NZ);
        double* dst = spb + (k * EPB + el) * nl + n1 * ln;
#pragma unroll
        for (int a = 0; a <= N; ++a) cp_async8(dst + a, p.P + g0 + a);
        const int ex = e % p.nelx, ey = (e / p.nelx) % p.nely, ez = e / (p.nelx * p.nely);
        for (int q = ln; q < 24; q += NL) {
            const int v = q / 3, i = q - 3 * v;
            const int vx = ex + (v & 1), vy = ey + ((v >> 1) & 1), vz = ez + (v >> 2);
            SEM_CHECK(vx <= p.nelx && vy <= p.nely && vz <= p.nelz);
            cp_async8(Xvb + (k * EPB + el) * 24 + q,
                      p.vlat + 3 * ((size_t)vx + (size_t)(p.nelx + 1) * ((size_t)vy + (size_t)(p.nely + 1) * vz)) + i);
        }
        return g0;
    };
    int gi = blockIdx.x, k = 0;
    long long g0 = stage(gi, 0);
    cp_async_commit();
    for (; gi < ngroups; gi += gridDim.x, k ^= 1) {
        cp_async_wait_all();
        __syncthreads();
        const long long gnext = stage(gi + gridDim.x, k ^ 1);   // overlaps this group's arithmetic
        cp_async_commit();
        const double* sp = spb + (k * EPB + el) * nl;
        const double* Xv = Xvb + (k * EPB + el) * 24;
        double* const f1 = sf1 + el * nl;
        double* const f2 = sf2 + el * nl;
        // ---- reference gradient on the line
        double cur[n1], gx[n1], gy[n1], gz[n1];
#if SEM_CV_LINES
        // y and z derivatives by line passes: thread ln also acts as the y-line (a, c) and the z-line
        // (a, b) with (a, c|b) = (ln % n1, ln / n1); the output index is a compile-time loop index, so the
        // D entries are immediates and each line is read once (6 + 6 loads instead of 36 + 36)
        {
            const int la = ln % n1, lo = ln / n1;
            double vy[n1], vz[n1];
#pragma unroll
            for (int j = 0; j <= N; ++j) {
                vy[j] = sp[la + n1 * (j + n1 * lo)];
                vz[j] = sp[la + n1 * (lo + n1 * j)];
            }
#pragma unroll
            for (int i = 0; i <= N; ++i) {
                double sy = 0.0, sz = 0.0;
#pragma unroll
                for (int j = 0; j <= N; ++j) {
                    sy = fma(RT.D[i][j], vy[j], sy);
                    sz = fma(RT.D[i][j], vz[j], sz);
                }
                f1[la + n1 * (i + n1 * lo)] = sy;
                f2[la + n1 * (lo + n1 * i)] = sz;
            }
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a <= N; ++a) {
            cur[a] = sp[a + n1 * ln];
            gy[a] = f1[a + n1 * ln];
            gz[a] = f2[a + n1 * ln];
        }
#pragma unroll
        for (int a = 0; a <= N; ++a) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j <= N; ++j) s = fma(RT.D[a][j], cur[j], s);
            gx[a] = s;
        }
#else
#pragma unroll
        for (int a = 0; a <= N; ++a) cur[a] = sp[a + n1 * ln];
#pragma unroll
        for (int a = 0; a <= N; ++a) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j <= N; ++j) s = fma(RT.D[a][j], cur[j], s);
            gx[a] = s;
            gy[a] = 0.0;
            gz[a] = 0.0;
        }
#pragma unroll
        for (int j = 0; j <= N; ++j) {
            const double dyj = Ds[b * n1 + j], dzj = Ds[c * n1 + j];
#pragma unroll
            for (int a = 0; a <= N; ++a) {
                gy[a] = fma(dyj, sp[a + n1 * (j + n1 * c)], gy[a]);
                gz[a] = fma(dzj, sp[a + n1 * (b + n1 * j)], gz[a]);
            }
        }
#endif
        // ---- Jacobian pieces of the line: J[:,0] constant, J[:,1] = P1 + xi Q1, J[:,2] = P2 + xi Q2
        double J0[3], P1[3], Q1[3], P2[3], Q2[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double X0 = Xv[i], X1 = Xv[3 + i], X2 = Xv[6 + i], X3 = Xv[9 + i];
            const double X4 = Xv[12 + i], X5 = Xv[15 + i], X6 = Xv[18 + i], X7 = Xv[21 + i];
            // x-edges k = (v1, v2): corners (2k, 2k+1); s_k = mean, h_k = half difference
            const double h0 = 0.5 * (X1 - X0), h1 = 0.5 * (X3 - X2), h2 = 0.5 * (X5 - X4), h3 = 0.5 * (X7 - X6);
            const double s0 = 0.5 * (X1 + X0), s1 = 0.5 * (X3 + X2), s2 = 0.5 * (X5 + X4), s3 = 0.5 * (X7 + X6);
            J0[i] = fma(lz1, fma(ly1, h3, ly0 * h2), lz0 * fma(ly1, h1, ly0 * h0));
            P1[i] = 0.5 * fma(lz1, s3 - s2, lz0 * (s1 - s0));
            Q1[i] = 0.5 * fma(lz1, h3 - h2, lz0 * (h1 - h0));
            P2[i] = 0.5 * fma(ly1, s3 - s1, ly0 * (s2 - s0));
            Q2[i] = 0.5 * fma(ly1, h3 - h1, ly0 * (h2 - h0));
        }
        double f0[n1];   // f1 / f2 overwrite this line's own gy / gz entries (already in registers)
#pragma unroll
        for (int a = 0; a <= N; ++a) {
            const double xa = RT.x[a];
            double J[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                J[i][0] = J0[i];
                J[i][1] = fma(xa, Q1[i], P1[i]);
                J[i][2] = fma(xa, Q2[i], P2[i]);
            }
            // adj = det J^-1 (rows: cofactors); |J| J^-1 J^-T = adj adj^T / det
            double A[3][3];
            A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
            A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
            A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
            A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
            A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
            A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
            A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
            A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
            A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
            const double det = J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
            const double sc = RT.w[a] * wbc / det;
            double u[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) u[i] = A[0][i] * gx[a] + A[1][i] * gy[a] + A[2][i] * gz[a];   // A^T gh
            f0[a] = sc * (A[0][0] * u[0] + A[0][1] * u[1] + A[0][2] * u[2]);
            f1[a + n1 * ln] = sc * (A[1][0] * u[0] + A[1][1] * u[1] + A[1][2] * u[2]);
            f2[a + n1 * ln] = sc * (A[2][0] * u[0] + A[2][1] * u[1] + A[2][2] * u[2]);
        }
        __syncthreads();
        // ---- D^T: x part on the line's registers, y and z parts from the other lines
        double r[n1];
#pragma unroll
        for (int a = 0; a <= N; ++a) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j <= N; ++j) s = fma(RT.D[j][a], f0[j], s);
            r[a] = s;
        }
#if SEM_CV_LINES
        // D^T along y and z by the same line passes, in place (a line's entries are read by its own
        // thread only), then the x-line adds its two entries
        {
            const int la = ln % n1, lo = ln / n1;
            double vy[n1], vz[n1];
#pragma unroll
            for (int j = 0; j <= N; ++j) {
                vy[j] = f1[la + n1 * (j + n1 * lo)];
                vz[j] = f2[la + n1 * (lo + n1 * j)];
            }
#pragma unroll
            for (int i = 0; i <= N; ++i) {
                double sy = 0.0, sz = 0.0;
#pragma unroll
                for (int j = 0; j <= N; ++j) {
                    sy = fma(RT.D[j][i], vy[j], sy);
                    sz = fma(RT.D[j][i], vz[j], sz);
                }
                f1[la + n1 * (i + n1 * lo)] = sy;
                f2[la + n1 * (lo + n1 * i)] = sz;
            }
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a <= N; ++a) r[a] += f1[a + n1 * ln] + f2[a + n1 * ln];
#else
#pragma unroll
        for (int j = 0; j <= N; ++j) {
            const double dyj = Ds[j * n1 + b], dzj = Ds[j * n1 + c];
#pragma unroll
            for (int a = 0; a <= N; ++a) {
                r[a] = fma(dyj, f1[a + n1 * (j + n1 * c)], r[a]);
                r[a] = fma(dzj, f2[a + n1 * (b + n1 * j)], r[a]);
            }
        }
#endif
        if (g0 >= 0) {
#pragma unroll
            for (int a = 0; a <= N; ++a) atomicAdd(p.res + g0 + a, r[a]);
        }
        g0 = gnext;
    }
    cp_async_wait_all();
}

static int device_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms < 1) sms = 1;
    }
    return sms;
}

int curved_grid(int N, int nel) {
    static int per_sm[kMaxN + 1] = {};
    const int sms = device_sms();
    if (N < 1 || N > kMaxN) return 1;
    int epb = 1;
    switch (N) {
#define SEM_CV_OCC(n)                                                                                      \
    case n:                                                                                                \
        epb = curved_epb<n>();                                                                             \
        if (!per_sm[n]) {                                                                                  \
            cudaFuncSetAttribute(curved_residual_kernel<n>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                 curved_smem<n>());                                                         \
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[n], curved_residual_kernel<n>,             \
                                                          curved_threads<n>(), curved_smem<n>());           \
        }                                                                                                  \
        break;
        SEM_CV_OCC(1) SEM_CV_OCC(2) SEM_CV_OCC(3) SEM_CV_OCC(4)
        SEM_CV_OCC(5) SEM_CV_OCC(6) SEM_CV_OCC(7) SEM_CV_OCC(8)
#undef SEM_CV_OCC
        default: break;
    }
    if (per_sm[N] < 1) per_sm[N] = 1;
    const long long groups = ((long long)nel + epb - 1) / epb;
    const long long g = (long long)sms * per_sm[N];
    return (int)(g < groups ? g : (groups > 0 ? groups : 1));
}

// b_j(t) = pwf_j s'(tau_j - t0), s(u) = exp(-u^2 / (2 sigma^2)) sin(om u), tau_j = t - pwd_j (reading R13)
__device__ __forceinline__ double curved_pw_load(const CurvedParams& p, double t1, long long j) {
    const double u = t1 - __ldg(p.pwd + j) - p.pw_t0;
    double sn, cs;
    sincos(p.pw_om * u, &sn, &cs);
    return __ldg(p.pwf + j) * (exp(-0.5 * u * u * p.pw_is2) * (-u * p.pw_is2 * sn + p.pw_om * cs));
}

// Incident plane wave on a curved box's top plane: res_j -= b_j(t^{n+1}) before the nodal update (a kernel
// of its own: inside curved_update_kernel the sincos / exp path doubled that kernel's spills under its
// 32-register cap and cost 4% of the curved step)
__global__ void __launch_bounds__(256) curved_pw_kernel(const __grid_constant__ CurvedParams p) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.NX * p.NY) return;
    const double t1 = (double)(__ldcg(p.step) + 1) * p.dt;
    const long long ix = j % p.NX, iy = j / p.NX;
    p.res[(p.NY * (p.NZ - 1) + iy) * p.PX + ix] -= curved_pw_load(p, t1, j);
}

// Nodal kick-drift of a curved box as one flat stream over the padded lattice (16-byte accesses,
// grid-stride over 8 resident blocks per SM -- the register cap keeps all of them resident, a second
// wave of blocks would double the time): pad entries carry minv = cdamp = res = 0 and w = p = 0.
__global__ void __launch_bounds__(256, 8) curved_update_kernel(const __grid_constant__ CurvedParams p) {
    const long long n2 = p.PX * p.NY * p.NZ / 2;   // PX is a multiple of 8
    const double2* __restrict__ W2 = reinterpret_cast<const double2*>(p.W);
    const double2* __restrict__ M2 = reinterpret_cast<const double2*>(p.minv);
    const double2* __restrict__ R2 = reinterpret_cast<const double2*>(p.res);
    const double2* __restrict__ C2 = reinterpret_cast<const double2*>(p.cdamp);
    const double2* __restrict__ P2 = reinterpret_cast<const double2*>(p.P);
#pragma unroll 1
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
        // read-only (non-coherent) loads: each element is read once, before this thread overwrites it
#if SEM_TWO_LEVEL   // w^n = (p^{n+1} - p^n) / dt; p^n is read here and overwritten by p^{n+2} below
        const double2 mi = __ldg(M2 + i), cd = __ldg(C2 + i), pv = __ldg(P2 + i);
        const double2 po = reinterpret_cast<const double2*>(p.Pn)[i];
        const double2 wv = make_double2((pv.x - po.x) * p.inv_dt, (pv.y - po.y) * p.inv_dt);
        (void)W2;
#else
        const double2 wv = __ldg(W2 + i), mi = __ldg(M2 + i), cd = __ldg(C2 + i), pv = __ldg(P2 + i);
#endif
        double2 r = __ldg(R2 + i);
        if (p.F && 2 * i < p.PX * p.NY) {   // z = 0 plane: PMUT forcing f = kappa B^T qdd (Eq. 11)
            const long long d = 2 * i, ix = d % p.PX, iy = d / p.PX;   // PX even: both nodes on one row
            if (ix < p.NX) r.x -= __ldg(p.F + iy * p.NX + ix) * __ldg(p.fmx + ix) * __ldg(p.fmy + iy);
            if (ix + 1 < p.NX) r.y -= __ldg(p.F + iy * p.NX + ix + 1) * __ldg(p.fmx + ix + 1) * __ldg(p.fmy + iy);
        }
        double2 wn, pn;
        wn.x = fma(p.dt, -mi.x * r.x - cd.x * wv.x, wv.x);
        wn.y = fma(p.dt, -mi.y * r.y - cd.y * wv.y, wv.y);
        pn.x = fma(p.dt, wn.x, pv.x);
        pn.y = fma(p.dt, wn.y, pv.y);
        // nodes of no fluid element (obstacle interiors, lattice padding) have M^-1 = 0: held at 0
        if (mi.x == 0.0) wn.x = pn.x = 0.0;
        if (mi.y == 0.0) wn.y = pn.y = 0.0;
        reinterpret_cast<double2*>(p.res)[i] = make_double2(0.0, 0.0);
        if (!SEM_TWO_LEVEL) reinterpret_cast<double2*>(p.W)[i] = wn;
        reinterpret_cast<double2*>(p.Pn)[i] = pn;
    }
}


void launch_curved(const CurvedParams& p, cudaStream_t s) {
    switch (p.N) {
#define SEM_CV_CASE(n) case n: curved_residual_kernel<n><<<p.grid, curved_threads<n>(), curved_smem<n>(), s>>>(p); break;
        SEM_CV_CASE(1) SEM_CV_CASE(2) SEM_CV_CASE(3) SEM_CV_CASE(4)
        SEM_CV_CASE(5) SEM_CV_CASE(6) SEM_CV_CASE(7) SEM_CV_CASE(8)
#undef SEM_CV_CASE
        default: break;
    }
    if (p.pwd) curved_pw_kernel<<<(unsigned)((p.NX * p.NY + 255) / 256), 256, 0, s>>>(p);
    const long long n2 = p.PX * p.NY * p.NZ / 2;
    const long long want = (n2 + 255) / 256, cap = 8LL * device_sms();
    curved_update_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(p);
}

// ------------------------------------------------------------------------------------------------
// General non-conforming SIPG interface (curved boxes, lattices that need not
// nest): one thread per fine-face quadrature point x_q (a fine face GLL node, reading R9), the owner
// coarse element and x_hat^- from Algorithm 3 (setup).  With J = p+ - p-(x_hat^-), A = 1/2 (c+^2 d_n p+
// + c-^2 d_n p-) (n = n+ on both sides), T = W (gamma J - A), S = -1/2 W J, the rows of the face matrix
// of Eq. 7 (the oracle's K_F) give
//   fine i:   r_i += T phi_i(x_q) + c+^2 S d_n phi_i(x_q)      (collocated: phi_i(x_q) = delta)
//   coarse i: r_i += -T phi_i(x_hat^-) + c-^2 S d_n phi_i(x_hat^-)
// with d_n phi = (J^-1 n) . grad_hat phi; added to the boxes' assembled residuals with FP64 atomics.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) iface_general_kernel(const __grid_constant__ GIfaceParams p) {
    const long long qp = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (qp >= p.nqp) return;
    const int Nf = p.Nf, Nc = p.Nc, q1 = Nf + 1, c1 = Nc + 1;
    const int q = (int)(qp % (q1 * q1)), a = q % q1, b = q / q1;
    const long long SF = p.PXf * p.NYf, SC = p.PXc * p.NYc;
    const long long fb = p.fbase[qp] + a + b * p.PXf + Nf * SF;   // fine node (a, b, Nf)
    SEM_CHECK(p.fbase[qp] >= 0 && fb < SF * (p.NZf_dbg > 0 ? p.NZf_dbg : 1) && p.cbase[qp] >= 0);
    const double pp = __ldg(p.Pf + fb);
    double dxi = 0.0, deta = 0.0, dzeta = 0.0;
    for (int j = 0; j <= Nf; ++j) {
        dxi = fma(p.Df[a][j], __ldg(p.Pf + fb + (j - a)), dxi);
        deta = fma(p.Df[b][j], __ldg(p.Pf + fb + (long long)(j - b) * p.PXf), deta);
        dzeta = fma(p.Df[Nf][j], __ldg(p.Pf + fb + (long long)(j - Nf) * SF), dzeta);
    }
    const double* G = p.geo + qp * 7;
    const double W = __ldg(G), gp0 = __ldg(G + 1), gp1 = __ldg(G + 2), gp2 = __ldg(G + 3);
    const double gm0 = __ldg(G + 4), gm1 = __ldg(G + 5), gm2 = __ldg(G + 6);
    const double dnp = gp0 * dxi + gp1 * deta + gp2 * dzeta;
    const double* B = p.bas + qp * 6 * c1;   // lx, dlx, ly, dly, lz, dlz
    const long long cb = p.cbase[qp];
    double pm = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int c = 0; c <= Nc; ++c)
        for (int bb = 0; bb <= Nc; ++bb) {
            const double ly = __ldg(B + 2 * c1 + bb), dly = __ldg(B + 3 * c1 + bb);
            const double lz = __ldg(B + 4 * c1 + c), dlz = __ldg(B + 5 * c1 + c);
            for (int aa = 0; aa <= Nc; ++aa) {
                const double v = __ldg(p.Pc + cb + aa + (long long)bb * p.PXc + (long long)c * SC);
                const double lx = __ldg(B + aa), dlx = __ldg(B + c1 + aa);
                pm = fma(lx * ly * lz, v, pm);
                gx = fma(dlx * ly * lz, v, gx);
                gy = fma(lx * dly * lz, v, gy);
                gz = fma(lx * ly * dlz, v, gz);
            }
        }
    const double dnm = gm0 * gx + gm1 * gy + gm2 * gz;
    const double J = pp - pm;
    const double A = 0.5 * (p.cf2 * dnp + p.cc2 * dnm);
    const double T = W * (p.gamma * J - A), S = -0.5 * W * J;
    atomicAdd(p.resF + fb, T);
    const double sF = p.cf2 * S;
    for (int j = 0; j <= Nf; ++j) {
        atomicAdd(p.resF + fb + (j - a), sF * gp0 * p.Df[a][j]);
        atomicAdd(p.resF + fb + (long long)(j - b) * p.PXf, sF * gp1 * p.Df[b][j]);
        atomicAdd(p.resF + fb + (long long)(j - Nf) * SF, sF * gp2 * p.Df[Nf][j]);
    }
    const double sC = p.cc2 * S;
    for (int c = 0; c <= Nc; ++c)
        for (int bb = 0; bb <= Nc; ++bb) {
            const double ly = __ldg(B + 2 * c1 + bb), dly = __ldg(B + 3 * c1 + bb);
            const double lz = __ldg(B + 4 * c1 + c), dlz = __ldg(B + 5 * c1 + c);
            for (int aa = 0; aa <= Nc; ++aa) {
                const double lx = __ldg(B + aa), dlx = __ldg(B + c1 + aa);
                const double v = -T * lx * ly * lz + sC * (gm0 * dlx * ly * lz + gm1 * lx * dly * lz + gm2 * lx * ly * dlz);
                atomicAdd(p.resC + cb + aa + (long long)bb * p.PXc + (long long)c * SC, v);
            }
        }
}

void launch_iface_general(const GIfaceParams& p, cudaStream_t s) {
    if (p.nqp > 0) iface_general_kernel<<<(unsigned)((p.nqp + 127) / 128), 128, 0, s>>>(p);
}

__global__ void step_bump_kernel(long long* step) { *step += 1; }

void launch_step_bump(long long* step, cudaStream_t s) { step_bump_kernel<<<1, 1, 0, s>>>(step); }

__global__ void set_state_kernel(const double* pprev, double* pcur, const double* w, long long NX, long long PX,
                                 long long rows, double dt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= NX * rows) return;
    const long long d = (i / NX) * PX + i % NX;
    pcur[d] = pprev[d] + dt * w[d];
}

void launch_set_state(const double* pprev, double* pcur, const double* w, long long NX, long long PX, long long rows,
                      double dt, cudaStream_t s) {
    const long long n = NX * rows;
    set_state_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pprev, pcur, w, NX, PX, rows, dt);
}

// Obstacle boxes: nodes of no fluid element (M^-1 = 0) are held at 0 (include/sem.h)
__global__ void zero_inactive_kernel(double* p0, double* p1, double* w, const double* minv, long long NX, long long PX,
                                     long long rows) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= NX * rows) return;
    const long long d = (i / NX) * PX + i % NX;
    if (minv[d] == 0.0) p0[d] = p1[d] = w[d] = 0.0;
}

void launch_zero_inactive(double* p0, double* p1, double* w, const double* minv, long long NX, long long PX,
                          long long rows, cudaStream_t s) {
    const long long n = NX * rows;
    zero_inactive_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p0, p1, w, minv, NX, PX, rows);
}

__global__ void gather_kernel(const double* src, const long long* idx, long long n, double* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}

void launch_gather(const double* src, const long long* idx, long long n, double* out, cudaStream_t s) {
    gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, idx, n, out);
}

__global__ void nonfinite_kernel(const double* p, long long NX, long long PX, long long rows, unsigned long long* flag) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    bool bad = false;
    for (; i < NX * rows; i += stride) bad |= !isfinite(p[(i / NX) * PX + i % NX]);
    if (bad) atomicOr(flag, 1ull);
}

void launch_nonfinite(const double* p, long long NX, long long PX, long long rows, unsigned long long* flag,
                      cudaStream_t s) {
    nonfinite_kernel<<<148 * 8, 256, 0, s>>>(p, NX, PX, rows, flag);
}

}  // namespace sem
