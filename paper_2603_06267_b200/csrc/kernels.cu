// sm_100a FP64 kernels of one leapfrog step (Algorithm 1) of the DG-SEM / PMUT model.
//
//  vol_kernel     volume stiffness (Eq. 7 first sum) in 1D-stiffness sum-factorised form on affine
//                 GLL elements, CG assembly in registers/shared memory (owner computes), fused with
//                 ABC (Eq. 8), PMUT forcing (Eq. 11), the SIPG layer terms and the kick-drift update.
//                 One CTA = 32 x TY node columns marching over z: the z-stencil lives in a register
//                 window, the x/y stencils read one shared-memory plane (with an N-node halo).
//  modal_kernel   one warp per PMUT: pressure projection (Eq. 12), modal predictor/solve/corrector
//                 (Eq. 10), force plane f = kappa B^T qdd (Eq. 11).
//  iface_*        SIPG flux of Eq. 7 on the 2:1 non-conforming face on the fine-face GLL lattice.
// See DESIGN.md for the derivation of every coefficient and the byte budget of each kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sem_internal.h"

namespace sem {

// ------------------------------------------------------------------------------------------------
// Volume + update kernel
// ------------------------------------------------------------------------------------------------
template <int N, int TY>
__global__ void __launch_bounds__(kTX* TY) vol_kernel(const __grid_constant__ VolParams p) {
    constexpr int SW = kTX + 2 * N;         // shared plane pitch (doubles)
    constexpr int SH = TY + 2 * N;
    constexpr int NT = kTX * TY;
    constexpr int HX = 2 * N * TY;          // x-halo cells per plane
    constexpr int H = HX + 2 * N * kTX;     // + y-halo cells
    constexpr int HPT = (H + NT - 1) / NT;  // halo cells per thread
    __shared__ double sbuf[2][SH * SW];

    const BoxTables& T = p.tab;
    const int lx = threadIdx.x, ly = threadIdx.y, tid = ly * kTX + lx;
    const long long NX = p.NX, NY = p.NY, NZ = p.NZ;
    const long long tx0 = (long long)blockIdx.x * kTX, ty0 = (long long)blockIdx.y * TY;
    const long long ix = tx0 + lx, iy = ty0 + ly;
    const bool valid = ix < NX && iy < NY;
    const long long S = NX * NY;
    const long long col = valid ? iy * NX + ix : 0;

    // ---- 1D row coefficients of this thread's x / y position (see sem_internal.h) ----
    int ax = 0, ay = 0;
    bool hxR = false, hxL = false, hyR = false, hyL = false;
    int rxR = 0, ryR = 0;
    if (valid) {
        if (ix == 0) { rxR = row_B0(N); hxR = true; }
        else if (ix == NX - 1) { hxL = true; }
        else { ax = (int)(ix % N); rxR = ax; hxR = true; hxL = (ax == 0); }
        if (iy == 0) { ryR = row_B0(N); hyR = true; }
        else if (iy == NY - 1) { hyL = true; }
        else { ay = (int)(iy % N); ryR = ay; hyR = true; hyL = (ay == 0); }
    }
    const int rxL = (ix == NX - 1) ? row_BN(N) : row_L(N);
    const int ryL = (iy == NY - 1) ? row_BN(N) : row_L(N);
    double cxR[N + 1], cxL[N + 1], cyR[N + 1], cyL[N + 1];
#pragma unroll
    for (int b = 0; b <= N; ++b) {
        cxR[b] = hxR ? T.G[0][rxR][b] : 0.0;
        cxL[b] = hxL ? T.G[0][rxL][b] : 0.0;
        cyR[b] = hyR ? T.G[1][ryR][b] : 0.0;
        cyL[b] = hyL ? T.G[1][ryL][b] : 0.0;
    }
    const int own = (ly + N) * SW + lx + N;
    const int bRx = own - ax, bLx = (ly + N) * SW + lx;
    const int bRy = (ly + N - ay) * SW + lx + N, bLy = ly * SW + lx + N;

    double dxy = 0.0;
    if (valid) {
        if (ix == 0) dxy += p.damp[0];
        if (ix == NX - 1) dxy += p.damp[1];
        if (iy == 0) dxy += p.damp[2];
        if (iy == NY - 1) dxy += p.damp[3];
    }

    // ---- halo slots ----
    int hs[HPT];
    long long hg[HPT];
#pragma unroll
    for (int k = 0; k < HPT; ++k) {
        const int h = tid + k * NT;
        hs[k] = -1;
        hg[k] = -1;
        if (h < H) {
            long long gx, gy;
            int sx, sy;
            if (h < HX) {
                const int side = h / (N * TY), rem = h % (N * TY), r = rem / N, c = rem % N;
                sy = r + N;
                sx = side ? kTX + N + c : c;
                gx = side ? tx0 + kTX + c : tx0 - N + c;
                gy = ty0 + r;
            } else {
                const int hh = h - HX, side = hh / (N * kTX), rem = hh % (N * kTX), r = rem / kTX,
                          c = rem % kTX;
                sy = side ? TY + N + r : r;
                sx = c + N;
                gx = tx0 + c;
                gy = side ? ty0 + TY + r : ty0 - N + r;
            }
            hs[k] = sy * SW + sx;
            if (gx >= 0 && gx < NX && gy >= 0 && gy < NY) hg[k] = gy * NX + gx;
        }
    }

    // ---- per-column extras ----
    const long long n = __ldcg(p.step);
    const double t1 = (double)(n + 1) * p.dt;
    const double fv = (p.F != nullptr && valid) ? p.F[col] : 0.0;
    double tauv = 0.0, sigv = 0.0;
    if (p.iface_side != 0 && valid) { tauv = p.tau[col]; sigv = p.sig[col]; }
    double pw_x = 0.0, pw_y = 0.0;
    if (p.pw_on && valid) { pw_x = p.xc[ix]; pw_y = p.yc[iy]; }

    const double* __restrict__ P = p.P;
    double zw[2 * N + 1];
#pragma unroll
    for (int k = 0; k <= 2 * N; ++k) {
        const long long pl = k - N;
        zw[k] = (valid && pl >= 0 && pl < NZ) ? __ldg(P + col + pl * S) : 0.0;
    }
    double hv[HPT];
#pragma unroll
    for (int k = 0; k < HPT; ++k) hv[k] = (hg[k] >= 0) ? __ldg(P + hg[k]) : 0.0;
    double wpre = valid ? __ldcs(p.W + col) : 0.0;

    const int nelz = p.nelz;
    for (int ez = 0; ez < nelz; ++ez) {
        const long long z0 = (long long)N * ez;
        const bool last = (ez == nelz - 1);
        double nxt[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const long long pl = z0 + N + 1 + j;
            nxt[j] = (valid && pl < NZ) ? __ldg(P + col + pl * S) : 0.0;
        }
#pragma unroll
        for (int c = 0; c <= N; ++c) {
            if (c == N && !last) break;
            const long long iz = z0 + c;
            double* sb = sbuf[iz & 1];
            const double v = zw[N + c];
            sb[own] = v;
#pragma unroll
            for (int k = 0; k < HPT; ++k)
                if (hs[k] >= 0) sb[hs[k]] = hv[k];
            const double wv = wpre;
            if (iz + 1 < NZ) {
#pragma unroll
                for (int k = 0; k < HPT; ++k) hv[k] = (hg[k] >= 0) ? __ldg(P + hg[k] + (iz + 1) * S) : 0.0;
                wpre = valid ? __ldcs(p.W + col + (iz + 1) * S) : 0.0;
            }
            __syncthreads();

            // z: register window (compile-time rows)
            double zp = 0.0;
            if (c == N) {
#pragma unroll
                for (int b = 0; b <= N; ++b) zp = fma(T.G[2][row_BN(N)][b], zw[N + b], zp);
            } else if (c == 0) {
                if (ez == 0) {
#pragma unroll
                    for (int b = 0; b <= N; ++b) zp = fma(T.G[2][row_B0(N)][b], zw[N + b], zp);
                } else {
#pragma unroll
                    for (int b = 0; b <= N; ++b) zp = fma(T.G[2][0][b], zw[N + b], zp);
#pragma unroll
                    for (int b = 0; b <= N; ++b) zp = fma(T.G[2][row_L(N)][b], zw[b], zp);
                }
            } else {
#pragma unroll
                for (int b = 0; b <= N; ++b) zp = fma(T.G[2][c][b], zw[N + b], zp);
            }
            // x, y: shared plane
            double xp = 0.0, yp = 0.0;
            if (hxR) {
#pragma unroll
                for (int b = 0; b <= N; ++b) xp = fma(cxR[b], sb[bRx + b], xp);
            }
            if (hxL) {
#pragma unroll
                for (int b = 0; b <= N; ++b) xp = fma(cxL[b], sb[bLx + b], xp);
            }
            if (hyR) {
#pragma unroll
                for (int b = 0; b <= N; ++b) yp = fma(cyR[b], sb[bRy + b * SW], yp);
            }
            if (hyL) {
#pragma unroll
                for (int b = 0; b <= N; ++b) yp = fma(cyL[b], sb[bLy + b * SW], yp);
            }
            double a = -(xp + yp + zp);
            double damp = dxy;
            if (iz == 0) damp += p.damp[4];
            if (iz == NZ - 1) damp += p.damp[5];
            a -= damp * wv;
            if (iz == 0) a += p.kF * fv;
            if (p.iface_side > 0 && iz >= NZ - 1 - N) {
                const int cc = (int)(iz - (NZ - 1 - N));
                a -= tauv * T.ktau[cc] + sigv * T.ksig[cc];
            } else if (p.iface_side < 0 && iz <= N) {
                const int cc = (int)iz;
                a -= tauv * T.ktau[cc] + sigv * T.ksig[cc];
            }
            if (p.pw_on && iz == NZ - 1) {
                const double tau = t1 - (p.pw_k[0] * (pw_x - p.pw_xref[0]) + p.pw_k[1] * (pw_y - p.pw_xref[1]) +
                                         p.pw_k[2] * (p.pw_ztop - p.pw_xref[2])) / p.pw_c;
                const double u = tau - p.pw_t0;
                const double is2 = 1.0 / (p.pw_sigma * p.pw_sigma);
                double sn, cs;
                sincos(p.pw_om * u, &sn, &cs);
                const double ds = exp(-0.5 * u * u * is2) * (-u * is2 * sn + p.pw_om * cs);
                a += p.pw_fac * ds;
            }
            const double wn = fma(p.dt, a, wv);
            const double pn = fma(p.dt, wn, v);
            if (valid) {
                __stcs(p.W + col + iz * S, wn);
                __stcs(p.Pn + col + iz * S, pn);
            }
        }
#pragma unroll
        for (int k = 0; k <= N; ++k) zw[k] = zw[k + N];
#pragma unroll
        for (int j = 0; j < N; ++j) zw[N + 1 + j] = nxt[j];
    }

    if (p.bump_step) {
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            const unsigned prev = atomicAdd(p.done, 1u);
            if (prev == p.total_blocks - 1) {
                *p.step = n + 1;
                *p.done = 0u;
                __threadfence();
            }
        }
    }
}

template <int N>
static void launch_vol_N(const VolParams& p, cudaStream_t s) {
    constexpr int TY = 8;
    dim3 blk(kTX, TY);
    dim3 grd((unsigned)((p.NX + kTX - 1) / kTX), (unsigned)((p.NY + TY - 1) / TY));
    vol_kernel<N, TY><<<grd, blk, 0, s>>>(p);
}

void launch_volume(const VolParams& p, int N, cudaStream_t s) {
    switch (N) {
        case 1: launch_vol_N<1>(p, s); break;
        case 2: launch_vol_N<2>(p, s); break;
        case 3: launch_vol_N<3>(p, s); break;
        case 4: launch_vol_N<4>(p, s); break;
        case 5: launch_vol_N<5>(p, s); break;
        case 6: launch_vol_N<6>(p, s); break;
        case 7: launch_vol_N<7>(p, s); break;
        case 8: launch_vol_N<8>(p, s); break;
        default: break;
    }
}

unsigned volume_blocks(long long NX, long long NY) {
    return (unsigned)(((NX + kTX - 1) / kTX) * ((NY + 8 - 1) / 8));
}

// ------------------------------------------------------------------------------------------------
// Modal kernel: one warp per PMUT
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double drive_tx(const ModalParams& p, double tp) {
    if (tp < 0.0 || tp > p.t_end) return 0.0;
    return p.amp * sin(p.om0 * tp) * 0.5 * (1.0 - cos(p.om0 * tp / p.ncyc));
}

__global__ void __launch_bounds__(128) modal_kernel(const ModalParams p) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (k >= p.n_pmut) return;
    const unsigned FULL = 0xffffffffu;
    const int M = p.n_modes;
    const long long n = __ldcg(p.step);
    const double dt = p.dt;
    const double t1 = (double)(n + 1) * dt, t0 = (double)n * dt;
    const int i0 = p.rect[4 * k], j0 = p.rect[4 * k + 1], ni = p.rect[4 * k + 2], nj = p.rect[4 * k + 3];
    const int L = p.lmax;
    const double* sxk = p.sx + (size_t)k * M * L;
    const double* syk = p.sy + (size_t)k * M * L;
    const double* wxk = p.wx + (size_t)k * L;
    const double* wyk = p.wy + (size_t)k * L;

    // pressure projection G_m = sum_ij m_x(i) S_x(i) m_y(j) S_y(j) p_ij   (Eq. 12: int p U.n = -G)
    double acc[kMaxModes];
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) acc[m] = 0.0;
    for (int ib = 0; ib < ni; ib += 32) {
        const int i = ib + lane;
        const bool on = i < ni;
        double bx[kMaxModes];
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m) bx[m] = (on && m < M) ? wxk[i] * sxk[m * L + i] : 0.0;
        for (int j = 0; j < nj; ++j) {
            const double val = on ? p.P[(long long)(j0 + j) * p.NX + i0 + i] : 0.0;
            const double wj = wyk[j];
#pragma unroll
            for (int m = 0; m < kMaxModes; ++m)
                if (m < M) acc[m] = fma(bx[m] * val, wj * syk[m * L + j], acc[m]);
        }
    }
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[m] += __shfl_xor_sync(FULL, acc[m], o);
    }
    double G = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m)
        if (lane == m) G = acc[m];

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
    double qv[kMaxModes];
#pragma unroll
    for (int m = 0; m < kMaxModes; ++m) qv[m] = __shfl_sync(FULL, qdd1, m);
    // force plane F = kappa sum_m qdd_m S_m  (Eq. 11; the 1/M factor is applied in vol_kernel)
    for (int j = 0; j < nj; ++j) {
        for (int ib = 0; ib < ni; ib += 32) {
            const int i = ib + lane;
            if (i < ni) {
                double f = 0.0;
#pragma unroll
                for (int m = 0; m < kMaxModes; ++m)
                    if (m < M) f = fma(qv[m], sxk[m * L + i] * syk[m * L + j], f);
                p.F[(long long)(j0 + j) * p.NX + i0 + i] = p.kappa * f;
            }
        }
    }
}

void launch_modal(const ModalParams& p, cudaStream_t s) {
    modal_kernel<<<(p.n_pmut + 3) / 4, 128, 0, s>>>(p);
}

// ------------------------------------------------------------------------------------------------
// Interface (SIPG, Eq. 7) on the 2:1 face, fine-face GLL lattice as quadrature (reading R9)
// ------------------------------------------------------------------------------------------------
__global__ void iface_coarse_trace(const IfaceParams p) {
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = p.NXc * p.NYc;
    if (id >= n) return;
    const long long S = n;
    double d = 0.0;
    for (int c = 0; c <= p.Nc; ++c) d = fma(p.dcB[c], p.Pc[id + c * S], d);
    p.trc[id] = p.Pc[id];
    p.drc[id] = d;
}

__device__ __forceinline__ void coarse_locate(long long i, int NfR, int nelc, int Nc, long long& base, int& q) {
    long long e = i / NfR;
    if (e > nelc - 1) e = nelc - 1;
    q = (int)(i - e * NfR);
    base = e * Nc;
}

__global__ void iface_fine(const IfaceParams p) {
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = p.NXf * p.NYf;
    if (id >= n) return;
    const long long ix = id % p.NXf, iy = id / p.NXf;
    const long long S = n;
    const long long top = (p.NZf - 1) * S;
    const int Nf = p.Nf, Nc = p.Nc, NfR = p.Nf * p.R, Nc1 = Nc + 1;
    // fine trace and normal derivative (n+ = +e_z)
    const double pp = p.Pf[top + id];
    double dpp = 0.0;
    for (int c = 0; c <= Nf; ++c) dpp = fma(p.dfT[c], p.Pf[top - (Nf - c) * S + id], dpp);
    // coarse trace / derivative interpolated to x_q
    long long bx, by;
    int qx, qy;
    coarse_locate(ix, NfR, p.nelcx, Nc, bx, qx);
    coarse_locate(iy, NfR, p.nelcy, Nc, by, qy);
    double pm = 0.0, dpm = 0.0;
    for (int b = 0; b <= Nc; ++b) {
        const double wy = p.I[qy * Nc1 + b];
        double rt = 0.0, rd = 0.0;
        for (int a = 0; a <= Nc; ++a) {
            const double wx = p.I[qx * Nc1 + a];
            const long long cid = (by + b) * p.NXc + bx + a;
            rt = fma(wx, p.trc[cid], rt);
            rd = fma(wx, p.drc[cid], rd);
        }
        pm = fma(wy, rt, pm);
        dpm = fma(wy, rd, dpm);
    }
    const double J = pp - pm;                              // [[p]].n+
    const double A = 0.5 * (p.cf2 * dpp + p.cc2 * dpm);     // {c^2 grad p}.n+
    const double Wq = p.mxf[ix] * p.myf[iy];                // assembled fine-face weights
    p.tauf[id] = p.gamma * J - A;
    p.sigf[id] = -0.5 * p.cf2 * J;
    p.g1[id] = Wq * (A - p.gamma * J);
    p.g2[id] = Wq * (-0.5 * p.cc2 * J);
}

// transposed interpolation along one lattice direction: out(j) = sum_i psi_j(x_i) in(i)
__device__ __forceinline__ void gather_range(long long j, int Nc, int NfR, int nelc, long long nf, long long& lo,
                                             long long& hi) {
    const long long e = j / Nc;
    const int b = (int)(j - e * Nc);
    lo = (b == 0 && e > 0) ? (e - 1) * NfR : e * NfR;
    hi = (e + 1) * NfR;
    if (hi > nf - 1) hi = nf - 1;
    if (lo > nf - 1) lo = nf - 1;
}

__device__ __forceinline__ double gather_weight(const IfaceParams& p, long long i, long long j, int NfR, int nelc) {
    long long e = i / NfR;
    if (e > nelc - 1) e = nelc - 1;
    const int q = (int)(i - e * NfR);
    const long long b = j - e * p.Nc;
    if (b < 0 || b > p.Nc) return 0.0;
    return p.I[q * (p.Nc + 1) + b];
}

__global__ void iface_gather_y(const IfaceParams p) {
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = p.NXf * p.NYc;
    if (id >= n) return;
    const long long ix = id % p.NXf, jy = id / p.NXf;
    const int NfR = p.Nf * p.R;
    long long lo, hi;
    gather_range(jy, p.Nc, NfR, p.nelcy, p.NYf, lo, hi);
    double s1 = 0.0, s2 = 0.0;
    for (long long iy = lo; iy <= hi; ++iy) {
        const double w = gather_weight(p, iy, jy, NfR, p.nelcy);
        s1 = fma(w, p.g1[iy * p.NXf + ix], s1);
        s2 = fma(w, p.g2[iy * p.NXf + ix], s2);
    }
    p.h1[id] = s1;
    p.h2[id] = s2;
}

__global__ void iface_gather_x(const IfaceParams p) {
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = p.NXc * p.NYc;
    if (id >= n) return;
    const long long jx = id % p.NXc, jy = id / p.NXc;
    const int NfR = p.Nf * p.R;
    long long lo, hi;
    gather_range(jx, p.Nc, NfR, p.nelcx, p.NXf, lo, hi);
    double s1 = 0.0, s2 = 0.0;
    for (long long ix = lo; ix <= hi; ++ix) {
        const double w = gather_weight(p, ix, jx, NfR, p.nelcx);
        s1 = fma(w, p.h1[jy * p.NXf + ix], s1);
        s2 = fma(w, p.h2[jy * p.NXf + ix], s2);
    }
    const double inv = 1.0 / (p.mxc[jx] * p.myc[jy]);
    p.tauc[id] = s1 * inv;
    p.sigc[id] = s2 * inv;
}

void launch_iface(const IfaceParams& p, cudaStream_t s) {
    const int T = 256;
    const long long nc = p.NXc * p.NYc, nf = p.NXf * p.NYf, nh = p.NXf * p.NYc;
    iface_coarse_trace<<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(p);
    iface_fine<<<(unsigned)((nf + T - 1) / T), T, 0, s>>>(p);
    iface_gather_y<<<(unsigned)((nh + T - 1) / T), T, 0, s>>>(p);
    iface_gather_x<<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(p);
}

// ------------------------------------------------------------------------------------------------
// State / test-hook kernels
// ------------------------------------------------------------------------------------------------
// Counter-based generator: splitmix64 finaliser of
// key = seed * 0xD1B54A32D192ED03 + box * 0x8CB92BA72F3D8DD7 + field * 0x9E3779B97F4A7C15
// advanced by (id + 1) * 0x9E3779B97F4A7C15; u = 2 (z >> 11) 2^-53 - 1 in [-1, 1).
__device__ __forceinline__ double cb_uniform(unsigned long long seed, int box, int field, long long id) {
    unsigned long long z = seed * 0xD1B54A32D192ED03ull + (unsigned long long)box * 0x8CB92BA72F3D8DD7ull +
                           (unsigned long long)field * 0x9E3779B97F4A7C15ull;
    z += ((unsigned long long)id + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}

__global__ void fill_random_kernel(double* pprev, double* w, double* pcur, long long n, unsigned long long seed,
                                   int box, double ps, double vs, double dt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p0 = ps * cb_uniform(seed, box, 0, i);
    const double v0 = vs * cb_uniform(seed, box, 1, i);
    pprev[i] = p0;
    w[i] = v0;
    pcur[i] = p0 + dt * v0;     // p^1 = p^0 + dt p'^0 (+ dt^2/2 p''^0 = 0)
}

void launch_fill_random(double* pprev, double* w, double* pcur, long long n, unsigned long long seed, int box,
                        double ps, double vs, double dt, cudaStream_t s) {
    fill_random_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pprev, w, pcur, n, seed, box, ps, vs, dt);
}

__global__ void set_state_kernel(const double* pprev, double* pcur, const double* w, long long n, double dt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pcur[i] = pprev[i] + dt * w[i];
}

void launch_set_state(double* pprev, double* pcur, double* w, const double*, const double*, long long n, double dt,
                      cudaStream_t s) {
    set_state_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pprev, pcur, w, n, dt);
}

__global__ void gather_kernel(const double* src, const long long* ids, long long n, double* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[ids[i]];
}

void launch_gather(const double* src, const long long* ids, long long n, double* out, cudaStream_t s) {
    gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, ids, n, out);
}

__global__ void nonfinite_kernel(const double* p, long long n, unsigned long long* flag) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    bool bad = false;
    for (; i < n; i += stride) bad |= !isfinite(p[i]);
    if (bad) atomicOr(flag, 1ull);
}

void launch_nonfinite(const double* p, long long n, unsigned long long* flag, cudaStream_t s) {
    nonfinite_kernel<<<148 * 8, 256, 0, s>>>(p, n, flag);
}

}  // namespace sem
