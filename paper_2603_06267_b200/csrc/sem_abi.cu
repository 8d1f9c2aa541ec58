// libsem host side: C ABI entry points (include/sem.h), validation, 1D GLL tables, PMUT and
// interface tables, device allocation, CUDA-graph step capture.  No compute runs on the host:
// every step of the method executes in kernels.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "sem_internal.h"

namespace sem {
int volume_tile_y();
}

using sem::Box;

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link needed).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3D FP64 map of a pitched box field: dims (NX, NY, NZ), row pitch PX doubles, box (bw, bh, 1),
// out-of-bounds elements zero-filled (the halo outside the box reads as p = 0 with zero weight).
bool make_map(CUtensorMap* m, double* base, const Box& b, int bw, int bh) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)b.NX, (cuuint64_t)b.NY, (cuuint64_t)b.NZ};
    cuuint64_t strides[2] = {(cuuint64_t)b.PX * 8, (cuuint64_t)b.PX * b.NY * 8};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- GLL (host, setup only)
// Nodes: Newton iteration on (1 - x^2) P_N'(x) through x P_N - P_{N-1} (Chebyshev-Gauss-Lobatto
// start), weights 2 / (N (N+1) P_N^2); ascending order.  P:L581.
void gll_rule(int N, std::vector<double>& x, std::vector<double>& w) {
    x.assign(N + 1, 0.0);
    w.assign(N + 1, 0.0);
    std::vector<double> xo(N + 1), Pn(N + 1), Pm(N + 1);
    for (int i = 0; i <= N; ++i) x[i] = std::cos(M_PI * i / N);
    for (int it = 0; it < 200; ++it) {
        double dmax = 0.0;
        for (int i = 0; i <= N; ++i) {
            double p0 = 1.0, p1 = x[i];
            for (int k = 2; k <= N; ++k) {
                const double p2 = ((2.0 * k - 1.0) * x[i] * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            Pn[i] = p1;
            Pm[i] = (N >= 1) ? p0 : 0.0;
            xo[i] = x[i];
            x[i] = xo[i] - (x[i] * Pn[i] - Pm[i]) / ((N + 1.0) * Pn[i]);
            dmax = std::max(dmax, std::fabs(x[i] - xo[i]));
        }
        if (dmax < 1e-16) break;
    }
    for (int i = 0; i <= N; ++i) {
        double p0 = 1.0, p1 = x[i];
        for (int k = 2; k <= N; ++k) {
            const double p2 = ((2.0 * k - 1.0) * x[i] * p1 - (k - 1.0) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        w[i] = 2.0 / (N * (N + 1.0) * p1 * p1);
    }
    std::reverse(x.begin(), x.end());
    std::reverse(w.begin(), w.end());
    x[0] = -1.0;
    x[N] = 1.0;
}

// barycentric weights lambda_j = 1 / prod_{k != j} (x_j - x_k)
std::vector<double> bary(const std::vector<double>& x) {
    const int n = (int)x.size();
    std::vector<double> l(n, 1.0);
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k)
            if (k != j) l[j] /= (x[j] - x[k]);
    return l;
}

// D[i][j] = ell_j'(x_i): (lambda_j / lambda_i) / (x_i - x_j), diagonal by negative row sum
std::vector<double> deriv_matrix(const std::vector<double>& x) {
    const int n = (int)x.size();
    const std::vector<double> l = bary(x);
    std::vector<double> D(n * n, 0.0);
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j)
            if (j != i) {
                D[i * n + j] = (l[j] / l[i]) / (x[i] - x[j]);
                s += D[i * n + j];
            }
        D[i * n + i] = -s;
    }
    return D;
}

// ell_j(t) by the second barycentric form
std::vector<double> lagrange_at(const std::vector<double>& x, double t) {
    const int n = (int)x.size();
    const std::vector<double> l = bary(x);
    std::vector<double> v(n, 0.0);
    for (int j = 0; j < n; ++j)
        if (t == x[j]) {
            v[j] = 1.0;
            return v;
        }
    double den = 0.0;
    for (int j = 0; j < n; ++j) den += l[j] / (t - x[j]);
    for (int j = 0; j < n; ++j) v[j] = (l[j] / (t - x[j])) / den;
    return v;
}

sem_status fail(sem_ctx* c, sem_status st, const std::string& msg) {
    if (c) c->err = msg;
    return st;
}

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? SEM_E_OOM : SEM_E_CUDA,            \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                      \
    } while (0)

template <typename T>
sem_status dalloc(sem_ctx* ctx, T** p, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
    if (e != cudaSuccess) return fail(ctx, SEM_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    ctx->allocs.push_back(q);
    *p = (T*)q;
    return SEM_OK;
}

template <typename T>
sem_status upload(sem_ctx* ctx, T** p, const std::vector<T>& h) {
    sem_status st = dalloc(ctx, p, h.size());
    if (st != SEM_OK) return st;
    CU(cudaMemcpy(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return SEM_OK;
}

// assembled 1D GLL weights along a direction with nel elements: w_asm(i)
std::vector<double> assembled_weights(int N, int nel, const std::vector<double>& w) {
    std::vector<double> a(N * nel + 1, 0.0);
    for (int e = 0; e < nel; ++e)
        for (int j = 0; j <= N; ++j) a[N * e + j] += w[j];
    return a;
}

void build_tables(Box& b) {
    const int N = b.N;
    std::vector<double> x, w;
    gll_rule(N, x, w);
    const std::vector<double> D = deriv_matrix(x);
    // A_hat[a][b] = sum_q w_q D[q][a] D[q][b]  (1D GLL stiffness on [-1, 1])
    std::vector<double> Ah((N + 1) * (N + 1), 0.0);
    for (int a = 0; a <= N; ++a)
        for (int c = 0; c <= N; ++c) {
            double s = 0.0;
            for (int q = 0; q <= N; ++q) s += w[q] * D[q * (N + 1) + a] * D[q * (N + 1) + c];
            Ah[a * (N + 1) + c] = s;
        }
    std::memset(&b.tab, 0, sizeof(b.tab));
    const double c2 = b.d.c * b.d.c;
    for (int d = 0; d < 3; ++d) {
        const double s = c2 * (2.0 / b.h[d]) * (2.0 / b.h[d]);
        for (int a = 0; a < N; ++a)
            for (int c = 0; c <= N; ++c) b.tab.G[d][a][c] = s * Ah[a * (N + 1) + c] / (a == 0 ? 2.0 * w[0] : w[a]);
        for (int c = 0; c <= N; ++c) {
            b.tab.G[d][sem::row_L(N)][c] = s * Ah[N * (N + 1) + c] / (2.0 * w[0]);
            b.tab.G[d][sem::row_B0(N)][c] = s * Ah[0 * (N + 1) + c] / w[0];
            b.tab.G[d][sem::row_BN(N)][c] = s * Ah[N * (N + 1) + c] / w[N];
        }
    }
    // node coordinates and face-mass factors m_d(i) = (h_d/2) w_asm(i)
    const std::vector<double> ax = assembled_weights(N, b.d.nel[0], w);
    const std::vector<double> ay = assembled_weights(N, b.d.nel[1], w);
    const std::vector<double> az = assembled_weights(N, b.d.nel[2], w);
    b.xh.resize(b.NX);
    b.yh.resize(b.NY);
    b.mxh.resize(b.NX);
    b.myh.resize(b.NY);
    b.mzh.resize(b.NZ);
    for (long long i = 0; i < b.NX; ++i) {
        const long long e = std::min<long long>(i / N, b.d.nel[0] - 1);
        b.xh[i] = b.d.origin[0] + b.h[0] * ((double)e + 0.5 * (x[i - e * N] + 1.0));
        b.mxh[i] = 0.5 * b.h[0] * ax[i];
    }
    for (long long i = 0; i < b.NY; ++i) {
        const long long e = std::min<long long>(i / N, b.d.nel[1] - 1);
        b.yh[i] = b.d.origin[1] + b.h[1] * ((double)e + 0.5 * (x[i - e * N] + 1.0));
        b.myh[i] = 0.5 * b.h[1] * ay[i];
    }
    for (long long i = 0; i < b.NZ; ++i) b.mzh[i] = 0.5 * b.h[2] * az[i];
}

sem_status check_box(sem_ctx* ctx, const sem_box_desc& d) {
    if (d.degree < 1 || d.degree > sem::kMaxN) return fail(ctx, SEM_E_ARG, "degree must be in 1..8");
    for (int k = 0; k < 3; ++k) {
        if (d.nel[k] < 1) return fail(ctx, SEM_E_ARG, "nel must be >= 1");
        if (!(d.extent[k] > 0)) return fail(ctx, SEM_E_ARG, "extent must be > 0");
    }
    if (!(d.c > 0)) return fail(ctx, SEM_E_ARG, "c must be > 0");
    if (!(d.rho >= 0)) return fail(ctx, SEM_E_ARG, "rho must be >= 0");
    for (int f = 0; f < 6; ++f)
        if (d.bc[f] < 0 || d.bc[f] > 2) return fail(ctx, SEM_E_ARG, "bad bc code");
    for (int f = 0; f < 4; ++f)
        if (d.bc[f] == SEM_BC_INTERFACE) return fail(ctx, SEM_E_ARG, "interface only on z faces");
    const long long nn = (long long)(d.degree * d.nel[0] + 1) * (d.degree * d.nel[1] + 1) * (d.degree * d.nel[2] + 1);
    if (nn > (1ll << 40)) return fail(ctx, SEM_E_ARG, "box too large");
    return SEM_OK;
}

sem::VolParams vol_params(sem_ctx* ctx, int bi, int cur) {
    Box& b = ctx->boxes[bi];
    sem::VolParams p{};
    p.tmP = b.tmP[cur];
    p.tmW = b.tmW;
    p.tab = b.tab;
    p.Pn = b.P[1 - cur];
    p.W = b.W;
    p.NX = b.NX;
    p.NY = b.NY;
    p.NZ = b.NZ;
    p.PX = b.PX;
    for (int d = 0; d < 3; ++d) p.sdir[d] = b.d.c * b.d.c * (2.0 / b.h[d]) * (2.0 / b.h[d]);
    p.nelz = b.d.nel[2];
    p.dt = ctx->dt;
    std::vector<double> x, w;
    gll_rule(b.N, x, w);
    for (int f = 0; f < 6; ++f) {
        const int d = f / 2;
        p.damp[f] = (b.d.bc[f] == SEM_BC_ABSORBING) ? b.d.c / (0.5 * b.h[d] * w[0]) : 0.0;
    }
    if (ctx->pm.on && ctx->pm.box == bi) {
        p.F = ctx->pm.F;
        p.kF = 1.0 / b.mzh[0];
    }
    p.iface_side = b.iface_side;
    p.tau = b.tau;
    p.sig = b.sig;
    if (ctx->pw.on && ctx->pw.box == bi) {
        const sem::PlaneWave& pw = ctx->pw;
        p.pw_on = 1;
        p.pw_fac = b.d.c * pw.amp * (1.0 - pw.k[2]) / b.mzh[b.NZ - 1];
        for (int k = 0; k < 3; ++k) {
            p.pw_k[k] = pw.k[k];
            p.pw_xref[k] = pw.xref[k];
        }
        p.pw_c = b.d.c;
        p.pw_t0 = pw.t0;
        p.pw_sigma = pw.sigma;
        p.pw_om = 2.0 * M_PI * pw.f0;
        p.pw_ztop = b.d.origin[2] + b.d.extent[2];
        p.xc = b.xc;
        p.yc = b.yc;
    }
    p.step = ctx->d_step;
    p.done = ctx->d_done;
    unsigned tot = 0;
    for (auto& bb : ctx->boxes) tot += sem::volume_blocks(bb.N, bb.NX, bb.NY);
    p.total_blocks = tot;
    p.bump_step = 1;
    return p;
}

sem::ModalParams modal_params(sem_ctx* ctx, int cur) {
    sem::Pmut& pm = ctx->pm;
    Box& b = ctx->boxes[pm.box];
    sem::ModalParams p{};
    p.n_pmut = pm.n_pmut;
    p.n_modes = pm.n_modes;
    p.lmax = pm.lmax;
    p.literal = (ctx->flags & SEM_F_COUPLING_LITERAL) ? 1 : 0;
    p.dt = ctx->dt;
    p.P = p.literal ? b.P[1 - cur] : b.P[cur];
    p.NX = b.NX;
    p.PX = b.PX;
    p.rect = pm.rect;
    p.sx = pm.sx;
    p.sy = pm.sy;
    p.wx = pm.wx;
    p.wy = pm.wy;
    p.omega2 = pm.omega2;
    p.twozw = pm.twozw;
    p.invmass = pm.invmass;
    p.eta = pm.eta;
    p.delay = pm.delay;
    p.amp = pm.amp;
    p.om0 = pm.om0;
    p.ncyc = pm.ncyc;
    p.t_end = pm.t_end;
    p.t_switch = pm.t_switch;
    p.invC = pm.invC;
    p.rx = pm.rx;
    p.kappa = pm.kappa;
    p.q = pm.q;
    p.qd = pm.qd;
    p.qdd = pm.qdd;
    p.phi = pm.phi;
    p.F = pm.F;
    p.step = ctx->d_step;
    return p;
}

// enqueue one step with parity `cur` on `s`; returns number of kernel launches
int enqueue_step(sem_ctx* ctx, int cur, cudaStream_t s, bool prof) {
    int nl = 0;
    auto mark = [&](int which, bool begin) {
        if (!prof) return;
        static thread_local cudaEvent_t pend = nullptr;
        cudaEvent_t e;
        if (ctx->ev_pool.empty()) {
            cudaEventCreate(&e);
        } else {
            e = ctx->ev_pool.back();
            ctx->ev_pool.pop_back();
        }
        cudaEventRecord(e, s);
        if (begin) {
            pend = e;
        } else {
            ctx->ev_pending.push_back({which, {pend, e}});
        }
    };
    if (ctx->pm.on) {
        mark(2, true);
        sem::launch_modal(modal_params(ctx, cur), s);
        mark(2, false);
        ++nl;
    }
    if (ctx->itf.on) {
        sem::IfaceParams ip = ctx->itf.prm;
        ip.Pf = ctx->boxes[ctx->itf.fine].P[cur];
        ip.Pc = ctx->boxes[ctx->itf.coarse].P[cur];
        mark(1, true);
        sem::launch_iface(ip, s);
        mark(1, false);
        nl += 4;
    }
    mark(0, true);
    for (int bi = 0; bi < (int)ctx->boxes.size(); ++bi) {
        sem::launch_volume(vol_params(ctx, bi, cur), ctx->boxes[bi].N, s);
        ++nl;
    }
    mark(0, false);
    return nl;
}

sem_status reset_dynamic(sem_ctx* ctx) {
    CU(cudaMemsetAsync(ctx->d_step, 0, sizeof(long long), ctx->stream));
    CU(cudaMemsetAsync(ctx->d_done, 0, sizeof(unsigned), ctx->stream));
    if (ctx->pm.on) {
        const size_t nm = (size_t)ctx->pm.n_pmut * ctx->pm.n_modes;
        CU(cudaMemsetAsync(ctx->pm.q, 0, nm * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(ctx->pm.qd, 0, nm * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(ctx->pm.qdd, 0, nm * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(ctx->pm.phi, 0, ctx->pm.n_pmut * sizeof(double), ctx->stream));
        Box& b = ctx->boxes[ctx->pm.box];
        CU(cudaMemsetAsync(ctx->pm.F, 0, b.NX * b.NY * sizeof(double), ctx->stream));
    }
    ctx->step = 0;
    return SEM_OK;
}

void drop_graphs(sem_ctx* ctx) {
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            if (ctx->graph[a][b]) {
                cudaGraphExecDestroy(ctx->graph[a][b]);
                ctx->graph[a][b] = nullptr;
            }
}

sem_status check_ctx(sem_ctx* ctx) {
    if (!ctx) return SEM_E_ARG;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return fail(ctx, SEM_E_CUDA, cudaGetErrorString(e));
    return SEM_OK;
}

}  // namespace

extern "C" {

sem_status sem_mesh_create(const sem_mesh_desc* desc, sem_ctx** out) {
    if (!out) return SEM_E_ARG;
    *out = nullptr;
    if (!desc || desc->n_boxes < 1 || desc->n_boxes > 2 || !desc->boxes) return SEM_E_ARG;
    sem_ctx* ctx = new (std::nothrow) sem_ctx();
    if (!ctx) return SEM_E_OOM;
    auto bail = [&](sem_status st) {
        sem_destroy(ctx);
        return st;
    };
    if (!(desc->dt > 0) || !std::isfinite(desc->dt)) return bail(SEM_E_ARG);
    if (desc->world != 1 || desc->rank != 0) return bail(SEM_E_PARTITION);
    ctx->device = desc->device;
    ctx->flags = desc->flags;
    ctx->dt = desc->dt;
    ctx->rank = desc->rank;
    ctx->world = desc->world;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return bail(SEM_E_CUDA);
    if (desc->stream) {
        ctx->stream = (cudaStream_t)desc->stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SEM_E_CUDA);
        ctx->own_stream = true;
    }
    for (int i = 0; i < desc->n_boxes; ++i) {
        if (check_box(ctx, desc->boxes[i]) != SEM_OK) return bail(SEM_E_ARG);
        Box b;
        b.d = desc->boxes[i];
        b.N = b.d.degree;
        b.NX = (long long)b.N * b.d.nel[0] + 1;
        b.NY = (long long)b.N * b.d.nel[1] + 1;
        b.NZ = (long long)b.N * b.d.nel[2] + 1;
        b.PX = (b.NX + 7) / 8 * 8;
        for (int k = 0; k < 3; ++k) b.h[k] = b.d.extent[k] / b.d.nel[k];
        build_tables(b);
        ctx->boxes.push_back(b);
    }
    for (size_t i = 0; i < ctx->boxes.size(); ++i) {
        Box& b = ctx->boxes[i];
        const size_t n = (size_t)b.nalloc();
        if (dalloc(ctx, &b.P[0], n) || dalloc(ctx, &b.P[1], n) || dalloc(ctx, &b.W, n)) return bail(SEM_E_OOM);
        if (cudaMemset(b.P[0], 0, n * 8) || cudaMemset(b.P[1], 0, n * 8) || cudaMemset(b.W, 0, n * 8))
            return bail(SEM_E_CUDA);
        const int TY = sem::volume_tile_y();
        sem::volume_prepare(b.N);
        if (!make_map(&b.tmP[0], b.P[0], b, sem::vol_pbox_w(b.N), TY + 2 * b.N) ||
            !make_map(&b.tmP[1], b.P[1], b, sem::vol_pbox_w(b.N), TY + 2 * b.N) ||
            !make_map(&b.tmW, b.W, b, sem::vol_wbox_w(b.N), TY)) {
            fprintf(stderr, "libsem: cuTensorMapEncodeTiled failed\n");
            return bail(SEM_E_CUDA);
        }
        if (upload(ctx, &b.xc, b.xh) || upload(ctx, &b.yc, b.yh) || upload(ctx, &b.mx, b.mxh) ||
            upload(ctx, &b.my, b.myh))
            return bail(SEM_E_CUDA);
    }
    if (dalloc(ctx, &ctx->d_step, 1) || dalloc(ctx, &ctx->d_done, 1) || dalloc(ctx, &ctx->d_flag, 1))
        return bail(SEM_E_OOM);
    if (reset_dynamic(ctx) != SEM_OK) return bail(SEM_E_CUDA);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return bail(SEM_E_CUDA);
    *out = ctx;
    return SEM_OK;
}

sem_status sem_pmut_attach(sem_ctx* ctx, const sem_pmut_desc* pd) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (!pd) return fail(ctx, SEM_E_ARG, "null pmut desc");
    if (ctx->pm.on) return fail(ctx, SEM_E_STATE, "PMUT array already attached");
    if (pd->box < 0 || pd->box >= (int)ctx->boxes.size()) return fail(ctx, SEM_E_ARG, "bad box");
    if (pd->face != 4) return fail(ctx, SEM_E_ARG, "PMUTs supported on the -z face only");
    if (pd->n_pmut < 1 || pd->n_modes < 1 || pd->n_modes > sem::kMaxModes)
        return fail(ctx, SEM_E_ARG, "n_pmut >= 1 and 1 <= n_modes <= 8 required");
    if (!(pd->side > 0) || !pd->center || !pd->mode_mn || !pd->freq_hz || !pd->modal_mass || !pd->damping_ratio ||
        !pd->eta || !pd->delay_s)
        return fail(ctx, SEM_E_ARG, "missing PMUT arrays");
    if (pd->rx && !(pd->capacitance > 0)) return fail(ctx, SEM_E_ARG, "RX requires capacitance > 0");
    if (pd->n_cycles < 1 || !(pd->f0_hz > 0)) return fail(ctx, SEM_E_ARG, "bad drive");
    Box& b = ctx->boxes[pd->box];
    if (b.d.bc[4] == SEM_BC_INTERFACE) return fail(ctx, SEM_E_ARG, "PMUT face is an interface");
    const int K = pd->n_pmut, M = pd->n_modes;
    const double a = pd->side;
    std::vector<int> rect(4 * K);
    std::vector<int> occ((size_t)b.NX * b.NY, -1);
    int lmax = 1;
    std::vector<std::vector<long long>> xi(K), yi(K);
    for (int k = 0; k < K; ++k) {
        const double x0 = pd->center[2 * k] - 0.5 * a, y0 = pd->center[2 * k + 1] - 0.5 * a;
        for (long long i = 0; i < b.NX; ++i) {
            const double xl = b.xh[i] - x0;
            if (xl >= 0 && xl <= a) xi[k].push_back(i);
        }
        for (long long j = 0; j < b.NY; ++j) {
            const double yl = b.yh[j] - y0;
            if (yl >= 0 && yl <= a) yi[k].push_back(j);
        }
        if (xi[k].empty() || yi[k].empty()) return fail(ctx, SEM_E_ARG, "membrane with no face node (or off the face)");
        if (x0 < b.d.origin[0] - 1e-12 * a || y0 < b.d.origin[1] - 1e-12 * a ||
            x0 + a > b.d.origin[0] + b.d.extent[0] + 1e-12 * a || y0 + a > b.d.origin[1] + b.d.extent[1] + 1e-12 * a)
            return fail(ctx, SEM_E_ARG, "membrane off the face");
        rect[4 * k] = (int)xi[k].front();
        rect[4 * k + 1] = (int)yi[k].front();
        rect[4 * k + 2] = (int)xi[k].size();
        rect[4 * k + 3] = (int)yi[k].size();
        lmax = std::max<int>(lmax, std::max(rect[4 * k + 2], rect[4 * k + 3]));
        for (long long j : yi[k])
            for (long long i : xi[k]) {
                int& o = occ[(size_t)j * b.NX + i];
                if (o >= 0) return fail(ctx, SEM_E_ARG, "membranes overlap");
                o = k;
            }
    }
    std::vector<double> sx((size_t)K * M * lmax, 0.0), sy((size_t)K * M * lmax, 0.0), wx((size_t)K * lmax, 0.0),
        wy((size_t)K * lmax, 0.0), om2((size_t)K * M), tzw((size_t)K * M), im(M), et(M), dl(K);
    for (int k = 0; k < K; ++k) {
        const double x0 = pd->center[2 * k] - 0.5 * a, y0 = pd->center[2 * k + 1] - 0.5 * a;
        for (int m = 0; m < M; ++m) {
            const int mm = pd->mode_mn[2 * m], nn = pd->mode_mn[2 * m + 1];
            for (size_t i = 0; i < xi[k].size(); ++i)
                sx[((size_t)k * M + m) * lmax + i] = std::sin(mm * M_PI * (b.xh[xi[k][i]] - x0) / a);
            for (size_t j = 0; j < yi[k].size(); ++j)
                sy[((size_t)k * M + m) * lmax + j] = std::sin(nn * M_PI * (b.yh[yi[k][j]] - y0) / a);
            const double om = 2.0 * M_PI * pd->freq_hz[(size_t)k * M + m];
            om2[(size_t)k * M + m] = om * om;
            tzw[(size_t)k * M + m] = 2.0 * pd->damping_ratio[m] * om;
        }
        for (size_t i = 0; i < xi[k].size(); ++i) wx[(size_t)k * lmax + i] = b.mxh[xi[k][i]];
        for (size_t j = 0; j < yi[k].size(); ++j) wy[(size_t)k * lmax + j] = b.myh[yi[k][j]];
        dl[k] = pd->delay_s[k];
    }
    for (int m = 0; m < M; ++m) {
        if (!(pd->modal_mass[m] > 0)) return fail(ctx, SEM_E_ARG, "modal mass must be > 0");
        im[m] = 1.0 / pd->modal_mass[m];
        et[m] = pd->eta[m];
    }
    sem::Pmut& pm = ctx->pm;
    pm.box = pd->box;
    pm.n_pmut = K;
    pm.n_modes = M;
    pm.lmax = lmax;
    if (upload(ctx, &pm.rect, rect) || upload(ctx, &pm.sx, sx) || upload(ctx, &pm.sy, sy) ||
        upload(ctx, &pm.wx, wx) || upload(ctx, &pm.wy, wy) || upload(ctx, &pm.omega2, om2) ||
        upload(ctx, &pm.twozw, tzw) || upload(ctx, &pm.invmass, im) || upload(ctx, &pm.eta, et) ||
        upload(ctx, &pm.delay, dl))
        return SEM_E_CUDA;
    const size_t nm = (size_t)K * M;
    if (dalloc(ctx, &pm.q, nm) || dalloc(ctx, &pm.qd, nm) || dalloc(ctx, &pm.qdd, nm) || dalloc(ctx, &pm.phi, K) ||
        dalloc(ctx, &pm.F, (size_t)b.NX * b.NY))
        return SEM_E_OOM;
    pm.amp = pd->amp_v;
    pm.om0 = 2.0 * M_PI * pd->f0_hz;
    pm.ncyc = pd->n_cycles;
    pm.t_end = pd->n_cycles / pd->f0_hz;
    pm.t_switch = pd->t_switch;
    pm.rx = pd->rx ? 1 : 0;
    pm.invC = pd->rx ? 1.0 / pd->capacitance : 0.0;
    pm.kappa = b.d.rho * b.d.c * b.d.c;   // kappa = rho c^2
    pm.on = true;
    drop_graphs(ctx);
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_dg_interface_build(sem_ctx* ctx, int fine_box, int coarse_box, double alpha, int quad_rule) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (ctx->itf.on) return fail(ctx, SEM_E_STATE, "interface already built");
    if (quad_rule != 0) return fail(ctx, SEM_E_ARG, "only quad_rule 0 (fine-face GLL nodes) is implemented");
    const int nb = (int)ctx->boxes.size();
    if (fine_box < 0 || coarse_box < 0 || fine_box >= nb || coarse_box >= nb || fine_box == coarse_box)
        return fail(ctx, SEM_E_ARG, "bad box indices");
    if (!(alpha > 0)) return fail(ctx, SEM_E_ARG, "penalty alpha must be > 0");
    Box& F = ctx->boxes[fine_box];
    Box& C = ctx->boxes[coarse_box];
    if (F.d.bc[5] != SEM_BC_INTERFACE || C.d.bc[4] != SEM_BC_INTERFACE)
        return fail(ctx, SEM_E_ARG, "fine +z and coarse -z faces must be tagged SEM_BC_INTERFACE");
    const double tol = 1e-9 * std::max(F.h[0], C.h[0]);
    for (int k = 0; k < 2; ++k) {
        if (std::fabs(F.d.origin[k] - C.d.origin[k]) > tol || std::fabs(F.d.extent[k] - C.d.extent[k]) > tol)
            return fail(ctx, SEM_E_UNMATCHED, "interface faces do not coincide laterally");
    }
    if (std::fabs(F.d.origin[2] + F.d.extent[2] - C.d.origin[2]) > tol)
        return fail(ctx, SEM_E_UNMATCHED, "boxes do not touch in z");
    if (F.d.nel[0] % C.d.nel[0] || F.d.nel[1] % C.d.nel[1] ||
        F.d.nel[0] / C.d.nel[0] != F.d.nel[1] / C.d.nel[1])
        return fail(ctx, SEM_E_UNMATCHED, "fine lattice does not nest in the coarse one (need h_c = R h_f)");
    const int R = F.d.nel[0] / C.d.nel[0];
    std::vector<double> xf, wf, xc, wc;
    gll_rule(F.N, xf, wf);
    gll_rule(C.N, xc, wc);
    const std::vector<double> Df = deriv_matrix(xf), Dc = deriv_matrix(xc);
    sem::IfaceParams& p = ctx->itf.prm;
    p = sem::IfaceParams{};
    p.NXf = F.NX;
    p.NYf = F.NY;
    p.NZf = F.NZ;
    p.NXc = C.NX;
    p.PXf = F.PX;
    p.PXc = C.PX;
    p.NYc = C.NY;
    p.Nf = F.N;
    p.Nc = C.N;
    p.R = R;
    p.nelcx = C.d.nel[0];
    p.nelcy = C.d.nel[1];
    const double cbar = 2.0 * F.d.c * C.d.c / (F.d.c + C.d.c);
    const double hmin = std::min(std::min(std::min(F.h[0], F.h[1]), F.h[2]), std::min(std::min(C.h[0], C.h[1]), C.h[2]));
    p.gamma = alpha * cbar * cbar * std::max(F.N, C.N) * std::max(F.N, C.N) / hmin;
    p.cf2 = F.d.c * F.d.c;
    p.cc2 = C.d.c * C.d.c;
    for (int c = 0; c <= F.N; ++c) p.dfT[c] = (2.0 / F.h[2]) * Df[F.N * (F.N + 1) + c];
    for (int c = 0; c <= C.N; ++c) p.dcB[c] = (2.0 / C.h[2]) * Dc[0 * (C.N + 1) + c];
    const int NfR = F.N * R;
    std::vector<double> I((size_t)(NfR + 1) * (C.N + 1), 0.0);
    for (int q = 0; q <= NfR; ++q) {
        int r = q / F.N, a = q % F.N;
        if (q == NfR) {
            r = R - 1;
            a = F.N;
        }
        const double xm = (2.0 * r + xf[a] + 1.0) / R - 1.0;   // x_hat^- of the fine node
        const std::vector<double> l = lagrange_at(xc, xm);
        for (int b = 0; b <= C.N; ++b) I[(size_t)q * (C.N + 1) + b] = l[b];
    }
    double* dI = nullptr;
    if (upload(ctx, &dI, I)) return SEM_E_CUDA;
    p.I = dI;
    p.mxf = F.mx;
    p.myf = F.my;
    p.mxc = C.mx;
    p.myc = C.my;
    const size_t nf = (size_t)F.NX * F.NY, nc = (size_t)C.NX * C.NY, nh = (size_t)F.NX * C.NY;
    if (dalloc(ctx, &p.trc, nc) || dalloc(ctx, &p.drc, nc) || dalloc(ctx, &p.tauf, nf) || dalloc(ctx, &p.sigf, nf) ||
        dalloc(ctx, &p.g1, nf) || dalloc(ctx, &p.g2, nf) || dalloc(ctx, &p.h1, nh) || dalloc(ctx, &p.h2, nh) ||
        dalloc(ctx, &p.tauc, nc) || dalloc(ctx, &p.sigc, nc))
        return SEM_E_OOM;
    // layer coefficients: a -= tau ktau[c] + sigma ksig[c]
    F.iface_side = +1;
    F.tau = p.tauf;
    F.sig = p.sigf;
    for (int c = 0; c <= F.N; ++c) {
        const long long iz = F.NZ - 1 - F.N + c;
        F.tab.ksig[c] = (2.0 / F.h[2]) * Df[F.N * (F.N + 1) + c] / F.mzh[iz];
        F.tab.ktau[c] = (c == F.N) ? 1.0 / F.mzh[iz] : 0.0;
    }
    C.iface_side = -1;
    C.tau = p.tauc;
    C.sig = p.sigc;
    for (int c = 0; c <= C.N; ++c) {
        C.tab.ksig[c] = (2.0 / C.h[2]) * Dc[0 * (C.N + 1) + c] / C.mzh[c];
        C.tab.ktau[c] = (c == 0) ? 1.0 / C.mzh[0] : 0.0;
    }
    ctx->itf.on = true;
    ctx->itf.fine = fine_box;
    ctx->itf.coarse = coarse_box;
    drop_graphs(ctx);
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_plane_wave_source(sem_ctx* ctx, int box, int face, double amp, double f0, double sigma, double t0,
                                 const double dir[3]) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->boxes.size() || face != 5 || !dir)
        return fail(ctx, SEM_E_ARG, "plane wave: +z face of an existing box only");
    Box& b = ctx->boxes[box];
    if (b.d.bc[5] != SEM_BC_ABSORBING) return fail(ctx, SEM_E_ARG, "plane wave needs an absorbing face");
    const double nk = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    if (!(nk > 0) || !(sigma > 0)) return fail(ctx, SEM_E_ARG, "bad plane-wave parameters");
    sem::PlaneWave& pw = ctx->pw;
    pw.box = box;
    pw.amp = amp;
    pw.f0 = f0;
    pw.sigma = sigma;
    pw.t0 = t0;
    for (int k = 0; k < 3; ++k) pw.k[k] = dir[k] / nk;
    // x_ref: the +z face corner the wavefront reaches first (min k.x), reading R13
    const double zt = b.d.origin[2] + b.d.extent[2];
    double best = std::numeric_limits<double>::infinity();
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double x = b.xh[i ? b.NX - 1 : 0], y = b.yh[j ? b.NY - 1 : 0];
            const double kx = pw.k[0] * x + pw.k[1] * y + pw.k[2] * zt;
            if (kx < best) {
                best = kx;
                pw.xref[0] = x;
                pw.xref[1] = y;
                pw.xref[2] = zt;
            }
        }
    pw.on = true;
    drop_graphs(ctx);
    return SEM_OK;
}

sem_status sem_step(sem_ctx* ctx, int n_steps) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (n_steps < 0) return fail(ctx, SEM_E_ARG, "n_steps < 0");
    long long launches = 0;
    const bool direct = ctx->profiling || (ctx->flags & SEM_F_NO_GRAPH);
    int left = n_steps;
    while (left > 0) {
        if (direct) {
            launches += enqueue_step(ctx, ctx->cur, ctx->stream, ctx->profiling);
            ctx->cur ^= 1;
            --left;
            continue;
        }
        const int len = left >= 2 ? 2 : 1;
        cudaGraphExec_t& g = ctx->graph[ctx->cur][len - 1];
        if (!g) {
            cudaGraph_t graph;
            CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            int nl = 0;
            for (int k = 0; k < len; ++k) nl += enqueue_step(ctx, ctx->cur ^ (k & 1), ctx->stream, false);
            CU(cudaStreamEndCapture(ctx->stream, &graph));
            cudaError_t e = cudaGraphInstantiate(&g, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) return fail(ctx, SEM_E_CUDA, std::string("graph: ") + cudaGetErrorString(e));
            ctx->graph_launches[ctx->cur][len - 1] = nl;
        }
        CU(cudaGraphLaunch(g, ctx->stream));
        launches += ctx->graph_launches[ctx->cur][len - 1];
        if (len == 2) {
            /* parity unchanged after two steps */
        } else {
            ctx->cur ^= 1;
        }
        left -= len;
    }
    CU(cudaGetLastError());
    ctx->step += n_steps;
    ctx->last_launches = launches;
    if (ctx->flags & SEM_F_NAN_CHECK) {
        CU(cudaMemsetAsync(ctx->d_flag, 0, 8, ctx->stream));
        for (auto& b : ctx->boxes)
            sem::launch_nonfinite(b.P[1 - ctx->cur], b.NX, b.PX, b.NY * b.NZ, ctx->d_flag, ctx->stream);
        unsigned long long f = 0;
        CU(cudaMemcpyAsync(&f, ctx->d_flag, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (f) return fail(ctx, SEM_E_NONFINITE, "non-finite pressure at step " + std::to_string(ctx->step));
    }
    return SEM_OK;
}

sem_status sem_sync(sem_ctx* ctx) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_read_pressure(sem_ctx* ctx, int box, double* host, size_t n) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->boxes.size() || !host) return fail(ctx, SEM_E_ARG, "bad box / buffer");
    Box& b = ctx->boxes[box];
    if (n != (size_t)b.ndof()) return fail(ctx, SEM_E_ARG, "n must equal the box node count");
    CU(cudaMemcpy2DAsync(host, b.NX * 8, b.P[1 - ctx->cur], b.PX * 8, b.NX * 8, b.NY * b.NZ, cudaMemcpyDeviceToHost,
                         ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_read_pressure_at(sem_ctx* ctx, int box, const long long* ids, size_t n, double* out) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->boxes.size() || (n && (!ids || !out))) return fail(ctx, SEM_E_ARG, "bad args");
    if (n == 0) return SEM_OK;
    Box& b = ctx->boxes[box];
    for (size_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= b.ndof()) return fail(ctx, SEM_E_ARG, "node id out of range");
    long long* dids = nullptr;
    double* dout = nullptr;
    CU(cudaMallocAsync(&dids, n * sizeof(long long), ctx->stream));
    CU(cudaMallocAsync(&dout, n * sizeof(double), ctx->stream));
    CU(cudaMemcpyAsync(dids, ids, n * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
    sem::launch_gather(b.P[1 - ctx->cur], dids, (long long)n, b.NX, b.PX, dout, ctx->stream);
    CU(cudaMemcpyAsync(out, dout, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaFreeAsync(dids, ctx->stream));
    CU(cudaFreeAsync(dout, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_read_modal(sem_ctx* ctx, double* q, double* qdot, double* v_rx, size_t n) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (!ctx->pm.on) return fail(ctx, SEM_E_STATE, "no PMUT array attached");
    const size_t nm = (size_t)ctx->pm.n_pmut * ctx->pm.n_modes;
    if (n != nm) return fail(ctx, SEM_E_ARG, "n must equal n_pmut * n_modes");
    if (q) CU(cudaMemcpyAsync(q, ctx->pm.q, nm * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (qdot) CU(cudaMemcpyAsync(qdot, ctx->pm.qd, nm * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (v_rx) CU(cudaMemcpyAsync(v_rx, ctx->pm.phi, ctx->pm.n_pmut * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_write_state(sem_ctx* ctx, int box, const double* p, const double* pdot, size_t n) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->boxes.size() || !p || !pdot) return fail(ctx, SEM_E_ARG, "bad args");
    Box& b = ctx->boxes[box];
    if (n != (size_t)b.ndof()) return fail(ctx, SEM_E_ARG, "n must equal the box node count");
    // p^S lives in P[1-cur]; p^{S+1} = p^S + dt w^S in P[cur]; w^0 = p'^0 + dt/2 p''^0 = p'^0
    double* pprev = b.P[1 - ctx->cur];
    double* pcur = b.P[ctx->cur];
    CU(cudaMemcpy2DAsync(pprev, b.PX * 8, p, b.NX * 8, b.NX * 8, b.NY * b.NZ, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpy2DAsync(b.W, b.PX * 8, pdot, b.NX * 8, b.NX * 8, b.NY * b.NZ, cudaMemcpyHostToDevice, ctx->stream));
    sem::launch_set_state(pprev, pcur, b.W, b.NX, b.PX, b.NY * b.NZ, ctx->dt, ctx->stream);
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_fill_random_state(sem_ctx* ctx, int box, unsigned long long seed, double ps, double vs) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->boxes.size()) return fail(ctx, SEM_E_ARG, "bad box");
    Box& b = ctx->boxes[box];
    sem::launch_fill_random(b.P[1 - ctx->cur], b.W, b.P[ctx->cur], b.NX, b.PX, b.NY * b.NZ, seed, box, ps, vs, ctx->dt,
                            ctx->stream);
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_query(sem_ctx* ctx, long long* n_dof, long long* step, double* t) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    long long nd = 0;
    for (auto& b : ctx->boxes) nd += b.ndof();
    if (n_dof) *n_dof = nd;
    if (step) *step = ctx->step;
    if (t) *t = ctx->step * ctx->dt;
    return SEM_OK;
}

sem_status sem_set_profiling(sem_ctx* ctx, int on) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    for (auto& pe : ctx->ev_pending) {
        ctx->ev_pool.push_back(pe.second.first);
        ctx->ev_pool.push_back(pe.second.second);
    }
    ctx->ev_pending.clear();
    for (int k = 0; k < 3; ++k) {
        ctx->kt_ms[k] = 0;
        ctx->kt_n[k] = 0;
    }
    ctx->profiling = on != 0;
    return SEM_OK;
}

sem_status sem_kernel_time(sem_ctx* ctx, int which, double* ms, long long* nl) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (which < 0 || which > 2) return fail(ctx, SEM_E_ARG, "which in 0..2");
    CU(cudaStreamSynchronize(ctx->stream));
    for (auto& pe : ctx->ev_pending) {
        float f = 0;
        CU(cudaEventElapsedTime(&f, pe.second.first, pe.second.second));
        ctx->kt_ms[pe.first] += f;
        ctx->kt_n[pe.first] += 1;
        ctx->ev_pool.push_back(pe.second.first);
        ctx->ev_pool.push_back(pe.second.second);
    }
    ctx->ev_pending.clear();
    if (ms) *ms = ctx->kt_ms[which];
    if (nl) *nl = ctx->kt_n[which];
    return SEM_OK;
}

sem_status sem_last_launch_count(sem_ctx* ctx, long long* n) {
    if (!ctx || !n) return SEM_E_ARG;
    *n = ctx->last_launches;
    return SEM_OK;
}

const char* sem_last_error(const sem_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void sem_destroy(sem_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drop_graphs(ctx);
    for (void* p : ctx->allocs) cudaFree(p);
    for (auto& pe : ctx->ev_pending) {
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

}  // extern "C"
