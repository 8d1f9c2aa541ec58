// libsem host side: C ABI entry points (include/sem.h), validation, 1D GLL tables, PMUT and
// interface tables, device allocation, CUDA-graph step capture.  No compute runs on the host:
// every step of the method executes in kernels.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "sem_internal.h"

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
// n-point Gauss-Legendre rule on [-1, 1] (ascending): roots of P_n by Newton, w = 2 / ((1 - x^2) P_n'(x)^2)
void gl_rule(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (z * p1 - p0) / (z * z - 1.0);
            const double dz = p1 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[n - 1 - i] = z;
        w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
}

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
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    if (ctx->dev_alloc) {
        q = ctx->dev_alloc(bytes, ctx->alloc_user);
        if (!q) return fail(ctx, SEM_E_OOM, "caller allocator returned NULL");
    } else {
        cudaError_t e = cudaMalloc(&q, bytes);
        if (e != cudaSuccess) return fail(ctx, SEM_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    ctx->allocs.push_back(q);
    *p = (T*)q;
    return SEM_OK;
}

template <typename T>
sem_status upload(sem_ctx* ctx, T** p, const std::vector<T>& h) {
    sem_status st = dalloc(ctx, p, h.size());
    if (st != SEM_OK) return st;
    // setup copies run on the context stream (not the legacy default stream, which does not order
    // with the non-blocking streams the steps use) and complete before the call returns
    CU(cudaMemcpyAsync(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
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

// ------------------------------------------------------------------------------------------------
// NCCL through dlopen (only needed for world > 1 without emulation; torch normally has it loaded)
// ------------------------------------------------------------------------------------------------
struct NcclUid { char internal[128]; };
struct NcclApi {
    bool ok = false;
    int (*getUniqueId)(NcclUid*) = nullptr;
    int (*commInitRank)(void**, int, NcclUid, int) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    const char* (*errStr)(int) = nullptr;
};
constexpr int kNcclDouble = 8;   // ncclFloat64 in nccl.h (ncclDouble == ncclFloat64 == 8)

NcclApi& nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.getUniqueId = (int (*)(NcclUid*))dlsym(h, "ncclGetUniqueId");
            api.commInitRank = (int (*)(void**, int, NcclUid, int))dlsym(h, "ncclCommInitRank");
            api.commDestroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
            api.send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclSend");
            api.recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclRecv");
            api.groupStart = (int (*)())dlsym(h, "ncclGroupStart");
            api.groupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
            api.errStr = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
            api.ok = api.getUniqueId && api.commInitRank && api.send && api.recv && api.groupStart && api.groupEnd;
        }
    }
    return api;
}

#define NC(call)                                                                                  \
    do {                                                                                          \
        int r_ = (call);                                                                          \
        if (r_ != 0)                                                                              \
            return fail(ctx, SEM_E_NCCL, std::string(#call) + ": " +                              \
                                             (nccl_api().errStr ? nccl_api().errStr(r_) : "?"));  \
    } while (0)

// ------------------------------------------------------------------------------------------------
// Slabs
// ------------------------------------------------------------------------------------------------
bool nccl_mode(const sem_ctx* ctx) { return ctx->world > 1 && !ctx->emulate; }

// ---- partition rules (shared by sem_mesh_create / sem_pmut_attach / sem_dg_interface_build and the
//      host-only sem_slab_plan): y-slabs, cuts at the same y for all boxes, given as box-0 element y
//      indices cuts[0] = 0 < cuts[1] < ... < cuts[G] = nel_y(box 0).
//      y (not x): a cut plane iy = const is, per z-plane, one contiguous lattice row, so the cut-plane
//      partial rows and fix-ups are coalesced (an x cut touches one node per row).
// box b's element index of box-0 element boundary k, or -1 if it is not an element boundary of box b
long long cut_in_box(const sem_box_desc& b0, const sem_box_desc& b, long long k) {
    const long long num = k * (long long)b.nel[1];
    return num % b0.nel[1] ? -1 : num / b0.nel[1];
}

const char* plan_invalid(const sem_box_desc* boxes, int n, const std::vector<long long>& cuts) {
    const int G = (int)cuts.size() - 1;
    if (G < 1 || cuts[0] != 0 || cuts[G] != boxes[0].nel[1]) return "slab plan must run from 0 to nel_y";
    for (int r = 0; r < G; ++r) {
        if (cuts[r + 1] <= cuts[r]) return "slab plan must be increasing";
        for (int i = 0; i < n; ++i)
            if (cut_in_box(boxes[0], boxes[i], cuts[r + 1]) < 0)
                return "every slab cut must be an element boundary of every box";
    }
    return nullptr;
}

// y position of box-0 element boundary k
double cut_y(const sem_box_desc& b0, long long k) { return b0.origin[1] + b0.extent[1] / b0.nel[1] * (double)k; }

// slab owning a membrane spanning [y0, y0 + a]; -1 if a cut crosses or touches it (membranes are never
// split across GPUs: the paper's membrane-preserving partition)
int membrane_slab(const sem_box_desc& b0, const std::vector<long long>& cuts, double y0, double a) {
    const double hy = b0.extent[1] / b0.nel[1];
    int slab = 0;
    for (size_t r = 1; r + 1 < cuts.size(); ++r) {
        const double cut = cut_y(b0, cuts[r]);
        if (y0 <= cut + 1e-9 * hy && y0 + a >= cut - 1e-9 * hy) return -1;
        if (y0 > cut) slab = (int)r;
    }
    return slab;
}

std::vector<long long> equal_plan(const sem_box_desc& b0, int G) {
    std::vector<long long> c(G + 1);
    for (int r = 0; r <= G; ++r) c[r] = (long long)b0.nel[1] * r / G;
    return c;
}

bool plan_ok(const sem_box_desc* boxes, int n, const std::vector<long long>& cuts, const sem_pmut_desc* pm) {
    if (plan_invalid(boxes, n, cuts)) return false;
    if (pm)
        for (int k = 0; k < pm->n_pmut; ++k)
            if (membrane_slab(boxes[0], cuts, pm->center[2 * k + 1] - 0.5 * pm->side, pm->side) < 0) return false;
    return true;
}

// equal slabs if admissible, else greedily the admissible cut nearest to each equal cut
bool auto_plan(const sem_box_desc* boxes, int n, int G, const sem_pmut_desc* pm, std::vector<long long>& cuts) {
    const long long nel = boxes[0].nel[1];
    if (G > nel) return false;
    if (nel % G == 0 && plan_ok(boxes, n, cuts = equal_plan(boxes[0], G), pm)) return true;
    std::vector<char> adm(nel + 1, 0);
    const double a = pm ? pm->side : 0.0;
    for (long long k = 1; k < nel; ++k) {
        bool ok = true;
        for (int i = 0; i < n && ok; ++i) ok = cut_in_box(boxes[0], boxes[i], k) >= 0;
        if (ok && pm)
            for (int m = 0; m < pm->n_pmut && ok; ++m) {
                const double y0 = pm->center[2 * m + 1] - 0.5 * a, hy = boxes[0].extent[1] / nel, cy = cut_y(boxes[0], k);
                ok = !(y0 <= cy + 1e-9 * hy && y0 + a >= cy - 1e-9 * hy);
            }
        adm[k] = ok ? 1 : 0;
    }
    // admissible boundaries, then the G-slab plan minimising the largest slab (dynamic programme over
    // the admissible positions; the largest slab bounds the step time of a strong-scaling run)
    std::vector<long long> P{0};
    for (long long k = 1; k < nel; ++k)
        if (adm[k]) P.push_back(k);
    P.push_back(nel);
    const int m = (int)P.size();
    const long long INF = 1LL << 60;
    std::vector<std::vector<long long>> dp(G + 1, std::vector<long long>(m, INF));
    std::vector<std::vector<int>> from(G + 1, std::vector<int>(m, -1));
    dp[0][0] = 0;
    for (int r = 1; r <= G; ++r)
        for (int j = 1; j < m; ++j)
            for (int i = 0; i < j; ++i) {
                if (dp[r - 1][i] >= INF) continue;
                const long long v = std::max(dp[r - 1][i], P[j] - P[i]);
                if (v < dp[r][j]) {
                    dp[r][j] = v;
                    from[r][j] = i;
                }
            }
    if (dp[G][m - 1] >= INF) return false;
    cuts.assign(G + 1, 0);
    for (int r = G, j = m - 1; r >= 1; --r) {
        cuts[r] = P[j];
        j = from[r][j];
    }
    return plan_ok(boxes, n, cuts, pm);
}

// Slab of global box g: elements [ey0, ey0 + nel_loc) along y.  1D tables (coordinates, face masses)
// are taken from the global lattice, so a cut node keeps its interior (two-sided) mass.
Box make_slab(const sem_box_desc& g, long long ey0, long long nel_loc, bool cutL, bool cutR) {
    Box gb;
    gb.d = g;
    gb.N = g.degree;
    gb.NX = (long long)gb.N * g.nel[0] + 1;
    gb.NY = (long long)gb.N * g.nel[1] + 1;
    gb.NZ = (long long)gb.N * g.nel[2] + 1;
    for (int k = 0; k < 3; ++k) gb.h[k] = g.extent[k] / g.nel[k];
    build_tables(gb);
    Box b = gb;
    b.d.origin[1] = g.origin[1] + gb.h[1] * (double)ey0;
    b.d.extent[1] = gb.h[1] * (double)nel_loc;
    b.d.nel[1] = (int)nel_loc;
    if (cutL) b.d.bc[2] = SEM_BC_RIGID;
    if (cutR) b.d.bc[3] = SEM_BC_RIGID;
    b.NY = (long long)b.N * nel_loc + 1;
    b.PX = (b.NX + 7) / 8 * 8;
    b.gy0 = (long long)b.N * ey0;
    b.NYg = gb.NY;
    b.cutL = cutL;
    b.cutR = cutR;
    b.yh.assign(gb.yh.begin() + b.gy0, gb.yh.begin() + b.gy0 + b.NY);
    b.myh.assign(gb.myh.begin() + b.gy0, gb.myh.begin() + b.gy0 + b.NY);
    return b;
}

// The fine face's d_z p hand-off (VolParams::dzf / IfaceParams::dzf): the structured fused interface on
// one GPU (no slabs: the cut fix-up would change p^{n+2} after the volume kernel) and no PML on the fine
// box (the PML fix-up would, too).
bool dzf_active(const sem_ctx* ctx, const sem::Part& pt) {
    if (!pt.itf.on || pt.itf.general || !pt.itf.dzf || ctx->world > 1 || ctx->parts.size() != 1) return false;
    if (pt.pml.on && pt.pml.box == pt.itf.fine) return false;
    if (pt.boxes[pt.itf.fine].curved || pt.boxes[pt.itf.coarse].curved) return false;
    return true;
}

// (re)compute d_z p at the fine face from the current state P[cur]
void dzf_refresh(sem_ctx* ctx) {
    for (auto& pt : ctx->parts)
        if (dzf_active(ctx, pt)) {
            sem::IfaceParams ip = pt.itf.prm;
            ip.Pf = pt.boxes[pt.itf.fine].P[ctx->cur];
            sem::launch_iface_dz_init(ip, pt.itf.dzf, ctx->stream);
        }
}

sem::VolParams vol_params(sem_ctx* ctx, sem::Part& pt, int bi, int cur) {
    Box& b = pt.boxes[bi];
    sem::VolParams p{};
    p.tmP = b.tmP[cur];
    p.tmW = SEM_TWO_LEVEL ? b.tmPw[1 - cur] : b.tmW;   // two-level: the p^n tile instead of w^n
    p.tab = b.tab;
    p.Pn = b.P[1 - cur];
    p.W = b.W;
    p.NX = b.NX;
    p.NY = b.NY;
    p.NZ = b.NZ;
    p.PX = b.PX;
    p.N = b.N;
    for (int d = 0; d < 3; ++d) p.sdir[d] = b.d.c * b.d.c * (2.0 / b.h[d]) * (2.0 / b.h[d]);
    p.nelz = b.d.nel[2];
    p.dt = ctx->dt;
    p.inv_dt = 1.0 / ctx->dt;
    std::vector<double> x, w;
    gll_rule(b.N, x, w);
    for (int f = 0; f < 6; ++f) {
        const int d = f / 2;
        p.damp[f] = (b.d.bc[f] == SEM_BC_ABSORBING) ? b.d.c / (0.5 * b.h[d] * w[0]) : 0.0;
    }
    p.cutL = b.cutL ? 1 : 0;
    p.cutR = b.cutR ? 1 : 0;
    if (pt.pm.on && pt.pm.box == bi) {
        p.F = pt.pm.F;
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
    if (pt.itf.on && bi == pt.itf.fine && dzf_active(ctx, pt)) {
        p.dzf = pt.itf.dzf;
        for (int c = 0; c <= b.N; ++c) p.dzc[c] = pt.itf.prm.dfT[c];
    }
    return p;
}

sem::ModalParams modal_params(sem_ctx* ctx, sem::Part& pt, int cur) {
    sem::Pmut& pm = pt.pm;
    Box& b = pt.boxes[pm.box];
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
    if (pm.toff) {
        p.toff = pm.toff;
        p.tidx = pm.tidx;
        p.tB = pm.tB;
        p.res = b.res;
        p.NY_dbg = b.NY;
    }
    return p;
}

// partial rows (side 0: this slab's first y plane, R0 row; side 1: last y plane, L row) of box bi
sem::CutParams cut_params(sem_ctx* ctx, sem::Part& pt, int side, int bi, int cur) {
    Box& b = pt.boxes[bi];
    sem::CutParams c{};
    c.side = side;
    c.N = b.N;
    c.NX = b.NX;
    c.NY = b.NY;
    c.NZ = b.NZ;
    c.PX = b.PX;
    c.P = b.P[cur];
    c.Pn = b.P[1 - cur];
    c.W = b.W;
    const int row = side == 0 ? 0 : sem::row_L(b.N);
    for (int k = 0; k <= b.N; ++k) c.row[k] = b.tab.G[1][row][k];   // y rows (scaled by c^2 (2/h_y)^2)
    c.dt = ctx->dt;
    if (b.iface_side < 0) {   // coarse box of the interface: SIPG partials (one face-lattice row) travel with it
        c.NXt = b.NX;
        c.NYt = b.NY;
        c.tau = b.tau;
        c.sig = b.sig;
        for (int k = 0; k <= b.N; ++k) {
            c.ktau[k] = b.tab.ktau[k];
            c.ksig[k] = b.tab.ksig[k];
        }
    }
    if (pt.pml.on && pt.pml.box == bi) c.pda = pt.pml.da;
    c.out = pt.send[side] + pt.xoff[bi];
    c.in = pt.recv[side] + pt.xoff[bi];
    return c;
}

sem::CurvedParams curved_params(sem_ctx* ctx, sem::Part& pt, int bi, int cur) {
    Box& b = pt.boxes[bi];
    sem::CurvedParams p{};
    p.N = b.N;
    p.NX = b.NX;
    p.NY = b.NY;
    p.NZ = b.NZ;
    p.PX = b.PX;
    p.nelx = b.d.nel[0];
    p.nely = b.d.nel[1];
    p.nelz = b.d.nel[2];
    p.grid = sem::curved_grid(b.N, p.nelx * p.nely * p.nelz);
    p.solid = b.solid;
    p.vlat = b.vlat;
    p.P = b.P[cur];
    p.res = b.res;
    p.W = b.W;
    p.Pn = b.P[1 - cur];
    p.minv = b.minv;
    p.cdamp = b.cdamp;
    std::vector<double> x, w;
    gll_rule(b.N, x, w);
    const std::vector<double> D = deriv_matrix(x);
    for (int i = 0; i <= b.N; ++i) {
        p.x[i] = x[i];
        p.w[i] = w[i];
        for (int j = 0; j <= b.N; ++j) p.D[i][j] = D[(size_t)i * (b.N + 1) + j];
    }
    p.c2 = b.d.c * b.d.c;
    p.dt = ctx->dt;
    p.inv_dt = 1.0 / ctx->dt;
    if (ctx->pw.on && ctx->pw.box == bi && b.pwd) {
        p.pwd = b.pwd;
        p.pwf = b.pwf;
        p.step = ctx->d_step;
        p.pw_t0 = ctx->pw.t0;
        p.pw_is2 = 1.0 / (ctx->pw.sigma * ctx->pw.sigma);
        p.pw_om = 2.0 * M_PI * ctx->pw.f0;
    }
    if (pt.pm.on && pt.pm.box == bi && !pt.pm.toff) {   // affine obstacle box: separable coupling
        p.F = pt.pm.F;
        p.fmx = b.mx;
        p.fmy = b.my;
    }
    return p;
}

sem::CutBatch cut_batch(sem_ctx* ctx, sem::Part& pt, int cur) {
    sem::CutBatch B{};
    for (int side = 0; side < 2; ++side)
        if (side == 0 ? pt.cutL : pt.cutR)
            for (int bi = 0; bi < (int)pt.boxes.size() && B.n < 4; ++bi) B.c[B.n++] = cut_params(ctx, pt, side, bi, cur);
    return B;
}

sem::PmlParams pml_params(sem_ctx* ctx, sem::Part& pt, int cur) {
    sem::PmlBox& m = pt.pml;
    Box& b = pt.boxes[m.box];
    sem::PmlParams p{};
    p.N = b.N;
    p.NX = b.NX;
    p.NY = b.NY;
    p.NZ = b.NZ;
    p.PX = b.PX;
    p.nelx = b.d.nel[0];
    p.nely = b.d.nel[1];
    p.nelz = b.d.nel[2];
    p.elems = m.elems;
    p.n_el = m.n_el;
    p.P = b.P[cur];
    p.W = b.W;
    p.Pn = b.P[1 - cur];
    p.Wn = b.W;
    p.psi_old = m.psi[cur];
    p.psi_new = m.psi[1 - cur];
    p.phi = m.phi;
    p.da = m.da;
    p.tx = m.tab[0];
    p.ty = m.tab[1];
    p.tz = m.tab[2];
    for (int i = 0; i <= b.N; ++i) {
        p.w[i] = m.w[i];
        for (int j = 0; j <= b.N; ++j) p.D[i][j] = m.D[(size_t)i * (b.N + 1) + j];
    }
    for (int d = 0; d < 3; ++d) p.s2h[d] = 2.0 / b.h[d];
    p.jac = 0.125 * b.h[0] * b.h[1] * b.h[2];
    p.c2 = b.d.c * b.d.c;
    p.dt = ctx->dt;
    p.inv_dt = 1.0 / ctx->dt;
    p.cutL = b.cutL ? 1 : 0;
    p.seg_start = m.seg_start;
    p.seg_len = m.seg_len;
    p.n_seg = m.n_seg;
    return p;
}

// enqueue one step with parity `cur` on ctx->stream; returns the number of kernel launches
int enqueue_step(sem_ctx* ctx, int cur, bool prof) {
    cudaStream_t s = ctx->stream;
    int nl = 0;
    auto mark = [&](int which, bool begin, cudaStream_t on) {
        if (!prof) return;
        static thread_local cudaEvent_t pend[4] = {nullptr, nullptr, nullptr, nullptr};
        cudaEvent_t e;
        if (ctx->ev_pool.empty()) {
            cudaEventCreate(&e);
        } else {
            e = ctx->ev_pool.back();
            ctx->ev_pool.pop_back();
        }
        cudaEventRecord(e, on);
        if (begin) pend[which] = e;
        else ctx->ev_pending.push_back({which, {pend[which], e}});
    };
    // modal ROM (a2-a4) and SIPG interface (a8) only read p^{n+1}: with both present the modal kernel
    // runs on the auxiliary stream, concurrently with the interface kernels (fork/join by events, also
    // inside the captured graph)
    // The modal ROM (a2-a4), the PML auxiliaries and the SIPG interface (a8) only read p^{n+1} (and
    // w^n): with interface work present the first two run on the auxiliary stream, concurrently with
    // the interface kernels (event fork/join, also inside the captured graph).
    bool any_pm = false, any_pml = false;
    for (auto& pt : ctx->parts) {
        any_pm = any_pm || pt.pm.on;
        any_pml = any_pml || pt.pml.on;
    }
    const bool fork = (any_pm || any_pml) && ctx->itf_on;
    cudaStream_t ms = s;
    if (fork) {
        cudaEventRecord(ctx->ev_mfork, s);
        cudaStreamWaitEvent(ctx->aux, ctx->ev_mfork, 0);
        ms = ctx->aux;
    }
    if (any_pm) {
        mark(2, true, ms);
        for (auto& pt : ctx->parts)
            if (pt.pm.on) {
                sem::launch_modal(modal_params(ctx, pt, cur), ms);
                ++nl;
            }
        mark(2, false, ms);
    }
    // PML auxiliaries and the PML acceleration (reads p^{n+1} and w^n: before the volume kernel)
    if (any_pml) {
        mark(3, true, ms);
        for (auto& pt : ctx->parts)
            if (pt.pml.on) {
                sem::launch_pml_elements(pml_params(ctx, pt, cur), ms);
                ++nl;
            }
        mark(3, false, ms);
    }
    if (fork) cudaEventRecord(ctx->ev_mjoin, ctx->aux);
    if (ctx->itf_on) {
        mark(1, true, s);
        for (auto& pt : ctx->parts) {
            if (pt.itf.general) {   // curved boxes: the face terms go straight into the residuals
                sem::GIfaceParams gp = pt.itf.gprm;
                gp.Pf = pt.boxes[pt.itf.fine].P[cur];
                gp.Pc = pt.boxes[pt.itf.coarse].P[cur];
                sem::launch_iface_general(gp, s);
                ++nl;
                continue;
            }
            sem::IfaceParams ip = pt.itf.prm;
            ip.Pf = pt.boxes[pt.itf.fine].P[cur];
            ip.Pc = pt.boxes[pt.itf.coarse].P[cur];
            ip.dzf = dzf_active(ctx, pt) ? pt.itf.dzf : nullptr;
            nl += sem::launch_iface(ip, s);
        }
        mark(1, false, s);
    }
    if (fork) cudaStreamWaitEvent(s, ctx->ev_mjoin, 0);
    const bool slabs = ctx->world > 1;
    if (slabs) {
        for (auto& pt : ctx->parts) {
            sem::CutBatch B = cut_batch(ctx, pt, cur);
            sem::launch_cut_partial(B, s);
            nl += B.n ? 1 : 0;
        }
        if (ctx->emulate) {   // device copies between the slabs of this context
            for (size_t r = 0; r < ctx->parts.size(); ++r) {
                sem::Part& pt = ctx->parts[r];
                const size_t bytes = (size_t)pt.xcount * 8;
                if (pt.cutL) cudaMemcpyAsync(pt.recv[0], ctx->parts[r - 1].send[1], bytes, cudaMemcpyDeviceToDevice, s);
                if (pt.cutR) cudaMemcpyAsync(pt.recv[1], ctx->parts[r + 1].send[0], bytes, cudaMemcpyDeviceToDevice, s);
            }
        } else {              // NCCL on the comm stream, overlapped with the volume kernels
            NcclApi& api = nccl_api();
            sem::Part& pt = ctx->parts[0];
            cudaEventRecord(ctx->ev_fork, s);
            cudaStreamWaitEvent(ctx->comm, ctx->ev_fork, 0);
            api.groupStart();
            if (pt.cutL) {
                api.send(pt.send[0], pt.xcount, kNcclDouble, ctx->rank - 1, ctx->nccl, ctx->comm);
                api.recv(pt.recv[0], pt.xcount, kNcclDouble, ctx->rank - 1, ctx->nccl, ctx->comm);
            }
            if (pt.cutR) {
                api.send(pt.send[1], pt.xcount, kNcclDouble, ctx->rank + 1, ctx->nccl, ctx->comm);
                api.recv(pt.recv[1], pt.xcount, kNcclDouble, ctx->rank + 1, ctx->nccl, ctx->comm);
            }
            api.groupEnd();
            cudaEventRecord(ctx->ev_join, ctx->comm);
        }
    }
    mark(0, true, s);
    {
        // persistent volume launches: both boxes of a slab in one launch when the degree pair is
        // instantiated (5/3 of configs 2-4), else one launch per box; each has its own scheduler pair
        std::vector<sem::VolLaunch> ls;
        for (auto& pt : ctx->parts) {
            const int nb = (int)pt.boxes.size();
            if (nb == 2 && sem::volume_pair_supported(pt.boxes[0].N, pt.boxes[1].N) && !pt.boxes[0].curved &&
                !pt.boxes[1].curved) {
                sem::VolLaunch L{};
                L.nbox = 2;
                L.box[0] = vol_params(ctx, pt, 0, cur);
                L.box[1] = vol_params(ctx, pt, 1, cur);
                ls.push_back(L);
            } else {
                for (int bi = 0; bi < nb; ++bi) {
                    if (pt.boxes[bi].curved) continue;   // element-scatter path below
                    sem::VolLaunch L{};
                    L.nbox = 1;
                    L.box[0] = vol_params(ctx, pt, bi, cur);
                    ls.push_back(L);
                }
            }
        }
        for (size_t i = 0; i < ls.size(); ++i) {
            ls[i].sched = ctx->d_sched + 2 * (i % sem_ctx::kSchedPairs);
            ls[i].step = ctx->d_step;
            ls[i].bump_step = i + 1 == ls.size() ? 1 : 0;
            // NCCL's send/recv kernel cannot co-reside with a volume CTA (smem, registers): keep a few SMs
            // free so the cut-plane exchange overlaps the volume launch instead of waiting for its end
            ls[i].reserve_sms = nccl_mode(ctx) ? 4 : 0;
            ls[i].ty = ctx->vol_ty;
            sem::launch_volume(ls[i], s);
            ++nl;
        }
        // curved boxes: element-by-element residual + nodal update (no structured volume launch)
        for (auto& pt : ctx->parts)
            for (int bi = 0; bi < (int)pt.boxes.size(); ++bi)
                if (pt.boxes[bi].curved) {
                    const sem::CurvedParams cp = curved_params(ctx, pt, bi, cur);
                    sem::launch_curved(cp, s);
                    nl += cp.pwd ? 3 : 2;
                }
        if (ls.empty()) {
            sem::launch_step_bump(ctx->d_step, s);
            ++nl;
        }
    }
    mark(0, false, s);
    if (slabs) {
        if (!ctx->emulate) cudaStreamWaitEvent(s, ctx->ev_join, 0);
        for (auto& pt : ctx->parts) {
            sem::CutBatch B = cut_batch(ctx, pt, cur);
            sem::launch_cut_fixup(B, s);
            nl += B.n ? 1 : 0;
        }
    }
    for (auto& pt : ctx->parts)
        if (pt.pml.on) {
            sem::launch_pml_fixup(pml_params(ctx, pt, cur), s);
            ++nl;
        }
    return nl;
}

sem_status reset_dynamic(sem_ctx* ctx) {
    CU(cudaMemsetAsync(ctx->d_step, 0, sizeof(long long), ctx->stream));
    CU(cudaMemsetAsync(ctx->d_sched, 0, 2 * sem_ctx::kSchedPairs * sizeof(unsigned), ctx->stream));
    for (auto& pt : ctx->parts) {
        if (!pt.pm.on) continue;
        const size_t nm = (size_t)pt.pm.n_pmut * pt.pm.n_modes;
        CU(cudaMemsetAsync(pt.pm.q, 0, nm * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(pt.pm.qd, 0, nm * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(pt.pm.qdd, 0, nm * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(pt.pm.phi, 0, pt.pm.n_pmut * sizeof(double), ctx->stream));
        Box& b = pt.boxes[pt.pm.box];
        CU(cudaMemsetAsync(pt.pm.F, 0, b.NX * b.NY * sizeof(double), ctx->stream));
    }
    for (auto& pt : ctx->parts) {
        sem::PmlBox& m = pt.pml;
        if (!m.on) continue;
        Box& b = pt.boxes[m.box];
        const size_t nl = (size_t)(b.N + 1) * (b.N + 1) * (b.N + 1);
        CU(cudaMemsetAsync(m.phi, 0, (size_t)m.n_el * 3 * nl * sizeof(double), ctx->stream));
        for (int k = 0; k < 2; ++k) CU(cudaMemsetAsync(m.psi[k], 0, (size_t)b.nalloc() * sizeof(double), ctx->stream));
        CU(cudaMemsetAsync(m.da, 0, (size_t)b.nalloc() * sizeof(double), ctx->stream));
    }
    ctx->step = 0;
    dzf_refresh(ctx);   // the state changed: the fine face's d_z p follows it
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

// owner slab of global lattice row gy of box bi (a shared cut row belongs to the lower slab)
int owner_part(sem_ctx* ctx, int bi, long long gy) {
    for (size_t r = 0; r < ctx->parts.size(); ++r) {
        const Box& b = ctx->parts[r].boxes[bi];
        if (gy >= b.gy0 && gy < b.gy0 + b.NY) return (int)r;
    }
    return -1;
}

// One y-slab (rows y_skip .. NY-1 of every z-plane) between the pitched device layout and the
// lexicographic host layout of the global box (x fastest), as one 3D copy.
cudaError_t copy_slab(double* host, double* dev, const Box& b, long long NYg, long long gy0, long long y_skip,
                      bool to_host, cudaStream_t s) {
    cudaMemcpy3DParms m = {};
    const cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)b.NX * 8, (size_t)b.NX * 8, (size_t)NYg);
    const cudaPitchedPtr dp = make_cudaPitchedPtr(dev, (size_t)b.PX * 8, (size_t)b.NX * 8, (size_t)b.NY);
    m.extent = make_cudaExtent((size_t)b.NX * 8, (size_t)(b.NY - y_skip), (size_t)b.NZ);
    if (to_host) {
        m.srcPtr = dp;
        m.srcPos = make_cudaPos(0, (size_t)y_skip, 0);
        m.dstPtr = hp;
        m.dstPos = make_cudaPos(0, (size_t)(gy0 + y_skip), 0);
        m.kind = cudaMemcpyDeviceToHost;
    } else {
        m.srcPtr = hp;
        m.srcPos = make_cudaPos(0, (size_t)(gy0 + y_skip), 0);
        m.dstPtr = dp;
        m.dstPos = make_cudaPos(0, (size_t)y_skip, 0);
        m.kind = cudaMemcpyHostToDevice;
    }
    return cudaMemcpy3DAsync(&m, s);
}

// exchange buffers: per box one NX x NZ cut plane + 2 NX for the coarse SIPG row (sized always) + one
// NX x NZ plane of PML acceleration for the PML box (after sem_pml_attach)
sem_status setup_exchange(sem_ctx* ctx, sem::Part& pt) {
    pt.xoff.clear();
    long long off = 0;
    for (int bi = 0; bi < (int)pt.boxes.size(); ++bi) {
        const Box& b = pt.boxes[bi];
        pt.xoff.push_back(off);
        off += b.NX * b.NZ + 2 * b.NX + ((pt.pml.on && pt.pml.box == bi) ? b.NX * b.NZ : 0);
    }
    pt.xcount = off;
    for (int s = 0; s < 2; ++s) {   // (buffers of an earlier layout stay allocated until sem_destroy)
        if (dalloc(ctx, &pt.send[s], (size_t)off) || dalloc(ctx, &pt.recv[s], (size_t)off)) return SEM_E_OOM;
        CU(cudaMemsetAsync(pt.send[s], 0, (size_t)off * 8, ctx->stream));
        CU(cudaMemsetAsync(pt.recv[s], 0, (size_t)off * 8, ctx->stream));
    }
    return SEM_OK;
}

sem_status setup_part_buffers(sem_ctx* ctx, sem::Part& pt) {
    for (auto& b : pt.boxes) {
        const size_t n = (size_t)b.nalloc();
        if (dalloc(ctx, &b.P[0], n) || dalloc(ctx, &b.P[1], n) || dalloc(ctx, &b.W, n)) return SEM_E_OOM;
        CU(cudaMemsetAsync(b.P[0], 0, n * 8, ctx->stream));
        CU(cudaMemsetAsync(b.P[1], 0, n * 8, ctx->stream));
        CU(cudaMemsetAsync(b.W, 0, n * 8, ctx->stream));
        if (upload(ctx, &b.xc, b.xh) || upload(ctx, &b.yc, b.yh) || upload(ctx, &b.mx, b.mxh) ||
            upload(ctx, &b.my, b.myh))
            return SEM_E_CUDA;
        const int TY = sem::volume_tile_y(ctx->world > 1 || ctx->parts.size() > 1);
        ctx->vol_ty = TY;
        sem::volume_prepare(b.N, TY);
        if (pt.boxes.size() == 2) sem::volume_pair_prepare(pt.boxes[0].N, pt.boxes[1].N, TY);
        if (!make_map(&b.tmP[0], b.P[0], b, sem::vol_pbox_w(b.N), TY + 2 * b.N) ||
            !make_map(&b.tmP[1], b.P[1], b, sem::vol_pbox_w(b.N), TY + 2 * b.N) ||
            !make_map(&b.tmW, b.W, b, sem::vol_wbox_w(b.N), TY) ||
            !make_map(&b.tmPw[0], b.P[0], b, sem::vol_wbox_w(b.N), TY) ||
            !make_map(&b.tmPw[1], b.P[1], b, sem::vol_wbox_w(b.N), TY))
            return fail(ctx, SEM_E_CUDA, "cuTensorMapEncodeTiled failed");
    }
    return setup_exchange(ctx, pt);
}

// the affine vertex lattice of a structured box (element-scatter path without set vertices)
void affine_lattice(Box& b, const sem_box_desc& g) {
    const int nx = g.nel[0] + 1, ny = g.nel[1] + 1, nz = g.nel[2] + 1;
    b.vlat_h.resize((size_t)3 * nx * ny * nz);
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int ijk[3] = {i, j, k};
                for (int d = 0; d < 3; ++d)
                    b.vlat_h[3 * ((size_t)i + (size_t)nx * ((size_t)j + (size_t)ny * k)) + d] =
                        g.origin[d] + g.extent[d] * ijk[d] / g.nel[d];
            }
}

// host trilinear map of an element: J[i][j] = dX_i / dxi_j at xi (vertex v = i + 2j + 4k at reference
// corner (2i-1, 2j-1, 2k-1))
void trilinear_jacobian(const double* V, const double xi[3], double J[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) J[i][j] = 0.0;
    for (int v = 0; v < 8; ++v) {
        const double s0 = (v & 1) ? 1.0 : -1.0, s1 = (v & 2) ? 1.0 : -1.0, s2 = (v & 4) ? 1.0 : -1.0;
        const double f0 = 1.0 + s0 * xi[0], f1 = 1.0 + s1 * xi[1], f2 = 1.0 + s2 * xi[2];
        const double dN[3] = {0.125 * s0 * f1 * f2, 0.125 * s1 * f0 * f2, 0.125 * s2 * f0 * f1};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) J[i][j] += dN[j] * V[3 * v + i];
    }
}

// x = J^-1 b (Cramer's rule; J is a positive-Jacobian element map)
void solve3(const double J[3][3], const double b[3], double x[3]) {
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    for (int c = 0; c < 3; ++c) {
        double M[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) M[i][j] = (j == c) ? b[i] : J[i][j];
        x[c] = (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0])) / det;
    }
}

// ell_j'(t) of the Lagrange basis on nodes x: sum_m 1/(x_j - x_m) prod_{k != j, m} (t - x_k)/(x_j - x_k)
std::vector<double> lagrange_deriv_at(const std::vector<double>& x, double t) {
    const int n = (int)x.size();
    std::vector<double> d(n, 0.0);
    for (int j = 0; j < n; ++j)
        for (int m = 0; m < n; ++m) {
            if (m == j) continue;
            double pr = 1.0 / (x[j] - x[m]);
            for (int k = 0; k < n; ++k)
                if (k != j && k != m) pr *= (t - x[k]) / (x[j] - x[k]);
            d[j] += pr;
        }
    return d;
}

// General non-conforming interface between two curved (element-scatter) boxes: Algorithm 3 on the
// GPU (sem_face_match: fine +z faces vs coarse -z faces) and per quadrature point the fine face
// weight W_q = w_a w_b |J_s|, the outward unit normal n+, J_F^-1 n+ at the fine node, J_C^-1 n+ and the
// coarse 1D basis values / derivatives at x_hat^- (reading R9).
sem_status build_general_interface(sem_ctx* ctx, int fb, int cb, double gamma) {
    sem::Part& pt = ctx->parts[0];
    Box& F = pt.boxes[fb];
    Box& C = pt.boxes[cb];
    const sem_box_desc& gF = ctx->gdesc[fb];
    const sem_box_desc& gC = ctx->gdesc[cb];
    const int Nf = gF.degree, Nc = gC.degree, q1 = Nf + 1, nq = q1 * q1, c1 = Nc + 1;
    auto verts_of = [](const Box& b, const sem_box_desc& g, int ex, int ey, int ez, double* out) {
        const long long nx = g.nel[0] + 1, ny = g.nel[1] + 1;
        for (int v = 0; v < 8; ++v) {
            const long long vx = ex + (v & 1), vy = ey + ((v >> 1) & 1), vz = ez + (v >> 2);
            for (int i = 0; i < 3; ++i) out[3 * v + i] = b.vlat_h[3 * (vx + nx * (vy + ny * vz)) + i];
        }
    };
    const int nfF = gF.nel[0] * gF.nel[1], nfC = gC.nel[0] * gC.nel[1];
    std::vector<double> fv((size_t)24 * nfF), cv((size_t)24 * nfC);
    std::vector<int> ff(nfF, 5), cf(nfC, 4);
    for (int ey = 0; ey < gF.nel[1]; ++ey)
        for (int ex = 0; ex < gF.nel[0]; ++ex) verts_of(F, gF, ex, ey, gF.nel[2] - 1, &fv[(size_t)24 * (ex + gF.nel[0] * ey)]);
    for (int ey = 0; ey < gC.nel[1]; ++ey)
        for (int ex = 0; ex < gC.nel[0]; ++ex) verts_of(C, gC, ex, ey, 0, &cv[(size_t)24 * (ex + gC.nel[0] * ey)]);
    const sem_face_set fs{nfF, fv.data(), ff.data()}, cs{nfC, cv.data(), cf.data()};
    const long long nqp = (long long)nfF * nq;
    std::vector<long long> owner((size_t)nqp);
    std::vector<double> xim((size_t)3 * nqp);
    CU(cudaStreamSynchronize(ctx->stream));
    // normal filter |n+ + n-| < 0.25 (opposite up to ~14 degrees: a curved interface's matching faces
    // need not have parallel centre normals; Newton containment decides)
    const sem_status ms = sem_face_match(ctx->device, &fs, &cs, Nf, 0.25, owner.data(), xim.data(), nullptr);
    if (ms == SEM_E_UNMATCHED) return fail(ctx, SEM_E_UNMATCHED, "orphan interface quadrature point (Algorithm 3)");
    if (ms != SEM_OK) return fail(ctx, ms, "interface face matching failed");
    std::vector<double> xf, wf, xc, wc;
    gll_rule(Nf, xf, wf);
    gll_rule(Nc, xc, wc);
    const std::vector<double> Df = deriv_matrix(xf);
    std::vector<long long> fbase((size_t)nqp), cbase((size_t)nqp);
    std::vector<double> geo((size_t)7 * nqp), bas((size_t)6 * c1 * nqp);
    for (int f = 0; f < nfF; ++f) {
        const int ex = f % gF.nel[0], ey = f / gF.nel[0], ez = gF.nel[2] - 1;
        for (int q = 0; q < nq; ++q) {
            const long long i = (long long)f * nq + q;
            const int a = q % q1, b = q / q1;
            const double xi[3] = {xf[a], xf[b], 1.0};
            double J[3][3];
            trilinear_jacobian(&fv[(size_t)24 * f], xi, J);
            // n+ |J_s| = J[:,0] x J[:,1] (outward: +zeta for a positive Jacobian)
            double cr[3] = {J[1][0] * J[2][1] - J[2][0] * J[1][1], J[2][0] * J[0][1] - J[0][0] * J[2][1],
                            J[0][0] * J[1][1] - J[1][0] * J[0][1]};
            const double js = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
            for (double& v : cr) v /= js;
            double gp[3], gm[3];
            solve3(J, cr, gp);
            const long long oc = owner[(size_t)i];
            const int cex = (int)(oc % gC.nel[0]), cey = (int)(oc / gC.nel[0]);
            const double* xm = &xim[(size_t)3 * i];
            double JC[3][3];
            trilinear_jacobian(&cv[(size_t)24 * oc], xm, JC);
            solve3(JC, cr, gm);
            double* G = &geo[(size_t)7 * i];
            G[0] = wf[a] * wf[b] * js;
            for (int k = 0; k < 3; ++k) {
                G[1 + k] = gp[k];
                G[4 + k] = gm[k];
            }
            double* Bq = &bas[(size_t)6 * c1 * i];
            for (int d = 0; d < 3; ++d) {
                const std::vector<double> l = lagrange_at(xc, xm[d]), dl = lagrange_deriv_at(xc, xm[d]);
                for (int k = 0; k <= Nc; ++k) {
                    Bq[(2 * d) * c1 + k] = l[k];
                    Bq[(2 * d + 1) * c1 + k] = dl[k];
                }
            }
            fbase[(size_t)i] = ((long long)Nf * ez * F.NY + (long long)Nf * ey) * F.PX + (long long)Nf * ex;
            cbase[(size_t)i] = ((long long)0 * C.NY + (long long)Nc * cey) * C.PX + (long long)Nc * cex;
        }
    }
    sem::GIfaceParams& g = pt.itf.gprm;
    g = sem::GIfaceParams{};
    g.Nf = Nf;
    g.Nc = Nc;
    g.nqp = nqp;
    g.resF = F.res;
    g.resC = C.res;
    g.PXf = F.PX;
    g.NYf = F.NY;
    g.PXc = C.PX;
    g.NYc = C.NY;
    long long *dfb = nullptr, *dcb = nullptr;
    double *dgeo = nullptr, *dbas = nullptr;
    if (upload(ctx, &dfb, fbase) || upload(ctx, &dcb, cbase) || upload(ctx, &dgeo, geo) || upload(ctx, &dbas, bas))
        return SEM_E_CUDA;
    g.fbase = dfb;
    g.cbase = dcb;
    g.geo = dgeo;
    g.bas = dbas;
    for (int i = 0; i <= Nf; ++i)
        for (int j = 0; j <= Nf; ++j) g.Df[i][j] = Df[(size_t)i * q1 + j];
    g.gamma = gamma;
    g.NZf_dbg = F.NZ;
    g.cf2 = gF.c * gF.c;
    g.cc2 = gC.c * gC.c;
    pt.itf.general = true;
    pt.itf.on = true;
    pt.itf.fine = fb;
    pt.itf.coarse = cb;
    F.iface_side = +1;
    C.iface_side = -1;
    return SEM_OK;
}

// Coupling table of a curved box (reading R4, Eqs. 11-12): B_{k,m,j} = sum over the -z faces of the
// face quadrature weight w_a w_b |J_s| (J_s of the trilinear map at zeta = -1) times S_{k,m} at the
// node's physical position (reading R19), for every face node of every PMUT with some S != 0.
sem_status pmut_tables(sem_ctx* ctx, sem::Part& pt, Box& b, const sem_pmut_desc& pd, const std::vector<int>& ks) {
    const sem_box_desc& g = b.d;
    const int N = b.N, M = pd.n_modes, KL = (int)ks.size();
    std::vector<double> x, w;
    gll_rule(N, x, w);
    const long long nx = g.nel[0] + 1, ny = g.nel[1] + 1;
    // assembled face weight and position of every z = 0 lattice node
    std::vector<double> fw((size_t)b.NX * b.NY, 0.0), fx((size_t)b.NX * b.NY), fy((size_t)b.NX * b.NY);
    for (int ey = 0; ey < g.nel[1]; ++ey)
        for (int ex = 0; ex < g.nel[0]; ++ex) {
            double V[24];
            for (int v = 0; v < 8; ++v) {
                const long long vx = ex + (v & 1), vy = ey + ((v >> 1) & 1), vz = (v >> 2);
                for (int i = 0; i < 3; ++i) V[3 * v + i] = b.vlat_h[3 * (vx + nx * (vy + ny * vz)) + i];
            }
            for (int bb = 0; bb <= N; ++bb)
                for (int a = 0; a <= N; ++a) {
                    const double xi[3] = {x[a], x[bb], -1.0};
                    double J[3][3];
                    trilinear_jacobian(V, xi, J);
                    const double cx = J[1][0] * J[2][1] - J[2][0] * J[1][1], cy = J[2][0] * J[0][1] - J[0][0] * J[2][1],
                                 cz = J[0][0] * J[1][1] - J[1][0] * J[0][1];
                    double X[3] = {0, 0, 0};
                    for (int v = 0; v < 8; ++v) {
                        const double sh = 0.125 * (1.0 + ((v & 1) ? 1 : -1) * xi[0]) * (1.0 + ((v & 2) ? 1 : -1) * xi[1]) *
                                          (1.0 + ((v & 4) ? 1 : -1) * xi[2]);
                        for (int i = 0; i < 3; ++i) X[i] += sh * V[3 * v + i];
                    }
                    const size_t j = (size_t)(N * ey + bb) * b.NX + (N * ex + a);
                    fw[j] += w[a] * w[bb] * std::sqrt(cx * cx + cy * cy + cz * cz);
                    fx[j] = X[0];
                    fy[j] = X[1];
                }
        }
    std::vector<int> off(KL + 1, 0);
    std::vector<long long> idx;
    std::vector<double> B;
    std::vector<int> used((size_t)b.NX * b.NY, -1);
    const double a = pd.side;
    // candidate nodes of a membrane: the face nodes whose PHYSICAL position lies in its square, whatever
    // the vertex lattice does to the node positions (a mapped lattice, e.g. square -> disc, moves nodes by
    // several elements).  Membranes are binned on a uniform grid of cell size a (a square meets <= 4
    // cells per axis pair), every node looks its cell up; nodes are visited in lattice order (y, then x),
    // so each membrane's rows keep that order.
    double bx0 = 1e300, by0 = 1e300, bx1 = -1e300, by1 = -1e300;
    for (int l = 0; l < KL; ++l) {
        const int k = ks[l];
        bx0 = std::min(bx0, pd.center[2 * k] - 0.5 * a);
        by0 = std::min(by0, pd.center[2 * k + 1] - 0.5 * a);
        bx1 = std::max(bx1, pd.center[2 * k] + 0.5 * a);
        by1 = std::max(by1, pd.center[2 * k + 1] + 0.5 * a);
    }
    const long long gnx = std::max<long long>(1, (long long)std::ceil((bx1 - bx0) / a)) + 1,
                    gny = std::max<long long>(1, (long long)std::ceil((by1 - by0) / a)) + 1;
    std::vector<std::vector<int>> cell((size_t)(gnx * gny));
    for (int l = 0; l < KL; ++l) {
        const int k = ks[l];
        const double x0 = pd.center[2 * k] - 0.5 * a, y0 = pd.center[2 * k + 1] - 0.5 * a;
        const long long cx0 = std::max<long long>(0, (long long)std::floor((x0 - bx0) / a) - 1),
                        cy0 = std::max<long long>(0, (long long)std::floor((y0 - by0) / a) - 1);
        for (long long cy = cy0; cy <= std::min(gny - 1, cy0 + 3); ++cy)
            for (long long cx = cx0; cx <= std::min(gnx - 1, cx0 + 3); ++cx) cell[(size_t)(cy * gnx + cx)].push_back(l);
    }
    std::vector<std::vector<long long>> midx(KL);
    std::vector<std::vector<double>> mB(KL);
    std::vector<double> row(M);
    for (long long jy = 0; jy < b.NY; ++jy)
        for (long long jx = 0; jx < b.NX; ++jx) {
            const size_t j = (size_t)jy * b.NX + (size_t)jx;
            if (!(fx[j] >= bx0 && fx[j] <= bx1 && fy[j] >= by0 && fy[j] <= by1)) continue;
            const long long cx = std::min(gnx - 1, (long long)std::floor((fx[j] - bx0) / a)),
                            cy = std::min(gny - 1, (long long)std::floor((fy[j] - by0) / a));
            for (int l : cell[(size_t)(cy * gnx + cx)]) {
                const int k = ks[l];
                const double xl = fx[j] - (pd.center[2 * k] - 0.5 * a), yl = fy[j] - (pd.center[2 * k + 1] - 0.5 * a);
                if (!(xl >= 0 && xl <= a && yl >= 0 && yl <= a)) continue;
                bool nz = false;
                for (int m = 0; m < M; ++m) {
                    const double S = pd.shape_fn
                                         ? pd.shape_fn(k, m, fx[j] - pd.center[2 * k], fy[j] - pd.center[2 * k + 1], pd.shape_user)
                                         : std::sin(pd.mode_mn[2 * m] * M_PI * xl / a) * std::sin(pd.mode_mn[2 * m + 1] * M_PI * yl / a);
                    if (!std::isfinite(S)) return fail(ctx, SEM_E_ARG, "shape_fn returned a non-finite value");
                    row[m] = fw[j] * S;
                    nz = nz || S != 0.0;
                }
                if (!nz) continue;
                if (used[j] >= 0) return fail(ctx, SEM_E_ARG, "membranes overlap");
                used[j] = l;
                midx[l].push_back((long long)(j / b.NX) * b.PX + (long long)(j % b.NX));   // pitched, plane z = 0
                mB[l].insert(mB[l].end(), row.begin(), row.end());
            }
        }
    for (int l = 0; l < KL; ++l) {
        idx.insert(idx.end(), midx[l].begin(), midx[l].end());
        B.insert(B.end(), mB[l].begin(), mB[l].end());
        off[l + 1] = (int)idx.size();
        if (off[l + 1] == off[l]) return fail(ctx, SEM_E_ARG, "membrane with no face node");
    }
    if (upload(ctx, &pt.pm.toff, off) || upload(ctx, &pt.pm.tidx, idx) || upload(ctx, &pt.pm.tB, B)) return SEM_E_CUDA;
    return SEM_OK;
}

// Incident plane wave on the +z face of a curved box (reading R13 on a vertex lattice): per top-face
// node the assembled face weight W_j = sum_F w_a w_b |J_s| and the physical position from the trilinear
// maps of the top element layer; x_ref = the corner of the face's bounding rectangle the wavefront
// reaches first; tables pwd_j = k.(x_j - x_ref)/c and pwf_j = c A (1 - n.k) W_j.  The face must be planar
// (n = +z), as the boxes' faces are in every supported configuration.
sem_status curved_plane_wave(sem_ctx* ctx, Box& b, double amp, const double kk[3]) {
    const sem_box_desc& g = b.d;
    const int N = b.N;
    std::vector<double> x, w;
    gll_rule(N, x, w);
    const long long nx = g.nel[0] + 1, ny = g.nel[1] + 1;
    const size_t nn = (size_t)b.NX * b.NY;
    std::vector<double> fw(nn, 0.0), fx(nn), fy(nn), fz(nn);
    const int ez = g.nel[2] - 1;
    for (int ey = 0; ey < g.nel[1]; ++ey)
        for (int ex = 0; ex < g.nel[0]; ++ex) {
            double V[24];
            for (int v = 0; v < 8; ++v) {
                const long long vx = ex + (v & 1), vy = ey + ((v >> 1) & 1), vz = ez + (v >> 2);
                for (int i = 0; i < 3; ++i) V[3 * v + i] = b.vlat_h[3 * (vx + nx * (vy + ny * vz)) + i];
            }
            for (int bb = 0; bb <= N; ++bb)
                for (int a = 0; a <= N; ++a) {
                    const double xi[3] = {x[a], x[bb], 1.0};
                    double J[3][3];
                    trilinear_jacobian(V, xi, J);
                    const double cx = J[1][0] * J[2][1] - J[2][0] * J[1][1], cy = J[2][0] * J[0][1] - J[0][0] * J[2][1],
                                 cz = J[0][0] * J[1][1] - J[1][0] * J[0][1];
                    double X[3] = {0, 0, 0};
                    for (int v = 0; v < 8; ++v) {
                        const double sh = 0.125 * (1.0 + ((v & 1) ? 1 : -1) * xi[0]) * (1.0 + ((v & 2) ? 1 : -1) * xi[1]) *
                                          (1.0 + ((v & 4) ? 1 : -1) * xi[2]);
                        for (int i = 0; i < 3; ++i) X[i] += sh * V[3 * v + i];
                    }
                    const size_t j = (size_t)(N * ey + bb) * b.NX + (N * ex + a);
                    fw[j] += w[a] * w[bb] * std::sqrt(cx * cx + cy * cy + cz * cz);
                    fx[j] = X[0];
                    fy[j] = X[1];
                    fz[j] = X[2];
                }
        }
    double lo[2] = {1e300, 1e300}, hi[2] = {-1e300, -1e300}, zmin = 1e300, zmax = -1e300;
    for (size_t j = 0; j < nn; ++j) {
        lo[0] = std::min(lo[0], fx[j]);
        hi[0] = std::max(hi[0], fx[j]);
        lo[1] = std::min(lo[1], fy[j]);
        hi[1] = std::max(hi[1], fy[j]);
        zmin = std::min(zmin, fz[j]);
        zmax = std::max(zmax, fz[j]);
    }
    if (zmax - zmin > 1e-9 * std::max(hi[0] - lo[0], hi[1] - lo[1]))
        return fail(ctx, SEM_E_ARG, "plane wave on a curved box: the +z face must be planar");
    double best = std::numeric_limits<double>::infinity();
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double cxr = i ? hi[0] : lo[0], cyr = j ? hi[1] : lo[1];
            const double kx = kk[0] * cxr + kk[1] * cyr + kk[2] * fz[0];
            if (kx < best) {
                best = kx;
                ctx->pw_xref_curved[0] = cxr;
                ctx->pw_xref_curved[1] = cyr;
                ctx->pw_xref_curved[2] = fz[0];
            }
        }
    std::vector<double> dl(nn), fc(nn);
    for (size_t j = 0; j < nn; ++j) {
        dl[j] = (kk[0] * (fx[j] - ctx->pw_xref_curved[0]) + kk[1] * (fy[j] - ctx->pw_xref_curved[1]) +
                 kk[2] * (fz[j] - ctx->pw_xref_curved[2])) / g.c;
        fc[j] = g.c * amp * (1.0 - kk[2]) * fw[j];
    }
    if (upload(ctx, &b.pwd, dl) || upload(ctx, &b.pwf, fc)) return SEM_E_CUDA;
    return SEM_OK;
}

}  // namespace

extern "C" {

sem_status sem_nccl_unique_id(void* out) {
    if (!out) return SEM_E_ARG;
    NcclApi& api = nccl_api();
    if (!api.ok) return SEM_E_NCCL;
    NcclUid id;
    if (api.getUniqueId(&id) != 0) return SEM_E_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return SEM_OK;
}

sem_status sem_slab_plan(const sem_box_desc* boxes, int n_boxes, int world, const sem_pmut_desc* pm,
                         long long* slab_y0) {
    if (!boxes || n_boxes < 1 || n_boxes > 2 || world < 1) return SEM_E_ARG;
    if (pm && (pm->box < 0 || pm->box >= n_boxes || !pm->center)) return SEM_E_ARG;
    std::vector<long long> cuts;
    if (!auto_plan(boxes, n_boxes, world, pm, cuts)) return SEM_E_PARTITION;
    if (slab_y0)
        for (int r = 0; r <= world; ++r) slab_y0[r] = cuts[r];
    return SEM_OK;
}

sem_status sem_mesh_create(const sem_mesh_desc* desc, sem_ctx** out) {
    if (!out) return SEM_E_ARG;
    *out = nullptr;
    if (!desc || desc->n_boxes < 1 || desc->n_boxes > 2 || !desc->boxes) return SEM_E_ARG;
    sem_ctx* ctx = new (std::nothrow) sem_ctx();
    if (!ctx) return SEM_E_OOM;
    auto bail = [&](sem_status st) {
        if (!ctx->err.empty()) fprintf(stderr, "libsem: sem_mesh_create: %s\n", ctx->err.c_str());
        sem_destroy(ctx);
        return st;
    };
    if (!(desc->dt > 0) || !std::isfinite(desc->dt)) return bail(SEM_E_ARG);
    if (desc->world < 1 || desc->rank < 0 || desc->rank >= desc->world) return bail(SEM_E_ARG);
    ctx->device = desc->device;
    ctx->flags = desc->flags;
    if (!desc->dev_alloc != !desc->dev_free) return bail(SEM_E_ARG);   // both or neither
    ctx->dev_alloc = desc->dev_alloc;
    ctx->dev_free = desc->dev_free;
    ctx->alloc_user = desc->alloc_user;
    ctx->dt = desc->dt;
    ctx->rank = desc->rank;
    ctx->world = desc->world;
    ctx->emulate = desc->world > 1 && (desc->flags & SEM_F_EMULATE_SLABS);
    if (ctx->emulate && desc->rank != 0) return bail(SEM_E_ARG);
    if (cudaSetDevice(ctx->device) != cudaSuccess) return bail(SEM_E_CUDA);
    if (desc->stream) {
        ctx->stream = (cudaStream_t)desc->stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SEM_E_CUDA);
        ctx->own_stream = true;
    }
    for (int i = 0; i < desc->n_boxes; ++i) {
        if (check_box(ctx, desc->boxes[i]) != SEM_OK) return bail(SEM_E_ARG);
        const sem_box_desc& g = desc->boxes[i];
        ctx->gdesc.push_back(g);
        ctx->gNX.push_back((long long)g.degree * g.nel[0] + 1);
        ctx->gNY.push_back((long long)g.degree * g.nel[1] + 1);
        ctx->gNZ.push_back((long long)g.degree * g.nel[2] + 1);
    }
    // slab decomposition along y: the caller's plan (sem_slab_plan) or equal slabs; the same slab
    // boundaries (in y) for all boxes
    const int G = ctx->world;
    if (desc->slab_y0) {
        ctx->cuts.assign(desc->slab_y0, desc->slab_y0 + G + 1);
    } else {
        if (ctx->gdesc[0].nel[1] % G) {
            ctx->err = "nel_y must be divisible by the number of slabs (or pass slab_y0 from sem_slab_plan)";
            return bail(SEM_E_PARTITION);
        }
        ctx->cuts = equal_plan(ctx->gdesc[0], G);
    }
    if (const char* why = plan_invalid(ctx->gdesc.data(), (int)ctx->gdesc.size(), ctx->cuts)) {
        ctx->err = why;
        return bail(SEM_E_PARTITION);
    }
    const int first = ctx->emulate ? 0 : ctx->rank;
    const int last = ctx->emulate ? G - 1 : ctx->rank;
    for (int r = first; r <= last; ++r) {
        sem::Part pt;
        pt.slab = r;
        pt.cutL = r > 0;
        pt.cutR = r < G - 1;
        for (auto& g : ctx->gdesc) {
            const long long e0 = cut_in_box(ctx->gdesc[0], g, ctx->cuts[r]), e1 = cut_in_box(ctx->gdesc[0], g, ctx->cuts[r + 1]);
            pt.boxes.push_back(make_slab(g, e0, e1 - e0, pt.cutL, pt.cutR));
        }
        ctx->parts.push_back(pt);
    }
    for (auto& pt : ctx->parts)
        if (setup_part_buffers(ctx, pt) != SEM_OK) return bail(SEM_E_OOM);
    if (dalloc(ctx, &ctx->d_step, 1) || dalloc(ctx, &ctx->d_sched, 2 * sem_ctx::kSchedPairs) || dalloc(ctx, &ctx->d_flag, 1))
        return bail(SEM_E_OOM);
    if (cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_mfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_mjoin, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking) != cudaSuccess)
        return bail(SEM_E_CUDA);
    if (nccl_mode(ctx)) {
        NcclApi& api = nccl_api();
        if (!api.ok || !desc->nccl_unique_id) {
            ctx->err = "world > 1 needs NCCL (libnccl.so.2) and an ncclUniqueId";
            return bail(SEM_E_NCCL);
        }
        if (cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking) != cudaSuccess) return bail(SEM_E_CUDA);
        NcclUid id;
        std::memcpy(&id, desc->nccl_unique_id, sizeof(id));
        if (api.commInitRank(&ctx->nccl, G, id, ctx->rank) != 0) {
            ctx->err = "ncclCommInitRank failed";
            return bail(SEM_E_NCCL);
        }
    }
    if (reset_dynamic(ctx) != SEM_OK) return bail(SEM_E_CUDA);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return bail(SEM_E_CUDA);
    *out = ctx;
    return SEM_OK;
}

sem_status sem_pmut_attach(sem_ctx* ctx, const sem_pmut_desc* pd) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (!pd) return fail(ctx, SEM_E_ARG, "null pmut desc");
    if (ctx->n_pmut) return fail(ctx, SEM_E_STATE, "PMUT array already attached");
    if (pd->box < 0 || pd->box >= (int)ctx->gdesc.size()) return fail(ctx, SEM_E_ARG, "bad box");
    if (pd->face != 4) return fail(ctx, SEM_E_ARG, "PMUTs supported on the -z face only");

    if (pd->n_pmut < 1 || pd->n_modes < 1 || pd->n_modes > sem::kMaxModes)
        return fail(ctx, SEM_E_ARG, "n_pmut >= 1 and 1 <= n_modes <= 8 required");
    if (!(pd->side > 0) || !pd->center || !pd->mode_mn || !pd->freq_hz || !pd->modal_mass || !pd->damping_ratio ||
        !pd->eta || !pd->delay_s)
        return fail(ctx, SEM_E_ARG, "missing PMUT arrays");
    if (pd->rx && !(pd->capacitance > 0)) return fail(ctx, SEM_E_ARG, "RX requires capacitance > 0");
    if (pd->n_cycles < 1 || !(pd->f0_hz > 0)) return fail(ctx, SEM_E_ARG, "bad drive");
    const sem_box_desc& g = ctx->gdesc[pd->box];
    if (g.bc[4] == SEM_BC_INTERFACE) return fail(ctx, SEM_E_ARG, "PMUT face is an interface");
    for (int m = 0; m < pd->n_modes; ++m)
        if (!(pd->modal_mass[m] > 0)) return fail(ctx, SEM_E_ARG, "modal mass must be > 0");
    const int K = pd->n_pmut, M = pd->n_modes;
    const double a = pd->side;
    // membranes must lie on the face, must not overlap, and must not touch a slab cut
    const int G = ctx->world;
    ctx->pm_lists.assign(G, {});
    for (int k = 0; k < K; ++k) {
        const double x0 = pd->center[2 * k] - 0.5 * a, y0 = pd->center[2 * k + 1] - 0.5 * a;
        if (x0 < g.origin[0] - 1e-12 * a || y0 < g.origin[1] - 1e-12 * a ||
            x0 + a > g.origin[0] + g.extent[0] + 1e-12 * a || y0 + a > g.origin[1] + g.extent[1] + 1e-12 * a)
            return fail(ctx, SEM_E_ARG, "membrane off the face");
        const int slab = membrane_slab(ctx->gdesc[0], ctx->cuts, y0, a);
        if (slab < 0) return fail(ctx, SEM_E_PARTITION, "a slab cut crosses a membrane");
        ctx->pm_lists[slab].push_back(k);
    }
    for (auto& pt : ctx->parts) {
        Box& b = pt.boxes[pd->box];
        const std::vector<int>& ks = ctx->pm_lists[pt.slab];
        pt.pm_global = ks;
        if (ks.empty()) continue;
        const int KL = (int)ks.size();
        std::vector<int> rect(4 * KL);
        std::vector<int> occ((size_t)b.NX * b.NY, -1);
        int lmax = 1;
        std::vector<std::vector<long long>> xi(KL), yi(KL);
        for (int l = 0; l < KL; ++l) {
            const int k = ks[l];
            const double x0 = pd->center[2 * k] - 0.5 * a, y0 = pd->center[2 * k + 1] - 0.5 * a;
            for (long long i = 0; i < b.NX; ++i) {
                const double xl = b.xh[i] - x0;
                if (xl >= 0 && xl <= a) xi[l].push_back(i);
            }
            for (long long j = 0; j < b.NY; ++j) {
                const double yl = b.yh[j] - y0;
                if (yl >= 0 && yl <= a) yi[l].push_back(j);
            }
            if (xi[l].empty() || yi[l].empty()) return fail(ctx, SEM_E_ARG, "membrane with no face node");
            rect[4 * l] = (int)xi[l].front();
            rect[4 * l + 1] = (int)yi[l].front();
            rect[4 * l + 2] = (int)xi[l].size();
            rect[4 * l + 3] = (int)yi[l].size();
            lmax = std::max<int>(lmax, std::max(rect[4 * l + 2], rect[4 * l + 3]));
            for (long long j : yi[l])
                for (long long i : xi[l]) {
                    int& o = occ[(size_t)j * b.NX + i];
                    if (o >= 0) return fail(ctx, SEM_E_ARG, "membranes overlap");
                    o = l;
                }
            if (!b.solid_h.empty()) {   // obstacle box: a membrane is a fluid boundary, never under a solid element
                const int N = b.N;
                for (long long j : yi[l])
                    for (long long i : xi[l])
                        for (long long ey = std::max<long long>(0, (j - 1) / N); ey <= std::min<long long>(b.d.nel[1] - 1, j / N); ++ey)
                            for (long long ex = std::max<long long>(0, (i - 1) / N); ex <= std::min<long long>(b.d.nel[0] - 1, i / N); ++ex)
                                if (b.solid_h[(size_t)ex + (size_t)b.d.nel[0] * (size_t)ey] &&
                                    i >= N * ex && i <= N * (ex + 1) && j >= N * ey && j <= N * (ey + 1))
                                    return fail(ctx, SEM_E_ARG, "membrane on the face of an obstacle element");
            }
        }
        if (pd->shape_fn && !b.verts_set)
            return fail(ctx, SEM_E_ARG, "caller-defined mode shapes need the tabulated coupling of a curved box (sem_box_set_vertices first)");
        if (b.verts_set) {   // curved box: tabulated coupling
            st = pmut_tables(ctx, pt, b, *pd, ks);
            if (st) return st;
        }
        std::vector<double> sx((size_t)KL * M * lmax, 0.0), sy((size_t)KL * M * lmax, 0.0), wx((size_t)KL * lmax, 0.0),
            wy((size_t)KL * lmax, 0.0), om2((size_t)KL * M), tzw((size_t)KL * M), im(M), et(M), dl(KL);
        for (int l = 0; l < KL; ++l) {
            const int k = ks[l];
            const double x0 = pd->center[2 * k] - 0.5 * a, y0 = pd->center[2 * k + 1] - 0.5 * a;
            for (int m = 0; m < M; ++m) {
                const int mm = pd->mode_mn[2 * m], nn = pd->mode_mn[2 * m + 1];
                for (size_t i = 0; i < xi[l].size(); ++i)
                    sx[((size_t)l * M + m) * lmax + i] = std::sin(mm * M_PI * (b.xh[xi[l][i]] - x0) / a);
                for (size_t j = 0; j < yi[l].size(); ++j)
                    sy[((size_t)l * M + m) * lmax + j] = std::sin(nn * M_PI * (b.yh[yi[l][j]] - y0) / a);
                const double om = 2.0 * M_PI * pd->freq_hz[(size_t)k * M + m];
                om2[(size_t)l * M + m] = om * om;
                tzw[(size_t)l * M + m] = 2.0 * pd->damping_ratio[m] * om;
            }
            for (size_t i = 0; i < xi[l].size(); ++i) wx[(size_t)l * lmax + i] = b.mxh[xi[l][i]];
            for (size_t j = 0; j < yi[l].size(); ++j) wy[(size_t)l * lmax + j] = b.myh[yi[l][j]];
            dl[l] = pd->delay_s[k];
        }
        for (int m = 0; m < M; ++m) {
            im[m] = 1.0 / pd->modal_mass[m];
            et[m] = pd->eta[m];
        }
        sem::Pmut& pm = pt.pm;
        pm.box = pd->box;
        pm.n_pmut = KL;
        pm.n_modes = M;
        pm.lmax = lmax;
        if (upload(ctx, &pm.rect, rect) || upload(ctx, &pm.sx, sx) || upload(ctx, &pm.sy, sy) ||
            upload(ctx, &pm.wx, wx) || upload(ctx, &pm.wy, wy) || upload(ctx, &pm.omega2, om2) ||
            upload(ctx, &pm.twozw, tzw) || upload(ctx, &pm.invmass, im) || upload(ctx, &pm.eta, et) ||
            upload(ctx, &pm.delay, dl))
            return SEM_E_CUDA;
        const size_t nm = (size_t)KL * M;
        if (dalloc(ctx, &pm.q, nm) || dalloc(ctx, &pm.qd, nm) || dalloc(ctx, &pm.qdd, nm) || dalloc(ctx, &pm.phi, KL) ||
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
    }
    ctx->n_pmut = K;
    ctx->n_modes = M;
    drop_graphs(ctx);
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status curved_setup(sem_ctx* ctx, Box& b, const sem_box_desc& g);   // below

sem_status sem_dg_interface_build(sem_ctx* ctx, int fine_box, int coarse_box, double alpha, int quad_rule) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (ctx->itf_on) return fail(ctx, SEM_E_STATE, "interface already built");
    if (quad_rule != 0 && quad_rule != 1)
        return fail(ctx, SEM_E_ARG, "quad_rule must be 0 (fine-face GLL nodes) or 1 (Gauss-Legendre points)");
    if (quad_rule == 1 && (ctx->world > 1 || ctx->parts.size() != 1))
        return fail(ctx, SEM_E_PARTITION, "the Gauss-Legendre interface rule is implemented for a single slab only");
    const int nb = (int)ctx->gdesc.size();
    if (fine_box < 0 || coarse_box < 0 || fine_box >= nb || coarse_box >= nb || fine_box == coarse_box)
        return fail(ctx, SEM_E_ARG, "bad box indices");
    if (!(alpha > 0)) return fail(ctx, SEM_E_ARG, "penalty alpha must be > 0");
    const sem_box_desc& gF = ctx->gdesc[fine_box];
    const sem_box_desc& gC = ctx->gdesc[coarse_box];
    if (gF.bc[5] != SEM_BC_INTERFACE || gC.bc[4] != SEM_BC_INTERFACE)
        return fail(ctx, SEM_E_ARG, "fine +z and coarse -z faces must be tagged SEM_BC_INTERFACE");
    const double hF[3] = {gF.extent[0] / gF.nel[0], gF.extent[1] / gF.nel[1], gF.extent[2] / gF.nel[2]};
    const double hC[3] = {gC.extent[0] / gC.nel[0], gC.extent[1] / gC.nel[1], gC.extent[2] / gC.nel[2]};
    {
        const bool cvF = ctx->parts[0].boxes[fine_box].curved, cvC = ctx->parts[0].boxes[coarse_box].curved;
        if (cvF || cvC) {   // curved boxes: general non-conforming interface (Algorithm 3 matching)
            if (!(cvF && cvC))
                return fail(ctx, SEM_E_STATE, "an interface with a curved box needs both boxes curved (set vertices)");
            if (ctx->world > 1 || ctx->parts.size() != 1)
                return fail(ctx, SEM_E_PARTITION, "the curved-box interface is implemented for a single slab only");
            if (quad_rule != 0) return fail(ctx, SEM_E_ARG, "the curved-box interface uses the GLL rule (quad_rule 0)");
            const double cbar = 2.0 * gF.c * gC.c / (gF.c + gC.c);
            const double hmin = std::min(std::min(std::min(hF[0], hF[1]), hF[2]), std::min(std::min(hC[0], hC[1]), hC[2]));
            const int Nm = std::max(gF.degree, gC.degree);
            st = build_general_interface(ctx, fine_box, coarse_box, alpha * cbar * cbar * Nm * Nm / hmin);
            if (st) return st;
            ctx->itf_on = true;
            drop_graphs(ctx);
            CU(cudaStreamSynchronize(ctx->stream));
            return SEM_OK;
        }
    }
    const double tol = 1e-9 * std::max(hF[0], hC[0]);
    for (int k = 0; k < 2; ++k) {
        if (std::fabs(gF.origin[k] - gC.origin[k]) > tol || std::fabs(gF.extent[k] - gC.extent[k]) > tol)
            return fail(ctx, SEM_E_UNMATCHED, "interface faces do not coincide laterally");
    }
    if (std::fabs(gF.origin[2] + gF.extent[2] - gC.origin[2]) > tol)
        return fail(ctx, SEM_E_UNMATCHED, "boxes do not touch in z");
    if (gF.nel[0] % gC.nel[0] || gF.nel[1] % gC.nel[1] || gF.nel[0] / gC.nel[0] != gF.nel[1] / gC.nel[1]) {
        // lattices that do not nest: both boxes move to the element-scatter path (their affine vertex
        // lattices) and take the general interface (Algorithm 3 matching, section 5.2e of DESIGN.md)
        sem::Part& pt0 = ctx->parts[0];
        if (ctx->world > 1 || ctx->parts.size() != 1 || quad_rule != 0 ||
            (pt0.pml.on && (pt0.pml.box == fine_box || pt0.pml.box == coarse_box)) ||
            (ctx->pw.on && (ctx->pw.box == fine_box || ctx->pw.box == coarse_box)))
            return fail(ctx, SEM_E_UNMATCHED,
                        "fine lattice does not nest in the coarse one (need h_c = R h_f; the general interface of "
                        "non-nested lattices is single-slab, GLL rule, without PML / plane wave on its boxes)");
        for (int bi : {fine_box, coarse_box}) {
            Box& b = pt0.boxes[bi];
            if (b.curved) continue;
            affine_lattice(b, ctx->gdesc[bi]);
            st = curved_setup(ctx, b, ctx->gdesc[bi]);
            if (st) return st;
        }
        const double cbar = 2.0 * gF.c * gC.c / (gF.c + gC.c);
        const double hmin = std::min(std::min(std::min(hF[0], hF[1]), hF[2]), std::min(std::min(hC[0], hC[1]), hC[2]));
        const int Nm = std::max(gF.degree, gC.degree);
        st = build_general_interface(ctx, fine_box, coarse_box, alpha * cbar * cbar * Nm * Nm / hmin);
        if (st) return st;
        ctx->itf_on = true;
        drop_graphs(ctx);
        CU(cudaStreamSynchronize(ctx->stream));
        return SEM_OK;
    }
    const int R = gF.nel[0] / gC.nel[0];
    for (size_t r = 1; r + 1 < ctx->cuts.size(); ++r)   // (sem_mesh_create checked every box; restated here)
        if (cut_in_box(ctx->gdesc[0], gC, ctx->cuts[r]) < 0)
            return fail(ctx, SEM_E_PARTITION, "slab cut not aligned to the coarse elements");
    std::vector<double> xf, wf, xc, wc;
    gll_rule(gF.degree, xf, wf);
    gll_rule(gC.degree, xc, wc);
    const std::vector<double> Df = deriv_matrix(xf), Dc = deriv_matrix(xc);
    const int Nf = gF.degree, Nc = gC.degree, NfR = Nf * R;
    std::vector<double> I((size_t)(NfR + 1) * (Nc + 1), 0.0);
    for (int q = 0; q <= NfR; ++q) {
        int r = q / Nf, a = q % Nf;
        if (q == NfR) {
            r = R - 1;
            a = Nf;
        }
        const double xm = (2.0 * r + xf[a] + 1.0) / R - 1.0;   // x_hat^- of the fine node
        const std::vector<double> l = lagrange_at(xc, xm);
        for (int b = 0; b <= Nc; ++b) I[(size_t)q * (Nc + 1) + b] = l[b];
    }
    const double cbar = 2.0 * gF.c * gC.c / (gF.c + gC.c);
    const double hmin = std::min(std::min(std::min(hF[0], hF[1]), hF[2]), std::min(std::min(hC[0], hC[1]), hC[2]));
    const double gamma = alpha * cbar * cbar * std::max(Nf, Nc) * std::max(Nf, Nc) / hmin;
    for (auto& pt : ctx->parts) {
        Box& F = pt.boxes[fine_box];
        Box& C = pt.boxes[coarse_box];
        sem::IfaceParams& p = pt.itf.prm;
        p = sem::IfaceParams{};
        p.NXf = F.NX;
        p.NYf = F.NY;
        p.NZf = F.NZ;
        p.NXc = C.NX;
        p.NYc = C.NY;
        p.PXf = F.PX;
        p.PXc = C.PX;
        p.Nf = Nf;
        p.Nc = Nc;
        p.R = R;
        p.nelcx = C.d.nel[0];
        p.nelcy = C.d.nel[1];
        p.gamma = gamma;
        p.cf2 = gF.c * gF.c;
        p.cc2 = gC.c * gC.c;
        p.skip_iy0 = F.cutL ? 1 : 0;
        for (int c = 0; c <= Nf; ++c) p.dfT[c] = (2.0 / hF[2]) * Df[Nf * (Nf + 1) + c];
        for (int c = 0; c <= Nc; ++c) p.dcB[c] = (2.0 / hC[2]) * Dc[0 * (Nc + 1) + c];
        double* dI = nullptr;
        if (upload(ctx, &dI, I)) return SEM_E_CUDA;
        p.I = dI;
        p.mxf = F.mx;
        p.myf = F.my;
        p.mxc = C.mx;
        p.myc = C.my;
        const size_t nf = (size_t)F.NX * F.NY, nc = (size_t)C.NX * C.NY, nh = (size_t)F.NX * C.NY;
        if (dalloc(ctx, &p.trc, nc) || dalloc(ctx, &p.drc, nc) || dalloc(ctx, &p.tauf, nf) ||
            dalloc(ctx, &p.sigf, nf) || dalloc(ctx, &p.h1, nh) ||
            dalloc(ctx, &p.h2, nh) || dalloc(ctx, &p.tauc, nc) || dalloc(ctx, &p.sigc, nc))
            return SEM_E_OOM;
        if (quad_rule == 1) {   // Gauss-Legendre points of the fine faces (R9's flag)
            const int nq = Nf + 1;
            std::vector<double> xq, wq;
            gl_rule(nq, xq, wq);
            std::vector<double> Lf((size_t)nq * (Nf + 1)), ILG((size_t)R * nq * (Nc + 1));
            for (int k = 0; k < nq; ++k) {
                const std::vector<double> l = lagrange_at(xf, xq[k]);
                for (int a = 0; a <= Nf; ++a) Lf[(size_t)k * (Nf + 1) + a] = l[a];
            }
            for (int r = 0; r < R; ++r)
                for (int k = 0; k < nq; ++k) {
                    const double xm = (2.0 * r + xq[k] + 1.0) / R - 1.0;   // x_hat^- of the LG point
                    const std::vector<double> l = lagrange_at(xc, xm);
                    for (int b = 0; b <= Nc; ++b) ILG[(size_t)(r * nq + k) * (Nc + 1) + b] = l[b];
                }
            p.lg = 1;
            p.nelfx = F.d.nel[0];
            p.nelfy = F.d.nel[1];
            p.NXq = (long long)p.nelfx * nq;
            p.NYq = (long long)p.nelfy * nq;
            for (int k = 0; k < nq; ++k) {
                p.wqx[k] = 0.5 * hF[0] * wq[k];
                p.wqy[k] = 0.5 * hF[1] * wq[k];
            }
            double *dLf = nullptr, *dILG = nullptr;
            if (upload(ctx, &dLf, Lf) || upload(ctx, &dILG, ILG)) return SEM_E_CUDA;
            p.Lf = dLf;
            p.ILG = dILG;
            const size_t nqq = (size_t)p.NXq * p.NYq, nqh = (size_t)p.NXq * C.NY;
            if (dalloc(ctx, &p.g1, nqq) || dalloc(ctx, &p.g2, nqq) || dalloc(ctx, &p.tacc, nf) ||
                dalloc(ctx, &p.sacc, nf) || dalloc(ctx, &p.q1, nqh) || dalloc(ctx, &p.q2, nqh))
                return SEM_E_OOM;
            CU(cudaMemsetAsync(p.tacc, 0, nf * sizeof(double), ctx->stream));
            CU(cudaMemsetAsync(p.sacc, 0, nf * sizeof(double), ctx->stream));
        }
        // layer coefficients: a -= tau ktau[c] + sigma ksig[c]
        F.iface_side = +1;
        F.tau = p.tauf;
        F.sig = p.sigf;
        for (int c = 0; c <= Nf; ++c) {
            const long long iz = F.NZ - 1 - Nf + c;
            F.tab.ksig[c] = (2.0 / hF[2]) * Df[Nf * (Nf + 1) + c] / F.mzh[iz];
            F.tab.ktau[c] = (c == Nf) ? 1.0 / F.mzh[iz] : 0.0;
        }
        C.iface_side = -1;
        C.tau = p.tauc;
        C.sig = p.sigc;
        for (int c = 0; c <= Nc; ++c) {
            C.tab.ksig[c] = (2.0 / hC[2]) * Dc[0 * (Nc + 1) + c] / C.mzh[c];
            C.tab.ktau[c] = (c == 0) ? 1.0 / C.mzh[0] : 0.0;
        }
        pt.itf.on = true;
        pt.itf.fine = fine_box;
        pt.itf.coarse = coarse_box;
        if (sem::iface_uses_dzf(Nf, Nc, R, quad_rule == 1 ? 1 : 0) && dalloc(ctx, &pt.itf.dzf, nf)) return SEM_E_OOM;
    }
    sem::iface_prepare(gF.degree, gC.degree, R);
    dzf_refresh(ctx);
    ctx->itf_on = true;
    drop_graphs(ctx);
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

// Element-scatter setup of a box (curved vertex lattice and/or obstacle): assembled lumped mass and
// ABC diagonal over the fluid elements from b.vlat_h / b.solid_h, device copies, kernel occupancy.
sem_status curved_setup(sem_ctx* ctx, Box& b, const sem_box_desc& g) {
    const int nx = g.nel[0] + 1, ny = g.nel[1] + 1;
    std::vector<double> x, w;
    gll_rule(b.N, x, w);
    const int N = b.N;
    // assembled lumped mass (sum_e w_q |det J|) and ABC diagonal (sum_F c w_s w_t |J_s|), Eq. 8
    std::vector<double> M((size_t)b.nalloc(), 0.0), Cd((size_t)b.nalloc(), 0.0);
    const double* verts = b.vlat_h.data();
    auto vtx = [&](int vx, int vy, int vz, int i) { return verts[3 * ((size_t)vx + (size_t)nx * ((size_t)vy + (size_t)ny * vz)) + i]; };
    for (int ez = 0; ez < g.nel[2]; ++ez)
        for (int ey = 0; ey < g.nel[1]; ++ey)
            for (int ex = 0; ex < g.nel[0]; ++ex) {
                if (!b.solid_h.empty() && b.solid_h[(size_t)ex + (size_t)g.nel[0] * ((size_t)ey + (size_t)g.nel[1] * ez)])
                    continue;   // obstacle element: not part of the fluid
                for (int c = 0; c <= N; ++c)
                    for (int bb = 0; bb <= N; ++bb)
                        for (int a = 0; a <= N; ++a) {
                            const double xi[3] = {x[a], x[bb], x[c]};
                            double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                            for (int v = 0; v < 8; ++v) {
                                const double s0 = (v & 1) ? 1.0 : -1.0, s1 = (v & 2) ? 1.0 : -1.0, s2 = (v & 4) ? 1.0 : -1.0;
                                const double f0 = 1.0 + s0 * xi[0], f1 = 1.0 + s1 * xi[1], f2 = 1.0 + s2 * xi[2];
                                const double dN[3] = {0.125 * s0 * f1 * f2, 0.125 * s1 * f0 * f2, 0.125 * s2 * f0 * f1};
                                for (int i = 0; i < 3; ++i)
                                    for (int j = 0; j < 3; ++j)
                                        J[i][j] += dN[j] * vtx(ex + (v & 1), ey + ((v >> 1) & 1), ez + (v >> 2), i);
                            }
                            const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                                               J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                                               J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                            if (!(det > 0.0)) return fail(ctx, SEM_E_ARG, "non-positive Jacobian at a GLL point");
                            const long long gx = (long long)N * ex + a, gy = (long long)N * ey + bb, gz = (long long)N * ez + c;
                            const size_t gi = (size_t)((gz * b.NY + gy) * b.PX + gx);
                            M[gi] += w[a] * w[bb] * w[c] * det;
                            // faces of the box (absorbing): surface element |dX/ds x dX/dt| at the node
                            const int loc[3] = {a, bb, c};
                            const int el[3] = {ex, ey, ez};
                            for (int f = 0; f < 6; ++f) {
                                if (g.bc[f] != SEM_BC_ABSORBING) continue;
                                const int d = f / 2, side = f % 2;
                                if (loc[d] != (side ? N : 0) || el[d] != (side ? g.nel[d] - 1 : 0)) continue;
                                const int t0 = d == 0 ? 1 : 0, t1 = d == 2 ? 1 : 2;
                                const double cx = J[1][t0] * J[2][t1] - J[2][t0] * J[1][t1];
                                const double cy = J[2][t0] * J[0][t1] - J[0][t0] * J[2][t1];
                                const double cz = J[0][t0] * J[1][t1] - J[1][t0] * J[0][t1];
                                Cd[gi] += g.c * w[loc[t0]] * w[loc[t1]] * std::sqrt(cx * cx + cy * cy + cz * cz);
                            }
                        }
            }
    for (size_t i = 0; i < M.size(); ++i) {
        if (M[i] > 0.0) {
            Cd[i] /= M[i];
            M[i] = 1.0 / M[i];
        }
    }
    auto put = [&](double** d, const std::vector<double>& h) -> sem_status {
        if (!*d) return upload(ctx, d, h);
        CU(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        return SEM_OK;
    };
    if (put(&b.vlat, b.vlat_h) || put(&b.minv, M) || put(&b.cdamp, Cd)) return SEM_E_CUDA;
    if (!b.solid_h.empty()) {
        if (!b.solid && dalloc(ctx, &b.solid, b.solid_h.size())) return SEM_E_OOM;
        CU(cudaMemcpyAsync(b.solid, b.solid_h.data(), b.solid_h.size(), cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    if (!b.res) {
        if (dalloc(ctx, &b.res, (size_t)b.nalloc())) return SEM_E_OOM;
        CU(cudaMemsetAsync(b.res, 0, (size_t)b.nalloc() * sizeof(double), ctx->stream));
    }
    b.curved = true;
    sem::curved_grid(b.N, g.nel[0] * g.nel[1] * g.nel[2]);   // occupancy query + smem opt-in, outside any capture
    drop_graphs(ctx);
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

// shared checks of sem_box_set_vertices / sem_box_set_obstacle
sem_status scatter_box_check(sem_ctx* ctx, int box, const void* data, const char* what) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->gdesc.size() || !data) return fail(ctx, SEM_E_ARG, std::string("bad box / ") + what);
    if (ctx->world > 1 || ctx->parts.size() != 1)
        return fail(ctx, SEM_E_PARTITION, "curved / obstacle boxes are implemented for a single slab (world 1) only");
    sem::Part& pt = ctx->parts[0];
    if (pt.boxes[box].iface_side != 0 || (pt.pml.on && pt.pml.box == box) || (ctx->pw.on && ctx->pw.box == box))
        return fail(ctx, SEM_E_STATE, "curved / obstacle boxes carry no interface / PML / plane wave");
    return SEM_OK;
}

sem_status sem_box_set_vertices(sem_ctx* ctx, int box, const double* verts, size_t n_verts) {
    sem_status st = scatter_box_check(ctx, box, verts, "vertices");
    if (st) return st;
    if (ctx->parts[0].pm.on && ctx->parts[0].pm.box == box)
        return fail(ctx, SEM_E_STATE, "set the vertices before attaching the PMUTs of their box");
    Box& b = ctx->parts[0].boxes[box];
    const sem_box_desc& g = ctx->gdesc[box];
    if (b.verts_set) return fail(ctx, SEM_E_STATE, "vertices already set");
    const size_t nv = (size_t)(g.nel[0] + 1) * (g.nel[1] + 1) * (g.nel[2] + 1);
    if (n_verts != nv) return fail(ctx, SEM_E_ARG, "n_verts must be (nel_x+1)(nel_y+1)(nel_z+1)");
    const std::vector<double> keep = b.vlat_h;
    b.vlat_h.assign(verts, verts + 3 * n_verts);
    st = curved_setup(ctx, b, g);
    if (st) b.vlat_h = keep;
    else b.verts_set = true;
    return st;
}

sem_status sem_box_set_obstacle(sem_ctx* ctx, int box, const unsigned char* solid, size_t n_el) {
    sem_status st = scatter_box_check(ctx, box, solid, "solid mask");
    if (st) return st;
    if (ctx->parts[0].pm.on && ctx->parts[0].pm.box == box)
        return fail(ctx, SEM_E_STATE, "set the obstacle before attaching the PMUTs of its box");
    Box& b = ctx->parts[0].boxes[box];
    const sem_box_desc& g = ctx->gdesc[box];
    if ((long long)n_el != (long long)g.nel[0] * g.nel[1] * g.nel[2])
        return fail(ctx, SEM_E_ARG, "n_el must be nel_x nel_y nel_z");
    if (!b.solid_h.empty()) return fail(ctx, SEM_E_STATE, "obstacle already set");
    size_t n_fluid = 0;
    for (size_t e = 0; e < n_el; ++e) n_fluid += solid[e] ? 0 : 1;
    if (n_fluid == 0) return fail(ctx, SEM_E_ARG, "every element is solid");
    if (b.vlat_h.empty()) affine_lattice(b, g);   // affine box: its own vertex lattice
    b.solid_h.assign(solid, solid + n_el);
    for (auto& v : b.solid_h) v = v ? 1 : 0;
    st = curved_setup(ctx, b, g);
    if (st) b.solid_h.clear();
    return st;
}

sem_status sem_pml_attach(sem_ctx* ctx, int box, const double* thickness, double R) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->gdesc.size() || !thickness) return fail(ctx, SEM_E_ARG, "bad box / thickness");
    if (!(R > 0.0 && R < 1.0)) return fail(ctx, SEM_E_ARG, "PML reflection coefficient must be in (0, 1)");
    for (auto& pt : ctx->parts) {
        if (pt.pml.on) return fail(ctx, SEM_E_STATE, "PML already attached");
        if (pt.boxes[box].curved) return fail(ctx, SEM_E_STATE, "PML on a curved box is not supported");
    }
    const sem_box_desc& g = ctx->gdesc[box];
    for (int f = 0; f < 6; ++f)
        if (!(thickness[f] >= 0.0) || !std::isfinite(thickness[f])) return fail(ctx, SEM_E_ARG, "thickness must be >= 0");
    for (int d = 0; d < 3; ++d)
        if (thickness[2 * d] + thickness[2 * d + 1] > g.extent[d] * (1.0 + 1e-12))
            return fail(ctx, SEM_E_ARG, "PML layers of opposite faces overlap");
    const int N = g.degree;
    std::vector<double> x, w;
    gll_rule(N, x, w);
    // 1D damping profiles z_d at the GLOBAL lattice nodes (reading R23): a y-slab takes its
    // rows of the y profile, so the layers sit at the global box faces, never at a slab cut
    const long long ng[3] = {(long long)N * g.nel[0] + 1, (long long)N * g.nel[1] + 1, (long long)N * g.nel[2] + 1};
    std::vector<double> zt[3];
    std::vector<char> epml[3];
    for (int d = 0; d < 3; ++d) {
        const int nel = g.nel[d];
        const double hd = g.extent[d] / nel;
        zt[d].assign(ng[d], 0.0);
        for (long long i = 0; i < ng[d]; ++i) {
            long long e = i / N;
            if (e > nel - 1) e = nel - 1;
            const int a = (int)(i - e * N);
            const double xc = g.origin[d] + hd * ((double)e + 0.5 * (x[a] + 1.0));
            for (int side = 0; side < 2; ++side) {
                const double ell = thickness[2 * d + side];
                if (ell <= 0.0) continue;
                const double lo = g.origin[d], hi = g.origin[d] + g.extent[d];
                const double dist = side ? xc - (hi - ell) : (lo + ell) - xc;
                if (dist <= 0.0) continue;
                const double sfrac = std::min(dist / ell, 1.0);
                const double ztl = g.c / ell * std::log(1.0 / R);
                zt[d][i] += ztl * (sfrac - std::sin(2.0 * M_PI * sfrac) / (2.0 * M_PI));
            }
        }
        epml[d].assign(nel, 0);
        for (int e = 0; e < nel; ++e)
            for (int a = 0; a <= N; ++a)
                if (zt[d][(size_t)e * N + a] > 0.0) epml[d][e] = 1;
    }
    for (auto& pt : ctx->parts) {
        Box& b = pt.boxes[box];
        sem::PmlBox& m = pt.pml;
        m.box = box;
        m.D = deriv_matrix(x);
        m.w = w;
        const long long ey0 = b.gy0 / N, nely = b.d.nel[1];
        // PML elements of this slab: every element with a node where some z_d > 0 (slab-local y index)
        std::vector<int> el;
        for (int ez = 0; ez < g.nel[2]; ++ez)
            for (long long ey = 0; ey < nely; ++ey)
                for (int ex = 0; ex < g.nel[0]; ++ex)
                    if (epml[0][ex] || epml[1][ey + ey0] || epml[2][ez]) {
                        el.push_back(ex);
                        el.push_back((int)ey);
                        el.push_back(ez);
                    }
        m.n_el = (int)(el.size() / 3);
        const size_t nl = (size_t)(N + 1) * (N + 1) * (N + 1);
        // per-axis node tables: z, CN factors, inverse assembled 1D mass (PmlParams::tx); slab rows in y
        const long long nn[3] = {b.NX, b.NY, b.NZ}, i0[3] = {0, b.gy0, 0};
        const std::vector<double>* m1[3] = {&b.mxh, &b.myh, &b.mzh};
        for (int d = 0; d < 3; ++d) {
            std::vector<double> t4((size_t)nn[d] * 4);
            for (long long i = 0; i < nn[d]; ++i) {
                const double zz = zt[d][i + i0[d]], den = 1.0 + 0.5 * ctx->dt * zz;
                t4[4 * i] = zz;
                t4[4 * i + 1] = (1.0 - 0.5 * ctx->dt * zz) / den;
                t4[4 * i + 2] = ctx->dt / den;
                t4[4 * i + 3] = 1.0 / (*m1[d])[i];
            }
            if (upload(ctx, &m.tab[d], t4)) return SEM_E_CUDA;
        }
        if (m.n_el > 0 && upload(ctx, &m.elems, el)) return SEM_E_CUDA;
        if (dalloc(ctx, &m.phi, (size_t)std::max(m.n_el, 1) * 3 * nl) || dalloc(ctx, &m.psi[0], (size_t)b.nalloc()) ||
            dalloc(ctx, &m.psi[1], (size_t)b.nalloc()) || dalloc(ctx, &m.da, (size_t)b.nalloc()))
            return SEM_E_OOM;
        // the region (nodes of PML elements) as x-row segments: node (ix, iy, iz) belongs to a PML element
        // iff some element containing it along some axis d has a damped node (element masks per axis)
        if (m.n_el > 0) {
            auto node_mask = [&](int d, long long n, long long off) {
                std::vector<char> nm((size_t)n, 0);
                for (long long i = 0; i < n; ++i) {
                    const long long ig = i + off;
                    const long long e1 = std::min<long long>(ig / N, g.nel[d] - 1), e0 = (ig % N == 0 && ig > 0) ? ig / N - 1 : e1;
                    nm[(size_t)i] = (epml[d][e0] || epml[d][e1]) ? 1 : 0;
                }
                return nm;
            };
            const std::vector<char> mx = node_mask(0, b.NX, 0), my = node_mask(1, b.NY, b.gy0), mz = node_mask(2, b.NZ, 0);
            std::vector<long long> ss;
            std::vector<int> sl;
            for (long long iz = 0; iz < b.NZ; ++iz)
                for (long long iy = 0; iy < b.NY; ++iy) {
                    const long long row = (iz * b.NY + iy) * b.PX;
                    if (my[(size_t)iy] || mz[(size_t)iz]) {
                        ss.push_back(row);
                        sl.push_back((int)b.NX);
                        continue;
                    }
                    for (long long ix = 0; ix < b.NX;) {
                        if (!mx[(size_t)ix]) {
                            ++ix;
                            continue;
                        }
                        long long e = ix;
                        while (e < b.NX && mx[(size_t)e]) ++e;
                        ss.push_back(row + ix);
                        sl.push_back((int)(e - ix));
                        ix = e;
                    }
                }
            if (upload(ctx, &m.seg_start, ss) || upload(ctx, &m.seg_len, sl)) return SEM_E_CUDA;
            m.n_seg = (long long)ss.size();
        }
        m.on = true;
        if (ctx->world > 1 && setup_exchange(ctx, pt) != SEM_OK) return SEM_E_OOM;   // + the PML da plane
    }
    drop_graphs(ctx);
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_plane_wave_source(sem_ctx* ctx, int box, int face, double amp, double f0, double sigma, double t0,
                                 const double dir[3]) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->gdesc.size() || face != 5 || !dir)
        return fail(ctx, SEM_E_ARG, "plane wave: +z face of an existing box only");
    const sem_box_desc& g = ctx->gdesc[box];
    if (g.bc[5] != SEM_BC_ABSORBING) return fail(ctx, SEM_E_ARG, "plane wave needs an absorbing face");
    const double nk = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    if (!(nk > 0) || !(sigma > 0)) return fail(ctx, SEM_E_ARG, "bad plane-wave parameters");
    if (ctx->parts[0].boxes[box].curved) {
        // element-scatter box: the load is tabulated per top-face node from the vertex lattice
        for (auto& b : ctx->parts[0].boxes)
            if (!b.curved) return fail(ctx, SEM_E_STATE, "a plane wave on a curved box needs every box on the element-scatter path");
        double kk[3];
        for (int k = 0; k < 3; ++k) kk[k] = dir[k] / nk;
        st = curved_plane_wave(ctx, ctx->parts[0].boxes[box], amp, kk);
        if (st) return st;
    }
    sem::PlaneWave& pw = ctx->pw;
    pw.box = box;
    pw.amp = amp;
    pw.f0 = f0;
    pw.sigma = sigma;
    pw.t0 = t0;
    for (int k = 0; k < 3; ++k) pw.k[k] = dir[k] / nk;
    // x_ref: the corner of the (global) +z face the wavefront reaches first (min k.x), reading R13
    const double zt = g.origin[2] + g.extent[2];
    double best = std::numeric_limits<double>::infinity();
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            const double x = i ? g.origin[0] + g.extent[0] : g.origin[0];
            const double y = j ? g.origin[1] + g.extent[1] : g.origin[1];
            const double kx = pw.k[0] * x + pw.k[1] * y + pw.k[2] * zt;
            if (kx < best) {
                best = kx;
                pw.xref[0] = x;
                pw.xref[1] = y;
                pw.xref[2] = zt;
            }
        }
    if (ctx->parts[0].boxes[box].curved)
        for (int k = 0; k < 3; ++k) pw.xref[k] = ctx->pw_xref_curved[k];
    pw.on = true;
    drop_graphs(ctx);
    return SEM_OK;
}

sem_status sem_step(sem_ctx* ctx, int n_steps) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (n_steps < 0) return fail(ctx, SEM_E_ARG, "n_steps < 0");
    long long launches = 0;
    int left = n_steps;
    while (left > 0) {
        const bool direct = ctx->profiling || (ctx->flags & SEM_F_NO_GRAPH) || ctx->graph_failed;
        if (direct) {
            launches += enqueue_step(ctx, ctx->cur, ctx->profiling);
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
            for (int k = 0; k < len; ++k) nl += enqueue_step(ctx, ctx->cur ^ (k & 1), false);
            cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
            if (e == cudaSuccess) {
                e = cudaGraphInstantiate(&g, graph, 0);
                cudaGraphDestroy(graph);
            }
            if (e != cudaSuccess) {
                g = nullptr;
                if (nccl_mode(ctx)) {   // NCCL build without capture support: direct launches from now on
                    (void)cudaGetLastError();
                    ctx->graph_failed = true;
                    continue;
                }
                return fail(ctx, SEM_E_CUDA, std::string("graph: ") + cudaGetErrorString(e));
            }
            ctx->graph_launches[ctx->cur][len - 1] = nl;
        }
        CU(cudaGraphLaunch(g, ctx->stream));
        launches += ctx->graph_launches[ctx->cur][len - 1];
        if (len == 1) ctx->cur ^= 1;
        left -= len;
    }
    CU(cudaGetLastError());
    ctx->step += n_steps;
    ctx->last_launches = launches;
    if (ctx->flags & SEM_F_NAN_CHECK) {
        CU(cudaMemsetAsync(ctx->d_flag, 0, 8, ctx->stream));
        for (auto& pt : ctx->parts)
            for (auto& b : pt.boxes)
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
    if (box < 0 || box >= (int)ctx->gdesc.size()) return fail(ctx, SEM_E_ARG, "bad box");
    const long long NXg = ctx->gNX[box], rows = ctx->gNY[box] * ctx->gNZ[box];
    const bool receiver = !nccl_mode(ctx) || ctx->rank == 0;
    if (receiver && (!host || n != (size_t)(NXg * rows))) return fail(ctx, SEM_E_ARG, "n must equal the box node count");
    const long long NYg = ctx->gNY[box];
    if (!nccl_mode(ctx)) {
        for (auto& pt : ctx->parts) {
            Box& b = pt.boxes[box];
            const long long skip = b.cutL ? 1 : 0;   // the shared cut row is reported by the lower slab
            CU(copy_slab(host, b.P[1 - ctx->cur], b, NYg, b.gy0, skip, true, ctx->stream));
        }
        CU(cudaStreamSynchronize(ctx->stream));
        return SEM_OK;
    }
    // NCCL: every rank sends its slab to rank 0, which assembles the global field
    NcclApi& api = nccl_api();
    Box& mine = ctx->parts[0].boxes[box];
    if (ctx->rank != 0) {
        NC(api.send(mine.P[1 - ctx->cur], (size_t)mine.nalloc(), kNcclDouble, 0, ctx->nccl, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        return SEM_OK;
    }
    CU(copy_slab(host, mine.P[1 - ctx->cur], mine, NYg, mine.gy0, 0, true, ctx->stream));
    // the other ranks' slabs (the plan may be uneven): their geometry from the plan, largest buffer once
    const sem_box_desc& g = ctx->gdesc[box];
    std::vector<Box> slabs;
    size_t most = 0;
    for (int r = 1; r < ctx->world; ++r) {
        const long long e0 = cut_in_box(ctx->gdesc[0], g, ctx->cuts[r]), e1 = cut_in_box(ctx->gdesc[0], g, ctx->cuts[r + 1]);
        slabs.push_back(make_slab(g, e0, e1 - e0, true, r < ctx->world - 1));
        most = std::max(most, (size_t)slabs.back().nalloc());
    }
    double* tmp = nullptr;
    CU(cudaMallocAsync(&tmp, most * 8, ctx->stream));
    for (int r = 1; r < ctx->world; ++r) {
        const Box& rb = slabs[r - 1];
        NC(api.recv(tmp, (size_t)rb.nalloc(), kNcclDouble, r, ctx->nccl, ctx->stream));
        CU(copy_slab(host, tmp, rb, NYg, rb.gy0, 1, true, ctx->stream));
    }
    CU(cudaFreeAsync(tmp, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_read_pressure_at(sem_ctx* ctx, int box, const long long* ids, size_t n, double* out) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->gdesc.size() || (n && (!ids || !out))) return fail(ctx, SEM_E_ARG, "bad args");
    if (nccl_mode(ctx)) return fail(ctx, SEM_E_STATE, "sampled readout is single-process only (world 1 or emulated)");
    if (n == 0) return SEM_OK;
    const long long NXg = ctx->gNX[box], NYg = ctx->gNY[box], total = NXg * NYg * ctx->gNZ[box];
    std::vector<std::vector<long long>> idx(ctx->parts.size()), pos(ctx->parts.size());
    for (size_t i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= total) return fail(ctx, SEM_E_ARG, "node id out of range");
        const long long gx = ids[i] % NXg, row = ids[i] / NXg, gy = row % NYg, gz = row / NYg;
        const int r = owner_part(ctx, box, gy);
        const Box& b = ctx->parts[r].boxes[box];
        idx[r].push_back((gz * b.NY + (gy - b.gy0)) * b.PX + gx);
        pos[r].push_back((long long)i);
    }
    std::vector<double> tmp(n);
    for (size_t r = 0; r < ctx->parts.size(); ++r) {
        const size_t m = idx[r].size();
        if (!m) continue;
        long long* didx = nullptr;
        double* dout = nullptr;
        CU(cudaMallocAsync(&didx, m * sizeof(long long), ctx->stream));
        CU(cudaMallocAsync(&dout, m * sizeof(double), ctx->stream));
        CU(cudaMemcpyAsync(didx, idx[r].data(), m * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
        sem::launch_gather(ctx->parts[r].boxes[box].P[1 - ctx->cur], didx, (long long)m, dout, ctx->stream);
        std::vector<double> got(m);
        CU(cudaMemcpyAsync(got.data(), dout, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaFreeAsync(didx, ctx->stream));
        CU(cudaFreeAsync(dout, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        for (size_t j = 0; j < m; ++j) out[pos[r][j]] = got[j];
    }
    return SEM_OK;
}

sem_status sem_read_modal(sem_ctx* ctx, double* q, double* qdot, double* v_rx, size_t n) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (!ctx->n_pmut) return fail(ctx, SEM_E_STATE, "no PMUT array attached");
    const int M = ctx->n_modes;
    const size_t nm = (size_t)ctx->n_pmut * M;
    const bool receiver = !nccl_mode(ctx) || ctx->rank == 0;
    if (receiver && n != nm) return fail(ctx, SEM_E_ARG, "n must equal n_pmut * n_modes");
    double* outs[3] = {q, qdot, v_rx};
    auto scatter = [&](const std::vector<int>& ks, const std::vector<double>& buf, int which) {
        const int per = which == 2 ? 1 : M;
        if (!outs[which]) return;
        for (size_t l = 0; l < ks.size(); ++l)
            for (int m = 0; m < per; ++m) outs[which][(size_t)ks[l] * per + m] = buf[l * per + m];
    };
    if (!nccl_mode(ctx)) {
        for (auto& pt : ctx->parts) {
            if (!pt.pm.on) continue;
            const size_t KL = pt.pm_global.size();
            const double* src[3] = {pt.pm.q, pt.pm.qd, pt.pm.phi};
            for (int w = 0; w < 3; ++w) {
                std::vector<double> buf(KL * (w == 2 ? 1 : M));
                CU(cudaMemcpyAsync(buf.data(), src[w], buf.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
                CU(cudaStreamSynchronize(ctx->stream));
                scatter(pt.pm_global, buf, w);
            }
        }
        return SEM_OK;
    }
    NcclApi& api = nccl_api();
    sem::Part& pt = ctx->parts[0];
    const double* src[3] = {pt.pm.q, pt.pm.qd, pt.pm.phi};
    if (ctx->rank != 0) {
        for (int w = 0; w < 3; ++w) {
            const size_t cnt = pt.pm_global.size() * (w == 2 ? 1 : M);
            if (cnt) NC(api.send(src[w], cnt, kNcclDouble, 0, ctx->nccl, ctx->stream));
        }
        CU(cudaStreamSynchronize(ctx->stream));
        return SEM_OK;
    }
    for (int r = 0; r < ctx->world; ++r) {
        const std::vector<int>& ks = ctx->pm_lists[r];
        for (int w = 0; w < 3; ++w) {
            const size_t cnt = ks.size() * (w == 2 ? 1 : M);
            if (!cnt) continue;
            std::vector<double> buf(cnt);
            if (r == 0) {
                CU(cudaMemcpyAsync(buf.data(), src[w], cnt * 8, cudaMemcpyDeviceToHost, ctx->stream));
            } else {
                double* tmp = nullptr;
                CU(cudaMallocAsync(&tmp, cnt * 8, ctx->stream));
                NC(api.recv(tmp, cnt, kNcclDouble, r, ctx->nccl, ctx->stream));
                CU(cudaMemcpyAsync(buf.data(), tmp, cnt * 8, cudaMemcpyDeviceToHost, ctx->stream));
                CU(cudaFreeAsync(tmp, ctx->stream));
            }
            CU(cudaStreamSynchronize(ctx->stream));
            scatter(ks, buf, w);
        }
    }
    return SEM_OK;
}

sem_status sem_write_state(sem_ctx* ctx, int box, const double* p, const double* pdot, size_t n) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->gdesc.size() || !p || !pdot) return fail(ctx, SEM_E_ARG, "bad args");
    const long long NXg = ctx->gNX[box], rows = ctx->gNY[box] * ctx->gNZ[box];
    if (n != (size_t)(NXg * rows)) return fail(ctx, SEM_E_ARG, "n must equal the box node count");
    // p^S lives in P[1-cur]; p^{S+1} = p^S + dt w^S in P[cur]; w^0 = p'^0 + dt/2 p''^0 = p'^0
    for (auto& pt : ctx->parts) {
        Box& b = pt.boxes[box];
        double* pprev = b.P[1 - ctx->cur];
        CU(copy_slab(const_cast<double*>(p), pprev, b, ctx->gNY[box], b.gy0, 0, false, ctx->stream));
        CU(copy_slab(const_cast<double*>(pdot), b.W, b, ctx->gNY[box], b.gy0, 0, false, ctx->stream));
        sem::launch_set_state(pprev, b.P[ctx->cur], b.W, b.NX, b.PX, b.NY * b.NZ, ctx->dt, ctx->stream);
        if (b.solid) sem::launch_zero_inactive(b.P[0], b.P[1], b.W, b.minv, b.NX, b.PX, b.NY * b.NZ, ctx->stream);
    }
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_fill_random_state(sem_ctx* ctx, int box, unsigned long long seed, double ps, double vs) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (box < 0 || box >= (int)ctx->gdesc.size()) return fail(ctx, SEM_E_ARG, "bad box");
    for (auto& pt : ctx->parts) {
        Box& b = pt.boxes[box];
        sem::launch_fill_random(b.P[1 - ctx->cur], b.W, b.P[ctx->cur], b.NX, b.PX, b.NY, b.NZ, b.gy0, b.NYg, seed, box,
                                ps, vs, ctx->dt, ctx->stream);
        if (b.solid) sem::launch_zero_inactive(b.P[0], b.P[1], b.W, b.minv, b.NX, b.PX, b.NY * b.NZ, ctx->stream);
    }
    st = reset_dynamic(ctx);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    return SEM_OK;
}

sem_status sem_query(sem_ctx* ctx, long long* n_dof, long long* step, double* t) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    long long nd = 0;
    for (size_t b = 0; b < ctx->gdesc.size(); ++b) nd += ctx->gNX[b] * ctx->gNY[b] * ctx->gNZ[b];
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
    for (int k = 0; k < 4; ++k) {
        ctx->kt_ms[k] = 0;
        ctx->kt_n[k] = 0;
    }
    ctx->profiling = on != 0;
    return SEM_OK;
}

sem_status sem_kernel_time(sem_ctx* ctx, int which, double* ms, long long* nl) {
    sem_status st = check_ctx(ctx);
    if (st) return st;
    if (which < 0 || which > 3) return fail(ctx, SEM_E_ARG, "which in 0..3");
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
    if (ctx->nccl && nccl_api().commDestroy) nccl_api().commDestroy(ctx->nccl);
    for (void* p : ctx->allocs) {
        if (ctx->dev_free) ctx->dev_free(p, ctx->alloc_user);
        else if (!ctx->dev_alloc) cudaFree(p);
    }
    for (auto& pe : ctx->ev_pending) {
        cudaEventDestroy(pe.second.first);
        cudaEventDestroy(pe.second.second);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_mfork) cudaEventDestroy(ctx->ev_mfork);
    if (ctx->ev_mjoin) cudaEventDestroy(ctx->ev_mjoin);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->comm) cudaStreamDestroy(ctx->comm);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

}  // extern "C"
