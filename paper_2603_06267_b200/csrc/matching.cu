// Algorithm 3 (face matching on the non-conforming interface) on the GPU.
//
// One thread per fine-face quadrature node x_q = X_{K+}(xhat_q+) (fine-face GLL nodes, reading R9).
// The paper's filters are applied unchanged -- opposite normals |n+ + n-| < tol and the one-vertex
// radius test |V_{K-} - x_q| < r, r = max(diam dK-, diam dK+) + eps -- followed by the Newton-Raphson
// inverse map xhat_q- = X_{K-}^{-1}(x_q) and the containment test xhat_q- in [-1,1]^3.
// The candidate set is taken from a uniform grid of cell size r_max over the coarse faces' vertices
// V_{K-} (the 27 cells around x_q hold every V within r_max), which replaces the paper's loop over all
// coarse faces; among the matching faces the lowest index wins (reading R26: the oracle's first match
// in index order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/sem.h"

namespace {

constexpr int kMaxQ1 = 9;   // degree <= 8

struct MatchParams {
    const double* fv;        // fine element vertices [nf][8][3]
    const int* ff;           // fine local faces [nf]
    const double* cv;        // coarse element vertices [nc][8][3]
    const int* cf;
    const double* cn;        // coarse face centre normals [nc][3]
    const double* cV;        // coarse face first vertices [nc][3]
    const double* cd;        // coarse face diameters [nc]
    const int* cell_start;   // [ncell + 1] CSR over grid cells
    const int* cell_face;    // coarse face ids sorted by cell
    int nf, nc, q1;          // q1 = degree + 1 nodes per face direction
    double xg[kMaxQ1];       // GLL nodes of the fine face
    double tol, eps;
    double lo[3], cell;      // grid origin and cell size
    int gd[3];               // grid dimensions
    long long* owner;        // [nf * q1^2]
    double* xi;              // [nf * q1^2][3]
};

__host__ __device__ inline int face_vertex(int face, int k) {   // k-th vertex (ascending id) of a local face
    const int d = face / 2, side = face % 2;
    int cnt = 0;
    for (int v = 0; v < 8; ++v) {
        const int bit = (v >> d) & 1;
        if (bit == side) {
            if (cnt == k) return v;
            ++cnt;
        }
    }
    return 0;
}

__device__ inline void trilinear(const double* V, const double xi[3], double x[3], double J[3][3]) {
    for (int i = 0; i < 3; ++i) {
        x[i] = 0.0;
        for (int j = 0; j < 3; ++j) J[i][j] = 0.0;
    }
    for (int v = 0; v < 8; ++v) {
        const double s[3] = {(v & 1) ? 1.0 : -1.0, (v & 2) ? 1.0 : -1.0, (v & 4) ? 1.0 : -1.0};
        const double f[3] = {1.0 + s[0] * xi[0], 1.0 + s[1] * xi[1], 1.0 + s[2] * xi[2]};
        const double N = 0.125 * f[0] * f[1] * f[2];
        const double dN[3] = {0.125 * s[0] * f[1] * f[2], 0.125 * s[1] * f[0] * f[2], 0.125 * s[2] * f[0] * f[1]};
        for (int i = 0; i < 3; ++i) {
            const double Xv = V[3 * v + i];
            x[i] = fma(N, Xv, x[i]);
            for (int j = 0; j < 3; ++j) J[i][j] = fma(dN[j], Xv, J[i][j]);
        }
    }
}

__device__ inline void face_frame(const double* V, int face, double n[3], double* diam) {
    const int d = face / 2, side = face % 2;
    double xi[3] = {0.0, 0.0, 0.0};
    xi[d] = side ? 1.0 : -1.0;
    double c[3], J[3][3];
    trilinear(V, xi, c, J);
    const int t0 = d == 0 ? 1 : 0, t1 = d == 2 ? 1 : 2;
    n[0] = J[1][t0] * J[2][t1] - J[2][t0] * J[1][t1];
    n[1] = J[2][t0] * J[0][t1] - J[0][t0] * J[2][t1];
    n[2] = J[0][t0] * J[1][t1] - J[1][t0] * J[0][t1];
    const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    double cen[3] = {0.0, 0.0, 0.0};
    for (int v = 0; v < 8; ++v)
        for (int i = 0; i < 3; ++i) cen[i] += 0.125 * V[3 * v + i];
    const double dot = (c[0] - cen[0]) * n[0] + (c[1] - cen[1]) * n[1] + (c[2] - cen[2]) * n[2];
    const double sg = dot < 0.0 ? -1.0 : 1.0;
    for (int i = 0; i < 3; ++i) n[i] *= sg / nn;
    if (diam) {
        double dm = 0.0;
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                const double* pa = V + 3 * face_vertex(face, a);
                const double* pb = V + 3 * face_vertex(face, b);
                const double e0 = pa[0] - pb[0], e1 = pa[1] - pb[1], e2 = pa[2] - pb[2];
                dm = fmax(dm, sqrt(e0 * e0 + e1 * e1 + e2 * e2));
            }
        *diam = dm;
    }
}

__global__ void coarse_face_kernel(const double* cv, const int* cf, int nc, double* cn, double* cV, double* cd) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nc) return;
    const double* V = cv + 24 * (size_t)j;
    double n[3], dm;
    face_frame(V, cf[j], n, &dm);
    const int v0 = face_vertex(cf[j], 0);
    for (int i = 0; i < 3; ++i) {
        cn[3 * j + i] = n[i];
        cV[3 * j + i] = V[3 * v0 + i];
    }
    cd[j] = dm;
}

// Newton-Raphson for X_K(xi) = x (the oracle's rule: until max |dxi| < 1e-14, at most 50 steps)
__device__ inline void inverse_map(const double* V, const double x[3], double xi[3]) {
    xi[0] = xi[1] = xi[2] = 0.0;
    for (int it = 0; it < 50; ++it) {
        double X[3], J[3][3];
        trilinear(V, xi, X, J);
        const double r[3] = {x[0] - X[0], x[1] - X[1], x[2] - X[2]};
        const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
        const double inv = 1.0 / det;
        const double d0 = (r[0] * c00 + J[0][1] * (r[2] * J[1][2] - r[1] * J[2][2]) +
                           J[0][2] * (r[1] * J[2][1] - r[2] * J[1][1])) * inv;
        const double d1 = (J[0][0] * (r[1] * J[2][2] - r[2] * J[1][2]) + r[0] * c01 +
                           J[0][2] * (r[2] * J[1][0] - r[1] * J[2][0])) * inv;
        const double d2 = (J[0][0] * (r[2] * J[1][1] - r[1] * J[2][1]) + J[0][1] * (r[1] * J[2][0] - r[2] * J[1][0]) +
                           r[0] * c02) * inv;
        xi[0] += d0;
        xi[1] += d1;
        xi[2] += d2;
        if (fmax(fabs(d0), fmax(fabs(d1), fabs(d2))) < 1e-14) break;
    }
}

__global__ void match_kernel(const __grid_constant__ MatchParams p) {
    const int nq = p.q1 * p.q1;
    const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (long long)p.nf * nq) return;
    const int f = (int)(id / nq), q = (int)(id - (long long)f * nq);
    const double* V = p.fv + 24 * (size_t)f;
    const int face = p.ff[f];
    double nplus[3], dplus;
    face_frame(V, face, nplus, &dplus);
    // x_q = X_{K+}(xhat_q+), s fastest
    const int d = face / 2, side = face % 2;
    const int t0 = d == 0 ? 1 : 0, t1 = d == 2 ? 1 : 2;
    double xr[3];
    xr[d] = side ? 1.0 : -1.0;
    xr[t0] = p.xg[q % p.q1];
    xr[t1] = p.xg[q / p.q1];
    double x[3], J[3][3];
    trilinear(V, xr, x, J);
    int best = -1;
    double bxi[3] = {0.0, 0.0, 0.0};
    int c0[3];
    for (int i = 0; i < 3; ++i) c0[i] = (int)floor((x[i] - p.lo[i]) / p.cell);
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int cx = c0[0] + dx, cy = c0[1] + dy, cz = c0[2] + dz;
                if (cx < 0 || cy < 0 || cz < 0 || cx >= p.gd[0] || cy >= p.gd[1] || cz >= p.gd[2]) continue;
                const int cell = cx + p.gd[0] * (cy + p.gd[1] * cz);
                for (int s = p.cell_start[cell]; s < p.cell_start[cell + 1]; ++s) {
                    const int j = p.cell_face[s];
                    if (best >= 0 && j >= best) continue;
                    const double* nm = p.cn + 3 * j;
                    const double s0 = nplus[0] + nm[0], s1 = nplus[1] + nm[1], s2 = nplus[2] + nm[2];
                    if (sqrt(s0 * s0 + s1 * s1 + s2 * s2) >= p.tol) continue;           // normal filter
                    const double* vv = p.cV + 3 * j;
                    const double e0 = vv[0] - x[0], e1 = vv[1] - x[1], e2 = vv[2] - x[2];
                    const double r = fmax(p.cd[j], dplus) + p.eps;
                    if (sqrt(e0 * e0 + e1 * e1 + e2 * e2) >= r) continue;              // radius filter
                    double xi[3];
                    inverse_map(p.cv + 24 * (size_t)j, x, xi);                          // Newton-Raphson
                    if (fmax(fabs(xi[0]), fmax(fabs(xi[1]), fabs(xi[2]))) <= 1.0 + 1e-9) {
                        best = j;
                        bxi[0] = xi[0];
                        bxi[1] = xi[1];
                        bxi[2] = xi[2];
                    }
                }
            }
    p.owner[id] = best;
    for (int i = 0; i < 3; ++i) p.xi[3 * id + i] = bxi[i];
}

void gll_nodes(int N, std::vector<double>& x) {   // ascending GLL nodes (Newton on (1-x^2) P_N')
    x.assign(N + 1, 0.0);
    for (int i = 0; i <= N; ++i) x[i] = -std::cos(M_PI * i / N);
    for (int it = 0; it < 100; ++it)
        for (int i = 1; i < N; ++i) {
            double p0 = 1.0, p1 = x[i];
            for (int k = 2; k <= N; ++k) {
                const double p2 = ((2.0 * k - 1.0) * x[i] * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            // (1 - x^2) P_N' = N (P_{N-1} - x P_N); derivative of it = -N (N+1) P_N
            const double g = N * (p0 - x[i] * p1), dg = -N * (N + 1.0) * p1;
            x[i] -= g / dg;
        }
    x[0] = -1.0;
    x[N] = 1.0;
}

}  // namespace

extern "C" sem_status sem_face_match(int device, const sem_face_set* fine, const sem_face_set* coarse, int degree,
                                     double normal_tol, long long* owner, double* xi_minus, double* elapsed_ms) {
    if (!fine || !coarse || !owner || !xi_minus || degree < 1 || degree > 8 || !(normal_tol > 0.0)) return SEM_E_ARG;
    if (fine->n < 0 || coarse->n <= 0 || (fine->n && (!fine->verts || !fine->face)) || !coarse->verts || !coarse->face)
        return SEM_E_ARG;
    for (int i = 0; i < fine->n; ++i)
        if (fine->face[i] < 0 || fine->face[i] > 5) return SEM_E_ARG;
    for (int i = 0; i < coarse->n; ++i)
        if (coarse->face[i] < 0 || coarse->face[i] > 5) return SEM_E_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return SEM_E_CUDA;
    const int nf = fine->n, nc = coarse->n, q1 = degree + 1, nq = q1 * q1;
    if (nf == 0) return SEM_OK;
    // host-side: coarse face first vertices, diameters (for the grid), fine diameters
    auto diam = [](const double* V, int face) {
        double dm = 0.0;
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                const double* pa = V + 3 * face_vertex(face, a);
                const double* pb = V + 3 * face_vertex(face, b);
                dm = std::max(dm, std::sqrt((pa[0] - pb[0]) * (pa[0] - pb[0]) + (pa[1] - pb[1]) * (pa[1] - pb[1]) +
                                            (pa[2] - pb[2]) * (pa[2] - pb[2])));
            }
        return dm;
    };
    double rmax = 0.0, lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    std::vector<double> Vh((size_t)nc * 3);
    for (int j = 0; j < nc; ++j) {
        const double* V = coarse->verts + 24 * (size_t)j;
        rmax = std::max(rmax, diam(V, coarse->face[j]));
        const double* v0 = V + 3 * face_vertex(coarse->face[j], 0);
        for (int i = 0; i < 3; ++i) {
            Vh[3 * (size_t)j + i] = v0[i];
            lo[i] = std::min(lo[i], v0[i]);
            hi[i] = std::max(hi[i], v0[i]);
        }
    }
    for (int f = 0; f < nf; ++f) rmax = std::max(rmax, diam(fine->verts + 24 * (size_t)f, fine->face[f]));
    const double eps = 1e-12 * std::max(rmax, 1e-300);
    const double cell = rmax * (1.0 + 1e-9) + eps;
    int gd[3];
    for (int i = 0; i < 3; ++i) {
        lo[i] -= cell;
        gd[i] = (int)std::floor((hi[i] + cell - lo[i]) / cell) + 1;
    }
    const long long ncell = (long long)gd[0] * gd[1] * gd[2];
    if (ncell > (1ll << 28)) return SEM_E_ARG;   // degenerate geometry (cells far smaller than the extent)
    std::vector<int> cnt(ncell + 1, 0), cface(nc), cid(nc);
    for (int j = 0; j < nc; ++j) {
        int c[3];
        for (int i = 0; i < 3; ++i) c[i] = (int)std::floor((Vh[3 * (size_t)j + i] - lo[i]) / cell);
        cid[j] = c[0] + gd[0] * (c[1] + gd[1] * c[2]);
        ++cnt[cid[j] + 1];
    }
    for (long long c = 0; c < ncell; ++c) cnt[c + 1] += cnt[c];
    {
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int j = 0; j < nc; ++j) cface[pos[cid[j]]++] = j;   // ascending j inside a cell
    }
    // device buffers
    MatchParams p{};
    double *dfv = nullptr, *dcv = nullptr, *dcn = nullptr, *dcV = nullptr, *dcd = nullptr, *dxi = nullptr;
    int *dff = nullptr, *dcf = nullptr, *dcs = nullptr, *dcface = nullptr;
    long long* down = nullptr;
    sem_status st = SEM_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto ok = [&](cudaError_t e) {
        if (e != cudaSuccess && st == SEM_OK) st = (e == cudaErrorMemoryAllocation) ? SEM_E_OOM : SEM_E_CUDA;
        return st == SEM_OK;
    };
    if (ok(cudaMalloc(&dfv, sizeof(double) * 24 * nf)) && ok(cudaMalloc(&dcv, sizeof(double) * 24 * nc)) &&
        ok(cudaMalloc(&dcn, sizeof(double) * 3 * nc)) && ok(cudaMalloc(&dcV, sizeof(double) * 3 * nc)) &&
        ok(cudaMalloc(&dcd, sizeof(double) * nc)) && ok(cudaMalloc(&dxi, sizeof(double) * 3 * (size_t)nf * nq)) &&
        ok(cudaMalloc(&dff, sizeof(int) * nf)) && ok(cudaMalloc(&dcf, sizeof(int) * nc)) &&
        ok(cudaMalloc(&dcs, sizeof(int) * (ncell + 1))) && ok(cudaMalloc(&dcface, sizeof(int) * nc)) &&
        ok(cudaMalloc(&down, sizeof(long long) * (size_t)nf * nq)) &&
        ok(cudaMemcpy(dfv, fine->verts, sizeof(double) * 24 * nf, cudaMemcpyHostToDevice)) &&
        ok(cudaMemcpy(dcv, coarse->verts, sizeof(double) * 24 * nc, cudaMemcpyHostToDevice)) &&
        ok(cudaMemcpy(dff, fine->face, sizeof(int) * nf, cudaMemcpyHostToDevice)) &&
        ok(cudaMemcpy(dcf, coarse->face, sizeof(int) * nc, cudaMemcpyHostToDevice)) &&
        ok(cudaMemcpy(dcs, cnt.data(), sizeof(int) * (ncell + 1), cudaMemcpyHostToDevice)) &&
        ok(cudaMemcpy(dcface, cface.data(), sizeof(int) * nc, cudaMemcpyHostToDevice)) &&
        ok(cudaEventCreate(&e0)) && ok(cudaEventCreate(&e1))) {
        std::vector<double> xg;
        gll_nodes(degree, xg);
        p.fv = dfv;
        p.ff = dff;
        p.cv = dcv;
        p.cf = dcf;
        p.cn = dcn;
        p.cV = dcV;
        p.cd = dcd;
        p.cell_start = dcs;
        p.cell_face = dcface;
        p.nf = nf;
        p.nc = nc;
        p.q1 = q1;
        for (int i = 0; i < q1; ++i) p.xg[i] = xg[i];
        p.tol = normal_tol;
        p.eps = eps;
        for (int i = 0; i < 3; ++i) {
            p.lo[i] = lo[i];
            p.gd[i] = gd[i];
        }
        p.cell = cell;
        p.owner = down;
        p.xi = dxi;
        cudaEventRecord(e0);
        coarse_face_kernel<<<(nc + 255) / 256, 256>>>(dcv, dcf, nc, dcn, dcV, dcd);
        const long long nt = (long long)nf * nq;
        match_kernel<<<(unsigned)((nt + 127) / 128), 128>>>(p);
        cudaEventRecord(e1);
        if (ok(cudaEventSynchronize(e1)) && ok(cudaGetLastError())) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (elapsed_ms) *elapsed_ms = ms;
            if (ok(cudaMemcpy(owner, down, sizeof(long long) * nt, cudaMemcpyDeviceToHost)) &&
                ok(cudaMemcpy(xi_minus, dxi, sizeof(double) * 3 * nt, cudaMemcpyDeviceToHost))) {
                for (long long i = 0; i < nt; ++i)
                    if (owner[i] < 0) {
                        st = SEM_E_UNMATCHED;
                        break;
                    }
            }
        }
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    for (void* ptr : {(void*)dfv, (void*)dcv, (void*)dcn, (void*)dcV, (void*)dcd, (void*)dxi, (void*)dff, (void*)dcf,
                      (void*)dcs, (void*)dcface, (void*)down})
        if (ptr) cudaFree(ptr);
    return st;
}
