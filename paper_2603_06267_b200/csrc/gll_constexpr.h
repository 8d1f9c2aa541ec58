// Compile-time GLL tables for the volume kernel (degree N is a template parameter there).
//
// The 1D operator rows of DESIGN.md "1D operator rows" are  G_d[row][b] = s_d * Ghat[row][b]  with the
// per-box scale s_d = c^2 (2/h_d)^2 and the reference rows Ghat (functions of N only):
//     R[a][b] = A[a][b] / w_asm(a)   (w_asm = 2 w_0 at a = 0, w_a otherwise)
//     L[b]    = A[N][b] / (2 w_0),   B0 = 2 R[0],   BN = 2 L
//     A       = D^T diag(w) D        (1D GLL stiffness on [-1, 1]),  D[i][j] = ell_j'(xi_i).
// Computing Ghat at compile time lets the kernel use literal coefficients (no parameter-bank traffic,
// no registers) and apply s_d once per direction.  Nodes: Newton on (1 - x^2) P_N'(x) from the
// Chebyshev-Gauss-Lobatto points, weights 2 / (N (N+1) P_N(x)^2).
#pragma once

namespace sem {
namespace gllc {

constexpr double kPi = 3.14159265358979323846264338327950288;

constexpr double cos_cx(double x) {   // |x| <= pi: Taylor series, 40 terms
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 40; ++k) {
        term *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
        sum += term;
    }
    return sum;
}

constexpr double abs_cx(double x) { return x < 0 ? -x : x; }

template <int N>
struct Tables {
    double x[N + 1];
    double w[N + 1];
    double R[N][N + 1];   // reference rows R[a], a = 0..N-1
    double L[N + 1];      // left-element row of a shared node
    double D[N + 1][N + 1];   // differentiation matrix D[i][j] = l_j'(x_i)
};

template <int N>
constexpr Tables<N> make_tables() {
    Tables<N> t{};
    // nodes (descending from the Newton iteration, then reversed to ascending)
    double x[N + 1] = {};
    for (int i = 0; i <= N; ++i) x[i] = cos_cx(kPi * i / N);
    for (int it = 0; it < 100; ++it) {
        for (int i = 0; i <= N; ++i) {
            double p0 = 1.0, p1 = x[i];
            for (int k = 2; k <= N; ++k) {
                const double p2 = ((2.0 * k - 1.0) * x[i] * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            x[i] = x[i] - (x[i] * p1 - p0) / ((N + 1.0) * p1);
        }
    }
    for (int i = 0; i <= N; ++i) t.x[i] = x[N - i];
    t.x[0] = -1.0;
    t.x[N] = 1.0;
    for (int i = 0; i <= N; ++i) {
        double p0 = 1.0, p1 = t.x[i];
        for (int k = 2; k <= N; ++k) {
            const double p2 = ((2.0 * k - 1.0) * t.x[i] * p1 - (k - 1.0) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        t.w[i] = 2.0 / (N * (N + 1.0) * p1 * p1);
    }
    // barycentric derivative matrix
    double lam[N + 1] = {};
    for (int j = 0; j <= N; ++j) {
        lam[j] = 1.0;
        for (int k = 0; k <= N; ++k)
            if (k != j) lam[j] /= (t.x[j] - t.x[k]);
    }
    double D[N + 1][N + 1] = {};
    for (int i = 0; i <= N; ++i) {
        double s = 0.0;
        for (int j = 0; j <= N; ++j)
            if (j != i) {
                D[i][j] = (lam[j] / lam[i]) / (t.x[i] - t.x[j]);
                s += D[i][j];
            }
        D[i][i] = -s;
    }
    for (int i = 0; i <= N; ++i)
        for (int j = 0; j <= N; ++j) t.D[i][j] = D[i][j];
    double A[N + 1][N + 1] = {};
    for (int a = 0; a <= N; ++a)
        for (int b = 0; b <= N; ++b) {
            double s = 0.0;
            for (int q = 0; q <= N; ++q) s += t.w[q] * D[q][a] * D[q][b];
            A[a][b] = s;
        }
    for (int a = 0; a < N; ++a)
        for (int b = 0; b <= N; ++b) t.R[a][b] = A[a][b] / (a == 0 ? 2.0 * t.w[0] : t.w[a]);
    for (int b = 0; b <= N; ++b) t.L[b] = A[N][b] / (2.0 * t.w[0]);
    return t;
}

template <int N>
struct Gll {
    static constexpr Tables<N> T = make_tables<N>();
};

}  // namespace gllc
}  // namespace sem
