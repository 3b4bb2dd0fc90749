// Smoothed-aggregation AMG setup (host, once per distinct diagonal block).
//
// The coarsening is the reference's own (BASELINE "AMG hierarchy setup with
// the reference's own coarsening"), restated so that aggregates, P, R and the
// Galerkin operators are bit-identical to amg.cpp:172-227 on the same input:
//   strength graph of |A| + |A|^T with a row-relative, non-strict threshold
//   (amg.cpp:15-42), three greedy aggregation passes (amg.cpp:44-74),
//   rho(D^-1 sym A) by 10 seeded power iterations (amg.cpp:80-98),
//   P = (I - w D^-1 A)^steps T (amg.cpp:207-216), R = P^T, A_c = R (A P).
// The coarsest operator is inverted densely here; the device applies that
// inverse in its coarse solve (the reference uses a sparse LU solve there,
// amg.cpp:149-151, which agrees to rounding).
#include <cmath>
#include <random>

#include "setup.hpp"

namespace irkb {
namespace {

std::vector<double> inverse_diagonal(const Csr& A) {
    std::vector<double> d(A.rows, 0.0);
    for (int i = 0; i < A.rows; ++i)
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
            if (A.idx[k] == i) d[i] = A.val[k];
    for (int i = 0; i < A.rows; ++i) {
        if (d[i] == 0.0)
            throw SingularError("amg_setup: zero diagonal at row " + std::to_string(i), i);
        d[i] = 1.0 / d[i];
    }
    return d;
}

Csr strength_weights(const Csr& A) {
    Csr B = A;
    for (double& v : B.val) v = std::fabs(v);
    return add(1.0, B, 1.0, transpose(B));
}

std::vector<int> aggregate(const Csr& C, double theta, int& n_agg) {
    const int n = C.rows;
    std::vector<double> rmax(n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int k = C.ptr[i]; k < C.ptr[i + 1]; ++k)
            if (C.idx[k] != i) rmax[i] = std::max(rmax[i], C.val[k]);
    auto strong = [&](int i, int k) {
        return C.idx[k] != i && C.val[k] >= theta * rmax[i];
    };
    std::vector<int> agg(n, -1);
    n_agg = 0;
    // Seeds: nodes whose whole strong neighbourhood is unassigned.
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        bool free_nbhd = true;
        for (int k = C.ptr[i]; k < C.ptr[i + 1] && free_nbhd; ++k)
            if (strong(i, k) && agg[C.idx[k]] >= 0) free_nbhd = false;
        if (!free_nbhd) continue;
        agg[i] = n_agg;
        for (int k = C.ptr[i]; k < C.ptr[i + 1]; ++k)
            if (strong(i, k)) agg[C.idx[k]] = n_agg;
        ++n_agg;
    }
    // Leftovers join their strongest already-aggregated strong neighbour.
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        int best = -1;
        double wbest = 0.0;
        for (int k = C.ptr[i]; k < C.ptr[i + 1]; ++k) {
            const int j = C.idx[k];
            if (j == i || agg[j] < 0) continue;
            if (strong(i, k) && C.val[k] > wbest) {
                wbest = C.val[k];
                best = agg[j];
            }
        }
        if (best >= 0) agg[i] = best;
    }
    // Isolated nodes become singletons.
    for (int i = 0; i < n; ++i)
        if (agg[i] < 0) agg[i] = n_agg++;
    return agg;
}

double spectral_radius(const Csr& A, const std::vector<double>& dinv) {
    const Csr S = add(0.5, A, 0.5, transpose(A));
    const int n = A.rows;
    std::mt19937_64 gen(0x1d872b41u);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::vector<double> x(n), y(n);
    for (double& v : x) v = dist(gen);
    double rho = 1.0;
    for (int it = 0; it < 10; ++it) {
        spmv(S, x.data(), y.data());
        for (int i = 0; i < n; ++i) y[i] *= dinv[i];
        rho = std::sqrt(blocked_dot(y.data(), y.data(), n));
        if (rho == 0.0) break;
        const double inv = 1.0 / rho;
        for (double& v : y) v *= inv;
        std::swap(x, y);
    }
    return std::max(rho, 1e-12);
}

}  // namespace

std::vector<double> dense_inverse_host(const Csr& A) {
    const int n = A.rows;
    std::vector<double> M(static_cast<std::size_t>(n) * n, 0.0), X(M.size(), 0.0);
    for (int i = 0; i < n; ++i) {
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) M[static_cast<std::size_t>(i) * n + A.idx[k]] += A.val[k];
        X[static_cast<std::size_t>(i) * n + i] = 1.0;
    }
    // Gauss-Jordan with partial pivoting on [M | I].
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(M[static_cast<std::size_t>(i) * n + k]) > std::fabs(M[static_cast<std::size_t>(p) * n + k])) p = i;
        if (M[static_cast<std::size_t>(p) * n + k] == 0.0)
            throw SingularError("amg coarse solve: matrix is singular at column " + std::to_string(k), k);
        if (p != k)
            for (int j = 0; j < n; ++j) {
                std::swap(M[static_cast<std::size_t>(k) * n + j], M[static_cast<std::size_t>(p) * n + j]);
                std::swap(X[static_cast<std::size_t>(k) * n + j], X[static_cast<std::size_t>(p) * n + j]);
            }
        const double inv = 1.0 / M[static_cast<std::size_t>(k) * n + k];
        for (int j = 0; j < n; ++j) {
            M[static_cast<std::size_t>(k) * n + j] *= inv;
            X[static_cast<std::size_t>(k) * n + j] *= inv;
        }
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            const double f = M[static_cast<std::size_t>(i) * n + k];
            if (f == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                M[static_cast<std::size_t>(i) * n + j] -= f * M[static_cast<std::size_t>(k) * n + j];
                X[static_cast<std::size_t>(i) * n + j] -= f * X[static_cast<std::size_t>(k) * n + j];
            }
        }
    }
    return X;
}

Hierarchy amg_setup(const Csr& A, const AmgParams& p) {
    check(A.rows == A.cols, "amg_setup: matrix must be square");
    check(A.rows > 0, "amg_setup: empty matrix");
    check(p.theta > 0.0 && p.theta < 1.0, "amg_setup: theta must be in (0,1)");
    check(p.pre_sweeps >= 1 && p.post_sweeps >= 1, "amg_setup: sweeps must be >= 1");
    check(p.smoother == 0 || p.smoother == 1, "amg_setup: unknown smoother");

    Hierarchy h;
    h.params = p;
    h.levels.push_back({A, inverse_diagonal(A), {}, {}, {}, {}});
    while (h.levels.back().A.rows > p.max_coarse && h.n_levels() < p.max_levels) {
        AmgLevel& fine = h.levels.back();
        const int n = fine.A.rows;
        int n_agg = 0;
        const std::vector<int> agg = aggregate(strength_weights(fine.A), p.theta, n_agg);
        if (n_agg == 0) throw NumericalError("amg_setup: aggregation stalled");
        if (n_agg > (9 * n) / 10) break;

        Csr P;
        P.rows = n;
        P.cols = n_agg;
        P.ptr.resize(n + 1);
        P.idx = agg;
        P.val.assign(n, 1.0);
        for (int i = 0; i <= n; ++i) P.ptr[i] = i;

        const double w = p.prolongation_weight / spectral_radius(fine.A, fine.inv_diag);
        for (int step = 0; step < p.prolongation_steps; ++step) {
            Csr AP = matmul(fine.A, P);
            for (int i = 0; i < n; ++i) {
                const double sc = w * fine.inv_diag[i];
                for (int k = AP.ptr[i]; k < AP.ptr[i + 1]; ++k) AP.val[k] *= sc;
            }
            P = add(1.0, P, -1.0, AP);
        }
        fine.P = std::move(P);
        fine.R = transpose(fine.P);
        Csr Ac = matmul(fine.R, matmul(fine.A, fine.P));
        std::vector<double> dinv = inverse_diagonal(Ac);
        h.levels.push_back({std::move(Ac), std::move(dinv), {}, {}, {}, {}});
    }
    h.coarse_inverse = dense_inverse_host(h.levels.back().A);
    attach_tail(h, tail_max_rows(h.params));
    attach_composed(h);
    return h;
}

}  // namespace irkb
