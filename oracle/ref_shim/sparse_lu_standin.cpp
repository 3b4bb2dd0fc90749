// TEST INFRASTRUCTURE ONLY (oracle/_ref).  Never linked into the product.
//
// Stand-in for the reference's Eigen-backed `irkprec::SparseLu`
// (/root/reference/proj/src/sparse_lu.cpp:1-66).  Eigen3 is not present in
// this image, so the reference cannot be compiled with its own sparse_lu.cpp.
// The reference hot path only uses SparseLu for the AMG coarsest-level solve
// (amg.cpp:150, amg.cpp:225), where n <= a few hundred, so a dense
// partial-pivot LU reproduces the *solution* contract pinned by the
// reference's tests (test_sparsela.cpp:73-134, test_amg.cpp:40-50), not
// Eigen's rounding.  Singular matrices throw SingularError like
// sparse_lu.cpp:30-32.
#include "irkprec/sparse_lu.hpp"

#include <cmath>
#include <string>
#include <vector>

namespace irkprec {

struct SparseLu::Impl {
    int n = 0;
    std::vector<double> lu;  // row-major packed L\U, L unit lower
    std::vector<int> perm;   // row permutation: row i of PA is row perm[i] of A
};

SparseLu::SparseLu(const CsrMatrix& A) : impl_(new Impl), n_(A.n_rows) {
    require(A.square(), "sparse_lu: matrix must be square");
    require(A.n_rows > 0, "sparse_lu: empty matrix");
    const int n = A.n_rows;
    Impl& f = *impl_;
    f.n = n;
    f.lu.assign(static_cast<std::size_t>(n) * n, 0.0);
    f.perm.resize(n);
    for (int i = 0; i < n; ++i) {
        f.perm[i] = i;
        for (int k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k)
            f.lu[static_cast<std::size_t>(i) * n + A.col_idx[k]] += A.vals[k];
    }
    auto at = [&](int i, int j) -> double& {
        return f.lu[static_cast<std::size_t>(i) * n + j];
    };
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(at(i, k)) > std::fabs(at(p, k))) p = i;
        if (at(p, k) == 0.0)
            throw SingularError("sparse_lu: matrix is structurally or numerically "
                                "singular: zero pivot in column " +
                                std::to_string(k));
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(at(k, j), at(p, j));
            std::swap(f.perm[k], f.perm[p]);
        }
        const double piv = at(k, k);
        for (int i = k + 1; i < n; ++i) {
            const double m = at(i, k) / piv;
            at(i, k) = m;
            if (m != 0.0)
                for (int j = k + 1; j < n; ++j) at(i, j) -= m * at(k, j);
        }
    }
}

SparseLu::~SparseLu() = default;
SparseLu::SparseLu(SparseLu&&) noexcept = default;
SparseLu& SparseLu::operator=(SparseLu&&) noexcept = default;

void SparseLu::solve(std::span<const double> b, std::span<double> x) const {
    require(static_cast<int>(b.size()) == n_, "lu_solve: rhs size mismatch");
    require(static_cast<int>(x.size()) == n_, "lu_solve: out size mismatch");
    const Impl& f = *impl_;
    const int n = f.n;
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) {
        double s = b[f.perm[i]];
        for (int j = 0; j < i; ++j) s -= f.lu[static_cast<std::size_t>(i) * n + j] * y[j];
        y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int j = i + 1; j < n; ++j) s -= f.lu[static_cast<std::size_t>(i) * n + j] * y[j];
        y[i] = s / f.lu[static_cast<std::size_t>(i) * n + i];
    }
    for (int i = 0; i < n; ++i) x[i] = y[i];
}

Vec SparseLu::solve(std::span<const double> b) const {
    Vec x(static_cast<std::size_t>(n_));
    solve(b, x);
    return x;
}

Vec SparseLu::solve_transposed(std::span<const double> b) const {
    require(static_cast<int>(b.size()) == n_, "lu_solve: rhs size mismatch");
    // A^T x = b with PA = LU:  U^T L^T P x = b.
    const Impl& f = *impl_;
    const int n = f.n;
    std::vector<double> y(b.begin(), b.end());
    for (int i = 0; i < n; ++i) {
        double s = y[i];
        for (int j = 0; j < i; ++j) s -= f.lu[static_cast<std::size_t>(j) * n + i] * y[j];
        y[i] = s / f.lu[static_cast<std::size_t>(i) * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int j = i + 1; j < n; ++j) s -= f.lu[static_cast<std::size_t>(j) * n + i] * y[j];
        y[i] = s;
    }
    Vec x(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) x[f.perm[i]] = y[i];
    return x;
}

Vec lu_solve(const SparseLu& f, std::span<const double> b) { return f.solve(b); }

SparseLu sparse_lu_factor(const CsrMatrix& A) { return SparseLu(A); }

} // namespace irkprec
