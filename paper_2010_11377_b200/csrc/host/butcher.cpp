// Butcher tableaux and block-preconditioner coefficients.
//
// Radau IIA (s = 1..7) and Lobatto IIIC (s = 2..5) are built as collocation
// methods from their quadrature nodes in long double (reference
// butcher.cpp:29-101); the pivot-free Doolittle LDU and the coefficient
// kinds J / GSL / DU / LD follow butcher.cpp:190-288.  All of this is s x s
// host arithmetic uploaded as constants.
#include <cmath>
#include <fstream>

#include "orthopoly.hpp"
#include "setup.hpp"

namespace irkb {
namespace {

// Partial-pivot Gaussian elimination in long double (n <= 7).
std::vector<long double> solve_ld(std::vector<long double> A, std::vector<long double> b, int n) {
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (fabsl(A[i * n + k]) > fabsl(A[p * n + k])) p = i;
        if (A[p * n + k] == 0.0L) throw SingularError("butcher: singular collocation system", k);
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
            std::swap(b[k], b[p]);
        }
        for (int i = k + 1; i < n; ++i) {
            const long double m = A[i * n + k] / A[k * n + k];
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= m * A[k * n + j];
            b[i] -= m * b[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        long double acc = b[i];
        for (int j = i + 1; j < n; ++j) acc -= A[i * n + j] * b[j];
        b[i] = acc / A[i * n + i];
    }
    return b;
}

}  // namespace

Tableau radau_iia(int s) {
    check(s >= 1 && s <= 7, "make_radau_iia: stage count must be in 1..7");
    std::vector<long double> c;
    if (s > 1) {
        auto f = [s](long double x) {
            long double p1, d1, p0, d0;
            legendre_ld(s, x, p1, d1);
            legendre_ld(s - 1, x, p0, d0);
            return p1 - p0;
        };
        auto df = [s](long double x) {
            long double p1, d1, p0, d0;
            legendre_ld(s, x, p1, d1);
            legendre_ld(s - 1, x, p0, d0);
            return d1 - d0;
        };
        for (long double x : roots_in_unit(f, df, s - 1)) c.push_back(0.5L * (x + 1.0L));
    }
    c.push_back(1.0L);

    Tableau t;
    t.s = s;
    t.q = 2 * s - 1;
    t.A.assign(s * s, 0.0);
    t.c.resize(s);
    for (int i = 0; i < s; ++i) t.c[i] = static_cast<double>(c[i]);
    // Collocation: sum_j a_ij c_j^(k-1) = c_i^k / k, k = 1..s.
    std::vector<long double> V(s * s);
    for (int k = 0; k < s; ++k)
        for (int j = 0; j < s; ++j) V[k * s + j] = powl(c[j], k);
    for (int i = 0; i < s; ++i) {
        std::vector<long double> rhs(s);
        for (int k = 0; k < s; ++k) rhs[k] = powl(c[i], k + 1) / (k + 1);
        const auto row = solve_ld(V, rhs, s);
        for (int j = 0; j < s; ++j) t.A[i * s + j] = static_cast<double>(row[j]);
    }
    t.b.assign(t.A.begin() + (s - 1) * s, t.A.end());
    return t;
}

Tableau lobatto_iiic(int s) {
    check(s >= 2 && s <= 5, "make_lobatto_iiic: stage count must be in 2..5");
    std::vector<long double> c{0.0L};
    if (s > 2) {
        auto f = [s](long double x) {
            long double p, dp;
            legendre_ld(s - 1, x, p, dp);
            return dp;
        };
        auto df = [s](long double x) {
            long double p, dp;
            legendre_ld(s - 1, x, p, dp);
            return (2.0L * x * dp - static_cast<long double>(s - 1) * s * p) / (1.0L - x * x);
        };
        for (long double x : roots_in_unit(f, df, s - 2)) c.push_back(0.5L * (x + 1.0L));
    }
    c.push_back(1.0L);

    Tableau t;
    t.s = s;
    t.q = 2 * s - 2;
    t.A.assign(s * s, 0.0);
    t.c.resize(s);
    t.b.resize(s);
    for (int i = 0; i < s; ++i) t.c[i] = static_cast<double>(c[i]);
    // Lobatto weights b_i = 1 / (s (s-1) P_{s-1}(x_i)^2), x = 2c - 1.
    std::vector<long double> bl(s);
    for (int i = 0; i < s; ++i) {
        long double p, dp;
        legendre_ld(s - 1, 2.0L * c[i] - 1.0L, p, dp);
        bl[i] = 1.0L / (static_cast<long double>(s) * (s - 1) * p * p);
        t.b[i] = static_cast<double>(bl[i]);
    }
    // Column 1 pinned to b_1; columns 2..s from collocation k = 1..s-1.
    const int m = s - 1;
    std::vector<long double> V(m * m);
    for (int k = 0; k < m; ++k)
        for (int j = 0; j < m; ++j) V[k * m + j] = powl(c[j + 1], k);
    for (int i = 0; i < s; ++i) {
        t.A[i * s] = static_cast<double>(bl[0]);
        std::vector<long double> rhs(m);
        for (int k = 0; k < m; ++k) {
            rhs[k] = powl(c[i], k + 1) / (k + 1);
            if (k == 0) rhs[k] -= bl[0];
        }
        const auto row = solve_ld(V, rhs, m);
        for (int j = 0; j < m; ++j) t.A[i * s + j + 1] = static_cast<double>(row[j]);
    }
    return t;
}

Tableau make_tableau(Scheme scheme, int s) {
    return scheme == Scheme::LobattoIIIC ? lobatto_iiic(s) : radau_iia(s);
}

Ldu ldu_factorize(int s, const std::vector<double>& A) {
    check(static_cast<int>(A.size()) == s * s, "ldu_factorize: not square");
    double amax = 0.0;
    for (double v : A) amax = std::max(amax, std::fabs(v));
    Ldu f;
    f.L.assign(s * s, 0.0);
    f.U.assign(s * s, 0.0);
    f.D.assign(s, 0.0);
    for (int i = 0; i < s; ++i) f.L[i * s + i] = f.U[i * s + i] = 1.0;
    auto L = [&](int i, int j) -> double& { return f.L[i * s + j]; };
    auto U = [&](int i, int j) -> double& { return f.U[i * s + j]; };
    for (int k = 0; k < s; ++k) {
        double d = A[k * s + k];
        for (int m = 0; m < k; ++m) d -= L(k, m) * f.D[m] * U(m, k);
        if (std::fabs(d) <= 1e-14 * amax)
            throw SingularError("ldu_factorize: zero pivot, leading principal minor " +
                                    std::to_string(k + 1) + " is singular",
                                k + 1);
        f.D[k] = d;
        for (int j = k + 1; j < s; ++j) {
            double u = A[k * s + j];
            for (int m = 0; m < k; ++m) u -= L(k, m) * f.D[m] * U(m, j);
            U(k, j) = u / d;
        }
        for (int i = k + 1; i < s; ++i) {
            double l = A[i * s + k];
            for (int m = 0; m < k; ++m) l -= L(i, m) * f.D[m] * U(m, k);
            L(i, k) = l / d;
        }
    }
    return f;
}

namespace {
void require_nonzero_diagonal(int s, const std::vector<double>& At) {
    for (int i = 0; i < s; ++i)
        if (At[i * s + i] == 0.0)
            throw InvalidArgument("coefficient matrix has a zero diagonal entry");
}
}  // namespace

Coeff precond_coeff(const Tableau& t, CoeffKind kind) {
    const int s = t.s;
    Coeff pc;
    pc.At.assign(s * s, 0.0);
    switch (kind) {
    case CoeffKind::Jacobi:
        for (int i = 0; i < s; ++i) pc.At[i * s + i] = t.A[i * s + i];
        pc.structure = Structure::Diagonal;
        break;
    case CoeffKind::GaussSeidelLower:
        for (int i = 0; i < s; ++i)
            for (int j = 0; j <= i; ++j) pc.At[i * s + j] = t.A[i * s + j];
        pc.structure = Structure::Lower;
        break;
    case CoeffKind::UpperFactor: {
        const Ldu f = ldu_factorize(s, t.A);
        for (int i = 0; i < s; ++i)
            for (int j = i; j < s; ++j) pc.At[i * s + j] = f.D[i] * f.U[i * s + j];
        pc.structure = Structure::Upper;
        break;
    }
    case CoeffKind::LowerFactor: {
        const Ldu f = ldu_factorize(s, t.A);
        for (int i = 0; i < s; ++i)
            for (int j = 0; j <= i; ++j) pc.At[i * s + j] = f.L[i * s + j] * f.D[j];
        pc.structure = Structure::Lower;
        break;
    }
    case CoeffKind::Custom:
        throw InvalidArgument("precond_coeff: use custom_coeff for user matrices");
    }
    require_nonzero_diagonal(s, pc.At);
    return pc;
}

Coeff custom_coeff(int s, const std::vector<double>& At) {
    check(static_cast<int>(At.size()) == s * s, "custom_coeff: not square");
    bool lower_zero = true, upper_zero = true;
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) {
            if (At[i * s + j] == 0.0) continue;
            if (i > j) lower_zero = false;
            if (i < j) upper_zero = false;
        }
    Coeff pc;
    if (lower_zero && upper_zero)
        pc.structure = Structure::Diagonal;
    else if (upper_zero)
        pc.structure = Structure::Lower;
    else if (lower_zero)
        pc.structure = Structure::Upper;
    else
        throw InvalidArgument("coefficient matrix is neither diagonal nor triangular");
    require_nonzero_diagonal(s, At);
    pc.At = At;
    return pc;
}

std::vector<double> read_coeff_file(const std::string& path, int& s) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open coefficient file: " + path);
    s = 0;
    if (!(in >> s) || s < 1) throw IoError("coefficient file: bad stage count");
    std::vector<double> At(static_cast<size_t>(s) * s);
    for (double& a : At)
        if (!(in >> a)) throw IoError("coefficient file: truncated matrix data");
    return At;
}

Coeff make_coeff(const Tableau& t, CoeffKind kind, const std::string& custom_path) {
    if (kind != CoeffKind::Custom) return precond_coeff(t, kind);
    if (custom_path.empty())
        throw InvalidArgument("custom preconditioner requested without --custom-coeff");
    int s = 0;
    std::vector<double> At = read_coeff_file(custom_path, s);
    if (s != t.s)
        throw InvalidArgument("custom coefficient matrix is " + std::to_string(s) + "x" +
                              std::to_string(s) + ", expected s = " + std::to_string(t.s));
    return custom_coeff(s, At);
}

void distinct_diagonals(int s, const std::vector<double>& At,
                        std::vector<int>& solver_of_block,
                        std::vector<double>& distinct) {
    solver_of_block.assign(s, -1);
    distinct.clear();
    for (int j = 0; j < s; ++j) {
        const double d = At[j * s + j];
        int idx = -1;
        for (std::size_t k = 0; k < distinct.size(); ++k)
            if (distinct[k] == d) idx = static_cast<int>(k);
        if (idx < 0) {
            idx = static_cast<int>(distinct.size());
            distinct.push_back(d);
        }
        solver_of_block[j] = idx;
    }
}

}  // namespace irkb
