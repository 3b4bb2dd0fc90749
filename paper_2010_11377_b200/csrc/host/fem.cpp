// P1 finite-element assembly on the structured SW-NE triangulation.
//
// The reference assembles with a 5x5 Gauss-Legendre rule collapsed onto the
// reference triangle (fem.cpp:14-33) and compresses triplets with a (row,col)
// sort (csr.cpp:55-88).  We evaluate the same quadrature in the same order so
// the assembled M and K are bit-identical to the reference's, which makes the
// strength-of-connection ties in the AMG coarsening (amg.cpp:40-42) resolve
// identically (tests/test_setup_parity.py).
#include <cmath>
#include <cstdint>

#include "orthopoly.hpp"
#include "setup.hpp"

namespace irkb {
namespace {

// Gauss-Legendre on [0,1]: roots of P_n by the shared bracketing finder,
// weights 2 / ((1 - x^2) P_n'(x)^2).
void gauss01(int n, std::vector<double>& pts, std::vector<double>& wts) {
    auto f = [n](long double x) {
        long double p, dp;
        legendre_ld(n, x, p, dp);
        return p;
    };
    auto df = [n](long double x) {
        long double p, dp;
        legendre_ld(n, x, p, dp);
        return dp;
    };
    const std::vector<long double> roots = roots_in_unit(f, df, n);
    pts.clear();
    wts.clear();
    for (long double x : roots) {
        long double p, dp;
        legendre_ld(n, x, p, dp);
        const long double w = 2.0L / ((1.0L - x * x) * dp * dp);
        pts.push_back(static_cast<double>(0.5L * (x + 1.0L)));
        wts.push_back(static_cast<double>(0.5L * w));
    }
}

struct TriRule {
    std::vector<double> xi, eta, w;
};

const TriRule& duffy25() {
    static const TriRule r = [] {
        std::vector<double> p, w;
        gauss01(5, p, w);
        TriRule t;
        for (std::size_t i = 0; i < p.size(); ++i)
            for (std::size_t j = 0; j < p.size(); ++j) {
                t.xi.push_back(p[i]);
                t.eta.push_back(p[j] * (1.0 - p[i]));
                t.w.push_back(w[i] * w[j] * (1.0 - p[i]));
            }
        return t;
    }();
    return r;
}

// Structured lattice: (n+1)^2 vertices, two triangles per cell split along
// the SW-NE diagonal, counterclockwise.
struct Lattice {
    int n;
    double x0, h;
    double x(int i) const { return x0 + i * h; }
    int vid(int i, int j) const { return j * (n + 1) + i; }
};

struct Geometry {
    double ax, ay, J00, J01, J10, J11, det, I00, I01, I10, I11;
};

Geometry geometry(const double* a, const double* b, const double* c) {
    Geometry g;
    g.ax = a[0];
    g.ay = a[1];
    g.J00 = b[0] - a[0];
    g.J01 = c[0] - a[0];
    g.J10 = b[1] - a[1];
    g.J11 = c[1] - a[1];
    g.det = g.J00 * g.J11 - g.J01 * g.J10;
    if (!(g.det > 1e-300)) throw InvalidArgument("assembly: degenerate triangle");
    const double inv = 1.0 / g.det;
    g.I00 = g.J11 * inv;
    g.I01 = -g.J01 * inv;
    g.I10 = -g.J10 * inv;
    g.I11 = g.J00 * inv;
    return g;
}

constexpr double kRefGrad[3][2] = {{-1.0, -1.0}, {1.0, 0.0}, {0.0, 1.0}};

// Visits every triangle in mesh order with its three vertex ids and coords.
template <class F>
void for_each_triangle(const Lattice& L, F&& f) {
    // element e = 2 (j n + i) + t in the reference's (row, cell, triangle)
    // order; cells are independent, so rows of cells run in parallel and each
    // element writes only its own triplet slots (9 e .. 9 e + 8)
#pragma omp parallel for schedule(static)
    for (int j = 0; j < L.n; ++j)
        for (int i = 0; i < L.n; ++i) {
            const long long e0 = 2LL * (static_cast<long long>(j) * L.n + i);
            const int v00 = L.vid(i, j), v10 = L.vid(i + 1, j);
            const int v11 = L.vid(i + 1, j + 1), v01 = L.vid(i, j + 1);
            const double p00[2] = {L.x(i), L.x(j)}, p10[2] = {L.x(i + 1), L.x(j)};
            const double p11[2] = {L.x(i + 1), L.x(j + 1)}, p01[2] = {L.x(i), L.x(j + 1)};
            {
                const int v[3] = {v00, v10, v11};
                const double* p[3] = {p00, p10, p11};
                f(e0, v, p);
            }
            {
                const int v[3] = {v00, v11, v01};
                const double* p[3] = {p00, p11, p01};
                f(e0 + 1, v, p);
            }
        }
}

struct FreeMap {
    std::vector<int> to_free;  // -1 on boundary nodes
    std::vector<int> free_ids;
};

FreeMap free_map(int n) {
    const int nps = n + 1;
    FreeMap m;
    m.to_free.assign(static_cast<std::size_t>(nps) * nps, -1);
    for (int j = 0; j < nps; ++j)
        for (int i = 0; i < nps; ++i) {
            if (i == 0 || j == 0 || i == nps - 1 || j == nps - 1) continue;
            m.to_free[j * nps + i] = static_cast<int>(m.free_ids.size());
            m.free_ids.push_back(j * nps + i);
        }
    return m;
}

Csr restrict_free(const Csr& A, const FreeMap& fm) {
    Csr R;
    const int nf = static_cast<int>(fm.free_ids.size());
    R.rows = R.cols = nf;
    R.ptr.assign(nf + 1, 0);
    for (int r = 0; r < nf; ++r) {
        const int i = fm.free_ids[r];
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int c = fm.to_free[A.idx[k]];
            if (c < 0) continue;
            R.idx.push_back(c);
            R.val.push_back(A.val[k]);
        }
        R.ptr[r + 1] = static_cast<int>(R.idx.size());
    }
    return R;
}

std::vector<double> lift_free(const Csr& A, const FreeMap& fm, const std::vector<double>& g) {
    std::vector<double> prod(A.rows);
    spmv(A, g.data(), prod.data());
    std::vector<double> out(fm.free_ids.size());
    for (std::size_t k = 0; k < out.size(); ++k) out[k] = prod[fm.free_ids[k]];
    return out;
}

void fill_coords(Problem& P, const Lattice& L, const FreeMap& fm) {
    const int nps = L.n + 1;
    P.coords.resize(fm.free_ids.size());
    for (std::size_t k = 0; k < fm.free_ids.size(); ++k) {
        const int id = fm.free_ids[k];
        P.coords[k] = {L.x(id % nps), L.x(id / nps)};
    }
}

}  // namespace

Problem make_heat_problem(int cells) {
    check(cells >= 2, "heat problem: cells >= 2");
    const Lattice L{cells, 0.0, 1.0 / cells};
    const int nv = (cells + 1) * (cells + 1);
    const TriRule& q = duffy25();
    Triplets tm(nv, nv), tk(nv, nv);
    tm.resize(static_cast<std::size_t>(18) * cells * cells);
    tk.resize(static_cast<std::size_t>(18) * cells * cells);
    for_each_triangle(L, [&](long long e, const int* v, const double* const* p) {
        const Geometry g = geometry(p[0], p[1], p[2]);
        double gx[3], gy[3];
        for (int a = 0; a < 3; ++a) {
            gx[a] = g.I00 * kRefGrad[a][0] + g.I10 * kRefGrad[a][1];
            gy[a] = g.I01 * kRefGrad[a][0] + g.I11 * kRefGrad[a][1];
        }
        double me[3][3] = {}, ke[3][3] = {};
        for (std::size_t k = 0; k < q.w.size(); ++k) {
            const double scale = q.w[k] * g.det;
            const double N[3] = {1.0 - q.xi[k] - q.eta[k], q.xi[k], q.eta[k]};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    me[a][b] += scale * (N[b] * N[a]);
                    ke[a][b] += scale * (1.0 * (gx[b] * gx[a] + gy[b] * gy[a]));
                }
        }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                tm.set(9 * e + 3 * a + b, v[a], v[b], me[a][b]);
                tk.set(9 * e + 3 * a + b, v[a], v[b], ke[a][b]);
            }
    });
    const Csr M = tm.compress(), K = tk.compress();
    const FreeMap fm = free_map(cells);
    Problem P;
    P.cells = cells;
    P.M = restrict_free(M, fm);
    P.K = restrict_free(K, fm);
    P.f_lift = lift_free(K, fm, std::vector<double>(nv, 0.0));
    fill_coords(P, L, fm);
    return P;
}

Problem make_double_glazing_problem(int cells, double eps) {
    check(cells >= 2, "double glazing: cells >= 2");
    check(eps > 0.0, "double glazing: eps must be positive");
    const Lattice L{cells, -1.0, 2.0 / cells};
    const int nv = (cells + 1) * (cells + 1);
    const TriRule& q = duffy25();
    auto wind = [](double x, double y, double w[2]) {
        w[0] = 2.0 * y * (1.0 - x * x);
        w[1] = -2.0 * x * (1.0 - y * y);
    };
    Triplets tf(nv, nv), tm(nv, nv);
    tf.resize(static_cast<std::size_t>(18) * cells * cells);
    tm.resize(static_cast<std::size_t>(18) * cells * cells);
    for_each_triangle(L, [&](long long e, const int* v, const double* const* p) {
        const Geometry g = geometry(p[0], p[1], p[2]);
        auto edge = [](const double* a, const double* b) {
            return std::hypot(b[0] - a[0], b[1] - a[1]);
        };
        const double he = std::max(std::max(edge(p[0], p[1]), edge(p[1], p[2])),
                                   edge(p[2], p[0]));
        double wc[2];
        wind((p[0][0] + p[1][0] + p[2][0]) / 3.0, (p[0][1] + p[1][1] + p[2][1]) / 3.0, wc);
        const double wmag = std::hypot(wc[0], wc[1]);
        double delta = 0.0;
        if (wmag > 0.0) {
            const double pe = wmag * he / (2.0 * eps);
            delta = he / (2.0 * wmag) * std::max(0.0, 1.0 - 1.0 / pe);
        }
        double gx[3], gy[3];
        for (int a = 0; a < 3; ++a) {
            gx[a] = g.I00 * kRefGrad[a][0] + g.I10 * kRefGrad[a][1];
            gy[a] = g.I01 * kRefGrad[a][0] + g.I11 * kRefGrad[a][1];
        }
        double fe[3][3] = {}, me[3][3] = {};
        for (std::size_t k = 0; k < q.w.size(); ++k) {
            const double scale = q.w[k] * g.det;
            const double N[3] = {1.0 - q.xi[k] - q.eta[k], q.xi[k], q.eta[k]};
            const double x = g.ax + g.J00 * q.xi[k] + g.J01 * q.eta[k];
            const double y = g.ay + g.J10 * q.xi[k] + g.J11 * q.eta[k];
            double w[2];
            wind(x, y, w);
            double conv[3];
            for (int a = 0; a < 3; ++a) conv[a] = w[0] * gx[a] + w[1] * gy[a];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    fe[a][b] += scale * (eps * (gx[b] * gx[a] + gy[b] * gy[a]) +
                                         conv[b] * N[a] + delta * (conv[b] * conv[a]));
                    me[a][b] += scale * (N[b] * N[a] + delta * (N[b] * conv[a]));
                }
        }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                tf.set(9 * e + 3 * a + b, v[a], v[b], fe[a][b]);
                tm.set(9 * e + 3 * a + b, v[a], v[b], me[a][b]);
            }
    });
    const Csr F = tf.compress(), M = tm.compress();
    const FreeMap fm = free_map(cells);
    // Wall data: East = 1, others 0; the East value wins at corners.
    std::vector<double> g(nv, 0.0);
    const int nps = cells + 1;
    for (int j = 0; j < nps; ++j)
        for (int i = 0; i < nps; ++i)
            if (i == nps - 1) g[j * nps + i] = 1.0;
    Problem P;
    P.cells = cells;
    P.M = restrict_free(M, fm);
    P.K = restrict_free(F, fm);
    P.f_lift = lift_free(F, fm, g);
    fill_coords(P, L, fm);
    return P;
}

std::vector<double> heat_initial(const Problem& p, double noise_amp,
                                 unsigned long long seed) {
    constexpr double pi = 3.14159265358979323846;
    std::uint64_t st = seed;
    auto next = [&st]() {
        std::uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    std::vector<double> u(p.coords.size());
    for (std::size_t k = 0; k < u.size(); ++k) {
        u[k] = std::sin(pi * p.coords[k][0]) * std::sin(pi * p.coords[k][1]);
        if (noise_amp != 0.0) {
            const double r = static_cast<double>(next() >> 11) * 0x1.0p-53;
            u[k] += noise_amp * (2.0 * r - 1.0);
        }
    }
    return u;
}

}  // namespace irkb
