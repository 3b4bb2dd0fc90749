// Legendre recurrence and a bracketing root finder in long double, shared by
// the quadrature (fem.cpp) and the collocation nodes (butcher.cpp); the
// node-finding strategy of the reference's orthopoly.cpp:27-69.
#pragma once

#include <vector>

#include "sparse.hpp"

namespace irkb {
namespace {

void legendre_ld(int n, long double x, long double& p, long double& dp) {
    if (n == 0) {
        p = 1.0L;
        dp = 0.0L;
        return;
    }
    long double a = 1.0L, b = x;
    for (int k = 2; k <= n; ++k) {
        const long double c = ((2 * k - 1) * x * b - (k - 1) * a) / k;
        a = b;
        b = c;
    }
    p = b;
    dp = n * (x * b - a) / (x * x - 1.0L);
}

// All simple roots of f in (-1,1): sign scan on 4096 cells, 80 bisection
// steps, 4 Newton steps.
template <class F, class D>
std::vector<long double> roots_in_unit(F f, D df, int expected) {
    std::vector<long double> out;
    const int grid = 4096;
    long double lo = -1.0L + 1e-12L, flo = f(lo);
    for (int g = 1; g <= grid; ++g) {
        const long double hi = -1.0L + 2.0L * g / grid - (g == grid ? 1e-12L : 0.0L);
        const long double fhi = f(hi);
        if (flo == 0.0L && (out.empty() || lo - out.back() > 1e-9L)) out.push_back(lo);
        if (flo != 0.0L && fhi != 0.0L && ((flo < 0.0L) != (fhi < 0.0L))) {
            long double a = lo, b = hi, fa = flo;
            for (int it = 0; it < 80; ++it) {
                const long double m = 0.5L * (a + b), fm = f(m);
                if ((fa < 0.0L) == (fm < 0.0L)) {
                    a = m;
                    fa = fm;
                } else {
                    b = m;
                }
            }
            long double x = 0.5L * (a + b);
            for (int it = 0; it < 4; ++it) {
                const long double d = df(x);
                if (d == 0.0L) break;
                x -= f(x) / d;
            }
            if (out.empty() || x - out.back() > 1e-9L) out.push_back(x);
        }
        lo = hi;
        flo = fhi;
    }
    if (static_cast<int>(out.size()) != expected)
        throw NumericalError("butcher: node root scan found the wrong count");
    return out;
}

}  // namespace
}  // namespace irkb
