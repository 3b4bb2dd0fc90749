// On-disk formats around the solve path: MatrixMarket
// coordinate files (csr.cpp:240-290) so the device path can consume
// reference-assembled M / K, and the study driver's CSV rows
// (study.cpp:334-360) so device runs can be tabulated beside reference runs.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "mmio.hpp"

namespace irkb {

void write_matrix_market(const Csr& A, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw IoError("cannot open for write: " + path);
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%d %d %d\n", A.rows, A.cols, A.nnz());
    for (int i = 0; i < A.rows; ++i)
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
            std::fprintf(f, "%d %d %.17g\n", i + 1, A.idx[k] + 1, A.val[k]);
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) throw IoError("write failed: " + path);
}

// C stdio parsing (strtod is correctly rounded, like the reference's
// istream extraction, so %.17g files round-trip exactly).
Csr read_matrix_market(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw IoError("cannot open for read: " + path);
    struct Closer {
        std::FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    std::string line;
    auto next_line = [&]() {
        line.clear();
        int ch;
        while ((ch = std::fgetc(f)) != EOF && ch != '\n') line.push_back(static_cast<char>(ch));
        return !(ch == EOF && line.empty());
    };
    bool header = false, symmetric = false, sized = false;
    long nr = 0, nc = 0, nz = 0;
    while (next_line()) {
        if (line.empty()) continue;
        if (line[0] == '%') {
            if (!header && line.compare(0, 14, "%%MatrixMarket") == 0) {
                header = true;
                symmetric = line.find("symmetric") != std::string::npos;
                check(line.find("coordinate") != std::string::npos &&
                          line.find("real") != std::string::npos,
                      "matrix market: only coordinate real supported");
            }
            continue;
        }
        sized = std::sscanf(line.c_str(), "%ld %ld %ld", &nr, &nc, &nz) == 3;
        break;
    }
    check(sized, "matrix market: bad size line");
    check(nr >= 0 && nc >= 0 && nz >= 0 && nr < (1L << 31) && nc < (1L << 31),
          "matrix market: bad size line");
    Triplets t(static_cast<int>(nr), static_cast<int>(nc));
    t.reserve(static_cast<size_t>(nz) * (symmetric ? 2 : 1));
    for (long e = 0; e < nz; ++e) {
        long i, j;
        char vbuf[128];
        if (std::fscanf(f, "%ld %ld %127s", &i, &j, vbuf) != 3)
            throw IoError("matrix market: truncated entry list");
        char* end = nullptr;
        const double v = std::strtod(vbuf, &end);
        if (end == vbuf) throw IoError("matrix market: truncated entry list");
        t.add(static_cast<int>(i - 1), static_cast<int>(j - 1), v);
        if (symmetric && i != j) t.add(static_cast<int>(j - 1), static_cast<int>(i - 1), v);
    }
    return t.compress();
}

namespace {

const char* scheme_name(int s) { return s == 0 ? "radau_iia" : s == 1 ? "lobatto_iiic" : "custom"; }

const char* kind_name(int k) {
    switch (k) {
    case 0: return "jacobi";
    case 1: return "gsl";
    case 2: return "du";
    case 3: return "ld";
    default: return "custom";
    }
}

}  // namespace

std::string csv_header() {
    return "scheme,s,hx_inv,ht,dof,precond,side,subsolver,iterations,"
           "true_residual,rel_error,seconds\n";
}

std::string csv_row(const CsvCell& c) {
    char buf[384];
    const int dof = c.s * c.n_free;
    const char* side = c.side == 0 ? "left" : "right";
    const char* sub = c.subsolver == 1 ? "lu" : "amg";
    if (c.failed)
        std::snprintf(buf, sizeof buf, "%s,%d,%d,%.12g,%d,%s,%s,%s,failed,,,\n",
                      scheme_name(c.scheme), c.s, c.hx_inv, c.ht, dof, kind_name(c.kind), side, sub);
    else
        std::snprintf(buf, sizeof buf, "%s,%d,%d,%.12g,%d,%s,%s,%s,%.10g,%.6e,%.6e,%.4f\n",
                      scheme_name(c.scheme), c.s, c.hx_inv, c.ht, dof, kind_name(c.kind), side, sub,
                      c.iterations, c.true_residual, c.rel_error, c.seconds);
    return buf;
}

}  // namespace irkb
