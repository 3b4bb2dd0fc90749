// MatrixMarket I/O (csr.cpp:240-290) and study CSV rows (study.cpp:334-360).
#pragma once

#include <string>

#include "sparse.hpp"

namespace irkb {

// "%%MatrixMarket matrix coordinate real general", 1-based, %.17g values.
void write_matrix_market(const Csr& A, const std::string& path);
// coordinate real (general or symmetric, mirrored); duplicates summed by the
// triplet compression (csr.cpp:55-90 order).
Csr read_matrix_market(const std::string& path);

struct CsvCell {
    int scheme = 0, s = 1, hx_inv = 0, n_free = 0, kind = 3, side = 1, subsolver = 0;
    double ht = 0.0, iterations = 0.0, true_residual = 0.0, rel_error = 0.0, seconds = 0.0;
    bool failed = false;
};

std::string csv_header();
std::string csv_row(const CsvCell& c);

}  // namespace irkb
