// Host-side sparse containers and the setup-time sparse algebra of the
// B200 IRK solve phase.  Nothing here is on the timed path: these routines
// build the operators that are uploaded once.
//
// Arithmetic order is chosen so that every integer structure and every value
// agrees bit-for-bit with the reference's CSR algebra
// (/root/reference/proj/src/csr.cpp) on the same inputs; the tests check this
// against oracle/_ref.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace irkb {

// Error classes mirror the reference's (common.hpp:16-41): the C ABI maps
// them onto distinct status codes and the C++ facade rethrows them.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct SingularError : std::runtime_error {
    int index;
    explicit SingularError(const std::string& w, int idx = -1)
        : std::runtime_error(w), index(idx) {}
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// File I/O and parse failures: the reference throws plain std::runtime_error
// (butcher.cpp:300-313, csr.cpp:240-290).
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(bool ok, const char* msg) {
    if (!ok) throw InvalidArgument(msg);
}

// CSR with int32 indices and fp64 values, strictly increasing columns per
// row (csr.hpp:15-32).
struct Csr {
    int rows = 0, cols = 0;
    std::vector<int> ptr;   // rows + 1
    std::vector<int> idx;   // nnz
    std::vector<double> val;

    int nnz() const { return static_cast<int>(val.size()); }
    bool same_pattern(const Csr& o) const {
        return rows == o.rows && cols == o.cols && ptr == o.ptr && idx == o.idx;
    }
    void validate() const;
};

// Coordinate accumulator; duplicates are summed in the order produced by a
// (row, col) std::sort of the insertion sequence, the order the reference's
// TripletBuilder::compress uses (csr.cpp:55-88).
class Triplets {
public:
    Triplets(int rows, int cols) : rows_(rows), cols_(cols) {}
    void reserve(std::size_t n) { r_.reserve(n); c_.reserve(n); v_.reserve(n); }
    void add(int r, int c, double v) { r_.push_back(r); c_.push_back(c); v_.push_back(v); }
    // fixed-slot filling (parallel assembly): the slot order is the add order
    void resize(std::size_t n) { r_.resize(n); c_.resize(n); v_.resize(n); }
    void set(std::size_t k, int r, int c, double v) { r_[k] = r; c_[k] = c; v_[k] = v; }
    Csr compress() const;

private:
    int rows_, cols_;
    std::vector<int> r_, c_;
    std::vector<double> v_;
};

Csr transpose(const Csr& A);
// alpha*A + beta*B over the union pattern (explicit zeros kept).
Csr add(double alpha, const Csr& A, double beta, const Csr& B);
// Row-wise Gustavson product, columns sorted per row.
Csr matmul(const Csr& A, const Csr& B);
void spmv(const Csr& A, const double* x, double* y);

// Fixed-block (4096) deterministic reduction, the association of the
// reference's dot (kernels.cpp:14-49); used only by setup-time estimates.
double blocked_dot(const double* x, const double* y, std::size_t n);

}  // namespace irkb
