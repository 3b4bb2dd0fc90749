#include "sparse.hpp"

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <numeric>

namespace irkb {

void Csr::validate() const {
    check(rows >= 0 && cols >= 0, "csr: negative dimension");
    check(static_cast<int>(ptr.size()) == rows + 1, "csr: row_ptr size mismatch");
    check(ptr.front() == 0 && ptr.back() == nnz(), "csr: row_ptr bounds");
    check(idx.size() == val.size(), "csr: col/val size mismatch");
    for (int i = 0; i < rows; ++i) {
        check(ptr[i] <= ptr[i + 1], "csr: row_ptr not nondecreasing");
        for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
            check(idx[k] >= 0 && idx[k] < cols, "csr: column index out of range");
            check(k == ptr[i] || idx[k - 1] < idx[k],
                  "csr: columns not strictly increasing in row");
        }
    }
}

Csr Triplets::compress() const {
    const std::size_t nt = v_.size();
    // The reference sorts an index permutation by (row, col) with std::sort
    // (csr.cpp:55-62) and sums duplicates in the resulting order.  Sorting
    // (key, value) pairs by key alone performs the same comparisons and
    // moves, hence leaves the values in the same order -- with contiguous
    // keys and a linear summation pass instead of indirect loads.
    struct KV {
        std::uint64_t key;
        double v;
    };
    std::vector<KV> kv(nt);
    for (std::size_t t = 0; t < nt; ++t) {
        check(r_[t] >= 0 && r_[t] < rows_ && c_[t] >= 0 && c_[t] < cols_, "triplets: index out of range");
        kv[t] = {(static_cast<std::uint64_t>(static_cast<std::uint32_t>(r_[t])) << 32) |
                     static_cast<std::uint32_t>(c_[t]),
                 v_[t]};
    }
    std::sort(kv.begin(), kv.end(), [](const KV& a, const KV& b) { return a.key < b.key; });
    Csr A;
    A.rows = rows_;
    A.cols = cols_;
    A.ptr.assign(rows_ + 1, 0);
    A.idx.reserve(nt);
    A.val.reserve(nt);
    std::uint64_t last = ~std::uint64_t{0};
    for (const KV& e : kv) {
        if (e.key == last) {
            A.val.back() += e.v;
            continue;
        }
        const int r = static_cast<int>(e.key >> 32), c = static_cast<int>(e.key & 0xffffffffu);
        A.idx.push_back(c);
        A.val.push_back(e.v);
        ++A.ptr[r + 1];
        last = e.key;
    }
    std::partial_sum(A.ptr.begin(), A.ptr.end(), A.ptr.begin());
    return A;
}

Csr transpose(const Csr& A) {
    Csr T;
    T.rows = A.cols;
    T.cols = A.rows;
    T.ptr.assign(T.rows + 1, 0);
    T.idx.resize(A.idx.size());
    T.val.resize(A.val.size());
    for (int c : A.idx) ++T.ptr[c + 1];
    std::partial_sum(T.ptr.begin(), T.ptr.end(), T.ptr.begin());
    std::vector<int> fill(T.ptr.begin(), T.ptr.end() - 1);
    for (int i = 0; i < A.rows; ++i)
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int at = fill[A.idx[k]]++;
            T.idx[at] = i;
            T.val[at] = A.val[k];
        }
    return T;
}

Csr add(double alpha, const Csr& A, double beta, const Csr& B) {
    check(A.rows == B.rows && A.cols == B.cols, "csr add: shape mismatch");
    Csr C;
    C.rows = A.rows;
    C.cols = A.cols;
    C.ptr.resize(A.rows + 1);
    C.ptr[0] = 0;
    C.idx.reserve(std::max(A.idx.size(), B.idx.size()));
    C.val.reserve(C.idx.capacity());
    for (int i = 0; i < A.rows; ++i) {
        int a = A.ptr[i], b = B.ptr[i];
        const int ae = A.ptr[i + 1], be = B.ptr[i + 1];
        while (a < ae || b < be) {
            const int ca = a < ae ? A.idx[a] : INT32_MAX;
            const int cb = b < be ? B.idx[b] : INT32_MAX;
            if (ca == cb) {
                C.idx.push_back(ca);
                C.val.push_back(alpha * A.val[a++] + beta * B.val[b++]);
            } else if (ca < cb) {
                C.idx.push_back(ca);
                C.val.push_back(alpha * A.val[a++]);
            } else {
                C.idx.push_back(cb);
                C.val.push_back(beta * B.val[b++]);
            }
        }
        C.ptr[i + 1] = static_cast<int>(C.idx.size());
    }
    return C;
}

Csr matmul(const Csr& A, const Csr& B) {
    check(A.cols == B.rows, "csr matmul: shape mismatch");
    Csr C;
    C.rows = A.rows;
    C.cols = B.cols;
    C.ptr.assign(A.rows + 1, 0);
    std::vector<double> acc(B.cols, 0.0);
    std::vector<int> seen(B.cols, -1);
    std::vector<int> touched;
    for (int i = 0; i < A.rows; ++i) {
        touched.clear();
        for (int ka = A.ptr[i]; ka < A.ptr[i + 1]; ++ka) {
            const int j = A.idx[ka];
            const double a = A.val[ka];
            for (int kb = B.ptr[j]; kb < B.ptr[j + 1]; ++kb) {
                const int c = B.idx[kb];
                if (seen[c] != i) {
                    seen[c] = i;
                    acc[c] = 0.0;
                    touched.push_back(c);
                }
                acc[c] += a * B.val[kb];
            }
        }
        std::sort(touched.begin(), touched.end());
        for (int c : touched) {
            C.idx.push_back(c);
            C.val.push_back(acc[c]);
        }
        C.ptr[i + 1] = static_cast<int>(C.idx.size());
    }
    return C;
}

void spmv(const Csr& A, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < A.rows; ++i) {
        double s = 0.0;
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) s += A.val[k] * x[A.idx[k]];
        y[i] = s;
    }
}

double blocked_dot(const double* x, const double* y, std::size_t n) {
    constexpr std::size_t kChunk = 4096;
    const std::size_t nb = (n + kChunk - 1) / kChunk;
    std::vector<double> part(nb);
#pragma omp parallel for schedule(static)
    for (std::ptrdiff_t b = 0; b < static_cast<std::ptrdiff_t>(nb); ++b) {
        const std::size_t lo = b * kChunk, hi = std::min(n, lo + kChunk);
        double s = 0.0;
        for (std::size_t i = lo; i < hi; ++i) s += x[i] * y[i];
        part[b] = s;
    }
    double s = 0.0;
    for (double p : part) s += p;
    return s;
}

}  // namespace irkb
