#include "sparse.hpp"

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <numeric>

#include <omp.h>

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

// Threads take contiguous row blocks; per-thread column counts give every
// (column, thread) pair its slot range, so entries land in row order inside
// each column exactly as in the sequential counting sort.
Csr transpose(const Csr& A) {
    Csr T;
    T.rows = A.cols;
    T.cols = A.rows;
    T.ptr.assign(T.rows + 1, 0);
    T.idx.resize(A.idx.size());
    T.val.resize(A.val.size());
    const int nt = A.idx.size() >= (1u << 16) ? omp_get_max_threads() : 1;
    std::vector<std::vector<int>> cnt(nt);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const int lo = static_cast<int>(static_cast<long long>(A.rows) * t / nt);
        const int hi = static_cast<int>(static_cast<long long>(A.rows) * (t + 1) / nt);
        std::vector<int>& c = cnt[t];
        c.assign(A.cols, 0);
        for (int k = A.ptr[lo]; k < A.ptr[hi]; ++k) ++c[A.idx[k]];
#pragma omp barrier
#pragma omp single
        {
            int run = 0;
            for (int col = 0; col < A.cols; ++col) {
                T.ptr[col] = run;
                for (int u = 0; u < nt; ++u) {
                    const int m = cnt[u][col];
                    cnt[u][col] = run;  // this thread's first slot in the column
                    run += m;
                }
            }
            T.ptr[A.cols] = run;
        }
        for (int i = lo; i < hi; ++i)
            for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
                const int at = c[A.idx[k]]++;
                T.idx[at] = i;
                T.val[at] = A.val[k];
            }
    }
    return T;
}

// alpha*A + beta*B over the union pattern: row counts, prefix sum, then every
// row merged independently (same expressions as the sequential merge).
Csr add(double alpha, const Csr& A, double beta, const Csr& B) {
    check(A.rows == B.rows && A.cols == B.cols, "csr add: shape mismatch");
    Csr C;
    C.rows = A.rows;
    C.cols = A.cols;
    C.ptr.assign(A.rows + 1, 0);
    auto merge = [&](int i, int* oi, double* ov) {
        int a = A.ptr[i], b = B.ptr[i], m = 0;
        const int ae = A.ptr[i + 1], be = B.ptr[i + 1];
        while (a < ae || b < be) {
            const int ca = a < ae ? A.idx[a] : INT32_MAX;
            const int cb = b < be ? B.idx[b] : INT32_MAX;
            if (ca == cb) {
                if (oi) {
                    oi[m] = ca;
                    ov[m] = alpha * A.val[a] + beta * B.val[b];
                }
                ++a;
                ++b;
            } else if (ca < cb) {
                if (oi) {
                    oi[m] = ca;
                    ov[m] = alpha * A.val[a];
                }
                ++a;
            } else {
                if (oi) {
                    oi[m] = cb;
                    ov[m] = beta * B.val[b];
                }
                ++b;
            }
            ++m;
        }
        return m;
    };
#pragma omp parallel for schedule(static)
    for (int i = 0; i < A.rows; ++i) C.ptr[i + 1] = merge(i, nullptr, nullptr);
    std::partial_sum(C.ptr.begin(), C.ptr.end(), C.ptr.begin());
    C.idx.resize(C.ptr.back());
    C.val.resize(C.ptr.back());
#pragma omp parallel for schedule(static)
    for (int i = 0; i < A.rows; ++i) merge(i, C.idx.data() + C.ptr[i], C.val.data() + C.ptr[i]);
    return C;
}

// Row-wise Gustavson product.  Rows are independent, so contiguous row blocks
// run on OpenMP threads with private accumulators and are concatenated in row
// order: every entry is accumulated exactly as in the sequential loop (k
// ascending), so the result is bit-identical for any thread count.
Csr matmul(const Csr& A, const Csr& B) {
    check(A.cols == B.rows, "csr matmul: shape mismatch");
    Csr C;
    C.rows = A.rows;
    C.cols = B.cols;
    C.ptr.assign(A.rows + 1, 0);
    const int nt = A.rows >= 4096 ? omp_get_max_threads() : 1;
    std::vector<std::vector<int>> bidx(nt);
    std::vector<std::vector<double>> bval(nt);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const int lo = static_cast<int>(static_cast<long long>(A.rows) * t / nt);
        const int hi = static_cast<int>(static_cast<long long>(A.rows) * (t + 1) / nt);
        std::vector<double> acc(B.cols, 0.0);
        std::vector<int> seen(B.cols, -1);
        std::vector<int> touched;
        std::vector<int>& oi = bidx[t];
        std::vector<double>& ov = bval[t];
        for (int i = lo; i < hi; ++i) {
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
                oi.push_back(c);
                ov.push_back(acc[c]);
            }
            C.ptr[i + 1] = static_cast<int>(touched.size());
        }
    }
    std::partial_sum(C.ptr.begin(), C.ptr.end(), C.ptr.begin());
    C.idx.reserve(C.ptr.back());
    C.val.reserve(C.ptr.back());
    for (int t = 0; t < nt; ++t) {
        C.idx.insert(C.idx.end(), bidx[t].begin(), bidx[t].end());
        C.val.insert(C.val.end(), bval[t].begin(), bval[t].end());
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
