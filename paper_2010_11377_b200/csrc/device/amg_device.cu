// Smoothed-aggregation AMG setup on the device (SURVEY.md §8 row f2,
// reference amg.cpp:172-227).  Produces the same hierarchy, bit for bit, as
// the reference's amg_setup and the host restatement (csrc/host/amg_setup.cpp)
// on the same input:
//
//   strength graph  |A| + |A|^T, row-relative non-strict threshold
//                   (amg.cpp:15-42)                         -> device
//   aggregation     three greedy passes (amg.cpp:44-74): the
//                   result depends on visiting order, so it
//                   runs sequentially on the host over the
//                   downloaded strong graph                  -> host
//   rho(D^-1 symA)  10 seeded power iterations with the
//                   reference's blocked dot (amg.cpp:80-98,
//                   kernels.cpp:25-49)                       -> device
//   P = (I - w D^-1 A) T, R = P^T, A_c = R (A P)
//                   (amg.cpp:207-221)                        -> device
//
// Bit-exactness of the sparse algebra:
//   * transpose: stable radix sort of the entries by column, so every column
//     lists its rows in increasing order (csr.cpp:128-145);
//   * add: one thread per row, the two-pointer merge of csr.cpp:147-186 with
//     the same alpha*a + beta*b expression;
//   * matmul (Gustavson with a dense accumulator, csr.cpp:188-216): every
//     product a_ik * b_kj is expanded in the reference's traversal order
//     (k along A's row, then along B's row k), stably sorted by (row, col),
//     and each (row, col) run is summed sequentially from 0.0 -- the
//     accumulator's exact association;
//   * all kernels are compiled with --fmad=false.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "amg_device.hpp"
#include "common.cuh"

namespace irkb {
namespace {

constexpr int kT = 256;

inline int nblk(long long n) { return static_cast<int>((n + kT - 1) / kT); }

int bits_for(long long v) {
    int b = 1;
    while ((1LL << b) <= v) ++b;
    return b;
}

// Stream-ordered device array from the setup's own memory pool (a release
// threshold of "never" keeps freed blocks for reuse; the default pool would
// hand them back to the driver at every synchronisation).
thread_local cudaMemPool_t g_pool = nullptr;

// One pool per device for the life of the process: mapping fresh physical
// memory costs far more than the setup's kernels, so blocks are kept for the
// next hierarchy (peak ~1.5 GB at C2).
cudaMemPool_t setup_pool(int device) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lock(mu);
    if (static_cast<int>(pools.size()) <= device) pools.resize(device + 1, nullptr);
    if (!pools[device]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        IRK_CUDA_CHECK(cudaMemPoolCreate(&pools[device], &props));
        uint64_t keep = ~0ULL;
        IRK_CUDA_CHECK(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep));
    }
    return pools[device];
}

template <class T>
class DA {
public:
    DA() = default;
    DA(long long n, cudaStream_t st) : n_(n), st_(st) {
        IRK_CUDA_CHECK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p_), sizeof(T) * std::max<long long>(n, 1),
                                               g_pool, st));
    }
    ~DA() { reset(); }
    DA(DA&& o) noexcept : p_(o.p_), n_(o.n_), st_(o.st_) { o.p_ = nullptr; o.n_ = 0; }
    DA& operator=(DA&& o) noexcept {
        if (this != &o) {
            reset();
            p_ = o.p_;
            n_ = o.n_;
            st_ = o.st_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    DA(const DA&) = delete;
    DA& operator=(const DA&) = delete;
    T* get() const { return p_; }
    long long size() const { return n_; }
    void reset() {
        if (p_) cudaFreeAsync(p_, st_);
        p_ = nullptr;
        n_ = 0;
    }

private:
    T* p_ = nullptr;
    long long n_ = 0;
    cudaStream_t st_ = nullptr;
};

struct DCsr {
    int rows = 0, cols = 0;
    long long nnz = 0;
    DA<int> ptr, idx;
    DA<double> val;
};

// CUB temporary storage, grown on demand.
struct Temp {
    cudaStream_t st;
    DA<unsigned char> buf;
    void* get(size_t bytes) {
        if (static_cast<long long>(bytes) > buf.size()) buf = DA<unsigned char>(static_cast<long long>(bytes), st);
        return buf.get();
    }
};

#define CUB_CALL(tmp, fn, ...)                                        \
    do {                                                              \
        size_t b__ = 0;                                               \
        IRK_CUDA_CHECK(fn(nullptr, b__, __VA_ARGS__));                \
        void* p__ = (tmp).get(b__);                                   \
        IRK_CUDA_CHECK(fn(p__, b__, __VA_ARGS__));                    \
    } while (0)

// ------------------------------------------------------------------ kernels
__global__ void k_row_of(int rows, const int* __restrict__ ptr, int* __restrict__ row_of) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) row_of[k] = i;
}

__global__ void k_iota(long long n, int* __restrict__ v) {
    const long long i = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (i < n) v[i] = static_cast<int>(i);
}

__global__ void k_gather_transpose(long long nnz, const int* __restrict__ perm, const int* __restrict__ row_of,
                                   const double* __restrict__ val, int* __restrict__ tidx,
                                   double* __restrict__ tval) {
    const long long p = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (p >= nnz) return;
    const int k = perm[p];
    tidx[p] = row_of[k];
    tval[p] = val[k];
}

// ptr[c] = first position whose key >= c (sorted int keys).
__global__ void k_lower_bound_i32(int nkeys, const int* __restrict__ keys, int nq, int* __restrict__ ptr) {
    const int c = blockIdx.x * kT + threadIdx.x;
    if (c > nq) return;
    int lo = 0, hi = nkeys;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (keys[m] < c) lo = m + 1; else hi = m;
    }
    ptr[c] = lo;
}

__global__ void k_lower_bound_u64_row(long long nkeys, const unsigned long long* __restrict__ keys, int rows,
                                      int* __restrict__ ptr) {
    const int r = blockIdx.x * kT + threadIdx.x;
    if (r > rows) return;
    const unsigned long long q = static_cast<unsigned long long>(r) << 32;
    long long lo = 0, hi = nkeys;
    while (lo < hi) {
        const long long m = (lo + hi) >> 1;
        if (keys[m] < q) lo = m + 1; else hi = m;
    }
    ptr[r] = static_cast<int>(lo);
}

// csr_add (csr.cpp:147-186): merged row lengths, then the merge itself.
__global__ void k_add_count(int rows, const int* __restrict__ ap, const int* __restrict__ ai,
                            const int* __restrict__ bp, const int* __restrict__ bi, int* __restrict__ cnt) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    int ka = ap[i], kb = bp[i];
    const int ea = ap[i + 1], eb = bp[i + 1];
    int c = 0;
    while (ka < ea || kb < eb) {
        if (kb >= eb || (ka < ea && ai[ka] < bi[kb])) ++ka;
        else if (ka >= ea || bi[kb] < ai[ka]) ++kb;
        else { ++ka; ++kb; }
        ++c;
    }
    cnt[i + 1] = c;
}

__global__ void k_add_fill(int rows, double alpha, const int* __restrict__ ap, const int* __restrict__ ai,
                           const double* __restrict__ av, double beta, const int* __restrict__ bp,
                           const int* __restrict__ bi, const double* __restrict__ bv,
                           const int* __restrict__ cp, int* __restrict__ ci, double* __restrict__ cv) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    int ka = ap[i], kb = bp[i];
    const int ea = ap[i + 1], eb = bp[i + 1];
    int o = cp[i];
    while (ka < ea || kb < eb) {
        int c;
        double v;
        if (kb >= eb || (ka < ea && ai[ka] < bi[kb])) {
            c = ai[ka];
            v = alpha * av[ka++];
        } else if (ka >= ea || bi[kb] < ai[ka]) {
            c = bi[kb];
            v = beta * bv[kb++];
        } else {
            c = ai[ka];
            v = alpha * av[ka++] + beta * bv[kb++];
        }
        ci[o] = c;
        cv[o] = v;
        ++o;
    }
}

// matmul: products per entry of A, expansion in traversal order, run sums.
__global__ void k_prod_count(long long nnz, const int* __restrict__ ai, const int* __restrict__ bp,
                             long long* __restrict__ cnt) {
    const long long k = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (k >= nnz) return;
    const int j = ai[k];
    cnt[k] = bp[j + 1] - bp[j];
}

__global__ void k_expand(long long nnz, const int* __restrict__ row_of, const int* __restrict__ ai,
                         const double* __restrict__ av, const int* __restrict__ bp, const int* __restrict__ bi,
                         const double* __restrict__ bv, const long long* __restrict__ off,
                         unsigned long long* __restrict__ keys, double* __restrict__ vals) {
    const long long k = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (k >= nnz) return;
    const unsigned long long r = static_cast<unsigned long long>(row_of[k]) << 32;
    const int j = ai[k];
    const double a = av[k];
    long long o = off[k];
    for (int q = bp[j]; q < bp[j + 1]; ++q, ++o) {
        keys[o] = r | static_cast<unsigned int>(bi[q]);
        vals[o] = a * bv[q];
    }
}

__global__ void k_run_sum(long long nruns, const long long* __restrict__ start, const int* __restrict__ len,
                          const unsigned long long* __restrict__ ukeys, const double* __restrict__ vals,
                          int* __restrict__ ci, double* __restrict__ cv) {
    const long long s = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (s >= nruns) return;
    double acc = 0.0;  // acc[c] = 0.0; acc[c] += a * b  (csr.cpp:203-208)
    const long long b = start[s];
    for (int q = 0; q < len[s]; ++q) acc += vals[b + q];
    ci[s] = static_cast<int>(ukeys[s] & 0xffffffffu);
    cv[s] = acc;
}

__global__ void k_abs(long long n, const double* __restrict__ v, double* __restrict__ o) {
    const long long k = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (k < n) o[k] = fabs(v[k]);
}

// Strong off-diagonal connections of C (amg.cpp:25-42): C_ij >= theta * max_{j'!=i} C_ij'.
__global__ void k_strong_count(int rows, const int* __restrict__ cp, const int* __restrict__ ci,
                               const double* __restrict__ cv, double theta, int* __restrict__ cnt) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    double mx = 0.0;
    for (int k = cp[i]; k < cp[i + 1]; ++k)
        if (ci[k] != i) mx = fmax(mx, cv[k]);
    const double th = theta * mx;
    int c = 0;
    for (int k = cp[i]; k < cp[i + 1]; ++k) c += (ci[k] != i && cv[k] >= th);
    cnt[i + 1] = c;
}

__global__ void k_strong_fill(int rows, const int* __restrict__ cp, const int* __restrict__ ci,
                              const double* __restrict__ cv, double theta, const int* __restrict__ sp,
                              int* __restrict__ si, double* __restrict__ sv) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    double mx = 0.0;
    for (int k = cp[i]; k < cp[i + 1]; ++k)
        if (ci[k] != i) mx = fmax(mx, cv[k]);
    const double th = theta * mx;
    int o = sp[i];
    for (int k = cp[i]; k < cp[i + 1]; ++k)
        if (ci[k] != i && cv[k] >= th) {
            si[o] = ci[k];
            sv[o] = cv[k];
            ++o;
        }
}

// inverse_diagonal (amg.cpp:100-113); the first zero diagonal is reported.
__global__ void k_inv_diag(int rows, const int* __restrict__ p, const int* __restrict__ ix,
                           const double* __restrict__ v, double* __restrict__ d, int* __restrict__ bad) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    double a = 0.0;
    for (int k = p[i]; k < p[i + 1]; ++k)
        if (ix[k] == i) a = v[k];
    if (a == 0.0) atomicMin(bad, i);
    d[i] = 1.0 / a;
}

// y = (S x) .* dinv: sequential row sums (csr.cpp:108-113), then y[i] *= dinv[i].
__global__ void k_spmv_scale(int rows, const int* __restrict__ p, const int* __restrict__ ix,
                             const double* __restrict__ v, const double* __restrict__ x,
                             const double* __restrict__ dinv, double* __restrict__ y) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    double s = 0.0;
    for (int k = p[i]; k < p[i + 1]; ++k) s += v[k] * x[ix[k]];
    y[i] = s * dinv[i];
}

// The reference's dot (kernels.cpp:25-49): sequential sums over blocks of
// 4096, then the block sums in order.
constexpr long long kDotBlock = 4096;
__global__ void k_block_sq(long long n, const double* __restrict__ y, double* __restrict__ part) {
    const long long b = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    const long long lo = b * kDotBlock;
    if (lo >= n) return;
    const long long hi = min(n, lo + kDotBlock);
    double s = 0.0;
    for (long long i = lo; i < hi; ++i) s += y[i] * y[i];
    part[b] = s;
}

__global__ void k_final_norm(long long nb, const double* __restrict__ part, double* __restrict__ out) {
    double s = 0.0;
    for (long long b = 0; b < nb; ++b) s += part[b];
    out[0] = sqrt(s);
}

__global__ void k_scal(long long n, double a, double* __restrict__ y) {
    const long long i = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (i < n) y[i] *= a;
}

// AP.vals[k] *= w * inv_diag[i] (amg.cpp:211-213).
__global__ void k_scale_rows(int rows, const int* __restrict__ p, double w, const double* __restrict__ dinv,
                             double* __restrict__ v) {
    const int i = blockIdx.x * kT + threadIdx.x;
    if (i >= rows) return;
    const double sc = w * dinv[i];
    for (int k = p[i]; k < p[i + 1]; ++k) v[k] *= sc;
}

__global__ void k_fill_d(long long n, double a, double* __restrict__ v) {
    const long long i = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
    if (i < n) v[i] = a;
}

// ------------------------------------------------------------------ algebra
// IRK_SETUP_TIMING=1: per-phase wall times on stderr (stream-synchronised)
struct PhaseClock {
    bool on = std::getenv("IRK_SETUP_TIMING") != nullptr;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(const char* what, int level) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "setup L%d %-12s %8.2f ms\n", level, what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};
thread_local PhaseClock* g_clk = nullptr;
void lap(const char* what, int level = -1) {
    if (g_clk) g_clk->lap(what, level);
}

struct Setup {
    cudaStream_t st;
    Temp tmp;

    explicit Setup(cudaStream_t s) : st(s), tmp{s, {}} {}

    // counts in ptr[1..rows] -> row pointers (ptr[0] = 0)
    void scan_ptr(DA<int>& ptr, int rows) {
        IRK_CUDA_CHECK(cudaMemsetAsync(ptr.get(), 0, sizeof(int), st));
        CUB_CALL(tmp, cub::DeviceScan::InclusiveSum, ptr.get() + 1, ptr.get() + 1, rows, st);
    }

    int read_int(const int* p) {
        int v = 0;
        IRK_CUDA_CHECK(cudaMemcpyAsync(&v, p, sizeof(int), cudaMemcpyDeviceToHost, st));
        IRK_CUDA_CHECK(cudaStreamSynchronize(st));
        return v;
    }

    DA<int> row_of(const DCsr& A) {
        DA<int> r(A.nnz, st);
        if (A.rows) k_row_of<<<nblk(A.rows), kT, 0, st>>>(A.rows, A.ptr.get(), r.get());
        return r;
    }

    DCsr upload(const Csr& A) {
        DCsr d;
        d.rows = A.rows;
        d.cols = A.cols;
        d.nnz = A.nnz();
        d.ptr = DA<int>(A.rows + 1, st);
        d.idx = DA<int>(d.nnz, st);
        d.val = DA<double>(d.nnz, st);
        IRK_CUDA_CHECK(cudaMemcpyAsync(d.ptr.get(), A.ptr.data(), sizeof(int) * (A.rows + 1), cudaMemcpyHostToDevice, st));
        if (d.nnz) {
            IRK_CUDA_CHECK(cudaMemcpyAsync(d.idx.get(), A.idx.data(), sizeof(int) * d.nnz, cudaMemcpyHostToDevice, st));
            IRK_CUDA_CHECK(cudaMemcpyAsync(d.val.get(), A.val.data(), sizeof(double) * d.nnz, cudaMemcpyHostToDevice, st));
        }
        IRK_CUDA_CHECK(cudaStreamSynchronize(st));  // host vectors may be temporaries
        return d;
    }

    Csr download(const DCsr& d) {
        Csr A;
        A.rows = d.rows;
        A.cols = d.cols;
        A.ptr.resize(d.rows + 1);
        A.idx.resize(d.nnz);
        A.val.resize(d.nnz);
        IRK_CUDA_CHECK(cudaMemcpyAsync(A.ptr.data(), d.ptr.get(), sizeof(int) * (d.rows + 1), cudaMemcpyDeviceToHost, st));
        if (d.nnz) {
            IRK_CUDA_CHECK(cudaMemcpyAsync(A.idx.data(), d.idx.get(), sizeof(int) * d.nnz, cudaMemcpyDeviceToHost, st));
            IRK_CUDA_CHECK(cudaMemcpyAsync(A.val.data(), d.val.get(), sizeof(double) * d.nnz, cudaMemcpyDeviceToHost, st));
        }
        IRK_CUDA_CHECK(cudaStreamSynchronize(st));
        return A;
    }

    std::vector<double> download(const DA<double>& v, long long n) {
        std::vector<double> h(n);
        if (n) IRK_CUDA_CHECK(cudaMemcpyAsync(h.data(), v.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        IRK_CUDA_CHECK(cudaStreamSynchronize(st));
        return h;
    }

    // csr_transpose (csr.cpp:128-145): stable sort of the entries by column.
    DCsr transpose(const DCsr& A) {
        DCsr T;
        T.rows = A.cols;
        T.cols = A.rows;
        T.nnz = A.nnz;
        T.ptr = DA<int>(T.rows + 1, st);
        T.idx = DA<int>(A.nnz, st);
        T.val = DA<double>(A.nnz, st);
        DA<int> rof = row_of(A), perm_in(A.nnz, st), perm(A.nnz, st), keys(A.nnz, st);
        if (A.nnz) {
            k_iota<<<nblk(A.nnz), kT, 0, st>>>(A.nnz, perm_in.get());
            CUB_CALL(tmp, cub::DeviceRadixSort::SortPairs, A.idx.get(), keys.get(), perm_in.get(), perm.get(),
                     A.nnz, 0, bits_for(A.cols), st);
            k_gather_transpose<<<nblk(A.nnz), kT, 0, st>>>(A.nnz, perm.get(), rof.get(), A.val.get(), T.idx.get(),
                                                           T.val.get());
        }
        k_lower_bound_i32<<<nblk(T.rows + 1), kT, 0, st>>>(static_cast<int>(A.nnz), keys.get(), T.rows, T.ptr.get());
        return T;
    }

    // csr_add (csr.cpp:147-186)
    DCsr add(double alpha, const DCsr& A, double beta, const DCsr& B) {
        check(A.rows == B.rows && A.cols == B.cols, "csr_add: shape mismatch");
        DCsr C;
        C.rows = A.rows;
        C.cols = A.cols;
        C.ptr = DA<int>(A.rows + 1, st);
        if (A.rows)
            k_add_count<<<nblk(A.rows), kT, 0, st>>>(A.rows, A.ptr.get(), A.idx.get(), B.ptr.get(), B.idx.get(),
                                                     C.ptr.get());
        scan_ptr(C.ptr, A.rows);
        C.nnz = read_int(C.ptr.get() + A.rows);
        C.idx = DA<int>(C.nnz, st);
        C.val = DA<double>(C.nnz, st);
        if (A.rows)
            k_add_fill<<<nblk(A.rows), kT, 0, st>>>(A.rows, alpha, A.ptr.get(), A.idx.get(), A.val.get(), beta,
                                                    B.ptr.get(), B.idx.get(), B.val.get(), C.ptr.get(),
                                                    C.idx.get(), C.val.get());
        return C;
    }

    // csr_matmul (csr.cpp:188-216) by expand / stable sort / ordered run sums.
    DCsr matmul(const DCsr& A, const DCsr& B) {
        check(A.cols == B.rows, "csr_matmul: shape mismatch");
        DCsr C;
        C.rows = A.rows;
        C.cols = B.cols;
        C.ptr = DA<int>(A.rows + 1, st);
        DA<long long> off(A.nnz + 1, st);
        IRK_CUDA_CHECK(cudaMemsetAsync(off.get(), 0, sizeof(long long), st));
        if (A.nnz) {
            k_prod_count<<<nblk(A.nnz), kT, 0, st>>>(A.nnz, A.idx.get(), B.ptr.get(), off.get() + 1);
            CUB_CALL(tmp, cub::DeviceScan::InclusiveSum, off.get() + 1, off.get() + 1, A.nnz, st);
        }
        long long np = 0;
        IRK_CUDA_CHECK(cudaMemcpyAsync(&np, off.get() + A.nnz, sizeof(long long), cudaMemcpyDeviceToHost, st));
        IRK_CUDA_CHECK(cudaStreamSynchronize(st));
        if (np == 0) {
            IRK_CUDA_CHECK(cudaMemsetAsync(C.ptr.get(), 0, sizeof(int) * (A.rows + 1), st));
            C.idx = DA<int>(0, st);
            C.val = DA<double>(0, st);
            return C;
        }
        DA<unsigned long long> k0(np, st), k1(np, st);
        DA<double> v0(np, st), v1(np, st);
        {
            DA<int> rof = row_of(A);
            k_expand<<<nblk(A.nnz), kT, 0, st>>>(A.nnz, rof.get(), A.idx.get(), A.val.get(), B.ptr.get(),
                                                 B.idx.get(), B.val.get(), off.get(), k0.get(), v0.get());
        }
        off.reset();
        // LSD radix sort is stable: equal (row, col) keys keep expansion order
        CUB_CALL(tmp, cub::DeviceRadixSort::SortPairs, k0.get(), k1.get(), v0.get(), v1.get(), np, 0,
                 32 + bits_for(A.rows), st);
        k0.reset();
        v0.reset();
        DA<unsigned long long> uk(np, st);
        DA<int> len(np, st), nruns_d(1, st);
        CUB_CALL(tmp, cub::DeviceRunLengthEncode::Encode, k1.get(), uk.get(), len.get(), nruns_d.get(), np, st);
        const int nruns = read_int(nruns_d.get());
        DA<long long> start(nruns, st);
        CUB_CALL(tmp, cub::DeviceScan::ExclusiveSum, len.get(), start.get(), nruns, st);
        C.nnz = nruns;
        C.idx = DA<int>(nruns, st);
        C.val = DA<double>(nruns, st);
        k_run_sum<<<nblk(nruns), kT, 0, st>>>(nruns, start.get(), len.get(), uk.get(), v1.get(), C.idx.get(),
                                              C.val.get());
        k_lower_bound_u64_row<<<nblk(A.rows + 1), kT, 0, st>>>(nruns, uk.get(), A.rows, C.ptr.get());
        return C;
    }

    DA<double> inverse_diagonal(const DCsr& A) {
        DA<double> d(A.rows, st);
        DA<int> bad(1, st);
        const int big = 0x7fffffff;
        IRK_CUDA_CHECK(cudaMemcpyAsync(bad.get(), &big, sizeof(int), cudaMemcpyHostToDevice, st));
        k_inv_diag<<<nblk(A.rows), kT, 0, st>>>(A.rows, A.ptr.get(), A.idx.get(), A.val.get(), d.get(), bad.get());
        const int b = read_int(bad.get());
        if (b != big) throw SingularError("amg_setup: zero diagonal at row " + std::to_string(b), b);
        return d;
    }

    // |A| + |A|^T, then its strong off-diagonal entries, downloaded as CSR.
    Csr strong_graph(const DCsr& A, double theta) {
        DCsr B;
        B.rows = A.rows;
        B.cols = A.cols;
        B.nnz = A.nnz;
        B.ptr = DA<int>(A.rows + 1, st);
        B.idx = DA<int>(A.nnz, st);
        B.val = DA<double>(A.nnz, st);
        IRK_CUDA_CHECK(cudaMemcpyAsync(B.ptr.get(), A.ptr.get(), sizeof(int) * (A.rows + 1), cudaMemcpyDeviceToDevice, st));
        if (A.nnz) {
            IRK_CUDA_CHECK(cudaMemcpyAsync(B.idx.get(), A.idx.get(), sizeof(int) * A.nnz, cudaMemcpyDeviceToDevice, st));
            k_abs<<<nblk(A.nnz), kT, 0, st>>>(A.nnz, A.val.get(), B.val.get());
        }
        DCsr C;
        {
            lap("  str:abs");
            DCsr BT = transpose(B);
            lap("  str:T");
            C = add(1.0, B, 1.0, BT);
            lap("  str:add");
        }
        DCsr S;
        S.rows = C.rows;
        S.cols = C.cols;
        S.ptr = DA<int>(C.rows + 1, st);
        k_strong_count<<<nblk(C.rows), kT, 0, st>>>(C.rows, C.ptr.get(), C.idx.get(), C.val.get(), theta,
                                                    S.ptr.get());
        scan_ptr(S.ptr, C.rows);
        S.nnz = read_int(S.ptr.get() + C.rows);
        S.idx = DA<int>(S.nnz, st);
        S.val = DA<double>(S.nnz, st);
        k_strong_fill<<<nblk(C.rows), kT, 0, st>>>(C.rows, C.ptr.get(), C.idx.get(), C.val.get(), theta,
                                                   S.ptr.get(), S.idx.get(), S.val.get());
        return download(S);
    }

    // spectral_radius_estimate (amg.cpp:80-98)
    double spectral_radius(const DCsr& A, const DA<double>& dinv) {
        DCsr S;
        {
            DCsr AT = transpose(A);
            lap("  rho:T");
            S = add(0.5, A, 0.5, AT);
        }
        lap("  rho:add");
        const int n = A.rows;
        std::mt19937_64 gen(0x1d872b41u);
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        std::vector<double> hx(n);
        for (double& v : hx) v = dist(gen);
        DA<double> x(n, st), y(n, st);
        IRK_CUDA_CHECK(cudaMemcpyAsync(x.get(), hx.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
        lap("  rho:x0");
        const long long nb = (n + kDotBlock - 1) / kDotBlock;
        DA<double> part(nb, st), rho_d(1, st);
        double rho = 1.0;
        for (int it = 0; it < 10; ++it) {
            k_spmv_scale<<<nblk(n), kT, 0, st>>>(n, S.ptr.get(), S.idx.get(), S.val.get(), x.get(), dinv.get(),
                                                 y.get());
            k_block_sq<<<nblk(nb), kT, 0, st>>>(n, y.get(), part.get());
            k_final_norm<<<1, 1, 0, st>>>(nb, part.get(), rho_d.get());
            IRK_CUDA_CHECK(cudaMemcpyAsync(&rho, rho_d.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
            IRK_CUDA_CHECK(cudaStreamSynchronize(st));
            if (rho == 0.0) break;
            k_scal<<<nblk(n), kT, 0, st>>>(n, 1.0 / rho, y.get());
            std::swap(x, y);
        }
        return std::max(rho, 1e-12);
    }
};

// Greedy aggregation (amg.cpp:44-74) over the strong graph: S lists, per
// row and in column order, exactly the entries for which the reference's
// strong(i, k) holds, with their weights.
std::vector<int> aggregate_strong(const Csr& S, int& n_agg) {
    const int n = S.rows;
    std::vector<int> agg(n, -1);
    n_agg = 0;
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        bool free_nbhd = true;
        for (int k = S.ptr[i]; k < S.ptr[i + 1] && free_nbhd; ++k)
            if (agg[S.idx[k]] >= 0) free_nbhd = false;
        if (!free_nbhd) continue;
        agg[i] = n_agg;
        for (int k = S.ptr[i]; k < S.ptr[i + 1]; ++k) agg[S.idx[k]] = n_agg;
        ++n_agg;
    }
    for (int i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        int best = -1;
        double wbest = 0.0;
        for (int k = S.ptr[i]; k < S.ptr[i + 1]; ++k) {
            const int j = S.idx[k];
            if (agg[j] < 0) continue;
            if (S.val[k] > wbest) {
                wbest = S.val[k];
                best = agg[j];
            }
        }
        if (best >= 0) agg[i] = best;
    }
    for (int i = 0; i < n; ++i)
        if (agg[i] < 0) agg[i] = n_agg++;
    return agg;
}

}  // namespace

Hierarchy amg_setup_device(const Csr& A, const AmgParams& p, int device) {
    check(A.rows == A.cols, "amg_setup: matrix must be square");
    check(A.rows > 0, "amg_setup: empty matrix");
    check(p.theta > 0.0 && p.theta < 1.0, "amg_setup: theta must be in (0,1)");
    check(p.pre_sweeps >= 1 && p.post_sweeps >= 1, "amg_setup: sweeps must be >= 1");
    check(p.smoother == 0 || p.smoother == 1, "amg_setup: unknown smoother");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CudaError("no CUDA device: amg_setup_device has no CPU fallback");
    DeviceScope on(device);
    cudaStream_t st = nullptr;
    IRK_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
            g_pool = nullptr;
            g_clk = nullptr;
        }
    } guard{st};
    g_pool = setup_pool(device);

    Hierarchy h;
    h.params = p;
    PhaseClock clk;
    clk.st = st;
    g_clk = clk.on ? &clk : nullptr;
    {
        Setup S(st);
        DCsr Af = S.upload(A);
        DA<double> dinv = S.inverse_diagonal(Af);
        h.levels.push_back({A, S.download(dinv, A.rows), {}, {}});
        clk.lap("upload", 0);
        while (Af.rows > p.max_coarse && h.n_levels() < p.max_levels) {
            const int n = Af.rows;
            int n_agg = 0;
            const int lv = h.n_levels() - 1;
            const Csr sg = S.strong_graph(Af, p.theta);
            clk.lap("strong", lv);
            const std::vector<int> agg = aggregate_strong(sg, n_agg);
            clk.lap("aggregate", lv);
            if (n_agg == 0) throw NumericalError("amg_setup: aggregation stalled");
            if (n_agg > (9 * n) / 10) break;

            // tentative piecewise-constant prolongator (amg.cpp:195-203)
            DCsr P;
            P.rows = n;
            P.cols = n_agg;
            P.nnz = n;
            P.ptr = DA<int>(n + 1, st);
            P.idx = DA<int>(n, st);
            P.val = DA<double>(n, st);
            k_iota<<<nblk(n + 1), kT, 0, st>>>(n + 1, P.ptr.get());
            IRK_CUDA_CHECK(cudaMemcpyAsync(P.idx.get(), agg.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
            k_fill_d<<<nblk(n), kT, 0, st>>>(n, 1.0, P.val.get());

            const double w = p.prolongation_weight / S.spectral_radius(Af, dinv);
            clk.lap("rho", lv);
            for (int step = 0; step < p.prolongation_steps; ++step) {
                DCsr AP = S.matmul(Af, P);
                k_scale_rows<<<nblk(n), kT, 0, st>>>(n, AP.ptr.get(), w, dinv.get(), AP.val.get());
                P = S.add(1.0, P, -1.0, AP);
            }
            clk.lap("smooth P", lv);
            DCsr R = S.transpose(P);
            DCsr Ac;
            {
                DCsr AP = S.matmul(Af, P);
                Ac = S.matmul(R, AP);
            }
            clk.lap("RAP", lv);
            AmgLevel& fine = h.levels.back();
            fine.P = S.download(P);
            fine.R = S.download(R);
            DA<double> dc = S.inverse_diagonal(Ac);
            h.levels.push_back({S.download(Ac), S.download(dc, Ac.rows), {}, {}, {}, {}});
            clk.lap("download", lv);
            Af = std::move(Ac);
            dinv = std::move(dc);
        }
    }
    h.coarse_inverse = dense_inverse_host(h.levels.back().A);
    attach_tail(h, tail_max_rows(h.params));
    attach_composed(h);
    clk.lap("coarse inv", h.n_levels() - 1);
    return h;
}

}  // namespace irkb
