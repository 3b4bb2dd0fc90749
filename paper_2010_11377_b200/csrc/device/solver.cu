// Device solver orchestration.  One CUDA stream per solver; one CUDA graph
// per IRK step holding the whole restarted GMRES as nested conditional WHILE
// nodes (outer: restart cycles, inner: Arnoldi iterations), so a step is one
// graph launch plus one small device->host read of the report.  The kernels
// read the iteration index from the device control block, which keeps the
// captured iteration body iteration-invariant.
#include <algorithm>
#include <atomic>
#include <unordered_map>
#include <unordered_set>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "amg_device.hpp"
#include "solver.hpp"

namespace irkb {

namespace dev {
void set_smem_limits();
}

using dev::VecRef;

DevBuf::DevBuf(size_t bytes) : n_(bytes) {
    if (bytes == 0) return;
    IRK_CUDA_CHECK(cudaMalloc(&p_, bytes));
}

DevBuf::~DevBuf() {
    if (p_) cudaFree(p_);
}

DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (p_) cudaFree(p_);
        p_ = o.p_;
        n_ = o.n_;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}

namespace {

VecRef block(VecRef v, long long off) {
    v.offset += off;
    return v;
}

VecRef slot(double* base, const int* idx, long long stride, int add) {
    return VecRef{base, idx, stride, add, 0};
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

void* DeviceSolver::raw_alloc(size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    bufs_.emplace_back(bytes);
    return bufs_.back().as<void>();
}

double* DeviceSolver::alloc(size_t count) {
    return static_cast<double*>(raw_alloc(sizeof(double) * count));
}

namespace {

// Exact value dictionary: distinct fp64 bit patterns (so +0.0 / -0.0 stay
// distinct and decoding reproduces every stored bit).
struct Dict {
    int vf = dev::kF64;
    std::vector<double> tab;
    std::vector<unsigned char> c8;
    std::vector<unsigned short> c16;
};

Dict encode(const std::vector<double>& v) {
    Dict d;
    const long long n = static_cast<long long>(v.size());
    std::vector<uint64_t> bits(v.size());
    std::memcpy(bits.data(), v.data(), v.size() * sizeof(double));
    // distinct bit patterns (thread-local sets, giving up past 65,536)
    std::vector<uint64_t> u;
    std::atomic<bool> too_many{false};
#pragma omp parallel
    {
        std::unordered_set<uint64_t> loc;
        uint64_t last = 0;
        bool have = false;
#pragma omp for schedule(static)
        for (long long i = 0; i < n; ++i) {
            if ((have && bits[i] == last) || too_many.load(std::memory_order_relaxed)) continue;
            loc.insert(bits[i]);
            last = bits[i];
            have = true;
            if (loc.size() > 65536) too_many.store(true, std::memory_order_relaxed);
        }
#pragma omp critical
        u.insert(u.end(), loc.begin(), loc.end());
    }
    if (too_many.load()) return d;
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    if (u.size() > 65536) return d;
    // Codes in order of first appearance (IRK_DICT_ORDER=0: sorted bit patterns):
    // the entries a warp decodes together -- consecutive entries of a few rows
    // with the same stencil -- then sit in adjacent dictionary slots, i.e. in
    // one or two cache lines instead of scattered over the table.
    std::vector<int> rank(u.size());
    for (size_t q = 0; q < u.size(); ++q) rank[q] = static_cast<int>(q);
    auto slot = [&](uint64_t b) {
        return static_cast<size_t>(std::lower_bound(u.begin(), u.end(), b) - u.begin());
    };
    if (dev::option("IRK_DICT_ORDER", 1) != 0) {
        std::vector<int> seen(u.size(), -1);
        int next = 0;
        uint64_t last = 0;
        bool have = false;
        for (long long i = 0; i < n && next < static_cast<int>(u.size()); ++i) {
            if (have && bits[i] == last) continue;
            last = bits[i];
            have = true;
            const size_t q = slot(bits[i]);
            if (seen[q] < 0) seen[q] = next++;
        }
        rank = seen;
    }
    d.tab.resize(u.size());
    for (size_t q = 0; q < u.size(); ++q) std::memcpy(&d.tab[rank[q]], &u[q], sizeof(double));
    auto code = [&](uint64_t b) { return static_cast<size_t>(rank[slot(b)]); };
    if (u.size() <= 256) {
        d.vf = dev::kU8;
        d.c8.resize(v.size());
#pragma omp parallel for schedule(static)
        for (long long i = 0; i < n; ++i) d.c8[i] = static_cast<unsigned char>(code(bits[i]));
    } else {
        d.vf = dev::kU16;
        d.c16.resize(v.size());
#pragma omp parallel for schedule(static)
        for (long long i = 0; i < n; ++i) d.c16[i] = static_cast<unsigned short>(code(bits[i]));
    }
    return d;
}

}  // namespace

template <class T>
const T* DeviceSolver::upload_array(const std::vector<T>& h) {
    T* p = static_cast<T*>(raw_alloc(sizeof(T) * h.size()));
    if (!h.empty()) IRK_CUDA_CHECK(cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return p;
}

// Stores the entry values (fp64 or dictionary codes) of an operator.
void DeviceSolver::upload_values(dev::Mat& m, const std::vector<double>& vals, double omega,
                                 std::vector<unsigned>* codes_out) {
    // Small operators keep fp64 values: their kernels are latency-bound and a
    // dictionary lookup is one more dependent memory trip.
    const long long min_rows = dev::option("IRK_CODES_MIN_ROWS", 100000);
    const bool small = std::max(m.rows, m.cols) < min_rows;
    Dict d = compress_values_ && !small ? encode(vals) : Dict{};
    // u16 dictionaries (up to 512 KB) are L2 gathers: only worth it where the
    // operator is big enough for its value bytes to dominate
    if (d.vf == dev::kU16 && std::max(m.rows, m.cols) < dev::option("IRK_U16_MIN_ROWS", 0)) d = Dict{};
    m.vf = d.vf;
    if (d.vf == dev::kF64) {
        m.val = upload_array(vals);
        m.bytes += vals.size() * sizeof(double);
        return;
    }
    m.tab = upload_array(d.tab);
    m.ntab = static_cast<int>(d.tab.size());
    // u8 dictionaries are read in place through L1 (a per-CTA shared-memory
    // copy costs a dependent prologue and a barrier; IRK_U8_TAB_SMEM=1 keeps it)
    static const bool tab_smem = std::getenv("IRK_U8_TAB_SMEM") != nullptr;
    m.tab_smem = tab_smem ? 1 : 0;
    int code_bits = 1;
    while ((size_t(1) << code_bits) < d.tab.size()) ++code_bits;
    if (codes_out && dev::option("IRK_PACK8", 1) != 0 && code_bits <= 16 &&
        static_cast<long long>(m.cols) <= (1LL << (32 - code_bits))) {
        // code and column share one index word (kP8); the caller packs them
        m.pk_shift = 32 - code_bits;
        if (d.vf == dev::kU8)
            codes_out->assign(d.c8.begin(), d.c8.end());
        else
            codes_out->assign(d.c16.begin(), d.c16.end());
    } else if (d.vf == dev::kU8) {
        m.val = upload_array(d.c8);
        m.bytes += d.c8.size();
    } else {
        m.val = upload_array(d.c16);
        m.bytes += 2 * d.c16.size();
    }
    if (omega > 0.0 && m.fmt == dev::kDia && d.vf == dev::kU8) {
        // omega * (1 / a_ii) per diagonal code: exactly the host's wd
        // (jacobi_weight * inv_diag[i], amg.cpp:100-113, 123).
        std::vector<double> wd(d.tab.size());
        for (size_t c = 0; c < d.tab.size(); ++c) wd[c] = omega * (1.0 / d.tab[c]);
        m.wdtab = upload_array(wd);
    }
}

void DeviceSolver::pack_codes(dev::Mat& m, std::vector<int>& idx, const std::vector<unsigned>& codes) {
    for (size_t e = 0; e < idx.size(); ++e) idx[e] = static_cast<int>(static_cast<unsigned>(idx[e]) | (codes[e] << m.pk_shift));
    m.vf = dev::kP8;
    m.val = nullptr;
}

namespace {

// DIA layout of a square operator: sorted offsets, aligned stride and the
// diagonal-major values (padding = 0.0); empty when the pattern has more
// than kMaxDiags diagonals or more than 15% padding.
struct DiaLayout {
    std::vector<int> offs;
    long long ds = 0;
    std::vector<double> v;
};

DiaLayout dia_layout(const Csr& A) {
    DiaLayout L;
    if (A.rows != A.cols || A.rows == 0) return L;
    std::vector<int>& offs = L.offs;
    for (int i = 0; i < A.rows; ++i)
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int o = A.idx[k] - i;
            if (std::find(offs.begin(), offs.end(), o) == offs.end()) {
                offs.push_back(o);
                if (static_cast<int>(offs.size()) > dev::kMaxDiags) {
                    offs.clear();
                    return L;
                }
            }
        }
    if (static_cast<double>(offs.size()) * A.rows > 1.15 * A.nnz() + 64) {
        offs.clear();
        return L;
    }
    std::sort(offs.begin(), offs.end());
    L.ds = (static_cast<long long>(A.rows) + 3) / 4 * 4;  // aligned stride
    L.v.assign(offs.size() * L.ds, 0.0);
    for (int i = 0; i < A.rows; ++i)
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int d = static_cast<int>(std::lower_bound(offs.begin(), offs.end(), A.idx[k] - i) - offs.begin());
            L.v[static_cast<size_t>(d) * L.ds + i] = A.val[k];
        }
    return L;
}

// Row classes: rows whose stencil values (over all `vals` operators) are the
// same fp64 bit patterns share a class; at most 256 classes (else false).
bool row_classes(const std::vector<const std::vector<double>*>& vals, int nd, int rows, long long ds,
                 std::vector<unsigned char>& cls, std::vector<std::vector<double>>& tabs) {
    const int nm = static_cast<int>(vals.size());
    const int w = nm * nd;
    std::vector<uint64_t> reps;  // class tuples, w words each
    std::unordered_map<uint64_t, std::vector<int>> by_hash;
    std::vector<uint64_t> t(w);
    cls.resize(rows);
    int prev = -1;
    for (int i = 0; i < rows; ++i) {
        uint64_t h = 1469598103934665603ULL;
        for (int m = 0; m < nm; ++m)
            for (int d = 0; d < nd; ++d) {
                uint64_t b;
                std::memcpy(&b, &(*vals[m])[static_cast<size_t>(d) * ds + i], sizeof(b));
                t[m * nd + d] = b;
                h = (h ^ b) * 1099511628211ULL;
            }
        auto same = [&](int c) { return std::equal(t.begin(), t.end(), reps.begin() + static_cast<size_t>(c) * w); };
        int c = -1;
        if (prev >= 0 && same(prev)) {
            c = prev;
        } else {
            std::vector<int>& cand = by_hash[h];
            for (int q : cand)
                if (same(q)) c = q;
            if (c < 0) {
                c = static_cast<int>(reps.size() / w);
                if (c >= 256) return false;
                reps.insert(reps.end(), t.begin(), t.end());
                cand.push_back(c);
            }
        }
        cls[i] = static_cast<unsigned char>(c);
        prev = c;
    }
    const int nc = static_cast<int>(reps.size() / w);
    tabs.assign(nm, std::vector<double>(static_cast<size_t>(nc) * nd));
    for (int c = 0; c < nc; ++c)
        for (int m = 0; m < nm; ++m)
            std::memcpy(&tabs[m][static_cast<size_t>(c) * nd], &reps[static_cast<size_t>(c) * w + m * nd],
                        sizeof(double) * nd);
    return true;
}

bool row_classes_enabled() {
    static const bool on = !(std::getenv("IRK_ROW_CLASSES") && std::string(std::getenv("IRK_ROW_CLASSES")) == "0");
    return on;
}

}  // namespace

// Re-stores DIA operators (7 diagonals, shared layout) as row classes: one
// class array (shared by all `mats`) and one value table per operator;
// `omega` > 0 adds the omega / diagonal table per class (hierarchy operators).
bool DeviceSolver::to_row_classes(std::vector<dev::Mat*> mats, const std::vector<const std::vector<double>*>& vals,
                                  double omega) {
    dev::Mat& m0 = *mats[0];
    if (!row_classes_enabled() || m0.fmt != dev::kDia || m0.nd != 7) return false;
    std::vector<unsigned char> cls;
    std::vector<std::vector<double>> tabs;
    if (!row_classes(vals, m0.nd, m0.rows, m0.dstride, cls, tabs)) return false;
    const unsigned char* dcls = upload_array(cls);
    // the most frequent class rides in the kernel parameters (dev::Mat::dom)
    int dom = 0;
    {
        std::vector<long long> cnt(256, 0);
        for (unsigned char c : cls) ++cnt[c];
        for (int c = 1; c < 256; ++c)
            if (cnt[c] > cnt[dom]) dom = c;
    }
    // a null entry in `mats`: its table is the neighbour omega / a_cc table
    // of mats[0] (same class array)
    for (size_t q = 0; q < mats.size(); ++q)
        if (!mats[q]) {
            mats[0]->nbwd = upload_array(tabs[q]);
            for (int d = 0; d < 7; ++d) mats[0]->dom_nbwd[d] = tabs[q][static_cast<size_t>(dom) * 7 + d];
        }
    for (size_t q = 0; q < mats.size(); ++q) {
        if (!mats[q]) continue;
        dev::Mat& m = *mats[q];
        m.vf = dev::kCls;
        m.val = dcls;
        m.tab = upload_array(tabs[q]);
        m.ntab = static_cast<int>(tabs[q].size() / m.nd);
        m.tab_smem = 0;
        m.bytes = (q == 0 ? cls.size() : 0) + sizeof(double) * tabs[q].size();
        m.wdtab = nullptr;
        m.dom = dom;
        for (int d = 0; d < 7; ++d) m.dom_tab[d] = tabs[q][static_cast<size_t>(dom) * 7 + d];
        if (omega > 0.0 && m.diag0 >= 0) {
            std::vector<double> wd(m.ntab);
            for (int c = 0; c < m.ntab; ++c) wd[c] = omega * (1.0 / tabs[q][static_cast<size_t>(c) * m.nd + m.diag0]);
            m.wdtab = upload_array(wd);
            m.dom_wd = wd[dom];
        }
    }
    return true;
}

// DIA when the pattern is <= 16 diagonals with <= 15% padding; else SELL-32.
// `omega` > 0 requests the omega/diag dictionary (hierarchy operators).
bool DeviceSolver::upload_rowsig(const Csr& A, int lanes, int split, dev::Mat& out) {
    // Opt-in (IRK_ROW_SIG bit mask: 1 the Q part of a 7-point up leg, 2 the
    // down legs G, 4 the split up legs).  Off by default: at C2 the table reads
    // are one more dependent level per row and the table of the up leg's Q
    // part (10,011 signatures, 960 KB) is not L1-resident -- hot V-cycle 65.9
    // us with it (exceptions skipped) vs 64.6 us without
    // (profiles/r2/ab_composed_vcycle.txt).
    const long long mask = dev::option("IRK_ROW_SIG", 0);
    const long long need = lanes < 2 ? 1 : split > 0 ? 4 : 2;
    if ((mask & need) == 0 || A.rows == 0) return false;
    const int n = A.rows;
    const int cut = split > 0 ? split : A.cols;  // columns >= cut: second operand
    std::vector<unsigned short> sig(n);
    std::vector<int> base0(n, 0), base1(n, 0);
    // signature store: offsets and value bits of each distinct row, in first-seen order
    std::vector<int> sptr{0}, soff;
    std::vector<uint64_t> sval;
    std::unordered_map<uint64_t, std::vector<int>> by_hash;
    std::vector<int> ro;
    std::vector<uint64_t> rv;
    const size_t max_sigs = std::min<size_t>(65535, static_cast<size_t>(n) / 4 + 1);
    int prev = -1;
    for (int i = 0; i < n; ++i) {
        const int lo = A.ptr[i], hi = A.ptr[i + 1];
        int b0 = -1, b1 = -1;
        for (int k = lo; k < hi; ++k) {
            if (A.idx[k] < cut) {
                if (b0 < 0) b0 = A.idx[k];
            } else if (b1 < 0) {
                b1 = A.idx[k] - cut;
            }
        }
        base0[i] = std::max(b0, 0);
        base1[i] = std::max(b1, 0);
        ro.resize(hi - lo);
        rv.resize(hi - lo);
        uint64_t h = 1469598103934665603ULL;
        for (int k = lo; k < hi; ++k) {
            const int c = A.idx[k];
            const int o = c < cut ? c - base0[i] : ((c - cut - base1[i]) | dev::kRsQ);
            uint64_t b;
            std::memcpy(&b, &A.val[k], sizeof(b));
            ro[k - lo] = o;
            rv[k - lo] = b;
            h = (h ^ static_cast<uint64_t>(static_cast<unsigned>(o))) * 1099511628211ULL;
            h = (h ^ b) * 1099511628211ULL;
        }
        auto same = [&](int c) {
            return sptr[c + 1] - sptr[c] == hi - lo && std::equal(ro.begin(), ro.end(), soff.begin() + sptr[c]) &&
                   std::equal(rv.begin(), rv.end(), sval.begin() + sptr[c]);
        };
        int c = -1;
        if (prev >= 0 && same(prev)) {
            c = prev;
        } else {
            std::vector<int>& cand = by_hash[h];
            for (int q : cand)
                if (same(q)) c = q;
            if (c < 0) {
                c = static_cast<int>(sptr.size()) - 1;
                if (static_cast<size_t>(c) >= max_sigs) return false;  // the rows do not repeat
                soff.insert(soff.end(), ro.begin(), ro.end());
                sval.insert(sval.end(), rv.begin(), rv.end());
                sptr.push_back(static_cast<int>(soff.size()));
                cand.push_back(c);
            }
        }
        sig[i] = static_cast<unsigned short>(c);
        prev = c;
    }
    const int ns = static_cast<int>(sptr.size()) - 1;
    int w = 1;
    for (int c = 0; c < ns; ++c) w = std::max(w, sptr[c + 1] - sptr[c]);
    if (static_cast<size_t>(ns) * w * 12 > (size_t(2) << 20)) return false;  // keep the table cache-resident
    std::vector<int> tlen(ns), toff(static_cast<size_t>(ns) * w, 0);
    std::vector<double> tval(static_cast<size_t>(ns) * w, 0.0);
    for (int c = 0; c < ns; ++c) {
        tlen[c] = sptr[c + 1] - sptr[c];
        for (int k = 0; k < tlen[c]; ++k) {
            toff[static_cast<size_t>(c) * w + k] = soff[sptr[c] + k];
            std::memcpy(&tval[static_cast<size_t>(c) * w + k], &sval[sptr[c] + k], sizeof(double));
        }
    }
    dev::Mat m;
    m.rows = A.rows;
    m.cols = A.cols;
    m.nnz = A.nnz();
    m.fmt = dev::kRowSig;
    m.vf = dev::kF64;
    m.lanes = lanes;
    m.tree = lanes >= 2 ? 4 : 0;
    m.rs_sig = upload_array(sig);
    m.rs_base0 = upload_array(base0);
    m.rs_base1 = split > 0 ? upload_array(base1) : nullptr;
    m.rs_len = upload_array(tlen);
    m.rs_off = upload_array(toff);
    m.rs_val = upload_array(tval);
    m.rs_w = w;
    m.rs_n = ns;
    m.bytes = static_cast<size_t>(n) * (split > 0 ? 10 : 6) + static_cast<size_t>(ns) * (4 + 12 * static_cast<size_t>(w));
    out = m;
    return true;
}

bool DeviceSolver::upload_up_cls(const Csr& U, int n, dev::Mat& Sm, dev::Mat& Qm) {
    if (!row_classes_enabled() || dev::option("IRK_UP_CLS", 1) == 0 || U.rows != n || U.cols <= n) return false;
    Csr S, Q;
    S.rows = S.cols = n;
    Q.rows = n;
    Q.cols = U.cols - n;
    S.ptr.assign(n + 1, 0);
    Q.ptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        int ns = 0;
        for (int k = U.ptr[i]; k < U.ptr[i + 1]; ++k) ns += U.idx[k] < n ? 1 : 0;
        S.ptr[i + 1] = S.ptr[i] + ns;
        Q.ptr[i + 1] = Q.ptr[i] + (U.ptr[i + 1] - U.ptr[i] - ns);
    }
    S.idx.resize(S.ptr[n]);
    S.val.resize(S.ptr[n]);
    Q.idx.resize(Q.ptr[n]);
    Q.val.resize(Q.ptr[n]);
    for (int i = 0; i < n; ++i) {
        int os = S.ptr[i], oq = Q.ptr[i];
        for (int k = U.ptr[i]; k < U.ptr[i + 1]; ++k) {
            if (U.idx[k] < n) {
                S.idx[os] = U.idx[k];
                S.val[os++] = U.val[k];
            } else {
                Q.idx[oq] = U.idx[k] - n;
                Q.val[oq++] = U.val[k];
            }
        }
    }
    const DiaLayout L = dia_layout(S);
    if (L.offs.size() != 7) return false;
    dev::Mat m;
    m.rows = m.cols = n;
    m.nnz = S.nnz();
    m.fmt = dev::kDia;
    m.dstride = L.ds;
    m.nd = 7;
    for (int d = 0; d < 7; ++d) {
        m.off[d] = L.offs[d];
        if (L.offs[d] == 0) m.diag0 = d;
    }
    if (!to_row_classes({&m}, {&L.v}, 0.0)) return false;
    Sm = m;
    if (!upload_rowsig(Q, 1, 0, Qm)) {
        pack_sell_ = true;  // k_up_cls reads packed entries
        Qm = upload(Q, false, 0.0, 1);
        pack_sell_ = false;
    }
    return true;
}

dev::Mat DeviceSolver::upload(const Csr& A, bool allow_dia, double omega, int tree_lanes) {
    dev::Mat m;
    m.rows = A.rows;
    m.cols = A.cols;
    m.nnz = A.nnz();
    if (tree_lanes >= 2) {
        m.fmt = dev::kCsrVec;
        m.lanes = tree_lanes;
        {
            // staged entries per lane: covers the 95th percentile row length
            std::vector<int> lens(A.rows);
            for (int i = 0; i < A.rows; ++i) lens[i] = A.ptr[i + 1] - A.ptr[i];
            int p95 = 0;
            if (!lens.empty()) {
                const size_t q = lens.size() * 95 / 100;
                std::nth_element(lens.begin(), lens.begin() + q, lens.end());
                p95 = lens[q];
            }
            const int mm = (p95 + tree_lanes - 1) / tree_lanes;
            m.tree = static_cast<int>(dev::option("IRK_LT_MM", std::min(std::max(mm, 4), 6)));
        }
        m.ptr = upload_array(A.ptr);
        m.bytes += sizeof(int) * (A.ptr.size() + A.idx.size());
        std::vector<unsigned> codes;
        upload_values(m, A.val, omega, &codes);
        if (!codes.empty()) {
            std::vector<int> idx = A.idx;
            pack_codes(m, idx, codes);
            m.idx = upload_array(idx);
        } else {
            m.idx = upload_array(A.idx);
        }
        return m;
    }
    DiaLayout L;
    if (allow_dia) L = dia_layout(A);
    if (!L.offs.empty()) {
        const int nd = static_cast<int>(L.offs.size());
        m.fmt = dev::kDia;
        m.dstride = L.ds;
        m.nd = nd;
        for (int d = 0; d < nd; ++d) {
            m.off[d] = L.offs[d];
            if (L.offs[d] == 0) m.diag0 = d;
        }
        // hierarchy operators: row classes when the stencil repeats; the
        // class also fixes omega / a_cc of every partner row (nbwd)
        if (omega > 0.0 && m.diag0 >= 0 && dev::option("IRK_NBWD", 1) != 0) {
            const long long ds = L.ds;
            std::vector<double> nbw(static_cast<size_t>(nd) * ds, 0.0);
            for (int i = 0; i < A.rows; ++i)
                for (int d = 0; d < nd; ++d) {
                    if (L.v[static_cast<size_t>(d) * ds + i] == 0.0) continue;
                    const int c = std::min(std::max(i + L.offs[d], 0), A.rows - 1);
                    nbw[static_cast<size_t>(d) * ds + i] = omega * (1.0 / L.v[static_cast<size_t>(m.diag0) * ds + c]);
                }
            if (to_row_classes({&m, nullptr}, {&L.v, &nbw}, omega)) return m;
        }
        if (omega > 0.0 && to_row_classes({&m}, {&L.v}, omega)) return m;
        upload_values(m, L.v, omega);
        return m;
    }
    // Long rows: CSR-vector with G lanes per row (G ~ average length / 3).
    const double avg = A.rows ? static_cast<double>(A.nnz()) / A.rows : 0.0;
    static const int force = std::getenv("IRK_SPARSE_FMT") ? std::atoi(std::getenv("IRK_SPARSE_FMT")) : -1;
    // (SELL wins when there are enough rows to fill the GPU with one thread
    // per row; small coarse operators need lanes per row to expose
    // memory-level parallelism.)
    // (big operators switch to CSR-vector above IRK_CSRV_BIG_AVG entries per row)
    static const double big_avg =
        std::getenv("IRK_CSRV_BIG_AVG") ? std::atof(std::getenv("IRK_CSRV_BIG_AVG")) : 24.0;
    const long long sell_min_rows = dev::option("IRK_SELL_MIN_ROWS", 65536);
    if (tree_lanes != 1 &&
        ((force < 0 && avg > 4.5 && (A.rows < sell_min_rows || avg > big_avg)) || force == dev::kCsrVec)) {
        // entries per lane (tenths; IRK_CSRV_PER_LANE10, default 30 = 3.0)
        const double per_lane = 0.1 * static_cast<double>(dev::option("IRK_CSRV_PER_LANE10", 30));
        int g = 2;
        while (g < 32 && per_lane * g < avg) g *= 2;
        // fewer lanes when the grid would spill just past one wave of
        // resident threads (a second, nearly empty wave costs a full row trip)
        if (dev::option("IRK_CSRV_WAVE_CAP", 1) != 0) {
            int dev_id = 0, sms = 148, tpm = 2048;
            cudaGetDevice(&dev_id);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id);
            cudaDeviceGetAttribute(&tpm, cudaDevAttrMaxThreadsPerMultiProcessor, dev_id);
            const long long wave = static_cast<long long>(sms) * tpm;
            const long long thr = static_cast<long long>(A.rows) * g;
            if (thr > wave && thr < 2 * wave && g > 2) g /= 2;
        }
        m.fmt = dev::kCsrVec;
        m.lanes = g;
        m.ptr = upload_array(A.ptr);
        m.idx = upload_array(A.idx);
        m.bytes += sizeof(int) * (A.ptr.size() + A.idx.size());
        upload_values(m, A.val, omega);
        return m;
    }
    // Short rows: SELL-32, slice = 32 consecutive rows padded to the slice's
    // longest row; padding entries repeat the row's last column with a zero.
    const int ns = (A.rows + 31) / 32;
    std::vector<int> sptr(ns + 1, 0);
    for (int sl = 0; sl < ns; ++sl) {
        int len = 0;
        for (int r = sl * 32; r < std::min(A.rows, sl * 32 + 32); ++r)
            len = std::max(len, A.ptr[r + 1] - A.ptr[r]);
        sptr[sl + 1] = sptr[sl] + 32 * len;
    }
    std::vector<int> idx(sptr[ns]);
    std::vector<double> v(sptr[ns], 0.0);
    for (int sl = 0; sl < ns; ++sl) {
        const int len = (sptr[sl + 1] - sptr[sl]) / 32;
        for (int lane = 0; lane < 32; ++lane) {
            const int r = sl * 32 + lane;
            const int lo = r < A.rows ? A.ptr[r] : 0, cnt = r < A.rows ? A.ptr[r + 1] - lo : 0;
            for (int k = 0; k < len; ++k) {
                const size_t e = static_cast<size_t>(sptr[sl]) + k * 32 + lane;
                if (k < cnt) {
                    idx[e] = A.idx[lo + k];
                    v[e] = A.val[lo + k];
                } else {
                    idx[e] = cnt > 0 ? A.idx[lo + cnt - 1] : 0;
                }
            }
        }
    }
    m.fmt = dev::kSell;
    m.sptr = upload_array(sptr);
    m.bytes += sizeof(int) * (sptr.size() + idx.size());
    std::vector<unsigned> codes;
    upload_values(m, v, omega, pack_sell_ ? &codes : nullptr);
    if (!codes.empty()) pack_codes(m, idx, codes);
    m.idx = upload_array(idx);
    return m;
}

DeviceSolver::DeviceSolver(const Csr& M, const Csr& K, int s, const std::vector<double>& A,
                           const std::vector<double>& b, const std::vector<double>& At,
                           Structure structure, double ht, const AmgParams& amg,
                           std::vector<Hierarchy> hiers, int device)
    : s_(s), device_(device), At_(At), structure_(structure), ht_(ht) {
    compress_values_ = dev::option("IRK_NO_VALUE_CODES", 0) == 0;
    {
        const char* o = std::getenv("IRK_ORTHO");
        ortho_ = (o && std::string(o) == "cgs2") ? 0 : 1;
    }
    const auto t0 = std::chrono::steady_clock::now();
    check(s >= 1 && s <= dev::kMaxStages, "device solver: s must be in 1..7");
    check(M.rows == M.cols && K.rows == K.cols && M.rows == K.rows,
          "block preconditioner: M, F size mismatch");
    check(static_cast<int>(A.size()) == s * s && static_cast<int>(At.size()) == s * s &&
              static_cast<int>(b.size()) == s,
          "device solver: coefficient size mismatch");
    check(ht > 0.0, "irk_step: ht must be positive");
    n_ = M.rows;
    sN_ = static_cast<long long>(s) * n_;
    stride_ = (sN_ + 63) / 64 * 64;

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CudaError("no CUDA device: the B200 solve phase has no CPU fallback");
    device_ = device;
    DeviceScope on(device_);
    IRK_CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    dev::set_smem_limits();

    // Hierarchies: one per distinct diagonal coefficient (stage.cpp:85-106).
    std::vector<double> distinct;
    distinct_diagonals(s, At, sob_, distinct);
    if (hiers.empty()) {
        // device setup (bit-identical; IRK_HOST_AMG_SETUP=1 selects the host one)
        static const bool host_setup = std::getenv("IRK_HOST_AMG_SETUP") != nullptr;
        for (double d : distinct)
            hiers.push_back(host_setup ? amg_setup(add(1.0, M, ht * d, K), amg)
                                       : amg_setup_device(add(1.0, M, ht * d, K), amg, device));
    }
    check(hiers.size() == distinct.size(), "device solver: hierarchy count mismatch");
    static const bool timing = std::getenv("IRK_SETUP_TIMING") != nullptr;
    auto lap = [&](const char* what) {
        if (timing) std::fprintf(stderr, "solver setup %-14s %8.1f ms\n", what, 1e3 * seconds_since(t0));
    };
    lap("hierarchies");
    hier_host_ = std::move(hiers);

    M_ = upload(M, true, 0.0);
    K_ = upload(K, true, 0.0);
    if (M_.fmt == dev::kDia && K_.fmt == dev::kDia && M_.nd == K_.nd &&
        std::equal(M_.off, M_.off + M_.nd, K_.off) &&
        !(M_.vf == K_.vf && (M_.vf == dev::kF64 || M_.vf == dev::kU8))) {
        // the fused stage operator needs M and K in one value format (fp64 or
        // u8 codes): e.g. SUPG K with > 256 distinct values -> both fp64
        const bool keep = compress_values_;
        compress_values_ = false;
        M_ = upload(M, true, 0.0);
        K_ = upload(K, true, 0.0);
        compress_values_ = keep;
    }
    lap("M, K");
    fused_op_ = M_.fmt == dev::kDia && K_.fmt == dev::kDia && M_.nd == K_.nd &&
                std::equal(M_.off, M_.off + M_.nd, K_.off) && M_.vf == K_.vf &&
                (M_.vf == dev::kF64 || M_.vf == dev::kU8);
    if (fused_op_ && M_.nd == 7) {
        // one joint row class per row for the stage operator and the sweeps
        const DiaLayout lm = dia_layout(M), lk = dia_layout(K);
        if (lm.ds == M_.dstride && lk.ds == K_.dstride) to_row_classes({&M_, &K_}, {&lm.v, &lk.v}, 0.0);
    }
    coef_.s = s;
    for (int i = 0; i < s * s; ++i) coef_.c[i] = ht * A[i];
    hb_.resize(s);
    for (int i = 0; i < s; ++i) hb_[i] = ht * b[i];

    for (const Hierarchy& h : hier_host_) {
        DevHier dh;
        dh.prm = h.params;
        const int L = h.n_levels();
        dh.lv.resize(L);
        for (int l = L - 1; l >= 0; --l) {
            const AmgLevel& lev = h.levels[l];
            DevLevel d;
            d.n = lev.A.rows;
            d.A = upload(lev.A, true, h.params.jacobi_weight);
            std::vector<double> wd(d.n);
            for (int i = 0; i < d.n; ++i) wd[i] = h.params.jacobi_weight * lev.inv_diag[i];
            d.wd = alloc(d.n);
            IRK_CUDA_CHECK(cudaMemcpy(d.wd, wd.data(), sizeof(double) * d.n, cudaMemcpyHostToDevice));
            if (l + 1 < L) {
                d.P = upload(lev.P, false, 0.0);
                d.R = upload(lev.R, false, 0.0);
                if (lev.G.rows > 0 && lev.U.rows > 0) {
                    if (lev.g_lanes < 2 || !upload_rowsig(lev.G, lev.g_lanes, 0, d.G))
                        d.G = upload(lev.G, false, 0.0, lev.g_lanes);
                    d.up_cls = lev.u_lanes == 1 && upload_up_cls(lev.U, d.n, d.US, d.UQ);
                    if (!d.up_cls && (lev.u_lanes < 2 || !upload_rowsig(lev.U, lev.u_lanes, d.n, d.U)))
                        d.U = upload(lev.U, false, 0.0, lev.u_lanes);
                    if (std::getenv("IRK_SETUP_TIMING"))
                        std::fprintf(stderr, "level %d composed: G fmt %d (%d sigs, w %d)  U %s fmt %d (%d sigs, w %d)\n", l,
                                     d.G.fmt, d.G.rs_n, d.G.rs_w, d.up_cls ? "cls+Q" : "split",
                                     d.up_cls ? d.UQ.fmt : d.U.fmt, d.up_cls ? d.UQ.rs_n : d.U.rs_n,
                                     d.up_cls ? d.UQ.rs_w : d.U.rs_w);
                }
            }
            d.t = alloc(d.n);
            d.u = alloc(d.n);
            if (h.params.pre_sweeps > 1 || h.params.smoother != 0) d.zp = alloc(d.n);
            if (h.params.smoother != 0 && l + 1 < L) {
                d.gsf = upload_gs(lev.A, lev.inv_diag, false);
                d.gsb = upload_gs(lev.A, lev.inv_diag, true);
                // gather scratch, shared by the level's (sequential) sweeps
                d.gsf.rs = d.gsb.rs = alloc(d.n);
                d.gsf.ps = d.gsb.ps = alloc(std::max<long long>(std::max(d.gsf.nnz, d.gsb.nnz), 1));
            }
            if (l > 0) {
                d.r = alloc(d.n);
                d.z = alloc(d.n);
                d.zr = alloc(d.n);
            }
            dh.lv[l] = d;
        }
        dh.nc = h.levels.back().A.rows;
        if (h.tail_from > 0) {
            dh.tail_from = h.tail_from;
            dh.tail_ld = h.tail_ld;
            dh.tail = alloc(h.tail.size());
            IRK_CUDA_CHECK(cudaMemcpy(dh.tail, h.tail.data(), sizeof(double) * h.tail.size(),
                                      cudaMemcpyHostToDevice));
        }
        build_bottom(dh, h);
        dh.cinv = alloc(static_cast<size_t>(dh.nc) * dh.nc);
        IRK_CUDA_CHECK(cudaMemcpy(dh.cinv, h.coarse_inverse.data(),
                                  sizeof(double) * dh.nc * dh.nc, cudaMemcpyHostToDevice));
        hier_.push_back(std::move(dh));
        lap("hierarchy up");
    }

    rhs_ = alloc(n_);
    fw_ = alloc(static_cast<size_t>(s) * n_);
    u_ = alloc(n_);
    lift_ = alloc(n_);
    unext_ = alloc(n_);
    ku_ = alloc(n_);
    b_ = alloc(stride_);
    x_ = alloc(stride_);
    r_ = alloc(stride_);
    ax_ = alloc(stride_);
    const long long nch = (sN_ + dev::kChunk - 1) / dev::kChunk;
    red_part_ = alloc(nch + 1);
    red_out_ = alloc(8);
    bufs_.emplace_back(sizeof(unsigned) * 16);
    red_cnt_ = bufs_.back().as<unsigned>();
    IRK_CUDA_CHECK(cudaMemset(red_cnt_, 0, sizeof(unsigned) * 16));
    IRK_CUDA_CHECK(cudaDeviceSynchronize());
    setup_seconds_ = seconds_since(t0);
}

DeviceSolver::~DeviceSolver() {
    DeviceScope on(device_);
    for (cudaGraphExec_t* e : {&exec_, &exec_iter_, &exec_pre_, &exec_cb_, &exec_ce_, &exec_post_})
        if (*e) cudaGraphExecDestroy(*e);
    for (Branches& b : branch_sets_) {
        for (cudaStream_t x : b.st)
            if (x) cudaStreamDestroy(x);
        for (cudaEvent_t e : b.ev)
            if (e) cudaEventDestroy(e);
    }
    if (ctl_host_) cudaFreeHost(ctl_host_);
    if (hist_host_) cudaFreeHost(hist_host_);
    if (st_) cudaStreamDestroy(st_);
}

int DeviceSolver::matrix_format(int which) const { return which == 0 ? M_.fmt : K_.fmt; }

// ------------------------------------------------------------------ recording
// One V(pre,post) cycle (amg.cpp:144-168) with fused kernels per level:
//   t = r - A (wd.*r)      pre-smooth from zero fused into the residual
//   r_{l+1} = R t          restriction
//   t = wd.*r + P z_{l+1}  prolongation fused with the pre-smoothed iterate
//   z = t + wd.*(r - A t)  post-smoothing sweep
// Packs the deepest levels whose operators fit one CTA's shared memory into
// the bottom kernel's blob (smallest first level b >= 1 that fits).
void DeviceSolver::build_bottom(DevHier& dh, const Hierarchy& h) {
    const int L = h.n_levels();
    if (dev::option("IRK_BOTTOM", 1) == 0 || L < 3) return;
    if (h.params.pre_sweeps != 1 || h.params.post_sweeps != 1 || h.params.smoother != 0) return;
    const int budget = 225 * 1024;
    bool force_csr = false;
    for (int b = 1; b <= L - 2; ++b) {
        if (L - 1 - b > dev::kMaxBot) continue;
        std::vector<char> blob;
        auto put = [&](const void* p, size_t bytes) {
            const int off = static_cast<int>(blob.size());
            blob.resize((blob.size() + bytes + 15) / 16 * 16, 0);
            if (bytes) std::memcpy(blob.data() + off, p, bytes);
            return off;
        };
        bool ok = true;
        auto put_csr = [&](const Csr& A, int& po, int& io, int& vo) {
            if (A.cols > 65535) ok = false;
            std::vector<unsigned short> ix(A.idx.begin(), A.idx.end());
            po = put(A.ptr.data(), sizeof(int) * A.ptr.size());
            io = put(ix.data(), sizeof(unsigned short) * ix.size());
            vo = put(A.val.data(), sizeof(double) * A.val.size());
        };
        // A_l as SELL-32 (conflict-free shared loads) unless the padding
        // would not fit, then CSR
        auto put_sell = [&](const Csr& A, dev::BotLevel& bl) {
            if (A.cols > 65535) ok = false;
            const int ns = (A.rows + 31) / 32;
            std::vector<int> sp(ns + 1, 0);
            std::vector<unsigned short> len(A.rows);
            for (int sl = 0; sl < ns; ++sl) {
                int mx = 0;
                for (int r = sl * 32; r < std::min(A.rows, sl * 32 + 32); ++r) {
                    len[r] = static_cast<unsigned short>(A.ptr[r + 1] - A.ptr[r]);
                    mx = std::max(mx, A.ptr[r + 1] - A.ptr[r]);
                }
                sp[sl + 1] = sp[sl] + 32 * mx;
            }
            std::vector<unsigned short> ix(sp[ns], 0);
            std::vector<double> vv(sp[ns], 0.0);
            for (int r = 0; r < A.rows; ++r)
                for (int q = 0; q < A.ptr[r + 1] - A.ptr[r]; ++q) {
                    const size_t e = static_cast<size_t>(sp[r / 32]) + 32 * q + (r % 32);
                    ix[e] = static_cast<unsigned short>(A.idx[A.ptr[r] + q]);
                    vv[e] = A.val[A.ptr[r] + q];
                }
            bl.a_sell = 1;
            bl.a_ptr = put(sp.data(), sizeof(int) * sp.size());
            bl.a_len = put(len.data(), sizeof(unsigned short) * len.size());
            bl.a_idx = put(ix.data(), sizeof(unsigned short) * ix.size());
            bl.a_val = put(vv.data(), sizeof(double) * vv.size());
        };
        const bool sell = dev::option("IRK_BOTTOM_SELL", 1) != 0 && !force_csr;
        dev::BotDesc d;
        d.nl = L - 1 - b;
        long long vec = 0;
        for (int q = 0; q < d.nl; ++q) {
            const AmgLevel& lev = h.levels[b + q];
            dev::BotLevel& bl = d.lv[q];
            bl.n = lev.A.rows;
            if (sell) {
                put_sell(lev.A, bl);
            } else {
                bl.a_sell = 0;
                bl.a_len = 0;
                put_csr(lev.A, bl.a_ptr, bl.a_idx, bl.a_val);
            }
            put_csr(lev.P, bl.p_ptr, bl.p_idx, bl.p_val);
            put_csr(lev.R, bl.r_ptr, bl.r_idx, bl.r_val);
            std::vector<double> wd(bl.n);
            for (int i = 0; i < bl.n; ++i) wd[i] = h.params.jacobi_weight * lev.inv_diag[i];
            bl.wd = put(wd.data(), sizeof(double) * wd.size());
            vec += 3LL * bl.n;
        }
        d.nc = h.levels.back().A.rows;
        {
            // column-major copy of the dense inverse
            const int nc = h.levels.back().A.rows;
            std::vector<double> ct(h.coarse_inverse.size());
            for (int i = 0; i < nc; ++i)
                for (int j = 0; j < nc; ++j) ct[static_cast<size_t>(j) * nc + i] = h.coarse_inverse[static_cast<size_t>(i) * nc + j];
            d.cinv = put(ct.data(), sizeof(double) * ct.size());
        }
        vec += 3LL * d.nc;
        d.bytes = static_cast<int>(blob.size());
        d.vec = d.bytes;
        {
            int off = d.vec;
            for (int q = 0; q <= d.nl; ++q) {
                const int nq = q < d.nl ? d.lv[q].n : d.nc;
                d.vr[q] = off;
                d.vt[q] = off + 8 * nq;
                d.vz[q] = off + 16 * nq;
                off += 24 * nq;
            }
        }
        const long long total = d.bytes + 8 * vec;
        if (std::getenv("IRK_SETUP_TIMING"))
            std::fprintf(stderr, "bottom candidate: levels %d..%d, A %s: %lld B%s\n", b, L - 1,
                         force_csr ? "CSR" : "SELL-32", total, total > budget ? " (too big)" : "");
        if (ok && total > budget && !force_csr) {
            force_csr = true;  // retry this b with CSR operators
            --b;
            continue;
        }
        force_csr = false;
        if (!ok || total > budget) continue;
        d.smem = static_cast<int>(total);
        if (std::getenv("IRK_SETUP_TIMING"))
            std::fprintf(stderr, "bottom kernel: levels %d..%d, A %s, blob %d B, smem %d B\n", b, L - 1,
                         d.lv[0].a_sell ? "SELL-32" : "CSR", d.bytes, d.smem);
        std::vector<char> padded = blob;
        d.blob = upload_array(padded);
        dh.bot = d;
        dh.bot_from = b;
        return;
    }
}

namespace {
// IRK_ZR=0: levels >= 1 recompute wd .* r on the fly instead of reading the
// copy the restriction wrote (A/B switch)
bool zr_on() { return dev::option("IRK_ZR", 1) != 0; }
}  // namespace

// Gauss-Seidel schedule of one level (amg.cpp:125-140): depth(i) = 1 + max
// depth(j) over the entries a_ij the sweep reads updated (j < i forward, j > i
// backward); positions sorted by depth (stable in i) and cut into chunks of
// <= kGsRows rows whose entries, padded to the chunk's longest row, fit
// kGsEnt; a chunk's entries column-major (dev::GsSweep), each row's in CSR
// column order without the diagonal, with their source codes.
dev::GsSweep DeviceSolver::upload_gs(const Csr& A, const std::vector<double>& inv_diag,
                                     bool backward) {
    const int n = A.rows;
    std::vector<int> depth(n, 0);
    int nlev = 0;
    for (int t = 0; t < n; ++t) {
        const int i = backward ? n - 1 - t : t;
        int d = 0;
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int c = A.idx[k];
            if (backward ? c > i : c < i) d = std::max(d, depth[c] + 1);
        }
        depth[i] = d;
        nlev = std::max(nlev, d + 1);
    }
    std::vector<int> lptr(nlev + 1, 0);
    for (int i = 0; i < n; ++i) ++lptr[depth[i] + 1];
    for (int l = 0; l < nlev; ++l) lptr[l + 1] += lptr[l];
    std::vector<int> order(n), pos(n);
    {
        std::vector<int> fill(lptr.begin(), lptr.end() - 1);
        for (int i = 0; i < n; ++i) order[fill[depth[i]]++] = i;
    }
    for (int q = 0; q < n; ++q) pos[order[q]] = q;
    std::vector<int> len(n);
    for (int q = 0; q < n; ++q) {
        const int i = order[q];
        int c = 0;
        for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) c += A.idx[k] != i;
        len[q] = c;
        check(c <= dev::kGsEnt, "gauss-seidel: row longer than the staging buffer");
    }
    // chunks: each depth cut into pieces whose padded entries fit a buffer
    std::vector<int> cptr{0}, width;
    for (int l = 0; l < nlev; ++l) {
        int rows = 0, w = 0;
        for (int q = lptr[l]; q < lptr[l + 1]; ++q) {
            const int w2 = std::max(w, len[q]);
            if (rows > 0 && (rows + 1 > dev::kGsRows || static_cast<long long>(w2) * (rows + 1) > dev::kGsEnt)) {
                cptr.push_back(q);
                width.push_back(w);
                rows = 0;
                w = 0;
            }
            ++rows;
            w = std::max(w, len[q]);
        }
        cptr.push_back(lptr[l + 1]);
        width.push_back(w);
    }
    const int nch = static_cast<int>(cptr.size()) - 1;
    std::vector<int> ceptr(nch + 1, 0), chunk_end(n);
    for (int c = 0; c < nch; ++c) {
        ceptr[c + 1] = ceptr[c] + width[c] * (cptr[c + 1] - cptr[c]);
        for (int q = cptr[c]; q < cptr[c + 1]; ++q) chunk_end[q] = cptr[c + 1];
    }
    const long long nnz = ceptr[nch];
    std::vector<int2> hdr(n);
    // padding entries: value 0, gather code 0, the ring's 1.0 slot (never summed)
    std::vector<int> ref(std::max<long long>(nnz, 1), 0), sref(std::max<long long>(nnz, 1), dev::kGsRing);
    std::vector<double> val(std::max<long long>(nnz, 1), 0.0), dinv(n);
    long long far = 0;
    for (int c = 0; c < nch; ++c) {
        const int nr = cptr[c + 1] - cptr[c];
        for (int q = cptr[c]; q < cptr[c + 1]; ++q) {
            const int i = order[q];
            hdr[q] = make_int2(i, len[q]);
            dinv[q] = inv_diag[i];
            int k = 0;
            for (int kk = A.ptr[i]; kk < A.ptr[i + 1]; ++kk) {
                const int col = A.idx[kk];
                if (col == i) continue;
                const long long e = ceptr[c] + static_cast<long long>(k) * nr + (q - cptr[c]);
                const bool updated = backward ? col > i : col < i;
                if (!updated) {
                    ref[e] = -(2 * col + 1);
                    sref[e] = dev::kGsRing;  // the gathered product x 1.0
                } else if (pos[col] + dev::kGsRing >= chunk_end[q]) {
                    // the ring slot survives until q's chunk ends
                    sref[e] = pos[col] & (dev::kGsRing - 1);
                } else {
                    sref[e] = -(col + 2);  // zout[col]
                    ++far;
                }
                val[e] = A.val[kk];
                ++k;
            }
        }
    }
    dev::GsSweep g;
    g.hdr = upload_array(hdr);
    g.ref = upload_array(ref);
    g.sref = upload_array(sref);
    g.val = upload_array(val);
    g.dinv = upload_array(dinv);
    g.cptr = upload_array(cptr);
    g.ceptr = upload_array(ceptr);
    g.nch = nch;
    g.n = n;
    g.nnz = nnz;
    g.far = far > 0;
    if (std::getenv("IRK_SETUP_TIMING")) {
        long long real = 0;
        for (int q = 0; q < n; ++q) real += len[q];
        std::fprintf(stderr, "gs %s: n %d, depths %d, chunks %d, entries %lld (stored %lld), %lld beyond the ring\n",
                     backward ? "bwd" : "fwd", n, nlev, nch, real, nnz, far);
    }
    return g;
}

// V(pre, post) cycle with the Gauss-Seidel smoother, the reference's own
// order (amg.cpp:144-168): pre forward sweeps from z = 0, t = r - A z,
// r_c = R t, the coarse cycle, z + P z_c, post backward sweeps.  Sweeps
// ping-pong between two level vectors (see gs_sweep); the tail operator and
// the dense coarsest inverse are shared with the Jacobi cycle.
void DeviceSolver::record_vcycle_gs(int k, VecRef r0, VecRef z0, int first) {
    DevHier& H = hier_[k];
    const int L = static_cast<int>(H.lv.size());
    const int pre = H.prm.pre_sweeps, post = H.prm.post_sweeps;
    auto rhs_of = [&](int l) { return l == first ? r0 : dev::plain(H.lv[l].r); };
    auto out_of = [&](int l) { return l == first ? z0 : dev::plain(H.lv[l].z); };
    const int tail = dev::option("IRK_TAIL", 1) != 0 && H.tail_from > first ? H.tail_from : -1;
    const int down_end = tail > 0 ? tail : L - 1;
    for (int l = first; l < down_end; ++l) {
        DevLevel& d = H.lv[l];
        // pre sweeps, the last one into zp
        const double* in = nullptr;
        for (int sw = 0; sw < pre; ++sw) {
            double* out = (pre - 1 - sw) % 2 == 0 ? d.zp : d.u;
            dev::gs_sweep(d.gsf, false, rhs_of(l), in, dev::plain(out), st_);
            in = out;
        }
        dev::SpmvArgs a;
        a.x = dev::plain(d.zp);
        a.r = rhs_of(l);
        a.y = dev::plain(d.t);
        dev::spmv(d.A, dev::kXPlain, dev::kEResid, a, st_);
        dev::SpmvArgs ra;
        ra.x = dev::plain(d.t);
        ra.y = dev::plain(H.lv[l + 1].r);
        dev::spmv(d.R, dev::kXPlain, dev::kEPlain, ra, st_);
    }
    if (tail > 0)
        dev::tail_mv(H.lv[tail].n, H.tail_ld, H.tail, H.lv[tail].r, H.lv[tail].z, st_);
    else
        dev::dense_mv(H.nc, H.cinv, rhs_of(L - 1), out_of(L - 1), st_);
    for (int l = down_end - 1; l >= first; --l) {
        DevLevel& d = H.lv[l];
        dev::SpmvArgs pa;
        pa.x = dev::plain(H.lv[l + 1].z);
        pa.zb = d.zp;
        pa.y = dev::plain(d.t);
        dev::spmv(d.P, dev::kXPlain, dev::kEProlong, pa, st_);
        double* cur = d.t;
        for (int sw = 0; sw < post; ++sw) {
            double* nxt = cur == d.t ? d.u : d.t;
            const VecRef out = sw == post - 1 ? out_of(l) : dev::plain(nxt);
            dev::gs_sweep(d.gsb, true, rhs_of(l), cur, out, st_);
            cur = nxt;
        }
    }
}

void DeviceSolver::record_vcycle(int k, VecRef r0, VecRef z0, int first) {
    DevHier& H = hier_[k];
    if (H.prm.smoother != 0) {
        record_vcycle_gs(k, r0, z0, first);
        return;
    }
    const int L = static_cast<int>(H.lv.size());
    const int pre = H.prm.pre_sweeps, post = H.prm.post_sweeps;
    // `first` > 0 runs only the part of the cycle below level `first` (timing)
    auto rhs_of = [&](int l) { return l == first ? r0 : dev::plain(H.lv[l].r); };
    // programmatic launches for the latency-bound levels >= 2
    // (IRK_PDL_COARSE=<level> moves the threshold, -1 turns it off)
    static const int pdl_from = std::getenv("IRK_PDL_COARSE") ? std::atoi(std::getenv("IRK_PDL_COARSE")) : 2;
    // IRK_PDL_FINE=1: the levels below pdl_from are launched programmatically
    // too, with the trigger at the end of each thread's work (SpmvArgs::late)
    const bool fine_late = dev::option("IRK_PDL_FINE", 1) != 0;
    auto scope = [&](int l) {
        const bool coarse = pdl_from >= 0 && l >= pdl_from;
        dev::set_pdl_scope(coarse);
        dev::set_pdl_late(!coarse && fine_late);
    };
    auto out_of = [&](int l) { return l == first ? z0 : dev::plain(H.lv[l].z); };
    // levels >= bot run in the single-CTA bottom kernel
    // levels >= tail are one dense matvec (IRK_TAIL=0: the recursive cycle)
    const int tail = dev::option("IRK_TAIL", 1) != 0 && H.tail_from > first ? H.tail_from : -1;
    // composed levels (compose.cpp): one kernel down (r_{l+1} = G r_l), one up
    // (z_l = U [r_l; z_{l+1}]); a composed hierarchy has no bottom kernel
    auto composed = [&](int l) { return pre == 1 && post == 1 && H.lv[l].G.rows > 0; };
    const int bot = tail < 0 && dev::option("IRK_BOTTOM", 1) != 0 && H.bot_from > first && pre == 1 &&
                            post == 1 && !composed(first)
                        ? H.bot_from : -1;
    const int down_end = tail > 0 ? tail : bot > 0 ? bot : L - 1;
    for (int l = first; l < down_end; ++l) {
        DevLevel& d = H.lv[l];
        scope(l);
        // the cycle's first kernel: programmatic only after a late-trigger
        // kernel (a block sweep), not after one that triggers at its start
        if (l == first && !vc_pdl_first_) dev::set_pdl_late(false);
        if (composed(l)) {
            dev::SpmvArgs ga;
            ga.x = rhs_of(l);
            ga.y = dev::plain(H.lv[l + 1].r);
            dev::spmv(d.G, dev::kXPlain, dev::kEPlain, ga, st_);
            continue;
        }
        dev::SpmvArgs a;
        a.r = rhs_of(l);
        a.wd = d.wd;
        a.y = dev::plain(d.t);
        // below the entry level the restriction already wrote wd .* r
        const bool zr = zr_on() && pre == 1 && l > first && d.zr;
        if (zr) {
            a.x = dev::plain(d.zr);
            dev::spmv(d.A, dev::kXPlain, dev::kEResid, a, st_);
        } else if (pre == 1) {
            dev::spmv(d.A, dev::kXWdR, dev::kEResid, a, st_);
        } else {
            dev::wd_times_r(d.n, d.wd, a.r, d.zp, st_);
            double* cur = d.zp;
            double* tmp = d.u;
            for (int sw = 1; sw < pre; ++sw) {
                dev::SpmvArgs sa = a;
                sa.x = dev::plain(cur);
                sa.y = dev::plain(tmp);
                dev::spmv(d.A, dev::kXPlain, dev::kESmooth, sa, st_);
                std::swap(cur, tmp);
            }
            if (cur != d.zp)
                IRK_CUDA_CHECK(cudaMemcpyAsync(d.zp, cur, sizeof(double) * d.n, cudaMemcpyDeviceToDevice, st_));
            a.x = dev::plain(d.zp);
            dev::spmv(d.A, dev::kXPlain, dev::kEResid, a, st_);
        }
        scope(l);
        dev::SpmvArgs ra;
        ra.x = dev::plain(d.t);
        ra.y = dev::plain(H.lv[l + 1].r);
        if (zr_on() && pre == 1 && l + 2 < L && l + 1 != bot && l + 1 != tail) {
            ra.y2 = H.lv[l + 1].zr;
            ra.wd2 = H.lv[l + 1].wd;
        }
        dev::spmv(d.R, dev::kXPlain, dev::kEPlain, ra, st_);
    }
    if (tail > 0) {
        scope(tail);
        dev::tail_mv(H.lv[tail].n, H.tail_ld, H.tail, H.lv[tail].r, H.lv[tail].z, st_);
    } else if (bot > 0) {
        scope(bot);
        dev::bottom_cycle(H.bot, H.lv[bot].r, H.lv[bot].z, st_);
    } else {
        scope(L - 1);
        dev::dense_mv(H.nc, H.cinv, rhs_of(L - 1), out_of(L - 1), st_);
    }
    for (int l = (tail > 0 ? tail - 1 : bot > 0 ? bot - 1 : L - 2); l >= first; --l) {
        DevLevel& d = H.lv[l];
        scope(l);
        if (composed(l)) {
            dev::SpmvArgs ua;
            ua.x = rhs_of(l);
            ua.x2 = dev::plain(H.lv[l + 1].z);
            ua.split = d.n;
            ua.y = out_of(l);
            if (d.up_cls)
                dev::up_cls(d.US, d.UQ, ua, st_);
            else
                dev::spmv(d.U, dev::kXSplit, dev::kEPlain, ua, st_);
            continue;
        }
        dev::SpmvArgs pa;
        pa.x = dev::plain(H.lv[l + 1].z);
        pa.r = rhs_of(l);
        pa.wd = d.wd;
        pa.zb = pre == 1 ? (zr_on() && l > first && d.zr ? d.zr : nullptr) : d.zp;
        pa.y = dev::plain(d.t);
        dev::spmv(d.P, dev::kXPlain, dev::kEProlong, pa, st_);
        double* cur = d.t;
        for (int sw = 0; sw < post; ++sw) {
            dev::SpmvArgs sa;
            sa.x = dev::plain(cur);
            sa.r = rhs_of(l);
            sa.wd = d.wd;
            const bool last = sw == post - 1;
            double* nxt = cur == d.t ? d.u : d.t;
            sa.y = last ? out_of(l) : dev::plain(nxt);
            dev::spmv(d.A, dev::kXPlain, dev::kESmooth, sa, st_);
            cur = nxt;
        }
    }
    dev::set_pdl_scope(false);
    dev::set_pdl_late(false);
}

// Block preconditioner apply (stage.cpp:138-182): diagonal, forward (LD,
// GSL) or backward (DU) block substitution, one V-cycle per block.  The
// off-diagonal K-products are fused into the sweep kernel that assembles the
// next block's right-hand side.
void DeviceSolver::record_precond(VecRef v, VecRef w) {
    const int s = s_;
    const long long n = n_;
    const int nh = static_cast<int>(hier_.size());
    static const bool serial = std::getenv("IRK_SERIAL_JACOBI") != nullptr;
    if (structure_ == Structure::Diagonal && nh > 1 && !serial) {
        // Block Jacobi (stage.cpp:151-153): the subsolves are independent, so
        // each distinct hierarchy gets its own stream branch (a fork/join in
        // the captured graph); blocks sharing a hierarchy share its level
        // buffers and run in stage order on that branch.
        // A stream that joined one capture stays in it until that capture
        // ends, so nested captures (outer and inner WHILE bodies) each take
        // a set of branch streams no capture is using.
        Branches* set = nullptr;
        for (Branches& b : branch_sets_) {
            bool busy = false;
            for (int k = 1; k < nh; ++k) {
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                IRK_CUDA_CHECK(cudaStreamIsCapturing(b.st[k], &cs));
                busy = busy || cs != cudaStreamCaptureStatusNone;
            }
            if (!busy) {
                set = &b;
                break;
            }
        }
        if (!set) {
            branch_sets_.emplace_back();
            set = &branch_sets_.back();
            set->st.assign(nh, nullptr);
            set->ev.assign(nh + 1, nullptr);
            for (int k = 1; k < nh; ++k)
                IRK_CUDA_CHECK(cudaStreamCreateWithFlags(&set->st[k], cudaStreamNonBlocking));
            for (auto& e : set->ev) IRK_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const std::vector<cudaStream_t>& branch_ = set->st;
        const std::vector<cudaEvent_t>& branch_ev_ = set->ev;
        cudaStream_t main = st_;
        IRK_CUDA_CHECK(cudaEventRecord(branch_ev_[0], main));
        for (int k = 0; k < nh; ++k) {
            st_ = k == 0 ? main : branch_[k];
            if (k > 0) IRK_CUDA_CHECK(cudaStreamWaitEvent(st_, branch_ev_[0], 0));
            for (int j = 0; j < s; ++j)
                if (sob_[j] == k) record_vcycle(k, block(v, j * n), block(w, j * n));
            if (k > 0) IRK_CUDA_CHECK(cudaEventRecord(branch_ev_[k], st_));
        }
        st_ = main;
        for (int k = 1; k < nh; ++k) IRK_CUDA_CHECK(cudaStreamWaitEvent(main, branch_ev_[k], 0));
        return;
    }
    auto e = [&](int j, int k) { return -ht_ * At_[j * s + k]; };
    const bool fine_late = dev::option("IRK_PDL_FINE", 1) != 0;
    for (int q = 0; q < s; ++q) {
        const int j = structure_ == Structure::Upper ? s - 1 - q : q;
        VecRef in = block(v, j * n);
        bool swept = false;
        if (structure_ != Structure::Diagonal && q > 0) {
            const int prev = structure_ == Structure::Upper ? j + 1 : j - 1;
            const int k0 = structure_ == Structure::Upper ? j + 1 : 0;
            const int k1 = structure_ == Structure::Upper ? s : j;
            // later stages that still need K w_prev
            bool later = false;
            for (int q2 = q + 1; q2 < s; ++q2) {
                const int j2 = structure_ == Structure::Upper ? s - 1 - q2 : q2;
                if (At_[j2 * s + prev] != 0.0) later = true;
            }
            dev::SweepTerms t{};
            bool fresh = false;
            for (int k = k0; k < k1; ++k) {
                if (At_[j * s + k] == 0.0) continue;
                t.coef[t.nt] = e(j, k);
                t.buf[t.nt] = k == prev ? nullptr : fw_ + k * n;
                if (k == prev) fresh = true;
                ++t.nt;
            }
            if (fresh || later) {
                double* store = later ? fw_ + prev * n : nullptr;
                if (K_.fmt == dev::kDia) {
                    // programmatic, late trigger: it follows the previous
                    // V-cycle's last (late-trigger) kernel
                    dev::set_pdl_late(fine_late);
                    dev::sweep_dia(K_, block(w, prev * n), in, t, store, dev::plain(rhs_), n_, st_);
                    dev::set_pdl_late(false);
                    swept = true;
                } else {
                    dev::SpmvArgs a;
                    a.x = block(w, prev * n);
                    a.y = dev::plain(fw_ + prev * n);
                    dev::spmv(K_, dev::kXPlain, dev::kEPlain, a, st_);
                    for (int q3 = 0; q3 < t.nt; ++q3)
                        if (!t.buf[q3]) t.buf[q3] = fw_ + prev * n;
                    dev::combine(in, t, dev::plain(rhs_), n_, st_);
                }
                in = dev::plain(rhs_);
            } else if (t.nt > 0) {
                dev::combine(in, t, dev::plain(rhs_), n_, st_);
                in = dev::plain(rhs_);
            }
        }
        vc_pdl_first_ = swept;
        record_vcycle(sob_[j], in, block(w, j * n));
        vc_pdl_first_ = false;
    }
}

// Stage operator (stage.cpp:28-44): fused single pass when M and K share a
// DIA pattern, otherwise s K-products, s M-products and s^2 axpys.
void DeviceSolver::record_stage_op(VecRef z, VecRef y) {
    if (fused_op_) {
        dev::stage_op_dia(M_, K_, coef_, z, y, n_, st_);
        return;
    }
    const long long n = n_;
    for (int j = 0; j < s_; ++j) {
        dev::SpmvArgs a;
        a.x = block(z, j * n);
        a.y = dev::plain(fw_ + j * n);
        dev::spmv(K_, dev::kXPlain, dev::kEPlain, a, st_);
    }
    for (int i = 0; i < s_; ++i) {
        dev::SpmvArgs a;
        a.x = block(z, i * n);
        a.y = block(y, i * n);
        dev::spmv(M_, dev::kXPlain, dev::kEPlain, a, st_);
        for (int j = 0; j < s_; ++j)
            dev::axpy(coef_.c[i * s_ + j], fw_ + j * n, block(y, i * n), n_, st_);
    }
}

// One Arnoldi iteration: Z_j = P^-1 V_j, V_{j+1} = A Z_j, CGS (+ conditional
// second pass), Givens, normalisation.
void DeviceSolver::record_iteration() {
    const int* jp = &gb_.ctl->j;
    if (side_ == 0) {
        // left (gmres.cpp:69-71): w = P^-1 (A vt_j); Z_j keeps the operator
        // input vt_j so that x += Z y in both sides' flexible form
        dev::copy_ref(slot(gb_.V, jp, stride_, 0), slot(gb_.Z, jp, stride_, 0), sN_, st_);
        record_stage_op(slot(gb_.V, jp, stride_, 0), dev::plain(ax_));
        record_precond(dev::plain(ax_), slot(gb_.V, jp, stride_, 1));
    } else {
        record_precond(slot(gb_.V, jp, stride_, 0), slot(gb_.Z, jp, stride_, 0));
        // after the last V-cycle's late-trigger smoother (not after the
        // block-Jacobi join)
        const bool late = dev::option("IRK_PDL_FINE", 1) != 0 &&
                          !(structure_ == Structure::Diagonal && hier_.size() > 1);
        dev::set_pdl_late(late);
        record_stage_op(slot(gb_.Z, jp, stride_, 0), slot(gb_.V, jp, stride_, 1));
        dev::set_pdl_late(false);
    }
    if (ortho_ == 1) {
        // programmatic launches: the block-dot's static loads overlap the
        // operator's tail, the update's the block-dot's scalar tail
        // (IRK_PDL_DGS=0 turns this off)
        dev::set_pdl_scope(dev::option("IRK_PDL_DGS", 1) != 0);
        dev::gm_dgs_dot(gb_, 0, st_);
        dev::gm_dgs_update(gb_, st_);
        dev::set_pdl_scope(false);
        return;
    }
    dev::gm_blockdot(gb_, 1, st_);
    dev::gm_update(gb_, 1, st_);
    dev::gm_blockdot(gb_, 2, st_);
    dev::gm_update(gb_, 2, st_);
    dev::gm_normalize(gb_, st_);
}

// ------------------------------------------------------------------ GMRES
void DeviceSolver::ensure_gmres(int restart, int max_iter) {
    check(restart <= dev::kMaxRestart, "gmres: restart exceeds the device capacity (512)");
    if (restart <= cap_restart_ && max_iter <= cap_iter_) return;
    for (cudaGraphExec_t* e : {&exec_, &exec_iter_, &exec_pre_, &exec_cb_, &exec_ce_, &exec_post_})
        if (*e) {
            cudaGraphExecDestroy(*e);
            *e = nullptr;
        }
    g_restart_ = -1;
    cap_restart_ = std::max(restart, cap_restart_);
    cap_iter_ = std::max(max_iter, cap_iter_);
    V_ = DevBuf(sizeof(double) * stride_ * (cap_restart_ + 1));
    Z_ = DevBuf(sizeof(double) * stride_ * cap_restart_);
    H_ = DevBuf(sizeof(double) * (cap_restart_ + 1) * (cap_restart_ + 1));
    hist_ = DevBuf(sizeof(double) * (cap_iter_ + 1));
    const int nch = static_cast<int>((sN_ + dev::kChunk - 1) / dev::kChunk);
    // k_dgs_dot writes nv = 2j + 2 per-chunk partials at inner index j < cap
    // (and the cycle-end finalize 2j + 4); size for the largest, like dgs_smem.
    part_ = DevBuf(sizeof(double) * static_cast<size_t>(2 * cap_restart_ + 4) * nch);
    ctl_ = DevBuf(sizeof(dev::GmresCtl));
    cnt_ = DevBuf(sizeof(unsigned) * 16);
    IRK_CUDA_CHECK(cudaMemset(cnt_.as<void>(), 0, sizeof(unsigned) * 16));
    IRK_CUDA_CHECK(cudaMemset(ctl_.as<void>(), 0, sizeof(dev::GmresCtl)));
    if (ctl_host_) cudaFreeHost(ctl_host_);
    if (hist_host_) cudaFreeHost(hist_host_);
    IRK_CUDA_CHECK(cudaMallocHost(&ctl_host_, sizeof(dev::GmresCtl)));
    IRK_CUDA_CHECK(cudaMallocHost(&hist_host_, sizeof(double) * (cap_iter_ + 1)));
    gb_.ctl = ctl_.as<dev::GmresCtl>();
    gb_.H = H_.as<double>();
    gb_.hist = hist_.as<double>();
    gb_.partials = part_.as<double>();
    gb_.counters = cnt_.as<unsigned>();
    gb_.V = V_.as<double>();
    gb_.Z = Z_.as<double>();
    gb_.sN = sN_;
    gb_.nchunks = nch;
    gb_.cap = cap_restart_;
}

namespace {

struct Capture {
    cudaStream_t st;
    cudaGraph_t g = nullptr;
};

cudaGraphExec_t instantiate(cudaGraph_t g) {
    cudaGraphExec_t e = nullptr;
    IRK_CUDA_CHECK(cudaGraphInstantiate(&e, g, 0));
    return e;
}

// Adds a WHILE conditional node at the current capture point of `st` and
// returns its body graph; `st` continues after the node.
cudaGraph_t add_while(cudaStream_t st, cudaGraphConditionalHandle* h, unsigned dflt) {
    cudaStreamCaptureStatus status;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    IRK_CUDA_CHECK(cudaStreamGetCaptureInfo(st, &status, nullptr, &cg, &deps, &ndeps));
    IRK_CUDA_CHECK(cudaGraphConditionalHandleCreate(h, cg, dflt, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = *h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    IRK_CUDA_CHECK(cudaGraphAddNode(&node, cg, deps, ndeps, &p));
    IRK_CUDA_CHECK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    return p.conditional.phGraph_out[0];
}

// Kernel nodes of a graph (memset / conditional nodes excluded).
int count_nodes(cudaGraph_t g) {
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    if (n) cudaGraphGetNodes(g, nodes.data(), &n);
    int k = 0;
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
}

// Kernel launches recorded by fn, counted from a throw-away capture.
// With `t`, also tallies the recorded kernels' algorithmic bytes.
template <class F>
int count_launches(cudaStream_t st, F&& fn, dev::Tally* t = nullptr) {
    cudaGraph_t g = nullptr;
    IRK_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    dev::tally_open(t);
    try {
        fn();
    } catch (...) {
        dev::tally_close();
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    dev::tally_close();
    IRK_CUDA_CHECK(cudaStreamEndCapture(st, &g));
    const int k = count_nodes(g);
    cudaGraphDestroy(g);
    return k;
}

}  // namespace

void DeviceSolver::build_graph(bool lift, bool forcing, int restart, int max_iter, double rtol,
                               bool use_cond) {
    for (cudaGraphExec_t* e : {&exec_, &exec_iter_, &exec_pre_, &exec_cb_, &exec_ce_, &exec_post_})
        if (*e) {
            cudaGraphExecDestroy(*e);
            *e = nullptr;
        }
    gb_.use_cond = use_cond ? 1 : 0;
    auto pre = [&]() {
        dev::SpmvArgs a;
        a.x = dev::plain(u_);
        a.y = dev::plain(ku_);
        dev::spmv(K_, dev::kXPlain, dev::kEPlain, a, st_);
        dev::stage_rhs_finish(ku_, lift ? lift_ : nullptr, forcing ? forcing_ : nullptr, b_, n_, s_,
                              st_);
        IRK_CUDA_CHECK(cudaMemsetAsync(x_, 0, sizeof(double) * sN_, st_));
        dev::gm_init(gb_, b_, r_, rtol, restart, max_iter, ortho_, side_, st_);
    };
    auto cycle_begin = [&]() {
        if (side_ == 0) {  // left: the cycle's base vector is P^-1 r (gmres.cpp:41-46)
            record_precond(dev::plain(r_), dev::plain(ax_));
            dev::gm_cycle_begin(gb_, ax_, st_);
        } else {
            dev::gm_cycle_begin(gb_, r_, st_);
        }
    };
    auto cycle_end = [&]() {
        if (ortho_ == 1) dev::gm_dgs_dot(gb_, 1, st_);
        dev::gm_solution(gb_, x_, st_);
        record_stage_op(dev::plain(x_), dev::plain(ax_));
        dev::gm_residual(gb_, b_, ax_, r_, st_);
    };
    auto post = [&]() { dev::irk_update(u_, x_, hb_.data(), n_, s_, unext_, st_); };

    tally_ = {};
    launch_counts_[0] = count_launches(st_, pre, &tally_[0]);
    launch_counts_[1] = count_launches(st_, [&] { cycle_begin(); cycle_end(); }, &tally_[1]);
    launch_counts_[2] = count_launches(st_, [&] { record_iteration(); }, &tally_[2]);
    launch_counts_[3] = count_launches(st_, post, &tally_[3]);
    if (use_cond) {
        cudaStream_t s2 = nullptr, s3 = nullptr;
        IRK_CUDA_CHECK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        IRK_CUDA_CHECK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
        cudaStream_t main = st_;
        cudaGraph_t top = nullptr;
        try {
            IRK_CUDA_CHECK(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
            // The outer handle must exist before the init kernel is recorded.
            cudaGraphConditionalHandle ho;
            {
                cudaStreamCaptureStatus status;
                cudaGraph_t cg = nullptr;
                IRK_CUDA_CHECK(cudaStreamGetCaptureInfo(main, &status, nullptr, &cg, nullptr, nullptr));
                IRK_CUDA_CHECK(cudaGraphConditionalHandleCreate(&ho, cg, 0, 0));
            }
            gb_.h_outer = ho;
            pre();
            // outer WHILE node (handle created above, on the top graph)
            cudaGraph_t outer_body;
            {
                cudaStreamCaptureStatus status;
                cudaGraph_t cg = nullptr;
                const cudaGraphNode_t* deps = nullptr;
                size_t ndeps = 0;
                IRK_CUDA_CHECK(cudaStreamGetCaptureInfo(main, &status, nullptr, &cg, &deps, &ndeps));
                cudaGraphNodeParams p = {};
                p.type = cudaGraphNodeTypeConditional;
                p.conditional.handle = ho;
                p.conditional.type = cudaGraphCondTypeWhile;
                p.conditional.size = 1;
                cudaGraphNode_t node;
                IRK_CUDA_CHECK(cudaGraphAddNode(&node, cg, deps, ndeps, &p));
                IRK_CUDA_CHECK(cudaStreamUpdateCaptureDependencies(main, &node, 1, cudaStreamSetCaptureDependencies));
                outer_body = p.conditional.phGraph_out[0];
            }
            // outer body: cycle begin -> inner WHILE -> cycle end
            st_ = s2;
            IRK_CUDA_CHECK(cudaStreamBeginCaptureToGraph(s2, outer_body, nullptr, nullptr, 0,
                                                         cudaStreamCaptureModeThreadLocal));
            cudaGraphConditionalHandle hi;
            {
                cudaStreamCaptureStatus status;
                cudaGraph_t cg = nullptr;
                IRK_CUDA_CHECK(cudaStreamGetCaptureInfo(s2, &status, nullptr, &cg, nullptr, nullptr));
                IRK_CUDA_CHECK(cudaGraphConditionalHandleCreate(&hi, cg, 0, 0));
            }
            gb_.h_inner = hi;
            cycle_begin();
            cudaGraph_t inner_body;
            {
                cudaStreamCaptureStatus status;
                cudaGraph_t cg = nullptr;
                const cudaGraphNode_t* deps = nullptr;
                size_t ndeps = 0;
                IRK_CUDA_CHECK(cudaStreamGetCaptureInfo(s2, &status, nullptr, &cg, &deps, &ndeps));
                cudaGraphNodeParams p = {};
                p.type = cudaGraphNodeTypeConditional;
                p.conditional.handle = hi;
                p.conditional.type = cudaGraphCondTypeWhile;
                p.conditional.size = 1;
                cudaGraphNode_t node;
                IRK_CUDA_CHECK(cudaGraphAddNode(&node, cg, deps, ndeps, &p));
                IRK_CUDA_CHECK(cudaStreamUpdateCaptureDependencies(s2, &node, 1, cudaStreamSetCaptureDependencies));
                inner_body = p.conditional.phGraph_out[0];
            }
            st_ = s3;
            IRK_CUDA_CHECK(cudaStreamBeginCaptureToGraph(s3, inner_body, nullptr, nullptr, 0,
                                                         cudaStreamCaptureModeThreadLocal));
            record_iteration();
            IRK_CUDA_CHECK(cudaStreamEndCapture(s3, &inner_body));
            launches_per_iter_ = count_nodes(inner_body);
            st_ = s2;
            cycle_end();
            IRK_CUDA_CHECK(cudaStreamEndCapture(s2, &outer_body));
            st_ = main;
            post();
            IRK_CUDA_CHECK(cudaStreamEndCapture(main, &top));
        } catch (...) {
            // leave no stream in capture mode and the solver on its own stream
            st_ = main;
            for (cudaStream_t x : {s3, s2, main}) {
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                if (cudaStreamIsCapturing(x, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
                    cudaGraph_t junk = nullptr;
                    cudaStreamEndCapture(x, &junk);
                    if (junk) cudaGraphDestroy(junk);
                }
            }
            cudaGetLastError();
            cudaStreamDestroy(s2);
            cudaStreamDestroy(s3);
            throw;
        }
        exec_ = instantiate(top);
        cudaGraphDestroy(top);
        cudaStreamDestroy(s2);
        cudaStreamDestroy(s3);
    } else {
        auto cap = [&](auto&& fn) {
            cudaGraph_t g = nullptr;
            IRK_CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
            fn();
            IRK_CUDA_CHECK(cudaStreamEndCapture(st_, &g));
            return g;
        };
        cudaGraph_t g;
        g = cap(pre); exec_pre_ = instantiate(g); cudaGraphDestroy(g);
        g = cap(cycle_begin); exec_cb_ = instantiate(g); cudaGraphDestroy(g);
        g = cap([&] { record_iteration(); });
        launches_per_iter_ = count_nodes(g);
        exec_iter_ = instantiate(g); cudaGraphDestroy(g);
        g = cap(cycle_end); exec_ce_ = instantiate(g); cudaGraphDestroy(g);
        g = cap(post); exec_post_ = instantiate(g); cudaGraphDestroy(g);
    }
    graph_mode_ = use_cond ? 1 : 0;
    g_lift_ = lift;
    g_forcing_ = forcing;
    g_side_ = side_;
    g_restart_ = restart;
    g_iter_ = max_iter;
    g_rtol_ = rtol;
}

SolveReport DeviceSolver::report_from(const dev::GmresCtl& c, const double* hist, int max_iter) {
    SolveReport rep;
    rep.iterations = c.total;
    rep.cycles = c.cycles;
    rep.n_reorth = c.n_reorth;
    rep.converged = c.converged;
    rep.final_rel = c.final_rel;
    rep.true_rel = c.true_rel;
    if (hist) {
        const int len = std::min(c.total, max_iter) + 1;
        rep.history.assign(hist, hist + len);
    }
    return rep;
}

int DeviceSolver::prepare(const GmresConfig& cfg, bool lift, bool forcing) {
    check(cfg.rel_tol > 0.0, "gmres: rel_tol must be positive");
    check(cfg.side == 0 || cfg.side == 1, "gmres: side must be 0 (left) or 1 (right)");
    if (cfg.side == 0 && ortho_ != 1)
        throw Unsupported("device gmres: left preconditioning runs with the delayed CGS2 scheme only");
    side_ = cfg.side;
    const int max_iter = cfg.max_iter;
    int restart = cfg.restart <= 0 || cfg.restart > max_iter ? max_iter : cfg.restart;
    if (restart < 1) restart = 1;
    ensure_gmres(restart, std::max(max_iter, 1));
    if (forcing && !forcing_) forcing_ = alloc(static_cast<size_t>(s_) * n_);
    // IRK_NO_COND_GRAPH=1 (environment or irk_set_option): host-driven loop
    // over plain graphs, whose kernels profilers can see
    const bool want_cond = dev::option("IRK_NO_COND_GRAPH", 0) == 0;
    if (g_restart_ != restart || g_iter_ != max_iter || g_rtol_ != cfg.rel_tol ||
        g_lift_ != lift || g_forcing_ != forcing || g_side_ != side_ ||
        (graph_mode_ == 1) != want_cond || g_opt_gen_ != dev::option_generation()) {
        g_opt_gen_ = dev::option_generation();
        bool ok = false;
        if (want_cond) {
            try {
                build_graph(lift, forcing, restart, max_iter, cfg.rel_tol, true);
                ok = true;
            } catch (const CudaError&) {
                cudaGetLastError();
                cudaStreamCaptureStatus stc;
                if (cudaStreamIsCapturing(st_, &stc) == cudaSuccess && stc != cudaStreamCaptureStatusNone) {
                    cudaGraph_t junk;
                    cudaStreamEndCapture(st_, &junk);
                }
            }
        }
        if (!ok) build_graph(lift, forcing, restart, max_iter, cfg.rel_tol, false);
    }
    return max_iter;
}

void DeviceSolver::launch_solve() {
    if (graph_mode_ == 1) {
        IRK_CUDA_CHECK(cudaGraphLaunch(exec_, st_));
        return;
    }
    IRK_CUDA_CHECK(cudaGraphLaunch(exec_pre_, st_));
    IRK_CUDA_CHECK(cudaMemcpyAsync(ctl_host_, gb_.ctl, sizeof(dev::GmresCtl), cudaMemcpyDeviceToHost, st_));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
    while (!ctl_host_->done) {
        IRK_CUDA_CHECK(cudaGraphLaunch(exec_cb_, st_));
        while (true) {
            IRK_CUDA_CHECK(cudaGraphLaunch(exec_iter_, st_));
            IRK_CUDA_CHECK(cudaMemcpyAsync(&ctl_host_->stop, &gb_.ctl->stop, sizeof(int),
                                           cudaMemcpyDeviceToHost, st_));
            IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
            if (ctl_host_->stop != 0) break;
        }
        IRK_CUDA_CHECK(cudaGraphLaunch(exec_ce_, st_));
        IRK_CUDA_CHECK(cudaMemcpyAsync(ctl_host_, gb_.ctl, sizeof(dev::GmresCtl), cudaMemcpyDeviceToHost, st_));
        IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
    }
    IRK_CUDA_CHECK(cudaGraphLaunch(exec_post_, st_));
}

SolveReport DeviceSolver::step(const double* u, const double* lift, const GmresConfig& cfg,
                               double* u_next, double* k_out, const double* forcing) {
    DeviceScope on(device_);
    const int max_iter = prepare(cfg, lift != nullptr, forcing != nullptr);
    const auto t0 = std::chrono::steady_clock::now();
    IRK_CUDA_CHECK(cudaMemcpyAsync(u_, u, sizeof(double) * n_, cudaMemcpyDefault, st_));
    if (lift) IRK_CUDA_CHECK(cudaMemcpyAsync(lift_, lift, sizeof(double) * n_, cudaMemcpyDefault, st_));
    if (forcing)
        IRK_CUDA_CHECK(cudaMemcpyAsync(forcing_, forcing, sizeof(double) * sN_, cudaMemcpyDefault, st_));
    launch_solve();
    if (u_next) IRK_CUDA_CHECK(cudaMemcpyAsync(u_next, unext_, sizeof(double) * n_, cudaMemcpyDefault, st_));
    if (k_out) IRK_CUDA_CHECK(cudaMemcpyAsync(k_out, x_, sizeof(double) * sN_, cudaMemcpyDefault, st_));
    IRK_CUDA_CHECK(cudaMemcpyAsync(ctl_host_, gb_.ctl, sizeof(dev::GmresCtl), cudaMemcpyDeviceToHost, st_));
    IRK_CUDA_CHECK(cudaMemcpyAsync(hist_host_, gb_.hist, sizeof(double) * (max_iter + 1),
                                   cudaMemcpyDeviceToHost, st_));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
    SolveReport rep = report_from(*ctl_host_, hist_host_, max_iter);
    rep.solve_seconds = seconds_since(t0);
    return rep;
}

SolveReport DeviceSolver::step_host(const double* u, const double* lift, const GmresConfig& cfg,
                                    double* u_next, double* k_out, const double* forcing) {
    // cudaMemcpyDefault handles pageable or pinned host pointers.
    return step(u, lift, cfg, u_next, k_out, forcing);
}

// ------------------------------------------------------- device-resident loop
namespace {

// Pinned host block, freed on scope exit.
struct Pinned {
    void* p = nullptr;
    explicit Pinned(size_t bytes) { IRK_CUDA_CHECK(cudaMallocHost(&p, bytes ? bytes : 1)); }
    ~Pinned() { cudaFreeHost(p); }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct Events {
    std::vector<cudaEvent_t> ev;
    explicit Events(size_t k) : ev(k, nullptr) {
        for (auto& e : ev) IRK_CUDA_CHECK(cudaEventCreate(&e));
    }
    ~Events() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

}  // namespace

void DeviceSolver::load_u(const double* u0) {
    DeviceScope on(device_);
    IRK_CUDA_CHECK(cudaMemcpyAsync(u_, u0, sizeof(double) * n_, cudaMemcpyDefault, st_));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
}

void DeviceSolver::store_u(double* dst) {
    DeviceScope on(device_);
    IRK_CUDA_CHECK(cudaMemcpyAsync(dst, u_, sizeof(double) * n_, cudaMemcpyDefault, st_));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
}

std::vector<SolveReport> DeviceSolver::run_segment(int nsteps, double* t, const double* lift,
                                                   ForcingFn forcing, void* user, const double* c,
                                                   const GmresConfig& cfg, bool want_history) {
    DeviceScope on(device_);
    check(nsteps >= 0, "integrate: negative step count");
    check(!forcing || c, "integrate: forcing needs the stage nodes c");
    const int max_iter = prepare(cfg, lift != nullptr, forcing != nullptr);
    if (lift) IRK_CUDA_CHECK(cudaMemcpyAsync(lift_, lift, sizeof(double) * n_, cudaMemcpyDefault, st_));
    const size_t hl = static_cast<size_t>(max_iter) + 1;
    Pinned ctl(sizeof(dev::GmresCtl) * nsteps);
    Pinned hist(want_history ? sizeof(double) * hl * nsteps : 0);
    Pinned stage(forcing ? sizeof(double) * 2 * sN_ : 0);
    Events ev(2 * static_cast<size_t>(nsteps) + 2);
    cudaEvent_t* staged = ev.ev.data() + 2 * nsteps;  // H2D of staging buffer k%2 done
    bool staged_used[2] = {false, false};
    for (int k = 0; k < nsteps; ++k) {
        if (forcing) {
            double* buf = stage.as<double>() + (k % 2) * sN_;
            if (staged_used[k % 2]) IRK_CUDA_CHECK(cudaEventSynchronize(staged[k % 2]));
            for (int i = 0; i < s_; ++i) {
                // sys.forcing(t_n + c_i ht), irk.cpp:26
                const int rc = forcing(*t + c[i] * ht_, buf + static_cast<long long>(i) * n_, n_, user);
                check(rc == 0, "stage_rhs: forcing callback failed");
            }
            IRK_CUDA_CHECK(cudaMemcpyAsync(forcing_, buf, sizeof(double) * sN_, cudaMemcpyHostToDevice, st_));
            IRK_CUDA_CHECK(cudaEventRecord(staged[k % 2], st_));
            staged_used[k % 2] = true;
        }
        IRK_CUDA_CHECK(cudaEventRecord(ev.ev[2 * k], st_));
        launch_solve();
        IRK_CUDA_CHECK(cudaEventRecord(ev.ev[2 * k + 1], st_));
        // u_n <- u_{n+1} stays on the device (irk.cpp:95)
        IRK_CUDA_CHECK(cudaMemcpyAsync(u_, unext_, sizeof(double) * n_, cudaMemcpyDeviceToDevice, st_));
        IRK_CUDA_CHECK(cudaMemcpyAsync(ctl.as<dev::GmresCtl>() + k, gb_.ctl, sizeof(dev::GmresCtl),
                                       cudaMemcpyDeviceToHost, st_));
        if (want_history)
            IRK_CUDA_CHECK(cudaMemcpyAsync(hist.as<double>() + hl * k, gb_.hist, sizeof(double) * hl,
                                           cudaMemcpyDeviceToHost, st_));
        *t += ht_;  // t += step (irk.cpp:97)
    }
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
    std::vector<SolveReport> out;
    out.reserve(nsteps);
    for (int k = 0; k < nsteps; ++k) {
        SolveReport r = report_from(ctl.as<dev::GmresCtl>()[k],
                                    want_history ? hist.as<double>() + hl * k : nullptr, max_iter);
        float ms = 0.f;
        IRK_CUDA_CHECK(cudaEventElapsedTime(&ms, ev.ev[2 * k], ev.ev[2 * k + 1]));
        r.solve_seconds = ms * 1e-3;
        out.push_back(std::move(r));
    }
    return out;
}

void DeviceSolver::stage_apply(const double* v, double* y) {
    DeviceScope on(device_);
    record_stage_op(dev::plain(v), dev::plain(y));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
}

void DeviceSolver::precond_apply(const double* v, double* w) {
    DeviceScope on(device_);
    record_precond(dev::plain(v), dev::plain(w));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
}

void DeviceSolver::vcycle(int k, const double* r, double* z) {
    DeviceScope on(device_);
    check(k >= 0 && k < static_cast<int>(hier_.size()), "vcycle: hierarchy index out of range");
    record_vcycle(k, dev::plain(r), dev::plain(z));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
}

double DeviceSolver::dot(const double* x, const double* y, long long n) {
    DeviceScope on(device_);
    const long long nch = (n + dev::kChunk - 1) / dev::kChunk;
    DevBuf part(sizeof(double) * std::max<long long>(nch, 1));
    dev::dot(x, y, n, part.as<double>(), red_cnt_, red_out_, st_);
    double out = 0.0;
    IRK_CUDA_CHECK(cudaMemcpyAsync(&out, red_out_, sizeof(double), cudaMemcpyDeviceToHost, st_));
    IRK_CUDA_CHECK(cudaStreamSynchronize(st_));
    return out;
}

namespace {
__global__ void k_empty() {}
}  // namespace

double DeviceSolver::time_kernel(int which, int reps) {
    DeviceScope on(device_);
    if (which >= 100 && which < 100 + 2 * dev::kMaxRestart) {
        // GMRES block-dot with j = which - 100 (CGS pass 1) or which - 600
        // (DCGS2 block-dot): j+2 vectors of sN streamed
        const bool dgs = which >= 600;
        const int j = dgs ? which - 600 : which - 100;
        ensure_gmres(std::max(50, j + 2), 500);
        IRK_CUDA_CHECK(cudaMemsetAsync(gb_.V, 0, sizeof(double) * stride_ * (j + 2), st_));
        IRK_CUDA_CHECK(cudaMemcpyAsync(&gb_.ctl->j, &j, sizeof(int), cudaMemcpyHostToDevice, st_));
        const int zero = 0;
        IRK_CUDA_CHECK(cudaMemcpyAsync(&gb_.ctl->reorth, &zero, sizeof(int), cudaMemcpyHostToDevice, st_));
        gb_.use_cond = 0;
        auto launch_once = [&]() {
            if (dgs)
                dev::gm_dgs_dot(gb_, 0, st_);
            else
                dev::gm_blockdot(gb_, 1, st_);
        };
        launch_once();
        cudaEvent_t e0, e1;
        IRK_CUDA_CHECK(cudaEventCreate(&e0));
        IRK_CUDA_CHECK(cudaEventCreate(&e1));
        IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
        for (int i = 0; i < reps; ++i) launch_once();
        IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
        IRK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        g_restart_ = -1;  // graphs captured the old use_cond; rebuild on the next step
        if (std::getenv("IRK_DGS_PROF_PRINT")) {
            long long t[8];
            dev::dgs_prof_read(t);
            std::fprintf(stderr, "dgs dot (last launch, ns from CTA 0 start): last CTA arrives %lld, elected %lld, "
                         "reduced %lld, scalars done %lld\n", t[0] - t[4], t[1] - t[4], t[2] - t[4], t[3] - t[4]);
        }
        return static_cast<double>(ms) / reps;
    }
    if (which >= 60 && which < 80) {
        // Gauss-Seidel sweep of hierarchy 0, level (which - 60) / 2, forward
        // (even) or backward (odd), on the level's work vectors
        DevHier& H = hier_[0];
        const int l = (which - 60) / 2;
        const bool back = (which - 60) % 2 == 1;
        check(H.prm.smoother != 0 && l + 1 < static_cast<int>(H.lv.size()),
              "time_kernel: no Gauss-Seidel sweep at that level");
        DevLevel& d = H.lv[l];
        const double* rr = l == 0 ? d.t : d.r;
        dev::GsSweep S = back ? d.gsb : d.gsf;
        DevBuf prof(std::getenv("IRK_GS_PROF") ? 5 * 64 * sizeof(long long) : 0);
        if (prof.bytes()) {
            IRK_CUDA_CHECK(cudaMemset(prof.as<void>(), 0, prof.bytes()));
            S.prof = prof.as<long long>();
        }
        auto once = [&]() { dev::gs_sweep(S, back, dev::plain(rr), d.u, dev::plain(d.zp), st_); };
        IRK_CUDA_CHECK(cudaMemsetAsync(d.u, 0, sizeof(double) * d.n, st_));
        once();
        cudaEvent_t e0, e1;
        IRK_CUDA_CHECK(cudaEventCreate(&e0));
        IRK_CUDA_CHECK(cudaEventCreate(&e1));
        IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
        for (int i = 0; i < reps; ++i) once();
        IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
        IRK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (prof.bytes()) {
            std::vector<long long> h(5 * 64);
            IRK_CUDA_CHECK(cudaMemcpy(h.data(), prof.as<void>(), prof.bytes(), cudaMemcpyDeviceToHost));
            double a[5] = {0, 0, 0, 0, 0};
            for (int c = 1; c < 64; ++c)
                for (int k = 0; k < 5; ++k) a[k] += static_cast<double>(h[5 * c + k]) / 63.0;
            std::fprintf(stderr, "gs sweep L%d %s: cycles per chunk (thread 0, 63 sampled chunks, mean "
                         "%.0f rows) phase clocks %.0f / %.0f / %.0f / %.0f (ws: chunk ready, "
                         "rows done, consumer barrier)\n", l, back ? "bwd" : "fwd", a[4], a[0], a[1], a[2], a[3]);
        }
        return static_cast<double>(ms) / reps;
    }
    if (which == 50 || which == 51) {
        // bottom kernel of hierarchy 0 back to back (50), or alternating with
        // the level-1 smoother SpMV (51: forces the shared-memory carveout to
        // switch between launches)
        DevHier& H = hier_[0];
        check(H.bot_from > 0, "time_kernel: hierarchy 0 has no bottom kernel");
        DevBuf prof(16 * sizeof(long long));
        const bool want_prof = std::getenv("IRK_BOT_PROF") != nullptr;
        if (want_prof) {
            IRK_CUDA_CHECK(cudaMemset(prof.as<void>(), 0, 16 * sizeof(long long)));
            H.bot.prof = prof.as<long long>();
        }
        cudaGraph_t gr;
        IRK_CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
        for (int r = 0; r < reps; ++r) {
            dev::bottom_cycle(H.bot, H.lv[H.bot_from].r, H.lv[H.bot_from].z, st_);
            if (which == 51) {
                dev::SpmvArgs a;
                a.x = dev::plain(H.lv[1].t);
                a.r = dev::plain(H.lv[1].r);
                a.wd = H.lv[1].wd;
                a.y = dev::plain(H.lv[1].u);
                dev::spmv(H.lv[1].A, dev::kXPlain, dev::kESmooth, a, st_);
            }
        }
        IRK_CUDA_CHECK(cudaStreamEndCapture(st_, &gr));
        cudaGraphExec_t ge;
        IRK_CUDA_CHECK(cudaGraphInstantiate(&ge, gr, 0));
        cudaGraphDestroy(gr);
        IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        cudaEvent_t e0, e1;
        IRK_CUDA_CHECK(cudaEventCreate(&e0));
        IRK_CUDA_CHECK(cudaEventCreate(&e1));
        IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
        IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
        IRK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGraphExecDestroy(ge);
        if (want_prof) {
            long long t[16];
            IRK_CUDA_CHECK(cudaMemcpy(t, prof.as<void>(), sizeof(t), cudaMemcpyDeviceToHost));
            std::fprintf(stderr, "bottom phases (ns from start):");
            for (int q = 1; q < 16 && t[q]; ++q) std::fprintf(stderr, " %lld", t[q] - t[0]);
            std::fprintf(stderr, "\n");
            H.bot.prof = nullptr;
        }
        return static_cast<double>(ms) / reps;
    }
    if (which >= 30 && which < 40) {
        // graph-captured repetitions of the V-cycle below level which-30
        DevBuf a(sizeof(double) * stride_), b(sizeof(double) * stride_);
        IRK_CUDA_CHECK(cudaMemsetAsync(a.as<void>(), 0, sizeof(double) * stride_, st_));
        const int first = std::min<int>(which - 30, static_cast<int>(hier_[0].lv.size()) - 1);
        cudaGraph_t gr;
        IRK_CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
        for (int r = 0; r < reps; ++r)
            record_vcycle(0, dev::plain(a.as<double>()), dev::plain(b.as<double>()), first);
        IRK_CUDA_CHECK(cudaStreamEndCapture(st_, &gr));
        cudaGraphExec_t ge;
        IRK_CUDA_CHECK(cudaGraphInstantiate(&ge, gr, 0));
        cudaGraphDestroy(gr);
        IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        cudaEvent_t e0, e1;
        IRK_CUDA_CHECK(cudaEventCreate(&e0));
        IRK_CUDA_CHECK(cudaEventCreate(&e1));
        IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
        IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
        IRK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaGraphExecDestroy(ge);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return static_cast<double>(ms) / reps;
    }
    if (which == 40) {
        // graph-captured dense tail matvecs, cycling through the hierarchies
        DevBuf a(sizeof(double) * stride_), b(sizeof(double) * stride_);
        IRK_CUDA_CHECK(cudaMemsetAsync(a.as<void>(), 0, sizeof(double) * stride_, st_));
        std::vector<int> ks;
        for (int k = 0; k < static_cast<int>(hier_.size()); ++k)
            if (hier_[k].tail) ks.push_back(k);
        if (ks.empty()) return 0.0;
        cudaGraph_t gr;
        IRK_CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
        for (int r = 0; r < reps; ++r) {
            const DevHier& H = hier_[ks[r % ks.size()]];
            dev::tail_mv(H.lv[H.tail_from].n, H.tail_ld, H.tail, a.as<double>(), b.as<double>(), st_);
        }
        IRK_CUDA_CHECK(cudaStreamEndCapture(st_, &gr));
        cudaGraphExec_t ge;
        IRK_CUDA_CHECK(cudaGraphInstantiate(&ge, gr, 0));
        cudaGraphDestroy(gr);
        IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        cudaEvent_t e0, e1;
        IRK_CUDA_CHECK(cudaEventCreate(&e0));
        IRK_CUDA_CHECK(cudaEventCreate(&e1));
        IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
        IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
        IRK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaGraphExecDestroy(ge);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return static_cast<double>(ms) / reps;
    }
    if (which == 20 || which == 21) {
        // launch floor: 100 dependent empty kernels, graph (20) or stream (21)
        cudaEvent_t e0, e1;
        IRK_CUDA_CHECK(cudaEventCreate(&e0));
        IRK_CUDA_CHECK(cudaEventCreate(&e1));
        cudaGraphExec_t ge = nullptr;
        if (which == 20) {
            cudaGraph_t g;
            IRK_CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
            for (int i = 0; i < 100; ++i) k_empty<<<1, 32, 0, st_>>>();
            IRK_CUDA_CHECK(cudaStreamEndCapture(st_, &g));
            IRK_CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
            cudaGraphDestroy(g);
            IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
        }
        IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
        for (int r = 0; r < reps; ++r) {
            if (ge)
                IRK_CUDA_CHECK(cudaGraphLaunch(ge, st_));
            else
                for (int i = 0; i < 100; ++i) k_empty<<<1, 32, 0, st_>>>();
        }
        IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
        IRK_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ge) cudaGraphExecDestroy(ge);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return static_cast<double>(ms) / (reps * 100.0);
    }
    DevBuf a(sizeof(double) * stride_), b(sizeof(double) * stride_);
    IRK_CUDA_CHECK(cudaMemsetAsync(a.as<void>(), 0, sizeof(double) * stride_, st_));
    auto once = [&]() {
        switch (which) {
        case 0: record_stage_op(dev::plain(a.as<double>()), dev::plain(b.as<double>())); break;
        case 1: {
            DevLevel& d = hier_[0].lv[0];
            dev::SpmvArgs sa;
            sa.x = dev::plain(a.as<double>());
            sa.r = dev::plain(a.as<double>());
            sa.wd = d.wd;
            sa.y = dev::plain(b.as<double>());
            dev::spmv(d.A, dev::kXPlain, dev::kESmooth, sa, st_);
            break;
        }
        case 2: record_precond(dev::plain(a.as<double>()), dev::plain(b.as<double>())); break;
        case 3: record_vcycle(0, dev::plain(a.as<double>()), dev::plain(b.as<double>())); break;
        case 7:
        case 8: {
            // the composed level-0 legs alone: r_1 = G_0 r (7), z = U_0 [r; z_1] (8)
            DevLevel& d = hier_[0].lv[0];
            check(d.G.rows > 0, "time_kernel: hierarchy 0 is not composed");
            dev::SpmvArgs sa;
            sa.x = dev::plain(a.as<double>());
            if (which == 7) {
                sa.y = dev::plain(hier_[0].lv[1].r);
                dev::spmv(d.G, dev::kXPlain, dev::kEPlain, sa, st_);
            } else {
                sa.x2 = dev::plain(hier_[0].lv[1].z);
                sa.split = d.n;
                sa.y = dev::plain(b.as<double>());
                if (d.up_cls)
                    dev::up_cls(d.US, d.UQ, sa, st_);
                else
                    dev::spmv(d.U, dev::kXSplit, dev::kEPlain, sa, st_);
            }
            break;
        }
        default: {  // 4, 5, ...: the V-cycle below level which-3
            const int first = std::min<int>(which - 3, static_cast<int>(hier_[0].lv.size()) - 1);
            record_vcycle(0, dev::plain(a.as<double>()), dev::plain(b.as<double>()), first);
            break;
        }
        }
    };
    {
        // algorithmic bytes of one application (stored formats), for the roofline
        dev::Tally t{};
        dev::tally_open(&t);
        once();
        dev::tally_close();
        last_timed_bytes_ = t.fixed;
    }
    cudaEvent_t e0, e1;
    IRK_CUDA_CHECK(cudaEventCreate(&e0));
    IRK_CUDA_CHECK(cudaEventCreate(&e1));
    IRK_CUDA_CHECK(cudaEventRecord(e0, st_));
    for (int i = 0; i < reps; ++i) once();
    IRK_CUDA_CHECK(cudaEventRecord(e1, st_));
    IRK_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return static_cast<double>(ms) / reps;
}

}  // namespace irkb
