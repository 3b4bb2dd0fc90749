// Fused coarse-level V-cycle kernels (levels with few rows).
//
// On the coarse levels every V-cycle phase is a few microseconds of launch and
// dependency latency around almost no work (profiles/r1/phases_v7.txt).  These
// kernels halve the number of launches per coarse level by recomputing the
// intermediate vector on the fly instead of materialising it:
//
//   down:  rc_J = sum_i R_Ji t_i,  t_i = r_i - sum_k A_ik (wd_k r_k)
//          (pre-smooth from zero + residual + restriction, amg.cpp:153-160)
//   up:    z_i  = t_i + wd_i (r_i - sum_k A_ik t_k),  t_k = wd_k r_k + (P zc)_k
//          (prolongation + correction + post-smoothing, amg.cpp:163-167);
//   On the level above the coarsest, the last CTA of the down kernel (elected
//   by an atomic counter) also applies the dense coarse inverse, so the
//   coarse solve needs no launch of its own.
//
// Every intermediate (t_i, (P zc)_k, zc_J) is evaluated with exactly the
// operation order of the unfused kernels -- sequential column-order sums from
// 0.0 -- so results are bit-identical to them (and to the oracle); only
// redundant work is added (each t is recomputed by every row that needs it),
// which is negligible at these sizes.
#include <string>

#include "../host/sparse.hpp"
#include "amg_fused.cuh"

namespace irkb {
namespace dev {
namespace {

__device__ __forceinline__ double fval(const TailCsr& A, int k) {
    switch (A.vf) {
    case kU8: return __ldg(A.tab + __ldg(static_cast<const unsigned char*>(A.val) + k));
    case kU16: return __ldg(A.tab + __ldg(static_cast<const unsigned short*>(A.val) + k));
    default: return __ldg(static_cast<const double*>(A.val) + k);
    }
}

// t_i = r_i - sum_k A_ik (wd_k r_k), sequential (the kEResid/kXWdR row).
__device__ __forceinline__ double resid_row(const TailCsr& A, const double* wd, const double* r,
                                            int i) {
    const int lo = __ldg(A.ptr + i), hi = __ldg(A.ptr + i + 1);
    double s = 0.0;
#pragma unroll 4
    for (int k = lo; k < hi; ++k) {
        const int c = __ldg(A.idx + k);
        s += fval(A, k) * (wd[c] * r[c]);
    }
    return r[i] - s;
}

// t_k = wd_k r_k + sum_J P_kJ zc_J (the kEProlong row).
__device__ __forceinline__ double prolong_row(const FusedLevel& v, const double* r, int k) {
    const int lo = __ldg(v.P.ptr + k), hi = __ldg(v.P.ptr + k + 1);
    double s = 0.0;
#pragma unroll 4
    for (int e = lo; e < hi; ++e) s += fval(v.P, e) * v.zc[__ldg(v.P.idx + e)];
    return v.wd[k] * r[k] + s;
}

// Lane-parallel row reduction: the G lanes of a group evaluate term(e) for
// the entries of [lo, lo+len) (MM per lane per chunk), then every lane adds
// them in entry order through shuffles.  Warp-uniform control flow required.
template <int G, int MM, class Term>
__device__ __forceinline__ double ordered_sum(int len, int lane, Term&& term) {
    int chunks = (len + G * MM - 1) / (G * MM);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) chunks = max(chunks, __shfl_xor_sync(0xffffffffu, chunks, o));
    double s = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
        double p[MM];
#pragma unroll
        for (int m = 0; m < MM; ++m) {
            const int q = ch * G * MM + m * G + lane;
            p[m] = q < len ? term(q) : 0.0;
        }
#pragma unroll
        for (int m = 0; m < MM; ++m)
#pragma unroll
            for (int l = 0; l < G; ++l) {
                const double val = __shfl_sync(0xffffffffu, p[m], l, G);
                if (ch * G * MM + m * G + l < len) s += val;
            }
    }
    return s;
}

template <int G>
__global__ void __launch_bounds__(256) k_amg_down(const __grid_constant__ FusedLevel v) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = t / G, lane = threadIdx.x % G;
    const bool live = J < v.nrc;
    const double* r = v.r.get();
    const int lo = live ? __ldg(v.R.ptr + J) : 0;
    const int len = live ? __ldg(v.R.ptr + J + 1) - lo : 0;
    const double s = ordered_sum<G, 2>(len, lane, [&](int q) {
        const int i = __ldg(v.R.idx + lo + q);
        return fval(v.R, lo + q) * resid_row(v.A, v.wd, r, i);
    });
    if (live && lane == 0) v.rc[J] = s;
    if (!v.cinv) return;
    // coarsest solve by the last CTA to finish: zc = Ainv rc (k_dense_mv rows)
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(v.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int row = threadIdx.x; row < v.nc; row += blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < v.nc; ++j)
            acc += v.cinv[static_cast<long long>(row) * v.nc + j] * __ldcg(v.rc + j);
        v.zcw[row] = acc;
    }
    if (threadIdx.x == 0) *v.counter = 0u;
}

template <int G>
__global__ void __launch_bounds__(256) k_amg_up(const __grid_constant__ FusedLevel v) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = t / G, lane = threadIdx.x % G;
    const bool live = i < v.n;
    const double* r = v.r.get();
    const int lo = live ? __ldg(v.A.ptr + i) : 0;
    const int len = live ? __ldg(v.A.ptr + i + 1) - lo : 0;
    const double s = ordered_sum<G, 1>(len, lane, [&](int q) {
        const int k = __ldg(v.A.idx + lo + q);
        return fval(v.A, lo + q) * prolong_row(v, r, k);
    });
    if (live && lane == 0) {
        const double ti = prolong_row(v, r, i);
        v.z.get()[i] = ti + v.wd[i] * (r[i] - s);
    }
}

inline int blocks(long long threads) { return static_cast<int>((threads + 255) / 256); }

}  // namespace

void amg_down_fused(const FusedLevel& v, cudaStream_t st) {
    k_amg_down<32><<<blocks(static_cast<long long>(v.nrc) * 32), 256, 0, st>>>(v);
}

void amg_up_fused(const FusedLevel& v, cudaStream_t st) {
    k_amg_up<16><<<blocks(static_cast<long long>(v.n) * 16), 256, 0, st>>>(v);
}

}  // namespace dev
}  // namespace irkb
