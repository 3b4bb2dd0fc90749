// Coarse tail of the AMG V-cycle in ONE launch ("bottom solver").
//
// Default: a single CTA of 1024 threads takes the levels with <= 512 rows
// plus the dense coarsest solve (5 launches per V-cycle at C2 become one).
// A 16-CTA cluster variant (IRK_TAIL_CLUSTER=1) was measured slower on B200:
// with tens of thousands of rows the phases are DRAM-latency bound and 70% of
// the warps' stall cycles were spent at the cluster barriers
// (profiles/r1/ncu_tail_cluster.txt).
//
// Below a few tens of thousands of rows every V-cycle phase (residual,
// restriction, coarse solve, prolongation, post-smoothing) is pure latency:
// as separate launches the coarse levels cost ~13 launches of a few
// microseconds each per V-cycle.  Here a thread-block cluster (16 CTAs x 1024
// threads, one GPC) runs all phases of levels >= Lc back to back, separated
// by cluster barriers (barrier.cluster, which also invalidates L1 so the
// next phase reads the other CTAs' results from L2).
//
// Row sums keep the reference's order: G lanes load a row's entries at once,
// then the products are added sequentially in column order through warp
// shuffles, exactly like k_spmv_csrv -- so the tail is bit-identical to the
// per-level kernels and to the oracle.
#include <cooperative_groups.h>

#include <string>

#include "../host/sparse.hpp"
#include "coarse_tail.cuh"

namespace cg = cooperative_groups;

namespace irkb {
namespace dev {
namespace {

__device__ __forceinline__ double tail_val(const TailCsr& A, int k) {
    switch (A.vf) {
    case kU8: return __ldg(A.tab + __ldg(static_cast<const unsigned char*>(A.val) + k));
    case kU16: return __ldg(A.tab + __ldg(static_cast<const unsigned short*>(A.val) + k));
    default: return __ldg(static_cast<const double*>(A.val) + k);
    }
}

// Sequential (column-order) row sum of A(row,:) . x with G lanes per row.
// XM = 1: x_c = wd[c] * r[c].  All 32 lanes of the warp must call this with
// warp-uniform control flow.
template <int G, int XM>
__device__ __forceinline__ double row_sum(const TailCsr& A, int row, bool live, int lane,
                                          const double* x, const double* wd, const double* r) {
    constexpr int MM = 4;
    const int lo = live ? __ldg(A.ptr + row) : 0;
    const int len = live ? __ldg(A.ptr + row + 1) - lo : 0;
    int chunks = (len + G * MM - 1) / (G * MM);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) chunks = max(chunks, __shfl_xor_sync(0xffffffffu, chunks, o));
    double s = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
        double p[MM];
#pragma unroll
        for (int m = 0; m < MM; ++m) {
            const int k = ch * G * MM + m * G + lane;
            p[m] = 0.0;
            if (k < len) {
                const int c = __ldg(A.idx + lo + k);
                const double xv = XM ? wd[c] * r[c] : x[c];
                p[m] = tail_val(A, lo + k) * xv;
            }
        }
#pragma unroll
        for (int m = 0; m < MM; ++m)
#pragma unroll
            for (int l = 0; l < G; ++l) {
                const double v = __shfl_sync(0xffffffffu, p[m], l, G);
                if (ch * G * MM + m * G + l < len) s += v;
            }
    }
    return s;
}

// Dense coarse row: sum_j Ainv[row, j] r[j] in j order.
template <int G>
__device__ __forceinline__ double dense_row(const double* Ainv, int n, int row, bool live,
                                            int lane, const double* r) {
    constexpr int MM = 4;
    const int chunks = (n + G * MM - 1) / (G * MM);
    double s = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
        double p[MM];
#pragma unroll
        for (int m = 0; m < MM; ++m) {
            const int k = ch * G * MM + m * G + lane;
            p[m] = (live && k < n) ? Ainv[static_cast<long long>(row) * n + k] * r[k] : 0.0;
        }
#pragma unroll
        for (int m = 0; m < MM; ++m)
#pragma unroll
            for (int l = 0; l < G; ++l) {
                const double v = __shfl_sync(0xffffffffu, p[m], l, G);
                if (ch * G * MM + m * G + l < n) s += v;
            }
    }
    return s;
}

// Distributes rows [0, n) over G-lane groups of the whole cluster.
template <int G, class F>
__device__ __forceinline__ void for_rows(int n, F&& f) {
    const int gt = cg::this_cluster().block_rank() * blockDim.x + threadIdx.x;
    const int total = cg::this_cluster().num_blocks() * blockDim.x;
    const int group = gt / G, lane = gt % G, ngroups = total / G;
    for (int base = 0; base < n; base += ngroups) {
        const int row = base + group;
        f(row, row < n, lane);
    }
}

// Phase barrier: a single CTA (the bottom solver) only needs __syncthreads.
struct PhaseSync {
    cg::cluster_group cl;
    bool single;
    __device__ void operator()() {
        if (single)
            __syncthreads();
        else
            cl.sync();
    }
};

__global__ void __launch_bounds__(1024) k_coarse_tail(const __grid_constant__ TailArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    PhaseSync cl{cg::this_cluster(), cg::this_cluster().num_blocks() == 1};
    const int L = a.nlev;
    auto rhs = [&](int l) -> const double* { return l == 0 ? a.r0.get() : a.lv[l].r; };
    // down: residual of the pre-smoothed iterate, restriction
    for (int l = 0; l + 1 < L; ++l) {
        const TailLevel& v = a.lv[l];
        const double* r = rhs(l);
        for_rows<4>(v.n, [&](int row, bool live, int lane) {
            const double s = row_sum<4, 1>(v.A, row, live, lane, nullptr, v.wd, r);
            if (live && lane == 0) v.t[row] = r[row] - s;
        });
        cl();
        double* rc = a.lv[l + 1].r;
        for_rows<8>(a.lv[l + 1].n, [&](int row, bool live, int lane) {
            const double s = row_sum<8, 0>(v.R, row, live, lane, v.t, nullptr, nullptr);
            if (live && lane == 0) rc[row] = s;
        });
        cl();
    }
    // coarsest direct solve
    {
        const double* r = rhs(L - 1);
        double* z = L == 1 ? a.z0.get() : a.lv[L - 1].z;
        for_rows<8>(a.nc, [&](int row, bool live, int lane) {
            const double s = dense_row<8>(a.cinv, a.nc, row, live, lane, r);
            if (live && lane == 0) z[row] = s;
        });
        cl();
    }
    // up: prolongation + correction, post-smoothing sweep
    for (int l = L - 2; l >= 0; --l) {
        const TailLevel& v = a.lv[l];
        const double* r = rhs(l);
        const double* zc = a.lv[l + 1].z;
        for_rows<4>(v.n, [&](int row, bool live, int lane) {
            const double s = row_sum<4, 0>(v.P, row, live, lane, zc, nullptr, nullptr);
            if (live && lane == 0) v.t[row] = v.wd[row] * r[row] + s;
        });
        cl();
        double* z = l == 0 ? a.z0.get() : v.z;
        for_rows<4>(v.n, [&](int row, bool live, int lane) {
            const double s = row_sum<4, 0>(v.A, row, live, lane, v.t, nullptr, nullptr);
            if (live && lane == 0) z[row] = v.t[row] + v.wd[row] * (r[row] - s);
        });
        if (l > 0) cl();
    }
}

int g_cluster = 0;  // 0 = not probed

}  // namespace

int coarse_tail_cluster_size() {
    if (g_cluster) return g_cluster;
    cudaFuncSetAttribute(k_coarse_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int best = 0;
    for (int cs : {16, 8, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(1024);
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = cs;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k_coarse_tail, &cfg) == cudaSuccess &&
            nclusters > 0) {
            best = cs;
            break;
        }
        cudaGetLastError();
    }
    g_cluster = best > 0 ? best : -1;
    return g_cluster;
}

void coarse_tail(const TailArgs& a, int cluster, cudaStream_t st) {
    const int cs = cluster > 1 ? coarse_tail_cluster_size() : 1;
    if (cs <= 0) throw CudaError("coarse tail: no cluster launch configuration available");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(1024);
    cfg.stream = st;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cs;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cudaLaunchAttribute attrs[2];
    int na = 0;
    if (cs > 1) attrs[na++] = at;
    if (pdl_enabled()) {
        attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    IRK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_coarse_tail, a));
}

}  // namespace dev
}  // namespace irkb
