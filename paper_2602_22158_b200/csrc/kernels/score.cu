// K3/K4 — update-magnitude scorer over FP32 master partitions.
//
// Contract (the reference has no scorer — its numeric anchor is
// the FP64 sum of squared steps in R/src/adamw.cpp:34-45): for module m and
// consecutive snapshots A=S_p, B=S_{p+1},
//     s_delta = sum (double(B) - double(A))^2,   s_ref = sum double(A)^2,
// over every master element of m's groups; score = sqrt(s_delta)/sqrt(s_ref).
// Shard padding is zero in every snapshot, so whole rank chunks can be summed.
//
// K3 reads each snapshot once (K snapshots -> K-1 pairs in one sweep) with
// 128-bit non-allocating loads, accumulates FP64 per thread, reduces with warp
// shuffles and a fixed warp order, and writes one partial per tile (no
// atomics). K4 sums each module's tile partials in a fixed lane/tree order.
// Results are bitwise reproducible for a given tile table, independent of the
// grid size and of scheduling.
#include <algorithm>

#include "tailor/device.hpp"

namespace tailor::dev {

namespace {

constexpr int kScoreThreads = 256;
constexpr int kWarps = kScoreThreads / 32;

__device__ __forceinline__ float4 ld_nc_f4(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int K>
__device__ __forceinline__ void accumulate(double (&acc)[2 * (K - 1)], const float (&x)[K]) {
#pragma unroll
    for (int p = 0; p < K - 1; ++p) {
        const double a = static_cast<double>(x[p]);
        const double d = static_cast<double>(x[p + 1]) - a;
        acc[2 * p] = fma(d, d, acc[2 * p]);
        acc[2 * p + 1] = fma(a, a, acc[2 * p + 1]);
    }
}

template <int K>
__global__ void __launch_bounds__(kScoreThreads) score_partials_kernel(const ScoreTile* __restrict__ tiles,
                                                                        std::uint32_t ntiles,
                                                                        const float* const* __restrict__ field_base,
                                                                        std::uint32_t nfields, int vec_ok,
                                                                        double* __restrict__ out) {
    constexpr int V = 2 * (K - 1);
    __shared__ double red[kWarps][V];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (std::uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const ScoreTile tile = tiles[t];
        const float* base[K];
#pragma unroll
        for (int k = 0; k < K; ++k) base[k] = field_base[k * nfields + tile.field] + tile.elem_start;
        double acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.0;
        const std::uint32_t n = tile.count;
        std::uint32_t i0 = 0;
        if (vec_ok) {
            const std::uint32_t n4 = n >> 2;
            for (std::uint32_t i = tid; i < n4; i += kScoreThreads) {
                float4 q[K];
#pragma unroll
                for (int k = 0; k < K; ++k) q[k] = ld_nc_f4(reinterpret_cast<const float4*>(base[k]) + i);
                float x[K];
#pragma unroll
                for (int k = 0; k < K; ++k) x[k] = q[k].x;
                accumulate<K>(acc, x);
#pragma unroll
                for (int k = 0; k < K; ++k) x[k] = q[k].y;
                accumulate<K>(acc, x);
#pragma unroll
                for (int k = 0; k < K; ++k) x[k] = q[k].z;
                accumulate<K>(acc, x);
#pragma unroll
                for (int k = 0; k < K; ++k) x[k] = q[k].w;
                accumulate<K>(acc, x);
            }
            i0 = n4 << 2;
        }
        for (std::uint32_t i = i0 + tid; i < n; i += kScoreThreads) {
            float x[K];
#pragma unroll
            for (int k = 0; k < K; ++k) x[k] = __ldg(base[k] + i);
            accumulate<K>(acc, x);
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double s = warp_sum(acc[v]);
            if (lane == 0) red[warp][v] = s;
        }
        __syncthreads();
        if (tid < V) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s += red[w][tid];
            out[static_cast<std::uint64_t>(t) * V + tid] = s;
        }
        __syncthreads();
    }
}

__global__ void score_combine_kernel(const double* __restrict__ partials, const std::uint32_t* __restrict__ begin, int M,
                                     int P, double* __restrict__ out) {
    const int V = 2 * P;
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= M * V) return;
    const int m = gw / V, v = gw % V;
    double s = 0.0;
    for (std::uint32_t t = begin[m] + lane; t < begin[m + 1]; t += 32) s += partials[static_cast<std::uint64_t>(t) * V + v];
    s = warp_sum(s);
    if (lane == 0) out[(static_cast<std::uint64_t>(v / 2) * M + m) * 2 + (v & 1)] = s;
}

template <int K>
cudaError_t launch_k(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                     std::uint32_t nfields, bool vec_ok, double* d_out, cudaStream_t stream) {
    static int per_sm = 0;
    if (per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score_partials_kernel<K>, kScoreThreads, 0);
        per_sm = std::max(1, per_sm);
    }
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ntiles, static_cast<std::uint64_t>(sm_count()) * per_sm));
    score_partials_kernel<K><<<grid, kScoreThreads, 0, stream>>>(d_tiles, ntiles, d_field_base, nfields, vec_ok ? 1 : 0, d_out);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_score_partials(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                                  std::uint32_t nfields, int K, bool vec_ok, double* d_out, cudaStream_t stream) {
    if (ntiles == 0) return cudaSuccess;
    switch (K) {
#define TG_K(k)                                                                          \
    case k:                                                                              \
        return launch_k<k>(d_tiles, ntiles, d_field_base, nfields, vec_ok, d_out, stream);
        TG_K(2) TG_K(3) TG_K(4) TG_K(5) TG_K(6) TG_K(7) TG_K(8) TG_K(9) TG_K(10) TG_K(11) TG_K(12) TG_K(13) TG_K(14)
            TG_K(15) TG_K(16)
#undef TG_K
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_score_combine(const double* d_tile_partials, const std::uint32_t* d_module_tile_begin, int M, int K,
                                 double* d_out, cudaStream_t stream) {
    const int warps = M * 2 * (K - 1);
    if (warps <= 0) return cudaSuccess;
    const int threads = 256;
    const unsigned grid = static_cast<unsigned>((warps * 32 + threads - 1) / threads);
    score_combine_kernel<<<grid, threads, 0, stream>>>(d_tile_partials, d_module_tile_begin, M, K - 1, d_out);
    return cudaGetLastError();
}

} // namespace tailor::dev
