// K3/K4 — update-magnitude scorer over FP32 master partitions.
//
// Contract (the reference has no scorer — its numeric anchor is
// the FP64 sum of squared steps in R/src/adamw.cpp:34-45): for module m and
// consecutive snapshots A=S_p, B=S_{p+1},
//     s_delta = sum (double(B) - double(A))^2,   s_ref = sum double(A)^2,
// over every master element of m's groups; score = sqrt(s_delta)/sqrt(s_ref).
// Shard padding is zero in every snapshot, so whole rank chunks can be summed.
//
// K3 reads each snapshot once (K snapshots -> K-1 pairs in one sweep) — by
// default through a warp-specialised TMA bulk ring (score_staged_kernel), else
// with 128-bit non-allocating register loads — accumulates FP64 per thread,
// reduces with warp shuffles and a fixed warp order, and writes one partial per
// tile (no atomics). K4 sums each module's tile partials in a fixed lane/tree order.
// Results are bitwise reproducible for a given tile table, independent of the
// grid size and of scheduling.
#include <algorithm>

#include "tailor/device.hpp"
#include "tma.cuh"

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

__device__ __forceinline__ float2 ld_nc_f2(const float2* p) {
    float2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}

// VW = floats per snapshot per load (4: 128-bit, 2: 64-bit). Large K uses VW=2
// with the snapshot base pointers in shared memory, which roughly halves the
// per-thread register footprint (K=16: 172 -> <=128 regs, two CTAs per SM) so
// twice the warps keep loads in flight while others run the FP64 accumulate.
// Min-blocks hint keeps small-K instances at 4 CTAs/SM (<= 64 regs): loads in
// flight scale with resident warps.
template <int K, int VW>
__global__ void __launch_bounds__(kScoreThreads, VW == 2 ? 2 : (K <= 4 ? 4 : (K <= 8 ? 2 : 1))) score_partials_kernel(
    const ScoreTile* __restrict__ tiles, std::uint32_t ntiles, const float* const* __restrict__ field_base,
    std::uint32_t nfields, int vec_ok, double* __restrict__ out) {
    constexpr int V = 2 * (K - 1);
    __shared__ double red[kWarps][V];
    __shared__ const float* sbase[K];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // Small K: base pointers straight from global into registers. Large K: staged
    // through smem once per tile (measured: K=16 0.896 -> 0.938 of peak).
    constexpr bool kSmemBase = VW == 2 || K > 8;
    for (std::uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const ScoreTile tile = tiles[t];
        if constexpr (kSmemBase) {
            if (tid < K) sbase[tid] = field_base[tid * nfields + tile.field] + tile.elem_start;
            __syncthreads();
        }
        const auto base_of = [&](int k) -> const float* {
            if constexpr (kSmemBase) return sbase[k];
            else return field_base[k * nfields + tile.field] + tile.elem_start;
        };
        double acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.0;
        const std::uint32_t n = tile.count;
        std::uint32_t i0 = 0;
        if (vec_ok) {
            if constexpr (VW == 4) {
                const float* base[K];
#pragma unroll
                for (int k = 0; k < K; ++k)
                    base[k] = base_of(k);
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
            } else {
                const std::uint32_t n2 = n >> 1;
                for (std::uint32_t i = tid; i < n2; i += kScoreThreads) {
                    float2 q[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) q[k] = ld_nc_f2(reinterpret_cast<const float2*>(sbase[k]) + i);
                    float x[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) x[k] = q[k].x;
                    accumulate<K>(acc, x);
#pragma unroll
                    for (int k = 0; k < K; ++k) x[k] = q[k].y;
                    accumulate<K>(acc, x);
                }
                i0 = n2 << 1;
            }
        }
        for (std::uint32_t i = i0 + tid; i < n; i += kScoreThreads) {
            float x[K];
#pragma unroll
            for (int k = 0; k < K; ++k) x[k] = __ldg(base_of(k) + i);
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


// ---- staged variant: TMA bulk copies into a shared-memory ring ------------------
// For large K the register-staged kernel above needs K float4 per thread in
// flight (222 registers at K=16 -> one 8-warp CTA per SM, latency-bound: issue
// 21%, FP64 pipe 25%). Here loads are decoupled from registers: a producer warp
// (one elected lane) streams 1024-element chunks of all K snapshots into an
// S-stage shared-memory ring with cp.async.bulk (completion by mbarrier
// transaction count), and 8 consumer warps reduce out of shared memory rolling
// over k (two float4 live) and release each stage through an `empty` mbarrier
// (one arrival per consumer warp) — no CTA-wide barrier in the stream. Same
// tile -> partial contract (one partial per tile, fixed order); the summation
// order inside a tile differs from the register kernel, so the two variants
// agree to ~1e-15, not bitwise.
constexpr int kStagedSmem = 192 * 1024;
// Ring geometry: G = 0 default, 1 half the rows per stage (smaller bulk copies, more
// stages; the round-1 default for K >= 4), 2 two CTAs per SM (each half the ring).
// CTAs per SM: small K runs two (each with half the ring) for more independent streams.
template <int K, int G = 0>
__host__ __device__ constexpr int staged_ctas() {
    return G == 2 ? 2 : (K < 4 ? 2 : 1);
}
constexpr int kStagedThreads = kScoreThreads + 32; // 8 consumer warps + 1 producer warp

// float4 per consumer thread per snapshot row in one stage: 8 KB per snapshot row for
// 3 <= K <= 8 (K=4: 32 KB stages x 6 = 192 KB in flight per SM; with 4 KB rows, 8 x 16 KB
// stages, B200 measured 0.90 of the read stream vs 1.00), 16 KB for K = 2, 4 KB for K >= 9
// (the stage must fit twice in shared memory).
template <int K, int G = 0>
__host__ __device__ constexpr int staged_rows() {
    constexpr int r = K >= 9 ? 1 : (K >= 3 ? 2 : 4);
    return G == 1 ? (r > 1 ? r / 2 : 1) : r;
}
template <int K, int G = 0>
__host__ __device__ constexpr int chunk_elems() {
    return 4 * kScoreThreads * staged_rows<K, G>();
}

template <int K, int G = 0>
__host__ __device__ constexpr int staged_stages() {
    constexpr int per = K * chunk_elems<K, G>() * 4;
    constexpr int s = kStagedSmem / staged_ctas<K, G>() / per;
    return s < 2 ? 2 : (s > 8 ? 8 : s);
}

template <int K, int G = 0>
__host__ __device__ constexpr std::size_t staged_smem_bytes() {
    return static_cast<std::size_t>(staged_stages<K, G>()) * K * chunk_elems<K, G>() * 4 + 16 * staged_stages<K, G>();
}

template <int K>
__device__ __forceinline__ void accumulate4(double (&acc)[2 * (K - 1)], int p, const float4& a, const float4& b) {
    const double ax = a.x, ay = a.y, az = a.z, aw = a.w;
    const double dx = static_cast<double>(b.x) - ax, dy = static_cast<double>(b.y) - ay;
    const double dz = static_cast<double>(b.z) - az, dw = static_cast<double>(b.w) - aw;
    acc[2 * p] = fma(dw, dw, fma(dz, dz, fma(dy, dy, fma(dx, dx, acc[2 * p]))));
    acc[2 * p + 1] = fma(aw, aw, fma(az, az, fma(ay, ay, fma(ax, ax, acc[2 * p + 1]))));
}

// Which tile and chunk a ring stage holds (written by the producer before the
// stage's bulk copies; published to the consumers by the full barrier's arrive).
struct StageDesc {
    std::uint32_t tile;  // ~0u: end of the stream
    std::uint32_t start; // first element of the chunk within the tile
    std::uint32_t n;     // elements in the chunk
    std::uint32_t last;  // last chunk of the tile: the consumers reduce and write its partial
};
constexpr std::uint32_t kNoTile = ~0u;

// Tiles are claimed dynamically (counter != nullptr: atomicAdd on a per-launch counter
// zeroed on the stream before the launch) — SMs do not stream at equal rates (ncu, cfg2
// K=2 with the static split: SM active 89.6% of elapsed, the rest a tail of CTAs still
// working) — or statically (b, b+G, ...) without a counter. Either way tile t's partial
// lands at out[t]: the results do not depend on which CTA ran which tile.
template <int K, int G>
__global__ void __launch_bounds__(kStagedThreads, 1) score_staged_kernel(const ScoreTile* __restrict__ tiles,
                                                                          std::uint32_t ntiles,
                                                                          const float* const* __restrict__ field_base,
                                                                          std::uint32_t nfields, double* __restrict__ out,
                                                                          unsigned int* __restrict__ counter) {
    using namespace tma;
    constexpr int S = staged_stages<K, G>();
    constexpr int V = 2 * (K - 1);
    constexpr int kChunkElems = chunk_elems<K, G>();
    constexpr int R = staged_rows<K, G>();
    extern __shared__ __align__(128) float ring[];
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(ring + S * K * kChunkElems);
    std::uint64_t* empty = full + S;
    __shared__ double red[kWarps][V];
    __shared__ StageDesc desc[S];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int st = 0; st < S; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], kWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kWarps) { // producer
        if (lane == 0) {
            std::uint32_t item = 0, claimed = 0;
            const auto claim = [&]() -> std::uint32_t {
                return counter ? atomicAdd(counter, 1u) : blockIdx.x + (claimed++) * gridDim.x;
            };
            const auto next_stage = [&]() { // wait until the stage of `item` is free
                const int stage = static_cast<int>(item % S);
                if (item >= static_cast<std::uint32_t>(S)) mbar_wait_parity(&empty[stage], ((item / S) - 1) & 1u);
                return stage;
            };
            std::uint32_t t = claim();
            while (t < ntiles) {
                const ScoreTile tl = tiles[t];
                const std::uint32_t t_next = claim(); // in flight while this tile's chunks are issued
                const float* base[K];
#pragma unroll
                for (int k = 0; k < K; ++k) base[k] = field_base[k * nfields + tl.field] + tl.elem_start;
                for (std::uint32_t start = 0;; start += kChunkElems, ++item) {
                    const int stage = next_stage();
                    const std::uint32_t n = tl.count > start ? min(static_cast<std::uint32_t>(kChunkElems), tl.count - start) : 0u;
                    const bool last = start + kChunkElems >= tl.count;
                    desc[stage] = {t, start, n, last ? 1u : 0u};
                    const std::uint32_t nb = (n & ~3u) * 4u;
                    if (nb) {
                        mbar_arrive_expect_tx(&full[stage], nb * K); // releases desc[stage] too
#pragma unroll
                        for (int k = 0; k < K; ++k)
                            bulk_load(ring + (stage * K + k) * kChunkElems, base[k] + start, nb, &full[stage]);
                    } else {
                        mbar_arrive(&full[stage]);
                    }
                    if (last) {
                        ++item;
                        break;
                    }
                }
                t = t_next;
            }
            const int stage = next_stage(); // end of stream
            desc[stage] = {kNoTile, 0u, 0u, 1u};
            mbar_arrive(&full[stage]);
        }
        return;
    }

    double acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0;
    for (std::uint32_t item = 0;; ++item) {
        const int stage = static_cast<int>(item % S);
        mbar_wait_parity(&full[stage], (item / S) & 1u);
        const StageDesc d = desc[stage];
        if (d.tile == kNoTile) break;
        const std::uint32_t n4 = d.n & ~3u;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const std::uint32_t e = (static_cast<std::uint32_t>(rr) * kScoreThreads + static_cast<std::uint32_t>(tid)) * 4u;
            if (e < n4) {
                const float* row = ring + stage * K * kChunkElems + e;
                float4 prev = *reinterpret_cast<const float4*>(row);
#pragma unroll
                for (int k = 1; k < K; ++k) {
                    const float4 cur = *reinterpret_cast<const float4*>(row + k * kChunkElems);
                    accumulate4<K>(acc, k - 1, prev, cur);
                    prev = cur;
                }
            }
        }
        __syncwarp();
        if (lane == 0) { // this warp is done with the stage: order its generic-proxy reads
            fence_proxy_async_smem(); // before the producer's next async-proxy (TMA) writes
            mbar_arrive(&empty[stage]);
        }
        if (static_cast<std::uint32_t>(tid) < d.n - n4) { // ragged tail straight from global
            const ScoreTile tl = tiles[d.tile];
            float x[K];
#pragma unroll
            for (int k = 0; k < K; ++k) x[k] = __ldg(field_base[k * nfields + tl.field] + tl.elem_start + d.start + n4 + tid);
            accumulate<K>(acc, x);
        }
        if (d.last) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const double sv = warp_sum(acc[v]);
                if (lane == 0) red[warp][v] = sv;
                acc[v] = 0.0;
            }
            named_bar_sync(1, kScoreThreads);
            if (tid < V) {
                double sv = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) sv += red[w][tid];
                out[static_cast<std::uint64_t>(d.tile) * V + tid] = sv;
            }
            named_bar_sync(1, kScoreThreads);
        }
    }
}

template <int K, int G>
cudaError_t launch_staged_g(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                            std::uint32_t nfields, double* d_out, unsigned int* d_counter, cudaStream_t stream) {
    static std::atomic<std::uint64_t> attr{0};
    constexpr std::size_t smem = staged_smem_bytes<K, G>();
    if (const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(score_staged_kernel<K, G>), smem, attr);
        e != cudaSuccess)
        return e;
    if (d_counter)
        if (const cudaError_t e = cudaMemsetAsync(d_counter, 0, sizeof(unsigned int), stream); e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>(
        std::min<std::uint64_t>(ntiles, static_cast<std::uint64_t>(sm_count()) * staged_ctas<K, G>()));
    score_staged_kernel<K, G><<<grid, kStagedThreads, smem, stream>>>(d_tiles, ntiles, d_field_base, nfields, d_out,
                                                                      d_counter);
    return cudaGetLastError();
}

// geometry: 0 default; kScoreStagedWide / kScoreStaged2Cta (K <= 8; larger K keep the default)
template <int K>
cudaError_t launch_staged(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                          std::uint32_t nfields, double* d_out, unsigned int* d_counter, cudaStream_t stream, int variant) {
    if constexpr (K <= 8) {
        if (variant == kScoreStagedWide)
            return launch_staged_g<K, 1>(d_tiles, ntiles, d_field_base, nfields, d_out, d_counter, stream);
        if (variant == kScoreStaged2Cta)
            return launch_staged_g<K, 2>(d_tiles, ntiles, d_field_base, nfields, d_out, d_counter, stream);
    }
    return launch_staged_g<K, 0>(d_tiles, ntiles, d_field_base, nfields, d_out, d_counter, stream);
}

template <int K, int VW>
cudaError_t launch_kv(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                      std::uint32_t nfields, bool vec_ok, double* d_out, cudaStream_t stream) {
    static const int per_sm = [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, score_partials_kernel<K, VW>, kScoreThreads, 0);
        return std::max(1, n);
    }();
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ntiles, static_cast<std::uint64_t>(sm_count()) * per_sm));
    score_partials_kernel<K, VW><<<grid, kScoreThreads, 0, stream>>>(d_tiles, ntiles, d_field_base, nfields, vec_ok ? 1 : 0,
                                                                     d_out);
    return cudaGetLastError();
}

template <int K>
cudaError_t launch_k(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                     std::uint32_t nfields, bool vec_ok, double* d_out, cudaStream_t stream, int variant) {
    const bool narrow = variant == kScoreNarrow || (variant != kScoreWide && K >= kNarrowMinK);
    return narrow ? launch_kv<K, 2>(d_tiles, ntiles, d_field_base, nfields, vec_ok, d_out, stream)
                  : launch_kv<K, 4>(d_tiles, ntiles, d_field_base, nfields, vec_ok, d_out, stream);
}

} // namespace

cudaError_t launch_score_partials(const ScoreTile* d_tiles, std::uint32_t ntiles, const float* const* d_field_base,
                                  std::uint32_t nfields, int K, bool vec_ok, double* d_out, cudaStream_t stream,
                                  int variant, unsigned int* d_counter) {
    if (ntiles == 0) return cudaSuccess;
    const bool staged = vec_ok && (variant == kScoreStaged || variant == kScoreStagedWide || variant == kScoreStaged2Cta ||
                                   (variant == kScoreAuto && K >= kStagedMinK));
    switch (K) {
#define TG_K(k)                                                                                           \
    case k:                                                                                               \
        return staged ? launch_staged<k>(d_tiles, ntiles, d_field_base, nfields, d_out, d_counter, stream, variant) \
                      : launch_k<k>(d_tiles, ntiles, d_field_base, nfields, vec_ok, d_out, stream, variant);
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
