// K2 — segmented gather/scatter of checkpoint payload bytes (the composite
// assembly of R/src/merge.cpp:244-303, which the reference performs as
// per-tensor std::vector copies). Pure data movement: HBM-bound, no tensor
// cores. Two implementations over the same segment table:
//
//  * bulk (default when every segment is 16-B aligned and the segments tile
//    the destination): a persistent CTA per SM whose single elected thread
//    drives the TMA copy engine — cp.async.bulk global->shared into a 3-stage
//    ring of 64 KB completed by mbarrier transaction counts, then cp.async.bulk
//    shared->global (bulk_group) out of the same stage. No register staging,
//    a handful of issue instructions per 64 KB.
//  * lsu: 256-thread CTAs, 16-B ld.global.nc / st.global with UNROLL loads in
//    flight per thread, head/tail peeling and 4/2/1-byte fallbacks for the
//    misaligned segments the reference's randomized shapes produce (12-B
//    chunks, 2-B bf16 tensors).
//
// Work split: the destination is cut into fixed tiles. The LSU kernel and a bulk
// launch without a counter use the static split (CTA b owns tiles b, b+G, ...); a
// bulk launch with a plan's counter claims tiles dynamically (faster SMs take more:
// 0.97 -> 1.06 of the measured copy peak at cfg3). Either way a tile's bytes land
// at the tile's own offset, so the output never depends on timing.
#include <algorithm>

#include "tailor/device.hpp"
#include "tma.cuh"

namespace tailor::dev {

namespace {

constexpr int kLsuThreads = 256;
constexpr std::uint64_t kLsuTile = 64 * 1024;
constexpr int kLsuUnroll = 8;

// Ring: 3 x 64 KB (sweep on B200, cfg3 shard gather: 3x64K 4.155 ms, 4x48K 4.20, 3x72K
// 4.18, 4x56K 4.22, 6x32K 4.19, 2 CTAs x 3x32K 4.20, 8x24K 4.32).
constexpr int kBulkStages = 3;
constexpr std::uint32_t kBulkStage = 64 * 1024;

__device__ __forceinline__ int seg_lookup(const GatherSeg* __restrict__ segs, std::uint32_t n, std::uint64_t x) {
    int lo = 0, hi = static_cast<int>(n) - 1, ans = -1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (segs[mid].dst_off <= x) {
            ans = mid;
            lo = mid + 1;
        } else {
            hi = mid - 1;
        }
    }
    return ans < 0 ? 0 : ans;
}

__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

template <typename W>
__device__ __forceinline__ void cta_copy_words(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t n) {
    // dst and src share alignment mod sizeof(W); peel to W alignment.
    const int tid = threadIdx.x;
    std::uint64_t head = (sizeof(W) - (reinterpret_cast<std::uintptr_t>(dst) & (sizeof(W) - 1))) & (sizeof(W) - 1);
    if (head > n) head = n;
    if (static_cast<std::uint64_t>(tid) < head) dst[tid] = src[tid];
    const std::uint64_t nw = (n - head) / sizeof(W);
    const W* s = reinterpret_cast<const W*>(src + head);
    W* d = reinterpret_cast<W*>(dst + head);
    for (std::uint64_t i = tid; i < nw; i += kLsuThreads) d[i] = s[i];
    const std::uint64_t done = head + nw * sizeof(W);
    if (static_cast<std::uint64_t>(tid) < n - done) dst[done + tid] = src[done + tid];
}

__device__ __forceinline__ void cta_copy(std::uint8_t* __restrict__ dst, const std::uint8_t* __restrict__ src,
                                         std::uint64_t n) {
    const std::uintptr_t mis = reinterpret_cast<std::uintptr_t>(dst) ^ reinterpret_cast<std::uintptr_t>(src);
    if ((mis & 15) == 0) {
        const int tid = threadIdx.x;
        std::uint64_t head = (16 - (reinterpret_cast<std::uintptr_t>(dst) & 15)) & 15;
        if (head > n) head = n;
        if (static_cast<std::uint64_t>(tid) < head) dst[tid] = src[tid];
        const std::uint64_t nv = (n - head) >> 4;
        const int4* s4 = reinterpret_cast<const int4*>(src + head);
        int4* d4 = reinterpret_cast<int4*>(dst + head);
        std::uint64_t i = tid;
        for (; i + static_cast<std::uint64_t>(kLsuUnroll - 1) * kLsuThreads < nv; i += kLsuUnroll * kLsuThreads) {
            int4 v[kLsuUnroll];
#pragma unroll
            for (int u = 0; u < kLsuUnroll; ++u) v[u] = ld_stream(s4 + i + u * kLsuThreads);
#pragma unroll
            for (int u = 0; u < kLsuUnroll; ++u) st_stream(d4 + i + u * kLsuThreads, v[u]);
        }
        for (; i < nv; i += kLsuThreads) st_stream(d4 + i, ld_stream(s4 + i));
        const std::uint64_t done = head + (nv << 4);
        if (static_cast<std::uint64_t>(tid) < n - done) dst[done + tid] = src[done + tid];
    } else if ((mis & 3) == 0) {
        cta_copy_words<std::uint32_t>(dst, src, n);
    } else if ((mis & 1) == 0) {
        cta_copy_words<std::uint16_t>(dst, src, n);
    } else {
        for (std::uint64_t i = threadIdx.x; i < n; i += kLsuThreads) dst[i] = src[i];
    }
}

__global__ void __launch_bounds__(kLsuThreads) gather_lsu_kernel(const GatherSeg* __restrict__ segs, std::uint32_t nseg,
                                                                  std::uint8_t* __restrict__ dst, std::uint64_t dst_bytes) {
    const std::uint64_t ntiles = (dst_bytes + kLsuTile - 1) / kLsuTile;
    for (std::uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        std::uint64_t lo = t * kLsuTile;
        const std::uint64_t hi = min(lo + kLsuTile, dst_bytes);
        for (int s = seg_lookup(segs, nseg, lo); lo < hi && s < static_cast<int>(nseg); ++s) {
            const GatherSeg g = segs[s];
            const std::uint64_t end = g.dst_off + g.bytes;
            if (end <= lo) continue;
            if (g.dst_off >= hi) break;
            const std::uint64_t a = max(lo, g.dst_off), b = min(hi, end);
            cta_copy(dst + a, g.src + (a - g.dst_off), b - a);
            lo = b;
        }
    }
}

// ---- TMA bulk path -----------------------------------------------------------
using namespace tma;

// Tile assignment: static (counter == nullptr: CTA b copies tiles b, b+G, ...) or
// dynamic (claimed one at a time from counter[0] with atomicAdd, the next claim in
// flight while the current tile streams, so faster SMs take more tiles and no SM
// idles at the tail). Dynamic launches leave the counter as they found it (zero):
// the last CTA to finish (counter[1] == grid - 1) resets both words, so launches
// that share a counter must be stream-ordered (each plan owns its counter). The
// bytes placed never depend on the assignment.
template <int STAGES, std::uint32_t STAGE>
__global__ void __launch_bounds__(32) gather_bulk_kernel(const GatherSeg* __restrict__ segs, std::uint32_t nseg,
                                                          std::uint8_t* __restrict__ dst, std::uint64_t dst_bytes,
                                                          unsigned int* __restrict__ counter) {
    extern __shared__ __align__(128) std::uint8_t smem[];
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + STAGES * STAGE);
    if (threadIdx.x != 0) return; // one thread drives the copy engine
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();

    const std::uint64_t ntiles = (dst_bytes + STAGE - 1) / STAGE;
    std::uint64_t claimed = 0; // static: tiles handed out to this CTA so far
    const auto claim = [&]() -> std::uint64_t {
        return counter ? static_cast<std::uint64_t>(atomicAdd(counter, 1u)) : blockIdx.x + (claimed++) * gridDim.x;
    };
    std::uint64_t tile_of[STAGES];

    const auto issue_load = [&](std::uint64_t tile, int stage) {
        const std::uint64_t lo = tile * STAGE;
        const std::uint64_t hi = min(lo + STAGE, dst_bytes);
        std::uint8_t* buf = smem + stage * STAGE;
        mbar_arrive_expect_tx(&bars[stage], static_cast<std::uint32_t>(hi - lo));
        std::uint64_t at = lo;
        for (int s = seg_lookup(segs, nseg, lo); at < hi && s < static_cast<int>(nseg); ++s) {
            const GatherSeg g = segs[s];
            const std::uint64_t end = g.dst_off + g.bytes;
            if (end <= at) continue;
            const std::uint64_t b = min(hi, end);
            bulk_load(buf + (at - lo), g.src + (at - g.dst_off), static_cast<std::uint32_t>(b - at), &bars[stage]);
            at = b;
        }
    };

    std::uint64_t next = claim(); // the claim after the tiles already issued (in flight)
    std::uint64_t issued = 0;
    for (; issued < STAGES - 1 && next < ntiles; ++issued) {
        tile_of[issued] = next;
        issue_load(next, static_cast<int>(issued));
        next = claim();
    }
    for (std::uint64_t i = 0; i < issued; ++i) {
        const int stage = static_cast<int>(i % STAGES);
        mbar_wait_parity(&bars[stage], static_cast<std::uint32_t>((i / STAGES) & 1));
        const std::uint64_t lo = tile_of[stage] * STAGE;
        const std::uint64_t hi = min(lo + STAGE, dst_bytes);
        bulk_store(dst + lo, smem + stage * STAGE, static_cast<std::uint32_t>(hi - lo));
        bulk_commit();
        if (next < ntiles) { // lands in tile i-1's stage
            const int ns = static_cast<int>(issued % STAGES);
            if (i >= 1) bulk_wait_read_1(); // store of tile i-1 has finished reading smem
            tile_of[ns] = next;
            issue_load(next, ns);
            ++issued;
            next = claim();
        }
    }
    bulk_wait_all();
    if (counter) {
        __threadfence();
        if (atomicAdd(counter + 1, 1u) == gridDim.x - 1) { // every other CTA has made its last claim
            counter[0] = 0;
            counter[1] = 0;
        }
    }
}

template <int STAGES, std::uint32_t STAGE>
cudaError_t launch_bulk(const GatherSeg* d_segs, std::uint32_t nseg, std::uint8_t* d_dst, std::uint64_t dst_bytes,
                        int ctas_per_sm, unsigned int* d_counter, cudaStream_t stream) {
    static std::atomic<std::uint64_t> attr{0};
    const std::size_t smem = STAGES * STAGE + STAGES * sizeof(std::uint64_t);
    if (const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gather_bulk_kernel<STAGES, STAGE>), smem, attr);
        e != cudaSuccess)
        return e;
    const std::uint64_t tiles = (dst_bytes + STAGE - 1) / STAGE;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(tiles, static_cast<std::uint64_t>(sm_count()) * ctas_per_sm));
    gather_bulk_kernel<STAGES, STAGE><<<grid, 32, smem, stream>>>(d_segs, nseg, d_dst, dst_bytes, d_counter);
    return cudaGetLastError();
}


// Read-only HBM stream reference (measurement only): persistent grid, 8 x 16-B
// streaming loads in flight per thread, XOR-folded into one word per block so
// the loads cannot be elided. Gives the denominator for read-only kernels (the
// scorer), for which the read+write copy peak understates what HBM delivers.
__global__ void __launch_bounds__(kLsuThreads) read_probe_kernel(const int4* __restrict__ src, std::uint64_t n16,
                                                                 unsigned int* __restrict__ sink) {
    int4 acc = make_int4(0, 0, 0, 0);
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * kLsuThreads;
    std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(kLsuThreads) + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc.x ^= v[u].x;
            acc.y ^= v[u].y;
            acc.z ^= v[u].z;
            acc.w ^= v[u].w;
        }
    }
    for (; i < n16; i += stride) {
        const int4 v = ld_stream(src + i);
        acc.x ^= v.x;
        acc.y ^= v.y;
        acc.z ^= v.z;
        acc.w ^= v.w;
    }
    unsigned int x = static_cast<unsigned int>(acc.x ^ acc.y ^ acc.z ^ acc.w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) atomicXor(sink, x);
}

} // namespace

cudaError_t launch_read_probe(const std::uint8_t* d_src, std::uint64_t bytes, unsigned int* d_sink, cudaStream_t stream) {
    if (bytes < 16) return cudaSuccess;
    read_probe_kernel<<<static_cast<unsigned>(sm_count()) * 4, kLsuThreads, 0, stream>>>(reinterpret_cast<const int4*>(d_src),
                                                                                           bytes / 16, d_sink);
    return cudaGetLastError();
}

int sm_count() {
    static const int n = [] {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms > 0 ? sms : 148;
    }();
    return n;
}

cudaError_t ensure_smem_attr(const void* fn, std::size_t smem, std::atomic<std::uint64_t>& done) {
    int dev = 0;
    if (const cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    const std::uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

cudaError_t launch_gather(const GatherSeg* d_segs, std::uint32_t nseg, std::uint8_t* d_dst, std::uint64_t dst_bytes,
                          int variant, bool bulk_ok, cudaStream_t stream, unsigned int* d_counter) {
    if (dst_bytes == 0 || nseg == 0) return cudaSuccess;
    if (variant == kGatherBulkStatic) {
        variant = kGatherBulk;
        d_counter = nullptr;
    }
    const int sms = sm_count();
    const bool bulk = variant >= kGatherBulk || (variant == kGatherAuto && bulk_ok);
    if (bulk && bulk_ok) {
        switch (variant) { // ring shapes for experiments; auto/2 = 3 x 64 KB, one CTA per SM
            case kGatherBulk6x32: return launch_bulk<6, 32 * 1024>(d_segs, nseg, d_dst, dst_bytes, 1, d_counter, stream);
            case kGatherBulk2Cta: return launch_bulk<3, 32 * 1024>(d_segs, nseg, d_dst, dst_bytes, 2, d_counter, stream);
            case kGatherBulk4x48: return launch_bulk<4, 48 * 1024>(d_segs, nseg, d_dst, dst_bytes, 1, d_counter, stream);
            case kGatherBulk8x24: return launch_bulk<8, 24 * 1024>(d_segs, nseg, d_dst, dst_bytes, 1, d_counter, stream);
            default: return launch_bulk<kBulkStages, kBulkStage>(d_segs, nseg, d_dst, dst_bytes, 1, d_counter, stream);
        }
    }
    static const int lsu_blocks_per_sm = [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gather_lsu_kernel, kLsuThreads, 0);
        return std::max(1, std::min(n, 4));
    }();
    const std::uint64_t tiles = (dst_bytes + kLsuTile - 1) / kLsuTile;
    const unsigned grid =
        static_cast<unsigned>(std::min<std::uint64_t>(tiles, static_cast<std::uint64_t>(sms) * lsu_blocks_per_sm));
    gather_lsu_kernel<<<grid, kLsuThreads, 0, stream>>>(d_segs, nseg, d_dst, dst_bytes);
    return cudaGetLastError();
}

} // namespace tailor::dev
