// Access-pattern ceiling of the K7 update pass (diagnostics, not product code): the
// trainer's w/m/v in-place float4 read-modify-write over 16384-element tiles, with no
// arithmetic beyond one FMUL per value, at the trainer's grid (8 x SMs blocks of 256)
// and at one resident wave (4 x SMs). If this runs near the copy peak the update pass is
// bound by its instruction stream; if it runs where the update pass does, by the
// pattern of 3 read + 3 write streams per block.
// rmw_bulk: the same read-modify-write through a per-CTA ring of S stages (w, m, v
// 4 KB chunks each): cp.async.bulk G->S (mbarrier tx-count), every thread updates one
// float4 per array in shared memory, cp.async.bulk S->G (bulk groups), loads L chunks ahead.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rmw_probe tools/rmw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2602_22158_b200/csrc/kernels/tma.cuh"

using namespace tailor::dev;

constexpr int kThreads = 256;
constexpr std::uint32_t kTile = 16384;

__global__ void __launch_bounds__(kThreads) rmw3(float* w, float* m, float* v, std::uint64_t n, std::uint32_t ntiles) {
    for (std::uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const std::uint64_t base = static_cast<std::uint64_t>(t) * kTile;
        const std::uint32_t n4 = static_cast<std::uint32_t>((n - base < kTile ? n - base : kTile) >> 2);
        float4* wp = reinterpret_cast<float4*>(w + base);
        float4* mp = reinterpret_cast<float4*>(m + base);
        float4* vp = reinterpret_cast<float4*>(v + base);
        for (std::uint32_t q = threadIdx.x; q < n4; q += kThreads) {
            float4 a = __ldcs(wp + q), b = __ldcs(mp + q), c = __ldcs(vp + q);
            a.x *= 0.999f; a.y *= 0.999f; a.z *= 0.999f; a.w *= 0.999f;
            b.x *= 0.999f; b.y *= 0.999f; b.z *= 0.999f; b.w *= 0.999f;
            c.x *= 0.999f; c.y *= 0.999f; c.z *= 0.999f; c.w *= 0.999f;
            __stcs(mp + q, b);
            __stcs(vp + q, c);
            __stcs(wp + q, a);
        }
    }
}

constexpr std::uint32_t kChunk = kThreads * 16; // bytes per array per chunk
constexpr std::uint32_t kChunksPerTile = kTile * 4 / kChunk;

template <int S, int L>
__global__ void __launch_bounds__(kThreads) rmw_bulk(float* w, float* m, float* v, std::uint32_t ntiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ std::uint64_t full[S];
    float4* st = reinterpret_cast<float4*>(smem); // [S][3][kThreads]
    const std::uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const std::uint32_t nch = my_tiles * kChunksPerTile;
    float* arr[3] = {w, m, v};
    const auto gaddr = [&](std::uint32_t c, int a) {
        const std::uint64_t tile = blockIdx.x + static_cast<std::uint64_t>(c / kChunksPerTile) * gridDim.x;
        return reinterpret_cast<char*>(arr[a]) + tile * kTile * 4 + (c % kChunksPerTile) * kChunk;
    };
    const auto issue = [&](std::uint32_t c) {
        const int s = c % S;
        tma::mbar_arrive_expect_tx(&full[s], 3 * kChunk);
        for (int a = 0; a < 3; ++a) tma::bulk_load(st + (s * 3 + a) * kThreads, gaddr(c, a), kChunk, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) tma::mbar_init(&full[s], 1);
        tma::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (std::uint32_t c = 0; c < L && c < nch; ++c) issue(c);
    for (std::uint32_t c = 0; c < nch; ++c) {
        const int s = c % S;
        tma::mbar_wait_parity(&full[s], (c / S) & 1);
        for (int a = 0; a < 3; ++a) {
            float4 x = st[(s * 3 + a) * kThreads + threadIdx.x];
            x.x *= 0.999f; x.y *= 0.999f; x.z *= 0.999f; x.w *= 0.999f;
            st[(s * 3 + a) * kThreads + threadIdx.x] = x;
        }
        tma::fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int a = 0; a < 3; ++a) tma::bulk_store(gaddr(c, a), st + (s * 3 + a) * kThreads, kChunk);
            tma::bulk_commit();
            if (c + L < nch) {
                // stage (c+L)%S last held chunk c+L-S, stored S-L iterations ago
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - L) : "memory");
                issue(c + L);
            }
        }
    }
    if (threadIdx.x == 0) tma::bulk_wait_all();
}

template <int S, int L>
void run_bulk(float* w, float* m, float* v, std::uint64_t n, int sms, int per_sm) {
    const std::uint32_t ntiles = static_cast<std::uint32_t>(n / kTile);
    const int smem = S * 3 * kChunk;
    cudaFuncSetAttribute(rmw_bulk<S, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const unsigned grid = static_cast<unsigned>(sms * per_sm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) rmw_bulk<S, L><<<grid, kThreads, smem>>>(w, m, v, ntiles);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) rmw_bulk<S, L><<<grid, kThreads, smem>>>(w, m, v, ntiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = ms / reps;
    std::printf("{\"bulk\": true, \"stages\": %d, \"ahead\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
                S, L, per_sm, per, 24.0 * (ntiles * static_cast<double>(kTile)) / (per * 1e-3) / 1e9,
                cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const std::uint64_t n = 1104445952ull; // one Llama-3.1-8B rank partition (bench --workload train)
    float *w, *m, *v;
    cudaMalloc(&w, n * 4);
    cudaMalloc(&m, n * 4);
    cudaMalloc(&v, n * 4);
    cudaMemset(w, 0, n * 4);
    cudaMemset(m, 0, n * 4);
    cudaMemset(v, 0, n * 4);
    const std::uint32_t ntiles = static_cast<std::uint32_t>((n + kTile - 1) / kTile);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int per_sm : {8, 4, 16}) {
        const unsigned grid = static_cast<unsigned>(sms * per_sm);
        for (int i = 0; i < 3; ++i) rmw3<<<grid, kThreads>>>(w, m, v, n, ntiles);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int i = 0; i < reps; ++i) rmw3<<<grid, kThreads>>>(w, m, v, n, ntiles);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double per = ms / reps;
        std::printf("{\"blocks_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, per, 24.0 * n / (per * 1e-3) / 1e9);
    }
    const std::uint64_t nb = n / kTile * kTile;
    run_bulk<4, 2>(w, m, v, nb, sms, 4);
    run_bulk<4, 2>(w, m, v, nb, sms, 3);
    run_bulk<6, 3>(w, m, v, nb, sms, 3);
    run_bulk<4, 3>(w, m, v, nb, sms, 4);
    run_bulk<8, 5>(w, m, v, nb, sms, 2);
    run_bulk<3, 1>(w, m, v, nb, sms, 5);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        std::printf("error: %s\n", cudaGetErrorString(err));
        return 1;
    }
    return 0;
}
