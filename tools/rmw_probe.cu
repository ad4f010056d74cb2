// Access-pattern ceiling of the K7 update pass (diagnostics, not product code): the
// trainer's w/m/v in-place float4 read-modify-write over 16384-element tiles, with no
// arithmetic beyond one FMUL per value, at the trainer's grid (8 x SMs blocks of 256)
// and at one resident wave (4 x SMs). If this runs near the copy peak the update pass is
// bound by its instruction stream; if it runs where the update pass does, by the
// pattern of 3 read + 3 write streams per block.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rmw_probe tools/rmw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        std::printf("error: %s\n", cudaGetErrorString(err));
        return 1;
    }
    return 0;
}
