// Host-link behaviour probe (diagnostic, not part of the library):
//  1. copy-engine ordering: does a small H2D on stream B wait behind a large H2D
//     on stream A (FIFO), delaying B's dependent D2H?
//  2. SM zero-copy reads of pinned host memory: bandwidth alone and while a CE
//     D2H runs.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/pcie_ce_probe tools/pcie_ce_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        dst[i] = a;
        dst[i + stride] = b;
        dst[i + 2 * stride] = c;
        dst[i + 3 * stride] = d;
    }
    for (; i < n; i += stride) dst[i] = src[i];
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) {
    float m = 0;
    cudaEventElapsedTime(&m, a, b);
    return m;
}

int main() {
    const size_t G = 1ull << 30;
    const size_t n = 2 * G;
    uint8_t *h1, *h2, *d1, *d2, *d3;
    CK(cudaHostAlloc(&h1, n, cudaHostAllocDefault));
    CK(cudaHostAlloc(&h2, n, cudaHostAllocDefault));
    CK(cudaMalloc(&d1, n));
    CK(cudaMalloc(&d2, n));
    CK(cudaMalloc(&d3, n));
    cudaStream_t a, b;
    CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, ea, eb;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&ea);
    cudaEventCreate(&eb);
    for (int rep = 0; rep < 2; ++rep) {
        // 1a. alone
        cudaEventRecord(e0, a);
        cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, a);
        cudaEventRecord(e1, a);
        CK(cudaDeviceSynchronize());
        const float h2d = ms_between(e0, e1);
        cudaEventRecord(e0, b);
        cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(e1, b);
        CK(cudaDeviceSynchronize());
        const float d2h = ms_between(e0, e1);
        // 1b. A: big H2D; B: small H2D then big D2H (B issued after A)
        cudaEventRecord(e0, a);
        cudaStreamWaitEvent(b, e0, 0);
        cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, a);
        cudaMemcpyAsync(d3, h1, 1 << 20, cudaMemcpyHostToDevice, b);
        cudaEventRecord(eb, b);
        cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(e1, b);
        cudaEventRecord(ea, a);
        CK(cudaDeviceSynchronize());
        std::printf("{\"test\":\"ce_order\",\"h2d_alone_ms\":%.2f,\"d2h_alone_ms\":%.2f,\"small_h2d_done_ms\":%.2f,"
                    "\"b_done_ms\":%.2f,\"a_done_ms\":%.2f}\n",
                    h2d, d2h, ms_between(e0, eb), ms_between(e0, e1), ms_between(e0, ea));
        // 2. SM zero-copy read of pinned host memory -> device
        const size_t n4 = n / 16;
        for (int blocks : {148, 296, 592, 1184}) {
            cudaEventRecord(e0, a);
            zc_read<<<blocks, 512, 0, a>>>(reinterpret_cast<const uint4*>(h1), reinterpret_cast<uint4*>(d1), n4);
            cudaEventRecord(e1, a);
            CK(cudaDeviceSynchronize());
            std::printf("{\"test\":\"zero_copy_read\",\"blocks\":%d,\"ms\":%.2f,\"gbs\":%.1f}\n", blocks, ms_between(e0, e1),
                        n / (ms_between(e0, e1) / 1e3) / 1e9);
        }
        // 3. zero-copy read concurrent with a CE D2H
        cudaEventRecord(e0, a);
        cudaStreamWaitEvent(b, e0, 0);
        zc_read<<<592, 512, 0, a>>>(reinterpret_cast<const uint4*>(h1), reinterpret_cast<uint4*>(d1), n4);
        cudaEventRecord(ea, a);
        cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(eb, b);
        CK(cudaDeviceSynchronize());
        std::printf("{\"test\":\"zc_read_with_ce_d2h\",\"read_ms\":%.2f,\"d2h_ms\":%.2f}\n", ms_between(e0, ea),
                    ms_between(e0, eb));
        // 4. CE H2D concurrent with CE D2H on two streams (reference point)
        cudaEventRecord(e0, a);
        cudaStreamWaitEvent(b, e0, 0);
        cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, a);
        cudaEventRecord(ea, a);
        cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(eb, b);
        CK(cudaDeviceSynchronize());
        std::printf("{\"test\":\"ce_h2d_with_ce_d2h\",\"h2d_ms\":%.2f,\"d2h_ms\":%.2f}\n", ms_between(e0, ea),
                    ms_between(e0, eb));
    }
    return 0;
}
