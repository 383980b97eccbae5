// fabric_bench.cu -- what bounds the one-pass C2 design: HBM read / write /
// copy rates, and a copy whose data also makes an L2 round trip through a
// ring (write the ring, read it back, as the A -> B hand-off of k_ab_st does).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fb scripts/fabric_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const float4* __restrict__ a, size_t n, float4* sink) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(a + i);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x == 1.2345f) sink[0] = acc;
}
__global__ void k_write(float4* __restrict__ a, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(a + i, make_float4(1, 2, 3, (float)i));
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(b + i, __ldcs(a + i));
}
// copy through an L2 ring: each element is written to ring[i % rn] then read
// back (by the same thread, ld.cg) before the final store
__global__ void k_copy_ring(const float4* __restrict__ a, float4* __restrict__ b, float4* ring, size_t rn, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(a + i);
        ring[i % rn] = v;
        float4 w = __ldcg(ring + ((i + 4096) % rn));
        __stcs(b + i, make_float4(v.x + w.x, v.y, v.z, v.w));
    }
}
// L2-only traffic: write + read a ring (no HBM stream)
__global__ void k_ring_only(float4* ring, size_t rn, size_t n, float4* sink) {
    float acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        ring[i % rn] = make_float4((float)i, 0, 0, 0);
        acc += __ldcg(ring + ((i + 4096) % rn)).x;
    }
    if (acc == 1.2345f) sink[0] = make_float4(acc, 0, 0, 0);
}

int main() {
    const size_t bytes = 2ull << 30, n = bytes / 16, rn = (48ull << 20) / 16;
    float4 *a, *b, *ring, *sink;
    cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&ring, rn * 16); cudaMalloc(&sink, 64);
    cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"read 2G", "write 2G", "copy 2G->2G", "copy+ring rt", "ring only (L2 w+r, 2G each)"};
    const double gbs[] = {2, 2, 4, 4, 4};  // GB of HBM-side (or ring) traffic per run, x 2^30 / 1e9
    for (int k = 0; k < 5; ++k) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(e0);
            dim3 g(sms * 4), t(512);
            if (k == 0) k_read<<<g, t>>>(a, n, sink);
            if (k == 1) k_write<<<g, t>>>(b, n);
            if (k == 2) k_copy<<<g, t>>>(a, b, n);
            if (k == 3) k_copy_ring<<<g, t>>>(a, b, ring, rn, n);
            if (k == 4) k_ring_only<<<g, t>>>(ring, rn, n, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-30s %8.3f ms  %8.0f GB/s\n", names[k], best, gbs[k] * 1.073741824e9 / (best / 1e3) / 1e9);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
