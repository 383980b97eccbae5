// strided tile copy: tiles of W consecutive float2 x R rows at stride S (elements)
#include <cstdio>
#include <cstdint>
template <int W, int R>
__global__ void __launch_bounds__(256) k(const float2* __restrict__ in, float2* __restrict__ out, int64_t S, int64_t ntiles_per_row) {
    const int64_t tile = blockIdx.x;
    const int64_t rowblk = tile / ntiles_per_row;   // which group of R rows
    const int64_t c0 = (tile % ntiles_per_row) * W;
    const float2* src = in + rowblk * R * S + c0;
    float2* dst = out + rowblk * R * S + c0;
    constexpr int PER = W * R / 256;
    float2 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) { int idx = threadIdx.x + i * 256; v[i] = src[(int64_t)(idx / W) * S + idx % W]; }
#pragma unroll
    for (int i = 0; i < PER; ++i) { int idx = threadIdx.x + i * 256; dst[(int64_t)(idx / W) * S + idx % W] = v[i]; }
}
template <int W, int R>
void run(const float2* a, float2* b, int64_t n, int64_t S) {
    int64_t rows = n / S;
    int64_t ntiles = (rows / R) * (S / W);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) k<W, R><<<(unsigned)ntiles, 256>>>(a, b, S, S / W);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 3; ++rep) k<W, R><<<(unsigned)ntiles, 256>>>(a, b, S, S / W);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    printf("W=%3d (%4d B runs) R=%4d stride=%9lld elems: %.3f ms  %.0f GB/s\n", W, W * 8, R, (long long)S, ms, 16.0 * n / ms / 1e6);
}
int main() {
    const int64_t n = 1ll << 29;  // 4 GiB per buffer
    float2 *a, *b;
    cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    for (int64_t S : {1ll << 20, 1ll << 15, 1ll << 12}) {
        run<4, 512>(a, b, n, S);
        run<8, 256>(a, b, n, S);
        run<16, 128>(a, b, n, S);
        run<32, 64>(a, b, n, S);
        run<64, 32>(a, b, n, S);
        run<8, 1024>(a, b, n, S);
    }
    return 0;
}
