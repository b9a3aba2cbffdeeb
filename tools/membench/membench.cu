// Streaming microbenchmark with the fused x-pass's HBM access pattern (no math):
// per tile of 32 x-lines x 128 voxels: 16 field rows read, 12 written (float2),
// plus 3 x 65 spectrum runs of 32 complex read and written.  Variant 1 drops the
// spectrum; variant 2 is a plain 1:1 copy of the same byte count.
#include <cuda_runtime.h>
#include <cstdio>

constexpr int TL = 32, M = 128, HX = 65;

__global__ void __launch_bounds__(256, 3) pat(const float* __restrict__ in, float* __restrict__ out, const float2* sin,
                                              float2* sout, long long N, long long lines, int spec) {
    const long long L0 = (long long)blockIdx.x * TL;
    const size_t base = (size_t)L0 * M;
    float acc = 0.f;
    if (spec) {
        for (int i = threadIdx.x; i < 3 * HX * TL; i += 256) {
            const int l = i & 31, cp = i >> 5;
            const float2 v = sin[(size_t)cp * lines + L0 + l];
            acc += v.x + v.y;
        }
    }
    for (int i0 = threadIdx.x * 2; i0 < TL * M; i0 += 512) {
        float2 r[16];
#pragma unroll
        for (int f = 0; f < 16; ++f) r[f] = *reinterpret_cast<const float2*>(in + (size_t)f * N + base + i0);
        float s = acc;
#pragma unroll
        for (int f = 0; f < 16; ++f) s += r[f].x * 1e-30f + r[f].y * 1e-30f;
#pragma unroll
        for (int f = 0; f < 12; ++f) *reinterpret_cast<float2*>(out + (size_t)f * N + base + i0) = make_float2(s, r[f].y);
    }
    if (spec) {
        for (int i = threadIdx.x; i < 3 * HX * TL; i += 256) {
            const int l = i & 31, cp = i >> 5;
            sout[(size_t)cp * lines + L0 + l] = make_float2(acc, 0.f);
        }
    }
}

__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    const long long N = 32LL * 1048576;  // 32 pairs worth of voxels per field row-set
    const long long lines = N / M;
    float *in, *out;
    float2 *sin, *sout;
    cudaMalloc(&in, sizeof(float) * 16 * N);
    cudaMalloc(&out, sizeof(float) * 12 * N);
    cudaMalloc(&sin, sizeof(float2) * 3 * HX * lines);
    cudaMalloc(&sout, sizeof(float2) * 3 * HX * lines);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int spec = 1; spec >= 0; --spec) {
        for (int r = 0; r < 2; ++r) pat<<<lines / TL, 256>>>(in, out, sin, sout, N, lines, spec);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) pat<<<lines / TL, 256>>>(in, out, sin, sout, N, lines, spec);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)N * 28 * 4 + (spec ? 2.0 * 3 * HX * lines * 8 : 0);
        printf("pattern spec=%d: %.3f ms  %.0f GB/s\n", spec, ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
    }
    const size_t n4 = (size_t)N * 14 / 4;  // same bytes as the 28-field pattern: 14 read + 14 write
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copyk<<<148 * 8, 512>>>((float4*)in, (float4*)out, n4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.3f ms  %.0f GB/s\n", ms / 5, 2.0 * n4 * 16 / (ms / 5 * 1e-3) / 1e9);
    return 0;
}
