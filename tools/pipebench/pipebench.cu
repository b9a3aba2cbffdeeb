// Issue/pipe throughput probe for the fp32 forms the FFT butterflies use on sm_100a:
// scalar FADD / FFMA / FMUL vs packed FADD2 / FFMA2 / FMUL2.  8 independent chains
// per thread, 148*8 CTAs x 256 threads, CUDA-event timed; prints ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void k(float* out, float a, float b) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-7f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if constexpr (OP == 0) { x[i] = x[i] + x[i + 1]; x[i + 1] = x[i + 1] + a; }
            else if constexpr (OP == 1) { x[i] = fmaf(x[i], x[i + 1], a); x[i + 1] = fmaf(x[i + 1], b, x[i]); }
            else if constexpr (OP == 2) { x[i] = x[i] * x[i + 1]; x[i + 1] = x[i + 1] * b; }
            else if constexpr (OP == 3) {
                float2 v = __fadd2_rn(make_float2(x[i], x[i + 1]), make_float2(a, b));
                x[i] = v.x; x[i + 1] = v.y;
            } else if constexpr (OP == 4) {
                float2 v = __ffma2_rn(make_float2(x[i], x[i + 1]), make_float2(a, b), make_float2(x[i + 1], x[i]));
                x[i] = v.x; x[i + 1] = v.y;
            } else if constexpr (OP == 5) {
                float2 v = __fmul2_rn(make_float2(x[i], x[i + 1]), make_float2(a, b));
                x[i] = v.x; x[i + 1] = v.y;
            } else if constexpr (OP == 6) { x[i] = fmaf(x[i], 1.0001f, x[i + 1]); x[i + 1] = fmaf(x[i + 1], 0.9999f, a); }
            else if constexpr (OP == 7) {  // packed with broadcast operand (complex multiply form)
                float2 v = __ffma2_rn(make_float2(x[i + 1], x[i + 1]), make_float2(a, b), make_float2(x[i], x[i + 1]));
                x[i] = v.x; x[i + 1] = v.y;
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float* o;
    cudaMalloc(&o, 4);
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const char* names[] = {"FADD", "FFMA(3reg)", "FMUL", "FADD2", "FFMA2", "FMUL2", "FFMA(imm)", "FFMA2(bcast)"};
    void (*ks[])(float*, float, float) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int op = 0; op < 8; ++op) {
        const int blocks = sms * 8, threads = 256;
        ks[op]<<<blocks, threads>>>(o, 1.0001f, 0.9999f);
        cudaEventRecord(e0);
        ks[op]<<<blocks, threads>>>(o, 1.0001f, 0.9999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        // scalar ops: 16 per inner iteration; packed: 8 instructions (16 lanes of work)
        const bool packed = (op == 3 || op == 4 || op == 5 || op == 7);
        const double instr = (double)blocks * threads / 32 * ITERS * (packed ? 8 : 16);
        const double cyc = ms * 1e-3 * clk * 1e3;  // at the nominal max clock
        printf("%-14s warp-instr/clk/SM %.2f  fp32-lane-ops/clk/SM %.1f  (%.3f ms)\n", names[op], instr / cyc / sms,
               instr * 32 * (packed ? 2 : 1) / cyc / sms, ms);
    }
    return 0;
}
