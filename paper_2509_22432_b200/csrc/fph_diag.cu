// fph_diag.cu -- FP32 throughput microbenchmark: the roofline denominator
// for the FFMA2-bound flooding kernel (MEASURED_PEAKS.json carries only HBM
// and bf16 tensor peaks).  Independent fma.rn.f32x2 chains, 4 flop each.
#include "fph_flood.cuh"

namespace fph {

namespace {

__global__ void __launch_bounds__(256) ffma2_burn(float* out, int iters, float seed) {
    float2 acc[8];
    float2 mul = make_float2(0.9999f, 1.0001f);
    float2 add = make_float2(1e-7f * seed, -1e-7f);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, seed + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = ffma2(acc[i], mul, add);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

}  // namespace

double ffma2_peak_tflops(int device) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        return 0.0;
    float* d = nullptr;
    if (cudaMalloc(&d, sizeof(float)) != cudaSuccess) return 0.0;
    const int blocks = sms * 8, iters = 1 << 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    ffma2_burn<<<blocks, 256>>>(d, 1024, 1.f);  // warm up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        ffma2_burn<<<blocks, 256>>>(d, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    double flop = (double)blocks * 256 * iters * 8 * 4;
    return flop / (best * 1e-3) / 1e12;
}

}  // namespace fph
