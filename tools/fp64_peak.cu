// FP64 issue ceiling of this B200: dependent-free DFMA chains, timed with CUDA events.
// The f64 P2G/G2P are co-limited by FP64 issue; bench.py scores them against the
// number this writes (profiles/fp64_peak.json) instead of the datasheet's 37 TFLOP/s.
// Build + run (one GPU):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/fp64_peak tools/fp64_peak.cu
//   gpurun_out/fp64_peak > gpurun_out/fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;  // independent accumulators per thread (covers the DFMA latency)
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) k_dfma(double* out, double b, double c)
{
    double a[CHAINS];
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
        a[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < CHAINS; ++j)
            a[j] = fma(a[j], b, c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
        s += a[j];
    if (s == 12345.678) // never true: keeps the chains live
        out[0] = s;
}

int main()
{
    int dev = 0, nsm = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    int best_per_sm = 0;
    for (int per_sm : {4, 8}) {
        const int blocks = nsm * per_sm;
        k_dfma<<<blocks, 256>>>(out, 0.999999, 1e-7); // warm-up
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0);
            k_dfma<<<blocks, 256>>>(out, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * CHAINS * ITERS * double(blocks) * 256;
            const double tf = flops / (ms * 1e-3) / 1e12;
            if (tf > best) {
                best = tf;
                best_per_sm = per_sm;
            }
        }
    }
    if (cudaGetLastError() != cudaSuccess) {
        fprintf(stderr, "fp64_peak: CUDA error\n");
        return 1;
    }
    printf("{\"fp64_tflops\": %.3f, \"ctas_per_sm\": %d, \"sms\": %d, \"clock_attr_mhz\": %d, "
           "\"how\": \"DFMA chains (%d per thread, %d iterations), 256-thread CTAs, best of 10 by CUDA events; "
           "2 flops per DFMA\"}\n",
           best, best_per_sm, nsm, clk / 1000, CHAINS, ITERS);
    return 0;
}
