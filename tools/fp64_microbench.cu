// FP64 pipe microbenchmarks on the box (not part of the library):
//   1. dependent-chain latency of DFMA / DADD / DMUL (one warp, clock64)
//   2. DFMA throughput per SM vs chains per thread (ILP) and warps per SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_microbench tools/fp64_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void latency_kernel(double* out, long long* cycles, int iters) {
    double a = out[0], b = 0.9999999, c = 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if (OP == 0) a = fma(a, b, c);
            if (OP == 1) a = a + c;
            if (OP == 2) a = a * b;
        }
    }
    long long t1 = clock64();
    out[1] = a;
    if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

template <int ILP>
__global__ void throughput_kernel(double* out, long long* cycles, int iters) {
    double a[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) a[k] = out[0] + k;
    const double b = 0.9999999, c = 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 64 / ILP; ++r) {
#pragma unroll
            for (int k = 0; k < ILP; ++k) a[k] = fma(a[k], b, c);
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += a[k];
    if (s == 1.2345) out[1] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

int main() {
    double* d;
    long long* cyc;
    cudaMalloc(&d, 16);
    cudaMalloc(&cyc, 8);
    double one = 1.0;
    cudaMemcpy(d, &one, 8, cudaMemcpyHostToDevice);
    long long h;
    const int iters = 1000;
    const char* names[3] = {"DFMA", "DADD", "DMUL"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) latency_kernel<0><<<1, 32>>>(d, cyc, iters);
            if (op == 1) latency_kernel<1><<<1, 32>>>(d, cyc, iters);
            if (op == 2) latency_kernel<2><<<1, 32>>>(d, cyc, iters);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("latency %s: %.2f cycles\n", names[op], double(h) / (iters * 32));
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps = 4; warps <= 32; warps *= 2) {
        for (int ilp : {1, 2, 4, 8}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            const int threads = 32 * warps;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (ilp == 1) throughput_kernel<1><<<sms, threads>>>(d, cyc, iters);
                if (ilp == 2) throughput_kernel<2><<<sms, threads>>>(d, cyc, iters);
                if (ilp == 4) throughput_kernel<4><<<sms, threads>>>(d, cyc, iters);
                if (ilp == 8) throughput_kernel<8><<<sms, threads>>>(d, cyc, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = double(sms) * threads * iters * 64.0;
            printf("warps/SM %2d ILP %d: %.2f DFMA lane-ops/cycle/SM (clock64), %.2f Tops/s\n",
                   warps, ilp, double(threads) * iters * 64.0 / double(h), ops / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
