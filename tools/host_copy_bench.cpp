// Host-side copy microbenchmark for the e2e pipeline's drain / fill legs:
// pinned staging buffer <-> pageable store, T threads, with and without
// first-touch, transparent huge pages and non-temporal stores.
// build: g++ -O3 -march=native -pthread tools/host_copy_bench.cpp -I/usr/local/cuda/include \
//          -L/usr/local/cuda/lib64 -lcudart -o /tmp/hcb
// usage: /tmp/hcb MB threads
#include <cuda_runtime.h>
#include <immintrin.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void copy_nt(char* dst, const char* src, size_t n) {
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63)) { dst[i] = src[i]; ++i; }
    for (; i + 64 <= n; i += 64) {
        __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}

template <class F>
static double par(int T, size_t n, F f) {
    std::vector<std::thread> th;
    const double t0 = now_ms();
    const size_t chunk = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        size_t a = std::min(n, t * chunk), b = std::min(n, a + chunk);
        th.emplace_back([=] { f(a, b); });
    }
    for (auto& x : th) x.join();
    return now_ms() - t0;
}

static char* fresh(size_t n, bool huge) {
    void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) { perror("mmap"); std::exit(1); }
    if (huge) madvise(p, n, MADV_HUGEPAGE);
    return static_cast<char*>(p);
}

int main(int argc, char** argv) {
    const size_t n = size_t(argc > 1 ? atol(argv[1]) : 2048) << 20;
    const int T = argc > 2 ? atoi(argv[2]) : 16;
    char* pin = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&pin), n, cudaHostAllocDefault) != cudaSuccess) {
        std::printf("cudaHostAlloc failed\n");
        return 1;
    }
    std::memset(pin, 1, n);
    const double gb = n / 1e9;
    auto report = [&](const char* what, double ms) {
        std::printf("%-44s %8.1f ms  %6.1f GB/s\n", what, ms, gb / (ms * 1e-3));
    };
    for (int huge = 0; huge < 2; ++huge) {
        for (int nt = 0; nt < 2; ++nt) {
            char* d = fresh(n, huge);
            char label[96];
            std::snprintf(label, sizeof label, "pinned->fresh   huge=%d nt=%d T=%d", huge, nt, T);
            report(label, par(T, n, [&](size_t a, size_t b) {
                       nt ? copy_nt(d + a, pin + a, b - a) : (void)std::memcpy(d + a, pin + a, b - a);
                   }));
            std::snprintf(label, sizeof label, "pinned->touched huge=%d nt=%d T=%d", huge, nt, T);
            report(label, par(T, n, [&](size_t a, size_t b) {
                       nt ? copy_nt(d + a, pin + a, b - a) : (void)std::memcpy(d + a, pin + a, b - a);
                   }));
            std::snprintf(label, sizeof label, "touched->pinned huge=%d nt=%d T=%d", huge, nt, T);
            report(label, par(T, n, [&](size_t a, size_t b) {
                       nt ? copy_nt(pin + a, d + a, b - a) : (void)std::memcpy(pin + a, d + a, b - a);
                   }));
            munmap(d, n);
        }
        char* d = fresh(n, huge);
        char label[96];
        std::snprintf(label, sizeof label, "first-touch memset huge=%d T=%d", huge, T);
        report(label, par(T, n, [&](size_t a, size_t b) { std::memset(d + a, 0, b - a); }));
        std::snprintf(label, sizeof label, "first-touch memset huge=%d T=1", huge);
        munmap(d, n);
        d = fresh(n, huge);
        report(label, par(1, n, [&](size_t a, size_t b) { std::memset(d + a, 0, b - a); }));
        munmap(d, n);
    }
    // direct DMA from / to registered pageable memory (no staging copy)
    void* dev = nullptr;
    if (cudaMalloc(&dev, n) != cudaSuccess) { std::printf("cudaMalloc failed\n"); return 1; }
    for (int huge = 0; huge < 2; ++huge) {
        for (int touched = 0; touched < 2; ++touched) {
            char* d = fresh(n, huge);
            if (touched) par(T, n, [&](size_t a, size_t b) { std::memset(d + a, 0, b - a); });
            char label[96];
            double t0 = now_ms();
            cudaError_t e = cudaHostRegister(d, n, cudaHostRegisterDefault);
            std::snprintf(label, sizeof label, "hostRegister huge=%d touched=%d (%s)", huge, touched,
                          cudaGetErrorName(e));
            report(label, now_ms() - t0);
            t0 = now_ms();
            cudaMemcpy(dev, d, n, cudaMemcpyHostToDevice);
            std::snprintf(label, sizeof label, "  H2D from registered huge=%d", huge);
            report(label, now_ms() - t0);
            t0 = now_ms();
            cudaMemcpy(d, dev, n, cudaMemcpyDeviceToHost);
            std::snprintf(label, sizeof label, "  D2H to registered huge=%d", huge);
            report(label, now_ms() - t0);
            t0 = now_ms();
            cudaHostUnregister(d);
            std::snprintf(label, sizeof label, "  hostUnregister huge=%d", huge);
            report(label, now_ms() - t0);
            munmap(d, n);
        }
    }
    double t0 = now_ms();
    cudaMemcpy(dev, pin, n, cudaMemcpyHostToDevice);
    report("H2D from pinned", now_ms() - t0);
    t0 = now_ms();
    cudaMemcpy(pin, dev, n, cudaMemcpyDeviceToHost);
    report("D2H to pinned", now_ms() - t0);
    {
        char* d = fresh(n, 0);
        par(T, n, [&](size_t a, size_t b) { std::memset(d + a, 0, b - a); });
        t0 = now_ms();
        cudaMemcpy(dev, d, n, cudaMemcpyHostToDevice);
        report("H2D from pageable (driver staged)", now_ms() - t0);
        t0 = now_ms();
        cudaMemcpy(d, dev, n, cudaMemcpyDeviceToHost);
        report("D2H to pageable (driver staged)", now_ms() - t0);
        munmap(d, n);
    }
    cudaFree(dev);
    cudaFreeHost(pin);
    return 0;
}
