// Host -> device copy rates of PAGEABLE memory on this box (the e2e leg uploads 18 GB of reference
// arrays per call): pinned DMA ceiling, staged copies with T threads, cudaHostRegister in place.
//   nvcc -O2 -o /tmp/upload_probe tools/upload_probe.cu && /tmp/upload_probe [GB]
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); exit(1);} } while (0)
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
    size_t gb = argc > 1 ? atoi(argv[1]) : 4;
    size_t bytes = gb << 30;
    char* src = (char*)malloc(bytes);
    memset(src, 1, bytes);
    char* dst; CK(cudaMalloc(&dst, bytes));
    // (1) pinned ceiling
    {
        char* pin; size_t pb = 1ull << 30; CK(cudaMallocHost(&pin, pb)); memset(pin, 2, pb);
        CK(cudaMemcpy(dst, pin, pb, cudaMemcpyHostToDevice));
        double t0 = now();
        for (int i = 0; i < 4; ++i) CK(cudaMemcpy(dst, pin, pb, cudaMemcpyHostToDevice));
        printf("pinned H2D: %.1f GB/s\n", 4.0 * pb / (now() - t0) / 1e9);
        CK(cudaFreeHost(pin));
    }
    // (2) plain pageable cudaMemcpy
    { double t0 = now(); CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)); printf("pageable cudaMemcpy: %.1f GB/s\n", bytes / (now() - t0) / 1e9); }
    // (3) host memcpy rate alone with T threads (pageable -> pinned ring, no DMA)
    for (int T : {1, 4, 8, 16}) {
        std::vector<char*> ring(T);
        for (auto& p : ring) CK(cudaMallocHost(&p, 8 << 20));
        double t0 = now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
            for (size_t o = (size_t)t * (4 << 20); o + (4 << 20) <= bytes; o += (size_t)T * (4 << 20)) memcpy(ring[t], src + o, 4 << 20);
        });
        for (auto& x : th) x.join();
        printf("host memcpy only, %2d threads: %.1f GB/s\n", T, bytes / (now() - t0) / 1e9);
        for (auto& p : ring) cudaFreeHost(p);
    }
    // (4) staged: T threads, 2 slots each of C MB
    for (int T : {4, 8, 16}) for (int C : {2, 4}) {
        size_t cb = (size_t)C << 20;
        std::vector<char*> ring(2 * T); std::vector<cudaEvent_t> ev(2 * T); std::vector<cudaStream_t> st(T);
        for (auto& p : ring) CK(cudaMallocHost(&p, cb));
        for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        double t0 = now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
            int turn = 0;
            for (size_t o = (size_t)t * cb; o < bytes; o += (size_t)T * cb, ++turn) {
                int slot = 2 * t + (turn & 1);
                if (turn >= 2) cudaEventSynchronize(ev[slot]);
                size_t n = std::min(cb, bytes - o);
                memcpy(ring[slot], src + o, n);
                cudaMemcpyAsync(dst + o, ring[slot], n, cudaMemcpyHostToDevice, st[t]);
                cudaEventRecord(ev[slot], st[t]);
            }
            cudaStreamSynchronize(st[t]);
        });
        for (auto& x : th) x.join();
        printf("staged %2d threads x %d MB: %.1f GB/s\n", T, C, bytes / (now() - t0) / 1e9);
        for (auto& p : ring) cudaFreeHost(p);
        for (auto& e : ev) cudaEventDestroy(e);
        for (auto& s : st) cudaStreamDestroy(s);
    }
    // (5) register in place: T threads, each registers a C MB piece, DMA, unregister
    for (int T : {1, 2, 4, 8}) for (int C : {64, 256}) {
        size_t cb = (size_t)C << 20;
        std::vector<cudaStream_t> st(T);
        for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        double t0 = now();
        std::vector<std::thread> th;
        std::vector<int> bad(T, 0);
        for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
            for (size_t o = (size_t)t * cb; o < bytes; o += (size_t)T * cb) {
                size_t n = std::min(cb, bytes - o);
                if (cudaHostRegister(src + o, n, cudaHostRegisterDefault) != cudaSuccess) { bad[t] = 1; cudaGetLastError(); return; }
                cudaMemcpyAsync(dst + o, src + o, n, cudaMemcpyHostToDevice, st[t]);
                cudaStreamSynchronize(st[t]);
                cudaHostUnregister(src + o);
            }
        });
        for (auto& x : th) x.join();
        int b = 0; for (int x : bad) b |= x;
        printf("register-in-place %d threads x %3d MB: %.1f GB/s%s\n", T, C, bytes / (now() - t0) / 1e9, b ? " (FAILED)" : "");
        for (auto& s : st) cudaStreamDestroy(s);
    }
    return 0;
}
