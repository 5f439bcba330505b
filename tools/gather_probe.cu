// Micro-benchmark: dependent random 32-byte record gathers from a table larger than L2, with the
// load-instruction variants available on sm_100a. Answers "how many DRAM bytes does one 32-byte
// random read cost, and which load form keeps it at one sector" (profiles/README.md, K1 notes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gather_probe gather_probe.cu
//   ./gather_probe [table_MB] [fetch_granularity]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

struct __align__(32) Rec {
    uint64_t a, b, c, d;
};

template <int V>
__device__ __forceinline__ void load(const Rec* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                     uint64_t& d) {
    if (V == 0)
        asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    else if (V == 1)
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    else if (V == 2) {
        asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2+16];" : "=l"(c), "=l"(d) : "l"(p));
    } else if (V == 3)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    else if (V == 4) {
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2+16];" : "=l"(c), "=l"(d) : "l"(p));
    } else if (V == 5) {
        asm volatile("ld.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        asm volatile("ld.global.v2.u64 {%0,%1}, [%2+16];" : "=l"(c), "=l"(d) : "l"(p));
    } else if (V == 6) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2+16];" : "=l"(c), "=l"(d) : "l"(p));
    } else if (V == 7) {  // only 16 bytes of the record
        asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        c = d = 0;
    } else if (V == 8)
        asm volatile("ld.global.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 29;
    return x;
}

template <int V>
__global__ void __launch_bounds__(256) chase(const Rec* __restrict__ t, uint64_t n, int steps,
                                             uint64_t* out) {
    uint64_t x = mix(blockIdx.x * 256ull + threadIdx.x + 1);
    uint64_t acc = 0;
    for (int i = 0; i < steps; ++i) {
        uint64_t a, b, c, d;
        load<V>(t + (x % n), a, b, c, d);
        acc += b ^ c ^ d;
        x = mix(x + a);
    }
    if (acc == 0x1234567) out[0] = x;
}

__global__ void fill(Rec* t, uint64_t n) {
    uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < n) t[i] = Rec{mix(i + 77), i, i * 3, i * 5};
}

template <int V>
void run(const char* name, const Rec* t, uint64_t n, uint64_t* out) {
    const int blocks = 148 * 8, steps = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chase<V><<<blocks, 256>>>(t, n, 16, out);
    cudaEventRecord(e0);
    chase<V><<<blocks, 256>>>(t, n, steps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double loads = (double)blocks * 256 * steps;
    printf("%-44s %8.3f ms  %7.2f G loads/s  %7.1f GB/s useful (32 B/load)  err=%s\n", name, ms,
           loads / ms / 1e6, loads * 32 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    uint64_t mb = argc > 1 ? strtoull(argv[1], nullptr, 10) : 512;
    if (argc > 2) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[2]));
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("fetch granularity request %s -> %s, now %zu\n", argv[2], cudaGetErrorString(e), got);
    }
    uint64_t n = mb * 1024 * 1024 / sizeof(Rec);
    Rec* t;
    uint64_t* out;
    cudaMalloc(&t, n * sizeof(Rec));
    cudaMalloc(&out, 8);
    fill<<<(unsigned)((n + 255) / 256), 256>>>(t, n);
    cudaDeviceSynchronize();
    printf("table %llu MB, %llu records\n", (unsigned long long)mb, (unsigned long long)n);
    run<0>("v0 ld.global.nc.v4.u64", t, n, out);
    run<1>("v1 ld.global.v4.u64", t, n, out);
    run<2>("v2 2x ld.global.nc.v2.u64", t, n, out);
    run<3>("v3 ld.global.nc.L1::no_allocate.v4.u64", t, n, out);
    run<4>("v4 2x ld.global.cg.v2.u64", t, n, out);
    run<5>("v5 2x ld.global.v2.u64", t, n, out);
    run<6>("v6 2x ld.global.nc.L1::no_allocate.v2.u64", t, n, out);
    run<7>("v7 1x ld.global.nc.v2.u64 (16 B only)", t, n, out);
    run<8>("v8 ld.global.L1::no_allocate.v4.u64", t, n, out);
    return 0;
}
