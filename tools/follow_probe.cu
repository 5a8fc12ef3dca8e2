// follow_probe.cu -- diagnostic micro-benchmark (not part of the library): what limits the
// converging path's follow walk on an L2-resident table (cfg5: 1024 states x 256 symbols,
// u16 entries, 512 KiB)?  One dependent lookup per input byte per chain:
//     e = tab[c * 1024 + (e & 1023)]
// Swept: chains per thread C (ILP), threads per SM (TLP), and where the symbol c comes from:
//   IN = 0  per-thread LCG (no input stream at all: the pure gather)
//   IN = 1  thread-per-chain stream of 16-byte loads, ld.global.nc.L1::no_allocate (the kernel's)
//   IN = 2  the same loads, default caching (allocate in L1)
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o follow_probe follow_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ld_na(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int C, int IN, int PF>
__global__ void __launch_bounds__(512) flw(const uint16_t* __restrict__ tab, const uint8_t* __restrict__ in, uint64_t L,
                                            uint32_t nvec, uint32_t* sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e[C], h[C], rng[C];
    const uint8_t* p[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        e[k] = (uint32_t)(tid * 2654435761u + 977u * k) & 1023u;
        h[k] = 0;
        rng[k] = (uint32_t)tid * 747796405u + 2891336453u * (k + 1);
        p[k] = in + (tid * C + k) * L;
    }
    uint4 ring[C][PF];
    if (IN)
#pragma unroll
        for (int k = 0; k < C; ++k)
#pragma unroll
            for (int u = 0; u < PF; ++u) ring[k][u] = IN == 1 ? ld_na(p[k] + 16 * u) : __ldg((const uint4*)(p[k] + 16 * u));
    for (uint32_t v = 0; v < nvec; v += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            uint32_t w[C][4];
#pragma unroll
            for (int k = 0; k < C; ++k) {
                if (IN) {
                    const uint4 x = ring[k][u];
                    w[k][0] = x.x; w[k][1] = x.y; w[k][2] = x.z; w[k][3] = x.w;
                    if (v + u + PF < nvec)
                        ring[k][u] = IN == 1 ? ld_na(p[k] + 16ull * (v + u + PF)) : __ldg((const uint4*)(p[k] + 16ull * (v + u + PF)));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        rng[k] = rng[k] * 1664525u + 1013904223u;
                        w[k][q] = rng[k] ^ (rng[k] >> 15);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (uint32_t b = 0; b < 4; ++b)
#pragma unroll
                    for (int k = 0; k < C; ++k) {
                        const uint32_t c = __byte_perm(w[k][q], 0u, 0x4440u | b);
                        e[k] = __ldg(tab + c * 1024u + (e[k] & 1023u));
                        h[k] += e[k] >> 15;
                    }
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= e[k] + h[k];
    if (a == sink[1]) sink[0] = a;
}


// pure gather (IN = 0 style) over a table of S states x 256 symbols (u16): L1-resident to L2-resident
__global__ void __launch_bounds__(512) sized(const uint16_t* __restrict__ tab, uint32_t S, uint32_t steps, uint32_t* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e = (tid * 2654435761u) & (S - 1u), h = 0, rng = tid * 747796405u + 2891336453u;
    for (uint32_t s = 0; s < steps; ++s) {
        rng = rng * 1664525u + 1013904223u;
        const uint32_t c = rng >> 24;
        e = __ldg(tab + c * S + (e & (S - 1u)));
        h += e >> 15;
    }
    if (e + h == sink[1]) sink[0] = e;
}

// branch-free hybrid: columns < CS in shared memory, the rest in global memory; lanes served
// from shared memory aim their global load at ONE dummy address (a single wavefront for all of
// them), lanes served from global memory aim their shared load at offset 0 (a broadcast)
template <int C>
__global__ void __launch_bounds__(512) hyb(const uint16_t* __restrict__ tab, uint32_t CS, uint32_t steps, uint32_t* sink) {
    extern __shared__ __align__(16) uint16_t hs[];
    for (uint32_t i = threadIdx.x; i < CS * 1024u; i += blockDim.x) hs[i] = tab[i];
    __syncthreads();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e[C], h[C], rng[C];
#pragma unroll
    for (int k = 0; k < C; ++k) { e[k] = (tid * 2654435761u + 977u * k) & 1023u; h[k] = 0; rng[k] = tid * 747796405u + 2891336453u * (k + 1); }
    const uint32_t lim = CS * 1024u;
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            rng[k] = rng[k] * 1664525u + 1013904223u;
            const uint32_t idx = (rng[k] >> 24) * 1024u + (e[k] & 1023u);
            const bool insm = idx < lim;
            const uint32_t vg = __ldg(tab + (insm ? lim : idx));
            const uint32_t vs = hs[insm ? idx : 0u];
            e[k] = insm ? vs : vg;
            h[k] += e[k] >> 15;
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= e[k] + h[k];
    if (a == sink[1]) sink[0] = a;
}


// cache-hint variants of the pure gather (S states x 256 symbols)
template <int H>
__device__ __forceinline__ uint32_t ldh(const uint16_t* p) {
    unsigned short v;
    if (H == 0) asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
    if (H == 1) asm volatile("ld.global.nc.L2::128B.u16 %0, [%1];" : "=h"(v) : "l"(p));
    if (H == 2) asm volatile("ld.global.nc.L1::evict_last.u16 %0, [%1];" : "=h"(v) : "l"(p));
    if (H == 3) asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
    if (H == 4) asm volatile("ld.global.nc.L1::evict_last.L2::128B.u16 %0, [%1];" : "=h"(v) : "l"(p));
    if (H == 5) asm volatile("ld.global.nc.L2::256B.u16 %0, [%1];" : "=h"(v) : "l"(p));
    if (H == 6) asm volatile("ld.global.nc.L2::64B.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
template <int H>
__global__ void __launch_bounds__(512) hinted(const uint16_t* __restrict__ tab, uint32_t S, uint32_t steps, uint32_t* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e = (tid * 2654435761u) & (S - 1u), h = 0, rng = tid * 747796405u + 2891336453u;
    for (uint32_t s = 0; s < steps; ++s) {
        rng = rng * 1664525u + 1013904223u;
        const uint32_t c = rng >> 24;
        e = ldh<H>(tab + c * S + (e & (S - 1u)));
        h += e >> 15;
    }
    if (e + h == sink[1]) sink[0] = e;
}
template <int H>
static void run_hinted(const uint16_t* big, uint32_t S, int sms, double ghz, uint32_t* sink) {
    for (int tps : {512, 1024}) {
        const uint32_t steps = 8192;
        CK(cudaFuncSetAttribute(hinted<H>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
        hinted<H><<<sms * tps / 512, 512>>>(big, S, steps, sink);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        hinted<H><<<sms * tps / 512, 512>>>(big, S, steps, sink);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double lk = (double)sms * tps * steps;
        printf("hint %d table %4u KiB thr/SM %4d : %.3f Tlookup/s  %.2f lookups/clk/SM\n", H, 256 * S * 2 / 1024, tps, lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9));
    }
}


// packed hybrid: 10-bit entries, 3 per 32-bit word (342 words per symbol column of 1024 states);
// the first WS words of every ... simpler: columns c < CS live in shared memory (packed), the
// rest are read from the plain u16 table in global memory.  Branch-free selection as in hyb.
template <int C>
__global__ void __launch_bounds__(512) pk(const uint16_t* __restrict__ tab, const uint32_t* __restrict__ ptab, uint32_t CS, uint32_t steps, uint32_t* sink) {
    extern __shared__ __align__(16) uint32_t ps[];
    for (uint32_t i = threadIdx.x; i < CS * 342u; i += blockDim.x) ps[i] = ptab[i];
    __syncthreads();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e[C], h[C], rng[C];
#pragma unroll
    for (int k = 0; k < C; ++k) { e[k] = (tid * 2654435761u + 977u * k) & 1023u; h[k] = 0; rng[k] = tid * 747796405u + 2891336453u * (k + 1); }
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            rng[k] = rng[k] * 1664525u + 1013904223u;
            const uint32_t c = rng[k] >> 24, st = e[k] & 1023u;
            const bool insm = c < CS;
            const uint32_t q = (st * 43691u) >> 17, r = st - 3u * q;
            const uint32_t vg = __ldg(tab + (insm ? 0u : c * 1024u + st));
            const uint32_t w = ps[insm ? c * 342u + q : 0u];
            const uint32_t vs = (w >> (r * 10u)) & 1023u;
            e[k] = insm ? vs : (vg & 1023u);
            h[k] += e[k] < 100u;
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= e[k] + h[k];
    if (a == sink[1]) sink[0] = a;
}

// packed table entirely in global memory (10-bit entries, 3 per word: 342 KiB instead of 512 KiB
// -- does the smaller footprint raise the L1 hit rate enough to pay for the unpacking?)
__global__ void __launch_bounds__(512) pkg(const uint32_t* __restrict__ ptab, uint32_t steps, uint32_t* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e = (tid * 2654435761u) & 1023u, h = 0, rng = tid * 747796405u + 2891336453u;
    for (uint32_t s = 0; s < steps; ++s) {
        rng = rng * 1664525u + 1013904223u;
        const uint32_t c = rng >> 24;
        const uint32_t q = (e * 43691u) >> 17, r = e - 3u * q;
        const uint32_t w = __ldg(ptab + c * 342u + q);
        e = (w >> (r * 10u)) & 1023u;
        h += e < 100u;
    }
    if (e + h == sink[1]) sink[0] = e;
}

// packed hybrid fed by the real input stream: thread-per-chain 16-byte loads (no L1 allocation),
// PF vectors in flight per chain -- does the small L1 left beside a 128-192 KiB table starve it?
template <int C, int PF>
__global__ void __launch_bounds__(512) pk_in(const uint16_t* __restrict__ tab, const uint32_t* __restrict__ ptab, uint32_t CS,
                                              const uint8_t* __restrict__ in, uint64_t L, uint32_t nvec, uint32_t* sink) {
    extern __shared__ __align__(16) uint32_t ps[];
    for (uint32_t i = threadIdx.x; i < CS * 342u; i += blockDim.x) ps[i] = ptab[i];
    __syncthreads();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e[C], h[C];
    const uint8_t* p[C];
    uint4 ring[C][PF];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        e[k] = (uint32_t)(tid * 2654435761u + 977u * k) & 1023u;
        h[k] = 0;
        p[k] = in + (tid * C + k) * L;
#pragma unroll
        for (int u = 0; u < PF; ++u) ring[k][u] = ld_na(p[k] + 16 * u);
    }
    for (uint32_t v = 0; v < nvec; v += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            uint32_t w[C][4];
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const uint4 x = ring[k][u];
                w[k][0] = x.x; w[k][1] = x.y; w[k][2] = x.z; w[k][3] = x.w;
                if (v + u + PF < nvec) ring[k][u] = ld_na(p[k] + 16ull * (v + u + PF));
            }
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (uint32_t b = 0; b < 4; ++b)
#pragma unroll
                    for (int k = 0; k < C; ++k) {
                        const uint32_t c = __byte_perm(w[k][q4], 0u, 0x4440u | b), st = e[k];
                        const bool insm = c < CS;
                        const uint32_t q = (st * 43691u) >> 17, r = st - 3u * q;
                        const uint32_t vg = __ldg(tab + (insm ? 0u : c * 1024u + st));
                        const uint32_t ww = ps[insm ? c * 342u + q : 0u];
                        const uint32_t vs = (ww >> (r * 10u)) & 1023u;
                        e[k] = insm ? vs : (vg & 1023u);
                        h[k] += e[k] < 100u;
                    }
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= e[k] + h[k];
    if (a == sink[1]) sink[0] = a;
}

template <int C, int PF>
static void run_pk_in(const uint16_t* tab, const uint32_t* ptab, uint32_t CS, const uint8_t* in, uint64_t nin, int sms, uint32_t* sink, double ghz) {
    const size_t smem = (size_t)CS * 342 * 4 + 16;
    CK(cudaFuncSetAttribute(pk_in<C, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint64_t chains = (uint64_t)sms * 512 * C;
    uint64_t L = nin / chains;
    if (L > 16384) L = 16384;
    L &= ~(uint64_t)63;
    if (L % 128 == 0) L -= 16;
    const uint32_t nvec = (uint32_t)(L / 16) / PF * PF;
    pk_in<C, PF><<<sms, 512, smem>>>(tab, ptab, CS, in, L, nvec, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    pk_in<C, PF><<<sms, 512, smem>>>(tab, ptab, CS, in, L, nvec, sink);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double lk = (double)chains * nvec * 16;
    printf("packed+input CS %3u (%3zu KiB smem) thr/SM 512 C %d PF %d : %.3f Tlookup/s  %.2f lookups/clk/SM\n", CS, smem / 1024, C, PF,
           lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9));
    fflush(stdout);
}

static uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_bytes(uint8_t* p, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 8; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull + 12345;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        reinterpret_cast<uint64_t*>(p)[i] = z ^ (z >> 31);
    }
}

template <int C, int IN, int PF>
static void run(const uint16_t* tab, const uint8_t* in, uint64_t nin, int sms, int thr_sm, int cta, uint32_t* sink, double ghz) {
    const int ctas = sms * (thr_sm / cta);
    const uint64_t chains = (uint64_t)ctas * cta * C;
    uint64_t L = nin / chains;
    if (L > 32768) L = 32768;
    L &= ~(uint64_t)63;
    if (L % 128 == 0) L -= 16;   // the kernel's stride rule
    const uint32_t nvec = (uint32_t)(L / 16) / PF * PF;
    CK(cudaFuncSetAttribute(flw<C, IN, PF>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    flw<C, IN, PF><<<ctas, cta>>>(tab, in, L, nvec, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) flw<C, IN, PF><<<ctas, cta>>>(tab, in, L, nvec, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 3;
    const double lk = (double)chains * nvec * 16;
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, flw<C, IN, PF>, cta, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, flw<C, IN, PF>);
    printf("regs %3d resident thr/SM %4d | ", fa.numRegs, bps * cta);
    printf("IN %d  C %d  PF %d  thr/SM %4d (cta %4d)  chains/SM %5d  L %6llu : %.3f Tlookup/s  %.2f lookups/clk/SM  %.3f ms\n", IN, C, PF,
           thr_sm, cta, thr_sm * C, (unsigned long long)L, lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9), ms);
    fflush(stdout);
}

int main() {
    int sms = 148, khz = 1965000;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = khz * 1e-6;
    const uint32_t entries = 256 * 1024;
    uint16_t* h = (uint16_t*)malloc(entries * 2);
    uint64_t s = 42;
    for (uint32_t i = 0; i < entries; ++i) h[i] = (uint16_t)(splitmix(s) & 0x83FF);
    uint16_t* tab;
    CK(cudaMalloc(&tab, entries * 2));
    CK(cudaMemcpy(tab, h, entries * 2, cudaMemcpyHostToDevice));
    const uint64_t nin = 4ull << 30;
    uint8_t* in;
    CK(cudaMalloc(&in, nin + 4096));
    fill_bytes<<<sms * 8, 256>>>(in, nin);
    uint32_t* sink;
    CK(cudaMalloc(&sink, 8));
    uint32_t hs[2] = {0, 0xFFFFFFFFu};
    CK(cudaMemcpy(sink, hs, 8, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    printf("SMs %d clock %.3f GHz\n", sms, ghz);
#define ROW(C, IN, PF)                                   \
    run<C, IN, PF>(tab, in, nin, sms, 512, 512, sink, ghz);  \
    run<C, IN, PF>(tab, in, nin, sms, 1024, 512, sink, ghz); \
    run<C, IN, PF>(tab, in, nin, sms, 2048, 512, sink, ghz);
    ROW(1, 0, 4)

    {
        uint16_t* big;
        const uint32_t be = 256u * 4096u;
        uint16_t* hb = (uint16_t*)malloc(be * 2);
        for (uint32_t S : {1024u}) {
            for (uint32_t i = 0; i < 256 * S; ++i) hb[i] = (uint16_t)((splitmix(s) & (S - 1)) | (splitmix(s) & 0x8000));
            CK(cudaMalloc(&big, be * 2));
            CK(cudaMemcpy(big, hb, 256 * S * 2, cudaMemcpyHostToDevice));
            run_hinted<0>(big, S, sms, ghz, sink); run_hinted<1>(big, S, sms, ghz, sink); run_hinted<2>(big, S, sms, ghz, sink);
            run_hinted<3>(big, S, sms, ghz, sink); run_hinted<4>(big, S, sms, ghz, sink); run_hinted<5>(big, S, sms, ghz, sink); run_hinted<6>(big, S, sms, ghz, sink);
            for (int tps : {512, 1024, 2048}) {
                const uint32_t steps = 8192;
                CK(cudaFuncSetAttribute(sized, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
                sized<<<sms * tps / 512, 512>>>(big, S, steps, sink);
                CK(cudaDeviceSynchronize());
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a);
                sized<<<sms * tps / 512, 512>>>(big, S, steps, sink);
                cudaEventRecord(b); CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b);
                const double lk = (double)sms * tps * steps;
                printf("sized table %4u KiB thr/SM %4d : %.3f Tlookup/s  %.2f lookups/clk/SM\n", 256 * S * 2 / 1024, tps, lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9));
            }
            CK(cudaFree(big));
        }
        free(hb);
    }
    for (uint32_t CS : {0u, 96u}) {
        for (int tps : {512}) {
            const size_t smem = (size_t)CS * 2048;
            const uint32_t steps = 8192;
            CK(cudaFuncSetAttribute(hyb<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem ? smem : 1)));
            CK(cudaFuncSetAttribute(hyb<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem ? smem : 1)));
            for (int C : {1, 2}) {
                const int ctas = sms;   // one CTA per SM (the table copy is per CTA)
                auto launch = [&]() { if (C == 1) hyb<1><<<ctas, tps, smem>>>(tab, CS, steps, sink); else hyb<2><<<ctas, tps, smem>>>(tab, CS, steps, sink); };
                launch();
                CK(cudaDeviceSynchronize());
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b); CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b);
                const double lk = (double)ctas * tps * C * steps;
                printf("hybrid CS %3u (%3zu KiB smem) thr/SM %4d C %d : %.3f Tlookup/s  %.2f lookups/clk/SM\n", CS, smem / 1024, tps, C, lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9));
            }
        }
    }

    {
        uint32_t* hp = (uint32_t*)malloc(256 * 342 * 4);
        for (uint32_t c = 0; c < 256; ++c)
            for (uint32_t q = 0; q < 342; ++q) {
                uint32_t w = 0;
                for (uint32_t r = 0; r < 3; ++r) { const uint32_t st = 3 * q + r; if (st < 1024) w |= (uint32_t)(h[c * 1024 + st] & 1023u) << (10 * r); }
                hp[c * 342 + q] = w;
            }
        uint32_t* ptab;
        CK(cudaMalloc(&ptab, 256 * 342 * 4));
        CK(cudaMemcpy(ptab, hp, 256 * 342 * 4, cudaMemcpyHostToDevice));
        for (int tps : {512, 1024}) {
            const uint32_t steps = 8192;
            CK(cudaFuncSetAttribute(pkg, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
            pkg<<<sms * tps / 512, 512>>>(ptab, steps, sink);
            CK(cudaDeviceSynchronize());
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            pkg<<<sms * tps / 512, 512>>>(ptab, steps, sink);
            cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double lk = (double)sms * tps * steps;
            printf("packed global (342 KiB) thr/SM %4d : %.3f Tlookup/s  %.2f lookups/clk/SM\n", tps, lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9));
        }
        for (uint32_t CS : {0u, 96u, 128u, 144u}) {
            run_pk_in<1, 4>(tab, ptab, CS, in, nin, sms, sink, ghz);
            run_pk_in<2, 2>(tab, ptab, CS, in, nin, sms, sink, ghz);
            run_pk_in<2, 4>(tab, ptab, CS, in, nin, sms, sink, ghz);
            run_pk_in<3, 2>(tab, ptab, CS, in, nin, sms, sink, ghz);
        }
        for (uint32_t CS : {0u, 144u}) {
            const size_t smem = (size_t)CS * 342 * 4 + 16;
            const uint32_t steps = 8192;
            CK(cudaFuncSetAttribute(pk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem ? smem : 1)));
            CK(cudaFuncSetAttribute(pk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem ? smem : 1)));
            for (int C : {1, 2}) {
                auto launch = [&]() { if (C == 1) pk<1><<<sms, 512, smem>>>(tab, ptab, CS, steps, sink); else pk<2><<<sms, 512, smem>>>(tab, ptab, CS, steps, sink); };
                launch();
                CK(cudaDeviceSynchronize());
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b); CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b);
                const double lk = (double)sms * 512 * C * steps;
                printf("packed CS %3u (%3zu KiB smem) thr/SM 512 C %d : %.3f Tlookup/s  %.2f lookups/clk/SM\n", CS, smem / 1024, C, lk / (ms * 1e-3) / 1e12, lk / (ms * 1e-3) / (sms * ghz * 1e9));
            }
        }
    }
    printf("done\n");
    return 0;
}
