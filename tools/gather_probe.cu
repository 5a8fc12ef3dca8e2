// gather_probe.cu -- diagnostic micro-benchmark (not part of the library): the rate of
// DEPENDENT random table lookups on B200, which bounds the converging path's follow walk
// (one lookup per input byte per chain) for the three places a large table can live:
//   glob<C>  : u16 table in global memory (L1/L2), C independent chains per thread;
//              swept over resident chains per SM (latency vs throughput curve)
//   dsmem<C> : the table striped over a thread-block cluster's shared memory, read with
//              mapa + ld.shared::cluster (the "stripe it across a cluster's DSMEM" option)
//   smem     : u16 random (bank conflicts) vs u8 lane-private ("bank-private": lane l's copy
//              lives in bank l only, conflict-free by construction)
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o gather_probe gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

static int g_sms = 148;
static double g_clk_ghz = 1.965;

template <int C, bool CG>
__global__ void glob_kernel(const uint16_t* __restrict__ tab, uint32_t mask, uint32_t steps, uint32_t* sink) {
    uint32_t x[C];
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = (tid * 2654435761u + 977u * k) & mask;
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            uint32_t v;
            if (CG) {
                unsigned short t;
                asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(t) : "l"(tab + x[k]));
                v = t;
            } else {
                v = __ldg(tab + x[k]);
            }
            x[k] = (v * 0x9E3779B1u + s) & mask;
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= x[k];
    if (a == sink[1]) sink[0] = a;   // sink[1] = 0xFFFFFFFF at run time
}

// cluster of CS CTAs; CTA r holds entries [r*slice, (r+1)*slice) of a u16 table
template <int C>
__global__ void dsmem_kernel(const uint16_t* __restrict__ tab, uint32_t slice_log2, uint32_t cs_log2, uint32_t steps,
                             uint32_t* sink) {
    extern __shared__ __align__(16) uint16_t st[];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t slice = 1u << slice_log2;
    for (uint32_t i = threadIdx.x; i < slice; i += blockDim.x) st[i] = tab[(rank << slice_log2) + i];
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(st);
    const uint32_t mask = (1u << (slice_log2 + cs_log2)) - 1u;
    uint32_t x[C];
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = (tid * 2654435761u + 977u * k) & mask;
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const uint32_t r = x[k] >> slice_log2, off = x[k] & (slice - 1u);
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + 2u * off), "r"(r));
            unsigned short t;
            asm volatile("ld.shared::cluster.u16 %0, [%1];" : "=h"(t) : "r"(ra));
            x[k] = ((uint32_t)t * 0x9E3779B1u + s) & mask;
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= x[k];
    if (a == sink[1]) sink[0] = a;   // sink[1] = 0xFFFFFFFF at run time
}

// shared memory: MODE 0 = u16 table, random (bank conflicts); MODE 1 = u8 lane-private
// (entry i of lane l at ((i >> 2) << 7) | l << 2 | (i & 3)); entries = 4096 (256 states x 16 columns)
template <int C, int MODE>
__global__ void smem_kernel(const uint16_t* __restrict__ tab, uint32_t entries, uint32_t steps, uint32_t* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t lane = threadIdx.x & 31u;
    if (MODE == 0) {
        uint16_t* t = reinterpret_cast<uint16_t*>(sm);
        for (uint32_t i = threadIdx.x; i < entries; i += blockDim.x) t[i] = tab[i];
    } else {
        for (uint32_t j = threadIdx.x; j < entries * 32u; j += blockDim.x) {
            const uint32_t l = j & 31u, i = j >> 5;
            sm[((i >> 2) << 7) | (l << 2) | (i & 3u)] = (uint8_t)tab[i];
        }
    }
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    uint32_t x[C];
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = (tid * 2654435761u + 977u * k) % entries;
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            uint32_t v;
            if (MODE == 0) {
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(base + 2u * x[k]));
                x[k] = (v * 0x9E3779B1u + s) & (entries - 1u);
            } else {
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(base + (((x[k] >> 2) << 7) | (lane << 2) | (x[k] & 3u))));
                x[k] = (((v ^ s) & 255u) | ((s + 5u * k) << 8)) & (entries - 1u);   // state v, column from s
            }
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= x[k];
    if (a == sink[1]) sink[0] = a;   // sink[1] = 0xFFFFFFFF at run time
}


// hybrid table: u16 entries [256 columns][1024 states]; columns < CS staged in shared memory,
// the rest read from global (L1/L2).  Next index = column(rand) * 1024 + state(entry).
template <int C>
__global__ void hybrid_kernel(const uint16_t* __restrict__ tab, uint32_t CS, uint32_t steps, uint32_t* sink) {
    extern __shared__ __align__(16) uint16_t hs[];
    for (uint32_t i = threadIdx.x; i < CS * 1024u; i += blockDim.x) hs[i] = tab[i];
    __syncthreads();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(hs);
    uint32_t st[C], cc[C];
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < C; ++k) { st[k] = (tid * 2654435761u + 977u * k) & 1023u; cc[k] = (tid * 40503u + k * 7u) & 255u; }
    for (uint32_t s = 0; s < steps; ++s) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const uint32_t idx = cc[k] * 1024u + st[k];
            uint32_t v;
            if (cc[k] < CS) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(sbase + 2u * idx));
            else v = __ldg(tab + idx);
            st[k] = v & 1023u;
            cc[k] = (cc[k] * 167u + s + 13u) & 255u;   // next symbol: a cheap sequence spread over 0..255
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) a ^= st[k];
    if (a == sink[1]) sink[0] = a;
}

// replicated 16-copy u16 fragments of a 256-state x 26-column table (the converging path's
// cfg3 follow layout): 6 ops per step as in the real kernel
template <int C>
__global__ void __launch_bounds__(1024, 1) rep16_kernel(const uint8_t* __restrict__ in, uint32_t steps, uint32_t* sink) {
    extern __shared__ __align__(16) unsigned char rs[];
    const uint32_t COL = 8192u;
    const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(rs);
    const uint32_t tbase = (sraw + COL - 1) / COL * COL;
    unsigned char* base = rs + (tbase - sraw);
    for (uint32_t i = threadIdx.x; i < 26u * 256u; i += blockDim.x) {
        const uint32_t c = i >> 8, s = i & 255u;
        const uint32_t d = (s * 97u + c * 31u + 7u) & 255u;
        for (uint32_t k = 0; k < 16; ++k) {
            const uint32_t f = ((s >> 2) << 7) | (((s >> 1) & 1u) << 6) | (k << 2) | ((s & 1u) << 1);
            const uint32_t fd = ((d >> 2) << 7) | (((d >> 1) & 1u) << 6) | (k << 2) | ((d & 1u) << 1);
            *reinterpret_cast<uint16_t*>(base + c * COL + f) = (uint16_t)(fd | ((d & 1u) << 15));
        }
    }
    __syncthreads();
    const uint32_t k16 = threadIdx.x & 15u;
    uint32_t e[C], h[C];
#pragma unroll
    for (int j = 0; j < C; ++j) { e[j] = (k16 << 2) | (j << 7); h[j] = 0; }
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint4* p = reinterpret_cast<const uint4*>(in) + (size_t)tid * C * (steps / 16);
    for (uint32_t v = 0; v < steps / 16; ++v) {
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const uint4 x = __ldg(p + (size_t)j * (steps / 16) + v);
            const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (uint32_t b = 0; b < 4; ++b) {
                    const uint32_t c = min(__byte_perm(w4[q], 0u, 0x4440u | b), 25u);
                    const uint32_t colc = c * COL + tbase;
                    uint32_t nv;
                    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(nv) : "r"((e[j] & 8191u) | colc));
                    e[j] = nv;
                    h[j] += nv >> 15;
                }
        }
    }
    uint32_t a = 0;
#pragma unroll
    for (int j = 0; j < C; ++j) a ^= e[j] + h[j];
    if (a == sink[1]) sink[0] = a;
}

static float time_launch(void (*launch)(void*), void* ctx, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch(ctx);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) launch(ctx);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

struct GlobCtx {
    const void* fn;
    unsigned grid, block;
    const uint16_t* tab;
    uint32_t mask, steps;
    uint32_t* sink;
};
static void glob_launch(void* p) {
    GlobCtx* c = (GlobCtx*)p;
    void* args[] = {(void*)&c->tab, (void*)&c->mask, (void*)&c->steps, (void*)&c->sink};
    CK(cudaLaunchKernel(c->fn, dim3(c->grid), dim3(c->block), args, 0, 0));
}

template <int C, bool CG>
static void run_glob(const uint16_t* tab, uint32_t entries, uint32_t* sink, int threads_per_sm) {
    GlobCtx c;
    c.fn = (const void*)glob_kernel<C, CG>;
    CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    c.block = 256;
    c.grid = g_sms * threads_per_sm / 256;
    c.tab = tab;
    c.mask = entries - 1;
    c.steps = 512;
    c.sink = sink;
    const float ms = time_launch(glob_launch, &c, 3);
    const double lk = (double)c.grid * c.block * C * c.steps;
    const double chains_sm = (double)threads_per_sm * C;
    printf("glob %s table %7u KiB  thr/SM %4d  C %d  chains/SM %5.0f : %7.3f Tlookup/s  step latency %6.0f cyc\n",
           CG ? "cg " : "nc ", entries * 2 / 1024, threads_per_sm, C, chains_sm, lk / (ms * 1e-3) / 1e12,
           ms * 1e-3 * g_clk_ghz * 1e9 / c.steps / C * C);
}

struct DsCtx {
    const void* fn;
    unsigned grid, block, cs;
    size_t smem;
    const uint16_t* tab;
    uint32_t sl, csl, steps;
    uint32_t* sink;
};
static void ds_launch(void* p) {
    DsCtx* c = (DsCtx*)p;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->grid);
    cfg.blockDim = dim3(c->block);
    cfg.dynamicSmemBytes = c->smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* args[] = {(void*)&c->tab, (void*)&c->sl, (void*)&c->csl, (void*)&c->steps, (void*)&c->sink};
    CK(cudaLaunchKernelExC(&cfg, c->fn, args));
}

template <int C>
static void run_dsmem(const uint16_t* tab, uint32_t table_log2, uint32_t cs_log2, uint32_t* sink, unsigned block) {
    DsCtx c;
    c.fn = (const void*)dsmem_kernel<C>;
    c.cs = 1u << cs_log2;
    c.sl = table_log2 - cs_log2;
    c.csl = cs_log2;
    c.smem = (size_t)2 << c.sl;
    CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
    if (c.cs > 8) CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    c.block = block;
    // as many clusters as fit: ask the occupancy API
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.cs);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = c.smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, c.fn, &cfg);
    if (e != cudaSuccess || ncl < 1) {
        printf("dsmem cluster %u: cannot launch (%s, %d clusters)\n", c.cs, cudaGetErrorString(e), ncl);
        cudaGetLastError();
        return;
    }
    c.grid = ncl * c.cs;
    c.tab = tab;
    c.steps = 512;
    c.sink = sink;
    const float ms = time_launch(ds_launch, &c, 3);
    const double lk = (double)c.grid * c.block * C * c.steps;
    printf("dsmem table %5u KiB cluster %2u (%3zu KiB/CTA) CTAs %4u thr/CTA %4u C %d : %7.3f Tlookup/s  step latency %6.0f cyc\n",
           (2u << table_log2) / 1024, c.cs, c.smem / 1024, c.grid, block, C, lk / (ms * 1e-3) / 1e12,
           ms * 1e-3 * g_clk_ghz * 1e9 / c.steps);
}

struct SmCtx {
    const void* fn;
    unsigned grid, block;
    size_t smem;
    const uint16_t* tab;
    uint32_t entries, steps;
    uint32_t* sink;
};
static void sm_launch(void* p) {
    SmCtx* c = (SmCtx*)p;
    void* args[] = {(void*)&c->tab, (void*)&c->entries, (void*)&c->steps, (void*)&c->sink};
    CK(cudaLaunchKernel(c->fn, dim3(c->grid), dim3(c->block), args, c->smem, 0));
}

template <int C, int MODE>
static void run_smem(const uint16_t* tab, uint32_t* sink, unsigned block) {
    SmCtx c;
    c.fn = (const void*)smem_kernel<C, MODE>;
    c.entries = 4096;   // 16 columns x 256 states
    c.smem = MODE == 0 ? 2 * 4096 : 4096 / 4 * 128;
    CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, c.fn, block, c.smem));
    c.grid = g_sms * bps;
    c.block = block;
    c.tab = tab;
    c.steps = 1024;
    c.sink = sink;
    const float ms = time_launch(sm_launch, &c, 3);
    const double lk = (double)c.grid * c.block * C * c.steps;
    printf("smem %s thr/SM %5u C %d : %7.3f Tlookup/s\n", MODE == 0 ? "u16 random      " : "u8 lane-private ",
           bps * block, C, lk / (ms * 1e-3) / 1e12);
}


struct HyCtx { const void* fn; unsigned grid, block; size_t smem; const uint16_t* tab; uint32_t CS, steps; uint32_t* sink; };
static void hy_launch(void* p) {
    HyCtx* c = (HyCtx*)p;
    void* args[] = {(void*)&c->tab, (void*)&c->CS, (void*)&c->steps, (void*)&c->sink};
    CK(cudaLaunchKernel(c->fn, dim3(c->grid), dim3(c->block), args, c->smem, 0));
}
template <int C>
static void run_hybrid(const uint16_t* tab, uint32_t CS, uint32_t* sink, unsigned block) {
    HyCtx c;
    c.fn = (const void*)hybrid_kernel<C>;
    c.smem = (size_t)CS * 2048;
    CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(c.smem ? c.smem : 1)));
    if (!c.smem) CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, c.fn, block, c.smem));
    if (bps > 2048 / (int)block) bps = 2048 / block;
    c.grid = g_sms * bps; c.block = block; c.tab = tab; c.CS = CS; c.steps = 1024; c.sink = sink;
    const float ms = time_launch(hy_launch, &c, 3);
    const double lk = (double)c.grid * c.block * C * c.steps;
    printf("hybrid 512 KiB table, %3u of 256 columns in smem  thr/SM %5u C %d : %7.3f Tlookup/s\n", CS, bps * block, C,
           lk / (ms * 1e-3) / 1e12);
}
struct RpCtx { const void* fn; unsigned grid, block; size_t smem; const uint8_t* in; uint32_t steps; uint32_t* sink; };
static void rp_launch(void* p) {
    RpCtx* c = (RpCtx*)p;
    void* args[] = {(void*)&c->in, (void*)&c->steps, (void*)&c->sink};
    CK(cudaLaunchKernel(c->fn, dim3(c->grid), dim3(c->block), args, c->smem, 0));
}
template <int C>
static void run_rep16(const uint8_t* in, uint32_t* sink, unsigned block, uint32_t steps) {
    RpCtx c;
    c.fn = (const void*)rep16_kernel<C>;
    c.smem = 26 * 8192 + 8192;
    CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
    c.grid = g_sms; c.block = block; c.in = in; c.steps = steps; c.sink = sink;
    const float ms = time_launch(rp_launch, &c, 3);
    const double lk = (double)c.grid * c.block * C * steps;
    printf("rep16 follow-like  thr/SM %5u C %d steps %u : %7.3f Tlookup/s  %6.1f cyc per warp-step\n", block, C, steps,
           lk / (ms * 1e-3) / 1e12, ms * 1e-3 * g_clk_ghz * 1e9 / (steps * C));
}

int main() {
    int dev = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    if (clk > 0) g_clk_ghz = clk / 1e6;
    printf("SMs %d  clock %.3f GHz\n", g_sms, g_clk_ghz);
    const uint32_t maxe = 1u << 20;   // 2 MiB u16
    uint16_t* h = (uint16_t*)malloc(maxe * 2);
    uint32_t s = 12345;
    for (uint32_t i = 0; i < maxe; ++i) {
        s = s * 1664525u + 1013904223u;
        h[i] = (uint16_t)(s >> 16);
    }
    uint16_t* tab;
    uint32_t* sink;
    CK(cudaMalloc(&tab, maxe * 2));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(sink, 0xFF, 64));
    CK(cudaMemcpy(tab, h, maxe * 2, cudaMemcpyHostToDevice));
    for (uint32_t ent : {1u << 18}) {
        for (int tps : {512, 1024, 2048}) {
            run_glob<1, false>(tab, ent, sink, tps);
            run_glob<2, false>(tab, ent, sink, tps);
            run_glob<4, false>(tab, ent, sink, tps);
            run_glob<8, false>(tab, ent, sink, tps);
        }
        run_glob<4, true>(tab, ent, sink, 2048);
        run_glob<8, true>(tab, ent, sink, 2048);
    }
    // 512 KiB over 4 / 8 CTAs, 256 KiB over 2, 2 MiB over 16 (non-portable)
    for (unsigned blk : {1024u}) {
        run_dsmem<1>(tab, 18, 2, sink, blk);
        run_dsmem<2>(tab, 18, 2, sink, blk);
        run_dsmem<4>(tab, 18, 2, sink, blk);
        run_dsmem<8>(tab, 18, 2, sink, blk);
    }
    run_dsmem<4>(tab, 18, 3, sink, 1024);
    run_dsmem<4>(tab, 17, 1, sink, 1024);
    run_dsmem<4>(tab, 20, 4, sink, 1024);
    for (unsigned blk : {256u, 512u, 1024u}) {
        run_smem<1, 0>(tab, sink, blk);
        run_smem<2, 0>(tab, sink, blk);
        run_smem<1, 1>(tab, sink, blk);
        run_smem<2, 1>(tab, sink, blk);
        run_smem<4, 1>(tab, sink, blk);
    }
    for (uint32_t CS : {0u, 64u, 108u}) {
        run_hybrid<1>(tab, CS, sink, 1024);
        run_hybrid<2>(tab, CS, sink, 1024);
        run_hybrid<2>(tab, CS, sink, 512);
    }
    {
        const size_t nb = (size_t)148 * 1024 * 2 * 16384;
        uint8_t* din;
        CK(cudaMalloc(&din, nb));
        CK(cudaMemset(din, 3, nb));
        run_rep16<1>(din, sink, 1024, 16384);
        run_rep16<2>(din, sink, 1024, 8192);
        run_rep16<1>(din, sink, 512, 16384);
        CK(cudaFree(din));
    }
    printf("done\n");
    return 0;
}
