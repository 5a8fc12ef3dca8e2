// stream_probe.cu -- diagnostic micro-benchmark (not part of the library): how fast can a
// THREAD-PER-CHUNK kernel stream its input on B200?  Each thread owns one contiguous chunk
// (the tiny kernel's layout); variants differ only in how the bytes reach the registers.
//   coalesced : grid-stride 16-B loads (the HBM ceiling for a plain read)
//   ldg<U>    : every thread walks its own chunk with U independent 16-B loads in flight
//   tma<W,S>  : per warp, 32 rows x W bytes boxes (cp.async.bulk.tensor.2d), S stages
//   bulk<W,S> : per lane, a 1-D cp.async.bulk of W contiguous bytes of its own chunk
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o stream_probe stream_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t a, uint4 v) { return a ^ v.x ^ (v.y * 3u) ^ (v.z * 5u) ^ (v.w * 7u); }

__global__ void coalesced(const uint4* __restrict__ in, uint64_t nv, uint32_t* out) {
    uint32_t a = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x)
        a = mix(a, __ldg(in + i));
    if (a == 0x12345678u) out[0] = a;
}

template <int U>
__global__ void ldg_chunk(const uint8_t* __restrict__ in, uint64_t L, uint32_t* out) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint4* p = reinterpret_cast<const uint4*>(in + t * L);
    const uint64_t nv = L / 16;
    uint32_t a = 0;
    for (uint64_t i = 0; i + U <= nv; i += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(p + i + u);
#pragma unroll
        for (int u = 0; u < U; ++u) a = mix(a, v[u]);
    }
    if (a == 0x12345678u) out[0] = a;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_tx_only(uint32_t a, uint32_t b) { asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(b) : "memory"); }
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t ph) { while (!mbar_try(a, ph)) {} }
__device__ __forceinline__ bool mbar_try_s(uint32_t a, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(a), "r"(ph), "r"(100000u) : "memory");
    return ok;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

template <int W, int S>
__global__ void tma_rows(const __grid_constant__ CUtensorMap map, uint64_t L, uint32_t* out) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t stage_bytes = 32 * W;
    const uint32_t buf0 = smem_u32(sm) + warp * S * stage_bytes;
    const uint32_t bar0 = smem_u32(sm) + nw * S * stage_bytes + warp * S * 8;
    const int row0 = (int)((blockIdx.x * (uint64_t)blockDim.x) + warp * 32);
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t nst = (uint32_t)(L / W);
    if (lane == 0)
        for (uint32_t s = 0; s < S && s < nst; ++s) {
            mbar_expect_tx(bar0 + 8 * s, stage_bytes);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(buf0 + s * stage_bytes), "l"((uint64_t)&map), "r"((int)(s * W)), "r"(row0), "r"(bar0 + 8 * s) : "memory");
        }
    uint32_t a = 0;
    for (uint32_t s = 0; s < nst; ++s) {
        const uint32_t slot = s % S;
        mbar_wait(bar0 + 8 * slot, (s / S) & 1);
        const uint32_t b = buf0 + slot * stage_bytes + lane * W;
#pragma unroll
        for (int u = 0; u < W / 16; ++u) a = mix(a, lds128(b + 16 * (u ^ (W == 64 ? ((lane >> 1) & 3) : W == 128 ? (lane & 7) : 0))));
        __syncwarp();
        if (lane == 0 && s + S < nst) {
            mbar_expect_tx(bar0 + 8 * slot, stage_bytes);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(buf0 + slot * stage_bytes), "l"((uint64_t)&map), "r"((int)((s + S) * W)), "r"(row0), "r"(bar0 + 8 * slot) : "memory");
        }
    }
    if (a == 0x12345678u) out[0] = a;
}

// RW rows per warp (RW/32 chunks per lane), box = RW rows x W bytes, S stages, suspend-hint waits
template <int W, int S, int RW>
__global__ void tma_rows2(const __grid_constant__ CUtensorMap map, uint64_t L, uint32_t* out) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    constexpr uint32_t stage_bytes = RW * W;
    const uint32_t buf0 = smem_u32(sm) + warp * S * stage_bytes;
    const uint32_t bar0 = smem_u32(sm) + nw * S * stage_bytes + warp * S * 8;
    const int row0 = (int)((blockIdx.x * (uint64_t)nw + warp) * RW);
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t nst = (uint32_t)(L / W);
    if (lane == 0)
        for (uint32_t s = 0; s < S && s < nst; ++s) {
            mbar_expect_tx(bar0 + 8 * s, stage_bytes);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(buf0 + s * stage_bytes), "l"((uint64_t)&map), "r"((int)(s * W)), "r"(row0), "r"(bar0 + 8 * s) : "memory");
        }
    uint32_t a = 0;
    for (uint32_t s = 0; s < nst; ++s) {
        const uint32_t slot = s % S;
        while (!mbar_try_s(bar0 + 8 * slot, (s / S) & 1)) {}
#pragma unroll
        for (int r = 0; r < RW / 32; ++r) {
            const uint32_t b = buf0 + slot * stage_bytes + (lane + 32 * r) * W;
#pragma unroll
            for (int u = 0; u < W / 16; ++u) a = mix(a, lds128(b + 16 * u));
        }
        __syncwarp();
        if (lane == 0 && s + S < nst) {
            mbar_expect_tx(bar0 + 8 * slot, stage_bytes);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(buf0 + slot * stage_bytes), "l"((uint64_t)&map), "r"((int)((s + S) * W)), "r"(row0), "r"(bar0 + 8 * slot) : "memory");
        }
    }
    if (a == 0x12345678u) out[0] = a;
}

template <int W, int S>
__global__ void bulk_rows(const uint8_t* __restrict__ in, uint64_t L, uint32_t* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t stage_bytes = 32 * W;
    const uint32_t buf0 = smem_u32(sm) + warp * S * stage_bytes;
    const uint32_t bar0 = smem_u32(sm) + nw * S * stage_bytes + warp * S * 8;
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint8_t* row = in + t * L;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t nst = (uint32_t)(L / W);
    auto issue = [&](uint32_t s, uint32_t slot) {
        if (lane == 0) mbar_expect_tx(bar0 + 8 * slot, stage_bytes);
        __syncwarp();
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(buf0 + slot * stage_bytes + lane * W), "l"(row + (uint64_t)s * W), "r"((uint32_t)W), "r"(bar0 + 8 * slot) : "memory");
    };
    for (uint32_t s = 0; s < S && s < nst; ++s) issue(s, s);
    uint32_t a = 0;
    for (uint32_t s = 0; s < nst; ++s) {
        const uint32_t slot = s % S;
        mbar_wait(bar0 + 8 * slot, (s / S) & 1);
        const uint32_t b = buf0 + slot * stage_bytes + lane * W;
#pragma unroll
        for (int u = 0; u < W / 16; ++u) a = mix(a, lds128(b + 16 * u));
        __syncwarp();
        if (s + S < nst) issue(s + S, slot);
    }
    if (a == 0x12345678u) out[0] = a;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float timeit(void (*launch)(void*), void* ctx, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(ctx);
    launch(ctx);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch(ctx);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    CK(cudaGetLastError());
    return ms / reps;
}

struct Ctx {
    const uint8_t* in;
    uint64_t n, L;
    uint32_t* out;
    int grid, block;
    size_t smem;
    CUtensorMap map;
    const void* fn;
};

static void launch_generic(void* p) {
    Ctx* c = (Ctx*)p;
    void* argsl[] = {(void*)&c->in, &c->L, &c->out};
    CK(cudaLaunchKernel(c->fn, c->grid, c->block, argsl, c->smem, 0));
}
static void launch_tma(void* p) {
    Ctx* c = (Ctx*)p;
    void* args[] = {&c->map, &c->L, &c->out};
    CK(cudaLaunchKernel(c->fn, c->grid, c->block, args, c->smem, 0));
}
static void launch_coal(void* p) {
    Ctx* c = (Ctx*)p;
    coalesced<<<c->grid, c->block>>>((const uint4*)c->in, c->n / 16, c->out);
}

int main(int argc, char** argv) {
    const uint64_t n = 1ull << 30;
    uint8_t* d;
    uint32_t* out;
    CK(cudaMalloc(&d, n));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(d, 0x5A, n));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    const int reps = 10;
    Ctx c;
    c.in = d;
    c.n = n;
    c.out = out;
    c.grid = sms * 4;
    c.block = 512;
    float ms = timeit(launch_coal, &c, reps);
    printf("coalesced          %8.1f GB/s\n", n / ms / 1e6);

    if (argc > 1 && argv[1][0] == 'L') {
        // stride sweep: thread-per-chunk ldg streams (75776 threads) and TMA row boxes (tiny geometry)
        for (uint64_t Lf = 13824; Lf <= 13824 + 352; Lf += 16) {
            Ctx x = c;
            x.fn = (const void*)ldg_chunk<4>;
            x.block = 512;
            x.grid = sms;
            uint64_t T = (uint64_t)x.grid * 512;
            x.L = Lf;
            x.smem = 0;
            float t = timeit(launch_generic, &x, reps);
            printf("ldg  L=%llu (mod256=%llu) %8.1f GB/s\n", (unsigned long long)Lf, (unsigned long long)(Lf % 256),
                   (double)(x.L * T) / t / 1e6);
        }
    }
    auto run_ldg = [&](const void* fn, const char* name, int block, int per_sm) {
        Ctx x = c;
        x.fn = fn;
        x.block = block;
        x.grid = sms * per_sm;
        uint64_t T = (uint64_t)x.grid * block;
        x.L = (n / T) & ~255ull;
        x.smem = 0;
        float t = timeit(launch_generic, &x, reps);
        printf("%-18s %8.1f GB/s  (threads %llu, L %llu)\n", name, (double)(x.L * T) / t / 1e6, (unsigned long long)T,
               (unsigned long long)x.L);
    };
    run_ldg((const void*)ldg_chunk<1>, "ldg<1> 512x2", 512, 2);
    run_ldg((const void*)ldg_chunk<2>, "ldg<2> 512x2", 512, 2);
    run_ldg((const void*)ldg_chunk<4>, "ldg<4> 512x2", 512, 2);
    run_ldg((const void*)ldg_chunk<8>, "ldg<8> 512x2", 512, 2);
    run_ldg((const void*)ldg_chunk<4>, "ldg<4> 512x4", 512, 4);
    run_ldg((const void*)ldg_chunk<8>, "ldg<8> 256x4", 256, 4);

    auto run_tma = [&](const void* fn, const char* name, int W, int S, int block, int per_sm, CUtensorMapSwizzle sw,
                       CUtensorMapL2promotion pr) {
        Ctx x = c;
        x.fn = fn;
        x.block = block;
        x.grid = sms * per_sm;
        uint64_t T = (uint64_t)x.grid * block;
        x.L = (n / T) / W * W;
        x.smem = (size_t)(block / 32) * S * 32 * W + (block / 32) * S * 8 + 1024;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)x.smem));
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, block, x.smem);
        if (bps < per_sm) {
            printf("%-18s does not fit (%d/SM, smem %zu)\n", name, bps, x.smem);
            return;
        }
        const cuuint64_t dims[2] = {x.L, T};
        const cuuint64_t str[1] = {x.L};
        const cuuint32_t box[2] = {(cuuint32_t)W, 32};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&x.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                sw, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("%-18s encode failed\n", name);
            return;
        }
        float t = timeit(launch_tma, &x, reps);
        printf("%-18s %8.1f GB/s  (threads %llu, L %llu, smem %zu)\n", name, (double)(x.L * T) / t / 1e6,
               (unsigned long long)T, (unsigned long long)x.L, x.smem);
    };
    auto P256 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B, P128 = CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
         PN = CU_TENSOR_MAP_L2_PROMOTION_NONE;
    run_tma((const void*)tma_rows<64, 2>, "tma<64,2> 512x2", 64, 2, 512, 2, CU_TENSOR_MAP_SWIZZLE_64B, P256);
    run_tma((const void*)tma_rows<64, 2>, "tma<64,2> p128", 64, 2, 512, 2, CU_TENSOR_MAP_SWIZZLE_64B, P128);
    run_tma((const void*)tma_rows<64, 2>, "tma<64,2> pnone", 64, 2, 512, 2, CU_TENSOR_MAP_SWIZZLE_64B, PN);
    run_tma((const void*)tma_rows<64, 3>, "tma<64,3> 512x2", 64, 3, 512, 2, CU_TENSOR_MAP_SWIZZLE_64B, P256);
    run_tma((const void*)tma_rows<64, 4>, "tma<64,4> 256x4", 64, 4, 256, 4, CU_TENSOR_MAP_SWIZZLE_64B, P256);
    run_tma((const void*)tma_rows<128, 2>, "tma<128,2> 256x4", 128, 2, 256, 4, CU_TENSOR_MAP_SWIZZLE_128B, P256);
    run_tma((const void*)tma_rows<128, 3>, "tma<128,3> 256x3", 128, 3, 256, 3, CU_TENSOR_MAP_SWIZZLE_128B, P256);
    run_tma((const void*)tma_rows<64, 2>, "tma<64,2> 256x4", 64, 2, 256, 4, CU_TENSOR_MAP_SWIZZLE_64B, P256);

    auto run_tma2 = [&](const void* fn, const char* name, int W, int S, int RW, int block, int per_sm,
                        CUtensorMapL2promotion pr, uint64_t Lforce = 0) {
        Ctx x = c;
        x.fn = fn;
        x.block = block;
        x.grid = sms * per_sm;
        uint64_t T = (uint64_t)x.grid * (block / 32) * RW;   // rows = chunks
        x.L = (n / T) / W * W;
        if (Lforce && Lforce <= x.L) x.L = Lforce;
        x.smem = (size_t)(block / 32) * S * RW * W + (block / 32) * S * 8 + 1024;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)x.smem));
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, block, x.smem);
        if (bps < per_sm) {
            printf("%-22s does not fit (%d/SM, smem %zu)\n", name, bps, x.smem);
            return;
        }
        const cuuint64_t dims[2] = {x.L, T};
        const cuuint64_t str[1] = {x.L};
        const cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)RW};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&x.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("%-22s encode failed\n", name);
            return;
        }
        float t = timeit(launch_tma, &x, reps);
        printf("%-22s %8.1f GB/s  (chunks %llu, L %llu, smem %zu)\n", name, (double)(x.L * T) / t / 1e6,
               (unsigned long long)T, (unsigned long long)x.L, x.smem);
    };
    run_tma2((const void*)tma_rows2<64, 2, 32>, "t2<64,2,32> 512x2", 64, 2, 32, 512, 2, P256);
    run_tma2((const void*)tma_rows2<32, 2, 64>, "t2<32,2,64> 512x2", 32, 2, 64, 512, 2, P256);
    run_tma2((const void*)tma_rows2<32, 3, 64>, "t2<32,3,64> 512x2", 32, 3, 64, 512, 2, P256);
    run_tma2((const void*)tma_rows2<32, 2, 64>, "t2<32,2,64> 256x4", 32, 2, 64, 256, 4, P256);
    run_tma2((const void*)tma_rows2<32, 2, 96>, "t2<32,2,96> 512x2", 32, 2, 96, 512, 2, P256);
    run_tma2((const void*)tma_rows2<16, 4, 64>, "t2<16,4,64> 512x2", 16, 4, 64, 512, 2, P256);
    run_tma2((const void*)tma_rows2<32, 2, 128>, "t2<32,2,128> 256x3", 32, 2, 128, 256, 3, P256);
    run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 256x3", 64, 2, 64, 256, 3, P256);
    run_tma2((const void*)tma_rows2<128, 2, 32>, "t2<128,2,32> 256x3", 128, 2, 32, 256, 3, P256);
    run_tma2((const void*)tma_rows2<256, 2, 32>, "t2<256,2,32> 128x3", 256, 2, 32, 128, 3, P256);
    run_tma2((const void*)tma_rows2<256, 2, 16>, "t2<256,2,16> 256x3", 256, 2, 16, 256, 3, P256);
    run_tma2((const void*)tma_rows2<512, 2, 8>, "t2<512,2,8> 256x3", 512, 2, 8, 256, 3, P256);
    if (argc > 1 && argv[1][0] == 'L') {
        for (uint64_t Lf = 6784; Lf <= 7072; Lf += 16) {
            char nm[64];
            snprintf(nm, 64, "tma L=%llu (mod256=%llu)", (unsigned long long)Lf, (unsigned long long)(Lf % 256));
            run_tma2((const void*)tma_rows2<64, 2, 64>, nm, 64, 2, 64, 512, 1, P256, Lf);
        }
        return 0;
    }
    if (argc > 1) {
        run_tma2((const void*)tma_rows2<64, 2, 32>, "t2<64,2,32> 256x3", 64, 2, 32, 256, 3, P256);
        run_tma2((const void*)tma_rows2<64, 3, 32>, "t2<64,3,32> 256x3", 64, 3, 32, 256, 3, P256);
        run_tma2((const void*)tma_rows2<64, 4, 32>, "t2<64,4,32> 256x3", 64, 4, 32, 256, 3, P256);
        run_tma2((const void*)tma_rows2<64, 4, 32>, "t2<64,4,32> 512x1", 64, 4, 32, 512, 1, P256);
        run_tma2((const void*)tma_rows2<64, 3, 32>, "t2<64,3,32> 768x1", 64, 3, 32, 768, 1, P256);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 768x1", 64, 2, 64, 768, 1, P256);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 256x3", 64, 2, 64, 256, 3, P256);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 384x2", 64, 2, 64, 384, 2, P256);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 512x1", 64, 2, 64, 512, 1, P256);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 256x2", 64, 2, 64, 256, 2, P256);
        run_tma2((const void*)tma_rows2<64, 3, 64>, "t2<64,3,64> 512x1", 64, 3, 64, 512, 1, P256);
        run_tma2((const void*)tma_rows2<64, 2, 96>, "t2<64,2,96> 512x1", 64, 2, 96, 512, 1, P256);
        run_tma2((const void*)tma_rows2<64, 2, 128>, "t2<64,2,128> 384x1", 64, 2, 128, 384, 1, P256);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 768x1 P128", 64, 2, 64, 768, 1, P128);
        run_tma2((const void*)tma_rows2<64, 2, 64>, "t2<64,2,64> 768x1 PN", 64, 2, 64, 768, 1, PN);
        return 0;
    }
    auto run_bulk = [&](const void* fn, const char* name, int W, int S, int block, int per_sm) {
        Ctx x = c;
        x.fn = fn;
        x.block = block;
        x.grid = sms * per_sm;
        uint64_t T = (uint64_t)x.grid * block;
        x.L = (n / T) / W * W;
        x.smem = (size_t)(block / 32) * S * 32 * W + (block / 32) * S * 8;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)x.smem));
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, block, x.smem);
        if (bps < per_sm) {
            printf("%-18s does not fit (%d/SM, smem %zu)\n", name, bps, x.smem);
            return;
        }
        float t = timeit(launch_generic, &x, reps);
        printf("%-18s %8.1f GB/s  (threads %llu, L %llu, smem %zu)\n", name, (double)(x.L * T) / t / 1e6,
               (unsigned long long)T, (unsigned long long)x.L, x.smem);
    };
    run_bulk((const void*)bulk_rows<64, 2>, "bulk<64,2> 512x2", 64, 2, 512, 2);
    run_bulk((const void*)bulk_rows<128, 2>, "bulk<128,2> 256x4", 128, 2, 256, 4);
    run_bulk((const void*)bulk_rows<256, 2>, "bulk<256,2> 128x8", 256, 2, 128, 8);
    run_bulk((const void*)bulk_rows<128, 3>, "bulk<128,3> 256x3", 128, 3, 256, 3);
    run_bulk((const void*)bulk_rows<256, 2>, "bulk<256,2> 256x3", 256, 2, 256, 3);
    printf("done\n");
    return 0;
}
