// Microbenchmark: tcgen05.mma issue-to-completion throughput of the prefill kernel's MMA shapes on
// sm_100a, one CTA per SM, single issuing thread, operands resident in SMEM / TMEM (no TMA, no
// softmax).  Reports cycles per 128x128x128 product (ideal: 512 = 128*128/256 per K16 x 8).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2502_12574_b200/csrc mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "hi_kernels.cuh"
#include "tc_ptx.cuh"
using namespace hi::ptx;

constexpr int BOX = 128 * 128;  // [128 rows][64 bf16] SW128 box
template <int MODE>
__global__ void __launch_bounds__(256, 1) kern(int iters, long long* cyc, int bg, const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, tbar[2], cbar[4];
    __shared__ uint32_t tmem_base;
    const uint32_t sb = smem_addr(smem);
    // A: 2 tiles x 2 boxes (64 KB), B (K/V): 2 boxes (32 KB) -> 96 KB, + bg scratch 64 KB
    for (int i = threadIdx.x; i < (160 << 10) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) {
        mbar_init(smem_addr(&bar), 1); mbar_init(smem_addr(&tbar[0]), 1); mbar_init(smem_addr(&tbar[1]), 1);
        for (int c = 0; c < 4; ++c) mbar_init(smem_addr(&cbar[c]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tmem_base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        constexpr uint32_t ID_S = idesc_bf16(128, 128, false);
        constexpr uint32_t ID_S256 = idesc_bf16(128, 256, false);
        constexpr uint32_t ID_O = idesc_bf16(128, 128, true);
        const uint64_t dq = sdesc(sb, 16, 1024), dk = sdesc(sb + 4 * BOX, 16, 1024), dv = sdesc(sb + 4 * BOX, BOX, 1024);
        for (int it = 0; it < iters; ++it) {
            for (int tt = 0; tt < (MODE == 4 ? 2 : 1); ++tt) {
                if (MODE == 0 || MODE == 2 || MODE == 4) {
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint32_t off = ((ks >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem + tt * 256, dq + ((tt * 2 * BOX) >> 4) + off, dk + off, ID_S, ks > 0);
                    }
                }
                if (MODE == 1 || MODE == 2 || MODE == 4) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_bf16_ts(tmem + tt * 256 + 128, tmem + tt * 256 + kk * 8, dv + ((kk * 16 * 128) >> 4), ID_O, 1u);
                }
                if (MODE >= 5 && MODE <= 8) {  // S + PV with (MODE - 4) commits per iteration to never-waited barriers
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint32_t off = ((ks >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem, dq + off, dk + off, ID_S, ks > 0);
                    }
                    umma_commit(smem_addr(&cbar[0]));
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_bf16_ts(tmem + 128, tmem + kk * 8, dv + ((kk * 16 * 128) >> 4), ID_O, 1u);
                    for (int c = 1; c < MODE - 4; ++c) umma_commit(smem_addr(&cbar[c]));
                }
                if (MODE == 9) {  // SS M128 N64 K128 (8 x K16)
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint32_t off = ((ks >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem, dq + off, dk + off, idesc_bf16(128, 64, false), ks > 0);
                    }
                }
                if (MODE == 10) {  // TS M128 N128 K64 (4 x K16)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_bf16_ts(tmem + 128, tmem + kk * 8, dv + ((kk * 16 * 128) >> 4), ID_O, 1u);
                }
                if (MODE == 11 || MODE == 13) {  // SS N128 / N256, K64 (4 x K16)
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint32_t off = ((ks >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem, dq + off, dk + off, MODE == 11 ? ID_S : ID_S256, ks > 0);
                    }
                }
                if (MODE == 12) {  // SS N64, 16 x K16
#pragma unroll
                    for (int ks = 0; ks < 16; ++ks) {
                        const uint32_t off = (((ks & 7) >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem, dq + off, dk + off, idesc_bf16(128, 64, false), ks > 0);
                    }
                }
                if (MODE == 14) {  // SS N64 K128 into two alternating D (cols 0 / 64)
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint32_t off = ((ks >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem + (it & 1) * 64, dq + off, dk + off, idesc_bf16(128, 64, false), ks > 0);
                    }
                }
                if (MODE == 3) {
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint32_t off = ((ks >> 2) * BOX + (ks & 3) * 32) >> 4;
                        umma_bf16(tmem, dq + off, dk + off, ID_S256, ks > 0);
                    }
                }
            }
        }
        umma_commit(smem_addr(&bar));
        mbar_wait(smem_addr(&bar), 0);
    } else if (bg >= 4 && threadIdx.x == 32) {
        // TMA stream into the scratch region: (bg - 3) x 32 KiB per MMA iteration, 2 buffers in flight
        const int n = iters * (bg - 3);
        for (int i = 0; i < n; ++i) {
            const int s = i & 1;
            if (i >= 2) mbar_wait(smem_addr(&tbar[s]), ((i >> 1) - 1) & 1);
            mbar_expect_tx(smem_addr(&tbar[s]), 2 * BOX);
            for (int c = 0; c < 2; ++c)
                tma_load_3d(sb + 96 * 1024 + (s * 2 + c) * BOX, &tm, smem_addr(&tbar[s]), c * 64, (i % 2048) * 128, 0);
        }
        for (int i = (n > 2 ? n - 2 : 0); i < n; ++i) mbar_wait(smem_addr(&tbar[i & 1]), (i >> 1) & 1);
    } else if (bg >= 2 && bg < 4 && threadIdx.x >= 128) {
        // TMEM traffic of a softmax warpgroup: per iteration ld 128 S columns + st 64 P columns per lane
        // (columns of tile 1's S region; lane quarter = warp % 4); bg = 2: once per iteration, 3: twice
        const uint32_t lane_q = static_cast<uint32_t>((threadIdx.x / 32) % 4 * 32) << 16;
        uint32_t v[32];
        uint32_t acc = 0;
        for (int it = 0; it < iters * (bg - 1); ++it) {
            for (int cb = 0; cb < 4; ++cb) {
                tmem_ld32(tmem + lane_q + 256 + 64 * 0 + cb * 32 - (cb >= 2 ? 0 : 0), v);
                tmem_wait_ld();
                acc += v[0] + v[31];
            }
            for (int cb = 0; cb < 2; ++cb) { v[0] = acc; tmem_st32(tmem + lane_q + 256 + cb * 32, v); }
            tmem_wait_st();
        }
        if (acc == 0x12345678u) cyc[0] = acc;
    } else if (bg == 1 && threadIdx.x >= 32) {
        // background shared-memory writes (TMA-like traffic into the K/V region's neighbour)
        uint4* dst = reinterpret_cast<uint4*>(smem + 96 * 1024);
        for (int it = 0; it < iters * bg; ++it)
            for (int i = threadIdx.x - 32; i < 4096; i += 96) dst[i] = make_uint4(it, i, 0, 0);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

static CUtensorMap g_tm;
template <int MODE>
void run(const char* name, double products_per_iter, int bg = 0) {
    const int iters = 2000, blocks = 148, smem = (160 << 10) + 1024;
    long long* d; cudaMalloc(&d, blocks * sizeof(long long));
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<MODE><<<blocks, 256, smem>>>(10, d, bg, g_tm);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<MODE><<<blocks, 256, smem>>>(iters, d, bg, g_tm);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s bg=%d: %8.1f cycles per 128x128x128 product (ideal 512)  kernel %.3f ms %s\n", name, bg,
           avg / iters / products_per_iter, ms, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    void* buf; cudaMalloc(&buf, size_t(262144) * 256);
    cudaMemset(buf, 0, size_t(262144) * 256);
    const cuuint64_t dims[3] = {128, 262144, 1};
    const cuuint64_t strides[2] = {256, (cuuint64_t)262144 * 256};
    const cuuint32_t box[3] = {64, 128, 1};
    if (!hi::make_tmap_bf16(&g_tm, buf, 3, dims, strides, box)) { printf("tmap failed\n"); return 1; }
    run<0>("S: SS M128 N128 K128", 1);
    run<1>("PV: TS M128 N128 K128 (A in TMEM)", 1);
    run<2>("S + PV (one tile)", 2);
    run<4>("S + PV x 2 tiles", 4);
    run<3>("SS M128 N256 K128", 2);
    run<0>("S: SS M128 N128 K128", 1, 1);
    run<4>("S + PV x 2 tiles", 4, 1);
    run<0>("S: SS M128 N128 K128", 1, 2);
    run<1>("PV: TS M128 N128 K128 (A in TMEM)", 1, 2);
    run<2>("S + PV (one tile)", 2, 2);
    run<2>("S + PV (one tile)", 2, 3);
    run<9>("SS M128 N64 K128", 0.5);
    run<11>("SS M128 N128 K64", 0.5);
    run<13>("SS M128 N256 K64", 1);
    run<12>("SS M128 N64 K256", 1);
    run<14>("SS M128 N64 K128 alternating D", 0.5);
    run<10>("TS M128 N128 K64", 0.5);
    run<5>("S + PV, 1 commit / iter", 2);
    run<6>("S + PV, 2 commits / iter", 2);
    run<8>("S + PV, 4 commits / iter", 2);
    run<0>("S: SS M128 N128 K128", 1, 4);
    run<0>("S: SS M128 N128 K128", 1, 5);
    run<1>("PV: TS M128 N128 K128 (A in TMEM)", 1, 4);
    run<2>("S + PV (one tile)", 2, 4);
    run<2>("S + PV (one tile)", 2, 5);
    run<4>("S + PV x 2 tiles", 4, 4);
    return 0;
}
