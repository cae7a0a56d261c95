// Microbenchmark: TMA (cp.async.bulk.tensor) inbound throughput per SM on sm_100a for the prefill
// kernels' K/V streaming pattern: every CTA (one per SM) streams the same [n_keys][128] bf16 tensor
// in 128-key tiles (2 SWIZZLE_128B boxes of 16 KiB) through an S-stage ring, optionally multicast to
// a cluster of CL CTAs (each issues its share of the boxes).  No compute: the consumer releases a stage
// as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2502_12574_b200/csrc tma_rate.cu \
//        ../../paper_2502_12574_b200/csrc/tmap.cu -o tma_rate
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "hi_kernels.cuh"
#include "tc_ptx.cuh"
using namespace hi::ptx;

constexpr int BOX = 128 * 128;  // [128 keys][64 bf16]
template <int S, int CL>
__global__ void __launch_bounds__(64, 1) kern(const __grid_constant__ CUtensorMap tm, int n_tiles, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[S], empty[S];
    const uint32_t sb = smem_addr(smem);
    const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(smem_addr(&full[s]), 1); mbar_init(smem_addr(&empty[s]), CL); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (CL > 1) cluster_sync(); else __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x == 0) {  // producer
        for (int i = 0; i < n_tiles; ++i) {
            const int s = i % S;
            if (i >= S) mbar_wait(smem_addr(&empty[s]), ((i / S) - 1) & 1);
            mbar_expect_tx(smem_addr(&full[s]), 2 * BOX);
            for (int c = 0; c < 2; ++c) {
                if constexpr (CL == 1) tma_load_3d(sb + (s * 2 + c) * BOX, &tm, smem_addr(&full[s]), c * 64, i * 128, 0);
                else if (c % CL == static_cast<int>(crank) || (CL > 2 && false))
                    tma_load_3d_mc(sb + (s * 2 + c) * BOX, &tm, smem_addr(&full[s]), c * 64, i * 128, 0, (1u << CL) - 1);
            }
        }
    } else if (threadIdx.x == 32) {  // consumer
        for (int i = 0; i < n_tiles; ++i) {
            const int s = i % S;
            mbar_wait(smem_addr(&full[s]), (i / S) & 1);
            if constexpr (CL == 1) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[s])) : "memory");
            } else {
                for (int rk = 0; rk < CL; ++rk) mbar_arrive_cluster(mapa_shared(smem_addr(&empty[s]), rk));
            }
        }
        for (int i = (n_tiles > S ? n_tiles - S : 0); i < n_tiles; ++i) mbar_wait(smem_addr(&empty[i % S]), (i / S) & 1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x] = t1 - t0;
    if constexpr (CL > 1) cluster_sync(); else __syncthreads();
}

template <int S, int CL>
void run(const CUtensorMap& tm, int n_tiles) {
    const int blocks = 148, smem = S * 2 * BOX + 1024;
    long long* d; cudaMalloc(&d, blocks * sizeof(long long));
    cudaFuncSetAttribute(kern<S, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern<S, CL>, tm, 8, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, kern<S, CL>, tm, n_tiles, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
    const double bytes_in = 32768.0 * n_tiles;  // received per SM
    printf("stages=%d cluster=%d: %7.1f cycles per 32 KiB tile -> %6.1f B/clk/SM received; L2 reads %6.2f TB/s, "
           "SM receive %6.2f TB/s  %s\n", S, CL, avg / n_tiles, bytes_in / (avg), bytes_in * blocks / CL / (ms * 1e-3) / 1e12,
           bytes_in * blocks / (ms * 1e-3) / 1e12, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    const int n_keys = 262144, n_tiles = n_keys / 128;
    void* buf; cudaMalloc(&buf, size_t(n_keys) * 128 * 2);
    cudaMemset(buf, 0, size_t(n_keys) * 128 * 2);
    CUtensorMap tm;
    const cuuint64_t dims[3] = {128, (cuuint64_t)n_keys, 1};
    const cuuint64_t strides[2] = {256, (cuuint64_t)n_keys * 256};
    const cuuint32_t box[3] = {64, 128, 1};
    if (!hi::make_tmap_bf16(&tm, buf, 3, dims, strides, box)) { printf("tmap failed\n"); return 1; }
    run<2, 1>(tm, n_tiles); run<3, 1>(tm, n_tiles); run<4, 1>(tm, n_tiles); run<6, 1>(tm, n_tiles);
    run<2, 2>(tm, n_tiles); run<3, 2>(tm, n_tiles); run<4, 2>(tm, n_tiles); run<6, 2>(tm, n_tiles);
    return 0;
}
