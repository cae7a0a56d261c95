// k_gemm.cu -- the NEXT-4 layer's projections (QKV, O, gate/up, down) on the 5th-gen tensor cores.
//
//   Y[n, mo] = (beta ? Y : 0) + X[n, kd] W[mo, kd]^T        bf16 in/out, fp32 accumulate, one rounding
//
// (include/hilayer.h; reading R19: the residual add is the epilogue, so x + a W^T is
// rounded once.)  X is the activation (row-major = K-major), W a PyTorch Linear weight [out, in] (K-major).
//
// gemm_tc2_kernel (n >= 2, the product; HI_GEMM_2CTA): CTA pairs with tcgen05.mma.cta_group::2 on 256 x 256 tiles --
// see its comment below; 1.07x cuBLAS over the Llama-3-8B projections (profiles/gemm_vs_cublas_r02_pair.json).
// gemm_tc_kernel (n >= 2 with HI_GEMM_2CTA=0; 0.93x cuBLAS): persistent, warp-specialised, one CTA per SM.  Tile 128 (tokens) x 256 (out features)
// x 64 (K), both operands TMA-loaded with SWIZZLE_128B into a 4-stage ring (48 KiB per stage); one thread issues
// tcgen05.mma M128 N256 K16 (4 per stage) into a TMEM accumulator of 256 fp32 columns, double-buffered (512
// columns), so the 4 epilogue warps drain tile i (tcgen05.ld -> + residual -> bf16 -> global) while the MMAs
// of tile i+1 run.  Tiles are visited in groups of 8 row-blocks so that a wave of 148 CTAs shares ~8 MiB of X
// and ~37 MiB of W in L2.
//
// gemv_kernel (n == 1, decode): HBM-bound: each warp streams 2 weight rows with 16-byte loads against x held
// in shared memory (fp32), warp-shuffle reduction, one rounding per output (+ residual).
// Both also write fp32 outputs without rounding (`out_f32`): the partial sums of a tensor-parallel layer, which
// are all-reduced across ranks before the residual add rounds once.
#include "hi_kernels.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

namespace hi {
namespace {

using namespace ptx;

constexpr int GM = 128, GN = 256, GK = 64;   // tile
constexpr int G_STAGES = 4;
constexpr int G_GROUP_M = 8;                 // row-blocks per tile group (L2 locality)
constexpr int G_EPI_WARPS = 4;
constexpr int G_THREADS = 32 * (2 + G_EPI_WARPS);   // warp 0: TMA, warp 1: TMEM alloc + MMA, warps 2-5: epilogue
constexpr int A_BYTES = GM * GK * 2;         // 16 KiB
constexpr int B_BYTES = GN * GK * 2;         // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;

struct __align__(8) GemmBars {
    uint64_t full[G_STAGES], empty[G_STAGES];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};
constexpr int G_SMEM = G_STAGES * STAGE_BYTES + static_cast<int>(sizeof(GemmBars)) + 1024;

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
    const int per_group = G_GROUP_M * tiles_n;
    const int grp = t / per_group;
    const int first_m = grp * G_GROUP_M;
    const int gm = min(G_GROUP_M, tiles_m - first_m);
    const int local = t - grp * per_group;
    mb = first_m + local % gm;
    nb = local / gm;
}

template <bool F32OUT>
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                   void* __restrict__ yv, int n, int mo, int kd, int beta) {
    extern __shared__ uint8_t g_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(g_raw) + 1023) & ~uintptr_t(1023));
    GemmBars* bars = reinterpret_cast<GemmBars*>(smem + G_STAGES * STAGE_BYTES);
    const uint32_t sbase = smem_addr(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_m = (n + GM - 1) / GM, tiles_n = (mo + GN - 1) / GN, tiles = tiles_m * tiles_n;
    const int kt = (kd + GK - 1) / GK;
    auto full = [&](int s) { return smem_addr(&bars->full[s]); };
    auto empty = [&](int s) { return smem_addr(&bars->empty[s]); };
    auto accf = [&](int b) { return smem_addr(&bars->acc_full[b]); };
    auto acce = [&](int b) { return smem_addr(&bars->acc_empty[b]); };
    if (threadIdx.x == 0) {
        for (int s = 0; s < G_STAGES; ++s) {
            mbar_init(full(s), 1);
            mbar_init(empty(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(accf(b), 1);
            mbar_init(acce(b), G_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&bars->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                int mb, nb;
                tile_coords(t, tiles_m, tiles_n, mb, nb);
                for (int k = 0; k < kt; ++k, ++it) {
                    const int s = it % G_STAGES;
                    if (it >= G_STAGES) mbar_wait(empty(s), ((it / G_STAGES) - 1) & 1);
                    mbar_expect_tx(full(s), STAGE_BYTES);   // OOB rows / columns are zero-filled, still counted
                    tma_load_2d(sbase + s * STAGE_BYTES, &tm_x, full(s), k * GK, mb * GM);
                    tma_load_2d(sbase + s * STAGE_BYTES + A_BYTES, &tm_w, full(s), k * GK, nb * GN);
                }
            }
        }
    } else if (warp == 1) {
        {   // ---------------- MMA issuer: the whole warp runs the loop, elect.sync issues (no waterfall per MMA)
            constexpr uint32_t IDESC = idesc_bf16(GM, GN, false);
            int it = 0, i = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
                const int b = i & 1;
                if (i >= 2) mbar_wait(acce(b), ((i >> 1) - 1) & 1);   // the epilogue drained this buffer
                tc_fence_after();
                const uint32_t acc = tmem + b * GN;
                for (int k = 0; k < kt; ++k, ++it) {
                    const int s = it % G_STAGES;
                    mbar_wait(full(s), (it / G_STAGES) & 1);
                    tc_fence_after();
                    const uint64_t da = sdesc(sbase + s * STAGE_BYTES, 16, 1024);
                    const uint64_t db = sdesc(sbase + s * STAGE_BYTES + A_BYTES, 16, 1024);
#pragma unroll
                    for (int kk = 0; kk < GK / 16; ++kk)   // 32-byte steps inside the 128-byte swizzle atom
                        umma_bf16_w(acc, da + (kk * 2), db + (kk * 2), IDESC, (k > 0 || kk > 0) ? 1u : 0u);
                    umma_commit_w(empty(s));   // the stage is free once these MMAs have read it
                }
                umma_commit_w(accf(b));        // accumulator complete
            }
        }
    } else {
        // ---------------- epilogue: warp w owns TMEM lanes 32*(w%4) .. +31 (rows of the tile)
        const int q = warp & 3;
        const int r_in = q * 32 + lane;
        int i = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
            int mb, nb;
            tile_coords(t, tiles_m, tiles_n, mb, nb);
            const int b = i & 1;
            mbar_wait(accf(b), (i >> 1) & 1);
            tc_fence_after();
            const int row = mb * GM + r_in;
            const bool live = row < n;
            const int64_t yoff = static_cast<int64_t>(row) * mo + nb * GN;
            const uint32_t taddr = tmem + b * GN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
            for (int c = 0; c < GN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(taddr + c * 32, v);
                tmem_wait_ld();
                const int col = nb * GN + c * 32;
                if (F32OUT && live && col < mo) {   // fp32 partial sums (tensor-parallel layer): no rounding here
                    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(yv) + yoff + c * 32);
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4)
                        dst[e4] = make_float4(__uint_as_float(v[4 * e4]), __uint_as_float(v[4 * e4 + 1]),
                                              __uint_as_float(v[4 * e4 + 2]), __uint_as_float(v[4 * e4 + 3]));
                } else if (live && col < mo) {   // mo is a multiple of 64: a 32-column chunk is all in or all out
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(yv) + yoff + c * 32);
                    float f[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(v[e]);
                    if (beta) {
#pragma unroll
                        for (int e8 = 0; e8 < 4; ++e8) {
                            const uint4 u = dst[e8];
                            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                f[e8 * 8 + 2 * h] += __uint_as_float(w4[h] << 16);
                                f[e8 * 8 + 2 * h + 1] += __uint_as_float(w4[h] & 0xffff0000u);
                            }
                        }
                    }
#pragma unroll
                    for (int e8 = 0; e8 < 4; ++e8) {
                        uint4 o;
                        o.x = pack_bf16(f[e8 * 8 + 0], f[e8 * 8 + 1]);
                        o.y = pack_bf16(f[e8 * 8 + 2], f[e8 * 8 + 3]);
                        o.z = pack_bf16(f[e8 * 8 + 4], f[e8 * 8 + 5]);
                        o.w = pack_bf16(f[e8 * 8 + 6], f[e8 * 8 + 7]);
                        dst[e8] = o;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce(b));   // this warp's lanes of the buffer are drained
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ---------------------------------------------------------------- CTA-pair GEMM (cta_group::2)
// gemm_tc2_kernel: a cluster of two CTAs computes 256 (tokens) x 256 (out features) tiles with
// tcgen05.mma.cta_group::2 M256 N256 K16: each CTA loads its own 128 activation rows and HALF of the 256 weight
// rows of every K step (the MMA reads the other half from the peer's shared memory at the same offset) and keeps
// its 128 x 256 fp32 accumulator rows in its own TMEM.  Per SM and K step that is 32 KiB of TMA and 32 KiB of
// operand reads instead of 48 + 48 KiB with a 128 x 256 tile per CTA: the shared-memory port, not the tensor
// pipe, bounded the single-CTA kernel.  The leader CTA's MMA warp issues for the pair; both CTAs' TMA bytes land
// on the leader's full[] barriers; commits are multicast to both CTAs (empty[], acc_full[]); both CTAs'
// epilogue warps release an accumulator buffer on the leader's acc_empty[].
#ifndef HI_GEMM_2CTA
#define HI_GEMM_2CTA 1
#endif
constexpr int P_GM = 256, P_GN = 256, P_GK = 64;    // pair tile; per CTA 128 rows of X, 128 rows of W per K step
constexpr int P_STAGES = 6;
constexpr int P_A_BYTES = 128 * P_GK * 2;           // 16 KiB: this CTA's activation rows
constexpr int P_B_BYTES = 128 * P_GK * 2;           // 16 KiB: this CTA's half of the weight rows
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
struct __align__(8) PairBars {
    uint64_t full[P_STAGES], empty[P_STAGES];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};
constexpr int P_SMEM = P_STAGES * P_STAGE_BYTES + static_cast<int>(sizeof(PairBars)) + 1024;

template <bool F32OUT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                    void* __restrict__ yv, int n, int mo, int kd, int beta) {
    extern __shared__ uint8_t g_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(g_raw) + 1023) & ~uintptr_t(1023));
    PairBars* bars = reinterpret_cast<PairBars*>(smem + P_STAGES * P_STAGE_BYTES);
    const uint32_t sbase = smem_addr(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int tiles_m = (n + P_GM - 1) / P_GM, tiles_n = (mo + P_GN - 1) / P_GN, tiles = tiles_m * tiles_n;
    const int kt = (kd + P_GK - 1) / P_GK;
    auto full = [&](int s) { return smem_addr(&bars->full[s]); };
    auto empty = [&](int s) { return smem_addr(&bars->empty[s]); };
    auto accf = [&](int b) { return smem_addr(&bars->acc_full[b]); };
    auto acce = [&](int b) { return smem_addr(&bars->acc_empty[b]); };
    if (threadIdx.x == 0) {
        for (int s = 0; s < P_STAGES; ++s) {
            mbar_init(full(s), 1);    // leader's: its producer's arrive.expect_tx; both CTAs' bytes
            mbar_init(empty(s), 1);   // both: one multicast commit per use
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(accf(b), 1);                  // both: one multicast commit per tile
            mbar_init(acce(b), 2 * G_EPI_WARPS);    // leader's: every epilogue warp of the pair
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&bars->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();   // both CTAs' barriers initialised and TMEM allocated before any cross-CTA traffic
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer (both CTAs): this CTA's X rows and half of the W rows
            int it = 0;
            for (int t = pair; t < tiles; t += n_pairs) {
                int mb, nb;
                tile_coords(t, tiles_m, tiles_n, mb, nb);
                for (int k = 0; k < kt; ++k, ++it) {
                    const int s = it % P_STAGES;
                    if (it >= P_STAGES) mbar_wait_cluster(empty(s), ((it / P_STAGES) - 1) & 1);
                    if (leader) mbar_expect_tx(full(s), 2 * P_STAGE_BYTES);   // OOB rows are zero-filled, still counted
                    const uint32_t full_l = mapa_shared(full(s), 0);
                    tma_load_2d_cg2(sbase + s * P_STAGE_BYTES, &tm_x, full_l, k * P_GK, mb * P_GM + static_cast<int>(rank) * 128);
                    tma_load_2d_cg2(sbase + s * P_STAGE_BYTES + P_A_BYTES, &tm_w, full_l, k * P_GK,
                                    nb * P_GN + static_cast<int>(rank) * 128);
                }
            }
            // tail: the leader's multicast commits for the last stages must have landed in this CTA's barriers
            // before it can exit (they fire asynchronously on MMA completion)
            for (int j = it > P_STAGES ? it - P_STAGES : 0; j < it; ++j)
                mbar_wait_cluster(empty(j % P_STAGES), (j / P_STAGES) & 1);
        }
    } else if (warp == 1) {
        if (leader) {   // ---------------- MMA issuer for the pair: the whole warp runs the loop, elect.sync issues
            constexpr uint32_t IDESC = idesc_bf16(P_GM, P_GN, false);
            int it = 0, i = 0;
            for (int t = pair; t < tiles; t += n_pairs, ++i) {
                const int b = i & 1;
                if (i >= 2) mbar_wait_cluster(acce(b), ((i >> 1) - 1) & 1);   // both epilogues drained this buffer
                tc_fence_after();
                const uint32_t acc = tmem + b * P_GN;
                for (int k = 0; k < kt; ++k, ++it) {
                    const int s = it % P_STAGES;
                    mbar_wait_cluster(full(s), (it / P_STAGES) & 1);
                    tc_fence_after();
                    const uint64_t da = sdesc(sbase + s * P_STAGE_BYTES, 16, 1024);
                    const uint64_t db = sdesc(sbase + s * P_STAGE_BYTES + P_A_BYTES, 16, 1024);
#pragma unroll
                    for (int kk = 0; kk < P_GK / 16; ++kk)
                        umma_bf16_cg2_w(acc, da + (kk * 2), db + (kk * 2), IDESC, (k > 0 || kk > 0) ? 1u : 0u);
                    umma_commit_cg2_mc_w(empty(s), 0x3);   // both CTAs' stage s is free once these MMAs have read it
                }
                umma_commit_cg2_mc_w(accf(b), 0x3);        // both CTAs' accumulator rows complete
            }
        }
    } else {
        // ---------------- epilogue (both CTAs): warp w owns TMEM lanes 32*(w%4) .. +31 = rows of this CTA's half
        const int q = warp & 3;
        const int r_in = static_cast<int>(rank) * 128 + q * 32 + lane;
        const uint32_t acce_l0 = mapa_shared(acce(0), 0), acce_l1 = mapa_shared(acce(1), 0);
        int i = 0;
        for (int t = pair; t < tiles; t += n_pairs, ++i) {
            int mb, nb;
            tile_coords(t, tiles_m, tiles_n, mb, nb);
            const int b = i & 1;
            mbar_wait_cluster(accf(b), (i >> 1) & 1);
            tc_fence_after();
            const int row = mb * P_GM + r_in;
            const bool live = row < n;
            const int64_t yoff = static_cast<int64_t>(row) * mo + nb * P_GN;
            const uint32_t taddr = tmem + b * P_GN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
            for (int c = 0; c < P_GN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(taddr + c * 32, v);
                tmem_wait_ld();
                const int col = nb * P_GN + c * 32;
                if (F32OUT && live && col < mo) {
                    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(yv) + yoff + c * 32);
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4)
                        dst[e4] = make_float4(__uint_as_float(v[4 * e4]), __uint_as_float(v[4 * e4 + 1]),
                                              __uint_as_float(v[4 * e4 + 2]), __uint_as_float(v[4 * e4 + 3]));
                } else if (live && col < mo) {
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(yv) + yoff + c * 32);
                    float f[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(v[e]);
                    if (beta) {
#pragma unroll
                        for (int e8 = 0; e8 < 4; ++e8) {
                            const uint4 u = dst[e8];
                            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                f[e8 * 8 + 2 * h] += __uint_as_float(w4[h] << 16);
                                f[e8 * 8 + 2 * h + 1] += __uint_as_float(w4[h] & 0xffff0000u);
                            }
                        }
                    }
#pragma unroll
                    for (int e8 = 0; e8 < 4; ++e8) {
                        uint4 o;
                        o.x = pack_bf16(f[e8 * 8 + 0], f[e8 * 8 + 1]);
                        o.y = pack_bf16(f[e8 * 8 + 2], f[e8 * 8 + 3]);
                        o.z = pack_bf16(f[e8 * 8 + 4], f[e8 * 8 + 5]);
                        o.w = pack_bf16(f[e8 * 8 + 6], f[e8 * 8 + 7]);
                        dst[e8] = o;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(b ? acce_l1 : acce_l0);   // this warp's rows of the buffer are drained
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();   // the pair's last MMAs wrote both CTAs' TMEM; free it only when both are done
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// y[o] = (beta ? y[o] : 0) + x . W[o, :]; 8 warps per CTA, 2 output rows per warp, x staged in shared memory
constexpr int GV_WARPS = 8, GV_ROWS = 2;

template <bool F32OUT>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_kernel(const __nv_bfloat16* __restrict__ w,
                                                             const __nv_bfloat16* __restrict__ x,
                                                             void* __restrict__ yv, int mo, int kd, int beta) {
    extern __shared__ float xs[];   // [kd]
    for (int i = threadIdx.x; i < kd; i += blockDim.x) xs[i] = __bfloat162float(x[i]);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int o0 = (blockIdx.x * GV_WARPS + warp) * GV_ROWS;
    const int k8 = kd / 8;
    float acc[GV_ROWS] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < GV_ROWS; ++r) {
        if (o0 + r >= mo) break;
        const uint4* wr = reinterpret_cast<const uint4*>(w + static_cast<int64_t>(o0 + r) * kd);
#pragma unroll 4
        for (int i = lane; i < k8; i += 32) {
            const uint4 u = __ldcs(wr + i);   // streamed once: do not keep in L2
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
            const float4 xa = reinterpret_cast<const float4*>(xs)[2 * i];
            const float4 xb = reinterpret_cast<const float4*>(xs)[2 * i + 1];
            const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                acc[r] = fmaf(__uint_as_float(w4[h] << 16), xv[2 * h], acc[r]);
                acc[r] = fmaf(__uint_as_float(w4[h] & 0xffff0000u), xv[2 * h + 1], acc[r]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < GV_ROWS; ++r) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
        if (lane == 0 && o0 + r < mo) {
            if constexpr (F32OUT) {
                static_cast<float*>(yv)[o0 + r] = acc[r];
            } else {
                __nv_bfloat16* y = static_cast<__nv_bfloat16*>(yv);
                const float base = beta ? __bfloat162float(y[o0 + r]) : 0.f;
                y[o0 + r] = __float2bfloat16_rn(base + acc[r]);
            }
        }
    }
}

template <bool F32OUT>
cudaError_t launch_gemm_t(const __nv_bfloat16* w, const __nv_bfloat16* x, void* y, int mo, int n, int kd, int beta,
                          cudaStream_t stream) {
    if (n == 1) {
        const int rows_per_cta = GV_WARPS * GV_ROWS;
        const size_t smem = static_cast<size_t>(kd) * sizeof(float);
        static std::atomic<unsigned long long> configured{0};
        if (smem > 48 * 1024)
            if (cudaError_t e = set_smem_attr_once(gemv_kernel<F32OUT>, 227 * 1024, configured); e != cudaSuccess) return e;
        gemv_kernel<F32OUT><<<(mo + rows_per_cta - 1) / rows_per_cta, GV_WARPS * 32, smem, stream>>>(w, x, y, mo, kd, beta);
        return cudaGetLastError();
    }
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (HI_GEMM_2CTA) {
        static std::atomic<unsigned long long> configured2{0};
        if (cudaError_t e = set_smem_attr_once(gemm_tc2_kernel<F32OUT>, P_SMEM, configured2); e != cudaSuccess) return e;
        CUtensorMap tx, tw;
        const cuuint64_t dx[2] = {static_cast<cuuint64_t>(kd), static_cast<cuuint64_t>(n)};
        const cuuint64_t dw[2] = {static_cast<cuuint64_t>(kd), static_cast<cuuint64_t>(mo)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kd) * 2};
        const cuuint32_t box[2] = {P_GK, 128};
        if (!make_tmap_bf16(&tx, x, 2, dx, strides, box)) return cudaErrorInvalidValue;
        if (!make_tmap_bf16(&tw, w, 2, dw, strides, box)) return cudaErrorInvalidValue;
        const int tiles = ((n + P_GM - 1) / P_GM) * ((mo + P_GN - 1) / P_GN);
        const int pairs = tiles < sms / 2 ? tiles : sms / 2;
        gemm_tc2_kernel<F32OUT><<<2 * pairs, G_THREADS, P_SMEM, stream>>>(tx, tw, y, n, mo, kd, beta);
        return cudaGetLastError();
    }
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = set_smem_attr_once(gemm_tc_kernel<F32OUT>, G_SMEM, configured); e != cudaSuccess) return e;
    CUtensorMap tx, tw;
    {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kd), static_cast<cuuint64_t>(n)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kd) * 2};
        const cuuint32_t box[2] = {GK, GM};
        if (!make_tmap_bf16(&tx, x, 2, dims, strides, box)) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kd), static_cast<cuuint64_t>(mo)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kd) * 2};
        const cuuint32_t box[2] = {GK, GN};
        if (!make_tmap_bf16(&tw, w, 2, dims, strides, box)) return cudaErrorInvalidValue;
    }
    const int tiles = ((n + GM - 1) / GM) * ((mo + GN - 1) / GN);
    gemm_tc_kernel<F32OUT><<<tiles < sms ? tiles : sms, G_THREADS, G_SMEM, stream>>>(tx, tw, y, n, mo, kd, beta);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm(const __nv_bfloat16* w, const __nv_bfloat16* x, void* y, int mo, int n, int kd, int beta,
                        int out_f32, cudaStream_t stream) {
    if (mo <= 0 || n <= 0 || kd <= 0 || mo % 64 || kd % 8 || (out_f32 && beta)) return cudaErrorInvalidValue;
    return out_f32 ? launch_gemm_t<true>(w, x, y, mo, n, kd, 0, stream) : launch_gemm_t<false>(w, x, y, mo, n, kd, beta, stream);
}

}  // namespace hi
