// k_prefill_tc2.cu -- sm_100a prefill attention over one KV segment with CTA-pair (cta_group::2) MMAs.
//
// Same contract and math as k_prefill_tc.cu (Eq. 9; resumable (O, m, l)
// state per key segment, causal across chunks, GQA-packed rows), but a cluster of two CTAs on one
// TPC computes M = 256 tiles: each CTA keeps its two 128-row Q tiles, and every
// tcgen05.mma.cta_group::2 multiplies the pair's 256 rows by a B operand whose N columns are split
// between the two CTAs' shared memory -- K rows (keys) for S = Q K^T, V columns (head dims) for
// O += P V.  So each SM loads and reads only half of every K/V tile: half the L2 -> SMEM traffic
// (which with one CTA per tile pair was ~40% of the kernel time even with no MMA at all) and half
// the B-operand SMEM reads of the single-CTA kernel, with one MMA issue per pair.
//
// Roles per CTA (384 threads): warps 0-7 softmax (thread = TMEM lane = row of its own tile), warp 8
// TMA producer, warp 9 TMEM allocator; the leader CTA's warp 9 lane 0 issues every MMA of the pair.
// Synchronisation: TMA bytes of both CTAs land on the LEADER's full[] barriers (cta_group::2 TMA);
// both CTAs' softmax threads arrive on the leader's p_full[] barriers (cluster-scope arrive); the
// MMA commits are multicast to the barrier at the same offset in both CTAs (s_full, o_done, empty).
// head_dim 128 only (each CTA's half of V is one 64-column SWIZZLE_128B box); d = 64 uses the
// single-CTA kernel.
#include "../hi_kernels.cuh"
#include "../tc_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <mutex>

namespace hi {
namespace {
using namespace ptx;

constexpr int D = 128;
constexpr int BM = 128;              // rows per Q tile (per CTA, per tile)
constexpr int BN = 128;              // keys per KV tile (pair-wide)
constexpr int NS = 4;                // K/V stages (each CTA: 16 KiB of K + 16 KiB of V per stage)
constexpr int NUM_THREADS = 384;
constexpr int WARP_TMA = 8, WARP_MMA = 9;
constexpr float RESCALE_THRESHOLD = 8.0f;
// HI_WARP_ISSUE (as in k_prefill_tc.cu): the whole MMA warp runs the issue loop, elect.sync picks the lane
#ifndef HI_WARP_ISSUE
#define HI_WARP_ISSUE 1
#endif
#if HI_WARP_ISSUE
#define umma_bf16_cg2 umma_bf16_cg2_w
#define umma_bf16_ts_cg2 umma_bf16_ts_cg2_w
#define umma_commit_cg2_mc umma_commit_cg2_mc_w
#endif

constexpr int QBOX = BM * 128;       // [128 rows][64 d] bf16 SW128 = 16 KiB
constexpr int KBOX = (BN / 2) * 128; // [64 keys][64 d] = 8 KiB  (this CTA's half of the keys)
constexpr int VBOX = BN * 128;       // [128 keys][64 d] = 16 KiB (this CTA's half of the dims)
constexpr int Q_OFF = 0;             // 2 tiles x 2 boxes
constexpr int K_OFF = Q_OFF + 2 * 2 * QBOX;
constexpr int V_OFF = K_OFF + NS * 2 * KBOX;
constexpr int BAR_OFF = V_OFF + NS * VBOX;

struct __align__(8) Bars {
    uint64_t q_full;                 // leader: both CTAs' Q bytes
    uint64_t full[NS];               // leader: both CTAs' K/V bytes of a stage
    uint64_t empty[NS];              // both: stage consumed (multicast commit)
    uint64_t s_full[2];              // both: S of tile tt ready (multicast commit)
    uint64_t p_full[2];              // leader: P of tile tt written by 2 x 128 softmax threads
    uint64_t o_done[2];              // both: last PV of tile tt done (multicast commit)
    uint32_t tmem_base;
};
constexpr int SMEM_BYTES = BAR_OFF + static_cast<int>(sizeof(Bars)) + 1024;

__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 208;"); }
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 88;"); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    prefill_tc2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const PrefillParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + BAR_OFF);
    const uint32_t sbase = smem_addr(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int g = p.g;
    const int n_rows = p.n_q * g;
    const int pair_row0 = (blockIdx.x >> 1) * (4 * BM);
    const int row0 = pair_row0 + static_cast<int>(rank) * (2 * BM);   // this CTA's 256 rows
    const bool first = p.flags & PF_FIRST, last = p.flags & PF_LAST, causal = p.flags & PF_CAUSAL;

    // KV tiles the pair streams for tile tt: set by the later-token CTA (rank 1) of the pair
    auto kt_count = [&](int r0) {
        const int t_hi = min(p.n_q - 1, (r0 + BM - 1) / g);
        int64_t e = p.n_k;
        if (causal) {
            const int64_t lim = p.q_pos0 + t_hi - p.k_pos0 + 1;
            e = lim < e ? lim : e;
        }
        e = e > 0 ? e : 0;
        return static_cast<int>((e + BN - 1) / BN);
    };
    const int nk_t[2] = {kt_count(pair_row0 + 2 * BM), kt_count(pair_row0 + 3 * BM)};
    const int n_kt = max(nk_t[0], nk_t[1]);

    auto A = [&](const void* ptr) { return smem_addr(ptr); };
    if (threadIdx.x == 0) {
        mbar_init(A(&bars->q_full), 1);
        for (int s = 0; s < NS; ++s) {
            mbar_init(A(&bars->full[s]), 1);
            mbar_init(A(&bars->empty[s]), 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(A(&bars->s_full[t]), 1);
            mbar_init(A(&bars->p_full[t]), 2 * 128);
            mbar_init(A(&bars->o_done[t]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(A(&bars->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any cross-CTA traffic
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp >= 8) {
        setmaxnreg_dec();
        if (warp == WARP_TMA && lane == 0 && n_kt > 0) {
            // ============================ TMA producer (both CTAs) ============================
            const uint32_t q_full_l = mapa_shared(A(&bars->q_full), 0);
            if (leader) mbar_expect_tx(A(&bars->q_full), 2 * 2 * 2 * QBOX);
            for (int tt = 0; tt < 2; ++tt)
                for (int c = 0; c < 2; ++c)
                    tma_load_3d_cg2(sbase + Q_OFF + (tt * 2 + c) * QBOX, &tm_q, q_full_l, c * 64, 0, (row0 + tt * BM) / g);
            for (int i = 0; i < n_kt; ++i) {
                const int s = i % NS;
                if (i >= NS) mbar_wait(A(&bars->empty[s]), ((i / NS) - 1) & 1);
                const uint32_t full_l = mapa_shared(A(&bars->full[s]), 0);
                if (leader) mbar_expect_tx(A(&bars->full[s]), 2 * (2 * KBOX + VBOX));
                // K: this CTA's 64 keys (all 128 dims); V: all 128 keys, this CTA's 64 dims
                for (int c = 0; c < 2; ++c)
                    tma_load_2d_cg2(sbase + K_OFF + (s * 2 + c) * KBOX, &tm_k, full_l, c * 64,
                                    i * BN + static_cast<int>(rank) * (BN / 2));
                tma_load_2d_cg2(sbase + V_OFF + s * VBOX, &tm_v, full_l, static_cast<int>(rank) * 64, i * BN);
            }
        } else if (warp == WARP_MMA && (HI_WARP_ISSUE || lane == 0) && leader && n_kt > 0) {
            // ============================ MMA issuer (leader CTA) ============================
            constexpr uint32_t ID_S = idesc_bf16(2 * BM, BN, false);  // M = 256 (pair), N = 128 keys
            constexpr uint32_t ID_O = idesc_bf16(2 * BM, D, true);    // M = 256, N = 128 dims
            const uint64_t dq0 = sdesc(sbase + Q_OFF, 16, 1024);
            const uint64_t dk0 = sdesc(sbase + K_OFF, 16, 1024);
            const uint64_t dv0 = sdesc(sbase + V_OFF, 16, 1024);
            mbar_wait_cluster(A(&bars->q_full), 0);
            auto issue_s = [&](int tt, int i) {
                const int s = i % NS;
                const uint64_t a0 = dq0 + ((tt * 2 * QBOX) >> 4);
                const uint64_t b0 = dk0 + ((s * 2 * KBOX) >> 4);
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t qo = ((ks >> 2) * QBOX + (ks & 3) * 32) >> 4;
                    const uint32_t ko = ((ks >> 2) * KBOX + (ks & 3) * 32) >> 4;
                    umma_bf16_cg2(tmem + tt * 256, a0 + qo, b0 + ko, ID_S, ks > 0);
                }
                umma_commit_cg2_mc(A(&bars->s_full[tt]), 0x3);
            };
            auto issue_pv = [&](int tt, int j) {
                const int s = j % NS;
                const uint64_t b0 = dv0 + ((s * VBOX) >> 4);
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk)
                    umma_bf16_ts_cg2(tmem + tt * 256 + 128, tmem + tt * 256 + kk * 8, b0 + ((kk * 16 * 128) >> 4), ID_O,
                                     (j > 0 || kk > 0 || !first) ? 1u : 0u);
                if (j + 1 == nk_t[tt]) umma_commit_cg2_mc(A(&bars->o_done[tt]), 0x3);
            };
            mbar_wait_cluster(A(&bars->full[0]), 0);
            tc_fence_after();
            for (int tt = 0; tt < 2; ++tt)
                if (nk_t[tt] > 0) issue_s(tt, 0);
            for (int j = 0; j < n_kt; ++j) {
                bool waited_next = false;
                for (int tt = 0; tt < 2; ++tt) {
                    if (j >= nk_t[tt]) continue;
                    mbar_wait_cluster(A(&bars->p_full[tt]), j & 1);
                    tc_fence_after();
                    issue_pv(tt, j);
                    if (j + 1 < nk_t[tt]) {
                        if (!waited_next) {
                            mbar_wait_cluster(A(&bars->full[(j + 1) % NS]), ((j + 1) / NS) & 1);
                            waited_next = true;
                        }
                        tc_fence_after();
                        issue_s(tt, j + 1);
                    }
                }
                umma_commit_cg2_mc(A(&bars->empty[j % NS]), 0x3);  // K/V stage j consumed by both tiles
            }
        }
    } else {
        // ====================== softmax / correction / epilogue (both CTAs, warps 0-7) ======================
        setmaxnreg_inc();
        const int tt = warp >> 2;
        const int wq = warp & 3;
        const int r = wq * 32 + lane;
        const int rg = row0 + tt * BM + r;
        const bool row_valid = rg < n_rows;
        const int t = row_valid ? rg / g : 0;
        const int64_t qpos = p.q_pos0 + t;
        const int nkt = nk_t[tt];
        const int t_lo = (row0 + tt * BM) / g;
        const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t t_s = tmem + tt * 256 + lane_addr;
        const uint32_t t_o = t_s + 128;
        const uint32_t p_full_l = mapa_shared(A(&bars->p_full[tt]), 0);
        const float sc = p.scale_log2;
        float m_run = -CUDART_INF_F, l_run = 0.f;
        if (!first) {
            m_run = row_valid ? p.m_acc[rg] : -CUDART_INF_F;
            l_run = row_valid ? p.l_acc[rg] : 0.f;
            if (nkt > 0) {
#pragma unroll
                for (int cb = 0; cb < D / 32; ++cb) {
                    uint32_t v[32];
                    const float4* src = reinterpret_cast<const float4*>(p.o_acc + static_cast<int64_t>(row_valid ? rg : 0) * D + cb * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float4 f = row_valid ? src[i] : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[4 * i] = __float_as_uint(f.x); v[4 * i + 1] = __float_as_uint(f.y);
                        v[4 * i + 2] = __float_as_uint(f.z); v[4 * i + 3] = __float_as_uint(f.w);
                    }
                    tmem_st32(t_o + cb * 32, v);
                }
                tmem_wait_st();
            }
        }
        for (int j = 0; j < nkt; ++j) {
            mbar_wait(A(&bars->s_full[tt]), j & 1);  // implies PV(j-1) of this tile is complete (in-order)
            tc_fence_after();
            uint32_t x[BN];
#pragma unroll
            for (int cb = 0; cb < BN / 32; ++cb)
                tmem_ld32(t_s + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
            tmem_wait_ld();
#ifdef HI_FAKE_SOFTMAX  // timing experiment only
            tc_fence_before();
            mbar_arrive_cluster(p_full_l);
            continue;
#endif
            const int key0 = j * BN;
            const bool need_mask = (key0 + BN > p.n_k) || (causal && p.k_pos0 + key0 + BN - 1 > p.q_pos0 + t_lo);
            if (need_mask) {
                const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                for (int i = 0; i < BN; ++i)
                    if (key0 + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
            }
            float mk[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
            for (int i = 8; i < BN; i += 8)
#pragma unroll
                for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
            const float mx = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])), fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
            const float mxs = mx * sc;
            float m_ref = m_run, alpha = 1.f;
            const bool grow = (mx != -CUDART_INF_F) && (m_run == -CUDART_INF_F || mxs > m_run + RESCALE_THRESHOLD);
            if (grow) {
                m_ref = mxs;
                alpha = (m_run == -CUDART_INF_F) ? 0.f : ex2(m_run - mxs);
            }
            const float neg_m = (m_ref == -CUDART_INF_F) ? 0.f : -m_ref;
            float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < BN; i += 2) {
                const float p0 = ex2(fmaf(__uint_as_float(x[i]), sc, neg_m));
                const float p1 = ex2(fmaf(__uint_as_float(x[i + 1]), sc, neg_m));
                ls[(i >> 1) & 3] += p0 + p1;
                x[i / 2] = pack_bf16(p0, p1);
            }
            tmem_st32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
            tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&x[32]));
            const bool o_live = !first || j > 0;
            if (o_live && __any_sync(0xffffffffu, grow)) {
#pragma unroll
                for (int cb = 0; cb < D / 32; ++cb) {
                    uint32_t v[32];
                    tmem_ld32(t_o + cb * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                    tmem_st32(t_o + cb * 32, v);
                }
            }
            tmem_wait_st();
            l_run = l_run * alpha + ((ls[0] + ls[1]) + (ls[2] + ls[3]));
            m_run = m_ref;
            tc_fence_before();
            mbar_arrive_cluster(p_full_l);
        }
        if (nkt > 0) {
            mbar_wait(A(&bars->o_done[tt]), 0);
            tc_fence_after();
        }
        if (last) {
            const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
            __nv_bfloat16* dst = p.out + static_cast<int64_t>(t) * p.o_tok_stride + (rg % g) * D;
#pragma unroll
            for (int cb = 0; cb < D / 32; ++cb) {
                uint32_t v[32];
                if (nkt > 0) {
                    tmem_ld32(t_o + cb * 32, v);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        v[i] = (row_valid && !first) ? __float_as_uint(p.o_acc[static_cast<int64_t>(rg) * D + cb * 32 + i]) : 0u;
                }
                if (row_valid) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        uint4 w;
                        w.x = pack_bf16(__uint_as_float(v[8 * i]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
                        w.y = pack_bf16(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
                        w.z = pack_bf16(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
                        w.w = pack_bf16(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
                        *reinterpret_cast<uint4*>(dst + cb * 32 + 8 * i) = w;
                    }
                }
            }
        } else if (nkt > 0) {
#pragma unroll
            for (int cb = 0; cb < D / 32; ++cb) {
                uint32_t v[32];
                tmem_ld32(t_o + cb * 32, v);
                tmem_wait_ld();
                if (row_valid) {
                    float4* dst = reinterpret_cast<float4*>(p.o_acc + static_cast<int64_t>(rg) * D + cb * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
            }
            if (row_valid) {
                p.m_acc[rg] = m_run;
                p.l_acc[rg] = l_run;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the pair's last MMAs wrote both CTAs' TMEM; free it only when both are done
    if (warp == WARP_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

}  // namespace

cudaError_t launch_prefill_tc2(const PrefillParams& p, int d, cudaStream_t stream) {
    if (d != D) return cudaErrorInvalidValue;
    const int n_rows = p.n_q * p.g;
    const int pairs = (n_rows + 4 * BM - 1) / (4 * BM);
    if (pairs == 0) return cudaSuccess;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(prefill_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap tq, tk, tv;
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.g), static_cast<cuuint64_t>(p.n_q)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(p.q_tok_stride) * 2};
        const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(p.g), static_cast<cuuint32_t>(BM / p.g)};
        if (!make_tmap_bf16(&tq, p.q, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.n_k)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.kv_row_stride) * 2};
        const cuuint32_t kbox[2] = {64, BN / 2};
        const cuuint32_t vbox[2] = {64, BN};
        if (!make_tmap_bf16(&tk, p.k, 2, dims, strides, kbox)) return cudaErrorInvalidValue;
        if (!make_tmap_bf16(&tv, p.v, 2, dims, strides, vbox)) return cudaErrorInvalidValue;
    }
    prefill_tc2_kernel<<<2 * pairs, NUM_THREADS, SMEM_BYTES, stream>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

}  // namespace hi
