// k_prefill_tc1.cu -- sm_100a prefill attention over one KV segment, one 128-row Q tile per CTA with a
// three-deep S/P ring in TMEM (TMA -> SMEM -> tcgen05.mma, fp32 online softmax on CUDA cores).
//
// Same contract and math as k_prefill_tc.cu (Eq. 9; resumable (O, m, l)
// state per key segment, causal across chunks, GQA-packed rows t*g+j, head groups on grid.y), different
// schedule.  In the two-tile kernel P(j) aliases S(j) in TMEM, so S(j+1) of a tile can only be issued
// after PV(j) has read P(j): every KV tile costs  softmax + PV + QK^T  in series per Q tile, and the
// tensor core idles while the softmax runs (profiles/trace_r01: ~3500 cycles per KV tile and tile pair
// vs 2048 of MMA work).  Here TMEM holds three S buffers (3 x 128 columns) + O (d columns): QK^T for KV
// tiles j+1 and j+2 is already computed while the softmax works on tile j, and PV(j) is issued as soon
// as P(j) is stored, so the per-tile cost is max(softmax, PV + QK^T) instead of their sum.  Eight
// softmax warps share the tile (warp w: TMEM lane quarter w%4 = rows, key half w/4 = 64 of the 128
// columns; the row max is exchanged through shared memory), which halves the softmax latency.  K/V
// tiles are multicast to a cluster of CL CTAs (consecutive row tiles of the same kv head), so the
// L2 -> SMEM traffic per FLOP equals the two-tile kernel's at CL = 2.
//
// TMEM columns (512 allocated): S/P buffer b in {0,1,2} at [128 b, 128 b + 128); O at [384, 384 + d).
// P(j) (bf16 pairs) overwrites the first 64 columns of buffer j%3 once both key halves have read S(j).
//
// Warps: 0-7 softmax / O correction / epilogue; 8 TMA (Q + K ring); 9 TMEM allocator + MMA issuer;
// 10 TMA (V ring); 11 idle.
#include "../hi_kernels.cuh"
#include "../tc_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <mutex>

namespace hi {
namespace {

constexpr int BM = 128;            // query rows per CTA (TMEM lanes)
constexpr int BN = 128;            // keys per KV tile
constexpr int NSB = 3;             // S/P buffers in TMEM
#ifndef HI_T1_NK
#define HI_T1_NK 3
#endif
#ifndef HI_T1_NV
#define HI_T1_NV 2
#endif
#ifndef HI_T1_CL
#define HI_T1_CL 1  // multicast measured 3x slower per SM than plain TMA (profiles/ubench_tma_rate_r01.txt)
#endif
#ifndef HI_T1_PACKED
#define HI_T1_PACKED 0  // FFMA2/FADD2 softmax (spills here: x[128] pairs need aligned register pairs)
#endif
constexpr int NK = HI_T1_NK;       // K ring stages
constexpr int NV = HI_T1_NV;       // V ring stages
constexpr int CL = HI_T1_CL;       // K/V multicast cluster size
constexpr int SOFTMAX_WARPS = 8;
constexpr int WARP_TMA = 8, WARP_MMA = 9, WARP_TMA_V = 10;
constexpr int NUM_THREADS = 384;
// setmaxnreg: softmax 256 threads x +40 = producers 128 x -80 (launch 168 = 64K / 384)
constexpr int REG_SOFTMAX = 208, REG_PRODUCER = 88;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units
// HI_WARP_ISSUE (as in k_prefill_tc.cu): the whole MMA warp runs the issue loop, elect.sync picks the lane
#ifndef HI_WARP_ISSUE
#define HI_WARP_ISSUE 1
#endif

#if HI_T1_CL > 1
#define HI_T1_CLUSTER_ATTR __cluster_dims__(HI_T1_CL, 1, 1)
#else
#define HI_T1_CLUSTER_ATTR
#endif

using namespace ptx;
#if HI_WARP_ISSUE
#define T1_UMMA umma_bf16_w
#define T1_UMMA_TS umma_bf16_ts_w
#define T1_UCOMMIT umma_commit_w
#else
#define T1_UMMA umma_bf16
#define T1_UMMA_TS umma_bf16_ts
#define T1_UCOMMIT umma_commit
#endif

// Optional timeline trace (variant builds with -DHI_TRACE): clock64() at pipeline events of CTA 0
// (blockIdx 0,0), read back with hi_debug_prefill_trace1(); off in the product build.
#ifdef HI_TRACE
__device__ unsigned long long g_hi_trace1[16][512];
#define T1_TR(ev, j) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 512) g_hi_trace1[ev][j] = clock64(); } while (0)
#else
#define T1_TR(ev, j) do { } while (0)
#endif

struct __align__(8) Barriers {
    uint64_t q_full;
    uint64_t k_full[NK], k_empty[NK], v_full[NV], v_empty[NV];
    uint64_t s_full[NSB], p_full[NSB];
    uint64_t pv_done[2];             // [j parity]: one phase per PV(j) of that parity (O holds every PV <= j)
    uint64_t o_done;                 // last PV complete
    uint32_t tmem_base;
    uint32_t pad;
    float xchg[2][1][BM];            // [warp set][row]: reference max handed to the other set / final m_l
    float xchg_l[2][BM];             // [warp set][row]: partial row sum (epilogue)
};

template <int D>
struct Smem {
    static constexpr int BOX = BM * 128;            // one [128 rows][64 bf16] SW128 box = 16 KiB
    static constexpr int Q_OFF = 0;                 // D/64 boxes
    static constexpr int K_OFF = Q_OFF + (D / 64) * BOX;
    static constexpr int V_OFF = K_OFF + NK * (D / 64) * BOX;
    static constexpr int BAR_OFF = V_OFF + NV * (D / 64) * BOX;
    static constexpr int BYTES = BAR_OFF + static_cast<int>(sizeof(Barriers));
    static constexpr int ALLOC = BYTES + 1024;      // slack for 1 KiB alignment
    static_assert(ALLOC <= 232448, "shared memory per CTA exceeds the sm_100 limit (227 KiB)");
};

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int D>
__global__ void HI_T1_CLUSTER_ATTR __launch_bounds__(NUM_THREADS, 1)
    prefill_tc1_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const PrefillParams p) {
    using L = Smem<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bars = reinterpret_cast<Barriers*>(smem + L::BAR_OFF);
    const uint32_t sbase = smem_addr(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = p.g;
    const int n_rows = p.n_q * g;
    const int row0 = blockIdx.x * BM;
    const int hh = blockIdx.y;                 // kv head within the launch's head group
    float* const o_acc = p.o_acc + static_cast<int64_t>(hh) * p.state_rows * D;
    float* const m_acc = p.m_acc + static_cast<int64_t>(hh) * p.state_rows;
    float* const l_acc = p.l_acc + static_cast<int64_t>(hh) * p.state_rows;
    const bool first = p.flags & PF_FIRST, last = p.flags & PF_LAST, causal = p.flags & PF_CAUSAL;
    const bool has_tile = row0 < n_rows;       // a CTA padding the grid to whole clusters has none
    const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;

    // KV tiles of the segment visible to the tile at packed row r0 (causal: key c visible to token t
    // iff k_pos0+c <= q_pos0+t); 0 for a tile past the last row
    auto kt_rows = [&](int r0) {
        if (r0 >= n_rows) return 0;
        const int t_hi = min(p.n_q - 1, (r0 + BM - 1) / g);
        int64_t e = p.n_k;
        if (causal) {
            const int64_t lim = p.q_pos0 + t_hi - p.k_pos0 + 1;
            e = lim < e ? lim : e;
        }
        e = e > 0 ? e : 0;
        return static_cast<int>((e + BN - 1) / BN);
    };
    const int nk_own = kt_rows(row0);
    // KV tiles streamed: the cluster's maximum (tiles past this CTA's own causal limit are received and
    // released unused)
    int n_kt = nk_own;
    if constexpr (CL > 1) {
        const int base = (blockIdx.x - crank) * BM;
        for (int c = 0; c < CL; ++c) n_kt = max(n_kt, kt_rows(base + c * BM));
    }

    const uint32_t bar_q = smem_addr(&bars->q_full);
    auto bar_k = [&](int s) { return smem_addr(&bars->k_full[s]); };
    auto bar_ke = [&](int s) { return smem_addr(&bars->k_empty[s]); };
    auto bar_v = [&](int s) { return smem_addr(&bars->v_full[s]); };
    auto bar_ve = [&](int s) { return smem_addr(&bars->v_empty[s]); };
    auto bar_s = [&](int b) { return smem_addr(&bars->s_full[b]); };
    auto bar_p = [&](int b) { return smem_addr(&bars->p_full[b]); };
    auto bar_pvd = [&](int par) { return smem_addr(&bars->pv_done[par]); };
    const uint32_t bar_od = smem_addr(&bars->o_done);

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < NK; ++s) {
            mbar_init(bar_k(s), 1);
            mbar_init(bar_ke(s), CL);
        }
        for (int s = 0; s < NV; ++s) {
            mbar_init(bar_v(s), 1);
            mbar_init(bar_ve(s), CL);
        }
        for (int b = 0; b < NSB; ++b) {
            mbar_init(bar_s(b), 1);
            mbar_init(bar_p(b), 4);  // one arrival per warp of the owning set
        }
        mbar_init(bar_pvd(0), 1);
        mbar_init(bar_pvd(1), 1);
        mbar_init(bar_od, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&bars->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    if constexpr (CL > 1) cluster_sync();  // every CTA's barriers initialised before any multicast lands
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp >= SOFTMAX_WARPS) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_PRODUCER));
        constexpr uint16_t MASK = static_cast<uint16_t>((1u << CL) - 1);
        // box b (K boxes 0..D/64-1, then V boxes) of every tile is issued by CTA rank b % CL (multicast)
        auto load_tile = [&](const CUtensorMap* map, uint32_t off, uint32_t bar, int i, int b0) {
            mbar_expect_tx(bar, (D / 64) * L::BOX);  // the whole tile lands here (own + peers' boxes)
            for (int c = 0; c < D / 64; ++c) {
                if constexpr (CL == 1) {
                    tma_load_3d(sbase + off + c * L::BOX, map, bar, c * 64, i * BN, hh);
                } else if ((b0 + c) % CL == static_cast<int>(crank)) {
                    tma_load_3d_mc(sbase + off + c * L::BOX, map, bar, c * 64, i * BN, hh, MASK);
                }
            }
        };
        if (warp == WARP_TMA && lane == 0 && n_kt > 0) {
            // ======================= TMA producer: Q, then the K ring =======================
            if (has_tile) {
                mbar_expect_tx(bar_q, (D / 64) * L::BOX);
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sbase + L::Q_OFF + c * L::BOX, &tm_q, bar_q, c * 64, hh * g, row0 / g);
            }
            for (int i = 0; i < n_kt; ++i) {
                const int s = i % NK;
                if (i >= NK) mbar_wait(bar_ke(s), ((i / NK) - 1) & 1);
                T1_TR(4, i);  // (slot 4 = K load issue; the softmax set-0 'arrive' stamp is dropped)
                load_tile(&tm_k, L::K_OFF + s * (D / 64) * L::BOX, bar_k(s), i, 0);
            }
        } else if (warp == WARP_TMA_V && lane == 0 && n_kt > 0) {
            // ======================= TMA producer: the V ring ===============================
            for (int i = 0; i < n_kt; ++i) {
                const int s = i % NV;
                if (i >= NV) mbar_wait(bar_ve(s), ((i / NV) - 1) & 1);
                load_tile(&tm_v, L::V_OFF + s * (D / 64) * L::BOX, bar_v(s), i, D / 64);
            }
        } else if (warp == WARP_MMA && (HI_WARP_ISSUE || lane == 0) && n_kt > 0) {
            // ============================ MMA issuer ==============================
            constexpr uint32_t ID_S = idesc_bf16(BM, BN, false);
            constexpr uint32_t ID_O = idesc_bf16(BM, D, true);
            if (has_tile) mbar_wait(bar_q, 0);
            const uint64_t dq0 = sdesc(sbase + L::Q_OFF, 16, 1024);
            const uint64_t dk0 = sdesc(sbase + L::K_OFF, 16, 1024);
            const uint64_t dv0 = sdesc(sbase + L::V_OFF, L::BOX, 1024);
            auto issue_s = [&](int i) {  // S(i) = Q K(i)^T -> buffer i % 3
                const uint64_t b0 = dk0 + (((i % NK) * (D / 64) * L::BOX) >> 4);
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = ((ks >> 2) * L::BOX + (ks & 3) * 32) >> 4;
                    T1_UMMA(tmem + (i % NSB) * 128, dq0 + off, b0 + off, ID_S, ks > 0);
                }
                T1_UCOMMIT(bar_s(i % NSB));
            };
            auto issue_pv = [&](int j) {  // O += P(j) V(j), P from TMEM buffer j % 3
                const uint64_t b0 = dv0 + (((j % NV) * (D / 64) * L::BOX) >> 4);
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk)
                    T1_UMMA_TS(tmem + 384, tmem + (j % NSB) * 128 + kk * 8, b0 + ((kk * 16 * 128) >> 4), ID_O,
                                 (j > 0 || kk > 0 || !first) ? 1u : 0u);
                T1_UCOMMIT(bar_pvd(j & 1));
                if (j + 1 == nk_own) T1_UCOMMIT(bar_od);
            };
            // release a ring slot once every MMA reading it is issued (the commit fires on completion).
            // Cluster: the round must also have fully landed here (this CTA may not have needed it), and
            // the release goes to every CTA of the cluster.
            auto release = [&](uint32_t full, uint32_t empty, uint32_t parity) {
                if constexpr (CL == 1) {
                    T1_UCOMMIT(empty);
                } else {
                    mbar_wait(full, parity);
                    umma_commit_mc(empty, MASK);
                }
            };
            auto do_s = [&](int i) {
                if (i < nk_own) {
                    mbar_wait(bar_k(i % NK), (i / NK) & 1);
                    T1_TR(14, i);
                    tc_fence_after();
                    issue_s(i);
                    T1_TR(15, i);
                }
                release(bar_k(i % NK), bar_ke(i % NK), (i / NK) & 1);
            };
            for (int i = 0; i < min(NSB, n_kt); ++i) do_s(i);
            for (int j = 0; j < n_kt; ++j) {
                if (j < nk_own) {
                    mbar_wait(bar_p(j % NSB), (j / NSB) & 1);
                    T1_TR(10, j);
                    mbar_wait(bar_v(j % NV), (j / NV) & 1);
                    T1_TR(11, j);
                    tc_fence_after();
                    issue_pv(j);
                    T1_TR(12, j);
                }
                release(bar_v(j % NV), bar_ve(j % NV), (j / NV) & 1);
                // S(j+3) reuses buffer j%3: issued after PV(j), which reads P(j) there (MMAs run in order)
                if (j + NSB < n_kt) do_s(j + NSB);
                T1_TR(13, j);
            }
            if constexpr (CL > 1) {
                // drain: every CTA's release of the last rounds has reached this CTA's barriers, so no
                // peer commit is still in flight towards this CTA's shared memory when it exits
                for (int j = max(0, n_kt - NK); j < n_kt; ++j) mbar_wait(bar_ke(j % NK), (j / NK) & 1);
                for (int j = max(0, n_kt - NV); j < n_kt; ++j) mbar_wait(bar_ve(j % NV), (j / NV) & 1);
            }
        }
    } else if (has_tile) {
        // ==== softmax / O correction / epilogue: warp w = lane quarter w%4 (rows), warp set w/4 ====
        // Set X in {0, 1} owns the KV tiles j = X, X+2, X+4, ... (all 128 columns of its rows).  The online
        // softmax chain crosses the sets only through the reference max: set X receives m_ref(j-1) from the
        // other set (shared memory + named barrier), decides m_ref(j), and hands it on before its exponentials,
        // so the two sets' exponential phases overlap on every SMSP (the MUFU unit is shared, the rest of
        // each set's work hides behind the other's exponentials).  Each set keeps its partial row sum
        // relative to the last reference it used; O is shared (one accumulator, rescaled by the owner of
        // the tile whose reference moved, after every earlier PV has landed).
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REG_SOFTMAX));
        constexpr int HD = D / 2;                   // O columns per thread in the epilogue
        const int wq = warp & 3, set = warp >> 2;
        const int r = wq * 32 + lane;               // row within the tile == TMEM lane
        const int rg = row0 + r;                    // packed row index t*g + j
        const bool row_valid = rg < n_rows;
        const int t = row_valid ? rg / g : 0;
        const int64_t qpos = p.q_pos0 + t;
        const int t_lo = row0 / g;
        const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t t_o = tmem + lane_addr + 384;  // O columns of this row
        const float sc = p.scale_log2;
        const uint32_t bar_to_other = 1 + set * 4 + wq;        // this set -> other set (m_ref handoff)
        const uint32_t bar_from_other = 1 + (set ^ 1) * 4 + wq;
        const uint32_t bar_pair = 9 + wq;                       // both sets of this lane quarter
        float m_init = -CUDART_INF_F, l_part = 0.f;
        if (!first) {
            m_init = row_valid ? m_acc[rg] : -CUDART_INF_F;
            l_part = (row_valid && set == 0) ? l_acc[rg] : 0.f;
            if (nk_own > 0) {  // running O -> TMEM (each set half the columns) before PV(0) accumulates
#pragma unroll
                for (int cb = 0; cb < HD / 32; ++cb) {
                    uint32_t v[32];
                    const float4* src = reinterpret_cast<const float4*>(
                        o_acc + static_cast<int64_t>(row_valid ? rg : 0) * D + set * HD + cb * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float4 f = row_valid ? src[i] : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[4 * i] = __float_as_uint(f.x); v[4 * i + 1] = __float_as_uint(f.y);
                        v[4 * i + 2] = __float_as_uint(f.z); v[4 * i + 3] = __float_as_uint(f.w);
                    }
                    tmem_st32(t_o + set * HD + cb * 32, v);
                }
                tmem_wait_st();
                tc_fence_before();
                named_bar_sync(bar_pair, 64);  // set 1's half is in TMEM before set 0 releases P(0)
            }
        }
        // the m_ref chain starts from the segment's incoming max; set 1 waits for set 0's first hand-off
        float m_prev = m_init;                  // m_ref of the previous tile (set 0, tile 0: the incoming max)
        float m_l = (set == 0) ? m_init : -CUDART_INF_F;  // reference of l_part
        for (int j = set; j < nk_own; j += 2) {
            const int b = j % NSB;
            const uint32_t t_s = tmem + lane_addr + b * 128;
            const int tre = (lane == 0 && wq == 0) ? set * 5 : -1;
            mbar_wait(bar_s(b), (j / NSB) & 1);
            if (tre >= 0) T1_TR(tre + 0, j);
            tc_fence_after();
#ifdef HI_FAKE_SOFTMAX  // timing experiment only: the MMA / TMA pipeline without the softmax
            if (lane == 0) mbar_arrive(bar_p(b));
            continue;
#endif
            uint32_t x[BN];
#pragma unroll
            for (int cb = 0; cb < BN / 32; ++cb)
                tmem_ld32(t_s + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
            tmem_wait_ld();
#ifdef HI_FAKE_SOFTMAX_LDST  // timing experiment only: TMEM traffic of the softmax, no math
            tmem_st32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
            tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&x[32]));
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_p(b));
            continue;
#endif
            // masking (causal diagonal / segment tail): keys past this row's limit -> -inf
            const bool need_mask = (j * BN + BN > p.n_k) || (causal && p.k_pos0 + j * BN + BN - 1 > p.q_pos0 + t_lo);
            if (need_mask) {
                const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                for (int i = 0; i < BN; ++i)
                    if (j * BN + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
            }
            float mk[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
            for (int i = 8; i < BN; i += 8)
#pragma unroll
                for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
            const float mx = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])), fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
            // reference of tile j-1 from the other set (tile 0: the incoming max)
            if (j > 0) {
                named_bar_sync(bar_from_other, 64);
                m_prev = bars->xchg[set ^ 1][0][r];
            }
            if (tre >= 0) T1_TR(tre + 1, j);
            const float mxs = mx * sc;  // log2-domain tile max
            // lazy rescale: move the reference max only when it grows by > 2^8
            const bool grow = (mx != -CUDART_INF_F) && (m_prev == -CUDART_INF_F || mxs > m_prev + RESCALE_THRESHOLD);
            const float m_ref = grow ? mxs : m_prev;
            if (j + 1 < nk_own) {  // hand m_ref(j) on to the owner of tile j+1
                bars->xchg[set][0][r] = m_ref;
                asm volatile("bar.arrive %0, %1;" ::"r"(bar_to_other), "r"(64) : "memory");
            }
            const float neg_m = (m_ref == -CUDART_INF_F) ? 0.f : -m_ref;
            // p = 2^(x*scale - m), packed to bf16 pairs in place (x[i/2] is dead once read)
            f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#if HI_T1_PACKED
            const f2 sc2{sc, sc}, nm2{neg_m, neg_m};
#pragma unroll
            for (int i = 0; i < BN; i += 2) {
                const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                const f2 pp{ex2(a.x), ex2(a.y)};
                acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                x[i / 2] = pack_bf16(pp.x, pp.y);
            }
#else
#pragma unroll
            for (int i = 0; i < BN; i += 2) {
                const float p0 = ex2(fmaf(__uint_as_float(x[i]), sc, neg_m));
                const float p1 = ex2(fmaf(__uint_as_float(x[i + 1]), sc, neg_m));
                acc[(i >> 1) & 3].x += p0;
                acc[(i >> 1) & 3].y += p1;
                x[i / 2] = pack_bf16(p0, p1);
            }
#endif
            if (tre >= 0) T1_TR(tre + 2, j);
            // P -> TMEM: packed columns [0, 64) of buffer b
            tmem_st32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
            tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&x[32]));
            if (tre >= 0) T1_TR(tre + 3, j);
            const bool o_live = !first || j > 0;
            if (o_live && __any_sync(0xffffffffu, grow)) {
                // O correction needs every earlier PV complete: wait for PV(j-1) (its commit fires after every
                // earlier MMA).  Waited only here (rarely), yet never ambiguous: the barrier of j's parity
                // class j-1 cannot be two phases behind (S(j), complete, was issued after PV(j-3)) nor
                // ahead (PV(j+1) needs P(j) first).
                if (j > 0) mbar_wait(bar_pvd((j - 1) & 1), ((j - 1) >> 1) & 1);
                const float alpha = (m_prev == -CUDART_INF_F) ? 0.f : ex2(m_prev - m_ref);
                tc_fence_after();
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
            const f2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
            const float sum = (s01.x + s01.y) + (s23.x + s23.y);
            // l_part is relative to m_l; bring it to m_ref (m_ref >= m_l: the reference never decreases)
            l_part = (m_l == -CUDART_INF_F ? 0.f : l_part * ex2(m_l - m_ref)) + sum;
            if (m_ref == -CUDART_INF_F) l_part = 0.f;
            m_l = m_ref;
            m_prev = m_ref;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_p(b));
            if (tre > 0) T1_TR(tre + 4, j);
        }
        // ---- epilogue: combine the two sets' partial sums at the final reference ----
        bars->xchg[set][0][r] = m_l;
        bars->xchg_l[set][r] = l_part;
        named_bar_sync(bar_pair, 64);
        const float m_o = bars->xchg[set ^ 1][0][r], l_o = bars->xchg_l[set ^ 1][r];
        const float m_fin = fmaxf(m_l, m_o);  // the last tile's reference (references never decrease)
        float l_tot = 0.f;
        if (m_fin != -CUDART_INF_F) {
            l_tot = (m_l == -CUDART_INF_F ? 0.f : l_part * ex2(m_l - m_fin)) +
                    (m_o == -CUDART_INF_F ? 0.f : l_o * ex2(m_o - m_fin));
        }
        if (nk_own > 0) {
            mbar_wait(bar_od, 0);
            tc_fence_after();
        }
        const uint32_t t_oh = t_o + set * HD;  // this set's half of the O columns
        if (last) {
            const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
            __nv_bfloat16* dst = p.out + static_cast<int64_t>(t) * p.o_tok_stride + (hh * g + rg % g) * D + set * HD;
#pragma unroll
            for (int cb = 0; cb < HD / 32; ++cb) {
                uint32_t v[32];
                if (nk_own > 0) {
                    tmem_ld32(t_oh + cb * 32, v);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        v[i] = (row_valid && !first)
                                   ? __float_as_uint(o_acc[static_cast<int64_t>(rg) * D + set * HD + cb * 32 + i])
                                   : 0u;
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
        } else if (nk_own > 0) {
#pragma unroll
            for (int cb = 0; cb < HD / 32; ++cb) {
                uint32_t v[32];
                tmem_ld32(t_oh + cb * 32, v);
                tmem_wait_ld();
                if (row_valid) {
                    float4* dst = reinterpret_cast<float4*>(o_acc + static_cast<int64_t>(rg) * D + set * HD + cb * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
            }
            if (row_valid && set == 0) {
                m_acc[rg] = m_fin;
                l_acc[rg] = l_tot;
            }
        }
    }
    tc_fence_before();
    if constexpr (CL > 1) cluster_sync();  // no multicast / remote commit targets this CTA any more
    else __syncthreads();
    if (warp == WARP_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ---------------------------------------------------------------- host side
template <int D>
cudaError_t launch_tc1(const PrefillParams& p, cudaStream_t stream) {
    const int n_rows = p.n_q * p.g;
    const int grid = ((n_rows + BM - 1) / BM + CL - 1) / CL * CL;  // whole clusters
    const int heads = p.n_heads > 0 ? p.n_heads : 1;
    if (n_rows == 0) return cudaSuccess;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(prefill_tc1_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<D>::ALLOC);
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap tq, tk, tv;
    {
        // (d, q heads of the launch's head group, tokens): head h's g rows start at coordinate h*g
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.g) * heads,
                                    static_cast<cuuint64_t>(p.n_q)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(p.q_tok_stride) * 2};
        const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(p.g), static_cast<cuuint32_t>(BM / p.g)};
        if (!make_tmap_bf16(&tq, p.q, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    {
        // (d, keys, kv heads of the group)
        const int64_t hs = heads > 1 ? p.kv_head_stride : static_cast<int64_t>(p.n_k) * p.kv_row_stride;
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.n_k), static_cast<cuuint64_t>(heads)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.kv_row_stride) * 2, static_cast<cuuint64_t>(hs) * 2};
        const cuuint32_t box[3] = {64, BN, 1};
        if (!make_tmap_bf16(&tk, p.k, 3, dims, strides, box)) return cudaErrorInvalidValue;
        if (!make_tmap_bf16(&tv, p.v, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    prefill_tc1_kernel<D><<<dim3(grid, heads), NUM_THREADS, Smem<D>::ALLOC, stream>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

}  // namespace

#ifdef HI_TRACE
extern "C" int hi_debug_prefill_trace1(void* dst, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_hi_trace1, bytes));
}
#endif

cudaError_t launch_prefill_tc1(const PrefillParams& p, int d, cudaStream_t stream) {
    if (d == 64) return launch_tc1<64>(p, stream);
    if (d == 128) return launch_tc1<128>(p, stream);
    return cudaErrorInvalidValue;
}

}  // namespace hi
