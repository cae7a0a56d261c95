// k_prefill_tcp.cu -- sm_100a prefill attention over one KV segment with P staged in SHARED memory, so that
// S(j+1) = Q K(j+1)^T can run while the softmax of S(j) is still computing.
//
// Same contract as k_prefill_tc.cu (Eq. 9; one launch folds one contiguous key
// segment into the running (O, m, l) state): same CTA (two 128-row GQA-packed Q tiles), same TMEM map
// (tile t: S at columns 256t .. +128, O at 256t + 128 .. +D), same masks, band, head maps, state and epilogue.
// What differs is where P goes.  In k_prefill_tc.cu P(j) overwrites S(j) in TMEM and the PV MMA reads it from
// there, so S(j+1) of a tile can only be issued once PV(j) has consumed P(j): per tile the chain is
// softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1), and the tensor pipe idles while both tiles' softmaxes run
// (profiles/trace_tc_r01.txt: 3600-cycle period per KV tile against 2048 cycles of MMAs).  Here the softmax
// releases the S columns as soon as S(j) is in registers (s_cons), the MMA warp issues S(j+1) right away, and
// the softmax writes P(j) as bf16 into a per-tile shared-memory tile laid out exactly like a TMA SWIZZLE_128B
// Q tile, from which PV(j) reads it as a K-major A operand (SS MMA).  The per-tile chain becomes
// softmax(j) -> softmax(j+1) with the MMAs in its shadow; the price is 64 KiB of shared memory for P (K and V
// share one 3-slot ring in consumption order) and an SS instead of a TS PV MMA.
//
// Pipeline: one thread issues every MMA, event-driven: a tile's S(j+1) as soon as its softmax has read S(j) and
// K(j+1) landed, its PV(j) as soon as P(j) is in shared memory and V(j) landed.
// Barriers: kv_full/kv_empty (3-slot K/V ring), per tile s_full (S(j) in TMEM),
// s_cons (S(j) read by the softmax), p_full (P(j) in shared memory, O corrected), pv_done (PV(j) complete:
// the P tile may be rewritten and O may be rescaled).
#include "../hi_kernels.cuh"
#include "../tc_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

namespace hi {
namespace {

using namespace ptx;

constexpr int BM = 128;            // query rows per tile (TMEM lanes)
constexpr int BN = 128;            // keys per KV tile
constexpr int KV_SLOTS = 3;        // one ring of K and V tiles in consumption order K(0), [K(i+1), V(i)] ...
constexpr int SOFTMAX_WARPS = 8;
constexpr int WARP_TMA = 8, WARP_MMA = 9;
constexpr int NUM_THREADS = 32 * 12;
constexpr int REG_SOFTMAX = 208, REG_PRODUCER = 88;   // setmaxnreg: 256 x +40 == 128 x -80
constexpr float RESCALE_THRESHOLD = 8.0f;

struct __align__(8) Barriers {
    uint64_t q_full;
    uint64_t kv_full[KV_SLOTS], kv_empty[KV_SLOTS];
    uint64_t s_full[2], s_cons[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
};

template <int D>
struct Smem {
    static constexpr int BOX = BM * 128;                 // [128 rows][64 bf16] SWIZZLE_128B = 16 KiB
    static constexpr int Q_OFF = 0;                      // 2 tiles x D/64 boxes
    static constexpr int P_OFF = Q_OFF + 2 * (D / 64) * BOX;   // 2 tiles x BN/64 boxes
    static constexpr int KV_OFF = P_OFF + 2 * (BN / 64) * BOX;  // KV_SLOTS x D/64 boxes
    static constexpr int BAR_OFF = KV_OFF + KV_SLOTS * (D / 64) * BOX;
    static constexpr int BYTES = BAR_OFF + static_cast<int>(sizeof(Barriers));
    static constexpr int ALLOC = BYTES + 1024;
};
static_assert(Smem<128>::ALLOC <= 232448, "shared memory per CTA");

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    prefill_tcp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const PrefillParams p) {
    using L = Smem<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bars = reinterpret_cast<Barriers*>(smem + L::BAR_OFF);
    const uint32_t sbase = smem_addr(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = p.g;
    const int n_rows = p.n_q * g;
    const int row0 = abs(p.row_rev - static_cast<int>(blockIdx.x)) * (2 * BM);   // LPT order for causal segments
    const int hh = blockIdx.y;
    const int hq = p.head_q[hh], hk = p.head_kv[hh];
    float* const o_acc = p.o_acc + static_cast<int64_t>(hh) * p.state_rows * D;
    float* const m_acc = p.m_acc + static_cast<int64_t>(hh) * p.state_rows;
    float* const l_acc = p.l_acc + static_cast<int64_t>(hh) * p.state_rows;
    const bool first = p.flags & PF_FIRST, last = p.flags & PF_LAST, causal = p.flags & PF_CAUSAL;
    const int n_tiles = (row0 + BM < n_rows) ? 2 : 1;

    const bool band = p.win > 0;
    int kt_lo = 0;
    if (band) {
        const int64_t c_lo = p.q_pos0 + row0 / g - p.win + 1 - p.k_pos0;
        kt_lo = c_lo > 0 ? static_cast<int>((c_lo < p.n_k ? c_lo : static_cast<int64_t>(p.n_k)) / BN) : 0;
    }
    const int kb = kt_lo * BN;
    auto kt_count = [&](int tt) {
        const int r0 = row0 + tt * BM;
        const int t_hi = min(p.n_q - 1, (r0 + BM - 1) / g);
        int64_t e = p.n_k;
        if (causal) {
            const int64_t lim = p.q_pos0 + t_hi - p.k_pos0 + 1;
            e = lim < e ? lim : e;
        }
        e = e > 0 ? e : 0;
        return max(0, static_cast<int>((e + BN - 1) / BN) - kt_lo);
    };
    const int n_kt0 = kt_count(0);
    const int n_kt1 = n_tiles == 2 ? kt_count(1) : 0;
    const int n_kt = max(n_kt0, n_kt1);

    const uint32_t bar_q = smem_addr(&bars->q_full);
    auto bar_kvf = [&](int s) { return smem_addr(&bars->kv_full[s]); };
    auto bar_kve = [&](int s) { return smem_addr(&bars->kv_empty[s]); };
    // ring item of K(i) and of V(i): K(0), then K(i+1) before V(i); an item waits for the one 3 places earlier
    auto item_k = [&](int i) { return i == 0 ? 0 : 2 * i - 1; };
    auto item_v = [&](int i) { return i + 1 < n_kt ? 2 * i + 2 : 2 * i + 1; };
    auto bar_s = [&](int t) { return smem_addr(&bars->s_full[t]); };
    auto bar_sc = [&](int t) { return smem_addr(&bars->s_cons[t]); };
    auto bar_p = [&](int t) { return smem_addr(&bars->p_full[t]); };
    auto bar_pv = [&](int t) { return smem_addr(&bars->pv_done[t]); };

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < KV_SLOTS; ++s) {
            mbar_init(bar_kvf(s), 1);
            mbar_init(bar_kve(s), 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(bar_s(t), 1);
            mbar_init(bar_sc(t), 128);
            mbar_init(bar_p(t), 128);
            mbar_init(bar_pv(t), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&bars->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp >= SOFTMAX_WARPS) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_PRODUCER));
        if (warp == WARP_TMA && lane == 0 && n_kt > 0) {
            // ============================ TMA producer: Q, then K(0), [K(i+1), V(i)] ...
            mbar_expect_tx(bar_q, n_tiles * (D / 64) * L::BOX);
            for (int tt = 0; tt < n_tiles; ++tt)
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sbase + L::Q_OFF + (tt * (D / 64) + c) * L::BOX, &tm_q, bar_q, c * 64, hq * g,
                                (row0 + tt * BM) / g);
            auto load = [&](int item, const CUtensorMap* map, int i) {
                const int s = item % KV_SLOTS;
                if (item >= KV_SLOTS) mbar_wait(bar_kve(s), ((item / KV_SLOTS) - 1) & 1);
                mbar_expect_tx(bar_kvf(s), (D / 64) * L::BOX);
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sbase + L::KV_OFF + (s * (D / 64) + c) * L::BOX, map, bar_kvf(s), c * 64, kb + i * BN, hk);
            };
            load(item_k(0), &tm_k, 0);
            for (int i = 0; i < n_kt; ++i) {
                if (i + 1 < n_kt) load(item_k(i + 1), &tm_k, i + 1);
                load(item_v(i), &tm_v, i);
            }
        } else if (warp == WARP_MMA && lane == 0 && n_kt > 0) {
            // ============================ MMA issuer
            constexpr uint32_t ID_S = idesc_bf16(BM, BN, false);
            constexpr uint32_t ID_O = idesc_bf16(BM, D, true);
            const int nk_t[2] = {n_kt0, n_kt1};
            const uint64_t dq0 = sdesc(sbase + L::Q_OFF, 16, 1024);
            const uint64_t dk0 = sdesc(sbase + L::KV_OFF, 16, 1024);
            const uint64_t dp0 = sdesc(sbase + L::P_OFF, 16, 1024);
            const uint64_t dv0 = sdesc(sbase + L::KV_OFF, L::BOX, 1024);
            auto issue_s = [&](int tt, int i) {   // S_tt(i) = Q_tt K(i)^T -> TMEM columns 256 tt
                const uint64_t a0 = dq0 + ((tt * (D / 64) * L::BOX) >> 4);
                const uint64_t b0 = dk0 + (((item_k(i) % KV_SLOTS) * (D / 64) * L::BOX) >> 4);
#pragma unroll 1   // rolled: the issuer runs on 88 registers, and one MMA takes 64 cycles to execute
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = ((ks >> 2) * L::BOX + (ks & 3) * 32) >> 4;
                    umma_bf16(tmem + tt * 256, a0 + off, b0 + off, ID_S, ks > 0);
                }
                umma_commit(bar_s(tt));
            };
            auto issue_pv = [&](int tt, int j) {  // O_tt += P_tt(j) V(j): A = P (shared, K-major), B = V (MN-major)
                const uint64_t a0 = dp0 + ((tt * (BN / 64) * L::BOX) >> 4);
                const uint64_t v0 = dv0 + (((item_v(j) % KV_SLOTS) * (D / 64) * L::BOX) >> 4);
#pragma unroll 1
                for (int kk = 0; kk < BN / 16; ++kk) {
                    const uint32_t aoff = ((kk >> 2) * L::BOX + (kk & 3) * 32) >> 4;
                    umma_bf16(tmem + tt * 256 + 128, a0 + aoff, v0 + ((kk * 16 * 128) >> 4), ID_O,
                              (j > 0 || kk > 0 || !first) ? 1u : 0u);
                }
                umma_commit(bar_pv(tt));
            };
            mbar_wait(bar_q, 0);
            // Event-driven issue: each tile's next S and next PV go to the tensor pipe as soon as their inputs are
            // ready, whatever the other tile is doing (a fixed S_A S_B PV_A PV_B order made each tile's S wait on
            // the other tile's P).  A ring slot is released when the last tile that reads it has issued its MMA;
            // the tiles cannot drift more than a few KV tiles apart (the ring holds 3), so 4 counters suffice.
            int ns[2] = {0, 0}, npv[2] = {0, 0};
            uint32_t kmask = 0, vmask = 0;   // bit (i & 3): one of two reading tiles has issued on K(i) / V(i)
            // true when this issue is the last read of the item (then its ring slot is released)
            auto last_user = [&](uint32_t& mask, int i) {
                if ((i < nk_t[0]) != (i < nk_t[1])) return true;   // only one tile reads it
                const uint32_t bit = 1u << (i & 3);
                const bool second = mask & bit;
                mask ^= bit;
                return second;
            };
            while (npv[0] < nk_t[0] || npv[1] < nk_t[1]) {
#pragma unroll
                for (int tt = 0; tt < 2; ++tt) {
                    const int j = ns[tt];
                    if (j < nk_t[tt] && (j == 0 || mbar_test(bar_sc(tt), (j - 1) & 1))) {   // S(j-1) read
                        const int it = item_k(j);
                        if (mbar_test(bar_kvf(it % KV_SLOTS), (it / KV_SLOTS) & 1)) {
                            tc_fence_after();
                            issue_s(tt, j);
                            ns[tt] = j + 1;
                            if (last_user(kmask, j)) umma_commit(bar_kve(it % KV_SLOTS));
                        }
                    }
                    const int jp = npv[tt];
                    if (jp < ns[tt] && mbar_test(bar_p(tt), jp & 1)) {   // P(jp) in shared memory, O corrected
                        const int iv = item_v(jp);
                        if (mbar_test(bar_kvf(iv % KV_SLOTS), (iv / KV_SLOTS) & 1)) {
                            tc_fence_after();
                            issue_pv(tt, jp);
                            npv[tt] = jp + 1;
                            if (last_user(vmask, jp)) umma_commit(bar_kve(iv % KV_SLOTS));
                        }
                    }
                }
            }
        }
    } else {
        // ====================== softmax / correction / epilogue: warps 0-3 tile 0, 4-7 tile 1
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REG_SOFTMAX));
        const int tt = warp >> 2;
        const int wq = warp & 3;
        const int r = wq * 32 + lane;               // row within the tile == TMEM lane
        const int rg = row0 + tt * BM + r;          // packed row t*g + j
        const bool row_valid = rg < n_rows;
        const int t = row_valid ? rg / g : 0;
        const int64_t qpos = p.q_pos0 + t;
        const int nkt = tt == 0 ? n_kt0 : n_kt1;
        const int t_lo = (row0 + tt * BM) / g;
        const int t_hi_tile = min(p.n_q - 1, (row0 + tt * BM + BM - 1) / g);
        const uint32_t t_s = tmem + tt * 256 + (static_cast<uint32_t>(wq * 32) << 16);
        const uint32_t t_o = t_s + 128;
        const uint32_t sp_row = sbase + L::P_OFF + tt * (BN / 64) * L::BOX + r * 128;   // this row of the P tile
        const float sc = p.scale_log2;
        float m_run = -CUDART_INF_F, l_run = 0.f;
        if (tt < n_tiles) {
            if (!first) {
                m_run = row_valid ? m_acc[rg] : -CUDART_INF_F;
                l_run = row_valid ? l_acc[rg] : 0.f;
                if (nkt > 0) {
#pragma unroll
                    for (int cb = 0; cb < D / 32; ++cb) {
                        uint32_t v[32];
                        const float4* src = reinterpret_cast<const float4*>(o_acc + static_cast<int64_t>(row_valid ? rg : 0) * D + cb * 32);
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
                mbar_wait(bar_s(tt), j & 1);
                tc_fence_after();
                uint32_t x[BN];
#pragma unroll
                for (int cb = 0; cb < BN / 32; ++cb) tmem_ld32(t_s + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(bar_sc(tt));   // the S columns may take S(j+1)
                const int key0 = kb + j * BN;
                const bool need_mask = (key0 + BN > p.n_k) || (causal && p.k_pos0 + key0 + BN - 1 > p.q_pos0 + t_lo);
                if (need_mask) {
                    const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                    const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                    for (int i = 0; i < BN; ++i)
                        if (key0 + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
                }
                if (band && p.k_pos0 + key0 <= p.q_pos0 + t_hi_tile - p.win) {
                    const int64_t lo = qpos - p.win - p.k_pos0;
#pragma unroll
                    for (int i = 0; i < BN; ++i)
                        if (key0 + i <= lo) x[i] = __float_as_uint(-CUDART_INF_F);
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
                const bool grow = (mx != -CUDART_INF_F) && (m_run == -CUDART_INF_F || mxs > m_run + RESCALE_THRESHOLD);
                const float mref = grow ? mxs : m_run;
                const float alpha = grow ? ((m_run == -CUDART_INF_F) ? 0.f : ex2(m_run - mxs)) : 1.f;
                bool pv_prev_done = j == 0;
                if ((!first || j > 0) && __any_sync(0xffffffffu, grow)) {   // O correction: PV(j-1) must be done
                    if (j > 0) {
                        mbar_wait(bar_pv(tt), (j - 1) & 1);
                        tc_fence_after();
                        pv_prev_done = true;
                    }
#pragma unroll
                    for (int cb = 0; cb < D / 32; ++cb) {
                        uint32_t v[32];
                        tmem_ld32(t_o + cb * 32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(t_o + cb * 32, v);
                    }
                    tmem_wait_st();
                }
                // p = 2^(x*scale - m), packed to bf16 pairs in place, row sum in fp32
                const float nm = (mref == -CUDART_INF_F) ? 0.f : -mref;
                f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                const f2 sc2{sc, sc}, nm2{nm, nm};
#ifdef HI_FAKE_SOFTMAX   // timing experiment only: the MMA / shared-memory ceiling of this pipeline without exps
                if (true) {
                } else
#endif
#pragma unroll
                for (int i = 0; i < BN; i += 2) {
                    const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                    const f2 pp{ex2(a.x), ex2(a.y)};
                    acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                    x[i / 2] = pack_bf16(pp.x, pp.y);
                }
                if (!pv_prev_done) mbar_wait(bar_pv(tt), (j - 1) & 1);   // PV(j-1) has read the P tile
                // P(j) -> shared memory, SWIZZLE_128B K-major (16-byte chunk c of the row at chunk c ^ (row % 8))
#pragma unroll
                for (int c = 0; c < BN / 8; ++c) {
                    const uint32_t addr = sp_row + (c >> 3) * L::BOX + (((c & 7) ^ (r & 7)) << 4);
                    st_shared_v4(addr, x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
                }
                fence_proxy_async_smem();   // generic-proxy stores visible to the tensor core (async proxy)
                tc_fence_before();
                mbar_arrive(bar_p(tt));
                const f2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
                l_run = l_run * alpha + ((s01.x + s01.y) + (s23.x + s23.y));
                m_run = mref;
            }
            // ---- epilogue (as k_prefill_tc.cu) ----
            if (nkt > 0) {
                mbar_wait(bar_pv(tt), (nkt - 1) & 1);   // the last PV
                tc_fence_after();
            }
            if (last) {
                const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
                __nv_bfloat16* dst = p.out + static_cast<int64_t>(t) * p.o_tok_stride + (hq * g + rg % g) * D;
#pragma unroll
                for (int cb = 0; cb < D / 32; ++cb) {
                    uint32_t v[32];
                    if (nkt > 0) {
                        tmem_ld32(t_o + cb * 32, v);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            v[i] = (row_valid && !first) ? __float_as_uint(o_acc[static_cast<int64_t>(rg) * D + cb * 32 + i]) : 0u;
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
                        float4* dst = reinterpret_cast<float4*>(o_acc + static_cast<int64_t>(rg) * D + cb * 32);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                 __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                    }
                }
                if (row_valid) {
                    m_acc[rg] = m_run;
                    l_acc[rg] = l_run;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == WARP_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

template <int D>
cudaError_t launch_tcp(const PrefillParams& p, cudaStream_t stream) {
    const int n_rows = p.n_q * p.g;
    const int grid = (n_rows + 2 * BM - 1) / (2 * BM);
    const int heads = p.n_heads > 0 ? p.n_heads : 1;
    if (grid == 0) return cudaSuccess;
    if (heads > MAX_LAUNCH_HEADS || p.q_span < 1 || p.kv_span < 1) return cudaErrorInvalidValue;
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = set_smem_attr_once(prefill_tcp_kernel<D>, Smem<D>::ALLOC, configured); e != cudaSuccess) return e;
    CUtensorMap tq, tk, tv;
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.g) * p.q_span,
                                    static_cast<cuuint64_t>(p.n_q)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(p.q_tok_stride) * 2};
        const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(p.g), static_cast<cuuint32_t>(BM / p.g)};
        if (!make_tmap_bf16(&tq, p.q, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    {
        const int64_t hs = p.kv_span > 1 ? p.kv_head_stride : static_cast<int64_t>(p.n_k) * p.kv_row_stride;
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.n_k), static_cast<cuuint64_t>(p.kv_span)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.kv_row_stride) * 2, static_cast<cuuint64_t>(hs) * 2};
        const cuuint32_t box[3] = {64, BN, 1};
        if (!make_tmap_bf16(&tk, p.k, 3, dims, strides, box)) return cudaErrorInvalidValue;
        if (!make_tmap_bf16(&tv, p.v, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    PrefillParams pl = p;
    pl.row_rev = (p.flags & PF_CAUSAL) ? grid - 1 : 0;
    prefill_tcp_kernel<D><<<dim3(grid, heads), NUM_THREADS, Smem<D>::ALLOC, stream>>>(tq, tk, tv, pl);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prefill_tcp(const PrefillParams& p, int d, cudaStream_t stream) {
    if (d == 64) return launch_tcp<64>(p, stream);
    if (d == 128) return launch_tcp<128>(p, stream);
    return cudaErrorInvalidValue;
}

}  // namespace hi
