// k_decode.cu -- decode attention: split-K partials over a staged history block + LSE combine.
//
// for each q head j of group h,
//   o = softmax(q . K[0..s]^T / sqrt(d)) V[0..s]         (Eq. 9; the new key included, R3)
// Decode is bandwidth-bound (AI ~ 1, App. C), so this runs on CUDA cores: 128-bit
// coalesced loads (a key row is d/8 lanes x 16 B), fp32 math, warp-shuffle dot reductions,
// online max/sum per lane, then a shared-memory merge per CTA.  Each CTA writes one partial
// record (m, l, o[d]) per q head; decode_combine merges all records of a head plus the new
// token's key by log-sum-exp and writes bf16.
#include "hi_kernels.cuh"

#include <cuda_bf16.h>
#include <math_constants.h>

namespace hi {
namespace {


__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}


// ---- PTX helpers: mbarrier + bulk async copy (TMA engine, non-tensor form) --------------------
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t it = 0;; ++it) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
        if (done) return;
        if (it > (1u << 31)) __trap();
    }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

constexpr int DM_CONSUMERS = 4;                       // consumer warps, 16 keys each per stage
constexpr int DM_THREADS = (DM_CONSUMERS + 1) * 32;   // + 1 TMA producer warp
constexpr int DM_CHUNK = 16 * DM_CONSUMERS;           // keys per pipeline stage
constexpr int DM_BOX = DM_CHUNK * 128;                // one [64 keys][64 bf16] SW128 box = 8 KiB
constexpr int DM_STAGES = 6;
constexpr float DM_RESCALE = 8.0f;                    // lazy O rescale threshold (log2 units)

template <int D>
constexpr int dm_smem_bytes() { return DM_STAGES * 2 * (D / 64) * DM_BOX + 2 * DM_STAGES * 8 + 1024 + 1024; }

// Fused combine (DecodePartialParams::combine): called by the 4 consumer warps of every CTA after its record is
// written.  The CTA that completes head blockIdx.y's last split merges all of that head's records with the new
// key (the token attends itself, reading R3) -- the same log-sum-exp as decode_combine_kernel -- and, with
// `append`, stores the new key/value row for the next step.
template <int D, int G>
__device__ __forceinline__ void combine_tail(const DecodePartialParams& p) {
    constexpr int NT = DM_CONSUMERS * 32;
    __shared__ int s_last;
    __shared__ float s_x[G];
    const int y = blockIdx.y, h = p.head[y];
    __threadfence();   // this CTA's record is visible device-wide before the counter says so
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (threadIdx.x == 0) s_last = atomicAdd(&p.counters[h], 1u) == gridDim.x - 1;
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (!s_last) return;
    __threadfence();   // acquire: every other CTA's record of head h
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const __nv_bfloat16* qg = p.q + h * p.q_head_stride;
    const __nv_bfloat16* kn = p.k_new + static_cast<int64_t>(h) * D;
    const __nv_bfloat16* vn = p.v_new + static_cast<int64_t>(h) * D;
    for (int j = warp; j < G; j += DM_CONSUMERS) {   // new key's score per q head (log2 domain)
        float prod = 0.f;
        for (int c = lane; c < D; c += 32) prod += __bfloat162float(qg[j * D + c]) * __bfloat162float(kn[c]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, off);
        if (lane == 0) s_x[j] = prod * p.scale_log2;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    const float* recs = p.parts + h * p.parts_head_stride;
    const int n = p.parts_total;
    for (int idx = threadIdx.x; idx < G * D; idx += NT) {
        const int j = idx / D, c = idx % D;
        const float* rj = recs + j * (D + 4);
        float M = s_x[j];
        for (int i = 0; i < n; ++i) M = fmaxf(M, __ldcg(rj + static_cast<int64_t>(i) * G * (D + 4)));
        const float a0 = fast_exp2(s_x[j] - M);
        float L = a0, O = a0 * __bfloat162float(vn[c]);
        for (int i = 0; i < n; ++i) {
            const float* r = rj + static_cast<int64_t>(i) * G * (D + 4);
            const float mi = __ldcg(r);
            const float a = (mi == -CUDART_INF_F) ? 0.f : fast_exp2(mi - M);
            L += a * __ldcg(r + 1);
            O += a * __ldcg(r + 4 + c);
        }
        p.out[(static_cast<int64_t>(h) * G + j) * D + c] = __float2bfloat16_rn(O / L);
    }
    if (p.append) {   // row n_k of this head's cache: outside every range this launch read
        __nv_bfloat16* kd = const_cast<__nv_bfloat16*>(p.k) + p.kvc[y] * p.kv_head_stride + static_cast<int64_t>(p.n_k) * D;
        __nv_bfloat16* vd = const_cast<__nv_bfloat16*>(p.v) + p.kvc[y] * p.kv_head_stride + static_cast<int64_t>(p.n_k) * D;
        for (int c = threadIdx.x; c < D; c += NT) {
            kd[c] = kn[c];
            vd[c] = vn[c];
        }
    }
    if (threadIdx.x == 0) p.counters[h] = 0u;   // ready for the next launch (stream-ordered)
}

// One CTA = keys [blockIdx.x*split_len, +split_len) of the block.  A single producer thread streams
// the CTA's K and V rows with 2-D TMA (SWIZZLE_128B boxes of 64 keys x 64 dims) into a 6-stage
// shared-memory ring -- up to 192 KiB in flight per SM, which is what HBM latency needs.  Each of the
// 4 consumer warps takes 16 keys of a stage and runs them through the tensor cores with warp-level
// mma.sync m16n8k16: S = Q K^T with the g query rows zero-padded to M = 16 (Q fragments in registers),
// online softmax on the fp32 accumulators (log2 domain, lazy rescale), O += P V with P re-packed from
// the S accumulators as the A operand (no shared-memory round trip).  On CUDA cores the same kernel
// was issue-bound at ~50% of HBM bandwidth (profiles/ncu_decode_r01.txt); with the contraction on the
// tensor pipe a key costs ~5 warp instructions instead of ~55.
template <int D, int G>
__global__ void __launch_bounds__(DM_THREADS, 1)
    decode_partial_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                          const DecodePartialParams p) {
    static_assert(G <= 8, "query group must fit the 8 live rows of an m16 tile");
    constexpr int NB = D / 64;                         // 64-dim boxes per key row
    constexpr int STAGE = 2 * NB * DM_BOX;
    extern __shared__ uint8_t dm_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DM_STAGES * STAGE);
    const uint32_t sbase = smem_u32(smem);
    auto bar_full = [&](int s) { return smem_u32(&bars[s]); };
    auto bar_empty = [&](int s) { return smem_u32(&bars[DM_STAGES + s]); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int k_begin = blockIdx.x * p.split_len;
    const int k_end = min(p.n_k, k_begin + p.split_len);
    const int n_chunks = (k_end - k_begin + DM_CHUNK - 1) / DM_CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < DM_STAGES; ++s) {
            mbar_init(bar_full(s), 1);
            mbar_init(bar_empty(s), DM_CONSUMERS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == DM_CONSUMERS) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % DM_STAGES;
                if (i >= DM_STAGES) mbar_wait(bar_empty(s), ((i / DM_STAGES) - 1) & 1);
                const int k0 = k_begin + i * DM_CHUNK;
                mbar_expect_tx(bar_full(s), STAGE);  // OOB rows of the last chunk are zero-filled, still counted
#pragma unroll
                for (int c = 0; c < NB; ++c) {
                    tma_load_3d(sbase + s * STAGE + c * DM_BOX, &tm_k, bar_full(s), c * 64, k0, p.kvc[blockIdx.y]);
                    tma_load_3d(sbase + s * STAGE + (NB + c) * DM_BOX, &tm_v, bar_full(s), c * 64, k0, p.kvc[blockIdx.y]);
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int gid = lane >> 2, tq = lane & 3;
    const bool row_live = gid < G;
    const __nv_bfloat16* qg = p.q + p.head[blockIdx.y] * p.q_head_stride;
    // Q fragments (A operand, rows = q heads of the group, zero-padded to 16), all of D
    uint32_t qa[D / 16][2];  // {a0a1 (row gid, k 0-7 of the step), a4a5 (row gid, k 8-15)}; rows gid+8 are 0
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
        qa[ks][0] = row_live ? *reinterpret_cast<const uint32_t*>(qg + gid * D + ks * 16 + tq * 2) : 0u;
        qa[ks][1] = row_live ? *reinterpret_cast<const uint32_t*>(qg + gid * D + ks * 16 + 8 + tq * 2) : 0u;
    }
    float o[D / 8][4];
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m_run = -CUDART_INF_F, l_run = 0.f;  // row gid (l: this thread's partial sum)
    const float sc = p.scale_log2;
    const int kb = warp * 16;                 // this warp's 16 keys within a stage
    for (int i = 0; i < n_chunks; ++i) {
        const int s = i % DM_STAGES;
        mbar_wait(bar_full(s), (i / DM_STAGES) & 1);
        const uint32_t sk = sbase + s * STAGE;
        const uint32_t sv = sk + NB * DM_BOX;
        const int nvalid = k_end - (k_begin + i * DM_CHUNK) - kb;  // keys of this warp's 16 that exist
        if (nvalid > 0) {
            // S = Q K^T over 16 keys (two n-tiles of 8)
            float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const int r = kb + (lane & 7) + ((lane >> 4) << 3);
                const int c = ((ks & 3) << 1) + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sk + (ks >> 2) * DM_BOX + r * 128 + ((c ^ (r & 7)) << 4), b0, b1, b2, b3);
                mma_bf16(sacc[0], qa[ks][0], 0u, qa[ks][1], 0u, b0, b1);
                mma_bf16(sacc[1], qa[ks][0], 0u, qa[ks][1], 0u, b2, b3);
            }
            // online softmax for row gid (elements 0,1 of each n-tile; 2,3 are the padded rows)
            float x[4];
            x[0] = sacc[0][0] * sc; x[1] = sacc[0][1] * sc; x[2] = sacc[1][0] * sc; x[3] = sacc[1][1] * sc;
            if (nvalid < 16) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if ((e >> 1) * 8 + tq * 2 + (e & 1) >= nvalid) x[e] = -CUDART_INF_F;
            }
            float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const bool grow = m_run == -CUDART_INF_F || mx > m_run + DM_RESCALE;
            if (__any_sync(0xffffffffu, grow)) {
                const float m_new = grow ? mx : m_run;
                const float alpha = (m_run == -CUDART_INF_F) ? 0.f : fast_exp2(m_run - m_new);
                l_run *= alpha;
#pragma unroll
                for (int nt = 0; nt < D / 8; ++nt) { o[nt][0] *= alpha; o[nt][1] *= alpha; }
                m_run = m_new;
            }
            float pr[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                pr[e] = fast_exp2(x[e] - m_run);
                l_run += pr[e];
            }
            const uint32_t pa0 = pack_bf16(pr[0], pr[1]);  // row gid, keys tq*2..   (k 0-7)
            const uint32_t pa2 = pack_bf16(pr[2], pr[3]);  // row gid, keys 8+tq*2.. (k 8-15)
            // O += P V (V rows = keys: transposed ldmatrix gives the k-major B fragments)
#pragma unroll
            for (int dn = 0; dn < D / 16; ++dn) {
                const int r = kb + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = dn * 2 + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(sv + (c >> 3) * DM_BOX + r * 128 + (((c & 7) ^ (r & 7)) << 4), b0, b1, b2, b3);
                mma_bf16(o[2 * dn], pa0, 0u, pa2, 0u, b0, b1);
                mma_bf16(o[2 * dn + 1], pa0, 0u, pa2, 0u, b2, b3);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty(s));
    }
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);

    // merge the consumer warps through shared memory (the ring is free: every chunk was consumed)
    float* sm_m = reinterpret_cast<float*>(smem);            // [W][G]
    float* sm_l = sm_m + DM_CONSUMERS * G;                   // [W][G]
    float* sm_o = sm_l + DM_CONSUMERS * G;                   // [W][G][D]
    asm volatile("bar.sync 1, %0;" ::"n"(DM_CONSUMERS * 32) : "memory");
    if (row_live) {
        if (tq == 0) { sm_m[warp * G + gid] = m_run; sm_l[warp * G + gid] = l_run; }
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
            sm_o[(warp * G + gid) * D + nt * 8 + tq * 2] = o[nt][0];
            sm_o[(warp * G + gid) * D + nt * 8 + tq * 2 + 1] = o[nt][1];
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(DM_CONSUMERS * 32) : "memory");
    float* rec = p.parts + p.head[blockIdx.y] * p.parts_head_stride + static_cast<int64_t>(blockIdx.x) * G * (D + 4);
    for (int idx = threadIdx.x; idx < G * D; idx += DM_CONSUMERS * 32) {
        const int j = idx / D, c = idx % D;
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < DM_CONSUMERS; ++w) mx = fmaxf(mx, sm_m[w * G + j]);
        float lsum = 0.f, osum = 0.f;
#pragma unroll
        for (int w = 0; w < DM_CONSUMERS; ++w) {
            const float mw = sm_m[w * G + j];
            const float a = (mw == -CUDART_INF_F) ? 0.f : fast_exp2(mw - mx);
            lsum += a * sm_l[w * G + j];
            osum += a * sm_o[(w * G + j) * D + c];
        }
        float* r = rec + j * (D + 4);
        r[4 + c] = osum;
        if (c == 0) { r[0] = mx; r[1] = lsum; }
    }
    if (p.combine) combine_tail<D, G>(p);
}

// One CTA (8 warps) per local q head: merge the n_parts records of its kv head with the new key.
// Pass 1: block max over the record maxima (and the new key's score); pass 2: each warp accumulates
// a strided subset of records (lane = D/32 consecutive columns, float4/float2 loads, 4 records in
// flight), then the warps are merged in shared memory.
constexpr int CB_WARPS = 8;

template <int D>
__global__ void __launch_bounds__(CB_WARPS * 32) decode_combine_kernel(const DecodeCombineParams p) {
    constexpr int CPL = D / 32;  // columns per lane
    const int jq = blockIdx.x;   // local q head
    const int h = jq / p.g, j = jq % p.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ float s_red[CB_WARPS];
    __shared__ float s_x;
    __shared__ float s_o[CB_WARPS][D];
    __shared__ float s_l[CB_WARPS];
    // score of the new key (the token attends itself, reading R3): warp 0
    if (warp == 0) {
        float prod = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int col = lane * CPL + c;
            prod += __bfloat162float(p.q[jq * D + col]) * __bfloat162float(p.k_new[h * D + col]);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, off);
        if (lane == 0) s_x = prod * p.scale_log2;
    }
    const int n_parts = p.n_parts[h];
    const float* recs = p.parts + (static_cast<int64_t>(h) * p.max_parts * p.g + j) * (D + 4);
    const int64_t rstride = static_cast<int64_t>(p.g) * (D + 4);
    float mx = -CUDART_INF_F;
    for (int i = threadIdx.x; i < n_parts; i += CB_WARPS * 32) mx = fmaxf(mx, recs[i * rstride]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    float M = s_x;
#pragma unroll
    for (int w = 0; w < CB_WARPS; ++w) M = fmaxf(M, s_red[w]);
    float o[CPL], lsum = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) o[c] = 0.f;
#pragma unroll 4
    for (int i = warp; i < n_parts; i += CB_WARPS) {
        const float* r = recs + i * rstride;
        const float mi = r[0];
        const float a = (mi == -CUDART_INF_F) ? 0.f : fast_exp2(mi - M);
        lsum += a * r[1];
        if constexpr (CPL == 4) {
            const float4 v = *reinterpret_cast<const float4*>(r + 4 + lane * 4);
            o[0] += a * v.x; o[1] += a * v.y; o[2] += a * v.z; o[3] += a * v.w;
        } else {
            const float2 v = *reinterpret_cast<const float2*>(r + 4 + lane * 2);
            o[0] += a * v.x; o[1] += a * v.y;
        }
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) s_o[warp][lane * CPL + c] = o[c];
    if (lane == 0) s_l[warp] = lsum;
    __syncthreads();
    if (threadIdx.x < D) {
        const int c = threadIdx.x;
        const float a0 = fast_exp2(s_x - M);
        float L = a0, O = a0 * __bfloat162float(p.v_new[h * D + c]);
#pragma unroll
        for (int w = 0; w < CB_WARPS; ++w) {
            L += s_l[w];
            O += s_o[w][c];
        }
        p.out[jq * D + c] = __float2bfloat16_rn(O / L);
    }
}

template <int D, int G>
cudaError_t launch_partial_dg(const DecodePartialParams& p, int n_splits, int n_heads, cudaStream_t s) {
    constexpr int smem = dm_smem_bytes<D>();
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = set_smem_attr_once(decode_partial_kernel<D, G>, smem, configured); e != cudaSuccess) return e;
    CUtensorMap tk, tv;
    const int64_t hs = p.kv_span > 1 ? p.kv_head_stride : static_cast<int64_t>(p.n_k) * D;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.n_k), static_cast<cuuint64_t>(p.kv_span)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(hs) * 2};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(DM_CHUNK), 1};
    if (!make_tmap_bf16(&tk, p.k, 3, dims, strides, box) || !make_tmap_bf16(&tv, p.v, 3, dims, strides, box))
        return cudaErrorInvalidValue;
    decode_partial_kernel<D, G><<<dim3(n_splits, n_heads), DM_THREADS, smem, s>>>(tk, tv, p);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_partial_d(const DecodePartialParams& p, int g, int n_splits, int n_heads, cudaStream_t s) {
    switch (g) {
        case 1: return launch_partial_dg<D, 1>(p, n_splits, n_heads, s);
        case 2: return launch_partial_dg<D, 2>(p, n_splits, n_heads, s);
        case 4: return launch_partial_dg<D, 4>(p, n_splits, n_heads, s);
        case 8: return launch_partial_dg<D, 8>(p, n_splits, n_heads, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_decode_partial(const DecodePartialParams& p, int d, int g, int n_splits, int n_heads,
                                  cudaStream_t stream) {
    if (n_splits <= 0 || n_heads <= 0) return cudaSuccess;
    if (n_heads > MAX_LAUNCH_HEADS || p.kv_span < 1) return cudaErrorInvalidValue;
    if (d == 64) return launch_partial_d<64>(p, g, n_splits, n_heads, stream);
    if (d == 128) return launch_partial_d<128>(p, g, n_splits, n_heads, stream);
    return cudaErrorInvalidValue;
}

cudaError_t launch_decode_combine(const DecodeCombineParams& p, int d, int hq_loc, cudaStream_t stream) {
    if (d == 64) decode_combine_kernel<64><<<hq_loc, CB_WARPS * 32, 0, stream>>>(p);
    else if (d == 128) decode_combine_kernel<128><<<hq_loc, CB_WARPS * 32, 0, stream>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace hi
