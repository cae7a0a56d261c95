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

constexpr int TD_CONSUMERS = 8;                       // consumer warps
constexpr int TD_THREADS = (TD_CONSUMERS + 1) * 32;   // + 1 producer warp
constexpr int TD_STAGES = 4;
template <int G>
constexpr int td_chunk() { return G >= 8 ? 32 : 64; }  // keys per pipeline stage (register budget at g = 8)

template <int D, int G>
constexpr int td_smem_bytes() { return TD_STAGES * 2 * td_chunk<G>() * D * 2 + 2 * TD_STAGES * 8 + 128; }

// One CTA = keys [blockIdx.x*split_len, +split_len) of the block.  One producer thread streams the
// CTA's contiguous K and V rows into a TD_STAGES-deep shared-memory ring with cp.async.bulk (the
// TMA engine: a few bulk requests keep >100 KiB in flight per SM, which is what HBM latency needs);
// 8 consumer warps compute from shared memory.  Lane layout: LPK = D/8 lanes hold one key row
// (16 B each); KPW = 32/LPK keys per warp step.
template <int D, int G>
__global__ void __launch_bounds__(TD_THREADS, 1) decode_partial_kernel(const DecodePartialParams p) {
    constexpr int LPK = D / 8;
    constexpr int KPW = 32 / LPK;
    constexpr int NW = TD_CONSUMERS;
    constexpr int TD_CHUNK = td_chunk<G>();
    constexpr int STAGE_BYTES = 2 * TD_CHUNK * D * 2;
    extern __shared__ __align__(128) uint8_t td_smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(td_smem + TD_STAGES * STAGE_BYTES);
    const uint32_t sbase = smem_u32(td_smem);
    auto bar_full = [&](int s) { return smem_u32(&bars[s]); };
    auto bar_empty = [&](int s) { return smem_u32(&bars[TD_STAGES + s]); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int k_begin = blockIdx.x * p.split_len;
    const int k_end = min(p.n_k, k_begin + p.split_len);
    const int n_chunks = (k_end - k_begin + TD_CHUNK - 1) / TD_CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TD_STAGES; ++s) {
            mbar_init(bar_full(s), 1);
            mbar_init(bar_empty(s), NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {
        // ---------------- producer: bulk copies of K and V rows into the ring ----------------
        if (lane == 0) {
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % TD_STAGES;
                if (i >= TD_STAGES) mbar_wait(bar_empty(s), ((i / TD_STAGES) - 1) & 1);
                const int k0 = k_begin + i * TD_CHUNK;
                const uint32_t bytes = static_cast<uint32_t>(min(TD_CHUNK, k_end - k0)) * D * 2;
                mbar_expect_tx(bar_full(s), 2 * bytes);
                bulk_g2s(sbase + s * STAGE_BYTES, p.k + static_cast<int64_t>(k0) * D, bytes, bar_full(s));
                bulk_g2s(sbase + s * STAGE_BYTES + TD_CHUNK * D * 2, p.v + static_cast<int64_t>(k0) * D, bytes,
                         bar_full(s));
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int sub = lane / LPK, part = lane % LPK;
    float q[G][8];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        float f[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(p.q + j * D + part * 8), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) q[j][i] = f[i] * p.scale_log2;  // fold log2(e)/sqrt(d) into q
    }
    float m[G], l[G], o[G][8];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        m[j] = -CUDART_INF_F;
        l[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[j][i] = 0.f;
    }
    constexpr int KEYS_PER_WARP = TD_CHUNK / NW;
    constexpr int U = KEYS_PER_WARP / KPW;                 // key steps per warp per chunk
    for (int i = 0; i < n_chunks; ++i) {
        const int s = i % TD_STAGES;
        mbar_wait(bar_full(s), (i / TD_STAGES) & 1);
        const int nk = min(TD_CHUNK, k_end - (k_begin + i * TD_CHUNK));
        const uint8_t* sk = td_smem + s * STAGE_BYTES;
        const uint8_t* sv = sk + TD_CHUNK * D * 2;
        uint4 kr[U], vr[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int key = warp * KEYS_PER_WARP + u * KPW + sub;
            valid[u] = key < nk;
            const int kk = valid[u] ? key : 0;
            kr[u] = *reinterpret_cast<const uint4*>(sk + kk * D * 2 + part * 16);
            vr[u] = *reinterpret_cast<const uint4*>(sv + kk * D * 2 + part * 16);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty(s));  // this warp's reads of stage s are done
        float x[U][G];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float kf[8];
            bf16x8_to_f32(kr[u], kf);
#pragma unroll
            for (int j = 0; j < G; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) acc = fmaf(q[j][e], kf[e], acc);
                x[u][j] = acc;
            }
        }
#pragma unroll
        for (int off = 1; off < LPK; off <<= 1)
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int j = 0; j < G; ++j) x[u][j] += __shfl_xor_sync(0xffffffffu, x[u][j], off);
#pragma unroll
        for (int j = 0; j < G; ++j) {
            float mx = m[j];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (valid[u]) mx = fmaxf(mx, x[u][j]);
            const float alpha = (m[j] == -CUDART_INF_F) ? 0.f : fast_exp2(m[j] - mx);
            m[j] = mx;
            l[j] *= alpha;
#pragma unroll
            for (int e = 0; e < 8; ++e) o[j][e] *= alpha;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!valid[u]) continue;
                const float pw = fast_exp2(x[u][j] - mx);
                l[j] += pw;
                float vf[8];
                bf16x8_to_f32(vr[u], vf);
#pragma unroll
                for (int e = 0; e < 8; ++e) o[j][e] = fmaf(pw, vf[e], o[j][e]);
            }
        }
    }

    // merge the KPW key slots of the warp (lanes with equal `part`)
#pragma unroll
    for (int off = LPK; off < 32; off <<= 1) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m[j], off);
            const float l2 = __shfl_xor_sync(0xffffffffu, l[j], off);
            const float mx = fmaxf(m[j], m2);
            const float a1 = (m[j] == -CUDART_INF_F) ? 0.f : fast_exp2(m[j] - mx);
            const float a2 = (m2 == -CUDART_INF_F) ? 0.f : fast_exp2(m2 - mx);
            l[j] = l[j] * a1 + l2 * a2;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float o2 = __shfl_xor_sync(0xffffffffu, o[j][e], off);
                o[j][e] = o[j][e] * a1 + o2 * a2;
            }
            m[j] = mx;
        }
    }
    // merge the consumer warps through shared memory (the ring is free: every chunk was consumed)
    float* sm_m = reinterpret_cast<float*>(td_smem);          // [NW][G]
    float* sm_l = sm_m + NW * G;                              // [NW][G]
    float* sm_o = sm_l + NW * G;                              // [NW][G][D]
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");  // all consumers done with the ring
    if (sub == 0) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
            if (part == 0) { sm_m[warp * G + j] = m[j]; sm_l[warp * G + j] = l[j]; }
#pragma unroll
            for (int e = 0; e < 8; ++e) sm_o[(warp * G + j) * D + part * 8 + e] = o[j][e];
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
    float* rec = p.parts + static_cast<int64_t>(blockIdx.x) * G * (D + 4);
    for (int idx = threadIdx.x; idx < G * D; idx += NW * 32) {
        const int j = idx / D, c = idx % D;
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < NW; ++w) mx = fmaxf(mx, sm_m[w * G + j]);
        float lsum = 0.f, osum = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float mw = sm_m[w * G + j];
            const float a = (mw == -CUDART_INF_F) ? 0.f : fast_exp2(mw - mx);
            lsum += a * sm_l[w * G + j];
            osum += a * sm_o[(w * G + j) * D + c];
        }
        float* r = rec + j * (D + 4);
        r[4 + c] = osum;
        if (c == 0) { r[0] = mx; r[1] = lsum; }
    }
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
    const int n_parts = h < p.h_lo ? p.n_parts_lo : p.n_parts;
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
cudaError_t launch_partial_dg(const DecodePartialParams& p, int n_splits, cudaStream_t s) {
    constexpr int smem = td_smem_bytes<D, G>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(decode_partial_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    decode_partial_kernel<D, G><<<n_splits, TD_THREADS, smem, s>>>(p);
    return cudaGetLastError();
}
template <int D>
cudaError_t launch_partial_d(const DecodePartialParams& p, int g, int n_splits, cudaStream_t s) {
    switch (g) {
        case 1: return launch_partial_dg<D, 1>(p, n_splits, s);
        case 2: return launch_partial_dg<D, 2>(p, n_splits, s);
        case 4: return launch_partial_dg<D, 4>(p, n_splits, s);
        case 8: return launch_partial_dg<D, 8>(p, n_splits, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_decode_partial(const DecodePartialParams& p, int d, int g, int n_splits, cudaStream_t stream) {
    if (n_splits <= 0) return cudaSuccess;
    if (d == 64) return launch_partial_d<64>(p, g, n_splits, stream);
    if (d == 128) return launch_partial_d<128>(p, g, n_splits, stream);
    return cudaErrorInvalidValue;
}

cudaError_t launch_decode_combine(const DecodeCombineParams& p, int d, int hq_loc, cudaStream_t stream) {
    if (d == 64) decode_combine_kernel<64><<<hq_loc, CB_WARPS * 32, 0, stream>>>(p);
    else if (d == 128) decode_combine_kernel<128><<<hq_loc, CB_WARPS * 32, 0, stream>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace hi
