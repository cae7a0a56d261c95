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

constexpr int DEC_THREADS = 128;
constexpr int DEC_UNROLL = 4;

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

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// One CTA = keys [blockIdx.x*split_len, +split_len) of the block.  Lane layout: LPK = D/8 lanes
// hold one key row (16 B each); KPW = 32/LPK keys per warp step.
template <int D, int G>
__global__ void __launch_bounds__(DEC_THREADS) decode_partial_kernel(const DecodePartialParams p) {
    constexpr int LPK = D / 8;
    constexpr int KPW = 32 / LPK;
    constexpr int NW = DEC_THREADS / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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

    const int k_begin = blockIdx.x * p.split_len;
    const int k_end = min(p.n_k, k_begin + p.split_len);
    // warp w handles keys k_begin + (step*NW + w)*KPW + sub
    for (int base = k_begin + warp * KPW; base < k_end; base += NW * KPW * DEC_UNROLL) {
        uint4 kr[DEC_UNROLL], vr[DEC_UNROLL];
        bool valid[DEC_UNROLL];
#pragma unroll
        for (int u = 0; u < DEC_UNROLL; ++u) {
            const int key = base + u * NW * KPW + sub;
            valid[u] = key < k_end;
            const int64_t off = static_cast<int64_t>(valid[u] ? key : k_begin) * D + part * 8;
            kr[u] = ld_stream(p.k + off);
            vr[u] = ld_stream(p.v + off);
        }
        float x[DEC_UNROLL][G];
#pragma unroll
        for (int u = 0; u < DEC_UNROLL; ++u) {
            float kf[8];
            bf16x8_to_f32(kr[u], kf);
#pragma unroll
            for (int j = 0; j < G; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) acc = fmaf(q[j][i], kf[i], acc);
                x[u][j] = acc;
            }
        }
#pragma unroll
        for (int off = 1; off < LPK; off <<= 1)
#pragma unroll
            for (int u = 0; u < DEC_UNROLL; ++u)
#pragma unroll
                for (int j = 0; j < G; ++j) x[u][j] += __shfl_xor_sync(0xffffffffu, x[u][j], off);
#pragma unroll
        for (int j = 0; j < G; ++j) {
            float mx = m[j];
#pragma unroll
            for (int u = 0; u < DEC_UNROLL; ++u)
                if (valid[u]) mx = fmaxf(mx, x[u][j]);
            const float alpha = (m[j] == -CUDART_INF_F) ? 0.f : fast_exp2(m[j] - mx);
            m[j] = mx;
            l[j] *= alpha;
#pragma unroll
            for (int i = 0; i < 8; ++i) o[j][i] *= alpha;
#pragma unroll
            for (int u = 0; u < DEC_UNROLL; ++u) {
                if (!valid[u]) continue;
                const float pw = fast_exp2(x[u][j] - mx);
                l[j] += pw;
                float vf[8];
                bf16x8_to_f32(vr[u], vf);
#pragma unroll
                for (int i = 0; i < 8; ++i) o[j][i] = fmaf(pw, vf[i], o[j][i]);
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
            for (int i = 0; i < 8; ++i) {
                const float o2 = __shfl_xor_sync(0xffffffffu, o[j][i], off);
                o[j][i] = o[j][i] * a1 + o2 * a2;
            }
            m[j] = mx;
        }
    }
    // merge the warps through shared memory
    __shared__ float sm_m[NW][G], sm_l[NW][G];
    __shared__ float sm_o[NW][G][D];
    if (sub == 0) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
            if (part == 0) { sm_m[warp][j] = m[j]; sm_l[warp][j] = l[j]; }
#pragma unroll
            for (int i = 0; i < 8; ++i) sm_o[warp][j][part * 8 + i] = o[j][i];
        }
    }
    __syncthreads();
    float* rec = p.parts + static_cast<int64_t>(blockIdx.x) * G * (D + 4);
    for (int idx = threadIdx.x; idx < G * D; idx += DEC_THREADS) {
        const int j = idx / D, c = idx % D;
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < NW; ++w) mx = fmaxf(mx, sm_m[w][j]);
        float lsum = 0.f, osum = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float a = (sm_m[w][j] == -CUDART_INF_F) ? 0.f : fast_exp2(sm_m[w][j] - mx);
            lsum += a * sm_l[w][j];
            osum += a * sm_o[w][j][c];
        }
        float* r = rec + j * (D + 4);
        r[4 + c] = osum;
        if (c == 0) { r[0] = mx; r[1] = lsum; }
    }
}

// One CTA per local q head: merge the n_parts records of its kv head with the new key.
template <int D>
__global__ void __launch_bounds__(D) decode_combine_kernel(const DecodeCombineParams p) {
    const int jq = blockIdx.x;          // local q head
    const int h = jq / p.g, j = jq % p.g;
    const int c = threadIdx.x;
    __shared__ float red[D / 32];
    __shared__ float s_x;
    // score of the new key (the token attends itself, reading R3)
    const float qc = __bfloat162float(p.q[jq * D + c]);
    const float kc = __bfloat162float(p.k_new[h * D + c]);
    float prod = qc * kc;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, off);
    if ((c & 31) == 0) red[c >> 5] = prod;
    __syncthreads();
    if (c == 0) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < D / 32; ++w) t += red[w];
        s_x = t * p.scale_log2;
    }
    __syncthreads();
    const float x = s_x;
    const float* recs = p.parts + (static_cast<int64_t>(h) * p.max_parts * p.g + j) * (D + 4);
    const int64_t rstride = static_cast<int64_t>(p.g) * (D + 4);
    float mx = x;
    for (int i = 0; i < p.n_parts; ++i) mx = fmaxf(mx, recs[i * rstride]);
    const float a0 = fast_exp2(x - mx);
    float lsum = a0;
    float osum = a0 * __bfloat162float(p.v_new[h * D + c]);
    for (int i = 0; i < p.n_parts; ++i) {
        const float* r = recs + i * rstride;
        const float mi = r[0];
        const float a = (mi == -CUDART_INF_F) ? 0.f : fast_exp2(mi - mx);
        lsum += a * r[1];
        osum += a * r[4 + c];
    }
    p.out[jq * D + c] = __float2bfloat16_rn(osum / lsum);
}

template <int D, int G>
cudaError_t launch_partial_dg(const DecodePartialParams& p, int n_splits, cudaStream_t s) {
    decode_partial_kernel<D, G><<<n_splits, DEC_THREADS, 0, s>>>(p);
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
    if (d == 64) decode_combine_kernel<64><<<hq_loc, 64, 0, stream>>>(p);
    else if (d == 128) decode_combine_kernel<128><<<hq_loc, 128, 0, stream>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace hi
