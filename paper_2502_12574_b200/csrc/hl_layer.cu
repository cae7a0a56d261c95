// hl_layer.cu -- NEXT-4: the synthetic Llama decoder layer around the head-wise offloaded attention path
// (include/hilayer.h; the paper's whole-model setting).
//
// Per call, on the caller's stream:
//   rmsnorm_kernel      xn = bf16(x * rsqrt(mean(x^2) + eps) * gamma)          (fp32 inside)
//   gemm (k_gemm.cu)    qkv = bf16(xn W_qkv^T)                                 (tcgen05, fp32 accumulate)
//   rope_split_kernel   Q, K = bf16(rope(q, k)), V = v, split head-major for the attention call
//   hi_prefill_chunk / hi_decode   a = attention(Q, K, V)                      (the offloaded path)
//   gemm                x = bf16(x + a W_o^T)          (beta = 1: the residual is the epilogue)
//   rmsnorm_kernel      xn = ... mlp_norm
//   gemm                gu = bf16(xn W_gate_up^T)
//   swiglu_kernel       act = bf16(silu(g) * u)
//   gemm                x = bf16(x + act W_down^T)
// The projections run on this library's tcgen05 GEMM (k_gemm.cu; a streaming GEMV for one decode token); the
// elementwise / normalisation steps are HBM-bound one-pass kernels with 16-byte accesses.  RoPE angles are reduced in fp64 (p * inv_freq reaches 1e6 rad
// at 1M context, where an fp32 product would already be off by ~0.06 rad), then sin/cos in fp32.
#include "../../include/hilayer.h"
#include "hi_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <map>
#include <string>
#include <tuple>

namespace {

thread_local std::string g_hl_error = "no error";
constexpr int MAX_HALF_D = 64;  // head_dim <= 128

struct RopeParams {
    const __nv_bfloat16* qkv;  // [n][(hq + 2 hkv) * d]
    __nv_bfloat16* q;          // [n][hq][d]
    __nv_bfloat16* k;          // [n][hkv][d]
    __nv_bfloat16* v;          // [n][hkv][d]
    int n, hq, hkv, d;
    int64_t pos0;
    double inv_freq[MAX_HALF_D];
};

__device__ __forceinline__ float bf(const __nv_bfloat16 x) { return __bfloat162float(x); }

// One CTA per row: sum of squares in fp32 (8 bf16 per 16-byte load), then one rounding per output.
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ gamma,
                                                      __nv_bfloat16* __restrict__ out, int h, float eps) {
    const int64_t row = blockIdx.x;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
    const uint4* gr = reinterpret_cast<const uint4*>(gamma);
    uint4* orow = reinterpret_cast<uint4*>(out + row * h);
    const int n8 = h / 8;
    float ss = 0.f;
    for (int i = threadIdx.x; i < n8; i += blockDim.x) {
        const uint4 u = xr[i];
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += bf(e[j]) * bf(e[j]);
    }
    __shared__ float red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += red[w];
    const float rinv = rsqrtf(tot / static_cast<float>(h) + eps);
    for (int i = threadIdx.x; i < n8; i += blockDim.x) {
        const uint4 u = xr[i], gu = gr[i];
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&u);
        const __nv_bfloat16* g = reinterpret_cast<const __nv_bfloat16*>(&gu);
        uint4 w;
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&w);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16_rn(bf(e[j]) * rinv * bf(g[j]));
        orow[i] = w;
    }
}

// One CTA per token: cos/sin of the token's d/2 angles once (fp64 range reduction), then every q and k
// head's pairs (i, i + d/2) rotated (rotate-half convention) and V copied, into head-major tensors.
__global__ void __launch_bounds__(256) rope_split_kernel(const RopeParams p) {
    __shared__ float cs[MAX_HALF_D], sn[MAX_HALF_D];
    const int t = blockIdx.x;
    const int half = p.d / 2;
    if (threadIdx.x < half) {
        const double two_pi = 6.283185307179586476925286766559;
        double a = static_cast<double>(p.pos0 + t) * p.inv_freq[threadIdx.x];
        a -= two_pi * floor(a / two_pi);
        float s, c;
        sincosf(static_cast<float>(a), &s, &c);
        cs[threadIdx.x] = c;
        sn[threadIdx.x] = s;
    }
    __syncthreads();
    const int row = (p.hq + 2 * p.hkv) * p.d;
    const __nv_bfloat16* in = p.qkv + static_cast<int64_t>(t) * row;
    const int h2 = half / 2;  // each thread rotates two adjacent pairs: 4-byte loads / stores
    const int rot = (p.hq + p.hkv) * h2;
    for (int i = threadIdx.x; i < rot; i += blockDim.x) {
        const int hd = i / h2, j = 2 * (i % h2);  // heads [0, hq) are q, [hq, hq + hkv) are k
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(in + hd * p.d + j));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(in + hd * p.d + j + half));
        __nv_bfloat16* dst = hd < p.hq ? p.q + (static_cast<int64_t>(t) * p.hq + hd) * p.d
                                       : p.k + (static_cast<int64_t>(t) * p.hkv + (hd - p.hq)) * p.d;
        *reinterpret_cast<__nv_bfloat162*>(dst + j) =
            __floats2bfloat162_rn(a.x * cs[j] - b.x * sn[j], a.y * cs[j + 1] - b.y * sn[j + 1]);
        *reinterpret_cast<__nv_bfloat162*>(dst + j + half) =
            __floats2bfloat162_rn(b.x * cs[j] + a.x * sn[j], b.y * cs[j + 1] + a.y * sn[j + 1]);
    }
    const int v8 = p.hkv * p.d / 8;
    const uint4* vin = reinterpret_cast<const uint4*>(in + (p.hq + p.hkv) * p.d);
    uint4* vout = reinterpret_cast<uint4*>(p.v + static_cast<int64_t>(t) * p.hkv * p.d);
    for (int i = threadIdx.x; i < v8; i += blockDim.x) vout[i] = vin[i];
}

// act[t][c] = bf16(silu(g) * u), g = gu[t][c], u = gu[t][inter + c]; 8 columns per thread.
__global__ void swiglu_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act, int n,
                              int inter) {
    const int c8 = inter / 8;
    const int64_t total = static_cast<int64_t>(n) * c8;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t t = i / c8;
        const int c = static_cast<int>(i % c8);
        const uint4 gv = reinterpret_cast<const uint4*>(gu + t * 2 * inter)[c];
        const uint4 uv = reinterpret_cast<const uint4*>(gu + t * 2 * inter + inter)[c];
        const __nv_bfloat16* g = reinterpret_cast<const __nv_bfloat16*>(&gv);
        const __nv_bfloat16* u = reinterpret_cast<const __nv_bfloat16*>(&uv);
        uint4 w;
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&w);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float x = bf(g[j]);
            o[j] = __float2bfloat16_rn(x / (1.f + expf(-x)) * bf(u[j]));
        }
        reinterpret_cast<uint4*>(act + t * inter)[c] = w;
    }
}

// x[i] = bf16(x[i] + y[i]): the residual add of a tensor-parallel layer after its fp32 partial sums were
// all-reduced (one rounding, as the fused GEMM epilogue of the single-rank layer)
__global__ void residual_add_kernel(__nv_bfloat16* __restrict__ x, const float* __restrict__ y, int64_t n8) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint4 u = reinterpret_cast<uint4*>(x)[i];
        const float4 a = reinterpret_cast<const float4*>(y)[2 * i], b = reinterpret_cast<const float4*>(y)[2 * i + 1];
        __nv_bfloat16* e = reinterpret_cast<__nv_bfloat16*>(&u);
        const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = __float2bfloat16_rn(bf(e[j]) + f[j]);
        reinterpret_cast<uint4*>(x)[i] = u;
    }
}

}  // namespace

struct hl_model {
    hi_ctx* ctx = nullptr;
    hi::CtxInfo ci{};
    int H = 0, I = 0;   // I = this rank's intermediate columns (inter / world)
    float eps = 0.f;
    double inv_freq[MAX_HALF_D] = {0};
    std::string err = "no error";
    __nv_bfloat16 *xn = nullptr, *qkv = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *attn = nullptr,
                  *gu = nullptr, *act = nullptr;
    int64_t launches = 0;
};

namespace {

hi_status hl_fail(hl_model* m, hi_status s, const std::string& msg) {
    if (m) m->err = msg;
    else g_hl_error = msg;
    return s;
}

hi_status ck(hl_model* m, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return HI_OK;
    cudaGetLastError();
    return hl_fail(m, HI_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Y[n, mo] (+)= X[n, k] W[mo, k]^T, all row-major bf16; beta 0 or 1 (1: Y holds the residual, the sum is rounded
// once in the epilogue).  k_gemm.cu: tcgen05 GEMM (n >= 2) or GEMV (n == 1, decode).
hi_status gemm(hl_model* m, const __nv_bfloat16* W, const __nv_bfloat16* X, void* Y, int mo, int n, int kd,
               float beta, cudaStream_t st, bool out_f32 = false) {
    ++m->launches;
    return ck(m, hi::launch_gemm(W, X, Y, mo, n, kd, beta != 0.f ? 1 : 0, out_f32 ? 1 : 0, st), "launch_gemm");
}

hi_status residual_add(hl_model* m, __nv_bfloat16* x, const float* y, int n, cudaStream_t st) {
    const int64_t n8 = static_cast<int64_t>(n) * m->H / 8;
    const int grid = static_cast<int>(std::min<int64_t>((n8 + 255) / 256, 148 * 8));
    residual_add_kernel<<<grid, 256, 0, st>>>(x, y, n8);
    ++m->launches;
    return ck(m, cudaGetLastError(), "residual_add_kernel");
}

hi_status rmsnorm(hl_model* m, const __nv_bfloat16* x, const void* gamma, __nv_bfloat16* out, int n, cudaStream_t st) {
    rmsnorm_kernel<<<n, 256, 0, st>>>(x, static_cast<const __nv_bfloat16*>(gamma), out, m->H, m->eps);
    ++m->launches;
    return ck(m, cudaGetLastError(), "rmsnorm_kernel");
}

hi_status check_layer(hl_model* m, int layer_idx, const hl_weights* w, const void* xv) {
    if (!m) return HI_ESHAPE;
    if (!w || !xv || !w->attn_norm || !w->w_qkv || !w->w_o || !w->mlp_norm || !w->w_gate_up || !w->w_down)
        return hl_fail(m, HI_ESHAPE, "NULL weight or activation pointer");
    if (layer_idx < 0 || layer_idx >= m->ci.L) return hl_fail(m, HI_ESHAPE, "layer out of range");
    return HI_OK;
}

// Attention half of the layer: xn = rmsnorm(x), this rank's q|k|v = xn W_qkv^T, RoPE, the offloaded attention
// (`attend`: hi_prefill_chunk / hi_decode), then the O projection: x = bf16(x + a W_o^T) in the GEMM epilogue
// (y == NULL, single rank), or the fp32 partial y = a W_o^T of this rank's heads (tensor parallel).
template <typename Attend>
hi_status attn_half(hl_model* m, int layer_idx, const hl_weights* w, __nv_bfloat16* x, int n, float* y, cudaStream_t st,
                    Attend attend) {
    const int64_t s = hi_seq_len(m->ctx, layer_idx);
    const int hq = m->ci.Hq_loc, hkv = m->ci.Hkv_loc, d = m->ci.d;
    hi_status r;
    if ((r = rmsnorm(m, x, w->attn_norm, m->xn, n, st)) != HI_OK) return r;
    if ((r = gemm(m, static_cast<const __nv_bfloat16*>(w->w_qkv), m->xn, m->qkv, (hq + 2 * hkv) * d, n, m->H, 0.f, st)) != HI_OK)
        return r;
    RopeParams rp{};
    rp.qkv = m->qkv;
    rp.q = m->q;
    rp.k = m->k;
    rp.v = m->v;
    rp.n = n;
    rp.hq = hq;
    rp.hkv = hkv;
    rp.d = d;
    rp.pos0 = s;
    for (int i = 0; i < d / 2; ++i) rp.inv_freq[i] = m->inv_freq[i];
    rope_split_kernel<<<n, 256, 0, st>>>(rp);
    ++m->launches;
    if ((r = ck(m, cudaGetLastError(), "rope_split_kernel")) != HI_OK) return r;
    if ((r = attend()) != HI_OK) {
        m->err = std::string("attention: ") + hi_last_error(m->ctx);
        return r;
    }
    if (y) return gemm(m, static_cast<const __nv_bfloat16*>(w->w_o), m->attn, y, m->H, n, hq * d, 0.f, st, true);
    return gemm(m, static_cast<const __nv_bfloat16*>(w->w_o), m->attn, x, m->H, n, hq * d, 1.f, st);
}

// MLP half: xn = rmsnorm(x), this rank's gate|up = xn W_gate_up^T, SwiGLU, down projection: x = bf16(x + act W_down^T)
// (z == NULL, single rank) or the fp32 partial z = act W_down^T of this rank's intermediate columns.
hi_status mlp_half(hl_model* m, const hl_weights* w, __nv_bfloat16* x, int n, float* z, cudaStream_t st) {
    hi_status r;
    if ((r = rmsnorm(m, x, w->mlp_norm, m->xn, n, st)) != HI_OK) return r;
    if ((r = gemm(m, static_cast<const __nv_bfloat16*>(w->w_gate_up), m->xn, m->gu, 2 * m->I, n, m->H, 0.f, st)) != HI_OK)
        return r;
    const int64_t work = static_cast<int64_t>(n) * (m->I / 8);
    const int grid = static_cast<int>(std::min<int64_t>((work + 255) / 256, 148 * 8));
    swiglu_kernel<<<grid, 256, 0, st>>>(m->gu, m->act, n, m->I);
    ++m->launches;
    if ((r = ck(m, cudaGetLastError(), "swiglu_kernel")) != HI_OK) return r;
    if (z) return gemm(m, static_cast<const __nv_bfloat16*>(w->w_down), m->act, z, m->H, n, m->I, 0.f, st, true);
    return gemm(m, static_cast<const __nv_bfloat16*>(w->w_down), m->act, x, m->H, n, m->I, 1.f, st);
}

// The whole single-rank layer; `attend` runs hi_prefill_chunk / hi_decode.
template <typename Attend>
hi_status layer(hl_model* m, int layer_idx, const hl_weights* w, void* xv, int n, cudaStream_t st, Attend attend) {
    hi_status r = check_layer(m, layer_idx, w, xv);
    if (r != HI_OK) return r;
    if (m->ci.world != 1)
        return hl_fail(m, HI_ESTATE, "head-sharded context: use hl_attn_partial / hl_mlp_partial / hl_residual_add");
    __nv_bfloat16* x = static_cast<__nv_bfloat16*>(xv);
    if ((r = attn_half(m, layer_idx, w, x, n, nullptr, st, attend)) != HI_OK) return r;
    return mlp_half(m, w, x, n, nullptr, st);
}

void destroy(hl_model* m) {
    if (!m) return;
    cudaDeviceSynchronize();
    for (__nv_bfloat16* p : {m->xn, m->qkv, m->q, m->k, m->v, m->attn, m->gu, m->act}) cudaFree(p);
    cudaGetLastError();
    delete m;
}

}  // namespace

extern "C" {

const char* hl_last_error(const hl_model* m) { return m ? m->err.c_str() : g_hl_error.c_str(); }

hi_status hl_create(hi_ctx* ctx, int hidden, int inter, double rope_theta, float rms_eps, hl_model** out) {
    if (!out) return hl_fail(nullptr, HI_EINVAL, "out is NULL");
    *out = nullptr;
    hi::CtxInfo ci{};
    if (!hi::ctx_info(ctx, &ci)) return hl_fail(nullptr, HI_EINVAL, "ctx is NULL");
    if (hidden <= 0 || inter <= 0 || hidden % 64 || inter % (64 * ci.world) || !(rope_theta > 0.0) || !(rms_eps > 0.f))
        return hl_fail(nullptr, HI_EINVAL, "hidden must be a positive multiple of 64, inter of 64 * world; "
                                           "rope_theta, rms_eps > 0");
    hl_model* m = new hl_model();
    m->ctx = ctx;
    m->ci = ci;
    m->H = hidden;
    m->I = inter / ci.world;   // tensor parallel: this rank's intermediate columns
    m->eps = rms_eps;
    for (int i = 0; i < ci.d / 2; ++i) m->inv_freq[i] = pow(rope_theta, -2.0 * i / ci.d);
    auto bail = [&](hi_status s, const char* msg) {
        cudaGetLastError();
        destroy(m);
        return hl_fail(nullptr, s, msg);
    };
    hi::DeviceGuard dg(ci.device);  // allocate on the context's device; the caller's device is restored
    const size_t c = static_cast<size_t>(ci.chunk);
    const size_t elems[8] = {c * hidden, c * (ci.Hq_loc + 2 * ci.Hkv_loc) * ci.d, c * ci.Hq_loc * ci.d,
                             c * ci.Hkv_loc * ci.d, c * ci.Hkv_loc * ci.d, c * ci.Hq_loc * ci.d,
                             c * 2 * static_cast<size_t>(m->I), c * static_cast<size_t>(m->I)};
    __nv_bfloat16** bufs[8] = {&m->xn, &m->qkv, &m->q, &m->k, &m->v, &m->attn, &m->gu, &m->act};
    for (int i = 0; i < 8; ++i)
        if (cudaMalloc(reinterpret_cast<void**>(bufs[i]), elems[i] * 2) != cudaSuccess)
            return bail(HI_ENOMEM_DEV, "cudaMalloc of a layer workspace failed");
    *out = m;
    return HI_OK;
}

hi_status hl_prefill_chunk(hl_model* m, int layer_idx, const hl_weights* w, void* x, int n, void* cuda_stream) {
    if (m && (n < 1 || n > m->ci.chunk)) return hl_fail(m, HI_ESHAPE, "n_tokens must be in [1, chunk]");
    hi::DeviceGuard dg(m ? m->ci.device : 0);
    return layer(m, layer_idx, w, x, n, static_cast<cudaStream_t>(cuda_stream), [&] {
        return hi_prefill_chunk(m->ctx, layer_idx, m->q, m->k, m->v, m->attn, n, cuda_stream);
    });
}

hi_status hl_decode(hl_model* m, int layer_idx, const hl_weights* w, void* x, void* cuda_stream) {
    hi::DeviceGuard dg(m ? m->ci.device : 0);
    return layer(m, layer_idx, w, x, 1, static_cast<cudaStream_t>(cuda_stream), [&] {
        return hi_decode(m->ctx, layer_idx, m->q, m->k, m->v, m->attn, cuda_stream);
    });
}

hi_status hl_attn_partial(hl_model* m, int layer_idx, const hl_weights* w, const void* x, int n, int decode, void* y_f32,
                          void* cuda_stream) {
    hi_status r = check_layer(m, layer_idx, w, x);
    if (r != HI_OK) return r;
    if (!y_f32 || n < 1 || n > m->ci.chunk || (decode && n != 1))
        return hl_fail(m, HI_ESHAPE, "y_f32 NULL, n_tokens outside [1, chunk], or decode with n != 1");
    hi::DeviceGuard dg(m->ci.device);
    // x is read, not written: rmsnorm reads it; the residual add happens in hl_mlp_partial after the all-reduce
    __nv_bfloat16* xb = const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(x));
    return attn_half(m, layer_idx, w, xb, n, static_cast<float*>(y_f32), static_cast<cudaStream_t>(cuda_stream), [&] {
        return decode ? hi_decode(m->ctx, layer_idx, m->q, m->k, m->v, m->attn, cuda_stream)
                      : hi_prefill_chunk(m->ctx, layer_idx, m->q, m->k, m->v, m->attn, n, cuda_stream);
    });
}

hi_status hl_mlp_partial(hl_model* m, int layer_idx, const hl_weights* w, void* x, const void* y_f32, int n, void* z_f32,
                         void* cuda_stream) {
    hi_status r = check_layer(m, layer_idx, w, x);
    if (r != HI_OK) return r;
    if (!y_f32 || !z_f32 || n < 1 || n > m->ci.chunk) return hl_fail(m, HI_ESHAPE, "NULL partial or n_tokens out of range");
    hi::DeviceGuard dg(m->ci.device);
    const cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    __nv_bfloat16* xb = static_cast<__nv_bfloat16*>(x);
    if ((r = residual_add(m, xb, static_cast<const float*>(y_f32), n, st)) != HI_OK) return r;
    return mlp_half(m, w, xb, n, static_cast<float*>(z_f32), st);
}

hi_status hl_residual_add(hl_model* m, void* x, const void* z_f32, int n, void* cuda_stream) {
    if (!m) return HI_ESHAPE;
    if (!x || !z_f32 || n < 1) return hl_fail(m, HI_ESHAPE, "NULL tensor or n < 1");
    hi::DeviceGuard dg(m->ci.device);
    return residual_add(m, static_cast<__nv_bfloat16*>(x), static_cast<const float*>(z_f32), n,
                        static_cast<cudaStream_t>(cuda_stream));
}

hi_status hl_gemm(const void* w, const void* x, void* y, int mo, int n, int kd, int beta, void* cuda_stream) {
    if (!w || !x || !y || mo <= 0 || n <= 0 || kd <= 0 || mo % 64 || kd % 8)
        return hl_fail(nullptr, HI_EINVAL, "hl_gemm: NULL pointer or sizes (mo % 64, kd % 8)");
    const cudaError_t e = hi::launch_gemm(static_cast<const __nv_bfloat16*>(w), static_cast<const __nv_bfloat16*>(x),
                                          y, mo, n, kd, beta ? 1 : 0, 0, static_cast<cudaStream_t>(cuda_stream));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return hl_fail(nullptr, HI_ECUDA, std::string("hl_gemm: ") + cudaGetErrorString(e));
    }
    return HI_OK;
}

hi_status hl_free(hl_model* m) {
    destroy(m);
    return HI_OK;
}

}  // extern "C"
