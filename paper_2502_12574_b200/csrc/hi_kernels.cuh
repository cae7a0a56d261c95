// hi_kernels.cuh -- internal launch interface between the host runtime (hi_runtime.cu)
// and the device kernels of libheadinfer.so.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

struct hi_ctx;  // include/headinfer.h

namespace hi {

// Every entry point runs on the context's device and gives the caller back the current device it had
// (one process may hold contexts on several GPUs; the caller's own device choice is not ours to change).
struct DeviceGuard {
    int prev = -1;
    bool switched = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) switched = cudaSetDevice(dev) == cudaSuccess;
        cudaGetLastError();
    }
    ~DeviceGuard() {
        if (switched) cudaSetDevice(prev);
    }
};

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device.  The attribute is per device,
// so the "done" flag is kept per device ordinal (a process may hold contexts on several GPUs); setting it
// twice from racing threads is harmless.
template <typename K>
cudaError_t set_smem_attr_once(K kernel, int bytes, std::atomic<unsigned long long>& done_mask) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done_mask.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Context geometry for the layer wrapper (hl_layer.cu, NEXT-4); false on NULL.
struct CtxInfo {
    int L, Hq_loc, Hkv_loc, d, chunk, world, device;
};
bool ctx_info(const hi_ctx* c, CtxInfo* out);

// TMA tensor map over a bf16 tensor, SWIZZLE_128B, (tmap.cu); dims/strides innermost-first, strides in
// bytes (rank-1 entries).  false if the driver entry point is unavailable or the encode fails.
bool make_tmap_bf16(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                    const cuuint32_t* box);

// ---- prefill attention over one KV segment -------------------------
// Computes, for the g q heads of one kv head group, rows r = t*g + j (token t of the chunk,
// group member j; GQA packing), the flash-attention update of the running state
// (O, m, l) with the keys of ONE contiguous segment [k_pos0, k_pos0 + n_k): either a history
// block sitting in a staging slot or the chunk's own K/V (causal).  Scores are kept in the
// log2 domain: x = (q.k) * log2(e)/sqrt(d); m is the running max of x, l = sum 2^(x-m),
// O = sum 2^(x-m) v.  FIRST initialises the state, LAST writes out = O / l as bf16.
enum PrefillFlags : int { PF_FIRST = 1, PF_LAST = 2, PF_CAUSAL = 4 };
constexpr int MAX_LAUNCH_HEADS = 64;  // kv heads one launch may cover (and the cap on kv_heads/world)

struct PrefillParams {
    const __nv_bfloat16* q;   // (token 0, first q head of the group); row (t,j) at q + t*q_tok_stride + j*d
    int64_t q_tok_stride;     // elements between consecutive tokens (Hq_loc * d)
    __nv_bfloat16* out;       // same addressing as q
    int64_t o_tok_stride;
    const __nv_bfloat16* k;   // key i of the segment at k + i*kv_row_stride
    const __nv_bfloat16* v;
    int64_t kv_row_stride;
    int n_q;                  // tokens in the chunk
    int n_k;                  // keys in this segment
    int64_t q_pos0;           // global position of token 0
    int64_t k_pos0;           // global position of key 0 of the segment
    int g;                    // q heads per kv head
    float scale_log2;         // log2(e) / sqrt(d)
    float* o_acc;             // [n_q*g][d] fp32 running O
    float* m_acc;             // [n_q*g]
    float* l_acc;             // [n_q*g]
    int flags;
    // head groups (NEXT-2): n_heads kv heads per launch (blockIdx.y); head h's q/out columns start at
    // (h*g)*d, its keys at k/v + h*kv_head_stride, its running state at + h*state_rows rows
    int n_heads;              // 1 = one kv head (k_prefill_mma.cu / k_prefill_tc2.cu support only 1)
    int64_t kv_head_stride;   // elements
    int64_t state_rows;       // rows of O/m/l state per head (>= n_q*g)
    // head maps (any set of kv heads per launch): blockIdx.y = hh takes q/out columns of kv head head_q[hh]
    // (q heads head_q[hh]*g ..), keys at k/v + head_kv[hh]*kv_head_stride, state rows hh*state_rows; the q/out
    // tensor map spans q_span kv heads' q columns, the k/v map kv_span heads.  set_identity_heads() = h0 + hh.
    int16_t head_q[MAX_LAUNCH_HEADS];
    int16_t head_kv[MAX_LAUNCH_HEADS];
    int q_span, kv_span;
    // NEXT-3 duo-attention streaming heads (reading R18): win > 0 restricts key i of the segment to
    // i > p - win for query position p (the recent window).  The runtime only passes win > 0 for segments
    // that hold no sink keys (k_pos0 >= n_sink); sink segments are plain (all visible).
    int win;
    int row_rev;              // set by the launcher: CTA x takes the rows of CTA |row_rev - x| (grid - 1 for causal
                              // segments: longest-first); 0 = in order
};
inline void set_identity_heads(PrefillParams& p, int n) {
    for (int i = 0; i < n && i < MAX_LAUNCH_HEADS; ++i) p.head_q[i] = p.head_kv[i] = static_cast<int16_t>(i);
    p.q_span = p.kv_span = n;
}
// sm_100a kernels: TMA + tcgen05.mma + TMEM.  k_prefill_tc.cu: one CTA per 256 rows (any head_dim) --
// the product path; k_prefill_tc2.cu: CTA pairs (cta_group::2, M = 256), head_dim 128, HI_FLAG_PREFILL_2CTA
cudaError_t launch_prefill_tc2(const PrefillParams& p, int d, cudaStream_t stream);
cudaError_t launch_prefill_tc(const PrefillParams& p, int d, cudaStream_t stream);
// variants/k_prefill_tcp.cu (variants build only): the same contract with P staged in shared memory
cudaError_t launch_prefill_tcp(const PrefillParams& p, int d, cudaStream_t stream);
// k_prefill_tc1.cu: one CTA per 128 rows, three S buffers in TMEM, K/V multicast to CTA pairs
cudaError_t launch_prefill_tc1(const PrefillParams& p, int d, cudaStream_t stream);
// baseline comparator: mma.sync m16n8k16 (k_prefill_mma.cu), selected by HI_FLAG_MMA_SYNC_PREFILL
cudaError_t launch_prefill_mma(const PrefillParams& p, int d, cudaStream_t stream);

// ---- decode: split-K partials over one history block + LSE combine (a8) ----------------
struct DecodePartialParams {
    const __nv_bfloat16* q;   // [g][d] q rows of the group (contiguous)
    const __nv_bfloat16* k;   // [n_k][d] block in a staging slot
    const __nv_bfloat16* v;
    int n_k;
    int split_len;            // keys per CTA
    float scale_log2;
    float* parts;             // records for this launch: parts + (blockIdx.x*g + j)*(d+4): {m, l, pad, pad, o[d]}
    // several kv heads in one launch (blockIdx.y = head; HBM-resident heads, NEXT-1): per-head strides
    int64_t kv_head_stride;   // elements between head h and h+1 in k and in v (0 when n_heads == 1)
    int64_t q_head_stride;    // elements between the q groups of consecutive heads (g*d)
    int64_t parts_head_stride;// floats between the record arrays of consecutive heads
    // head maps: blockIdx.y = y reads q group head[y] (q + head[y]*q_head_stride), writes records at
    // parts + head[y]*parts_head_stride, and streams keys of k/v head coordinate kvc[y] (stride
    // kv_head_stride; the tensor map spans kv_span heads)
    int16_t head[MAX_LAUNCH_HEADS];
    int16_t kvc[MAX_LAUNCH_HEADS];
    int kv_span;
    // Fused combine (the launch holds EVERY record of its heads, e.g. all-resident layers, NEXT-1): the last CTA
    // of head y to finish (per-head completion counter, self-resetting) merges records [0, parts_total) of head
    // head[y] with the new key by log-sum-exp and writes out rows head[y]*g .. +g; with `append` it also writes
    // the new key/value as row n_k of kv coordinate kvc[y] (the cache row the next decode step reads).
    int combine;
    int append;
    int parts_total;
    unsigned* counters;           // [>= max head index + 1], zero between launches
    const __nv_bfloat16* k_new;   // [*][d]: head head[y] at k_new + head[y]*d
    const __nv_bfloat16* v_new;
    __nv_bfloat16* out;           // [*][d]: q head head[y]*g + j
};
inline void set_identity_heads(DecodePartialParams& p, int n) {
    for (int i = 0; i < n && i < MAX_LAUNCH_HEADS; ++i) p.head[i] = p.kvc[i] = static_cast<int16_t>(i);
    p.kv_span = n;
}
cudaError_t launch_decode_partial(const DecodePartialParams& p, int d, int g, int n_splits, int n_heads,
                                  cudaStream_t stream);

struct DecodeCombineParams {
    const __nv_bfloat16* q;      // [Hq_loc][d]
    const __nv_bfloat16* k_new;  // [Hkv_loc][d]  the new token's key (attends itself, reading R3)
    const __nv_bfloat16* v_new;  // [Hkv_loc][d]
    const float* parts;          // [Hkv_loc][max_parts][g][d+4]
    int max_parts;
    int32_t n_parts[MAX_LAUNCH_HEADS];  // records per local kv head (offloaded / resident / streaming differ)
    int g;
    float scale_log2;
    __nv_bfloat16* out;          // [Hq_loc][d]
};
cudaError_t launch_decode_combine(const DecodeCombineParams& p, int d, int hq_loc, cudaStream_t stream);

// ---- pack the chunk's K and V [n][Hkv][d] into head-major [Hkv][2][n][d] (a2, K5b) ------
cudaError_t launch_pack_kv(const __nv_bfloat16* k, const __nv_bfloat16* v, __nv_bfloat16* packed,
                           int n, int hkv, int d, cudaStream_t stream);

// ---- NEXT-3: append new K/V rows of the duo streaming heads into their device sink + ring buffers ----
// For each listed kv head heads[y] and new position p in [pos0, pos0+n): rows p < n_sink go to sink row p,
// rows p >= max(n_sink, pos0+n-ring) to ring row n_sink + (p-n_sink) % ring (the rest are overwritten in the
// same call and skipped).  Source row (y, t) at src_k/src_v + heads[y]*src_head_stride + t*src_row_stride;
// destination head h at dst + h*dst_head_stride (K rows, then V rows dst_v_off elements later).
struct DuoAppendParams {
    const __nv_bfloat16* src_k;
    const __nv_bfloat16* src_v;
    int64_t src_head_stride, src_row_stride;
    __nv_bfloat16* dst;
    int64_t dst_head_stride, dst_v_off;
    int64_t pos0;
    int n, n_sink, ring, n_heads;
    int16_t heads[MAX_LAUNCH_HEADS];
};
cudaError_t launch_duo_append(const DuoAppendParams& p, int d, cudaStream_t stream);

// ---- fill with a NaN bit pattern (poison mode, race detection) --------------------------
cudaError_t launch_poison(void* ptr, size_t bytes, cudaStream_t stream);
cudaError_t launch_spin(uint64_t ns, cudaStream_t stream);

// ---- NEXT-4 layer projections (k_gemm.cu): y[n, mo] = (beta ? y : 0) + x[n, kd] w[mo, kd]^T, bf16 in/out, fp32
// accumulate; tcgen05 persistent GEMM for n >= 2, an HBM-streaming GEMV for n == 1.  mo % 64 == 0, kd % 8 == 0.
// out_f32: y is fp32 and written unrounded (beta must be 0) -- the tensor-parallel layer's partial sums.
cudaError_t launch_gemm(const __nv_bfloat16* w, const __nv_bfloat16* x, void* y, int mo, int n, int kd, int beta,
                        int out_f32, cudaStream_t stream);
cudaError_t launch_fault(bool trap, cudaStream_t stream);

}  // namespace hi
