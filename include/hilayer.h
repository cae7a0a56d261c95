/*
 * hilayer.h -- C ABI of the synthetic Llama decoder layer around the head-wise offloaded attention
 * path ("Full synthetic transformer layer around the path (QKV/O GEMMs, RoPE,
 * MLP)", the paper's whole-model setting, §5, Tab. 6/7 P:L568-606).  Exported by the
 * same libheadinfer.so as headinfer.h.
 *
 * One layer, in the paper's model family (Llama-3), inference only (weights are the caller's,
 * random-init in benches and tests: no trained weights exist here).  For hidden states x [n, hidden]
 * at global positions s .. s+n-1 (s = hi_seq_len(ctx, layer) before the call):
 *
 *   xn   = rmsnorm(x) * attn_norm                  (RMSNorm, eps rms_eps)
 *   q|k|v = xn W_qkv^T                             (row-major weight [(Hq + 2 Hkv) d, hidden])
 *   q, k = rope(q, k, position)                    (rotate-half RoPE, inv_freq_i = theta^(-2i/d))
 *   a    = attention(q, k, v)                      (hi_prefill_chunk / hi_decode: the offloaded path)
 *   x    = x + a W_o^T                             ([hidden, Hq d])
 *   xn   = rmsnorm(x) * mlp_norm
 *   g|u  = xn W_gate_up^T                          ([2 inter, hidden]: gate rows, then up rows)
 *   x    = x + (silu(g) * u) W_down^T              ([hidden, inter])
 *
 * Storage is bf16 at every op boundary above (reading R19 in DESIGN.md); arithmetic inside an op is
 * fp32 (the projections on this library's tcgen05 GEMM with fp32 accumulation -- a streaming GEMV for a
 * single decode token -- and the norm / RoPE / SwiGLU in its one-pass kernels).
 * Layout: every tensor is row-major, contiguous, bf16, on the context's device.  x is updated in place.
 *
 * Tensor parallelism (a context created with world W > 1, SURVEY.md §8(f) NEXT-4 "70B via TP"): the layer
 * splits like the attention path -- rank r owns the q / kv heads of its head shard and the intermediate
 * columns [r*inter/W, (r+1)*inter/W).  Its weights are the matching shards: w_qkv = the rank's q-head rows, then
 * its k-head rows, then its v-head rows ([(Hq_loc + 2 Hkv_loc) d, hidden]); w_o = the rank's q-head columns
 * ([hidden, Hq_loc d]); w_gate_up = the rank's gate rows then its up rows ([2 inter/W, hidden]); w_down = the
 * rank's intermediate columns ([hidden, inter/W]); the norms are replicated.  x is replicated.  A layer is then
 *   hl_attn_partial   -> y  (fp32 [n, hidden]: this rank's a W_o^T, unrounded)      caller: all-reduce(y, sum)
 *   hl_mlp_partial    -> x = bf16(x + y); z (fp32: this rank's act W_down^T)        caller: all-reduce(z, sum)
 *   hl_residual_add   -> x = bf16(x + z)
 * which is the single-rank layer with the two residual sums rounded once each, up to the fp32 order of the sum
 * over ranks (at W = 1 the three calls are bit-identical to hl_prefill_chunk / hl_decode).  The collectives are
 * the caller's (NCCL through torch.distributed); hl_prefill_chunk / hl_decode need world == 1 (HI_ESTATE otherwise).
 *
 * Ownership: the caller owns x and the weights; the model owns its workspaces (sized for the context's
 * chunk) and never retains caller pointers.  All work is ordered on the caller's stream.
 * Errors: hi_status codes as in headinfer.h; a CUDA or cuBLAS failure returns HI_ECUDA.
 */
#ifndef HILAYER_H_
#define HILAYER_H_

#include "headinfer.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hl_model hl_model; /* opaque; one per hi_ctx */

/* One decoder layer's weights: device pointers, bf16, row-major [out, in] (PyTorch Linear layout). */
typedef struct hl_weights {
    const void* attn_norm;  /* [hidden] */
    const void* w_qkv;      /* [(Hq + 2 Hkv) * head_dim, hidden]: q heads, then k heads, then v heads */
    const void* w_o;        /* [hidden, Hq * head_dim] */
    const void* mlp_norm;   /* [hidden] */
    const void* w_gate_up;  /* [2 * inter, hidden]: gate rows [0, inter), up rows [inter, 2 inter) */
    const void* w_down;     /* [hidden, inter] */
} hl_weights;

/*
 * hl_create -- workspaces (for up to the context's `chunk` tokens) for layers around `ctx`'s attention.
 * hidden: multiple of 64; inter: multiple of 64 * world; rope_theta > 0; rms_eps > 0.
 * Errors: HI_EINVAL (sizes), HI_ENOMEM_DEV, HI_ECUDA.
 */
hi_status hl_create(hi_ctx* ctx, int hidden, int inter, double rope_theta, float rms_eps, hl_model** out);

/* One prefill chunk of one layer: x [n, hidden] in place (n in [1, chunk]); the attention step is
 * hi_prefill_chunk on the same layer (so seq_len[layer] advances by n).  Errors as hi_prefill_chunk. */
hi_status hl_prefill_chunk(hl_model* m, int layer, const hl_weights* w, void* x, int n, void* cuda_stream);

/* One decode token of one layer: x [hidden] in place; the attention step is hi_decode. */
hi_status hl_decode(hl_model* m, int layer, const hl_weights* w, void* x, void* cuda_stream);

/* Tensor-parallel halves of one layer (see above).  decode != 0: one token (n must be 1), attention = hi_decode.
 * y_f32 / z_f32: fp32 [n, hidden] device buffers the call writes.  Errors as hl_prefill_chunk. */
hi_status hl_attn_partial(hl_model* m, int layer, const hl_weights* w, const void* x, int n, int decode, void* y_f32,
                          void* cuda_stream);
hi_status hl_mlp_partial(hl_model* m, int layer, const hl_weights* w, void* x, const void* y_f32, int n, void* z_f32,
                         void* cuda_stream);
hi_status hl_residual_add(hl_model* m, void* x, const void* z_f32, int n, void* cuda_stream);

/* The layer's projection as a stand-alone call (tests and benches): y[n, mo] = (beta ? y : 0) + x[n, kd] w[mo, kd]^T,
 * row-major bf16 device tensors, fp32 accumulation, ONE rounding to bf16 (the residual add is the epilogue).
 * n >= 2: persistent tcgen05 GEMM (128 x 256 x 64 tiles, TMA, TMEM accumulators); n == 1: streaming GEMV.
 * mo must be a multiple of 64, kd of 8; w, x, y 16-byte aligned; ordered on cuda_stream.
 * Errors: HI_EINVAL (sizes), HI_ECUDA. */
hi_status hl_gemm(const void* w, const void* x, void* y, int mo, int n, int kd, int beta, void* cuda_stream);

/* Release the workspaces (the hi_ctx is not freed).  NULL is a no-op. */
hi_status hl_free(hl_model* m);

/* Message describing the model's last failure (or of the last failed hl_create when m is NULL). */
const char* hl_last_error(const hl_model* m);

#ifdef __cplusplus
}
#endif

#endif /* HILAYER_H_ */
