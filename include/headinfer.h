/*
 * headinfer.h -- C ABI of libheadinfer.so, the B200-native hot path of HeadInfer
 * (arXiv 2502.12574): causal GQA attention computed one KV head at a time, with
 * every head's K/V cache held in NUMA-local pinned host RAM and streamed to the
 * GPU through ping-pong staging slots.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (section / equation /
 * algorithm named alongside); SURVEY.md §8(b) fixes names and argument order.
 *
 * General conventions (apply to every call below)
 *  - Types: all tensors are bf16 (IEEE bfloat16 bit patterns), row-major, dense.
 *  - Head sharding: a context created with (rank, world) owns the
 *    kv heads [rank*kv_heads/world, (rank+1)*kv_heads/world) and the matching q heads
 *    [rank*q_heads/world, (rank+1)*q_heads/world).  Hkv_loc = kv_heads/world,
 *    Hq_loc = q_heads/world, g = q_heads/kv_heads.  "Local" head indices start at 0.
 *  - GQA (reading R4): local q head j reads local kv head floor(j/g).
 *  - Ownership: the caller owns Q/K/V/out (device pointers on the context's device,
 *    16-byte aligned).  The library owns the host KV store and all device staging and
 *    workspaces, and never retains caller pointers after a call returns.  Every call
 *    is stream-ordered on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *    stream): the library's internal streams wait for the caller's prior work, and
 *    the caller's stream is made to wait for every internal operation that reads a
 *    caller input or writes `out`, so buffers may be reused/freed in stream order.
 *    Calls return as soon as the work is enqueued (no host synchronisation).
 *  - Errors: return codes only, never an abort or exception across the ABI.  Argument
 *    validation happens before any state change (a failed call leaves the context
 *    untouched).  A CUDA error poisons the context ("sticky"): every later call
 *    except hi_free / hi_status_str / hi_last_error returns HI_ECUDA.
 *  - Threading: one host thread per context at a time.  No CPU fallback exists: on a
 *    machine without a usable CUDA device hi_init returns HI_ECUDA.
 */
#ifndef HEADINFER_H_
#define HEADINFER_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hi_ctx hi_ctx; /* opaque; one per (process, GPU) */

typedef enum {
    HI_OK = 0,
    HI_EINVAL = 1,      /* bad configuration: sizes <= 0, q_heads % kv_heads, kv_heads % world, head_dim not 64/128 */
    HI_ESHAPE = 2,      /* bad call shape: layer out of range, n_tokens < 1 or > chunk, NULL pointer */
    HI_ECAPACITY = 3,   /* seq_len[layer] + n would exceed max_ctx ("CapacityExceeded") */
    HI_ENOMEM_HOST = 4, /* host KV store could not be allocated / pinned */
    HI_ENOMEM_DEV = 5,  /* device staging / workspace allocation failed */
    HI_ECUDA = 6,       /* CUDA runtime error (context is now sticky-failed) */
    HI_ESTATE = 7       /* call not valid in the current state */
} hi_status;

/* Advanced options for hi_init_ex (tests and benches); zero-initialise, then set fields.
 * Any field left 0 takes the default shown. */
typedef struct hi_options {
    int n_slots;          /* staging slots per context (default 4, min 2: "ping-pong", Fig. 4) */
    int64_t slot_tokens;  /* tokens per slot and head.  Default: floor(max_ctx/(n_slots*head_group)), so that
                             n_slots*head_group*slot_tokens*4*head_dim <= one head's K+V at max_ctx (Eq. 11
                             P:L235) for every head group, but at least min(max_ctx/2, 32768) (short contexts:
                             fewer, longer copies); multiples of 64.  An explicit value is used as given */
    int device;           /* CUDA device ordinal (default: the current device) */
    int flags;            /* HI_FLAG_* bits */
    int numa_policy;      /* 0 = bind the host store to the GPU's NUMA node (sysfs), 1 = no binding,
                             2 = bind to numa_node */
    int numa_node;        /* used when numa_policy == 2 */
    int resident_kv_heads; /* NEXT-1 (Alg. 1 H_on, l.1 and l.7-8 / l.22-23): the first R (layer,
                              local kv head) pairs in layer-major order keep their whole KV cache in HBM
                              (2*max_ctx*head_dim bf16 each) -- updated in place, never offloaded, attended
                              straight from HBM; the rest are offloaded as usual.  0 (default) = pure head-
                              wise offload; HI_RESIDENT_AUTO = as many pairs as fit in free HBM minus ~12 GiB */
    int head_group;       /* NEXT-2 (§4 "adaptive head-wise offloading"; App. D; Tab. 5-7
                              P:L513-606): kv heads moved and computed per unit (one H2D per block carries
                              `head_group` heads; one kernel launch covers them).  Default 1 = finest
                              head-wise offload; kv_heads/world = layer-wise offload.  With the default
                              slot size the staging ring stays one head's K+V at max_ctx (shorter blocks);
                              with an explicit slot_tokens it grows head_group-fold.  Must divide kv_heads/world, or be
                              HI_GROUP_AUTO (-1): the smallest divisor whose chunk launch fills
                              >= 8 waves of 128-row tiles, staging capped at 1/32 of HBM; or
                              HI_GROUP_PAPER (-2): the paper's schedule by max_ctx (see below). */
    /* NEXT-3 head-wise sparsity (duo-attention, §4; App. D; Tab. "Prefill 1M, Decoding
     * with 1M KV cache" P:L988-1000): streaming_heads points at layers*kv_heads bytes (GLOBAL kv head index,
     * layer-major; the context reads its shard), nonzero = streaming head.  A streaming head is never
     * offloaded: its K/V live in HBM as duo_sink attention-sink rows plus a ring of the duo_window most
     * recent rows ("keep the streaming head in the GPU"), and a query at position p attends exactly
     * the keys i <= p with i < duo_sink or i > p - duo_window (reading R18).  The other (retrieval) heads
     * keep the full cache and are offloaded / resident / grouped as above.  The caller's array is copied.
     * NULL (default) = no streaming heads. */
    const unsigned char* streaming_heads;
    int duo_sink;         /* attention-sink tokens kept by streaming heads: 0 = default 64, < 0 = none */
    int duo_window;       /* recent-window tokens kept by streaming heads (>= 1): 0 = default 256 */
} hi_options;

#define HI_RESIDENT_AUTO (-1)
#define HI_GROUP_AUTO (-1)
#define HI_GROUP_PAPER (-2)  /* head_group: the paper's context-range schedule (§4): max_ctx <= 512K ->
                                all kv heads in one unit, <= 1M -> 2 groups, <= 2M -> 4, else 8 groups (bounds
                                2^19/2^20/2^21 plus a 64K-token decode tail); a unit is kv_heads/groups heads,
                                capped at this shard's kv heads */

#define HI_FLAG_POISON_SLOTS 0x1 /* fill each staging slot with NaN before every H2D (race detection) */
#define HI_FLAG_NO_HUGEPAGE 0x2  /* do not madvise(MADV_HUGEPAGE) the host store */
#define HI_FLAG_SERIALIZE 0x4    /* synchronise after every internal step (debug; destroys overlap) */
#define HI_FLAG_TIMING 0x8       /* bracket every attention kernel launch with timing events on the
                                    compute stream; durations are summed into hi_stats at the next
                                    hi_synchronize / hi_get_stats (bench roofline evidence) */
/* Comparison prefill kernels (A/B measurements only; csrc/variants/).  They exist only in the variants
 * build (build.build_variant, HI_LIB_VARIANT); the product libheadinfer.so rejects these flags with HI_EINVAL. */
#define HI_FLAG_PREFILL_2CTA 0x20     /* head_dim 128: the CTA-pair (cta_group::2, M = 256) tcgen05 prefill kernel
                                         instead of the single-CTA one (measured slower) */
#define HI_FLAG_PREFILL_TC1 0x40      /* the one-tile / three-S-buffer tcgen05 prefill kernel (measured slower) */
#define HI_FLAG_JITTER 0x80     /* hazard testing: before every history H2D block, write-back D2H and
                                   attention launch, hold that stream for a pseudo-random 0-200 us (counter hash);
                                   outputs must be bit-identical to a run without it */
#define HI_FLAG_FAULT_SKIP_RAW 0x100 /* NEGATIVE CONTROL, tests only: drop the compute stream's wait on each landed
                                        staging block (the RAW edge of Alg. 1 l.10/13) and delay the H2D stream by
                                        2 ms per block, so attention reads slots before their bytes land; parity
                                        must FAIL (proves the tests see a missing dependency) */
#define HI_FLAG_FAULT_SKIP_BLOCK 0x800 /* NEGATIVE CONTROL, tests only: prefill skips the attention launch over the
                                          FIRST history block of every offloaded unit (when a call has >= 2 blocks);
                                          the parity bar (relative L2 per q head) must FAIL where the absolute bounds
                                          alone cannot see it (near-uniform attention at long context) */
#define HI_FLAG_PREFILL_PSMEM 0x1000   /* variants build only: the prefill kernel with P staged in shared memory
                                          (variants/k_prefill_tcp.cu): S(j+1) overlaps the softmax of S(j); parity-green
                                          but 18 % slower per launch (measured; the SS PV MMA doubles shared-memory reads) */
#define HI_FLAG_FAULT_LAUNCH 0x200   /* FAULT INJECTION, tests only: the second hi_prefill_chunk / hi_decode call of the
                                        context makes a kernel launch with an invalid configuration (a synchronous
                                        CUDA error; the CUDA context survives), so the context must turn sticky */
#define HI_FLAG_FAULT_TRAP 0x400     /* FAULT INJECTION, tests only: as above, but the injected kernel executes `trap`
                                        (an asynchronous device fault that loses the process's CUDA context) */
#define HI_FLAG_MMA_SYNC_PREFILL 0x10 /* variants build only: prefill attention on the legacy mma.sync kernel
                                         instead of the tcgen05/TMEM/TMA kernel (baseline comparator) */

typedef struct hi_stats {
    int64_t host_store_bytes;     /* pinned host KV bytes (L * Hkv_loc * max_ctx * 4 * d) */
    int64_t staging_bytes;        /* device staging slots, total */
    int64_t staging_bound_bytes;  /* default slot size: one head at max_ctx, 4*d*max_ctx (Eq. 11, reading R8),
                                     unless the minimum block length makes the ring larger (short contexts);
                                     explicit slot_tokens: head_group heads at max_ctx */
    int64_t workspace_bytes;      /* other device buffers (pack, accumulators, partials) */
    int64_t h2d_bytes;            /* cumulative history bytes streamed host->device */
    int64_t d2h_bytes;            /* cumulative new-K/V bytes written back device->host */
    int64_t prefill_calls, decode_calls;
    int64_t kernel_launches;      /* cumulative launches of this library's kernels */
    /* HI_FLAG_TIMING only: attention kernels, device time from CUDA events on the compute stream */
    double prefill_attn_ms;       /* summed duration of prefill attention launches */
    double prefill_attn_flops;    /* their algorithmic FLOPs: 4*d*g*(visible (query,key) pairs) */
    int64_t prefill_attn_launches;
    double decode_attn_ms;        /* summed duration of decode split-K partial launches */
    double decode_attn_bytes;     /* their algorithmic HBM bytes: 4*d per key read */
    int64_t decode_attn_launches;
    double init_seconds;          /* wall time of hi_init (host pinning dominates) */
    int numa_node;                /* node the host store is bound to (-1: none / unknown) */
    int n_slots;
    int64_t slot_tokens;
    int resident_kv_heads;        /* H_on pairs held in HBM (NEXT-1) */
    int64_t resident_bytes;       /* their device KV bytes */
    int head_group;               /* kv heads per offload unit (NEXT-2) */
    int streaming_kv_heads;       /* local (layer, kv head) pairs that are duo streaming heads (NEXT-3) */
    int64_t streaming_bytes;      /* their device sink + window KV bytes */
    /* HI_FLAG_TIMING only: copy-engine busy time, from CUDA events on the copy streams around each
     * history block's H2D (§8(a) a3/a7) and each prefill write-back's D2H (a2) */
    double h2d_copy_ms;
    double d2h_copy_ms;
} hi_stats;

/*
 * hi_init -- pre-allocate everything (Alg. 1 lines 1-2; "pre-allocates the
 * CPU's KV cache memory and the GPU's ping-pong memory", §4).
 *   layers, q_heads, kv_heads, head_dim: model shape (head_dim in {64,128}).
 *   max_ctx: tokens per (layer, kv head) the host store holds (Eq. 4 P:L169 sizes it).
 *   chunk:   largest n_tokens a hi_prefill_chunk call may pass (§3.3 chunked prefill).
 *   rank, world: head shard (see conventions).  *out receives the handle (NULL on failure).
 * Host store: one contiguous K region and one V region of max_ctx*head_dim bf16 per
 * (layer, local kv head) (Eq. 7-8: "each head stores its keys and values in a
 * contiguous memory space"), mmap'd, bound to the GPU's NUMA node, pinned.
 * Errors: HI_EINVAL, HI_ENOMEM_HOST, HI_ENOMEM_DEV, HI_ECUDA (e.g. no GPU).
 */
hi_status hi_init(int layers, int q_heads, int kv_heads, int head_dim, int64_t max_ctx, int chunk,
                  int rank, int world, hi_ctx** out);
hi_status hi_init_ex(int layers, int q_heads, int kv_heads, int head_dim, int64_t max_ctx, int chunk,
                     int rank, int world, const hi_options* opt, hi_ctx** out);

/*
 * hi_prefill_chunk -- one chunk of the prefill phase for one layer (Alg. 1 lines 3-17,
 * P:L316-333): for every local kv head h, write the chunk's K/V of head h back to host
 * rows [s, s+n) (line 11 "Async Update CPU KV cache", delta write-back, reading R7),
 * stream head h's history rows [0, s) in through the staging slots (line 10 "Async
 * Prefetch"), and compute causal attention (line 13, Eq. 9) for the g q heads of
 * the group over history + chunk; outputs land in their q-head columns of `out`
 * (line 15 "Concatenate").  s = hi_seq_len(layer) before the call; it advances by n.
 *   Q   [n_tokens, Hq_loc, head_dim]   bf16 device, q heads of this shard, global positions s..s+n-1
 *   K,V [n_tokens, Hkv_loc, head_dim]  bf16 device
 *   out [n_tokens, Hq_loc, head_dim]   bf16 device (written)
 *   n_tokens in [1, chunk]; the last chunk may be partial (reading R11).
 * Errors: HI_ESHAPE, HI_ECAPACITY, HI_ECUDA, HI_ESTATE.
 */
hi_status hi_prefill_chunk(hi_ctx* ctx, int layer, const void* Q, const void* K, const void* V, void* out,
                           int n_tokens, void* cuda_stream);

/*
 * hi_decode -- one generated token for one layer (Alg. 1 lines 18-32): append
 * k, v at position s (host row s, D2H) and attend q to keys 0..s, the new key included
 * (reading R3), streaming each head's history [0, s) through the slots; split-K partials
 * merged by log-sum-exp.  s advances by 1.  s = 0 is allowed (out = v).
 *   q [Hq_loc, head_dim], k, v [Hkv_loc, head_dim], out [Hq_loc, head_dim]: bf16 device.
 * Errors: HI_ESHAPE, HI_ECAPACITY, HI_ECUDA, HI_ESTATE.
 */
hi_status hi_decode(hi_ctx* ctx, int layer, const void* q, const void* k, const void* v, void* out,
                    void* cuda_stream);

/* hi_free -- synchronise, unpin and release everything.  NULL is a no-op (HI_OK). */
hi_status hi_free(hi_ctx* ctx);

/* ---- verification / introspection / bench preparation (not on the hot path) ---- */

/* Copy KV rows [pos, pos+n) of (layer, local kv head) into host buffers k_dst, v_dst ([n, head_dim]
 * bf16 each) from wherever they live (host store, or HBM for resident pairs).  Waits for pending
 * write-backs first.  HI_ESHAPE on bad range.  Streaming heads (NEXT-3) hold only rows p < duo_sink and
 * the last duo_window rows below seq_len; asking for any other row is HI_ESTATE. */
hi_status hi_read_host_kv(hi_ctx* ctx, int layer, int kv_head_local, int64_t pos, int64_t n,
                          void* k_dst, void* v_dst);

/* Write host KV rows [pos, pos+n) of (layer, local kv head) from k_src, v_src ([n, head_dim]
 * bf16 each; device pointers if from_device != 0, else host).  Synchronous; with a device source, all
 * work already enqueued on the device (any stream) completes before the copy reads it.  Does not move
 * seq_len.  For a streaming head (NEXT-3) rows p < duo_sink go to its sink and rows p >= duo_sink to its
 * window ring (only the last duo_window of the range are kept).  This is the "helper for simulating or preparing decoding with large context"
 * (App. E): benches fill a long history without timing a full prefill. */
hi_status hi_write_host_kv(hi_ctx* ctx, int layer, int kv_head_local, int64_t pos, int64_t n,
                           const void* k_src, const void* v_src, int from_device);

/* seq_len[layer]: tokens cached for `layer` (all local kv heads share it).  -1 on bad args. */
int64_t hi_seq_len(const hi_ctx* ctx, int layer);

/* Set seq_len[layer] = s (0 <= s <= max_ctx).  Rows below s are taken as valid history;
 * used to rewind a bench to an earlier position (host history is immutable, so re-running
 * a chunk rewrites identical bytes).  Waits for in-flight work of the context. */
hi_status hi_set_seq_len(hi_ctx* ctx, int layer, int64_t s);

/* Snapshot of counters; waits for in-flight work of the context.  On a sticky-failed context the counters
 * are still filled in (without waiting) and the call returns HI_ECUDA. */
hi_status hi_get_stats(hi_ctx* ctx, hi_stats* out);

/* Blocks until all work the context enqueued has finished. */
hi_status hi_synchronize(hi_ctx* ctx);

const char* hi_status_str(hi_status s);

/* Message describing the last failure on this context (or of the last failed hi_init when
 * ctx is NULL).  Never NULL. */
const char* hi_last_error(const hi_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* HEADINFER_H_ */
