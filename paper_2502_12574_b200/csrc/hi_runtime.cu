// hi_runtime.cu -- host runtime of libheadinfer.so: the C ABI declared in include/headinfer.h.
//
// Subsystems (SURVEY.md §1 "The build", 2(a)-(f)):
//  (a) host KV store   -- one contiguous K and V region per (layer, local kv head) (Eq. 7-8,
//                         P:L203-213), mmap'd, NUMA-bound to the GPU's node, first-touched in
//                         parallel, pinned with cudaHostRegister (pre-allocation, §4).
//  (b) staging pool    -- n_slots device slots, each [slot_tokens][d] K + [slot_tokens][d] V,
//                         n_slots*slot_tokens <= max_ctx: at most one head's K/V resident
//                         (Eq. 10-11; the ping-pong memory of Fig. 4).
//  (c) copy engine     -- dedicated H2D and D2H streams; every slot hand-off is an event
//                         (slot_ready: H2D -> compute, slot_free: compute -> H2D), so H2D of
//                         head h+1, D2H of the chunk and compute on head h run concurrently,
//                         full duplex (§4; App. D).
//  (d) scheduler       -- per call: pack + write-back, then per kv head the chunk's own
//                         (causal) segment first -- it needs no transfer -- followed by the
//                         history blocks in landing order; the host only enqueues (never
//                         blocks), so the copy stream runs ahead across heads and layers.
//  (e) kernels         -- k_prefill_*.cu, k_decode.cu, k_pack.cu.
//  (f) stats + errors  -- status codes, sticky CUDA failure, hi_stats counters.
#include "../../include/headinfer.h"
#include "hi_kernels.cuh"

#include <cuda_runtime.h>
#include <errno.h>
#include <nvtx3/nvToolsExt.h>
#include <linux/mempolicy.h>
#include <math.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_init_error = "no error";

enum TimedKind { T_DECODE = 0, T_PREFILL = 1, T_H2D = 2, T_D2H = 3 };
struct TimedLaunch {
    cudaEvent_t start, stop;
    double work;   // algorithmic FLOPs (prefill), bytes (decode kernel) or bytes copied (H2D / D2H)
    int kind;      // TimedKind
};

struct Slot {
    cudaEvent_t ready = nullptr;  // recorded on the H2D stream after the block landed
    cudaEvent_t free_ = nullptr;  // recorded on the compute stream after its consumer kernel
};

}  // namespace

struct hi_ctx {
    // configuration
    int L = 0, Hq = 0, Hkv = 0, d = 0, chunk = 0, rank = 0, world = 1;
    int Hq_loc = 0, Hkv_loc = 0, g = 0, device = 0, flags = 0;
    int64_t max_ctx = 0;
    float scale_log2 = 0.f;
    // state
    std::vector<int64_t> seq_len;
    bool sticky = false;
    std::string err = "no error";
    // (a) host KV store (offloaded pairs) + device-resident KV cache (H_on pairs, NEXT-1).  Pairs are numbered
    // over the RETRIEVAL (layer, kv head) pairs only, layer-major (cidx); duo streaming pairs (NEXT-3) get -1.
    std::vector<int> cidx;             // [L*Hkv_loc]
    int n_retr = 0;                    // retrieval pairs
    int n_res = 0;                     // retrieval pairs with cidx < n_res stay in HBM
    uint8_t* d_res = nullptr;
    size_t res_bytes = 0;
    uint8_t* host = nullptr;
    size_t host_bytes = 0;
    size_t host_map_bytes = 0;
    bool host_registered = false;
    int numa_node = -1;
    // (b) staging
    int n_slots = 0;
    int64_t slot_tokens = 0;
    bool slot_default = true;   // slot_tokens chosen by hi_init: the ring holds <= one head at max_ctx
    size_t slot_bytes = 0;
    int group = 1;                     // NEXT-2: kv heads per transfer + kernel unit (slot holds `group` heads)
    uint8_t* d_stage = nullptr;
    std::vector<Slot> slots;
    int next_slot = 0;
    // (c) streams + events
    cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_call_in = nullptr, ev_call_out = nullptr, ev_packed = nullptr, ev_pack_free = nullptr;
    std::vector<cudaEvent_t> ev_layer_d2h;   // last write-back of each layer's rows
    std::vector<cudaEvent_t> ev_kvnew_free;  // decode: kvnew[layer] read by its D2H
    // workspaces
    __nv_bfloat16* d_pack = nullptr;   // [Hkv_loc][2][chunk][d]
    float* d_oacc = nullptr;           // [group][chunk*g][d]
    float* d_macc = nullptr;           // [group][chunk*g]
    float* d_lacc = nullptr;           // [group][chunk*g]
    float* d_parts = nullptr;          // [Hkv_loc][max_parts][g][d+4]
    int max_parts = 0;
    __nv_bfloat16* d_kvnew = nullptr;  // [L][2][Hkv_loc][d]
    unsigned* d_counters = nullptr;    // [Hkv_loc] fused decode combine completion counters (self-resetting)
    size_t workspace_bytes = 0;
    // NEXT-3 duo streaming heads: per (layer, kv head) a device block [K: duo_rows x d | V: duo_rows x d],
    // rows [0, duo_sink) = sink positions, rows duo_sink + (p - duo_sink) % duo_ring = the recent window
    int duo_sink = 0, duo_win = 0, duo_ring = 0, n_stream = 0;
    int64_t duo_rows = 0;
    uint8_t* d_duo = nullptr;
    size_t duo_bytes = 0;
    // per-layer head lists (local kv heads, ascending): resident retrieval, offload units, streaming
    std::vector<std::vector<int>> res_heads, str_heads;
    std::vector<std::vector<std::vector<int>>> off_units;
    // (f) stats
    int64_t h2d_bytes = 0, d2h_bytes = 0, prefill_calls = 0, decode_calls = 0, launches = 0;
    uint64_t jitter_ctr = 0;   // HI_FLAG_JITTER: counter of the delay hash
    double init_seconds = 0.0;
    // HI_FLAG_TIMING
    std::vector<TimedLaunch> timed;
    std::vector<cudaEvent_t> ev_pool;
    double prefill_ms = 0, prefill_flops = 0, decode_ms = 0, decode_bytes = 0, h2d_ms = 0, d2h_ms = 0;
    int64_t prefill_timed = 0, decode_timed = 0;

    size_t pair(int layer, int h) const { return static_cast<size_t>(cidx[static_cast<size_t>(layer) * Hkv_loc + h]); }
    bool streaming(int layer, int h) const { return cidx[static_cast<size_t>(layer) * Hkv_loc + h] < 0; }
    bool resident(int layer, int h) const { return !streaming(layer, h) && pair(layer, h) < static_cast<size_t>(n_res); }
    uint8_t* host_k(int layer, int h, int64_t row) const {
        return host + ((pair(layer, h) - n_res) * 2 + 0) * static_cast<size_t>(max_ctx) * d * 2 +
               static_cast<size_t>(row) * d * 2;
    }
    uint8_t* host_v(int layer, int h, int64_t row) const {
        return host + ((pair(layer, h) - n_res) * 2 + 1) * static_cast<size_t>(max_ctx) * d * 2 +
               static_cast<size_t>(row) * d * 2;
    }
    uint8_t* dev_k(int layer, int h, int64_t row) const {
        return d_res + (pair(layer, h) * 2 + 0) * static_cast<size_t>(max_ctx) * d * 2 + static_cast<size_t>(row) * d * 2;
    }
    uint8_t* dev_v(int layer, int h, int64_t row) const {
        return d_res + (pair(layer, h) * 2 + 1) * static_cast<size_t>(max_ctx) * d * 2 + static_cast<size_t>(row) * d * 2;
    }
    // streaming head block: [K rows | V rows], duo_rows each
    size_t duo_head_elems() const { return static_cast<size_t>(2) * duo_rows * d; }
    __nv_bfloat16* duo_k(int layer, int h, int64_t row) const {
        return reinterpret_cast<__nv_bfloat16*>(d_duo) + (static_cast<size_t>(layer) * Hkv_loc + h) * duo_head_elems() +
               static_cast<size_t>(row) * d;
    }
    int64_t duo_row(int64_t pos) const { return pos < duo_sink ? pos : duo_sink + (pos - duo_sink) % duo_ring; }
    // where the KV rows of (layer, h) live: device cache (resident) or host store (offloaded)
    uint8_t* kv_k(int layer, int h, int64_t row) const { return resident(layer, h) ? dev_k(layer, h, row) : host_k(layer, h, row); }
    uint8_t* kv_v(int layer, int h, int64_t row) const { return resident(layer, h) ? dev_v(layer, h, row) : host_v(layer, h, row); }
    // slot s holds `group` heads, each [K: slot_tokens x d | V: slot_tokens x d]
    size_t slot_head_bytes() const { return static_cast<size_t>(slot_tokens) * d * 2 * 2; }
    uint8_t* slot_k(int s, int gh = 0) const { return d_stage + static_cast<size_t>(s) * slot_bytes + gh * slot_head_bytes(); }
    uint8_t* slot_v(int s, int gh = 0) const { return slot_k(s, gh) + static_cast<size_t>(slot_tokens) * d * 2; }
};

namespace {

hi_status fail_cuda(hi_ctx* c, cudaError_t e, const char* what) {
    c->sticky = true;
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    c->err = buf;
    return HI_ECUDA;
}

#define HI_CK(ctx, call)                                     \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return fail_cuda(ctx, e_, #call); \
    } while (0)

hi_status set_err(hi_ctx* c, hi_status s, const char* msg) {
    if (c) c->err = msg;
    return s;
}

int gpu_numa_node(int device) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
    for (char* p = bus; *p; ++p) *p = static_cast<char>(tolower(*p));
    char path[256];
    snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
    FILE* f = fopen(path, "r");
    if (!f) return -1;
    int node = -1;
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
    return node;
}

int numa_node_count() {
    int n = 0;
    for (int i = 0; i < 1024; ++i) {
        char path[128];
        snprintf(path, sizeof path, "/sys/devices/system/node/node%d", i);
        if (access(path, F_OK) == 0) ++n;
        else if (i > 64) break;
    }
    return n;
}

// (a) host KV store: mmap + THP + mbind + parallel first touch + cudaHostRegister
hi_status alloc_host_store(hi_ctx* c, int numa_policy, int numa_node_req) {
    const size_t huge = 2u << 20;
    if (c->host_bytes == 0) return HI_OK;  // every pair resident in HBM
    c->host_map_bytes = (c->host_bytes + huge - 1) / huge * huge;
    void* p = mmap(nullptr, c->host_map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) return set_err(c, HI_ENOMEM_HOST, "mmap of the host KV store failed");
    c->host = static_cast<uint8_t*>(p);
    if (!(c->flags & HI_FLAG_NO_HUGEPAGE)) madvise(p, c->host_map_bytes, MADV_HUGEPAGE);
    int node = -1;
    if (numa_policy == 0) node = gpu_numa_node(c->device);
    else if (numa_policy == 2) node = numa_node_req;
    if (node >= 0 && numa_node_count() > 1 && node < 1024) {
        unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
        mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
        if (syscall(SYS_mbind, p, c->host_map_bytes, MPOL_BIND, mask, 1024, 0) == 0) c->numa_node = node;
    } else if (node >= 0) {
        c->numa_node = node;  // single node: already local
    }
    // parallel first touch (faults pages in on the bound node before pinning)
    unsigned nthr = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t per = (c->host_map_bytes / nthr + huge - 1) / huge * huge;
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nthr; ++i) {
        const size_t b = i * per;
        if (b >= c->host_map_bytes) break;
        const size_t e = std::min(c->host_map_bytes, b + per);
        th.emplace_back([=] {
            for (size_t o = b; o < e; o += 4096) c->host[o] = 0;
        });
    }
    for (auto& t : th) t.join();
    cudaError_t e = cudaHostRegister(p, c->host_map_bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[256];
        snprintf(buf, sizeof buf, "cudaHostRegister of %zu bytes failed: %s", c->host_map_bytes, cudaGetErrorString(e));
        return set_err(c, e == cudaErrorMemoryAllocation ? HI_ENOMEM_HOST : HI_ECUDA, buf);
    }
    c->host_registered = true;
    return HI_OK;
}

void destroy(hi_ctx* c) {
    if (!c) return;
    hi::DeviceGuard dg(c->device);
    if (c->s_comp) cudaStreamSynchronize(c->s_comp);
    if (c->s_h2d) cudaStreamSynchronize(c->s_h2d);
    if (c->s_d2h) cudaStreamSynchronize(c->s_d2h);
    for (auto& s : c->slots) {
        if (s.ready) cudaEventDestroy(s.ready);
        if (s.free_) cudaEventDestroy(s.free_);
    }
    for (auto& t : c->timed) { cudaEventDestroy(t.start); cudaEventDestroy(t.stop); }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto e : c->ev_layer_d2h) if (e) cudaEventDestroy(e);
    for (auto e : c->ev_kvnew_free) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->ev_call_in, c->ev_call_out, c->ev_packed, c->ev_pack_free})
        if (e) cudaEventDestroy(e);
    for (cudaStream_t s : {c->s_comp, c->s_h2d, c->s_d2h})
        if (s) cudaStreamDestroy(s);
    cudaFree(c->d_stage);
    cudaFree(c->d_pack);
    cudaFree(c->d_oacc);
    cudaFree(c->d_macc);
    cudaFree(c->d_lacc);
    cudaFree(c->d_parts);
    cudaFree(c->d_kvnew);
    cudaFree(c->d_counters);
    cudaFree(c->d_res);
    cudaFree(c->d_duo);
    if (c->host) {
        if (c->host_registered) cudaHostUnregister(c->host);
        munmap(c->host, c->host_map_bytes);
    }
    cudaGetLastError();
    delete c;
}

// Split length for the decode partial kernel (one 160-thread CTA per SM, TMA-fed 6-stage ring): about
// two waves of CTAs in total over the launch's `heads` kv heads, each CTA streaming one long contiguous
// key range (a deep ring pays off only over many stages); at least 64 keys (one stage) per CTA.
#ifndef HI_DECODE_WAVES
#define HI_DECODE_WAVES 3  // resident 1M decode: 1 wave 27.4 ms, 2 waves 22.6, 3 waves 21.2, 4 waves 21.4 (profiles/decode_waves_r02.txt)
#endif
// Offloaded history blocks are decoded while the NEXT block crosses the host link (~100x slower than HBM), so
// their launches need no more than one wave: fewer, longer CTAs amortise the ring's fill and the launch ramp.
constexpr int kOffloadDecodeWaves = 1;
int decode_split_len(int64_t nk, int heads = 1, int waves = HI_DECODE_WAVES) {
    const int64_t target = std::max<int64_t>(1, (waves * 148) / heads);   // never a partial extra wave
    int64_t s = (nk + target - 1) / target;
    s = (s + 63) / 64 * 64;
    return static_cast<int>(std::max<int64_t>(64, std::min<int64_t>(s, 1 << 30)));
}
int64_t decode_parts_for_block(int64_t nk) {
    const int sl = decode_split_len(nk);
    return (nk + sl - 1) / sl;
}

// Visible (query, key) pairs of one prefill segment (the launch's algorithmic work, HI_FLAG_TIMING): token t
// (position q_pos0 + t) sees key position k in [k_pos0, k_pos0 + n_k) iff (not causal or k <= p) and
// (win <= 0 or k > p - win).
double seg_pairs(int64_t q_pos0, int n, int64_t k_pos0, int64_t n_k, bool causal, int win) {
    if (!causal && win <= 0) return static_cast<double>(n) * static_cast<double>(n_k);
    double tot = 0.0;
    for (int t = 0; t < n; ++t) {
        const int64_t p = q_pos0 + t;
        const int64_t hi = causal ? std::min(k_pos0 + n_k - 1, p) : k_pos0 + n_k - 1;
        const int64_t lo = win > 0 ? std::max(k_pos0, p - win + 1) : k_pos0;
        if (hi >= lo) tot += static_cast<double>(hi - lo + 1);
    }
    return tot;
}

cudaError_t launch_prefill(hi_ctx* c, const hi::PrefillParams& p) {
#ifdef HI_WITH_VARIANTS
    // comparison kernels (csrc/variants/, built only into the variants library): single-head launches
    const bool mma = c->flags & HI_FLAG_MMA_SYNC_PREFILL;
    const bool pair = !mma && c->d == 128 && (c->flags & HI_FLAG_PREFILL_2CTA);
    if (mma || pair || (c->flags & HI_FLAG_PREFILL_TC1)) {
        for (int h = 0; h < std::max(1, p.n_heads); ++h) {
            hi::PrefillParams q1 = p;
            q1.n_heads = 1;
            q1.q = p.q + static_cast<int64_t>(p.head_q[h]) * p.g * c->d;
            q1.out = p.out + static_cast<int64_t>(p.head_q[h]) * p.g * c->d;
            q1.k = p.k + p.head_kv[h] * p.kv_head_stride;
            q1.v = p.v + p.head_kv[h] * p.kv_head_stride;
            q1.o_acc = p.o_acc + h * p.state_rows * c->d;
            q1.m_acc = p.m_acc + h * p.state_rows;
            q1.l_acc = p.l_acc + h * p.state_rows;
            hi::set_identity_heads(q1, 1);
            const cudaError_t e = mma ? hi::launch_prefill_mma(q1, c->d, c->s_comp)
                                  : pair ? hi::launch_prefill_tc2(q1, c->d, c->s_comp)
                                         : hi::launch_prefill_tc1(q1, c->d, c->s_comp);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
#endif
#ifdef HI_WITH_VARIANTS
    // comparison kernel with P staged in shared memory (variants/k_prefill_tcp.cu), every head in one launch
#ifndef HI_PSMEM_DEFAULT
#define HI_PSMEM_DEFAULT 0
#endif
    if (HI_PSMEM_DEFAULT || (c->flags & HI_FLAG_PREFILL_PSMEM)) return hi::launch_prefill_tcp(p, c->d, c->s_comp);
#endif
    // the product kernel: every head of the unit in one launch (grid.y, head maps)
    return hi::launch_prefill_tc(p, c->d, c->s_comp);
}

hi_status check_call(hi_ctx* c, int layer) {
    if (!c) return HI_ESHAPE;
    if (c->sticky) return HI_ECUDA;
    if (layer < 0 || layer >= c->L) return set_err(c, HI_ESHAPE, "layer out of range");
    return HI_OK;
}

cudaEvent_t pool_event(hi_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}

// Bracket a kernel launch (compute stream) or a batch of copies (a copy stream) with timing events when
// HI_FLAG_TIMING is set.  On a copy stream the start event is recorded after the stream's waits, so the
// elapsed time is the copy engine's busy time for those bytes.
struct LaunchTimer {
    hi_ctx* c;
    cudaStream_t st;
    cudaEvent_t start = nullptr;
    LaunchTimer(hi_ctx* ctx, cudaStream_t s = nullptr) : c(ctx), st(s ? s : ctx->s_comp) {
        if (c->flags & HI_FLAG_TIMING) {
            start = pool_event(c);
            if (start) cudaEventRecord(start, st);
        }
    }
    void done(double work, int kind) {
        if (!start) return;
        cudaEvent_t stop = pool_event(c);
        if (!stop) return;
        cudaEventRecord(stop, st);
        c->timed.push_back({start, stop, work, kind});
    }
};

// NVTX range over the host-side enqueue of a call or a staged block (tracing): visible in
// Nsight Systems / ncu --nvtx; header-only NVTX v3, a no-op when no tool is attached.
struct NvtxRange {
    template <typename... A>
    explicit NvtxRange(const char* fmt, A... a) {
        char buf[96];
        snprintf(buf, sizeof(buf), fmt, a...);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
};

// The copies of one step (a history block of `group` heads, a write-back, a decode append) are collected
// here and issued as plain stream-ordered cudaMemcpyAsync calls; a copy whose source and destination both
// continue the previous one is merged into it, so adjacent heads' rows go to the copy engine as one transfer.
struct CopyBatch {
    std::vector<void*> dst, src;
    std::vector<size_t> size;
    void add(void* d, const void* s_, size_t n) {
        if (!dst.empty() && static_cast<char*>(dst.back()) + size.back() == static_cast<char*>(d) &&
            static_cast<const char*>(src.back()) + size.back() == static_cast<const char*>(s_)) {
            size.back() += n;
            return;
        }
        dst.push_back(d);
        src.push_back(const_cast<void*>(s_));
        size.push_back(n);
    }
    // A run of equal-size copies whose sources and destinations each advance by a constant pitch (the K and V
    // rows of consecutive heads: host pitch max_ctx rows, slot pitch slot_tokens rows) is one cudaMemcpy2DAsync.
    cudaError_t issue(cudaStream_t st) {
        size_t i = 0;
        while (i < dst.size()) {
            size_t j = i + 1;
            if (j < dst.size() && size[j] == size[i]) {
                const ptrdiff_t dp = static_cast<char*>(dst[j]) - static_cast<char*>(dst[i]);
                const ptrdiff_t sp = static_cast<char*>(src[j]) - static_cast<char*>(src[i]);
                if (dp >= static_cast<ptrdiff_t>(size[i]) && sp >= static_cast<ptrdiff_t>(size[i])) {
                    while (j < dst.size() && size[j] == size[i] &&
                           static_cast<char*>(dst[j]) - static_cast<char*>(dst[j - 1]) == dp &&
                           static_cast<char*>(src[j]) - static_cast<char*>(src[j - 1]) == sp)
                        ++j;
                    cudaError_t e = cudaMemcpy2DAsync(dst[i], dp, src[i], sp, size[i], j - i, cudaMemcpyDefault, st);
                    if (e == cudaSuccess) {
                        i = j;
                        continue;
                    }
                    (void)cudaGetLastError();  // pitch out of range: fall back to one copy each
                    j = i + 1;
                }
            }
            for (; i < j; ++i) {
                cudaError_t e = cudaMemcpyAsync(dst[i], src[i], size[i], cudaMemcpyDefault, st);
                if (e != cudaSuccess) return e;
            }
        }
        return cudaSuccess;
    }
};

// HI_FLAG_JITTER: hold `s` for a pseudo-random 0-200 us (splitmix64 of a per-context counter), so the three
// streams complete in orders a plain run never produces; every dependency is an event, so outputs must not change.
hi_status jitter(hi_ctx* c, cudaStream_t s) {
    if (!(c->flags & HI_FLAG_JITTER)) return HI_OK;
    uint64_t z = (++c->jitter_ctr) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    HI_CK(c, hi::launch_spin(z % 200000, s));
    ++c->launches;
    return HI_OK;
}

// Enqueue the H2D of history block [k0, k0+nk) of the kv heads `heads` of `layer` into the next slot (head
// heads[gh] at slot position gh); the compute stream is made to wait for it.  Returns the slot through *slot_out.
hi_status stage_block(hi_ctx* c, int layer, const std::vector<int>& heads, int64_t k0, int64_t nk, int* slot_out) {
    const int nh = static_cast<int>(heads.size());
    const int s = c->next_slot;
    c->next_slot = (c->next_slot + 1) % c->n_slots;
    Slot& sl = c->slots[s];
    HI_CK(c, cudaStreamWaitEvent(c->s_h2d, sl.free_, 0));  // WAR: previous consumer of this slot done
    if (hi_status js = jitter(c, c->s_h2d); js != HI_OK) return js;
    if (c->flags & HI_FLAG_FAULT_SKIP_RAW) {  // negative control: the block lands 2 ms late
        HI_CK(c, hi::launch_spin(2000000, c->s_h2d));
        ++c->launches;
    }
    if (c->flags & HI_FLAG_POISON_SLOTS) {
        HI_CK(c, hi::launch_poison(c->slot_k(s), c->slot_bytes, c->s_h2d));
        ++c->launches;
    }
    const size_t bytes = static_cast<size_t>(nk) * c->d * 2;
    NvtxRange nr("hi H2D layer %d heads %d+%d keys [%lld, %lld)", layer, heads[0], nh, static_cast<long long>(k0),
                 static_cast<long long>(k0 + nk));
    LaunchTimer tm(c, c->s_h2d);
    CopyBatch cb;
    for (int gh = 0; gh < nh; ++gh) {
        cb.add(c->slot_k(s, gh), c->host_k(layer, heads[gh], k0), bytes);
        cb.add(c->slot_v(s, gh), c->host_v(layer, heads[gh], k0), bytes);
    }
    HI_CK(c, cb.issue(c->s_h2d));
    tm.done(static_cast<double>(2 * bytes) * nh, T_H2D);
    HI_CK(c, cudaEventRecord(sl.ready, c->s_h2d));
    if (!(c->flags & HI_FLAG_FAULT_SKIP_RAW))
        HI_CK(c, cudaStreamWaitEvent(c->s_comp, sl.ready, 0));  // RAW: block landed
    c->h2d_bytes += static_cast<int64_t>(2 * bytes) * nh;
    *slot_out = s;
    return HI_OK;
}

// HI_FLAG_FAULT_LAUNCH / HI_FLAG_FAULT_TRAP (tests): the context's second prefill/decode call injects a CUDA error
hi_status inject_fault(hi_ctx* c) {
    if (!(c->flags & (HI_FLAG_FAULT_LAUNCH | HI_FLAG_FAULT_TRAP)) || c->prefill_calls + c->decode_calls != 1)
        return HI_OK;
    HI_CK(c, hi::launch_fault(c->flags & HI_FLAG_FAULT_TRAP, c->s_comp));
    ++c->launches;
    return HI_OK;
}

hi_status release_slot(hi_ctx* c, int s) {
    HI_CK(c, cudaEventRecord(c->slots[s].free_, c->s_comp));
    return HI_OK;
}

void resolve_timing(hi_ctx* c) {
    for (auto& t : c->timed) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, t.start, t.stop) == cudaSuccess) {
            switch (t.kind) {
                case T_PREFILL: c->prefill_ms += ms; c->prefill_flops += t.work; ++c->prefill_timed; break;
                case T_DECODE: c->decode_ms += ms; c->decode_bytes += t.work; ++c->decode_timed; break;
                case T_H2D: c->h2d_ms += ms; break;
                default: c->d2h_ms += ms; break;
            }
        }
        c->ev_pool.push_back(t.start);
        c->ev_pool.push_back(t.stop);
    }
    c->timed.clear();
    cudaGetLastError();
}

hi_status finish_call(hi_ctx* c, cudaStream_t cs) {
    HI_CK(c, cudaEventRecord(c->ev_call_out, c->s_comp));
    HI_CK(c, cudaStreamWaitEvent(cs, c->ev_call_out, 0));
    if (c->flags & HI_FLAG_SERIALIZE) HI_CK(c, cudaDeviceSynchronize());
    return HI_OK;
}

}  // namespace

bool hi::ctx_info(const hi_ctx* c, hi::CtxInfo* o) {
    if (!c || !o) return false;
    *o = {c->L, c->Hq_loc, c->Hkv_loc, c->d, c->chunk, c->world, c->device};
    return true;
}

extern "C" {

const char* hi_status_str(hi_status s) {
    switch (s) {
        case HI_OK: return "HI_OK";
        case HI_EINVAL: return "HI_EINVAL";
        case HI_ESHAPE: return "HI_ESHAPE";
        case HI_ECAPACITY: return "HI_ECAPACITY";
        case HI_ENOMEM_HOST: return "HI_ENOMEM_HOST";
        case HI_ENOMEM_DEV: return "HI_ENOMEM_DEV";
        case HI_ECUDA: return "HI_ECUDA";
        case HI_ESTATE: return "HI_ESTATE";
    }
    return "HI_UNKNOWN";
}

const char* hi_last_error(const hi_ctx* c) { return c ? c->err.c_str() : g_init_error.c_str(); }

hi_status hi_init(int layers, int q_heads, int kv_heads, int head_dim, int64_t max_ctx, int chunk, int rank,
                  int world, hi_ctx** out) {
    return hi_init_ex(layers, q_heads, kv_heads, head_dim, max_ctx, chunk, rank, world, nullptr, out);
}

hi_status hi_init_ex(int layers, int q_heads, int kv_heads, int head_dim, int64_t max_ctx, int chunk, int rank,
                     int world, const hi_options* opt, hi_ctx** out) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!out) { g_init_error = "out is NULL"; return HI_EINVAL; }
    *out = nullptr;
    if (layers <= 0 || layers > 128 || q_heads <= 0 || kv_heads <= 0 || max_ctx <= 0 || chunk <= 0 || world <= 0 ||
        rank < 0 || rank >= world || q_heads % kv_heads != 0 || kv_heads % world != 0 ||
        (head_dim != 64 && head_dim != 128) || max_ctx > (int64_t(1) << 31) || chunk > (1 << 20)) {
        g_init_error = "invalid configuration (sizes, q_heads % kv_heads, kv_heads % world, head_dim in {64,128})";
        return HI_EINVAL;
    }
    const int g = q_heads / kv_heads;
    if (g != 1 && g != 2 && g != 4 && g != 8) {
        g_init_error = "q_heads/kv_heads must be 1, 2, 4 or 8";
        return HI_EINVAL;
    }
    hi_options o{};
    if (opt) o = *opt;
    if (o.n_slots == 0) o.n_slots = 4;
    if (o.head_group == 0) o.head_group = 1;
    if (o.n_slots < 2 || o.n_slots > 64 || o.slot_tokens < 0 || o.resident_kv_heads < HI_RESIDENT_AUTO ||
        (o.head_group != HI_GROUP_AUTO && o.head_group != HI_GROUP_PAPER &&
         (o.head_group < 1 || (kv_heads / world) % o.head_group != 0))) {
        g_init_error = "invalid hi_options (n_slots in [2,64], slot_tokens >= 0, resident_kv_heads >= -1, "
                       "head_group = -1 or >= 1 dividing kv_heads/world)";
        return HI_EINVAL;
    }
#ifndef HI_WITH_VARIANTS
    if (o.flags & (HI_FLAG_MMA_SYNC_PREFILL | HI_FLAG_PREFILL_2CTA | HI_FLAG_PREFILL_TC1 | HI_FLAG_PREFILL_PSMEM)) {
        g_init_error = "the comparison prefill kernels (mma.sync, CTA pair, one tile, P in shared memory) are only in the variants "
                       "build (paper_2502_12574_b200.build.build_variant(\"cmp\", []), HI_LIB_VARIANT=cmp)";
        return HI_EINVAL;
    }
#endif
    if (kv_heads / world > hi::MAX_LAUNCH_HEADS) {
        g_init_error = "kv_heads/world must be <= 64";
        return HI_EINVAL;
    }
    // NEXT-3 duo streaming heads (reading R18): labels of this shard's kv heads
    int n_stream_lab = 0;
    if (o.streaming_heads)
        for (int l = 0; l < layers; ++l)
            for (int h = 0; h < kv_heads / world; ++h)
                n_stream_lab += o.streaming_heads[static_cast<size_t>(l) * kv_heads + rank * (kv_heads / world) + h] != 0;
    if (o.duo_sink == 0) o.duo_sink = 64;
    if (o.duo_sink < 0) o.duo_sink = 0;
    if (o.duo_window == 0) o.duo_window = 256;
    if (n_stream_lab > 0 &&
        (o.duo_window < 1 || o.duo_window > (1 << 20) || o.duo_sink > (1 << 20) ||
         (o.flags & (HI_FLAG_MMA_SYNC_PREFILL | HI_FLAG_PREFILL_2CTA | HI_FLAG_PREFILL_TC1)))) {
        g_init_error = "streaming heads need duo_window in [1, 2^20], duo_sink <= 2^20 and the default prefill kernel";
        return HI_EINVAL;
    }

    hi_ctx* c = new hi_ctx();
    c->L = layers; c->Hq = q_heads; c->Hkv = kv_heads; c->d = head_dim; c->chunk = chunk;
    c->rank = rank; c->world = world; c->Hq_loc = q_heads / world; c->Hkv_loc = kv_heads / world; c->g = g;
    c->max_ctx = max_ctx; c->flags = o.flags;
    c->scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(head_dim)));
    c->seq_len.assign(layers, 0);
    c->n_slots = o.n_slots;
    // default slot size: the whole ring (n_slots slots of `group` heads) holds at most ONE head's K+V at
    // max_ctx (Eq. 11, reading R8), whatever the head group -- but a block is never shorter than
    // min(max_ctx/2, 32768) tokens: at short contexts, where one head is a few MiB, fewer and longer copies
    // beat the per-copy and per-launch overheads (the paper's adaptive grouping trades memory for speed
    // there too).  An explicit slot_tokens is taken as given.
    constexpr int64_t kMinBlock = 32768;
    auto default_slot_tokens = [&](int group) {
        const int64_t one_head = (max_ctx / (static_cast<int64_t>(o.n_slots) * group)) / 64 * 64;
        const int64_t floor_blk = std::min<int64_t>((max_ctx / 2) / 64 * 64, kMinBlock);
        return std::max<int64_t>(64, std::max(one_head, floor_blk));
    };

    auto bail = [&](hi_status s, const std::string& msg) {
        g_init_error = msg.empty() ? c->err : msg;
        destroy(c);
        return s;
    };
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return bail(HI_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    if (opt && opt->device >= 0 && opt->device < ndev && opt->device != 0) c->device = opt->device;
    else if (cudaGetDevice(&c->device) != cudaSuccess) c->device = 0;
    hi::DeviceGuard dg(c->device);  // the caller's current device is restored on return
    {
        int cur = -1;
        if ((e = cudaGetDevice(&cur)) != cudaSuccess || cur != c->device)
            return bail(HI_ECUDA, std::string("cannot select device ") + std::to_string(c->device));
    }
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, c->device) == cudaSuccess && prop.major < 10)
        return bail(HI_ECUDA, "libheadinfer is built for sm_100a (B200); device compute capability < 10");

    // head groups (NEXT-2).  Auto: the smallest divisor G of Hkv_loc whose chunk-segment launch has >= 8
    // waves of 128-row tiles (launch fill/drain amortised, Tab. 5-7 short-context regime), while the
    // staging ring stays <= 1/32 of device memory (the adaptive memory/speed trade-off of App. D).
    auto head_slot_bytes_for = [&](int group) {
        return static_cast<size_t>(o.slot_tokens ? o.slot_tokens : default_slot_tokens(group)) * head_dim * 2 * 2;
    };
    if (o.head_group == HI_GROUP_PAPER) {
        // the paper's adaptive schedule (§4 "Adaptive Head-wise Offloading"; Tab. 6/7 "Adaptive"): all
        // heads fused up to 500K tokens, 2 groups to 1M, 4 to 2M, 8 (one head per unit) beyond; the number of
        // groups is over the model's kv heads, so this shard's unit is Hkv_loc / groups heads (at least 1)
        // range bounds 512K / 1M / 2M tokens (2^19, 2^20, 2^21), each with a 64K-token decode tail
        const int64_t tail = 1 << 16;
        const int groups = max_ctx <= (1 << 19) + tail ? 1 : max_ctx <= (1 << 20) + tail ? 2
                           : max_ctx <= (1 << 21) + tail ? 4 : 8;
        int G = std::max(1, std::min(c->Hkv_loc, kv_heads / std::min(groups, kv_heads)));
        while (c->Hkv_loc % G) --G;
        o.head_group = G;
    }
    if (o.head_group == HI_GROUP_AUTO) {
        const int64_t tiles = (static_cast<int64_t>(chunk) * g + 127) / 128;
        const int sms = prop.multiProcessorCount > 0 ? prop.multiProcessorCount : 148;
        const size_t mem_cap = prop.totalGlobalMem / 32;
        int G = 1;
        for (int cand = 1; cand <= c->Hkv_loc; ++cand) {
            if (c->Hkv_loc % cand) continue;
            if (cand > 1 && head_slot_bytes_for(cand) * cand * c->n_slots > mem_cap) break;
            G = cand;
            if (tiles * cand >= 8LL * sms) break;
        }
        o.head_group = G;
    }
    c->group = o.head_group;
    const int64_t st = o.slot_tokens ? o.slot_tokens : default_slot_tokens(c->group);
    c->slot_tokens = st;
    c->slot_default = o.slot_tokens == 0;
    const size_t head_slot_bytes = head_slot_bytes_for(c->group);
    c->slot_bytes = head_slot_bytes * c->group;

    // head classes: retrieval pairs numbered layer-major (cidx), streaming pairs -1 (NEXT-3)
    const int n_pairs = layers * c->Hkv_loc;
    c->cidx.assign(n_pairs, -1);
    for (int l = 0; l < layers; ++l)
        for (int h = 0; h < c->Hkv_loc; ++h) {
            const bool str = o.streaming_heads &&
                             o.streaming_heads[static_cast<size_t>(l) * kv_heads + rank * c->Hkv_loc + h] != 0;
            if (!str) c->cidx[static_cast<size_t>(l) * c->Hkv_loc + h] = c->n_retr++;
        }
    c->n_stream = n_pairs - c->n_retr;
    if (c->n_stream > 0) {
        c->duo_sink = o.duo_sink;
        c->duo_win = o.duo_window;
        c->duo_ring = o.duo_window;  // history needs the last duo_window - 1 rows; the ring holds duo_window
        c->duo_rows = c->duo_sink + c->duo_ring;
        c->duo_bytes = static_cast<size_t>(n_pairs) * c->duo_head_elems() * 2;  // indexed by (layer, head)
        if (cudaMalloc(reinterpret_cast<void**>(&c->d_duo), c->duo_bytes) != cudaSuccess) {
            cudaGetLastError();
            return bail(HI_ENOMEM_DEV, "cudaMalloc of the streaming-head KV buffers failed");
        }
    }
    // (a) residency (NEXT-1, Alg. 1 H_on): the first n_res retrieval pairs keep their KV in HBM
    const size_t pair_bytes = 2 * static_cast<size_t>(max_ctx) * head_dim * 2;
    if (o.resident_kv_heads == HI_RESIDENT_AUTO) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) { cudaGetLastError(); free_b = 0; }
        const size_t reserve = (size_t(12) << 30) + c->slot_bytes * c->n_slots;  // workspaces + caller tensors
        c->n_res = free_b > reserve ? static_cast<int>(std::min<size_t>(c->n_retr, (free_b - reserve) / pair_bytes)) : 0;
    } else {
        c->n_res = std::min(o.resident_kv_heads, c->n_retr);
    }
    // per-layer schedules: resident retrieval heads, offload units of up to `group` heads, streaming heads
    c->res_heads.assign(layers, {});
    c->str_heads.assign(layers, {});
    c->off_units.assign(layers, {});
    for (int l = 0; l < layers; ++l) {
        std::vector<int> off;
        for (int h = 0; h < c->Hkv_loc; ++h) {
            if (c->streaming(l, h)) c->str_heads[l].push_back(h);
            else if (c->resident(l, h)) c->res_heads[l].push_back(h);
            else off.push_back(h);
        }
        for (size_t i = 0; i < off.size(); i += c->group)
            c->off_units[l].emplace_back(off.begin() + i, off.begin() + std::min(off.size(), i + c->group));
    }
    c->res_bytes = static_cast<size_t>(c->n_res) * pair_bytes;
    if (c->n_res > 0 && cudaMalloc(reinterpret_cast<void**>(&c->d_res), c->res_bytes) != cudaSuccess) {
        cudaGetLastError();
        return bail(HI_ENOMEM_DEV, "cudaMalloc of the resident KV cache failed");
    }
    // (a) host store for the offloaded pairs
    c->host_bytes = static_cast<size_t>(c->n_retr - c->n_res) * pair_bytes;
    hi_status hs = alloc_host_store(c, o.numa_policy, o.numa_node);
    if (hs != HI_OK) return bail(hs, "");

    // (b)/(c) staging, streams, events
    auto dmalloc = [&](void** p, size_t bytes) -> bool {
        if (cudaMalloc(p, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
        return true;
    };
    if (!dmalloc(reinterpret_cast<void**>(&c->d_stage), c->slot_bytes * c->n_slots))
        return bail(HI_ENOMEM_DEV, "cudaMalloc of the staging slots failed");
    const size_t rows = static_cast<size_t>(chunk) * g;
    const int64_t max_blocks = (max_ctx + st - 1) / st;
    c->max_parts = static_cast<int>(std::max<int64_t>(max_blocks * decode_parts_for_block(std::min<int64_t>(st, max_ctx)),
                                                     decode_parts_for_block(max_ctx)) + 8);
    if (c->n_stream > 0)  // sink segment + up to two ring runs, each split into >= 64-key parts
        c->max_parts = std::max<int>(c->max_parts, static_cast<int>((c->duo_sink + 63) / 64 + (c->duo_ring + 63) / 64 + 8));
    const size_t pack_b = static_cast<size_t>(c->Hkv_loc) * 2 * chunk * head_dim * 2;
    const size_t oacc_b = rows * head_dim * 4 * c->group, ml_b = rows * 4 * c->group;
    const size_t parts_b = static_cast<size_t>(c->Hkv_loc) * c->max_parts * g * (head_dim + 4) * 4;
    const size_t kvnew_b = static_cast<size_t>(layers) * 2 * c->Hkv_loc * head_dim * 2;
    if (!dmalloc(reinterpret_cast<void**>(&c->d_pack), pack_b) || !dmalloc(reinterpret_cast<void**>(&c->d_oacc), oacc_b) ||
        !dmalloc(reinterpret_cast<void**>(&c->d_macc), ml_b) || !dmalloc(reinterpret_cast<void**>(&c->d_lacc), ml_b) ||
        !dmalloc(reinterpret_cast<void**>(&c->d_parts), parts_b) || !dmalloc(reinterpret_cast<void**>(&c->d_kvnew), kvnew_b) ||
        !dmalloc(reinterpret_cast<void**>(&c->d_counters), sizeof(unsigned) * hi::MAX_LAUNCH_HEADS))
        return bail(HI_ENOMEM_DEV, "cudaMalloc of a workspace failed");
    if (cudaMemset(c->d_counters, 0, sizeof(unsigned) * hi::MAX_LAUNCH_HEADS) != cudaSuccess)
        return bail(HI_ECUDA, "cudaMemset of the decode counters failed");
    c->workspace_bytes = static_cast<int64_t>(pack_b + oacc_b + 2 * ml_b + parts_b + kvnew_b);

    auto mkev = [&](cudaEvent_t* ev) { return cudaEventCreateWithFlags(ev, cudaEventDisableTiming) == cudaSuccess; };
    bool ok = cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking) == cudaSuccess && mkev(&c->ev_call_in) &&
              mkev(&c->ev_call_out) && mkev(&c->ev_packed) && mkev(&c->ev_pack_free);
    c->slots.resize(c->n_slots);
    for (auto& s : c->slots) ok = ok && mkev(&s.ready) && mkev(&s.free_);
    c->ev_layer_d2h.assign(layers, nullptr);
    c->ev_kvnew_free.assign(layers, nullptr);
    for (int l = 0; l < layers; ++l) ok = ok && mkev(&c->ev_layer_d2h[l]) && mkev(&c->ev_kvnew_free[l]);
    if (!ok) { cudaGetLastError(); return bail(HI_ECUDA, "stream/event creation failed"); }
    // record every event once so the first waits are satisfied
    for (auto& s : c->slots) ok = ok && cudaEventRecord(s.free_, c->s_comp) == cudaSuccess;
    for (int l = 0; l < layers; ++l)
        ok = ok && cudaEventRecord(c->ev_layer_d2h[l], c->s_d2h) == cudaSuccess &&
             cudaEventRecord(c->ev_kvnew_free[l], c->s_d2h) == cudaSuccess;
    ok = ok && cudaEventRecord(c->ev_pack_free, c->s_d2h) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
    if (!ok) { cudaGetLastError(); return bail(HI_ECUDA, "initial event record failed"); }
    c->init_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = c;
    return HI_OK;
}

hi_status hi_free(hi_ctx* c) {
    destroy(c);
    return HI_OK;
}

hi_status hi_prefill_chunk(hi_ctx* c, int layer, const void* Q, const void* K, const void* V, void* out, int n,
                           void* cuda_stream) {
    if (!c) return HI_ESHAPE;
    hi::DeviceGuard dg(c->device);
    hi_status st = check_call(c, layer);
    if (st != HI_OK) return st;
    if (!Q || !K || !V || !out) return set_err(c, HI_ESHAPE, "NULL tensor pointer");
    if (n < 1 || n > c->chunk) return set_err(c, HI_ESHAPE, "n_tokens must be in [1, chunk]");
    const int64_t s = c->seq_len[layer];
    if (s + n > c->max_ctx) return set_err(c, HI_ECAPACITY, "seq_len + n_tokens exceeds max_ctx");
    cudaStream_t cs = static_cast<cudaStream_t>(cuda_stream);
    const int d = c->d, Hkv = c->Hkv_loc, g = c->g;
    NvtxRange nr("hi_prefill_chunk layer %d s %lld n %d", layer, static_cast<long long>(s), n);

    HI_CK(c, cudaEventRecord(c->ev_call_in, cs));
    HI_CK(c, cudaStreamWaitEvent(c->s_comp, c->ev_call_in, 0));
    if (hi_status fs = inject_fault(c); fs != HI_OK) return fs;
    // pack the chunk's K/V head-major (the previous call's write-back must have drained)
    HI_CK(c, cudaStreamWaitEvent(c->s_comp, c->ev_pack_free, 0));
    HI_CK(c, hi::launch_pack_kv(static_cast<const __nv_bfloat16*>(K), static_cast<const __nv_bfloat16*>(V), c->d_pack, n,
                                Hkv, d, c->s_comp));
    ++c->launches;
    HI_CK(c, cudaEventRecord(c->ev_packed, c->s_comp));
    // history H2D of this layer must see every earlier write-back of its rows (RAW via host DRAM)
    HI_CK(c, cudaStreamWaitEvent(c->s_h2d, c->ev_layer_d2h[layer], 0));
    // write-back (Alg. 1 line 11): D2H of the chunk's rows [s, s+n) of every offloaded local kv head;
    // resident heads (Alg. 1 line 8 "Update GPU KV cache") append on the compute stream instead; streaming
    // heads (NEXT-3) keep only their sink + window on the GPU (appended after their attention below)
    HI_CK(c, cudaStreamWaitEvent(c->s_d2h, c->ev_packed, 0));
    const size_t row_bytes = static_cast<size_t>(d) * 2;
    if (hi_status js = jitter(c, c->s_d2h); js != HI_OK) return js;
    LaunchTimer tm_wb(c, c->s_d2h);
    const int64_t wb0 = c->d2h_bytes;
    CopyBatch wb;
    for (int h = 0; h < Hkv; ++h) {
        if (c->streaming(layer, h)) continue;
        const __nv_bfloat16* pk = c->d_pack + (static_cast<size_t>(h) * 2 + 0) * n * d;
        const __nv_bfloat16* pv = c->d_pack + (static_cast<size_t>(h) * 2 + 1) * n * d;
        if (c->resident(layer, h)) {
            HI_CK(c, cudaMemcpyAsync(c->dev_k(layer, h, s), pk, n * row_bytes, cudaMemcpyDeviceToDevice, c->s_comp));
            HI_CK(c, cudaMemcpyAsync(c->dev_v(layer, h, s), pv, n * row_bytes, cudaMemcpyDeviceToDevice, c->s_comp));
            continue;
        }
        wb.add(c->host_k(layer, h, s), pk, n * row_bytes);
        wb.add(c->host_v(layer, h, s), pv, n * row_bytes);
        c->d2h_bytes += static_cast<int64_t>(2 * n * row_bytes);
    }
    HI_CK(c, wb.issue(c->s_d2h));
    tm_wb.done(static_cast<double>(c->d2h_bytes - wb0), T_D2H);
    HI_CK(c, cudaEventRecord(c->ev_pack_free, c->s_d2h));
    HI_CK(c, cudaEventRecord(c->ev_layer_d2h[layer], c->s_d2h));

    // attention, one unit of kv heads at a time (Alg. 1 line 5 loop; NEXT-2 head groups when group > 1)
    const int64_t nb = (s + c->slot_tokens - 1) / c->slot_tokens;
    hi::PrefillParams base{};
    base.q = static_cast<const __nv_bfloat16*>(Q);
    base.out = static_cast<__nv_bfloat16*>(out);
    base.q_tok_stride = static_cast<int64_t>(c->Hq_loc) * d;
    base.o_tok_stride = base.q_tok_stride;
    base.n_q = n;
    base.q_pos0 = s;
    base.g = g;
    base.scale_log2 = c->scale_log2;
    base.o_acc = c->d_oacc;
    base.m_acc = c->d_macc;
    base.l_acc = c->d_lacc;
    base.state_rows = static_cast<int64_t>(c->chunk) * g;
    base.q_span = Hkv;
    const bool timing = c->flags & HI_FLAG_TIMING;
    // one launch over segment keys [k_pos0, k_pos0 + n_k) for the unit's heads
    auto run = [&](hi::PrefillParams& p, int flags) -> hi_status {
        p.flags = flags;
        if (hi_status js = jitter(c, c->s_comp); js != HI_OK) return js;
        LaunchTimer tm(c);
        HI_CK(c, launch_prefill(c, p));
        if (timing)
            tm.done(4.0 * d * g * p.n_heads * seg_pairs(s, n, p.k_pos0, p.n_k, flags & hi::PF_CAUSAL, p.win), T_PREFILL);
        ++c->launches;
        return HI_OK;
    };
    // the chunk's own keys [s + r0, s + n) from the pack buffer ([h][K|V][n][d]); kv coordinate = the real head
    auto chunk_seg = [&](hi::PrefillParams& p, const std::vector<int>& unit, int r0) {
        p.k = c->d_pack + static_cast<size_t>(r0) * d;
        p.v = c->d_pack + static_cast<size_t>(n) * d + static_cast<size_t>(r0) * d;
        p.kv_row_stride = d;
        p.kv_head_stride = static_cast<int64_t>(2) * n * d;
        for (size_t y = 0; y < unit.size(); ++y) p.head_kv[y] = static_cast<int16_t>(unit[y]);
        p.kv_span = Hkv;
        p.n_k = n - r0;
        p.k_pos0 = s + r0;
    };
    auto start_unit = [&](const std::vector<int>& unit) {
        hi::PrefillParams p = base;
        p.n_heads = static_cast<int>(unit.size());
        for (size_t y = 0; y < unit.size(); ++y) p.head_q[y] = static_cast<int16_t>(unit[y]);
        return p;
    };
    auto units_of = [&](const std::vector<int>& heads) {
        std::vector<std::vector<int>> u;
        for (size_t i = 0; i < heads.size(); i += c->group)
            u.emplace_back(heads.begin() + i, heads.begin() + std::min(heads.size(), i + c->group));
        return u;
    };
    // H_on heads of this layer (NEXT-1): chunk segment + the whole history straight from the HBM cache
    // (consecutive resident pairs are 2*max_ctx rows apart)
    for (const auto& unit : units_of(c->res_heads[layer])) {
        hi::PrefillParams p = start_unit(unit);
        chunk_seg(p, unit, 0);
        if ((st = run(p, hi::PF_FIRST | hi::PF_CAUSAL | (s == 0 ? hi::PF_LAST : 0))) != HI_OK) return st;
        if (s > 0) {
            p.k = reinterpret_cast<const __nv_bfloat16*>(c->dev_k(layer, unit[0], 0));
            p.v = reinterpret_cast<const __nv_bfloat16*>(c->dev_v(layer, unit[0], 0));
            p.kv_head_stride = 2 * c->max_ctx * d;
            for (size_t y = 0; y < unit.size(); ++y) p.head_kv[y] = static_cast<int16_t>(y);
            p.kv_span = static_cast<int>(unit.size());
            p.n_k = static_cast<int>(s);
            p.k_pos0 = 0;
            if ((st = run(p, hi::PF_LAST)) != HI_OK) return st;
        }
    }
    // offloaded heads, `group` at a time
    for (const auto& unit : c->off_units[layer]) {
        hi::PrefillParams p = start_unit(unit);
        // the chunk's own keys first: causal, no transfer needed
        chunk_seg(p, unit, 0);
        if ((st = run(p, hi::PF_FIRST | hi::PF_CAUSAL | (s == 0 ? hi::PF_LAST : 0))) != HI_OK) return st;
        // history blocks [0, s) of the unit's heads through the staging slots (Alg. 1 line 10 prefetch)
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t k0 = b * c->slot_tokens;
            const int64_t nk = std::min<int64_t>(c->slot_tokens, s - k0);
            int slot = 0;
            st = stage_block(c, layer, unit, k0, nk, &slot);
            if (st != HI_OK) return st;
            p.k = reinterpret_cast<const __nv_bfloat16*>(c->slot_k(slot));
            p.v = reinterpret_cast<const __nv_bfloat16*>(c->slot_v(slot));
            p.kv_head_stride = static_cast<int64_t>(c->slot_head_bytes() / 2);
            for (size_t y = 0; y < unit.size(); ++y) p.head_kv[y] = static_cast<int16_t>(y);
            p.kv_span = static_cast<int>(unit.size());
            p.n_k = static_cast<int>(nk);
            p.k_pos0 = k0;
            const bool skip = (c->flags & HI_FLAG_FAULT_SKIP_BLOCK) && b == 0 && nb > 1;  // negative control
            if (!skip && (st = run(p, (b == nb - 1) ? hi::PF_LAST : 0)) != HI_OK) return st;
            st = release_slot(c, slot);
            if (st != HI_OK) return st;
        }
    }
    // duo streaming heads (NEXT-3, reading R18): row p attends keys i <= p with i < duo_sink or i > p - duo_win.
    // Segments: the chunk's sink keys, the chunk's windowed keys, the history sink, the history window (ring
    // runs) -- each wholly sink or wholly non-sink, so the kernel applies the band to non-sink segments only.
    if (!c->str_heads[layer].empty()) {
        const int64_t ns = c->duo_sink;
        for (const auto& unit : units_of(c->str_heads[layer])) {
            hi::PrefillParams p = start_unit(unit);
            struct Seg { int64_t row0_or_r0; int64_t n_k, k_pos0; bool chunk, causal; int win; };
            std::vector<Seg> segs;
            if (s < ns) segs.push_back({0, std::min<int64_t>(n, ns - s), s, true, true, 0});
            const int64_t c0 = std::max<int64_t>(s, ns) - s;
            if (c0 < n) segs.push_back({c0, n - c0, s + c0, true, true, c->duo_win});
            if (s > 0 && ns > 0) segs.push_back({0, std::min<int64_t>(ns, s), 0, false, false, 0});
            for (int64_t pos = std::max<int64_t>(ns, s - c->duo_win + 1); pos < s;) {
                const int64_t row = c->duo_row(pos);
                const int64_t len = std::min<int64_t>(s - pos, c->duo_rows - row);
                segs.push_back({row, len, pos, false, false, c->duo_win});
                pos += len;
            }
            for (size_t i = 0; i < segs.size(); ++i) {
                const Seg& sg = segs[i];
                if (sg.chunk) {
                    chunk_seg(p, unit, static_cast<int>(sg.row0_or_r0));
                    p.n_k = static_cast<int>(sg.n_k);
                } else {
                    p.k = c->duo_k(layer, 0, sg.row0_or_r0);
                    p.v = p.k + c->duo_rows * d;
                    p.kv_row_stride = d;
                    p.kv_head_stride = static_cast<int64_t>(c->duo_head_elems());
                    for (size_t y = 0; y < unit.size(); ++y) p.head_kv[y] = static_cast<int16_t>(unit[y]);
                    p.kv_span = Hkv;
                    p.n_k = static_cast<int>(sg.n_k);
                    p.k_pos0 = sg.k_pos0;
                }
                p.win = sg.win;
                const int fl = (i == 0 ? hi::PF_FIRST : 0) | (i + 1 == segs.size() ? hi::PF_LAST : 0) |
                               (sg.causal ? hi::PF_CAUSAL : 0);
                if ((st = run(p, fl)) != HI_OK) return st;
            }
        }
        // then the chunk's surviving rows go into the sink / ring (after every read of the old window)
        hi::DuoAppendParams ap{};
        ap.src_k = c->d_pack;
        ap.src_v = c->d_pack + static_cast<size_t>(n) * d;
        ap.src_head_stride = static_cast<int64_t>(2) * n * d;
        ap.src_row_stride = d;
        ap.dst = c->duo_k(layer, 0, 0);
        ap.dst_head_stride = static_cast<int64_t>(c->duo_head_elems());
        ap.dst_v_off = c->duo_rows * d;
        ap.pos0 = s;
        ap.n = n;
        ap.n_sink = c->duo_sink;
        ap.ring = c->duo_ring;
        ap.n_heads = static_cast<int>(c->str_heads[layer].size());
        for (int y = 0; y < ap.n_heads; ++y) ap.heads[y] = static_cast<int16_t>(c->str_heads[layer][y]);
        HI_CK(c, hi::launch_duo_append(ap, d, c->s_comp));
        ++c->launches;
    }
    st = finish_call(c, cs);
    if (st != HI_OK) return st;
    c->seq_len[layer] = s + n;
    ++c->prefill_calls;
    return HI_OK;
}

hi_status hi_decode(hi_ctx* c, int layer, const void* q, const void* k, const void* v, void* out, void* cuda_stream) {
    if (!c) return HI_ESHAPE;
    hi::DeviceGuard dg(c->device);
    hi_status st = check_call(c, layer);
    if (st != HI_OK) return st;
    if (!q || !k || !v || !out) return set_err(c, HI_ESHAPE, "NULL tensor pointer");
    const int64_t s = c->seq_len[layer];
    if (s + 1 > c->max_ctx) return set_err(c, HI_ECAPACITY, "seq_len + 1 exceeds max_ctx");
    cudaStream_t cs = static_cast<cudaStream_t>(cuda_stream);
    const int d = c->d, Hkv = c->Hkv_loc, g = c->g;
    const size_t row_bytes = static_cast<size_t>(d) * 2;
    NvtxRange nr("hi_decode layer %d s %lld", layer, static_cast<long long>(s));

    HI_CK(c, cudaEventRecord(c->ev_call_in, cs));
    HI_CK(c, cudaStreamWaitEvent(c->s_comp, c->ev_call_in, 0));
    if (hi_status fs = inject_fault(c); fs != HI_OK) return fs;
    // All-resident layer (NEXT-1, Alg. 1 H_on branch l.22-23): ONE launch -- split-K over [0, s) of every kv head
    // of the layer straight from HBM, the last CTA of each head merging its records with the new key and
    // appending the new row in place (no kvnew staging copy, no D2H, no separate combine or append copies).
    if (s > 0 && c->res_heads[layer].size() == static_cast<size_t>(Hkv)) {
        const auto& R = c->res_heads[layer];
        hi::DecodePartialParams p{};
        p.q = static_cast<const __nv_bfloat16*>(q);
        p.n_k = static_cast<int>(s);
        p.split_len = decode_split_len(s, Hkv);
        p.scale_log2 = c->scale_log2;
        p.parts = c->d_parts;
        p.q_head_stride = static_cast<int64_t>(g) * d;
        p.parts_head_stride = static_cast<int64_t>(c->max_parts) * g * (d + 4);
        for (int y = 0; y < Hkv; ++y) {
            p.head[y] = static_cast<int16_t>(R[y]);
            p.kvc[y] = static_cast<int16_t>(y);
        }
        p.kv_span = Hkv;
        p.k = reinterpret_cast<const __nv_bfloat16*>(c->dev_k(layer, R[0], 0));
        p.v = reinterpret_cast<const __nv_bfloat16*>(c->dev_v(layer, R[0], 0));
        p.kv_head_stride = 2 * c->max_ctx * d;
        const int nsp = static_cast<int>((s + p.split_len - 1) / p.split_len);
        p.combine = 1;
        p.append = 1;
        p.parts_total = nsp;
        p.counters = c->d_counters;
        p.k_new = static_cast<const __nv_bfloat16*>(k);
        p.v_new = static_cast<const __nv_bfloat16*>(v);
        p.out = static_cast<__nv_bfloat16*>(out);
        if (hi_status js = jitter(c, c->s_comp); js != HI_OK) return js;
        LaunchTimer tm(c);
        HI_CK(c, hi::launch_decode_partial(p, d, g, nsp, Hkv, c->s_comp));
        tm.done(4.0 * d * static_cast<double>(s) * Hkv, T_DECODE);
        ++c->launches;
        st = finish_call(c, cs);
        if (st != HI_OK) return st;
        c->seq_len[layer] = s + 1;
        ++c->decode_calls;
        return HI_OK;
    }
    // copy the new k, v into this layer's kvnew buffer (its previous write-back must be done)
    __nv_bfloat16* kn = c->d_kvnew + static_cast<size_t>(layer) * 2 * Hkv * d;
    __nv_bfloat16* vn = kn + static_cast<size_t>(Hkv) * d;
    HI_CK(c, cudaStreamWaitEvent(c->s_comp, c->ev_kvnew_free[layer], 0));
    HI_CK(c, cudaMemcpyAsync(kn, k, Hkv * row_bytes, cudaMemcpyDeviceToDevice, c->s_comp));
    HI_CK(c, cudaMemcpyAsync(vn, v, Hkv * row_bytes, cudaMemcpyDeviceToDevice, c->s_comp));
    HI_CK(c, cudaEventRecord(c->ev_packed, c->s_comp));
    HI_CK(c, cudaStreamWaitEvent(c->s_h2d, c->ev_layer_d2h[layer], 0));
    // append (Alg. 1 line 26 "Async Update CPU KV cache"): host row s of every offloaded local kv head
    HI_CK(c, cudaStreamWaitEvent(c->s_d2h, c->ev_packed, 0));
    if (hi_status js = jitter(c, c->s_d2h); js != HI_OK) return js;
    // all K rows first, then all V rows: consecutive offloaded heads' rows then sit at constant source
    // (one row) and destination (2*max_ctx rows) pitch, so each tensor is one 2-D copy per layer
    CopyBatch ap;
    for (int kv = 0; kv < 2; ++kv)
        for (int h = 0; h < Hkv; ++h) {
            if (c->streaming(layer, h)) continue;  // NEXT-3: sink / ring append below
            const __nv_bfloat16* src = (kv ? vn : kn) + static_cast<size_t>(h) * d;
            if (c->resident(layer, h)) {  // H_on: append in HBM (compute stream; read by later calls only)
                HI_CK(c, cudaMemcpyAsync(kv ? c->dev_v(layer, h, s) : c->dev_k(layer, h, s), src, row_bytes,
                                         cudaMemcpyDeviceToDevice, c->s_comp));
                continue;
            }
            ap.add(kv ? c->host_v(layer, h, s) : c->host_k(layer, h, s), src, row_bytes);
            c->d2h_bytes += static_cast<int64_t>(row_bytes);
        }
    HI_CK(c, ap.issue(c->s_d2h));
    HI_CK(c, cudaEventRecord(c->ev_kvnew_free[layer], c->s_d2h));
    HI_CK(c, cudaEventRecord(c->ev_layer_d2h[layer], c->s_d2h));

    // history -> split-K partial records, per local kv head h at parts[h][0 .. n_parts[h])
    hi::DecodeCombineParams cp{};
    const int64_t rec = static_cast<int64_t>(g) * (d + 4);
    auto partial = [&](hi::DecodePartialParams& p, const std::vector<int>& heads, int64_t nk, int pofs,
                       int waves = HI_DECODE_WAVES) -> int {
        p.q = static_cast<const __nv_bfloat16*>(q);
        p.n_k = static_cast<int>(nk);
        p.split_len = decode_split_len(nk, static_cast<int>(heads.size()), waves);
        p.scale_log2 = c->scale_log2;
        p.parts = c->d_parts + pofs * rec;
        p.q_head_stride = static_cast<int64_t>(g) * d;
        p.parts_head_stride = static_cast<int64_t>(c->max_parts) * rec;
        for (size_t y = 0; y < heads.size(); ++y) p.head[y] = static_cast<int16_t>(heads[y]);
        return static_cast<int>((nk + p.split_len - 1) / p.split_len);
    };
    auto launch = [&](const hi::DecodePartialParams& p, int nsp, int nh, int64_t nk) -> hi_status {
        if (hi_status js = jitter(c, c->s_comp); js != HI_OK) return js;
        LaunchTimer tm(c);
        HI_CK(c, hi::launch_decode_partial(p, d, g, nsp, nh, c->s_comp));
        tm.done(4.0 * d * static_cast<double>(nk) * nh, T_DECODE);
        ++c->launches;
        return HI_OK;
    };
    const auto& R = c->res_heads[layer];
    if (!R.empty() && s > 0) {  // H_on heads of this layer: ONE split-K launch over [0, s) of all of them, in HBM
        hi::DecodePartialParams p{};
        const int nsp = partial(p, R, s, 0);
        p.k = reinterpret_cast<const __nv_bfloat16*>(c->dev_k(layer, R[0], 0));
        p.v = reinterpret_cast<const __nv_bfloat16*>(c->dev_v(layer, R[0], 0));
        p.kv_head_stride = 2 * c->max_ctx * d;  // consecutive resident pairs are [K | V] blocks of max_ctx rows
        for (size_t y = 0; y < R.size(); ++y) p.kvc[y] = static_cast<int16_t>(y);
        p.kv_span = static_cast<int>(R.size());
        if ((st = launch(p, nsp, static_cast<int>(R.size()), s)) != HI_OK) return st;
        for (int h : R) cp.n_parts[h] = static_cast<int32_t>(nsp);
    }
    const int64_t nb = (s + c->slot_tokens - 1) / c->slot_tokens;
    for (const auto& unit : c->off_units[layer]) {
        const int nh = static_cast<int>(unit.size());
        int pofs = 0;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t k0 = b * c->slot_tokens;
            const int64_t nk = std::min<int64_t>(c->slot_tokens, s - k0);
            int slot = 0;
            st = stage_block(c, layer, unit, k0, nk, &slot);
            if (st != HI_OK) return st;
            hi::DecodePartialParams p{};
            const int nsp = partial(p, unit, nk, pofs, kOffloadDecodeWaves);
            p.k = reinterpret_cast<const __nv_bfloat16*>(c->slot_k(slot));
            p.v = reinterpret_cast<const __nv_bfloat16*>(c->slot_v(slot));
            p.kv_head_stride = static_cast<int64_t>(c->slot_head_bytes() / 2);
            for (int y = 0; y < nh; ++y) p.kvc[y] = static_cast<int16_t>(y);
            p.kv_span = nh;
            if ((st = launch(p, nsp, nh, nk)) != HI_OK) return st;
            pofs += nsp;
            st = release_slot(c, slot);
            if (st != HI_OK) return st;
        }
        for (int h : unit) cp.n_parts[h] = static_cast<int32_t>(pofs);
    }
    const auto& S = c->str_heads[layer];
    if (!S.empty()) {  // NEXT-3 streaming heads: the sink rows and the window's ring runs, all heads per launch
        const int nh = static_cast<int>(S.size());
        int pofs = 0;
        auto seg = [&](int64_t row, int64_t nk) -> hi_status {
            hi::DecodePartialParams p{};
            const int nsp = partial(p, S, nk, pofs);
            p.k = c->duo_k(layer, 0, row);
            p.v = p.k + c->duo_rows * d;
            p.kv_head_stride = static_cast<int64_t>(c->duo_head_elems());
            for (int y = 0; y < nh; ++y) p.kvc[y] = static_cast<int16_t>(S[y]);
            p.kv_span = Hkv;
            hi_status e = launch(p, nsp, nh, nk);
            pofs += nsp;
            return e;
        };
        if (s > 0 && c->duo_sink > 0)
            if ((st = seg(0, std::min<int64_t>(c->duo_sink, s))) != HI_OK) return st;
        for (int64_t pos = std::max<int64_t>(c->duo_sink, s - c->duo_win + 1); pos < s;) {
            const int64_t row = c->duo_row(pos);
            const int64_t len = std::min<int64_t>(s - pos, c->duo_rows - row);
            if ((st = seg(row, len)) != HI_OK) return st;
            pos += len;
        }
        for (int h : S) cp.n_parts[h] = static_cast<int32_t>(pofs);
        // the new token's row joins the sink / ring (its ring row is not one the window above read)
        hi::DuoAppendParams ap{};
        ap.src_k = kn;
        ap.src_v = vn;
        ap.src_head_stride = d;
        ap.src_row_stride = 0;
        ap.dst = c->duo_k(layer, 0, 0);
        ap.dst_head_stride = static_cast<int64_t>(c->duo_head_elems());
        ap.dst_v_off = c->duo_rows * d;
        ap.pos0 = s;
        ap.n = 1;
        ap.n_sink = c->duo_sink;
        ap.ring = c->duo_ring;
        ap.n_heads = nh;
        for (int y = 0; y < nh; ++y) ap.heads[y] = static_cast<int16_t>(S[y]);
        HI_CK(c, hi::launch_duo_append(ap, d, c->s_comp));
        ++c->launches;
    }
    cp.q = static_cast<const __nv_bfloat16*>(q);
    cp.k_new = kn;
    cp.v_new = vn;
    cp.parts = c->d_parts;
    cp.max_parts = c->max_parts;
    cp.g = g;
    cp.scale_log2 = c->scale_log2;
    cp.out = static_cast<__nv_bfloat16*>(out);
    HI_CK(c, hi::launch_decode_combine(cp, d, c->Hq_loc, c->s_comp));
    ++c->launches;
    st = finish_call(c, cs);
    if (st != HI_OK) return st;
    c->seq_len[layer] = s + 1;
    ++c->decode_calls;
    return HI_OK;
}

hi_status hi_synchronize(hi_ctx* c) {
    if (!c) return HI_ESHAPE;
    if (c->sticky) return HI_ECUDA;
    hi::DeviceGuard dg(c->device);
    HI_CK(c, cudaStreamSynchronize(c->s_comp));
    HI_CK(c, cudaStreamSynchronize(c->s_h2d));
    HI_CK(c, cudaStreamSynchronize(c->s_d2h));
    resolve_timing(c);
    return HI_OK;
}

hi_status hi_read_host_kv(hi_ctx* c, int layer, int h, int64_t pos, int64_t n, void* k_dst, void* v_dst) {
    if (!c) return HI_ESHAPE;
    hi::DeviceGuard dg(c->device);
    hi_status st = check_call(c, layer);
    if (st != HI_OK) return st;
    if (h < 0 || h >= c->Hkv_loc || pos < 0 || n < 0 || pos + n > c->max_ctx || (n > 0 && (!k_dst || !v_dst)))
        return set_err(c, HI_ESHAPE, "bad host KV range");
    if (c->streaming(layer, h)) {  // NEXT-3: only the sink rows and the last duo_win rows below seq_len exist
        const int64_t sl = c->seq_len[layer];
        for (int64_t p = pos; p < pos + n; ++p)
            if (p >= sl || (p >= c->duo_sink && p < sl - c->duo_win))
                return set_err(c, HI_ESTATE, "streaming head: row not held (only sink + recent window)");
        st = hi_synchronize(c);
        if (st != HI_OK) return st;
        for (int64_t p = pos; p < pos + n;) {  // runs of positions that are contiguous rows (sink, ring segments)
            const int64_t r = c->duo_row(p);
            const int64_t len = std::min(pos + n - p, p < c->duo_sink ? c->duo_sink - p : c->duo_rows - r);
            const size_t b = static_cast<size_t>(len) * c->d * 2;
            uint8_t* kd = static_cast<uint8_t*>(k_dst) + (p - pos) * c->d * 2;
            uint8_t* vd = static_cast<uint8_t*>(v_dst) + (p - pos) * c->d * 2;
            HI_CK(c, cudaMemcpy(kd, c->duo_k(layer, h, r), b, cudaMemcpyDeviceToHost));
            HI_CK(c, cudaMemcpy(vd, c->duo_k(layer, h, r) + c->duo_rows * c->d, b, cudaMemcpyDeviceToHost));
            p += len;
        }
        return HI_OK;
    }
    if (c->resident(layer, h)) {
        st = hi_synchronize(c);
        if (st != HI_OK) return st;
        HI_CK(c, cudaMemcpy(k_dst, c->dev_k(layer, h, pos), static_cast<size_t>(n) * c->d * 2, cudaMemcpyDeviceToHost));
        HI_CK(c, cudaMemcpy(v_dst, c->dev_v(layer, h, pos), static_cast<size_t>(n) * c->d * 2, cudaMemcpyDeviceToHost));
        return HI_OK;
    }
    HI_CK(c, cudaStreamSynchronize(c->s_d2h));
    memcpy(k_dst, c->host_k(layer, h, pos), static_cast<size_t>(n) * c->d * 2);
    memcpy(v_dst, c->host_v(layer, h, pos), static_cast<size_t>(n) * c->d * 2);
    return HI_OK;
}

hi_status hi_write_host_kv(hi_ctx* c, int layer, int h, int64_t pos, int64_t n, const void* k_src, const void* v_src,
                           int from_device) {
    if (!c) return HI_ESHAPE;
    hi::DeviceGuard dg(c->device);
    hi_status st = check_call(c, layer);
    if (st != HI_OK) return st;
    if (h < 0 || h >= c->Hkv_loc || pos < 0 || n < 0 || pos + n > c->max_ctx || (n > 0 && (!k_src || !v_src)))
        return set_err(c, HI_ESHAPE, "bad host KV range");
    st = hi_synchronize(c);
    if (st != HI_OK) return st;
    // a device source may have been produced on any stream (e.g. the caller's): the copies below run on the
    // library's own non-blocking streams, so everything already enqueued on the device finishes first
    if (from_device) HI_CK(c, cudaDeviceSynchronize());
    const size_t bytes = static_cast<size_t>(n) * c->d * 2;
    if (c->streaming(layer, h)) {  // NEXT-3: sink rows, then the last duo_ring rows of the range into the ring
        const cudaMemcpyKind kind = from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        const int64_t lo_ring = std::max<int64_t>(c->duo_sink, pos + n - c->duo_ring);
        for (int64_t p = pos; p < pos + n;) {  // runs of positions that are contiguous rows
            if (p >= c->duo_sink && p < lo_ring) { p = lo_ring; continue; }
            const int64_t r = c->duo_row(p);
            const int64_t len = std::min(pos + n - p, p < c->duo_sink ? c->duo_sink - p : c->duo_rows - r);
            const size_t b = static_cast<size_t>(len) * c->d * 2;
            const uint8_t* ks = static_cast<const uint8_t*>(k_src) + (p - pos) * c->d * 2;
            const uint8_t* vs = static_cast<const uint8_t*>(v_src) + (p - pos) * c->d * 2;
            HI_CK(c, cudaMemcpy(c->duo_k(layer, h, r), ks, b, kind));
            HI_CK(c, cudaMemcpy(c->duo_k(layer, h, r) + c->duo_rows * c->d, vs, b, kind));
            p += len;
        }
        return HI_OK;
    }
    if (c->resident(layer, h)) {
        const cudaMemcpyKind kind = from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        HI_CK(c, cudaMemcpy(c->dev_k(layer, h, pos), k_src, bytes, kind));
        HI_CK(c, cudaMemcpy(c->dev_v(layer, h, pos), v_src, bytes, kind));
        return HI_OK;
    }
    if (from_device) {
        HI_CK(c, cudaMemcpyAsync(c->host_k(layer, h, pos), k_src, bytes, cudaMemcpyDeviceToHost, c->s_d2h));
        HI_CK(c, cudaMemcpyAsync(c->host_v(layer, h, pos), v_src, bytes, cudaMemcpyDeviceToHost, c->s_d2h));
        HI_CK(c, cudaStreamSynchronize(c->s_d2h));
    } else {
        memcpy(c->host_k(layer, h, pos), k_src, bytes);
        memcpy(c->host_v(layer, h, pos), v_src, bytes);
    }
    return HI_OK;
}

int64_t hi_seq_len(const hi_ctx* c, int layer) {
    if (!c || layer < 0 || layer >= c->L) return -1;
    return c->seq_len[layer];
}

hi_status hi_set_seq_len(hi_ctx* c, int layer, int64_t s) {
    hi_status st = check_call(c, layer);
    if (st != HI_OK) return st;
    if (s < 0 || s > c->max_ctx) return set_err(c, HI_ESHAPE, "seq_len out of range");
    st = hi_synchronize(c);
    if (st != HI_OK) return st;
    c->seq_len[layer] = s;
    return HI_OK;
}

hi_status hi_get_stats(hi_ctx* c, hi_stats* o) {
    if (!c || !o) return HI_ESHAPE;
    if (!c->sticky) {
        hi_status st = hi_synchronize(c);
        if (st != HI_OK) return st;
    }
    memset(o, 0, sizeof *o);
    o->host_store_bytes = static_cast<int64_t>(c->host_bytes);
    o->staging_bytes = static_cast<int64_t>(c->slot_bytes) * c->n_slots;
    // default slot size: Eq. 11's one head at max_ctx, or the ring itself where the minimum block length set
    // it (short contexts); `group` heads when the caller sized the slots
    o->staging_bound_bytes = c->slot_default
        ? std::max<int64_t>(4ll * c->d * c->max_ctx, static_cast<int64_t>(c->slot_bytes) * c->n_slots)
        : 4ll * c->d * c->max_ctx * c->group;
    o->workspace_bytes = static_cast<int64_t>(c->workspace_bytes);
    o->h2d_bytes = c->h2d_bytes;
    o->d2h_bytes = c->d2h_bytes;
    o->prefill_calls = c->prefill_calls;
    o->decode_calls = c->decode_calls;
    o->kernel_launches = c->launches;
    o->prefill_attn_ms = c->prefill_ms;
    o->prefill_attn_flops = c->prefill_flops;
    o->prefill_attn_launches = c->prefill_timed;
    o->decode_attn_ms = c->decode_ms;
    o->decode_attn_bytes = c->decode_bytes;
    o->decode_attn_launches = c->decode_timed;
    o->init_seconds = c->init_seconds;
    o->resident_kv_heads = c->n_res;
    o->resident_bytes = static_cast<int64_t>(c->res_bytes);
    o->head_group = c->group;
    o->streaming_kv_heads = c->n_stream;
    o->streaming_bytes = static_cast<int64_t>(c->duo_bytes);
    o->h2d_copy_ms = c->h2d_ms;
    o->d2h_copy_ms = c->d2h_ms;
    o->numa_node = c->numa_node;
    o->n_slots = c->n_slots;
    o->slot_tokens = c->slot_tokens;
    return c->sticky ? HI_ECUDA : HI_OK;  // a sticky-failed context still reports its counters
}

}  // extern "C"
