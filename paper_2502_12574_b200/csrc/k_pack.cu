// k_pack.cu -- gather the chunk's K and V [n][Hkv][d] into head-major [Hkv][2][n][d]
// (SURVEY.md §2B K5b), so each head's write-back to host (Alg. 1 line 11) is one
// contiguous D2H per tensor and the chunk's own keys are a contiguous segment for the
// prefill kernel.  Pure data movement: 16-byte vector loads/stores, fully coalesced.
#include "hi_kernels.cuh"

namespace hi {
namespace {

__global__ void pack_kv_kernel(const uint4* __restrict__ k, const uint4* __restrict__ v, uint4* __restrict__ packed,
                               int n, int hkv, int cpr /* 16-byte chunks per row */) {
    const int64_t total = static_cast<int64_t>(n) * hkv * cpr;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cpr);
        const int64_t th = i / cpr;  // token*hkv + head
        const int h = static_cast<int>(th % hkv);
        const int64_t t = th / hkv;
        const int64_t dk = ((static_cast<int64_t>(h) * 2 + 0) * n + t) * cpr + c;
        const int64_t dv = ((static_cast<int64_t>(h) * 2 + 1) * n + t) * cpr + c;
        packed[dk] = k[i];
        packed[dv] = v[i];
    }
}

__global__ void poison_kernel(uint4* p, int64_t n16) {
    const uint4 nan4 = make_uint4(0x7fc07fc0u, 0x7fc07fc0u, 0x7fc07fc0u, 0x7fc07fc0u);  // bf16 qNaN pairs
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = nan4;
}

// NEXT-3: new K/V rows of the streaming heads -> device sink rows / ring rows (DuoAppendParams).  Only the
// rows that survive the call are written: p < n_sink (sink) or p >= pos0 + n - ring (the last `ring` rows).
__global__ void duo_append_kernel(const DuoAppendParams p, int cpr /* 16-byte chunks per row */) {
    const int64_t skip_lo = p.pos0 + p.n - p.ring;  // rows >= max(n_sink, skip_lo) stay in the ring
    const int64_t total = static_cast<int64_t>(p.n_heads) * p.n * cpr;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cpr);
        const int64_t yt = i / cpr;
        const int t = static_cast<int>(yt % p.n);
        const int y = static_cast<int>(yt / p.n);
        const int64_t pos = p.pos0 + t;
        int64_t row;
        if (pos < p.n_sink) row = pos;
        else if (pos >= skip_lo) row = p.n_sink + (pos - p.n_sink) % p.ring;
        else continue;
        const int h = p.heads[y];
        const int64_t so = h * p.src_head_stride + t * p.src_row_stride;
        __nv_bfloat16* dk = p.dst + h * p.dst_head_stride + row * (cpr * 8);
        reinterpret_cast<uint4*>(dk)[c] = reinterpret_cast<const uint4*>(p.src_k + so)[c];
        reinterpret_cast<uint4*>(dk + p.dst_v_off)[c] = reinterpret_cast<const uint4*>(p.src_v + so)[c];
    }
}

}  // namespace

cudaError_t launch_duo_append(const DuoAppendParams& p, int d, cudaStream_t stream) {
    const int cpr = d / 8;
    const int64_t total = static_cast<int64_t>(p.n_heads) * p.n * cpr;
    if (total == 0) return cudaSuccess;
    if (p.ring < 1 || p.n_heads > MAX_LAUNCH_HEADS) return cudaErrorInvalidValue;
    const int threads = 256;
    const int64_t want = (total + threads - 1) / threads;
    duo_append_kernel<<<static_cast<int>(want < 148 * 8 ? want : 148 * 8), threads, 0, stream>>>(p, cpr);
    return cudaGetLastError();
}

cudaError_t launch_pack_kv(const __nv_bfloat16* k, const __nv_bfloat16* v, __nv_bfloat16* packed, int n, int hkv,
                           int d, cudaStream_t stream) {
    const int cpr = d / 8;
    const int64_t total = static_cast<int64_t>(n) * hkv * cpr;
    if (total == 0) return cudaSuccess;
    const int threads = 256;
    const int64_t want = (total + threads - 1) / threads;
    const int grid = static_cast<int>(want < 148 * 8 ? want : 148 * 8);
    pack_kv_kernel<<<grid, threads, 0, stream>>>(reinterpret_cast<const uint4*>(k), reinterpret_cast<const uint4*>(v),
                                                 reinterpret_cast<uint4*>(packed), n, hkv, cpr);
    return cudaGetLastError();
}

cudaError_t launch_poison(void* ptr, size_t bytes, cudaStream_t stream) {
    const int64_t n16 = static_cast<int64_t>(bytes / 16);
    if (n16 == 0) return cudaSuccess;
    const int64_t want = (n16 + 255) / 256;
    poison_kernel<<<static_cast<int>(want < 148 * 8 ? want : 148 * 8), 256, 0, stream>>>(reinterpret_cast<uint4*>(ptr), n16);
    return cudaGetLastError();
}

// Hazard testing (HI_FLAG_JITTER / HI_FLAG_FAULT_SKIP_RAW): one thread holds its stream for
// `ns` nanoseconds of %globaltimer, delaying everything queued behind it on that stream.
__global__ void spin_kernel(uint64_t ns) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

cudaError_t launch_spin(uint64_t ns, cudaStream_t stream) {
    spin_kernel<<<1, 1, 0, stream>>>(ns);
    return cudaGetLastError();
}

// Fault injection (HI_FLAG_FAULT_LAUNCH / HI_FLAG_FAULT_TRAP, sticky-failure tests, SURVEY.md §8(b) "a CUDA
// error makes the ctx sticky-failed"): `trap` = a kernel that executes `trap` (asynchronous device fault, the
// CUDA context is lost); otherwise a launch with an invalid configuration (synchronous launch error, the CUDA
// context survives).
__global__ void trap_kernel() { asm volatile("trap;"); }

cudaError_t launch_fault(bool trap, cudaStream_t stream) {
    if (trap) {
        trap_kernel<<<1, 1, 0, stream>>>();
        return cudaGetLastError();
    }
    spin_kernel<<<1, 4096, 0, stream>>>(0);  // 4096 threads per block: cudaErrorInvalidConfiguration
    return cudaGetLastError();
}

}  // namespace hi
