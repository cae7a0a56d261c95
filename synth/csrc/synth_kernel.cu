// synth_kernel.cu -- CUDA twin of synth/gen.py (seeded counter-hash bf16 generator).
// Shared TEST/BENCH infrastructure: holds none of the method's arithmetic.  Must produce the
// same bits as gen_block() (pinned by tests/test_gpu_synth.py).  C ABI:
//   int synth_fill(void* dst, uint64_t seed, int tensor, int dist, int layer, int head0, int n_heads,
//                  int64_t pos0, int64_t n_pos, int d, int64_t tok_stride, void* stream)
// writes dst[(t*tok_stride) + h*d + c] for t < n_pos, h < n_heads, c < d  (bf16 bits).
// dist: 0=U 1=P 2=S 3=ONE; tensor: 0=Q 1=K 2=V.  Returns 0 or a cudaError_t.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t bf16_rne(float x) {
    const uint32_t u = __float_as_uint(x);
    return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

__global__ void synth_kernel(uint16_t* dst, uint64_t seedmix, int tensor, int dist, int layer, int head0, int n_heads,
                             int64_t pos0, int64_t n_pos, int d, int64_t tok_stride) {
    const int64_t total = n_pos * n_heads * d;
    const float scale = (dist == 1 && tensor == 0) ? 16.f : 1.f;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % d);
        const int h = static_cast<int>((i / d) % n_heads);
        const int64_t t = i / (static_cast<int64_t>(d) * n_heads);
        const int64_t pos = pos0 + t;
        uint16_t bits;
        if ((dist == 3 && tensor == 2) || (dist == 2 && tensor == 1 && pos == 0)) {
            bits = 0x3F80;
        } else {
            const uint64_t key =
                ((((static_cast<uint64_t>(tensor * 128 + layer) * 128 + static_cast<uint64_t>(head0 + h)) << 23) |
                  static_cast<uint64_t>(pos))
                 << 8) |
                static_cast<uint64_t>(c);
            const uint64_t hsh = splitmix64(key ^ seedmix);
            const int64_t v = static_cast<int64_t>(hsh >> 40) - (1 << 23);
            float x = static_cast<float>(v) * (1.0f / 8388608.0f) * scale;
            if (dist == 2 && tensor == 0) x = fabsf(x);
            bits = bf16_rne(x);
        }
        dst[t * tok_stride + static_cast<int64_t>(h) * d + c] = bits;
    }
}

}  // namespace

extern "C" int synth_fill(void* dst, uint64_t seed, int tensor, int dist, int layer, int head0, int n_heads,
                          int64_t pos0, int64_t n_pos, int d, int64_t tok_stride, void* stream) {
    const int64_t total = n_pos * n_heads * d;
    if (total <= 0) return 0;
    const uint64_t seedmix = seed * 0x9E3779B97F4A7C15ull;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    synth_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint16_t*>(dst), seedmix, tensor, dist, layer, head0, n_heads, pos0, n_pos, d, tok_stride);
    return static_cast<int>(cudaGetLastError());
}
