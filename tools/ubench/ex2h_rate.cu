// Microbenchmark: exponentials per cycle per SMSP on sm_100a for the softmax's element pair
// sequences.  MODE 0: the product sequence (FFMA2 scale-and-shift, 2x MUFU ex2.f32, FADD2 row sum,
// F2FP bf16x2 pack).  MODE 1: packed half2 MUFU (ex2.approx.f16x2: one MUFU op per element pair),
// with FFMA2 -> cvt f16x2 -> ex2.f16x2 -> unpack to f32 -> FADD2 + F2FP bf16x2.  MODE 2: bare
// ex2.approx.f16x2.  MODE 3: bare ex2.approx.ftz.bf16x2.  MODE 4: bare ex2.approx.ftz.f32.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ex2h_rate.cu -o ex2h_rate
#include <cstdio>
#include <cuda_runtime.h>

struct f2 { float x, y; };
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r)
                 : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
                   "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<f2*>(&r);
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
    unsigned long long r;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r)
                 : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<f2*>(&r);
}
__device__ __forceinline__ unsigned pack_bf16(float lo, float hi) {
    unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r;
}

template <int MODE>
__global__ void kern(float* out, int iters, long long* cyc) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-4f + i * 1e-3f - 3.f;
    f2 acc[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    unsigned pk = 0;
    const f2 sc{1.0001f, 1.0001f}, nm{-0.5f, -0.5f};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (MODE == 0) {
                const f2 s = ffma2(f2{a[i], a[i + 1]}, sc, nm);
                float p0, p1;
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(s.x));
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(s.y));
                acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], f2{p0, p1});
                pk ^= pack_bf16(p0, p1);
                a[i] = p0 - 3.f; a[i + 1] = p1 - 3.f;
            } else if (MODE == 1) {
                const f2 s = ffma2(f2{a[i], a[i + 1]}, sc, nm);
                unsigned h, e;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(s.y), "f"(s.x));
                asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
                float p0, p1;
                asm volatile("{.reg .f16 l, u; mov.b32 {l, u}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, u;}"
                             : "=f"(p0), "=f"(p1) : "r"(e));
                acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], f2{p0, p1});
                pk ^= pack_bf16(p0, p1);
                a[i] = p0 - 3.f; a[i + 1] = p1 - 3.f;
            } else if (MODE == 2) {
                unsigned h = __float_as_uint(a[i]), e;
                asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
                a[i] = __uint_as_float(e ^ 0x3c003c00u);
            } else if (MODE == 3) {
                unsigned h = __float_as_uint(a[i]), e;
                asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(e) : "r"(h));
                a[i] = __uint_as_float(e ^ 0x3f803f80u);
            } else {
                float y0, y1;
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(a[i]));
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(a[i + 1]));
                a[i] = y0 - 3.f; a[i + 1] = y1 - 3.f;
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 64 + threadIdx.x / 32] = t1 - t0;
    float s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc[0].x + acc[1].y + acc[2].x + acc[3].y + pk;
}

template <int MODE>
void run(const char* name, int warps) {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 64 * 8);
    const int iters = 4096;
    kern<MODE><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    kern<MODE><<<148, warps * 32>>>(out, iters, cyc);
    long long h[64];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int w = 0; w < warps; ++w) c += h[w];
    c /= warps;
    const double elems = 32.0 * (warps / 4) * iters * 16;  // elements per SMSP
    printf("%-26s warps/SMSP=%d: %.2f elements (exponentials) per cycle per SMSP\n", name, warps / 4, elems / c);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8}) {
        run<0>("softmax pair f32 MUFU", w);
        run<1>("softmax pair f16x2 MUFU", w);
        run<2>("ex2.approx.f16x2", w);
        run<3>("ex2.approx.ftz.bf16x2", w);
        run<4>("ex2.approx.ftz.f32", w);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
