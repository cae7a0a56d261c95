// Microbenchmark: issue throughput of ex2.approx (MUFU), cvt.rn.bf16x2.f32 (F2FP) and FFMA per SMSP
// on sm_100a, with 1 or 2 warps per SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 xu_rate.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(float* out, int iters, long long* cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f - 3.f;
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {  // MUFU ex2
                float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y - 3.f;
            } else if (MODE == 1) {  // F2FP pack
                __nv_bfloat162 h = __floats2bfloat162_rn(a[i], a[(i + 1) & 7]);
                acc += *reinterpret_cast<unsigned*>(&h);
                a[i] += 1e-7f;
            } else if (MODE == 2) {  // FFMA
                a[i] = fmaf(a[i], 1.0001f, -1e-5f);
            } else {  // MUFU + F2FP interleaved (softmax-like)
                float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
                __nv_bfloat162 h = __floats2bfloat162_rn(y, a[(i + 1) & 7]);
                acc += *reinterpret_cast<unsigned*>(&h);
                a[i] = y - 3.f;
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 64 + threadIdx.x / 32] = t1 - t0;
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

template <int MODE>
void run(const char* name, int warps) {
    float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 64 * 8);
    int iters = 4096;
    kern<MODE><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    kern<MODE><<<148, warps * 32>>>(out, iters, cyc);
    long long h[64]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int w = 0; w < warps; ++w) c += h[w]; c /= warps;
    double per_instr = c / (iters * 8.0);
    printf("%-12s warps/CTA=%2d (warps/SMSP=%d): %.2f cycles per warp-instr per warp; SMSP rate %.2f lanes/cycle\n",
           name, warps, warps / 4, per_instr, 32.0 * (warps / 4) / per_instr);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>("ex2", w);
        run<1>("f2fp_bf16x2", w);
        run<2>("ffma", w);
        run<3>("ex2+f2fp", w);
    }
    return 0;
}
