// k_prefill_mma.cu -- prefill attention over one KV segment, resumable flash-attention state.
//
// for q head j of group h and chunk positions p in [s, s+n),
//   o = sum_{i<=p} softmax_i(q_p . k_i / sqrt(d)) v_i          (Eq. 9)
// over history (staging-slot blocks) U chunk (causal, reading R2).  Each launch folds one
// contiguous key segment into the running state (O, m, l) kept in HBM, so history blocks can
// be consumed in the order the copy engine lands them (Alg. 1 line 10/13).
//
// BASELINE COMPARATOR (HI_FLAG_MMA_SYNC_PREFILL): the pre-Blackwell tensor-core path: warp-level mma.sync m16n8k16 bf16 with
// fp32 accumulation, cp.async double-buffered K/V tiles, XOR-swizzled shared memory and
// ldmatrix operand loads.  Tile: 128 query rows (GQA-packed: rows r = t*g + j) x 64 keys,
// 8 warps x 16 rows.
#include "../hi_kernels.cuh"

#include <cuda_bf16.h>
#include <math_constants.h>

namespace hi {
namespace {

constexpr int BM = 128;
constexpr int BN = 64;
constexpr int NWARPS = 8;
constexpr int NTHREADS = NWARPS * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
    return y;
}

// Swizzled byte offset of 16-byte chunk `c` in row `r` of a [rows][D] bf16 tile.
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
    return static_cast<uint32_t>(r * (D * 2) + ((c ^ (r & 7)) << 4));
}

template <int D>
__global__ void __launch_bounds__(NTHREADS, 2) prefill_mma_kernel(const PrefillParams p) {
    constexpr int CH = D / 8;  // 16-byte chunks per row
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* sQ = smem;                       // BM x D
    uint8_t* sK = sQ + BM * D * 2;            // 2 stages x BN x D
    uint8_t* sV = sK + 2 * BN * D * 2;        // 2 stages x BN x D

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int g = p.g;
    const int n_rows = p.n_q * g;
    const int row0 = blockIdx.x * BM;
    const bool first = p.flags & PF_FIRST;
    const bool last = p.flags & PF_LAST;
    const bool causal = p.flags & PF_CAUSAL;

    // ---- keys visible to this tile: key c (segment-relative) visible to token t iff
    //      k_pos0 + c <= q_pos0 + t  (bottom-right / global causal, reading R2)
    const int t_lo = row0 / g;
    const int t_hi = min(p.n_q - 1, (row0 + BM - 1) / g);
    int n_k_eff = p.n_k;
    if (causal) {
        const int64_t lim = p.q_pos0 + t_hi - p.k_pos0 + 1;
        int64_t e = lim < n_k_eff ? lim : static_cast<int64_t>(n_k_eff);
        n_k_eff = static_cast<int>(e > 0 ? e : 0);
    }
    const int n_kt = (n_k_eff + BN - 1) / BN;

    // ---- load Q tile (GQA packed rows) ------------------------------------------------
    for (int i = tid; i < BM * CH; i += NTHREADS) {
        const int r = i / CH, c = i % CH;
        const int rg = row0 + r;
        const bool valid = rg < n_rows;
        const int t = valid ? rg / g : 0, j = valid ? rg % g : 0;
        const __nv_bfloat16* src = p.q + static_cast<int64_t>(t) * p.q_tok_stride + j * D + c * 8;
        cp_async16(smem_u32(sQ + swz<D>(r, c)), src, valid);
    }
    auto load_kv = [&](int stage, int kt) {
        uint8_t* dk = sK + stage * BN * D * 2;
        uint8_t* dv = sV + stage * BN * D * 2;
        for (int i = tid; i < BN * CH; i += NTHREADS) {
            const int r = i / CH, c = i % CH;
            const int key = kt * BN + r;
            const bool valid = key < n_k_eff;
            const int64_t off = static_cast<int64_t>(valid ? key : 0) * p.kv_row_stride + c * 8;
            cp_async16(smem_u32(dk + swz<D>(r, c)), p.k + off, valid);
            cp_async16(smem_u32(dv + swz<D>(r, c)), p.v + off, valid);
        }
    };
    if (n_kt > 0) load_kv(0, 0);
    cp_async_commit();

    // ---- running state: rows rA = warp*16 + lane/4 and rB = rA + 8 ----------------------
    const int gid = lane >> 2, tq = lane & 3;
    const int rA = row0 + warp * 16 + gid, rB = rA + 8;
    float o[D / 8][4];
    float m_r[2], l_r[2];
    if (first) {
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
        m_r[0] = m_r[1] = -CUDART_INF_F;
        l_r[0] = l_r[1] = 0.f;
    } else {
        const bool va = rA < n_rows, vb = rB < n_rows;
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
            const int col = nt * 8 + tq * 2;
            float2 a = va ? *reinterpret_cast<const float2*>(p.o_acc + static_cast<int64_t>(rA) * D + col) : make_float2(0.f, 0.f);
            float2 b = vb ? *reinterpret_cast<const float2*>(p.o_acc + static_cast<int64_t>(rB) * D + col) : make_float2(0.f, 0.f);
            o[nt][0] = a.x; o[nt][1] = a.y; o[nt][2] = b.x; o[nt][3] = b.y;
        }
        m_r[0] = va ? p.m_acc[rA] : -CUDART_INF_F;
        m_r[1] = vb ? p.m_acc[rB] : -CUDART_INF_F;
        // l is kept as per-thread partial sums (reduced across the quad at the end)
        l_r[0] = (va && tq == 0) ? p.l_acc[rA] : 0.f;
        l_r[1] = (vb && tq == 0) ? p.l_acc[rB] : 0.f;
    }

    cp_async_wait<0>();
    __syncthreads();
    // positions for masking
    const int tA = rA / g, tB = rB / g;
    const int64_t posA = p.q_pos0 + tA, posB = p.q_pos0 + tB;
    const int64_t pos_lo = p.q_pos0 + t_lo;

    for (int kt = 0; kt < n_kt; ++kt) {
        const int stage = kt & 1;
        if (kt + 1 < n_kt) load_kv(stage ^ 1, kt + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const uint8_t* cK = sK + stage * BN * D * 2;
        const uint8_t* cV = sV + stage * BN * D * 2;

        // S = Q K^T  (16 rows x 64 keys per warp)
        float s[BN / 8][4];
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            uint32_t qf[4];  // Q fragment (16 rows x 16 dims), re-read from shared memory
            ldsm_x4(smem_u32(sQ + swz<D>(warp * 16 + (lane & 15), ks * 2 + (lane >> 4))), qf[0], qf[1], qf[2], qf[3]);
#pragma unroll
            for (int np = 0; np < BN / 16; ++np) {
                const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
                const int c = ks * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(smem_u32(cK + swz<D>(key, c)), b0, b1, b2, b3);
                mma_bf16(s[2 * np], qf, b0, b1);
                mma_bf16(s[2 * np + 1], qf, b2, b3);
            }
        }
        // scale to log2 domain + mask
        const int key0 = kt * BN;
        const int64_t kpos_hi = p.k_pos0 + key0 + BN - 1;
        const bool need_mask = (key0 + BN > n_k_eff) || (causal && kpos_hi > pos_lo);
        float mx[2] = {-CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float x = s[nt][e] * p.scale_log2;
                if (need_mask) {
                    const int key = key0 + nt * 8 + tq * 2 + (e & 1);
                    const int64_t kp = p.k_pos0 + key;
                    const int64_t qp = (e < 2) ? posA : posB;
                    if (key >= n_k_eff || (causal && kp > qp)) x = -CUDART_INF_F;
                }
                s[nt][e] = x;
                mx[e >> 1] = fmaxf(mx[e >> 1], x);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
        }
        float alpha[2], muse[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float m_new = fmaxf(m_r[h], mx[h]);
            muse[h] = (m_new == -CUDART_INF_F) ? 0.f : m_new;
            alpha[h] = fast_exp2(m_r[h] - muse[h]);  // m_r = -inf -> 0
            m_r[h] = m_new;
            l_r[h] *= alpha[h];
        }
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
            o[nt][0] *= alpha[0]; o[nt][1] *= alpha[0];
            o[nt][2] *= alpha[1]; o[nt][3] *= alpha[1];
        }
        // P = 2^(x - m), as bf16 A fragments; O += P V
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
            float p0 = fast_exp2(s[2 * kk][0] - muse[0]), p1 = fast_exp2(s[2 * kk][1] - muse[0]);
            float p2 = fast_exp2(s[2 * kk][2] - muse[1]), p3 = fast_exp2(s[2 * kk][3] - muse[1]);
            float p4 = fast_exp2(s[2 * kk + 1][0] - muse[0]), p5 = fast_exp2(s[2 * kk + 1][1] - muse[0]);
            float p6 = fast_exp2(s[2 * kk + 1][2] - muse[1]), p7 = fast_exp2(s[2 * kk + 1][3] - muse[1]);
            l_r[0] += p0 + p1 + p4 + p5;
            l_r[1] += p2 + p3 + p6 + p7;
            uint32_t a[4] = {pack_bf16(p0, p1), pack_bf16(p2, p3), pack_bf16(p4, p5), pack_bf16(p6, p7)};
#pragma unroll
            for (int dn = 0; dn < D / 16; ++dn) {
                const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = dn * 2 + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(smem_u32(cV + swz<D>(key, c)), b0, b1, b2, b3);
                mma_bf16(o[2 * dn], a, b0, b1);
                mma_bf16(o[2 * dn + 1], a, b2, b3);
            }
        }
        __syncthreads();
    }

    // ---- epilogue ----------------------------------------------------------------------
    if (last) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
            l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
        }
        const float invA = l_r[0] > 0.f ? 1.f / l_r[0] : 0.f;
        const float invB = l_r[1] > 0.f ? 1.f / l_r[1] : 0.f;
        if (rA < n_rows) {
            __nv_bfloat16* dst = p.out + static_cast<int64_t>(tA) * p.o_tok_stride + (rA % g) * D;
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt)
                *reinterpret_cast<uint32_t*>(dst + nt * 8 + tq * 2) = pack_bf16(o[nt][0] * invA, o[nt][1] * invA);
        }
        if (rB < n_rows) {
            __nv_bfloat16* dst = p.out + static_cast<int64_t>(tB) * p.o_tok_stride + (rB % g) * D;
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt)
                *reinterpret_cast<uint32_t*>(dst + nt * 8 + tq * 2) = pack_bf16(o[nt][2] * invB, o[nt][3] * invB);
        }
    } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
            l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
        }
        if (rA < n_rows) {
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt)
                *reinterpret_cast<float2*>(p.o_acc + static_cast<int64_t>(rA) * D + nt * 8 + tq * 2) = make_float2(o[nt][0], o[nt][1]);
            if (tq == 0) { p.m_acc[rA] = m_r[0]; p.l_acc[rA] = l_r[0]; }
        }
        if (rB < n_rows) {
#pragma unroll
            for (int nt = 0; nt < D / 8; ++nt)
                *reinterpret_cast<float2*>(p.o_acc + static_cast<int64_t>(rB) * D + nt * 8 + tq * 2) = make_float2(o[nt][2], o[nt][3]);
            if (tq == 0) { p.m_acc[rB] = m_r[1]; p.l_acc[rB] = l_r[1]; }
        }
    }
}

template <int D>
cudaError_t launch_d(const PrefillParams& p, cudaStream_t stream) {
    const size_t smem = (BM + 4 * BN) * D * 2;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(prefill_mma_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int n_rows = p.n_q * p.g;
    const int grid = (n_rows + BM - 1) / BM;
    if (grid == 0) return cudaSuccess;
    prefill_mma_kernel<D><<<grid, NTHREADS, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prefill_mma(const PrefillParams& p, int d, cudaStream_t stream) {
    if (d == 64) return launch_d<64>(p, stream);
    if (d == 128) return launch_d<128>(p, stream);
    return cudaErrorInvalidValue;
}

}  // namespace hi
