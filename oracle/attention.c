/*
 * oracle/attention.c -- fp64 CPU oracle for HeadInfer's attention hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2502_12574_b200/); the only common dependency is the seeded input
 * generator in synth/, which holds none of the method's arithmetic.
 *
 * What it computes ("Definition"): HeadInfer is exact
 * ("exact mathematical equivalence", §1), so the oracle is plain
 * causal attention of one query row against the KV cache of ONE head:
 *
 *   Eq. 3 / Eq. 9:
 *       A_t^(h) = Softmax( Q_t^(h) K_cache^(h)T / sqrt(d_k) ) V_cache^(h)
 *
 *   written out step by step, for a query row q at global position p
 *   (keys 0..p are visible -- reading R2, bottom-right/global causal):
 *       s_i = (q . k_i) / sqrt(d)          0 <= i <= p      (d_k = head_dim, R1)
 *       m   = max_i s_i
 *       w_i = exp(s_i - m)
 *       o   = (sum_i w_i v_i) / (sum_i w_i)
 *
 * Every input is a bf16 bit pattern converted EXACTLY to double
 * (uint16 << 16 -> float -> double); every sum is a plain sequential loop in
 * key order; no blocking, fusion or reordering.  Build: -O2, no fast-math.
 *
 * Head-wise decomposition (Eq. 7-9) and GQA (reading R4,
 * kv(j) = floor(j/g)) are applied by the caller (oracle/oracle.py), which
 * passes each query row with the K/V of the kv head it reads.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double bf16_bits_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/*
 * oracle_attention_rows
 *   q_rows   [n_rows][d]        bf16 bits, query rows (row stride q_stride elements)
 *   last_key [n_rows]           p: the row attends keys 0..p inclusive (p < n_keys)
 *   K, V                        bf16 bits; key i's row starts at K + i*kv_stride
 *   out      [n_rows][d]        fp64 result
 * returns 0 on success, -1 on bad arguments, -2 on allocation failure.
 */
int oracle_attention_rows(const uint16_t* q_rows, int64_t n_rows, int64_t q_stride,
                          const int64_t* last_key,
                          const uint16_t* K, const uint16_t* V, int64_t n_keys, int64_t kv_stride,
                          int d, double* out) {
    if (n_rows < 0 || d <= 0 || n_keys < 0) return -1;
    for (int64_t r = 0; r < n_rows; ++r)
        if (last_key[r] < 0 || last_key[r] >= n_keys) return -1;
    int err = 0;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
#pragma omp parallel
    {
        double* s = NULL;
        int64_t s_cap = 0;
        double* q = (double*)malloc(sizeof(double) * (size_t)d);
        double* acc = (double*)malloc(sizeof(double) * (size_t)d);
        if (!q || !acc) {
#pragma omp atomic write
            err = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < n_rows; ++r) {
            if (err) continue;
            const int64_t p = last_key[r];
            if (p + 1 > s_cap) {
                free(s);
                s_cap = p + 1;
                s = (double*)malloc(sizeof(double) * (size_t)s_cap);
                if (!s) {
#pragma omp atomic write
                    err = -2;
                    s_cap = 0;
                    continue;
                }
            }
            for (int c = 0; c < d; ++c) q[c] = bf16_bits_to_double(q_rows[r * q_stride + c]);
            /* s_i = (q . k_i) / sqrt(d) */
            for (int64_t i = 0; i <= p; ++i) {
                const uint16_t* k = K + i * kv_stride;
                double dot = 0.0;
                for (int c = 0; c < d; ++c) dot += q[c] * bf16_bits_to_double(k[c]);
                s[i] = dot * inv_sqrt_d;
            }
            /* m = max_i s_i */
            double m = s[0];
            for (int64_t i = 1; i <= p; ++i)
                if (s[i] > m) m = s[i];
            /* w_i = exp(s_i - m);  o = sum w_i v_i / sum w_i */
            double wsum = 0.0;
            for (int c = 0; c < d; ++c) acc[c] = 0.0;
            for (int64_t i = 0; i <= p; ++i) {
                const double w = exp(s[i] - m);
                const uint16_t* v = V + i * kv_stride;
                wsum += w;
                for (int c = 0; c < d; ++c) acc[c] += w * bf16_bits_to_double(v[c]);
            }
            for (int c = 0; c < d; ++c) out[r * d + c] = acc[c] / wsum;
        }
        free(s);
        free(q);
        free(acc);
    }
    return err;
}

/*
 * oracle_attention_rows_duo -- the same row attention for a duo-attention STREAMING head
 * (NEXT-3; §4 "truncating less important heads to a fixed length", App. D;
 * DuoAttention's streaming heads keep the attention-sink tokens and a window of recent tokens,
 * reading R18 in DESIGN.md).  A query row at position p attends exactly the keys
 *       V(p) = { i : i <= p  and  ( i < n_sink  or  i > p - win ) }
 * (win <= 0: no truncation, V(p) = {0..p}, the retrieval-head rule above), written out as
 *       s_i = (q . k_i) / sqrt(d)   i in V(p)
 *       m = max_{i in V(p)} s_i;  w_i = exp(s_i - m);  o = sum w_i v_i / sum w_i
 * in key order, fp64, no blocking.  Arguments as oracle_attention_rows.
 */
int oracle_attention_rows_duo(const uint16_t* q_rows, int64_t n_rows, int64_t q_stride,
                              const int64_t* last_key, int64_t n_sink, int64_t win,
                              const uint16_t* K, const uint16_t* V, int64_t n_keys, int64_t kv_stride,
                              int d, double* out) {
    if (n_rows < 0 || d <= 0 || n_keys < 0 || n_sink < 0) return -1;
    for (int64_t r = 0; r < n_rows; ++r)
        if (last_key[r] < 0 || last_key[r] >= n_keys) return -1;
    int err = 0;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
#pragma omp parallel
    {
        double* q = (double*)malloc(sizeof(double) * (size_t)d);
        double* acc = (double*)malloc(sizeof(double) * (size_t)d);
        if (!q || !acc) {
#pragma omp atomic write
            err = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < n_rows; ++r) {
            if (err) continue;
            const int64_t p = last_key[r];
            for (int c = 0; c < d; ++c) q[c] = bf16_bits_to_double(q_rows[r * q_stride + c]);
            /* m = max over the visible keys of s_i (first pass), then the weighted sum (second pass) */
            double m = 0.0;
            int have = 0;
            for (int64_t i = 0; i <= p; ++i) {
                if (!(win <= 0 || i < n_sink || i > p - win)) continue;
                const uint16_t* k = K + i * kv_stride;
                double dot = 0.0;
                for (int c = 0; c < d; ++c) dot += q[c] * bf16_bits_to_double(k[c]);
                const double si = dot * inv_sqrt_d;
                if (!have || si > m) m = si;
                have = 1;
            }
            double wsum = 0.0;
            for (int c = 0; c < d; ++c) acc[c] = 0.0;
            for (int64_t i = 0; i <= p; ++i) {
                if (!(win <= 0 || i < n_sink || i > p - win)) continue;
                const uint16_t* k = K + i * kv_stride;
                double dot = 0.0;
                for (int c = 0; c < d; ++c) dot += q[c] * bf16_bits_to_double(k[c]);
                const double w = exp(dot * inv_sqrt_d - m);
                const uint16_t* v = V + i * kv_stride;
                wsum += w;
                for (int c = 0; c < d; ++c) acc[c] += w * bf16_bits_to_double(v[c]);
            }
            for (int c = 0; c < d; ++c) out[r * d + c] = acc[c] / wsum;
        }
        free(q);
        free(acc);
    }
    return err;
}

/* Threads the OpenMP runtime will use (reported as cpu_baseline.cores). */
int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
