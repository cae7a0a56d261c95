// k_prefill_tc.cu -- sm_100a prefill attention over one KV segment: TMA -> SMEM -> tcgen05.mma
// with S and O accumulators in TMEM, fp32 online softmax on CUDA cores, warp-specialised.
//
// for q head j of group h and chunk positions p in [s, s+n),
//   o = sum_{i<=p} softmax_i(q_p . k_i / sqrt(d)) v_i                  (Eq. 9)
// over history (staging-slot blocks) and the chunk itself (causal, reading R2).  A launch folds
// ONE contiguous key segment into the running state (O, m, l) held in HBM (same contract as the
// baseline k_prefill_mma.cu), so history blocks are consumed in the order the copy engine lands
// them (Alg. 1 line 10/13).  Prefill is a dense contraction (compute-bound for
// S >= 10K, §5), so both products run on the 5th-gen tensor cores:
//
//   S = Q K^T   tcgen05.mma kind::f16, A = Q tile (SMEM, K-major SW128), B = K tile (SMEM,
//               K-major SW128), D = S in TMEM (fp32, 128 lanes x 128 cols per Q tile)
//   O += P V    A = P (bf16, in TMEM over the S columns, written by the softmax warps),
//               B = V tile (SMEM, MN-major SW128), D = O in TMEM (fp32, 128 lanes x d cols)
//
// CTA = two 128-row Q tiles (GQA-packed: row r = t*g + j, loaded by one 3-D TMA box per 64
// columns) sharing every K/V tile of 128 keys (halves the K/V SMEM/L2 traffic per FLOP).  Warps 0-3
// own tile 0 and warps 4-7 tile 1 (softmax + O correction + epilogue; thread i owns TMEM lane /
// row 32*(w%4)+i); warp 8: TMA producer (K and V stages released on separate barriers); warp 9: TMEM
// allocator + MMA issuer (the whole warp runs the issue loop, elect.sync issues).  P is written back into
// the S columns of TMEM as packed bf16 in two 64-key halves, each consumed from TMEM by its part of the PV
// MMA (A operand in TMEM), so P never touches shared memory; the MMA issuer alternates between the two
// tiles, so one tile's softmax overlaps the other tile's QK^T / PV on the tensor core.
// Online softmax in the log2 domain with lazy rescaling (the O correction is applied only when a
// row max grows by more than 2^8), which is exact: O/l does not depend on the reference max.
//
// Compile-time switches.  The product build uses the defaults; every other setting is an A/B experiment built only
// through build.build_variant (-D...), kept with its measurement so the choice stays checkable
// (profiles/prefill_probe_r02.jsonl; TFLOP/s per GHz in the sustained 1M probe, product ~760):
//   HI_WARP_ISSUE=1      whole-warp MMA issue, elect.sync per MMA          (lane-0 issue: -10.7 % per clock)
//   HI_SPLIT_S=2         P released in two halves, PV(j)_lo early           (=0 one piece 679; =1 S_lo early 731)
//   HI_P_SPLIT_KEYS=64   split point                                         (96: -0.3 %)
//   HI_P_PARTS=2         halves                                              (4 quarters: 742)
//   HI_KV_JOINT=0        K and V stages released separately                  (joint: -1.8 %, fake-softmax -8 %)
//   HI_SOFTMAX_SPLIT=1   one softmax warp per row quarter and tile           (2: spills, 0.85-0.9x in round 1)
//   HI_SUMCHECK=0        max-first lazy rescale                              (sum-checked: 668)
//   HI_PINGPONG=0        free-running exponential phases                     (MUFU token ping-pong: 670)
//   HI_POLY_MASK8/PAIRS  all exponentials on MUFU                             (1/8 on the FMA pipe: +0.8 %/clk, -clock)
//   HI_SPEC_EXP/SPLIT=0  max before the exponentials                          (speculative first half: -3 %)
//   HI_TWO_ISSUERS=0     one MMA issuer warp                                 (one per tile: 523)
//   HI_DESC_LO=0         64-bit descriptors                                  (low words: 743)
//   HI_TILE_MIX=0        tile 1 = warps 4-7 (wins issue arbitration on every SMSP)  (interleaved: 744)
//   HI_O_COMMIT_FIRST=1  final O commit before the last stage release        (after it: 748 vs 759)
//   HI_MMA_SPIN=0, HI_WAIT_HINT(_MMA)=0: try_wait without a suspend hint     (polling: 711; 2 us hint on the MMA warp: -5 %)
//   HI_FAKE_SOFTMAX / HI_FAKE_MAX / HI_SKIP_S / HI_SKIP_PV: timing-only (wrong results), never in the product
//   HI_TRACE: CTA-0 clock64() timeline (hi_debug_prefill_trace), tools/trace_prefill.py
#include "hi_kernels.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdio>
#include <mutex>
#include <type_traits>

namespace hi {
namespace {

constexpr int BM = 128;            // query rows per CTA (TMEM lanes)
constexpr int BN = 128;            // keys per KV tile
constexpr int NS = 2;              // K/V pipeline stages
#ifndef HI_SOFTMAX_SPLIT
#define HI_SOFTMAX_SPLIT 1
#endif
#ifndef HI_SPEC_EXP
#define HI_SPEC_EXP 0  // measured: no gain (profiles/ab_prefill_r01.txt)
#endif
constexpr bool SPEC_EXP = HI_SPEC_EXP != 0;
// Speculative first half on the split schedule (the tile max off the critical path), see the softmax.
#ifndef HI_SPEC_SPLIT
#define HI_SPEC_SPLIT 0
#endif
constexpr bool SPEC_SPLIT = HI_SPEC_SPLIT != 0;
// SPLIT softmax warps per TMEM lane quarter and tile, each owning BN/SPLIT S columns of its rows
// (and D/SPLIT O columns).  MUFU ex2 issues at 4 lanes/clk/SMSP (profiles/ubench_xu_rate_r01.txt), so
// with one softmax warp per SMSP and tile the exponentials of a 128 x 128 tile alone take 1024 cycles
// = the tensor time of PV + the next QK^T; a second warp per SMSP lets the FMA-pipe polynomial of one
// warp issue while the other waits on MUFU, and halves each warp's serial chain.
constexpr int SPLIT = HI_SOFTMAX_SPLIT;
constexpr int SOFTMAX_WARPS = 8 * SPLIT;
constexpr int WARP_TMA = SOFTMAX_WARPS, WARP_MMA = SOFTMAX_WARPS + 1;
constexpr int NUM_THREADS = 32 * (SOFTMAX_WARPS + 4);  // + one warpgroup: TMA warp, MMA warp, 2 idle
// Register budget (setmaxnreg).  setmaxnreg.inc only draws on registers that setmaxnreg.dec released
// in the same CTA (it blocks forever otherwise), so  softmax threads x (inc - launch)  must equal at
// most  producer threads x (launch - dec):
//   SPLIT=1, d=128: launch 168 x 384; softmax 208 (+40 x 256), producer 88 (-80 x 128)
//   SPLIT=1, d=64:  softmax 216 (+48 x 256), producer 72 (-96 x 128): the d = 64 issuer needs fewer descriptor
//                   registers and its softmax loop spills its counter at 208 (the d = 128 issuer spills at 72)
//   SPLIT=2: launch  96 x 640; softmax 104 (+8 x 512), producer 64 (-32 x 128)
#ifndef HI_REG_SOFTMAX
#define HI_REG_SOFTMAX (SPLIT == 1 ? (D == 64 ? 216 : 208) : 104)
#endif
#ifndef HI_REG_PRODUCER
#define HI_REG_PRODUCER (SPLIT == 1 ? (D == 64 ? 72 : 88) : 64)
#endif
template <int D> constexpr int REG_SOFTMAX = HI_REG_SOFTMAX;
template <int D> constexpr int REG_PRODUCER = HI_REG_PRODUCER;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units
// HI_WARP_ISSUE: the MMA warp runs the issue loop with all 32 lanes and elect.sync picks the issuing lane inside
// each tcgen05.mma / commit.  From a lane-0-only region ptxas wraps every UTCHMMA in a waterfall loop (ELECT,
// R2UR.BROADCAST, BRA.U.ANY) whose cost per MMA is close to the 64 cycles an M128 N128 K16 MMA runs, so the
// issuer throttled the tensor pipe: measured +5.3 % TFLOP/s (+10.7 % per clock) in the sustained 1M probe
// (profiles/prefill_probe_r02.jsonl, 3 interleaved repetitions); a rolled issue loop, the other direction,
// costs 12 %.  0 = the round-1 lane-0 issue.
#ifndef HI_WARP_ISSUE
#define HI_WARP_ISSUE 1
#endif
// HI_DESC_LO=1 (A/B, off; with HI_WARP_ISSUE): pass only the descriptors' low words (the high word is the constant
// DESC_HI): ~13 instead of ~19 issuer instructions per tcgen05.mma, parity-green, but 743 vs 765 TFLOP/s per GHz in
// the sustained probe (job AO) -- a faster issuer is not a faster kernel here (see also HI_MMA_SPIN)
#ifndef HI_DESC_LO
#define HI_DESC_LO 0
#endif
#if HI_WARP_ISSUE && HI_DESC_LO
#define HI_UMMA(d, a, b, i, acc) umma_bf16_wl(d, static_cast<uint32_t>(a), static_cast<uint32_t>(b), i, acc)
#define HI_UMMA_TS(d, a, b, i, acc) umma_bf16_ts_wl(d, a, static_cast<uint32_t>(b), i, acc)
#define HI_UCOMMIT umma_commit_w
#elif HI_WARP_ISSUE
#define HI_UMMA umma_bf16_w
#define HI_UMMA_TS umma_bf16_ts_w
#define HI_UCOMMIT umma_commit_w
#else
#define HI_UMMA umma_bf16
#define HI_UMMA_TS umma_bf16_ts
#define HI_UCOMMIT umma_commit
#endif
// HI_SUMCHECK=1 (A/B, off): on unmasked tiles the split schedule exponentiates against the running reference and
// checks each half's row sum against 2^8 instead of taking the 128-key row max first (see the softmax).  Exact and
// parity-green, but measured 9 % slower per clock (668 vs 730 TFLOP/s per GHz, profiles/prefill_probe_r02.jsonl,
// job AH): without the max phase the two tiles' exponential phases collide on the MUFU more often.
#ifndef HI_SUMCHECK
#define HI_SUMCHECK 0
#endif
// HI_TWO_ISSUERS=1 (A/B): each Q tile's MMAs are issued by its own warp (warp 9: tile 0, warp 10: tile 1), each
// waiting only on its own tile's barriers (no fixed A-then-B issue order), with per-tile K/V release barriers
#ifndef HI_TWO_ISSUERS
#define HI_TWO_ISSUERS 0
#endif
#ifndef HI_TILE_MIX
#define HI_TILE_MIX 0
#endif
static_assert(!HI_TILE_MIX || HI_SOFTMAX_SPLIT == 1, "tile mix: one softmax warp per row quarter");
// HI_O_COMMIT_FIRST=1 (default): the final O commit precedes the last stage release.  The reverse order (=0, the
// CTA's last commit is the one its epilogue waits for) measured 1.3 % slower per clock (748 vs 759, job AZ); the
// stage-release arrival tracks the same MMAs and lands while the epilogue drains O (thousands of cycles)
#ifndef HI_O_COMMIT_FIRST
#define HI_O_COMMIT_FIRST 1
#endif
// HI_KV_JOINT=1 (A/B only): the producer loads K(i) only once V(i - NS) is released too, in K(i), V(i) order -- the
// round-1 prefetch distance (one tile step for K) with the separate barriers
#ifndef HI_KV_JOINT
#define HI_KV_JOINT 0
#endif
// HI_WAIT_HINT=<ns> (A/B): the softmax warps wait for S with a suspend-time hint
#ifndef HI_WAIT_HINT
#define HI_WAIT_HINT 0
#endif
// HI_WAIT_HINT_MMA=<ns> (A/B): the same for the MMA warp's waits (it has the highest warp id on its SMSP, and the
// scheduler issues highest-wid-first, so a polling issuer takes slots from softmax warps 1 and 5)
#ifndef HI_WAIT_HINT_MMA
#define HI_WAIT_HINT_MMA 0
#endif
#ifndef HI_MMA_SPIN
#define HI_MMA_SPIN 0   // A/B: the MMA warp polls with the non-blocking test_wait instead of try_wait
#endif
#if HI_WAIT_HINT_MMA
#define MMA_WAIT(bar, par) mbar_wait_hint(bar, par, HI_WAIT_HINT_MMA)
#elif HI_MMA_SPIN
#define MMA_WAIT(bar, par) do { while (!mbar_test(bar, par)) { } } while (0)
#else
#define MMA_WAIT(bar, par) mbar_wait(bar, par)
#endif
// HI_ROLL_ISSUE: keep the MMA issuer's K-step loops rolled (fewer live descriptors: no spills at the 64 registers
// the issuer gets with SPLIT = 2)
#ifndef HI_ROLL_ISSUE
#define HI_ROLL_ISSUE 0
#endif
#if HI_ROLL_ISSUE
#define HI_ISSUE_UNROLL _Pragma("unroll 1")
#else
#define HI_ISSUE_UNROLL _Pragma("unroll")
#endif

// Optional timeline trace (variant builds with -DHI_TRACE): clock64() at pipeline events of CTA 0,
// read back with hi_debug_prefill_trace(); off in the product build.
#ifdef HI_TRACE
__device__ unsigned long long g_hi_trace[16][512];
#define HI_TR(ev, j) do { if (blockIdx.x == 0 && (threadIdx.x & 127) == 0 && (j) < 512) g_hi_trace[ev][j] = clock64(); } while (0)
#define HI_TR_MMA(ev, j) do { if (blockIdx.x == 0 && (j) < 512) g_hi_trace[ev][j] = clock64(); } while (0)
// stamp once register v has arrived (a TMEM load completes through the scoreboard, not at tcgen05.wait::ld)
#define HI_TR_DEP(ev, j, v) do { uint32_t z_; asm volatile("and.b32 %0, %1, 0;" : "=r"(z_) : "r"(v)); \
    if (blockIdx.x == 0 && (threadIdx.x & 127) == 0 && (j) < 512) g_hi_trace[ev][j] = clock64() + z_; } while (0)
#else
#define HI_TR_DEP(ev, j, v) do { } while (0)
#define HI_TR(ev, j) do { } while (0)
#define HI_TR_MMA(ev, j) do { } while (0)
#endif
#ifndef HI_EX2_POLY_EVERY
#define HI_EX2_POLY_EVERY 1000000  // off: MUFU + polynomial measured slower (profiles/ab_prefill_r01.txt)
#endif
constexpr int EX2_POLY_EVERY = HI_EX2_POLY_EVERY;  // 2 of every 16 exponentials on the FMA pipe (see ex2_poly)
// Packed softmax (sm_100 FFMA2/FADD2): of every 4 element pairs, POLY_PAIRS go through the packed
// FMA-pipe polynomial (ex2_poly2), the rest through MUFU; -1 = the scalar loop.  Measured (131K probe,
// profiles/ab_prefill_r01.txt): packed 0 +1.3% over scalar; 1 and 2 polynomial pairs slower.
#ifndef HI_POLY_PAIRS
#define HI_POLY_PAIRS 0
#endif
constexpr int POLY_PAIRS = HI_POLY_PAIRS;
// Finer choice of the polynomial pairs on the split schedule: bit k of HI_POLY_MASK8 sends element pair i
// (i % 8 == k) to ex2_poly2 (tools/ubench/softmax_row.cu: one warp per SMSP, 3 pairs in 8 = 0x52 run a row's
// exponentials at 3.43/cycle against 2.90 all-MUFU).  0 = all MUFU (or HI_POLY_PAIRS).
#ifndef HI_POLY_MASK8
#define HI_POLY_MASK8 0
#endif
constexpr unsigned POLY_MASK8 = HI_POLY_MASK8;
__device__ __forceinline__ constexpr bool poly_pair(int pair) {
    return POLY_MASK8 ? ((POLY_MASK8 >> (pair & 7)) & 1u) != 0 : (pair & 3) < POLY_PAIRS;
}
// Split schedule (SPLIT == 1): P(j) goes to the upper 64 S columns, so QK^T of the next KV tile's first 64
// keys (S_lo, columns 0-63) can run as soon as the softmax has read S(j) into registers; the softmax
// releases P in two key halves, so PV(j) over the first 64 keys overlaps the second half's
// exponentials.  What remains in series per tile is softmax -> PV(j)_hi + S(j+1)_hi (512 cycles of MMA
// instead of 1024).
// HI_SPLIT_S = 2: only PV is split (P stays in the lower S columns; S(j+1) is one N = 128 MMA after
// PV(j)_hi).  Measured: SS MMAs with N = 64 run at 2/3 rate (A + B operand reads exceed SMEM bandwidth,
// profiles/ubench_mma_rate_r01.txt), so mode 1's S halves cost more than they overlap.
#ifndef HI_SPLIT_S
#define HI_SPLIT_S 2
#endif
constexpr bool SPLIT_S = HI_SPLIT_S != 0;
// Ping-pong of the exponential phases (split schedule): the two tiles' softmax warps on one SMSP (warps q and
// q + 4) take turns on the MUFU -- tile 0's exponentials of KV tile j, then tile 1's of j, then tile 0's of
// j + 1 ... -- through a token mbarrier per SMSP and direction, so one tile's chain runs at the full MUFU rate
// while the other tile's MMAs run, instead of both crawling at half rate when their phases overlap.
#ifndef HI_PINGPONG
#define HI_PINGPONG 0
#endif
constexpr bool PINGPONG = HI_PINGPONG != 0;
constexpr bool SPLIT_S_LO = HI_SPLIT_S == 1;  // S(j+1)_lo issued early (P in the upper 64 columns)
constexpr int P_COL = SPLIT_S_LO ? 64 : 0;    // first packed P column
// keys whose P is released first (PV(j)_lo covers them; only PV over the rest stays on the chain)
#ifndef HI_P_SPLIT_KEYS
#define HI_P_SPLIT_KEYS 64
#endif
constexpr int KS = HI_P_SPLIT_KEYS;
// HI_P_PARTS=4 (A/B): P released in four 32-key quarters (PV(j) issued in four parts; only the last 32 keys' PV
// stays on the chain) instead of two halves
#ifndef HI_P_PARTS
#define HI_P_PARTS 2
#endif
constexpr int P_PARTS = HI_P_PARTS;
static_assert(P_PARTS == 2 || (P_PARTS == 4 && KS == 64 && HI_SPLIT_S == 2 && SPLIT == 1), "quarters: product split only");
static_assert(!HI_TWO_ISSUERS || (HI_SPLIT_S == 2 && !HI_KV_JOINT), "two issuers: the product split schedule only");
constexpr bool SUMCHECK = HI_SUMCHECK != 0 && HI_SPLIT_S == 2 && !HI_PINGPONG && !HI_SPEC_SPLIT && HI_P_SPLIT_KEYS == 64;
static_assert(KS == 64 || KS == 96, "P split at 64 or 96 keys");
static_assert(SPLIT == 1 || !SPLIT_S || (KS == 64 && !SPLIT_S_LO), "two warps per row split P at their 64-key boundary");
static_assert(!SPEC_SPLIT || (KS == 64 && HI_SPLIT_S == 2),
              "the speculative first half covers keys [0, 64) + [64, 128) of one warp's 128-column row");

using namespace ptx;

struct __align__(8) Barriers {
    uint64_t q_full;
    uint64_t k_full[NS], v_full[NS], k_empty[NS], v_empty[NS];  // K and V stages are released separately
    uint64_t k_empty2[2][NS], v_empty2[2][NS];                      // HI_TWO_ISSUERS: released per tile
    uint64_t s_full[2], p_full[2], o_done[2];
    uint64_t s_cons[2], p_lo[2];  // split schedule: S(j) read into registers / P(j) keys 0-63 stored
    uint64_t pv_lo[2];            // SUMCHECK: PV(j)_lo of tile t complete (a second-half rescale waits for it)
    uint64_t p_q[2][2];           // P_PARTS == 4: P(j) keys 32..63 / 64..95 stored (quarter 0 = p_lo, 3 = p_full)
    uint64_t tok[2][4];           // PINGPONG: MUFU token for tile t's warp on SMSP q (arrived by the other tile)
    uint32_t tmem_base;
    volatile int tile_done[2];    // PINGPONG: tile t has taken its last turn (its partner stops waiting for it)
    float xchg[2][2][BM];   // [tile][half][row]: partial row max, SPLIT=2
    float xchg_l[2][2][BM]; // [tile][half][row]: partial row sum (epilogue), SPLIT=2
    int row_t[2][BM];       // [tile][row]: the row's chunk token t, re-read by the mask paths (a live copy spills)
};

template <int D>
struct Smem {
    static constexpr int BOX = BM * 128;            // one [128 rows][64 bf16] SW128 box = 16 KiB
    static constexpr int Q_OFF = 0;                 // 2 Q tiles x D/64 boxes
    static constexpr int K_OFF = Q_OFF + 2 * (D / 64) * BOX;
    static constexpr int V_OFF = K_OFF + NS * (D / 64) * BOX;
    static constexpr int BAR_OFF = V_OFF + NS * (D / 64) * BOX;
    static constexpr int BYTES = BAR_OFF + static_cast<int>(sizeof(Barriers));
    static constexpr int ALLOC = BYTES + 1024;      // slack for 1 KiB alignment
};

template <int D>
__device__ __forceinline__ void setmaxnreg_softmax() {
    if constexpr (REG_SOFTMAX<D> > (SPLIT == 1 ? 168 : 96)) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REG_SOFTMAX<D>));
}
template <int D>
__device__ __forceinline__ void setmaxnreg_producer() {
    if constexpr (REG_PRODUCER<D> < (SPLIT == 1 ? 168 : 96)) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_PRODUCER<D>));
}
__device__ __forceinline__ int ld_shared_s32(uint32_t addr) {  // volatile: re-read where used, not kept live
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// TMEM column map (512 allocated): tile tt in {0,1}: S/P at [256*tt, 256*tt+128), O at [256*tt+128, +D).
// P (bf16, packed in pairs) overwrites the first 64 columns of S after the row has been read.
template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const PrefillParams p) {
    using L = Smem<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Barriers* bars = reinterpret_cast<Barriers*>(smem + L::BAR_OFF);
    const uint32_t sbase = smem_addr(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = p.g;
    const int n_rows = p.n_q * g;
    // causal segment: CTA x's work grows with its rows, so the launcher sets row_rev = grid - 1 and the grid runs
    // longest-first (LPT): the short CTAs fill the tail instead of the long ones starting last
    const int row0 = abs(p.row_rev - static_cast<int>(blockIdx.x)) * (2 * BM);
    const int hh = blockIdx.y;                 // kv head within the launch's head group (state index)
    const int hq = p.head_q[hh], hk = p.head_kv[hh];  // its q/out columns and k/v coordinate (head maps)
    float* const o_acc = p.o_acc + static_cast<int64_t>(hh) * p.state_rows * D;
    float* const m_acc = p.m_acc + static_cast<int64_t>(hh) * p.state_rows;
    float* const l_acc = p.l_acc + static_cast<int64_t>(hh) * p.state_rows;
    const bool first = p.flags & PF_FIRST, last = p.flags & PF_LAST, causal = p.flags & PF_CAUSAL;
    const int n_tiles = (row0 + BM < n_rows) ? 2 : 1;  // second Q tile may be empty at the tail

    // duo streaming band (NEXT-3): key c visible to token t only if k_pos0+c > q_pos0+t-win.  The CTA skips
    // the KV tiles wholly below the band of its first row: its loop covers tiles kt_lo .. (key base kb).
    const bool band = p.win > 0;
    int kt_lo = 0;
    if (band) {
        const int64_t c_lo = p.q_pos0 + row0 / g - p.win + 1 - p.k_pos0;  // first visible key of the first row
        kt_lo = c_lo > 0 ? static_cast<int>((c_lo < p.n_k ? c_lo : static_cast<int64_t>(p.n_k)) / BN) : 0;
    }
    const int kb = kt_lo * BN;
    // keys of the segment visible to tile tt (causal: key c visible to token t iff k_pos0+c <= q_pos0+t)
    auto kt_count = [&](int tt) {
        const int r0 = row0 + tt * BM;
        const int t_hi = min(p.n_q - 1, (r0 + BM - 1) / g);
        int64_t e = p.n_k;
        if (causal) {
            const int64_t lim = p.q_pos0 + t_hi - p.k_pos0 + 1;
            e = lim < e ? lim : e;
        }
        e = e > 0 ? e : 0;
        return max(0, static_cast<int>((e + BN - 1) / BN) - kt_lo);
    };
    const int n_kt0 = kt_count(0);
    const int n_kt1 = n_tiles == 2 ? kt_count(1) : 0;
    const int n_kt = max(n_kt0, n_kt1);  // KV tiles streamed through shared memory

    const uint32_t bar_q = smem_addr(&bars->q_full);
    auto bar_k = [&](int s) { return smem_addr(&bars->k_full[s]); };
    auto bar_v = [&](int s) { return smem_addr(&bars->v_full[s]); };
    auto bar_ke = [&](int s) { return smem_addr(&bars->k_empty[s]); };
    auto bar_ve = [&](int s) { return smem_addr(&bars->v_empty[s]); };
    auto bar_ke2 = [&](int t, int s) { return smem_addr(&bars->k_empty2[t][s]); };
    auto bar_ve2 = [&](int t, int s) { return smem_addr(&bars->v_empty2[t][s]); };
    auto bar_s = [&](int t) { return smem_addr(&bars->s_full[t]); };
    auto bar_p = [&](int t) { return smem_addr(&bars->p_full[t]); };
    auto bar_o = [&](int t) { return smem_addr(&bars->o_done[t]); };
    auto bar_sc = [&](int t) { return smem_addr(&bars->s_cons[t]); };
    auto bar_pl = [&](int t) { return smem_addr(&bars->p_lo[t]); };
    auto bar_pvl = [&](int t) { return smem_addr(&bars->pv_lo[t]); };
    auto bar_pq = [&](int t, int q) { return smem_addr(&bars->p_q[t][q]); };

    if (threadIdx.x == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < NS; ++s) {
            mbar_init(bar_k(s), 1);
            mbar_init(bar_v(s), 1);
            mbar_init(bar_ke(s), 1);
            mbar_init(bar_ve(s), 1);
            mbar_init(bar_ke2(0, s), 1);
            mbar_init(bar_ke2(1, s), 1);
            mbar_init(bar_ve2(0, s), 1);
            mbar_init(bar_ve2(1, s), 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(bar_s(t), 1);
            // split P release with two warps per row (SPLIT == 2): hf = 0 and hf = 1 both arrive on p_lo, only
            // hf = 1 on p_full (see the softmax)
            mbar_init(bar_p(t), (SPLIT_S && SPLIT == 2) ? 128 : 128 * SPLIT);
            mbar_init(bar_o(t), 1);
            mbar_init(bar_sc(t), 128);
            mbar_init(bar_pl(t), 128 * SPLIT);
            mbar_init(bar_pvl(t), 1);
            mbar_init(bar_pq(t, 0), 128);
            mbar_init(bar_pq(t, 1), 128);
            for (int q = 0; q < 4; ++q) mbar_init(smem_addr(&bars->tok[t][q]), 1);
        }
        // a tile without KV tiles never takes a turn (its partner must not wait for it)
        bars->tile_done[0] = n_kt0 == 0;
        bars->tile_done[1] = n_kt1 == 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&bars->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
#if HI_SUMCHECK || HI_TILE_MIX
    // the TMEM base is re-read from shared memory where each role needs it (with the sum-checked softmax, one copy
    // live across the role split spills to local memory)
#define tmem static_cast<uint32_t>(ld_shared_s32(smem_addr(&bars->tmem_base)))
#else
    const uint32_t tmem = bars->tmem_base;
#endif

    if (warp >= SOFTMAX_WARPS) {
        setmaxnreg_producer<D>();
        if (warp == WARP_TMA && lane == 0 && n_kt > 0) {
            // ============================ TMA producer ============================
            mbar_expect_tx(bar_q, n_tiles * (D / 64) * L::BOX);
            for (int tt = 0; tt < n_tiles; ++tt)
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sbase + L::Q_OFF + (tt * (D / 64) + c) * L::BOX, &tm_q, bar_q, c * 64, hq * g,
                                (row0 + tt * BM) / g);
            // K(i) is consumed by the S = Q K^T MMAs, V(i) only one tile step later by the PV MMAs, and each is released
            // on its own barrier: a K stage frees once S(i) of both tiles is done, so K(i+2) streams in while
            // PV(i), S(i+1), PV(i+1) run (2.5 tile steps of prefetch instead of 1 with a joint K/V release).  Order:
            // K(0), then K(i+1) ahead of V(i).
            auto load_k = [&](int i) {
                const int s = i % NS;
                if (HI_TWO_ISSUERS && i >= NS) {  // every tile that read K(i - NS) released it
                    for (int t = 0; t < n_tiles; ++t)
                        if ((t == 0 ? n_kt0 : n_kt1) > i - NS) mbar_wait(bar_ke2(t, s), ((i / NS) - 1) & 1);
                } else if (i >= NS) {
                    mbar_wait(bar_ke(s), ((i / NS) - 1) & 1);
                }
                if (HI_KV_JOINT && i >= NS) mbar_wait(bar_ve(s), ((i / NS) - 1) & 1);  // A/B: the round-1 joint release
                mbar_expect_tx(bar_k(s), (D / 64) * L::BOX);
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sbase + L::K_OFF + (s * (D / 64) + c) * L::BOX, &tm_k, bar_k(s), c * 64, kb + i * BN, hk);
            };
            if (!HI_KV_JOINT) load_k(0);
            for (int i = 0; i < n_kt; ++i) {
                if (HI_KV_JOINT) load_k(i);
                else if (i + 1 < n_kt) load_k(i + 1);
                const int s = i % NS;
                if (HI_TWO_ISSUERS && i >= NS) {
                    for (int t = 0; t < n_tiles; ++t)
                        if ((t == 0 ? n_kt0 : n_kt1) > i - NS) mbar_wait(bar_ve2(t, s), ((i / NS) - 1) & 1);
                } else if (i >= NS) {
                    mbar_wait(bar_ve(s), ((i / NS) - 1) & 1);
                }
                mbar_expect_tx(bar_v(s), (D / 64) * L::BOX);
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sbase + L::V_OFF + (s * (D / 64) + c) * L::BOX, &tm_v, bar_v(s), c * 64, kb + i * BN, hk);
            }
        } else if ((warp == WARP_MMA || (HI_TWO_ISSUERS && warp == WARP_MMA + 1 && n_tiles == 2)) && (HI_WARP_ISSUE || lane == 0) &&
                   n_kt > 0) {
            // ============================ MMA issuer ==============================
            const uint32_t tmem_m = tmem;  // read once: the issue loop must not wait on shared memory
            constexpr uint32_t ID_S = idesc_bf16(BM, BN, false);
            constexpr uint32_t ID_O = idesc_bf16(BM, D, true);
            const int nk_t[2] = {n_kt0, n_kt1};
            MMA_WAIT(bar_q, 0);
            // descriptors precomputed once; a K-step / stage offset is added to the 14-bit start-address
            // field (shared-memory addresses < 256 KiB, so the field never carries)
            const uint64_t dq0 = sdesc(sbase + L::Q_OFF, 16, 1024);
            const uint64_t dk0 = sdesc(sbase + L::K_OFF, 16, 1024);
            const uint64_t dv0 = sdesc(sbase + L::V_OFF, L::BOX, 1024);
            if (HI_DESC_LO && ((dq0 >> 32) != DESC_HI || (dk0 >> 32) != DESC_HI || (dv0 >> 32) != DESC_HI)) __trap();
            auto issue_s = [&](int tt, int i) {  // S_tt(i) = Q_tt K(i)^T
                const int s = i % NS;
                const uint64_t a0 = dq0 + ((tt * (D / 64) * L::BOX) >> 4);
                const uint64_t b0 = dk0 + ((s * (D / 64) * L::BOX) >> 4);
#ifndef HI_SKIP_S  // timing experiment switch
                HI_ISSUE_UNROLL
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = ((ks >> 2) * L::BOX + (ks & 3) * 32) >> 4;
                    HI_UMMA(tmem_m + tt * 256, a0 + off, b0 + off, ID_S, ks > 0);
                }
#endif
                HI_UCOMMIT(bar_s(tt));
            };
            auto issue_pv = [&](int tt, int j) {  // O_tt += P_tt(j) V(j), P from TMEM
                const int s = j % NS;
                const uint64_t b0 = dv0 + ((s * (D / 64) * L::BOX) >> 4);
#ifndef HI_SKIP_PV  // timing experiment switch
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk)
                    HI_UMMA_TS(tmem_m + tt * 256 + 128, tmem_m + tt * 256 + kk * 8, b0 + ((kk * 16 * 128) >> 4), ID_O,
                                 (j > 0 || kk > 0 || !first) ? 1u : 0u);
#endif
                if (j + 1 == nk_t[tt]) HI_UCOMMIT(bar_o(tt));  // O final: the epilogue's only wait
            };
            // HI_TWO_ISSUERS: this warp's tile; otherwise every tile
            const int tt_lo = HI_TWO_ISSUERS ? warp - WARP_MMA : 0;
            const int tt_hi = HI_TWO_ISSUERS ? tt_lo + 1 : n_tiles;
            const int j_end = HI_TWO_ISSUERS ? nk_t[tt_lo] : n_kt;
            MMA_WAIT(bar_k(0), 0);
            tc_fence_after();
            for (int tt = tt_lo; tt < tt_hi; ++tt)
                if (nk_t[tt] > 0) issue_s(tt, 0);
            if (HI_TWO_ISSUERS) {
                if (j_end > 0) HI_UCOMMIT(bar_ke2(tt_lo, 0));
            } else {
                HI_UCOMMIT(bar_ke(0));  // K(0) consumed once S(0) of every tile is done
            }
            // the last tile that reads V(j) (tiles run to nk_t[tt] key tiles; tile 1's rows are the later ones)
            auto last_v_tile = [&](int j) { return (n_tiles == 2 && j < nk_t[1]) ? 1 : 0; };
            if constexpr (SPLIT_S) {
                constexpr uint32_t ID_S64 = idesc_bf16(BM, 64, false);
                // S_tt(i), keys 64h .. 64h+63 -> S columns [64h, 64h+64): B = rows 64h.. of the K boxes
                auto issue_s_half = [&](int tt, int i, int h) {
                    const uint64_t a0 = dq0 + ((tt * (D / 64) * L::BOX) >> 4);
                    const uint64_t b0 = dk0 + (((i % NS) * (D / 64) * L::BOX + h * 64 * 128) >> 4);
                    HI_ISSUE_UNROLL
                    for (int ks = 0; ks < D / 16; ++ks) {
                        const uint32_t off = ((ks >> 2) * L::BOX + (ks & 3) * 32) >> 4;
                        HI_UMMA(tmem_m + tt * 256 + 64 * h, a0 + off, b0 + off, ID_S64, ks > 0);
                    }
                };
                // O_tt += P_tt(j)[keys 16 kk0 .. 16 kk1) V(j)[same keys]
                auto issue_pv_range = [&](int tt, int j, int kk0, int kk1) {
                    const uint64_t b0 = dv0 + (((j % NS) * (D / 64) * L::BOX) >> 4);
                    for (int kk = kk0; kk < kk1; ++kk)
                        HI_UMMA_TS(tmem_m + tt * 256 + 128, tmem_m + tt * 256 + P_COL + kk * 8, b0 + ((kk * 16 * 128) >> 4), ID_O,
                                   (j > 0 || kk > 0 || !first) ? 1u : 0u);
                };
                (void)issue_pv_range;
                // O_tt += P_tt(j)[keys 64h ..] V(j)[keys 64h ..]; P at packed columns 64 + 32h ..
                auto issue_pv_half = [&](int tt, int j, int h) {
                    const uint64_t b0 = dv0 + (((j % NS) * (D / 64) * L::BOX) >> 4);
                    HI_ISSUE_UNROLL
                    for (int kk = (h ? KS / 16 : 0); kk < (h ? BN / 16 : KS / 16); ++kk)
                        HI_UMMA_TS(tmem_m + tt * 256 + 128, tmem_m + tt * 256 + P_COL + kk * 8, b0 + ((kk * 16 * 128) >> 4), ID_O,
                                     (j > 0 || kk > 0 || !first) ? 1u : 0u);
                };
                for (int j = 0; j < j_end; ++j) {
                    const int s = j % NS;
                    bool waited_v = false, have_k = false;
                    for (int tt = tt_lo; tt < tt_hi; ++tt) {
                        if (j >= nk_t[tt]) continue;
                        const bool next = j + 1 < nk_t[tt];
                        bool lo_done = false;
                        if (next && SPLIT_S_LO) {
                            // S(j+1)_lo as soon as the softmax holds S(j) in registers -- if K(j+1) has landed
                            MMA_WAIT(bar_sc(tt), j & 1);
                            if (!have_k) have_k = mbar_test(bar_k((j + 1) % NS), ((j + 1) / NS) & 1);
                            if (have_k) {
                                tc_fence_after();
                                issue_s_half(tt, j + 1, 0);
                                lo_done = true;
                            }
                        }
                        MMA_WAIT(bar_pl(tt), j & 1);
                        if (!waited_v) { MMA_WAIT(bar_v(s), (j / NS) & 1); waited_v = true; }
                        tc_fence_after();
                        if constexpr (P_PARTS == 4) {
                            issue_pv_range(tt, j, 0, 2);
                            MMA_WAIT(bar_pq(tt, 0), j & 1);
                            tc_fence_after();
                            issue_pv_range(tt, j, 2, 4);
                            MMA_WAIT(bar_pq(tt, 1), j & 1);
                            tc_fence_after();
                            issue_pv_range(tt, j, 4, 6);
                            MMA_WAIT(bar_p(tt), j & 1);
                            HI_TR_MMA(12 + 2 * tt, j);
                            tc_fence_after();
                            issue_pv_range(tt, j, 6, 8);
                        } else {
                        issue_pv_half(tt, j, 0);
                        if constexpr (SUMCHECK) HI_UCOMMIT(bar_pvl(tt));  // PV(j)_lo done (a rare second-half rescale)
                        MMA_WAIT(bar_p(tt), j & 1);
                        HI_TR_MMA(12 + 2 * tt, j);
                        tc_fence_after();
                        issue_pv_half(tt, j, 1);
                        }
                        if (HI_O_COMMIT_FIRST && j + 1 == nk_t[tt]) HI_UCOMMIT(bar_o(tt));  // A/B: the old order
                        if (HI_TWO_ISSUERS) HI_UCOMMIT(bar_ve2(tt, s));  // this tile is done with V(j)
                        else if (tt == last_v_tile(j)) HI_UCOMMIT(bar_ve(s));  // V(j) consumed by every tile
                        // O final (HI_O_COMMIT_FIRST=0 order): the epilogue's only wait
                        if (!HI_O_COMMIT_FIRST && j + 1 == nk_t[tt]) HI_UCOMMIT(bar_o(tt));
                        if (next) {
                            if (!have_k) { MMA_WAIT(bar_k((j + 1) % NS), ((j + 1) / NS) & 1); have_k = true; }
                            tc_fence_after();
                            if (SPLIT_S_LO) {
                                if (!lo_done) issue_s_half(tt, j + 1, 0);
                                issue_s_half(tt, j + 1, 1);
                                HI_UCOMMIT(bar_s(tt));
                            } else {
                                issue_s(tt, j + 1);  // commits s_full
                            }
                            HI_TR_MMA(12 + 2 * tt + 1, j);
                            if (HI_TWO_ISSUERS) HI_UCOMMIT(bar_ke2(tt, (j + 1) % NS));  // this tile is done with K(j+1)
                        }
                    }
                    if (!HI_TWO_ISSUERS && j + 1 < n_kt) HI_UCOMMIT(bar_ke((j + 1) % NS));  // K(j+1) consumed by every tile's S(j+1)
                }
            } else {
            for (int j = 0; j < n_kt; ++j) {
                const int s = j % NS;
                bool waited_v = false, waited_k = false;
                for (int tt = 0; tt < n_tiles; ++tt) {
                    if (j >= nk_t[tt]) continue;
                    MMA_WAIT(bar_p(tt), j & 1);
                    HI_TR_MMA(12 + 2 * tt, j);
                    if (!waited_v) { MMA_WAIT(bar_v(s), (j / NS) & 1); waited_v = true; }
                    tc_fence_after();
                    issue_pv(tt, j);
                    if (tt == last_v_tile(j)) HI_UCOMMIT(bar_ve(s));  // V(j) consumed by every tile
                    if (j + 1 < nk_t[tt]) {
                        if (!waited_k) { MMA_WAIT(bar_k((j + 1) % NS), ((j + 1) / NS) & 1); waited_k = true; }
                        tc_fence_after();
                        issue_s(tt, j + 1);
                        HI_TR_MMA(12 + 2 * tt + 1, j);
                    }
                }
                if (j + 1 < n_kt) HI_UCOMMIT(bar_ke((j + 1) % NS));  // K(j+1) consumed by every tile's S(j+1)
            }
            }
        }
    } else {
        // ====================== softmax / correction / epilogue: warps 0-3 tile 0, 4-7 tile 1 ======================
        setmaxnreg_softmax<D>();
        // HI_TILE_MIX (A/B): tile 0 = warps {0, 2, 5, 7}, tile 1 = {1, 3, 4, 6}, so each tile's softmax warps win the
        // highest-warp-id-first issue arbitration on two of the four SMSPs instead of tile 1 winning on all four
        const int tt = HI_TILE_MIX ? (((warp >> 2) ^ warp) & 1) : warp / (4 * SPLIT);
        const int hf = (warp / 4) % SPLIT;          // which BN/SPLIT S columns (and D/SPLIT O columns)
        const int wq = warp & 3;                    // TMEM lane quarter
        const int ttr = tt * 5;  // trace slot base (HI_TRACE builds)
        (void)ttr;
        constexpr int HN = BN / SPLIT;              // S columns per thread
        constexpr int HD = D / SPLIT;               // O columns per thread
        const int r = wq * 32 + lane;               // row within the tile == TMEM lane
        const int rg = row0 + tt * BM + r;          // packed row index t*g + j
        const bool row_valid = rg < n_rows;
        const int t = row_valid ? rg / g : 0;
        // the row's global position; the masks re-read t from shared memory (keeping it live costs a spill)
        bars->row_t[tt][r] = t;  // SPLIT == 2: both warps of the row store the same value before reading it
        // (SPLIT == 1: row_t[tt][r] is word threadIdx.x, re-derived at the use instead of kept in a register)
#define t_row (ld_shared_s32(smem_addr(&bars->row_t[0][0]) + 4u * (SPLIT == 1 && !HI_TILE_MIX ? threadIdx.x : tt * BM + r)))
#define qpos (p.q_pos0 + t_row)
        const int nkt = tt == 0 ? n_kt0 : n_kt1;
        const int t_lo = (row0 + tt * BM) / g;
        const int t_hi_tile = min(p.n_q - 1, (row0 + tt * BM + BM - 1) / g);
        const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t t_s = tmem + tt * 256 + lane_addr;        // S / P columns of this row
        const uint32_t t_o = t_s + 128 + hf * HD;                // this thread's O columns
        float* x_mine = &bars->xchg[tt][hf][r];
        const float* x_other = &bars->xchg[tt][hf ^ 1][r];
        const float sc = p.scale_log2;
        float m_run = -CUDART_INF_F, l_run = 0.f;  // l_run: this thread's partial row sum
        if (tt < n_tiles) {
            if (!first) {
                m_run = row_valid ? m_acc[rg] : -CUDART_INF_F;
                l_run = (row_valid && hf == 0) ? l_acc[rg] : 0.f;
                if (nkt > 0) {  // running O -> TMEM before the first PV accumulates onto it
#pragma unroll
                    for (int cb = 0; cb < HD / 32; ++cb) {
                        uint32_t v[32];
                        const float4* src = reinterpret_cast<const float4*>(
                            o_acc + static_cast<int64_t>(row_valid ? rg : 0) * D + hf * HD + cb * 32);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            float4 f = row_valid ? src[i] : make_float4(0.f, 0.f, 0.f, 0.f);
                            v[4 * i] = __float_as_uint(f.x); v[4 * i + 1] = __float_as_uint(f.y);
                            v[4 * i + 2] = __float_as_uint(f.z); v[4 * i + 3] = __float_as_uint(f.w);
                        }
                        tmem_st32(t_o + cb * 32, v);
                    }
                    tmem_wait_st();
                }
            }
            for (int j = 0; j < nkt; ++j) {
#if HI_WAIT_HINT
                mbar_wait_hint(bar_s(tt), j & 1, HI_WAIT_HINT);
#else
                mbar_wait(bar_s(tt), j & 1);   // also implies PV(j-1) of this tile is complete (in-order MMAs)
#endif
                HI_TR(10 + tt, j);
                tc_fence_after();
                uint32_t x[HN];
#pragma unroll
                for (int cb = 0; cb < HN / 32; ++cb)
                    tmem_ld32(t_s + hf * HN + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
                tmem_wait_ld();
                HI_TR_DEP(ttr + 0, j, x[0] ^ x[HN - 1]);
                // row max of the raw scores (scale > 0 commutes with max); masking where needed
                const int key0 = kb + j * BN + hf * HN;
                const int kt0 = kb + j * BN;  // first key of the tile
                const bool need_mask = (kt0 + BN > p.n_k) || (causal && p.k_pos0 + kt0 + BN - 1 > p.q_pos0 + t_lo);
                if (need_mask) {
                    const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                    const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                    for (int i = 0; i < HN; ++i)
                        if (key0 + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
                }
                // band lower edge: keys c <= qpos - win - k_pos0 fall out of the recent window
                if (band && p.k_pos0 + kt0 <= p.q_pos0 + t_hi_tile - p.win) {
                    const int64_t lo = qpos - p.win - p.k_pos0;
#pragma unroll
                    for (int i = 0; i < HN; ++i)
                        if (key0 + i <= lo) x[i] = __float_as_uint(-CUDART_INF_F);
                }
                if constexpr (SPLIT_S && SPLIT == 2) {
                    // Two softmax warps per TMEM lane quarter and tile: this warp owns keys [64 hf, 64 hf + 64) of
                    // its 32 rows and packs their P into columns [32 hf, 32 hf + 32).  The partner warp (same
                    // tile and lane quarter, other hf) is met at a 64-thread named barrier to combine the row max.
                    // hf = 0's P release opens PV(j)_lo, hf = 1's opens PV(j)_hi.  PV(j)_lo accumulates into
                    // every O column, so bar_pl also takes hf = 1's arrival once its O columns are rescaled.
                    const uint32_t pair_bar = 3 + tt * 4 + wq;
                    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                    const f2 sc2{sc, sc};
                    f2 nm2{0.f, 0.f};
                    auto exp_keys = [&]() {
#pragma unroll
                        for (int i = 0; i < HN; i += 2) {
                            const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                            const f2 pp{ex2(a.x), ex2(a.y)};
                            acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                            x[i / 2] = pack_bf16(pp.x, pp.y);
                        }
                    };
                    auto half_max = [&]() {  // 4 chains: the register budget is 96 per thread at SPLIT == 2
                        float mk[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
                        for (int i = 4; i < HN; i += 4)
#pragma unroll
                            for (int c = 0; c < 4; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
                        return fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3]));
                    };
                    auto row_max = [&](float mine) {  // combine with the partner warp's half
                        *x_mine = mine;
                        named_bar_sync(pair_bar, 64);
                        return fmaxf(mine, *x_other);
                    };
                    bool spec_ok = false;
                    float mx_row;
                    // both warps of the pair hold the same m_run per row, so they take the same branch
                    if (SPEC_SPLIT && __all_sync(0xffffffffu, m_run != -CUDART_INF_F)) {
                        // speculative: exponentiate against the current reference while the max is reduced in
                        // the MUFU shadow (exact unless a row max grows by > 2^8, see the SPLIT == 1 path)
                        nm2 = f2{-m_run, -m_run};
                        float mk[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
                        for (int i = 0; i < HN; i += 2) {
                            if (i >= 4) {
                                mk[i & 3] = fmaxf(mk[i & 3], __uint_as_float(x[i]));
                                mk[(i + 1) & 3] = fmaxf(mk[(i + 1) & 3], __uint_as_float(x[i + 1]));
                            }
                            const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                            const f2 pp{ex2(a.x), ex2(a.y)};
                            acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                            x[i / 2] = pack_bf16(pp.x, pp.y);
                        }
                        mx_row = row_max(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])));
                        spec_ok = !__any_sync(0xffffffffu, mx_row * sc > m_run + RESCALE_THRESHOLD);
                        if (!spec_ok) {
                            // re-read the raw scores the packing overwrote (no P is stored yet: hf = 1 writes
                            // columns 32-63, hf = 0's scores, only after the second pair barrier)
                            acc[0] = acc[1] = acc[2] = acc[3] = f2{0.f, 0.f};
#pragma unroll
                            for (int cb = 0; cb < HN / 32; ++cb)
                                tmem_ld32(t_s + hf * HN + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
                            tmem_wait_ld();
                            if (need_mask) {
                                const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                                const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                                for (int i = 0; i < HN; ++i)
                                    if (key0 + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
                            }
                            if (band && p.k_pos0 + kt0 <= p.q_pos0 + t_hi_tile - p.win) {
                                const int64_t lo = qpos - p.win - p.k_pos0;
#pragma unroll
                                for (int i = 0; i < HN; ++i)
                                    if (key0 + i <= lo) x[i] = __float_as_uint(-CUDART_INF_F);
                            }
                            named_bar_sync(pair_bar, 64);
                        }
                    } else {
                        mx_row = row_max(half_max());
                    }
                    HI_TR(ttr + 1, j);
                    float mref = m_run, alp = 1.f;
                    if (!spec_ok) {
                        const float mxs = mx_row * sc;
                        const bool grw = (mx_row != -CUDART_INF_F) && (m_run == -CUDART_INF_F || mxs > m_run + RESCALE_THRESHOLD);
                        mref = grw ? mxs : m_run;
                        alp = grw ? ((m_run == -CUDART_INF_F) ? 0.f : ex2(m_run - mxs)) : 1.f;
                        if ((!first || j > 0) && __any_sync(0xffffffffu, grw)) {  // this warp's O columns
#pragma unroll 1
                            for (int cb = 0; cb < HD / 16; ++cb) {  // 16 columns at a time: x[] is live (96 regs)
                                uint32_t v[16];
                                tmem_ld16(t_o + cb * 16, v);
                                tmem_wait_ld();
#pragma unroll
                                for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alp);
                                tmem_st16(t_o + cb * 16, v);
                            }
                        }
                        nm2 = (mref == -CUDART_INF_F) ? f2{0.f, 0.f} : f2{-mref, -mref};
                    }
                    if (hf == 1) {  // O columns [64, 128) rescaled: PV(j)_lo may accumulate
                        tmem_wait_st();
                        tc_fence_before();
                        mbar_arrive(bar_pl(tt));
                    }
                    if (!spec_ok) exp_keys();
                    tmem_st32(t_s + hf * (HN / 2), *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(hf == 0 ? bar_pl(tt) : bar_p(tt));
                    HI_TR(ttr + 4, j);
                    const f2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
                    l_run = l_run * alp + ((s01.x + s01.y) + (s23.x + s23.y));
                    m_run = mref;
                    continue;
                }
                if constexpr (SPLIT_S && SPLIT == 1 && SUMCHECK) {
#ifdef HI_FAKE_SOFTMAX  // timing experiment only: the pipeline without the softmax math (P = raw S bits)
                    tc_fence_before();
                    mbar_arrive(bar_pl(tt));
                    mbar_arrive(bar_p(tt));
                    continue;
#endif
                    // Sum-checked lazy rescale.  The max-first rule moves the reference m only when the tile's row
                    // max exceeds it by more than 2^8, so when it does not, every p = 2^(s*scale - m_run) <= 2^8.
                    // Conversely a half whose sum of p is <= 2^8 has every p <= 2^8 (p >= 0): then the reference
                    // stays, exactly as the max-first path would decide, and the half's max is never needed.  So on
                    // unmasked tiles with a finite reference the softmax exponentiates each half against m_run
                    // straight away and checks its sum; only a half whose sum exceeds 2^8 takes its max:
                    //   first half (P not released yet): the raw scores the packing overwrote are re-read from TMEM
                    //     (S is intact) and the tile takes the max-first path;
                    //   second half (P_lo released, PV(j)_lo accumulating at m_run): its max comes from the raw
                    //     scores still in registers; if the reference must move, the warp waits for PV(j)_lo,
                    //     rescales O (and the running sum) by 2^(m_run - m_new) and redoes the half.
                    // Masked tiles (causal diagonal, segment tail, duo band edge) and the first tile keep max-first.
                    constexpr float THR = 256.f;  // 2^RESCALE_THRESHOLD
                    f2 acc[4];
                    const f2 sc2{sc, sc};
                    f2 nm2{-m_run, -m_run};
                    auto exp_keys = [&](auto lo_c, auto hi_c) {  // keys [LO, HI) -> packed pairs x[i/2]; sum in acc
                        constexpr int LO = decltype(lo_c)::value, HI = decltype(hi_c)::value;
                        acc[0] = acc[1] = acc[2] = acc[3] = f2{0.f, 0.f};
#pragma unroll
                        for (int i = LO; i < HI; i += 2) {
                            const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                            const f2 pp = poly_pair(i >> 1) ? ex2_poly2(a) : f2{ex2(a.x), ex2(a.y)};
                            acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                            x[i / 2] = pack_bf16(pp.x, pp.y);
                        }
                        const f2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
                        return (s01.x + s01.y) + (s23.x + s23.y);
                    };
                    auto o_rescale = [&](float a) {  // O *= a (this thread's row)
#pragma unroll
                        for (int cb = 0; cb < HD / 32; ++cb) {
                            uint32_t v[32];
                            tmem_ld32(t_o + cb * 32, v);
                            tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * a);
                            tmem_st32(t_o + cb * 32, v);
                        }
                    };
                    const bool band_edge = band && p.k_pos0 + kt0 <= p.q_pos0 + t_hi_tile - p.win;
                    bool fast = !need_mask && !band_edge && __all_sync(0xffffffffu, m_run != -CUDART_INF_F);
                    float mref = m_run, l_part = 0.f;
                    // ---- keys [0, KS): max-first, or sum-checked against m_run (a failed check retries max-first)
#pragma unroll 1
                    for (int pass = 0; pass < 2; ++pass) {
                        float alp = 1.f;
                        if (!fast) {
                            float mk[8];
#pragma unroll
                            for (int c = 0; c < 8; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
                            for (int i = 8; i < HN; i += 8)
#pragma unroll
                                for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
#ifdef HI_FAKE_MAX  // timing experiment only (wrong results): the row max of 8 scores instead of 128
                            const float mx = fmaxf(fmaxf(fmaxf(__uint_as_float(x[0]), __uint_as_float(x[1])), fmaxf(__uint_as_float(x[2]), __uint_as_float(x[3]))),
                                                   fmaxf(fmaxf(__uint_as_float(x[4]), __uint_as_float(x[5])), fmaxf(__uint_as_float(x[6]), __uint_as_float(x[7]))));
#else
                            const float mx = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])), fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
#endif
                            const float mxs = mx * sc;
                            const bool grw = (mx != -CUDART_INF_F) && (m_run == -CUDART_INF_F || mxs > m_run + RESCALE_THRESHOLD);
                            mref = grw ? mxs : m_run;
                            alp = grw ? ((m_run == -CUDART_INF_F) ? 0.f : ex2(m_run - mxs)) : 1.f;
                            HI_TR(ttr + 1, j);
                            // O correction before PV(j)_lo may accumulate (PV(j-1) is complete: S(j) was issued after it)
                            if ((!first || j > 0) && __any_sync(0xffffffffu, grw)) o_rescale(alp);
                            const float nm = (mref == -CUDART_INF_F) ? 0.f : -mref;
                            nm2 = f2{nm, nm};
                        }
                        const float s_lo = exp_keys(std::integral_constant<int, 0>{}, std::integral_constant<int, KS>{});
                        if (fast && __any_sync(0xffffffffu, !(s_lo <= THR))) {
                            // restore the raw scores of keys [0, KS/2) that the packing overwrote; retry max-first
                            tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                            tmem_wait_ld();
                            fast = false;
                            continue;
                        }
                        l_part = l_run * alp + s_lo;
                        break;
                    }
                    tmem_st32(t_s + P_COL, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(bar_pl(tt));  // PV(j)_lo may start
                    HI_TR(ttr + 2, j);
                    // ---- keys [KS, 128)
                    float s_hi = 0.f;
#pragma unroll 1
                    for (int pass = 0; pass < 2; ++pass) {
                        s_hi = exp_keys(std::integral_constant<int, KS>{}, std::integral_constant<int, BN>{});
                        if (fast && pass == 0 && __any_sync(0xffffffffu, !(s_hi <= THR))) {
                            float mk[8];  // max of the half's raw scores x[KS..127] (the packing wrote x[KS/2..63])
#pragma unroll
                            for (int c = 0; c < 8; ++c) mk[c] = __uint_as_float(x[KS + c]);
#pragma unroll
                            for (int i = KS + 8; i < HN; i += 8)
#pragma unroll
                                for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
                            const float mxs = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])),
                                                    fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7]))) * sc;
                            const bool grw = mxs > m_run + RESCALE_THRESHOLD;
                            if (__any_sync(0xffffffffu, grw)) {
                                const float alp2 = grw ? ex2(m_run - mxs) : 1.f;
                                mref = grw ? mxs : m_run;
                                mbar_wait(bar_pvl(tt), j & 1);  // O holds PV(j)_lo at the old reference
                                tc_fence_after();
                                o_rescale(alp2);
                                l_part *= alp2;
                                nm2 = f2{-mref, -mref};
                                continue;
                            }
                        }
                        break;
                    }
                    tmem_st32(t_s + P_COL + 32, *reinterpret_cast<uint32_t(*)[32]>(&x[32]));
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(bar_p(tt));
                    HI_TR(ttr + 4, j);
                    l_run = l_part + s_hi;
                    m_run = mref;
                    continue;
                } else if constexpr (SPLIT_S && SPLIT == 1) {
#ifdef HI_FAKE_SOFTMAX  // timing experiment only: the pipeline without the softmax math (P = raw S bits)
                    tc_fence_before();
                    mbar_arrive(bar_pl(tt));
                    mbar_arrive(bar_p(tt));
                    continue;
#endif
                    if constexpr (SPLIT_S_LO) {  // S(j) is in registers: columns 0-63 may take S(j+1)_lo
                        tc_fence_before();
                        mbar_arrive(bar_sc(tt));
                    }
                    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                    f2 sc2{sc, sc}, nm2{0.f, 0.f};
                    // exponentials of keys [LO, HI) packed in place (x[i/2]); compile-time bounds keep x[] in
                    // registers
                    auto exp_keys = [&](auto lo_c, auto hi_c) {
                        constexpr int LO = decltype(lo_c)::value, HI = decltype(hi_c)::value;
#pragma unroll
                        for (int i = LO; i < HI; i += 2) {
                            const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                            // POLY_PAIRS / POLY_MASK8 (experiment): some pairs on the FMA-pipe polynomial
                            const f2 pp = poly_pair(i >> 1) ? ex2_poly2(a) : f2{ex2(a.x), ex2(a.y)};
                            acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                            x[i / 2] = pack_bf16(pp.x, pp.y);
                        }
                    };
                    float mk[8];
                    bool spec_ok = false;
                    if constexpr (SPEC_SPLIT) {
                        // Speculative first half: exponentiate keys [0, KS) against the CURRENT reference max
                        // while the tile max over all keys is reduced in the MUFU shadow, so the max is off the
                        // critical path.  Exact whenever no row max grows by > 2^8 (the lazy-rescale rule): then
                        // the reference would not have moved anyway.  Otherwise (rare after the first tiles) the
                        // raw scores of keys [0, KS/2) that the packing overwrote are re-read from TMEM (S is
                        // intact: no P has been stored yet) and the tile takes the normal path.
                        if (__all_sync(0xffffffffu, m_run != -CUDART_INF_F)) {
                            nm2 = f2{-m_run, -m_run};
#pragma unroll
                            for (int c = 0; c < 8; ++c) mk[c] = fmaxf(__uint_as_float(x[c]), __uint_as_float(x[KS + c]));
#pragma unroll
                            for (int i = 0; i < KS; i += 2) {
                                if (i >= 8) mk[i & 7] = fmaxf(mk[i & 7], __uint_as_float(x[i]));
                                if (i + 1 >= 8) mk[(i + 1) & 7] = fmaxf(mk[(i + 1) & 7], __uint_as_float(x[i + 1]));
                                if (KS + i >= KS + 8 && KS + i < HN) mk[(KS + i) & 7] = fmaxf(mk[(KS + i) & 7], __uint_as_float(x[KS + i]));
                                if (KS + i + 1 >= KS + 8 && KS + i + 1 < HN)
                                    mk[(KS + i + 1) & 7] = fmaxf(mk[(KS + i + 1) & 7], __uint_as_float(x[KS + i + 1]));
                                const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                                const f2 pp{ex2(a.x), ex2(a.y)};
                                acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                                x[i / 2] = pack_bf16(pp.x, pp.y);
                            }
#pragma unroll
                            for (int i = 2 * KS; i < HN; i += 8)  // keys beyond 2*KS (KS = 64: none)
#pragma unroll
                                for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
                            const float mxs0 = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])),
                                                     fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7]))) * sc;
                            spec_ok = !__any_sync(0xffffffffu, mxs0 > m_run + RESCALE_THRESHOLD);
                            HI_TR(ttr + 1, j);
                            if (!spec_ok) {
                                acc[0] = acc[1] = acc[2] = acc[3] = f2{0.f, 0.f};
                                tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                                tmem_wait_ld();
                                if (need_mask) {
                                    const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                                    const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                                    for (int i = 0; i < 32; ++i)
                                        if (key0 + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
                                }
                                if (band && p.k_pos0 + kt0 <= p.q_pos0 + t_hi_tile - p.win) {
                                    const int64_t lo = qpos - p.win - p.k_pos0;
#pragma unroll
                                    for (int i = 0; i < 32; ++i)
                                        if (key0 + i <= lo) x[i] = __float_as_uint(-CUDART_INF_F);
                                }
                            }
                        }
                    }
                    float mref = m_run, alp = 1.f;
                    if (!spec_ok) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
                    for (int i = 8; i < HN; i += 8)
#pragma unroll
                        for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
#ifdef HI_FAKE_MAX  // timing experiment only (wrong results): the row max of 8 scores instead of 128
                    const float mx = fmaxf(fmaxf(fmaxf(__uint_as_float(x[0]), __uint_as_float(x[1])), fmaxf(__uint_as_float(x[2]), __uint_as_float(x[3]))),
                                           fmaxf(fmaxf(__uint_as_float(x[4]), __uint_as_float(x[5])), fmaxf(__uint_as_float(x[6]), __uint_as_float(x[7]))));
#else
                    const float mx = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])), fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
#endif
                    const float mxs = mx * sc;
                    const bool grw = (mx != -CUDART_INF_F) && (m_run == -CUDART_INF_F || mxs > m_run + RESCALE_THRESHOLD);
                    mref = grw ? mxs : m_run;
                    alp = grw ? ((m_run == -CUDART_INF_F) ? 0.f : ex2(m_run - mxs)) : 1.f;
                    HI_TR(ttr + 1, j);
                    // O correction before PV(j)_lo may accumulate (PV(j-1) is complete: S(j) was issued after it)
                    if ((!first || j > 0) && __any_sync(0xffffffffu, grw)) {
#pragma unroll
                        for (int cb = 0; cb < HD / 32; ++cb) {
                            uint32_t v[32];
                            tmem_ld32(t_o + cb * 32, v);
                            tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alp);
                            tmem_st32(t_o + cb * 32, v);
                        }
                    }
                    const float nm = (mref == -CUDART_INF_F) ? 0.f : -mref;
                    nm2 = f2{nm, nm};
                    }
                    auto release_p = [&](uint32_t bar) {
                        tmem_wait_st();
                        tc_fence_before();
                        mbar_arrive(bar);
                    };
                    const bool pp = PINGPONG && n_tiles == 2;
                    if (pp && (tt == 1 || j > 0) && !bars->tile_done[tt ^ 1]) {
                        // my turn: tile 0 before KV tile j waits for tile 1's turn j-1, tile 1 for tile 0's turn j
                        mbar_wait(smem_addr(&bars->tok[tt][wq]), tt == 0 ? ((j - 1) & 1) : (j & 1));
                    }
                    if constexpr (P_PARTS == 4) {
                        // quarter q: keys [32 q, 32 q + 32) -> packed columns [P_COL + 16 q, + 16), released on
                        // p_lo / p_q[0] / p_q[1] / p_full
                        exp_keys(std::integral_constant<int, 0>{}, std::integral_constant<int, 32>{});
                        tmem_st16(t_s + P_COL, &x[0]);
                        release_p(bar_pl(tt));
                        exp_keys(std::integral_constant<int, 32>{}, std::integral_constant<int, 64>{});
                        tmem_st16(t_s + P_COL + 16, &x[16]);
                        release_p(bar_pq(tt, 0));
                        exp_keys(std::integral_constant<int, 64>{}, std::integral_constant<int, 96>{});
                        tmem_st16(t_s + P_COL + 32, &x[32]);
                        release_p(bar_pq(tt, 1));
                        exp_keys(std::integral_constant<int, 96>{}, std::integral_constant<int, 128>{});
                        tmem_st16(t_s + P_COL + 48, &x[48]);
                        release_p(bar_p(tt));
                        HI_TR(ttr + 4, j);
                        const f2 q01 = fadd2(acc[0], acc[1]), q23 = fadd2(acc[2], acc[3]);
                        l_run = l_run * alp + ((q01.x + q01.y) + (q23.x + q23.y));
                        m_run = mref;
                        continue;
                    }
                    // keys [0, KS) -> packed columns [P_COL, P_COL + KS/2): PV(j)_lo may start
                    if (!spec_ok) exp_keys(std::integral_constant<int, 0>{}, std::integral_constant<int, KS>{});
                    tmem_st32(t_s + P_COL, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                    if constexpr (KS == 96) tmem_st16(t_s + P_COL + 32, &x[32]);
                    release_p(bar_pl(tt));
                    HI_TR(ttr + 2, j);
                    // keys [KS, 128) -> packed columns [P_COL + KS/2, P_COL + 64)
                    exp_keys(std::integral_constant<int, KS>{}, std::integral_constant<int, BN>{});
                    if (pp) {   // pass the MUFU to the other tile's warp on this SMSP
                        __syncwarp();
                        if (lane == 0) {
                            if (j + 1 == nkt) {   // last turn: announce it BEFORE the arrive that wakes the partner
                                bars->tile_done[tt] = 1;
                                __threadfence_block();
                            }
                            mbar_arrive(smem_addr(&bars->tok[tt ^ 1][wq]));
                        }
                    }
                    if constexpr (KS == 64) tmem_st32(t_s + P_COL + 32, *reinterpret_cast<uint32_t(*)[32]>(&x[32]));
                    else tmem_st16(t_s + P_COL + 48, &x[48]);
                    release_p(bar_p(tt));
                    HI_TR(ttr + 4, j);
                    const f2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
                    l_run = l_run * alp + ((s01.x + s01.y) + (s23.x + s23.y));
                    m_run = mref;
                    continue;
                }
                float m_ref = m_run, alpha = 1.f;
                bool grow = false;
                float ls[4] = {0.f, 0.f, 0.f, 0.f};
#ifdef HI_FAKE_SOFTMAX  // timing experiment only: tensor-core / pipeline bound without the softmax math
                tc_fence_before();
                mbar_arrive(bar_p(tt));
                continue;
#endif
                // Speculative pass (SPLIT == 1): exponentiate against the CURRENT reference max while the
                // tile max is reduced alongside, so the max is off the critical path.  With lazy rescaling the
                // reference moves only when a row max grows by > 2^8; then (rarely) the warp re-reads S from
                // TMEM (still intact: P is not stored yet) and redoes the pass with the new reference.
                bool done = false;
                if constexpr (SPLIT == 1 && SPEC_EXP) {
                    if (__all_sync(0xffffffffu, m_run != -CUDART_INF_F)) {
                        const float neg_m = -m_run;
                        float mk[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) mk[c] = -CUDART_INF_F;
#pragma unroll
                        for (int i = 0; i < HN; i += 2) {
                            const float r0 = __uint_as_float(x[i]), r1 = __uint_as_float(x[i + 1]);
                            mk[(i >> 1) & 7] = fmaxf(mk[(i >> 1) & 7], fmaxf(r0, r1));
                            const float p0 = ex2(fmaf(r0, sc, neg_m));
                            const float p1 = ex2(fmaf(r1, sc, neg_m));
                            ls[(i >> 1) & 3] += p0 + p1;
                            x[i / 2] = pack_bf16(p0, p1);
                        }
                        const float mx = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])),
                                               fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
                        grow = (mx != -CUDART_INF_F) && (mx * sc > m_run + RESCALE_THRESHOLD);
                        done = !__any_sync(0xffffffffu, grow);
                        if (!done) {  // re-read S (TMEM untouched) for the slow path
                            ls[0] = ls[1] = ls[2] = ls[3] = 0.f;
#pragma unroll
                            for (int cb = 0; cb < HN / 32; ++cb)
                                tmem_ld32(t_s + hf * HN + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
                            tmem_wait_ld();
                            if (need_mask) {
                                const int64_t lim = causal ? qpos - p.k_pos0 : static_cast<int64_t>(p.n_k) - 1;
                                const int64_t lim2 = lim < p.n_k - 1 ? lim : static_cast<int64_t>(p.n_k) - 1;
#pragma unroll
                                for (int i = 0; i < HN; ++i)
                                    if (key0 + i > lim2) x[i] = __float_as_uint(-CUDART_INF_F);
                            }
                        }
                    }
                }
                if (!done) {
                // 8 independent max chains (short dependency chain), then combine
                float mk[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) mk[c] = __uint_as_float(x[c]);
#pragma unroll
                for (int i = 8; i < HN; i += 8)
#pragma unroll
                    for (int c = 0; c < 8; ++c) mk[c] = fmaxf(mk[c], __uint_as_float(x[i + c]));
                float mx = fmaxf(fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3])), fmaxf(fmaxf(mk[4], mk[5]), fmaxf(mk[6], mk[7])));
                if constexpr (SPLIT == 2) {
                    // combine the two halves' maxima; after this barrier both halves have finished reading
                    // S, so P may overwrite any S column of the row
                    *x_mine = mx;
                    named_bar_sync(1 + tt, 256);
                    mx = fmaxf(mx, *x_other);
                }
                HI_TR(ttr + 1, j);
                const float mxs = mx * sc;  // log2-domain tile max
                // lazy rescale: move the reference max only when it grows by > 2^8
                grow = (mx != -CUDART_INF_F) && (m_run == -CUDART_INF_F || mxs > m_run + RESCALE_THRESHOLD);
                if (grow) {
                    m_ref = mxs;
                    alpha = (m_run == -CUDART_INF_F) ? 0.f : ex2(m_run - mxs);
                }
                const float neg_m = (m_ref == -CUDART_INF_F) ? 0.f : -m_ref;
                // p = 2^(x*scale - m): packed to bf16 pairs in place (x[i/2] is dead once read).  Two
                // elements in EX2_POLY_EVERY go through the FMA-pipe polynomial, the rest through MUFU.
                if constexpr (POLY_PAIRS >= 0) {
                    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                    const f2 sc2{sc, sc}, nm2{neg_m, neg_m};
#pragma unroll
                    for (int i = 0; i < HN; i += 2) {
                        const f2 a = ffma2(f2{__uint_as_float(x[i]), __uint_as_float(x[i + 1])}, sc2, nm2);
                        const f2 pp = ((i >> 1) & 3) < POLY_PAIRS ? ex2_poly2(a) : f2{ex2(a.x), ex2(a.y)};
                        acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], pp);
                        x[i / 2] = pack_bf16(pp.x, pp.y);
                    }
                    const f2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
                    ls[0] = s01.x; ls[1] = s01.y; ls[2] = s23.x; ls[3] = s23.y;
                } else {
#pragma unroll
                    for (int i = 0; i < HN; i += 2) {
                        const float a0 = fmaf(__uint_as_float(x[i]), sc, neg_m);
                        const float a1 = fmaf(__uint_as_float(x[i + 1]), sc, neg_m);
                        const float p0 = ((i % EX2_POLY_EVERY) == EX2_POLY_EVERY - 2) ? ex2_poly(a0) : ex2(a0);
                        const float p1 = (((i + 1) % EX2_POLY_EVERY) == EX2_POLY_EVERY - 1) ? ex2_poly(a1) : ex2(a1);
                        ls[(i >> 1) & 3] += p0 + p1;
                        x[i / 2] = pack_bf16(p0, p1);
                    }
                }
                }
                HI_TR(ttr + 2, j);
                // P -> TMEM: this thread's keys are packed columns [hf*HN/2, (hf+1)*HN/2)
#pragma unroll
                for (int cb = 0; cb < HN / 64; ++cb)
                    tmem_st32(t_s + hf * (HN / 2) + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&x[cb * 32]));
                const bool o_live = !first || j > 0;
                if (o_live && __any_sync(0xffffffffu, grow)) {
#pragma unroll
                    for (int cb = 0; cb < HD / 32; ++cb) {
                        uint32_t v[32];
                        tmem_ld32(t_o + cb * 32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st32(t_o + cb * 32, v);
                    }
                }
                tmem_wait_st();
                HI_TR(ttr + 3, j);
                l_run = l_run * alpha + ((ls[0] + ls[1]) + (ls[2] + ls[3]));
                m_run = m_ref;
                tc_fence_before();
                mbar_arrive(bar_p(tt));
                HI_TR(ttr + 4, j);
            }
            // ---- epilogue ----
            float l_tot = l_run;
            if constexpr (SPLIT == 2) {
                bars->xchg_l[tt][hf][r] = l_run;
                named_bar_sync(1 + tt, 256);
                l_tot += bars->xchg_l[tt][hf ^ 1][r];
            }
            if (nkt > 0) {
                mbar_wait(bar_o(tt), 0);
                tc_fence_after();
            }
            if (last) {
                const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
#if HI_SUMCHECK || HI_TILE_MIX
                __nv_bfloat16* dst = p.out + static_cast<int64_t>(t_row) * p.o_tok_stride + (hq * g + rg % g) * D + hf * HD;
#else
                __nv_bfloat16* dst = p.out + static_cast<int64_t>(t) * p.o_tok_stride + (hq * g + rg % g) * D + hf * HD;
#endif
#pragma unroll
                for (int cb = 0; cb < HD / 32; ++cb) {
                    uint32_t v[32];
                    if (nkt > 0) {
                        tmem_ld32(t_o + cb * 32, v);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            v[i] = (row_valid && !first)
                                       ? __float_as_uint(o_acc[static_cast<int64_t>(rg) * D + hf * HD + cb * 32 + i])
                                       : 0u;
                    }
                    if (row_valid) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            uint4 w;
                            w.x = pack_bf16(__uint_as_float(v[8 * i]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
                            w.y = pack_bf16(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
                            w.z = pack_bf16(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
                            w.w = pack_bf16(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
                            *reinterpret_cast<uint4*>(dst + cb * 32 + 8 * i) = w;
                        }
                    }
                }
            } else if (nkt > 0) {
#pragma unroll
                for (int cb = 0; cb < HD / 32; ++cb) {
                    uint32_t v[32];
                    tmem_ld32(t_o + cb * 32, v);
                    tmem_wait_ld();
                    if (row_valid) {
                        float4* dst = reinterpret_cast<float4*>(o_acc + static_cast<int64_t>(rg) * D + hf * HD + cb * 32);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                 __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                    }
                }
                if (row_valid && hf == 0) {
                    m_acc[rg] = m_run;
                    l_acc[rg] = l_tot;
                }
            }
        }
    }
#undef qpos
#undef t_row
    tc_fence_before();
    __syncthreads();
    if (warp == WARP_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
#if HI_SUMCHECK || HI_TILE_MIX
#undef tmem
#endif
    }
}

// ---------------------------------------------------------------- host side
template <int D>
cudaError_t launch_tc(const PrefillParams& p, cudaStream_t stream) {
    const int n_rows = p.n_q * p.g;
    const int grid = (n_rows + 2 * BM - 1) / (2 * BM);
    const int heads = p.n_heads > 0 ? p.n_heads : 1;
    if (grid == 0) return cudaSuccess;
    if (heads > MAX_LAUNCH_HEADS || p.q_span < 1 || p.kv_span < 1) return cudaErrorInvalidValue;
    static std::atomic<unsigned long long> configured{0};
    if (cudaError_t e = set_smem_attr_once(prefill_tc_kernel<D>, Smem<D>::ALLOC, configured); e != cudaSuccess) return e;
    CUtensorMap tq, tk, tv;
    {
        // (d, q heads spanned by the head map, tokens): kv head h's g rows start at coordinate h*g
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.g) * p.q_span,
                                    static_cast<cuuint64_t>(p.n_q)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(p.q_tok_stride) * 2};
        const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(p.g), static_cast<cuuint32_t>(BM / p.g)};
        if (!make_tmap_bf16(&tq, p.q, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    {
        // (d, keys, kv heads spanned by the head map)
        const int64_t hs = p.kv_span > 1 ? p.kv_head_stride : static_cast<int64_t>(p.n_k) * p.kv_row_stride;
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(p.n_k), static_cast<cuuint64_t>(p.kv_span)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.kv_row_stride) * 2, static_cast<cuuint64_t>(hs) * 2};
        const cuuint32_t box[3] = {64, BN, 1};
        if (!make_tmap_bf16(&tk, p.k, 3, dims, strides, box)) return cudaErrorInvalidValue;
        if (!make_tmap_bf16(&tv, p.v, 3, dims, strides, box)) return cudaErrorInvalidValue;
    }
    PrefillParams pl = p;
#ifndef HI_NO_LPT
    pl.row_rev = (p.flags & PF_CAUSAL) ? grid - 1 : 0;
#else
    pl.row_rev = 0;   // A/B: causal CTAs in launch order
#endif
    prefill_tc_kernel<D><<<dim3(grid, heads), NUM_THREADS, Smem<D>::ALLOC, stream>>>(tq, tk, tv, pl);
    return cudaGetLastError();
}

}  // namespace

#ifdef HI_TRACE
extern "C" int hi_debug_prefill_trace(void* dst, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_hi_trace, bytes));
}
#endif

cudaError_t launch_prefill_tc(const PrefillParams& p, int d, cudaStream_t stream) {
    if (d == 64) return launch_tc<64>(p, stream);
    if (d == 128) return launch_tc<128>(p, stream);
    return cudaErrorInvalidValue;
}

}  // namespace hi
