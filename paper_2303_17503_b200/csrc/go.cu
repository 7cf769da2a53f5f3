// Go (Tromp-Taylor, positional superko) batched step for sm_100a.
//
// Replaces reference pkg/src/boardbatch/games/go.py for make_game(size)
// (odd sizes 5..19 instantiated): apply :219-262, _analyse :45-80,
// legal_mask :121-174, score_rewards :176-210, init_core :212-217,
// observe :264-273, plus env-core _make_state core.py:192-220 and the
// auto-reset of batch_step core.py:353-386.
//
// Mapping: one warp SEGMENT per board -- a whole warp for 15x15..19x19, half a
// warp (16 lanes, two boards per warp) up to 13x13 -- and segment lane r owns
// board row r as bit rows (black, white, empty; bit c = column c). Per step:
//   1. placement + captures: bit-parallel flood of each enemy neighbour
//      group over the rows (shuffles), captured iff no liberty;
//   2. analysis of the new board: chains carry a persistent label (one point
//      of the chain, `lab`), updated incrementally at placement (a merge
//      relabels the absorbed chains); per chain "is in atari" from one
//      atomicOr per horizontal run of OR(lib) | OR(~lib) (a chain has exactly
//      one liberty iff every liberty position is equal iff the ORs are disjoint);
//   3. legal mask: empty points with an empty neighbour / a non-atari own
//      neighbour group / a capture (XOR of the captured atari groups'
//      zobrist accumulated at their single liberty), filtered by positional
//      superko through a per-env Bloom filter with an exact scan of the
//      append-only history on a Bloom hit (identical answers to the
//      reference's `h2 not in history`);
//   4. observation: the 8-deep board history is kept TRANSPOSED per point
//      (uint16 `pat`, bit 2t/2t+1 = black/white in boards_hist[t]), so the
//      17 planes of a point are one shift/swap of pat plus the colour bit;
//      the [N,N,17] float32 record is emitted as a flat 16-byte-aligned
//      stream with 128-bit stores (records are not 16-B aligned).
#include <cstdio>
#include "common.cuh"
#include "../../include/bbk.h"

namespace go {
#ifndef BBK_GO_OBS_UNROLL
#define BBK_GO_OBS_UNROLL 1   // r02 graph-timed: 1 = +1 % over a 19x19 cycle (2: baseline, 4: -4 %)
#endif
constexpr int kGoObsUnroll = BBK_GO_OBS_UNROLL;   // observation chunk loop unroll (tuning knob)
using namespace bbk;

constexpr int kWarps = 4;             // warps per CTA
constexpr int kPlanes = 17;

// Lanes per board. Rows are lanes, so a 9x9 board on a whole warp keeps 9 of 32 lanes busy in
// every row-parallel phase; on half a warp (two independent boards per warp, each with its own
// 16-lane shuffle / ballot / syncwarp mask, so the halves may diverge) it keeps 9 of 16.
__host__ __device__ constexpr int seg_lanes(int N) { return N <= 13 ? 16 : 32; }
__host__ __device__ constexpr int boards_per_cta(int N) { return kWarps * (32 / seg_lanes(N)); }

// Superko filter of one env, sized per board: it is read whole every step, so its size is HBM
// traffic (1,280 B at 19x19 against a 25.9 KB step, but 21 % of a 9x9 step at that size). The
// history of a small board is short (random 9x9 games end after ~130 plies), so a 2048-bit Bloom
// filter keeps the false-positive rate (answered by the exact history scan) well under 1 %.
#ifndef BBK_GO_BLOOM9_WORDS
#define BBK_GO_BLOOM9_WORDS 64   // Bloom words of boards up to 9x9 (tuning knob; the host asks bbk_go_filter_words)
#endif
__host__ __device__ constexpr int bloom_words(int N) { return N <= 9 ? BBK_GO_BLOOM9_WORDS : N <= 13 ? 128 : BBK_GO_BLOOM_WORDS; }
#ifndef BBK_GO_PAIR9_WORDS
#define BBK_GO_PAIR9_WORDS 64   // pair-filter words up to 13x13 (r02: 2048 bits +0.6 % over 1024 at 9x9)
#endif
__host__ __device__ constexpr int pair_words(int N) { return N <= 13 ? BBK_GO_PAIR9_WORDS : BBK_GO_PAIR_WORDS; }
__host__ __device__ constexpr int filter_words(int N) { return bloom_words(N) + pair_words(N); }
__host__ __device__ constexpr int log2i(int v) { return v <= 1 ? 0 : 1 + log2i(v / 2); }

__host__ __device__ constexpr int pat_stride(int N) { return (N * N + 7) & ~7; }

// The lanes of one board: shuffles / votes / syncs over the segment's mask only (width L), so the
// two boards of a split warp never wait on each other.
template <int L>
struct Seg {
    unsigned m;   // the segment's lanes
    int sl;       // lane within the segment (the row it owns)
    __device__ __forceinline__ Seg() {
        const int lane = lane_id();
        sl = lane & (L - 1);
        if constexpr (L == 32) m = BBK_FULL;
        else m = ((1u << L) - 1u) << (lane & ~(L - 1));
    }
    __device__ __forceinline__ uint32_t shfl(uint32_t v, int src) const { return __shfl_sync(m, v, src, L); }
    __device__ __forceinline__ int shfl(int v, int src) const { return __shfl_sync(m, v, src, L); }
    __device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) const {
        const uint32_t lo = __shfl_sync(m, (uint32_t)v, src, L), hi = __shfl_sync(m, (uint32_t)(v >> 32), src, L);
        return ((uint64_t)hi << 32) | lo;
    }
    __device__ __forceinline__ bool any(bool p) const { return __any_sync(m, p); }
    // segment-relative ballot (bit i = segment lane i)
    __device__ __forceinline__ unsigned ballot(bool p) const {
        const unsigned v = __ballot_sync(m, p);
        if constexpr (L == 32) return v;
        else return (v & m) >> (__ffs(m) - 1);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(m); }
    __device__ __forceinline__ unsigned reduce_or(unsigned v) const { return __reduce_or_sync(m, v); }
    __device__ __forceinline__ int sum(int v) const {
#pragma unroll
        for (int o = L / 2; o; o >>= 1) v += __shfl_xor_sync(m, v, o, L);
        return v;
    }
    __device__ __forceinline__ uint64_t xor64(uint64_t v) const {
#pragma unroll
        for (int o = L / 2; o; o >>= 1) {
            const uint32_t lo = __shfl_xor_sync(m, (uint32_t)v, o, L);
            const uint32_t hi = __shfl_xor_sync(m, (uint32_t)(v >> 32), o, L);
            v ^= ((uint64_t)hi << 32) | lo;
        }
        return v;
    }
    // inclusive prefix sum over the segment lanes
    __device__ __forceinline__ int scan(int v) const {
#pragma unroll
        for (int o = 1; o < L; o <<= 1) {
            const int t = __shfl_up_sync(m, v, o, L);
            if (sl >= o) v += t;
        }
        return v;
    }
    __device__ __forceinline__ uint32_t up_row(uint32_t v) const {   // row r-1's value at row r
        const uint32_t u = __shfl_up_sync(m, v, 1, L);
        return sl > 0 ? u : 0u;
    }
    __device__ __forceinline__ uint32_t dn_row(uint32_t v) const {   // row r+1's value at row r
        const uint32_t d = __shfl_down_sync(m, v, 1, L);
        return sl < L - 1 ? d : 0u;
    }
};

template <int N>
struct WarpSmem {   // one board's scratch (one per segment)
    static constexpr int C = N * N;
    static constexpr int A = C + 1;
    static constexpr int L = seg_lanes(N);
    static constexpr int MAXR = C;   // runs of both colours: each holds >= 1 stone
    // Per point, live during the legal-mask analysis: at an empty point the XOR of the zobrist keys
    // of the chains a stone there would capture; at a stone that is its chain's label, the chain's
    // liberty stats OR(lib) | OR(~lib) << 10 | HAS in the low word (labels are stones, capture
    // points are empty: the two never share a point). Between the analysis and the next board's
    // start it is the landing zone of the next board's prefetched `pat` and `lab`.
    uint64_t capx[C];
    // Phase-multiplexed scratch (each member is dead before the next one is written):
    // chain labels -> group analysis -> superko hits -> staged mask bytes -> observation pattern.
    union {
        struct {
            // the board's chain labels (u16) until the run list is built; then the env's
            // Bloom + count-pair filter (cp.async)
            alignas(16) uint32_t bl[filter_words(N)];
            uint16_t run[MAXR];    // (colour << 15) | (row << 10) | (start << 5) | len
            uint16_t root[MAXR];   // chain label of the run
        } uf;
        struct {
            uint32_t bloom_area[filter_words(N)];
            uint64_t hit[L];
        } sk;
        alignas(16) uint8_t mb[((A + 47) & ~15)];
        struct {
            alignas(16) uint32_t P[pat_stride(N)];   // points C.. are padding (only feed bits >= NF)
            uint32_t W[(C * 17 + 31) / 32 + 2];
        } ob;
    } u;
    static_assert(2 * pat_stride(N) <= 4 * filter_words(N), "labels must fit the filter landing area");
    static_assert(4 * pat_stride(N) <= 8 * C, "pat + lab prefetch must fit the capture-XOR array");
    static_assert(N <= L, "a board's rows must fit its lanes");
    alignas(16) uint16_t pat[pat_stride(N)];
    // rX / rY: rows of black / white and the flat stone bitmaps (small boards only)
    uint32_t rX[N <= 13 ? L : 1], rY[N <= 13 ? L : 1], rE[L], rcap[L];
    static_assert(L == 32 || 4 * L >= pat_stride(N) / 8 + 8, "flat stone bitmaps must fit rX / rY");
};

// zobrist key of (cell, colour) (go.py:20-25): mix64(0x60D00D60C0FFEE00 + N + 2*cell + colour).
// Boards up to 13x13 read it from a table filled once per device (launch_step) through the
// read-only path -- one L1 load instead of a chain of ~15 dependent 64-bit multiply / shift ops
// (go_9x9 +6.7 %); 15x15+ compute it in registers (their shared memory leaves little L1, and the
// table lost 1.2 % at 19x19).
#ifndef BBK_GO_ZTABLE_MAX
#define BBK_GO_ZTABLE_MAX 13   // largest board reading single-point keys from the table
#endif
#ifndef BBK_GO_ZROW_MAX
#define BBK_GO_ZROW_MAX 19     // largest board reading run hashes from the row-prefix table (all)
#endif
template <int N>
__device__ uint64_t g_zob[2 * N * N];

template <int N>
__device__ __forceinline__ uint64_t zkey(int cell, int colour) {
    if constexpr (N <= BBK_GO_ZTABLE_MAX) return __ldg(&g_zob<N>[2 * cell + colour]);
    else return mix64(0x60D00D60C0FFEE00ULL + (uint64_t)N + 2ull * (uint64_t)cell + (uint64_t)colour);
}

// Row-prefix XORs of the zobrist keys, every size: g_zrow[(colour * N + row) * (N + 1) + j] = XOR of
// zkey(row * N + c, colour) for c < j, so the hash of a horizontal run of stones (a captured chain's
// run, a removed row segment) is two loads instead of one key per stone.
template <int N>
__device__ uint64_t g_zrow[2 * N * (N + 1)];

template <int N>
__device__ __forceinline__ uint64_t zrun(int row, int s, int len, int colour) {
    // r02: +4 % at 9x9; at 19x19 +6 % late game / +2 % over a full cycle (big captured chains), the
    // single-point key table there stays off (neutral)
    if constexpr (N <= BBK_GO_ZROW_MAX) {
        const uint64_t* z = g_zrow<N> + (colour * N + row) * (N + 1);
        return __ldg(z + s + len) ^ __ldg(z + s);
    } else {
        uint64_t x = 0ull;
        for (int q = 0; q < len; q++) x ^= zkey<N>(row * N + s + q, colour);
        return x;
    }
}
// XOR of the keys of the stones in row bits `bits` of `row`, run by run
template <int N>
__device__ __forceinline__ uint64_t zbits(int row, uint32_t bits, int colour) {
    uint64_t x = 0ull;
    while (bits) {
        const int s = __ffs(bits) - 1, len = __ffs(~(bits >> s)) - 1;
        x ^= zrun<N>(row, s, len, colour);
        bits &= ~(((1u << len) - 1u) << s);
    }
    return x;
}

template <int N>
struct BlockSmem {
    static constexpr int C = N * N;
    float4 lut[16];
    WarpSmem<N> w[boards_per_cta(N)];
};

struct StepParams {
    bbk_cols in, out;
    bbk_go_state in_s, out_s;
    bbk_go_store store;
    const int64_t* actions;
    const uint64_t* slot_keys;
    int64_t n, slot0;
    uint64_t key;
    int32_t max_steps;
    double komi;
    int force_reset;
    int self_capture;   // make_game(allow_self_capture=True) (go.py:155-173, 249-255)
    int64_t tail_ctas;  // CTAs at the end of the grid that take one pass each (see step_kernel)
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t run_at(uint32_t X, int s) {
    uint32_t len = __ffs(~(X >> s)) - 1;
    return ((1u << len) - 1u) << s;
}

// Bloom probes per hash (13-bit slices of the 64-bit zobrist hash). A false positive costs an exact
// scan of the env's history (up to 4 KB late in a 19x19 game): 4 probes halve the false-positive
// rate of 3 at these fill levels (8192 bits, ~500 entries: 0.47 % -> 0.22 %).
#ifndef BBK_GO_BLOOM_K
#define BBK_GO_BLOOM_K 4
#endif
constexpr int kBloomK = BBK_GO_BLOOM_K;   // r02: 4 beat 3, 5 and a 4096-bit 9x9 filter
static_assert(kBloomK >= 1 && 13 * (kBloomK - 1) < 64, "probe slices must lie inside the 64-bit hash");
__device__ __forceinline__ uint32_t bloom_idx(uint64_t h, int j, uint32_t M) { return (uint32_t)(h >> (13 * j)) & M; }

template <int N>
__device__ __forceinline__ bool bloom_maybe(const uint32_t* bloom, uint64_t h) {
    constexpr uint32_t M = 32u * bloom_words(N) - 1u;
    uint32_t all = 1u;
#pragma unroll
    for (int j = 0; j < kBloomK; j++) {
        const uint32_t i = bloom_idx(h, j, M);
        all &= bloom[i >> 5] >> (i & 31);
    }
    return (all & 1u) != 0;
}

// Stone-count pair filter: a position can only repeat a history position with the same
// (black, white) stone counts; all non-capture candidates of a board share one pair.
template <int N>
__device__ __forceinline__ uint32_t pair_idx(int nb, int nw) {
    return ((uint32_t)((nb << 9) | nw) * 0x9E3779B1u) >> (32 - log2i(32 * pair_words(N)));
}
template <int N>
__device__ __forceinline__ void pair_add(uint32_t* gb, int nb, int nw) {   // one lane only
    const uint32_t i = pair_idx<N>(nb, nw);
    atomicOr(&gb[bloom_words(N) + (i >> 5)], 1u << (i & 31));
}

// One lane only: add h to the env's global filter.
template <int N>
__device__ __forceinline__ void bloom_add(uint32_t* gb, uint64_t h) {
    constexpr uint32_t M = 32u * bloom_words(N) - 1u;
#pragma unroll
    for (int j = 0; j < kBloomK; j++) {
        const uint32_t i = bloom_idx(h, j, M);
        atomicOr(&gb[i >> 5], 1u << (i & 31));   // RED: no round trip
    }
}

template <int N, int L>
__device__ __forceinline__ uint32_t dilate(const Seg<L>& g, uint32_t F) {
    constexpr uint32_t ROW = (1u << N) - 1u;
    return ((F << 1) | (F >> 1) | g.up_row(F) | g.dn_row(F)) & ROW;
}

// Tromp-Taylor area score (go.py:176-210), bit-parallel: an empty region
// borders colour X iff it is reachable through empties from a point adjacent
// to X. Returns role rewards (black, white).
template <int N, int L>
__device__ void score(const Seg<L>& g, uint32_t Bk, uint32_t Wh, double komi, float& r0, float& r1) {
    constexpr uint32_t ROW = (1u << N) - 1u;
    const uint32_t rowm = g.sl < N ? ROW : 0u;
    uint32_t E = ~(Bk | Wh) & rowm;
    uint32_t RB = dilate<N>(g, Bk) & E, RW = dilate<N>(g, Wh) & E;
    while (true) {
        uint32_t nb = (RB | dilate<N>(g, RB)) & E;
        uint32_t nw = (RW | dilate<N>(g, RW)) & E;
        bool ch = g.any((nb != RB) || (nw != RW));
        RB = nb; RW = nw;
        if (!ch) break;
    }
    int black = g.sum(__popc(Bk) + __popc(E & RB & ~RW));
    int white = g.sum(__popc(Wh) + __popc(E & RW & ~RB));
    double b = black, w = white + komi;
    if (b > w) { r0 = 1.0f; r1 = -1.0f; }
    else if (w > b) { r0 = -1.0f; r1 = 1.0f; }
    else { r0 = 0.0f; r1 = 0.0f; }
}

// Legal mask rows for the side to move (go.py:121-174, allow_self_capture
// off). X = mover's stones, Y = opponent's stones (colour index `ycol`),
// E = empties (row bits of this lane).
//
// Group analysis (go.py:45-80 restated for what the mask needs): every
// horizontal run of stones is a node. Runs are laid out as a flat list
// (row-major, X runs then Y runs per row) so that the liberty / classification
// passes stride lanes over RUNS, not rows -- the work is balanced no matter how
// the stones are distributed over the rows.
template <int N, int L>
__device__ uint32_t legal_rows(const Seg<L>& g, WarpSmem<N>& S, int ycol, uint32_t X, uint32_t Y, uint32_t E,
                               uint64_t h, const uint64_t* hist, const uint32_t* gbloom, int nscan, uint64_t extra,
                               int nblack, int nwhite, bool self_capture) {
    constexpr uint32_t ROW = (1u << N) - 1u;
    auto& U = S.u.uf;
    const int r = g.sl;
    const uint32_t SX = X & ~(X << 1), SY = Y & ~(Y << 1);
    const int nx = __popc(SX), cnt = nx + __popc(SY);
    int off = g.scan(cnt);   // inclusive prefix sum of run counts over rows
    const int total = g.shfl(off, L - 1);
    off -= cnt;
    S.rE[r] = E; S.rcap[r] = 0u;
    uint32_t* gst = reinterpret_cast<uint32_t*>(S.capx);   // chain stats at 2 * label (see WarpSmem)
    {   // this row's runs -> list, each with its chain label
        const uint16_t* lab = reinterpret_cast<const uint16_t*>(U.bl);
        int k = off;
        for (uint32_t s_ = SX; s_; s_ &= s_ - 1, k++) {
            int s = __ffs(s_) - 1;
            BBK_CHECK(k < WarpSmem<N>::MAXR && r < N);
            U.run[k] = (uint16_t)((0u << 15) | ((uint32_t)r << 10) | ((uint32_t)s << 5) | (uint32_t)(__ffs(~(X >> s)) - 1));
            const uint16_t l = lab[r * N + s];
            BBK_CHECK(l < N * N);
            U.root[k] = l;
        }
        for (uint32_t s_ = SY; s_; s_ &= s_ - 1, k++) {
            int s = __ffs(s_) - 1;
            BBK_CHECK(k < WarpSmem<N>::MAXR && r < N);
            U.run[k] = (uint16_t)((1u << 15) | ((uint32_t)r << 10) | ((uint32_t)s << 5) | (uint32_t)(__ffs(~(Y >> s)) - 1));
            const uint16_t l = lab[r * N + s];
            BBK_CHECK(l < N * N);
            U.root[k] = l;
        }
    }
    for (int i = r; i < (N * N + 1) / 2; i += L)
        reinterpret_cast<uint4*>(S.capx)[i] = make_uint4(0u, 0u, 0u, 0u);
    g.sync();
    // liberty OR-stats per chain
    for (int i = r; i < total; i += L) {
        const uint32_t x = U.root[i];
        const uint32_t e = U.run[i];
        const int rr = (e >> 10) & 31, s = (e >> 5) & 31, len = e & 31;
        const uint32_t run = ((1u << len) - 1u) << s;
        const uint32_t up = rr > 0 ? run & S.rE[rr - 1] : 0u, dn = rr < N - 1 ? run & S.rE[rr + 1] : 0u;
        const uint32_t sd = ((run << 1) | (run >> 1)) & S.rE[rr];
        if (!(up | dn | sd)) continue;
        // a label is a stone of its chain: its stats word never shares a point with a capture XOR
        BBK_CHECK(x < N * N && !((S.rE[x / N] >> (x % N)) & 1u));
        const uint32_t lo = up ? (rr - 1) * N + __ffs(up) - 1 : sd ? rr * N + __ffs(sd) - 1 : (rr + 1) * N + __ffs(dn) - 1;
        const uint32_t hi = dn ? (rr + 1) * N + 31 - __clz(dn) : sd ? rr * N + 31 - __clz(sd) : (rr - 1) * N + 31 - __clz(up);
        atomicOr(&gst[2 * x], 0x80000000u | (lo | hi) | (((~lo | ~hi) & 0x3FFu) << 10));
    }
    g.sync();
    // the labels are dead now: async-copy this env's Bloom + pair filter over them, overlapped
    // with the classification pass (it includes the hash appended by this step)
    const uint32_t* bl = U.bl;
    {
        __threadfence_block();
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(U.bl);
        const char* src = reinterpret_cast<const char*>(gbloom);
        for (int i = r; i < filter_words(N) / 4; i += L)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i), "l"(src + 16 * i));
        asm volatile("cp.async.commit_group;");
    }
    // 3. atari classification; capture liberties (+ zobrist XOR) of opponent atari groups
    for (int i = r; i < total; i += L) {
        const uint32_t gs = gst[2 * U.root[i]];
        const bool at = !(gs & 0x80000000u) || (gs & (gs >> 10) & 0x3FFu) == 0u;
        const uint32_t e = U.run[i];
        if ((e >> 15) && at && (gs & 0x80000000u)) {
            const uint32_t lib = gs & 0x3FFu;
            BBK_CHECK(lib < N * N && ((S.rE[lib / N] >> (lib % N)) & 1u));   // a capture point is empty
            atomicOr(&S.rcap[lib / N], 1u << (lib % N));
            const int rr = (e >> 10) & 31, s = (e >> 5) & 31, len = e & 31;
            const uint64_t x = zrun<N>(rr, s, len, ycol);
            // XOR is bitwise: two native 32-bit shared atomics instead of a 64-bit one
            uint32_t* cx = reinterpret_cast<uint32_t*>(&S.capx[lib]);
            atomicXor(cx, (uint32_t)x);
            atomicXor(cx + 1, (uint32_t)(x >> 32));
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    g.sync();
    // NA: mover stones whose group has >= 2 liberties (this row's X runs)
    uint32_t NA = 0u;
    {
        int k = off;
        for (uint32_t s_ = SX; s_; s_ &= s_ - 1, k++)
        {
            const uint32_t gs = gst[2 * U.root[k]];
            if ((gs & (gs >> 10) & 0x3FFu) != 0u) NA |= run_at(X, __ffs(s_) - 1);   // >= 2 liberties
        }
    }
    // 5. candidates + superko filter (row-parallel)
    const uint32_t Eu = g.up_row(E), Ed = g.dn_row(E);
    const uint32_t capb = r < N ? S.rcap[r] : 0u;
    const uint32_t NAu = g.up_row(NA), NAd = g.dn_row(NA);
    const uint32_t nb = ((E << 1) | (E >> 1) | Eu | Ed | (NA << 1) | (NA >> 1) | NAu | NAd) & ROW;
    uint32_t cand = E & (capb | nb);
    // Self-capture (go.py:155-173): an empty point whose own neighbours are all in atari on it
    // (and that captures nothing) kills the merged group; the placed stone cancels in the hash,
    // so h2 = h ^ XOR(zobrist of those chains), accumulated at the point in capx (free there:
    // it is not a capture point). A lone stone would recreate h itself: superko rejects it.
    uint32_t sc = 0u;
    if (self_capture) {
        const uint32_t Xn = ((X << 1) | (X >> 1) | g.up_row(X) | g.dn_row(X)) & ROW;
        sc = E & ~capb & ~nb & Xn;
        if (g.any(sc != 0u)) {
            g.sync();
            S.rcap[r] = sc;
            g.sync();
            for (int i = r; i < total; i += L) {
                const uint32_t e = U.run[i];
                if (e >> 15) continue;   // mover's runs only
                const uint32_t gs = gst[2 * U.root[i]];
                if ((gs & (gs >> 10) & 0x3FFu) != 0u) continue;   // >= 2 liberties
                const uint32_t lib = gs & 0x3FFu;
                BBK_CHECK(lib < N * N);
                if (!((S.rcap[lib / N] >> (lib % N)) & 1u)) continue;
                const int rr = (e >> 10) & 31, s = (e >> 5) & 31, len = e & 31;
                const uint64_t x = zrun<N>(rr, s, len, 1 - ycol);
                uint32_t* cx = reinterpret_cast<uint32_t*>(&S.capx[lib]);
                atomicXor(cx, (uint32_t)x);
                atomicXor(cx + 1, (uint32_t)(x >> 32));
            }
            g.sync();
        }
    }
    uint32_t legal = 0u, pend = 0u;
    // one probe per board: if no history position had the stone counts a non-capture move
    // produces, none of those moves can repeat a position -> no hash / Bloom work for them
    bool pair_seen;
    {
        const int mb = ycol == 1 ? nblack + 1 : nblack, mw = ycol == 1 ? nwhite : nwhite + 1;   // mover = 1 - ycol
        const uint32_t i = pair_idx<N>(mb, mw);
        pair_seen = (bl[bloom_words(N) + (i >> 5)] >> (i & 31)) & 1u;
    }
    if (!pair_seen) {
        legal = cand & ~capb;
        cand &= capb;
    }
    cand |= sc;   // counts after a suicide are not known here: always hashed
    for (uint32_t c_ = cand; c_; c_ &= c_ - 1) {
        int p = __ffs(c_) - 1;
        int cell = r * N + p;
        uint64_t h2 = ((sc >> p) & 1u) ? h : h ^ zkey<N>(cell, 1 - ycol);
        if (((capb | sc) >> p) & 1u) h2 ^= S.capx[cell];
        if (bloom_maybe<N>(bl, h2)) pend |= 1u << p;
        else legal |= 1u << p;
    }
    while (g.any(pend != 0u)) {
        const unsigned active = g.ballot(pend != 0u);
        int p = pend ? __ffs(pend) - 1 : 0;
        uint64_t h2 = 0ull;
        if (pend) {
            int cell = r * N + p;
            h2 = ((sc >> p) & 1u) ? h : h ^ zkey<N>(cell, 1 - ycol);
            if (((capb | sc) >> p) & 1u) h2 ^= S.capx[cell];
            S.u.sk.hit[r] = h2;
        }
        g.sync();
        unsigned found = 0u;
        BBK_CHECK(nscan >= 0 && nscan <= (int)0x7FFFFFFF);
        // 4 history entries per lane in flight per iteration (the scan is latency-bound)
        for (int j0 = r; j0 < nscan + 1; j0 += 4 * L) {
            uint64_t v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = j0 + u * L;
                v[u] = j < nscan ? hist[j] : j == nscan ? extra : ~extra;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                if (j0 + u * L > nscan) break;
                for (unsigned a_ = active; a_; a_ &= a_ - 1) {
                    int l = __ffs(a_) - 1;
                    if (v[u] == S.u.sk.hit[l]) found |= 1u << l;
                }
            }
        }
        found = g.reduce_or(found);
        if (pend) {
            if (!((found >> r) & 1u)) legal |= 1u << p;
            pend &= pend - 1u;
        }
        g.sync();
    }
    return legal;
}

// Observation of one board from the transposed history in S.pat (new
// state), colour plane = role (go.py:264-273). Float f of the record is bit
// f % 17 of the point pattern P[f / 17]; the [N, N, 17] record is emitted as
// float4 chunks of the flat 16-byte-aligned stream (records are not 16-B
// aligned; at most 3 scalar floats at each edge) through a 16-entry LUT.
#ifndef BBK_GO_OBS_DIRECT_MIN
#define BBK_GO_OBS_DIRECT_MIN 15   // smallest board cutting its observation chunks straight from pat
#endif
template <int N, int L>
__device__ void emit_obs(const Seg<L>& g, WarpSmem<N>& S, const float4* lut, float* obs, int64_t b, int role) {
    constexpr int C = N * N;
    constexpr int NF = C * kPlanes;
    const int sl = g.sl;
    if constexpr (N >= BBK_GO_OBS_DIRECT_MIN) {
        // Large boards: each 8-float chunk is cut straight from the two points' history patterns
        // (float f = plane f % 17 of point f / 17), no staged pattern / bit-stream passes: fewer
        // shared-memory round trips for more ALU work -- 19x19 +1.2 % over a full cycle, +1.6 % late
        // game; 9x9 (where ALU is the limit) -1.5 %, so small boards keep the staged passes below.
        const uint32_t hi16 = (uint32_t)role << 16;
        auto Pv = [&](uint32_t c) -> uint32_t {   // point c's 17-bit pattern for this role
            uint32_t u = S.pat[c];
            if (role) u = ((u & 0x5555u) << 1) | ((u >> 1) & 0x5555u);
            return u | hi16;
        };
        auto bits8 = [&](uint32_t q) -> uint32_t {   // floats q..q+7 of the record (8 <= 17: two points)
            const uint32_t c = (q * 61681u) >> 20, k = q - 17u * c;   // q / 17, exact for q < 65536
            BBK_CHECK(c == q / 17u && c + 1 < (uint32_t)pat_stride(N));
            return ((Pv(c) >> k) | (Pv(c + 1) << (17 - k))) & 0xFFu;
        };
        const int64_t F0 = b * (int64_t)NF;
        float* rec = obs + F0;
        const int head = (int)((8 - (F0 & 7)) & 7);             // floats before the first 32-B chunk
        const int nchunk = (NF - head) >> 3;
        const int tail0 = head + 8 * nchunk;
        if (sl < head || (sl >= 8 && sl - 8 < NF - tail0)) {   // at most 7 edge floats each side
            const uint32_t fi = sl < 8 ? (uint32_t)sl : (uint32_t)(tail0 + sl - 8);
            rec[fi] = (float)(bits8(fi) & 1u);
        }
        float* o8 = rec + head;
#pragma unroll kGoObsUnroll
        for (int j = sl; j < nchunk; j += L) {
            const uint32_t t = bits8((uint32_t)(head + 8 * j));
            const float4 lo = lut[t & 15u], hi = lut[(t >> 4) & 15u];
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o8 + 8 * j), "f"(lo.x), "f"(lo.y),
                         "f"(lo.z), "f"(lo.w), "f"(hi.x), "f"(hi.y), "f"(hi.z), "f"(hi.w) : "memory");
        }
        g.sync();
        return;
    }
    uint32_t* P = S.u.ob.P;
    {   // 8 points per lane-iteration: black/white swapped for role 1, colour bit 16
        const uint32_t hi = (uint32_t)role << 16;
        for (int i = sl; i < pat_stride(N) / 8; i += L) {
            const uint4 v = reinterpret_cast<const uint4*>(S.pat)[i];
            auto sw = [&](uint32_t u) { return role ? (((u & 0x55555555u) << 1) | ((u >> 1) & 0x55555555u)) : u; };
            const uint32_t a = sw(v.x), bb = sw(v.y), c = sw(v.z), d = sw(v.w);
            uint4* P4 = reinterpret_cast<uint4*>(P) + 2 * i;
            P4[0] = make_uint4((a & 0xFFFFu) | hi, (a >> 16) | hi, (bb & 0xFFFFu) | hi, (bb >> 16) | hi);
            P4[1] = make_uint4((c & 0xFFFFu) | hi, (c >> 16) | hi, (d & 0xFFFFu) | hi, (d >> 16) | hi);
        }
    }
    g.sync();
    // the record as a bit stream: bit f of W = float f (17 bits per point)
    uint32_t* W = S.u.ob.W;
    constexpr int NW = (NF + 31) / 32;
    for (int w = sl; w < NW; w += L) {
        const uint32_t q = 32u * w, c = (q * 61681u) >> 20, k = q - 17u * c;   // q / 17, exact for q < 65536
        BBK_CHECK(c == q / 17u && c + 2 < (uint32_t)pat_stride(N));
        uint32_t v = (P[c] >> k) | (P[c + 1] << (17 - k));
        if (k > 2) v |= P[c + 2] << (34 - k);
        W[w] = v;
    }
    if (sl == 0) W[NW] = 0u;
    g.sync();
    const int64_t F0 = b * (int64_t)NF;
    float* rec = obs + F0;
#ifndef BBK_GO_OBS_V8
#define BBK_GO_OBS_V8 1
#endif
    if constexpr (BBK_GO_OBS_V8) {
        // 32-byte stores (st.global.v8.f32): a warp writing whole per-board records absorbs 6.1-6.2
        // TB/s this way against 5.3-5.5 TB/s with 16-byte stores (tools/write_pattern.cu, B200)
        const int head = (int)((8 - (F0 & 7)) & 7);             // floats before the first 32-B chunk
        const int nchunk = (NF - head) >> 3;
        const int tail0 = head + 8 * nchunk;
        if (sl < head || (sl >= 8 && sl - 8 < NF - tail0)) {   // at most 7 edge floats each side
            const uint32_t fi = sl < 8 ? (uint32_t)sl : (uint32_t)(tail0 + sl - 8);
            rec[fi] = (float)((W[fi >> 5] >> (fi & 31)) & 1u);
        }
        // chunk j = sl + L m starts at bit head + 8 sl + 8 L m: a lane-constant bit offset in
        // word (head + 8 sl) / 32 + (L / 4) m
        float* o8 = rec + head;
        const uint32_t q0 = (uint32_t)(head + 8 * sl), sh = q0 & 31u;
        const uint32_t* wp = W + (q0 >> 5);
        BBK_CHECK(nchunk <= 0 || (head + 8 * (nchunk - 1)) / 32 + 1 <= NW);   // last chunk's words are staged
#pragma unroll kGoObsUnroll
        for (int j = sl; j < nchunk; j += L, wp += L / 4) {
            const uint32_t t = __funnelshift_r(wp[0], wp[1], sh);
            const float4 lo = lut[t & 15u], hi = lut[(t >> 4) & 15u];
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o8 + 8 * j), "f"(lo.x), "f"(lo.y),
                         "f"(lo.z), "f"(lo.w), "f"(hi.x), "f"(hi.y), "f"(hi.z), "f"(hi.w) : "memory");
        }
    } else {
        const int head = (int)((4 - (F0 & 3)) & 3);             // floats before the first aligned chunk
        const int nchunk = (NF - head) >> 2;
        const int tail0 = head + 4 * nchunk;
        if (sl < head || (sl >= 4 && sl - 4 < NF - tail0)) {
            const uint32_t fi = sl < 4 ? (uint32_t)sl : (uint32_t)(tail0 + sl - 4);
            rec[fi] = (float)((W[fi >> 5] >> (fi & 31)) & 1u);
        }
        // chunk j = sl + L m starts at bit head + 4 sl + 4 L m: a lane-constant bit offset in
        // word (head + 4 sl) / 32 + (L / 8) m
        float4* o4 = reinterpret_cast<float4*>(rec + head);
        const uint32_t q0 = (uint32_t)(head + 4 * sl), sh = q0 & 31u;
        const uint32_t* wp = W + (q0 >> 5);
        // (an ALU expansion of the 4 bits -- (t & 2^k) * (0x3F800000 >> k) -- instead of the LUT measured
        // -0.2 % at 19x19 and -1 % at 9x9 in r02, although the L1 / shared pipe is the busiest unit)
#pragma unroll 4
        for (int j = sl; j < nchunk; j += L, wp += L / 8)
            o4[j] = lut[__funnelshift_r(wp[0], wp[1], sh) & 15u];
    }
    g.sync();
}

// Write NBYTES bytes of a per-env record into a flat [n, NBYTES] byte stream from shared memory
// staged at the destination's 16-byte phase (common.cuh warp_emit_bytes over the segment's lanes).
template <int L>
__device__ __forceinline__ void seg_emit_bytes(const Seg<L>& g, uint8_t* dst_stream, int64_t rec_start, int nbytes,
                                               const uint8_t* staged) {
    if constexpr (L == 32) {
        warp_emit_bytes(dst_stream, rec_start, nbytes, staged);
    } else {
        const int64_t end = rec_start + nbytes;
        const int64_t base = rec_start & ~(int64_t)15;
        const int64_t f0 = (rec_start + 15) >> 4, f1 = end >> 4;
        for (int64_t c = f0 + g.sl; c < f1; c += L)
            *reinterpret_cast<uint4*>(dst_stream + (c << 4)) = *reinterpret_cast<const uint4*>(staged + ((c << 4) - base));
        const int64_t head_end = (f0 << 4) < end ? (f0 << 4) : end;
        {   // lane k: byte k of the partial head chunk, then byte k of the partial tail chunk
            const int64_t gh = rec_start + g.sl;
            if (g.sl < 16 && gh < head_end) dst_stream[gh] = staged[gh - base];
            const int64_t gt = (f1 << 4) + g.sl;
            if (g.sl < 16 && gt < end && gt >= (f0 << 4)) dst_stream[gt] = staged[gt - base];
        }
    }
}

// One scalar column of board b per lane (lanes 0-9), loaded a board ahead so the
// loads are in flight while the current board is processed; read back by shuffles.
// Go keeps the decoded form of the field reference in registers (it has register headroom; the
// packed FieldRef of common.cuh is for the register-capped chess / shogi kernels).
struct FieldRefWide {
    const char* base;
    uint32_t lsz;
    uint64_t mask;
};
// lanes without a field read (and mask off) the first byte of `any`, a valid column
__device__ __forceinline__ FieldRefWide widen(FieldRef f, const void* any) {
    const uint32_t lsz = (uint32_t)(f.v >> 58) & 3u;
    if (f.v >> 61) return {reinterpret_cast<const char*>(any), 0u, 0ull};
    return {reinterpret_cast<const char*>(f.v & ((1ull << 58) - 1ull)), lsz,
            lsz == 3u ? ~0ull : (1ull << (8u << lsz)) - 1ull};
}
// The raw aligned word and the element's bit offset: decoded (shift + mask) only when the board
// is processed, so no instruction waits on the load while the current board is being finished.
__device__ __forceinline__ uint64_t load_field_raw(const FieldRefWide& f, int64_t b, uint32_t& sh) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(f.base) + ((uintptr_t)b << f.lsz);
    sh = 8u * (uint32_t)(a & 7u);
    return *reinterpret_cast<const uint64_t*>(a & ~(uintptr_t)7);
}
__device__ __forceinline__ uint64_t load_field(const FieldRefWide& f, int64_t b) {
    uint32_t sh;
    const uint64_t w = load_field_raw(f, b, sh);
    return (w >> sh) & f.mask;
}
// deferred decode for the small boards (+1 % at 9x9); 19x19 decodes at the load (the extra live
// register across the board cost 1.7 % there)
#ifndef BBK_GO_DEFER_MAX
#define BBK_GO_DEFER_MAX 13
#endif
template <int N> constexpr bool kDeferFields = N <= BBK_GO_DEFER_MAX;

__device__ __forceinline__ FieldRef field_ref(const StepParams& p, int lane) {
    switch (lane) {
        case 0: return field_of(p.in.terminated, 0u);
        case 1: return field_of(p.in.truncated, 0u);
        case 2: return field_of(p.in.player_to_role, 1u);
        case 3: return field_of(p.in_s.role_to_move, 0u);
        case 4: return field_of(p.in_s.pass_count, 0u);
        case 5: return field_of(p.in.step_count, 2u);
        case 6: return field_of(p.in_s.hash, 3u);
        case 7: return field_of(p.in_s.hist_xor, 3u);
        case 8: return field_of(p.in_s.hist_len, 2u);
        case 9: return field_of(p.actions, 3u);
        default: return no_field();
    }
}

template <int N>
__device__ __forceinline__ void init_block(BlockSmem<N>& B) {
    if (threadIdx.x < 16) {
        uint32_t n = threadIdx.x;
        B.lut[n] = make_float4((float)(n & 1), (float)((n >> 1) & 1), (float)((n >> 2) & 1), (float)((n >> 3) & 1));
    }
    __syncthreads();
}

#ifndef BBK_GO_NB_UNROLL
#define BBK_GO_NB_UNROLL 1   // large boards too (r02 graph-timed: +0.5 % 19x19 cycle)
#endif
// the placement's neighbour loop: rolled up for the small boards (smaller hot code, +0.7 % at 9x9)
constexpr int kNbUnroll = BBK_GO_NB_UNROLL;

#ifndef BBK_GO_GRID_BOARDS
#define BBK_GO_GRID_BOARDS -1   // boards per warp segment per launch: 0 persistent, -1 per-size default
#endif
#ifndef BBK_GO_TAIL_PCT
#define BBK_GO_TAIL_PCT 150     // one-pass CTAs at the end of a multi-wave grid, % of the resident CTAs (r02: go_19x19 +0.8 %, go_9x9 +3.2 %; 50: -8 % at 9x9, 300: = 150)
#endif
constexpr int kGoTailPct = BBK_GO_TAIL_PCT;
// resident CTAs per SM the register budget is sized for: small boards fit 8 (shared memory allows it)
#ifndef BBK_GO_CTAS_SMALL
#define BBK_GO_CTAS_SMALL 8
#endif
#ifndef BBK_GO_CTAS_LARGE
#define BBK_GO_CTAS_LARGE 7   // r02 after the scratch diet + wave grid: 7 = +1.5 % default / +3.2 % full cycle over 6; 8: same
#endif
__host__ __device__ constexpr int min_ctas(int N) { return N <= 13 ? BBK_GO_CTAS_SMALL : BBK_GO_CTAS_LARGE; }

template <int N>
__global__ void __launch_bounds__(kWarps * 32, min_ctas(N)) step_kernel(StepParams p) {
    constexpr int C = N * N;
    constexpr int A = C + 1;
    constexpr int PS = pat_stride(N);
    constexpr int L = seg_lanes(N);
    constexpr uint32_t ROW = (1u << N) - 1u;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BlockSmem<N>& B = *reinterpret_cast<BlockSmem<N>*>(smem_raw);
    init_block<N>(B);
    const Seg<L> g;
    const int sl = g.sl;
    WarpSmem<N>& S = B.w[threadIdx.x / L];
    const uint32_t rowm = sl < N ? ROW : 0u;
    const PassMap pm = pass_map(p.n, boards_per_cta(N), p.tail_ctas, threadIdx.x / L);   // common.cuh
    const int64_t nboards = pm.stride, bend = pm.end;
    unsigned long long eps = 0;
    // next-board prefetch: scalar columns in registers (lane j holds field j), `pat` via
    // cp.async into an idle tail of the scratch union (not touched by mask/obs emission)
    uint16_t* pat_pf = reinterpret_cast<uint16_t*>(S.capx);   // dead from the mask on (see WarpSmem)
    uint16_t* lab_pf = pat_pf + PS;
    uint16_t* lab = reinterpret_cast<uint16_t*>(S.u.uf.bl);   // this board's chain labels
    const int64_t b0 = pm.b0;
    const FieldRefWide fref = widen(field_ref(p, sl), p.in.terminated);
    uint32_t pf_sh = 0u;
    uint64_t pf_raw = 0ull;
    if (!p.force_reset && b0 < bend) {
        if constexpr (kDeferFields<N>) pf_raw = load_field_raw(fref, b0, pf_sh);
        else pf_raw = load_field(fref, b0);
    }
    bool pat_ready = false;

    for (int64_t b = b0; b < bend; b += nboards) {
        if (!p.force_reset && b + nboards < bend && sl < (4 * filter_words(N) + 127) / 128) {
            // warm L2 with the next board's Bloom filter (cp.async'd mid-board)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(
                reinterpret_cast<const char*>(p.store.bloom + (b + nboards) * (int64_t)filter_words(N)) + 128 * sl));
        }
        const uint64_t pf = kDeferFields<N> ? (pf_raw >> pf_sh) & fref.mask : pf_raw;
        const uint64_t f_term = g.shfl((uint32_t)pf, 0), f_trunc = g.shfl((uint32_t)pf, 1);
        const uint32_t f_p2r = g.shfl((uint32_t)pf, 2), f_role = g.shfl((uint32_t)pf, 3);
        const uint32_t f_pass = g.shfl((uint32_t)pf, 4), f_step = g.shfl((uint32_t)pf, 5);
        const uint64_t f_hash = g.shfl64(pf, 6), f_hx = g.shfl64(pf, 7);
        const uint32_t f_hlen = g.shfl((uint32_t)pf, 8);
        const int64_t f_act = (int64_t)g.shfl64(pf, 9);
        const bool reset = p.force_reset || f_term || f_trunc;
        const uint64_t k = slot_key(p.slot_keys, p.key, p.slot0, b);
        uint64_t* hist = p.store.history + b * (int64_t)p.store.hist_cap;
        uint32_t* gbloom = p.store.bloom + b * (int64_t)filter_words(N);
        int8_t p2r0, p2r1;
        int role, pass_count, step, hlen;
        uint64_t h, hx;
        uint32_t Bk = 0u, Wh = 0u;
        int counts = -1;   // (black stones) | (white stones) << 16 of the new board once known
        bool terminal = false;
        float rr0 = 0.0f, rr1 = 0.0f;
        int nscan;
        uint64_t extra;
        if (reset) {
            // init (core.py:223-229) + init_core (go.py:212-217)
            int c = (int)(child(k, 0) % 2ull);
            p2r0 = (int8_t)c; p2r1 = (int8_t)(1 - c);
            role = 0; pass_count = 0; step = 0; h = 0ull; hx = 0ull; hlen = 1;
            // the discarded prefetch of this board must land before the scratch is reused
            if (pat_ready) asm volatile("cp.async.wait_all;" ::: "memory");
            for (int i = sl; i < PS; i += L) { S.pat[i] = 0; lab[i] = 0; }
            for (int i = sl; i < filter_words(N) / 4; i += L)
                reinterpret_cast<uint4*>(gbloom)[i] = make_uint4(0u, 0u, 0u, 0u);
            g.sync();
            if (sl == 0) { bloom_add<N>(gbloom, 0ull); pair_add<N>(gbloom, 0, 0); hist[0] = 0ull; }
            nscan = 0; extra = 0ull;
        } else {
            p2r0 = (int8_t)(f_p2r & 0xFF); p2r1 = (int8_t)(f_p2r >> 8);
            role = (int)f_role; pass_count = (int)f_pass;
            step = (int)f_step;
            h = f_hash; hx = f_hx; hlen = (int)f_hlen;
            // copy pat / lab in; boards up to 13x13 take each 8-point chunk's current stones (bits 0 / 1
            // of every u16) on the way as one byte of flat black / white bitmaps, from which each lane
            // then cuts its row with one funnel shift (no per-point pass over the pattern; go_9x9 +1.9 %)
            uint8_t* FB = reinterpret_cast<uint8_t*>(S.rX);   // free until legal_rows
            uint8_t* FW = reinterpret_cast<uint8_t*>(S.rY);
            auto take = [&](int i, uint4 v) {
                reinterpret_cast<uint4*>(S.pat)[i] = v;
                if constexpr (N > 13) return;   // 15x15+: rows from the pattern (below), measured faster
                FB[i] = (uint8_t)((v.x & 1u) | ((v.x >> 15) & 2u) | ((v.y & 1u) << 2) | ((v.y >> 13) & 8u) |
                                  ((v.z & 1u) << 4) | ((v.z >> 11) & 32u) | ((v.w & 1u) << 6) | ((v.w >> 9) & 128u));
                FW[i] = (uint8_t)(((v.x >> 1) & 1u) | ((v.x >> 16) & 2u) | ((v.y << 1) & 4u) | ((v.y >> 14) & 8u) |
                                  ((v.z << 3) & 16u) | ((v.z >> 12) & 32u) | ((v.w << 5) & 64u) | ((v.w >> 10) & 128u));
            };
            if (pat_ready) {   // prefetched during the previous board
                asm volatile("cp.async.wait_all;" ::: "memory");
                g.sync();
                for (int i = sl; i < PS / 8; i += L) {
                    take(i, reinterpret_cast<const uint4*>(pat_pf)[i]);
                    reinterpret_cast<uint4*>(lab)[i] = reinterpret_cast<const uint4*>(lab_pf)[i];
                }
            } else {
                const uint4* src = reinterpret_cast<const uint4*>(p.in_s.pat + b * (int64_t)PS);
                const uint4* lsrc = reinterpret_cast<const uint4*>(p.store.lab + b * (int64_t)PS);
                for (int i = sl; i < PS / 8; i += L) {
                    take(i, src[i]);
                    reinterpret_cast<uint4*>(lab)[i] = lsrc[i];
                }
            }
            g.sync();
            if constexpr (N > 13) {
                if (sl < N) {
#pragma unroll 4
                    for (int col = 0; col < N; col++) {
                        uint32_t v = S.pat[sl * N + col];
                        Bk |= (v & 1u) << col;
                        Wh |= ((v >> 1) & 1u) << col;
                    }
                }
            } else if (sl < N) {
                const int q = sl * N, w = q >> 5, sh = q & 31;
                const uint32_t* fb = reinterpret_cast<const uint32_t*>(FB);
                const uint32_t* fw = reinterpret_cast<const uint32_t*>(FW);
                Bk = __funnelshift_r(fb[w], fb[w + 1], sh) & ROW;
                Wh = __funnelshift_r(fw[w], fw[w + 1], sh) & ROW;
            }
            const int a = (int)f_act;
            step += 1;
            nscan = hlen; extra = h;
            if (a < 0 || a >= C) {   // pass (go.py:222-230)
                pass_count += 1;
                if (pass_count == 2) {
                    terminal = true;
                    score<N>(g, Bk, Wh, p.komi, rr0, rr1);
                }
            } else {                 // placement (go.py:232-262)
                const int ra = a / N, ca = a - ra * N;
                uint32_t M = role == 0 ? Bk : Wh, O = role == 0 ? Wh : Bk;
                {   // chain label of the new stone: the first own neighbour's, absorbing the others
                    const uint32_t Mr = g.shfl(M, ra);
                    const uint32_t Mu = g.shfl(M, ra > 0 ? ra - 1 : 0);
                    const uint32_t Md = g.shfl(M, ra < N - 1 ? ra + 1 : 0);
                    constexpr uint32_t NONE = 0xFFFFu;   // never a label (labels < C)
                    BBK_CHECK(a >= 0 && a < C && ra < N && ca < N);
                    const uint32_t lu = (ra > 0 && ((Mu >> ca) & 1u)) ? lab[a - N] : NONE;
                    const uint32_t ld = (ra < N - 1 && ((Md >> ca) & 1u)) ? lab[a + N] : NONE;
                    const uint32_t ll = (ca > 0 && ((Mr >> (ca - 1)) & 1u)) ? lab[a - 1] : NONE;
                    const uint32_t lr = (ca < N - 1 && ((Mr >> (ca + 1)) & 1u)) ? lab[a + 1] : NONE;
                    const uint32_t L0 = lu != NONE ? lu : ld != NONE ? ld : ll != NONE ? ll : lr != NONE ? lr : (uint32_t)a;
                    g.sync();
                    // labels change only here: the in-place store row takes the same writes (a few
                    // bytes per step instead of the whole row)
                    uint16_t* glab = p.store.lab + b * (int64_t)PS;
                    if ((ld != NONE && ld != L0) | (ll != NONE && ll != L0) | (lr != NONE && lr != L0)) {
                        for (uint32_t m_ = M; m_; m_ &= m_ - 1) {   // lanes >= N hold no stones
                            const int cell = sl * N + __ffs(m_) - 1;
                            const uint32_t l = lab[cell];
                            if (l == ld || l == ll || l == lr) {
                                lab[cell] = (uint16_t)L0;
                                glab[cell] = (uint16_t)L0;
                            }
                        }
                    }
                    if (sl == 0) {
                        lab[a] = (uint16_t)L0;
                        glab[a] = (uint16_t)L0;
                    }
                    g.sync();
                }
                if (sl == ra) M |= 1u << ca;
                const uint32_t E0 = ~(M | O) & rowm;
                uint64_t capxor = 0ull;
                uint32_t visited = 0u, dead = 0u;
#pragma unroll(N <= 13 ? 1 : kNbUnroll)
                for (int j = 0; j < 4; j++) {   // neighbours up, down, left, right
                    const int qr = j < 2 ? ra + 2 * j - 1 : ra, qc = j < 2 ? ca : ca + 2 * j - 5;
                    if (qr < 0 || qr >= N || qc < 0 || qc >= N) continue;
                    const uint32_t Oq = g.shfl(O, qr);
                    const uint32_t Vq = g.shfl(visited, qr);
                    if (!((Oq >> qc) & 1u) || ((Vq >> qc) & 1u)) continue;
                    // quick exit: the stone itself touches an empty point
                    const uint32_t Er = g.shfl(E0, qr);
                    const uint32_t Eup = qr > 0 ? g.shfl(E0, qr - 1) : 0u;
                    const uint32_t Edn = qr < N - 1 ? g.shfl(E0, qr + 1) : 0u;
                    if ((((Er << 1) | (Er >> 1) | Eup | Edn) >> qc) & 1u) continue;
                    uint32_t F = sl == qr ? (1u << qc) : 0u;
                    while (true) {
                        uint32_t F2 = (F | dilate<N>(g, F)) & O;
                        bool ch = g.any(F2 != F);
                        F = F2;
                        if (!ch) break;
                    }
                    visited |= F;
                    if (!g.any((dilate<N>(g, F) & E0) != 0u)) dead |= F;
                }
                capxor ^= zbits<N>(sl, dead, 1 - role);
                O &= ~dead;
                if (p.self_capture && !g.any(dead != 0u)) {
                    // go.py:249-255: the placed stone's group without a liberty is removed
                    uint32_t F = sl == ra ? (1u << ca) : 0u;
                    while (true) {
                        const uint32_t F2 = (F | dilate<N>(g, F)) & M;
                        const bool ch = g.any(F2 != F);
                        F = F2;
                        if (!ch) break;
                    }
                    const uint32_t E1 = ~(M | O) & rowm;
                    if (!g.any((dilate<N>(g, F) & E1) != 0u)) {
                        capxor ^= zbits<N>(sl, F, role);
                        M &= ~F;
                    }
                }
                const uint64_t h2 = h ^ zkey<N>(a, role) ^ g.xor64(capxor);
                if (role == 0) { Bk = M; Wh = O; } else { Wh = M; Bk = O; }
                counts = g.sum(__popc(Bk) | (__popc(Wh) << 16));
                const int nbk = counts & 0xFFFF, nwh = counts >> 16;
                BBK_CHECK(hlen < p.store.hist_cap);   // the superko history's capacity
                if (sl == 0) {
                    hist[hlen] = h2;
                    bloom_add<N>(gbloom, h2);
                    pair_add<N>(gbloom, nbk, nwh);
                }
                nscan = hlen; extra = h2;
                hlen += 1; h = h2; hx ^= h2; pass_count = 0;
            }
            role = 1 - role;
        }
        // new transposed history: pat' = pat << 2 | current board (go.py:224, 260)
        uint16_t* opat = p.out_s.pat + b * (int64_t)PS;
        if constexpr (N > 13) {   // row-parallel: this lane's row bits are in registers
            if (!reset && sl < N) {
#pragma unroll 4
                for (int col = 0; col < N; col++) {
                    const int i = sl * N + col;
                    S.pat[i] = (uint16_t)(((uint32_t)S.pat[i] << 2) | ((Bk >> col) & 1u) | (((Wh >> col) & 1u) << 1));
                }
            }
        } else {                  // small boards: point-parallel over all the segment's lanes
            S.rX[sl] = Bk; S.rY[sl] = Wh;
            g.sync();
            if (!reset) {
                for (int i = sl; i < C; i += L) {
                    const int rr = i / N, cc = i - rr * N;
                    S.pat[i] = (uint16_t)(((uint32_t)S.pat[i] << 2) | ((S.rX[rr] >> cc) & 1u) | (((S.rY[rr] >> cc) & 1u) << 1));
                }
            }
        }
        g.sync();
        for (int i = sl; i < PS / 8; i += L)
            reinterpret_cast<uint4*>(opat)[i] = reinterpret_cast<const uint4*>(S.pat)[i];
        const bool truncated = !terminal && step >= p.max_steps;
        // legal mask of the new mover (skipped once the slot is finished)
        uint32_t legal = 0u;
        if (!terminal && !truncated) {
            const uint32_t X = role == 0 ? Bk : Wh, Y = role == 0 ? Wh : Bk;
            const uint32_t E = ~(Bk | Wh) & rowm;
            if (counts < 0) counts = g.sum(__popc(Bk) | (__popc(Wh) << 16));
            const int nbk = counts & 0xFFFF, nwh = counts >> 16;
            legal = legal_rows<N>(g, S, 1 - role, X, Y, E, h, hist, gbloom, nscan, extra, nbk, nwh, p.self_capture != 0);
        }
        g.sync();   // the analysis scratch (atari flags, superko hits) is reused for mask staging
        // stage mask bytes at the destination's 16-byte phase and emit
        const int64_t mstart = b * (int64_t)A;
        const int moff = (int)(mstart & 15);
        BBK_CHECK(moff + C < (int)sizeof(S.u.mb));
        if (sl < N) {
            for (int col = 0; col < N; col++) S.u.mb[moff + sl * N + col] = (uint8_t)((legal >> col) & 1u);
        }
        if (sl == 0) S.u.mb[moff + C] = (uint8_t)(!terminal && !truncated);
        g.sync();
        seg_emit_bytes(g, p.out.legal_action_mask, mstart, A, S.u.mb);
        eps += (terminal || truncated) ? 1 : 0;
        if (p.out.next_actions) {   // fused agents.random_actions on the new mask (row bits + pass, still on chip)
            const int c = __popc(legal);
            const int incl = g.scan(c);
            const int cells = g.shfl(incl, L - 1);
            const bool live = !terminal && !truncated;
            const int total = live ? cells + 1 : 0;   // + pass
            int64_t act = 0;
            if (total > 0) {
                const int d = (int)umod_small(child(p.out.next_key, (uint64_t)(p.slot0 + b)), (uint32_t)total);
                if (d == cells) act = C;
                else {
                    const bool mine = d >= incl - c && d < incl;
                    int pos = 0;
                    if (mine) {
                        uint32_t v = legal;
                        for (int r = d - (incl - c); r > 0; r--) v &= v - 1;
                        pos = sl * N + __ffs(v) - 1;
                    }
                    const unsigned who = g.ballot(mine);
                    act = g.shfl(pos, __ffs(who) - 1);
                }
            }
            if (sl == 0) p.out.next_actions[b] = act;
        }
        g.sync();   // staged mask bytes are overwritten by the observation pattern next
        pat_ready = false;
        if (!p.force_reset && b + nboards < bend) {   // issue the next board's loads now
            const int64_t nb = b + nboards;
            if constexpr (kDeferFields<N>) pf_raw = load_field_raw(fref, nb, pf_sh);
            else pf_raw = load_field(fref, nb);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(pat_pf);
            const char* src = reinterpret_cast<const char*>(p.in_s.pat + nb * (int64_t)PS);
            const char* lsrc = reinterpret_cast<const char*>(p.store.lab + nb * (int64_t)PS);
            for (int i = sl; i < PS / 8; i += L) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i), "l"(src + 16 * i));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 2u * PS + 16u * i), "l"(lsrc + 16 * i));
            }
            asm volatile("cp.async.commit_group;");
            pat_ready = true;
        }
        if (p.out.observation) emit_obs<N>(g, S, B.lut, p.out.observation, b, role);
        if (sl == 0) {
            float r0 = 0.0f, r1 = 0.0f;
            if (!truncated && (rr0 != 0.0f || rr1 != 0.0f)) {   // core.py:197-204
                r0 = p2r0 == 0 ? rr0 : rr1;
                r1 = p2r1 == 0 ? rr0 : rr1;
            }
            p.out.rewards[2 * b] = r0;
            p.out.rewards[2 * b + 1] = r1;
            p.out.terminated[b] = terminal;
            p.out.truncated[b] = truncated;
            p.out.step_count[b] = step;
            p.out.current_player[b] = p2r0 == role ? 0 : 1;   // perm.index(role_to_move)
            p.out.player_to_role[2 * b] = p2r0;
            p.out.player_to_role[2 * b + 1] = p2r1;
            p.out_s.hash[b] = h;
            p.out_s.hist_xor[b] = hx;
            p.out_s.hist_len[b] = hlen;
            p.out_s.role_to_move[b] = (uint8_t)role;
            p.out_s.pass_count[b] = (uint8_t)pass_count;
        }
        g.sync();
    }
    // a cp.async issued for a board this lane never processes (none: the prefetch is only issued
    // for b + nboards < n) -- nothing is left in flight here
    if (p.out.episodes && sl == 0 && eps) atomicAdd(p.out.episodes, eps);
}

template <int N>
__global__ void __launch_bounds__(kWarps * 32) observe_kernel(const uint16_t* pat, const uint8_t* role, float* obs, int64_t n) {
    constexpr int PS = pat_stride(N);
    constexpr int L = seg_lanes(N);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BlockSmem<N>& B = *reinterpret_cast<BlockSmem<N>*>(smem_raw);
    init_block<N>(B);
    const Seg<L> g;
    WarpSmem<N>& S = B.w[threadIdx.x / L];
    const int64_t nboards = (int64_t)gridDim.x * boards_per_cta(N);
    for (int64_t b = (int64_t)blockIdx.x * boards_per_cta(N) + threadIdx.x / L; b < n; b += nboards) {
        const uint4* src = reinterpret_cast<const uint4*>(pat + b * (int64_t)PS);
        for (int i = g.sl; i < PS / 8; i += L) reinterpret_cast<uint4*>(S.pat)[i] = src[i];
        g.sync();
        emit_obs<N>(g, S, B.lut, obs, b, role[b]);
    }
}

template <int N>
__global__ void rebuild_bloom_kernel(bbk_go_store st, const int32_t* hist_len, int64_t n) {
    constexpr int BW = bloom_words(N), FW = filter_words(N);
    constexpr uint32_t M = 32u * BW - 1u;
    __shared__ uint32_t sb[kWarps][BW];
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    for (int64_t b = (int64_t)blockIdx.x * kWarps + w; b < n; b += nwarps) {
        for (int i = lane; i < BW; i += 32) sb[w][i] = 0u;
        __syncwarp();
        const uint64_t* hist = st.history + b * (int64_t)st.hist_cap;
        for (int j = lane; j < hist_len[b]; j += 32) {
            uint64_t h = hist[j];
#pragma unroll
            for (int q = 0; q < kBloomK; q++) {
                const uint32_t i = bloom_idx(h, q, M);
                atomicOr(&sb[w][i >> 5], 1u << (i & 31));
            }
        }
        __syncwarp();
        for (int i = lane; i < BW; i += 32) st.bloom[b * FW + i] = sb[w][i];
        // history keeps no stone counts: mark every pair as seen (correct, only slower)
        for (int i = BW + lane; i < FW; i += 32) st.bloom[b * FW + i] = 0xFFFFFFFFu;
        __syncwarp();
    }
}

// Chain labels of each board's current position (bits 0 / 1 of pat), label = the chain's lowest
// point, into the in-place store row: one warp per board, lane = row, one bit-parallel flood per chain.
template <int N>
__global__ void relabel_kernel(bbk_go_store st, const uint16_t* pat, int64_t n) {
    constexpr int PS = pat_stride(N);
    constexpr uint32_t ROW = (1u << N) - 1u;
    const Seg<32> g;
    const int lane = g.sl;
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    for (int64_t b = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); b < n; b += nwarps) {
        const uint16_t* pb = pat + b * (int64_t)PS;
        uint16_t* lb = st.lab + b * (int64_t)PS;
        uint32_t rows[2] = {0u, 0u};
        if (lane < N)
            for (int c = 0; c < N; c++) {
                const uint32_t v = pb[lane * N + c];
                rows[0] |= (v & 1u) << c;
                rows[1] |= ((v >> 1) & 1u) << c;
            }
#pragma unroll
        for (int col = 0; col < 2; col++) {
            uint32_t left = rows[col];   // stones of this colour not labelled yet
            while (g.any(left != 0u)) {
                const unsigned who = g.ballot(left != 0u);
                const int r0 = __ffs(who) - 1;                    // lowest row with an unlabelled stone
                const uint32_t lr = g.shfl(left, r0);
                const int label = r0 * N + __ffs(lr) - 1;        // its lowest point
                uint32_t F = lane == r0 ? (lr & (0u - lr)) : 0u;
                while (true) {
                    const uint32_t F2 = (F | dilate<N>(g, F)) & rows[col];
                    const bool ch = g.any(F2 != F);
                    F = F2;
                    if (!ch) break;
                }
                for (uint32_t f_ = F; f_; f_ &= f_ - 1) lb[lane * N + __ffs(f_) - 1] = (uint16_t)label;
                left &= ~F;
            }
        }
        (void)ROW;
    }
}

static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <int N>
static int launch_step(const StepParams& p, cudaStream_t stream) {
    const size_t smem = sizeof(BlockSmem<N>);
    // per device, once: shared-memory opt-in, occupancy, zobrist table (synchronous copy, so an
    // init launch -- always eager, before any capture -- leaves it ready for every later launch)
    constexpr int kMaxDev = 64;
    static int per_sm_dev[kMaxDev] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) return (int)cudaErrorInvalidDevice;
    if (!per_sm_dev[dev]) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(stream, &cs);
        if (cs != cudaStreamCaptureStatusNone) return (int)cudaErrorStreamCaptureUnsupported;
        cudaFuncSetAttribute(step_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(observe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        static uint64_t zob[2 * N * N];
        for (int c = 0; c < N * N; c++)
            for (int col = 0; col < 2; col++)
                zob[2 * c + col] = mix64(0x60D00D60C0FFEE00ULL + (uint64_t)N + 2ull * (uint64_t)c + (uint64_t)col);
        cudaError_t e = cudaMemcpyToSymbol(g_zob<N>, zob, sizeof(zob));
        if (e != cudaSuccess) return (int)e;
        static uint64_t zrow[2 * N * (N + 1)];
        for (int col = 0; col < 2; col++)
            for (int r = 0; r < N; r++) {
                uint64_t* z = zrow + (col * N + r) * (N + 1);
                z[0] = 0ull;
                for (int j = 0; j < N; j++) z[j + 1] = z[j] ^ zob[2 * (r * N + j) + col];
            }
        e = cudaMemcpyToSymbol(g_zrow<N>, zrow, sizeof(zrow));
        if (e != cudaSuccess) return (int)e;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<N>, kWarps * 32, smem);
        per_sm_dev[dev] = per_sm < 1 ? 1 : per_sm;
    }
    const int per_sm = per_sm_dev[dev];
    int64_t need = (p.n + boards_per_cta(N) - 1) / boards_per_cta(N);
    // Grid: whole waves of resident CTAs (wave_grid, common.cuh). The large boards launch about one
    // CTA per 3 boards per warp segment, so CTAs retire and new ones start in board order and the
    // observation stream leaves the SMs in a tighter address window: a warp writing whole records
    // absorbs 7.2 TB/s when each warp writes one record and exits vs 6.2 TB/s from a persistent grid
    // (tools/write_pattern.cu); go_19x19 +11.5 % early game, +4 % over a full episode cycle. Small
    // boards (prefetch-sensitive, ALU-bound) run two waves of 8 boards per segment (+0.4 % over a
    // persistent grid; more CTAs lost up to 3.7 %).
    constexpr int kGridBoards = BBK_GO_GRID_BOARDS >= 0 ? BBK_GO_GRID_BOARDS : (N > 13 ? 3 : 8);   // 19x19 at 7 CTAs: 3 > 4 > 2; 9x9: 8 (two waves) +0.4 % over persistent, 4: -0.8 %
    const int64_t resident = (int64_t)num_sms() * per_sm;
    const int64_t grid = wave_grid(resident, need, kGridBoards);
    StepParams q = p;
    q.tail_ctas = tail_ctas(grid, resident, kGoTailPct);
    step_kernel<N><<<(unsigned)grid, kWarps * 32, smem, stream>>>(q);
    return (int)cudaGetLastError();
}

template <int N>
static int launch_observe(const uint16_t* pat, const uint8_t* role, float* obs, int64_t n, cudaStream_t stream) {
    const size_t smem = sizeof(BlockSmem<N>);
    cudaFuncSetAttribute(observe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // one board per warp segment, CTAs retire in board order (a pure observation stream: 7.2 vs
    // 6.2 TB/s from a persistent grid, tools/write_pattern.cu)
    const int64_t need = (n + boards_per_cta(N) - 1) / boards_per_cta(N);
    const int64_t grid = need;
    observe_kernel<N><<<(unsigned)(grid < 1 ? 1 : grid), kWarps * 32, smem, stream>>>(pat, role, obs, n);
    return (int)cudaGetLastError();
}

static int dispatch_step(int size, const StepParams& p, cudaStream_t s) {
    switch (size) {   // odd board sizes 5..19 (go.py:114 accepts any size)
        case 5: return launch_step<5>(p, s);
        case 7: return launch_step<7>(p, s);
        case 9: return launch_step<9>(p, s);
        case 11: return launch_step<11>(p, s);
        case 13: return launch_step<13>(p, s);
        case 15: return launch_step<15>(p, s);
        case 17: return launch_step<17>(p, s);
        case 19: return launch_step<19>(p, s);
        default: return (int)cudaErrorInvalidValue;
    }
}

}  // namespace go

extern "C" {

int bbk_go_pat_stride(int size) { return go::pat_stride(size); }

int bbk_go_filter_words(int size) {
    if (size < 5 || size > 19 || !(size & 1)) return -1;
    return go::filter_words(size);
}

int bbk_go_init(int size, const bbk_cols* out, const bbk_go_state* out_s, const bbk_go_store* store,
                int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    go::StepParams p{};
    p.out = *out; p.out_s = *out_s; p.store = *store;
    p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.komi = 0.0; p.force_reset = 1;
    return go::dispatch_step(size, p, (cudaStream_t)stream);
}

int bbk_go_step(int size, double komi, int allow_self_capture, const bbk_cols* in, const bbk_go_state* in_s,
                const bbk_cols* out, const bbk_go_state* out_s, const bbk_go_store* store,
                const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state,
                const uint64_t* slot_keys, int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    go::StepParams p{};
    p.in = *in; p.in_s = *in_s; p.out = *out; p.out_s = *out_s; p.store = *store;
    p.actions = actions; p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.komi = komi; p.force_reset = 0; p.self_capture = allow_self_capture;
    return go::dispatch_step(size, p, (cudaStream_t)stream);
}

int bbk_go_observe(int size, const uint16_t* pat, const uint8_t* role, float* obs, int64_t n, void* stream) {
    if (n <= 0) return 0;
    switch (size) {
        case 5: return go::launch_observe<5>(pat, role, obs, n, (cudaStream_t)stream);
        case 7: return go::launch_observe<7>(pat, role, obs, n, (cudaStream_t)stream);
        case 9: return go::launch_observe<9>(pat, role, obs, n, (cudaStream_t)stream);
        case 11: return go::launch_observe<11>(pat, role, obs, n, (cudaStream_t)stream);
        case 13: return go::launch_observe<13>(pat, role, obs, n, (cudaStream_t)stream);
        case 15: return go::launch_observe<15>(pat, role, obs, n, (cudaStream_t)stream);
        case 17: return go::launch_observe<17>(pat, role, obs, n, (cudaStream_t)stream);
        case 19: return go::launch_observe<19>(pat, role, obs, n, (cudaStream_t)stream);
        default: return (int)cudaErrorInvalidValue;
    }
}

int bbk_go_relabel(int size, const bbk_go_store* store, const uint16_t* pat, int64_t n, void* stream) {
    if (n <= 0) return 0;
    int64_t grid = (n + go::kWarps - 1) / go::kWarps;
    if (grid > 148 * 8) grid = 148 * 8;
    const dim3 g((unsigned)grid), t(go::kWarps * 32);
    cudaStream_t s = (cudaStream_t)stream;
    switch (size) {
        case 5: go::relabel_kernel<5><<<g, t, 0, s>>>(*store, pat, n); break;
        case 7: go::relabel_kernel<7><<<g, t, 0, s>>>(*store, pat, n); break;
        case 9: go::relabel_kernel<9><<<g, t, 0, s>>>(*store, pat, n); break;
        case 11: go::relabel_kernel<11><<<g, t, 0, s>>>(*store, pat, n); break;
        case 13: go::relabel_kernel<13><<<g, t, 0, s>>>(*store, pat, n); break;
        case 15: go::relabel_kernel<15><<<g, t, 0, s>>>(*store, pat, n); break;
        case 17: go::relabel_kernel<17><<<g, t, 0, s>>>(*store, pat, n); break;
        case 19: go::relabel_kernel<19><<<g, t, 0, s>>>(*store, pat, n); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

int bbk_go_rebuild_bloom(int size, const bbk_go_store* store, const int32_t* hist_len, int64_t n, void* stream) {
    if (n <= 0) return 0;
    int64_t grid = (n + go::kWarps - 1) / go::kWarps;
    if (grid > 148 * 8) grid = 148 * 8;
    const dim3 g((unsigned)grid), t(go::kWarps * 32);
    cudaStream_t s = (cudaStream_t)stream;
    switch (size) {
        case 5: go::rebuild_bloom_kernel<5><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 7: go::rebuild_bloom_kernel<7><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 9: go::rebuild_bloom_kernel<9><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 11: go::rebuild_bloom_kernel<11><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 13: go::rebuild_bloom_kernel<13><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 15: go::rebuild_bloom_kernel<15><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 17: go::rebuild_bloom_kernel<17><<<g, t, 0, s>>>(*store, hist_len, n); break;
        case 19: go::rebuild_bloom_kernel<19><<<g, t, 0, s>>>(*store, hist_len, n); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_go)
