// Chess batched step for sm_100a (no reference engine: PAPER.md:781-856 +
// DESIGN.md §3.3 conventions; CPU twin oracle/orc_chess.c, perft-pinned).
//
// One warp per board. Lane l owns squares l and l+32 of the 64-byte board in
// shared memory. Per step:
//   1. lane 0 applies the action (AlphaZero 64x73 code in the mover's frame);
//   2. legal moves of the side to move, check/pin filtered: the opponent's
//      attack map (king removed) is an OR-reduction of per-lane ray scans;
//      lanes 0-7 walk the 8 rays out of the king to find checkers, block
//      squares and pins, lanes 8-17 test knight/pawn checkers; every lane
//      then emits its pieces' moves into a 4672-byte mask staged in shared
//      memory (en passant gets a full discovered-check test);
//   3. repetition: lanes compare the packed position against the ring
//      entries inside the half-move window in parallel (threefold = draw),
//      then mate / stalemate / insufficient material / 50-move rule;
//   4. observation: the 8 x 8 x 119 record is 7616 floats, almost all 0/1.
//      Lanes build it as a 7616-bit stream in shared memory (even squares,
//      then odd squares, so no two lanes touch one word), and emit float4
//      chunks through a 16-entry LUT; the two count planes are patched in.
#include "common.cuh"
#include "../../include/bbk.h"

namespace chess {
#ifndef BBK_CHESS_PASS_UNROLL
#define BBK_CHESS_PASS_UNROLL 1   // r02: rolled up +2 % (i-cache: 23 % of chess stalls are no-instruction)
#endif
constexpr int kChessPassUnroll = BBK_CHESS_PASS_UNROLL;   // the observation pattern's two square passes
#ifndef BBK_CHESS_OR_UNROLL
#define BBK_CHESS_OR_UNROLL 4
#endif
#ifndef BBK_CHESS_PAST_UNROLL
#define BBK_CHESS_PAST_UNROLL 1   // r02: rolled +2.8 % (2: +1.7 %, 4: +0.3 %)
#endif
constexpr int kChessOrUnroll = BBK_CHESS_OR_UNROLL, kChessPastUnroll = BBK_CHESS_PAST_UNROLL;
#ifndef BBK_CHESS_OBS_UNROLL
#define BBK_CHESS_OBS_UNROLL 2   // r02 (with the pass loop rolled): 2 = +1.9 % over 4, 1 = 0
#endif
constexpr int kChessObsUnroll = BBK_CHESS_OBS_UNROLL;   // observation chunk loop (tuning knob)
using namespace bbk;

constexpr int A = 4672;
constexpr int NF = 8 * 8 * 119;      // floats per record (7616)
constexpr int RING = 128;
constexpr int HIST_BYTES = RING * 32 + RING * 4;   // per env: packed boards + meta
constexpr int kWarps = 4;

enum { EMPTY = 0, P = 1, N = 2, B = 3, R = 4, Q = 5, K = 6 };

__device__ __constant__ int8_t KN_DR[8] = {2, 1, -1, -2, -2, -1, 1, 2};
__device__ __constant__ int8_t KN_DF[8] = {1, 2, 2, 1, -1, -2, -2, -1};
__device__ __constant__ int8_t DIR_DR[8] = {1, 1, 0, -1, -1, -1, 0, 1};
__device__ __constant__ int8_t DIR_DF[8] = {0, 1, 1, 1, 0, -1, -1, -1};
// square deltas of the knight jumps / king steps above (dr * 8 + df)
__device__ __constant__ int8_t KN_DELTA[8] = {17, 10, -6, -15, -17, -10, 6, 15};
__device__ __constant__ int8_t KG_DELTA[8] = {8, 9, 1, -7, -8, -9, -1, 7};
// knight / king target sets per square (read through the read-only path: lanes index them divergently)
__device__ const uint64_t KN_ATT[64] = {
    0x0000000000020400ull, 0x0000000000050800ull, 0x00000000000A1100ull, 0x0000000000142200ull,
    0x0000000000284400ull, 0x0000000000508800ull, 0x0000000000A01000ull, 0x0000000000402000ull,
    0x0000000002040004ull, 0x0000000005080008ull, 0x000000000A110011ull, 0x0000000014220022ull,
    0x0000000028440044ull, 0x0000000050880088ull, 0x00000000A0100010ull, 0x0000000040200020ull,
    0x0000000204000402ull, 0x0000000508000805ull, 0x0000000A1100110Aull, 0x0000001422002214ull,
    0x0000002844004428ull, 0x0000005088008850ull, 0x000000A0100010A0ull, 0x0000004020002040ull,
    0x0000020400040200ull, 0x0000050800080500ull, 0x00000A1100110A00ull, 0x0000142200221400ull,
    0x0000284400442800ull, 0x0000508800885000ull, 0x0000A0100010A000ull, 0x0000402000204000ull,
    0x0002040004020000ull, 0x0005080008050000ull, 0x000A1100110A0000ull, 0x0014220022140000ull,
    0x0028440044280000ull, 0x0050880088500000ull, 0x00A0100010A00000ull, 0x0040200020400000ull,
    0x0204000402000000ull, 0x0508000805000000ull, 0x0A1100110A000000ull, 0x1422002214000000ull,
    0x2844004428000000ull, 0x5088008850000000ull, 0xA0100010A0000000ull, 0x4020002040000000ull,
    0x0400040200000000ull, 0x0800080500000000ull, 0x1100110A00000000ull, 0x2200221400000000ull,
    0x4400442800000000ull, 0x8800885000000000ull, 0x100010A000000000ull, 0x2000204000000000ull,
    0x0004020000000000ull, 0x0008050000000000ull, 0x00110A0000000000ull, 0x0022140000000000ull,
    0x0044280000000000ull, 0x0088500000000000ull, 0x0010A00000000000ull, 0x0020400000000000ull,
};
__device__ const uint64_t KG_ATT[64] = {
    0x0000000000000302ull, 0x0000000000000705ull, 0x0000000000000E0Aull, 0x0000000000001C14ull,
    0x0000000000003828ull, 0x0000000000007050ull, 0x000000000000E0A0ull, 0x000000000000C040ull,
    0x0000000000030203ull, 0x0000000000070507ull, 0x00000000000E0A0Eull, 0x00000000001C141Cull,
    0x0000000000382838ull, 0x0000000000705070ull, 0x0000000000E0A0E0ull, 0x0000000000C040C0ull,
    0x0000000003020300ull, 0x0000000007050700ull, 0x000000000E0A0E00ull, 0x000000001C141C00ull,
    0x0000000038283800ull, 0x0000000070507000ull, 0x00000000E0A0E000ull, 0x00000000C040C000ull,
    0x0000000302030000ull, 0x0000000705070000ull, 0x0000000E0A0E0000ull, 0x0000001C141C0000ull,
    0x0000003828380000ull, 0x0000007050700000ull, 0x000000E0A0E00000ull, 0x000000C040C00000ull,
    0x0000030203000000ull, 0x0000070507000000ull, 0x00000E0A0E000000ull, 0x00001C141C000000ull,
    0x0000382838000000ull, 0x0000705070000000ull, 0x0000E0A0E0000000ull, 0x0000C040C0000000ull,
    0x0003020300000000ull, 0x0007050700000000ull, 0x000E0A0E00000000ull, 0x001C141C00000000ull,
    0x0038283800000000ull, 0x0070507000000000ull, 0x00E0A0E000000000ull, 0x00C040C000000000ull,
    0x0302030000000000ull, 0x0705070000000000ull, 0x0E0A0E0000000000ull, 0x1C141C0000000000ull,
    0x3828380000000000ull, 0x7050700000000000ull, 0xE0A0E00000000000ull, 0xC040C00000000000ull,
    0x0203000000000000ull, 0x0507000000000000ull, 0x0A0E000000000000ull, 0x141C000000000000ull,
    0x2838000000000000ull, 0x5070000000000000ull, 0xA0E0000000000000ull, 0x40C0000000000000ull,
};

struct WarpSmem {
    alignas(16) uint32_t mbits[A / 32];   // legal mask staged as bits (action a = bit a)
    alignas(16) uint32_t bits[(NF / 32 + 4 + 3) & ~3];   // zeroed as uint4
    alignas(16) uint8_t bd[64];
    alignas(16) uint8_t packed[32];
    alignas(16) uint8_t past[8][64];   // boards of history steps t = 0..7 (absolute squares)
    uint8_t prep[8];
    uint64_t pinray[8];
    int8_t pinsq[8];
    uint16_t task[2][96];              // (piece, ray) work units: own [0], opponent [1] (<= 9Q 2R 2B 2N K = 91)
    // next-board prefetch (cp.async): board, packed past boards t = 1..7, ring meta by ply
    alignas(16) uint8_t pf_bd[64];
    alignas(16) uint8_t pf_past[7][32];
    alignas(16) uint32_t pf_meta[RING];
};

struct Params {
    bbk_cols in, out;
    bbk_chess_state in_s, out_s;
    const int64_t* actions;
    const uint64_t* slot_keys;
    int64_t n, slot0;
    uint64_t key;
    int32_t max_steps;
    int force_reset;
    const uint8_t* load_board;   // kLoad: positions to start from, [n, 64] / [n, 8] (stm, castle, ep, half-move)
    const uint8_t* load_misc;
    int64_t tail_ctas;   // one-pass CTAs at the end of the grid (common.cuh pass_map)
};

__device__ __forceinline__ bool on(int r, int f) { return (unsigned)r < 8u && (unsigned)f < 8u; }
__device__ __forceinline__ int color(uint8_t pc) { return pc >> 3; }
__device__ __forceinline__ int type(uint8_t pc) { return pc & 7; }
__device__ __forceinline__ uint8_t mk(int c, int t) { return (uint8_t)((c << 3) | t); }

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
    uint32_t lo = __reduce_or_sync(BBK_FULL, (uint32_t)v), hi = __reduce_or_sync(BBK_FULL, (uint32_t)(v >> 32));
    return ((uint64_t)hi << 32) | lo;
}

// Attack test on a modified board (en passant legality): is `sq` attacked by
// side `by` when squares e1/e2 are emptied and `add` holds `add_pc`?
__device__ bool attacked_mod(const uint8_t* bd, int sq, int by, int e1, int e2, int add, uint8_t add_pc) {
    auto at = [&](int s) -> uint8_t { return s == add ? add_pc : (s == e1 || s == e2) ? (uint8_t)0 : bd[s]; };
    int r = sq >> 3, f = sq & 7;
    int pr = by == 0 ? r - 1 : r + 1;
    for (int df = -1; df <= 1; df += 2)
        if (on(pr, f + df) && at(pr * 8 + f + df) == mk(by, P)) return true;
    for (int k = 0; k < 8; k++) {
        int rr = r + KN_DR[k], ff = f + KN_DF[k];
        if (on(rr, ff) && at(rr * 8 + ff) == mk(by, N)) return true;
    }
    for (int d = 0; d < 8; d++) {
        int rr = r + DIR_DR[d], ff = f + DIR_DF[d];
        if (on(rr, ff) && at(rr * 8 + ff) == mk(by, K)) return true;
        bool diag = DIR_DR[d] != 0 && DIR_DF[d] != 0;
        while (on(rr, ff)) {
            uint8_t pc = at(rr * 8 + ff);
            if (pc) {
                if (color(pc) == by && (type(pc) == Q || type(pc) == (diag ? B : R))) return true;
                break;
            }
            rr += DIR_DR[d]; ff += DIR_DF[d];
        }
    }
    return false;
}

// (dr+2)*5 + (df+2) -> knight plane 56+k (KN_DR/KN_DF order), or -1;
// (sr+1)*3 + (sf+1) -> queen direction index (DIR_DR/DIR_DF order)
__device__ __constant__ int8_t KN_PLANE[25] = {-1, 60, -1, 59, -1, 61, -1, -1, -1, 58, -1, -1, -1, -1, -1,
                                               62, -1, -1, -1, 57, -1, 63, -1, 56, -1};
__device__ __constant__ int8_t QDIR[9] = {5, 4, 3, 6, -1, 2, 7, 0, 1};

// AlphaZero action index in the mover's frame.
__device__ __forceinline__ int action_of(int fl, int from, int to, int promo) {
    const int f = from ^ fl, t = to ^ fl;
    const int dr = (t >> 3) - (f >> 3), df = (t & 7) - (f & 7);
    int plane;
    if (promo && promo != Q) {
        plane = 64 + 3 * (promo == N ? 0 : promo == B ? 1 : 2) + (df + 1);
    } else {
        const int adr = dr < 0 ? -dr : dr, adf = df < 0 ? -df : df;
        const int kn = (adr <= 2 && adf <= 2) ? KN_PLANE[(dr + 2) * 5 + (df + 2)] : -1;
        if (kn >= 0) {
            plane = kn;
        } else {
            const int dist = adr > adf ? adr : adf;
            const int d = QDIR[((dr > 0) - (dr < 0) + 1) * 3 + ((df > 0) - (df < 0) + 1)];
            plane = d * 7 + dist - 1;
        }
    }
    return f * 73 + plane;
}

// ------------------------------------------------------------ task lists
// Work is distributed over (piece, ray) TASKS instead of squares: a slider
// contributes one task per direction, a knight / king / pawn one task. All 32
// lanes then stride over the task list, so the (few, uneven) pieces do not
// serialise the warp. Task = square | dir << 6 (dir 8 = whole piece).
__device__ __constant__ int8_t FLIPD[8] = {4, 3, 2, 1, 0, 7, 6, 5};   // vertical flip of a queen direction

__device__ __forceinline__ void setm(uint32_t* m, int a) { atomicOr(&m[a >> 5], 1u << (a & 31)); }

__device__ __forceinline__ int ntasks_of(uint8_t pc) {
    const int t = pc & 7;
    return !pc ? 0 : t == Q ? 8 : (t == R || t == B) ? 4 : 1;
}

// Build both task lists (own = `side`, opponent) with one packed warp scan.
__device__ void build_tasks(const uint8_t* bd, int side, uint16_t (*task)[96], int& n_own, int& n_opp, int lane) {
    const uint8_t p0 = bd[lane], p1 = bd[lane + 32];
    const int o0 = (p0 && color(p0) == side) ? ntasks_of(p0) : 0, o1 = (p1 && color(p1) == side) ? ntasks_of(p1) : 0;
    const int x0 = (p0 && color(p0) != side) ? ntasks_of(p0) : 0, x1 = (p1 && color(p1) != side) ? ntasks_of(p1) : 0;
    const int mine = (o0 + o1) | ((x0 + x1) << 16);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(BBK_FULL, incl, o);
        if (lane >= o) incl += t;
    }
    const int tot = __shfl_sync(BBK_FULL, incl, 31);
    n_own = tot & 0xFFFF; n_opp = tot >> 16;
    int ko = (incl - mine) & 0xFFFF, kx = (incl - mine) >> 16;
    BBK_CHECK(n_own <= 96 && n_opp <= 96);   // task list capacity (WarpSmem::task)
    auto put = [&](uint16_t* list, int& k, int sq, uint8_t pc, int n) {
        const int t = pc & 7;
        if (n == 1) { list[k++] = (uint16_t)(sq | (8 << 6)); return; }
        const int d0 = t == B ? 1 : 0, stp = t == Q ? 1 : 2;
        for (int d = d0; d < 8; d += stp) list[k++] = (uint16_t)(sq | (d << 6));
    };
    if (o0) put(task[0], ko, lane, p0, o0);
    if (o1) put(task[0], ko, lane + 32, p1, o1);
    if (x0) put(task[1], kx, lane, p0, x0);
    if (x1) put(task[1], kx, lane + 32, p1, x1);
}

// Attack bits of one opponent task (our king `ksq` is transparent to sliders).
__device__ __forceinline__ uint64_t task_attacks(const uint8_t* bd, uint16_t tk, uint64_t occ_nk) {
    const int sq = tk & 63, d = tk >> 6, r = sq >> 3, f = sq & 7;
    uint64_t a = 0ull;
    if (d < 8) {   // walk the ray on the occupancy bitboard (our king transparent): no board reads
        const int dr = DIR_DR[d], df = DIR_DF[d];
        int rr = r + dr, ff = f + df;
        while (on(rr, ff)) {
            const int to = rr * 8 + ff;
            a |= 1ull << to;
            if ((occ_nk >> to) & 1ull) break;
            rr += dr; ff += df;
        }
        return a;
    }
    const uint8_t pc = bd[sq];
    const int t = type(pc), by = color(pc);
    if (t == N) {
        a = __ldg(&KN_ATT[sq]);
    } else if (t == K) {
        a = __ldg(&KG_ATT[sq]);
    } else {   // pawn
        const int rr = by == 0 ? r + 1 : r - 1;
        if (on(rr, f - 1)) a |= 1ull << (rr * 8 + f - 1);
        if (on(rr, f + 1)) a |= 1ull << (rr * 8 + f + 1);
    }
    return a;
}

struct GenCtx {
    const uint8_t* bd;
    uint32_t* mask;   // bit per action
    int side, fl, ksq, ep;
    uint64_t att, checkmask, own, occ, pinned;   // own: side to move's squares; occ: all pieces
    const int8_t* pinsq;
    const uint64_t* pinray;
};

// Emit the legal moves of one own task into the staged mask; returns the count.
__device__ int task_moves(const GenCtx& c, uint16_t tk, bool& ep_legal) {
    const int sq = tk & 63, d = tk >> 6, r = sq >> 3, f = sq & 7;
    const uint8_t pc = c.bd[sq];
    const int t = type(pc), side = c.side;
    const int from = (sq ^ c.fl) * 73;
    int cnt = 0;
    if (t == K) {
        // a wrapped square sq + delta is never a king target of sq, so the set test is exact
        const uint64_t m = __ldg(&KG_ATT[sq]) & ~c.own & ~c.att;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int to = sq + KG_DELTA[k];
            if ((unsigned)to < 64u && ((m >> to) & 1ull)) { setm(c.mask, from + (c.fl ? (12 - k) & 7 : k) * 7); cnt++; }
        }
        return cnt;
    }
    uint64_t allow = c.checkmask;
    if ((c.pinned >> sq) & 1ull)   // the 8 pin slots are read only for a pinned piece
        for (int j = 0; j < 8; j++) if (c.pinsq[j] == sq) allow &= c.pinray[j];
    if (d < 8) {   // slider ray
        const int dm = (c.fl ? FLIPD[d] : d) * 7;
        const int dr = DIR_DR[d], df = DIR_DF[d];
        int rr = r + dr, ff = f + df, k = 0;
        while (on(rr, ff)) {
            const int to = rr * 8 + ff;
            if ((c.own >> to) & 1ull) break;
            if ((allow >> to) & 1ull) { setm(c.mask, from + dm + k); cnt++; }
            if ((c.occ >> to) & 1ull) break;
            rr += dr; ff += df; k++;
        }
        return cnt;
    }
    if (t == N) {
        const uint64_t m = __ldg(&KN_ATT[sq]) & ~c.own & allow;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int to = sq + KN_DELTA[k];
            if ((unsigned)to < 64u && ((m >> to) & 1ull)) { setm(c.mask, from + 56 + (c.fl ? (11 - k) & 7 : k)); cnt++; }
        }
        return cnt;
    }
    // pawn (mover frame: forward = N, captures NW / NE)
    const int dr = side == 0 ? 1 : -1, last = side == 0 ? 7 : 0, start = side == 0 ? 1 : 6;
    const int r1 = r + dr;
    auto emit = [&](int to, int df, int plane_q) {
        if (r1 == last) {
            setm(c.mask, from + plane_q);                       // queen promotion = queen-move plane
            setm(c.mask, from + 64 + 0 * 3 + df + 1);           // N, B, R under-promotions
            setm(c.mask, from + 64 + 1 * 3 + df + 1);
            setm(c.mask, from + 64 + 2 * 3 + df + 1);
            cnt += 4;
        } else {
            setm(c.mask, from + plane_q); cnt++;
        }
    };
    const int to1 = r1 * 8 + f;
    if (!((c.occ >> to1) & 1ull)) {
        if ((allow >> to1) & 1ull) emit(to1, 0, 0 * 7 + 0);
        const int to2 = (r + 2 * dr) * 8 + f;
        if (r == start && !((c.occ >> to2) & 1ull) && ((allow >> to2) & 1ull)) emit(to2, 0, 0 * 7 + 1);
    }
    for (int df = -1; df <= 1; df += 2) {
        if (!on(r1, f + df)) continue;
        const int to = r1 * 8 + f + df;
        const int plane = (df < 0 ? 7 : 1) * 7;               // NW / NE, distance 1
        if (((c.occ & ~c.own) >> to) & 1ull) {
            if ((allow >> to) & 1ull) emit(to, df, plane);
        } else if (to == c.ep) {
            const int cap = side == 0 ? to - 8 : to + 8;
            if (!attacked_mod(c.bd, c.ksq, 1 - side, sq, cap, to, pc)) {
                setm(c.mask, from + plane); cnt++;
                ep_legal = true;
            }
        }
    }
    return cnt;
}

// Apply a move encoded in the mover's frame (mirrors oracle make()).
__device__ void apply_action(uint8_t* bd, int& stm, int& castle, int& ep, int& halfmove, int a) {
    const int fl = stm ? 56 : 0;
    const int fromv = a / 73, plane = a - 73 * fromv;
    int dr, df, promo = 0;
    if (plane < 56) { int d = plane / 7, dist = plane - 7 * d + 1; dr = DIR_DR[d] * dist; df = DIR_DF[d] * dist; }
    else if (plane < 64) { dr = KN_DR[plane - 56]; df = KN_DF[plane - 56]; }
    else { int u = plane - 64; promo = u / 3 == 0 ? N : u / 3 == 1 ? B : R; df = u % 3 - 1; dr = 1; }
    const int tov = fromv + dr * 8 + df;
    const int from = fromv ^ fl, to = tov ^ fl;
    const uint8_t pc = bd[from], cap = bd[to];
    const int side = color(pc), t = type(pc);
    const bool reset = t == P || cap != EMPTY;
    if (t == P && !promo && ((to >> 3) == 7 || (to >> 3) == 0)) promo = Q;
    if (t == P && to == ep && cap == EMPTY && (from & 7) != (to & 7)) bd[side == 0 ? to - 8 : to + 8] = EMPTY;
    bd[to] = promo ? mk(side, promo) : pc;
    bd[from] = EMPTY;
    if (t == K && ((to & 7) - (from & 7) == 2 || (from & 7) - (to & 7) == 2)) {
        int rank = from & ~7;
        if ((to & 7) == 6) { bd[rank + 5] = bd[rank + 7]; bd[rank + 7] = EMPTY; }
        else { bd[rank + 3] = bd[rank + 0]; bd[rank + 0] = EMPTY; }
    }
    auto clr = [](int s) -> int { return s == 0 ? 2 : s == 4 ? 3 : s == 7 ? 1 : s == 56 ? 8 : s == 60 ? 12 : s == 63 ? 4 : 0; };
    castle &= ~(clr(from) | clr(to));
    ep = -1;
    if (t == P && (to - from == 16 || from - to == 16)) ep = (from + to) / 2;
    halfmove = reset ? 0 : halfmove + 1;
    stm ^= 1;
}

// One scalar field of board b per lane (lanes 0-4), loaded a board ahead.
__device__ __forceinline__ FieldRef field_ref(const Params& p, int lane) {
    switch (lane) {
        case 0: return field_of(p.in.terminated, 0u);
        case 1: return field_of(p.in.player_to_role, 1u);
        case 2: return field_of(p.in_s.misc, 3u);
        case 3: return field_of(p.in.step_count, 2u);
        case 4: return field_of(p.actions, 3u);
        case 5: return field_of(p.in.truncated, 0u);
        default: return no_field();
    }
}

// cp.async board b's state and the ring entries its step reads into the prefetch
// area: the board, the packed boards of plies step-1..step-7 (step = in step + 1)
// and the ring meta of plies [step - M, step) with M covering both the
// observation history and the repetition window (half-move clock + 1 bound).
__device__ __forceinline__ void issue_prefetch(WarpSmem& S, const Params& p, int64_t b, uint64_t f, int lane) {
    const uint32_t term = (uint32_t)__shfl_sync(BBK_FULL, (uint32_t)f, 0);
    const uint64_t misc = shfl64(f, 2);
    const int in_step = (int)__shfl_sync(BBK_FULL, (uint32_t)f, 3);
    const char* bsrc = reinterpret_cast<const char*>(p.in_s.board + b * 64);
    if (lane < 4) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(S.pf_bd) + 16u * lane;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(bsrc + 16 * lane));
    }
    if (!(term & 0xFFFFu)) {
        const uint8_t* hist = p.out_s.hist + b * (int64_t)HIST_BYTES;
        const int step = in_step + 1;
        if (lane < 14) {   // past boards t = 1 + lane / 2
            const int ply = step - 1 - (lane >> 1);
            if (ply >= 0) {
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&S.pf_past[lane >> 1][0]) + 16u * (lane & 1);
                const char* src = reinterpret_cast<const char*>(hist + (ply & (RING - 1)) * 32) + 16 * (lane & 1);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
            }
        }
        const int hm1 = (int)((misc >> 24) & 0xFF) + 1;
        int M = hm1 > 7 ? hm1 : 7;
        if (M > step) M = step;
        const uint32_t* meta = reinterpret_cast<const uint32_t*>(hist + RING * 32);
        for (int j = lane; j < M; j += 32) {
            const int ply = (step - 1 - j) & (RING - 1);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&S.pf_meta[ply]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(meta + ply));
        }
    }
    asm volatile("cp.async.commit_group;");
}

// kLoad: a reset that starts from p.load_board / p.load_misc instead of the initial position
// (bbk_chess_load, the device twin of the oracle's orc_chess_set_fen test hook); a separate
// instantiation so the hot kernel's code is unchanged.
template <bool kLoad>
#ifndef BBK_CHESS_MIN_CTAS
#define BBK_CHESS_MIN_CTAS 9
#endif
__global__ void __launch_bounds__(kWarps * 32, BBK_CHESS_MIN_CTAS) step_kernel(Params p) {   // 56 registers, no spills
    __shared__ WarpSmem sm[kWarps];
    __shared__ float4 lut[16];
    if (threadIdx.x < 16) {
        uint32_t q = threadIdx.x;
        lut[q] = make_float4((float)(q & 1), (float)((q >> 1) & 1), (float)((q >> 2) & 1), (float)((q >> 3) & 1));
    }
    __syncthreads();
    WarpSmem& S = sm[threadIdx.x >> 5];
    const int lane = lane_id();
    const PassMap pm = pass_map(p.n, kWarps, p.tail_ctas, threadIdx.x >> 5);
    const int64_t nwarps = pm.stride, bend = pm.end;
    unsigned long long eps = 0;
    const int64_t b0 = pm.b0;
    uint64_t cur = 0ull;   // this board's scalar fields (lane j holds field j)
    bool pf_ready = false;
    const FieldRef fref = field_ref(p, lane_id());
    for (int64_t b = b0; b < bend; b += nwarps) {
        if (!p.force_reset && !pf_ready) {   // first board of the warp: fetch synchronously
            cur = load_field(fref, b);
            issue_prefetch(S, p, b, cur, lane);
        }
        // the next board's scalars are in flight while this board is processed
        const int64_t nb = b + nwarps;
        const uint64_t nxt = (!p.force_reset && nb < bend) ? load_field(fref, nb) : 0ull;
        const uint32_t f_term = __shfl_sync(BBK_FULL, (uint32_t)cur, 0) | (__shfl_sync(BBK_FULL, (uint32_t)cur, 5) << 8);
        const bool reset = p.force_reset || (f_term & 0xFFFFu) != 0u;
        if (!p.force_reset) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const uint64_t k = slot_key(p.slot_keys, p.key, p.slot0, b);
        uint8_t* hist = p.out_s.hist + b * (int64_t)HIST_BYTES;
        uint32_t* hmeta = reinterpret_cast<uint32_t*>(hist + RING * 32);
        int8_t p2r0, p2r1;
        int stm, castle, ep, halfmove, step;
        if (reset) {
            int c = (int)(child(k, 0) % 2ull);
            p2r0 = (int8_t)c; p2r1 = (int8_t)(1 - c);
            if (kLoad) {
                S.bd[lane] = p.load_board[b * 64 + lane];
                S.bd[lane + 32] = p.load_board[b * 64 + lane + 32];
                const uint8_t* lm = p.load_misc + b * 8;
                stm = lm[0] & 1; castle = lm[1] & 15; ep = (int8_t)lm[2]; halfmove = lm[3];
            } else {
                constexpr uint32_t back = 0x42365324u;   // R N B Q K B N R, nibble f = file f
                for (int s = lane; s < 64; s += 32) {
                    int r = s >> 3, f = s & 7;
                    const int bk = (int)((back >> (4 * f)) & 15u);
                    uint8_t v = r == 0 ? mk(0, bk) : r == 1 ? mk(0, P) : r == 6 ? mk(1, P) : r == 7 ? mk(1, bk) : 0;
                    S.bd[s] = v;
                }
                stm = 0; castle = 15; ep = -1; halfmove = 0;
            }
            step = 0;
        } else {
            const uint32_t f_p2r = __shfl_sync(BBK_FULL, (uint32_t)cur, 1);
            const uint64_t misc = shfl64(cur, 2);
            const int f_step = (int)__shfl_sync(BBK_FULL, (uint32_t)cur, 3);
            const int f_act = (int)shfl64(cur, 4);
            p2r0 = (int8_t)(f_p2r & 0xFF); p2r1 = (int8_t)(f_p2r >> 8);
            S.bd[lane] = S.pf_bd[lane]; S.bd[lane + 32] = S.pf_bd[lane + 32];
            stm = (int)(misc & 0xFF); castle = (int)((misc >> 8) & 0xFF); ep = (int8_t)((misc >> 16) & 0xFF);
            halfmove = (int)((misc >> 24) & 0xFF);
            step = f_step + 1;
            // past boards t = 1..7 from the prefetched packed copies (two squares per byte): word w
            // of the packed area is 8 squares of board t = w / 8 + 1, unpacked by two byte permutes
            for (int w = lane; w < 7 * 8; w += 32) {
                const int t = (w >> 3) + 1;
                const uint32_t x = step - t >= 0 ? reinterpret_cast<const uint32_t*>(S.pf_past)[w] : 0u;
                const uint32_t e = x & 0x0F0F0F0Fu, o = (x >> 4) & 0x0F0F0F0Fu;
                reinterpret_cast<uint2*>(&S.past[1][0])[w] = make_uint2(__byte_perm(e, o, 0x5140), __byte_perm(e, o, 0x7362));
            }
            if (lane >= 1 && lane < 8)
                S.prep[lane] = step - lane >= 0 ? (uint8_t)(S.pf_meta[(step - lane) & (RING - 1)] >> 24) : (uint8_t)0;
            __syncwarp();
            if (lane == 0) apply_action(S.bd, stm, castle, ep, halfmove, f_act);
            stm = __shfl_sync(BBK_FULL, stm, 0); castle = __shfl_sync(BBK_FULL, castle, 0);
            ep = __shfl_sync(BBK_FULL, ep, 0); halfmove = __shfl_sync(BBK_FULL, halfmove, 0);
        }
        // zero the mask staging area while the board settles
        for (int i = lane; i < A / 128; i += 32) reinterpret_cast<uint4*>(S.mbits)[i] = make_uint4(0, 0, 0, 0);
        if (lane < (A / 32) % 4) S.mbits[A / 32 - 1 - lane] = 0u;
        __syncwarp();
        const int side = stm, opp = 1 - side, fl = side ? 56 : 0;
        // ---- king, attack map, checks, pins
        const unsigned kb0 = __ballot_sync(BBK_FULL, S.bd[lane] == mk(side, K));
        const unsigned kb1 = __ballot_sync(BBK_FULL, S.bd[lane + 32] == mk(side, K));
        const int ksq = kb0 ? __ffs(kb0) - 1 : kb1 ? 32 + __ffs(kb1) - 1 : 0;
        uint64_t own_bb, occ_bb;
        {
            const uint8_t q0 = S.bd[lane], q1 = S.bd[lane + 32];
            own_bb = (uint64_t)__ballot_sync(BBK_FULL, q0 && color(q0) == side) |
                     ((uint64_t)__ballot_sync(BBK_FULL, q1 && color(q1) == side) << 32);
            occ_bb = (uint64_t)__ballot_sync(BBK_FULL, q0 != 0) | ((uint64_t)__ballot_sync(BBK_FULL, q1 != 0) << 32);
        }
        int n_own, n_opp;
        build_tasks(S.bd, side, S.task, n_own, n_opp, lane);
        __syncwarp();
        uint64_t att_l = 0ull;
        const uint64_t occ_nk = occ_bb & ~(1ull << ksq);   // our king is transparent to sliders
        for (int i = lane; i < n_opp; i += 32) att_l |= task_attacks(S.bd, S.task[1][i], occ_nk);
        const uint64_t att = warp_or64(att_l);
        const bool in_check = (att >> ksq) & 1ull;
        bool checker = false;
        uint64_t block = 0ull;
        if (lane < 8) {          // ray d = lane out of the king
            const int d = lane;
            const bool diag = DIR_DR[d] != 0 && DIR_DF[d] != 0;
            int rr = (ksq >> 3) + DIR_DR[d], ff = (ksq & 7) + DIR_DF[d];
            uint64_t ray = 0ull;
            int own = -1;
            int8_t pin = -1;
            uint64_t pray = 0ull;
            const int dr = DIR_DR[d], df = DIR_DF[d];
            while (on(rr, ff)) {
                int s = rr * 8 + ff;
                ray |= 1ull << s;
                if ((occ_bb >> s) & 1ull) {   // the board is read only at the (at most two) blockers
                    const uint8_t pc = S.bd[s];
                    bool slider = color(pc) == opp && (type(pc) == Q || type(pc) == (diag ? B : R));
                    if (own < 0) {
                        if (color(pc) == side) own = s;
                        else { if (slider) { checker = true; block = ray; } break; }
                    } else {
                        if (slider) { pin = (int8_t)own; pray = ray; }
                        break;
                    }
                }
                rr += dr; ff += df;
            }
            S.pinsq[d] = pin;
            S.pinray[d] = pray;
        } else if (lane < 16) {  // knight checkers
            const int j = lane - 8;
            int rr = (ksq >> 3) + KN_DR[j], ff = (ksq & 7) + KN_DF[j];
            if (on(rr, ff) && S.bd[rr * 8 + ff] == mk(opp, N)) { checker = true; block = 1ull << (rr * 8 + ff); }
        } else if (lane < 18) {  // pawn checkers
            int rr = (ksq >> 3) + (side == 0 ? 1 : -1), ff = (ksq & 7) + (lane == 16 ? -1 : 1);
            if (on(rr, ff) && S.bd[rr * 8 + ff] == mk(opp, P)) { checker = true; block = 1ull << (rr * 8 + ff); }
        }
        const int nchecks = __popc(__ballot_sync(BBK_FULL, checker));
        const uint64_t blockall = warp_or64(block);
        const uint64_t pinned_bb = warp_or64(lane < 8 && S.pinsq[lane] >= 0 ? 1ull << S.pinsq[lane] : 0ull);
        __syncwarp();
        GenCtx c;
        c.bd = S.bd; c.mask = S.mbits; c.side = side; c.fl = fl; c.ksq = ksq; c.att = att; c.ep = ep;
        c.checkmask = nchecks == 0 ? ~0ull : nchecks == 1 ? blockall : 0ull;
        c.pinsq = S.pinsq; c.pinray = S.pinray; c.pinned = pinned_bb;
        c.own = own_bb; c.occ = occ_bb;
        bool ep_legal = false;
        int cnt = 0;
        for (int i = lane; i < n_own; i += 32) cnt += task_moves(c, S.task[0][i], ep_legal);
        if (lane == 0 && !in_check) {   // castling (oracle gen_pseudo castling rules)
            const int rank = side == 0 ? 0 : 56, kbit = side == 0 ? 1 : 4, qbit = side == 0 ? 2 : 8;
            if (ksq == rank + 4) {
                if ((castle & kbit) && S.bd[rank + 7] == mk(side, R) && !S.bd[rank + 5] && !S.bd[rank + 6] &&
                    !((att >> (rank + 5)) & 1ull) && !((att >> (rank + 6)) & 1ull)) {
                    setm(S.mbits, action_of(fl, ksq, rank + 6, 0)); cnt++;
                }
                if ((castle & qbit) && S.bd[rank + 0] == mk(side, R) && !S.bd[rank + 1] && !S.bd[rank + 2] &&
                    !S.bd[rank + 3] && !((att >> (rank + 3)) & 1ull) && !((att >> (rank + 2)) & 1ull)) {
                    setm(S.mbits, action_of(fl, ksq, rank + 2, 0)); cnt++;
                }
            }
        }
        const int nlegal = warp_sum(cnt);
        const bool any_ep = __any_sync(BBK_FULL, ep_legal);
        const int ep_eff = any_ep ? ep : -1;
        // ---- packed position + repetition within the half-move window
        {
            uint8_t byte = (uint8_t)(S.bd[2 * lane] | (S.bd[2 * lane + 1] << 4));
            S.packed[lane] = byte;
        }
        __syncwarp();
        const uint32_t meta_key = (uint32_t)side | ((uint32_t)castle << 8) | ((uint32_t)(uint8_t)ep_eff << 16);
        int reps = 0;
        const int window = halfmove < step ? halfmove : step;
        BBK_CHECK(window < RING);   // the scanned plies are still in the ring (half-move clock <= 100)
        for (int j = lane; 2 * (j + 1) <= window; j += 32) {
            const int ply = step - 2 * (j + 1);
            const uint32_t m = S.pf_meta[ply & (RING - 1)];   // window <= half-move clock: prefetched
            if ((m & 0xFFFFFFu) == meta_key) {
                const uint4* hb = reinterpret_cast<const uint4*>(hist + (ply & (RING - 1)) * 32);
                const uint4* cb = reinterpret_cast<const uint4*>(S.packed);
                uint4 x0 = hb[0], x1 = hb[1], y0 = cb[0], y1 = cb[1];
                if (x0.x == y0.x && x0.y == y0.y && x0.z == y0.z && x0.w == y0.w && x1.x == y1.x && x1.y == y1.y &&
                    x1.z == y1.z && x1.w == y1.w) reps++;
            }
        }
        reps = warp_sum(reps);
        const int rep = reps > 2 ? 2 : reps;
        __syncwarp();   // the prefetch area (board, past boards, ring meta) is free now: issue the next board's state
        pf_ready = false;
        if (!p.force_reset && nb < bend) {
            issue_prefetch(S, p, nb, nxt, lane);
            cur = nxt;
            pf_ready = true;
        }
        // ---- insufficient material (oracle insufficient())
        int minors = 0, heavy = 0, knights = 0, blight = 0, bdark = 0;
        for (int s = lane; s < 64; s += 32) {
            uint8_t pc = S.bd[s];
            int t = type(pc);
            if (!pc || t == K) continue;
            if (t == P || t == R || t == Q) heavy++;
            else {
                minors++;
                if (t == N) knights++;
                else if ((((s >> 3) + (s & 7)) & 1)) blight++;
                else bdark++;
            }
        }
        {   // one reduction of the five counts (each <= 32) packed in 6-bit fields
            const int sum = warp_sum(heavy | (minors << 6) | (knights << 12) | (blight << 18) | (bdark << 24));
            heavy = sum & 63; minors = (sum >> 6) & 63; knights = (sum >> 12) & 63;
            blight = (sum >> 18) & 63; bdark = (sum >> 24) & 63;
        }
        const bool insufficient = heavy == 0 && (minors <= 1 || (knights == 0 && (blight == 0 || bdark == 0)));
        bool terminal = false;
        float rr0 = 0.0f, rr1 = 0.0f;
        if (nlegal == 0) {
            terminal = true;
            if (in_check) { if (side == 0) { rr0 = -1.0f; rr1 = 1.0f; } else { rr0 = 1.0f; rr1 = -1.0f; } }
        } else if (insufficient || halfmove >= 100 || reps >= 2) {
            terminal = true;
        }
        const bool truncated = !terminal && step >= p.max_steps;
        eps += (terminal || truncated) ? 1 : 0;
        if (p.out.next_actions) {   // fused agents.random_actions on the new mask (still in shared memory)
            __syncwarp();
            const int64_t a = warp_sample_bits(S.mbits, A / 32, (terminal || truncated) ? 0 : nlegal, p.out.next_key,
                                                p.slot0 + b);
            if (lane == 0) p.out.next_actions[b] = a;
        }
        // ---- history entry for this ply, then the past boards for the observation
        if (lane < 2) reinterpret_cast<uint4*>(hist + (step & (RING - 1)) * 32)[lane] =
            reinterpret_cast<const uint4*>(S.packed)[lane];
        if (lane == 0) hmeta[step & (RING - 1)] = meta_key | ((uint32_t)rep << 24);
        reinterpret_cast<uint16_t*>(S.past[0])[lane] = reinterpret_cast<const uint16_t*>(S.bd)[lane];
        if (reset) {
            for (int t = 1; t < 8; t++) { S.past[t][lane] = 0; S.past[t][lane + 32] = 0; }
            if (lane < 8) S.prep[lane] = 0;
        }
        if (lane == 0) S.prep[0] = (uint8_t)rep;
        for (int i = lane; i < (int)(sizeof(S.bits) / 16); i += 32) reinterpret_cast<uint4*>(S.bits)[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        // ---- observation bitstream: square v (mover frame) owns bits [119 v, 119 v + 119)
        const int own_k = side ? 4 : 1, own_q = side ? 8 : 2, opp_k = side ? 1 : 4, opp_q = side ? 2 : 8;
        const uint32_t cbits = ((uint32_t)side << 0) | ((uint32_t)((castle & own_k) != 0) << 2) |
                               ((uint32_t)((castle & own_q) != 0) << 3) | ((uint32_t)((castle & opp_k) != 0) << 4) |
                               ((uint32_t)((castle & opp_q) != 0) << 5);   // planes 112.. relative
        // square-independent planes, once per board: repetition planes 14 t + 12 / 13 and
        // 112.. colour, [113 count], castling x4, [118 count]
        uint64_t clo = 0ull, chi = (uint64_t)cbits << (112 - 64);
#pragma unroll
        for (int t = 0; t < 8; t++) {
            const int base = 14 * t;
            const uint8_t rp = S.prep[t];
            const uint64_t r1 = rp >= 1 ? 1ull : 0ull, r2 = rp >= 2 ? 1ull : 0ull;
            if (base + 13 < 64) clo |= (r1 << (base + 12)) | (r2 << (base + 13));
            else if (base + 12 >= 64) chi |= (r1 << (base + 12 - 64)) | (r2 << (base + 13 - 64));
            else { clo |= r1 << (base + 12); chi |= r2 << (base + 13 - 64); }
        }
#pragma unroll kChessPassUnroll
        for (int pass = 0; pass < 2; pass++) {
            const int v = 2 * lane + pass;
            const int sabs = v ^ fl;
            // 119-bit pattern of square v (bit k = plane k) in two registers
            uint64_t plo = clo, phi = chi;
#pragma unroll kChessPastUnroll
            for (int t = 0; t < 8; t++) {
                const uint8_t pc = S.past[t][sabs];
                const int base = 14 * t;
                if (pc) {
                    const int bit = base + (color(pc) == side ? 0 : 6) + type(pc) - 1;
                    plo |= bit < 64 ? 1ull << bit : 0ull;
                    phi |= bit >= 64 ? 1ull << (bit - 64) : 0ull;
                }
            }
            const uint32_t w[4] = {(uint32_t)plo, (uint32_t)(plo >> 32), (uint32_t)phi, (uint32_t)(phi >> 32)};
            // OR the 119-bit pattern into the stream at bit offset 119 v
            const int off = 119 * v, wi = off >> 5, sh = off & 31;
#pragma unroll kChessOrUnroll
            for (int j = 0; j < 4; j++) {
                uint32_t lo = w[j] << sh;
                uint32_t hi = sh ? (w[j] >> (32 - sh)) : 0u;
                S.bits[wi + j] |= lo;
                if (hi) S.bits[wi + j + 1] |= hi;
            }
            __syncwarp();
        }
        if (p.out.observation) {
            // binary planes through the LUT, then the two count planes (113, 118) of the
            // 64 squares as scalar stores, ordered after the vector stores by __syncwarp
            float* orec = p.out.observation + b * (int64_t)NF;
#ifndef BBK_CHESS_OBS_V8
#define BBK_CHESS_OBS_V8 0   // 32-byte stores measured -1.6 % here (r02 A/B; +3.2 % shogi, +2.9 % go_19x19)
#endif
            if constexpr (BBK_CHESS_OBS_V8) {
                // 32-byte stores (records are 30,464 B: every one is 32-B aligned); chunk j = lane + 32 m:
                // word lane / 4 + 8 m, lane-constant byte (lane % 4)
                static_assert(NF % 8 == 0, "chess records are whole 32-byte chunks");
                const uint32_t* wp = S.bits + (lane >> 2);
                const uint32_t bsh = (uint32_t)(lane & 3) * 8u;
#pragma unroll 2
                for (int j = lane; j < NF / 8; j += 32, wp += 8) {
                    const uint32_t t = *wp >> bsh;
                    const float4 lo = lut[t & 15u], hi = lut[(t >> 4) & 15u];
                    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(orec + 8 * j), "f"(lo.x),
                                 "f"(lo.y), "f"(lo.z), "f"(lo.w), "f"(hi.x), "f"(hi.y), "f"(hi.z), "f"(hi.w) : "memory");
                }
            } else {
                float4* o4 = reinterpret_cast<float4*>(orec);
                // chunk j = lane + 32 m: word lane / 8 + 4 m, lane-constant nibble (lane % 8)
                const uint32_t* wp = S.bits + (lane >> 3);
                const uint32_t nsh = (uint32_t)(lane & 7) * 4u;
#pragma unroll kChessObsUnroll
                for (int j = lane; j < NF / 4; j += 32, wp += 4) o4[j] = lut[(*wp >> nsh) & 15u];
            }
            __syncwarp();
            const float cnt113 = (float)step / 512.0f, cnt118 = (float)halfmove / 100.0f;
            orec[119 * lane + 113] = cnt113;
            orec[119 * (lane + 32) + 113] = cnt113;
            orec[119 * lane + 118] = cnt118;
            orec[119 * (lane + 32) + 118] = cnt118;
        }
        // ---- mask: zero when finished, else the staged bytes
        // mask bytes from the staged bits: 16 actions per 16-byte store, zero when finished
        uint4* m4 = reinterpret_cast<uint4*>(p.out.legal_action_mask + b * (int64_t)A);
        const bool live = !(terminal || truncated);
        for (int i = lane; i < A / 16; i += 32) {
            const uint32_t v = live ? (S.mbits[i >> 1] >> (16 * (i & 1))) & 0xFFFFu : 0u;
            m4[i] = make_uint4(spread4(v & 15u), spread4((v >> 4) & 15u), spread4((v >> 8) & 15u), spread4(v >> 12));
        }
        uint8_t* ob = p.out_s.board + b * 64;
        reinterpret_cast<uint16_t*>(ob)[lane] = reinterpret_cast<const uint16_t*>(S.bd)[lane];
        if (lane == 0) {
            uint8_t* m = p.out_s.misc + b * 8;
            m[0] = (uint8_t)stm; m[1] = (uint8_t)castle; m[2] = (uint8_t)ep; m[3] = (uint8_t)halfmove;
            m[4] = (uint8_t)rep; m[5] = 0; m[6] = 0; m[7] = 0;
            float r0 = 0.0f, r1 = 0.0f;
            if (!truncated && (rr0 != 0.0f || rr1 != 0.0f)) {
                r0 = p2r0 == 0 ? rr0 : rr1;
                r1 = p2r1 == 0 ? rr0 : rr1;
            }
            p.out.rewards[2 * b] = r0; p.out.rewards[2 * b + 1] = r1;
            p.out.terminated[b] = terminal; p.out.truncated[b] = truncated;
            p.out.step_count[b] = step;
            p.out.current_player[b] = p2r0 == stm ? 0 : 1;
            p.out.player_to_role[2 * b] = p2r0; p.out.player_to_role[2 * b + 1] = p2r1;
        }
        __syncwarp();
    }
    if (p.out.episodes && lane_id() == 0 && eps) atomicAdd(p.out.episodes, eps);
}

// observe(state, player) for an explicit role: rebuild from board + history.
__global__ void observe_kernel(bbk_chess_state st, const int32_t* step_count, const uint8_t* role, float* obs, int64_t n) {
    // Simple (non-hot) path: one thread per output float.
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * NF) return;
    int64_t b = idx / NF;
    int f = (int)(idx - b * NF);
    int v = f / 119, kpl = f - 119 * v;
    const int side = role[b], fl = side ? 56 : 0, sabs = v ^ fl;
    const int step = step_count[b];
    const uint8_t* m = st.misc + b * 8;
    const int castle = m[1], halfmove = m[3];
    const uint8_t* hist = st.hist + b * (int64_t)HIST_BYTES;
    const uint32_t* hmeta = reinterpret_cast<const uint32_t*>(hist + RING * 32);
    float val = 0.0f;
    if (kpl < 112) {
        int t = kpl / 14, j = kpl - 14 * t;
        if (step - t >= 0) {
            int ply = (step - t) & (RING - 1);
            uint8_t byte = hist[ply * 32 + (sabs >> 1)];
            uint8_t pc = (sabs & 1) ? byte >> 4 : byte & 15;
            int rp = (int)(hmeta[ply] >> 24);
            if (j < 12) val = (pc && ((color(pc) == side ? 0 : 6) + type(pc) - 1) == j) ? 1.0f : 0.0f;
            else val = rp >= j - 11 ? 1.0f : 0.0f;
        }
    } else if (kpl == 112) val = (float)side;
    else if (kpl == 113) val = (float)step / 512.0f;
    else if (kpl == 118) val = (float)halfmove / 100.0f;
    else {
        const int own_k = side ? 4 : 1, own_q = side ? 8 : 2, opp_k = side ? 1 : 4, opp_q = side ? 2 : 8;
        int bit = kpl == 114 ? own_k : kpl == 115 ? own_q : kpl == 116 ? opp_k : opp_q;
        val = (castle & bit) ? 1.0f : 0.0f;
    }
    obs[idx] = val;
}

#ifndef BBK_CHESS_GRID_BOARDS
#define BBK_CHESS_GRID_BOARDS 3   // boards per warp per launch (common.cuh step_grid); 0: persistent grid (r02: 3 = +6.3 %, 4 = +6 %, 6 = +4 %, 8 = +3 %)
#endif
#ifndef BBK_CHESS_TAIL_PCT
#define BBK_CHESS_TAIL_PCT 150   // one-pass CTAs at the end of the grid, % of the resident CTAs (r02: +2.3 %; 100: +1.6 %)
#endif
template <bool kLoad>
static void launch_grid(const Params& p, cudaStream_t s) {
    const int64_t need = (p.n + kWarps - 1) / kWarps;
    const int64_t resident = resident_ctas(step_kernel<kLoad>, kWarps * 32, 0);
    const int64_t grid = wave_grid(resident, need, BBK_CHESS_GRID_BOARDS);
    Params q = p;
    q.tail_ctas = tail_ctas(grid, resident, BBK_CHESS_TAIL_PCT);
    step_kernel<kLoad><<<(unsigned)grid, kWarps * 32, 0, s>>>(q);
}
static int launch(const Params& p, cudaStream_t s) {
    if (p.load_board) launch_grid<true>(p, s);
    else launch_grid<false>(p, s);
    return (int)cudaGetLastError();
}

}  // namespace chess

extern "C" {

int bbk_chess_init(const bbk_cols* out, const bbk_chess_state* out_s, int64_t n, int64_t slot0, uint64_t key_state,
                   const uint64_t* slot_keys, int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    chess::Params p{};
    p.out = *out; p.out_s = *out_s; p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.force_reset = 1;
    return chess::launch(p, (cudaStream_t)stream);
}

int bbk_chess_load(const bbk_cols* out, const bbk_chess_state* out_s, const uint8_t* boards, const uint8_t* misc,
                   int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys, int32_t max_steps,
                   void* stream) {
    if (n <= 0) return 0;
    if (!boards || !misc) return (int)cudaErrorInvalidValue;
    chess::Params p{};
    p.out = *out; p.out_s = *out_s; p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.force_reset = 1; p.load_board = boards; p.load_misc = misc;
    return chess::launch(p, (cudaStream_t)stream);
}

int bbk_chess_step(const bbk_cols* in, const bbk_chess_state* in_s, const bbk_cols* out, const bbk_chess_state* out_s,
                   const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                   int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    chess::Params p{};
    p.in = *in; p.in_s = *in_s; p.out = *out; p.out_s = *out_s; p.actions = actions; p.slot_keys = slot_keys;
    p.n = n; p.slot0 = slot0; p.key = key_state; p.max_steps = max_steps; p.force_reset = 0;
    return chess::launch(p, (cudaStream_t)stream);
}

int bbk_chess_observe(const bbk_chess_state* s, const int32_t* step_count, const uint8_t* role, float* obs, int64_t n,
                      void* stream) {
    if (n <= 0) return 0;
    int64_t tot = n * (int64_t)chess::NF;
    chess::observe_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*s, step_count, role, obs, n);
    return (int)cudaGetLastError();
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_chess)
